out=gpurun_out/pcie.txt
: > $out
nvidia-smi topo -m >> $out 2>&1
lscpu | grep -iE "numa|socket|model name" >> $out
for n in 1 2 4; do
  timeout 300 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2964$n tools/pcie_probe.py >> $out 2>/dev/null
done
