# copy lanes of the SUMMA pulls: 4 (round-2 default) vs 2 vs 1, per-rank anatomy at N=4
for l in 4 1 2; do
  PROBE_LANES=$l timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2969$l tools/summa_probe.py > gpurun_out/summa_probe_l$l.json 2>/dev/null
done
