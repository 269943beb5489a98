# stencil per-GPU rate: single GPU at the per-GPU rectangle sizes, then 4 GPUs per tile height
python tools/stencil_probe.py 16384 > gpurun_out/stm.txt 2>&1
for tr in 16 32 64; do
  for shape in "32768 32768" "16384 65536"; do
    PM_STENCIL_TR=$tr timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
      --master-addr 127.0.0.1 --master-port $((29400 + RANDOM % 300)) tools/stencil_multi_probe.py $shape \
      >> gpurun_out/stm.txt 2>> gpurun_out/stm.err
  done
done
