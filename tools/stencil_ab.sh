# A/B of two libmapple builds on the stencil (single GPU + all GPUs of the box)
for lib in paper_2507_17087_b200/libmapple_b200.so paper_2507_17087_b200/csrc/build/oldst/lib.so; do
  echo "== $lib" >> gpurun_out/stencil_ab.txt
  MAPPLE_B200_LIB=$lib python tools/stencil_probe.py 16384 >> gpurun_out/stencil_ab.txt 2>&1
  MAPPLE_B200_LIB=$lib python tools/stencil_probe.py 16384 >> gpurun_out/stencil_ab.txt 2>&1
  n=$(nvidia-smi -L | wc -l)
  for shape in "32768 32768" "16384 65536"; do
    MAPPLE_B200_LIB=$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29400 + RANDOM % 300)) tools/stencil_multi_probe.py $shape >> gpurun_out/stencil_ab.txt 2>> gpurun_out/stencil_ab.err
  done
done
