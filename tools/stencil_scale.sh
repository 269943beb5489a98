# stencil ms/sweep per mapping on this box's GPUs: square and 1:4 aspect (configs[4])
n=$(nvidia-smi -L | wc -l)
for shape in "32768 32768" "16384 65536"; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29400 + RANDOM % 300)) tools/stencil_multi_probe.py $shape >> gpurun_out/stencil_scale.txt 2>> gpurun_out/stencil_scale.err
done
