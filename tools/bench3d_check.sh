o=gpurun_out/b3d
mkdir -p $o
for n in 4 2; do
  timeout 900 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2972$n bench.py --gpus $n --no-kernels --no-stencil --no-cannon --no-circuit --no-hydro --no-cpu --no-e2e > $o/n$n.json 2> $o/n$n.err
done
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --no-kernels --no-stencil --no-cannon --no-circuit --no-hydro --no-cpu --no-e2e > $o/n1.json 2> $o/n1.err
