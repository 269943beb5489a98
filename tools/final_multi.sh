# 4-GPU box: the whole GPU suite (multi-rank cases at their real world sizes), then the
# N=4 and N=2 bench lines
o=gpurun_out/multi_r02c
mkdir -p $o
timeout 2400 python -m pytest tests -m gpu -x -q > $o/pytest_gpu_4gpu.log 2>&1; echo "rc=$?" >> $o/pytest_gpu_4gpu.log
timeout 1200 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29671 bench.py --gpus 4 > $o/bench_n4.json 2> $o/bench_n4.err
timeout 1200 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29672 bench.py --gpus 2 > $o/bench_n2.json 2> $o/bench_n2.err
echo done
