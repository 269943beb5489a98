# after the add-launch wave change: GEMM + multi-rank parity, then N=4 and N=2 bench lines
o=gpurun_out/final_r02b
mkdir -p $o
timeout 1500 python -m pytest -q -x tests/test_gpu_gemm.py tests/test_gpu_stencil_multi.py > $o/pytest.log 2>&1; echo "rc=$?" >> $o/pytest.log
timeout 1200 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29711 bench.py --gpus 4 > $o/bench_n4.json 2> $o/bench_n4.err
timeout 1200 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29712 bench.py --gpus 2 > $o/bench_n2.json 2> $o/bench_n2.err
echo done
