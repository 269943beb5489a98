# SUMMA / PUMMA K-rotated buffers: parity (real ranks, 8 ranks sharing GPUs, N=1), then the
# SUMMA / PUMMA bench legs with e2e at N=4 and N=2
o=gpurun_out/krot
mkdir -p $o
timeout 1500 python -m pytest -q -x tests/test_gpu_summa.py tests/test_gpu_multi.py tests/test_gpu_stencil_multi.py -k "summa or multi" > $o/pytest.log 2>&1; echo "rc=$?" >> $o/pytest.log
for n in 4 2; do
  timeout 900 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2973$n bench.py --gpus $n --no-kernels --no-stencil --no-cannon --no-circuit --no-hydro --no-cpu > $o/n$n.json 2> $o/n$n.err
done
