# Cannon checks (N=4 and 8 ranks on 4 GPUs) + configs[0] timing at N=4
export PM_HANG_DUMP_S=200
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29641 tests/dist_cannon_check.py > gpurun_out/cp4.out 2> gpurun_out/cp4.err; echo "n4 rc $? $(grep '^{' gpurun_out/cp4.out | cut -c1-20)" > gpurun_out/cp.log
PM_TEST_BACKEND=gloo timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29642 tests/dist_cannon_check.py > gpurun_out/cp8.out 2> gpurun_out/cp8.err; echo "n8 rc $? $(grep '^{' gpurun_out/cp8.out | cut -c1-20)" >> gpurun_out/cp.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29643 bench.py --gpus 4 --steps 4 --warmup 3 --no-3d --no-stencil --no-circuit --no-hydro --no-kernels --no-cpu --no-e2e --decompose-only > gpurun_out/cpb.json 2> gpurun_out/cpb.err; echo "bench rc $?" >> gpurun_out/cp.log
