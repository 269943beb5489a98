export PM_TEST_BACKEND=gloo
for s in 1 5 20; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port $((29300 + RANDOM % 300)) tools/hydro_diag.py $s > gpurun_out/hd_$s.out 2> gpurun_out/hd_$s.err
done
