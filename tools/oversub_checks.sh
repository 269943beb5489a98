# 8 ranks on the box's GPUs (2 per GPU on a 4-GPU box) with gloo host collectives:
# exercises the N=8 executor paths (2.5D c=2, 2x2x2 grids, (2,4) SUMMA, 8-way stencil)
export PM_TEST_BACKEND=gloo PM_HANG_DUMP_S=240
for t in cannon grid3d summa stencil circuit hydro; do
  echo "== $t" >> gpurun_out/ov.log
  timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
    --master-port $((29300 + RANDOM % 300)) tests/dist_${t}_check.py > gpurun_out/ov_$t.out 2> gpurun_out/ov_$t.err
  echo "rc $?" >> gpurun_out/ov.log
  grep '^{' gpurun_out/ov_$t.out | tail -1 | cut -c1-300 >> gpurun_out/ov.log
done
