export PM_HANG_DUMP_S=100
for t in cannon circuit hydro distmap; do
  echo "== $t" >> gpurun_out/c4.log
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tests/dist_${t}_check.py > gpurun_out/c4_$t.out 2> gpurun_out/c4_$t.err
  echo "rc $?" >> gpurun_out/c4.log
  tail -c 300 gpurun_out/c4_$t.out >> gpurun_out/c4.log
done
