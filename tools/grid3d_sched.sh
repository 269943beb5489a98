# grid3d schedule (plan_3d: one copy lane in need order, sub-products): parity, then timing
out=gpurun_out/grid3d_sched.txt
: > $out
timeout 900 python -m pytest -q -x tests/test_gpu_stencil_multi.py -k grid3d >> $out 2>&1
for rep in 1 2; do
  timeout 300 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 tools/grid3d_probe.py >> $out 2>/dev/null
done
timeout 300 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 tools/grid3d_probe.py >> $out 2>/dev/null
