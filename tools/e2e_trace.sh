# e2e pipeline timeline at N=2 and N=4 (PM_E2E_TRACE: per-step H2D / multiply / D2H marks)
out=gpurun_out/e2e_trace.txt
: > $out
for n in 4 2; do
  echo "== N=$n" >> $out
  PM_E2E_TRACE=1 timeout 600 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2965$n bench.py --gpus $n --steps 10 --warmup 3 --no-kernels --decompose-only --no-3d --no-stencil --no-cannon --no-circuit --no-hydro --no-cpu > gpurun_out/e2e_n$n.json 2> gpurun_out/e2e_n$n.err
  grep e2e_trace gpurun_out/e2e_n$n.err >> $out
  python -c "import json;d=json.loads(open('gpurun_out/e2e_n$n.json').read().strip().splitlines()[-1]);print(d['value'],json.dumps(d['e2e']))" >> $out
done
