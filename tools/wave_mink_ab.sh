# (historical: PM_GEMM_WAVE_MIN_K was removed -- the wave barrier on every launch measured better for SUMMA at N=2/N=4)
# wave barrier only for K >= 24576 (default) vs always (PM_GEMM_WAVE_MIN_K=0): N=4 and N=2
# SUMMA / PUMMA / 3-D legs, interleaved on one box
out=gpurun_out/wave_mink.txt
: > $out
for rep in 1 2; do
for n in 4 2; do
for mk in 24576 0; do
  PM_GEMM_WAVE_MIN_K=$mk timeout 900 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2969$n bench.py --gpus $n --no-kernels --no-stencil --no-cannon --no-circuit --no-hydro --no-cpu --no-e2e > gpurun_out/wm.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/wm.json').read().strip().splitlines()[-1]);w=d['workloads_3d'];p=d['pumma'];print('N=$n mink=$mk', round(d['value']), round(d['decompose_vs_heuristic']['heuristic_tflops']), 'pumma', round(p['decompose']['tflops']), round(p['heuristic']['tflops']), 'johnson', round(w['johnson3d']['decompose']['tflops']), round(w['johnson3d']['heuristic']['tflops']), 'cosma', round(w['cosma']['decompose']['tflops']), round(w['cosma']['heuristic']['tflops']))" >> $out 2>&1
done
done
done
