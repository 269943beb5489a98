# (historical: PM_SUMMA_LEGACY was removed after this A/B -- new schedule +0.4-1.1%)
# SUMMA schedule A/B on one box (PM_SUMMA_LEGACY=1: the earlier schedule), N=4 and N=2
out=gpurun_out/summa_ab2.txt
: > $out
for rep in 1 2; do
for n in 4 2; do
for leg in 0 1; do
  PM_SUMMA_LEGACY=$leg timeout 900 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2968$n bench.py --gpus $n --no-kernels --no-3d --no-stencil --no-cannon --no-circuit --no-hydro --no-cpu --no-e2e > gpurun_out/summa_n$n.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/summa_n$n.json').read().strip().splitlines()[-1]);print('N=$n legacy=$leg', round(d['value']), round(d['ms_per_step'],3), d['gpu_launches'], round(d['roofline']['achieved']), round(d['decompose_vs_heuristic']['heuristic_tflops']), round(d['pumma']['decompose']['tflops']) if 'pumma' in d else None)" >> $out 2>&1
done
done
done
