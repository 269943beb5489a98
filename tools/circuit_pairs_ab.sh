# (historical: the packed-FP32 pair kernel was removed after this A/B -- slower)
# circuit wires: packed FP32 pairs (FFMA2) vs scalar; bit-exactness; parity tests
out=gpurun_out/circuit_pairs.txt
: > $out
for rep in 1 2; do
  echo "== pairs $(timeout 300 python tools/circuit_probe.py 2>&1 | tail -1)" >> $out
  echo "== scalar $(PM_CIRCUIT_SCALAR=1 timeout 300 python tools/circuit_probe.py 2>&1 | tail -1)" >> $out
done
timeout 300 python tools/circuit_exact.py gpurun_out/c_pairs.npz >> $out 2>&1
PM_CIRCUIT_SCALAR=1 timeout 300 python tools/circuit_exact.py gpurun_out/c_scalar.npz >> $out 2>&1
python -c "
import numpy as np
a=np.load('gpurun_out/c_pairs.npz'); b=np.load('gpurun_out/c_scalar.npz')
print('bit-exact', {k: bool((a[k].view(np.uint32)==b[k].view(np.uint32)).all()) for k in a.files})
" >> $out 2>&1
timeout 900 python -m pytest -q -x tests/test_gpu_stencil_multi.py -k circuit >> $out 2>&1
