# (historical: the PM_HYDRO_PAIRS kernel and zone reorder were removed after this A/B)
# A/B: one zone per thread with row shuffle merge (default) vs row-pair zones (PM_HYDRO_PAIRS=1),
# vs no merge (var_hz0); then the hydro parity checks under the pairs kernel.
out=gpurun_out/hydro_ab2.txt
: > $out
for rep in 1 2; do
  echo "== row-merge" >> $out; timeout 120 python tools/hydro_probe.py >> $out 2>&1
  echo "== pairs" >> $out; PM_HYDRO_PAIRS=1 timeout 120 python tools/hydro_probe.py >> $out 2>&1
  echo "== no-merge" >> $out; MAPPLE_B200_LIB=paper_2507_17087_b200/csrc/build/var_hz0/lib.so timeout 120 python tools/hydro_probe.py >> $out 2>&1
done
PM_HYDRO_PAIRS=1 timeout 900 python -m pytest -q -x tests/test_gpu_stencil_multi.py -k hydro >> $out 2>&1
timeout 900 python -m pytest -q -x tests/test_gpu_stencil_multi.py -k hydro >> $out 2>&1
