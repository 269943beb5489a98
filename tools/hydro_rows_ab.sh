# (historical: the diagnostic knobs and the two-row kernel were removed after these runs)
# hydro zones: two-row CTAs (zones_w hint) vs the 1-D kernel (PM_HYDRO_1D=1), then parity
out=gpurun_out/hydro_rows.txt
: > $out
for rep in 1 2 3; do
  echo "== rows $(timeout 120 python tools/hydro_probe.py 2>&1 | tail -1)" >> $out
  echo "== 1d $(PM_HYDRO_1D=1 timeout 120 python tools/hydro_probe.py 2>&1 | tail -1)" >> $out
done
timeout 900 python -m pytest -q -x tests/test_gpu_stencil_multi.py -k hydro >> $out 2>&1
