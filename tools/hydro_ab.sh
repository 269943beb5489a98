# A/B of hydro kernel variants (csrc/build/var_hz*/): per-phase times, twice each, interleaved,
# then the hydro GPU tests on the default build.
out=gpurun_out/hydro_ab.txt
: > $out
for rep in 1 2; do
for lib in paper_2507_17087_b200/libmapple_b200.so "$@"; do
  echo "== $lib" >> $out
  MAPPLE_B200_LIB=$lib timeout 120 python tools/hydro_probe.py >> $out 2>&1
done
done
timeout 600 python -m pytest -q -x tests/test_gpu_stencil_multi.py -k hydro >> $out 2>&1
