# (historical: PM_HYDRO_PAIR_ATOMICS was removed after this A/B -- slower)
# hydro zones: paired 16-byte force atomics vs one 8-byte atomic per merged corner, then parity
out=gpurun_out/hydro_pair.txt
: > $out
for rep in 1 2 3; do
  echo "== pair $(timeout 120 python tools/hydro_probe.py 2>&1 | tail -1)" >> $out
  echo "== nopair $(MAPPLE_B200_LIB=paper_2507_17087_b200/csrc/build/hp0/lib.so timeout 120 python tools/hydro_probe.py 2>&1 | tail -1)" >> $out
done
timeout 900 python -m pytest -q -x tests/test_gpu_stencil_multi.py -k hydro >> $out 2>&1
