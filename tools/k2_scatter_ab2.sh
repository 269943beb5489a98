# A/B of the scatter prologue / tiles per CTA on K2 and the fused K1+K2 (block + cyclic)
out=gpurun_out/k2sc2.txt
: > $out
B=paper_2507_17087_b200/csrc/build
for rep in 1 2; do
for lib in paper_2507_17087_b200/libmapple_b200.so $B/sc2_s1/lib.so $B/sc2_s4/lib.so; do
  echo "== $lib" >> $out
  MAPPLE_B200_LIB=$lib timeout 200 python tools/k12_probe.py >> $out 2>&1
done
done
timeout 900 python -m pytest -q -x tests/test_gpu_partition.py tests/test_gpu_map_partition.py tests/test_gpu_halo.py >> $out 2>&1
