# (historical: variants built by tools/build_variant.sh; PM_SCATTER_TILES=2 became the default)
# A/B of the K2 scatter: tiles per CTA (PM_SCATTER_TILES) and streaming vs plain iota stores
out=gpurun_out/k2sc.txt
: > $out
B=paper_2507_17087_b200/csrc/build
for rep in 1 2; do
for lib in paper_2507_17087_b200/libmapple_b200.so $B/sc_t2/lib.so $B/sc_t4/lib.so $B/sc_t8/lib.so $B/sc_t1nocs/lib.so $B/sc_t4nocs/lib.so; do
  echo "== $lib $(MAPPLE_B200_LIB=$lib timeout 120 python tools/k2_probe.py 2>&1 | tail -1)" >> $out
done
done
MAPPLE_B200_LIB=$B/sc_t4/lib.so timeout 900 python -m pytest -q -x tests/test_gpu_partition.py tests/test_gpu_map_partition.py tests/test_gpu_halo.py >> $out 2>&1
