# A/B of the K2 histogram-pass L2 prefetch distance (PM_HIST_PREFETCH_TILES variants built
# under csrc/build/var_hpf*/): block-structured and random ids, twice each, interleaved.
out=gpurun_out/k2pf.txt
: > $out
for rep in 1 2; do
for lib in paper_2507_17087_b200/libmapple_b200.so paper_2507_17087_b200/csrc/build/var_hpf600/lib.so paper_2507_17087_b200/csrc/build/var_hpf1200/lib.so paper_2507_17087_b200/csrc/build/var_hpf2400/lib.so; do
  echo "== $lib" >> $out
  MAPPLE_B200_LIB=$lib timeout 120 python tools/k2_probe.py >> $out 2>&1
  MAPPLE_B200_LIB=$lib timeout 120 python tools/halo_probe.py >> $out 2>&1
done
done
MAPPLE_B200_LIB=paper_2507_17087_b200/csrc/build/var_hpf1200/lib.so timeout 600 python -m pytest -q -x tests/test_gpu_partition.py tests/test_gpu_map_partition.py tests/test_gpu_halo.py >> $out 2>&1
