# A/B of the K2 histogram: one warp per tile (loads in flight per lane) vs one CTA per tile
out=gpurun_out/k2histwarp.txt
: > $out
B=paper_2507_17087_b200/csrc/build
for rep in 1 2; do
  echo "== warp8 $(timeout 200 python tools/k12_probe.py 2>&1 | head -2 | tr '\n' ' ')" >> $out
  echo "== cta $(PM_HIST_CTA=1 timeout 200 python tools/k12_probe.py 2>&1 | head -2 | tr '\n' ' ')" >> $out
  echo "== warp4 $(MAPPLE_B200_LIB=$B/hw_w4/lib.so timeout 200 python tools/k12_probe.py 2>&1 | head -2 | tr '\n' ' ')" >> $out
  echo "== warp16 $(MAPPLE_B200_LIB=$B/hw_w16/lib.so timeout 200 python tools/k12_probe.py 2>&1 | head -2 | tr '\n' ' ')" >> $out
done
timeout 200 python tools/kernel_times.py 2>/dev/null | grep -E "k_small|k_halo2d_count|pm_map" | cut -c1-75,150-185 >> $out
timeout 1200 python -m pytest -q -x tests/test_gpu_partition.py tests/test_gpu_map_partition.py tests/test_gpu_halo.py >> $out 2>&1
