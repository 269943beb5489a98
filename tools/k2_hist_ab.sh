# A/B of the K2 histogram: tiles per CTA (PM_HIST_TILES), prefetch distance
out=gpurun_out/k2hist.txt
: > $out
B=paper_2507_17087_b200/csrc/build
for rep in 1 2; do
for lib in paper_2507_17087_b200/libmapple_b200.so $B/hv_h2/lib.so $B/hv_h4/lib.so $B/hv_h2pf1200/lib.so; do
  echo "== $lib $(MAPPLE_B200_LIB=$lib timeout 200 python tools/k12_probe.py 2>&1 | tr '\n' ' ')" >> $out
done
done
