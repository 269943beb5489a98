# (historical: the diagnostic knobs and the two-row kernel were removed after these runs)
# where the hydro zones kernel's time goes: without the force atomics, without the point
# gathers, without both (diagnostic builds, results invalid)
out=gpurun_out/hydro_diag.txt
: > $out
B=paper_2507_17087_b200/csrc/build
for rep in 1 2; do
for lib in paper_2507_17087_b200/libmapple_b200.so $B/hd_noat/lib.so $B/hd_nog/lib.so $B/hd_both/lib.so; do
  echo "== $lib $(MAPPLE_B200_LIB=$lib timeout 120 python tools/hydro_probe.py 2>&1 | tail -1)" >> $out
done
done
