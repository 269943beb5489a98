# (historical: the PM_K1_* knobs were folded into the default -- 4 iterations per thread -- after these A/Bs)
# A/B of K1 (pm_map_points) grid size: groups of 4 points per thread (PM_K1_ITERS) on the
# 32768^2 block launch, and the cyclic launch for the chosen ones
out=gpurun_out/k1ab3.txt
: > $out
for rep in 1 2; do
for v in "PM_X=0" "PM_K1_CTAS=512" "PM_K1_ITERS=2" "PM_K1_ITERS=4" "PM_K1_ITERS=8" "PM_K1_ITERS=16" "PM_K1_ITERS=32"; do
  echo "== $v $(env $v timeout 200 python tools/k12_probe.py 2>&1 | head -2 | tr '\n' ' ')" >> $out
done
done
