# late round-2 ncu full captures of the mapping kernels changed last: K1 (short-lived CTAs),
# K2 histogram (warp per tile) and scatter (2 tiles per CTA), fused K1+K2 scatter
o=gpurun_out/ncu_r02c
mkdir -p $o
python tools/k12_probe.py 2 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"pm_map_points|k_small_hist_warp|k_small_scatter|pm_map_scatter" -c 4 -o $o/mapping python tools/k12_probe.py 2 > $o/mapping.log 2>&1
echo done
