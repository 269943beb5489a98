# wide GEMM: raster group x wave barrier -- sustained TF/s / clock / power (power_probe)
# and DRAM bytes per launch (ncu), at 16384^3 and 32768^3
out=gpurun_out/gemm_wave.txt
for n in 32768 16384; do
  for cfg in "0 0" "1 8" "1 4" "1 16" "0 8"; do
    set -- $cfg
    echo "== n=$n wavesync=$1 group=$2" >> $out
    if [ "$2" = "0" ]; then unset PM_GEMM_GROUP; else export PM_GEMM_GROUP=$2; fi
    PM_GEMM_WAVESYNC=$1 timeout 120 python tools/power_probe.py $n 3 2>&1 | head -2 >> $out
    PM_GEMM_WAVESYNC=$1 timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum \
      --clock-control none -k regex:k_gemm_bf16_wide -c 1 python tools/gemm_one.py $n 2>&1 \
      | grep -E "dram__bytes_read|gpu__time" >> $out
  done
done
unset PM_GEMM_GROUP
