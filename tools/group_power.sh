#!/bin/bash
# sustained pm_gemm TF/s + clock per raster group (wide kernel, dynamic scheduler)
for n in 16384 32768; do for g in 2 3 4 6; do
  echo -n "n=$n g=$g: "; PM_GEMM_GROUP=$g timeout -s KILL 120 python tools/power_probe.py $n 3 2>&1 | head -1
done; done
