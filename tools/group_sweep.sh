#!/bin/bash
# raster group sweep: DRAM bytes (ncu) and sustained TF/s / clock / power per PM_GEMM_GROUP
for g in 4 8 16; do
  echo "== group $g"
  PM_GEMM_GROUP=$g timeout 120 python tools/power_probe.py 16384 3 2>&1 | head -1
done
