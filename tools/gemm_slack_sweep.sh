for n in 16384 32768; do for sl in 0 4 16 37; do
  echo "== n=$n slack=$sl" >> gpurun_out/gemm_slack.txt
  PM_GEMM_WAVE_SLACK=$sl timeout 120 python tools/power_probe.py $n 3 2>&1 | head -2 >> gpurun_out/gemm_slack.txt
done; done
