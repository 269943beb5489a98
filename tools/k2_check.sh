out=gpurun_out/k2check.txt
: > $out
timeout 200 python tools/k12_probe.py >> $out 2>&1
timeout 200 python tools/kernel_times.py 2>/dev/null | grep -E "k_small|k_halo2d_count|pm_map" | cut -c1-75,150-185 >> $out
timeout 1200 python -m pytest -q -x tests/test_gpu_partition.py tests/test_gpu_map_partition.py tests/test_gpu_halo.py >> $out 2>&1
