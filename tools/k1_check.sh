out=gpurun_out/k1check.txt
: > $out
timeout 200 python tools/k12_probe.py >> $out 2>&1
timeout 1200 python -m pytest -q -x tests/test_gpu_mapping.py tests/test_gpu_map_partition.py tests/test_gpu_partition.py tests/test_gpu_reference_consumers.py >> $out 2>&1
