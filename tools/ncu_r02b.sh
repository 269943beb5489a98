# round-2 late captures: K2 after the histogram L2 prefetch, hydro zones after the shuffle merge,
# then the 1-GPU test suite, the bench line and its launch list (each ncu after a clean run)
set -x
o=gpurun_out/ncu_r02b
mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -x -q > $o/pytest_gpu.log 2>&1
python bench.py > $o/bench_n1.json 2> $o/bench_n1.err
python tools/k2_probe.py && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_small -c 2 -o $o/k2 python tools/k2_probe.py > $o/k2.log 2>&1
python tools/hydro_probe.py && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hydro -c 2 -o $o/hydro python tools/hydro_probe.py > $o/hydro.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_bench_n1.csv python bench.py --steps 3 --warmup 3 --no-cpu > $o/bench_under_ncu.log 2>&1
echo done
