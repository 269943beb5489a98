# round-2 ncu captures (each after its own command ran clean): full sets of the changed
# kernels + the bench launch list
set -x
o=gpurun_out/ncu_r02
mkdir -p $o
python tools/gemm_one.py 32768 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_bf16_wide -c 1 -o $o/gemm_wide_32768 python tools/gemm_one.py 32768 > $o/gemm.log 2>&1
python tools/halo_probe.py && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_halo2d -c 2 -o $o/k3 python tools/halo_probe.py > $o/k3.log 2>&1
python tools/hydro_probe.py && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hydro -c 2 -o $o/hydro python tools/hydro_probe.py > $o/hydro.log 2>&1
python tools/circuit_probe.py 200 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_circuit_wires -c 1 -o $o/circuit python tools/circuit_probe.py 200 > $o/circuit.log 2>&1
python tools/stencil_probe.py 16384 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_jacobi -c 1 -o $o/stencil python tools/stencil_probe.py 16384 > $o/stencil.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu > $o/bench_plain.json 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_bench_n1.csv python bench.py --steps 3 --warmup 3 --no-cpu > $o/bench_under_ncu.log 2>&1
echo done
