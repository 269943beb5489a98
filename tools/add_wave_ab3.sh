# (the default since this A/B: reduce-adding launches without the wave barrier; PM_GEMM_ADD_WAVE=1 restores it)
# reduce-adding launches without the wave barrier (default) vs with (PM_GEMM_ADD_WAVE=1):
# Johnson / COSMA at N=2 and N=4, interleaved on one box, 3 reps
out=gpurun_out/add_wave3.txt
: > $out
export PROBE_SHAPES=johnson PROBE_MAPPINGS=decompose
for rep in 1 2 3; do
for n in 2 4; do
  echo "== N=$n nowave $(timeout 300 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2964$n tools/grid3d_probe.py 2>/dev/null | grep world)" >> $out
  echo "== N=$n wave $(PM_GEMM_ADD_WAVE=1 timeout 300 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2965$n tools/grid3d_probe.py 2>/dev/null | grep world)" >> $out
done
done
