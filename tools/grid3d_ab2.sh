# (historical: the PM_GEMM_ADD_* knobs were removed after this A/B -- no difference beyond noise)
# Johnson decompose (K-split grids) at N=2 and N=4: reduce-adding launches with / without the
# wave barrier and with a slack (tools/grid3d_probe.py)
out=gpurun_out/grid3d_ab2.txt
: > $out
export PROBE_SHAPES=johnson PROBE_MAPPINGS=decompose
run() { n=$1; shift; echo "== N=$n $*" >> $out; env "$@" timeout 300 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n tools/grid3d_probe.py >> $out 2>>gpurun_out/grid3d_err.txt; }
for n in 2 4; do
  run $n PM_X=0
  run $n PM_GEMM_ADD_WAVE=1
  run $n PM_GEMM_ADD_WAVE=1 PM_GEMM_ADD_SLACK=37
  run $n PM_GEMM_ADD_WAVE=1 PM_GEMM_ADD_SLACK=18
  run $n PM_X=0
  run $n PM_GEMM_ADD_WAVE=1
done
