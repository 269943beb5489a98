# (historical: the PM_GEMM_ADD_* knobs were removed after this A/B -- no difference beyond noise)
# A/B at N=4 of GEMM knobs for the reduce-adding 3-D grids (tools/grid3d_probe.py)
out=gpurun_out/grid3d_ab.txt
: > $out
run() { echo "== $*" >> $out; env "$@" timeout 300 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 tools/grid3d_probe.py >> $out 2>gpurun_out/grid3d_err.txt; }
run PM_X=0
run PM_GEMM_ADD_NOWAVE=1  # (knob folded into the default after this A/B)
run PM_GEMM_WAVESYNC=0
run PM_X=0
run PM_GEMM_ADD_NOWAVE=1  # (knob folded into the default after this A/B)
