# hydro 8-rank diagnosis: host barrier vs peer barrier, and 4 ranks on 2 GPUs
export PM_TEST_BACKEND=gloo PM_HANG_DUMP_S=240
run() {  # label nproc
  timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 \
    --master-port $((29300 + RANDOM % 300)) tests/dist_hydro_check.py > gpurun_out/ovh_$1.out 2> gpurun_out/ovh_$1.err
  echo "$1 rc $? $(grep '^{' gpurun_out/ovh_$1.out | tail -1 | cut -c1-30)" >> gpurun_out/ov2.log
}
PM_HOST_BARRIER=1 run hostbar8 8
run peer8 8
CUDA_VISIBLE_DEVICES=0,1 run peer4on2 4
CUDA_VISIBLE_DEVICES=0,1 PM_HOST_BARRIER=1 run hostbar4on2 4
