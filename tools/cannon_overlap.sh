# Cannon / 2.5D with the shift pulls overlapping the GEMMs: parity (real ranks and 8 ranks
# sharing GPUs), then the Cannon bench leg at N=4
out=gpurun_out/cannon_overlap.txt
: > $out
timeout 1200 python -m pytest -q -x tests/test_gpu_stencil_multi.py -k "cannon or ranks_sharing" >> $out 2>&1
timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29684 bench.py --gpus 4 --no-kernels --no-3d --no-stencil --no-circuit --no-hydro --no-cpu --no-e2e > gpurun_out/cannon_n4.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/cannon_n4.json').read().strip().splitlines()[-1]);print(json.dumps(d['cannon']))" >> $out 2>&1
