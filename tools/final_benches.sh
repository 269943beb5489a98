# final round-2 bench lines: N=4, N=2 (torchrun) then N=1, plus the reference arm at N=1
o=gpurun_out/final_r02c
mkdir -p $o
timeout 1200 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29701 bench.py --gpus 4 > $o/bench_n4.json 2> $o/bench_n4.err
timeout 1200 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29702 bench.py --gpus 2 > $o/bench_n2.json 2> $o/bench_n2.err
CUDA_VISIBLE_DEVICES=0 timeout 1200 python bench.py > $o/bench_n1.json 2> $o/bench_n1.err
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference > $o/bench_ref_n1.json 2> $o/bench_ref_n1.err
echo done
