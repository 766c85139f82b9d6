#!/bin/bash
# Balanced co-location of the 8 devices at N=2 / N=4 (gpurun --gpus 4): bench lines for
# both placements, live + ncu DRAM traffic of the balanced placement. gpurun_out/r02co/.
O=gpurun_out/r02co; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29991 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err
timeout 900 $TR --nproc-per-node 4 --master-port 29992 bench.py --gpus 4 > $O/bench_n4.json 2> $O/bench_n4.err
timeout 900 $TR --nproc-per-node 4 --master-port 29993 bench.py --gpus 4 --placement contiguous --no-cpu-baseline > $O/bench_n4_contig.json 2> $O/bench_n4_contig.err
CUDA_VISIBLE_DEVICES=0,1 timeout 600 python tools/p2p_profile.py --layers 32 --reps 3 --gpus 2 --placement balanced > $O/live_n2.json 2> $O/live_n2.err
timeout 600 python tools/p2p_profile.py --layers 32 --reps 3 --gpus 4 --placement balanced > $O/live_n4.json 2> $O/live_n4.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
CUDA_VISIBLE_DEVICES=0,1 timeout 1200 ncu --replay-mode application --metrics $M --clock-control none -k regex:copy_tiles -c 2 --csv \
    --log-file $O/ncu_n2.csv python tools/p2p_profile.py --layers 32 --reps 1 --gpus 2 --placement balanced > $O/ncu_n2.out 2>&1
timeout 1200 ncu --replay-mode application --metrics $M --clock-control none -k regex:copy_tiles -c 4 --csv \
    --log-file $O/ncu_n4.csv python tools/p2p_profile.py --layers 32 --reps 1 --gpus 4 --placement balanced > $O/ncu_n4.out 2>&1
