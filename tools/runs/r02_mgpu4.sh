#!/bin/bash
# Round-2 multi-GPU batch 4 (gpurun --gpus 4): outputs under gpurun_out/r02m4/.
O=gpurun_out/r02m4; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
CUDA_VISIBLE_DEVICES=0,1 RS_TIMING=1 timeout 600 $TR --nproc-per-node 2 --master-port 29901 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_n2.json 2> $O/bench_n2.err
RS_TIMING=1 timeout 600 $TR --nproc-per-node 4 --master-port 29902 bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_n4.json 2> $O/bench_n4.err
timeout 600 $TR --nproc-per-node 4 --master-port 29903 bench.py --impl reference --gpus 4 --steps 3 --warmup 1 > $O/ref_n4.json 2> $O/ref_n4.err
timeout 900 $TR --nproc-per-node 4 --master-port 29904 tools/configs_bench.py --config 1 --reps 20 > $O/configs_c1_n4.jsonl 2> $O/configs_c1.err
timeout 900 $TR --nproc-per-node 4 --master-port 29905 tools/configs_bench.py --config 4 --layers 24 --reps 3 > $O/configs_c4_n4.jsonl 2> $O/configs_c4.err
timeout 900 $TR --nproc-per-node 4 --master-port 29906 tools/configs_bench.py --config 3 --reps 3 > $O/configs_c3_n4.jsonl 2> $O/configs_c3.err
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/configs_bench.py --config 1 --reps 20 > $O/configs_c1_n1.jsonl 2> $O/configs_c1_n1.err
timeout 900 $TR --nproc-per-node 4 --master-port 29907 tools/bcast_bench.py --layers 32 --reps 3 > $O/bcast_config3_n4_L32.json 2> $O/bcast.err
timeout 1800 python -m pytest tests -m gpu -q -rs --durations=10 > $O/pytest_gpu.txt 2>&1; echo rc=$? >> $O/pytest_gpu.txt
