#!/bin/bash
# Stage-boundary cost of the memory-aware arena at N=4 (gpurun --gpus 4): outputs under
# gpurun_out/r02so/. SynchronizeAll latency, then the north star forced through ladder
# levels with 1 to many stages (caps not binding), device vs host barriers.
O=gpurun_out/r02so; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 300 $TR --nproc-per-node 4 --master-port 29971 tools/configs_bench.py --barrier-probe 1000 > $O/barrier_n4.json 2> $O/barrier_n4.err
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $TR --nproc-per-node 2 --master-port 29972 tools/configs_bench.py --barrier-probe 1000 > $O/barrier_n2.json 2> $O/barrier_n2.err
timeout 1500 $TR --nproc-per-node 4 --master-port 29973 tools/configs_bench.py --config 2 --layers 32 --arena-cap 170 \
    --level 0 --level 19 --level 36 --level 21 --level 38 --level 30 --both-barriers --reps 5 > $O/levels_n4.jsonl 2> $O/levels_n4.err
