#!/bin/bash
# 2-GPU check after host-side descriptor changes (gpurun --gpus 2): outputs under gpurun_out/r02c2/.
O=gpurun_out/r02c2; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -rs > $O/pytest_gpu.txt 2>&1; echo rc=$? >> $O/pytest_gpu.txt
RS_TIMING=1 timeout 900 $TR --nproc-per-node 2 --master-port 29981 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_n2_timing.json 2> $O/bench_n2_timing.err
timeout 900 $TR --nproc-per-node 2 --master-port 29982 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err
CUDA_VISIBLE_DEVICES=0 RS_TIMING=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_n1_timing.json 2> $O/bench_n1_timing.err
