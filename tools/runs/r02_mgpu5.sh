#!/bin/bash
# Round-2 multi-GPU batch 5 (gpurun --gpus 4): outputs under gpurun_out/r02m5/.
O=gpurun_out/r02m5; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
CUDA_VISIBLE_DEVICES=0 RS_TIMING=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_n1.json 2> $O/bench_n1.err
for v in 0 1; do
  CUDA_VISIBLE_DEVICES=0,1 RS_INTERLEAVE_TILES=$v RS_TIMING=1 timeout 600 $TR --nproc-per-node 2 --master-port $((29910+v)) bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_n2_tiles$v.json 2> $O/bench_n2_tiles$v.err
  RS_INTERLEAVE_TILES=$v RS_TIMING=1 timeout 600 $TR --nproc-per-node 4 --master-port $((29920+v)) bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_n4_tiles$v.json 2> $O/bench_n4_tiles$v.err
done
timeout 1800 python -m pytest tests -m gpu -q -rs --durations=10 > $O/pytest_gpu.txt 2>&1; echo rc=$? >> $O/pytest_gpu.txt
