#!/bin/bash
O=gpurun_out/r02m7; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
for rep in 1 2; do
for v in 0 1; do
  CUDA_VISIBLE_DEVICES=0,1 RS_INTERLEAVE_TILES=$v timeout 600 $TR --nproc-per-node 2 --master-port $((29940+v+10*rep)) bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_n2_tiles${v}_$rep.json 2> $O/bench_n2_tiles${v}_$rep.err
  RS_INTERLEAVE_TILES=$v timeout 600 $TR --nproc-per-node 4 --master-port $((29950+v+10*rep)) bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_n4_tiles${v}_$rep.json 2> $O/bench_n4_tiles${v}_$rep.err
done
done
timeout 900 python -m pytest tests/test_gpu_exec.py -m gpu -q -k "multi_gpu or collectives or staged or eight" > $O/pytest_mgpu.txt 2>&1; echo rc=$? >> $O/pytest_mgpu.txt
