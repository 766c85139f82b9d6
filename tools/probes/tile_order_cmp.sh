# usage: bash tools/probes/tile_order_cmp.sh "<gpu counts>"  -- fused executor, op order vs lane interleave
for n in ${1:-4 2}; do for o in op interleave; do
RS_TIMING=1 RS_TILE_ORDER=$o timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n bench.py --gpus $n --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/o_${n}_$o.log 2>&1
echo "N=$n order=$o $(grep '^{' gpurun_out/o_${n}_$o.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["reconfig_s"], d["reconfig_back_s"], d["verified_mismatches"], d["roofline"]["achieved"], d["e2e"]["value"])')"
grep "prepare:\|e2e step" gpurun_out/o_${n}_$o.log | tail -8
done; done
