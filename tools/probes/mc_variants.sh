# multicast executor variants on config 3 grow (4 GPUs): serial/concurrent, CTAs per SM
for v in "RS_MC_SERIAL=1 RS_MC_CTAS_PER_SM=1" "RS_MC_SERIAL=1 RS_MC_CTAS_PER_SM=3" "RS_MC_CTAS_PER_SM=1" "RS_MC_CTAS_PER_SM=2"; do
env $v RS_TIMING=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 tools/bcast_bench.py --layers ${1:-32} > gpurun_out/mcv.log 2>&1
echo "== $v: $(grep '^{' gpurun_out/mcv.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["push"]["ms_min"], d["multicast"]["ms_min"], d["multicast"]["ms_per_rank"], d["multicast"]["mismatches"])')"
grep "run: multicast" gpurun_out/mcv.log | tail -1
done
