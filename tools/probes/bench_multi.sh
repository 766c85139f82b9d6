# bench lines at N=2 and N=4 (plain allocations), and N=2 under an HBM cap (multi-GPU arena)
run() { n=$1; shift; timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2959$n bench.py --gpus $n --steps 5 --warmup 3 "$@" 2>/dev/null | grep "^{"; }
run 4 --no-cpu-baseline > gpurun_out/bench_n4.json
run 2 > gpurun_out/bench_n2.json
run 2 --no-cpu-baseline --arena-multi --hbm-cap 100000000000 > gpurun_out/bench_n2_cap100.json
run 2 --no-cpu-baseline --arena-multi --hbm-cap 80000000000 > gpurun_out/bench_n2_cap80.json
for f in gpurun_out/bench_n4.json gpurun_out/bench_n2.json gpurun_out/bench_n2_cap100.json gpurun_out/bench_n2_cap80.json; do
python -c "import json,sys; d=json.load(open('$f')); r=d['roofline']; print('$f', d['value'], d['reconfig_s'], d['reconfig_back_s'], d['verified_mismatches'], r['achieved'], r['frac'], r['frac_of_nominal_900'], d['e2e']['value'], d.get('memory', {}).get('physical_gb'), d.get('memory', {}).get('stage_groups'))" || echo "$f failed"
done
