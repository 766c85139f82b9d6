# bench.py at N=1, 2, 4 back to back (the driver's scaling run, up to this box's GPUs)
python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | grep "^{" > gpurun_out/scale_1.json
for n in 2 4; do
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | grep "^{" > gpurun_out/scale_$n.json
done
python - <<'PY'
import json
rows = [json.load(open(f"gpurun_out/scale_{n}.json")) for n in (1, 2, 4)]
out = {"metric": rows[0]["metric"], "unit": rows[0]["unit"],
       "runs": [{"n_gpus": r["n_gpus"], "value": r["value"], "ms_per_step": r["ms_per_step"], "reconfig_s": r["reconfig_s"],
                 "e2e": r["e2e"]["value"], "roofline_frac": r["roofline"]["frac"], "verified_mismatches": r["verified_mismatches"],
                 "clocks": r["clocks"]} for r in rows]}
json.dump(out, open("gpurun_out/scale.json", "w"), indent=1)
for r in out["runs"]: print(r["n_gpus"], r["value"], r["reconfig_s"], r["e2e"], r["roofline_frac"], r["verified_mismatches"])
PY
