#!/bin/bash
# Round-2 final one-GPU validation (what the driver runs): outputs under gpurun_out/r02z/.
O=gpurun_out/${OUT:-r02z}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=10 > $O/pytest_gpu.txt 2>&1; echo rc=$? >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo rc=$? >> $O/smoke.txt
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
timeout 900 python bench.py --impl reference > $O/ref_n1.json 2> $O/ref_n1.err
RS_TIMING=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_n1_timing.json 2> $O/bench_n1_timing.err
