"""Latency of a small (launch-bound) transition: plain launches vs CUDA-graph replay."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_18815_b200 import _capi as A  # noqa: E402
from paper_2605_18815_b200 import scenarios as S  # noqa: E402
from paper_2605_18815_b200.api import Executor, RoutingPlan  # noqa: E402

out = {}
for name, sc in (("config1", S.config1()), ("config1-zero", S.config1(zero=True))):
    plan = RoutingPlan.from_scenario(sc, allow_oversourced=True)
    ex = Executor(plan)
    ex.alloc()
    ex.fill(A.SIDE_SRC, 1)
    ex.prepare()
    st = torch.cuda.Stream()
    res = {}
    for mode, fn in (("launches", ex.run), ("graph", ex.run_graph)):
        for _ in range(20):
            fn(st.cuda_stream)
        st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(200):
            fn(st.cuda_stream)
        e1.record(st)
        st.synchronize()
        res[mode + "_us"] = round(e0.elapsed_time(e1) / 200 * 1e3, 2)
    res["bytes"] = plan.bytes_moved() + plan.bytes_retained()
    res["kernels_per_run"] = ex.stats().launches
    res["mismatches"] = ex.verify(A.SIDE_DST, 1)[0]
    out[name] = res
print(json.dumps(out))
