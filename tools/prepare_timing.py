"""Where does per-reconfiguration host time go (plan, descriptors, upload)?"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["RS_TIMING"] = "1"
from paper_2605_18815_b200 import scenarios as S  # noqa: E402
from paper_2605_18815_b200.api import Arena, Executor, RoutingPlan  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32
sc = S.config2(L)
t0 = time.perf_counter()
ab = RoutingPlan.from_scenario(sc)
t1 = time.perf_counter()
ba = RoutingPlan.from_scenario(sc.reversed(), allow_oversourced=True)
t2 = time.perf_counter()
print(f"plan ab {1e3*(t1-t0):.1f} ms, plan ba (D2 ext) {1e3*(t2-t1):.1f} ms", flush=True)
arena = Arena(ab, ba)
t3 = time.perf_counter()
print(f"arena {1e3*(t3-t2):.1f} ms", flush=True)
e1, e2 = Executor(ab), Executor(ba)
arena.bind(e1, e2)
for i in range(3):
    t0 = time.perf_counter()
    e1.prepare()
    t1 = time.perf_counter()
    e2.prepare()
    t2 = time.perf_counter()
    e1.run(); e2.run(); torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"prepare fwd {1e3*(t1-t0):.1f} ms, bwd {1e3*(t2-t1):.1f} ms, run both {1e3*(t3-t2):.1f} ms", flush=True)
