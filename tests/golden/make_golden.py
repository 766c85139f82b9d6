"""Generate tests/golden/ from the REFERENCE itself (oracle/_ref/ref_plan).

ref_plan compiles the unmodified reference headers from /root/reference/proj/include
(plus the one-line D1 shim, oracle/ref_plan.cpp). This script runs it on a fixed
list of scenarios and records, per scenario: the scenario text, the exit code, the
sha256 of the plan dump, counts/bytes, and (for small plans) the full dump. Only run
in the build container (the GPU box has no /root/reference); the outputs are
committed.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_2605_18815_b200 import scenarios as S  # noqa: E402
import pyoracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
FULL_DUMP_MAX_LINES = 400


def kat_scenarios():
    T, M, Cfg, Sc = S.Tensor, S.Model, S.Cfg, S.Scenario
    out = []
    # SPEC.md:76 VPS offsets: A[4,4], B[8] -> off(B)=16, total 24
    m = M("kat-vps", [T("A", (4, 4), 0), T("B", (8,), 0)])
    out.append(Sc(m, Cfg(), Cfg(), name="kat.vps.identity"))
    # W[4,4] axis-0 sharded, tp 2 -> 4
    m = M("kat-w", [T("W", (4, 4), 0, tp=0)])
    out.append(Sc(m, Cfg(tp=2), Cfg(tp=4), name="kat.tp2-to-tp4"))
    out.append(Sc(m, Cfg(tp=4), Cfg(tp=2), name="kat.tp4-to-tp2"))
    # pure replication dp=k
    out.append(Sc(m, Cfg(dp=3), Cfg(dp=2), name="kat.dp3-to-dp2"))
    # ZeRO A(30), B(45), C(25)
    m = M("kat-abc", [T("A", (30,), 0), T("B", (45,), 0), T("C", (25,), 0)])
    out.append(Sc(m, Cfg(dp=2, zero=True), Cfg(dp=3, zero=True), name="kat.zero-abc.dp2-to-dp3"))
    out.append(Sc(m, Cfg(dp=4, zero=True), Cfg(dp=2, zero=True), name="kat.zero-abc.dp4-to-dp2"))
    out.append(Sc(m, Cfg(dp=2, zero=True), Cfg(dp=4, zero=True), name="kat.zero-abc.dp2-to-dp4"))
    # SPEC.md:185 / Fig. 4: (TP,PP) = (2,2) -> (4,1)
    fig = M("fig4", [T("l0.w1", (8, 8), 0, tp=0), T("l0.w2", (8, 8), 0, tp=1), T("l0.n", (8,), 0),
                     T("l1.w1", (8, 8), 1, tp=0), T("l1.w2", (8, 8), 1, tp=1), T("l1.n", (8,), 1)], layers=2)
    out.append(Sc(fig, Cfg(tp=2, pp=2), Cfg(tp=4), name="fig4.tp2pp2-to-tp4"))
    out.append(Sc(fig, Cfg(tp=2, pp=2, zero=True), Cfg(tp=4, zero=True), name="fig4.tp2pp2-to-tp4.zero-D2"))
    out.append(Sc(fig, Cfg(tp=2, pp=2, dp=2, zero=True), Cfg(tp=4, dp=2, zero=True), name="fig4.dp2.zero-D2"))
    out.append(Sc(fig, Cfg(tp=1, pp=2, dp=2, zero=True), Cfg(tp=2, pp=1, dp=2, zero=True), name="fig4.tp1pp2dp2-to-tp2dp2.zero"))
    # dp 1 -> 2 replication with proximity over 2 nodes
    m = M("kat-prox", [T("W", (4, 4), 0, tp=0), T("b", (4,), 0)])
    out.append(Sc(m, Cfg(dp=2), Cfg(dp=4), nodes=2, rpn=2, name="kat.prox.dp2-to-dp4.2nodes"))
    out.append(Sc(m, Cfg(dp=2), Cfg(dp=4), nodes=2, rpn=2, balance=True, name="kat.prox.balance"))
    out.append(Sc(m, Cfg(dp=2, tp=2), Cfg(dp=1, tp=4), grads="migrate", name="kat.migrate"))
    # world-map join/leave (worldmap.hpp:30-79)
    out.append(Sc(m, Cfg(dp=4), Cfg(dp=2), world_src=[0, 1, 2, 3], world_dst=[3, 1], name="kat.world.shrink-renumber"))
    out.append(Sc(m, Cfg(dp=2, zero=True), Cfg(dp=4, zero=True), world_src=[5, 2], world_dst=[0, 2, 4, 5], name="kat.world.grow-zero"))
    # errors
    out.append(Sc(m, Cfg(tp=3), Cfg(tp=2), name="err.tp3"))
    out.append(Sc(m, Cfg(dp=2, zero=True), Cfg(dp=2), name="err.zero-toggle"))
    out.append(Sc(m, Cfg(dp=2, order="pp-dp-xx"), Cfg(dp=2), name="err.order"))
    return out


def baseline_scenarios():
    out = [S.config1(False), S.config1(True), S.config2(1), S.config2(2)]
    shrink, grow = S.config3(32)
    out += [shrink, grow]
    out.append(S.config4(1))
    out.append(S.config5(2))
    return out


def campaign_scenarios(n: int = 80, seed: int = 2605):
    rng = random.Random(seed)
    out = []
    for i in range(n):
        experts = rng.choice([1, 1, 1, 4])
        m = S.toy_model(rng, experts=experts, with_replicated=rng.random() < 0.5)
        zero = rng.random() < 0.5
        src = S.random_cfg(rng, m, zero=zero)
        dst = S.random_cfg(rng, m, zero=zero)
        sc = S.Scenario(m, src, dst, name=f"campaign.{i:03d}")
        r = rng.random()
        if r < 0.15:
            # shuffled renumbering with joins/leaves over a pool of devices
            pool = list(range(max(src.world(), dst.world()) + 2))
            sc.world_src = rng.sample(pool, src.world())
            sc.world_dst = rng.sample(pool, dst.world())
        if rng.random() < 0.2:
            sc.nodes, sc.rpn = 4, 4
        if rng.random() < 0.15:
            sc.balance = True
        if rng.random() < 0.15:
            sc.grads = "migrate"
        out.append(sc)
    return out


def main() -> None:
    """Regenerate every group, or with `--append GROUP` add/replace one group in place."""
    if not pyoracle.ref_available():
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"])
    all_groups = {"kat": kat_scenarios, "baseline": baseline_scenarios, "campaign": campaign_scenarios,
                  "edge": S.edge_scenarios}
    entries = []
    groups = [(g, f()) for g, f in all_groups.items()]
    if len(sys.argv) > 2 and sys.argv[1] == "--append":
        with open(os.path.join(OUT, "ref_plans.json")) as f:
            entries = [e for e in json.load(f)["entries"] if e["group"] != sys.argv[2]]
        groups = [(sys.argv[2], all_groups[sys.argv[2]]())]
    for group, scs in groups:
        for sc in scs:
            text = sc.text()
            t0 = time.time()
            rc, out = pyoracle.ref_plan(text, timeout=3600)
            dt = time.time() - t0
            lines = out.splitlines()
            tail = lines[-1] if lines else ""
            body = "\n".join(lines[:-1]) + ("\n" if len(lines) > 1 else "")
            e = {"name": sc.name, "group": group, "scenario": text, "rc": rc, "ref_seconds": round(dt, 3)}
            if rc == 0:
                kv = dict(x.split("=") for x in tail[2:].split())
                e.update(transfers=int(kv["transfers"]), bytes_moved=int(kv["bytes_moved"]),
                         bytes_retained=int(kv["bytes_retained"]),
                         sha256=hashlib.sha256(body.encode()).hexdigest(),
                         head=lines[:3])
                if len(lines) - 1 <= FULL_DUMP_MAX_LINES:
                    e["dump"] = body
            else:
                e["error"] = tail
            if group == "kat" and rc == 0:
                for side in ("src", "dst"):
                    rrc, reg = pyoracle.ref_plan(text, cmd=f"regions-{side}")
                    e[f"regions_{side}"] = reg
            entries.append(e)
            print(f"{sc.name:50s} rc={rc} {tail[:90]} ({dt:.1f}s)", flush=True)
    with open(os.path.join(OUT, "ref_plans.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py via oracle/_ref/ref_plan (reference headers + D1 shim)",
                   "entries": entries}, f, indent=1)


if __name__ == "__main__":
    main()
