"""The reference's C++ routing API surface (routing.hpp:93-193) as a drop-in: the caller
tools/cpp_example/routes_dump.cpp reads routes[*].params / .optim CategorySets
(src, dst, send, recv, retain), route_of(), the pending fragments with their candidates,
the ScalarBroadcast (scalars->recv_phys ...), then resolve_peers' transfers,
bytes_moved() and bytes_retained(space). Compiled against csrc/reshard/ and linked to
libreshard_b200.so, its output must equal the same file compiled against the reference
headers (tests/golden/ref_routes.json, made by make_routes_golden.py) on every golden
scenario: KATs, BASELINE configs (incl. D2 errors), the random campaign, edge cases."""
import hashlib
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_DIR = os.path.join(ROOT, "paper_2605_18815_b200", "_lib")


@pytest.fixture(scope="module")
def routes_dump(tmp_path_factory):
    from paper_2605_18815_b200 import _capi
    _capi.lib()  # built
    exe = str(tmp_path_factory.mktemp("cpp") / "routes_dump")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "paper_2605_18815_b200", "csrc"),
                    "-I", os.path.join(ROOT, "tools", "cpp_example"),
                    os.path.join(ROOT, "tools", "cpp_example", "routes_dump.cpp"), "-L", LIB_DIR, "-lreshard_b200",
                    f"-Wl,-rpath,{LIB_DIR}", "-o", exe], check=True)
    return exe


def test_routes_pending_scalars_match_reference(routes_dump, golden, tmp_path):
    with open(os.path.join(ROOT, "tests", "golden", "ref_routes.json")) as f:
        ref = {e["name"]: e for e in json.load(f)["entries"]}
    n = full = 0
    for e in golden:
        want = ref[e["name"]]
        p = tmp_path / "s.txt"
        p.write_text(e["scenario"])
        r = subprocess.run([routes_dump, str(p)], capture_output=True, text=True, timeout=300)
        assert r.returncode == want["rc"], (e["name"], r.stdout[-300:])
        if "text" in want:
            assert r.stdout == want["text"], e["name"]
            full += 1
        assert hashlib.sha256(r.stdout.encode()).hexdigest() == want["sha256"], (e["name"], want["last"])
        n += 1
    assert n >= 100 and full >= 30


def test_routes_fields_are_populated(routes_dump, tmp_path):
    """Fig. 4 with ZeRO on both sides but dp=1 on the source (no D2): every route has a
    parameter and an optimizer category set, pending is consumed by resolve_peers, and
    the scalar broadcast reaches every other destination device."""
    from paper_2605_18815_b200 import scenarios as S
    fig = S.Model("fig4", [S.Tensor("l0.w1", (8, 8), 0, tp=0), S.Tensor("l0.w2", (8, 8), 0, tp=1),
                           S.Tensor("l1.w1", (8, 8), 1, tp=0), S.Tensor("l1.w2", (8, 8), 1, tp=1)], layers=2)
    sc = S.Scenario(fig, S.Cfg(tp=2, pp=2, zero=True), S.Cfg(tp=4, zero=True))
    p = tmp_path / "s.txt"
    p.write_text(sc.text())
    out = subprocess.run([routes_dump, str(p)], capture_output=True, text=True, check=True).stdout
    assert out.count("route phys=") == 4
    assert "  optim.recv flat" in out and "  params.retain box" in out and "pending optim - [" in out
    assert "scalars root_phys=0 root_src_rank=0 words=8 bytes_per_rank=64 recv=1,2,3" in out
    assert "resolved=1 pending=0 " in out
