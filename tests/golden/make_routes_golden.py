"""Generate tests/golden/ref_routes.json from the REFERENCE itself: the C++ caller
tools/cpp_example/routes_dump.cpp compiled against the unmodified reference headers
(oracle/_ref/routes_dump, D1 shim only) prints the whole RoutingPlan surface —
routes[*].params/optim CategorySets, route_of, pending with candidates, the
ScalarBroadcast, and the resolved transfers — for every scenario of ref_plans.json.
Only run in the build container (the GPU box has no /root/reference); the output is
committed.

    python tests/golden/make_routes_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.dirname(os.path.abspath(__file__))
FULL_MAX_LINES = 150


def main() -> None:
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"])
    exe = os.path.join(ROOT, "oracle", "_ref", "routes_dump")
    with open(os.path.join(OUT, "ref_plans.json")) as f:
        scenarios = [(e["name"], e["scenario"]) for e in json.load(f)["entries"]]
    entries = []
    for name, text in scenarios:
        with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as f:
            f.write(text)
        try:
            r = subprocess.run([exe, f.name], capture_output=True, text=True, timeout=600)
        finally:
            os.unlink(f.name)
        lines = r.stdout.splitlines()
        e = {"name": name, "rc": r.returncode, "sha256": hashlib.sha256(r.stdout.encode()).hexdigest(),
             "lines": len(lines), "last": lines[-1] if lines else ""}
        if len(lines) <= FULL_MAX_LINES:
            e["text"] = r.stdout
        entries.append(e)
        print(f"{name:50s} rc={r.returncode} lines={len(lines)}", flush=True)
    with open(os.path.join(OUT, "ref_routes.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_routes_golden.py via oracle/_ref/routes_dump "
                                "(tools/cpp_example/routes_dump.cpp against the reference headers + D1 shim)",
                   "entries": entries}, f, indent=1)


if __name__ == "__main__":
    main()
