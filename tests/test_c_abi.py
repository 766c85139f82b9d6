"""The drop-in boundary is a real C ABI: every function include/reshard_b200.h declares
is exported by libreshard_b200.so, and a plain-C caller reproduces the reference's own
plan dumps (output format of the reference CLI, incl. exit code 2 on ConfigError)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "reshard_b200.h")
LIB = os.path.join(ROOT, "paper_2605_18815_b200", "_lib", "libreshard_b200.so")


def declared():
    text = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(rs_[a-z_0-9]+)\s*\(", text, re.M)))


def test_every_declared_symbol_is_exported():
    from paper_2605_18815_b200 import _capi
    _capi.lib()
    names = declared()
    assert len(names) >= 40
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(rs_[a-z_0-9]+)$", out, re.M))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    # and the Python binding knows all of them
    assert set(_capi.EXPORTED) <= exported


@pytest.fixture(scope="module")
def c_caller(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("c") / "plan_dump")
    lib_dir = os.path.dirname(LIB)
    subprocess.run(["cc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tools", "c_example", "plan_dump.c"), "-L", lib_dir, "-lreshard_b200",
                    f"-Wl,-rpath,{lib_dir}", "-o", exe], check=True)
    return exe


def test_c_caller_reproduces_reference_dumps(c_caller, golden, tmp_path):
    n = 0
    for e in golden:
        if "dump" not in e and e["rc"] == 0:
            continue
        p = tmp_path / "s.txt"
        p.write_text(e["scenario"])
        r = subprocess.run([c_caller, str(p)], capture_output=True, text=True)
        assert r.returncode == e["rc"], (e["name"], r.stdout[-300:])
        if e["rc"] == 0:
            body, tail = r.stdout.rsplit("# transfers", 1)
            assert body == e["dump"], e["name"]
            assert f"bytes_moved={e['bytes_moved']}" in tail
        else:
            assert r.stdout.strip() == e["error"], e["name"]
        n += 1
    assert n >= 80


def test_cpp_caller_of_the_reference_routing_api(golden, tmp_path):
    """A C++ program written against the reference's routing API (plan_parameters,
    plan_optimizer, plan_scalars, resolve_peers, format_transfer) builds against this repo
    by switching its include path and prints the reference's own dump of config 1; with
    ZeRO it throws the reference's ConfigError (D2)."""
    exe = str(tmp_path / "routing_dump")
    lib_dir = os.path.dirname(LIB)
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "paper_2605_18815_b200", "csrc"),
                    os.path.join(ROOT, "tools", "cpp_example", "routing_dump.cpp"), "-L", lib_dir, "-lreshard_b200",
                    f"-Wl,-rpath,{lib_dir}", "-o", exe], check=True)
    ref = {e["name"]: e for e in golden}
    r = subprocess.run([exe], capture_output=True, text=True)
    body, tail = r.stdout.rsplit("# transfers", 1)
    e = ref["tiny-gpt.dp2tp2-to-tp4"]
    assert r.returncode == 0 and body == e["dump"]
    assert f"bytes_moved={e['bytes_moved']}" in tail and f"bytes_retained={e['bytes_retained']}" in tail
    r = subprocess.run([exe, "zero"], capture_output=True, text=True)
    assert r.returncode == 2 and r.stdout.strip() == ref["tiny-gpt.dp2tp2-to-tp4-zero1"]["error"]
