"""The tile cutter the executor runs on the host (counts, tile-level interleave) and on the
GPU (cut_kernel) is one definition (csrc/reshard/tiles.hpp); this host check pins it on
20,000 random copies: exact coverage, kTile bounds, alignment classes, and the record
splitting behind the record-level lane interleave cuts into identical tiles."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_tile_cutter_properties(tmp_path):
    exe = str(tmp_path / "tiles_check")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "paper_2605_18815_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "tiles_check.cpp"), "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("TILES_OK"), r.stdout + r.stderr


def test_host_pool_runs_each_index_once(tmp_path):
    """The persistent worker pool behind the planner and the descriptor build: 20,000
    back-to-back loops, every index exactly once (a worker leaving one loop must not claim
    an index of the next), exceptions propagated, nested loops inline."""
    exe = str(tmp_path / "pool_check")
    csrc = os.path.join(ROOT, "paper_2605_18815_b200", "csrc")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Werror", "-pthread", "-I", csrc,
                    os.path.join(ROOT, "tests", "cpp", "pool_check.cpp"), os.path.join(csrc, "pool.cpp"), "-o", exe],
                   check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("POOL_OK"), r.stdout + r.stderr
