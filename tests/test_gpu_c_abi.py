"""The C ABI from plain C (no Python binding): examples/c_abi_demo.c compiled
with gcc against include/af.h and libautofreeze.so reproduces the closed-form
tiny trace and a cache round trip with evict-on-read."""
import json
import os
import subprocess

import pytest

import paper_2102_01386_b200 as af

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_program_reproduces_closed_form_trace(tmp_path, golden):
    exe = tmp_path / "c_abi_demo"
    lib_dir = os.path.dirname(af.LIB_PATH)
    cmd = ["gcc", "-O2", "-std=c11", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "c_abi_demo.c"), "-L", lib_dir, "-l:libautofreeze.so",
           "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib_dir}", "-lm", "-o", str(exe)]
    subprocess.run(cmd, check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    bounds = [int(ln.split()[3]) for ln in lines if ln.startswith("T ")]
    assert bounds == golden("tiny_trace.json")["boundary_after"]
    assert lines[-1].startswith("cache roundtrip ok depths 2 2 2 valid_after_evict 0 err 0")


def test_training_loop_example_runs_and_freezes_monotonically():
    """examples/autofreeze_loop.py (small): the frozen prefix only grows, some
    layers freeze, and the cache serves hits from the epoch after a freeze."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("loop", os.path.join(ROOT, "examples", "autofreeze_loop.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    trace, hits = mod.run(epochs=3, small=True, verbose=False)
    assert trace == sorted(trace) and trace[-1] >= 1
    assert hits > 0


def test_zero_example_runs_and_freezes_monotonically():
    """examples/zero_loop.py at world 1 (the fused reduce-scatter + AdamW path):
    the frozen prefix only grows and some layers freeze."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("zero", os.path.join(ROOT, "examples", "zero_loop.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    trace = mod.run(intervals=8, verbose=False)
    assert trace == sorted(trace) and trace[-1] >= 1, trace
