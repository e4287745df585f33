"""bench.py's contract on CPU: the reference arm (the fp64 oracle, the only arm
that runs without a GPU) prints ONE JSON line with the driver's keys, and under
torchrun (world 2, gloo) rank 0 alone prints it while the other rank exits 0."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e")


def _lines(out):
    return [json.loads(x) for x in out.strip().splitlines() if x.startswith("{")]


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "bert-base-bf16", "--steps",
                        "1", "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1
    d = lines[0]
    for k in KEYS:
        assert k in d, k
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"] == "bert-base-bf16"


def test_reference_arm_rank0_only_under_torchrun():
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29641", "bench.py", "--impl", "reference",
                        "--workload", "bert-base-bf16", "--gpus", "2", "--steps", "1", "--warmup", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1 and lines[0]["impl"] == "reference"


def test_gpus_flag_self_launches_torchrun():
    # `python bench.py --gpus 2` without torchrun re-launches itself under
    # torch.distributed.run (one rank per GPU); the reference arm prints on rank 0 only
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "bert-base-bf16", "--gpus",
                        "2", "--steps", "1", "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env={k: v for k, v in dict(os.environ, CUDA_VISIBLE_DEVICES="").items()
                            if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
