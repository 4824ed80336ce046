"""bench.py's launch contract: one JSON line from rank 0 under torchrun; the reference arm
on CPU; the N > 1 path with two ranks sharing one GPU (gloo; SPECDEC_BENCH_SHARE_GPU)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(n, args, env=None, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(ROOT, "bench.py"), "--gpus", str(n)] + args
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT,
                       env={**os.environ, **(env or {})})
    assert r.returncode == 0, r.stderr[-2000:]
    return [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]


def test_reference_arm_rank0_only():
    """--impl reference under torchrun: rank 0 alone prints one line (the oracle timed on
    the host); the other rank exits 0 without work."""
    lines = _torchrun(2, ["--impl", "reference", "--config", "toy", "--steps", "2", "--warmup", "1"])
    assert len(lines) == 1
    d = lines[0]
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "rounds/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["toy", "pool"])
def test_two_ranks_share_one_gpu(config):
    extra = ["--steps", "5", "--warmup", "3", "--no-cpu-baseline"]
    if config == "pool":
        extra += ["--config", "pool", "--pool-n", "32", "--max-new", "24"]
    else:
        extra += ["--config", "toy"]
    lines = _torchrun(2, extra, env={"SPECDEC_BENCH_SHARE_GPU": "1"})
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    if config == "pool":
        assert d["scaling"] == "strong"
    else:
        assert d["scaling"] == "weak" and d["e2e"]["value"] > 0
