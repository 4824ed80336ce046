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


@pytest.mark.gpu
def test_default_line_has_the_contract_keys():
    """`python bench.py` (N=1) prints one JSON line with every key the driver reads:
    value / unit / timing fields, roofline (bound, achieved, peak, unit, frac, traffic),
    cpu_baseline (oracle), e2e (host-buffer copies counted), gpu_launches, clocks."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "6", "--warmup", "3"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
                "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 6 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["config"]["workload"] and d["data"] == "synthetic" and d["dtype"] == "bf16"
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9 and 0.5 < rf["frac"] < 1.2
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 14_000_000 and e["d2h_bytes_per_step"] > 0
    from paper_2510_22876_b200 import _abi
    assert d["gpu_launches"] == (2 + _abi.specdec_verify_kernels(False)) * 6      # K1, K3, K2
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert d["bytes_moved_check"]["value_region"] == d["bytes_moved_check"]["kernel_region"]
    kp = d["k2_per_launch"]                    # per-launch K2 rates (region B's 6 launches)
    assert kp["launches"] == 6 and kp["GBps_quartiles"][2] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["epoch", "alg3", "pipelined"])
def test_pool_line_drain_matches_the_oracle(mode):
    """The pool line's timed drain (native executor with the default deferred fallback; Alg. 3:
    the graph-replayed device loop; pipelined: R28) against the oracle's own plan-driven drain
    of the same workload (the cpu_baseline leg): batches, same-length batches and members,
    fallback members and KV bytes, exactly; the whole-drain byte roofline is reported."""
    extra = ["--pool-pipeline", "1"] if mode == "pipelined" else ["--pool-mode", mode]
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "pool", "--pool-n", "192",
                        "--max-new", "64"] + extra, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    chk = d["oracle_drain_check"]
    assert chk["match"], chk
    assert d["cpu_baseline"]["kind"] == "oracle" and d["gpu_launches"] > 0 and d["status"] == 0
    dr = d["roofline"]["drain"]
    assert dr["bytes"] == dr["kv_bytes"] + dr["logit_bytes"] and 0 < dr["frac"] < 1.2
