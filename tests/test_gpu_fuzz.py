"""Seeded random-configuration parity: many small EqSpec episodes whose shape (B, k, ragged V,
layers, KV heads, head_dim, logit / KV dtypes, length spread), acceptance pattern, EOS,
budget, ZERO_PADS and anchored-origin options are all drawn from one RNG, each compared
round by round with the oracle (tests/test_gpu_round._run_rounds: accept / bonus / emit /
finished / kept, L', pads, lengths, tokens, masks, positions, every defined KV entry,
moved bytes, output buffers).  SPECDEC_FUZZ_CASES=n widens the sweep (2000 ran green)."""
import numpy as np
import pytest

from synth import workloads as W
from tests.test_gpu_round import _run_rounds

pytestmark = pytest.mark.gpu

N_CASES = int(__import__("os").environ.get("SPECDEC_FUZZ_CASES", "24"))


def draw_case(i: int):
    rng = np.random.default_rng(10_000 + i)
    k = int(rng.integers(1, 9))
    V = int(rng.integers(k + 2, 20_000))           # ragged: any residue mod 8
    B = int(rng.integers(1, 13))
    layers = int(rng.integers(1, 3))
    H = int(rng.integers(1, 4))
    D = int(rng.choice([8, 16, 64, 72, 128]))       # D * 2 bytes % 16 == 0
    kv_dtype = str(rng.choice(["bf16", "fp16"]))
    logit_dtype = str(rng.choice(["bf16", "fp16", "fp32"]))
    lo = int(rng.integers(1, 120))
    hi = lo + int(rng.integers(0, 200))
    shape = W.Shape(f"fuzz{i}", V, layers, H, D, kv_dtype, logit_dtype, B, k, hi, lo, hi)
    pattern = str(rng.choice(W.ACCEPT_PATTERNS))
    rounds = int(rng.integers(1, 9))
    max_new = int(rng.choice([0, 0, int(rng.integers(1, 4 * (k + 1)))]))
    eos_id = -1
    if rng.random() < 0.4:  # a token round 0 drafts for row 0: a hit whenever it is accepted
        eos_id = int(W.gen_round_truth(i, 0, B, k, V, pattern).draft[0, 0])
    anchor = int(rng.choice([0, 0, k + 2, 64]))
    zero_pads = bool(anchor == 0 and rng.random() < 0.3)
    return dict(shape=shape, B=B, rounds=rounds, pattern=pattern, seed=i, max_new=max_new,
                eos_id=eos_id, zero_pads=zero_pads, anchor_slack=anchor)


@pytest.mark.parametrize("i", range(N_CASES))
def test_fuzz_episode(cuda, i):
    c = draw_case(i)
    _run_rounds(cuda, c["shape"], c["B"], c["rounds"], c["pattern"], seed=c["seed"],
                max_new=c["max_new"], eos_id=c["eos_id"], zero_pads=c["zero_pads"],
                anchor_slack=c["anchor_slack"])


# 3029: separate pinned logits / drafts that the caching host allocator placed back to back
# -- a single copy spanning both allocations failed (inputs_packed is now explicit)
@pytest.mark.parametrize("i", sorted(set(range(N_CASES)) | {3029}))
def test_fuzz_episode_native_drivers(cuda, i):
    """The same episodes through the native round driver, the host-buffer driver (separate
    or packed inputs) and graph replay of the captured round, in turn, with the KV mode
    drawn too (ping-pong when not anchored)."""
    c = draw_case(i)
    rng = np.random.default_rng(20_000 + i)
    kv_mode = "pingpong" if (c["anchor_slack"] == 0 and not c["zero_pads"] and rng.random() < 0.4) else "inplace"
    _run_rounds(cuda, c["shape"], c["B"], c["rounds"], c["pattern"], seed=c["seed"],
                max_new=c["max_new"], eos_id=c["eos_id"], zero_pads=c["zero_pads"],
                anchor_slack=c["anchor_slack"], kv_mode=kv_mode,
                drive=("native", "host", "graph", "host_packed")[i % 4])
