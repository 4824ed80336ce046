"""The CUDA path (libspecdec.so through the C ABI) against the hand-worked fixtures in
tests/golden/: the EqSpec round of eqspec_round.json (K1 -> K3 -> K2) in every logit
dtype, and the pool plans of pool_plans.json (K4)."""
import json
import os

import numpy as np
import pytest
import torch

from paper_2510_22876_b200.eqspec import EqSpecBatch
from tests.gpu_helpers import bits_to_torch
from tests.test_golden import _round_inputs
from tests.test_gpu_pool import _check_plan, _plan_gpu
from tests.test_gpu_verify import run_verify

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


@pytest.mark.parametrize("dtype", ["fp32", "fp16", "bf16"])
def test_gpu_golden_verify(cuda, dtype):
    g = load("eqspec_round.json")
    B = len(g["n"])
    for c in g["cases"]:
        r = run_verify(cuda, _round_inputs(g, dtype), dtype, g["draft"], g["n"], np.ones(B, np.uint8),
                       eos_id=c["eos_id"], budget=c["budget"], pad_id=g["pad_id"])
        for key in ("pred", "accept", "bonus", "emit", "finished", "n_new", "pad_new", "kept", "kept_draft"):
            assert r[key].tolist() == c[key], (dtype, c["name"], key)
        assert int(r["plan_L"][0]) == c["L_new"] and r["ws_clean"]


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("case", [0, 1])
def test_gpu_golden_round(cuda, dtype, case):
    """One whole round through EqSpecBatch: tokens', mask, pos and every defined KV entry."""
    g = load("eqspec_round.json")
    c = g["cases"][case]
    k, cap, L, B = g["k"], g["cap"], g["L"], len(g["n"])
    H, D = 1, 8                                    # 16-byte bf16 rows (specdec.h)
    bt = EqSpecBatch(B, k, cap, 1, H, D, "bf16", cuda, max_new=32, eos_id=c["eos_id"], pad_id=g["pad_id"])
    tokens = np.full((B, cap), g["pad_id"], np.int64)
    tokens[:, :L] = g["tokens_before"]
    # KV entry (plane p, row i, column c) = 1000 p + 100 i + c in every head_dim lane
    val = (1000 * np.arange(2)[:, None, None] + 100 * np.arange(B)[None, :, None]
           + np.arange(cap)[None, None, :]).astype(np.uint16)
    kv = np.broadcast_to(val[:, :, None, :, None], (2, B, H, cap, D)).copy()
    bt.load(tokens, np.array(g["n"]), bits_to_torch(kv, "bf16", cuda))
    if c["budget"] is not None:
        bt.budget.copy_(torch.tensor(c["budget"], dtype=torch.int32))
    bt.step(bits_to_torch(_round_inputs(g, dtype), dtype, cuda),
            torch.tensor(g["draft"], dtype=torch.int64, device=cuda))
    torch.cuda.synchronize()
    Ln = c["L_new"]
    assert bt.accept.tolist() == c["accept"] and bt.bonus.tolist() == c["bonus"]
    assert int(bt.plan_L.item()) == Ln
    assert bt.tokens[:, :Ln].tolist() == c["tokens_after"]
    assert bt.mask[:, :Ln + k].tolist() == c["mask"] and bt.pos[:, :Ln + k].tolist() == c["pos"]
    got = bt.kv.cpu().view(torch.int16).numpy().view(np.uint16)
    for i_s, row in c["kv_after"].items():
        for col_s, v in row.items():
            i, col = int(i_s), int(col_s)
            for p in range(2):
                assert (got[p, i, :, col, :] == 1000 * p + v).all(), (i, col, p)
    assert int(bt.status.item()) == 0


def test_gpu_golden_pool_plans(cuda):
    for c in load("pool_plans.json")["cases"]:
        gp = _plan_gpu(cuda, c["lens"], c["active"], c["order"], c["W"], c["B"], c["min_group"])
        _check_plan(gp, c, np.array(c["lens"]), c["B"])
