"""Host-side driver logic of EqSpecBatch / SequencePool that needs no GPU: buffer modes,
parity bookkeeping, option validation, launch counts (CPU tensors; no kernel is called)."""
import os

import pytest
import torch

from paper_2510_22876_b200.eqspec import EqSpecBatch
from paper_2510_22876_b200.exspec import SequencePool


def test_pingpong_buffers_follow_parity():
    bt = EqSpecBatch(3, 4, 64, 1, 2, 8, "bf16", "cpu", kv_mode="pingpong", draft=(1, 1, 8))
    assert len(bt._kvbuf) == 2 and len(bt._dkvbuf) == 2
    k0, d0 = bt.kv, bt.dkv
    bt.cur = 1
    assert bt.kv is not k0 and bt.kv is bt._kvbuf[1] and bt.dkv is bt._dkvbuf[1]
    bt.cur = 0
    assert bt.kv is k0 and bt.dkv is d0
    ip = EqSpecBatch(3, 4, 64, 1, 2, 8, "bf16", "cpu")
    k = ip.kv
    ip.cur = 1
    assert ip.kv is k                      # in place: one buffer whatever the parity


def test_option_validation():
    with pytest.raises(ValueError):
        EqSpecBatch(2, 4, 64, 1, 1, 8, "bf16", "cpu", kv_mode="bogus")
    with pytest.raises(ValueError):
        EqSpecBatch(2, 4, 64, 1, 1, 8, "bf16", "cpu", kv_mode="pingpong", anchor_slack=8)
    bt = EqSpecBatch(2, 4, 64, 1, 1, 8, "bf16", "cpu", kv_mode="pingpong")
    bt.zero_pads = True
    with pytest.raises(ValueError):        # ZERO_PADS is in place only; raised before any launch
        bt.realign()


def test_kernels_per_round():
    from paper_2510_22876_b200 import _abi
    k1 = _abi.specdec_verify_kernels(False)     # argmax grid + epilogue kernel (default): 2
    assert k1 == (1 if os.environ.get("SPECDEC_K1_SPLIT", "1").split(",")[0] in ("0", "2") else 2)
    assert EqSpecBatch(1, 4, 64, 1, 1, 8, "bf16", "cpu").kernels_per_round == k1 + 1     # B=1: no K2
    assert EqSpecBatch(1, 4, 64, 1, 1, 8, "bf16", "cpu", kv_mode="pingpong").kernels_per_round == k1 + 2
    assert EqSpecBatch(4, 4, 64, 1, 1, 8, "bf16", "cpu").kernels_per_round == k1 + 2
    assert EqSpecBatch(4, 4, 64, 1, 1, 8, "bf16", "cpu", draft=(1, 1, 8)).kernels_per_round == k1 + 3


def test_result_sets_per_parity():
    bt = EqSpecBatch(2, 4, 64, 1, 1, 8, "bf16", "cpu")
    bt._accept[0].fill_(1)
    bt._accept[1].fill_(2)
    bt._last = 0
    assert int(bt.accept[0]) == 1
    bt._last = 1
    assert int(bt.accept[0]) == 2 and bt.emit.data_ptr() == bt._emit[1].data_ptr()


def test_pool_dense_consumer_flag():
    sp = SequencePool(6, 16, 1, 1, 8, 3, W=4, B=2, device="cpu", dense_consumer=True)
    assert sp.dense_consumer
    calls = []
    sp.gather = lambda b, s=None: calls.append(("g", b))
    sp.scatter = lambda b, blen, s=None: calls.append(("s", b))
    sp.verify_writeback = lambda *a, **k: calls.append(("vw",))
    seen = []
    sp.run_batch(0, 1, 5, None, None, forward=lambda pool, b, zero_copy, blen: seen.append(zero_copy))
    assert calls == [("g", 0), ("vw",), ("s", 0)] and seen == [False]
    sp.consumer = "zero-copy"
    calls.clear()
    seen.clear()
    sp.run_batch(0, 1, 5, None, None, forward=lambda pool, b, zero_copy, blen: seen.append(zero_copy))
    assert calls == [("vw",)] and seen == [True]
    calls.clear()
    sp.run_batch(0, 0, 5, None, None)                  # a mixed-length batch is gathered
    assert calls == [("g", 0), ("vw",), ("s", 0)]
    sp.consumer = "slot"                               # slot-indexed consumer: never
    calls.clear()
    seen.clear()
    sp.run_batch(0, 0, 5, None, None, forward=lambda pool, b, zero_copy, blen: seen.append(zero_copy))
    assert calls == [("vw",)] and seen == [True]
    assert torch.equal(sp.order, torch.arange(6, dtype=torch.int32))
    with pytest.raises(ValueError):
        SequencePool(6, 16, 1, 1, 8, 3, W=4, B=2, device="cpu", consumer="paged")
