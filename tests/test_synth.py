"""The shared input generator: numpy and torch forms produce identical bits."""
import numpy as np
import torch

from synth.hashgen import hash_np, hash_torch, splitmix64_int, to_u64_np
from synth import workloads as W


def test_splitmix64_known_vector():
    # SplitMix64 seeded with state 0: first output (Steele et al. 2014 reference impl.)
    assert splitmix64_int(0) == 0xE220A8397B1DCDAF


def test_hash_numpy_equals_torch_cpu():
    idx = np.arange(0, 100_000, 7, dtype=np.uint64)
    a = hash_np(3, 5, idx)
    b = to_u64_np(hash_torch(3, 5, torch.from_numpy(idx.astype(np.int64))))
    assert np.array_equal(a, b)


def test_logits_numpy_equals_torch_cpu():
    for dt in ("bf16", "fp16", "fp32"):
        a = W.gen_logits_np(1, 2, 3, 4, 257, dt)
        t = W.gen_logits_torch(1, 2, 3, 4, 257, dt, "cpu")
        if dt == "fp32":
            b = t.numpy()
        else:
            b = t.view(torch.int16).numpy().view(np.uint16)
        assert np.array_equal(a, b), dt


def test_kv_numpy_equals_torch_cpu():
    shape = (2, 3, 2, 37, 8)
    a = W.gen_kv_bits_np(4, int(np.prod(shape)))
    b = W.gen_kv_torch(4, shape, torch.bfloat16, "cpu").view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(a, b.reshape(-1))
    # finite: exponent never all-ones
    assert not np.any((a & 0x7F80) == 0x7F80)
    # offset windows agree with the full stream
    assert np.array_equal(W.gen_kv_bits_np(4, 50, offset=13), a[13:63])


def test_planted_truth_consistency():
    rt = W.gen_round_truth(0, 3, 8, 5, 1000, "alpha")
    assert rt.draft.shape == (8, 5)
    for i in range(8):
        a = rt.accept[i]
        assert np.array_equal(rt.draft[i, :a], rt.pred[i, :a])
        if a < 5:
            assert rt.draft[i, a] != rt.pred[i, a]
