"""The thread-parallel oracle driver (CPU baseline timing) computes exactly
what the serial oracle composition computes: every verify output, the plan, tokens',
masks, positions and every KV byte, on random rounds with EOS, budgets and inactive rows."""
import numpy as np

from oracle import align as OA
from oracle import driver as OD
from oracle import verify as OV
from synth import workloads as W


def test_parallel_round_equals_serial():
    rng = np.random.default_rng(3)
    with OD.make_pool(4) as pool:
        for t in range(40):
            B, k, V = int(rng.integers(1, 9)), int(rng.integers(1, 6)), 53
            n = rng.integers(1, 30, B).astype(np.int32)
            L = int(n.max())
            pad = (L - n).astype(np.int32)
            cap = L + 3 * (k + 1)
            tokens = np.zeros((B, cap), np.int64)
            for i in range(B):
                tokens[i, pad[i]:L] = rng.integers(2, V, n[i])
            bits = W.gen_logits_np(t, 0, B, k, V, "bf16")
            draft = W.gen_round_truth(t, 0, B, k, V, "alpha").draft
            act = (rng.random(B) < 0.8).astype(np.uint8)
            eos = int(rng.integers(2, V)) if rng.random() < 0.3 else -1
            budget = rng.integers(0, 8, B) if rng.random() < 0.4 else None
            kv = rng.integers(0, 1 << 15, size=(3, B, 2, cap, 4)).astype(np.uint16)
            v = OV.batch_verify(bits, "bf16", draft, n, pad, act, eos, budget)
            tok_s, mask_s, pos_s = OA.repad_tokens(tokens, cap, k, pad, L, v)
            kv_s = OA.realign_kv_inplace(kv.copy(), pad, v["pad_new"], v["kept"])
            kv_p = kv.copy()
            vp, tok_p, mask_p, pos_p = OD.eqspec_round_parallel(pool, bits, "bf16", draft, tokens, cap, k, n, pad,
                                                                 L, act, kv_p, eos, budget)
            for key in ("pred", "accept", "bonus", "emit", "finished", "n_new", "pad_new", "kept", "kept_draft"):
                assert np.array_equal(v[key], vp[key]), key
            assert v["E"] == vp["E"] and v["L_new"] == vp["L_new"] and v["nan"] == vp["nan"]
            assert np.array_equal(tok_s, tok_p) and np.array_equal(mask_s, mask_p) and np.array_equal(pos_s, pos_p)
            assert np.array_equal(kv_s, kv_p)
