"""Helpers shared by the -m gpu parity tests: build inputs with synth/, run the oracle
on host copies of the SAME bytes, compare element by element."""
from __future__ import annotations

import numpy as np
import torch

from synth import workloads as W

TDT = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}


def bits_to_torch(bits: np.ndarray, dtype: str, device) -> torch.Tensor:
    if dtype == "fp32":
        return torch.from_numpy(np.ascontiguousarray(bits, np.float32)).to(device)
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).to(device).view(TDT[dtype])


def torch_to_bits(t: torch.Tensor) -> np.ndarray:
    t = t.detach().cpu()
    if t.dtype == torch.float32:
        return t.numpy()
    return t.view(torch.int16).numpy().view(np.uint16)


def padded_logits(bits: np.ndarray, dtype: str, device, extra: int = 0) -> torch.Tensor:
    """[B, k+1, V] bits -> device tensor with row stride V + extra (tail filled with +inf,
    which must never be read)."""
    B, K1, V = bits.shape
    t = bits_to_torch(bits, dtype, device)
    ve = 4 if dtype == "fp32" else 8
    if not extra and V % ve == 0:
        return t
    rs = (V + extra + ve - 1) // ve * ve       # 16-byte aligned rows (specdec.h)
    out = torch.full((B, K1, rs), float("inf"), dtype=TDT[dtype], device=device)
    out[:, :, :V] = t
    return out


def initial_state(shape: W.Shape, seed: int, B: int, cap: int):
    lengths = W.gen_lengths(shape, seed, B)
    tokens = W.left_padded_tokens(lengths, cap, seed, shape.V)
    return lengths, tokens
