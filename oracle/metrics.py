"""Oracle: closed forms and equivalence scores.

Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations


def expected_tokens_per_iteration(alpha: float, k: int) -> float:
    """(1 - alpha^(k+1)) / (1 - alpha)  (§3.1, after Leviathan et al.)."""
    if not 0.0 <= alpha < 1.0:
        raise ValueError("alpha must be in [0, 1)")
    return (1.0 - alpha ** (k + 1)) / (1.0 - alpha)


def score_equivalence(candidate, reference):
    """Exact match and partial match (§4.1): exact = fraction
    of sequences fully equal; partial = mean of common-prefix length / reference length."""
    if len(candidate) != len(reference):
        raise ValueError("id mismatch")
    exact, partial = 0, 0.0
    for c, r in zip(candidate, reference):
        exact += int(list(c) == list(r))
        m = 0
        while m < min(len(c), len(r)) and c[m] == r[m]:
            m += 1
        partial += min(1.0, m / len(r)) if len(r) else 1.0
    return exact / len(reference), partial / len(reference)
