"""Seeded inputs for edge-cost generation, shared by the
CUDA path's tests and the oracle.  Holds none of the method's arithmetic:
it only draws bandwidth profiles (the measurements of P:668-671), tensor
shapes and query index triples.

Profile recipe: for a group of 2^c devices the bandwidth at
2^i bytes follows a saturating curve bw = peak_c * 2^i / (2^i + half_c)
(latency-dominated small messages, "latency could dominate the
communication time when transferring small tensors"), peak_c falling with
group size (contention), times a seeded +-5 % jitter; integer bytes/s.
"""
from __future__ import annotations

from typing import Dict, List, Tuple

import numpy as np

MAXL, MAXP, MAXD = 6, 46, 4


def profile(seed: int = 0, L: int = 5, P: int = 40, peak: float = 4.5e11,
            half: float = 2.0 ** 20, jitter: float = 0.05, monotone: bool = False) -> Dict:
    """Bandwidth profile dict {L, P, lat[MAXL+1], bw[MAXL+1][MAXP+1]} (int64)."""
    rng = np.random.default_rng(seed)
    lat = np.zeros(MAXL + 1, np.int64)
    bw = np.ones((MAXL + 1, MAXP + 1), np.int64)
    for c in range(1, L + 1):
        lat[c] = int(2000 + 1500 * c + rng.integers(0, 500))
        pk = peak / (1.0 + 0.15 * (c - 1))
        h = half * (1.0 + 0.5 * (c - 1))
        for i in range(P + 1):
            s = float(2 ** i)
            v = pk * s / (s + h)
            if not monotone:
                v *= 1.0 + jitter * (2.0 * rng.random() - 1.0)
            bw[c, i] = max(1, int(v))
    return {"L": L, "P": P, "lat": lat, "bw": bw}


def tensors(seed: int, n: int, L: int, max_ndims: int = 4) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """n tensors: ndims[n] int32, dims[n, MAXD] int64 (unused dims = 1), elem_bytes[n] int64.
    Dims are products of a power of two (0..L+1) and a small odd factor, so
    some dims cannot be split 2^L ways (exercises the divisibility rule)."""
    rng = np.random.default_rng(seed)
    nd = rng.integers(1, max_ndims + 1, n).astype(np.int32)
    dims = np.ones((n, MAXD), np.int64)
    for x in range(n):
        for j in range(nd[x]):
            dims[x, j] = int(2 ** rng.integers(0, L + 2)) * int(rng.choice([1, 3, 5, 7, 48, 96]))
    eb = rng.choice([2, 4], n).astype(np.int64)
    return nd, dims, eb


def queries(seed: int, n_states: List[int], n_q: int) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """n_q (tensor, from, to) index triples with from/to < n_states[tensor]."""
    rng = np.random.default_rng(seed)
    qt = rng.integers(0, len(n_states), n_q).astype(np.int32)
    ns = np.asarray(n_states, np.int64)[qt]
    qf = (rng.random(n_q) * ns).astype(np.int32)
    qo = (rng.random(n_q) * ns).astype(np.int32)
    return qt, qf, qo
