"""Walsh-Hadamard transform oracle -- TEST INFRASTRUCTURE ONLY (same rules as
oracle/paro_oracle.py: imported only by tests/, smoke() and bench.py's oracle legs; no code
shared with paper_2511_10645_b200/).

The comparison transform of the paper's kernel experiment (fig:kernel-speedup,
PAPER.md:200-209: "the fast Hadamard transform", Hadamard-based rotation
methods), with SPEC.md:336-344's conventions: the unnormalised transform, and the randomised
variant that applies +-1 signs first and scales after.  Written as the definition: the
Sylvester matrix H_1 = [1], H_2m = [[H_m, H_m], [H_m, -H_m]] times the vector, in fp64.

Pins (tests/test_hadamard.py): scipy.linalg.hadamard, SPEC.md:341's [1,0,0,0] -> [1,1,1,1],
H H^T = n I (and the involution fwht(fwht(v)) = n v), the closed form
H[i, j] = (-1)^popcount(i & j).
"""
from __future__ import annotations

import numpy as np


def hadamard_matrix(n: int) -> np.ndarray:
    """Sylvester's construction, n a power of two."""
    if n < 1 or n & (n - 1):
        raise ValueError("n must be a power of two")
    H = np.ones((1, 1))
    while H.shape[0] < n:
        H = np.block([[H, H], [H, -H]])
    return H


def fwht(x: np.ndarray, signs: np.ndarray | None = None, scale: float = 1.0) -> np.ndarray:
    """y = scale * H_n diag(signs) x for every row x of x [T, n] (fp64)."""
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[-1]
    if signs is not None:
        x = x * np.asarray(signs, dtype=np.float64)
    return scale * (x @ hadamard_matrix(n).T)
