"""Alg. A1 ("Selection of Independent Channel Pairs") oracle -- TEST INFRASTRUCTURE ONLY.

Same rules as oracle/paro_oracle.py: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module; it shares no code with
paper_2511_10645_b200/ (the C++ paro_select_pairs in csrc/pairs.cpp is written
independently and compared with this one bit for bit).

Plain Python, step by step in the paper's order and notation:

  * PAPER.md:509-553 (Alg. A1): P = {(i, j) | 1 <= i < j <= g}; P_shuffled = Shuffle(P);
    A = ones(g, g) - I; for r = 1..K: A_rot = Copy(A); for each (i, j) in P_shuffled:
    if |P_r| = N: break; if A_rot[i, j] = 0: continue; append (i, j) to P_r; zero rows and
    columns i and j of A_rot; A[i, j] = A[j, i] = 0.
  * PAPER.md:170 ("skip pairs that have already been selected") -- later rotations may
    fall short of N; absent slots are (-1, -1).
  * The random Shuffle (reading Q20): SplitMix64 seeding a
    xoshiro256** generator, both by their public reference definitions; the Fisher-Yates
    shuffle from the last element down with an unbiased bounded draw; P enumerated in
    lexicographic order before the shuffle; group gamma's generator state is outputs
    4 gamma .. 4 gamma + 3 of the SplitMix64 stream seeded with `seed` (counter-based, so
    groups are independent).

Pins (tests/test_alg_a1.py): SplitMix64's published first output for seed 0, xoshiro256**'s
published output sequence for the state {1, 2, 3, 4}, hand-derived Alg. A1 runs on a fixed
order (including a short rotation), exhaustive properties (Def. 1 per rotation, no pair
repeated across rotations, greedy maximality), the uniformity of the shuffle on tiny n.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def splitmix64(seed: int, n: int) -> list[int]:
    """First n outputs of SplitMix64 seeded with `seed` (Steele, Lea, Flood 2014; the
    reference C routine: x += 0x9e3779b97f4a7c15, then two xor-shift-multiplies)."""
    out = []
    x = seed & MASK64
    for _ in range(n):
        x = (x + GOLDEN) & MASK64
        z = x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        out.append(z ^ (z >> 31))
    return out


def _rotl(v: int, k: int) -> int:
    return ((v << k) | (v >> (64 - k))) & MASK64


class Xoshiro256ss:
    """xoshiro256** 1.0 (Blackman & Vigna), the reference next()."""

    def __init__(self, state):
        self.s = [int(v) & MASK64 for v in state]

    def next(self) -> int:
        s = self.s
        result = (_rotl((s[1] * 5) & MASK64, 7) * 9) & MASK64
        t = (s[1] << 17) & MASK64
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = _rotl(s[3], 45)
        return result

    def bounded(self, m: int) -> int:
        """Uniform integer in [0, m): draws below 2^64 mod m are rejected, then r mod m."""
        lim = (1 << 64) % m
        while True:
            r = self.next()
            if r >= lim:
                return r % m


def group_rng(seed: int, gamma: int) -> Xoshiro256ss:
    """Generator of group gamma: state = SplitMix64(seed) outputs 4 gamma .. 4 gamma + 3."""
    return Xoshiro256ss(splitmix64(seed, 4 * gamma + 4)[4 * gamma:])


def shuffle(seq: list, rng: Xoshiro256ss) -> list:
    """Fisher-Yates: for i = n-1 down to 1, swap element i with element bounded(i + 1)."""
    a = list(seq)
    for i in range(len(a) - 1, 0, -1):
        j = rng.bounded(i + 1)
        a[i], a[j] = a[j], a[i]
    return a


def all_pairs(g: int) -> list[tuple[int, int]]:
    """P = {(i, j) | 1 <= i < j <= g} (0-based here), lexicographic order."""
    return [(i, j) for i in range(g) for j in range(i + 1, g)]


def select_pairs_from_order(order, g: int, K: int, N: int):
    """Alg. A1's loop on a given shuffled pair list; returns K lists."""
    A = np.ones((g, g), dtype=np.int8) - np.eye(g, dtype=np.int8)
    P = [[] for _ in range(K)]
    for r in range(K):
        A_rot = A.copy()                      # tracks available channels within this rotation
        for (i, j) in order:
            if len(P[r]) == N:
                break
            if A_rot[i, j] == 0:
                continue
            P[r].append((i, j))               # select the next available pair
            A_rot[i, :] = 0
            A_rot[:, i] = 0
            A_rot[j, :] = 0
            A_rot[:, j] = 0                   # block channels
            A[i, j] = 0
            A[j, i] = 0                       # block pair
    return P


def select_pairs(n_groups: int, g: int, K: int, N: int, seed: int) -> np.ndarray:
    """Alg. A1 for every group of a linear (Alg. A2 calls it once per group):
    int16 [n_groups, K, N, 2], 0-based, i < j, (-1, -1) in the slots of a short rotation."""
    if g < 2 or K < 1 or not (1 <= N <= g // 2) or n_groups < 0:
        raise ValueError("select_pairs: need g >= 2, K >= 1, 1 <= N <= g/2")
    out = np.full((n_groups, K, N, 2), -1, dtype=np.int16)
    for gamma in range(n_groups):
        order = shuffle(all_pairs(g), group_rng(seed, gamma))
        for r, lst in enumerate(select_pairs_from_order(order, g, K, N)):
            for p, (i, j) in enumerate(lst):
                out[gamma, r, p] = (i, j)
    return out
