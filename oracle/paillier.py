"""CPU oracle for PC-MM over the Paillier scheme.

TEST INFRASTRUCTURE (same rules as `oracle/__init__.py`: only tests/, smoke()
and bench.py's reference legs may use it; the product path never does).

Plain Python big integers, written from the paper:
  * KeyGen / Encrypt / Decrypt: Sec. 2.5, with g = n + 1
    (R19: the paper samples g at random subject to
    gcd(n, L(g^lambda mod n^2)) = 1; n + 1 satisfies it and is the usual choice);
  * the homomorphism prod_i c_i^{s_i} = Enc(sum_i s_i m_i): Eq. 6, PAPER.md:207-213;
  * schoolbook PC-MM: C_ij = prod_k c_kj^{a_ik} mod n^2;
  * exponentiation by the Montgomery powering ladder: Alg. 4, PAPER.md:607-620;
  * Cussen PC-MM: Alg. 3 with point addition replaced by
    multiplication mod n^2 and ECSM by exponentiation: the
    per-column compression plan is the oracle's Alg. 2 (`oracle.cussen_plan`),
    reconstruction = level-N exponentiations, then prefix PRODUCTS, un-sort by
    tracking pointer, and the accumulation multiplies the m reconstructed
    ciphertexts of column k into row accumulators.
Plaintexts A are non-negative (R20: a negative scalar would need
c^{-1} mod n^2, which the paper does not discuss).
"""
from __future__ import annotations

from math import gcd

import numpy as np

from . import cussen_plan


def L_fn(x: int, n: int) -> int:
    """L(x) = (x - 1) / n."""
    return (x - 1) // n


def keygen(p: int, q: int):
    """-> (n, g, lam, mu) for primes p, q."""
    n = p * q
    n2 = n * n
    g = n + 1
    lam = (p - 1) * (q - 1) // gcd(p - 1, q - 1)
    mu = pow(L_fn(pow(g, lam, n2), n), -1, n)
    return n, g, lam, mu


def encrypt(n: int, g: int, m: int, r: int) -> int:
    """c = g^m r^n mod n^2."""
    n2 = n * n
    return pow(g, m % n, n2) * pow(r, n, n2) % n2


def decrypt(n: int, lam: int, mu: int, c: int) -> int:
    """m = L(c^lambda mod n^2) mu mod n."""
    return L_fn(pow(c, lam, n * n), n) * mu % n


def ladder_pow(g: int, k: int, t: int, mod: int) -> int:
    """Alg. 4: Montgomery powering ladder over t bits of k."""
    r = [1, g % mod]
    for i in range(t - 1, -1, -1):
        b = (k >> i) & 1
        r[1 - b] = r[1] * r[0] % mod
        r[b] = r[b] * r[b] % mod
    return r[0]


def pcmm_schoolbook(A: np.ndarray, C: list[list[int]], n2: int, t: int) -> list[list[int]]:
    """C_out[i][j] = prod_k C[k][j]^{a_ik} mod n^2, exponentiation by Alg. 4."""
    m, nn = A.shape
    l = len(C[0])
    out = [[1] * l for _ in range(m)]
    for i in range(m):
        for j in range(l):
            acc = 1
            for k in range(nn):
                a = int(A[i, k])
                if a:
                    acc = acc * ladder_pow(C[k][j], a, t, n2) % n2
            out[i][j] = acc
    return out


def _reconstruct(levels, N: int, t: int, c: int, n2: int, m: int) -> list[int]:
    """Alg. 3 lines 5-6 for one (k, j): out[i] = c^{a_ik} (1 for a_ik = 0)."""
    sN = [int(v) for v in levels[N - 1][0]]
    b = [ladder_pow(c, v, t, n2) for v in sN]                       # line 5
    for w in range(N, 0, -1):
        vals, ptr = levels[w - 1]
        if w != N:
            for i in range(len(b) - 1):                              # prefix products
                b[i + 1] = b[i + 1] * b[i] % n2
        prev = m if w == 1 else len(levels[w - 2][0])
        b = [1 if int(ptr[e]) < 0 else b[int(ptr[e])] for e in range(prev)]
    return b


def pcmm_cussen(A: np.ndarray, C: list[list[int]], n2: int, t: int, N: int = 4) -> list[list[int]]:
    """Alg. 3 in the multiplicative group mod n^2."""
    m, nn = A.shape
    l = len(C[0])
    out = [[1] * l for _ in range(m)]
    for k in range(nn):
        if (A[:, k] < 0).any():
            raise ValueError("Paillier PC-MM takes non-negative plaintexts (R20)")
        levels = cussen_plan(A[:, k].astype(np.int64), N)
        for j in range(l):
            col = _reconstruct(levels, N, t, C[k][j], n2, m)
            for i in range(m):
                out[i][j] = out[i][j] * col[i] % n2
    return out
