"""Pins of the Paillier oracle (NEXT-4, oracle/paillier.py) against the paper's
definitions and plain integer arithmetic (SURVEY.md §8(c) style):
decryption inverts encryption, Eq. 6's homomorphism
(PAPER.md:207-213), Alg. 4 == Python's pow, and PC-MM: Cussen == schoolbook ==
the closed form g^(c_ij) (prod_k r_kj^a_ik)^n, decrypting to A.B."""
import numpy as np
import pytest

import synth
from oracle import paillier as pl


@pytest.fixture(scope="module")
def key():
    p, q = synth.paillier_primes(5, 256)
    n, g, lam, mu = pl.keygen(p, q)
    assert n.bit_length() == 256 and p != q
    return n, g, lam, mu


def test_primes_are_prime():
    p, q = synth.paillier_primes(6, 128)
    for v in (p, q):
        assert all(pow(a, v - 1, v) == 1 for a in (2, 3, 5, 7, 11))
        assert all(v % d for d in range(3, 2000, 2))


def test_roundtrip_and_eq6(key):
    n, g, lam, mu = key
    rs = synth.paillier_random_units(1, n, 40)
    ms = [0, 1, n - 1, 12345] + [int(v) for v in synth.SplitMix64(2).small(0, 2**40, 36)]
    cs = [pl.encrypt(n, g, m, r) for m, r in zip(ms, rs)]
    assert [pl.decrypt(n, lam, mu, c) for c in cs] == [m % n for m in ms]
    s = [int(v) for v in synth.SplitMix64(3).small(0, 255, 40)]
    prod = 1
    for c, si in zip(cs, s):
        prod = prod * pow(c, si, n * n) % (n * n)
    assert pl.decrypt(n, lam, mu, prod) == sum(si * mi for si, mi in zip(s, ms)) % n


def test_ladder_alg4_equals_pow():
    g = synth.SplitMix64(4)
    mod = (2**255 - 19) * (2**127 - 1)
    for t in (1, 4, 8, 12, 16):
        for k in [0, 1, (1 << t) - 1] + [int(v) for v in g.small(0, (1 << t) - 1, 20)]:
            b = int(g.small(2, 2**62, 1)[0]) ** 3
            assert pl.ladder_pow(b, k, t, mod) == pow(b, k, mod)


@pytest.mark.parametrize("shape,t", [((5, 7, 3), 4), ((6, 5, 4), 8), ((9, 4, 2), 2)])
def test_pcmm_cussen_schoolbook_closed_form(key, shape, t):
    n, g, lam, mu = key
    n2 = n * n
    m, nn, l = shape
    gen = synth.SplitMix64(100 + t)
    A = gen.small(0, (1 << t) - 1, m * nn).reshape(m, nn)
    A[0, :] = 0
    A[1, 0] = (1 << t) - 1
    B = gen.small(0, 255, nn * l).reshape(nn, l)
    R = synth.paillier_random_units(7 + t, n, nn * l)
    C = [[pl.encrypt(n, g, int(B[k, j]), R[k * l + j]) for j in range(l)] for k in range(nn)]
    cs = pl.pcmm_cussen(A, C, n2, t)
    sb = pl.pcmm_schoolbook(A, C, n2, t)
    assert cs == sb
    AB = A.astype(object) @ B.astype(object)
    for i in range(m):
        for j in range(l):
            rp = 1
            for k in range(nn):
                rp = rp * pow(R[k * l + j], int(A[i, k]), n2) % n2
            assert cs[i][j] == pow(g, int(AB[i, j]), n2) * pow(rp, n, n2) % n2     # Eq. 6
            assert pl.decrypt(n, lam, mu, cs[i][j]) == int(AB[i, j])


def test_rejects_negative_plaintexts(key):
    n, g, _, _ = key
    with pytest.raises(ValueError):
        pl.pcmm_cussen(np.array([[-1]]), [[pl.encrypt(n, g, 1, 3)]], n * n, 4)
