"""Pins of the oracle's EC-ElGamal and homomorphic identities
(Eq. 1, Eq. 3, Eq. 5) against OpenSSL k*G."""
import random

import numpy as np

import oracle
import synth
from tests import ecref

rng = random.Random(7)


def _r(n):
    return [rng.randrange(1, ecref.Q) for _ in range(n)]


def test_keygen_and_encrypt_vs_openssl():
    x = synth.keygen_secret(0)
    assert 1 <= x < ecref.Q
    H = oracle.pubkey(x)
    assert H == ecref.mulG(x)                                       # H = x G
    b = np.array([0, 1, 3, 255, -8, 72], dtype=np.int64)
    r = _r(b.size)
    ct = oracle.encrypt(H, b, synth.scalars_to_be_bytes(r))
    for e in range(b.size):
        # (r G, r H + b G) = (r G, (r x + b) G)
        assert ct[e].tobytes() == ecref.enc_closed_form(x, r[e], int(b[e]))


def test_decrypt_roundtrip_and_bound():
    x = rng.randrange(1, ecref.Q)
    H = oracle.pubkey(x)
    b = np.arange(-5, 20, dtype=np.int64)
    ct = oracle.encrypt(H, b, synth.scalars_to_be_bytes(_r(b.size)))
    m, st = oracle.decrypt(x, ct, -5, 19)
    assert (st == 0).all() and (m == b).all()
    m, st = oracle.decrypt(x, ct, 0, 10)                             # out of range -> decode failure
    assert ((st == oracle.PCMM_EDECODE) == ((b < 0) | (b > 10))).all()
    assert (m[st == 0] == b[st == 0]).all()


def test_homomorphic_identities_p4():
    x = rng.randrange(1, ecref.Q)
    H = oracle.pubkey(x)
    for _ in range(5):
        a, b = rng.randrange(0, 1000), rng.randrange(0, 1000)
        r1, r2 = _r(2)
        ca = oracle.encrypt(H, np.array([a]), synth.scalars_to_be_bytes([r1]))[0].tobytes()
        cb = oracle.encrypt(H, np.array([b]), synth.scalars_to_be_bytes([r2]))[0].tobytes()
        # Eq. 1: Enc(a; r1) (+) Enc(b; r2) = Enc(a + b; r1 + r2), component-wise point adds
        s = oracle.point_add(ca[:64], cb[:64]) + oracle.point_add(ca[64:], cb[64:])
        assert s == ecref.enc_closed_form(x, r1 + r2, a + b)
        # Eq. 3: k (x) Enc(a; r) = Enc(k a; k r)
        k = rng.randrange(0, 64)
        km = oracle.scalar_mul(k, ca[:64]) + oracle.scalar_mul(k, ca[64:])
        assert km == ecref.enc_closed_form(x, k * r1, k * a)


def test_closed_form_eq5_vs_openssl():
    x = rng.randrange(1, ecref.Q)
    n = 6
    a = np.array([rng.randrange(-8, 8) for _ in range(n)], dtype=np.int8)
    b = np.array([rng.randrange(0, 256) for _ in range(n)], dtype=np.int64)
    r = _r(n)
    R = sum(int(a[k]) * r[k] for k in range(n))
    c = sum(int(a[k]) * int(b[k]) for k in range(n))
    assert oracle.closed_form(x, a, b, synth.scalars_to_be_bytes(r)) == ecref.enc_closed_form(x, R, c)
