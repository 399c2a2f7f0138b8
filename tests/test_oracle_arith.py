"""Pins of the oracle's field, scalar and group arithmetic.

Every expected value comes from something other than the oracle: Python's
arbitrary-precision integers (a textbook special case of modular arithmetic),
the published curve constants, and k*G from OpenSSL via `cryptography`.
"""
import random

import numpy as np
import pytest

import oracle
from tests import ecref

rng = random.Random(20250419)
EDGE = [0, 1, 2, 3, 2**32 - 1, 2**64, 2**128 + 5, 2**255, ecref.P - 1, ecref.P - 2, ecref.Q - 1, 2**256 - 1]


def test_curve_constants_p1():
    # p = 2^256 - 2^224 + 2^192 + 2^96 - 1 and y^2 = x^3 - 3x + b
    assert ecref.P == int("ffffffff00000001000000000000000000000000ffffffffffffffffffffffff", 16)
    assert (ecref.GY ** 2 - (ecref.GX ** 3 - 3 * ecref.GX + ecref.B)) % ecref.P == 0
    G = oracle.generator()
    assert G == ecref.GX.to_bytes(32, "big") + ecref.GY.to_bytes(32, "big")
    assert oracle.on_curve(G)
    # q G = infinity and (q-1) G = -G
    assert oracle.scalar_mul_base(ecref.Q) == ecref.INF
    assert oracle.scalar_mul_base(ecref.Q - 1) == ecref.mulG(ecref.Q - 1)


@pytest.mark.parametrize("which,mod", [(oracle.FIELD_P, ecref.P), (oracle.ORDER_Q, ecref.Q)])
def test_modular_ops_vs_python_ints_p2(which, mod):
    vals = [v % (2**256) for v in EDGE] + [rng.randrange(2**256) for _ in range(60)]
    for a in vals:
        b = rng.choice(vals)
        ar, br = a % mod, b % mod
        assert oracle.modop(which, "add", a, b) == (ar + br) % mod
        assert oracle.modop(which, "sub", a, b) == (ar - br) % mod
        assert oracle.modop(which, "mul", a, b) == (ar * br) % mod
        e = rng.randrange(2**256)
        assert oracle.modop(which, "pow", a, e) == pow(ar, e, mod)
        if ar:
            assert oracle.modop(which, "inv", a) == pow(ar, -1, mod)


def test_scalar_mul_base_vs_openssl_p3():
    for k in [1, 2, 3, 7, 255, 2**64 + 13] + [rng.randrange(1, ecref.Q) for _ in range(12)]:
        assert oracle.scalar_mul_base(k) == ecref.mulG(k)


def test_group_law_vs_openssl():
    for _ in range(12):
        a, b = rng.randrange(1, ecref.Q), rng.randrange(1, ecref.Q)
        Pa, Pb = ecref.mulG(a), ecref.mulG(b)
        assert oracle.point_add(Pa, Pb) == ecref.mulG(a + b)
        assert oracle.point_dbl(Pa) == ecref.mulG(2 * a)
        assert oracle.point_neg(Pa) == ecref.mulG(-a)
        k = rng.randrange(2**256)
        assert oracle.scalar_mul(k, Pa) == ecref.mulG(k * a)


def test_exceptional_cases():
    a = rng.randrange(1, ecref.Q)
    Pa = ecref.mulG(a)
    assert oracle.point_add(Pa, ecref.INF) == Pa                      # P + inf = P
    assert oracle.point_add(ecref.INF, Pa) == Pa
    assert oracle.point_add(ecref.INF, ecref.INF) == ecref.INF
    assert oracle.point_add(Pa, ecref.mulG(-a)) == ecref.INF          # P + (-P) = inf
    assert oracle.point_add(Pa, Pa) == oracle.point_dbl(Pa) == ecref.mulG(2 * a)
    assert oracle.point_dbl(ecref.INF) == ecref.INF
    assert not oracle.on_curve(bytes(63) + b"\x01")
    bad = bytearray(Pa); bad[63] ^= 1
    assert not oracle.on_curve(bytes(bad))


def test_group_invariants():
    pts = [ecref.mulG(rng.randrange(1, ecref.Q)) for _ in range(3)]
    P, Q, R = pts
    assert oracle.point_add(P, Q) == oracle.point_add(Q, P)
    assert oracle.point_add(oracle.point_add(P, Q), R) == oracle.point_add(P, oracle.point_add(Q, R))


def test_ladder_alg1_counts_and_values_p10():
    # Alg. 1: exactly t additions and t doublings; equals k-fold addition
    a = rng.randrange(1, ecref.Q)
    Pa = ecref.mulG(a)
    acc = ecref.INF
    for k in range(0, 65):
        t = max(1, k.bit_length())
        for tt in (t, 8):
            pt, (adds, dbls, ecsm, bits) = oracle.ladder_mul(k, tt, Pa)
            assert pt == acc == ecref.mulG(k * a)
            assert (adds, dbls, ecsm, bits) == (tt, tt, 1, tt)
        acc = oracle.point_add(acc, Pa)
