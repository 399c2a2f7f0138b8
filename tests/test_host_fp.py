"""CPU unit tests of the CUDA path's portable field / curve ALGORITHMS (fp.cuh,
ec.cuh compiled for the host by nvcc): Montgomery reduction specialised to
P-256, the inversion addition chain, the RCB complete formulas and the
canonical encodings, against Python ints and OpenSSL k*G."""
import ctypes
import os
import random
import shutil
import subprocess

import pytest

from tests import ecref

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "host_fp", "host_fp.cu")
LIB = os.path.join(HERE, "host_fp", "libhost_fp.so")
CSRC = os.path.join(os.path.dirname(HERE), "paper_2504_14497_b200", "csrc")

pytestmark = pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not available")


def _lib():
    deps = [SRC] + [os.path.join(CSRC, f) for f in ("fp.cuh", "ec.cuh")]
    if not os.path.exists(LIB) or any(os.path.getmtime(d) > os.path.getmtime(LIB) for d in deps):
        subprocess.check_call(["nvcc", "-O2", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC", "-shared", "-o", LIB, SRC])
    return ctypes.CDLL(LIB)


L = None


def lib():
    global L
    if L is None:
        L = _lib()
    return L


rng = random.Random(3)


def b32(v):
    return (v % 2**256).to_bytes(32, "big")


def call(fn, *args, n=32):
    out = ctypes.create_string_buffer(n)
    rc = fn(*args, out)
    assert rc == 0
    return out.raw


def test_field_ops_vs_python_ints():
    P = ecref.P
    vals = [0, 1, 2, 3, P - 1, P - 2, P - 3, 2**224, 2**192 - 1, 2**96, 2**255 % P, 2**30, 2**30 - 1, 2**60 + 1,
            (P + 1) // 2, P // 3] + [rng.randrange(P) for _ in range(600)] + [rng.randrange(2**40) for _ in range(50)]
    for a in vals:
        b = rng.choice(vals)
        get = lambda op: int.from_bytes(call(lib().hfp_op, op, b32(a), b32(b)), "big")
        assert get(0) == (a + b) % P
        assert get(1) == (a - b) % P
        assert get(2) == (a * b) % P
        assert get(4) == (-a) % P
        if a:
            assert get(3) == pow(a, -1, P)                 # divsteps (Bernstein-Yang)
            assert get(5) == pow(a, -1, P)                 # Fermat chain
            assert get(6) == pow(a, -1, P)                 # variable-time divsteps
        else:
            assert get(3) == 0 and get(5) == 0 and get(6) == 0


def test_inversions_many_inputs():
    # divsteps (20 batches of 30 half-delta steps), variable-time divsteps and Fermat agree with
    # pow(a, -1, p) on structured inputs (runs of zero / one bits, tiny and near-p values) and
    # thousands of random ones
    P = ecref.P
    vals = [1, 2, 3, P - 1, P - 2, 2**255 % P, P >> 1, (P + 1) >> 1]
    vals += [2**k for k in range(0, 256)] + [(2**k - 1) % P for k in range(1, 257)]
    vals += [P - 2**k for k in range(0, 200, 7)] + [rng.randrange(1, 2**rng.randrange(1, 256)) for _ in range(500)]
    vals += [rng.randrange(1, P) for _ in range(3000)]
    for a in vals:
        a %= P
        if a == 0:
            continue
        want = pow(a, -1, P)
        assert int.from_bytes(call(lib().hfp_op, 3, b32(a), b32(1)), "big") == want, hex(a)
        assert int.from_bytes(call(lib().hfp_op, 6, b32(a), b32(1)), "big") == want, hex(a)
        # the plain-domain cores directly: constant-time (20 x 30 half-delta divsteps) and variable-time, both
        # with the (d, e) update that keeps d, e in (-2p, p) without a per-batch reduction
        want_plain = pow(a, -1, P)
        assert int.from_bytes(call(lib().hfp_inv_plain, 1, b32(a)), "big") == want_plain, hex(a)
        assert int.from_bytes(call(lib().hfp_inv_plain, 0, b32(a)), "big") == want_plain, hex(a)
    assert int.from_bytes(call(lib().hfp_op, 6, b32(0), b32(1)), "big") == 0
    assert int.from_bytes(call(lib().hfp_inv_plain, 1, b32(0)), "big") == 0
    assert int.from_bytes(call(lib().hfp_inv_plain, 0, b32(0)), "big") == 0


def test_montgomery_raw_bound():
    # fe_mul is a Montgomery product a b 2^-256 mod p, fully reduced
    P = ecref.P
    Rinv = pow(2**256, -1, P)
    for _ in range(300):
        a, b = rng.randrange(P), rng.randrange(P)
        r = int.from_bytes(call(lib().hfp_mont_mul_raw, b32(a), b32(b)), "big")
        assert r == a * b * Rinv % P


def test_points_vs_openssl():
    for _ in range(20):
        a, b = rng.randrange(1, ecref.Q), rng.randrange(1, ecref.Q)
        Pa, Pb = ecref.mulG(a), ecref.mulG(b)
        assert call(lib().hpt_add, Pa, Pb, n=64) == ecref.mulG(a + b)
        assert call(lib().hpt_dbl, Pa, n=64) == ecref.mulG(2 * a)
        v = rng.randrange(-300, 300)
        assert call(lib().hpt_mul_small, v, Pa, n=64) == ecref.mulG(v * a)
        k = rng.randrange(2**256)
        assert call(lib().hpt_mul_scalar, b32(k), Pa, n=64) == ecref.mulG(k * a)


def test_complete_formulas_exceptional_cases():
    a = rng.randrange(1, ecref.Q)
    Pa, Na, I = ecref.mulG(a), ecref.mulG(-a), ecref.INF
    assert call(lib().hpt_add, Pa, Pa, n=64) == ecref.mulG(2 * a)     # P + P through the ADD formula
    assert call(lib().hpt_add, Pa, Na, n=64) == I                     # P + (-P)
    assert call(lib().hpt_add, Pa, I, n=64) == Pa
    assert call(lib().hpt_add, I, Pa, n=64) == Pa
    assert call(lib().hpt_add, I, I, n=64) == I
    assert call(lib().hpt_dbl, I, n=64) == I
    assert call(lib().hpt_mul_small, 0, Pa, n=64) == I
    assert lib().hpt_on_curve(Pa) == 1 and lib().hpt_on_curve(I) == 1
    bad = bytearray(Pa); bad[10] ^= 4
    assert lib().hpt_on_curve(bytes(bad)) == 0
    over = b32(ecref.P) + Pa[32:]                                     # x = p is not reduced
    assert lib().hpt_on_curve(over) == 0
