"""End-to-end pins of the oracle's PC-MM engines:
Cussen == schoolbook, both == the Eq. 5 closed form computed from the
plaintext inputs with OpenSSL k*G, and the tiny config decrypts to A.B."""
import numpy as np
import pytest

import oracle
import synth
from tests import ecref


def _encrypt(I):
    H = oracle.pubkey(I.x)
    assert H == ecref.mulG(I.x)
    return oracle.encrypt(H, I.B.reshape(-1), I.r_be)


def _closed(I, i, j):
    n, l = I.cfg.n, I.cfg.l
    r = [int.from_bytes(I.r_be[k * l + j].tobytes(), "big") for k in range(n)]
    R = sum(int(I.A[i, k]) * r[k] for k in range(n))
    c = sum(int(I.A[i, k]) * int(I.B[k, j]) for k in range(n))
    return ecref.enc_closed_form(I.x, R, c)


def test_tiny_config_all_checks_p6():
    I = synth.make_instance(synth.CONFIGS["tiny"])
    ct = _encrypt(I)
    oc, _ = oracle.pcmm(oracle.CUSSEN, I.A, ct, 8, 2)
    os_, _ = oracle.pcmm(oracle.SCHOOLBOOK, I.A, ct, 8, 2)
    assert (oc == os_).all()
    for i in range(8):
        for j in range(8):
            assert oc[i * 8 + j].tobytes() == _closed(I, i, j)
    m, st = oracle.decrypt(I.x, oc, 0, 72)                  # BASELINE tiny: max value 8*3*3 = 72
    assert (st == 0).all()
    assert (m.reshape(8, 8) == I.A.astype(np.int64) @ I.B.astype(np.int64)).all()


def test_rectangular_signed():
    cfg = synth.CONFIGS["ml"]
    I = synth.make_instance(cfg, m=8, n=16, l=4, seed=99)
    ct = _encrypt(I)
    oc, _ = oracle.pcmm(oracle.CUSSEN, I.A, ct, 4, 4)
    os_, _ = oracle.pcmm(oracle.SCHOOLBOOK, I.A, ct, 4, 4)
    assert (oc == os_).all()
    for i in range(8):
        for j in range(4):
            assert oc[i * 4 + j].tobytes() == _closed(I, i, j)
    m, st = oracle.decrypt(I.x, oc, -16 * 8 * 255, 16 * 8 * 255)
    assert (st == 0).all() and (m.reshape(8, 4) == I.A.astype(np.int64) @ I.B.astype(np.int64)).all()


def test_degenerate_matrices():
    I = synth.make_instance(synth.CONFIGS["c64"], m=8, n=8, l=3, seed=5)
    ct = _encrypt(I)
    Z = np.zeros((8, 8), dtype=np.int8)
    for path in (oracle.CUSSEN, oracle.SCHOOLBOOK):
        o, _ = oracle.pcmm(path, Z, ct, 3, 4)
        assert (o == 0).all()                                 # all-zero A -> (inf, inf)
        o, _ = oracle.pcmm(path, np.eye(8, dtype=np.int8), ct, 3, 4)
        assert (o == ct).all()                                 # A = I -> Enc(B) itself
        one = np.ones((1, 1), dtype=np.int8)
        o, _ = oracle.pcmm(path, one, ct[:1], 1, 4)
        assert (o == ct[:1]).all()                             # 1x1x1


def test_c64_cussen_equals_schoolbook_p5():
    I = synth.make_instance(synth.CONFIGS["c64"])
    ct = _encrypt(I)
    oc, _ = oracle.pcmm(oracle.CUSSEN, I.A, ct, 64, 4)
    os_, _ = oracle.pcmm(oracle.SCHOOLBOOK, I.A, ct, 64, 4)
    assert (oc == os_).all()
    for (i, j) in [(0, 0), (17, 42), (63, 63)]:
        assert oc[i * 64 + j].tobytes() == _closed(I, i, j)
    assert oracle.inner_product(I.A[17], ct.reshape(64, 64, 128)[:, 42]) == oc[17 * 64 + 42].tobytes()


@pytest.mark.parametrize("t,signed", [(12, False), (16, False), (16, True)])
def test_wide_plaintexts_t12_t16(t, signed):
    # the paper's t = 12, 16 grid (Table A9): plaintexts wider than a byte, unsigned
    # 16-bit values above 2^15 included; Cussen == schoolbook == Eq. 5 closed form
    cfg = synth.Config(f"w{t}", 6, 7, 3, t, signed, 0, 255, 41 + t)
    I = synth.make_instance(cfg)
    assert I.A.dtype == np.int32
    A = I.A.copy()
    if not signed:
        A[0, 0], A[1, 0], A[2, 1] = (1 << t) - 1, (1 << t) - 2, 1 << (t - 1)
    else:
        A[0, 0], A[1, 0] = -(1 << (t - 1)), (1 << (t - 1)) - 1
    ct = _encrypt(I)
    oc, _ = oracle.pcmm(oracle.CUSSEN, A, ct, 3, t)
    os_, _ = oracle.pcmm(oracle.SCHOOLBOOK, A, ct, 3, t)
    assert (oc == os_).all()
    n = 7
    for i in range(6):
        for j in range(3):
            r = [int.from_bytes(I.r_be[k * 3 + j].tobytes(), "big") for k in range(n)]
            R = sum(int(A[i, k]) * r[k] for k in range(n))
            c = sum(int(A[i, k]) * int(I.B[k, j]) for k in range(n))
            assert oc[i * 3 + j].tobytes() == ecref.enc_closed_form(I.x, R, c)
