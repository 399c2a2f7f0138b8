"""GPU parity tests: the CUDA path through the C ABI vs the CPU oracle (oracle/).

Bar (north_star): BIT-EXACT canonical affine bytes for every output
compared -- all of this is integer work, there is no tolerance.  Expected values
come only from `oracle/` (and, for scalar multiples, OpenSSL via tests/ecref.py)
applied to the seeded synthetic inputs of `synth`; never from the CUDA path.

* small configs (tiny, 64^3, ragged shapes): every output, oracle-encrypted inputs;
* full BASELINE sizes (256^3, 512^3, ML): the launch configuration bench.py uses,
  EVERY output compared byte for byte with the oracle's Cussen PC-MM (Alg. 3,
  P:430-449) on oracle-encrypted inputs (the oracle, all host cores, ~1 min in
  total on a 16-core box), the GPU encryption of the same (B, r) compared with
  the oracle's over all n*l ciphertexts, and a sample of outputs checked a second,
  independent way against the Eq. 5 closed form evaluated from (x, A, B, r) alone.
"""
import functools
import random

import numpy as np
import pytest
import torch

import oracle
import synth
from tests import ecref

pytestmark = pytest.mark.gpu

P = None


def setup_module(_m):
    global P
    from paper_2504_14497_b200 import pcmm
    P = pcmm
    P.load()


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


rng = random.Random(1234)


# ------------------------------------------------------------------ field / points
def test_field_ops_bit_exact():
    vals = [0, 1, 2, ecref.P - 1, ecref.P - 2, 2**224, 2**96 - 1] + [rng.randrange(ecref.P) for _ in range(4000)]
    # structured inputs for the variable-time inversion (long runs of zero / one bits)
    vals += [2**k for k in range(256)] + [(2**k - 1) % ecref.P for k in range(1, 257)] + [ecref.P - 2**k for k in range(0, 224, 5)]
    a = vals
    b = [rng.choice(vals) for _ in vals]
    A = cuda(np.frombuffer(b"".join(v.to_bytes(32, "big") for v in a), dtype=np.uint8).reshape(-1, 32))
    B = cuda(np.frombuffer(b"".join(v.to_bytes(32, "big") for v in b), dtype=np.uint8).reshape(-1, 32))
    for op, f in [(0, lambda x, y: (x + y) % ecref.P), (1, lambda x, y: (x - y) % ecref.P),
                  (2, lambda x, y: x * y % ecref.P), (4, lambda x, y: (-x) % ecref.P),
                  (5, lambda x, y: x * x % ecref.P), (6, lambda x, y: x * y % ecref.P)]:
        out = P.test_field(op, A, B).cpu().numpy()
        for i in range(len(a)):
            assert int.from_bytes(out[i].tobytes(), "big") == f(a[i], b[i]), (op, i)
    for op in (3, 7):                                       # divsteps, Fermat
        out = P.test_field(op, A, B).cpu().numpy()
        for i in range(len(a)):
            exp = pow(a[i], -1, ecref.P) if a[i] else 0
            assert int.from_bytes(out[i].tobytes(), "big") == exp, (op, i)


def test_lazy_field_ops():
    # the accumulate loop's almost-reduced arithmetic (fp_fast.cuh fe_*_lz): operands in [0, 2^256),
    # including non-canonical representatives x + p (ops 8-12 denormalise odd Montgomery forms below
    # 2^256 - p); results must be congruent mod p (fully reduced by the harness afterwards), and the
    # zero test must accept both 0 and p.  Edge forms: 0, 1, the largest below 2^256 - p (double wrap
    # of the sum: both operands near 2^256), small even minus small odd (difference below -p).
    Pm = ecref.P
    R = 2**256
    Rinv = pow(R, -1, Pm)
    delta = R - Pm
    forms = [0, 1, 2, 3, delta - 1, delta - 2, delta - 3, delta - 5, 5, 7, Pm - 1, Pm - 2]
    forms += [rng.randrange(delta) for _ in range(1500)] + [rng.randrange(Pm) for _ in range(1500)]
    a = [f * Rinv % Pm for f in forms]                      # plain values whose Montgomery forms are `forms`
    b = [a[(i * 7 + 3) % len(a)] for i in range(len(a))]
    b[: 12] = [a[4], a[4], a[6], a[2], a[4], a[0], a[1], a[3], a[6], a[0], a[11], a[10]]
    A = cuda(np.frombuffer(b"".join(v.to_bytes(32, "big") for v in a), dtype=np.uint8).reshape(-1, 32))
    B = cuda(np.frombuffer(b"".join(v.to_bytes(32, "big") for v in b), dtype=np.uint8).reshape(-1, 32))
    for op, f in [(8, lambda x, y: x * y % Pm), (9, lambda x, y: x * x % Pm), (10, lambda x, y: (x + y) % Pm),
                  (11, lambda x, y: (x - y) % Pm)]:
        out = P.test_field(op, A, B).cpu().numpy()
        for i in range(len(a)):
            assert int.from_bytes(out[i].tobytes(), "big") == f(a[i], b[i]), (op, i)
    out = P.test_field(12, A, B).cpu().numpy()
    for i in range(len(a)):
        assert int.from_bytes(out[i].tobytes(), "big") == (1 if a[i] == 0 else 2), i


def _pts(scalars):
    return cuda(np.frombuffer(b"".join(ecref.mulG(s) for s in scalars), dtype=np.uint8).reshape(-1, 64))


def test_point_ops_vs_openssl():
    n = 64
    a = [rng.randrange(1, ecref.Q) for _ in range(n)]
    b = [rng.randrange(1, ecref.Q) for _ in range(n)]
    b[0], b[1], b[2] = a[0], ecref.Q - a[1], 0           # P+P, P+(-P), P+inf through the add formula
    a[3] = 0                                               # inf + Q
    Pa, Pb = _pts(a), _pts(b)
    add = P.test_point(0, Pa, Pb).cpu().numpy()
    dbl = P.test_point(1, Pa).cpu().numpy()
    v = [rng.randrange(-40000, 40000) for _ in range(n)]
    v[4], v[5] = 0, 1
    mul = P.test_point(2, Pa, v=cuda(np.array(v, dtype=np.int32))).cpu().numpy()
    k = [rng.randrange(2**256) for _ in range(n)]
    k[6], k[7], k[8], k[9] = 0, 1, 15, 2**256 - 1          # empty, single, one-window and all-ones scalars
    K = cuda(np.frombuffer(b"".join(x.to_bytes(32, "big") + bytes(32) for x in k), dtype=np.uint8).reshape(-1, 64))
    kmul = P.test_point(3, Pa, K).cpu().numpy()
    kmul2 = P.test_point(4, Pa, K).cpu().numpy()
    assert (kmul == kmul2).all()
    for i in range(n):
        assert add[i].tobytes() == ecref.mulG(a[i] + b[i]), i
        assert dbl[i].tobytes() == ecref.mulG(2 * a[i]), i
        assert mul[i].tobytes() == ecref.mulG(v[i] * a[i]), i
        assert kmul[i].tobytes() == ecref.mulG(k[i] * a[i]), i


# ------------------------------------------------------------------ EC-ElGamal boundary
def test_keygen_matches_generator_and_openssl():
    for seed in (0, 1, 2, 3, 4, 12345):
        sk, pk = P.keygen(seed)
        x = synth.keygen_secret(seed)
        assert int.from_bytes(sk, "big") == x
        assert pk == ecref.mulG(x) == oracle.pubkey(x)


def test_encrypt_matches_oracle():
    I = synth.make_instance(synth.CONFIGS["c64"], m=4, n=16, l=16, seed=77)
    sk, pk = P.keygen(77)
    b = I.B.reshape(-1).astype(np.int32)
    b[:4] = [0, 1, -1, -255]
    ct = P.encrypt(pk, cuda(b), cuda(I.r_be)).cpu().numpy()
    exp = oracle.encrypt(pk, b.astype(np.int64), I.r_be)
    assert (ct == exp).all()


def test_decrypt_small():
    I = synth.make_instance(synth.CONFIGS["c64"], m=4, n=8, l=8, seed=5)
    sk, pk = P.keygen(5)
    b = np.arange(-20, 44, dtype=np.int32)
    ct = oracle.encrypt(pk, b.astype(np.int64), I.r_be[:64])
    m, st = P.decrypt_small(sk, cuda(ct), -20, 43)
    assert (st.cpu().numpy() == 0).all() and (m.cpu().numpy() == b).all()
    m, st = P.decrypt_small(sk, cuda(ct), 0, 10)
    st = st.cpu().numpy()
    assert ((st == P.PCMM_EDECODE) == ((b < 0) | (b > 10))).all()


# ------------------------------------------------------------------ step a1: compression plan
@pytest.mark.parametrize("w,signed", [(1, False), (2, False), (3, False), (4, False), (4, True), (2, True),
                                      (5, False), (6, True), (8, False), (8, True)])
def test_plan_matches_oracle(w, signed):
    g = np.random.default_rng(w * 10 + signed)
    lo, hi = (-(1 << (w - 1)), (1 << (w - 1)) - 1) if signed else (0, (1 << w) - 1)
    m, n = (77, 40) if w <= 4 else (300, 24)
    A = g.integers(lo, hi + 1, (m, n)).astype(np.int8 if signed else np.uint8)
    A[:, 0] = 0                                   # all-zero column
    A[:, 1] = hi                                  # constant column
    A[::3, 2] = 0                                 # many zeros
    for N in (1, 2, 3, 4):
        levels, sN, rank = P.test_plan(cuda(A), w, signed, N)
        levels, sN, rank = levels.cpu().numpy(), sN.cpu().numpy(), rank.cpu().numpy()
        for k in range(n):
            lev = oracle.cussen_plan(A[:, k].astype(np.int64), N)
            assert list(levels[k, :N]) == [len(s) for s, _ in lev], (N, k)
            assert list(sN[k, : len(lev[-1][0])]) == list(lev[-1][0])
            exp_rank = np.where(lev[0][1] < 0, 0, lev[0][1] + 1)
            assert (rank[k] == exp_rank).all()


# ------------------------------------------------------------------ full PC-MM, small sizes: every output
def _gpu_pcmm(A, ct, l, w, signed, path, iters=4):
    return P.pcmm(cuda(A), cuda(ct), l, w, signed, path=path, iters=iters).cpu().numpy()


def test_tiny_config_both_paths_and_decrypt():
    I = synth.make_instance(synth.CONFIGS["tiny"])
    sk, pk = P.keygen(0)
    ct = oracle.encrypt(pk, I.B.reshape(-1), I.r_be)
    exp, _ = oracle.pcmm(oracle.CUSSEN, I.A, ct, 8, 2)
    for path in (P.CUSSEN, P.SCHOOLBOOK):
        out = _gpu_pcmm(I.A, ct, 8, 2, False, path)
        assert (out == exp).all(), path
    # P6: brute-force dlog of the GPU output = A.B
    m, st = P.decrypt_small(sk, cuda(exp), 0, 72)
    assert (st.cpu().numpy() == 0).all()
    assert (m.cpu().numpy().reshape(8, 8) == I.A.astype(np.int64) @ I.B.astype(np.int64)).all()


def test_tiny_forced_real_ecsm_column():
    # force a column whose compression ends in a value != 1 (a real ECSM, step a2)
    I = synth.make_instance(synth.CONFIGS["tiny"])
    A = I.A.copy()
    A[:, 3] = [0, 3, 3, 0, 3, 0, 0, 3]            # level values {3} -> ECSM by 3
    A[:, 5] = [2, 0, 2, 2, 0, 0, 2, 0]            # {2}
    sk, pk = P.keygen(0)
    ct = oracle.encrypt(pk, I.B.reshape(-1), I.r_be)
    exp, _ = oracle.pcmm(oracle.SCHOOLBOOK, A, ct, 8, 2)
    for path in (P.CUSSEN, P.SCHOOLBOOK):
        assert (_gpu_pcmm(A, ct, 8, 2, False, path) == exp).all()


def test_c64_config_every_output():
    I = synth.make_instance(synth.CONFIGS["c64"])
    sk, pk = P.keygen(1)
    ct = oracle.encrypt(pk, I.B.reshape(-1), I.r_be)
    exp, _ = oracle.pcmm(oracle.CUSSEN, I.A, ct, 64, 4)
    for path in (P.CUSSEN, P.SCHOOLBOOK):
        assert (_gpu_pcmm(I.A, ct, 64, 4, False, path) == exp).all(), path


@pytest.mark.parametrize("shape,w,signed,iters", [((100, 37, 45), 3, True, 4), ((129, 70, 33), 4, False, 4),
                                                  ((1, 1, 1), 4, False, 4), ((1, 200, 3), 4, True, 2),
                                                  ((260, 5, 1), 2, False, 1), ((33, 64, 130), 4, True, 3),
                                                  ((140, 20, 9), 8, False, 4), ((64, 16, 40), 8, True, 4),
                                                  ((300, 9, 5), 6, False, 2), ((50, 30, 3), 5, True, 1),
                                                  ((256, 12, 7), 7, False, 3)])
def test_ragged_shapes_every_output(shape, w, signed, iters):
    m, n, l = shape
    cfg = synth.Config("ragged", m, n, l, w, signed, 0, 255, 1000 + m + w)
    I = synth.make_instance(cfg)
    x = synth.keygen_secret(cfg.seed)
    ct = oracle.encrypt(ecref.mulG(x), I.B.reshape(-1), I.r_be)
    exp, _ = oracle.pcmm(oracle.SCHOOLBOOK if n * m * l < 20000 else oracle.CUSSEN, I.A, ct, l, w)
    for path in (P.CUSSEN, P.SCHOOLBOOK):
        assert (_gpu_pcmm(I.A, ct, l, w, signed, path, iters) == exp).all(), path


def test_degenerate_matrices():
    I = synth.make_instance(synth.CONFIGS["c64"], m=16, n=16, l=8, seed=9)
    x = synth.keygen_secret(9)
    ct = oracle.encrypt(ecref.mulG(x), I.B.reshape(-1), I.r_be)
    Z = np.zeros((16, 16), dtype=np.uint8)
    E = np.eye(16, dtype=np.uint8)
    C = np.full((16, 16), 15, dtype=np.uint8)
    for path in (P.CUSSEN, P.SCHOOLBOOK):
        assert (_gpu_pcmm(Z, ct, 8, 4, False, path) == 0).all()                 # (inf, inf)
        assert (_gpu_pcmm(E, ct, 8, 4, False, path) == ct).all()                # A = I -> Enc(B)
        exp, _ = oracle.pcmm(oracle.CUSSEN, C, ct, 8, 4)
        assert (_gpu_pcmm(C, ct, 8, 4, False, path) == exp).all()
    # an infinity ciphertext in the input
    ct2 = ct.copy()
    ct2[5] = 0
    exp, _ = oracle.pcmm(oracle.CUSSEN, I.A, ct2, 8, 4)
    assert (_gpu_pcmm(I.A, ct2, 8, 4, False, P.CUSSEN) == exp).all()


@pytest.mark.parametrize("w,l", [(2, 128), (4, 128), (4, 130)])
def test_consecutive_column_tables_mixed(w, l):
    # A launch large enough for the consecutive-column kernels (2 n l >= 65536): columns whose
    # level-1 set is {1..n1} (k_tables_coz by default: co-Z prefix chain converted to affine in the
    # same kernel; PCMM_TABLES_COZ=0: XYZZ prefix sums converted by k_affine's XYZZ branch) next to
    # columns that are not (k_tables + homogeneous k_affine), an all-zero column, identity
    # ciphertexts in a consecutive column, n1 = 1, 5, 7 (not powers of two), and l = 130 so that
    # warps straddle columns k with different n1.
    m, n = 8, 256
    cfg = synth.Config("mixed", m, n, l, w, False, 0, 255, 77 + w)
    I = synth.make_instance(cfg)
    A = I.A.copy()
    top = (1 << w) - 1
    A[:, 0] = [(i % top) + 1 for i in range(m)]        # consecutive, n1 = min(m, top)
    A[:, 1] = 2                                          # {2}: not consecutive
    A[:, 2] = 0                                          # empty column
    A[:, 3] = [1, 3] * (m // 2)                          # {1, 3}: not consecutive
    A[:, 4] = [1, 2] * (m // 2)                          # consecutive, n1 = 2
    A[:, 5] = 1                                          # consecutive, n1 = 1 (no rounds)
    A[:, 6] = [(i % 5) + 1 for i in range(m)] if w > 2 else 3 - (np.arange(m) % 3)   # n1 = 5 (w = 2: 3)
    A[:, 7] = [(i % 7) + 1 for i in range(m)] if w > 2 else 1 + (np.arange(m) % 2)   # n1 = 7 (w = 2: 2)
    x = synth.keygen_secret(cfg.seed)
    ct = oracle.encrypt(ecref.mulG(x), I.B.reshape(-1), I.r_be).reshape(n, l, 128)
    ct[0, 5] = 0                                         # (inf, inf) in consecutive column k = 0
    ct[4, :7, 64:] = 0                                   # C2 = inf in k = 4
    ct = np.ascontiguousarray(ct.reshape(n * l, 128))
    exp, _ = oracle.pcmm(oracle.CUSSEN, A, ct, l, w)
    assert (_gpu_pcmm(A, ct, l, w, False, P.CUSSEN) == exp).all()


@pytest.mark.parametrize("w,l", [(4, 128), (8, 130), (3, 128)])
def test_signed_chain_columns_mixed(w, l):
    # Signed A in a launch large enough for k_tables_coz (2 n l >= 65536): columns whose magnitudes are
    # {1..M} in either sign (R10b: one chain P..MP, the entry of -v is the negated entry of
    # v) next to columns with a gap in the magnitudes (k_tables + k_affine), only negative values,
    # only positive values, the most negative value -2^(w-1), an all-zero column, M = 1, and identity
    # ciphertexts in chain columns.
    m, n = (136, 256) if w == 8 else (24, 256)
    cfg = synth.Config("smixed", m, n, l, w, True, 0, 255, 91 + w)
    I = synth.make_instance(cfg)
    A = I.A.copy().astype(np.int8)
    lo, hi = -(1 << (w - 1)), (1 << (w - 1)) - 1
    r = np.arange(m)
    A[:, 0] = np.where(r % 2 == 0, (r % hi) + 1, -((r % hi) + 1))       # +-1..hi mixed signs
    A[:, 1] = -((r % min(hi, 5)) + 1)                                    # only negatives, M = min(hi, 5)
    A[:, 2] = 0                                                          # empty column
    A[:, 3] = np.where(r % 2 == 0, 1, -3)                                # magnitudes {1, 3}: gap -> general
    A[:, 4] = np.where(r % 3 == 0, lo, -((r % (-lo - 1)) + 1) if lo < -1 else lo)   # includes -2^(w-1)
    A[:, 5] = np.where(r % 2 == 0, 1, -1)                                # M = 1, both signs
    A[:, 6] = (r % hi) + 1                                               # only positives 1..hi
    A[:, 7] = np.where(r % 2 == 0, 2, -1)                                # {-1, 2}: magnitudes {1, 2}
    A[:, 8] = np.where(r % 2 == 0, 3, -3)                                # {-3, 3}: gap (1, 2 missing) -> general
    if w == 8:
        A[:, 9] = -np.minimum(r + 1, 128)                                # -1..-128: chain of 128, all negative
    x = synth.keygen_secret(cfg.seed)
    ct = oracle.encrypt(ecref.mulG(x), I.B.reshape(-1), I.r_be).reshape(n, l, 128)
    ct[0, 5] = 0                                         # (inf, inf) in chain column k = 0
    ct[7, :7, 64:] = 0                                   # C2 = inf in k = 7
    ct[3, 2] = 0                                         # (inf, inf) in a general column
    ct = np.ascontiguousarray(ct.reshape(n * l, 128))
    exp, _ = oracle.pcmm(oracle.CUSSEN, A, ct, l, w)
    assert (_gpu_pcmm(A, ct, l, w, True, P.CUSSEN) == exp).all()


@pytest.mark.parametrize("w,signed", [(8, False), (7, True)])
def test_xyzz_level1_tables_with_identities(w, signed):
    # k_tables_x (2^w >= 128 slots, many tables): level-2 entries made affine by a warp-shared inversion,
    # level-1 prefix sums as XYZZ mixed additions; identity ciphertexts (both or one component) and
    # repeated ciphertexts in the inputs
    m, n, l = 40, 24, 16
    cfg = synth.Config("x", m, n, l, w, signed, 0, 255, 300 + w)
    I = synth.make_instance(cfg)
    x = synth.keygen_secret(cfg.seed)
    ct = oracle.encrypt(ecref.mulG(x), I.B.reshape(-1), I.r_be).reshape(n, l, 128)
    ct[3, 2] = 0                                         # (inf, inf)
    ct[5, :4, :64] = 0                                   # C1 = inf
    ct[7] = ct[6]                                        # equal ciphertexts in consecutive k
    ct = np.ascontiguousarray(ct.reshape(n * l, 128))
    exp, _ = oracle.pcmm(oracle.CUSSEN, I.A, ct, l, w)
    for path in (P.CUSSEN, P.SCHOOLBOOK):
        assert (_gpu_pcmm(I.A, ct, l, w, signed, path) == exp).all(), path


@pytest.mark.parametrize("w", [4, 6])
def test_accumulator_exceptional_cases(w):
    # Equal ciphertexts in rows k = 0..3 make the accumulated sum equal to +-(the next
    # table entry): the Jacobian + affine mixed addition of the accumulate kernel hits
    # H = 0 (doubling, and cancellation to the identity followed by more additions),
    # which its general path must handle.  w = 4: shared-memory kernel, w = 6: the
    # global-gather kernel.
    m, n, l = 8, 8, 4
    I = synth.make_instance(synth.CONFIGS["c64"], m=m, n=n, l=l, seed=21)
    x = synth.keygen_secret(21)
    ct = oracle.encrypt(ecref.mulG(x), I.B.reshape(-1), I.r_be).reshape(n, l, 128)
    ct[1] = ct[0]
    ct[2] = ct[0]
    ct[3] = ct[0]
    ct = np.ascontiguousarray(ct.reshape(n * l, 128))
    A = np.array([[1, 1, 0, 0, 3, 2, 1, 0],          # Q + Q
                  [1, -1, 0, 0, 5, 0, 0, 2],         # Q - Q = identity, then more
                  [2, 0, -2, 0, 0, 0, 0, 1],         # 2Q - 2Q
                  [1, 1, -2, 0, 0, 0, 0, 0],         # Q + Q - 2Q = identity at the end
                  [3, -1, -2, 0, 0, 1, 0, 0],
                  [-1, -1, -1, 3, 0, 0, 0, 0],       # -Q - Q - Q + 3Q
                  [7, -8, 1, 0, 1, 1, 1, 1],
                  [-8, 7, 1, 1, -1, 2, -3, 4]], dtype=np.int8)
    if w == 6:
        A = A.astype(np.int16) * 3
        A[6, 0], A[6, 1] = 31, -32
        A = A.astype(np.int8)
    exp, _ = oracle.pcmm(oracle.SCHOOLBOOK, A, ct, l, w)
    for path in (P.CUSSEN, P.SCHOOLBOOK):
        assert (_gpu_pcmm(A, ct, l, w, True, path) == exp).all(), path
    assert (exp[3 * l:4 * l] == 0).all()            # row 3 sums to the identity in every column


def test_all_identity_ciphertexts_consecutive_tables():
    # Every ciphertext is (inf, inf) (64 + 64 zero bytes are valid input) in a launch that takes
    # k_tables_fast (unsigned, consecutive columns, 2 n l >= 65536): every table entry is the identity,
    # so no CTA of k_affine has anything to invert, and every output must be (inf, inf)
    m, n, l = 8, 256, 128
    cfg = synth.Config("allinf", m, n, l, 4, False, 0, 255, 4242)
    I = synth.make_instance(cfg)
    A = I.A.copy()
    A[:, :] = (np.arange(m)[:, None] % 15) + 1          # every column consecutive {1..8}
    ct = np.zeros((n * l, 128), dtype=np.uint8)
    exp, _ = oracle.pcmm(oracle.CUSSEN, A, ct, l, 4)
    assert (exp == 0).all()
    assert (_gpu_pcmm(A, ct, l, 4, False, P.CUSSEN) == 0).all()
    # and half of the columns identity, half not: mixed CTAs
    x = synth.keygen_secret(cfg.seed)
    ct2 = oracle.encrypt(ecref.mulG(x), I.B.reshape(-1), I.r_be).reshape(n, l, 128)
    ct2[: n // 2] = 0
    ct2 = np.ascontiguousarray(ct2.reshape(n * l, 128))
    exp2, _ = oracle.pcmm(oracle.CUSSEN, A, ct2, l, 4)
    assert (_gpu_pcmm(A, ct2, l, 4, False, P.CUSSEN) == exp2).all()


def test_encrypt_rejects_off_curve_key():
    sk, pk = P.keygen(3)
    bad = bytearray(pk)
    bad[40] ^= 4
    b = torch.zeros(4, dtype=torch.int32, device="cuda")
    r = torch.ones((4, 32), dtype=torch.uint8, device="cuda")
    with pytest.raises(P.PCMMError) as e:
        P.encrypt(bytes(bad), b, r)
    assert e.value.code == P.PCMM_ENOTONCURVE
    assert P.encrypt(pk, b, r).shape == (4, 128)


def test_error_reporting():
    I = synth.make_instance(synth.CONFIGS["c64"], m=8, n=8, l=8, seed=3)
    x = synth.keygen_secret(3)
    ct = oracle.encrypt(ecref.mulG(x), I.B.reshape(-1), I.r_be)
    bad = I.A.copy()
    bad[2, 3] = 16
    for path in (P.CUSSEN, P.SCHOOLBOOK):
        with pytest.raises(P.PCMMError) as e:
            _gpu_pcmm(bad, ct, 8, 4, False, path)
        assert e.value.code == P.PCMM_EBOUND
    cbad = ct.copy()
    cbad[7, 10] ^= 1
    with pytest.raises(P.PCMMError) as e:
        _gpu_pcmm(I.A, cbad, 8, 4, False, P.CUSSEN)
    assert e.value.code == P.PCMM_ENOTONCURVE
    with pytest.raises(P.PCMMError) as e:
        _gpu_pcmm(I.A, ct, 8, 9, False, P.CUSSEN)
    assert e.value.code == P.PCMM_EINVAL
    with pytest.raises(P.PCMMError) as e:
        _gpu_pcmm(I.A, ct, 8, 4, False, P.CUSSEN, iters=5)
    assert e.value.code == P.PCMM_ENOTSUP


# ------------------------------------------------------------------ full BASELINE sizes: sampled outputs
def _full_size(name, path, samples):
    cfg = synth.CONFIGS[name]
    I = synth.make_instance(cfg)
    sk, pk = P.keygen(cfg.seed)
    n, l = cfg.n, cfg.l
    ctd = P.encrypt(pk, cuda(I.B.reshape(-1).astype(np.int32)), cuda(I.r_be))
    ct = ctd.cpu().numpy()
    g = np.random.default_rng(cfg.seed)
    idx = g.choice(n * l, 24, replace=False)
    exp_ct = oracle.encrypt(pk, I.B.reshape(-1)[idx].astype(np.int64), I.r_be[idx])
    assert (ct[idx] == exp_ct).all()                                  # GPU encryption vs oracle
    out = P.pcmm(cuda(I.A), ctd, l, cfg.w, cfg.signed, path=path).cpu().numpy()
    r = I.r_be.reshape(n, l, 32)
    picks = [(0, 0), (cfg.m - 1, l - 1)] + [(int(g.integers(cfg.m)), int(g.integers(l))) for _ in range(samples)]
    for (i, j) in picks:
        exp = oracle.closed_form(I.x, I.A[i], I.B[:, j], r[:, j])
        assert out[i * l + j].tobytes() == exp, (name, i, j)
    return out


@functools.lru_cache(maxsize=None)
def _oracle_full(name):
    """The oracle's answer for a BASELINE config: (instance, pk, Enc(B), C) with Enc(B) from
    oracle.encrypt and C = oracle.pcmm(CUSSEN) (Alg. 3 step by step, all host cores)."""
    cfg = synth.CONFIGS[name]
    I = synth.make_instance(cfg)
    pk = oracle.pubkey(I.x)
    ct = oracle.encrypt(pk, I.B.reshape(-1), I.r_be)
    exp, _ = oracle.pcmm(oracle.CUSSEN, I.A, ct, cfg.l, cfg.w)
    return I, pk, ct, exp


def _every_output(name, path):
    cfg = synth.CONFIGS[name]
    I, pk, ct, exp = _oracle_full(name)
    out = P.pcmm(cuda(I.A), cuda(ct), cfg.l, cfg.w, cfg.signed, path=path).cpu().numpy()
    bad = np.nonzero((out != exp).any(axis=1))[0]
    assert bad.size == 0, (name, path, bad.size, [(int(e) // cfg.l, int(e) % cfg.l) for e in bad[:8]])
    return I, out


@pytest.mark.parametrize("name", ["c256", "c512", "ml"])
def test_full_size_cussen_every_output(name):
    # north_star: bit-exact agreement with the CPU oracle on every BASELINE config (Cussen
    # "always performs exact reconstruction"); every one of the m*l outputs, launch configuration of bench.py
    cfg = synth.CONFIGS[name]
    I, out = _every_output(name, P.CUSSEN)
    # second, independent check of a sample: the Eq. 5 closed form from (x, A, B, r) alone
    r = I.r_be.reshape(cfg.n, cfg.l, 32)
    g = np.random.default_rng(cfg.seed)
    for (i, j) in [(0, 0), (cfg.m - 1, cfg.l - 1)] + [(int(g.integers(cfg.m)), int(g.integers(cfg.l)))
                                                      for _ in range(6)]:
        assert out[i * cfg.l + j].tobytes() == oracle.closed_form(I.x, I.A[i], I.B[:, j], r[:, j]), (name, i, j)


def test_full_size_c256_schoolbook_every_output():
    # the comparison path on the headline config, every output
    _every_output("c256", P.SCHOOLBOOK)


@pytest.mark.parametrize("name", ["c256", "c512", "ml"])
def test_full_size_gpu_encryption_every_ciphertext(name):
    # pcmm_encrypt on the full B of each config equals the oracle's Encrypt for every ciphertext
    I, pk, ct, _ = _oracle_full(name)
    got = P.encrypt(pk, cuda(I.B.reshape(-1).astype(np.int32)), cuda(I.r_be)).cpu().numpy()
    assert (got == ct).all()


def test_full_size_gpu_encrypted_inputs_sampled():
    # the bench's own input path (B encrypted on the GPU) at 256^3, sampled vs Eq. 5
    _full_size("c256", P.CUSSEN, 8)


@pytest.mark.parametrize("name,path", [("c512", "schoolbook"), ("ml", "schoolbook"), ("c256", "strassen"),
                                       ("ml", "strassen")])
def test_full_size_comparison_paths_sampled(name, path):
    # the comparison paths at BASELINE sizes, sampled outputs vs the Eq. 5 closed form
    _full_size(name, P.SCHOOLBOOK if path == "schoolbook" else P.STRASSEN, 8)


# ------------------------------------------------------------------ edge cases
def test_empty_and_invalid_sizes():
    z = torch.zeros(0, dtype=torch.uint8, device="cuda")
    assert P.normalize(torch.zeros(0, dtype=torch.uint8, device="cuda"), 0).shape == (0, 128)
    sk, pk = P.keygen(1)
    assert P.encrypt(pk, torch.zeros(0, dtype=torch.int32, device="cuda"), z).shape == (0, 128)
    m, st = P.decrypt_small(sk, torch.zeros((0, 128), dtype=torch.uint8, device="cuda"), 0, 10)
    assert m.numel() == 0 and st.numel() == 0
    L = P.load()
    for dims in ((0, 4, 4), (4, 0, 4), (4, 4, 0), (-1, 4, 4)):
        rc = L.pcmm_mul_cussen(1, dims[0], dims[1], dims[2], 4, 0, 4, 16, 16, 256, 1 << 20, None)
        assert rc == P.PCMM_EDIM
    assert L.pcmm_workspace_bytes(4, 4, 4, 4, 1) > 0


def test_extreme_values_and_shapes():
    # extreme plaintexts (all max / all min signed), many rows (16 row blocks), long k (split-k)
    # (m = 4200 > 4096: k_rowperm sorts per 128-row block instead of the whole column, 33 row blocks, ragged tail)
    for (m, n, l, w, signed) in ((2048, 6, 2, 4, False), (40, 2048, 2, 4, True), (16, 8, 3, 8, True),
                                 (4200, 7, 2, 3, False)):
        cfg = synth.Config("edge", m, n, l, w, signed, 0, 255, 31 + m)
        I = synth.make_instance(cfg)
        lo, hi = cfg.a_range
        A = I.A.copy()
        A[:, 0] = hi
        A[:, 1] = lo if signed else 0
        A[0, :] = hi
        if signed:
            A[1, :] = lo
        x = synth.keygen_secret(cfg.seed)
        ct = oracle.encrypt(ecref.mulG(x), I.B.reshape(-1), I.r_be)
        out = _gpu_pcmm(A, ct, l, w, signed, P.CUSSEN)
        sb = _gpu_pcmm(A, ct, l, w, signed, P.SCHOOLBOOK)
        assert (out == sb).all()
        r = I.r_be.reshape(n, l, 32)
        for (i, j) in [(0, 0), (1, l - 1), (m - 1, 0), (m // 2, l // 2)]:
            assert out[i * l + j].tobytes() == oracle.closed_form(x, A[i], I.B[:, j], r[:, j]), (m, n, i, j)


# ------------------------------------------------------------------ NEXT-3: Strassen comparison path
@pytest.mark.parametrize("shape,w,signed,leaf", [((16, 16, 16), 4, False, 4), ((32, 32, 32), 2, False, 8),
                                                 ((24, 40, 12), 4, True, 3), ((8, 8, 8), 8, True, 1),
                                                 ((30, 18, 10), 3, False, 2)])
def test_strassen_every_output(shape, w, signed, leaf):
    m, n, l = shape
    cfg = synth.Config("strassen", m, n, l, w, signed, 0, 255, 500 + m + w)
    I = synth.make_instance(cfg)
    x = synth.keygen_secret(cfg.seed)
    ct = oracle.encrypt(ecref.mulG(x), I.B.reshape(-1), I.r_be)
    exp, _ = oracle.pcmm(oracle.CUSSEN, I.A, ct, l, w)
    out = P.pcmm(cuda(I.A), cuda(ct), l, w, signed, path=P.STRASSEN, iters=leaf).cpu().numpy()
    assert (out == exp).all()


def test_strassen_c64_every_output():
    I = synth.make_instance(synth.CONFIGS["c64"])
    sk, pk = P.keygen(1)
    ct = oracle.encrypt(pk, I.B.reshape(-1), I.r_be)
    exp, _ = oracle.pcmm(oracle.CUSSEN, I.A, ct, 64, 4)
    out = P.pcmm(cuda(I.A), cuda(ct), 64, 4, False, path=P.STRASSEN, iters=16).cpu().numpy()
    assert (out == exp).all()


# ------------------------------------------------------------------ NEXT-1: wide plaintexts (t = 12, 16)
@pytest.mark.parametrize("shape,t,signed", [((20, 24, 6), 12, False), ((33, 17, 5), 16, False),
                                            ((16, 40, 3), 16, True), ((64, 64, 64), 16, False),
                                            ((40, 48, 8), 12, True)])
def test_wide_every_output(shape, t, signed):
    # the paper's t = 12, 16 grid (Table A9): int32 plaintexts, up to min(m, 2^t - 1)
    # distinct values per column; unsigned 16-bit values above 2^15 included
    m, n, l = shape
    cfg = synth.Config("wide", m, n, l, t, signed, 0, 255, 700 + m + t)
    I = synth.make_instance(cfg)
    A = I.A.copy()
    if signed:
        A[0, 0], A[1, 0], A[2, 0] = -(1 << (t - 1)), (1 << (t - 1)) - 1, 0
    else:
        A[0, 0], A[1, 0], A[2, 0] = (1 << t) - 1, 1 << (t - 1), 0
    A[3, :] = A[4, :]                               # repeated rows / values
    x = synth.keygen_secret(cfg.seed)
    ct = oracle.encrypt(ecref.mulG(x), I.B.reshape(-1), I.r_be)
    exp, _ = oracle.pcmm(oracle.SCHOOLBOOK if m * n * l > 60000 else oracle.CUSSEN, A, ct, l, t)
    for path in (P.CUSSEN, P.SCHOOLBOOK):
        out = _gpu_pcmm(A, ct, l, t, signed, path)
        assert (out == exp).all(), path
    if m % 2 == 0 and n % 2 == 0 and l % 2 == 0:
        assert (_gpu_pcmm(A, ct, l, t, signed, P.STRASSEN, iters=4) == exp).all()   # leaf 4


def test_wide_chunked_equals_byte_path():
    # the wide path at w <= 8 (several k-chunks forced by a tiny table budget) equals the
    # byte path bit for bit, and an out-of-range plaintext is reported as EBOUND
    import os
    I = synth.make_instance(synth.CONFIGS["c64"], m=48, n=40, l=24, seed=77)
    x = synth.keygen_secret(77)
    ct = oracle.encrypt(ecref.mulG(x), I.B.reshape(-1), I.r_be)
    ref = _gpu_pcmm(I.A, ct, 24, 4, False, P.CUSSEN)
    os.environ["PCMM_WIDE_BUDGET_MB"] = "1"
    try:
        out = _gpu_pcmm(I.A.astype(np.int32), ct, 24, 4, False, P.CUSSEN)
    finally:
        del os.environ["PCMM_WIDE_BUDGET_MB"]
    assert (out == ref).all()
    bad = I.A.astype(np.int32)
    bad[5, 7] = 1 << 12
    with pytest.raises(P.PCMMError) as e:
        _gpu_pcmm(bad, ct, 24, 12, False, P.CUSSEN)
    assert e.value.code == P.PCMM_EBOUND


# ------------------------------------------------------------------ NEXT-2: comb encryption, BSGS decryption
def test_encrypt_comb_matches_oracle():
    x = synth.keygen_secret(31)
    pk = ecref.mulG(x)
    ctx = P.enc_ctx(pk)
    g = synth.SplitMix64(31)
    count = 3000
    b = g.small(-(2**31), 2**31 - 1, count)
    b[:8] = [0, 1, -1, 2**31 - 1, -(2**31), 255, -256, 65536]
    b = b.astype(np.int32)
    rs = g.scalars256(count)
    rs[:6] = [1, ecref.Q - 1, 2**255, 256, 2**64 - 1, 0x0100000000000000000000000000000000000000000000000000000000000001]
    r_be = synth.scalars_to_be_bytes(rs)
    exp = oracle.encrypt(pk, b, r_be)
    out = P.encrypt_ctx(ctx, cuda(b), cuda(r_be)).cpu().numpy()
    assert (out == exp).all()
    assert (P.encrypt(pk, cuda(b), cuda(r_be)).cpu().numpy() == exp).all()


def test_enc_ctx_rejects_bad_key():
    bad = bytearray(ecref.mulG(5))
    bad[63] ^= 1
    with pytest.raises(P.PCMMError) as e:
        P.enc_ctx(bytes(bad))
    assert e.value.code == P.PCMM_ENOTONCURVE
    with pytest.raises(P.PCMMError) as e:
        P.enc_ctx(bytes(64))
    assert e.value.code == P.PCMM_ENOTONCURVE


def test_decrypt_bsgs_ranges():
    x = synth.keygen_secret(32)
    sk = x.to_bytes(32, "big")
    pk = ecref.mulG(x)
    g = synth.SplitMix64(32)
    lo, hi = -(2**29) + 7, 2**30 - 3
    s = 2**20
    msgs = [lo, hi, lo + s, lo + 5 * s, lo + 5 * s - 1, 0, 1, -1, lo + 1, hi - 1]
    msgs += [int(v) for v in g.small(lo, hi, 200)]
    out_of_range = [lo - 1, hi + 1, -(2**31), 2**31 - 1]
    b = np.array(msgs + out_of_range, dtype=np.int64).astype(np.int32)
    ct = oracle.encrypt(pk, b, synth.scalars_to_be_bytes(g.scalars256(len(b))))
    ctx = P.bsgs_ctx(20)
    m, st = P.decrypt_bsgs(sk, ctx, 20, cuda(ct), lo, hi)
    m, st = m.cpu().numpy(), st.cpu().numpy()
    n_in = len(msgs)
    assert (st[:n_in] == 0).all() and (m[:n_in] == np.array(msgs)).all()
    assert (st[n_in:] == P.PCMM_EDECODE).all()
    # agrees with the exact-table decryption on a small range, and reports a bad point
    small = np.array([-5, 0, 3, 100, 999], dtype=np.int32)
    ct2 = oracle.encrypt(pk, small, synth.scalars_to_be_bytes(g.scalars256(5)))
    ct2[4, 100] ^= 1
    m1, s1 = P.decrypt_small(sk, cuda(ct2), -10, 1000)
    m2, s2 = P.decrypt_bsgs(sk, ctx, 20, cuda(ct2), -10, 1000)
    assert (m1.cpu() == m2.cpu()).all() and (s1.cpu() == s2.cpu()).all()
    assert list(s2.cpu().numpy()) == [0, 0, 0, 0, P.PCMM_ENOTONCURVE]


def test_pcmm_output_decrypts_with_bsgs():
    I = synth.make_instance(synth.CONFIGS["c64"], m=16, n=64, l=8, seed=33)
    sk, pk = P.keygen(33)
    ctx = P.enc_ctx(pk)
    ct = P.encrypt_ctx(ctx, cuda(I.B.reshape(-1).astype(np.int32)), cuda(I.r_be))
    out = P.pcmm(cuda(I.A), ct, 8, 4, False, P.CUSSEN)
    bctx = P.bsgs_ctx(12)
    m, st = P.decrypt_bsgs(sk, bctx, 12, out, 0, 64 * 15 * 255)
    assert (st.cpu().numpy() == 0).all()
    assert (m.cpu().numpy().reshape(16, 8) == I.A.astype(np.int64) @ I.B.astype(np.int64)).all()


# ------------------------------------------------------------------ NEXT-4: Paillier PC-MM
@pytest.mark.parametrize("nbits,shape,w", [(512, (9, 7, 5), 4), (1024, (6, 10, 3), 8), (3072, (8, 8, 8), 4),
                                           (2048, (5, 6, 4), 2)])
def test_paillier_every_output(nbits, shape, w):
    from oracle import paillier as pl
    m, nn, l = shape
    p, q = synth.paillier_primes(nbits, nbits // 2)
    n, g, lam, mu = pl.keygen(p, q)
    n2 = n * n
    assert n2.bit_length() in (nbits, nbits - 1)
    gen = synth.SplitMix64(nbits + w)
    A = gen.small(0, (1 << w) - 1, m * nn).reshape(m, nn).astype(np.uint8)
    A[0, :] = 0
    A[1, 0] = (1 << w) - 1
    A[2, :] = A[3, :]
    B = gen.small(0, 255, nn * l).reshape(nn, l)
    R = synth.paillier_random_units(nbits, n, nn * l)
    C = [[pl.encrypt(n, g, int(B[k, j]), R[k * l + j]) for j in range(l)] for k in range(nn)]
    exp = pl.pcmm_schoolbook(A, C, n2, w)
    ct = P.to_words([C[k][j] for k in range(nn) for j in range(l)], nbits // 32).cuda()
    for path in (P.SCHOOLBOOK, P.CUSSEN):
        out = P.from_words(P.paillier_mul(path, cuda(A), ct, l, w, n2))
        assert out == [exp[i][j] for i in range(m) for j in range(l)], path
    AB = A.astype(np.int64) @ B.astype(np.int64)
    assert pl.decrypt(n, lam, mu, out[0 * l + 1]) == AB[0, 1] == 0
    assert pl.decrypt(n, lam, mu, out[4 * l + 2]) == AB[4, 2]


def test_paillier_per_thread_kernels():
    # the per-thread Paillier kernels (used for large launches at 1024 / 2048 bits) on the same
    # every-output cases, in a subprocess with the warp-cooperative kernels switched off
    import os
    import subprocess
    import sys
    env = dict(os.environ, PCMM_PAILLIER_WARP="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", __file__,
                        "-k", "test_paillier_every_output"], env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_paillier_errors():
    p, q = synth.paillier_primes(512, 256)
    n2 = (p * q) ** 2
    A = np.ones((2, 2), dtype=np.uint8)
    ct = P.to_words([n2 - 1, 2, 3, n2 + 5 - n2], 16).cuda()
    ok = P.paillier_mul(P.CUSSEN, cuda(A), ct, 2, 4, n2)
    assert ok.shape == (4, 16)
    bad = P.to_words([n2 + 1, 2, 3, 4], 16).cuda()            # a value >= n^2
    with pytest.raises(P.PCMMError) as e:
        P.paillier_mul(P.CUSSEN, cuda(A), bad, 2, 4, n2)
    assert e.value.code == P.PCMM_ENOTONCURVE
    with pytest.raises(P.PCMMError) as e:
        P.paillier_mul(P.SCHOOLBOOK, cuda(np.full((2, 2), 16, dtype=np.uint8)), ct, 2, 4, n2)
    assert e.value.code == P.PCMM_EBOUND


def test_wide_full_grid_size_sampled():
    # the grid's 256^3 t = 16 run (tools/grid.py), in the launch configuration bench.py uses
    # (default 2 GiB table budget -> several k-chunks): sampled outputs vs the Eq. 5 closed form
    cfg = synth.Config("w16", 256, 256, 256, 16, False, 0, 255, 1616)
    I = synth.make_instance(cfg)
    sk, pk = P.keygen(cfg.seed)
    ctd = P.encrypt(pk, cuda(I.B.reshape(-1).astype(np.int32)), cuda(I.r_be))
    out = P.pcmm(cuda(I.A), ctd, 256, 16, False, path=P.CUSSEN).cpu().numpy()
    r = I.r_be.reshape(256, 256, 32)
    g = np.random.default_rng(16)
    for (i, j) in [(0, 0), (255, 255)] + [(int(g.integers(256)), int(g.integers(256))) for _ in range(6)]:
        assert out[i * 256 + j].tobytes() == oracle.closed_form(I.x, I.A[i], I.B[:, j], r[:, j]), (i, j)


def test_paillier_3072_64cube_sampled():
    # 64^3, t = 4, n^2 of 3072 bits, random residues mod n^2 as ciphertexts (any unit is the
    # encryption of some message): sampled outputs vs the oracle's definition prod_k c^a mod n^2
    from oracle import paillier as pl
    p, q = synth.paillier_primes(3072, 1536)
    n2 = (p * q) ** 2
    g = synth.SplitMix64(64)
    A = g.small(0, 15, 64 * 64).reshape(64, 64).astype(np.uint8)
    vals = [pow(int(v), 5, n2) for v in g.small(2, 2**62, 64 * 64)]
    ct = P.to_words(vals, 96).cuda()
    for path in (P.CUSSEN, P.SCHOOLBOOK):
        out = P.from_words(P.paillier_mul(path, cuda(A), ct, 64, 4, n2))
        for (i, j) in [(0, 0), (63, 63), (17, 5), (40, 33)]:
            C = [[vals[k * 64 + j]] for k in range(64)]
            assert out[i * 64 + j] == pl.pcmm_schoolbook(A[i:i + 1], C, n2, 4)[0][0], (path, i, j)


@pytest.mark.parametrize("t", [4, 12])
def test_vector_times_ciphertext_scalars(t):
    # NEXT-1's vector workload (Tables A7/A8): an n x 1 plaintext vector times a 1 x l row of ciphertexts
    _vector_case(37, 5, t)


@pytest.mark.parametrize("m,l,t", [(300, 3, 16), (1000, 1, 16), (700, 2, 12)])
def test_vector_long_tables_block_scan(m, l, t):
    # few tables with hundreds of entries: the wide path's one-CTA-per-table block-scan kernel
    # (runs of several entries per thread, a 128-wide scan of run totals)
    _vector_case(m, l, t)


def test_wide_block_scan_forced():
    # the block-scan table kernel on the every-output wide cases (PCMM_WIDE_SCAN=2 forces it)
    import os
    import subprocess
    import sys
    env = dict(os.environ, PCMM_WIDE_SCAN="2")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", __file__,
                        "-k", "test_wide_every_output or test_wide_chunked"], env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("mode", ["0", "2"])
def test_consecutive_table_kernels_forced(mode):
    # PCMM_TABLES_COZ=0: the XYZZ consecutive-column kernel (k_tables_fast + k_affine's XYZZ branch);
    # 2: the fused co-Z kernel (k_tables_coz) for every unsigned launch, also the small ones
    import os
    import subprocess
    import sys
    env = dict(os.environ, PCMM_TABLES_COZ=mode)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", __file__, "-k",
                        "test_ragged_shapes or test_tiny or test_c64_config or test_degenerate or "
                        "test_consecutive_column or test_all_identity or test_vector_times"],
                       env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("m,n,l,w,signed", [(64, 128, 128, 4, False), (48, 128, 128, 6, True), (40, 64, 64, 8, False)])
def test_general_fused_tables_every_output(m, n, l, w, signed):
    # launches of the size at which the default picks k_tables_gz (32,768 tables; 8,192 of 2^w >= 64
    # slots) but not k_tables_coz: every column, chain columns included, goes through the fused
    # general kernel (doubling steps T[2] = P + P, gaps, signed level sets); identity ciphertexts and
    # a repeated ciphertext in the inputs; every output against the oracle
    cfg = synth.Config("gz", m, n, l, w, signed, 0, 255, 500 + w)
    I = synth.make_instance(cfg)
    x = synth.keygen_secret(cfg.seed)
    ct = oracle.encrypt(ecref.mulG(x), I.B.reshape(-1), I.r_be).reshape(n, l, 128)
    ct[3, 2] = 0                                         # (inf, inf)
    ct[5, :4, :64] = 0                                   # C1 = inf
    ct[7] = ct[6]                                        # equal ciphertexts in consecutive k
    ct = np.ascontiguousarray(ct.reshape(n * l, 128))
    exp, _ = oracle.pcmm(oracle.CUSSEN, I.A, ct, l, w)
    assert (_gpu_pcmm(I.A, ct, l, w, signed, P.CUSSEN) == exp).all()


@pytest.mark.parametrize("mode", ["0", "2"])
def test_general_table_kernels_forced(mode):
    # PCMM_TABLES_GZ=2: the fused general-column kernel (k_tables_gz: XYZZ level-1 prefix sum with the
    # affine conversion, doubling steps, identity components) for every launch, also the small ones;
    # 0: k_tables / k_tables_x + k_affine everywhere (the default picks by launch size)
    import os
    import subprocess
    import sys
    env = dict(os.environ, PCMM_TABLES_GZ=mode)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", __file__, "-k",
                        "test_ragged_shapes or test_tiny or test_c64_config or test_degenerate or "
                        "test_consecutive_column or test_signed_chain or test_xyzz_level1 or test_all_identity or "
                        "test_extreme_values or test_vector_times or test_accumulator_exceptional"],
                       env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_rowperm_per_block_forced():
    # PCMM_ROWPERM_ALL=0: rows sorted inside each 128-row block (the path of m > 4096) on the every-output
    # cases with m > 64, incl. 256^3 and ML
    import os
    import subprocess
    import sys
    env = dict(os.environ, PCMM_ROWPERM_ALL="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", __file__, "-k",
                        "test_ragged_shapes or (test_full_size_cussen_every_output and not c512) or "
                        "test_extreme_values or test_signed_chain or test_byte_path_k_chunks"],
                       env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("mode", ["0", "1", "2"])
def test_accumulate_modes_forced(mode):
    # PCMM_ACC_MODE: 0 = k_accum (tables staged in shared memory; the default only for m <= 64),
    # 1 = k_accum_g (gather) for every w, 2 = k_rowperm + k_accum_g2 with the 4-group step
    # (default: 3, the pipelined step), on every-output cases incl. 256^3 (modes 0, 2) and the exceptional
    # accumulator cases
    import os
    import subprocess
    import sys
    env = dict(os.environ, PCMM_ACC_MODE=mode)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", __file__, "-k",
                        "test_ragged_shapes or test_accumulator_exceptional or test_degenerate or "
                        + ("" if mode == "1" else "(test_full_size_cussen_every_output and c256) or ") +
                        "test_signed_chain or test_general_fused or test_byte_path_k_chunks or test_extreme_values"],
                       env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_xyzz_schoolbook_forced():
    # the XYZZ schoolbook kernel (school.cu, PCMM_SCHOOL_XYZZ=1) on the every-output cases, including the
    # exceptional accumulator cases (equal and opposite terms) and identity ciphertexts
    import os
    import subprocess
    import sys
    env = dict(os.environ, PCMM_SCHOOL_XYZZ="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", __file__, "-k",
                        "test_ragged_shapes or test_tiny or test_c64_config or test_degenerate or "
                        "test_accumulator_exceptional or test_xyzz_level1 or test_extreme_values"],
                       env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_byte_path_k_chunks_forced():
    # a tiny table budget (PCMM_BYTE_BUDGET_MB=1) forces the byte path's k-chunking (tables built and
    # consumed chunk by chunk, each chunk's sums added into the running output) on the every-output cases
    import os
    import subprocess
    import sys
    env = dict(os.environ, PCMM_BYTE_BUDGET_MB="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", __file__, "-k",
                        "test_ragged_shapes or test_c64_config or test_degenerate or test_consecutive_column or "
                        "test_accumulator_exceptional or test_xyzz_level1"],
                       env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_c256_chunked_direct_every_output():
    # 256^3 w = 4 with a 100 MB table budget: k-chunks large enough that each chunk's accumulation fills the
    # GPU, so k_accum adds each chunk straight into the running output (no split-k, no k_reduce); every
    # output against the oracle
    import os
    import subprocess
    import sys
    env = dict(os.environ, PCMM_BYTE_BUDGET_MB="100")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", __file__, "-k",
                        "test_full_size_cussen_every_output and c256"],
                       env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "1 passed" in r.stdout, r.stdout[-500:]


def test_c512_w8_chunked_sampled():
    # 512^3 at w = 8 (tables of all k would take ~21 GB): the default 2 GiB budget chunks k;
    # sampled outputs vs the Eq. 5 closed form
    cfg = synth.Config("w8", 512, 512, 512, 8, False, 0, 255, 888)
    I = synth.make_instance(cfg)
    sk, pk = P.keygen(cfg.seed)
    ctd = P.encrypt(pk, cuda(I.B.reshape(-1).astype(np.int32)), cuda(I.r_be))
    assert P.workspace_bytes(512, 512, 512, 8, P.CUSSEN) <= 2 << 30
    out = P.pcmm(cuda(I.A), ctd, 512, 8, False, path=P.CUSSEN).cpu().numpy()
    r = I.r_be.reshape(512, 512, 32)
    g = np.random.default_rng(8)
    for (i, j) in [(0, 0), (511, 511), (0, 511)] + [(int(g.integers(512)), int(g.integers(512))) for _ in range(5)]:
        assert out[i * 512 + j].tobytes() == oracle.closed_form(I.x, I.A[i], I.B[:, j], r[:, j]), (i, j)


def test_checked_build():
    # the device bounds-check build (libpcmm_checked.so, PCMM_CHECKED=1: shared-memory staging and scans,
    # table slots, scratch entries, plan bitmaps, CTA-inverse layout, chain-column slots, the row
    # permutation) on the every-output cases incl. the signed chain columns, the fused general-column
    # kernel and the k-chunked byte path; a failed check traps the launch.  Stands in for compute-sanitizer memcheck, which the GPU pool does not run.
    import os
    import subprocess
    import sys
    env = dict(os.environ, PCMM_LIB_VARIANT="checked")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", __file__, "-k",
                        "(test_ragged_shapes or test_tiny or test_c64_config or test_degenerate or test_consecutive_column "
                        "or test_all_identity or test_accumulator_exceptional or test_xyzz_level1 or test_vector "
                        "or test_wide_every_output or test_wide_chunked or test_strassen_every or test_plan_matches "
                        "or test_extreme_values or test_byte_path_k_chunks or test_paillier_every "
                        "or test_signed_chain or test_general_fused "
                        "or test_full_size_comparison_paths_sampled or test_c512_w8_chunked_sampled "
                        "or test_full_size_gpu_encrypted_inputs_sampled or test_wide_full_grid_size_sampled) "
                        "and not test_checked_build"],
                       env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "PCMM_DCHECK failed" not in r.stdout


def test_byte_block_scan_forced():
    # the byte path's block-scan table kernel (k_tables_scan) forced on the every-output cases
    import os
    import subprocess
    import sys
    env = dict(os.environ, PCMM_TABLES_SCAN="2")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", __file__, "-k",
                        "test_ragged_shapes or test_tiny or test_c64_config or test_degenerate or "
                        "test_accumulator_exceptional or test_vector_times"],
                       env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def _vector_case(m, l, t):
    cfg = synth.Config("vec", m, 1, l, t, False, 0, 255, 900 + t + m)
    I = synth.make_instance(cfg)
    x = synth.keygen_secret(cfg.seed)
    ct = oracle.encrypt(ecref.mulG(x), I.B.reshape(-1), I.r_be)
    exp, _ = oracle.pcmm(oracle.CUSSEN, I.A, ct, l, t)
    for path in (P.CUSSEN, P.SCHOOLBOOK):
        assert (_gpu_pcmm(I.A, ct, l, t, False, path) == exp).all(), path


def test_step_is_cuda_graph_capturable():
    # the Cussen step (mul + normalize) is stream-ordered with no host synchronisation, so it can be
    # captured once into a CUDA graph and replayed (serving-style launch-overhead removal)
    I = synth.make_instance(synth.CONFIGS["c64"], m=32, n=48, l=16, seed=41)
    x = synth.keygen_secret(41)
    ct = cuda(oracle.encrypt(ecref.mulG(x), I.B.reshape(-1), I.r_be))
    A = cuda(I.A)
    ref = P.pcmm(A, ct, 16, 4, False, P.CUSSEN).cpu()
    ws = P.alloc_workspace(32, 48, 16, 4, P.CUSSEN)
    proj = torch.empty(P.proj_bytes(32 * 16), dtype=torch.uint8, device="cuda")
    out = torch.empty((32 * 16, 128), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):                       # warm-up outside capture (first-call attribute setup)
        P.mul_cussen(A, ct, 16, 4, False, 4, out_proj=proj, ws=ws)
        P.normalize(proj, 32 * 16, out=out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        P.mul_cussen(A, ct, 16, 4, False, 4, out_proj=proj, ws=ws)
        P.normalize(proj, 32 * 16, out=out)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out.cpu(), ref)
    P.status(ws)
