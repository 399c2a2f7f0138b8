"""The oracle's paper-model cost functions reproduce the paper's deterministic
tables exactly: A3/A4 (plaintext counts), A5/A6 (equivalent
point additions), using the printed A1/A2 cells for the Cussen columns."""
import os

import numpy as np
import pytest

import oracle
from tests.test_oracle_cussen import A1, A2, NS

HERE = os.path.dirname(os.path.abspath(__file__))


def _golden():
    a5, a6 = {}, {}
    with open(os.path.join(HERE, "golden", "tables_a5_a6.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            p = line.split()
            t, n = int(p[1]), int(p[2])
            vals = [int(v) for v in p[3:]]
            (a5 if p[0] == "A5" else a6)[(t, n)] = vals
    return a5, a6


A5, A6 = _golden()


def strassen_mults(n):
    return 7 ** int(np.log2(n))


def strassen_ct_adds(n):            # T(n) = 7 T(n/2) + 13 (n/2)^2, T(1) = 0
    return 0 if n == 1 else 7 * strassen_ct_adds(n // 2) + 13 * (n // 2) ** 2


def test_table_a3_a4_closed_forms():
    # A3 and A4 cells for n = 8 and 512, every column
    a3 = {8: [512, 343, 64, 256, 512, 512], 512: [134217728, 40353607, 262144, 262144, 524288, 1835008]}
    a4 = {8: [448, 1674, 1152, 1792, 1984, 1984], 512: [133955584, 240548778, 138412032, 192937984, 271056896,
                                                        338690048]}
    for n in (8, 512):
        ni = NS.index(n)
        assert a3[n][0] == n ** 3 and a3[n][1] == strassen_mults(n)
        assert a3[n][2:] == [n * n * A1[t][ni] for t in (4, 8, 12, 16)]
        assert a4[n][0] == n * n * (n - 1)
        assert a4[n][2:] == [n * n * A2[t][ni] + n * n * (n - 1) for t in (4, 8, 12, 16)]


@pytest.mark.parametrize("t", [4, 8, 12, 16])
def test_table_a5_a6_exact(t):
    for ni, n in enumerate(NS):
        school5, prop5 = A5[(t, n)]
        assert school5 == 4 * n * t                                   # 2n ECSMs of 2t each
        assert prop5 == 4 * t * A1[t][ni] + 2 * A2[t][ni]             # 2 n_N ECSMs + 2 sum n_w adds
        school6, strassen6, prop6 = A6[(t, n)]
        assert school6 == oracle.paper_model_equiv_adds_schoolbook(t, n, n, n)
        assert strassen6 == 4 * t * strassen_mults(n) + 2 * strassen_ct_adds(n)
        # the proposed column: every column k of A with (n_N, sum n_w) = the A1/A2 cells
        lev = [[A2[t][ni], 0, 0, A1[t][ni]]] * n                      # sum(lev[:3]) = A2, lev[3] = A1
        assert prop6 == oracle.paper_model_equiv_adds_cussen(lev, t, n, n, n)


def test_oracle_run_counts_follow_model():
    # Counters of a real oracle run obey the schoolbook law of P:232-233: m n l plaintext-
    # ciphertext multiplications = 2 m n l ladders of width t.
    import synth
    I = synth.make_instance(synth.CONFIGS["tiny"])
    H = oracle.pubkey(I.x)
    ct = oracle.encrypt(H, I.B.reshape(-1), I.r_be)
    _, (adds, dbls, ecsm, bits) = oracle.pcmm(oracle.SCHOOLBOOK, I.A, ct, 8, 2)
    assert ecsm == 2 * 8 * 8 * 8 and bits == 2 * 2 * 8 * 8 * 8
    # Cussen: ladders only for the compressed values, 2 per (k, j)
    _, (adds_c, dbls_c, ecsm_c, bits_c) = oracle.pcmm(oracle.CUSSEN, I.A, ct, 8, 2)
    n_mults = sum(oracle.cussen_counts(I.A[:, k].astype(np.int64))[0] for k in range(8))
    assert ecsm_c == 2 * 8 * n_mults


def test_bench_counts_match_oracle_compression():
    # bench.py's host-side work counts (the roofline numerator's table ops and the paper-model
    # equivalent additions it reports) agree with the oracle's Alg. 2 compression of every column
    import bench
    import synth
    for name in ("tiny", "c64", "ml"):
        cfg = synth.CONFIGS[name]
        I = synth.make_instance(cfg) if name != "ml" else synth.make_instance(cfg, m=32, n=48, l=5)
        m, n = I.A.shape
        l = I.B.shape[1]
        levels = [oracle.cussen_counts(I.A[:, k])[3] for k in range(n)]
        assert bench.paper_model_adds(I.A, l, cfg.w) == oracle.paper_model_equiv_adds_cussen(levels, cfg.w, m, n, l)
        # executed prefix additions: sum over levels w < N of (|s^(w)| - 1), per (k, j, c)
        _, tbl_adds, _ = bench.algorithmic_counts(I.A, l, cfg.w)
        exec_prefix = 2 * l * sum(max(lv[w] - 1, 0) for lv in levels for w in range(3))
        assert tbl_adds >= exec_prefix
