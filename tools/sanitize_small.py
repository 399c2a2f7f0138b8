"""Small end-to-end runs of every kernel family for compute-sanitizer (one tool per invocation).

Covers, on shapes that take each launch path (api.cu / kernels.cu dispatch):
  k_import, k_plan, k_tables (unsigned / signed), k_tables_fast + k_affine (XYZZ branch),
  k_tables_x (2^w >= 128 slots), k_tables_scan (few long tables), k_accum<S> for S = 4, 8, 16
  (shared-memory staging, several k-chunks, split-k) + k_reduce, k_accum_g (w > 4),
  k_normalize, k_school, the wide path (k_plan_wide, k_tables_wide, k_tables_wide_scan,
  k_accum_gw), Strassen, comb encryption, BSGS and table decryption, Paillier (warp and per-thread).
Every run is also checked Cussen == schoolbook (bytes), so a silent corruption fails here too.

  compute-sanitizer --tool memcheck python tools/sanitize_small.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2504_14497_b200 import pcmm as P  # noqa: E402


def run(name, m, n, l, w, signed, seed, wide=False, strassen=False):
    cfg = synth.Config(name, m, n, l, w, signed, 0, 255, seed)
    I = synth.make_instance(cfg)
    sk, pk = P.keygen(seed)
    ct = P.encrypt(pk, torch.from_numpy(I.B.reshape(-1).astype(np.int32)).cuda(), torch.from_numpy(I.r_be).cuda())
    A = torch.from_numpy(I.A).cuda()
    c1 = P.pcmm(A, ct, l, w, signed, path=P.CUSSEN)
    c2 = P.pcmm(A, ct, l, w, signed, path=P.SCHOOLBOOK)
    assert torch.equal(c1, c2), name
    if strassen:
        c3 = P.pcmm(A, ct, l, w, signed, path=P.STRASSEN, iters=4)
        assert torch.equal(c1, c3), name
    torch.cuda.synchronize()
    print(name, (m, n, l, w, signed), "ok", flush=True)
    return sk, pk, c1


only = set(sys.argv[1:])
cases = [
    ("tiny", 8, 8, 8, 2, False, 0, False, True),
    ("k_tables+accum16", 40, 70, 33, 4, False, 1, False, False),
    ("signed+splitk", 130, 512, 3, 4, True, 4, False, False),        # k_tables<true>, many k-chunks, split-k + k_reduce
    ("tables_fast+affine", 8, 256, 128, 4, False, 5, False, False),   # 2 n l >= 65536: k_tables_fast, XYZZ k_affine
    ("accum_S4", 70, 96, 5, 2, False, 6, False, False),               # k_accum<4>
    ("accum_S8", 33, 80, 4, 3, True, 7, False, False),                # k_accum<8>
    ("accum_g", 20, 24, 6, 6, False, 8, False, False),                # w > 4: k_accum_g
    ("tables_x", 40, 16, 12, 8, True, 9, False, False),               # 2^w >= 128 slots: k_tables_x
    ("tables_scan", 300, 1, 1, 8, False, 10, False, False),           # few long tables: k_tables_scan
    ("wide12", 20, 24, 6, 12, False, 11, True, False),                # wide path
    ("wide_scan16", 300, 1, 2, 16, False, 12, True, False),           # k_tables_wide_scan
    ("strassen", 16, 16, 16, 4, False, 13, False, True),
]
for c in cases:
    if only and c[0] not in only:
        continue
    sk, pk, out = run(*c[:7], wide=c[7], strassen=c[8])
    if c[0] == "tiny":
        mm, st = P.decrypt_small(sk, out, 0, 8 * 3 * 255)        # B in [0, 255] here
        assert int(st.abs().sum()) == 0
        ctx = P.enc_ctx(pk)
        g = synth.SplitMix64(5)
        b = torch.from_numpy(g.small(-1000, 1000, 64).astype(np.int32)).cuda()
        r = torch.from_numpy(synth.scalars_to_be_bytes(g.scalars256(64))).cuda()
        e1 = P.encrypt_ctx(ctx, b, r)
        assert torch.equal(e1, P.encrypt(pk, b, r))
        bctx = P.bsgs_ctx(8)
        mb, sb = P.decrypt_bsgs(sk, bctx, 8, e1, -1000, 1000)
        assert int(sb.abs().sum()) == 0 and torch.equal(mb.cpu(), b.cpu().long())
        print("next2 ok", flush=True)
if not only or "paillier" in only:
    # NEXT-4: warp-cooperative (3072-bit) and per-thread (1024-bit, PCMM_PAILLIER_WARP=0 in the env) kernels;
    # random units as ciphertexts (the arithmetic does not depend on what they encrypt); Cussen == schoolbook
    for nbits, (m, nn, l), w in ((3072, (4, 6, 3), 4), (1024, (6, 10, 3), 8)):
        p_, q_ = synth.paillier_primes(nbits, nbits // 2)
        n = p_ * q_
        gen = synth.SplitMix64(nbits + w)
        A = torch.from_numpy(gen.small(0, (1 << w) - 1, m * nn).reshape(m, nn).astype(np.uint8)).cuda()
        R = synth.paillier_random_units(nbits, n, nn * l)
        ct = P.to_words([x * x % (n * n) for x in R], nbits // 32).cuda()
        o1 = P.from_words(P.paillier_mul(P.CUSSEN, A, ct, l, w, n * n))
        o2 = P.from_words(P.paillier_mul(P.SCHOOLBOOK, A, ct, l, w, n * n))
        assert o1 == o2, nbits
        print("paillier", nbits, "ok", flush=True)
torch.cuda.synchronize()
print("all ok")
