"""NEXT-2 throughput on one GPU: encryption (ladder vs comb context) and decryption
(exact table vs BSGS) of the 256^3 workload's 65,536 ciphertexts / outputs.
Prints a markdown table.  Run on the GPU box."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2504_14497_b200 import pcmm as P  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


cfg = synth.CONFIGS["c256"]
I = synth.make_instance(cfg)
sk, pk = P.keygen(cfg.seed)
b = torch.from_numpy(I.B.reshape(-1).astype(np.int32)).cuda()
r = torch.from_numpy(I.r_be).cuda()
count = b.numel()
rows = ["| step | implementation | ms | items/s |", "|---|---|---|---|"]
t0 = time.time()
ctx = P.enc_ctx(pk)
torch.cuda.synchronize()
t_ctx = (time.time() - t0) * 1e3
ms_l = timed(lambda: P.encrypt(pk, b, r))
ms_c = timed(lambda: P.encrypt_ctx(ctx, b, r))
assert (P.encrypt(pk, b, r) == P.encrypt_ctx(ctx, b, r)).all()
rows.append(f"| encrypt 65,536 | two 256-bit 4-bit-window ECSMs (pcmm_encrypt) | {ms_l:.3f} | {count / ms_l * 1e3:,.0f} |")
rows.append(f"| encrypt 65,536 | comb context (pcmm_encrypt_ctx) | {ms_c:.3f} | {count / ms_c * 1e3:,.0f} |")
rows.append(f"| comb context build (once per key, wall) | pcmm_enc_ctx_init | {t_ctx:.1f} | |")
ct = P.encrypt_ctx(ctx, b, r)
out = P.pcmm(torch.from_numpy(I.A).cuda(), ct, cfg.l, cfg.w, False, P.CUSSEN)
hi = cfg.n * 15 * 255
ms_s = timed(lambda: P.decrypt_small(sk, out, 0, hi), reps=2)
for lb in (16, 20, 22):
    t0 = time.time()
    bctx = P.bsgs_ctx(lb)
    torch.cuda.synchronize()
    t_b = (time.time() - t0) * 1e3
    ms_b = timed(lambda: P.decrypt_bsgs(sk, bctx, lb, out, 0, hi), reps=2)
    m, st = P.decrypt_bsgs(sk, bctx, lb, out, 0, hi)
    exp = (I.A.astype(np.int64) @ I.B.astype(np.int64)).reshape(-1)
    assert (st.cpu().numpy() == 0).all() and (m.cpu().numpy() == exp).all()
    rows.append(f"| decrypt 65,536 outputs in [0, {hi}] | BSGS, s = 2^{lb} (table build {t_b:.1f} ms wall) | "
                f"{ms_b:.3f} | {count / ms_b * 1e3:,.0f} |")
rows.append(f"| decrypt 65,536 outputs in [0, {hi}] | BSGS with a per-call table (pcmm_decrypt_small, incl. build) | "
            f"{ms_s:.3f} | {count / ms_s * 1e3:,.0f} |")
print("\n".join(rows))
