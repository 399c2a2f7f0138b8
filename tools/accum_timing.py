"""Per-kernel times of pcmm_mul_cussen on the c256 shape with arbitrary (not necessarily on-curve)
ciphertext bytes -- for measurement-only builds whose arithmetic is deliberately wrong (e.g.
PCMM_REDC_FAKE), where the encryption and status checks of bench.py would fail.  Run on the GPU box."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2504_14497_b200 import pcmm as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c256"
cfg = synth.CONFIGS[name]
I = synth.make_instance(cfg)
g = np.random.default_rng(5)
ct = g.integers(0, 256, size=(cfg.n * cfg.l, 128), dtype=np.uint8)
ct[:, 0] = 0x7f
ct[:, 32] = 0x7f
ct[:, 64] = 0x7f
ct[:, 96] = 0x7f
A = torch.from_numpy(I.A).cuda()
ctd = torch.from_numpy(ct).cuda()
ws = P.alloc_workspace(cfg.m, cfg.n, cfg.l, cfg.w, P.CUSSEN)
out = torch.empty(P.proj_bytes(cfg.m * cfg.l), dtype=torch.uint8, device="cuda")
for _ in range(3):
    P.mul_cussen(A, ctd, cfg.l, cfg.w, cfg.signed, out_proj=out, ws=ws)
torch.cuda.synchronize()
P.profile_enable(True)
reps = 10
for _ in range(reps):
    P.mul_cussen(A, ctd, cfg.l, cfg.w, cfg.signed, out_proj=out, ws=ws)
torch.cuda.synchronize()
recs = P.profile_read()
P.profile_enable(False)
tot = {}
for n_, ms in recs:
    tot[n_] = tot.get(n_, 0.0) + ms / reps
print(name, {k: round(v, 3) for k, v in tot.items()})
