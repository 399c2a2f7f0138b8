"""Debug helper: the mixed consecutive-column test case, reporting mismatching outputs."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import oracle, synth
from tests import ecref
from paper_2504_14497_b200 import pcmm as P

w = int(sys.argv[1]) if len(sys.argv) > 1 else 2
m, n, l = 8, 256, 128
cfg = synth.Config("mixed", m, n, l, w, False, 0, 255, 77 + w)
I = synth.make_instance(cfg)
A = I.A.copy()
top = (1 << w) - 1
A[:, 0] = [(i % top) + 1 for i in range(m)]
A[:, 1] = 2
A[:, 2] = 0
A[:, 3] = [1, 3] * (m // 2)
A[:, 4] = [1, 2] * (m // 2)
x = synth.keygen_secret(cfg.seed)
ct = oracle.encrypt(ecref.mulG(x), I.B.reshape(-1), I.r_be).reshape(n, l, 128)
if len(sys.argv) > 2 and sys.argv[2] == "inf":
    ct[0, 5] = 0
    ct[4, :7, 64:] = 0
ct = np.ascontiguousarray(ct.reshape(n * l, 128))
exp, _ = oracle.pcmm(oracle.CUSSEN, A, ct, l, w)
out = P.pcmm(torch.from_numpy(A).cuda(), torch.from_numpy(ct).cuda(), l, w, False, path=P.CUSSEN).cpu().numpy()
bad = np.nonzero((out != exp).any(axis=1))[0]
print("w", w, "mismatches", len(bad), "of", out.shape[0], "first", [(int(b) // l, int(b) % l) for b in bad[:10]])
