"""Small end-to-end runs of every kernel for compute-sanitizer (one tool per invocation)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2504_14497_b200 import pcmm as P  # noqa: E402

for name, shape in (("tiny", None), ("c64", (40, 70, 33)), ("ml", (20, 64, 9)), ("c64", (8, 256, 128))):
    cfg = synth.CONFIGS[name]
    I = synth.make_instance(cfg) if shape is None else synth.make_instance(cfg, m=shape[0], n=shape[1], l=shape[2])
    m, n, l = I.A.shape[0], I.A.shape[1], I.B.shape[1]
    sk, pk = P.keygen(cfg.seed)
    ct = P.encrypt(pk, torch.from_numpy(I.B.reshape(-1).astype(np.int32)).cuda(), torch.from_numpy(I.r_be).cuda())
    A = torch.from_numpy(I.A).cuda()
    c1 = P.pcmm(A, ct, l, cfg.w, cfg.signed, path=P.CUSSEN)
    c2 = P.pcmm(A, ct, l, cfg.w, cfg.signed, path=P.SCHOOLBOOK)
    assert torch.equal(c1, c2)
    if name == "tiny":
        mm, st = P.decrypt_small(sk, c1, 0, 72)
        assert int(st.abs().sum()) == 0
    torch.cuda.synchronize()
    print(name, "ok")
