"""Latency of one field inversion per lane (test-field op 3 = fe_inv, op 7 = Fermat) and of a plain
product (op 2), one warp, min over repetitions: python tools/inv_latency.py.  Run on the GPU box."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_14497_b200 import pcmm as P  # noqa: E402

rng = np.random.default_rng(1)
A = torch.from_numpy(rng.integers(0, 255, size=(32, 32), dtype=np.uint8)).cuda()
A[:, 0] = 0x3f
B = A.clone()
for op, name in ((2, "fe_mul"), (3, "fe_inv (default)"), (7, "fe_inv_fermat")):
    for _ in range(3):
        P.test_field(op, A, B)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(50):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        P.test_field(op, A, B)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    print(f"{name:20s} one warp, one call: {best * 1e3:.1f} us (incl. launch)")
