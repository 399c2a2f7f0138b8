"""Per-kernel times of the Paillier PC-MM (profile hooks) for a few sizes: python tools/paillier_prof.py [nbits]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2504_14497_b200 import pcmm as P  # noqa: E402

NB = int(sys.argv[1]) if len(sys.argv) > 1 else 3072
p, q = synth.paillier_primes(NB, NB // 2)
n2 = (p * q) ** 2
L = NB // 32
for t, nn in ((4, 8), (4, 64), (4, 256)):
    g = synth.SplitMix64(1000 * t + nn)
    A = torch.from_numpy(g.small(0, (1 << t) - 1, nn * nn).reshape(nn, nn).astype(np.uint8)).cuda()
    vals = [pow(int(v) % n2, 3, n2) for v in g.small(1, 2**62, nn * nn)]
    ct = P.to_words(vals, L).cuda()
    for path in (P.CUSSEN, P.SCHOOLBOOK):
        P.paillier_mul(path, A, ct, nn, t, n2, check=False)
        torch.cuda.synchronize()
        P.profile_enable(True)
        P.paillier_mul(path, A, ct, nn, t, n2, check=False)
        torch.cuda.synchronize()
        recs = P.profile_read()
        P.profile_enable(False)
        print(t, nn, "cussen" if path == P.CUSSEN else "school", {k: round(v, 3) for k, v in recs})
