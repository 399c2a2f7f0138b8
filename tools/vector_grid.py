"""The paper's vector x ciphertext-scalar workload on one B200 (NEXT-1; Tables A7/A8,
PAPER.md:886-949): a plaintext vector a of length n times Enc(b), i.e. the PC-MM of an
n x 1 matrix by a 1 x l row of ciphertexts.  Two numbers per (t, n): one vector times one
ciphertext (latency: a single table of up to 2^t - 1 entries is built by one thread), and
one vector times 1024 ciphertexts (throughput per vector-scalar product).  Cussen vs
schoolbook; the RPi 5 numbers of Table A7 beside them.  Prints a markdown table."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2504_14497_b200 import pcmm as P  # noqa: E402

A7 = {4: [(929.364, 250.138), (1853.07, 261.694), (3700.836, 296.418), (7400.958, 318.018), (14837.766, 335.144),
          (29592.7, 353.944), (59153.174, 399.094)],
      8: [(1194.568, 723.292), (2386.114, 588.268), (4765.696, 551.734), (9526.752, 615.192), (19047.554, 765.108),
          (38086.59, 1071.834), (76327.824, 1473.63)],
      12: [(1460.39, 1472.122), (2917.274, 1905.484), (5830.14, 1563.06), (11652.792, 1458.826),
           (23298.534, 1583.76), (46590.522, 1978.638), (93181.214, 3044.194)],
      16: [(1729.608, 1814.146), (3445.01, 3502.018), (6884.118, 4633.108), (13775.728, 3949.804),
           (27523.884, 3692.986), (55047.72, 4172.836), (110086.372, 5272.712)]}   # microseconds
NS = [8, 16, 32, 64, 128, 256, 512]


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3          # microseconds


sk, pk = P.keygen(7)
rows = ["| t | n | 1 vector x 1 ct: Cussen / schoolbook us | 1 vector x 1024 cts: Cussen / schoolbook us per product "
        "| RPi5 Cussen / schoolbook us (A7) |", "|---|---|---|---|---|"]
for t in (4, 8, 12, 16):
    for q, n in enumerate(NS):
        g = synth.SplitMix64(100 * t + n)
        a = g.small(0, (1 << t) - 1, n).reshape(n, 1).astype(np.uint8 if t <= 8 else np.int32)
        A = torch.from_numpy(a).cuda()
        res = []
        for l in (1, 1024):
            b = torch.from_numpy(g.small(0, 255, l).astype(np.int32)).cuda()
            r = torch.from_numpy(synth.scalars_to_be_bytes(g.scalars256(l))).cuda()
            ct = P.encrypt(pk, b, r)
            for path in (P.CUSSEN, P.SCHOOLBOOK):
                us = timed(lambda: P.pcmm(A, ct, l, t, False, path=path, check=False), 5)
                res.append(us / l)
        rows.append(f"| {t} | {n} | {res[0]:.1f} / {res[1]:.1f} | {res[2]:.3f} / {res[3]:.3f} | "
                    f"{A7[t][q][1]} / {A7[t][q][0]} |")
        print(rows[-1], file=sys.stderr, flush=True)
print("\n".join(rows))
