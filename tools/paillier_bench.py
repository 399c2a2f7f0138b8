"""NEXT-4 timing on one GPU: Paillier PC-MM, n^2 of 3072 bits (n of 1536 bits),
square n x n x n, t in {4, 8}: Cussen vs schoolbook (the paper predicts speedups
"quite similar" to EC-ElGamal's, but never measures them).
Ciphertexts are random residues mod n^2 (the PC-MM arithmetic does not depend on
the plaintexts they encrypt).  Prints a markdown table.  Run on the GPU box."""
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
rows = [f"| t | n | GPU Cussen ms | GPU schoolbook ms | speedup | Cussen mod-mults/s |", "|---|---|---|---|---|---|"]
for t in (4, 8):
    for nn in (8, 16, 32, 64, 128, 256):
        g = synth.SplitMix64(1000 * t + nn)
        A = torch.from_numpy(g.small(0, (1 << t) - 1, nn * nn).reshape(nn, nn).astype(np.uint8)).cuda()
        vals = [int(v) % n2 for v in g.small(1, 2**62, nn * nn)]
        vals = [pow(v, 3, n2) for v in vals]
        ct = P.to_words(vals, L).cuda()

        def run(path):
            P.paillier_mul(path, A, ct, nn, t, n2, check=False)

        res = {}
        for path in (P.CUSSEN, P.SCHOOLBOOK):
            run(path)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 3 if nn >= 64 else 5
            s.record()
            for _ in range(reps):
                run(path)
            e.record()
            torch.cuda.synchronize()
            res[path] = s.elapsed_time(e) / reps
        a = A.cpu().numpy()
        nnz = int((a != 0).sum())
        mults = nnz * nn + nn * nn * 2 ** t          # accumulate + table products (upper bound)
        rows.append(f"| {t} | {nn} | {res[P.CUSSEN]:.3f} | {res[P.SCHOOLBOOK]:.3f} | "
                    f"{res[P.SCHOOLBOOK] / res[P.CUSSEN]:.2f}x | {mults / res[P.CUSSEN] * 1e3:,.0f} |")
        print(rows[-1], file=sys.stderr, flush=True)
print("\n".join(rows))
