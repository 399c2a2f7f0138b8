"""fp_mul / fe_add throughput probe (k_bench_fp_mul): G ops/s per variant."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2504_14497_b200 import pcmm as P

for v, name in ((0, "fe_mul (default)"), (3, "fe_mul other prod"), (1, "fe_mul_portable"), (2, "fe_add")):
    for blocks in (148 * 4, 148 * 8):
        P.bench_fp_mul(v, blocks, 128, 16)
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); P.bench_fp_mul(v, blocks, 128, 2000); e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e); n = blocks * 128 * 2000 * 4
        print(f"{name:18s} blocks {blocks:5d}  {n / ms / 1e6:8.1f} G/s")
