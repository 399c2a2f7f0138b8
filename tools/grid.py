"""The paper's PC-MM grid on one B200 (NEXT-1): square n x n x n, t = w in {4, 8, 12, 16}
(int8 plaintexts for t <= 8, the int32 wide path above), Cussen vs schoolbook vs Strassen, next to the paper's Raspberry Pi 5 numbers
(Table A9; speedups Table A10).
Writes a markdown table to stdout.  Run on the GPU box."""
import json
import subprocess
import sys

# Table A9: (t, n) -> (Cussen s, schoolbook s) on RPi 5
A9 = {(4, 8): (0.02, 0.06), (4, 16): (0.09, 0.49), (4, 32): (0.43, 3.93), (4, 64): (2.46, 31.43),
      (4, 128): (14.31, 251.74), (4, 256): (95.5, 2017.64), (4, 512): (687.85, 16139.04),
      (8, 8): (0.05, 0.08), (8, 16): (0.18, 0.63), (8, 32): (0.70, 5.02), (8, 64): (3.65, 40.13),
      (8, 128): (20.96, 321.82), (8, 256): (139.56, 2571.89), (8, 512): (932.97, 20577.63),
      (12, 8): (0.1, 0.1), (12, 16): (0.5, 0.76), (12, 32): (1.71, 6.11), (12, 64): (7.13, 48.92),
      (12, 128): (34.53, 391.16), (12, 256): (198.54, 3134.81), (12, 512): (1305.7, 25079.63),
      (16, 8): (0.12, 0.11), (16, 16): (0.91, 0.9), (16, 32): (4.93, 7.19), (16, 64): (17.14, 57.61),
      (16, 128): (69.5, 461.59), (16, 256): (334.51, 3687.85), (16, 512): (1862.09, 29503.38)}

rows = ["| t | n | GPU Cussen ms | GPU schoolbook ms | GPU Strassen ms | speedup vs schoolbook | vs Strassen "
        "| RPi5 Cussen s | RPi5 vs schoolbook | RPi5 vs Strassen |",
        "|---|---|---|---|---|---|---|---|---|---|"]
A9S = {(4, 8): 0.05, (4, 16): 0.4, (4, 32): 2.95, (4, 64): 21.73, (4, 128): 158.82, (4, 256): 1161.86,
       (4, 512): 8480.31, (8, 8): 0.07, (8, 16): 0.48, (8, 32): 3.51, (8, 64): 25.66, (8, 128): 186.59,
       (8, 256): 1355.63, (8, 512): 9824.45, (12, 8): 0.08, (12, 16): 0.56, (12, 32): 4.07, (12, 64): 29.52,
       (12, 128): 213.63, (12, 256): 1544.58, (12, 512): 11292.73, (16, 8): 0.09, (16, 16): 0.64,
       (16, 32): 4.63, (16, 64): 33.43, (16, 128): 241.41, (16, 256): 1759.8,
       (16, 512): 12489.93}   # Table A9 Strassen column
TS = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [4, 8, 12, 16]
NS = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [8, 16, 32, 64, 128, 256, 512]
for t in TS:
    for n in NS:
        steps = "5" if n >= 256 else "10"
        leaf = "32"   # deeper recursion leaves tiny, under-filled leaf blocks (measured slower)
        out = subprocess.run([sys.executable, "bench.py", "--custom", f"{n},{n},{n},{t}", "--steps", steps,
                              "--warmup", "3", "--no-cpu-baseline", "--leaf", leaf], capture_output=True, text=True)
        try:
            d = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception:
            rows.append(f"| {t} | {n} | error | | | | | |")
            continue
        cu, sb, sv = d["ms_per_step"], d["schoolbook"]["ms_per_step"], d["strassen"]["ms_per_step"]
        pc, ps = A9[(t, n)]
        pst = A9S[(t, n)]
        rows.append(f"| {t} | {n} | {cu:.3f} | {sb:.3f} | {sv:.3f} | {sb / cu:.2f}x | {sv / cu:.2f}x | {pc} | "
                    f"{ps / pc:.2f}x | {pst / pc:.2f}x |")
        print(rows[-1], file=sys.stderr, flush=True)
print("\n".join(rows))
