#!/usr/bin/env python3
"""bench.py -- PC-MM C = A . Enc(B) on B200 (the driver's benchmark contract).

One "step" = one pass of the whole hot path over one
batch: pcmm_mul_cussen (import, compression plan, tables, shared-memory gather +
accumulate, split-k reduce) + pcmm_normalize (batch inversion to canonical bytes),
inputs already resident in HBM.  Workload at N=1: the headline 256x256x256, w=4
configuration (BASELINE.json configs[2], north_star's 50%-of-roofline target).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c256] [--path cussen|schoolbook]
  python bench.py --impl reference ...     # the CPU oracle (oracle/) as the reference arm

value = output ciphertexts (entries) per second, whole job (all ranks).
Timing: CUDA events on the launching stream per step, L2 flushed (256 MiB memset)
before every timed step outside the event pair, barrier + synchronize around the
timed region, max over ranks.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "encrypted output entries/s and EC point-adds/s; % of INT32-IMAD fp_mul roofline"
UNIT = "entries/s"
# Roofline denominator: 32x32->64 products / clk / SM on the
# IMAD pipe (IMAD.WIDE.U32 issues at half the IMAD rate; K11 probe, profiles/k11_imad.txt)
P_PROD = 32.0
LIMB_PRODUCTS_PER_FPMUL = 64.0
FPMUL_PER_ADD = 14          # RCB16 Alg. 4: 12M + 2 m_b (table build)
# k_accum: XYZZ + affine mixed addition (madd-2008-s) 8M + 2S; the two squares of
# the hot loop (P^2, R^2) run through the 36-product squaring:
# 8 products + 2 x 36/64 = 9.125 fp_mul-equivalents of IMAD work per addition
FPMUL_PER_ACC_ADD = 8 + 2 * 36 / 64
FPMUL_PER_AFFINE = 6        # k_affine: 5 products per table entry + the warp-shared inversion (amortised)
FPMUL_PER_DBL = 13          # RCB16 Alg. 6: 8M + 3S + 2 m_b
FPMUL_PER_NORM = 6          # batch inversion + x, y + from-Montgomery (amortised)


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def workload_config(cfg, path: str, world: int) -> dict:
    """The `config` object of the JSON line (shared by both arms)."""
    return {"workload": f"{cfg.name}: PC-MM {cfg.m}x{cfg.n} by {cfg.n}x{cfg.l}, w={cfg.w}"
                        f"{' signed' if cfg.signed else ''}, B in [{cfg.b_lo},{cfg.b_hi}], P-256 EC-ElGamal, "
                        f"seed {cfg.seed}",
            "m": cfg.m, "n": cfg.n, "l": cfg.l, "w": cfg.w, "path": path, "iters": 4,
            "parallelism": f"independent problem per GPU x{world} (no data-path collective)",
            "l2": "flushed (256 MiB memset) before every timed step, outside the events"}


def rank_instance_seed(cfg, rank: int) -> int:
    """Weak scaling: every rank runs its own independent problem of the same shape
    (no data-path exchange); rank r uses seed cfg.seed + 1000 r."""
    return cfg.seed + 1000 * rank


def reduce_max(value: float, dist, device) -> float:
    """Max over ranks (the slowest rank defines the step time)."""
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def algorithmic_counts(A: np.ndarray, l: int, w: int):
    """Algorithmic work of the Cussen path fixed by the input:
    useful accumulate adds (terms with a_ik != 0; n_i - 1 adds per output and
    component), table-build ops (prefix adds of every level + binary-ECSM ops of
    the last level), normalisation points.  Counted from the compression of A."""
    m, n = A.shape
    nnz = (A != 0).sum(axis=1)
    acc_adds = 2 * l * int(np.maximum(nnz - 1, 0).sum())
    tbl_adds = 0
    tbl_dbls = 0
    for k in range(n):
        col = A[:, k].astype(np.int64)
        v = col
        sizes, last = [], None
        for lev in range(4):
            s = np.unique(v)
            s = s[s != 0]
            sizes.append(len(s))
            last = s
            if lev < 3:
                v = np.diff(np.concatenate([[0], s]))
        tbl_adds += sum(max(x - 1, 0) for x in sizes[:3])
        for val in last:
            a = abs(int(val))
            if a > 1:
                tbl_dbls += a.bit_length() - 1
                tbl_adds += bin(a).count("1") - 1
    tbl_adds *= 2 * l
    tbl_dbls *= 2 * l
    return acc_adds, tbl_adds, tbl_dbls


def paper_model_adds(A: np.ndarray, l: int, w: int) -> int:
    """The paper's cost model for the Cussen run (SURVEY.md §8(c) counts; Table A6 form):
    per column k, l x (4 t |s^(N)_k| + 2 sum_{w<N} |s^(w)_k|) equivalent point additions (an ECSM of width
    t = w is t additions + t doublings per component) plus the dense accumulation 2 m l (n - 1)."""
    m, n = A.shape
    tot = 2 * m * l * (n - 1)
    for k in range(n):
        v = A[:, k].astype(np.int64)
        sizes = []
        for lev in range(4):
            s = np.unique(v)
            s = s[s != 0]
            sizes.append(len(s))
            if lev < 3:
                v = np.diff(np.concatenate([[0], s]))
        tot += l * (4 * w * sizes[3] + 2 * sum(sizes[:3]))
    return tot


def table_entries(A: np.ndarray, l: int) -> int:
    """Non-identity table entries (distinct nonzero values per column x 2 l)."""
    return 2 * l * sum(len(np.setdiff1d(np.unique(A[:, k]), [0])) for k in range(A.shape[1]))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            try:
                pw.append(float(f[2]))
            except ValueError:
                pass
            for nm, val in zip(names, f[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s in sm if mx and s > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_median": statistics.median(pw) if pw else None}


def oracle_baseline(cfg, l_sample: int, path: str):
    """The CPU oracle (oracle/, as it stands) on a bounded sample of the workload:
    all m rows, all n inner indices, the first `l_sample` output columns."""
    import oracle
    I = synth.make_instance(cfg, l=l_sample)
    threads = os.cpu_count() or 1
    pk = oracle.pubkey(I.x)
    ct = oracle.encrypt(pk, I.B.reshape(-1), I.r_be)
    t0 = time.perf_counter()
    oracle.pcmm(oracle.CUSSEN if path == "cussen" else oracle.SCHOOLBOOK, I.A, ct, l_sample, cfg.w,
                threads=threads)
    dt = time.perf_counter() - t0
    return {"value": cfg.m * l_sample / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{cfg.name}: all {cfg.m} rows x {cfg.n} k, first {l_sample} of {cfg.l} output columns "
                      f"({cfg.m * l_sample} entries, {path} path, {dt:.2f} s wall on {threads} threads)"}


def run_reference(args, cfg, rank):
    if rank != 0:
        return
    l_sample = args.ref_cols
    vals = []
    for _ in range(args.warmup and 1):
        oracle_baseline(cfg, max(1, l_sample // 8), args.path)
    for _ in range(args.steps):
        vals.append(oracle_baseline(cfg, l_sample, args.path))
    v = statistics.median([x["value"] for x in vals])
    cb = dict(vals[-1])
    cb["value"] = v
    ms = cfg.m * cfg.l / v * 1e3
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": dict(workload_config(cfg, args.path, max(1, args.gpus)),
                       note="oracle on host cores; each step a bounded sample (first --ref-cols output columns); "
                            "ms_per_step extrapolated to the full workload"),
        "cpu_baseline": cb, "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c256", choices=list(synth.CONFIGS))
    ap.add_argument("--path", default="cussen", choices=["cussen", "schoolbook", "strassen"])
    ap.add_argument("--leaf", type=int, default=32, help="Strassen recursion leaf block size")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-cols", type=int, default=48, help="output columns in the oracle's bounded sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-schoolbook", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="time the step as eager launches instead of one CUDA-graph replay per step")
    ap.add_argument("--custom", default=None, help="ad-hoc workload m,n,l,w[,signed] (A and B ranges from w / 8 bits)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    cfg = synth.CONFIGS[args.config]
    if args.custom:
        f = [int(x) for x in args.custom.split(",")]
        m_, n_, l_, w_ = f[:4]
        sg = bool(f[4]) if len(f) > 4 else False
        cfg = synth.Config(f"custom{m_}x{n_}x{l_}w{w_}{'s' if sg else ''}", m_, n_, l_, w_, sg, 0, 255, 7)
    if args.impl == "reference":
        return run_reference(args, cfg, rank)

    import torch
    from paper_2504_14497_b200 import pcmm as P

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    # ---- inputs (seeded, synthetic; encrypted on the GPU, outside any timing) ----
    seed = rank_instance_seed(cfg, rank)
    I = synth.make_instance(cfg, seed=seed)
    sk, pk = P.keygen(seed)
    A_h = torch.from_numpy(I.A).pin_memory()
    A = A_h.to(dev)
    ctB = P.encrypt(pk, torch.from_numpy(I.B.reshape(-1).astype(np.int32)).to(dev),
                    torch.from_numpy(I.r_be).to(dev))
    ctB_h = ctB.cpu().pin_memory()
    m, n, l, w = cfg.m, cfg.n, cfg.l, cfg.w
    count = m * l
    path = {"cussen": P.CUSSEN, "schoolbook": P.SCHOOLBOOK, "strassen": P.STRASSEN}[args.path]
    wide = w > 8                         # int32 plaintexts: pcmm_mul_*_wide (NEXT-1, t = 12, 16)
    ws = P.alloc_workspace(m, n, l, w, path, dev, wide=wide)
    proj = torch.empty(P.proj_bytes(count), dtype=torch.uint8, device=dev)
    out = torch.empty((count, 128), dtype=torch.uint8, device=dev)
    out_h = torch.empty((count, 128), dtype=torch.uint8).pin_memory()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step(A=A, ctB=ctB, out=out):
        if path == P.CUSSEN:
            P.mul_cussen(A, ctB, l, w, cfg.signed, 4, out_proj=proj, ws=ws)
        elif path == P.STRASSEN:
            P.mul_strassen(A, ctB, l, w, cfg.signed, args.leaf, out_proj=proj, ws=ws)
        else:
            P.mul_schoolbook(A, ctB, l, w, cfg.signed, out_proj=proj, ws=ws)
        P.normalize(proj, count, out=out)

    # pipelined end to end: two device input/output sets; the host->device copy of
    # step k+1's inputs and the device->host copy of step k's result run on a copy
    # stream while step k computes (every step still copies its own inputs and result)
    copy_stream = torch.cuda.Stream(device=dev)
    sets = [(A, ctB, out, out_h), (torch.empty_like(A), torch.empty_like(ctB), torch.empty_like(out),
                                   torch.empty_like(out_h).pin_memory())]

    def e2e_pipelined(K):
        h2d = [torch.cuda.Event() for _ in range(2)]
        comp = [torch.cuda.Event() for _ in range(2)]
        d2h = [torch.cuda.Event() for _ in range(2)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0.record(copy_stream)
        with torch.cuda.stream(copy_stream):
            sets[0][0].copy_(A_h, non_blocking=True)
            sets[0][1].copy_(ctB_h, non_blocking=True)
        h2d[0].record(copy_stream)
        for k in range(K):
            a_d, c_d, o_d, o_h = sets[k % 2]
            stream.wait_event(h2d[k % 2])
            if k >= 2:
                stream.wait_event(d2h[k % 2])          # the result buffer of step k-2 has been read
            if graphs:
                graphs[k % 2].replay()
            else:
                step(a_d, c_d, o_d)
            comp[k % 2].record(stream)
            if k + 1 < K:
                nxt = sets[(k + 1) % 2]
                if k >= 1:
                    copy_stream.wait_event(comp[(k + 1) % 2])   # step k-1 no longer reads that set
                with torch.cuda.stream(copy_stream):
                    nxt[0].copy_(A_h, non_blocking=True)
                    nxt[1].copy_(ctB_h, non_blocking=True)
                h2d[(k + 1) % 2].record(copy_stream)
            copy_stream.wait_event(comp[k % 2])
            with torch.cuda.stream(copy_stream):
                o_h.copy_(o_d, non_blocking=True)
            d2h[k % 2].record(copy_stream)
        t1.record(copy_stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        return reduce_max(t0.elapsed_time(t1) / K, dist, dev)

    def step_e2e():
        A.copy_(A_h, non_blocking=True)
        ctB.copy_(ctB_h, non_blocking=True)
        step()
        out_h.copy_(out, non_blocking=True)

    for _ in range(args.warmup):
        step()
    P.status(ws)

    def timed(fn, K, profile=False):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        if profile:
            P.profile_enable(True)
        for a, b in evs:
            flush.zero_()
            a.record(stream)
            fn()
            b.record(stream)
        torch.cuda.synchronize()
        prof = P.profile_read() if profile else []
        if profile:
            P.profile_enable(False)
        if dist:
            dist.barrier()
        ms = reduce_max(sum(a.elapsed_time(b) for a, b in evs) / K, dist, dev)
        return ms, prof

    # The step is captured once into a CUDA graph per device buffer set (every kernel of the
    # step is a graph node; the library's argument checks run at capture time) and replayed
    # per step; the per-kernel breakdown comes from a separate profiled eager pass.
    graphs = []
    if not args.no_graph and path != P.STRASSEN:           # Strassen allocates per call (stream-ordered pool)
        cap = torch.cuda.Stream(device=dev)
        for st_set in sets:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                step(st_set[0], st_set[1], st_set[2])
            graphs.append(g)
        torch.cuda.synchronize()
    run = graphs[0].replay if graphs else step
    with ClockSampler(local) as clk:
        ms, _ = timed(run, args.steps)
    clocks = clk.summary()
    P.status(ws)
    _, prof = timed(step, args.steps, profile=True)
    P.status(ws)
    ms_e2e_serial, _ = timed(step_e2e, max(3, args.steps // 2))
    P.status(ws)
    e2e_pipelined(2)
    ms_e2e = e2e_pipelined(max(3, args.steps // 2))
    P.status(ws)
    assert torch.equal(sets[1][3], out_h), "pipelined e2e results differ"

    # ---- kernel breakdown and roofline of the dominant kernel ----
    per = {}
    for name, t in prof:
        per.setdefault(name, []).append(t)
    launches = len(prof)
    kern = {k: {"ms_per_step": sum(v) / args.steps, "launches_per_step": len(v) / args.steps} for k, v in per.items()}
    dom = max(kern, key=lambda k: kern[k]["ms_per_step"]) if kern else None
    acc_adds, tbl_adds, tbl_dbls = algorithmic_counts(I.A, l, w)
    peaks = measured_peaks()
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_fpmul = nsm * P_PROD * f_max / LIMB_PRODUCTS_PER_FPMUL / 1e9          # G fp_mul/s
    F_total = (FPMUL_PER_ACC_ADD * acc_adds + FPMUL_PER_ADD * tbl_adds + FPMUL_PER_DBL * tbl_dbls
               + FPMUL_PER_AFFINE * table_entries(I.A, l) + FPMUL_PER_NORM * 2 * count)
    roof = None
    if path == P.CUSSEN and "accum" in kern:
        t_acc = kern["accum"]["ms_per_step"] + kern.get("reduce", {"ms_per_step": 0})["ms_per_step"]
        F_acc = FPMUL_PER_ACC_ADD * acc_adds
        achieved = F_acc / (t_acc * 1e-3) / 1e9
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                traffic = json.load(f).get(args.config, {}).get("accum_dram_bytes")
        except Exception:
            pass
        roof = {"bound": "alu", "kernel": "k_accum (+k_reduce)", "achieved": achieved, "peak": peak_fpmul,
                "unit": "G fp_mul/s", "frac": achieved / peak_fpmul, "traffic": traffic,
                "peak_note": f"{nsm} SM x {P_PROD:.0f} 32x32->64 products/clk/SM x {f_max / 1e9:.3f} GHz (sm_max) "
                             f"/ 64 products per fp_mul; IMAD.WIDE half-rate measured by tools/k11_imad_probe.cu",
                "algorithmic": f"{FPMUL_PER_ACC_ADD} fp_mul-equivalents (8M + 2S XYZZ + affine; squares at "
                               f"36/64) x {acc_adds} useful "
                               f"accumulate adds (a_ik != 0)"}

    value = world * count / (ms * 1e-3)
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": workload_config(cfg, args.path, world),
        "point_adds_per_s": world * (acc_adds + tbl_adds + tbl_dbls) / (ms * 1e-3),
        "paper_model_adds_per_s": world * paper_model_adds(I.A, l, w) / (ms * 1e-3),
        "fp_mul_per_s": world * F_total / (ms * 1e-3),
        "roofline_whole_step": {"achieved": F_total / (ms * 1e-3) / 1e9, "peak": peak_fpmul,
                                "frac": F_total / (ms * 1e-3) / 1e9 / peak_fpmul, "unit": "G fp_mul/s"},
        "roofline": roof,
        "kernels": kern, "dominant_kernel": dom,
        "gpu_launches": launches,
        "launch": (f"one CUDA-graph replay per step ({launches // max(args.steps, 1)} kernels captured once per "
                   f"device buffer set)") if graphs else "eager launches",
        "clocks": clocks,
        "e2e": {"value": world * count / (ms_e2e * 1e-3), "unit": UNIT, "ms_per_step": ms_e2e,
                "h2d_bytes_per_step": int(A.numel() + ctB.numel()), "d2h_bytes_per_step": int(out.numel()),
                "mode": "pipelined: step k+1's H2D and step k's D2H on a copy stream overlap step k's compute "
                        "(pinned host buffers, two device buffer sets, continuous timed region over all steps)",
                "serial_ms_per_step": ms_e2e_serial,
                "serial_value": world * count / (ms_e2e_serial * 1e-3)},
    }
    if path == P.CUSSEN and not args.no_schoolbook:
        def sb():
            P.mul_schoolbook(A, ctB, l, w, cfg.signed, out_proj=proj, ws=ws_sb)
            P.normalize(proj, count, out=out)
        ws_sb = P.alloc_workspace(m, n, l, w, P.SCHOOLBOOK, dev, wide=wide)
        ws_st = P.alloc_workspace(m, n, l, w, P.STRASSEN, dev, wide=wide)
        sb()
        ms_sb, _ = timed(sb, max(2, args.steps // 5))
        res["schoolbook"] = {"ms_per_step": ms_sb, "value": world * count / (ms_sb * 1e-3),
                             "cussen_speedup": ms_sb / ms}

        def st():
            P.mul_strassen(A, ctB, l, w, cfg.signed, args.leaf, out_proj=proj, ws=ws_st)
            P.normalize(proj, count, out=out)
        st()
        ms_st, _ = timed(st, max(2, args.steps // 5))
        res["strassen"] = {"ms_per_step": ms_st, "value": world * count / (ms_st * 1e-3), "leaf": args.leaf,
                           "cussen_speedup": ms_st / ms}
    if rank == 0 and not args.no_cpu_baseline:
        res["cpu_baseline"] = oracle_baseline(cfg, min(args.ref_cols, cfg.l), args.path)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
