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
# Roofline denominator (DESIGN.md §6 "Machine model"): 32x32->64 products / clk / SM, the best measured
# rate of the product instruction in the form the field product issues it (carry chains of
# IMAD.WIDE.U32 + IMAD.WIDE.U32.X): 52.2 at 48-64 warps per SM (tools/k12_chain_probe.cu,
# profiles/r02_k12_chain_probe_nc2.txt).  Round 1 used 32.0 from K11's mul.wide probe
# (profiles/r01_k11_imad.txt), whose operands came from one register pair; K12 supersedes it.
P_PROD = 52.2
P_PROD_K11 = 32.0
LIMB_PRODUCTS_PER_FPMUL = 64.0
# Algorithmic work numerator F of SURVEY.md §8(d) (fixed per input, not per implementation):
#   F = 14 (useful complete adds) + 13 (doublings) + 6 (normalised points)
F_ADD = 14                  # complete addition (RCB16 Alg. 4: 12M + 2 m_b)
F_DBL = 13                  # complete doubling (RCB16 Alg. 6: 8M + 3S + 2 m_b)
F_NORM = 6                  # normalisation per point
# Executed IMAD work of the accumulate step actually run (k_accum): XYZZ + affine mixed addition
# (madd-2008-s) 8M + 2S, the squares through the 36-product squaring: 8 + 2 x 36/64 = 9.125
# fp_mul-equivalents per addition -> `frac_executed_products` (the utilisation of the products issued)
EXEC_PER_ACC_ADD = 8 + 2 * 36 / 64


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def workload_config(cfg, path: str, world: int) -> dict:
    """The `config` object of the JSON line (shared, identical, by both arms)."""
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


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def algorithmic_counts(A: np.ndarray, l: int, w: int):
    """Algorithmic work of the Cussen path fixed by the input:
    useful accumulate adds (terms with a_ik != 0; n_i - 1 adds per output and
    component), table-build ops (prefix adds of every level + binary-ECSM ops of
    the last level; x1 is free), counted from the compression of A."""
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


def work_numerators(A: np.ndarray, l: int, w: int) -> dict:
    """SURVEY.md §8(d)'s fixed numerator F for the whole step and for the dominant kernel."""
    m = A.shape[0]
    acc_adds, tbl_adds, tbl_dbls = algorithmic_counts(A, l, w)
    points = 2 * m * l
    return {"acc_adds": acc_adds, "tbl_adds": tbl_adds, "tbl_dbls": tbl_dbls, "points": points,
            "F_step": F_ADD * (acc_adds + tbl_adds) + F_DBL * tbl_dbls + F_NORM * points,
            "F_accum": F_ADD * acc_adds, "exec_accum": EXEC_PER_ACC_ADD * acc_adds,
            "point_ops": acc_adds + tbl_adds + tbl_dbls}


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


def lib_sha16() -> str | None:
    """Identity of the library build: sha256 over its sources (csrc/, include/pcmm.h) and build.py (flags),
    so that a rebuild of the same sources (e.g. the driver's build()) keeps the identity of an ncu capture."""
    import hashlib
    try:
        from paper_2504_14497_b200 import build as _b
        h = hashlib.sha256()
        for path in sorted(_b._deps()):
            h.update(os.path.basename(path).encode())
            with open(path, "rb") as f:
                h.update(f.read())
        return h.hexdigest()[:16]
    except Exception:
        return None


def dram_traffic(config_name: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per k_accum launch from an `ncu --set full` capture
    (profiles/traffic.json, written by tools/traffic.py from the .ncu-rep).  Used only when the capture
    was taken of a library built from THESE sources (same source sha256): a number from other code is stale -> null."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)
    except Exception:
        return None, "no capture"
    sha = lib_sha16()
    e = d.get(config_name)
    if not e:
        return None, "no capture for this config"
    if e.get("lib_sha16") != sha:
        return None, f"capture of another build ({e.get('lib_sha16')}, this one {sha})"
    return float(e["accum_dram_bytes"]), e.get("source", "")


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


# ---------------------------------------------------------------- the CPU oracle (baseline, reference arm)
def oracle_inputs(cfg, lcols: int | None = None):
    """Oracle-side inputs of a config: the full seeded instance, restricted to the first `lcols`
    output columns, encrypted by the ORACLE's Encrypt (nothing from the CUDA path)."""
    import oracle
    I = synth.make_instance(cfg)
    lc = cfg.l if lcols is None else min(lcols, cfg.l)
    B = I.B[:, :lc]
    r = I.r_be.reshape(cfg.n, cfg.l, 32)[:, :lc].reshape(-1, 32)
    pk = oracle.pubkey(I.x)
    ct = oracle.encrypt(pk, B.reshape(-1), r)
    return I, lc, ct


def oracle_time(cfg, path: str, lcols: int | None = None, inputs=None) -> dict:
    """Time the oracle (oracle/ as it stands: C, own bignum, all host threads) on all m rows and
    n inner indices of `cfg` and the first `lcols` output columns (all of them when None)."""
    import oracle
    I, lc, ct = inputs if inputs is not None else oracle_inputs(cfg, lcols)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    _, cnt = oracle.pcmm(oracle.CUSSEN if path == "cussen" else oracle.SCHOOLBOOK, I.A, ct, lc, cfg.w,
                         threads=threads)
    dt = time.perf_counter() - t0
    entries = cfg.m * lc
    return {"value": entries / dt, "unit": UNIT, "cores": threads, "kind": "oracle", "path": path,
            "seconds": dt, "point_ops_per_s": (cnt[0] + cnt[1]) / dt,
            "sample": (f"{cfg.name}: full workload ({entries} entries)" if lc == cfg.l else
                       f"{cfg.name}: all {cfg.m} rows x {cfg.n} k, first {lc} of {cfg.l} output columns "
                       f"({entries} entries, {100.0 * lc / cfg.l:.1f} % of the workload)") +
                      f", {path} path, {dt:.2f} s wall on {threads} threads"}


# Per-config samples of the CPU baseline (output columns; None = the full workload), sized so that
# both oracle paths over all five configs take ~30-40 s on a 16-core host
CPU_SAMPLE_COLS = {"tiny": (None, None), "c64": (None, None), "c256": (None, 32), "c512": (64, 16),
                   "ml": (None, 16)}


def cpu_baseline_all(primary: str) -> dict:
    """Both oracle paths on every BASELINE config; the top-level value is the
    oracle's Cussen path on the primary config's full workload."""
    out = {"cpu_model": cpu_model(), "cores": os.cpu_count() or 1, "configs": {}}
    for name, (lc_c, lc_s) in CPU_SAMPLE_COLS.items():
        cfg = synth.CONFIGS[name]
        inp = oracle_inputs(cfg, max(lc or cfg.l for lc in (lc_c, lc_s)) if (lc_c or lc_s) else None)
        per = {}
        for path, lc in (("cussen", lc_c), ("schoolbook", lc_s)):
            I, lcmax, ct = inp
            lc = lcmax if lc is None else min(lc, lcmax)
            ctc = ct.reshape(cfg.n, lcmax, 128)[:, :lc].reshape(-1, 128).copy()
            r = oracle_time(cfg, path, inputs=(I, lc, ctc))
            per[path] = {k: r[k] for k in ("value", "seconds", "point_ops_per_s", "sample")}
        out["configs"][name] = per
    top = out["configs"][primary]["cussen"]
    out.update({"value": top["value"], "unit": UNIT, "kind": "oracle", "sample": top["sample"]})
    return out


def run_reference(args, cfg, rank):
    """--impl reference: the CPU oracle as the reference arm (there is no installable reference code:
    /root/reference holds only the paper).  Rank 0 alone; each step is the FULL workload of `cfg`
    (the oracle's Cussen path), the inputs encrypted by the oracle once before timing."""
    if rank != 0:
        return
    inp = oracle_inputs(cfg)
    for _ in range(args.warmup):
        oracle_time(cfg, args.path if args.path != "strassen" else "cussen", inputs=inp)
    vals = [oracle_time(cfg, args.path if args.path != "strassen" else "cussen", inputs=inp)
            for _ in range(args.steps)]
    secs = [v["seconds"] for v in vals]
    ms = statistics.mean(secs) * 1e3
    v = cfg.m * cfg.l / (ms * 1e-3)
    cb = {"value": v, "unit": UNIT, "cores": vals[-1]["cores"], "kind": "oracle", "cpu_model": cpu_model(),
          "sample": f"{cfg.name}: the full workload every step ({cfg.m * cfg.l} entries), "
                    f"{args.path} path, {vals[-1]['cores']} threads"}
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": workload_config(cfg, args.path, max(1, args.gpus)),
        "cpu_baseline": cb, "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference arm = the CPU oracle (oracle/oracle.c, plain C, all host threads) on the same "
                "workload: the paper ships no code; its Raspberry Pi 5 numbers are context in BASELINE.md",
    }), flush=True)


class Gpu:
    """Device-side plumbing shared by the measured configs (one rank, one device)."""

    def __init__(self, local: int, dist):
        import torch
        from paper_2504_14497_b200 import pcmm as P
        self.torch, self.P, self.dist = torch, P, dist
        self.dev = torch.device("cuda", local)
        self.stream = torch.cuda.current_stream()
        self.flush = torch.empty(256 << 20, dtype=torch.uint8, device=self.dev)
        peaks = measured_peaks()
        self.f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
        self.nsm = torch.cuda.get_device_properties(self.dev).multi_processor_count
        self.peak = self.nsm * P_PROD * self.f_max / LIMB_PRODUCTS_PER_FPMUL / 1e9       # G fp_mul/s

    def timed(self, fn, K, profile=False):
        """K steps, L2 flushed before each (outside the events), CUDA events on the launching stream,
        barrier + synchronize on both sides, max over ranks."""
        torch, P, dist = self.torch, self.P, self.dist
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        if profile:
            P.profile_enable(True)
        for a, b in evs:
            self.flush.zero_()
            a.record(self.stream)
            fn()
            b.record(self.stream)
        torch.cuda.synchronize()
        prof = P.profile_read() if profile else []
        if profile:
            P.profile_enable(False)
        if dist:
            dist.barrier()
        ms = reduce_max(sum(a.elapsed_time(b) for a, b in evs) / K, dist, self.dev)
        return ms, prof


class Problem:
    """One configuration's device buffers and its step (a0-a6: mul + normalize)."""

    def __init__(self, g: Gpu, cfg, path_name: str, seed: int, leaf: int = 32):
        torch, P = g.torch, g.P
        self.g, self.cfg, self.path_name, self.leaf = g, cfg, path_name, leaf
        I = synth.make_instance(cfg, seed=seed)
        self.I = I
        sk, pk = P.keygen(seed)
        self.A_h = torch.from_numpy(I.A).pin_memory()
        self.A = self.A_h.to(g.dev)
        self.ctB = P.encrypt(pk, torch.from_numpy(I.B.reshape(-1).astype(np.int32)).to(g.dev),
                             torch.from_numpy(I.r_be).to(g.dev))
        self.ctB_h = self.ctB.cpu().pin_memory()
        m, n, l, w = cfg.m, cfg.n, cfg.l, cfg.w
        self.count = m * l
        self.path = {"cussen": P.CUSSEN, "schoolbook": P.SCHOOLBOOK, "strassen": P.STRASSEN}[path_name]
        self.wide = w > 8
        self.ws = P.alloc_workspace(m, n, l, w, self.path, g.dev, wide=self.wide)
        self.proj = torch.empty(P.proj_bytes(self.count), dtype=torch.uint8, device=g.dev)
        self.out = torch.empty((self.count, 128), dtype=torch.uint8, device=g.dev)
        self.out_h = torch.empty((self.count, 128), dtype=torch.uint8).pin_memory()
        self.graphs = []

    def step(self, A=None, ctB=None, out=None, path=None, ws=None):
        P, cfg = self.g.P, self.cfg
        A = self.A if A is None else A
        ctB = self.ctB if ctB is None else ctB
        out = self.out if out is None else out
        path = self.path if path is None else path
        ws = self.ws if ws is None else ws
        if path == P.CUSSEN:
            P.mul_cussen(A, ctB, cfg.l, cfg.w, cfg.signed, 4, out_proj=self.proj, ws=ws)
        elif path == P.STRASSEN:
            P.mul_strassen(A, ctB, cfg.l, cfg.w, cfg.signed, self.leaf, out_proj=self.proj, ws=ws)
        else:
            P.mul_schoolbook(A, ctB, cfg.l, cfg.w, cfg.signed, out_proj=self.proj, ws=ws)
        P.normalize(self.proj, self.count, out=out)

    def capture(self, sets):
        """One CUDA graph per device buffer set (every kernel of the step is a graph node; the
        library's argument checks run at capture time)."""
        torch = self.g.torch
        if self.path == self.g.P.STRASSEN:          # Strassen allocates per call (stream-ordered pool)
            return
        cap = torch.cuda.Stream(device=self.g.dev)
        for st in sets:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=cap):
                self.step(st[0], st[1], st[2])
            self.graphs.append(gr)
        torch.cuda.synchronize()

    def measure(self, steps: int, warmup: int, with_school: bool = True):
        """Device-timed step, per-kernel breakdown (library events, separate eager pass), roofline
        per SURVEY.md §8(d), and the schoolbook path on the same inputs."""
        g, P, cfg = self.g, self.g.P, self.cfg
        for _ in range(warmup):
            self.step()
        P.status(self.ws)
        if not self.graphs:
            self.capture([(self.A, self.ctB, self.out)])
        run = self.graphs[0].replay if self.graphs else self.step
        ms, _ = g.timed(run, steps)
        P.status(self.ws)
        _, prof = g.timed(self.step, steps, profile=True)
        P.status(self.ws)
        per = {}
        for name, t in prof:
            per.setdefault(name, []).append(t)
        kern = {k: {"ms_per_step": sum(v) / steps, "launches_per_step": len(v) / steps} for k, v in per.items()}
        W = work_numerators(self.I.A, cfg.l, cfg.w)
        world = max(1, g.dist.get_world_size()) if g.dist else 1
        res = {"ms_per_step": ms, "value": world * self.count / (ms * 1e-3),
               "point_adds_per_s": world * W["point_ops"] / (ms * 1e-3),
               "fp_mul_per_s": world * W["F_step"] / (ms * 1e-3),
               "paper_model_adds_per_s": world * paper_model_adds(self.I.A, cfg.l, cfg.w) / (ms * 1e-3),
               "kernels": kern, "gpu_launches": len(prof),
               "dominant_kernel": max(kern, key=lambda k: kern[k]["ms_per_step"]) if kern else None,
               "roofline_whole_step": {"achieved": W["F_step"] / (ms * 1e-3) / 1e9, "peak": g.peak,
                                       "frac": W["F_step"] / (ms * 1e-3) / 1e9 / g.peak, "unit": "G fp_mul/s",
                                       "numerator": "SURVEY.md §8(d) F = 14 (useful adds) + 13 (doublings) "
                                                    f"+ 6 (points) = {W['F_step']:.4g} fp_mul"}}
        if self.path == P.CUSSEN and "accum" in kern:
            t_acc = (kern["accum"]["ms_per_step"] + kern.get("reduce", {"ms_per_step": 0})["ms_per_step"] +
                     kern.get("rowperm", {"ms_per_step": 0})["ms_per_step"])
            ach = W["F_accum"] / (t_acc * 1e-3) / 1e9
            ex = W["exec_accum"] / (t_acc * 1e-3) / 1e9
            traffic, tsrc = dram_traffic(cfg.name)
            res["roofline"] = {
                "bound": "alu", "kernel": ("k_accum_g2 (+k_rowperm, k_reduce)" if "rowperm" in kern else "k_accum (+k_reduce)"), "achieved": ach, "peak": g.peak,
                "unit": "G fp_mul/s", "frac": ach / g.peak, "traffic": traffic, "traffic_source": tsrc,
                "frac_executed_products": ex / g.peak,
                "frac_vs_r01_peak": ach / (g.peak * P_PROD_K11 / P_PROD),
                "algorithmic": f"SURVEY.md §8(d): 14 fp_mul per useful complete addition x {W['acc_adds']} "
                               f"useful accumulate additions (a_ik != 0) over the kernel time {t_acc:.4f} ms "
                               f"(library CUDA events on the launching stream)",
                "executed": f"frac_executed_products: the products the kernel issues, {EXEC_PER_ACC_ADD} "
                            f"fp_mul-equivalents per XYZZ + affine mixed addition (8M + 2S, squares at 36/64)",
                "peak_note": f"{g.nsm} SM x {P_PROD:.1f} 32x32->64 products/clk/SM x {g.f_max / 1e9:.3f} GHz "
                             f"(sm_max) / 64 products per fp_mul; {P_PROD:.1f} = IMAD.WIDE.U32(.X) carry chains "
                             f"alone at 48-64 warps per SM (tools/k12_chain_probe.cu, "
                             f"profiles/r02_k12_chain_probe_nc2.txt); the kernel's own instruction mix "
                             f"(1.8 ALU instructions per IMAD.WIDE, issue costs add: DESIGN.md §6) bounds it "
                             f"at ~0.47 of this peak at full issue efficiency; frac_vs_r01_peak is against "
                             f"round 1's {P_PROD_K11:.0f}/clk/SM (K11's mul.wide probe, superseded)"}
        if with_school and self.path == P.CUSSEN:
            ws_sb = P.alloc_workspace(cfg.m, cfg.n, cfg.l, cfg.w, P.SCHOOLBOOK, g.dev, wide=self.wide)

            def sb():
                self.step(path=P.SCHOOLBOOK, ws=ws_sb)
            sb()
            ms_sb, _ = g.timed(sb, max(2, min(steps // 5, 6)))
            res["schoolbook"] = {"ms_per_step": ms_sb, "value": world * self.count / (ms_sb * 1e-3),
                                 "cussen_speedup": ms_sb / ms}
            del ws_sb
        return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c256", choices=list(synth.CONFIGS))
    ap.add_argument("--path", default="cussen", choices=["cussen", "schoolbook", "strassen"])
    ap.add_argument("--leaf", type=int, default=32, help="Strassen recursion leaf block size")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-schoolbook", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the other BASELINE configs' sub-objects")
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
        args.no_configs = True
    if args.impl == "reference":
        return run_reference(args, cfg, rank)

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    g = Gpu(local, dist)
    P = g.P
    pr = Problem(g, cfg, args.path, rank_instance_seed(cfg, rank), args.leaf)
    stream = g.stream

    # pipelined end to end: two device input/output sets; the host->device copy of step k+1's
    # inputs and the device->host copy of step k's result run on a copy stream while step k
    # computes (every step still copies its own inputs and result)
    copy_stream = torch.cuda.Stream(device=g.dev)
    sets = [(pr.A, pr.ctB, pr.out, pr.out_h), (torch.empty_like(pr.A), torch.empty_like(pr.ctB),
                                              torch.empty_like(pr.out), torch.empty_like(pr.out_h).pin_memory())]
    if not args.no_graph:
        pr.capture(sets)

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
            sets[0][0].copy_(pr.A_h, non_blocking=True)
            sets[0][1].copy_(pr.ctB_h, non_blocking=True)
        h2d[0].record(copy_stream)
        for k in range(K):
            a_d, c_d, o_d, o_h = sets[k % 2]
            stream.wait_event(h2d[k % 2])
            if k >= 2:
                stream.wait_event(d2h[k % 2])          # the result buffer of step k-2 has been read
            if pr.graphs:
                pr.graphs[k % 2].replay()
            else:
                pr.step(a_d, c_d, o_d)
            comp[k % 2].record(stream)
            if k + 1 < K:
                nxt = sets[(k + 1) % 2]
                if k >= 1:
                    copy_stream.wait_event(comp[(k + 1) % 2])   # step k-1 no longer reads that set
                with torch.cuda.stream(copy_stream):
                    nxt[0].copy_(pr.A_h, non_blocking=True)
                    nxt[1].copy_(pr.ctB_h, non_blocking=True)
                h2d[(k + 1) % 2].record(copy_stream)
            copy_stream.wait_event(comp[k % 2])
            with torch.cuda.stream(copy_stream):
                o_h.copy_(o_d, non_blocking=True)
            d2h[k % 2].record(copy_stream)
        t1.record(copy_stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        return reduce_max(t0.elapsed_time(t1) / K, dist, g.dev)

    def step_e2e():
        pr.A.copy_(pr.A_h, non_blocking=True)
        pr.ctB.copy_(pr.ctB_h, non_blocking=True)
        pr.step()
        pr.out_h.copy_(pr.out, non_blocking=True)

    for _ in range(args.warmup):
        pr.step()
    P.status(pr.ws)
    run = pr.graphs[0].replay if pr.graphs else pr.step
    with ClockSampler(local) as clk:
        ms, _ = g.timed(run, args.steps)
    clocks = clk.summary()
    P.status(pr.ws)
    detail = pr.measure(args.steps, 0, with_school=not args.no_schoolbook)
    ms_e2e_serial, _ = g.timed(step_e2e, max(3, args.steps // 2))
    P.status(pr.ws)
    e2e_pipelined(2)
    ms_e2e = e2e_pipelined(max(3, args.steps // 2))
    P.status(pr.ws)
    assert torch.equal(sets[1][3], pr.out_h), "pipelined e2e results differ"

    W = work_numerators(pr.I.A, cfg.l, cfg.w)
    count = pr.count
    value = world * count / (ms * 1e-3)
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": workload_config(cfg, args.path, world),
        "point_adds_per_s": world * W["point_ops"] / (ms * 1e-3),
        "paper_model_adds_per_s": world * paper_model_adds(pr.I.A, cfg.l, cfg.w) / (ms * 1e-3),
        "fp_mul_per_s": world * W["F_step"] / (ms * 1e-3),
        "roofline_whole_step": {"achieved": W["F_step"] / (ms * 1e-3) / 1e9, "peak": g.peak,
                                "frac": W["F_step"] / (ms * 1e-3) / 1e9 / g.peak, "unit": "G fp_mul/s",
                                "numerator": detail["roofline_whole_step"]["numerator"]},
        "roofline": detail.get("roofline"),
        "kernels": detail["kernels"], "dominant_kernel": detail["dominant_kernel"],
        "gpu_launches": detail["gpu_launches"],
        "launch": (f"one CUDA-graph replay per step ({detail['gpu_launches'] // max(args.steps, 1)} kernels "
                   f"captured once per device buffer set)") if pr.graphs else "eager launches",
        "clocks": clocks,
        "e2e": {"value": world * count / (ms_e2e * 1e-3), "unit": UNIT, "ms_per_step": ms_e2e,
                "h2d_bytes_per_step": int(pr.A.numel() + pr.ctB.numel()), "d2h_bytes_per_step": int(pr.out.numel()),
                "mode": "pipelined: step k+1's H2D and step k's D2H on a copy stream overlap step k's compute "
                        "(pinned host buffers, two device buffer sets, continuous timed region over all steps)",
                "serial_ms_per_step": ms_e2e_serial,
                "serial_value": world * count / (ms_e2e_serial * 1e-3)},
    }
    if "schoolbook" in detail:
        res["schoolbook"] = detail["schoolbook"]
    if pr.path == P.CUSSEN and not args.no_schoolbook:
        ws_st = P.alloc_workspace(cfg.m, cfg.n, cfg.l, cfg.w, P.STRASSEN, g.dev, wide=pr.wide)

        def st():
            P.mul_strassen(pr.A, pr.ctB, cfg.l, cfg.w, cfg.signed, args.leaf, out_proj=pr.proj, ws=ws_st)
            P.normalize(pr.proj, count, out=pr.out)
        st()
        ms_st, _ = g.timed(st, max(2, args.steps // 5))
        res["strassen"] = {"ms_per_step": ms_st, "value": world * count / (ms_st * 1e-3), "leaf": args.leaf,
                           "cussen_speedup": ms_st / ms}
        del ws_st
    # the other BASELINE configs, same protocol, as sub-objects of this line
    if not args.no_configs and args.path == "cussen":
        res["configs"] = {}
        for name, c in synth.CONFIGS.items():
            if name == cfg.name:
                continue
            pc = Problem(g, c, "cussen", rank_instance_seed(c, rank))
            d = pc.measure(max(5, args.steps // 2), 3, with_school=not args.no_schoolbook)
            d["workload"] = workload_config(c, "cussen", world)["workload"]
            res["configs"][name] = d
            del pc
            torch.cuda.empty_cache()
    res["gpu_launches_total"] = res["gpu_launches"] + sum(d["gpu_launches"] for d in res.get("configs", {}).values())
    if rank == 0 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline_all(cfg.name) if cfg.name in CPU_SAMPLE_COLS else \
            oracle_time(cfg, "cussen" if args.path == "strassen" else args.path, lcols=min(48, cfg.l))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
