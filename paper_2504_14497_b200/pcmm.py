"""Thin Python binding of libpcmm.so (include/pcmm.h) -- argument marshalling only.

Every step of the PC-MM path runs in the library's sm_100a kernels; this module
only checks tensor dtypes / devices / shapes, allocates outputs and workspaces
with PyTorch (device memory + streams are PyTorch's job here), and passes raw
pointers and the current CUDA stream through ctypes.  There is no CPU fallback:
if the library cannot be built / loaded, or no CUDA device is present, calls
raise `PCMMError`.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

from . import build as _build

PCMM_OK = 0
PCMM_EINVAL = -1
PCMM_EDIM = -2
PCMM_EBOUND = -3
PCMM_ENOTONCURVE = -4
PCMM_EDECODE = -5
PCMM_ECUDA = -6
PCMM_ENOMEM = -7
PCMM_ENOTSUP = -8
SCHOOLBOOK, CUSSEN, STRASSEN = 0, 1, 2

EXPORTS = [
    "pcmm_last_error", "pcmm_version", "pcmm_proj_bytes", "pcmm_keygen", "pcmm_encrypt", "pcmm_workspace_bytes",
    "pcmm_mul_schoolbook", "pcmm_mul_cussen", "pcmm_mul_strassen", "pcmm_normalize", "pcmm_decrypt_small", "pcmm_status",
    "pcmm_profile_enable", "pcmm_profile_read", "pcmm_test_field", "pcmm_test_point", "pcmm_test_plan",
    "pcmm_bench_fp_mul", "pcmm_workspace_bytes_wide", "pcmm_mul_cussen_wide", "pcmm_mul_schoolbook_wide",
    "pcmm_mul_strassen_wide", "pcmm_enc_ctx_bytes", "pcmm_enc_ctx_init", "pcmm_encrypt_ctx", "pcmm_bsgs_ctx_bytes",
    "pcmm_bsgs_init", "pcmm_decrypt_bsgs", "pcmm_paillier_workspace_bytes", "pcmm_paillier_mul",
]


class PCMMError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"pcmm error {code}: {msg}")
        self.code = code


_lock = threading.Lock()
_lib = None


def lib_path() -> str:
    return _build.LIB


def load(build_if_needed: bool = True) -> ctypes.CDLL:
    """Load libpcmm.so (building it with nvcc first if it is missing or stale)."""
    global _lib
    with _lock:
        if _lib is None:
            checked = os.environ.get("PCMM_LIB_VARIANT", "") == "checked"    # device bounds-check build
            lib = _build.LIB_CHECKED if checked else _build.LIB
            if build_if_needed and _build.needs_build(checked):
                _build.build(checked=checked)
            if not os.path.exists(lib):
                raise PCMMError(PCMM_ECUDA, f"{lib} is missing (run __graft_entry__.build())")
            L = ctypes.CDLL(lib)
            vp, sz, i64, i32, u64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64
            L.pcmm_last_error.restype = ctypes.c_char_p
            L.pcmm_version.restype = ctypes.c_char_p
            L.pcmm_proj_bytes.restype = sz
            L.pcmm_proj_bytes.argtypes = [i64]
            L.pcmm_keygen.argtypes = [u64, vp, vp]
            L.pcmm_encrypt.argtypes = [vp, vp, vp, i64, vp, vp]
            L.pcmm_workspace_bytes.restype = sz
            L.pcmm_workspace_bytes.argtypes = [i32] * 5
            L.pcmm_mul_schoolbook.argtypes = [vp, i32, i32, i32, i32, i32, vp, vp, vp, sz, vp]
            L.pcmm_mul_cussen.argtypes = [vp, i32, i32, i32, i32, i32, i32, vp, vp, vp, sz, vp]
            L.pcmm_mul_strassen.argtypes = [vp, i32, i32, i32, i32, i32, i32, vp, vp, vp, sz, vp]
            L.pcmm_normalize.argtypes = [vp, i64, vp, vp, sz, vp]
            L.pcmm_decrypt_small.argtypes = [vp, vp, i64, i64, i64, vp, vp, vp]
            L.pcmm_status.argtypes = [vp, vp]
            L.pcmm_profile_enable.argtypes = [i32]
            L.pcmm_profile_read.argtypes = [vp, vp, i32]
            L.pcmm_test_field.argtypes = [i32, vp, vp, vp, i64, vp]
            L.pcmm_test_point.argtypes = [i32, vp, vp, vp, vp, i64, vp]
            L.pcmm_test_plan.argtypes = [vp, i32, i32, i32, i32, i32, vp, vp, vp, vp]
            L.pcmm_bench_fp_mul.argtypes = [i32, i32, i32, i32, vp, vp]
            L.pcmm_workspace_bytes_wide.restype = sz
            L.pcmm_workspace_bytes_wide.argtypes = [i32] * 5
            L.pcmm_mul_cussen_wide.argtypes = [vp, i32, i32, i32, i32, i32, i32, vp, vp, vp, sz, vp]
            L.pcmm_mul_schoolbook_wide.argtypes = [vp, i32, i32, i32, i32, i32, vp, vp, vp, sz, vp]
            L.pcmm_mul_strassen_wide.argtypes = [vp, i32, i32, i32, i32, i32, i32, vp, vp, vp, sz, vp]
            L.pcmm_enc_ctx_bytes.restype = sz
            L.pcmm_enc_ctx_bytes.argtypes = []
            L.pcmm_enc_ctx_init.argtypes = [vp, vp, vp]
            L.pcmm_encrypt_ctx.argtypes = [vp, vp, vp, i64, vp, vp]
            L.pcmm_bsgs_ctx_bytes.restype = sz
            L.pcmm_bsgs_ctx_bytes.argtypes = [i32]
            L.pcmm_bsgs_init.argtypes = [i32, vp, vp]
            L.pcmm_decrypt_bsgs.argtypes = [vp, vp, i32, vp, i64, i64, i64, vp, vp, vp]
            L.pcmm_paillier_workspace_bytes.restype = sz
            L.pcmm_paillier_workspace_bytes.argtypes = [i32] * 6
            L.pcmm_paillier_mul.argtypes = [i32, vp, i32, i32, i32, i32, i32, vp, i32, vp, vp, vp, sz, vp]
            _lib = L
    return _lib


def _check(rc: int):
    if rc != PCMM_OK:
        raise PCMMError(rc, load().pcmm_last_error().decode())


def _stream(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _dev(t: torch.Tensor, dtype, name: str) -> int:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise PCMMError(PCMM_EINVAL, f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise PCMMError(PCMM_EINVAL, f"{name} must have dtype {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise PCMMError(PCMM_EINVAL, f"{name} must be contiguous")
    return t.data_ptr()


def _require_cuda():
    if not torch.cuda.is_available():
        raise PCMMError(PCMM_ECUDA, "no CUDA device: libpcmm has no CPU fallback")


def version() -> str:
    return load().pcmm_version().decode()


# ------------------------------------------------------------------ EC-ElGamal
def keygen(seed: int) -> tuple[bytes, bytes]:
    """KeyGen: -> (sk = x, 32 B BE; pk = H = xG, 64 B canonical)."""
    _require_cuda()
    sk = ctypes.create_string_buffer(32)
    pk = ctypes.create_string_buffer(64)
    _check(load().pcmm_keygen(seed & (2**64 - 1), sk, pk))
    return sk.raw, pk.raw


def encrypt(pk: bytes, b: torch.Tensor, r: torch.Tensor, out: torch.Tensor | None = None, stream=None):
    """Encrypt: b int32 [count] (cuda), r uint8 [count, 32] -> uint8 [count, 128]."""
    _require_cuda()
    count = b.numel()
    if r.numel() != 32 * count:
        raise PCMMError(PCMM_EINVAL, "r must hold 32 bytes per plaintext")
    if out is None:
        out = torch.empty((count, 128), dtype=torch.uint8, device=b.device)
    pkb = ctypes.create_string_buffer(bytes(pk), 64)
    _check(load().pcmm_encrypt(pkb, _dev(b, torch.int32, "b"), _dev(r, torch.uint8, "r"), count,
                               _dev(out, torch.uint8, "out"), _stream(stream)))
    return out


def decrypt_small(sk: bytes, ct: torch.Tensor, lo: int, hi: int, stream=None):
    """Decrypt by exact table lookup over [lo, hi] -> (m int64, status int32)."""
    _require_cuda()
    count = ct.numel() // 128
    m = torch.empty(count, dtype=torch.int64, device=ct.device)
    st = torch.empty(count, dtype=torch.int32, device=ct.device)
    skb = ctypes.create_string_buffer(bytes(sk), 32)
    _check(load().pcmm_decrypt_small(skb, _dev(ct, torch.uint8, "ct"), count, lo, hi, m.data_ptr(), st.data_ptr(),
                                     _stream(stream)))
    return m, st


# ------------------------------------------------------------------ NEXT-2: comb encryption, BSGS decryption
def enc_ctx(pk: bytes, device="cuda", stream=None) -> torch.Tensor:
    """Fixed-base comb tables for G and H = pk: a device context (synchronises the stream)."""
    _require_cuda()
    ctx = torch.empty(int(load().pcmm_enc_ctx_bytes()), dtype=torch.uint8, device=device)
    pkb = ctypes.create_string_buffer(bytes(pk), 64)
    _check(load().pcmm_enc_ctx_init(pkb, ctx.data_ptr(), _stream(stream)))
    return ctx


def encrypt_ctx(ctx: torch.Tensor, b: torch.Tensor, r: torch.Tensor, out: torch.Tensor | None = None, stream=None):
    """Encrypt with a comb context: same bytes as `encrypt` (b int32 [count], r uint8 [count, 32])."""
    _require_cuda()
    count = b.numel()
    if r.numel() != 32 * count:
        raise PCMMError(PCMM_EINVAL, "r must hold 32 bytes per plaintext")
    if out is None:
        out = torch.empty((count, 128), dtype=torch.uint8, device=b.device)
    _check(load().pcmm_encrypt_ctx(_dev(ctx, torch.uint8, "ctx"), _dev(b, torch.int32, "b"),
                                   _dev(r, torch.uint8, "r"), count, _dev(out, torch.uint8, "out"), _stream(stream)))
    return out


def bsgs_ctx(log2_baby: int, device="cuda", stream=None) -> torch.Tensor:
    """Baby-step table { jG : 1 <= j < 2^log2_baby } as a device hash table."""
    _require_cuda()
    nb = int(load().pcmm_bsgs_ctx_bytes(log2_baby))
    if nb == 0:
        raise PCMMError(PCMM_EINVAL, "log2_baby must be in [1, 28]")
    ctx = torch.empty(nb, dtype=torch.uint8, device=device)
    _check(load().pcmm_bsgs_init(log2_baby, ctx.data_ptr(), _stream(stream)))
    return ctx


def decrypt_bsgs(sk: bytes, ctx: torch.Tensor, log2_baby: int, ct: torch.Tensor, lo: int, hi: int, stream=None):
    """Decrypt messages in [lo, hi] by baby-step giant-step -> (m int64, status int32)."""
    _require_cuda()
    count = ct.numel() // 128
    m = torch.empty(count, dtype=torch.int64, device=ct.device)
    st = torch.empty(count, dtype=torch.int32, device=ct.device)
    skb = ctypes.create_string_buffer(bytes(sk), 32)
    _check(load().pcmm_decrypt_bsgs(skb, _dev(ctx, torch.uint8, "ctx"), log2_baby, _dev(ct, torch.uint8, "ct"),
                                    count, lo, hi, m.data_ptr(), st.data_ptr(), _stream(stream)))
    return m, st


# ------------------------------------------------------------------ NEXT-4: Paillier PC-MM
def paillier_mul(path: int, A: torch.Tensor, ctB: torch.Tensor, l: int, w: int, n2: int, iters: int = 4,
                 check: bool = True, stream=None) -> torch.Tensor:
    """C_ij = prod_k c_kj^{a_ik} mod n^2 on the device.
    A uint8 [m, n] (cuda), ctB int32 [n*l, L] little-endian words of residues < n2 (cuda),
    n2 a Python int of 512 / 1024 / 2048 / 3072 bits.  Returns int32 [m*l, L] (same word layout)."""
    _require_cuda()
    m, n = A.shape
    nbits = 32 * ctB.shape[-1]
    if n2.bit_length() > nbits:
        raise PCMMError(PCMM_EINVAL, "n2 does not fit the ciphertext width")
    L = nbits // 32
    words = (ctypes.c_uint32 * L)(*[(n2 >> (32 * i)) & 0xFFFFFFFF for i in range(L)])
    nb = int(load().pcmm_paillier_workspace_bytes(m, n, l, w, nbits, path))
    if nb == 0:
        raise PCMMError(PCMM_EINVAL, "invalid Paillier PC-MM arguments")
    ws = torch.empty(nb, dtype=torch.uint8, device=A.device)
    out = torch.empty((m * l, L), dtype=torch.int32, device=A.device)
    _check(load().pcmm_paillier_mul(path, _dev(A, torch.uint8, "A"), m, n, l, w, iters, words, nbits,
                                    _dev(ctB, torch.int32, "ctB"), out.data_ptr(), ws.data_ptr(), nb,
                                    _stream(stream)))
    if check:
        status(ws, stream)
    return out


def to_words(vals, L: int) -> torch.Tensor:
    """Python ints -> int32 [len, L] little-endian 32-bit words (host tensor)."""
    import numpy as np
    a = np.zeros((len(vals), L), dtype=np.uint32)
    for e, v in enumerate(vals):
        for i in range(L):
            a[e, i] = (v >> (32 * i)) & 0xFFFFFFFF
    return torch.from_numpy(a.view(np.int32))


def from_words(t: torch.Tensor) -> list:
    """int32 [count, L] words -> Python ints."""
    import numpy as np
    a = t.cpu().numpy().view(np.uint32)
    return [sum(int(a[e, i]) << (32 * i) for i in range(a.shape[1])) for e in range(a.shape[0])]


# ------------------------------------------------------------------ PC-MM
def workspace_bytes(m: int, n: int, l: int, w: int, path: int, wide: bool = False) -> int:
    """Workspace of pcmm_mul_* (wide=False: int8 / uint8 A, w <= 8) or pcmm_mul_*_wide (int32 A, w <= 16)."""
    if wide:
        return int(load().pcmm_workspace_bytes_wide(m, n, l, w, path))
    return int(load().pcmm_workspace_bytes(m, n, l, w, path))


def proj_bytes(count: int) -> int:
    return int(load().pcmm_proj_bytes(count))


def alloc_workspace(m: int, n: int, l: int, w: int, path: int, device="cuda", wide: bool = False) -> torch.Tensor:
    nb = workspace_bytes(m, n, l, w, path, wide)
    if nb == 0:
        raise PCMMError(PCMM_EINVAL, "invalid dimensions for workspace")
    return torch.empty(nb, dtype=torch.uint8, device=device)   # caching allocator: 512 B aligned


def _mul(path: int, A: torch.Tensor, ctB: torch.Tensor, l: int, w: int, is_signed: bool, iters: int,
         out_proj: torch.Tensor | None, ws: torch.Tensor | None, stream):
    _require_cuda()
    if A.dim() != 2:
        raise PCMMError(PCMM_EINVAL, "A must be [m, n]")
    m, n = A.shape
    if ctB.numel() != n * l * 128:
        raise PCMMError(PCMM_EDIM, "ctB must hold n*l canonical ciphertexts")
    if out_proj is None:
        out_proj = torch.empty(proj_bytes(m * l), dtype=torch.uint8, device=A.device)
    if A.dtype == torch.int32:                     # wide plaintexts (w <= 16): pcmm_mul_*_wide
        if ws is None:
            ws = alloc_workspace(m, n, l, w, path, A.device, wide=True)
        L = load()
        a = (_dev(A, torch.int32, "A"), m, n, l, w, int(bool(is_signed)))
        if path == SCHOOLBOOK:
            rc = L.pcmm_mul_schoolbook_wide(*a, _dev(ctB, torch.uint8, "ctB"), out_proj.data_ptr(), ws.data_ptr(),
                                            ws.numel(), _stream(stream))
        elif path == STRASSEN:
            rc = L.pcmm_mul_strassen_wide(*a, iters, _dev(ctB, torch.uint8, "ctB"), out_proj.data_ptr(),
                                          ws.data_ptr(), ws.numel(), _stream(stream))
        else:
            rc = L.pcmm_mul_cussen_wide(*a, iters, _dev(ctB, torch.uint8, "ctB"), out_proj.data_ptr(),
                                        ws.data_ptr(), ws.numel(), _stream(stream))
        _check(rc)
        return out_proj, ws
    if ws is None:
        ws = alloc_workspace(m, n, l, w, path, A.device)
    # A's bytes are read as int8 (is_signed) or uint8 (unsigned, w up to 8)
    args = (_dev(A, A.dtype if A.dtype in (torch.int8, torch.uint8) else torch.int8, "A"), m, n, l, w,
            int(bool(is_signed)))
    L = load()
    if path == SCHOOLBOOK:
        rc = L.pcmm_mul_schoolbook(*args, _dev(ctB, torch.uint8, "ctB"), out_proj.data_ptr(), ws.data_ptr(),
                                   ws.numel(), _stream(stream))
    elif path == STRASSEN:
        rc = L.pcmm_mul_strassen(*args, iters, _dev(ctB, torch.uint8, "ctB"), out_proj.data_ptr(), ws.data_ptr(),
                                 ws.numel(), _stream(stream))
    else:
        rc = L.pcmm_mul_cussen(*args, iters, _dev(ctB, torch.uint8, "ctB"), out_proj.data_ptr(), ws.data_ptr(),
                               ws.numel(), _stream(stream))
    _check(rc)
    return out_proj, ws


def mul_schoolbook(A, ctB, l, w, is_signed=False, out_proj=None, ws=None, stream=None):
    """Schoolbook PC-MM -> (projective output, workspace)."""
    return _mul(SCHOOLBOOK, A, ctB, l, w, is_signed, 0, out_proj, ws, stream)


def mul_cussen(A, ctB, l, w, is_signed=False, iters=4, out_proj=None, ws=None, stream=None):
    """Cussen PC-MM (Alg. 3) -> (projective output, workspace)."""
    return _mul(CUSSEN, A, ctB, l, w, is_signed, iters, out_proj, ws, stream)


def mul_strassen(A, ctB, l, w, is_signed=False, leaf=32, out_proj=None, ws=None, stream=None):
    """Strassen PC-MM down to `leaf`-sized blocks -> (projective output, workspace)."""
    return _mul(STRASSEN, A, ctB, l, w, is_signed, leaf, out_proj, ws, stream)


def normalize(proj: torch.Tensor, count: int, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Projective -> canonical affine bytes uint8 [count, 128]."""
    _require_cuda()
    if out is None:
        out = torch.empty((count, 128), dtype=torch.uint8, device=proj.device)
    _check(load().pcmm_normalize(proj.data_ptr(), count, _dev(out, torch.uint8, "out"), None, 0, _stream(stream)))
    return out


def status(ws: torch.Tensor, stream=None) -> int:
    """Synchronise and return the device-side status of the last mul on `ws` (raises on error)."""
    rc = load().pcmm_status(ws.data_ptr(), _stream(stream))
    _check(rc)
    return rc


def pcmm(A: torch.Tensor, ctB: torch.Tensor, l: int, w: int, is_signed: bool = False, path: int = CUSSEN,
         iters: int = 4, check: bool = True, stream=None) -> torch.Tensor:
    """C = A . Enc(B) end to end on the device: mul (Cussen, schoolbook or Strassen) + normalise.
    `iters` = Cussen's N, or Strassen's leaf block size.
    Returns canonical ciphertexts uint8 [m*l, 128] (c_ij at row i*l + j)."""
    m = A.shape[0]
    proj, ws = _mul(path, A, ctB, l, w, is_signed, iters, None, None, stream)
    out = normalize(proj, m * l, stream=stream)
    if check:
        status(ws, stream)
    return out


# ------------------------------------------------------------------ measurement hooks
def profile_enable(on: bool = True):
    _check(load().pcmm_profile_enable(int(on)))


def profile_read(max_records: int = 4096):
    names = ctypes.create_string_buffer(48 * max_records)
    ms = (ctypes.c_float * max_records)()
    n = load().pcmm_profile_read(names, ms, max_records)
    if n < 0:
        _check(n)
    out = []
    for i in range(n):
        nm = names.raw[48 * i: 48 * (i + 1)].split(b"\0", 1)[0].decode()
        out.append((nm, float(ms[i])))
    return out


# ------------------------------------------------------------------ test hooks
def test_field(op: int, a: torch.Tensor, b: torch.Tensor, stream=None) -> torch.Tensor:
    count = a.numel() // 32
    out = torch.empty((count, 32), dtype=torch.uint8, device=a.device)
    _check(load().pcmm_test_field(op, _dev(a, torch.uint8, "a"), _dev(b, torch.uint8, "b"), out.data_ptr(), count,
                                  _stream(stream)))
    return out


def test_point(op: int, p: torch.Tensor, q: torch.Tensor | None = None, v: torch.Tensor | None = None,
               stream=None) -> torch.Tensor:
    count = p.numel() // 64
    out = torch.empty((count, 64), dtype=torch.uint8, device=p.device)
    qp = _dev(q, torch.uint8, "q") if q is not None else None
    vp = _dev(v, torch.int32, "v") if v is not None else None
    _check(load().pcmm_test_point(op, _dev(p, torch.uint8, "p"), qp, vp, out.data_ptr(), count, _stream(stream)))
    return out


def test_plan(A: torch.Tensor, w: int, is_signed: bool, iters: int = 4, stream=None):
    m, n = A.shape
    levels = torch.zeros((n, 4), dtype=torch.int32, device=A.device)
    sN = torch.zeros((n, 256), dtype=torch.int16, device=A.device)
    rank = torch.zeros((n, m), dtype=torch.uint8, device=A.device)
    _check(load().pcmm_test_plan(_dev(A, A.dtype if A.dtype in (torch.int8, torch.uint8) else torch.int8, "A"), m,
                                 n, w, int(is_signed), iters, levels.data_ptr(),
                                 sN.data_ptr(), rank.data_ptr(), _stream(stream)))
    return levels, sN, rank


def bench_fp_mul(variant: int, blocks: int, threads: int, iters: int, stream=None) -> torch.Tensor:
    out = torch.empty(blocks * threads * 8, dtype=torch.int32, device="cuda")
    _check(load().pcmm_bench_fp_mul(variant, blocks, threads, iters, out.data_ptr(), _stream(stream)))
    return out
