"""CPU oracle for PC-MM over EC-ElGamal / NIST P-256 (arXiv 2504.14497).

TEST INFRASTRUCTURE.  Only `tests/`, `__graft_entry__.smoke()` and bench.py's
`cpu_baseline` / `--impl reference` legs may import this package.  The product
path (`paper_2504_14497_b200/`) never imports, links or executes it, and the two
share no code (see oracle/oracle.c's header for the passages followed).

The arithmetic lives in `oracle/oracle.c` (plain C: own 4x64-bit bignum,
Jacobian curve arithmetic with explicit special cases, Alg. 1 ladder, Alg. 2 /
Alg. 3); this module only builds it with gcc and marshals numpy arrays.

Parity status: every exported function is pinned by `tests/test_oracle_*.py`
(closed forms, library-checked scalar multiples, homomorphic identities,
brute-force tiny cases, the paper's appendix tables).  The paper's Fig. 2 / Fig.
4 toy vectors exist only as images: those worked
examples are "parity unpinned" beyond their printed operation counts.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

PCMM_EDECODE = -5


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc -O2 (plain C, pthreads)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread",
                               "-fvisibility=hidden", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            u8p = ctypes.POINTER(ctypes.c_uint8)
            i64p = ctypes.POINTER(ctypes.c_int64)
            u64p = ctypes.POINTER(ctypes.c_uint64)
            L.oracle_modop.argtypes = [ctypes.c_int, ctypes.c_int, u8p, u8p, u8p]
            L.oracle_point_on_curve.argtypes = [u8p]
            L.oracle_point_add.argtypes = [u8p, u8p, u8p]
            L.oracle_point_dbl.argtypes = [u8p, u8p]
            L.oracle_point_neg.argtypes = [u8p, u8p]
            L.oracle_scalar_mul.argtypes = [u8p, u8p, u8p]
            L.oracle_scalar_mul_base.argtypes = [u8p, u8p]
            L.oracle_ladder_mul.argtypes = [ctypes.c_uint64, ctypes.c_int, u8p, u8p, u64p]
            L.oracle_generator.argtypes = [u8p]
            L.oracle_pubkey.argtypes = [u8p, u8p]
            L.oracle_encrypt.argtypes = [u8p, ctypes.c_int64, i64p, u8p, u8p, ctypes.c_int]
            L.oracle_closed_form.argtypes = [u8p, ctypes.c_int, ctypes.POINTER(ctypes.c_int32), i64p, u8p, u8p]
            L.oracle_decrypt.argtypes = [u8p, ctypes.c_int64, u8p, ctypes.c_int64, ctypes.c_int64, i64p,
                                         ctypes.POINTER(ctypes.c_int32)]
            L.oracle_cussen_counts.argtypes = [i64p, ctypes.c_int, ctypes.c_int, i64p, ctypes.POINTER(ctypes.c_int)]
            L.oracle_cussen_plan.argtypes = [i64p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int), i64p,
                                             ctypes.POINTER(ctypes.c_int)]
            L.oracle_cussen_vs_mul_plain.argtypes = [i64p, ctypes.c_int, ctypes.c_int64, ctypes.c_int, i64p]
            L.oracle_cussen_vs_mul_encrypted.argtypes = [i64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, u8p, u8p,
                                                         u64p]
            L.oracle_pcmm.argtypes = [ctypes.c_int] * 6 + [ctypes.POINTER(ctypes.c_int32), u8p, u8p, ctypes.c_int,
                                                          u64p]
            L.oracle_inner_product.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int32), u8p, u8p]
            L.oracle_init()
            _lib = L
    return _lib


def _p(a: np.ndarray, ct=ctypes.c_uint8):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _b32(v: int) -> np.ndarray:
    return np.frombuffer(int(v).to_bytes(32, "big"), dtype=np.uint8).copy()


def _buf(n: int) -> np.ndarray:
    return np.zeros(n, dtype=np.uint8)


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"oracle {what} failed with status {rc}")


# ------------------------------------------------------------ field / scalars
FIELD_P, ORDER_Q = 0, 1


def modop(which: int, op: str, a: int, b: int = 0) -> int:
    code = {"add": 0, "sub": 1, "mul": 2, "inv": 3, "pow": 4}[op]
    out = _buf(32)
    _check(lib().oracle_modop(which, code, _p(_b32(a)), _p(_b32(b)), _p(out)), "modop")
    return int.from_bytes(out.tobytes(), "big")


# ------------------------------------------------------------- group ops
def generator() -> bytes:
    out = _buf(64)
    lib().oracle_generator(_p(out))
    return out.tobytes()


def _pt(b: bytes) -> np.ndarray:
    a = np.frombuffer(bytes(b), dtype=np.uint8).copy()
    assert a.size == 64
    return a


def on_curve(pt: bytes) -> bool:
    return bool(lib().oracle_point_on_curve(_p(_pt(pt))))


def point_add(p: bytes, q: bytes) -> bytes:
    out = _buf(64)
    _check(lib().oracle_point_add(_p(_pt(p)), _p(_pt(q)), _p(out)), "point_add")
    return out.tobytes()


def point_dbl(p: bytes) -> bytes:
    out = _buf(64)
    _check(lib().oracle_point_dbl(_p(_pt(p)), _p(out)), "point_dbl")
    return out.tobytes()


def point_neg(p: bytes) -> bytes:
    out = _buf(64)
    _check(lib().oracle_point_neg(_p(_pt(p)), _p(out)), "point_neg")
    return out.tobytes()


def scalar_mul(k: int, p: bytes) -> bytes:
    out = _buf(64)
    _check(lib().oracle_scalar_mul(_p(_b32(k % (1 << 256))), _p(_pt(p)), _p(out)), "scalar_mul")
    return out.tobytes()


def scalar_mul_base(k: int) -> bytes:
    out = _buf(64)
    _check(lib().oracle_scalar_mul_base(_p(_b32(k % (1 << 256))), _p(out)), "scalar_mul_base")
    return out.tobytes()


def ladder_mul(k: int, t: int, p: bytes):
    """Alg. 1 ladder; returns (point, (adds, dbls, ecsm, bits))."""
    out = _buf(64)
    cnt = np.zeros(4, dtype=np.uint64)
    _check(lib().oracle_ladder_mul(k, t, _p(_pt(p)), _p(out), _p(cnt, ctypes.c_uint64)), "ladder")
    return out.tobytes(), tuple(int(c) for c in cnt)


# ------------------------------------------------------------- EC-ElGamal
def pubkey(x: int) -> bytes:
    out = _buf(64)
    _check(lib().oracle_pubkey(_p(_b32(x)), _p(out)), "pubkey")
    return out.tobytes()


def encrypt(H: bytes, b: np.ndarray, r_be: np.ndarray, threads: int | None = None) -> np.ndarray:
    """b: int [count]; r_be: uint8 [count, 32].  -> uint8 [count, 128]."""
    b = np.ascontiguousarray(np.asarray(b).reshape(-1), dtype=np.int64)
    r = np.ascontiguousarray(r_be, dtype=np.uint8).reshape(-1, 32)
    assert r.shape[0] == b.size
    out = np.zeros((b.size, 128), dtype=np.uint8)
    th = threads if threads else (os.cpu_count() or 1)
    _check(lib().oracle_encrypt(_p(_pt(H)), b.size, _p(b, ctypes.c_int64), _p(r), _p(out), th), "encrypt")
    return out


def closed_form(x: int, a_row, b_col, r_col_be) -> bytes:
    """Eq. 5: Enc(sum a_k b_k) = (R G, (x R + c) G), R = sum a_k r_k mod q."""
    a = np.ascontiguousarray(np.asarray(a_row).astype(np.int32)).reshape(-1)
    b = np.ascontiguousarray(b_col, dtype=np.int64).reshape(-1)
    r = np.ascontiguousarray(r_col_be, dtype=np.uint8).reshape(a.size, 32)
    out = _buf(128)
    _check(lib().oracle_closed_form(_p(_b32(x)), a.size, _p(a, ctypes.c_int32), _p(b, ctypes.c_int64), _p(r),
                                    _p(out)), "closed_form")
    return out.tobytes()


def decrypt(x: int, ct: np.ndarray, lo: int, hi: int):
    """-> (m int64 [count], status int32 [count]); status -5 = not in [lo, hi]."""
    ct = np.ascontiguousarray(ct, dtype=np.uint8).reshape(-1, 128)
    m = np.zeros(ct.shape[0], dtype=np.int64)
    st = np.zeros(ct.shape[0], dtype=np.int32)
    _check(lib().oracle_decrypt(_p(_b32(x)), ct.shape[0], _p(ct), lo, hi, _p(m, ctypes.c_int64),
                                _p(st, ctypes.c_int32)), "decrypt")
    return m, st


# ------------------------------------------------------------- Cussen
def cussen_counts(a, N: int = 4):
    """-> (mults = n_N, paper-model adds = sum_{w<N} n_w, executed adds, [n_1..n_N])."""
    a = np.ascontiguousarray(np.asarray(a).reshape(-1), dtype=np.int64)
    out = np.zeros(3, dtype=np.int64)
    lev = (ctypes.c_int * N)()
    _check(lib().oracle_cussen_counts(_p(a, ctypes.c_int64), a.size, N, _p(out, ctypes.c_int64), lev), "counts")
    return int(out[0]), int(out[1]), int(out[2]), list(lev)


def cussen_plan(a, N: int = 4):
    """-> list over levels w=1..N of (s^(w) sorted values, ptr^(w) for elements of level w-1)."""
    a = np.ascontiguousarray(np.asarray(a).reshape(-1), dtype=np.int64)
    L = max(a.size, 1)
    n = (ctypes.c_int * N)()
    s = np.zeros(N * L, dtype=np.int64)
    ptr = np.zeros(N * L, dtype=np.int32)
    _check(lib().oracle_cussen_plan(_p(a, ctypes.c_int64), a.size, N, n, _p(s, ctypes.c_int64),
                                    ptr.ctypes.data_as(ctypes.POINTER(ctypes.c_int))), "plan")
    levels = []
    prev = a.size
    for w in range(N):
        levels.append((s[w * L: w * L + n[w]].copy(), ptr[w * L: w * L + prev].copy()))
        prev = n[w]
    return levels


def cussen_vs_mul_plain(a, C: int, N: int = 4) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a).reshape(-1), dtype=np.int64)
    out = np.zeros(a.size, dtype=np.int64)
    _check(lib().oracle_cussen_vs_mul_plain(_p(a, ctypes.c_int64), a.size, C, N, _p(out, ctypes.c_int64)),
           "vs_mul_plain")
    return out


def cussen_vs_mul_encrypted(a, t: int, ct: bytes, N: int = 4):
    a = np.ascontiguousarray(np.asarray(a).reshape(-1), dtype=np.int64)
    c = np.frombuffer(bytes(ct), dtype=np.uint8).copy()
    out = np.zeros((a.size, 128), dtype=np.uint8)
    cnt = np.zeros(4, dtype=np.uint64)
    _check(lib().oracle_cussen_vs_mul_encrypted(_p(a, ctypes.c_int64), a.size, t, N, _p(c), _p(out),
                                                _p(cnt, ctypes.c_uint64)), "vs_mul_encrypted")
    return out, tuple(int(x) for x in cnt)


# ------------------------------------------------------------- PC-MM
SCHOOLBOOK, CUSSEN = 0, 1


def pcmm(path: int, A: np.ndarray, ct: np.ndarray, l: int, t: int, N: int = 4, threads: int | None = None):
    """A: integer [m, n] (int8 / uint8 / wider, |a| < 2^31); ct: uint8 [n*l, 128] canonical, (k, j) row-major.
    -> (out uint8 [m*l, 128], (adds, dbls, ecsm, ecsm_bits))."""
    A = np.ascontiguousarray(np.asarray(A).astype(np.int32))
    m, n = A.shape
    ct = np.ascontiguousarray(ct, dtype=np.uint8).reshape(n * l, 128)
    out = np.zeros((m * l, 128), dtype=np.uint8)
    cnt = np.zeros(4, dtype=np.uint64)
    th = threads if threads else (os.cpu_count() or 1)
    _check(lib().oracle_pcmm(path, m, n, l, t, N, _p(A, ctypes.c_int32), _p(ct), _p(out), th,
                             _p(cnt, ctypes.c_uint64)), "pcmm")
    return out, tuple(int(x) for x in cnt)


def inner_product(a_row: np.ndarray, ct_col: np.ndarray) -> bytes:
    """Enc(sum_k a_k b_k) from a row of A and a column of n ciphertexts (definition)."""
    a = np.ascontiguousarray(np.asarray(a_row).astype(np.int32)).reshape(-1)
    c = np.ascontiguousarray(ct_col, dtype=np.uint8).reshape(a.size, 128)
    out = _buf(128)
    _check(lib().oracle_inner_product(a.size, _p(a, ctypes.c_int32), _p(c), _p(out)), "inner_product")
    return out.tobytes()


# ------------------------------------------------------------- cost model
def paper_model_equiv_adds_cussen(levels_per_col, t: int, m: int, n: int, l: int, N: int = 4) -> int:
    """Equivalent point additions of Alg. 3 under the paper's cost model (P:419-420,
    Table A6): per column k and output column j, 2 * n_N ECSMs of 2t each plus
    2 * sum_{w<N} n_w reconstruction adds; plus 2 m l (n-1) accumulation adds."""
    tot = 0
    for lev in levels_per_col:
        tot += l * (4 * t * lev[N - 1] + 2 * sum(lev[: N - 1]))
    return tot + 2 * m * l * (n - 1)


def paper_model_equiv_adds_schoolbook(t: int, m: int, n: int, l: int) -> int:
    """m n l plaintext-ciphertext multiplications (2 ECSMs of 2t each) and
    m l (n-1) ciphertext additions (2 point adds each)."""
    return 4 * t * m * n * l + 2 * m * l * (n - 1)
