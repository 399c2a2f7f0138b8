"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no field, curve, ElGamal or
PC-MM code).  It only draws the random numbers the method consumes, so that
the CPU oracle (`oracle/`) and the CUDA path (`paper_2504_14497_b200/`) see
exactly the same inputs while sharing no code with each other.

Randomness (reading R12; the paper fixes no PRNG, PAPER.md:179-180
only says x and r are "sampled uniformly at random from [1, q-1]"):

* generator: SplitMix64(seed), one 64-bit draw per call;
* draw order: secret key x; then A row-major (m x n); then B row-major (n x l);
  then the per-ciphertext randomness r row-major over (k, j);
* a 256-bit value is 4 consecutive draws concatenated big-endian and is
  rejected (and redrawn) unless it lies in [1, q-1];
* a small entry in [lo, hi] is lo + (draw mod (hi - lo + 1)); all ranges used
  here have power-of-two sizes, so this is unbiased.

`libpcmm.so`'s `pcmm_keygen(seed)` re-derives x with its own SplitMix64 (same
counter-based generator, separate implementation), which the GPU tests check.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# Group order of NIST P-256 (a constant of the curve; hex from
# SEC 2 / `openssl ecparam -name prime256v1 -param_enc explicit`).  Used only
# for rejection sampling of x and r.
P256_ORDER = int("ffffffff00000000ffffffffffffffffbce6faada7179e84f3b9cac2fc632551", 16)

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_MASK64 = (1 << 64) - 1


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


class SplitMix64:
    """SplitMix64 (Steele, Lea, Flood 2014): state += gamma; output = mix(state)."""

    def __init__(self, seed: int):
        self.state = seed & _MASK64

    def next_block(self, count: int) -> np.ndarray:
        """The next `count` draws as a uint64 array (vectorised; counter-based)."""
        if count <= 0:
            return np.zeros(0, dtype=np.uint64)
        idx = np.arange(1, count + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            states = np.uint64(self.state) + idx * _GAMMA
            out = _mix(states)
        self.state = int(states[-1])
        return out

    def next(self) -> int:
        return int(self.next_block(1)[0])

    def small(self, lo: int, hi: int, count: int) -> np.ndarray:
        span = hi - lo + 1
        d = self.next_block(count)
        return (lo + (d % np.uint64(span)).astype(np.int64)).astype(np.int64)

    def scalar256(self) -> int:
        while True:
            d = self.next_block(4)
            v = (int(d[0]) << 192) | (int(d[1]) << 128) | (int(d[2]) << 64) | int(d[3])
            if 1 <= v <= P256_ORDER - 1:
                return v

    def scalars256(self, count: int) -> list[int]:
        """`count` scalars in [1, q-1], in draw order (fast path + exact fallback)."""
        d = self.next_block(4 * count)
        words = d.reshape(count, 4) if count else d.reshape(0, 4)
        out: list[int] = []
        for i in range(count):
            w = words[i]
            v = (int(w[0]) << 192) | (int(w[1]) << 128) | (int(w[2]) << 64) | int(w[3])
            if not (1 <= v <= P256_ORDER - 1):
                # Rejection (probability ~2^-32 per value): rewind to just after
                # this value's 4 draws and continue sequentially from there.
                self.state = (int(self.state) - (4 * (count - i - 1)) * int(_GAMMA)) & _MASK64
                rest = [self.scalar256()] + self.scalars256(count - i - 1)
                return out + rest
            out.append(v)
        return out


def scalars_to_be_bytes(vals: list[int]) -> np.ndarray:
    """[count] ints -> uint8 [count, 32] big-endian."""
    out = np.zeros((len(vals), 32), dtype=np.uint8)
    for i, v in enumerate(vals):
        out[i] = np.frombuffer(v.to_bytes(32, "big"), dtype=np.uint8)
    return out


@dataclass(frozen=True)
class Config:
    """One BASELINE.json configuration."""
    name: str
    m: int
    n: int
    l: int
    w: int                # plaintext bit width of A
    signed: bool          # A in [-2^(w-1), 2^(w-1)) instead of [0, 2^w)
    b_lo: int
    b_hi: int
    seed: int

    @property
    def a_range(self) -> tuple[int, int]:
        if self.signed:
            return -(1 << (self.w - 1)), (1 << (self.w - 1)) - 1
        return 0, (1 << self.w) - 1


CONFIGS = {
    "tiny": Config("tiny", 8, 8, 8, 2, False, 0, 3, 0),
    "c64": Config("c64", 64, 64, 64, 4, False, 0, 15, 1),
    "c256": Config("c256", 256, 256, 256, 4, False, 0, 255, 2),
    "c512": Config("c512", 512, 512, 512, 2, False, 0, 255, 3),
    "ml": Config("ml", 128, 1024, 64, 4, True, 0, 255, 4),
}


@dataclass
class Instance:
    cfg: Config
    x: int                 # secret key, in [1, q-1]
    A: np.ndarray          # [m, n] int8 (signed) or uint8 (unsigned), the boundary's byte layout
    B: np.ndarray          # int32 [n, l]
    r_be: np.ndarray       # uint8 [n*l, 32]  big-endian encryption randomness, (k, j) row-major
    x_be: bytes


def make_instance(cfg: Config, m: int | None = None, n: int | None = None, l: int | None = None,
                  seed: int | None = None) -> Instance:
    """Draw (x, A, B, r) for `cfg` (optionally with overridden shape / seed)."""
    m = cfg.m if m is None else m
    n = cfg.n if n is None else n
    l = cfg.l if l is None else l
    seed = cfg.seed if seed is None else seed
    g = SplitMix64(seed)
    x = g.scalar256()
    lo, hi = cfg.a_range
    # w <= 8: one byte per entry (int8 signed / uint8 unsigned, the pcmm_mul_* ABI);
    # w > 8 (the paper's t = 12, 16 grid): int32 (the pcmm_mul_*_wide ABI)
    dt = (np.int8 if cfg.signed else np.uint8) if cfg.w <= 8 else np.int32
    A = g.small(lo, hi, m * n).reshape(m, n).astype(dt)
    B = g.small(cfg.b_lo, cfg.b_hi, n * l).reshape(n, l).astype(np.int32)
    r = g.scalars256(n * l)
    c = Config(cfg.name, m, n, l, cfg.w, cfg.signed, cfg.b_lo, cfg.b_hi, seed)
    return Instance(c, x, A, B, scalars_to_be_bytes(r), x.to_bytes(32, "big"))


def keygen_secret(seed: int) -> int:
    """The secret key x that `make_instance(seed=...)` (and pcmm_keygen) derive."""
    return SplitMix64(seed).scalar256()


# ------------------------------------------------------------- NEXT-4: Paillier key material
def _probable_prime(v: int, g: "SplitMix64", rounds: int = 24) -> bool:
    """Miller-Rabin with bases drawn from `g` (key material only, not the method's arithmetic)."""
    if v < 4:
        return v in (2, 3)
    if v % 2 == 0:
        return False
    for sp in (3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if v % sp == 0:
            return v == sp
    d, s = v - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for _ in range(rounds):
        a = 2 + g.next() % (v - 3)
        x = pow(a, d, v)
        if x in (1, v - 1):
            continue
        for _ in range(s - 1):
            x = x * x % v
            if x == v - 1:
                break
        else:
            return False
    return True


def paillier_primes(seed: int, nbits: int) -> tuple[int, int]:
    """Deterministic primes p != q of nbits/2 bits each (top two bits set so that n = p q has
    exactly nbits bits) with gcd(p q, (p-1)(q-1)) = 1."""
    from math import gcd
    g = SplitMix64(seed ^ 0x5A5A5A5A5A5A5A5A)
    half = nbits // 2
    out = []
    while len(out) < 2:
        words = [g.next() for _ in range((half + 63) // 64)]
        v = 0
        for w in words:
            v = (v << 64) | w
        v &= (1 << half) - 1
        v |= (3 << (half - 2)) | 1
        if _probable_prime(v, g) and v not in out:
            out.append(v)
    p, q = out
    assert gcd(p * q, (p - 1) * (q - 1)) == 1
    return p, q


def paillier_random_units(seed: int, n: int, count: int) -> list[int]:
    """`count` values r in [1, n-1] with gcd(r, n) = 1 (encryption randomness)."""
    from math import gcd
    g = SplitMix64(seed ^ 0x3C3C3C3C3C3C3C3C)
    words = (n.bit_length() + 63) // 64
    out = []
    while len(out) < count:
        v = 0
        for _ in range(words):
            v = (v << 64) | g.next()
        v %= n
        if v and gcd(v, n) == 1:
            out.append(v)
    return out
