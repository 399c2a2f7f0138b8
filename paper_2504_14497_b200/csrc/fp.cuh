// fp.cuh -- NIST P-256 prime-field arithmetic for sm_100a, 8 x 32-bit limbs.
//
// Field: p = 2^256 - 2^224 + 2^192 + 2^96 - 1 (arXiv 2504.14497).
// Representation: Montgomery form x * 2^256 mod p, little-endian 32-bit limbs,
// always fully reduced to [0, p) ("canonical"), so that equal field elements
// have equal limbs.
//
// Montgomery reduction is specialised to P-256: -p^{-1} mod 2^32 = 1, so each
// reduction quotient limb is the current low limb q, and q * p * 2^{32 i} only
// contributes +q at limbs i+3 and i+6 and +q*(2^32-1) at limbs i+7..i+8 (the -q
// at limb i cancels the limb exactly).  No multiplications are needed in the
// reduction; the 8 x 8 operand product is the only multiply work (64 products).
//
// Everything here is __host__ __device__ portable C so that the same source can
// be unit-tested on the host (tests/host_fp); device-only fast paths live in
// fp_fast.cuh and are selected under __CUDA_ARCH__.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define PCMM_HD __host__ __device__ __forceinline__
#define PCMM_HD_NOINLINE static __host__ __device__ __noinline__
#else
#define PCMM_HD inline
#define PCMM_HD_NOINLINE static
#endif

namespace pcmm {

struct fe {
    uint32_t v[8];
};

// p, little-endian limbs
#define PCMM_P0 0xffffffffu
#define PCMM_P1 0xffffffffu
#define PCMM_P2 0xffffffffu
#define PCMM_P3 0x00000000u
#define PCMM_P4 0x00000000u
#define PCMM_P5 0x00000000u
#define PCMM_P6 0x00000001u
#define PCMM_P7 0xffffffffu

PCMM_HD uint32_t p_limb(int i) {
    return (i < 3) ? 0xffffffffu : (i < 6) ? 0u : (i == 6) ? 1u : 0xffffffffu;
}

PCMM_HD void fe_zero(fe &r) {
#pragma unroll
    for (int i = 0; i < 8; i++) r.v[i] = 0;
}

// 2^256 mod p  (= 1 in Montgomery form)
PCMM_HD void fe_one_mont(fe &r) {
    r.v[0] = 0x00000001u; r.v[1] = 0x00000000u; r.v[2] = 0x00000000u; r.v[3] = 0xffffffffu;
    r.v[4] = 0xffffffffu; r.v[5] = 0xffffffffu; r.v[6] = 0xfffffffeu; r.v[7] = 0x00000000u;
}

// 2^512 mod p (to-Montgomery multiplier)
PCMM_HD void fe_r2(fe &r) {
    r.v[0] = 0x00000003u; r.v[1] = 0x00000000u; r.v[2] = 0xffffffffu; r.v[3] = 0xfffffffbu;
    r.v[4] = 0xfffffffeu; r.v[5] = 0xffffffffu; r.v[6] = 0xfffffffdu; r.v[7] = 0x00000004u;
}

// curve coefficient b in Montgomery form (b * 2^256 mod p)
PCMM_HD void fe_b_mont(fe &r) {
    r.v[0] = 0x29c4bddfu; r.v[1] = 0xd89cdf62u; r.v[2] = 0x78843090u; r.v[3] = 0xacf005cdu;
    r.v[4] = 0xf7212ed6u; r.v[5] = 0xe5a220abu; r.v[6] = 0x04874834u; r.v[7] = 0xdc30061du;
}

PCMM_HD bool fe_is_zero(const fe &a) {
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) x |= a.v[i];
    return x == 0;
}

PCMM_HD bool fe_eq(const fe &a, const fe &b) {
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) x |= a.v[i] ^ b.v[i];
    return x == 0;
}

// r = (a >= p) ? a - p : a  for a < 2^256 (single conditional subtraction),
// with an extra incoming carry bit `hi` (value = hi * 2^256 + a, < 2p).
PCMM_HD void fe_cond_sub_p(fe &r, const fe &a, uint32_t hi) {
    uint32_t d[8];
    uint64_t borrow = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        uint64_t x = (uint64_t)a.v[i] - p_limb(i) - borrow;
        d[i] = (uint32_t)x;
        borrow = (x >> 63) & 1;
    }
    // keep d iff hi == 1 or no borrow
    uint32_t use_d = hi | (uint32_t)(borrow ^ 1);
    uint32_t mask = 0u - use_d;
#pragma unroll
    for (int i = 0; i < 8; i++) r.v[i] = (d[i] & mask) | (a.v[i] & ~mask);
}

// r = a + b mod p, a, b in [0, p)
PCMM_HD void fe_add_portable(fe &r, const fe &a, const fe &b) {
    fe s;
    uint64_t c = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        c += (uint64_t)a.v[i] + b.v[i];
        s.v[i] = (uint32_t)c;
        c >>= 32;
    }
    fe_cond_sub_p(r, s, (uint32_t)c);
}

// r = a - b mod p, a, b in [0, p)
PCMM_HD void fe_sub_portable(fe &r, const fe &a, const fe &b) {
    uint32_t d[8];
    uint64_t borrow = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        uint64_t x = (uint64_t)a.v[i] - b.v[i] - borrow;
        d[i] = (uint32_t)x;
        borrow = (x >> 63) & 1;
    }
    uint32_t mask = 0u - (uint32_t)borrow;   // add p back iff a < b
    uint64_t c = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        c += (uint64_t)d[i] + (p_limb(i) & mask);
        r.v[i] = (uint32_t)c;
        c >>= 32;
    }
}

// Montgomery multiplication r = a * b * 2^-256 mod p (portable reference form).
PCMM_HD void fe_mul_portable(fe &r, const fe &a, const fe &b) {
    uint32_t t[17];
#pragma unroll
    for (int k = 0; k < 17; k++) t[k] = 0;
    // 8 x 8 operand-scanning product
#pragma unroll
    for (int i = 0; i < 8; i++) {
        uint64_t carry = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            uint64_t x = (uint64_t)a.v[i] * b.v[j] + t[i + j] + carry;
            t[i + j] = (uint32_t)x;
            carry = x >> 32;
        }
        t[i + 8] = (uint32_t)carry;
    }
    // P-256 Montgomery reduction, one limb per round
#pragma unroll
    for (int i = 0; i < 8; i++) {
        uint32_t q = t[i];
        uint32_t lo = 0u - q;               // low word of q * (2^32 - 1)
        uint32_t hi = q - (q != 0u);        // high word of q * (2^32 - 1)
        uint64_t c = (uint64_t)t[i + 3] + q;
        t[i + 3] = (uint32_t)c; c >>= 32;
        c += t[i + 4]; t[i + 4] = (uint32_t)c; c >>= 32;
        c += t[i + 5]; t[i + 5] = (uint32_t)c; c >>= 32;
        c += (uint64_t)t[i + 6] + q; t[i + 6] = (uint32_t)c; c >>= 32;
        c += (uint64_t)t[i + 7] + lo; t[i + 7] = (uint32_t)c; c >>= 32;
        c += (uint64_t)t[i + 8] + hi; t[i + 8] = (uint32_t)c; c >>= 32;
#pragma unroll
        for (int k = i + 9; k < 17; k++) { c += t[k]; t[k] = (uint32_t)c; c >>= 32; }
        t[i] = 0;
    }
    fe hiw;
#pragma unroll
    for (int i = 0; i < 8; i++) hiw.v[i] = t[8 + i];
    fe_cond_sub_p(r, hiw, t[16]);
}

}  // namespace pcmm

#if defined(__CUDA_ARCH__)
#include "fp_fast.cuh"
#endif

namespace pcmm {

PCMM_HD void fe_mul(fe &r, const fe &a, const fe &b) {
#if defined(__CUDA_ARCH__) && defined(PCMM_HAVE_FAST_MUL)
    fe_mul_fast(r, a, b);
#else
    fe_mul_portable(r, a, b);
#endif
}

PCMM_HD void fe_add(fe &r, const fe &a, const fe &b) {
#if defined(__CUDA_ARCH__) && defined(PCMM_HAVE_FAST_MUL)
    fe_add_fast(r, a, b);
#else
    fe_add_portable(r, a, b);
#endif
}

PCMM_HD void fe_sub(fe &r, const fe &a, const fe &b) {
#if defined(__CUDA_ARCH__) && defined(PCMM_HAVE_FAST_MUL)
    fe_sub_fast(r, a, b);
#else
    fe_sub_portable(r, a, b);
#endif
}

PCMM_HD void fe_neg(fe &r, const fe &a) {
    fe z;
    fe_zero(z);
    fe_sub(r, z, a);
}

PCMM_HD void fe_sqr(fe &r, const fe &a) {
#if defined(__CUDA_ARCH__) && defined(PCMM_HAVE_FAST_MUL)
    fe_sqr_fast(r, a);
#else
    fe_mul_portable(r, a, a);
#endif
}

PCMM_HD void fe_to_mont(fe &r, const fe &a) {
    fe r2;
    fe_r2(r2);
    fe_mul(r, a, r2);
}

PCMM_HD void fe_from_mont(fe &r, const fe &a) {
    fe one;
    fe_zero(one);
    one.v[0] = 1;
    fe_mul(r, a, one);
}

PCMM_HD_NOINLINE void fe_sqr_n(fe &r, const fe &a, int n) {
    r = a;
#pragma unroll 1
    for (int i = 0; i < n; i++) fe_sqr(r, r);
}

// r = a^(p-2) = a^-1 (Montgomery in / out; 0 -> 0).
// p - 2 = ffffffff 00000001 00000000 00000000 00000000 ffffffff ffffffff fffffffd
// addition chain: 255 squarings + 12 multiplications.
PCMM_HD_NOINLINE void fe_inv_fermat(fe &r, const fe &a) {
    fe x2, x3, x6, x12, x15, x30, x32, t;
    fe_sqr(x2, a);          fe_mul(x2, x2, a);       // 2^2 - 1
    fe_sqr(x3, x2);         fe_mul(x3, x3, a);       // 2^3 - 1
    fe_sqr_n(x6, x3, 3);    fe_mul(x6, x6, x3);      // 2^6 - 1
    fe_sqr_n(x12, x6, 6);   fe_mul(x12, x12, x6);    // 2^12 - 1
    fe_sqr_n(x15, x12, 3);  fe_mul(x15, x15, x3);    // 2^15 - 1
    fe_sqr_n(x30, x15, 15); fe_mul(x30, x30, x15);   // 2^30 - 1
    fe_sqr_n(x32, x30, 2);  fe_mul(x32, x32, x2);    // 2^32 - 1
    fe_sqr_n(t, x32, 32);   fe_mul(t, t, a);         // ffffffff 00000001
    fe_sqr_n(t, t, 96);                              // ... 00000000 x3
    fe_sqr_n(t, t, 32);     fe_mul(t, t, x32);       // ffffffff
    fe_sqr_n(t, t, 32);     fe_mul(t, t, x32);       // ffffffff
    fe_sqr_n(t, t, 30);     fe_mul(t, t, x30);       // 30 ones of fffffffd
    fe_sqr_n(t, t, 2);      fe_mul(r, t, a);         // "01"
}

// ---- inversion by divsteps (Bernstein and Yang, "Fast constant-time gcd
// computation and modular inversion", TCHES 2019), the default fe_inv: the
// latency of one inversion bounds the normalisation / affine passes of small
// problems, and 25 batches of 30 divsteps are ~4x shorter than the 255
// dependent squarings of Fermat's chain.
//
// State: (zeta, f, g, d, e) with f = d x and g = e x (mod p), starting from
// (-1, p, x, 0, 1).  One divstep (zeta = -(delta + 1/2)):
//   zeta < 0 and g odd:  (f, g, d, e) <- (g, (g - f)/2, e, (e - d)/2), zeta <- -zeta - 2
//   g odd otherwise:     (f, g, d, e) <- (f, (g + f)/2, d, (e + d)/2), zeta <- zeta - 1
//   g even:              (f, g, d, e) <- (f, g/2, d, e/2),              zeta <- zeta - 1
// (halvings of d, e are mod p).  30 divsteps depend only on the low 30 bits of
// f and g, so they are run on 32-bit words and collected in a 2x2 integer matrix
// M (entries <= 2^30): (f, g) <- M (f, g) / 2^30 exactly, and (d, e) <- M (d, e)
// / 2^30 mod p.  After 750 divsteps (> the 590 needed for 256-bit inputs) g = 0
// and f = +-1, so x^-1 = +-d.  Big integers are 9 signed radix-2^30 limbs.
struct s30 {
    int32_t v[9];                  // limbs 0..7 in [0, 2^30), limb 8 signed
};

constexpr int32_t kM30 = 0x3fffffff;

PCMM_HD void s30_from_words(s30 &r, const fe &a) {
    for (int i = 0; i < 9; i++) {
        const int bit = 30 * i, w = bit >> 5, sh = bit & 31;
        const uint64_t lo = w < 8 ? a.v[w] : 0, hi = w + 1 < 8 ? a.v[w + 1] : 0;
        r.v[i] = (int32_t)(((lo | (hi << 32)) >> sh) & (uint64_t)kM30);
    }
}

PCMM_HD void s30_to_words(fe &r, const s30 &a) {              // a in [0, 2^256)
    uint64_t acc = 0;
    int nb = 0, w = 0;
    for (int i = 0; i < 9; i++) {
        acc |= (uint64_t)(uint32_t)a.v[i] << nb;
        nb += 30;
        while (nb >= 32 && w < 8) {
            r.v[w++] = (uint32_t)acc;
            acc >>= 32;
            nb -= 32;
        }
    }
    while (w < 8) {
        r.v[w++] = (uint32_t)acc;
        acc >>= 32;
    }
}

// r = a + s b (s = +-1), limbs renormalised; top limb keeps the sign
PCMM_HD void s30_addmul(s30 &r, const s30 &a, const s30 &b, int32_t s) {
    int64_t c = 0;
    for (int i = 0; i < 8; i++) {
        c += (int64_t)a.v[i] + (int64_t)s * b.v[i];
        r.v[i] = (int32_t)(c & kM30);
        c >>= 30;
    }
    r.v[8] = (int32_t)(c + a.v[8] + (int64_t)s * b.v[8]);
}

PCMM_HD bool s30_neg(const s30 &a) { return a.v[8] < 0; }

// zeta, 30 divsteps on the low words of f and g -> M = (u, v; q, r)
PCMM_HD int32_t divsteps30(int32_t zeta, uint32_t f, uint32_t g, int32_t M[4]) {
    uint32_t u = 1, v = 0, q = 0, r = 1;
    for (int i = 0; i < 30; i++) {
        const uint32_t odd = 0u - (g & 1u);                       // all ones if g odd
        const uint32_t swap = odd & (uint32_t)(zeta >> 31);       // ... and zeta < 0
        // g <- g + (swap ? -f : f) when odd; the swap case then moves the old g into f
        const uint32_t fs = (f ^ swap) - swap, us = (u ^ swap) - swap, vs = (v ^ swap) - swap;
        const uint32_t g1 = g + (fs & odd), q1 = q + (us & odd), r1 = r + (vs & odd);
        // swap: f <- old g = g1 + f (g1 = g - f), u <- old q, v <- old r
        f += g1 & swap;
        u += q1 & swap;
        v += r1 & swap;
        zeta = swap ? -zeta - 2 : zeta - 1;
        g = g1 >> 1;
        q = q1;
        r = r1;
        u <<= 1;
        v <<= 1;
    }
    M[0] = (int32_t)u;
    M[1] = (int32_t)v;
    M[2] = (int32_t)q;
    M[3] = (int32_t)r;
    return zeta;
}

// (f, g) <- M (f, g) / 2^30 (exact)
PCMM_HD void s30_apply_fg(s30 &f, s30 &g, const int32_t M[4]) {
    int64_t cf = (int64_t)M[0] * f.v[0] + (int64_t)M[1] * g.v[0];
    int64_t cg = (int64_t)M[2] * f.v[0] + (int64_t)M[3] * g.v[0];
    cf >>= 30;
    cg >>= 30;
    for (int i = 1; i < 9; i++) {
        cf += (int64_t)M[0] * f.v[i] + (int64_t)M[1] * g.v[i];
        cg += (int64_t)M[2] * f.v[i] + (int64_t)M[3] * g.v[i];
        f.v[i - 1] = (int32_t)(cf & kM30);
        g.v[i - 1] = (int32_t)(cg & kM30);
        cf >>= 30;
        cg >>= 30;
    }
    f.v[8] = (int32_t)cf;
    g.v[8] = (int32_t)cg;
}

// x in (-1.5 p, 1.5 p) -> [0, p): two conditional additions and one subtraction of p
PCMM_HD void s30_reduce_1p5(s30 &x, const s30 &P) {
    if (s30_neg(x)) s30_addmul(x, x, P, 1);
    if (s30_neg(x)) s30_addmul(x, x, P, 1);
    s30 y;
    s30_addmul(y, x, P, -1);
    if (!s30_neg(y)) x = y;
}

// (d, e) <- M (d, e) / 2^30 mod p for d, e in [0, p); results in [0, p).  The
// division is made exact by adding k p with k = the low 30 bits of M (d, e)
// (sign-extended): p = -1 mod 2^30, so k p = -k mod 2^30 cancels them.
PCMM_HD void s30_apply_de(s30 &d, s30 &e, const int32_t M[4], const s30 &P) {
    int64_t cd = (int64_t)M[0] * d.v[0] + (int64_t)M[1] * e.v[0];
    int64_t ce = (int64_t)M[2] * d.v[0] + (int64_t)M[3] * e.v[0];
    const int64_t kd = (int64_t)((int32_t)((uint32_t)cd << 2) >> 2);
    const int64_t ke = (int64_t)((int32_t)((uint32_t)ce << 2) >> 2);
    cd = (cd + kd * P.v[0]) >> 30;
    ce = (ce + ke * P.v[0]) >> 30;
    for (int i = 1; i < 9; i++) {
        cd += (int64_t)M[0] * d.v[i] + (int64_t)M[1] * e.v[i] + kd * P.v[i];
        ce += (int64_t)M[2] * d.v[i] + (int64_t)M[3] * e.v[i] + ke * P.v[i];
        d.v[i - 1] = (int32_t)(cd & kM30);
        e.v[i - 1] = (int32_t)(ce & kM30);
        cd >>= 30;
        ce >>= 30;
    }
    d.v[8] = (int32_t)cd;
    e.v[8] = (int32_t)ce;
    s30_reduce_1p5(d, P);
    s30_reduce_1p5(e, P);
}

// (d, e) <- (u d + v e + md p, q d + r e + me p) / 2^30 for d, e in (-2p, p), without a reduction per
// batch: md, me add p for each negative input (u [d < 0] + v [e < 0], ...) and are then corrected so that
// the sums are multiples of 2^30 (p^-1 = -1 mod 2^30: md -= (md - cd) mod 2^30); with |u| + |v| and
// |q| + |r| <= 2^30 (30 divsteps) the results stay in (-2p, p) (the bound of Bernstein-Yang's analysis as
// used by libsecp256k1's modinv32).  Two 9-limb multiply-accumulate chains, no conditional passes.
PCMM_HD void s30_update_de(s30 &d, s30 &e, const int32_t M[4], const s30 &P) {
    const int32_t u = M[0], v = M[1], q = M[2], r = M[3];
    const int32_t sd = d.v[8] >> 31, se = e.v[8] >> 31;
    int32_t md = (u & sd) + (v & se);
    int32_t me = (q & sd) + (r & se);
    int64_t cd = (int64_t)u * d.v[0] + (int64_t)v * e.v[0];
    int64_t ce = (int64_t)q * d.v[0] + (int64_t)r * e.v[0];
    md -= (int32_t)(((uint32_t)md - (uint32_t)cd) & (uint32_t)kM30);
    me -= (int32_t)(((uint32_t)me - (uint32_t)ce) & (uint32_t)kM30);
    cd += (int64_t)P.v[0] * md;
    ce += (int64_t)P.v[0] * me;
    cd >>= 30;
    ce >>= 30;
#pragma unroll
    for (int i = 1; i < 9; i++) {
        cd += (int64_t)u * d.v[i] + (int64_t)v * e.v[i] + (int64_t)P.v[i] * md;
        ce += (int64_t)q * d.v[i] + (int64_t)r * e.v[i] + (int64_t)P.v[i] * me;
        d.v[i - 1] = (int32_t)(cd & kM30);
        e.v[i - 1] = (int32_t)(ce & kM30);
        cd >>= 30;
        ce >>= 30;
    }
    d.v[8] = (int32_t)cd;
    e.v[8] = (int32_t)ce;
}

// x^-1 = sign(f) d with d in (-2p, p) -> [0, p)
PCMM_HD void s30_finish_inverse(fe &r, s30 d, const s30 &f, const s30 &P) {
    if (s30_neg(f)) {
        s30 z;
        for (int i = 0; i < 9; i++) z.v[i] = 0;
        s30_addmul(d, z, d, -1);                              // -d in (-p, 2p)
    }
    if (s30_neg(d)) s30_addmul(d, d, P, 1);
    if (s30_neg(d)) s30_addmul(d, d, P, 1);
    s30 y;
    s30_addmul(y, d, P, -1);
    if (!s30_neg(y)) d = y;                                   // [0, 2p) -> [0, p)
    s30_to_words(r, d);
}

#ifndef PCMM_INV_LAZY_DE
#define PCMM_INV_LAZY_DE 1      // 1: s30_update_de (no per-batch reduction of d, e), 0: s30_apply_de
#endif

// plain (non-Montgomery) x^-1 mod p for x in [0, p) (0 -> 0)
PCMM_HD void fe_inv_plain_divsteps(fe &r, const fe &x) {
    fe pw;
    for (int i = 0; i < 8; i++) pw.v[i] = p_limb(i);
    s30 P, f, g, d, e;
    s30_from_words(P, pw);
    f = P;
    s30_from_words(g, x);
    for (int i = 0; i < 9; i++) {
        d.v[i] = 0;
        e.v[i] = i == 0 ? 1 : 0;
    }
    int32_t zeta = -1;
    // zeta = -(delta + 1/2) with delta starting at 1/2: the "half-delta" divstep, for which
    // 590 divsteps suffice for 256-bit inputs (Bernstein-Yang's bound, as used by
    // libsecp256k1's constant-time modinv): 20 batches of 30
#pragma unroll 1
    for (int it = 0; it < 20; it++) {
        int32_t M[4];
        zeta = divsteps30(zeta, (uint32_t)f.v[0] | ((uint32_t)f.v[1] << 30), (uint32_t)g.v[0] | ((uint32_t)g.v[1] << 30),
                          M);
#if PCMM_INV_LAZY_DE
        s30_update_de(d, e, M, P);
#else
        s30_apply_de(d, e, M, P);
#endif
        s30_apply_fg(f, g, M);
    }
#if PCMM_INV_LAZY_DE
    s30_finish_inverse(r, d, f, P);
    return;
#endif
    // f = +-1 (or p for x = 0, where d = 0): x^-1 = sign(f) d
    if (s30_neg(f)) {
        s30 z;
        for (int i = 0; i < 9; i++) z.v[i] = 0;
        s30_addmul(d, z, d, -1);                             // -d in (-p, 0]
        if (s30_neg(d)) s30_addmul(d, d, P, 1);
    }
    s30_to_words(r, d);
}

// Variable-time divsteps (original delta, eta = -delta starting at -1): runs of even g
// are shifted out at once (count trailing zeros) and an odd g has its low
// min(eta + 1, remaining, 8) bits cancelled by adding w f, w = -g / f mod 2^8 (f^-1 by
// two Newton steps) -- the same 30-divstep transition matrix as divsteps30 in far
// fewer loop trips.  Side channels are out of scope (DESIGN R11).
PCMM_HD int ctz32_hd(uint32_t x) {
#ifdef __CUDA_ARCH__
    return __ffs((int)x) - 1;
#else
    return __builtin_ctz(x);
#endif
}

PCMM_HD int32_t divsteps30_var(int32_t eta, uint32_t f, uint32_t g, int32_t M[4]) {
    uint32_t u = 1, v = 0, q = 0, r = 1;
    int i = 30;
    for (;;) {
        const int zeros = ctz32_hd(g | (0xffffffffu << i));
        g >>= zeros;
        u <<= zeros;
        v <<= zeros;
        eta -= zeros;
        i -= zeros;
        if (i == 0) break;
        if (eta < 0) {                                          // (f, g) <- (g, -f)
            uint32_t t;
            eta = -eta;
            t = f; f = g; g = 0u - t;
            t = u; u = q; q = 0u - t;
            t = v; v = r; r = 0u - t;
        }
        const int limit = (eta + 1) > i ? i : (eta + 1);
        const uint32_t m = (0xffffffffu >> (32 - limit)) & 255u;
        uint32_t fi = f;                                         // f odd: f f = 1 mod 8
        fi *= 2u - f * fi;                                       // f^-1 mod 2^6
        fi *= 2u - f * fi;                                       // f^-1 mod 2^12
        const uint32_t w = (0u - g * fi) & m;
        g += f * w;
        q += u * w;
        r += v * w;
    }
    M[0] = (int32_t)u;
    M[1] = (int32_t)v;
    M[2] = (int32_t)q;
    M[3] = (int32_t)r;
    return eta;
}

PCMM_HD bool s30_is_zero(const s30 &a) {
    int32_t o = 0;
    for (int i = 0; i < 9; i++) o |= a.v[i];
    return o == 0;
}

// plain x^-1 mod p by variable-time divsteps, stopping as soon as g = 0 (<= 25
// batches: the original divstep needs <= 741 steps for 256-bit inputs)
PCMM_HD void fe_inv_plain_divsteps_var(fe &r, const fe &x) {
    fe pw;
    for (int i = 0; i < 8; i++) pw.v[i] = p_limb(i);
    s30 P, f, g, d, e;
    s30_from_words(P, pw);
    f = P;
    s30_from_words(g, x);
    for (int i = 0; i < 9; i++) {
        d.v[i] = 0;
        e.v[i] = i == 0 ? 1 : 0;
    }
    int32_t eta = -1;
#pragma unroll 1
    for (int it = 0; it < 26 && !s30_is_zero(g); it++) {
        int32_t M[4];
        eta = divsteps30_var(eta, (uint32_t)f.v[0] | ((uint32_t)f.v[1] << 30), (uint32_t)g.v[0] | ((uint32_t)g.v[1] << 30),
                             M);
#if PCMM_INV_LAZY_DE
        s30_update_de(d, e, M, P);
#else
        s30_apply_de(d, e, M, P);
#endif
        s30_apply_fg(f, g, M);
    }
#if PCMM_INV_LAZY_DE
    s30_finish_inverse(r, d, f, P);
    return;
#endif
    if (s30_neg(f)) {
        s30 z;
        for (int i = 0; i < 9; i++) z.v[i] = 0;
        s30_addmul(d, z, d, -1);
        if (s30_neg(d)) s30_addmul(d, d, P, 1);
    }
    s30_to_words(r, d);
}

PCMM_HD_NOINLINE void fe_inv_var(fe &r, const fe &a) {
    fe inv, r2;
    fe_inv_plain_divsteps_var(inv, a);
    fe_r2(r2);
    fe_mul(inv, inv, r2);
    fe_mul(r, inv, r2);
}

// r = a^-1 in Montgomery form: plain inverse of the Montgomery residue a R, times R^3
// (two Montgomery products by R^2 mod p): (a R)^-1 R^2 = a^-1 R.  0 -> 0.
#ifndef PCMM_INV_VAR
#define PCMM_INV_VAR 1          // 1: fe_inv runs the variable-time divsteps (256^3: k_normalize 0.091 -> 0.082 ms, k_affine 0.302 -> 0.289; tiny 0.200 -> 0.188 ms); 0: constant-time
#endif
PCMM_HD_NOINLINE void fe_inv(fe &r, const fe &a) {
    fe inv, r2;
#if PCMM_INV_VAR
    fe_inv_plain_divsteps_var(inv, a);
#else
    fe_inv_plain_divsteps(inv, a);
#endif
    fe_r2(r2);
    fe_mul(inv, inv, r2);
    fe_mul(r, inv, r2);
}

// big-endian 32 bytes -> limbs (no reduction); returns 1 iff value < p
PCMM_HD int fe_from_be_bytes(fe &r, const uint8_t *b) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const uint8_t *w = b + 28 - 4 * i;
        r.v[i] = ((uint32_t)w[0] << 24) | ((uint32_t)w[1] << 16) | ((uint32_t)w[2] << 8) | (uint32_t)w[3];
    }
    uint64_t borrow = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        uint64_t x = (uint64_t)r.v[i] - p_limb(i) - borrow;
        borrow = (x >> 63) & 1;
    }
    return (int)borrow;
}

PCMM_HD void fe_to_be_bytes(uint8_t *b, const fe &a) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
        uint8_t *w = b + 28 - 4 * i;
        w[0] = (uint8_t)(a.v[i] >> 24); w[1] = (uint8_t)(a.v[i] >> 16);
        w[2] = (uint8_t)(a.v[i] >> 8);  w[3] = (uint8_t)a.v[i];
    }
}

}  // namespace pcmm
