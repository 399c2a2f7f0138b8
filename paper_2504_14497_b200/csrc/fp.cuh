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
PCMM_HD_NOINLINE void fe_inv(fe &r, const fe &a) {
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
