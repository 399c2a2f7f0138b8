// fp_fast.cuh -- sm_100a fast paths for fp.cuh (device only; included by fp.cuh
// under __CUDA_ARCH__).  Same representation and results as the portable code:
// Montgomery form, fully reduced to [0, p).
//
// SASS shape (tools/k11_imad_probe.cu measured on B200): IMAD.WIDE.U32 issues at
// half the IMAD rate (2 slots of the FMA pipe) and is the only 32x32->64 product
// form worth using (IMAD + IMAD.HI costs 3 slots); carries live on the ALU pipe
// (IADD3 / IADD3.X).  PTX carry flags do not survive between asm statements, so
// every carry chain below is a single asm statement.
//
//  * product: operand scanning, 8 rows; in row i the 64-bit product
//    a_i*b_j + T[i+j] never overflows, so each IMAD.WIDE also absorbs the
//    running column word; the row's high words are then added with one carry
//    chain (8 ALU ops per row, 64 IMAD.WIDE total);
//  * reduction: P-256 Montgomery with 64-bit quotient digits (-p^-1 = 1 mod
//    2^64): 4 rounds, each one 7-word carry chain; carries deferred between
//    rounds (see below);
//  * final conditional subtraction of p with a LOP3 select.
#pragma once

#define PCMM_HAVE_FAST_MUL 1


namespace pcmm {

// operand scanning (V3): IMAD.WIDE folds the running column word; per-row add chain
__device__ __forceinline__ void fe_prod_os(uint32_t T[16], const fe &a, const fe &b) {
    uint32_t l[8], h[8];
    // ---- row 0
#pragma unroll
    for (int j = 0; j < 8; j++) {
        uint64_t p = (uint64_t)a.v[0] * b.v[j];
        l[j] = (uint32_t)p;
        h[j] = (uint32_t)(p >> 32);
    }
    T[0] = l[0];
    asm("add.cc.u32 %0, %8, %9;\n\t"
        "addc.cc.u32 %1, %10, %11;\n\t"
        "addc.cc.u32 %2, %12, %13;\n\t"
        "addc.cc.u32 %3, %14, %15;\n\t"
        "addc.cc.u32 %4, %16, %17;\n\t"
        "addc.cc.u32 %5, %18, %19;\n\t"
        "addc.cc.u32 %6, %20, %21;\n\t"
        "addc.u32 %7, %22, 0;"
        : "=r"(T[1]), "=r"(T[2]), "=r"(T[3]), "=r"(T[4]), "=r"(T[5]), "=r"(T[6]), "=r"(T[7]), "=r"(T[8])
        : "r"(l[1]), "r"(h[0]), "r"(l[2]), "r"(h[1]), "r"(l[3]), "r"(h[2]), "r"(l[4]), "r"(h[3]), "r"(l[5]),
          "r"(h[4]), "r"(l[6]), "r"(h[5]), "r"(l[7]), "r"(h[6]), "r"(h[7]));
    // ---- rows 1..7
#pragma unroll
    for (int i = 1; i < 8; i++) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            uint64_t p = (uint64_t)a.v[i] * b.v[j] + T[i + j];
            l[j] = (uint32_t)p;
            h[j] = (uint32_t)(p >> 32);
        }
        T[i] = l[0];
        asm("add.cc.u32 %0, %8, %9;\n\t"
            "addc.cc.u32 %1, %10, %11;\n\t"
            "addc.cc.u32 %2, %12, %13;\n\t"
            "addc.cc.u32 %3, %14, %15;\n\t"
            "addc.cc.u32 %4, %16, %17;\n\t"
            "addc.cc.u32 %5, %18, %19;\n\t"
            "addc.cc.u32 %6, %20, %21;\n\t"
            "addc.u32 %7, %22, 0;"
            : "=r"(T[i + 1]), "=r"(T[i + 2]), "=r"(T[i + 3]), "=r"(T[i + 4]), "=r"(T[i + 5]), "=r"(T[i + 6]),
              "=r"(T[i + 7]), "=r"(T[i + 8])
            : "r"(l[1]), "r"(h[0]), "r"(l[2]), "r"(h[1]), "r"(l[3]), "r"(h[2]), "r"(l[4]), "r"(h[3]), "r"(l[5]),
              "r"(h[4]), "r"(l[6]), "r"(h[5]), "r"(l[7]), "r"(h[6]), "r"(h[7]));
    }
}

// Even/odd product scanning: the 64 products a_j b_i are summed into two
// accumulators, E (products at even word offsets, i + j even) and O (odd
// offsets, stored one word down so that its pairs are aligned too).  A row i of
// either accumulator is a chain of four mad.lo.cc / madc.hi.cc pairs, which
// ptxas fuses into IMAD.WIDE.U32(.X) with the aligned 64-bit accumulator pair as
// addend and the carry in a predicate: no zeroed high words and no separate add
// chain per row.  The carry out of a chain lands in the word above it, which
// holds at most earlier carries (never a product word) at that point, so
// `addc` there cannot overflow.  T = E + O 2^32 at the end (one add chain).
#define PCMM_CHAIN4C(d0, d1, d2, d3, d4, d5, d6, d7, c, x0, x1, x2, x3, y)                        \
    asm("mad.lo.cc.u32 %0, %9, %13, %0;\n\t"                                                      \
        "madc.hi.cc.u32 %1, %9, %13, %1;\n\t"                                                     \
        "madc.lo.cc.u32 %2, %10, %13, %2;\n\t"                                                    \
        "madc.hi.cc.u32 %3, %10, %13, %3;\n\t"                                                    \
        "madc.lo.cc.u32 %4, %11, %13, %4;\n\t"                                                    \
        "madc.hi.cc.u32 %5, %11, %13, %5;\n\t"                                                    \
        "madc.lo.cc.u32 %6, %12, %13, %6;\n\t"                                                    \
        "madc.hi.cc.u32 %7, %12, %13, %7;\n\t"                                                    \
        "addc.u32 %8, %8, 0;"                                                                     \
        : "+r"(d0), "+r"(d1), "+r"(d2), "+r"(d3), "+r"(d4), "+r"(d5), "+r"(d6), "+r"(d7), "+r"(c) \
        : "r"(x0), "r"(x1), "r"(x2), "r"(x3), "r"(y))
#define PCMM_CHAIN4(d0, d1, d2, d3, d4, d5, d6, d7, x0, x1, x2, x3, y)                            \
    asm("mad.lo.cc.u32 %0, %8, %12, %0;\n\t"                                                      \
        "madc.hi.cc.u32 %1, %8, %12, %1;\n\t"                                                     \
        "madc.lo.cc.u32 %2, %9, %12, %2;\n\t"                                                     \
        "madc.hi.cc.u32 %3, %9, %12, %3;\n\t"                                                     \
        "madc.lo.cc.u32 %4, %10, %12, %4;\n\t"                                                    \
        "madc.hi.cc.u32 %5, %10, %12, %5;\n\t"                                                    \
        "madc.lo.cc.u32 %6, %11, %12, %6;\n\t"                                                    \
        "madc.hi.u32 %7, %11, %12, %7;"                                                           \
        : "+r"(d0), "+r"(d1), "+r"(d2), "+r"(d3), "+r"(d4), "+r"(d5), "+r"(d6), "+r"(d7)          \
        : "r"(x0), "r"(x1), "r"(x2), "r"(x3), "r"(y))

__device__ __forceinline__ void fe_prod_eo(uint32_t T[16], const fe &a, const fe &b) {
    uint32_t E[16], O[16];                       // O[k] = word k + 1
    // row 0: plain products
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const uint64_t pe = (uint64_t)a.v[2 * j] * b.v[0];
        const uint64_t po = (uint64_t)a.v[2 * j + 1] * b.v[0];
        E[2 * j] = (uint32_t)pe;
        E[2 * j + 1] = (uint32_t)(pe >> 32);
        O[2 * j] = (uint32_t)po;
        O[2 * j + 1] = (uint32_t)(po >> 32);
    }
#pragma unroll
    for (int k = 8; k < 16; k++) {
        E[k] = 0;
        O[k] = 0;
    }
    const uint32_t a0 = a.v[0], a1 = a.v[1], a2 = a.v[2], a3 = a.v[3];
    const uint32_t a4 = a.v[4], a5 = a.v[5], a6 = a.v[6], a7 = a.v[7];
#pragma unroll
    for (int i = 1; i < 8; i++) {
        const uint32_t bi = b.v[i];
        if (i & 1) {
            // even a-limbs -> odd offsets i..i+7 = O[i-1..i+6], carry O[i+7]
            PCMM_CHAIN4C(O[i - 1], O[i], O[i + 1], O[i + 2], O[i + 3], O[i + 4], O[i + 5], O[i + 6], O[i + 7],
                         a0, a2, a4, a6, bi);
            // odd a-limbs -> even offsets i+1..i+8 = E[i+1..i+8], carry E[i+9] (none for i = 7)
            if (i < 7) {
                PCMM_CHAIN4C(E[i + 1], E[i + 2], E[i + 3], E[i + 4], E[i + 5], E[i + 6], E[i + 7], E[i + 8],
                             E[(i + 9) & 15], a1, a3, a5, a7, bi);
            } else {
                PCMM_CHAIN4(E[8], E[9], E[10], E[11], E[12], E[13], E[14], E[15], a1, a3, a5, a7, bi);
            }
        } else {
            // even a-limbs -> even offsets E[i..i+7], carry E[i+8]
            PCMM_CHAIN4C(E[i], E[i + 1], E[i + 2], E[i + 3], E[i + 4], E[i + 5], E[i + 6], E[i + 7], E[i + 8],
                         a0, a2, a4, a6, bi);
            // odd a-limbs -> odd offsets i+1..i+8 = O[i..i+7], carry O[i+8]
            PCMM_CHAIN4C(O[i], O[i + 1], O[i + 2], O[i + 3], O[i + 4], O[i + 5], O[i + 6], O[i + 7], O[i + 8],
                         a1, a3, a5, a7, bi);
        }
    }
    // T = E + O 2^32 (< 2^512: no carry out of word 15)
    T[0] = E[0];
    asm("add.cc.u32 %0, %15, %30;\n\t"
        "addc.cc.u32 %1, %16, %31;\n\t"
        "addc.cc.u32 %2, %17, %32;\n\t"
        "addc.cc.u32 %3, %18, %33;\n\t"
        "addc.cc.u32 %4, %19, %34;\n\t"
        "addc.cc.u32 %5, %20, %35;\n\t"
        "addc.cc.u32 %6, %21, %36;\n\t"
        "addc.cc.u32 %7, %22, %37;\n\t"
        "addc.cc.u32 %8, %23, %38;\n\t"
        "addc.cc.u32 %9, %24, %39;\n\t"
        "addc.cc.u32 %10, %25, %40;\n\t"
        "addc.cc.u32 %11, %26, %41;\n\t"
        "addc.cc.u32 %12, %27, %42;\n\t"
        "addc.cc.u32 %13, %28, %43;\n\t"
        "addc.u32 %14, %29, %44;"
        : "=r"(T[1]), "=r"(T[2]), "=r"(T[3]), "=r"(T[4]), "=r"(T[5]), "=r"(T[6]), "=r"(T[7]), "=r"(T[8]),
          "=r"(T[9]), "=r"(T[10]), "=r"(T[11]), "=r"(T[12]), "=r"(T[13]), "=r"(T[14]), "=r"(T[15])
        : "r"(E[1]), "r"(E[2]), "r"(E[3]), "r"(E[4]), "r"(E[5]), "r"(E[6]), "r"(E[7]), "r"(E[8]), "r"(E[9]),
          "r"(E[10]), "r"(E[11]), "r"(E[12]), "r"(E[13]), "r"(E[14]), "r"(E[15]),
          "r"(O[0]), "r"(O[1]), "r"(O[2]), "r"(O[3]), "r"(O[4]), "r"(O[5]), "r"(O[6]), "r"(O[7]), "r"(O[8]),
          "r"(O[9]), "r"(O[10]), "r"(O[11]), "r"(O[12]), "r"(O[13]), "r"(O[14]));
}

#ifndef PCMM_MUL_PRODUCT
#define PCMM_MUL_PRODUCT 1        // 1: even/odd product scanning, 0: operand scanning
#endif

// Montgomery reduction of a 512-bit T (T < 2^512) to T 2^-256 mod p: in [0, p)
// (kLazy = false), or in [0, 2^256) (kLazy = true: "almost reduced", see below)
template <bool kLazy = false>
__device__ __forceinline__ void fe_redc_t(fe &r, uint32_t T[16]) {
    // ---- reduction, 64-bit quotient digits: -p^-1 = 1 mod 2^64 (p = -1 mod 2^96),
    // so round r (base b = 2r) takes q = T[b] + 2^32 T[b+1] and adds
    //   q p 2^(32b) = -q + q 2^96 + u 2^192,  u = q (2^64 - 2^32 + 1) < 2^128.
    // The -q cancels T[b], T[b+1] exactly; q 2^96 and u 2^192 go to words
    // b+3..b+4 and b+6..b+9 in one carry chain.  The chain's carry out (word
    // b+10) is deferred into the next round's u (word 2 of u' is word b+10;
    // u' + 2^64 < 2^128), so no chain runs to the top.
    uint32_t E = 0;
#pragma unroll
    for (int r = 0; r < 4; r++) {
        const int b = 2 * r;
        const uint32_t q0 = T[b], q1 = T[b + 1];
        uint32_t w1, w2, w3;
        asm("sub.cc.u32 %0, %3, %4;\n\t"
            "subc.cc.u32 %1, %4, %3;\n\t"
            "subc.u32 %2, %3, 0;"
            : "=r"(w1), "=r"(w2), "=r"(w3)
            : "r"(q1), "r"(q0));
        if (r > 0) {
            asm("add.cc.u32 %0, %0, %2;\n\t"
                "addc.u32 %1, %1, 0;"
                : "+r"(w2), "+r"(w3)
                : "r"(E));
        }
        asm("add.cc.u32 %0, %0, %8;\n\t"
            "addc.cc.u32 %1, %1, %9;\n\t"
            "addc.cc.u32 %2, %2, 0;\n\t"
            "addc.cc.u32 %3, %3, %8;\n\t"
            "addc.cc.u32 %4, %4, %10;\n\t"
            "addc.cc.u32 %5, %5, %11;\n\t"
            "addc.cc.u32 %6, %6, %12;\n\t"
            "addc.u32 %7, 0, 0;"
            : "+r"(T[b + 3]), "+r"(T[b + 4]), "+r"(T[b + 5]), "+r"(T[b + 6]), "+r"(T[b + 7]), "+r"(T[b + 8]),
              "+r"(T[b + 9]), "=r"(E)
            : "r"(q0), "r"(q1), "r"(w1), "r"(w2), "r"(w3));
    }
    if (kLazy) {
        // ---- result V = E 2^256 + T[8..15] < 2^256 + p.  Lazy: keep V mod 2^256 when E = 0,
        // else V - p = T[8..15] + (2^256 - p) (< 2^256 because then T[8..15] < p):
        // 2^256 - p = (1, 0, 0, ffffffff, ffffffff, ffffffff, fffffffe, 0) little-endian words.
        // One masked add chain instead of a subtraction and eight selects.
        const uint32_t m = 0u - E;
        asm("add.cc.u32 %0, %8, %16;\n\t"
            "addc.cc.u32 %1, %9, 0;\n\t"
            "addc.cc.u32 %2, %10, 0;\n\t"
            "addc.cc.u32 %3, %11, %17;\n\t"
            "addc.cc.u32 %4, %12, %17;\n\t"
            "addc.cc.u32 %5, %13, %17;\n\t"
            "addc.cc.u32 %6, %14, %18;\n\t"
            "addc.u32 %7, %15, 0;"
            : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]), "=r"(r.v[6]),
              "=r"(r.v[7])
            : "r"(T[8]), "r"(T[9]), "r"(T[10]), "r"(T[11]), "r"(T[12]), "r"(T[13]), "r"(T[14]), "r"(T[15]),
              "r"(m & 1u), "r"(m), "r"(m & 0xfffffffeu));
        return;
    }
    // ---- result = E*2^256 + T[8..15] < 2^256 + p (< 2p for inputs < p); subtract p if it is >= p
    // (inputs < 2^256 but not < p give E = 1 with T[8..15] < p: the same subtraction is exact)
    uint32_t t[8], m;
    asm("sub.cc.u32 %0, %9, 0xffffffff;\n\t"
        "subc.cc.u32 %1, %10, 0xffffffff;\n\t"
        "subc.cc.u32 %2, %11, 0xffffffff;\n\t"
        "subc.cc.u32 %3, %12, 0;\n\t"
        "subc.cc.u32 %4, %13, 0;\n\t"
        "subc.cc.u32 %5, %14, 0;\n\t"
        "subc.cc.u32 %6, %15, 1;\n\t"
        "subc.cc.u32 %7, %16, 0xffffffff;\n\t"
        "subc.u32 %8, %17, 0;"
        : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3]), "=r"(t[4]), "=r"(t[5]), "=r"(t[6]), "=r"(t[7]), "=r"(m)
        : "r"(T[8]), "r"(T[9]), "r"(T[10]), "r"(T[11]), "r"(T[12]), "r"(T[13]), "r"(T[14]), "r"(T[15]), "r"(E));
    // m = E - borrow: 0 -> take t (value >= p), 0xffffffff -> keep T (value < p)
#pragma unroll
    for (int k = 0; k < 8; k++) r.v[k] = (T[8 + k] & m) | (t[k] & ~m);
}

__device__ __forceinline__ void fe_redc_fast(fe &r, uint32_t T[16]) { fe_redc_t<false>(r, T); }

#ifndef PCMM_REDC_FAKE
#define PCMM_REDC_FAKE 0        // MEASUREMENT ONLY (wrong results): 1 skips the reduction, 2 also the final subtraction
#endif
template <int PV>
__device__ __forceinline__ void fe_mul_fast_v(fe &r, const fe &a, const fe &b) {
    uint32_t T[16];
    if (PV == 1) fe_prod_eo(T, a, b);
    else fe_prod_os(T, a, b);
#if PCMM_REDC_FAKE == 2
#pragma unroll
    for (int k = 0; k < 8; k++) r.v[k] = T[8 + k] ^ T[k];
#elif PCMM_REDC_FAKE == 1
    uint32_t t[8], m;
    asm("sub.cc.u32 %0, %9, 0xffffffff;\n\t"
        "subc.cc.u32 %1, %10, 0xffffffff;\n\t"
        "subc.cc.u32 %2, %11, 0xffffffff;\n\t"
        "subc.cc.u32 %3, %12, 0;\n\t"
        "subc.cc.u32 %4, %13, 0;\n\t"
        "subc.cc.u32 %5, %14, 0;\n\t"
        "subc.cc.u32 %6, %15, 1;\n\t"
        "subc.cc.u32 %7, %16, 0xffffffff;\n\t"
        "subc.u32 %8, %17, 0;"
        : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3]), "=r"(t[4]), "=r"(t[5]), "=r"(t[6]), "=r"(t[7]), "=r"(m)
        : "r"(T[8] ^ T[0]), "r"(T[9] ^ T[1]), "r"(T[10] ^ T[2]), "r"(T[11] ^ T[3]), "r"(T[12] ^ T[4]), "r"(T[13] ^ T[5]),
          "r"(T[14] ^ T[6]), "r"(T[15] ^ T[7]), "r"(0u));
#pragma unroll
    for (int k = 0; k < 8; k++) r.v[k] = ((T[8 + k] ^ T[k]) & m) | (t[k] & ~m);
#else
    fe_redc_fast(r, T);
#endif
}

__device__ __forceinline__ void fe_mul_fast(fe &r, const fe &a, const fe &b) { fe_mul_fast_v<PCMM_MUL_PRODUCT>(r, a, b); }

// ---- "almost reduced" (lazy) arithmetic for the accumulate loop: operands and
// results anywhere in [0, 2^256) (congruent mod p, not canonical).  The product
// skips the final conditional subtraction (fe_redc_t<true>), the sum folds its
// carry back as + (2^256 - p), the difference adds p (twice in the rare case
// b - a > p); an element is zero iff it is 0 or p.  Canonical values are
// produced again by any non-lazy product (fe_mul_fast accepts inputs < 2^256).
__device__ __forceinline__ void fe_mul_lz(fe &r, const fe &a, const fe &b) {
    uint32_t T[16];
    fe_prod_eo(T, a, b);
    fe_redc_t<true>(r, T);
}

__device__ __forceinline__ bool fe_is_zero_lz(const fe &a) {
    const uint32_t z = a.v[0] | a.v[1] | a.v[2] | a.v[3] | a.v[4] | a.v[5] | a.v[6] | a.v[7];
    const uint32_t pp = ~a.v[0] | ~a.v[1] | ~a.v[2] | a.v[3] | a.v[4] | a.v[5] | (a.v[6] ^ 1u) | ~a.v[7];
    return z == 0 || pp == 0;
}

// r = a + b (mod p), a, b, r in [0, 2^256)
__device__ __forceinline__ void fe_add_lz(fe &r, const fe &a, const fe &b) {
    uint32_t s[8], c;
    asm("add.cc.u32 %0, %9, %17;\n\t"
        "addc.cc.u32 %1, %10, %18;\n\t"
        "addc.cc.u32 %2, %11, %19;\n\t"
        "addc.cc.u32 %3, %12, %20;\n\t"
        "addc.cc.u32 %4, %13, %21;\n\t"
        "addc.cc.u32 %5, %14, %22;\n\t"
        "addc.cc.u32 %6, %15, %23;\n\t"
        "addc.cc.u32 %7, %16, %24;\n\t"
        "addc.u32 %8, 0, 0;"
        : "=r"(s[0]), "=r"(s[1]), "=r"(s[2]), "=r"(s[3]), "=r"(s[4]), "=r"(s[5]), "=r"(s[6]), "=r"(s[7]), "=r"(c)
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(a.v[6]), "r"(a.v[7]),
          "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]), "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    uint32_t m = 0u - c;                          // carry: + (2^256 - p)
    asm("add.cc.u32 %0, %0, %9;\n\t"
        "addc.cc.u32 %1, %1, 0;\n\t"
        "addc.cc.u32 %2, %2, 0;\n\t"
        "addc.cc.u32 %3, %3, %10;\n\t"
        "addc.cc.u32 %4, %4, %10;\n\t"
        "addc.cc.u32 %5, %5, %10;\n\t"
        "addc.cc.u32 %6, %6, %11;\n\t"
        "addc.cc.u32 %7, %7, 0;\n\t"
        "addc.u32 %8, 0, 0;"
        : "+r"(s[0]), "+r"(s[1]), "+r"(s[2]), "+r"(s[3]), "+r"(s[4]), "+r"(s[5]), "+r"(s[6]), "+r"(s[7]), "=r"(c)
        : "r"(m & 1u), "r"(m), "r"(m & 0xfffffffeu));
    if (c) {                                      // a second wrap: only when a + b - p >= 2^256 - (2^256 - p)
        asm("add.cc.u32 %0, %0, 1;\n\t"
            "addc.cc.u32 %1, %1, 0;\n\t"
            "addc.cc.u32 %2, %2, 0;\n\t"
            "addc.cc.u32 %3, %3, 0xffffffff;\n\t"
            "addc.cc.u32 %4, %4, 0xffffffff;\n\t"
            "addc.cc.u32 %5, %5, 0xffffffff;\n\t"
            "addc.cc.u32 %6, %6, 0xfffffffe;\n\t"
            "addc.u32 %7, %7, 0;"
            : "+r"(s[0]), "+r"(s[1]), "+r"(s[2]), "+r"(s[3]), "+r"(s[4]), "+r"(s[5]), "+r"(s[6]), "+r"(s[7]));
    }
#pragma unroll
    for (int k = 0; k < 8; k++) r.v[k] = s[k];
}

// r = a - b (mod p), a, b, r in [0, 2^256)
__device__ __forceinline__ void fe_sub_lz(fe &r, const fe &a, const fe &b) {
    uint32_t d[8], m, c;
    asm("sub.cc.u32 %0, %9, %17;\n\t"
        "subc.cc.u32 %1, %10, %18;\n\t"
        "subc.cc.u32 %2, %11, %19;\n\t"
        "subc.cc.u32 %3, %12, %20;\n\t"
        "subc.cc.u32 %4, %13, %21;\n\t"
        "subc.cc.u32 %5, %14, %22;\n\t"
        "subc.cc.u32 %6, %15, %23;\n\t"
        "subc.cc.u32 %7, %16, %24;\n\t"
        "subc.u32 %8, 0, 0;"
        : "=&r"(d[0]), "=&r"(d[1]), "=&r"(d[2]), "=&r"(d[3]), "=&r"(d[4]), "=&r"(d[5]), "=&r"(d[6]), "=&r"(d[7]),
          "=&r"(m)
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(a.v[6]), "r"(a.v[7]),
          "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]), "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    // borrow: + p (limbs m, m, m, 0, 0, 0, m & 1, m); carry out c = 1 iff the result is now >= 0
    asm("add.cc.u32 %0, %0, %9;\n\t"
        "addc.cc.u32 %1, %1, %9;\n\t"
        "addc.cc.u32 %2, %2, %9;\n\t"
        "addc.cc.u32 %3, %3, 0;\n\t"
        "addc.cc.u32 %4, %4, 0;\n\t"
        "addc.cc.u32 %5, %5, 0;\n\t"
        "addc.cc.u32 %6, %6, %10;\n\t"
        "addc.cc.u32 %7, %7, %9;\n\t"
        "addc.u32 %8, 0, 0;"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3]), "+r"(d[4]), "+r"(d[5]), "+r"(d[6]), "+r"(d[7]), "=r"(c)
        : "r"(m), "r"(m & 1u));
    if (m & ~(0u - c)) {                          // still negative (b - a > p: only for b >= p): + p again
        asm("add.cc.u32 %0, %0, 0xffffffff;\n\t"
            "addc.cc.u32 %1, %1, 0xffffffff;\n\t"
            "addc.cc.u32 %2, %2, 0xffffffff;\n\t"
            "addc.cc.u32 %3, %3, 0;\n\t"
            "addc.cc.u32 %4, %4, 0;\n\t"
            "addc.cc.u32 %5, %5, 0;\n\t"
            "addc.cc.u32 %6, %6, 1;\n\t"
            "addc.u32 %7, %7, 0xffffffff;"
            : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3]), "+r"(d[4]), "+r"(d[5]), "+r"(d[6]), "+r"(d[7]));
    }
#pragma unroll
    for (int k = 0; k < 8; k++) r.v[k] = d[k];
}

// ---- squaring: the 28 cross products a_i a_j (i < j) once, in the even/odd
// accumulators (row i: j - i odd -> O, j - i even -> E; chains of 1..4 pairs),
// C = E + O 2^32, T = 2 C + sum a_i^2 2^(64 i) (the diagonal as one fused
// IMAD.WIDE.U32.X chain over all 16 words): 36 products instead of 64.
#define PCMM_CH1C(d0, d1, c, x0, y)                                \
    asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"                       \
        "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"                      \
        "addc.u32 %2, %2, 0;"                                      \
        : "+r"(d0), "+r"(d1), "+r"(c)                              \
        : "r"(x0), "r"(y))
#define PCMM_CH2C(d0, d1, d2, d3, c, x0, x1, y)                    \
    asm("mad.lo.cc.u32 %0, %5, %7, %0;\n\t"                       \
        "madc.hi.cc.u32 %1, %5, %7, %1;\n\t"                      \
        "madc.lo.cc.u32 %2, %6, %7, %2;\n\t"                      \
        "madc.hi.cc.u32 %3, %6, %7, %3;\n\t"                      \
        "addc.u32 %4, %4, 0;"                                      \
        : "+r"(d0), "+r"(d1), "+r"(d2), "+r"(d3), "+r"(c)          \
        : "r"(x0), "r"(x1), "r"(y))
#define PCMM_CH3C(d0, d1, d2, d3, d4, d5, c, x0, x1, x2, y)        \
    asm("mad.lo.cc.u32 %0, %7, %10, %0;\n\t"                      \
        "madc.hi.cc.u32 %1, %7, %10, %1;\n\t"                     \
        "madc.lo.cc.u32 %2, %8, %10, %2;\n\t"                     \
        "madc.hi.cc.u32 %3, %8, %10, %3;\n\t"                     \
        "madc.lo.cc.u32 %4, %9, %10, %4;\n\t"                     \
        "madc.hi.cc.u32 %5, %9, %10, %5;\n\t"                     \
        "addc.u32 %6, %6, 0;"                                      \
        : "+r"(d0), "+r"(d1), "+r"(d2), "+r"(d3), "+r"(d4), "+r"(d5), "+r"(c) \
        : "r"(x0), "r"(x1), "r"(x2), "r"(y))

template <bool kLazy>
__device__ __forceinline__ void fe_sqr_fast_t(fe &r, const fe &a) {
    const uint32_t a0 = a.v[0], a1 = a.v[1], a2 = a.v[2], a3 = a.v[3];
    const uint32_t a4 = a.v[4], a5 = a.v[5], a6 = a.v[6], a7 = a.v[7];
    uint32_t E[16], O[16];                       // E[k] = word k (k >= 2), O[k] = word k + 1
    // row 0: plain products; O[0..7] = a0 (a1, a3, a5, a7), E[2..7] = a0 (a2, a4, a6)
    {
        uint64_t p;
        p = (uint64_t)a0 * a1; O[0] = (uint32_t)p; O[1] = (uint32_t)(p >> 32);
        p = (uint64_t)a0 * a3; O[2] = (uint32_t)p; O[3] = (uint32_t)(p >> 32);
        p = (uint64_t)a0 * a5; O[4] = (uint32_t)p; O[5] = (uint32_t)(p >> 32);
        p = (uint64_t)a0 * a7; O[6] = (uint32_t)p; O[7] = (uint32_t)(p >> 32);
        p = (uint64_t)a0 * a2; E[2] = (uint32_t)p; E[3] = (uint32_t)(p >> 32);
        p = (uint64_t)a0 * a4; E[4] = (uint32_t)p; E[5] = (uint32_t)(p >> 32);
        p = (uint64_t)a0 * a6; E[6] = (uint32_t)p; E[7] = (uint32_t)(p >> 32);
    }
#pragma unroll
    for (int k = 8; k < 16; k++) {
        E[k] = 0;
        O[k] = 0;
    }
    // row i: O-chain over j = i+1, i+3, .. at O[2i ..], E-chain over j = i+2, .. at E[2i+2 ..]
    PCMM_CH3C(O[2], O[3], O[4], O[5], O[6], O[7], O[8], a2, a4, a6, a1);        // i = 1
    PCMM_CH3C(E[4], E[5], E[6], E[7], E[8], E[9], E[10], a3, a5, a7, a1);
    PCMM_CH3C(O[4], O[5], O[6], O[7], O[8], O[9], O[10], a3, a5, a7, a2);       // i = 2
    PCMM_CH2C(E[6], E[7], E[8], E[9], E[10], a4, a6, a2);
    PCMM_CH2C(O[6], O[7], O[8], O[9], O[10], a4, a6, a3);                       // i = 3
    PCMM_CH2C(E[8], E[9], E[10], E[11], E[12], a5, a7, a3);
    PCMM_CH2C(O[8], O[9], O[10], O[11], O[12], a5, a7, a4);                     // i = 4
    PCMM_CH1C(E[10], E[11], E[12], a6, a4);
    PCMM_CH1C(O[10], O[11], O[12], a6, a5);                                     // i = 5
    PCMM_CH1C(E[12], E[13], E[14], a7, a5);
    PCMM_CH1C(O[12], O[13], O[14], a7, a6);                                     // i = 6
    // C = E + O 2^32 (C[0] = 0, C[1] = O[0]); C < 2^511
    uint32_t C[16];
    C[0] = 0;
    C[1] = O[0];
    asm("add.cc.u32 %0, %14, %28;\n\t"
        "addc.cc.u32 %1, %15, %29;\n\t"
        "addc.cc.u32 %2, %16, %30;\n\t"
        "addc.cc.u32 %3, %17, %31;\n\t"
        "addc.cc.u32 %4, %18, %32;\n\t"
        "addc.cc.u32 %5, %19, %33;\n\t"
        "addc.cc.u32 %6, %20, %34;\n\t"
        "addc.cc.u32 %7, %21, %35;\n\t"
        "addc.cc.u32 %8, %22, %36;\n\t"
        "addc.cc.u32 %9, %23, %37;\n\t"
        "addc.cc.u32 %10, %24, %38;\n\t"
        "addc.cc.u32 %11, %25, %39;\n\t"
        "addc.cc.u32 %12, %26, %40;\n\t"
        "addc.u32 %13, %27, %41;"
        : "=r"(C[2]), "=r"(C[3]), "=r"(C[4]), "=r"(C[5]), "=r"(C[6]), "=r"(C[7]), "=r"(C[8]), "=r"(C[9]),
          "=r"(C[10]), "=r"(C[11]), "=r"(C[12]), "=r"(C[13]), "=r"(C[14]), "=r"(C[15])
        : "r"(E[2]), "r"(E[3]), "r"(E[4]), "r"(E[5]), "r"(E[6]), "r"(E[7]), "r"(E[8]), "r"(E[9]), "r"(E[10]),
          "r"(E[11]), "r"(E[12]), "r"(E[13]), "r"(E[14]), "r"(E[15]),
          "r"(O[1]), "r"(O[2]), "r"(O[3]), "r"(O[4]), "r"(O[5]), "r"(O[6]), "r"(O[7]), "r"(O[8]), "r"(O[9]),
          "r"(O[10]), "r"(O[11]), "r"(O[12]), "r"(O[13]), "r"(O[14]));
    uint32_t T[16];
    T[0] = 0;
#pragma unroll
    for (int k = 1; k < 16; k++) T[k] = __funnelshift_l(C[k - 1], C[k], 1);   // 2 C
    asm("mad.lo.cc.u32 %0, %16, %16, %0;\n\t"
        "madc.hi.cc.u32 %1, %16, %16, %1;\n\t"
        "madc.lo.cc.u32 %2, %17, %17, %2;\n\t"
        "madc.hi.cc.u32 %3, %17, %17, %3;\n\t"
        "madc.lo.cc.u32 %4, %18, %18, %4;\n\t"
        "madc.hi.cc.u32 %5, %18, %18, %5;\n\t"
        "madc.lo.cc.u32 %6, %19, %19, %6;\n\t"
        "madc.hi.cc.u32 %7, %19, %19, %7;\n\t"
        "madc.lo.cc.u32 %8, %20, %20, %8;\n\t"
        "madc.hi.cc.u32 %9, %20, %20, %9;\n\t"
        "madc.lo.cc.u32 %10, %21, %21, %10;\n\t"
        "madc.hi.cc.u32 %11, %21, %21, %11;\n\t"
        "madc.lo.cc.u32 %12, %22, %22, %12;\n\t"
        "madc.hi.cc.u32 %13, %22, %22, %13;\n\t"
        "madc.lo.cc.u32 %14, %23, %23, %14;\n\t"
        "madc.hi.u32 %15, %23, %23, %15;"
        : "+r"(T[0]), "+r"(T[1]), "+r"(T[2]), "+r"(T[3]), "+r"(T[4]), "+r"(T[5]), "+r"(T[6]), "+r"(T[7]),
          "+r"(T[8]), "+r"(T[9]), "+r"(T[10]), "+r"(T[11]), "+r"(T[12]), "+r"(T[13]), "+r"(T[14]), "+r"(T[15])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(a4), "r"(a5), "r"(a6), "r"(a7));
    fe_redc_t<kLazy>(r, T);
}

__device__ __forceinline__ void fe_sqr_fast(fe &r, const fe &a) { fe_sqr_fast_t<false>(r, a); }
__device__ __forceinline__ void fe_sqr_lz(fe &r, const fe &a) { fe_sqr_fast_t<true>(r, a); }


// r = a + b mod p (a, b < p)
__device__ __forceinline__ void fe_add_fast(fe &r, const fe &a, const fe &b) {
    uint32_t s[8], t[8], m;
    asm("add.cc.u32 %0, %17, %25;\n\t"
        "addc.cc.u32 %1, %18, %26;\n\t"
        "addc.cc.u32 %2, %19, %27;\n\t"
        "addc.cc.u32 %3, %20, %28;\n\t"
        "addc.cc.u32 %4, %21, %29;\n\t"
        "addc.cc.u32 %5, %22, %30;\n\t"
        "addc.cc.u32 %6, %23, %31;\n\t"
        "addc.cc.u32 %7, %24, %32;\n\t"
        "addc.u32 %16, 0, 0;\n\t"
        "sub.cc.u32 %8, %0, 0xffffffff;\n\t"
        "subc.cc.u32 %9, %1, 0xffffffff;\n\t"
        "subc.cc.u32 %10, %2, 0xffffffff;\n\t"
        "subc.cc.u32 %11, %3, 0;\n\t"
        "subc.cc.u32 %12, %4, 0;\n\t"
        "subc.cc.u32 %13, %5, 0;\n\t"
        "subc.cc.u32 %14, %6, 1;\n\t"
        "subc.cc.u32 %15, %7, 0xffffffff;\n\t"
        "subc.u32 %16, %16, 0;"
        : "=&r"(s[0]), "=&r"(s[1]), "=&r"(s[2]), "=&r"(s[3]), "=&r"(s[4]), "=&r"(s[5]), "=&r"(s[6]), "=&r"(s[7]),
          "=&r"(t[0]), "=&r"(t[1]), "=&r"(t[2]), "=&r"(t[3]), "=&r"(t[4]), "=&r"(t[5]), "=&r"(t[6]), "=&r"(t[7]),
          "=&r"(m)
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(a.v[6]), "r"(a.v[7]),
          "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]), "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    // m = carry - borrow: 0xffffffff -> a + b < p (keep s), 0 -> take s - p
#pragma unroll
    for (int k = 0; k < 8; k++) r.v[k] = (s[k] & m) | (t[k] & ~m);
}

// r = a - b mod p (a, b < p)
__device__ __forceinline__ void fe_sub_fast(fe &r, const fe &a, const fe &b) {
    uint32_t d[8], m, m1;
    asm("sub.cc.u32 %0, %9, %17;\n\t"
        "subc.cc.u32 %1, %10, %18;\n\t"
        "subc.cc.u32 %2, %11, %19;\n\t"
        "subc.cc.u32 %3, %12, %20;\n\t"
        "subc.cc.u32 %4, %13, %21;\n\t"
        "subc.cc.u32 %5, %14, %22;\n\t"
        "subc.cc.u32 %6, %15, %23;\n\t"
        "subc.cc.u32 %7, %16, %24;\n\t"
        "subc.u32 %8, 0, 0;"
        : "=&r"(d[0]), "=&r"(d[1]), "=&r"(d[2]), "=&r"(d[3]), "=&r"(d[4]), "=&r"(d[5]), "=&r"(d[6]), "=&r"(d[7]),
          "=&r"(m)
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(a.v[6]), "r"(a.v[7]),
          "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]), "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    m1 = m & 1u;
    // add p & m: limbs (m, m, m, 0, 0, 0, m & 1, m)
    asm("add.cc.u32 %0, %0, %8;\n\t"
        "addc.cc.u32 %1, %1, %8;\n\t"
        "addc.cc.u32 %2, %2, %8;\n\t"
        "addc.cc.u32 %3, %3, 0;\n\t"
        "addc.cc.u32 %4, %4, 0;\n\t"
        "addc.cc.u32 %5, %5, 0;\n\t"
        "addc.cc.u32 %6, %6, %9;\n\t"
        "addc.u32 %7, %7, %8;"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3]), "+r"(d[4]), "+r"(d[5]), "+r"(d[6]), "+r"(d[7])
        : "r"(m), "r"(m1));
#pragma unroll
    for (int k = 0; k < 8; k++) r.v[k] = d[k];
}

// Out-of-line Montgomery product, arguments and result in registers.  The hot
// accumulate loop calls this instead of inlining 14 copies of fe_mul_fast into
// every point addition: the inlined loop body (~80 KB of SASS) thrashed the
// instruction cache ("no_instructions" was the top stall reason in ncu).
__device__ __noinline__ fe fe_mul_call(const fe a, const fe b) {
    fe r;
    fe_mul_fast(r, a, b);
    return r;
}

struct fe2 {
    fe x, y;
};

// Two independent Montgomery products in one out-of-line call: ptxas
// interleaves the two dependency chains (twice the ILP of a single call).
__device__ __noinline__ fe2 fe_mul2_call(const fe a0, const fe b0, const fe a1, const fe b1) {
    fe2 r;
    fe_mul_fast(r.x, a0, b0);
    fe_mul_fast(r.y, a1, b1);
    return r;
}

// One product and one square in one out-of-line call: (a b, c^2).
__device__ __noinline__ fe2 fe_mulsqr_call(const fe a, const fe b, const fe c) {
    fe2 r;
    fe_mul_fast(r.x, a, b);
    fe_sqr_fast(r.y, c);
    return r;
}

struct fe3 {
    fe x, y, z;
};

// The accumulate step's product groups (jac.cuh jac_add_aff).  Inlined by default
// (PCMM_INLINE_ACCUM=1): with the even/odd product the whole step is ~40 KB of
// SASS, just past the 32 KB L1.5 instruction cache, and the call glue (argument
// moves on the FMA-heavy pipe) costs more than the misses: measured at 4 CTAs per
// SM, 256^3 / 512^3 / ML accumulate 1.7 / 4.9 / 4.3 % faster than out of line.
#ifndef PCMM_INLINE_ACCUM
#define PCMM_INLINE_ACCUM 1
#endif
#if PCMM_INLINE_ACCUM
#define PCMM_HOTCALL __forceinline__
#else
#define PCMM_HOTCALL __noinline__
#endif

struct fe4 {
    fe x, y, z, w;
};

// (a b, c^2, d^2) in one out-of-line call
__device__ __noinline__ fe3 fe_m1s2_call(const fe a, const fe b, const fe c, const fe d) {
    fe3 r;
    fe_mul_fast(r.x, a, b);
    fe_sqr_fast(r.y, c);
    fe_sqr_fast(r.z, d);
    return r;
}

// (a b, c d, e^2, f^2) in one out-of-line call
__device__ __noinline__ fe4 fe_m2s2_call(const fe a, const fe b, const fe c, const fe d, const fe e, const fe f) {
    fe4 r;
    fe_mul_fast(r.x, a, b);
    fe_mul_fast(r.y, c, d);
    fe_sqr_fast(r.z, e);
    fe_sqr_fast(r.w, f);
    return r;
}


// Three independent Montgomery products in one out-of-line call (the Jacobian
// accumulate step has a stage with three independent products).
__device__ __noinline__ fe3 fe_mul3_call(const fe a0, const fe b0, const fe a1, const fe b1, const fe a2,
                                         const fe b2) {
    fe3 r;
    fe_mul_fast(r.x, a0, b0);
    fe_mul_fast(r.y, a1, b1);
    fe_mul_fast(r.z, a2, b2);
    return r;
}

}  // namespace pcmm

namespace pcmm {

__device__ PCMM_HOTCALL fe2 fe_mul2_hot(const fe a0, const fe b0, const fe a1, const fe b1) {
    fe2 r;
    fe_mul_fast(r.x, a0, b0);
    fe_mul_fast(r.y, a1, b1);
    return r;
}

__device__ PCMM_HOTCALL fe2 fe_mulsqr_hot(const fe a, const fe b, const fe c) {
    fe2 r;
    fe_mul_fast(r.x, a, b);
    fe_sqr_fast(r.y, c);
    return r;
}

__device__ PCMM_HOTCALL fe2 fe_sqr2_hot(const fe a, const fe b) {
    fe2 r;
    fe_sqr_fast(r.x, a);
    fe_sqr_fast(r.y, b);
    return r;
}

// (c^2, a0 b0, a1 b1, a2 b2) and four products: the software-pipelined XYZZ step
#ifndef PCMM_SQRMUL3_IL
#define PCMM_SQRMUL3_IL 0       // 1: the square as a general product in a phase-interleaved 4-product group
#endif
template <int K>
__device__ __forceinline__ void fe_mul_il(fe *r, const fe *a, const fe *b);
__device__ PCMM_HOTCALL fe4 fe_sqr_mul3_hot(const fe c, const fe a0, const fe b0, const fe a1, const fe b1,
                                            const fe a2, const fe b2) {
    fe4 r;
#if PCMM_SQRMUL3_IL
    const fe a[4] = {c, a0, a1, a2}, b[4] = {c, b0, b1, b2};
    fe o[4];
    fe_mul_il<4>(o, a, b);
    r.x = o[0];
    r.y = o[1];
    r.z = o[2];
    r.w = o[3];
#else
    fe_sqr_fast(r.x, c);
    fe_mul_fast(r.y, a0, b0);
    fe_mul_fast(r.z, a1, b1);
    fe_mul_fast(r.w, a2, b2);
#endif
    return r;
}

// (c^2, a0 b0, a1 b1): the XYZZ doubling's third group (jac.cuh xyzz_dbl)
__device__ PCMM_HOTCALL fe3 fe_sqr_mul2_hot(const fe c, const fe a0, const fe b0, const fe a1, const fe b1) {
    fe3 r;
    fe_sqr_fast(r.x, c);
    fe_mul_fast(r.y, a0, b0);
    fe_mul_fast(r.z, a1, b1);
    return r;
}

#ifndef PCMM_MUL4_IL
#define PCMM_MUL4_IL 0          // 1: the 4-product group written phase by phase (fe_mul_il<4>, below)
#endif
template <int K>
__device__ __forceinline__ void fe_mul_il(fe *r, const fe *a, const fe *b);
__device__ PCMM_HOTCALL fe4 fe_mul4_hot(const fe a0, const fe b0, const fe a1, const fe b1, const fe a2,
                                        const fe b2, const fe a3, const fe b3) {
    fe4 r;
#if PCMM_MUL4_IL
    const fe a[4] = {a0, a1, a2, a3}, b[4] = {b0, b1, b2, b3};
    fe o[4];
    fe_mul_il<4>(o, a, b);
    r.x = o[0];
    r.y = o[1];
    r.z = o[2];
    r.w = o[3];
#else
    fe_mul_fast(r.x, a0, b0);
    fe_mul_fast(r.y, a1, b1);
    fe_mul_fast(r.z, a2, b2);
    fe_mul_fast(r.w, a3, b3);
#endif
    return r;
}

__device__ PCMM_HOTCALL fe3 fe_mul3_hot(const fe a0, const fe b0, const fe a1, const fe b1, const fe a2,
                                        const fe b2) {
    fe3 r;
    fe_mul_fast(r.x, a0, b0);
    fe_mul_fast(r.y, a1, b1);
    fe_mul_fast(r.z, a2, b2);
    return r;
}

// lazy (almost reduced) forms of the software-pipelined XYZZ step's product groups (jac.cuh)
__device__ PCMM_HOTCALL fe2 fe_mulsqr_lz_hot(const fe a, const fe b, const fe c) {
    fe2 r;
    fe_mul_lz(r.x, a, b);
    fe_sqr_lz(r.y, c);
    return r;
}

__device__ PCMM_HOTCALL fe4 fe_sqr_mul3_lz_hot(const fe c, const fe a0, const fe b0, const fe a1, const fe b1,
                                               const fe a2, const fe b2) {
    fe4 r;
    fe_sqr_lz(r.x, c);
    fe_mul_lz(r.y, a0, b0);
    fe_mul_lz(r.z, a1, b1);
    fe_mul_lz(r.w, a2, b2);
    return r;
}

__device__ PCMM_HOTCALL fe4 fe_mul4_lz_hot(const fe a0, const fe b0, const fe a1, const fe b1, const fe a2,
                                           const fe b2, const fe a3, const fe b3) {
    fe4 r;
    fe_mul_lz(r.x, a0, b0);
    fe_mul_lz(r.y, a1, b1);
    fe_mul_lz(r.z, a2, b2);
    fe_mul_lz(r.w, a3, b3);
    return r;
}

// ---- K independent products written phase by phase (all K products' E/O rows, then all merges, then
// reduction round by round across the K products, then the K final subtractions), so that the
// instruction stream ptxas starts from is already interleaved (PCMM_MUL4_IL: the accumulate step's
// 4-product group).  Same arithmetic and results as K calls of fe_mul_fast.
template <int K>
__device__ __forceinline__ void fe_mul_il(fe *r, const fe *a, const fe *b) {
    uint32_t E[K][16], O[K][16];
#pragma unroll
    for (int q = 0; q < K; q++) {
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint64_t pe = (uint64_t)a[q].v[2 * j] * b[q].v[0];
            const uint64_t po = (uint64_t)a[q].v[2 * j + 1] * b[q].v[0];
            E[q][2 * j] = (uint32_t)pe;
            E[q][2 * j + 1] = (uint32_t)(pe >> 32);
            O[q][2 * j] = (uint32_t)po;
            O[q][2 * j + 1] = (uint32_t)(po >> 32);
        }
#pragma unroll
        for (int k = 8; k < 16; k++) {
            E[q][k] = 0;
            O[q][k] = 0;
        }
    }
#pragma unroll
    for (int i = 1; i < 8; i++) {
#pragma unroll
        for (int q = 0; q < K; q++) {
            const uint32_t bi = b[q].v[i];
            const uint32_t a0 = a[q].v[0], a1 = a[q].v[1], a2 = a[q].v[2], a3 = a[q].v[3];
            const uint32_t a4 = a[q].v[4], a5 = a[q].v[5], a6 = a[q].v[6], a7 = a[q].v[7];
            if (i & 1) {
                PCMM_CHAIN4C(O[q][i - 1], O[q][i], O[q][i + 1], O[q][i + 2], O[q][i + 3], O[q][i + 4], O[q][i + 5],
                             O[q][i + 6], O[q][i + 7], a0, a2, a4, a6, bi);
                if (i < 7) {
                    PCMM_CHAIN4C(E[q][i + 1], E[q][i + 2], E[q][i + 3], E[q][i + 4], E[q][i + 5], E[q][i + 6],
                                 E[q][i + 7], E[q][i + 8], E[q][(i + 9) & 15], a1, a3, a5, a7, bi);
                } else {
                    PCMM_CHAIN4(E[q][8], E[q][9], E[q][10], E[q][11], E[q][12], E[q][13], E[q][14], E[q][15], a1, a3,
                                a5, a7, bi);
                }
            } else {
                PCMM_CHAIN4C(E[q][i], E[q][i + 1], E[q][i + 2], E[q][i + 3], E[q][i + 4], E[q][i + 5], E[q][i + 6],
                             E[q][i + 7], E[q][i + 8], a0, a2, a4, a6, bi);
                PCMM_CHAIN4C(O[q][i], O[q][i + 1], O[q][i + 2], O[q][i + 3], O[q][i + 4], O[q][i + 5], O[q][i + 6],
                             O[q][i + 7], O[q][i + 8], a1, a3, a5, a7, bi);
            }
        }
    }
    uint32_t T[K][16];
#pragma unroll
    for (int q = 0; q < K; q++) {
        T[q][0] = E[q][0];
        asm("add.cc.u32 %0, %15, %30;\n\t"
            "addc.cc.u32 %1, %16, %31;\n\t"
            "addc.cc.u32 %2, %17, %32;\n\t"
            "addc.cc.u32 %3, %18, %33;\n\t"
            "addc.cc.u32 %4, %19, %34;\n\t"
            "addc.cc.u32 %5, %20, %35;\n\t"
            "addc.cc.u32 %6, %21, %36;\n\t"
            "addc.cc.u32 %7, %22, %37;\n\t"
            "addc.cc.u32 %8, %23, %38;\n\t"
            "addc.cc.u32 %9, %24, %39;\n\t"
            "addc.cc.u32 %10, %25, %40;\n\t"
            "addc.cc.u32 %11, %26, %41;\n\t"
            "addc.cc.u32 %12, %27, %42;\n\t"
            "addc.cc.u32 %13, %28, %43;\n\t"
            "addc.u32 %14, %29, %44;"
            : "=r"(T[q][1]), "=r"(T[q][2]), "=r"(T[q][3]), "=r"(T[q][4]), "=r"(T[q][5]), "=r"(T[q][6]), "=r"(T[q][7]),
              "=r"(T[q][8]), "=r"(T[q][9]), "=r"(T[q][10]), "=r"(T[q][11]), "=r"(T[q][12]), "=r"(T[q][13]),
              "=r"(T[q][14]), "=r"(T[q][15])
            : "r"(E[q][1]), "r"(E[q][2]), "r"(E[q][3]), "r"(E[q][4]), "r"(E[q][5]), "r"(E[q][6]), "r"(E[q][7]),
              "r"(E[q][8]), "r"(E[q][9]), "r"(E[q][10]), "r"(E[q][11]), "r"(E[q][12]), "r"(E[q][13]), "r"(E[q][14]),
              "r"(E[q][15]), "r"(O[q][0]), "r"(O[q][1]), "r"(O[q][2]), "r"(O[q][3]), "r"(O[q][4]), "r"(O[q][5]),
              "r"(O[q][6]), "r"(O[q][7]), "r"(O[q][8]), "r"(O[q][9]), "r"(O[q][10]), "r"(O[q][11]), "r"(O[q][12]),
              "r"(O[q][13]), "r"(O[q][14]));
    }
    uint32_t Ec[K];
#pragma unroll
    for (int q = 0; q < K; q++) Ec[q] = 0;
#pragma unroll
    for (int rr = 0; rr < 4; rr++) {
        const int bb = 2 * rr;
#pragma unroll
        for (int q = 0; q < K; q++) {
            const uint32_t q0 = T[q][bb], q1 = T[q][bb + 1];
            uint32_t w1, w2, w3;
            asm("sub.cc.u32 %0, %3, %4;\n\t"
                "subc.cc.u32 %1, %4, %3;\n\t"
                "subc.u32 %2, %3, 0;"
                : "=r"(w1), "=r"(w2), "=r"(w3)
                : "r"(q1), "r"(q0));
            if (rr > 0) {
                asm("add.cc.u32 %0, %0, %2;\n\t"
                    "addc.u32 %1, %1, 0;"
                    : "+r"(w2), "+r"(w3)
                    : "r"(Ec[q]));
            }
            asm("add.cc.u32 %0, %0, %8;\n\t"
                "addc.cc.u32 %1, %1, %9;\n\t"
                "addc.cc.u32 %2, %2, 0;\n\t"
                "addc.cc.u32 %3, %3, %8;\n\t"
                "addc.cc.u32 %4, %4, %10;\n\t"
                "addc.cc.u32 %5, %5, %11;\n\t"
                "addc.cc.u32 %6, %6, %12;\n\t"
                "addc.u32 %7, 0, 0;"
                : "+r"(T[q][bb + 3]), "+r"(T[q][bb + 4]), "+r"(T[q][bb + 5]), "+r"(T[q][bb + 6]), "+r"(T[q][bb + 7]),
                  "+r"(T[q][bb + 8]), "+r"(T[q][bb + 9]), "=r"(Ec[q])
                : "r"(q0), "r"(q1), "r"(w1), "r"(w2), "r"(w3));
        }
    }
#pragma unroll
    for (int q = 0; q < K; q++) {
        uint32_t t[8], m;
        asm("sub.cc.u32 %0, %9, 0xffffffff;\n\t"
            "subc.cc.u32 %1, %10, 0xffffffff;\n\t"
            "subc.cc.u32 %2, %11, 0xffffffff;\n\t"
            "subc.cc.u32 %3, %12, 0;\n\t"
            "subc.cc.u32 %4, %13, 0;\n\t"
            "subc.cc.u32 %5, %14, 0;\n\t"
            "subc.cc.u32 %6, %15, 1;\n\t"
            "subc.cc.u32 %7, %16, 0xffffffff;\n\t"
            "subc.u32 %8, %17, 0;"
            : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3]), "=r"(t[4]), "=r"(t[5]), "=r"(t[6]), "=r"(t[7]), "=r"(m)
            : "r"(T[q][8]), "r"(T[q][9]), "r"(T[q][10]), "r"(T[q][11]), "r"(T[q][12]), "r"(T[q][13]), "r"(T[q][14]),
              "r"(T[q][15]), "r"(Ec[q]));
#pragma unroll
        for (int k = 0; k < 8; k++) r[q].v[k] = (T[q][8 + k] & m) | (t[k] & ~m);
    }
}

}  // namespace pcmm
