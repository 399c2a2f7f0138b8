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

__device__ __forceinline__ void fe_mul_fast(fe &r, const fe &a, const fe &b) {
    uint32_t T[17];
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
    // ---- result = E*2^256 + T[8..15] < 2p; subtract p if it is >= p
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

struct fe3 {
    fe x, y, z;
};

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
