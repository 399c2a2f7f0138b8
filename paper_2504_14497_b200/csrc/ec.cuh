// ec.cuh -- NIST P-256 group law in homogeneous projective coordinates
// (x = X/Z, y = Y/Z; identity = (0 : 1 : 0)) with the COMPLETE formulas of
// Renes, Costello and Batina, "Complete addition formulas for prime order
// elliptic curves" (EUROCRYPT 2016), Algorithm 4 (addition, a = -3,
// 12M + 2m_b) and Algorithm 6 (doubling, a = -3, 8M + 3S + 2m_b).
//
// Completeness matters on this hot path: Cussen's prefix sums hit P + P
// (2P = P + P) and zero plaintext entries add the identity
// (R1), and both must be handled without branches.
//
// The group law, identity and ECSM are those of PAPER.md:150-155 (Sec. 2.3).
#pragma once
#include "fp.cuh"

namespace pcmm {

struct pt {
    fe X, Y, Z;
};

PCMM_HD void pt_identity(pt &r) {
    fe_zero(r.X);
    fe_one_mont(r.Y);
    fe_zero(r.Z);
}

PCMM_HD bool pt_is_identity(const pt &a) { return fe_is_zero(a.Z); }

// multiplication policies for the group law: inlined, or (device, hot loop) an
// out-of-line call that keeps the loop body inside the instruction cache
struct MulInline {
    static PCMM_HD void mul(fe &r, const fe &a, const fe &b) { fe_mul(r, a, b); }
};
#if defined(__CUDA_ARCH__) && defined(PCMM_HAVE_FAST_MUL)
struct MulCall {
    static __device__ __forceinline__ void mul(fe &r, const fe &a, const fe &b) { r = fe_mul_call(a, b); }
};
#else
typedef MulInline MulCall;
#endif

#if defined(__CUDA_ARCH__) && defined(PCMM_HAVE_FAST_MUL)
// RCB16 Algorithm 4 with its 14 products grouped into 7 independent pairs
// (same operations as pt_add_g, reordered along the data flow; each pair is one
// out-of-line call that interleaves two Montgomery products).
__device__ __forceinline__ void mul2(fe &r0, const fe &a0, const fe &b0, fe &r1, const fe &a1, const fe &b1) {
    fe2 r = fe_mul2_call(a0, b0, a1, b1);
    r0 = r.x;
    r1 = r.y;
}

__device__ __forceinline__ void pt_add_pair(pt &R, const pt &P, const pt &Q) {
    fe m1, m2, m3, m4, m5, m6, s0, s1, b;
    fe_b_mont(b);
    mul2(m1, P.X, Q.X, m2, P.Y, Q.Y);              // t0 = X1 X2, t1 = Y1 Y2
    fe_add(s0, P.X, P.Y);
    fe_add(s1, Q.X, Q.Y);
    mul2(m3, P.Z, Q.Z, m4, s0, s1);                // t2 = Z1 Z2, t3 = (X1+Y1)(X2+Y2)
    fe_add(s0, P.Y, P.Z);
    fe_add(s1, Q.Y, Q.Z);
    fe a0, a1;
    fe_add(a0, P.X, P.Z);
    fe_add(a1, Q.X, Q.Z);
    mul2(m5, s0, s1, m6, a0, a1);                  // t4 = (Y1+Z1)(Y2+Z2), X3 = (X1+Z1)(X2+Z2)
    fe t3, t4, y3;
    fe_add(s0, m1, m2);
    fe_sub(t3, m4, s0);                            // t3 = t3 - (t0 + t1)
    fe_add(s0, m2, m3);
    fe_sub(t4, m5, s0);                            // t4 = t4 - (t1 + t2)
    fe_add(s0, m1, m3);
    fe_sub(y3, m6, s0);                            // Y3 = X3 - (t0 + t2)
    fe m7, m8;
    mul2(m7, b, m3, m8, b, y3);                    // Z3 = b t2, Y3 = b Y3
    fe x3, z3;
    fe_sub(x3, y3, m7);                            // X3 = Y3 - Z3
    fe_add(z3, x3, x3);
    fe_add(x3, x3, z3);                            // X3 = 3 X3
    fe_sub(z3, m2, x3);                            // Z3 = t1 - X3
    fe_add(x3, m2, x3);                            // X3 = t1 + X3
    fe t2b;
    fe_add(s0, m3, m3);
    fe_add(t2b, s0, m3);                           // t2 = 3 t2
    fe_sub(y3, m8, t2b);
    fe_sub(y3, y3, m1);                            // Y3 = Y3 - t2 - t0
    fe_add(s0, y3, y3);
    fe_add(y3, s0, y3);                            // Y3 = 3 Y3
    fe t0b;
    fe_add(s0, m1, m1);
    fe_add(t0b, s0, m1);
    fe_sub(t0b, t0b, t2b);                         // t0 = 3 t0 - t2
    fe m9, m10, m11, m12, m13, m14;
    mul2(m9, t4, y3, m10, t0b, y3);                // t1 = t4 Y3, t2 = t0 Y3
    mul2(m11, x3, z3, m12, t3, x3);                // Y3 = X3 Z3, X3 = t3 X3
    mul2(m13, t4, z3, m14, t3, t0b);               // Z3 = t4 Z3, t1 = t3 t0
    fe_add(R.Y, m11, m10);
    fe_sub(R.X, m12, m9);
    fe_add(R.Z, m13, m14);
}

// RCB16 Algorithm 5: complete MIXED addition R = P + Q for a = -3 with Q affine
// (Z2 = 1, Q != infinity): Alg. 4 with Z2 = 1, 11M + 2m_b.  The 13 products are
// grouped into 6 independent pairs + 1.  Not on the hot path: measured in
// k_accum it saves only 1.5 % (the loop is latency-bound), less than converting
// the tables to affine coordinates would cost.
__device__ __forceinline__ void pt_madd_pair(pt &R, const pt &P, const fe &X2, const fe &Y2) {
    fe b;
    fe_b_mont(b);
    fe m1, m6, m2, m8, m4, m5, m7, s0, s1, y3;
    mul2(m1, P.X, X2, m6, X2, P.Z);               // t0 = X1 X2, Y3 = X2 Z1
    fe_add(y3, m6, P.X);                          // Y3 = X2 Z1 + X1
    mul2(m2, P.Y, Y2, m8, b, y3);                 // t1 = Y1 Y2, Y3' = b Y3 (step 18 operand)
    fe_add(s0, X2, Y2);
    fe_add(s1, P.X, P.Y);
    mul2(m4, s0, s1, m5, Y2, P.Z);                // t3 = (X2+Y2)(X1+Y1), t4 = Y2 Z1
    m7 = fe_mul_call(b, P.Z);                     // Z3 = b Z1
    fe t3, t4, x3, z3, t2, t0;
    fe_add(s0, m1, m2);
    fe_sub(t3, m4, s0);                           // t3 = t3 - (t0 + t1)
    fe_add(t4, m5, P.Y);                          // t4 = Y2 Z1 + Y1
    fe_sub(x3, y3, m7);                           // X3 = Y3 - Z3
    fe_add(z3, x3, x3);
    fe_add(x3, x3, z3);                           // X3 = 3 X3
    fe_sub(z3, m2, x3);                           // Z3 = t1 - X3
    fe_add(x3, m2, x3);                           // X3 = t1 + X3
    fe_add(s0, P.Z, P.Z);
    fe_add(t2, s0, P.Z);                          // t2 = 3 Z1
    fe_sub(y3, m8, t2);
    fe_sub(y3, y3, m1);                           // Y3 = b Y3 - t2 - t0
    fe_add(s0, y3, y3);
    fe_add(y3, s0, y3);                           // Y3 = 3 Y3
    fe_add(s0, m1, m1);
    fe_add(t0, s0, m1);
    fe_sub(t0, t0, t2);                           // t0 = 3 t0 - t2
    fe m9, m10, m11, m12, m13, m14;
    mul2(m9, t4, y3, m10, t0, y3);                // t1 = t4 Y3, t2 = t0 Y3
    mul2(m11, x3, z3, m12, t3, x3);               // Y3 = X3 Z3, X3 = t3 X3
    mul2(m13, t4, z3, m14, t3, t0);               // Z3 = t4 Z3, t1 = t3 t0
    fe_add(R.Y, m11, m10);
    fe_sub(R.X, m12, m9);
    fe_add(R.Z, m13, m14);
}

// RCB16 Algorithm 6 (doubling, a = -3) with its 13 products grouped into 6
// independent pairs + 1 (same operations, reordered along the data flow).
__device__ __forceinline__ void pt_dbl_pair(pt &R, const pt &P) {
    fe b;
    fe_b_mont(b);
    fe t0, t1, t2, t3, z3, yz;
    mul2(t0, P.X, P.X, t1, P.Y, P.Y);            // t0 = X^2, t1 = Y^2
    mul2(t2, P.Z, P.Z, t3, P.X, P.Y);            // t2 = Z^2, t3 = X Y
    mul2(z3, P.X, P.Z, yz, P.Y, P.Z);            // Z3 = X Z, t0' = Y Z (step 28)
    fe_add(t3, t3, t3);                          // t3 = 2 X Y
    fe_add(z3, z3, z3);                          // Z3 = 2 X Z
    fe y3, bz;
    mul2(y3, b, t2, bz, b, z3);                  // Y3 = b t2, Z3 = b Z3
    fe x3, s;
    fe_sub(y3, y3, z3);                          // Y3 = Y3 - Z3
    fe_add(x3, y3, y3);
    fe_add(y3, x3, y3);                          // Y3 = 3 Y3
    fe_sub(x3, t1, y3);                          // X3 = t1 - Y3
    fe_add(y3, t1, y3);                          // Y3 = t1 + Y3
    fe_add(s, t2, t2);
    fe_add(t2, t2, s);                           // t2 = 3 t2
    fe_sub(bz, bz, t2);
    fe_sub(bz, bz, t0);                          // Z3 = b Z3 - t2 - t0
    fe_add(s, bz, bz);
    fe_add(bz, bz, s);                           // Z3 = 3 Z3
    fe_add(s, t0, t0);
    fe_add(t0, s, t0);
    fe_sub(t0, t0, t2);                          // t0 = 3 t0 - t2
    fe_add(yz, yz, yz);                          // t0' = 2 Y Z
    fe m7, m8, m10, m12;
    mul2(m7, x3, y3, m8, x3, t3);                // Y3 = X3 Y3, X3 = X3 t3
    mul2(m10, t0, bz, m12, yz, bz);              // t0 = t0 Z3, Z3 = t0' Z3
    fe m13 = fe_mul_call(yz, t1);                // Z3 = t0' t1
    fe_add(R.Y, m7, m10);                        // Y3 = Y3 + t0
    fe_sub(R.X, m8, m12);                        // X3 = X3 - Z3
    fe_add(m13, m13, m13);
    fe_add(R.Z, m13, m13);                       // Z3 = 4 t0' t1
}

PCMM_HD void pt_neg(pt &R, const pt &P);

// v * P for a small signed v with warp-uniform v (schoolbook): binary double-and-add
// with the paired formulas.
__device__ __forceinline__ void pt_mul_small_pair(pt &R, int v, const pt &P) {
    const unsigned a = v < 0 ? (unsigned)(-v) : (unsigned)v;
    pt acc;
    pt_identity(acc);
    if (a != 0) {
        const int top = 31 - __clz(a);
        acc = P;
        for (int i = top - 1; i >= 0; i--) {
            pt_dbl_pair(acc, acc);
            if ((a >> i) & 1u) pt_add_pair(acc, acc, P);
        }
        if (v < 0) pt_neg(acc, acc);
    }
    R = acc;
}
#else
template <class M> PCMM_HD void pt_add_g(pt &R, const pt &P, const pt &Q);
struct MulInline;
PCMM_HD void pt_add_pair(pt &R, const pt &P, const pt &Q) { pt_add_g<MulInline>(R, P, Q); }
template <class M> PCMM_HD void pt_dbl_g(pt &R, const pt &P);
template <class M> PCMM_HD void pt_mul_small_g(pt &R, int v, const pt &P);
PCMM_HD void pt_dbl_pair(pt &R, const pt &P) { pt_dbl_g<MulInline>(R, P); }
PCMM_HD void pt_madd_pair(pt &R, const pt &P, const fe &X2, const fe &Y2) {
    pt Q;
    Q.X = X2;
    Q.Y = Y2;
    fe_one_mont(Q.Z);
    pt_add_g<MulInline>(R, P, Q);
}
PCMM_HD void pt_mul_small_pair(pt &R, int v, const pt &P) { pt_mul_small_g<MulInline>(R, v, P); }
#endif

// RCB16 Algorithm 4: complete projective addition for a = -3.
template <class M>
PCMM_HD void pt_add_g(pt &R, const pt &P, const pt &Q) {
    fe t0, t1, t2, t3, t4, X3, Y3, Z3, b;
    fe_b_mont(b);
    M::mul(t0, P.X, Q.X);
    M::mul(t1, P.Y, Q.Y);
    M::mul(t2, P.Z, Q.Z);
    fe_add(t3, P.X, P.Y);
    fe_add(t4, Q.X, Q.Y);
    M::mul(t3, t3, t4);
    fe_add(t4, t0, t1);
    fe_sub(t3, t3, t4);
    fe_add(t4, P.Y, P.Z);
    fe_add(X3, Q.Y, Q.Z);
    M::mul(t4, t4, X3);
    fe_add(X3, t1, t2);
    fe_sub(t4, t4, X3);
    fe_add(X3, P.X, P.Z);
    fe_add(Y3, Q.X, Q.Z);
    M::mul(X3, X3, Y3);
    fe_add(Y3, t0, t2);
    fe_sub(Y3, X3, Y3);
    M::mul(Z3, b, t2);
    fe_sub(X3, Y3, Z3);
    fe_add(Z3, X3, X3);
    fe_add(X3, X3, Z3);
    fe_sub(Z3, t1, X3);
    fe_add(X3, t1, X3);
    M::mul(Y3, b, Y3);
    fe_add(t1, t2, t2);
    fe_add(t2, t1, t2);
    fe_sub(Y3, Y3, t2);
    fe_sub(Y3, Y3, t0);
    fe_add(t1, Y3, Y3);
    fe_add(Y3, t1, Y3);
    fe_add(t1, t0, t0);
    fe_add(t0, t1, t0);
    fe_sub(t0, t0, t2);
    M::mul(t1, t4, Y3);
    M::mul(t2, t0, Y3);
    M::mul(Y3, X3, Z3);
    fe_add(Y3, Y3, t2);
    M::mul(X3, t3, X3);
    fe_sub(X3, X3, t1);
    M::mul(Z3, t4, Z3);
    M::mul(t1, t3, t0);
    fe_add(Z3, Z3, t1);
    R.X = X3;
    R.Y = Y3;
    R.Z = Z3;
}

PCMM_HD void pt_add(pt &R, const pt &P, const pt &Q) { pt_add_g<MulInline>(R, P, Q); }

// RCB16 Algorithm 6: complete projective doubling for a = -3.
template <class M>
PCMM_HD void pt_dbl_g(pt &R, const pt &P) {
    fe t0, t1, t2, t3, X3, Y3, Z3, b;
    fe_b_mont(b);
    M::mul(t0, P.X, P.X);
    M::mul(t1, P.Y, P.Y);
    M::mul(t2, P.Z, P.Z);
    M::mul(t3, P.X, P.Y);
    fe_add(t3, t3, t3);
    M::mul(Z3, P.X, P.Z);
    fe_add(Z3, Z3, Z3);
    M::mul(Y3, b, t2);
    fe_sub(Y3, Y3, Z3);
    fe_add(X3, Y3, Y3);
    fe_add(Y3, X3, Y3);
    fe_sub(X3, t1, Y3);
    fe_add(Y3, t1, Y3);
    M::mul(Y3, X3, Y3);
    M::mul(X3, X3, t3);
    fe_add(t3, t2, t2);
    fe_add(t2, t2, t3);
    M::mul(Z3, b, Z3);
    fe_sub(Z3, Z3, t2);
    fe_sub(Z3, Z3, t0);
    fe_add(t3, Z3, Z3);
    fe_add(Z3, Z3, t3);
    fe_add(t3, t0, t0);
    fe_add(t0, t3, t0);
    fe_sub(t0, t0, t2);
    M::mul(t0, t0, Z3);
    fe_add(Y3, Y3, t0);
    M::mul(t0, P.Y, P.Z);
    fe_add(t0, t0, t0);
    M::mul(Z3, t0, Z3);
    fe_sub(X3, X3, Z3);
    M::mul(Z3, t0, t1);
    fe_add(Z3, Z3, Z3);
    fe_add(Z3, Z3, Z3);
    R.X = X3;
    R.Y = Y3;
    R.Z = Z3;
}

PCMM_HD void pt_dbl(pt &R, const pt &P) { pt_dbl_g<MulInline>(R, P); }

// Out-of-line copies for the cold paths (table build, schoolbook ECSMs, encrypt,
// decrypt): keeps compile time and code size bounded; the hot accumulate loop
// uses the inlined forms above.
PCMM_HD_NOINLINE void pt_add_nl(pt &R, const pt &P, const pt &Q) { pt_add(R, P, Q); }
PCMM_HD_NOINLINE void pt_dbl_nl(pt &R, const pt &P) { pt_dbl(R, P); }

PCMM_HD void pt_neg(pt &R, const pt &P) {
    R.X = P.X;
    fe_neg(R.Y, P.Y);
    R.Z = P.Z;
}

// v * P for a small signed integer v (|v| < 2^31): left-to-right binary
// double-and-add over the bits of |v|, then negation for v < 0 (R10:
// -(|v| P) is the group element (q - |v|) P).  v = 0 gives the identity.
template <class M>
PCMM_HD void pt_mul_small_g(pt &R, int v, const pt &P) {
    unsigned a = v < 0 ? (unsigned)(-v) : (unsigned)v;
    pt acc;
    pt_identity(acc);
    int top = 31;
    while (top >= 0 && !((a >> top) & 1u)) top--;
    for (int i = top; i >= 0; i--) {
        if (i != top) pt_dbl_g<M>(acc, acc);
        if ((a >> i) & 1u) {
            if (i == top) acc = P;
            else pt_add_g<M>(acc, acc, P);
        }
    }
    if (v < 0) pt_neg(acc, acc);
    R = acc;
}

PCMM_HD void pt_mul_small(pt &R, int v, const pt &P) {
    unsigned a = v < 0 ? (unsigned)(-v) : (unsigned)v;
    pt acc;
    pt_identity(acc);
    int top = 31;
    while (top >= 0 && !((a >> top) & 1u)) top--;
    for (int i = top; i >= 0; i--) {
        if (i != top) pt_dbl_nl(acc, acc);
        if ((a >> i) & 1u) {
            if (i == top) acc = P;
            else pt_add_nl(acc, acc, P);
        }
    }
    if (v < 0) pt_neg(acc, acc);
    R = acc;
}

// k * P for a 256-bit scalar k (8 little-endian 32-bit words), MSB-first
// double-and-add with complete formulas (used by encrypt / keygen / decrypt,
// not by the PC-MM hot path).
PCMM_HD void pt_mul_scalar(pt &R, const uint32_t k[8], const pt &P) {
    pt acc;
    pt_identity(acc);
    bool started = false;
    for (int i = 255; i >= 0; i--) {
        if (started) pt_dbl_nl(acc, acc);
        if ((k[i >> 5] >> (i & 31)) & 1u) {
            if (started) pt_add_nl(acc, acc, P);
            else { acc = P; started = true; }
        }
    }
    R = acc;
}

// (x, y) affine in Montgomery form -> projective with Z = 1
PCMM_HD void pt_from_affine(pt &R, const fe &x, const fe &y) {
    R.X = x;
    R.Y = y;
    fe_one_mont(R.Z);
}

// y^2 == x^3 - 3x + b (Montgomery form inputs)
PCMM_HD bool affine_on_curve(const fe &x, const fe &y) {
    fe y2, x3, t, b;
    fe_sqr(y2, y);
    fe_sqr(x3, x);
    fe_mul(x3, x3, x);
    fe_add(t, x, x);
    fe_add(t, t, x);
    fe_sub(x3, x3, t);
    fe_b_mont(b);
    fe_add(x3, x3, b);
    return fe_eq(x3, y2);
}

// canonical 64-byte point (x||y big-endian, identity = 64 zero bytes) -> projective
// Montgomery point.  Returns 0 ok, 1 if not on the curve / not reduced.
PCMM_HD int pt_from_canonical(pt &R, const uint8_t *b64) {
    uint32_t any = 0;
    for (int i = 0; i < 64; i++) any |= b64[i];
    if (any == 0) {
        pt_identity(R);
        return 0;
    }
    fe x, y;
    int okx = fe_from_be_bytes(x, b64);
    int oky = fe_from_be_bytes(y, b64 + 32);
    fe_to_mont(x, x);
    fe_to_mont(y, y);
    pt_from_affine(R, x, y);
    return (okx && oky && affine_on_curve(x, y)) ? 0 : 1;
}

// projective Montgomery point with known inverse zi = 1/Z (Montgomery) ->
// canonical bytes; the identity (Z = 0) gives 64 zero bytes.
PCMM_HD void pt_to_canonical_with_inv(uint8_t *b64, const pt &P, const fe &zi) {
    if (pt_is_identity(P)) {
        for (int i = 0; i < 64; i++) b64[i] = 0;
        return;
    }
    fe x, y;
    fe_mul(x, P.X, zi);
    fe_mul(y, P.Y, zi);
    fe_from_mont(x, x);
    fe_from_mont(y, y);
    fe_to_be_bytes(b64, x);
    fe_to_be_bytes(b64 + 32, y);
}

PCMM_HD void pt_to_canonical(uint8_t *b64, const pt &P) {
    fe zi;
    fe_inv(zi, P.Z);
    pt_to_canonical_with_inv(b64, P, zi);
}

}  // namespace pcmm
