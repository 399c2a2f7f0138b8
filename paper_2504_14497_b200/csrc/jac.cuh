// jac.cuh -- Jacobian accumulator + affine mixed addition with a complete
// fallback (used by the accumulate kernels in hot.cu and the fixed-base comb
// encryption / BSGS decryption in next2.cu).
#pragma once
#include "ec.cuh"
#include "internal.h"

namespace pcmm {

// ------------------------------------------------------------ Jacobian accumulator
// The accumulate loop adds affine table entries (k_affine writes
// the tables as (x, y)) into a Jacobian accumulator (x = X/Z^2, y = Y/Z^3) that
// carries ZZ = Z^2: the mixed addition below is 8M + 3S with five out-of-line
// product calls of two or three independent products each, against 12M + 2m_b
// in seven calls for the complete homogeneous addition.  The mixed formula is
// not complete: the identity (accumulator or entry) and H = 0 (acc = +-Q) take
// the out-of-line general path, which runs the complete RCB16 addition
// (ec.cuh) on homogeneous images of both points, so every input is handled.
struct jacc {
    fe X, Y, Z, ZZ;
    uint32_t inf;                 // 1 while the accumulator is the identity
};

// affine table entry = 16 words (x, y); the identity has x = all ones (never a
// residue in [0, p): p's top two words are 0xffffffff, 0x00000001)
__device__ __forceinline__ bool aff_is_inf(const fe &x) { return (x.v[7] & x.v[6]) == 0xffffffffu; }

static __device__ __noinline__ jacc jac_add_slow(jacc A, const fe x2, const fe y2) {
#ifdef __CUDA_ARCH__
    if (aff_is_inf(x2)) return A;
    if (A.inf) {
        A.X = x2;
        A.Y = y2;
        fe_one_mont(A.Z);
        A.ZZ = A.Z;
        A.inf = 0;
        return A;
    }
    pt P, Q, R;
    mul2(P.X, A.X, A.Z, P.Z, A.Z, A.ZZ);          // (X Z : Y : Z^3) = the same point, homogeneous
    P.Y = A.Y;
    Q.X = x2;
    Q.Y = y2;
    fe_one_mont(Q.Z);
    pt_add_pair(R, P, Q);                         // complete (RCB16 Alg. 4)
    if (fe_is_zero(R.Z)) {
        A.inf = 1;
        return A;
    }
    A.Z = R.Z;                                    // back to Jacobian: (X Z, Y Z^2, Z)
    A.ZZ = fe_mul_call(R.Z, R.Z);
    mul2(A.X, R.X, R.Z, A.Y, R.Y, A.ZZ);
#endif
    return A;
}

#ifndef PCMM_JAC_FORMULA
#define PCMM_JAC_FORMULA 1       // 1: 8M + 3S, 2: 7M + 4S (madd-2007-bl; measured 2.7 % slower at 256^3 w=4, 2 % faster at 512^3 w=2)
#endif

// A += (x2, y2), U1 = X1, S1 = Y1 (Z2 = 1).
// Formula 1: U2 = x2 Z1^2, S2 = y2 Z1^3, H = U2 - X1, R = S2 - Y1,
//   X3 = R^2 - H^3 - 2 X1 H^2, Y3 = R (X1 H^2 - X3) - Y1 H^3, Z3 = Z1 H, ZZ3 = Z1^2 H^2.
// Formula 2 (madd-2007-bl): HH = H^2, I = 4 HH, J = H I, r = 2 (S2 - Y1), V = X1 I,
//   X3 = r^2 - J - 2V, Y3 = r (V - X3) - 2 Y1 J, Z3 = (Z1 + H)^2 - Z1^2 - HH, ZZ3 = Z3^2:
//   7 products + 4 squares (the squares at 36/64 of a product) in four calls of 2, 3, 4, 2.
__device__ __forceinline__ void jac_add_aff(jacc &A, const fe &x2, const fe &y2) {
#ifdef __CUDA_ARCH__
    if (A.inf | aff_is_inf(x2)) {
        A = jac_add_slow(A, x2, y2);
        return;
    }
    const fe2 ut = fe_mul2_hot(x2, A.ZZ, A.Z, A.ZZ);   // U2 = x2 ZZ, T1 = Z^3
    const fe &U2 = ut.x, &T1 = ut.y;
    fe H;
    fe_sub(H, U2, A.X);
    if (fe_is_zero(H)) {
        A = jac_add_slow(A, x2, y2);
        return;
    }
#if PCMM_JAC_FORMULA == 1
    const fe2 sh = fe_mulsqr_hot(y2, T1, H);     // S2 = y2 Z^3, HH = H^2
    const fe &S2 = sh.x, &HH = sh.y;
    fe R;
    fe_sub(R, S2, A.Y);
    const fe3 t = fe_mul3_hot(H, HH, A.X, HH, A.ZZ, HH);  // H^3, V = X1 H^2, ZZ3
    const fe2 zr = fe_mulsqr_hot(A.Z, H, R);     // Z3 = Z1 H, R^2
    const fe &Z3 = zr.x, &R2 = zr.y;
    fe X3, V2, D;
    fe_add(V2, t.y, t.y);
    fe_sub(X3, R2, t.x);
    fe_sub(X3, X3, V2);                           // X3 = R^2 - H^3 - 2V
    fe_sub(D, t.y, X3);
    const fe2 yy = fe_mul2_hot(R, D, A.Y, t.x);   // R (V - X3), Y1 H^3
    fe_sub(A.Y, yy.x, yy.y);
    A.X = X3;
    A.Z = Z3;
    A.ZZ = t.z;
#else
    fe ZH;
    fe_add(ZH, A.Z, H);
    const fe3 s = fe_m1s2_call(y2, T1, H, ZH);    // S2 = y2 Z^3, HH = H^2, (Z1 + H)^2
    const fe &S2 = s.x, &HH = s.y;
    fe r, I, Z3;
    fe_sub(r, S2, A.Y);
    fe_add(r, r, r);                              // r = 2 (S2 - Y1)
    fe_add(I, HH, HH);
    fe_add(I, I, I);                              // I = 4 HH
    fe_sub(Z3, s.z, A.ZZ);
    fe_sub(Z3, Z3, HH);                           // Z3 = (Z1 + H)^2 - ZZ - HH
    const fe4 q = fe_m2s2_call(H, I, A.X, I, r, Z3);   // J = H I, V = X1 I, r^2, ZZ3 = Z3^2
    const fe &J = q.x, &V = q.y;
    fe X3, V2, D;
    fe_add(V2, V, V);
    fe_sub(X3, q.z, J);
    fe_sub(X3, X3, V2);                           // X3 = r^2 - J - 2V
    fe_sub(D, V, X3);
    fe P1, P2;
    mul2(P1, r, D, P2, A.Y, J);                   // r (V - X3), Y1 J
    fe_add(P2, P2, P2);
    fe_sub(A.Y, P1, P2);                          // Y3 = r (V - X3) - 2 Y1 J
    A.X = X3;
    A.Z = Z3;
    A.ZZ = q.w;
#endif
#endif
}

__device__ __forceinline__ void jac_init(jacc &A) {
    fe_zero(A.X);
    fe_zero(A.Y);
    fe_zero(A.Z);
    fe_zero(A.ZZ);
    A.inf = 1;
}

// Jacobian -> homogeneous projective (X Z : Y : Z^3) for the output buffer
__device__ __forceinline__ void jac_to_proj(pt &o, const jacc &A) {
#ifdef __CUDA_ARCH__
    if (A.inf) {
        pt_identity(o);
    } else {
        mul2(o.X, A.X, A.Z, o.Z, A.Z, A.ZZ);
        o.Y = A.Y;
    }
#endif
}

// A <- 2A (a = -3, dbl-2001-b with ZZ carried): gamma = Y^2, beta = X gamma,
// alpha = 3 (X - ZZ)(X + ZZ), X3 = alpha^2 - 8 beta, Z3 = (Y + Z)^2 - gamma - ZZ,
// Y3 = alpha (4 beta - X3) - 8 gamma^2, ZZ3 = Z3^2: 3M + 5S.  Complete for
// P-256 (no point of order 2); the identity stays the identity.
__device__ __forceinline__ void jac_dbl(jacc &A) {
#ifdef __CUDA_ARCH__
    if (A.inf) return;
    fe gamma, t0, t1, alpha, yz, beta, a2, g2, x3, z3, u;
    fe_sqr(gamma, A.Y);
    fe_sub(t0, A.X, A.ZZ);
    fe_add(t1, A.X, A.ZZ);
    fe_mul(t0, t0, t1);
    fe_add(alpha, t0, t0);
    fe_add(alpha, alpha, t0);                     // alpha = 3 (X - ZZ)(X + ZZ)
    fe_add(yz, A.Y, A.Z);
    fe_sqr(yz, yz);
    fe_mul(beta, A.X, gamma);
    fe_sqr(a2, alpha);
    fe_sqr(g2, gamma);
    fe_add(u, beta, beta);
    fe_add(u, u, u);                              // 4 beta
    fe_add(t1, u, u);                             // 8 beta
    fe_sub(x3, a2, t1);                           // X3 = alpha^2 - 8 beta
    fe_sub(z3, yz, gamma);
    fe_sub(z3, z3, A.ZZ);                         // Z3 = (Y + Z)^2 - gamma - ZZ
    fe_sub(u, u, x3);
    fe_mul(u, alpha, u);                          // alpha (4 beta - X3)
    fe_add(g2, g2, g2);
    fe_add(g2, g2, g2);
    fe_add(g2, g2, g2);                           // 8 gamma^2
    fe_sub(A.Y, u, g2);
    A.X = x3;
    A.Z = z3;
    fe_sqr(A.ZZ, z3);
#endif
}

// ------------------------------------------------------------ XYZZ accumulator
// x = X/ZZ, y = Y/ZZZ with ZZ^3 = ZZZ^2 (Chudnovsky-style "XYZZ" coordinates).
// Mixed addition of an affine entry (madd-2008-s): U2 = x2 ZZ1, S2 = y2 ZZZ1,
// P = U2 - X1, R = S2 - Y1, PP = P^2, PPP = P PP, Q = X1 PP,
// X3 = R^2 - PPP - 2Q, Y3 = R (Q - X3) - Y1 PPP, ZZ3 = ZZ1 PP, ZZZ3 = ZZZ1 PPP:
// 8M + 2S in four groups of 2, 2 (squares), 3, 3 independent products, one
// product fewer than the Jacobian step above (which also has to form Z^3 and
// Z3 = Z1 H).  Same exceptional cases as jac_add_aff (identity, P = 0), which
// take the complete RCB16 path on homogeneous images.
#ifndef PCMM_ACC_PERM
// 1 (default): product order / operand order of the pipelined step from PCMM_G1, _G2, _G3, _SWAPM;
// 0: the grouped calls in their original order.  Measured with k_accum_g2 (256^3 / 512^3 / ML step):
// 0: 3.960 / 22.69 / 2.156 ms; 1 with the orders below: 3.930 / 22.34 / 2.145
#define PCMM_ACC_PERM 1
#endif
#ifndef PCMM_G1
#define PCMM_G1 12
#endif
#ifndef PCMM_G2
#define PCMM_G2 2341            // PPP, Q, ZZ3, R^2
#endif
#ifndef PCMM_G3
#define PCMM_G3 4123            // U2', R (Q - X3), Y PPP, ZZZ3
#endif
#ifndef PCMM_SWAPM
#define PCMM_SWAPM 8            // ZZ3 = PP ZZ (operands swapped): 256^3 3.931 -> 3.913 ms, 512^3 22.33 -> 22.21
#endif
#ifndef PCMM_ACC_LZ3
#define PCMM_ACC_LZ3 0          // 1: PP, ZZ3, ZZZ3 of the pipelined step without the final conditional subtraction
#endif
struct xyzz {
    fe X, Y, ZZ, ZZZ;
    uint32_t inf;                 // 1 while the accumulator is the identity
};

__device__ __forceinline__ void xyzz_init(xyzz &A) {
    fe_zero(A.X);
    fe_zero(A.Y);
    fe_zero(A.ZZ);
    fe_zero(A.ZZZ);
    A.inf = 1;
}

// A = 2 (x, y) for an affine input (mdbl-2008-s-1, a = -3): U = 2y, V = U^2,
// W = U V, S = x V, M = 3 (x^2 - 1), X3 = M^2 - 2S, Y3 = M (S - X3) - W y,
// ZZ3 = V, ZZZ3 = W: 4M + 3S.  y != 0 on P-256 (no point of order 2).
__device__ __forceinline__ void xyzz_dbl_aff(xyzz &A, const fe &x, const fe &y) {
    fe U, V, W, Sv, M, x2, t, X3, D;
    fe_add(U, y, y);                               // U = 2y
    fe_sqr(V, U);                                  // V = U^2
    fe_mul(W, U, V);                               // W = U V
    fe_mul(Sv, x, V);                              // S = x V
    fe_sqr(x2, x);
    fe one;
    fe_one_mont(one);
    fe_sub(t, x2, one);
    fe_add(M, t, t);
    fe_add(M, M, t);                               // M = 3 (x^2 - 1) = 3 x^2 + a, a = -3
    fe_sqr(X3, M);
    fe_sub(X3, X3, Sv);
    fe_sub(X3, X3, Sv);                            // X3 = M^2 - 2S
    fe_sub(D, Sv, X3);
    fe_mul(D, M, D);
    fe_mul(t, W, y);
    fe_sub(A.Y, D, t);                             // Y3 = M (S - X3) - W y
    A.X = X3;
    A.ZZ = V;
    A.ZZZ = W;
    A.inf = 0;
}

// A <- 2A in XYZZ (dbl-2008-s-1, a = -3): U = 2Y, V = U^2, W = U V, S = X V,
// M = 3 (X - ZZ)(X + ZZ), X3 = M^2 - 2S, Y3 = M (S - X3) - W Y, ZZ3 = V ZZ,
// ZZZ3 = W ZZZ: 7M + 2S.  The identity stays the identity.
__device__ __forceinline__ void xyzz_dbl(xyzz &A) {
#ifdef __CUDA_ARCH__
    if (A.inf) return;
    fe U, V, t0, t1, M, X3, D;
    fe_add(U, A.Y, A.Y);
    fe_sqr(V, U);
    fe_sub(t0, A.X, A.ZZ);
    fe_add(t1, A.X, A.ZZ);
    const fe4 g = fe_mul4_hot(U, V, A.X, V, t0, t1, V, A.ZZ);    // W, S, (X - ZZ)(X + ZZ), ZZ3
    const fe &W = g.x, &Sv = g.y;
    fe_add(M, g.z, g.z);
    fe_add(M, M, g.z);                                            // M = 3 (X - ZZ)(X + ZZ)
    const fe3 h = fe_sqr_mul2_hot(M, W, A.Y, W, A.ZZZ);          // M^2, W Y, ZZZ3
    fe_sub(X3, h.x, Sv);
    fe_sub(X3, X3, Sv);                                           // X3 = M^2 - 2S
    fe_sub(D, Sv, X3);
    fe MD;
    fe_mul(MD, M, D);                                             // M (S - X3)
    fe_sub(A.Y, MD, h.y);                                         // Y3 = M (S - X3) - W Y
    A.X = X3;
    A.ZZ = g.w;
    A.ZZZ = h.z;
#endif
}

// homogeneous (X : Y : Z), Z != 0  ->  XYZZ (X Z, Y Z^2, Z^2, Z^3)
__device__ __forceinline__ void xyzz_from_proj(xyzz &A, const pt &o) {
#ifdef __CUDA_ARCH__
    A.ZZ = fe_mul_call(o.Z, o.Z);
    mul2(A.X, o.X, o.Z, A.Y, o.Y, A.ZZ);
    A.ZZZ = fe_mul_call(A.ZZ, o.Z);
    A.inf = 0;
#endif
}

// XYZZ -> homogeneous (X ZZZ : Y ZZ : ZZ ZZZ) (x = X/ZZ, y = Y/ZZZ)
__device__ __forceinline__ void xyzz_to_proj(pt &o, const xyzz &A) {
#ifdef __CUDA_ARCH__
    if (A.inf) {
        pt_identity(o);
    } else {
#if PCMM_ACC_LZ3
        fe zz, zzz;                               // ZZ, ZZZ may be in [p, 2^256) (xyzz_add_aff_pipe)
        fe_cond_sub_p(zz, A.ZZ, 0);
        fe_cond_sub_p(zzz, A.ZZZ, 0);
        mul2(o.X, A.X, zzz, o.Y, A.Y, zz);
        o.Z = fe_mul_call(zz, zzz);
#else
        mul2(o.X, A.X, A.ZZZ, o.Y, A.Y, A.ZZ);
        o.Z = fe_mul_call(A.ZZ, A.ZZZ);
#endif
    }
#endif
}

static __device__ __noinline__ xyzz xyzz_add_slow(xyzz A, const fe x2, const fe y2) {
#ifdef __CUDA_ARCH__
    if (aff_is_inf(x2)) return A;
    if (A.inf) {
        A.X = x2;
        A.Y = y2;
        fe_one_mont(A.ZZ);
        A.ZZZ = A.ZZ;
        A.inf = 0;
        return A;
    }
    pt P, Q, R;
    xyzz_to_proj(P, A);
    Q.X = x2;
    Q.Y = y2;
    fe_one_mont(Q.Z);
    pt_add_pair(R, P, Q);                         // complete (RCB16 Alg. 4)
    if (fe_is_zero(R.Z)) {
        A.inf = 1;
        return A;
    }
    xyzz_from_proj(A, R);
#endif
    return A;
}

__device__ __forceinline__ void xyzz_add_aff(xyzz &A, const fe &x2, const fe &y2) {
#ifdef __CUDA_ARCH__
    if (A.inf | aff_is_inf(x2)) {
        A = xyzz_add_slow(A, x2, y2);
        return;
    }
    const fe2 us = fe_mul2_hot(x2, A.ZZ, y2, A.ZZZ);   // U2 = x2 ZZ, S2 = y2 ZZZ
    fe P, R;
    fe_sub(P, us.x, A.X);
    if (fe_is_zero(P)) {
        A = xyzz_add_slow(A, x2, y2);
        return;
    }
    fe_sub(R, us.y, A.Y);
    const fe2 sq = fe_sqr2_hot(P, R);                  // PP = P^2, R^2
    const fe &PP = sq.x;
    const fe3 t = fe_mul3_hot(P, PP, A.X, PP, A.ZZ, PP);   // PPP, Q = X1 PP, ZZ3
    fe X3, Q2, D;
    fe_add(Q2, t.y, t.y);
    fe_sub(X3, sq.y, t.x);
    fe_sub(X3, X3, Q2);                           // X3 = R^2 - PPP - 2Q
    fe_sub(D, t.y, X3);
    const fe3 u = fe_mul3_hot(R, D, A.Y, t.x, A.ZZZ, t.x);  // R (Q - X3), Y1 PPP, ZZZ3
    fe_sub(A.Y, u.x, u.y);
    A.X = X3;
    A.ZZ = t.z;
    A.ZZZ = u.z;
#endif
}

// Software-pipelined form for the shared-memory accumulate loop: the next entry's
// U2' = x2' ZZ3 needs only ZZ3, so it joins the last product group of this step,
// and S2 = y2 ZZZ joins P^2:  {S2, PP} | {R^2, PPP, Q, ZZ3} | {R (Q - X3), Y1 PPP,
// ZZZ3, U2'}: three dependent groups of 2, 4, 4 products per step instead of four
// of 2, 2, 3, 3, the same 8M + 2S (U2' is this step's share of the next one).
// have_u2: U2 holds x2 ZZ for the current accumulator (false after the general
// path or at the start of a chunk: then it is computed here).  xn: the next
// entry's x (any residue when there is none: the extra product is discarded).
__device__ __forceinline__ void xyzz_add_aff_pipe(xyzz &A, const fe &x2, const fe &y2, fe &U2, bool &have_u2,
                                                  const fe &xn) {
#ifdef __CUDA_ARCH__
    if (A.inf | aff_is_inf(x2)) {
        A = xyzz_add_slow(A, x2, y2);
        have_u2 = false;
        return;
    }
    if (!have_u2) U2 = fe_mul_call(x2, A.ZZ);
    fe P, R;
    fe_sub(P, U2, A.X);
    if (fe_is_zero(P)) {
        A = xyzz_add_slow(A, x2, y2);
        have_u2 = false;
        return;
    }
#if PCMM_ACC_LZ3
    // PP, ZZ3 and ZZZ3 feed only products: they skip the final conditional subtraction (values in
    // [0, 2^256)); every product with one canonical operand is canonical again (fp_fast.cuh).
    fe2 sp;
    fe_mul_fast(sp.x, y2, A.ZZZ);                            // S2 = y2 ZZZ
    fe_sqr_lz(sp.y, P);                                      // PP = P^2 (lazy)
    fe_sub(R, sp.x, A.Y);
    fe4 t;
    fe_sqr_fast(t.x, R);                                     // R^2
    fe_mul_fast(t.y, P, sp.y);                               // PPP
    fe_mul_fast(t.z, A.X, sp.y);                             // Q = X1 PP
    fe_mul_lz(t.w, A.ZZ, sp.y);                              // ZZ3 (lazy)
    fe X3, Q2, D;
    fe_add(Q2, t.z, t.z);
    fe_sub(X3, t.x, t.y);
    fe_sub(X3, X3, Q2);                                     // X3 = R^2 - PPP - 2Q
    fe_sub(D, t.z, X3);
    fe4 u;
    fe_mul_fast(u.x, R, D);                                  // R (Q - X3)
    fe_mul_fast(u.y, A.Y, t.y);                              // Y1 PPP
    fe_mul_lz(u.z, A.ZZZ, t.y);                              // ZZZ3 (lazy)
    fe_mul_fast(u.w, xn, t.w);                               // U2'
#elif PCMM_ACC_PERM
    // the same ten products in a source order chosen by macros (schedule search, tools/perm_search.sh):
    // PCMM_G1 / PCMM_G2 / PCMM_G3 = the order of each group's products as decimal digits,
    // PCMM_SWAPM = bit mask swapping the operands of the eight general products
    fe2 sp;
#pragma unroll
    for (int st = 0; st < 2; st++) {
        const int d = st == 0 ? (PCMM_G1 / 10) % 10 : PCMM_G1 % 10;
        if (d == 1) { if (PCMM_SWAPM & 1) fe_mul_fast(sp.x, A.ZZZ, y2); else fe_mul_fast(sp.x, y2, A.ZZZ); }
        if (d == 2) fe_sqr_fast(sp.y, P);
    }
    fe_sub(R, sp.x, A.Y);
    fe4 t;
#pragma unroll
    for (int st = 0; st < 4; st++) {
        const int d = st == 0 ? (PCMM_G2 / 1000) % 10 : st == 1 ? (PCMM_G2 / 100) % 10 : st == 2 ? (PCMM_G2 / 10) % 10 : PCMM_G2 % 10;
        if (d == 1) fe_sqr_fast(t.x, R);
        if (d == 2) { if (PCMM_SWAPM & 2) fe_mul_fast(t.y, sp.y, P); else fe_mul_fast(t.y, P, sp.y); }
        if (d == 3) { if (PCMM_SWAPM & 4) fe_mul_fast(t.z, sp.y, A.X); else fe_mul_fast(t.z, A.X, sp.y); }
        if (d == 4) { if (PCMM_SWAPM & 8) fe_mul_fast(t.w, sp.y, A.ZZ); else fe_mul_fast(t.w, A.ZZ, sp.y); }
    }
    fe X3, Q2, D;
    fe_add(Q2, t.z, t.z);
    fe_sub(X3, t.x, t.y);
    fe_sub(X3, X3, Q2);                                     // X3 = R^2 - PPP - 2Q
    fe_sub(D, t.z, X3);
    fe4 u;
#pragma unroll
    for (int st = 0; st < 4; st++) {
        const int d = st == 0 ? (PCMM_G3 / 1000) % 10 : st == 1 ? (PCMM_G3 / 100) % 10 : st == 2 ? (PCMM_G3 / 10) % 10 : PCMM_G3 % 10;
        if (d == 1) { if (PCMM_SWAPM & 16) fe_mul_fast(u.x, D, R); else fe_mul_fast(u.x, R, D); }
        if (d == 2) { if (PCMM_SWAPM & 32) fe_mul_fast(u.y, t.y, A.Y); else fe_mul_fast(u.y, A.Y, t.y); }
        if (d == 3) { if (PCMM_SWAPM & 64) fe_mul_fast(u.z, t.y, A.ZZZ); else fe_mul_fast(u.z, A.ZZZ, t.y); }
        if (d == 4) { if (PCMM_SWAPM & 128) fe_mul_fast(u.w, t.w, xn); else fe_mul_fast(u.w, xn, t.w); }
    }
#else
    const fe2 sp = fe_mulsqr_hot(y2, A.ZZZ, P);              // S2 = y2 ZZZ, PP = P^2
    fe_sub(R, sp.x, A.Y);
    const fe4 t = fe_sqr_mul3_hot(R, P, sp.y, A.X, sp.y, A.ZZ, sp.y);   // R^2, PPP, Q = X1 PP, ZZ3
    fe X3, Q2, D;
    fe_add(Q2, t.z, t.z);
    fe_sub(X3, t.x, t.y);
    fe_sub(X3, X3, Q2);                                     // X3 = R^2 - PPP - 2Q
    fe_sub(D, t.z, X3);
    const fe4 u = fe_mul4_hot(R, D, A.Y, t.y, A.ZZZ, t.y, xn, t.w);   // R (Q - X3), Y1 PPP, ZZZ3, U2'
#endif
    fe_sub(A.Y, u.x, u.y);
    A.X = X3;
    A.ZZ = t.w;
    A.ZZZ = u.z;
    U2 = u.w;
    have_u2 = true;
#endif
}

// The same step on almost-reduced values (fp_fast.cuh fe_*_lz: the accumulator,
// U2 and every intermediate anywhere in [0, 2^256), products without the final
// conditional subtraction).  Table entries are canonical; the exceptional path
// and xyzz_to_proj use non-lazy products, whose outputs are canonical again.
// P = 0 is tested as P in {0, p}.
__device__ __forceinline__ void xyzz_add_aff_pipe_lz(xyzz &A, const fe &x2, const fe &y2, fe &U2, bool &have_u2,
                                                     const fe &xn) {
#ifdef __CUDA_ARCH__
    if (A.inf | aff_is_inf(x2)) {
        A = xyzz_add_slow(A, x2, y2);
        have_u2 = false;
        return;
    }
    if (!have_u2) U2 = fe_mul_call(x2, A.ZZ);
    fe P, R;
    fe_sub_lz(P, U2, A.X);
    if (fe_is_zero_lz(P)) {
        A = xyzz_add_slow(A, x2, y2);
        have_u2 = false;
        return;
    }
    const fe2 sp = fe_mulsqr_lz_hot(y2, A.ZZZ, P);           // S2 = y2 ZZZ, PP = P^2
    fe_sub_lz(R, sp.x, A.Y);
    const fe4 t = fe_sqr_mul3_lz_hot(R, P, sp.y, A.X, sp.y, A.ZZ, sp.y);   // R^2, PPP, Q = X1 PP, ZZ3
    fe X3, Q2, D;
    fe_add_lz(Q2, t.z, t.z);
    fe_sub_lz(X3, t.x, t.y);
    fe_sub_lz(X3, X3, Q2);                                   // X3 = R^2 - PPP - 2Q
    fe_sub_lz(D, t.z, X3);
    const fe4 u = fe_mul4_lz_hot(R, D, A.Y, t.y, A.ZZZ, t.y, xn, t.w);   // R (Q - X3), Y1 PPP, ZZZ3, U2'
    fe_sub_lz(A.Y, u.x, u.y);
    A.X = X3;
    A.ZZ = t.w;
    A.ZZZ = u.z;
    U2 = u.w;
    have_u2 = true;
#endif
}

// The accumulate kernels' accumulator (hot.cu): PCMM_ACC_XYZZ=1 (default) XYZZ
// (8M + 2S per step), 0 the Jacobian step above (9M + 2S).
#ifndef PCMM_ACC_XYZZ
#define PCMM_ACC_XYZZ 1
#endif
#if PCMM_ACC_XYZZ
typedef xyzz acc_t;
__device__ __forceinline__ void acc_init(acc_t &A) { xyzz_init(A); }
__device__ __forceinline__ void acc_add_aff(acc_t &A, const fe &x, const fe &y) { xyzz_add_aff(A, x, y); }
__device__ __forceinline__ void acc_to_proj(pt &o, const acc_t &A) { xyzz_to_proj(o, A); }
__device__ __forceinline__ void acc_from_proj(acc_t &A, const pt &o) { xyzz_from_proj(A, o); }
#else
typedef jacc acc_t;
__device__ __forceinline__ void acc_init(acc_t &A) { jac_init(A); }
__device__ __forceinline__ void acc_add_aff(acc_t &A, const fe &x, const fe &y) { jac_add_aff(A, x, y); }
__device__ __forceinline__ void acc_to_proj(pt &o, const acc_t &A) { jac_to_proj(o, A); }
__device__ __forceinline__ void acc_from_proj(acc_t &A, const pt &o) {
#ifdef __CUDA_ARCH__
    A.Z = o.Z;
    A.ZZ = fe_mul_call(o.Z, o.Z);
    mul2(A.X, o.X, o.Z, A.Y, o.Y, A.ZZ);
    A.inf = 0;
#endif
}
#endif

// R = k P for a 256-bit k (little-endian words) and an affine P (x, y) (pinf:
// the identity): 4-bit fixed windows over precomputed affine multiples 1..15 P
// (14 mixed additions, one simultaneous inversion), 252 Jacobian doublings and
// <= 64 mixed additions (complete fallback inside jac_add_aff): ~2,400 products
// against ~5,100 for binary double-and-add with the complete formulas.
static __device__ __noinline__ jacc jac_mul_scalar_aff(const uint32_t k[8], const fe x, const fe y, int pinf) {
    jacc A;
    jac_init(A);
#ifdef __CUDA_ARCH__
    if (pinf) return A;
    fe tx[16], ty[16];                            // slot v = v P (affine); slot 0 unused
    tx[1] = x;
    ty[1] = y;
    jacc T[16];
    jac_init(T[1]);
    jac_add_aff(T[1], x, y);                      // T[1] = P (Z = 1)
    for (int v = 2; v < 16; v++) {
        T[v] = T[v - 1];
        jac_add_aff(T[v], x, y);
    }
    // batch inversion of Z for v = 2..15 (identity multiples cannot occur: q is prime > 15)
    fe pre[16], acc;
    fe_one_mont(acc);
    for (int v = 2; v < 16; v++) {
        pre[v] = acc;
        fe_mul(acc, acc, T[v].Z);
    }
    fe inv;
    fe_inv(inv, acc);
    for (int v = 15; v >= 2; v--) {
        fe zi, z2;
        fe_mul(zi, inv, pre[v]);
        fe_mul(inv, inv, T[v].Z);
        fe_sqr(z2, zi);
        fe_mul(tx[v], T[v].X, z2);
        fe_mul(z2, z2, zi);
        fe_mul(ty[v], T[v].Y, z2);
    }
    for (int wdx = 63; wdx >= 0; wdx--) {
        if (wdx != 63) {
            jac_dbl(A);
            jac_dbl(A);
            jac_dbl(A);
            jac_dbl(A);
        }
        const int v = (k[wdx >> 3] >> (4 * (wdx & 7))) & 15;
        if (v) jac_add_aff(A, tx[v], ty[v]);
    }
#endif
    return A;
}

// R = k P for P with Z = 1 (an imported / decoded point) or the identity
__device__ __forceinline__ void pt_mul_scalar_win(pt &R, const uint32_t k[8], const pt &P) {
    const jacc J = jac_mul_scalar_aff(k, P.X, P.Y, pt_is_identity(P) ? 1 : 0);
    jac_to_proj(R, J);
}

}  // namespace pcmm
