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

// A += (x2, y2).  U1 = X1, S1 = Y1 (Z2 = 1): U2 = x2 Z1^2, S2 = y2 Z1^3,
// H = U2 - X1, R = S2 - Y1, X3 = R^2 - H^3 - 2 X1 H^2,
// Y3 = R (X1 H^2 - X3) - Y1 H^3, Z3 = Z1 H, ZZ3 = Z1^2 H^2.
__device__ __forceinline__ void jac_add_aff(jacc &A, const fe &x2, const fe &y2) {
#ifdef __CUDA_ARCH__
    if (A.inf | aff_is_inf(x2)) {
        A = jac_add_slow(A, x2, y2);
        return;
    }
    fe U2, T1;
    mul2(U2, x2, A.ZZ, T1, A.Z, A.ZZ);            // U2 = x2 ZZ, T1 = Z^3
    fe H;
    fe_sub(H, U2, A.X);
    if (fe_is_zero(H)) {
        A = jac_add_slow(A, x2, y2);
        return;
    }
    const fe2 sh = fe_mulsqr_call(y2, T1, H);     // S2 = y2 Z^3, HH = H^2
    const fe &S2 = sh.x, &HH = sh.y;
    fe R;
    fe_sub(R, S2, A.Y);
    const fe3 t = fe_mul3_call(H, HH, A.X, HH, A.ZZ, HH);  // H^3, V = X1 H^2, ZZ3
    const fe2 zr = fe_mulsqr_call(A.Z, H, R);     // Z3 = Z1 H, R^2
    const fe &Z3 = zr.x, &R2 = zr.y;
    fe X3, V2, D;
    fe_add(V2, t.y, t.y);
    fe_sub(X3, R2, t.x);
    fe_sub(X3, X3, V2);                           // X3 = R^2 - H^3 - 2V
    fe_sub(D, t.y, X3);
    fe Y3a, YH;
    mul2(Y3a, R, D, YH, A.Y, t.x);                // R (V - X3), Y1 H^3
    fe_sub(A.Y, Y3a, YH);
    A.X = X3;
    A.Z = Z3;
    A.ZZ = t.z;
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

}  // namespace pcmm
