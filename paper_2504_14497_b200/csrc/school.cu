// school.cu -- row s1 of SURVEY.md §8(a): schoolbook PC-MM, the comparison path
// (§3.1): Enc(c_ij) = sum_k a_ik Enc(b_kj), each term an
// independent small-scalar multiplication of the ciphertext followed by one
// accumulator addition (P:232-233's cost model: n^3 ECSMs and n^2 (n - 1)
// additions per component).
//
// Same coordinate machinery as the Cussen accumulate (jac.cuh), so that the
// comparison is like for like: the ciphertext component P is affine (k_import),
// the term V = |a| P is built in XYZZ by left-to-right binary (an affine-input
// doubling 4M + 3S, then XYZZ doublings 7M + 2S and mixed additions of P
// 8M + 2S; a = 2^t - 1, t >= 3, as 2^t P - P), and added to the XYZZ accumulator
// with add-2008-s (12M + 2S), or with the mixed addition when |a| = 1.
// a < 0 negates P first (R10).  Average over a uniform w = 4 entry
// (zeros included): 36.2 fp_mul-equivalents per term, against 49 for the
// complete homogeneous formulas of k_school (kernels.cu).  Measured at 256^3:
// 40.7 ms against k_school's 27.4 ms -- fewer products, but the call structure
// this code size needs (below) costs more than it saves -- so k_school stays the
// comparison path and this kernel is selected by PCMM_SCHOOL_XYZZ=1 (kept
// parity-tested).
//
// Lanes <-> output columns j (coalesced loads of Enc(b_kj)), warp <-> row i, so
// a_ik is warp-uniform and the double-and-add control flow never diverges.
#include "canon.cuh"
#include "ec.cuh"
#include "internal.h"
#include "jac.cuh"

namespace pcmm {

namespace {

// A += B, both XYZZ, B not the identity, complete: the identity accumulator and
// P = U2 - U1 = 0 (A = +-B) take the complete RCB16 addition on homogeneous images.
__device__ __noinline__ xyzz xyzz_add_slow2(xyzz A, const xyzz B) {
#ifdef __CUDA_ARCH__
    if (A.inf) return B;
    pt P, Q, R;
    xyzz_to_proj(P, A);
    xyzz_to_proj(Q, B);
    pt_add_pair(R, P, Q);
    if (fe_is_zero(R.Z)) {
        A.inf = 1;
        return A;
    }
    xyzz_from_proj(A, R);
#endif
    return A;
}

// add-2008-s: U1 = X1 ZZ2, U2 = X2 ZZ1, S1 = Y1 ZZZ2, S2 = Y2 ZZZ1, P = U2 - U1,
// R = S2 - S1, PP = P^2, PPP = P PP, Q = U1 PP, X3 = R^2 - PPP - 2Q,
// Y3 = R (Q - X3) - S1 PPP, ZZ3 = ZZ1 ZZ2 PP, ZZZ3 = ZZZ1 ZZZ2 PPP: 12M + 2S in
// four groups of 4, 2, 4, 4 independent products.
__device__ __forceinline__ void xyzz_add_xyzz(xyzz &A, const xyzz &B) {
#ifdef __CUDA_ARCH__
    if (A.inf) {
        A = xyzz_add_slow2(A, B);
        return;
    }
    const fe4 g = fe_mul4_hot(A.X, B.ZZ, B.X, A.ZZ, A.Y, B.ZZZ, B.Y, A.ZZZ);   // U1, U2, S1, S2
    fe P, R;
    fe_sub(P, g.y, g.x);
    if (fe_is_zero(P)) {
        A = xyzz_add_slow2(A, B);
        return;
    }
    fe_sub(R, g.w, g.z);
    const fe2 sq = fe_sqr2_hot(P, R);                                         // PP, R^2
    const fe4 h = fe_mul4_hot(P, sq.x, g.x, sq.x, A.ZZ, B.ZZ, A.ZZZ, B.ZZZ);  // PPP, Q, ZZ1 ZZ2, ZZZ1 ZZZ2
    fe X3, Q2, D;
    fe_add(Q2, h.y, h.y);
    fe_sub(X3, sq.y, h.x);
    fe_sub(X3, X3, Q2);                                                       // X3 = R^2 - PPP - 2Q
    fe_sub(D, h.y, X3);
    const fe4 u = fe_mul4_hot(R, D, g.z, h.x, h.z, sq.x, h.w, h.x);           // R (Q - X3), S1 PPP, ZZ3, ZZZ3
    fe_sub(A.Y, u.x, u.y);
    A.X = X3;
    A.ZZ = u.z;
    A.ZZZ = u.w;
#endif
}

// Out-of-line point operations: the schoolbook's term loop calls each of them
// from several places, and inlined copies of their product groups overflow the
// instruction cache (measured: 315 KB of SASS, 256^3 69 ms vs 27 ms for the
// homogeneous kernel).  With the product groups out of line as well
// (build.py compiles this unit with PCMM_INLINE_ACCUM=0) the loop is small.
// (By-value signatures, arguments and results in registers: 44.8 ms; inlined
// point operations with out-of-line products: 53 ms; everything inlined: 68 ms.)
__device__ __noinline__ void sc_dbl_aff(xyzz &V, const fe x, const fe y) { xyzz_dbl_aff(V, x, y); }
__device__ __noinline__ void sc_dbl(xyzz &V) { xyzz_dbl(V); }
__device__ __noinline__ void sc_madd(xyzz &V, const fe x, const fe y) { xyzz_add_aff(V, x, y); }
__device__ __noinline__ void sc_add(xyzz &A, const xyzz B) { xyzz_add_xyzz(A, B); }

// V = av P for an affine P and av >= 2 (left-to-right binary; 2^t - 1 as 2^t P - P)
__device__ __forceinline__ void xyzz_mul_small(xyzz &V, int av, const fe &x, const fe &y) {
    const int top = 31 - __clz(av);                                           // av >= 2: top >= 1
    sc_dbl_aff(V, x, y);                                                    // 2P
    if (top >= 2 && av == (1 << (top + 1)) - 1) {
        for (int i = 1; i <= top; i++) sc_dbl(V);                           // 2^(top+1) P
        fe ny;
        fe_neg(ny, y);
        sc_madd(V, x, ny);                                               // - P
        return;
    }
    if ((av >> (top - 1)) & 1) sc_madd(V, x, y);
    for (int i = top - 2; i >= 0; i--) {
        sc_dbl(V);
        if ((av >> i) & 1) sc_madd(V, x, y);
    }
}

}  // namespace

#ifndef PCMM_SCHOOL_MINB
#define PCMM_SCHOOL_MINB 3
#endif
__global__ void __launch_bounds__(128, PCMM_SCHOOL_MINB) k_school_xyzz(const int8_t *__restrict__ A, int m, int n, int l, int w,
                                                     int is_signed, const uint32_t *__restrict__ bsoa,
                                                     uint32_t *__restrict__ out, int *__restrict__ status) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // block b = (c, row block, column block), column block fastest
    const int jblocks = (l + 31) / 32, rblocks = (m + 3) / 4;
    int64_t b = blockIdx.x;
    const int jb = (int)(b % jblocks);
    b /= jblocks;
    const int rb = (int)(b % rblocks);
    const int c = (int)(b / rblocks);
    const int i = rb * 4 + warp;
    if (i >= m) return;
    const int j = jb * 32 + lane;
    const int jj = min(j, l - 1);
    const int lo = is_signed ? -(1 << (w - 1)) : 0;
    const int hi = is_signed ? (1 << (w - 1)) - 1 : (1 << w) - 1;
    const int64_t cnt = (int64_t)n * l;
    const uint32_t *bc = bsoa + (int64_t)c * kPtWords * cnt;
    xyzz acc;
    xyzz_init(acc);
    bool bad = false;
    for (int k = 0; k < n; k++) {
        int v = is_signed ? (int)A[(int64_t)i * n + k] : (int)(uint8_t)A[(int64_t)i * n + k];
        if (v < lo || v > hi) {
            bad = true;
            v = 0;
        }
        if (v == 0) continue;                                                 // 0 * ct = (inf, inf), warp-uniform
        pt P;
        soa_load(P, bc, cnt, (int64_t)k * l + jj);
        if (pt_is_identity(P)) continue;                                      // (per lane) v * inf = inf
        if (v < 0) fe_neg(P.Y, P.Y);
        const int av = v < 0 ? -v : v;
        if (av == 1) {
            sc_madd(acc, P.X, P.Y);                                           // the term is P itself
        } else {
            xyzz V;
            xyzz_mul_small(V, av, P.X, P.Y);                                  // one ECSM per term
            sc_add(acc, V);
        }
    }
    if (bad && lane == 0) atomicOr(status, kStatusBound);
    if (j < l) {
        const int64_t oc = (int64_t)m * l;
        pt o;
        xyzz_to_proj(o, acc);
        soa_store(out + (int64_t)c * kPtWords * oc, oc, (int64_t)i * l + j, o);
    }
}

cudaError_t launch_schoolbook_xyzz(const int8_t *A, int m, int n, int l, int w, int is_signed, const uint32_t *bsoa,
                                   uint32_t *out, int *status, cudaStream_t s) {
    const int64_t blocks = (int64_t)((l + 31) / 32) * ((m + 3) / 4) * 2;
    k_school_xyzz<<<(unsigned)blocks, 128, 0, s>>>(A, m, n, l, w, is_signed, bsoa, out, status);
    return cudaGetLastError();
}

}  // namespace pcmm
