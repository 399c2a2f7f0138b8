// shared.cuh -- device helpers shared by kernels.cu (table kernels) and affine.cu (k_affine).
#pragma once
#include "ec.cuh"
#include "internal.h"

namespace pcmm {

// Column k's tables are built by k_tables_fast (below) when its level-1 set is
// {1, ..., n1}; k_tables / k_affine then skip it.  (k_affine: plans == nullptr, no skipping)
__device__ __forceinline__ bool col_consecutive(const ColPlan &pl, int N) {
    (void)N;
    return pl.coz > 0;          // set by k_plan (N >= 2; unsigned {1..n1} or signed magnitudes {1..M})
}

#ifndef PCMM_TFAST_PROJ
#define PCMM_TFAST_PROJ 0       // 1: k_tables_fast stores homogeneous (X ZZZ : Y ZZ : ZZ ZZZ) entries instead
#endif


__device__ __forceinline__ fe fe_shfl_up(const fe &a, int d) {
    fe r;
#pragma unroll
    for (int i = 0; i < 8; i++) r.v[i] = __shfl_up_sync(0xffffffffu, a.v[i], d);
    return r;
}

__device__ __forceinline__ fe fe_shfl_down(const fe &a, int d) {
    fe r;
#pragma unroll
    for (int i = 0; i < 8; i++) r.v[i] = __shfl_down_sync(0xffffffffu, a.v[i], d);
    return r;
}

__device__ __forceinline__ void st_aff_inf(uint32_t *d) {
    uint4 *q = reinterpret_cast<uint4 *>(d);
    const uint4 ones = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
    q[0] = ones;
    q[1] = ones;
    q[2] = make_uint4(0, 0, 0, 0);
    q[3] = make_uint4(0, 0, 0, 0);
}

// One inversion per CTA (128 lanes x `batch` entries): lane products -> warp
// prefix/suffix products (shuffles) -> the four warp totals -> lane 0 of warp 0
// inverts their product and hands each warp the inverse of its total; each lane
// then recovers 1 / (its product) = inv(warp total) x (prefix before it) x
// (suffix after it).  The other warps wait at the barrier while other CTAs run.
// kFermat: the CTA's one inversion by Fermat's chain (fewer registers: 3+ CTAs per
// SM keep the two passes busy on large tables) or by divsteps (4x shorter latency:
// small tables, where that one inversion is the kernel's critical path)
template <bool kFermat>
__device__ __forceinline__ fe cta_inverse(const fe &acc, fe *wtot, fe *winv) {
    const int lane = (int)(threadIdx.x & 31), warp = (int)(threadIdx.x >> 5);
    PCMM_DCHECK(blockDim.x == 128);                    // wtot[4], winv[4]
    fe one;
    fe_one_mont(one);
    // warp-inclusive prefix (Q) and suffix (S) products of the lane products
    fe Q = acc, S = acc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const fe q = fe_shfl_up(Q, d), sv = fe_shfl_down(S, d);
        fe qm, sm;
        fe_mul(qm, Q, q);
        fe_mul(sm, S, sv);
        if (lane >= d) Q = qm;
        if (lane + d < 32) S = sm;
    }
    if (lane == 31) wtot[warp] = Q;
    __syncthreads();
    if (threadIdx.x == 0) {
        fe p1 = wtot[0], p2, p3, tot, s2, s1, inv, x;
        fe_mul(p2, p1, wtot[1]);
        fe_mul(p3, p2, wtot[2]);
        fe_mul(tot, p3, wtot[3]);
        fe_mul(s2, wtot[2], wtot[3]);
        fe_mul(s1, wtot[1], s2);
        if (kFermat) fe_inv_fermat(inv, tot);
        else fe_inv(inv, tot);
        fe_mul(winv[0], inv, s1);                  // 1 / W0
        fe_mul(x, inv, p1);
        fe_mul(winv[1], x, s2);                    // 1 / W1
        fe_mul(x, inv, p2);
        fe_mul(winv[2], x, wtot[3]);               // 1 / W2
        fe_mul(winv[3], inv, p3);                  // 1 / W3
    }
    __syncthreads();
    fe qprev = fe_shfl_up(Q, 1), snext = fe_shfl_down(S, 1);
    if (lane == 0) qprev = one;
    if (lane == 31) snext = one;
    fe inv;
    fe_mul(inv, winv[warp], qprev);
    fe_mul(inv, inv, snext);                       // 1 / acc (this lane's product)
    return inv;
}

}  // namespace pcmm
