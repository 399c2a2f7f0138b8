// shared.cuh -- device helpers shared by kernels.cu (table kernels) and affine.cu (k_affine).
#pragma once
#include "ec.cuh"
#include "internal.h"

namespace pcmm {

// Column k's tables are built by k_tables_fast (below) when its level-1 set is
// {1, ..., n1}; k_tables / k_affine then skip it.  (k_affine: plans == nullptr, no skipping)
__device__ __forceinline__ bool col_consecutive(const ColPlan &pl, int N) {
    return N >= 2 && pl.n[0] >= 1 && pl.n[1] == 1 && pl.sN[0] == 1;
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

}  // namespace pcmm
