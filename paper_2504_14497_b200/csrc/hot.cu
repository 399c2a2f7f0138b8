// hot.cu -- the dominant kernel of the Cussen path (step a4 of SURVEY.md §8(a))
// and the fp_mul throughput probe, in their own translation unit (parallel
// compilation; the hot loop inlines the complete addition and fe_mul).
#include <stdlib.h>

#include "ec.cuh"
#include "internal.h"

namespace pcmm {

__device__ __forceinline__ void soa_store_hot(uint32_t *base, int64_t stride, int64_t idx, const pt &P) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
        base[(0 * 8 + i) * stride + idx] = P.X.v[i];
        base[(1 * 8 + i) * stride + idx] = P.Y.v[i];
        base[(2 * 8 + i) * stride + idx] = P.Z.v[i];
    }
}

// ------------------------------------------------------------ a4: accumulate
// CTA = (output column j, component c, row block, k-split).  Thread = row i.
// Per k-chunk the CTA stages KCH tables (1536 B each, [coord][limb][slot]) in
// shared memory; a warp reads, for one k, at most 15 distinct words per
// (coord, limb) within 16 consecutive banks: conflict-free gathers.
template <int ROWS, int KCH, int MINB>
__global__ void __launch_bounds__(ROWS, MINB) k_accum(const uint32_t *__restrict__ tables, const uint8_t *__restrict__ rank,
                                                int m, int n, int l, int ksplit, uint32_t *__restrict__ out,
                                                int64_t split_stride) {
    extern __shared__ uint4 smem4[];
    const uint32_t *smem = reinterpret_cast<const uint32_t *>(smem4);
    int b = blockIdx.x;
    const int j = b % l; b /= l;
    const int c = b & 1; b >>= 1;
    const int rowblocks = (m + ROWS - 1) / ROWS;
    const int rb = b % rowblocks;
    const int s = b / rowblocks;
    const int i = rb * ROWS + (int)threadIdx.x;
    const int kb = (int)((int64_t)s * n / ksplit), ke = (int)((int64_t)(s + 1) * n / ksplit);
    pt acc;
    pt_identity(acc);
    for (int k0 = kb; k0 < ke; k0 += KCH) {
        const int kc = min(KCH, ke - k0);
        __syncthreads();
        for (int t = threadIdx.x; t < kc * (kTableWords / 4); t += ROWS) {
            const int kk = t / (kTableWords / 4), wd = t % (kTableWords / 4);
            const uint4 *src = reinterpret_cast<const uint4 *>(
                tables + (((int64_t)c * n + (k0 + kk)) * l + j) * kTableWords);
            smem4[kk * (kTableWords / 4) + wd] = src[wd];
        }
        __syncthreads();
        if (i < m) {
            for (int kk = 0; kk < kc; kk++) {
                const int u = rank[(int64_t)(k0 + kk) * m + i];
                const uint32_t *T = smem + kk * kTableWords + u;
                pt Q;
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    Q.X.v[q] = T[(0 * 8 + q) * kSlots];
                    Q.Y.v[q] = T[(1 * 8 + q) * kSlots];
                    Q.Z.v[q] = T[(2 * 8 + q) * kSlots];
                }
                pt_add_pair(acc, acc, Q);
            }
        }
    }
    if (i < m) {
        const int64_t cnt = (int64_t)m * l;
        soa_store_hot(out + (int64_t)s * split_stride + (int64_t)c * kPtWords * cnt, cnt, (int64_t)i * l + j, acc);
    }
}

template <int VARIANT>
__global__ void __launch_bounds__(128) k_bench_fp_mul(int iters, uint32_t *__restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    fe x[4], y;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        y.v[i] = (uint32_t)(t * 2654435761u + i * 40503u) & 0x7fffffffu;
#pragma unroll
        for (int c = 0; c < 4; c++) x[c].v[i] = (uint32_t)(t * 97u + i * 131u + c * 7u) & 0x7fffffffu;
    }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int c = 0; c < 4; c++) {
            if (VARIANT == 1) fe_mul_portable(x[c], x[c], y);
            else if (VARIANT == 2) fe_add(x[c], x[c], y);
            else fe_mul(x[c], x[c], y);
        }
    }
#pragma unroll
    for (int i = 0; i < 8; i++) out[t * 8 + i] = x[0].v[i] ^ x[1].v[i] ^ x[2].v[i] ^ x[3].v[i];
}

constexpr int kChunk = 32;
constexpr int kRows = 128;

static int accum_minb() {
    static int minb = -1;
    if (minb < 0) {
        const char *e = getenv("PCMM_ACCUM_MINB");
        minb = e ? atoi(e) : 3;
    }
    return minb;
}

// resident k_accum CTAs per SM (for wave-balanced split-k choice)
int accum_ctas_per_sm() {
    static int occ = 0;
    if (!occ) {
        const size_t smem = (size_t)kChunk * kTableWords * 4;
        cudaError_t e;
        if (accum_minb() == 4) {
            cudaFuncSetAttribute(k_accum<kRows, kChunk, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_accum<kRows, kChunk, 4>, kRows, smem);
        } else {
            cudaFuncSetAttribute(k_accum<kRows, kChunk, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_accum<kRows, kChunk, 3>, kRows, smem);
        }
        if (e != cudaSuccess || occ <= 0) occ = 3;
    }
    return occ;
}

int accum_rows() { return kRows; }

cudaError_t launch_accum(const uint32_t *tables, const uint8_t *rank, int m, int n, int l, int rows, int ksplit,
                         uint32_t *out, int64_t out_stride_split, cudaStream_t s) {
    (void)rows;
    const int rowblocks = (m + kRows - 1) / kRows;
    const unsigned grid = (unsigned)((int64_t)l * 2 * rowblocks * ksplit);
    const size_t smem = (size_t)kChunk * kTableWords * 4;
    cudaError_t err;
    if (accum_minb() == 4) {
        err = cudaFuncSetAttribute(k_accum<kRows, kChunk, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (err) return err;
        k_accum<kRows, kChunk, 4><<<grid, kRows, smem, s>>>(tables, rank, m, n, l, ksplit, out, out_stride_split);
    } else {
        err = cudaFuncSetAttribute(k_accum<kRows, kChunk, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (err) return err;
        k_accum<kRows, kChunk, 3><<<grid, kRows, smem, s>>>(tables, rank, m, n, l, ksplit, out, out_stride_split);
    }
    return cudaGetLastError();
}

cudaError_t launch_bench_fp_mul(int variant, int blocks, int threads, int iters, uint32_t *out, cudaStream_t s) {
    if (variant == 1) k_bench_fp_mul<1><<<blocks, threads, 0, s>>>(iters, out);
    else if (variant == 2) k_bench_fp_mul<2><<<blocks, threads, 0, s>>>(iters, out);
    else k_bench_fp_mul<0><<<blocks, threads, 0, s>>>(iters, out);
    return cudaGetLastError();
}

}  // namespace pcmm
