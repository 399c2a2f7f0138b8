// strassen.cu -- Strassen PC-MM, the paper's second comparison path (NEXT-3,
// arXiv 2504.14497 Sec. 3.1).
//
// Breadth-first schedule: level d holds all 7^d subproblems and each step of a
// level is one batched launch (k_down_a, k_down_b, k_school_batched, k_up_c).
// One recursion level splits A (plaintext), Enc(B) and Enc(C) into 2 x 2 blocks
// and forms
//   M1 = (A11 + A22)(B11 + B22)   M2 = (A21 + A22) B11     M3 = A11 (B12 - B22)
//   M4 = A22 (B21 - B11)          M5 = (A11 + A12) B22     M6 = (A21 - A11)(B11 + B12)
//   M7 = (A12 - A22)(B21 + B22)
//   C11 = M1 + M4 - M5 + M7   C12 = M3 + M5   C21 = M2 + M4   C22 = M1 - M2 + M3 + M6
// i.e. 7 block PC-MMs, 5 plaintext block additions / subtractions and 13
// ciphertext block additions / subtractions.  The recursion stops
// at blocks of <= `leaf` rows / inner / columns (or an odd dimension) and runs the
// schoolbook kernel there.  Plaintext sums grow by one bit per level, so the
// recursion carries int32 plaintexts; ciphertext blocks are projective
// Montgomery SoA ([c][X,Y,Z][limb][r * cols + col]).
#include <vector>

#include "ec.cuh"
#include "internal.h"

namespace pcmm {

namespace {

__device__ __forceinline__ void soa_ld(pt &P, const uint32_t *base, int64_t stride, int64_t idx) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
        P.X.v[i] = base[(0 * 8 + i) * stride + idx];
        P.Y.v[i] = base[(1 * 8 + i) * stride + idx];
        P.Z.v[i] = base[(2 * 8 + i) * stride + idx];
    }
}

__device__ __forceinline__ void soa_st(uint32_t *base, int64_t stride, int64_t idx, const pt &P) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
        base[(0 * 8 + i) * stride + idx] = P.X.v[i];
        base[(1 * 8 + i) * stride + idx] = P.Y.v[i];
        base[(2 * 8 + i) * stride + idx] = P.Z.v[i];
    }
}

// widen A to int32 and check the w-bit range (EBOUND); A is int8 / uint8 (byte
// API) or int32 (wide API, w <= 16)
__device__ __forceinline__ int a_value(const int8_t *A, int64_t t, int is_signed) {
    return is_signed ? (int)A[t] : (int)(uint8_t)A[t];
}
__device__ __forceinline__ int a_value(const int32_t *A, int64_t t, int) { return A[t]; }

template <typename TA>
__global__ void k_a_widen(const TA *__restrict__ A, int64_t count, int w, int is_signed,
                          int32_t *__restrict__ out, int *__restrict__ status) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= count) return;
    const int v = a_value(A, t, is_signed);
    const int lo = is_signed ? -(1 << (w - 1)) : 0;
    const int hi = is_signed ? (1 << (w - 1)) - 1 : (1 << w) - 1;
    const bool ok = v >= lo && v <= hi;
    if (!ok) atomicOr(status, kStatusBound);
    out[t] = ok ? v : 0;
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// Coefficients of the 7 products on the 2 x 2 blocks (11, 12, 21, 22)
__constant__ int8_t kCoefA[7][4] = {{1, 0, 0, 1}, {0, 0, 1, 1}, {1, 0, 0, 0}, {0, 0, 0, 1},
                                    {1, 1, 0, 0}, {-1, 0, 1, 0}, {0, 1, 0, -1}};
__constant__ int8_t kCoefB[7][4] = {{1, 0, 0, 1}, {1, 0, 0, 0}, {0, 1, 0, -1}, {-1, 0, 1, 0},
                                    {0, 0, 0, 1}, {1, 1, 0, 0}, {0, 0, 1, 1}};
// C blocks from M1..M7
__constant__ int8_t kCoefC[4][7] = {{1, 0, 0, 1, -1, 0, 1}, {0, 0, 1, 0, 1, 0, 0},
                                    {0, 1, 0, 1, 0, 0, 0}, {1, -1, 1, 0, 0, 1, 0}};

// level d -> d+1 plaintext operands: child (p*7+q) = sum_b coefA[q][b] * block_b(parent p)
__global__ void k_down_a(const int32_t *__restrict__ A, int64_t P, int h, int w, int32_t *__restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per = (int64_t)h * w;
    if (t >= P * 7 * per) return;
    const int64_t child = t / per, e = t % per;
    const int64_t p = child / 7;
    const int q = (int)(child % 7);
    const int r = (int)(e / w), c = (int)(e % w);
    const int32_t *Ap = A + p * 4 * per;              // parent is (2h) x (2w), row-major
    int v = 0;
#pragma unroll
    for (int b = 0; b < 4; b++) {
        const int co = kCoefA[q][b];
        if (co) v += co * (int)Ap[(int64_t)((b >> 1) * h + r) * (2 * w) + (b & 1) * w + c];
    }
    out[t] = (int32_t)v;
}

// level d -> d+1 ciphertext operands (at most two blocks per combination: one point op)
__global__ void k_down_b(const uint32_t *__restrict__ B, int64_t P, int h, int w, uint32_t *__restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per = (int64_t)h * w, cnt_out = P * 7 * per, cnt_in = P * 4 * per;
    if (t >= 2 * cnt_out) return;
    const int comp = (int)(t / cnt_out);
    const int64_t i = t % cnt_out;
    const int64_t child = i / per, e = i % per;
    const int64_t p = child / 7;
    const int q = (int)(child % 7);
    const int r = (int)(e / w), c = (int)(e % w);
    const uint32_t *Bc = B + (int64_t)comp * kPtWords * cnt_in;
    pt acc;
    bool first = true;
#pragma unroll
    for (int b = 0; b < 4; b++) {
        const int co = kCoefB[q][b];
        if (!co) continue;
        pt X;
        soa_ld(X, Bc, cnt_in, p * 4 * per + (int64_t)((b >> 1) * h + r) * (2 * w) + (b & 1) * w + c);
        if (co < 0) pt_neg(X, X);
        if (first) {
            acc = X;
            first = false;
        } else {
            pt_add_pair(acc, acc, X);
        }
    }
    soa_st(out + (int64_t)comp * kPtWords * cnt_out, cnt_out, i, acc);
}

// level d+1 -> d: parent block b = sum_q coefC[b][q] * M_q (children p*7+q)
__global__ void k_up_c(const uint32_t *__restrict__ M, int64_t P, int h, int w, uint32_t *__restrict__ C) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per = (int64_t)h * w, cnt_out = P * 4 * per, cnt_in = P * 7 * per;
    if (t >= 2 * cnt_out) return;
    const int comp = (int)(t / cnt_out);
    const int64_t i = t % cnt_out;
    const int64_t p = i / (4 * per);
    const int64_t rem = i % (4 * per);
    const int R = (int)(rem / (2 * w)), Cc = (int)(rem % (2 * w));   // position in the (2h) x (2w) parent
    const int b = (R >= h ? 2 : 0) + (Cc >= w ? 1 : 0);
    const int64_t e = (int64_t)(R % h) * w + (Cc % w);
    const uint32_t *Mc = M + (int64_t)comp * kPtWords * cnt_in;
    pt acc;
    bool first = true;
#pragma unroll
    for (int q = 0; q < 7; q++) {
        const int co = kCoefC[b][q];
        if (!co) continue;
        pt X;
        soa_ld(X, Mc, cnt_in, (p * 7 + q) * per + e);
        if (co < 0) pt_neg(X, X);
        if (first) {
            acc = X;
            first = false;
        } else {
            pt_add_pair(acc, acc, X);
        }
    }
    soa_st(C + (int64_t)comp * kPtWords * cnt_out, cnt_out, i, acc);
}

// batched leaf schoolbook: problem z / 2, component z % 2; problem p's A block is
// A + p m n (int32), its B block starts at index p n l of the level's SoA
__global__ void __launch_bounds__(128) k_school_batched(const int32_t *__restrict__ A, int m, int n, int l,
                                                         int64_t P, const uint32_t *__restrict__ B,
                                                         uint32_t *__restrict__ out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // 1-D grid, problem-major (all CTAs of one subproblem adjacent: its B block stays in L2)
    const int jblocks = (l + 31) / 32, mblocks = (m + 3) / 4;
    const int64_t z = blockIdx.x / ((int64_t)jblocks * mblocks);   // problem * 2 + component
    const int rem = (int)(blockIdx.x % ((int64_t)jblocks * mblocks));
    const int64_t p = z >> 1;
    const int c = (int)(z & 1);
    const int i = (rem / jblocks) * 4 + warp;
    if (i >= m) return;
    const int j = (rem % jblocks) * 32 + lane;
    const int jj = min(j, l - 1);
    const int64_t cnt = P * n * l;
    const uint32_t *bc = B + (int64_t)c * kPtWords * cnt + p * n * l;
    const int32_t *Ap = A + p * m * n;
    pt acc, X, T;
    pt_identity(acc);
    for (int k = 0; k < n; k++) {
        const int v = Ap[(int64_t)i * n + k];
        if (v == 0) continue;                                       // warp-uniform
        soa_ld(X, bc, cnt, (int64_t)k * l + jj);
        pt_mul_small_pair(T, v, X);
        pt_add_pair(acc, acc, T);
    }
    if (j < l) {
        const int64_t oc = P * m * l;
        soa_st(out + (int64_t)c * kPtWords * oc + p * m * l, oc, (int64_t)i * l + j, acc);
    }
}

}  // namespace

cudaError_t run_strassen(const void *A, int a_is_i32, int m, int n, int l, int w, int is_signed,
                         const uint32_t *bsoa, int leaf, uint32_t *out, int *status, cudaStream_t s) {
    // breadth-first: level d holds all 7^d subproblems, so every step of a level is
    // ONE batched launch (a GPU-friendly schedule of the same Strassen recursion)
    if (leaf < 1) leaf = 1;
    int D = 0;
    while (D < 8 && ((m >> D) % 2 == 0) && ((n >> D) % 2 == 0) && ((l >> D) % 2 == 0) && (m >> (D + 1)) >= leaf &&
           (n >> (D + 1)) >= leaf && (l >> (D + 1)) >= leaf)
        D++;
    cudaError_t err = cudaSuccess;
    {
        // keep the stream-ordered pool's memory mapped between calls: the per-level blocks are
        // re-allocated every call, and returning them to the OS at each synchronisation made
        // some calls 50x slower (measured in tools/grid.py)
        static bool pool_tuned = false;
        int dev = 0;
        cudaMemPool_t pool;
        if (!pool_tuned && cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            pool_tuned = true;
        }
    }
    auto note = [&](cudaError_t e) {
        if (err == cudaSuccess && e != cudaSuccess) err = e;
    };
    std::vector<int32_t *> As(D + 1, nullptr);
    std::vector<uint32_t *> Bs(D + 1, nullptr), Cs(D + 1, nullptr);
    int64_t P = 1;
    note(cudaMallocAsync((void **)&As[0], (size_t)m * n * 4 + 4, s));
    if (err) return err;
    if (a_is_i32)
        k_a_widen<int32_t><<<nblk((int64_t)m * n, 256), 256, 0, s>>>((const int32_t *)A, (int64_t)m * n, w,
                                                                     is_signed, As[0], status);
    else
        k_a_widen<int8_t><<<nblk((int64_t)m * n, 256), 256, 0, s>>>((const int8_t *)A, (int64_t)m * n, w,
                                                                    is_signed, As[0], status);
    note(cudaGetLastError());
    Bs[0] = const_cast<uint32_t *>(bsoa);
    for (int d = 0; d < D && err == cudaSuccess; d++) {               // down: operands of the 7 products
        const int h = m >> (d + 1), kk = n >> (d + 1), ww = l >> (d + 1);
        note(cudaMallocAsync((void **)&As[d + 1], (size_t)P * 7 * h * kk * 4 + 4, s));
        note(cudaMallocAsync((void **)&Bs[d + 1], (size_t)P * 7 * kk * ww * 2 * kPtWords * 4, s));
        if (err) break;
        k_down_a<<<nblk(P * 7 * h * kk, 256), 256, 0, s>>>(As[d], P, h, kk, As[d + 1]);
        note(cudaGetLastError());
        k_down_b<<<nblk(2 * P * 7 * kk * ww, 64), 64, 0, s>>>(Bs[d], P, kk, ww, Bs[d + 1]);
        note(cudaGetLastError());
        P *= 7;
    }
    const int mD = m >> D, nD = n >> D, lD = l >> D;
    if (err == cudaSuccess) {                                            // leaves: batched schoolbook
        if (D == 0) Cs[0] = out;
        else note(cudaMallocAsync((void **)&Cs[D], (size_t)P * mD * lD * 2 * kPtWords * 4, s));
        if (err == cudaSuccess) {
            dim3 grid((unsigned)((int64_t)nblk(lD, 32) * nblk(mD, 4) * 2 * P));
            k_school_batched<<<grid, 128, 0, s>>>(As[D], mD, nD, lD, P, Bs[D], Cs[D]);
            note(cudaGetLastError());
        }
    }
    for (int d = D - 1; d >= 0 && err == cudaSuccess; d--) {             // up: C blocks from M1..M7
        P /= 7;
        const int h = m >> (d + 1), ww = l >> (d + 1);
        if (d == 0) Cs[0] = out;
        else note(cudaMallocAsync((void **)&Cs[d], (size_t)P * 4 * h * ww * 2 * kPtWords * 4, s));
        if (err) break;
        k_up_c<<<nblk(2 * P * 4 * h * ww, 64), 64, 0, s>>>(Cs[d + 1], P, h, ww, Cs[d]);
        note(cudaGetLastError());
        cudaFreeAsync(Cs[d + 1], s);
    }
    for (int d = 0; d <= D; d++) {
        if (As[d]) cudaFreeAsync(As[d], s);
        if (d > 0 && Bs[d]) cudaFreeAsync(Bs[d], s);
    }
    return err;
}

}  // namespace pcmm
