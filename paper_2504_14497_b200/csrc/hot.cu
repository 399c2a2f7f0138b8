// hot.cu -- the dominant kernel of the Cussen path (step a4 of SURVEY.md §8(a))
// and the fp_mul throughput probe, in their own translation unit (parallel
// compilation; the hot loop inlines the complete addition and fe_mul).
#include <algorithm>

#include "ec.cuh"
#include "internal.h"
#include "jac.cuh"

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
// Tables hold S = 2^w affine slots per (k, j, c) (entry-major [slot][16 words],
// slot 0 = the identity).  Per chunk of KCH = min(128, 512/S) columns the CTA
// stages the tables and the rank bytes of its rows in shared memory (entries
// padded to 17 words: lanes gathering different slots hit different banks);
// each lane then walks ITS OWN nonzero entries of the chunk (a_ik = 0 adds the
// identity and is skipped, R1), so a warp runs max-over-lanes of the
// nonzero count instead of KCH additions (25% zeros at w = 2).
#ifndef PCMM_ACCUM_CHUNK_SLOTS
#define PCMM_ACCUM_CHUNK_SLOTS 512  // table slots staged per chunk: k-chunk = this / 2^w (32 at w = 4)
#endif
#ifndef PCMM_ACC_UNROLL2
#define PCMM_ACC_UNROLL2 0      // 1: two pipelined steps per loop trip, entry registers alternating roles
#endif
#ifndef PCMM_ACC_LAZY
// 1: almost-reduced values in the pipelined step (jac.cuh xyzz_add_aff_pipe_lz: no final conditional
// subtraction in the products, lazy sums / differences).  Measured 8 % slower at 256^3 (3.95 vs
// 3.67 ms): the rare second-correction branches of the lazy add / subtract split the straight-line
// step into basic blocks that ptxas no longer interleaves, and the masked fold-back costs about what
// the subtraction saved.  Kept as a measured variant (parity-tested by test_lazy_field_ops).
#define PCMM_ACC_LAZY 0
#endif
#ifndef PCMM_ACC_PIPE
#define PCMM_ACC_PIPE 1         // software-pipelined XYZZ step (jac.cuh xyzz_add_aff_pipe); needs PCMM_ACC_XYZZ
#endif
#if !PCMM_ACC_XYZZ
#undef PCMM_ACC_PIPE
#define PCMM_ACC_PIPE 0
#endif
#ifndef PCMM_ACCUM_MINB
// resident CTAs per SM the register allocation targets (3: 168 regs, 4: 128, 5: 96).  The pipelined
// step's 4-product groups spill at 128 registers (256^3 accumulate +6 %); at 3 CTAs per SM it is 1.7 %
// faster than the 4-group step at 4 CTAs per SM (which is 2 % slower at 3)
#if PCMM_ACC_PIPE
#define PCMM_ACCUM_MINB 3
#else
#define PCMM_ACCUM_MINB 4
#endif
#endif

#ifndef PCMM_ACC_ROWS
#define PCMM_ACC_ROWS 128       // rows of A (threads) per k_accum CTA
#endif
#ifndef PCMM_ACC_EW
#define PCMM_ACC_EW 17          // shared-memory words per 16-word table entry (17: odd stride; 20: 16-B vector loads)
#endif
template <int S, int R = PCMM_ACC_ROWS>
struct AccumCfg {
    static constexpr int kRows = R;
    static constexpr int kChunk = (PCMM_ACCUM_CHUNK_SLOTS / S) < 128 ? (PCMM_ACCUM_CHUNK_SLOTS / S) : 128;
    static constexpr int kTW = kAffWords * S;                      // words per table (global, entry-major)
    static constexpr int kEW = PCMM_ACC_EW;                        // shared-memory entry stride
    static constexpr int kTWs = kEW * S;                           // words per table in shared memory
    static constexpr size_t kSmem = (size_t)kChunk * kTWs * 4 + (size_t)kChunk * kRows;
};

template <int EW>
__device__ __forceinline__ void ld_entry(fe &x, fe &y, const uint32_t *T) {
    if constexpr (EW % 4 == 0) {
        const uint4 *q = reinterpret_cast<const uint4 *>(T);
        const uint4 a = q[0], b = q[1], c = q[2], d = q[3];
        x = fe{{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w}};
        y = fe{{c.x, c.y, c.z, c.w, d.x, d.y, d.z, d.w}};
    } else {
#pragma unroll
        for (int q = 0; q < 8; q++) {
            x.v[q] = T[q];
            y.v[q] = T[8 + q];
        }
    }
}

// Stage one k-chunk: tables and the rank bytes of the CTA's rows.  Out of line so
// that the staging code does not perturb the hot loop's register allocation.
template <int S, int R>
__device__ __noinline__ void stage_chunk(const uint32_t *__restrict__ tables, const uint8_t *__restrict__ rank,
                                         uint4 *smem4, uint8_t *rsm, int m, int n, int l, int c, int j, int rb,
                                         int k0, int kc, int tid) {
    constexpr int ROWS = AccumCfg<S, R>::kRows, TW = AccumCfg<S, R>::kTW;
    constexpr int EW = AccumCfg<S, R>::kEW, TWS = AccumCfg<S, R>::kTWs;
    uint32_t *tsw = reinterpret_cast<uint32_t *>(smem4);
    for (int t = tid; t < kc * (TW / 4); t += ROWS) {
        const int kk = t / (TW / 4), r = t % (TW / 4);
        const int slot = r / (kAffWords / 4), q4 = (r % (kAffWords / 4)) * 4;
        const uint4 v = reinterpret_cast<const uint4 *>(tables + (((int64_t)c * n + (k0 + kk)) * l + j) * TW)[r];
        PCMM_DCHECK(kk < kc && kk * TWS + slot * EW + q4 + 3 < AccumCfg<S, R>::kChunk * TWS && k0 + kk < n);
        uint32_t *d = tsw + kk * TWS + slot * EW + q4;
        d[0] = v.x;
        d[1] = v.y;
        d[2] = v.z;
        d[3] = v.w;
    }
    for (int t = tid; t < kc * ROWS; t += ROWS) {
        const int row = rb * ROWS + (t % ROWS);
        PCMM_DCHECK(t < AccumCfg<S, R>::kChunk * ROWS);
        rsm[t] = row < m ? rank[(int64_t)(k0 + t / ROWS) * m + row] : (uint8_t)0;
        PCMM_DCHECK(rsm[t] < S);
    }
}

// The running output of earlier k-chunks (byte path, chunked, ksplit = 1): homogeneous (X : Y : Z) ->
// the accumulator (Z = 0: the identity stays the initial value)
__device__ __forceinline__ void acc_load_running(acc_t &acc, const uint32_t *ob, int64_t cnt, int64_t oi) {
#ifdef __CUDA_ARCH__
    pt o;
#pragma unroll
    for (int q = 0; q < 8; q++) {
        o.X.v[q] = ob[(0 * 8 + q) * cnt + oi];
        o.Y.v[q] = ob[(1 * 8 + q) * cnt + oi];
        o.Z.v[q] = ob[(2 * 8 + q) * cnt + oi];
    }
    if (!fe_is_zero(o.Z)) acc_from_proj(acc, o);
#endif
}

// R = rows per CTA (128, or 64 for m <= 64: twice the resident CTAs, no idle half-CTA)
template <int S, int R>
__global__ void __launch_bounds__(R, PCMM_ACCUM_MINB * (PCMM_ACC_ROWS / R))
    k_accum(const uint32_t *__restrict__ tables, const uint8_t *__restrict__ rank, int m, int n, int l, int ksplit,
            uint32_t *__restrict__ out, int64_t split_stride, int acc_in) {
    constexpr int ROWS = AccumCfg<S, R>::kRows, KCH = AccumCfg<S, R>::kChunk;
    constexpr int EW = AccumCfg<S, R>::kEW, TWS = AccumCfg<S, R>::kTWs;
    extern __shared__ uint4 smem4[];
    const uint32_t *tsm = reinterpret_cast<const uint32_t *>(smem4);
    uint8_t *rsm = reinterpret_cast<uint8_t *>(smem4) + (size_t)KCH * TWS * 4;
    int b = blockIdx.x;
    const int j = b % l; b /= l;
    const int c = b & 1; b >>= 1;
    const int rowblocks = (m + ROWS - 1) / ROWS;
    const int rb = b % rowblocks;
    const int s = b / rowblocks;
    const int tid = (int)threadIdx.x;
    const int i = rb * ROWS + tid;
    const int kb = (int)((int64_t)s * n / ksplit), ke = (int)((int64_t)(s + 1) * n / ksplit);
    PCMM_DCHECK(blockDim.x == ROWS && s < ksplit && c < 2);
    acc_t acc;
    acc_init(acc);
    if (acc_in && i < m) acc_load_running(acc, out + (int64_t)c * kPtWords * m * l, (int64_t)m * l, (int64_t)i * l + j);
    for (int k0 = kb; k0 < ke; k0 += KCH) {
        const int kc = min(KCH, ke - k0);
        __syncthreads();
        stage_chunk<S, R>(tables, rank, smem4, rsm, m, n, l, c, j, rb, k0, kc, tid);
        __syncthreads();
        // each lane walks its own nonzero entries (zeros are the identity, skipped)
        int kk = 0;
        while (kk < kc && rsm[kk * ROWS + tid] == 0) kk++;
#if PCMM_ACC_PIPE
        if (kk < kc) {
            fe x2, y2, U2;
            bool have_u2 = false;
            ld_entry<EW>(x2, y2, tsm + kk * TWS + rsm[kk * ROWS + tid] * EW);
#if PCMM_ACC_UNROLL2
            // two steps per trip with the entry registers alternating roles (no x2 = xn copies)
            fe xn, yn;
            while (true) {
                int kn = kk + 1;
                while (kn < kc && rsm[kn * ROWS + tid] == 0) kn++;
                bool more = kn < kc;
                ld_entry<EW>(xn, yn, tsm + (more ? kn * TWS + rsm[kn * ROWS + tid] * EW : kk * TWS + rsm[kk * ROWS + tid] * EW));
                xyzz_add_aff_pipe(acc, x2, y2, U2, have_u2, xn);
                if (!more) break;
                kk = kn;
                kn = kk + 1;
                while (kn < kc && rsm[kn * ROWS + tid] == 0) kn++;
                more = kn < kc;
                ld_entry<EW>(x2, y2, tsm + (more ? kn * TWS + rsm[kn * ROWS + tid] * EW : kk * TWS + rsm[kk * ROWS + tid] * EW));
                xyzz_add_aff_pipe(acc, xn, yn, U2, have_u2, x2);
                if (!more) break;
                kk = kn;
            }
#else
            while (true) {
                int kn = kk + 1;
                while (kn < kc && rsm[kn * ROWS + tid] == 0) kn++;
                const bool more = kn < kc;
                const uint32_t *T = tsm + (more ? kn * TWS + rsm[kn * ROWS + tid] * EW : kk * TWS + rsm[kk * ROWS + tid] * EW);
                fe xn, yn;
                ld_entry<EW>(xn, yn, T);
#if PCMM_ACC_LAZY
                xyzz_add_aff_pipe_lz(acc, x2, y2, U2, have_u2, xn);
#else
                xyzz_add_aff_pipe(acc, x2, y2, U2, have_u2, xn);
#endif
                if (!more) break;
                x2 = xn;
                y2 = yn;
                kk = kn;
            }
#endif
        }
#else
        while (kk < kc) {
            const uint32_t *T = tsm + kk * TWS + rsm[kk * ROWS + tid] * EW;
            fe x2, y2;
#pragma unroll
            for (int q = 0; q < 8; q++) {
                x2.v[q] = T[q];
                y2.v[q] = T[8 + q];
            }
            acc_add_aff(acc, x2, y2);
            kk++;
            while (kk < kc && rsm[kk * ROWS + tid] == 0) kk++;
        }
#endif
    }
    if (i < m) {
        const int64_t cnt = (int64_t)m * l;
        pt o;
        acc_to_proj(o, acc);
        soa_store_hot(out + (int64_t)s * split_stride + (int64_t)c * kPtWords * cnt, cnt, (int64_t)i * l + j, o);
    }
}

// ------------------------------------------------------------ a4 for w > 4: global gather
// Tables of up to 2^w = 256 slots (16 KB per (k, j, c)) do not fit in shared
// memory in useful chunks; each lane gathers its 64-byte entry straight from the
// L2-resident tables (4 x 16-byte loads), the next entry prefetched while the
// current addition runs.  Zero entries (slot 0) are skipped per lane.
__device__ __forceinline__ void load_aff(fe &x, fe &y, const uint32_t *e) {
    const uint4 *q = reinterpret_cast<const uint4 *>(e);
    const uint4 a = q[0], b = q[1], c = q[2], d = q[3];
    x.v[0] = a.x; x.v[1] = a.y; x.v[2] = a.z; x.v[3] = a.w;
    x.v[4] = b.x; x.v[5] = b.y; x.v[6] = b.z; x.v[7] = b.w;
    y.v[0] = c.x; y.v[1] = c.y; y.v[2] = c.z; y.v[3] = c.w;
    y.v[4] = d.x; y.v[5] = d.y; y.v[6] = d.z; y.v[7] = d.w;
}

constexpr int kRowsG = 128;

__global__ void __launch_bounds__(kRowsG, 3)
    k_accum_g(const uint32_t *__restrict__ tables, const uint8_t *__restrict__ rank, int m, int n, int l, int S,
              int ksplit, uint32_t *__restrict__ out, int64_t split_stride, int acc_in) {
    int b = blockIdx.x;
    const int j = b % l; b /= l;
    const int c = b & 1; b >>= 1;
    const int rowblocks = (m + kRowsG - 1) / kRowsG;
    const int rb = b % rowblocks;
    const int s = b / rowblocks;
    const int i = rb * kRowsG + (int)threadIdx.x;
    if (i >= m) return;
    const int kb = (int)((int64_t)s * n / ksplit), ke = (int)((int64_t)(s + 1) * n / ksplit);
    const int64_t tstride = (int64_t)l * S * kAffWords;                  // words between consecutive k
    const uint32_t *tb = tables + (((int64_t)c * n) * l + j) * (int64_t)S * kAffWords;
    acc_t acc;
    acc_init(acc);
    if (acc_in) acc_load_running(acc, out + (int64_t)c * kPtWords * m * l, (int64_t)m * l, (int64_t)i * l + j);
    int k = kb;
    while (k < ke && rank[(int64_t)k * m + i] == 0) k++;
    if (k < ke) {
        fe x2, y2;
        PCMM_DCHECK(rank[(int64_t)k * m + i] < S);
        load_aff(x2, y2, tb + k * tstride + rank[(int64_t)k * m + i] * kAffWords);
        while (true) {
            int kn = k + 1;
            while (kn < ke && rank[(int64_t)kn * m + i] == 0) kn++;
            fe xn, yn;
            PCMM_DCHECK(kn >= ke || rank[(int64_t)kn * m + i] < S);
            if (kn < ke) load_aff(xn, yn, tb + kn * tstride + rank[(int64_t)kn * m + i] * kAffWords);
            acc_add_aff(acc, x2, y2);
            if (kn >= ke) break;
            x2 = xn;
            y2 = yn;
            k = kn;
        }
    }
    const int64_t cnt = (int64_t)m * l;
    pt o;
    acc_to_proj(o, acc);
    soa_store_hot(out + (int64_t)s * split_stride + (int64_t)c * kPtWords * cnt, cnt, (int64_t)i * l + j, o);
}

// ------------------------------------------------------------ a4, gather kernel with sorted rows
// Every lane skips its own zero entries (a_ik = 0 adds the identity, R1), so a warp runs the
// maximum over its lanes of the nonzero count: with rows in matrix order that is 6 % (256^3, 1/16
// zeros) to 10 % (512^3, w = 2: 1/4 zeros) more steps than the mean.  k_rowperm sorts the rows of
// each 128-row block by their nonzero count over the k-range of each split (the permutation serves
// every output column j and both components), so the lanes of a warp finish together; k_accum_g2 is
// k_accum_g with the row of a thread taken from that permutation and the software-pipelined step
// (jac.cuh xyzz_add_aff_pipe).  Which output a thread accumulates changes; what it adds does not.
__global__ void __launch_bounds__(kRowsG) k_rowperm(const uint8_t *__restrict__ rank, int m, int n, int ksplit,
                                                    int *__restrict__ perm) {
    __shared__ uint32_t key[kRowsG];
    const int rowblocks = (m + kRowsG - 1) / kRowsG;
    const int rb = (int)blockIdx.x % rowblocks, s = (int)blockIdx.x / rowblocks;
    const int tid = (int)threadIdx.x;
    const int i = rb * kRowsG + tid;
    const int kb = (int)((int64_t)s * n / ksplit), ke = (int)((int64_t)(s + 1) * n / ksplit);
    uint32_t cnt = 0;
    if (i < m)
        for (int k = kb; k < ke; k++) cnt += rank[(int64_t)k * m + i] != 0;
    PCMM_DCHECK(cnt < (1u << 24));
    key[tid] = (cnt << 8) | (uint32_t)tid;                  // rows >= m: count 0, sorted last
    __syncthreads();
    for (int size = 2; size <= kRowsG; size <<= 1) {        // bitonic sort, descending
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const int p = tid ^ stride;
            if (p > tid) {
                const uint32_t a = key[tid], b = key[p];
                const bool desc = (tid & size) == 0;
                if (desc ? a < b : a > b) {
                    key[tid] = b;
                    key[p] = a;
                }
            }
            __syncthreads();
        }
    }
    perm[((int64_t)s * rowblocks + rb) * kRowsG + tid] = rb * kRowsG + (int)(key[tid] & 0xffu);
}

// m <= 4096: all rows of a split sorted together (one CTA per split, bitonic sort of the next power of
// two >= the padded row count in shared memory), so that a warp's 32 rows are 32 consecutive order
// statistics of the whole column of counts instead of a quarter of one 128-row block's
// (512^3, w = 2: the spread of the counts inside a warp drops from ~1 sigma to ~0.3 sigma).
__global__ void __launch_bounds__(1024) k_rowperm_all(const uint8_t *__restrict__ rank, int m, int n, int ksplit,
                                                      int np, int *__restrict__ perm) {
    extern __shared__ uint32_t keys[];
    const int s = (int)blockIdx.x, tid = (int)threadIdx.x, nt = (int)blockDim.x;
    const int mpad = ((m + kRowsG - 1) / kRowsG) * kRowsG;
    const int kb = (int)((int64_t)s * n / ksplit), ke = (int)((int64_t)(s + 1) * n / ksplit);
    PCMM_DCHECK(np <= 4096 && mpad <= np);
    for (int idx = tid; idx < np; idx += nt) {
        uint32_t cnt = 0;
        if (idx < m) {
            cnt = 1;                                        // every valid row sorts before the padding
            for (int k = kb; k < ke; k++) cnt += rank[(int64_t)k * m + idx] != 0;
        }
        PCMM_DCHECK(cnt < (1u << 20));
        keys[idx] = (cnt << 12) | (uint32_t)idx;
    }
    __syncthreads();
    for (int size = 2; size <= np; size <<= 1) {            // bitonic sort, descending
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int idx = tid; idx < np; idx += nt) {
                const int p = idx ^ stride;
                if (p > idx) {
                    const uint32_t a = keys[idx], b = keys[p];
                    const bool desc = (idx & size) == 0;
                    if (desc ? a < b : a > b) {
                        keys[idx] = b;
                        keys[p] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int idx = tid; idx < mpad; idx += nt) perm[(int64_t)s * mpad + idx] = (int)(keys[idx] & 0xfffu);
}

template <bool kPipe>
__global__ void __launch_bounds__(kRowsG, 3)
    k_accum_g2(const uint32_t *__restrict__ tables, const uint8_t *__restrict__ rank, int m, int n, int l, int S,
               int ksplit, uint32_t *__restrict__ out, int64_t split_stride, int acc_in,
               const int *__restrict__ perm) {
    int b = blockIdx.x;
    const int j = b % l; b /= l;
    const int c = b & 1; b >>= 1;
    const int rowblocks = (m + kRowsG - 1) / kRowsG;
    const int rb = b % rowblocks;
    const int s = b / rowblocks;
    const int i = perm[((int64_t)s * rowblocks + rb) * kRowsG + (int)threadIdx.x];
    PCMM_DCHECK(i >= 0 && i < rowblocks * kRowsG + 4096);
    if (i >= m) return;
    const int kb = (int)((int64_t)s * n / ksplit), ke = (int)((int64_t)(s + 1) * n / ksplit);
    const int64_t tstride = (int64_t)l * S * kAffWords;                  // words between consecutive k
    const uint32_t *tb = tables + (((int64_t)c * n) * l + j) * (int64_t)S * kAffWords;
    acc_t acc;
    acc_init(acc);
    if (acc_in) acc_load_running(acc, out + (int64_t)c * kPtWords * m * l, (int64_t)m * l, (int64_t)i * l + j);
    int k = kb;
    while (k < ke && rank[(int64_t)k * m + i] == 0) k++;
    if (k < ke) {
        fe x2, y2;
        PCMM_DCHECK(rank[(int64_t)k * m + i] < S);
        load_aff(x2, y2, tb + k * tstride + rank[(int64_t)k * m + i] * kAffWords);
#if PCMM_ACC_XYZZ
        fe U2;
        bool have_u2 = false;
#endif
        while (true) {
            int kn = k + 1;
            while (kn < ke && rank[(int64_t)kn * m + i] == 0) kn++;
            fe xn = x2, yn = y2;
            PCMM_DCHECK(kn >= ke || rank[(int64_t)kn * m + i] < S);
            if (kn < ke) load_aff(xn, yn, tb + kn * tstride + rank[(int64_t)kn * m + i] * kAffWords);
#if PCMM_ACC_XYZZ
            if (kPipe) xyzz_add_aff_pipe(acc, x2, y2, U2, have_u2, xn);
            else acc_add_aff(acc, x2, y2);
#else
            acc_add_aff(acc, x2, y2);
#endif
            if (kn >= ke) break;
            x2 = xn;
            y2 = yn;
            k = kn;
        }
    }
    const int64_t cnt = (int64_t)m * l;
    pt o;
    acc_to_proj(o, acc);
    soa_store_hot(out + (int64_t)s * split_stride + (int64_t)c * kPtWords * cnt, cnt, (int64_t)i * l + j, o);
}

cudaError_t launch_rowperm(const uint8_t *rank, int m, int n, int ksplit, int *perm, cudaStream_t s) {
    const int rowblocks = (m + kRowsG - 1) / kRowsG;
    static int all_env = -1;                                  // PCMM_ROWPERM_ALL=0: per-block sort always
    if (all_env < 0) {
        const char *e = getenv("PCMM_ROWPERM_ALL");
        all_env = e ? atoi(e) : 1;
    }
    if (all_env && rowblocks * kRowsG <= 4096) {
        int np = 128;
        while (np < rowblocks * kRowsG) np <<= 1;
        k_rowperm_all<<<(unsigned)ksplit, std::min(1024, np), (size_t)np * 4, s>>>(rank, m, n, ksplit, np, perm);
    } else {
        k_rowperm<<<(unsigned)(rowblocks * ksplit), kRowsG, 0, s>>>(rank, m, n, ksplit, perm);
    }
    return cudaGetLastError();
}

cudaError_t launch_accum_sorted(const uint32_t *tables, const uint8_t *rank, int m, int n, int l, int slots,
                                int ksplit, uint32_t *out, int64_t out_stride_split, cudaStream_t s, int acc_in,
                                const int *perm, int pipe) {
    const int rowblocks = (m + kRowsG - 1) / kRowsG;
    const unsigned grid = (unsigned)((int64_t)l * 2 * rowblocks * ksplit);
    if (pipe)
        k_accum_g2<true><<<grid, kRowsG, 0, s>>>(tables, rank, m, n, l, slots, ksplit, out, out_stride_split, acc_in,
                                                 perm);
    else
        k_accum_g2<false><<<grid, kRowsG, 0, s>>>(tables, rank, m, n, l, slots, ksplit, out, out_stride_split, acc_in,
                                                  perm);
    return cudaGetLastError();
}

// ------------------------------------------------------------ a4 (wide path, NEXT-1): one k-chunk
// As k_accum_g for the chunk k0 .. k0+kc-1 of the wide path (wide.cu): uint16
// rank, tables [c][kk][j][slot][16].  The accumulator starts from the running
// output (homogeneous (X : Y : Z) -> XYZZ (X Z, Y Z^2, Z^2, Z^3)) unless this is
// the first chunk, and the chunk's sum is written back to it.
__global__ void __launch_bounds__(kRowsG, 3)
    k_accum_gw(const uint32_t *__restrict__ tables, const uint16_t *__restrict__ rank, int m, int l, int S, int k0,
               int kc, int first, uint32_t *__restrict__ out) {
    int b = blockIdx.x;
    const int j = b % l; b /= l;
    const int c = b & 1; b >>= 1;
    const int i = b * kRowsG + (int)threadIdx.x;
    if (i >= m) return;
    const int64_t cnt = (int64_t)m * l;
    uint32_t *ob = out + (int64_t)c * kPtWords * cnt;
    const int64_t oi = (int64_t)i * l + j;
    acc_t acc;
    acc_init(acc);
#ifdef __CUDA_ARCH__
    if (!first) {
        pt o;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            o.X.v[q] = ob[(0 * 8 + q) * cnt + oi];
            o.Y.v[q] = ob[(1 * 8 + q) * cnt + oi];
            o.Z.v[q] = ob[(2 * 8 + q) * cnt + oi];
        }
        if (!fe_is_zero(o.Z)) acc_from_proj(acc, o);
    }
#endif
    const int64_t tstride = (int64_t)l * S * kAffWords;                  // words between consecutive kk
    const uint32_t *tb = tables + (((int64_t)c * kc) * l + j) * (int64_t)S * kAffWords;
    const uint16_t *rk = rank + (int64_t)k0 * m + i;
    int k = 0;
    while (k < kc && rk[(int64_t)k * m] == 0) k++;
    if (k < kc) {
        fe x2, y2;
        load_aff(x2, y2, tb + k * tstride + (int64_t)rk[(int64_t)k * m] * kAffWords);
#if PCMM_ACC_XYZZ
        fe U2;
        bool have_u2 = false;
#endif
        while (true) {
            int kn = k + 1;
            while (kn < kc && rk[(int64_t)kn * m] == 0) kn++;
            fe xn = x2, yn = y2;
            if (kn < kc) load_aff(xn, yn, tb + kn * tstride + (int64_t)rk[(int64_t)kn * m] * kAffWords);
#if PCMM_ACC_XYZZ
            xyzz_add_aff_pipe(acc, x2, y2, U2, have_u2, xn);          // the software-pipelined step (as k_accum_g2)
#else
            acc_add_aff(acc, x2, y2);
#endif
            if (kn >= kc) break;
            x2 = xn;
            y2 = yn;
            k = kn;
        }
    }
    pt o;
    acc_to_proj(o, acc);
    soa_store_hot(ob, cnt, oi, o);
}

cudaError_t launch_accum_wide(const uint32_t *atables, const uint16_t *rank, int m, int l, int S, int k0, int kc,
                              int first, uint32_t *out, cudaStream_t s) {
    const int rowblocks = (m + kRowsG - 1) / kRowsG;
    const unsigned grid = (unsigned)((int64_t)l * 2 * rowblocks);
    k_accum_gw<<<grid, kRowsG, 0, s>>>(atables, rank, m, l, S, k0, kc, first, out);
    return cudaGetLastError();
}

int accum_global_ctas_per_sm() {
    static int occ = 0;
    if (!occ) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_accum_g, kRowsG, 0) != cudaSuccess || occ <= 0)
            occ = 3;
    }
    return occ;
}

cudaError_t launch_accum_global(const uint32_t *tables, const uint8_t *rank, int m, int n, int l, int slots,
                                int ksplit, uint32_t *out, int64_t out_stride_split, cudaStream_t s, int acc_in) {
    const int rowblocks = (m + kRowsG - 1) / kRowsG;
    const unsigned grid = (unsigned)((int64_t)l * 2 * rowblocks * ksplit);
    k_accum_g<<<grid, kRowsG, 0, s>>>(tables, rank, m, n, l, slots, ksplit, out, out_stride_split, acc_in);
    return cudaGetLastError();
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
#ifdef __CUDA_ARCH__
            else if (VARIANT == 3) fe_mul_fast_v<1 - PCMM_MUL_PRODUCT>(x[c], x[c], y);
#endif
            else fe_mul(x[c], x[c], y);
        }
    }
#pragma unroll
    for (int i = 0; i < 8; i++) out[t * 8 + i] = x[0].v[i] ^ x[1].v[i] ^ x[2].v[i] ^ x[3].v[i];
}

template <int S, int R>
static int ctas_per_sm_s() {
    int occ = 0;
    cudaFuncSetAttribute(k_accum<S, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)AccumCfg<S, R>::kSmem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_accum<S, R>, R, AccumCfg<S, R>::kSmem) != cudaSuccess ||
        occ <= 0)
        occ = 3;
    return occ;
}

// rows per k_accum CTA for m rows: 64 when m <= 64 (PCMM_ACC_SMALL=0 disables)
int accum_rows(int m) {
    static int small = -1;
    if (small < 0) {
        const char *e = getenv("PCMM_ACC_SMALL");
        small = e ? atoi(e) : 1;
    }
    return (small && m <= 64 && PCMM_ACC_ROWS == 128) ? 64 : AccumCfg<16>::kRows;
}

// resident k_accum CTAs per SM for table slot count S = 2^w and the CTA's rows (wave-balanced split-k)
int accum_ctas_per_sm(int slots, int rows) {
    static int occ[2][17] = {{0}};
    if (slots < 2 || slots > 16) slots = 16;
    const int r = rows == 64 && PCMM_ACC_ROWS == 128 ? 1 : 0;
    if (!occ[r][slots]) {
#if PCMM_ACC_ROWS == 128
        if (r) {
            switch (slots) {
                case 2: occ[r][slots] = ctas_per_sm_s<2, 64>(); break;
                case 4: occ[r][slots] = ctas_per_sm_s<4, 64>(); break;
                case 8: occ[r][slots] = ctas_per_sm_s<8, 64>(); break;
                default: occ[r][slots] = ctas_per_sm_s<16, 64>(); break;
            }
        } else
#endif
        {
            switch (slots) {
                case 2: occ[r][slots] = ctas_per_sm_s<2, PCMM_ACC_ROWS>(); break;
                case 4: occ[r][slots] = ctas_per_sm_s<4, PCMM_ACC_ROWS>(); break;
                case 8: occ[r][slots] = ctas_per_sm_s<8, PCMM_ACC_ROWS>(); break;
                default: occ[r][slots] = ctas_per_sm_s<16, PCMM_ACC_ROWS>(); break;
            }
        }
    }
    return occ[r][slots];
}

int accum_chunk(int slots) {
    switch (slots) {
        case 2: return AccumCfg<2>::kChunk;
        case 4: return AccumCfg<4>::kChunk;
        case 8: return AccumCfg<8>::kChunk;
        default: return AccumCfg<16>::kChunk;
    }
}

template <int S, int R>
static cudaError_t launch_accum_s(const uint32_t *tables, const uint8_t *rank, int m, int n, int l, int ksplit,
                                  uint32_t *out, int64_t stride, cudaStream_t s, int acc_in) {
    const int rowblocks = (m + R - 1) / R;
    const unsigned grid = (unsigned)((int64_t)l * 2 * rowblocks * ksplit);
    cudaError_t err =
        cudaFuncSetAttribute(k_accum<S, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)AccumCfg<S, R>::kSmem);
    if (err) return err;
    k_accum<S, R><<<grid, R, AccumCfg<S, R>::kSmem, s>>>(tables, rank, m, n, l, ksplit, out, stride, acc_in);
    return cudaGetLastError();
}

template <int R>
static cudaError_t launch_accum_r(const uint32_t *tables, const uint8_t *rank, int m, int n, int l, int slots,
                                  int ksplit, uint32_t *out, int64_t out_stride_split, cudaStream_t s, int acc_in) {
    switch (slots) {
        case 2: return launch_accum_s<2, R>(tables, rank, m, n, l, ksplit, out, out_stride_split, s, acc_in);
        case 4: return launch_accum_s<4, R>(tables, rank, m, n, l, ksplit, out, out_stride_split, s, acc_in);
        case 8: return launch_accum_s<8, R>(tables, rank, m, n, l, ksplit, out, out_stride_split, s, acc_in);
        default: return launch_accum_s<16, R>(tables, rank, m, n, l, ksplit, out, out_stride_split, s, acc_in);
    }
}

cudaError_t launch_accum(const uint32_t *tables, const uint8_t *rank, int m, int n, int l, int slots, int ksplit,
                         uint32_t *out, int64_t out_stride_split, cudaStream_t s, int acc_in) {
#if PCMM_ACC_ROWS == 128
    if (accum_rows(m) == 64)
        return launch_accum_r<64>(tables, rank, m, n, l, slots, ksplit, out, out_stride_split, s, acc_in);
#endif
    return launch_accum_r<PCMM_ACC_ROWS>(tables, rank, m, n, l, slots, ksplit, out, out_stride_split, s, acc_in);
}

cudaError_t launch_bench_fp_mul(int variant, int blocks, int threads, int iters, uint32_t *out, cudaStream_t s) {
    if (variant == 1) k_bench_fp_mul<1><<<blocks, threads, 0, s>>>(iters, out);
    else if (variant == 2) k_bench_fp_mul<2><<<blocks, threads, 0, s>>>(iters, out);
    else if (variant == 3) k_bench_fp_mul<3><<<blocks, threads, 0, s>>>(iters, out);
    else k_bench_fp_mul<0><<<blocks, threads, 0, s>>>(iters, out);
    return cudaGetLastError();
}

}  // namespace pcmm
