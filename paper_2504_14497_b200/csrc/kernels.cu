// kernels.cu -- sm_100a kernels of the PC-MM hot path and of
// the boundary calls around it.  Launched only through api.cu.
//
//   k_import       a0: canonical big-endian ciphertexts -> Montgomery SoA
//   k_plan         a1: Alg. 2 compression of every column of A
//   k_tables       a2+a3: per (k, j, component) ECSMs of the level-N values and
//                  reconstruction prefix sums -> T_kj[v] = v * Enc(b_kj)
//                  (Alg. 3 lines 5-6, Alg. 2 lines 13-23)
//   k_accum        a4: un-sort / re-insert + accumulation C_ij += T_kj[a_ik]
//                  from shared-memory table chunks (Alg. 3 lines 6-9)
//   k_reduce       a5: split-k partial sums
//   k_normalize    a6: batch inversion -> canonical affine bytes
//   k_school       s1: schoolbook PC-MM
//   k_encrypt / k_pubkey: boundary; decryption: next2.cu (BSGS)

#include <algorithm>

#include "canon.cuh"
#include "jac.cuh"
#include "ec.cuh"
#include "internal.h"
#include "shared.cuh"

namespace pcmm {

// ------------------------------------------------------------ a0: import
__global__ void k_import(const uint8_t *__restrict__ ct, int64_t count, uint32_t *__restrict__ soa,
                         int *__restrict__ status) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * count) return;
    int64_t e = t >> 1;
    int c = (int)(t & 1);
    pt P;
    bool ok = load_canonical_point(P, ct + e * 128 + c * 64);
    if (!ok) atomicOr(status, kStatusCurve);
    soa_store(soa + (int64_t)c * kPtWords * count, count, e, P);
}

// ------------------------------------------------------------ a1: compression plan
// One warp per column k of A (values in [-128, 255]).  Level 1: the set of
// distinct nonzero values is a presence bitmap over [-128, 255] (12 words, bit
// v + 128) OR-reduced across the warp; rank[k][i] = 1 + (number of set bits
// below a_ik).  Lane 0 then builds levels 2..N the same way over [-128, 895]
// (32-word bitmap): level w values are differences of sorted level w-1 values.
constexpr int kBmOff = 128;

__device__ __forceinline__ int bm_rank(const uint32_t *bm, int bit) {
    int r = 0;
    for (int q = 0; q < (bit >> 5); q++) r += __popc(bm[q]);
    return r + __popc(bm[bit >> 5] & ((1u << (bit & 31)) - 1u));
}

__global__ void k_plan(const int8_t *__restrict__ A, int m, int n, int w, int is_signed, int N,
                       ColPlan *__restrict__ plans, uint8_t *__restrict__ rank, int *__restrict__ status) {
    int warp = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    int lane = threadIdx.x & 31;
    if (warp >= n) return;
    const int k = warp;
    const int lo = is_signed ? -(1 << (w - 1)) : 0;
    const int hi = is_signed ? (1 << (w - 1)) - 1 : (1 << w) - 1;
    uint32_t bm[12];
#pragma unroll
    for (int q = 0; q < 12; q++) bm[q] = 0;
    bool bad = false;
    for (int i = lane; i < m; i += 32) {
        const int a = is_signed ? (int)A[(int64_t)i * n + k] : (int)(uint8_t)A[(int64_t)i * n + k];
        if (a < lo || a > hi) bad = true;
        else if (a != 0) {
            const int b = a + kBmOff;
            PCMM_DCHECK(b >= 0 && (b >> 5) < 12);
#pragma unroll
            for (int q = 0; q < 12; q++)
                if ((b >> 5) == q) bm[q] |= 1u << (b & 31);
        }
    }
#pragma unroll
    for (int q = 0; q < 12; q++) bm[q] = __reduce_or_sync(0xffffffffu, bm[q]);
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, kStatusBound);
    // rank[k][i] = 1 + index of a_ik in the sorted distinct nonzero values (0 for a_ik = 0)
    for (int i = lane; i < m; i += 32) {
        const int a = is_signed ? (int)A[(int64_t)i * n + k] : (int)(uint8_t)A[(int64_t)i * n + k];
        uint8_t r = 0;
        if (a != 0 && a >= lo && a <= hi) r = (uint8_t)(1 + bm_rank(bm, a + kBmOff));
        rank[(int64_t)k * m + i] = r;
    }
    if (lane != 0) return;
    ColPlan *P = plans + k;
    int16_t s[kPlanCap], v[kPlanCap];
    int ns = 0;
    for (int q = 0; q < 12; q++)                                          // level 1 (R1), ascending
        for (uint32_t x = bm[q]; x; x &= x - 1u) s[ns++] = (int16_t)(32 * q + __ffs(x) - 1 - kBmOff);
    for (int q = 0; q < 4; q++) P->n[q] = 0;
    for (int q = 0; q < 12; q++) P->bm1[q] = bm[q];
    // chain columns (k_tables_coz): unsigned {1..ns}; signed with every magnitude 1..M present in some sign
    int coz = 0, sgn = 0;
    if (N >= 2 && ns >= 1) {
        if (!is_signed) {
            if (s[ns - 1] == ns) coz = ns;
        } else {
            const int M = max(abs((int)s[0]), abs((int)s[ns - 1]));
            bool ok = true;
            for (int u = 1; u <= M; u++) {
                const int bp = kBmOff + u, bn = kBmOff - u;
                if (!(((bm[bp >> 5] >> (bp & 31)) | (bm[bn >> 5] >> (bn & 31))) & 1u)) ok = false;
            }
            if (ok) {
                coz = M;
                sgn = 1;
            }
        }
    }
    P->coz = (int16_t)coz;
    P->sgn = (int16_t)sgn;
    for (int lev = 1; lev <= N; lev++) {
        if (lev > 1) {
            // level lev: sorted distinct values of the differenced level lev-1 (v, ns entries)
            uint32_t b2[32];
            for (int q = 0; q < 32; q++) b2[q] = 0;
            const int nv = ns;
            for (int e = 0; e < nv; e++) {
                const int b = v[e] + kBmOff;
                PCMM_DCHECK(b >= 0 && (b >> 5) < 32);
                b2[b >> 5] |= 1u << (b & 31);
            }
            ns = 0;
            for (int q = 0; q < 32; q++)
                for (uint32_t x = b2[q]; x; x &= x - 1u) s[ns++] = (int16_t)(32 * q + __ffs(x) - 1 - kBmOff);
            for (int e = 0; e < nv; e++) P->ptr[lev - 2][e] = (uint8_t)bm_rank(b2, v[e] + kBmOff);   // R3
        }
        PCMM_DCHECK(ns <= kPlanCap);
        P->n[lev - 1] = (int16_t)ns;
        if (lev < N) {                                          // differences, first element kept (R6)
            for (int e = 0; e < ns; e++) v[e] = (int16_t)(e == 0 ? s[0] : s[e] - s[e - 1]);
        } else {
            for (int e = 0; e < ns; e++) P->sN[e] = s[e];
        }
    }
    // status[1]: some column is not consecutive (k_tables / k_affine have work beside k_tables_coz)
    if (!col_consecutive(*P, N)) atomicOr(status + 1, 1);
}

// ------------------------------------------------------------ a2 + a3: tables
// Thread per (component c, column k, output column j); j fastest so that the
// loads of Enc(b_kj) are coalesced.  Reconstruction (Alg. 2 lines 14-23) in the
// recursive form b^(w)[u] = b^(w)[u-1] + b^(w+1)[ptr^(w)[u]] (R3, R7): levels
// >= 2 (at most 8 entries for w <= 4) live in a small local array; level 1 is
// produced as a running prefix sum and written straight to the table.

// Table entry (projective point) store, entry-major: 24 contiguous words per
// slot, written as 6 x 16-byte vector stores.
__device__ __forceinline__ void table_store(uint32_t *block, int slot, const pt &q) {
    PCMM_DCHECK(slot >= 0 && slot < kPlanCap);
    uint4 *d = reinterpret_cast<uint4 *>(block + slot * kPtWords);
    d[0] = make_uint4(q.X.v[0], q.X.v[1], q.X.v[2], q.X.v[3]);
    d[1] = make_uint4(q.X.v[4], q.X.v[5], q.X.v[6], q.X.v[7]);
    d[2] = make_uint4(q.Y.v[0], q.Y.v[1], q.Y.v[2], q.Y.v[3]);
    d[3] = make_uint4(q.Y.v[4], q.Y.v[5], q.Y.v[6], q.Y.v[7]);
    d[4] = make_uint4(q.Z.v[0], q.Z.v[1], q.Z.v[2], q.Z.v[3]);
    d[5] = make_uint4(q.Z.v[4], q.Z.v[5], q.Z.v[6], q.Z.v[7]);
}

// Upper-level scratch: entry e of (c, k, j) at words [((c n + k) 2 kMaxUpper + e) 24 + q] l + j,
// i.e. j innermost so that a warp (32 consecutive j, same k) reads and writes
// whole 128-byte lines; all indices are warp-uniform (same column plan).
__device__ __forceinline__ void scr_store(uint32_t *scr, int64_t base, int e, int64_t l, const pt &q) {
    PCMM_DCHECK(e >= 0 && e < 2 * 32);                       // two ping-pong levels of max_upper(w) <= 32
    uint32_t *d = scr + (base + (int64_t)e * kPtWords) * l;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        d[(0 * 8 + i) * l] = q.X.v[i];
        d[(1 * 8 + i) * l] = q.Y.v[i];
        d[(2 * 8 + i) * l] = q.Z.v[i];
    }
}

__device__ __forceinline__ void scr_load(pt &q, const uint32_t *scr, int64_t base, int e, int64_t l) {
    PCMM_DCHECK(e >= 0 && e < 2 * 32);
    const uint32_t *d = scr + (base + (int64_t)e * kPtWords) * l;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        q.X.v[i] = d[(0 * 8 + i) * l];
        q.Y.v[i] = d[(1 * 8 + i) * l];
        q.Z.v[i] = d[(2 * 8 + i) * l];
    }
}

// Alg. 3 line 5 for signed columns (k_tables<true>): v P for the level-N values
// sN[0..cnt) (ascending) into upper-level scratch.  A value whose magnitude equals
// the previous one's, or exceeds it by 1, reuses the previous product (|v| P =
// |v'| P or |v'| P + P, then the sign): the ML columns' {-8, 8, 9} cost 3 doublings
// + 1 addition instead of 9 + 1.  Out of line and only in the signed kernel: in
// the unsigned kernel (s^(N) = {1} in practice) it cost registers for nothing.
__device__ __noinline__ void level_n_products_shared(const int16_t *sN, int cnt, const pt P, uint32_t *sj,
                                                     int64_t sbase, int64_t l, int src) {
    pt prevabs, e;
    int prevmag = -1;
    for (int u = 0; u < cnt; u++) {
        const int v = sN[u];
        const int mag = v < 0 ? -v : v;
        if (mag == prevmag) {
            e = prevabs;
        } else if (prevmag > 0 && mag == prevmag + 1) {
            pt_add_pair(e, prevabs, P);
        } else {
            pt_mul_small_g<MulCall>(e, mag, P);
        }
        prevabs = e;
        prevmag = mag;
        if (v < 0) pt_neg(e, e);
        scr_store(sj, sbase, src + u, l, e);
    }
}

#ifndef PCMM_TABLES_MINB
#define PCMM_TABLES_MINB 2       // 236 registers, no spills: ML (signed) tables 0.679 -> 0.642 ms against 3 (168 registers + spills)
#endif
template <bool kSigned>
__global__ void __launch_bounds__(128, PCMM_TABLES_MINB) k_tables(const uint32_t *__restrict__ bsoa, const ColPlan *__restrict__ plans,
                                                   int n, int l, int N, int S, int maxup,
                                                   uint32_t *__restrict__ tables, uint32_t *__restrict__ scr,
                                                   int skip_fast, const int *__restrict__ general) {
    if (skip_fast && general != nullptr && *general == 0) return;      // every column consecutive (k_plan's flag)
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = 2LL * n * l;
    if (t >= total) return;
    const int j = (int)(t % l);
    const int k = (int)((t / l) % n);
    const int c = (int)(t / ((int64_t)l * n));
    const int64_t cnt = (int64_t)n * l;
    pt P;
    soa_load(P, bsoa + (int64_t)c * kPtWords * cnt, cnt, (int64_t)k * l + j);
    const ColPlan &pl = plans[k];
    if (skip_fast && col_consecutive(pl, N)) return;                 // k_tables_fast
    if (pl.n[0] == 0) return;            // all-zero column: no table (k_affine writes its identity markers);
                                         // its tracking pointers were never written (found by the checked build)
    uint32_t *blk = tables + (((int64_t)c * n + k) * l + j) * (int64_t)(kPtWords * S);
    uint32_t *sj = scr + j;
    const int64_t sbase = ((int64_t)c * n + k) * 2 * maxup * kPtWords;   // in units of l-strided words
    const int n1 = pl.n[0];                  // slot 0 and slots > n1: identity markers written by k_affine
    if (N == 1) {
        for (int u = 0; u < n1; u++) {                                      // Alg. 3 line 5 only
            pt e;
            pt_mul_small_g<MulCall>(e, pl.sN[u], P);
            table_store(blk, u + 1, e);
        }
    } else {
        // level N (Alg. 3 line 5): buffer A = entries [0, 8), buffer B = [8, 16)
        int src = 0;
        const int nN = pl.n[N - 1];
        if (kSigned) {
            level_n_products_shared(pl.sN, nN, P, sj, sbase, l, src);
        } else {
            for (int u = 0; u < nN; u++) {
                pt e;
                pt_mul_small_g<MulCall>(e, pl.sN[u], P);
                scr_store(sj, sbase, src + u, l, e);
            }
        }
        for (int lev = N - 1; lev >= 2; lev--) {                            // prefix sums, levels N-1 .. 2
            const int dst = maxup - src;
            const int nl = pl.n[lev - 1];
            pt run, g;
            scr_load(run, sj, sbase, src + pl.ptr[lev - 1][0], l);
            scr_store(sj, sbase, dst, l, run);
            for (int u = 1; u < nl; u++) {
                scr_load(g, sj, sbase, src + pl.ptr[lev - 1][u], l);
                pt_add_pair(run, run, g);
                scr_store(sj, sbase, dst + u, l, run);
            }
            src = dst;
        }
        pt run, g;                                                          // level 1 -> the table
        scr_load(run, sj, sbase, src + pl.ptr[0][0], l);
        table_store(blk, 1, run);
        for (int u = 1; u < n1; u++) {
            scr_load(g, sj, sbase, src + pl.ptr[0][u], l);
            pt_add_pair(run, run, g);
            table_store(blk, u + 1, run);
        }
    }
}

// ------------------------------------------------------------ a2 + a3, few tables: one CTA per table
// As k_tables for launches with few (c, k, j) tables -- a plaintext vector times one
// or a few ciphertexts (Tables A7/A8) -- where one thread per table is a
// serial chain of up to 2^w - 2 complete additions: the level-N ECSMs run in
// parallel and each level's prefix sum (Alg. 2 l.14-23, any addition order: R7)
// is a block scan (runs of consecutive elements per thread, Hillis-Steele over
// the run totals in shared memory, then each run adds its exclusive prefix).
constexpr int kTScanT = 128;

__device__ __forceinline__ void tsm_store(uint32_t *sm, int i, const pt &q) {
    PCMM_DCHECK(i >= 0 && i < kTScanT);
#pragma unroll
    for (int w = 0; w < 8; w++) {
        sm[(0 * 8 + w) * kTScanT + i] = q.X.v[w];
        sm[(1 * 8 + w) * kTScanT + i] = q.Y.v[w];
        sm[(2 * 8 + w) * kTScanT + i] = q.Z.v[w];
    }
}

__device__ __forceinline__ void tsm_load(pt &q, const uint32_t *sm, int i) {
    PCMM_DCHECK(i >= 0 && i < kTScanT);
#pragma unroll
    for (int w = 0; w < 8; w++) {
        q.X.v[w] = sm[(0 * 8 + w) * kTScanT + i];
        q.Y.v[w] = sm[(1 * 8 + w) * kTScanT + i];
        q.Z.v[w] = sm[(2 * 8 + w) * kTScanT + i];
    }
}

__device__ __forceinline__ void table_load(pt &q, const uint32_t *block, int slot) {
    PCMM_DCHECK(slot >= 0 && slot < kPlanCap);
    const uint4 *d = reinterpret_cast<const uint4 *>(block + slot * kPtWords);
    const uint4 x0 = d[0], x1 = d[1], y0 = d[2], y1 = d[3], z0 = d[4], z1 = d[5];
    q.X = fe{{x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w}};
    q.Y = fe{{y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w}};
    q.Z = fe{{z0.x, z0.y, z0.z, z0.w, z1.x, z1.y, z1.z, z1.w}};
}

__global__ void __launch_bounds__(kTScanT) k_tables_scan(const uint32_t *__restrict__ bsoa,
                                                         const ColPlan *__restrict__ plans, int n, int l, int N, int S,
                                                         int maxup, uint32_t *__restrict__ tables,
                                                         uint32_t *__restrict__ scr) {
    __shared__ uint32_t sm[kPtWords * kTScanT];
    const int64_t t = blockIdx.x;                                       // table (c, k, j), j fastest
    const int tid = (int)threadIdx.x;
    PCMM_DCHECK(blockDim.x == kTScanT && t < 2LL * n * l);
    const int j = (int)(t % l);
    const int k = (int)((t / l) % n);
    const int c = (int)(t / ((int64_t)l * n));
    const int64_t cnt = (int64_t)n * l;
    pt P;
    soa_load(P, bsoa + (int64_t)c * kPtWords * cnt, cnt, (int64_t)k * l + j);
    const ColPlan &pl = plans[k];
    uint32_t *blk = tables + t * (int64_t)(kPtWords * S);
    uint32_t *sj = scr + j;
    const int64_t sbase = ((int64_t)c * n + k) * 2 * maxup * kPtWords;
    pt id;
    pt_identity(id);
    const int n1 = pl.n[0];
    if (tid == 0) table_store(blk, 0, id);
    for (int slot = n1 + 1 + tid; slot < S; slot += kTScanT) table_store(blk, slot, id);
    if (N == 1) {
        for (int u = tid; u < n1; u += kTScanT) {
            pt e;
            pt_mul_small_g<MulCall>(e, pl.sN[u], P);                       // Alg. 3 l.5
            table_store(blk, u + 1, e);
        }
        return;
    }
    int src = 0;
    for (int u = tid; u < pl.n[N - 1]; u += kTScanT) {
        pt e;
        pt_mul_small_g<MulCall>(e, pl.sN[u], P);                           // Alg. 3 l.5 (v < 0: -(|v| P))
        scr_store(sj, sbase, src + u, l, e);
    }
    __syncthreads();
    for (int lev = N - 1; lev >= 1; lev--) {                                // levels N-1 .. 1
        const int nlv = pl.n[lev - 1];
        const uint8_t *pp = pl.ptr[lev - 1];
        const int dst = maxup - src;
        const int E = (nlv + kTScanT - 1) / kTScanT;
        const int u0 = min(tid * E, nlv), u1 = min(u0 + E, nlv);
        pt run = id, g;
        for (int u = u0; u < u1; u++) {                                    // own run, inclusive
            PCMM_DCHECK(src + pp[u] < 2 * maxup && dst + u < 2 * maxup + kPlanCap);
            scr_load(g, sj, sbase, src + pp[u], l);
            pt_add_nl(run, run, g);
            if (lev == 1) table_store(blk, u + 1, run);
            else scr_store(sj, sbase, dst + u, l, run);
        }
        tsm_store(sm, tid, run);
        __syncthreads();
        for (int d = 1; d < kTScanT; d <<= 1) {                            // Hillis-Steele over run totals
            pt o;
            if (tid >= d) tsm_load(o, sm, tid - d);
            __syncthreads();
            if (tid >= d) {
                pt_add_nl(run, run, o);
                tsm_store(sm, tid, run);
            }
            __syncthreads();
        }
        if (tid > 0) {
            pt excl;
            tsm_load(excl, sm, tid - 1);
            for (int u = u0; u < u1; u++) {                                // + exclusive prefix
                pt v;
                if (lev == 1) table_load(v, blk, u + 1);
                else scr_load(v, sj, sbase, dst + u, l);
                pt_add_nl(v, excl, v);
                if (lev == 1) table_store(blk, u + 1, v);
                else scr_store(sj, sbase, dst + u, l, v);
            }
        }
        __syncthreads();
        src = dst;
    }
}

// ------------------------------------------------------------ a2 + a3 for consecutive columns
// When s^(1)_k = {1, ..., n1} (every unsigned w <= 4 column of a dense random A),
// Alg. 2 gives s^(2) = ... = s^(N) = {1}: no ECSM (x1 is free, Alg. 3 line 5) and
// the level-1 reconstruction is the prefix sum T[u] = T[u-1] + P with the
// ciphertext component P itself as every addend (Alg. 2 lines 14-23).  P is
// affine (k_import: Z = 1), so each step is an XYZZ mixed addition (8M + 2S,
// jac.cuh) instead of a complete projective addition (12M + 2m_b), and T[2] = 2P
// an affine-input doubling (4M + 3S).  The XYZZ entries go to k_affine (6M + 1S
// per entry there, against 5M for a homogeneous one).  Other columns: k_tables.

__device__ __forceinline__ void st_fe2(uint32_t *d, const fe &a, const fe &b) {
    uint4 *q = reinterpret_cast<uint4 *>(d);
    q[0] = make_uint4(a.v[0], a.v[1], a.v[2], a.v[3]);
    q[1] = make_uint4(a.v[4], a.v[5], a.v[6], a.v[7]);
    q[2] = make_uint4(b.v[0], b.v[1], b.v[2], b.v[3]);
    q[3] = make_uint4(b.v[4], b.v[5], b.v[6], b.v[7]);
}

__device__ __forceinline__ void ld_fe2(fe &a, fe &b, const uint32_t *d) {
    const uint4 *q = reinterpret_cast<const uint4 *>(d);
    const uint4 a0 = q[0], a1 = q[1], b0 = q[2], b1 = q[3];
    a = fe{{a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w}};
    b = fe{{b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w}};
}


// ------------------------------------------------------------ a2 + a3 for 2^w >= 128 slots: XYZZ level 1
// As k_tables (levels N .. 2 identical, projective), then the level-2 entries --
// the only addends of the level-1 prefix sum (Alg. 2 l.14-23), a handful of small
// multiples v P -- are made affine with one batch inversion shared by the warp
// (lane products of their Z, prefix / suffix products by shuffles, one fe_inv of
// the warp total run by all lanes), and the level-1 prefix sum, up to 2^w - 2
// additions, runs as XYZZ mixed additions (8M + 2S instead of 12M + 2m_b).  Its
// entries are converted to homogeneous coordinates (3M) for k_affine.
template <bool kSigned>
__global__ void __launch_bounds__(128, PCMM_TABLES_MINB)
    k_tables_x(const uint32_t *__restrict__ bsoa, const ColPlan *__restrict__ plans, int n, int l, int N, int S,
               int maxup, uint32_t *__restrict__ tables, uint32_t *__restrict__ scr, int skip_fast) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = (int)(threadIdx.x & 31);
    const int64_t total = 2LL * n * l;
    bool valid = t < total;
    const int64_t tt = valid ? t : total - 1;
    const int j = (int)(tt % l);
    const int k = (int)((tt / l) % n);
    const int c = (int)(tt / ((int64_t)l * n));
    const int64_t cnt = (int64_t)n * l;
    const ColPlan &pl = plans[k];
    if (skip_fast && col_consecutive(pl, N)) valid = false;          // k_tables_fast
    if (pl.n[0] == 0) valid = false;                                   // all-zero column (pointers unset)
    uint32_t *sj = scr + j;
    const int64_t sbase = ((int64_t)c * n + k) * 2 * maxup * kPtWords;
    int src = 0, n2 = 0;
    if (valid) {
        pt P;
        soa_load(P, bsoa + (int64_t)c * kPtWords * cnt, cnt, (int64_t)k * l + j);
        const int nN = pl.n[N - 1];
        if (kSigned) {
            level_n_products_shared(pl.sN, nN, P, sj, sbase, l, src);
        } else {
            for (int u = 0; u < nN; u++) {
                pt e;
                pt_mul_small_g<MulCall>(e, pl.sN[u], P);
                scr_store(sj, sbase, src + u, l, e);
            }
        }
        for (int lev = N - 1; lev >= 2; lev--) {                        // prefix sums, levels N-1 .. 2
            const int dst = maxup - src;
            const int nl = pl.n[lev - 1];
            pt run, g;
            scr_load(run, sj, sbase, src + pl.ptr[lev - 1][0], l);
            scr_store(sj, sbase, dst, l, run);
            for (int u = 1; u < nl; u++) {
                scr_load(g, sj, sbase, src + pl.ptr[lev - 1][u], l);
                pt_add_pair(run, run, g);
                scr_store(sj, sbase, dst + u, l, run);
            }
            src = dst;
        }
        n2 = pl.n[1];
    }
    // level-2 entries -> affine: prefix products parked in the Z words of the other buffer
    const int dst = maxup - src;
    auto zword = [&](int e, int q) -> uint32_t * { return sj + (sbase + (int64_t)e * kPtWords + 16 + q) * l; };
    fe one;
    fe_one_mont(one);
    fe acc = one;
    for (int u = 0; u < n2; u++) {
        fe z;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            z.v[q] = *zword(src + u, q);
            *zword(dst + u, q) = acc.v[q];
        }
        if (!fe_is_zero(z)) fe_mul(acc, acc, z);
    }
    fe Q = acc, Sx = acc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const fe q = fe_shfl_up(Q, d), sv = fe_shfl_down(Sx, d);
        fe qm, sm;
        fe_mul(qm, Q, q);
        fe_mul(sm, Sx, sv);
        if (lane >= d) Q = qm;
        if (lane + d < 32) Sx = sm;
    }
    fe tot, inv;
#pragma unroll
    for (int i = 0; i < 8; i++) tot.v[i] = __shfl_sync(0xffffffffu, Q.v[i], 31);
    fe qprev = fe_shfl_up(Q, 1), snext = fe_shfl_down(Sx, 1);
    if (lane == 0) qprev = one;
    if (lane == 31) snext = one;
    fe_inv(inv, tot);                                                   // one inversion per warp
    fe_mul(inv, inv, qprev);
    fe_mul(inv, inv, snext);                                            // 1 / (this lane's product)
    for (int u = n2 - 1; u >= 0; u--) {
        pt e;
        scr_load(e, sj, sbase, src + u, l);
        fe pre, x, y, zi;
#pragma unroll
        for (int q = 0; q < 8; q++) pre.v[q] = *zword(dst + u, q);
        uint32_t *ex = sj + (sbase + (int64_t)(dst + u) * kPtWords) * l;   // affine (x, y) in words 0..15
        if (fe_is_zero(e.Z)) {                                          // the identity (P = identity)
#pragma unroll
            for (int q = 0; q < 8; q++) {
                ex[q * l] = 0xffffffffu;
                ex[(8 + q) * l] = 0;
            }
            continue;
        }
        fe_mul(zi, inv, pre);
        fe_mul(inv, inv, e.Z);
        fe_mul(x, e.X, zi);
        fe_mul(y, e.Y, zi);
#pragma unroll
        for (int q = 0; q < 8; q++) {
            ex[q * l] = x.v[q];
            ex[(8 + q) * l] = y.v[q];
        }
    }
    if (!valid) return;
    // level 1: XYZZ prefix sum of the affine level-2 entries (gathered by tracking pointer), each
    // entry stored homogeneous (X ZZZ : Y ZZ : ZZ ZZZ) for k_affine (the affine slots overlap other
    // tables' upper-level scratch while this kernel runs, so nothing is parked there)
    const int n1 = pl.n[0];
    uint32_t *blk = tables + (((int64_t)c * n + k) * l + j) * (int64_t)(kPtWords * S);
    xyzz run;
    xyzz_init(run);
    for (int u = 0; u < n1; u++) {
        const uint32_t *ex = sj + (sbase + (int64_t)(dst + pl.ptr[0][u]) * kPtWords) * l;
        fe x, y;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            x.v[q] = ex[q * l];
            y.v[q] = ex[(8 + q) * l];
        }
        xyzz_add_aff(run, x, y);
        pt h;
        xyzz_to_proj(h, run);                                           // the identity: Z = 0
        table_store(blk, u + 1, h);
    }
}

#ifndef PCMM_TFAST_MINB
#define PCMM_TFAST_MINB 3
#endif
__global__ void __launch_bounds__(128, PCMM_TFAST_MINB)
    k_tables_fast(const uint32_t *__restrict__ bsoa, const ColPlan *__restrict__ plans, int n, int l, int N, int S,
                  uint32_t *__restrict__ tables, uint32_t *__restrict__ atab) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = 2LL * n * l;
    if (t >= total) return;
    const int j = (int)(t % l);
    const int k = (int)((t / l) % n);
    const int c = (int)(t / ((int64_t)l * n));
    const ColPlan &pl = plans[k];
    if (!col_consecutive(pl, N)) return;                              // k_tables + k_affine
    const int64_t cnt = (int64_t)n * l;
    pt P;
    soa_load(P, bsoa + (int64_t)c * kPtWords * cnt, cnt, (int64_t)k * l + j);
    const int64_t tb = ((int64_t)c * n + k) * l + j;
    uint32_t *blk = tables + tb * (int64_t)(kPtWords * S);
    uint32_t *ablk = atab + tb * (int64_t)(kAffWords * S);
    const int n1 = pl.n[0];
    fe zero;
    fe_zero(zero);
    st_aff_inf(ablk);                                                 // slot 0 = the identity
    for (int u = n1 + 1; u < S; u++) st_aff_inf(ablk + u * kAffWords);
    if (pt_is_identity(P)) {                                          // every multiple is the identity
        st_aff_inf(ablk + kAffWords);
        for (int u = 2; u <= n1; u++) {
#if PCMM_TFAST_PROJ
            pt id;
            pt_identity(id);
            table_store(blk, u, id);
#else
            st_fe2(ablk + u * kAffWords, zero, zero);                 // ZZZ = 0: k_affine -> identity
#endif
        }
        return;
    }
    st_fe2(ablk + kAffWords, P.X, P.Y);                               // T[1] = P (Z = 1)
    xyzz run;
    for (int u = 2; u <= n1; u++) {
        if (u == 2) xyzz_dbl_aff(run, P.X, P.Y);
        else xyzz_add_aff(run, P.X, P.Y);
        if (run.inf) {                                                // only off the curve
#if PCMM_TFAST_PROJ
            pt id;
            pt_identity(id);
            table_store(blk, u, id);
#else
            st_fe2(ablk + u * kAffWords, zero, zero);
#endif
            continue;
        }
        uint32_t *e = blk + u * kPtWords;
#if PCMM_TFAST_PROJ
        pt h;
        xyzz_to_proj(h, run);
        table_store(blk, u, h);
#else
        st_fe2(e, run.X, run.Y);
        uint4 *z = reinterpret_cast<uint4 *>(e + 16);
        z[0] = make_uint4(run.ZZ.v[0], run.ZZ.v[1], run.ZZ.v[2], run.ZZ.v[3]);
        z[1] = make_uint4(run.ZZ.v[4], run.ZZ.v[5], run.ZZ.v[6], run.ZZ.v[7]);
        st_fe2(ablk + u * kAffWords, run.ZZZ, zero);                  // ZZZ parked in the affine slot
#endif
    }
}

// ------------------------------------------------------------ a5: split-k reduce
__global__ void k_reduce(const uint32_t *__restrict__ partial, int ksplit, int64_t count, uint32_t *__restrict__ out,
                         int accumulate) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * count) return;
    const int c = (int)(t / count);
    const int64_t e = t % count;
    const int64_t split_stride = 2LL * kPtWords * count;
    pt acc, q;
    soa_load(acc, partial + (int64_t)c * kPtWords * count, count, e);
    for (int s = 1; s < ksplit; s++) {
        soa_load(q, partial + s * split_stride + (int64_t)c * kPtWords * count, count, e);
        pt_add_nl(acc, acc, q);
    }
    if (accumulate) {                                      // the running output of earlier k-chunks
        soa_load(q, out + (int64_t)c * kPtWords * count, count, e);
        pt_add_nl(acc, acc, q);
    }
    soa_store(out + (int64_t)c * kPtWords * count, count, e, acc);
}

// ------------------------------------------------------------ s1: schoolbook
// lanes <-> output columns j (coalesced loads of Enc(b_kj)), warp <-> row i, so
// a_ik is warp-uniform and the double-and-add control flow never diverges.
__global__ void __launch_bounds__(128) k_school(const int8_t *__restrict__ A, int m, int n, int l, int w,
                                               int is_signed, const uint32_t *__restrict__ bsoa,
                                               uint32_t *__restrict__ out, int *__restrict__ status) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int jblocks = (l + 31) / 32, rblocks = (m + 3) / 4;            // 1-D grid: (c, row block, j block)
    int64_t bb = blockIdx.x;
    const int jb = (int)(bb % jblocks);
    bb /= jblocks;
    const int c = (int)(bb / rblocks);
    const int i = (int)(bb % rblocks) * 4 + warp;
    if (i >= m) return;
    const int j = jb * 32 + lane;
    const int jj = min(j, l - 1);
    const int lo = is_signed ? -(1 << (w - 1)) : 0;
    const int hi = is_signed ? (1 << (w - 1)) - 1 : (1 << w) - 1;
    const int64_t cnt = (int64_t)n * l;
    const uint32_t *bc = bsoa + (int64_t)c * kPtWords * cnt;
    pt acc, P, T;
    pt_identity(acc);
    bool bad = false;
    for (int k = 0; k < n; k++) {
        int v = is_signed ? (int)A[(int64_t)i * n + k] : (int)(uint8_t)A[(int64_t)i * n + k];
        if (v < lo || v > hi) { bad = true; v = 0; }
        if (v == 0) continue;                                  // 0 * ct = (inf, inf), warp-uniform
        soa_load(P, bc, cnt, (int64_t)k * l + jj);
        pt_mul_small_pair(T, v, P);                           // one ECSM per term
        pt_add_pair(acc, acc, T);
    }
    if (bad && lane == 0) atomicOr(status, kStatusBound);
    if (j < l) {
        const int64_t oc = (int64_t)m * l;
        soa_store(out + (int64_t)c * kPtWords * oc, oc, (int64_t)i * l + j, acc);
    }
}

// ------------------------------------------------------------ a6: normalise
// Montgomery batch inversion over kBatch points per thread (3 fe_mul per point
// + one inversion per batch); Z = 0 (infinity) is replaced by 1 in the batch.
constexpr int kBatch = 8;

__global__ void __launch_bounds__(128) k_normalize(const uint32_t *__restrict__ proj, int64_t count,
                                                   uint8_t *__restrict__ ct) {
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = 2 * count;
    fe pre[kBatch];
    fe one;
    fe_one_mont(one);
    fe acc = one;
    int nb = 0;
#pragma unroll
    for (int r = 0; r < kBatch; r++) {
        const int64_t p = t + r * nthreads;
        if (p < total) {
            const int c = (int)(p / count);
            const int64_t e = p % count;
            fe z;
#pragma unroll
            for (int q = 0; q < 8; q++) z.v[q] = proj[(int64_t)c * kPtWords * count + (2 * 8 + q) * count + e];
            if (fe_is_zero(z)) z = one;
            fe_mul(acc, acc, z);
            nb = r + 1;
        }
        pre[r] = acc;
    }
    if (nb == 0) return;
    fe inv;
    fe_inv(inv, pre[nb - 1]);
#pragma unroll
    for (int r = kBatch - 1; r >= 0; r--) {
        if (r >= nb) continue;
        const int64_t p = t + r * nthreads;
        const int c = (int)(p / count);
        const int64_t e = p % count;
        pt P;
        soa_load(P, proj + (int64_t)c * kPtWords * count, count, e);
        fe zi;
        if (r > 0) fe_mul(zi, inv, pre[r - 1]);
        else zi = inv;
        const bool isinf = fe_is_zero(P.Z);
        if (r > 0) fe_mul(inv, inv, isinf ? one : P.Z);
        uint8_t *dst = ct + e * 128 + c * 64;
        if (isinf) {
            uint32_t wz[16] = {0};
            store64(dst, wz);
        } else {
            fe x, y;
            fe_mul(x, P.X, zi);
            fe_mul(y, P.Y, zi);
            store_canonical_xy(dst, x, y);
        }
    }
}

// ------------------------------------------------------------ boundary kernels
struct Pk64 {
    uint8_t b[64];
};

__global__ void k_encrypt(const __grid_constant__ Pk64 pk, const int32_t *__restrict__ bvals, const uint8_t *__restrict__ r, int64_t count,
                          uint8_t *__restrict__ ct) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= count) return;
    pt G, H, C1, C2, bG;
    generator_mont(G);
    uint8_t pkb[64];
#pragma unroll
    for (int i = 0; i < 64; i++) pkb[i] = pk.b[i];
    pt_from_canonical(H, pkb);
    uint32_t k[8];
    be32_to_words(r + e * 32, k);
    pt_mul_scalar_win(C1, k, G);              // r G
    pt_mul_scalar_win(C2, k, H);              // r H
    pt_mul_small(bG, bvals[e], G);            // phi(b) = b G
    pt_add_nl(C2, C2, bG);
    store_canonical_point(ct + e * 128, C1);
    store_canonical_point(ct + e * 128 + 64, C2);
}

__global__ void k_pubkey(const uint32_t x0, const uint32_t x1, const uint32_t x2, const uint32_t x3,
                         const uint32_t x4, const uint32_t x5, const uint32_t x6, const uint32_t x7,
                         uint8_t *__restrict__ out) {
    uint32_t k[8] = {x0, x1, x2, x3, x4, x5, x6, x7};
    pt G, H;
    generator_mont(G);
    pt_mul_scalar(H, k, G);
    store_canonical_point(out, H);
}


// ------------------------------------------------------------ test hooks
// x + p without reduction (x < 2^256 - p): the non-canonical representative of x
__device__ __forceinline__ void fe_add_portable_nored(fe &r, const fe &x) {
    uint64_t c = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const uint64_t t = (uint64_t)x.v[i] + p_limb(i) + c;
        r.v[i] = (uint32_t)t;
        c = t >> 32;
    }
}

__global__ void k_test_field(int op, const uint8_t *__restrict__ a, const uint8_t *__restrict__ b,
                             uint8_t *__restrict__ out, int64_t count) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= count) return;
    fe x, y, r;
    fe_from_be_bytes(x, a + e * 32);
    fe_from_be_bytes(y, b + e * 32);
    fe_to_mont(x, x);
    fe_to_mont(y, y);
    switch (op) {
        case 0: fe_add(r, x, y); break;
        case 1: fe_sub(r, x, y); break;
        case 2: fe_mul(r, x, y); break;
        case 3: fe_inv(r, x); break;
#ifdef __CUDA_ARCH__
        case 5: fe_sqr_fast(r, x); break;
        case 6: fe_mul_fast_v<1 - PCMM_MUL_PRODUCT>(r, x, y); break;
        case 7: fe_inv_fermat(r, x); break;
        // lazy (almost-reduced) arithmetic: inputs whose Montgomery form is odd and below 2^256 - p are
        // denormalised to form + p (in [p, 2^256)) first; outputs fully reduced by fe_from_mont below
        case 8: case 9: case 10: case 11: case 12: {
            fe xd = x, yd = y;
            if (x.v[7] == 0 && x.v[6] < 0xfffffffeu && (x.v[0] & 1u)) fe_add_portable_nored(xd, x);   // odd forms
            if (y.v[7] == 0 && y.v[6] < 0xfffffffeu && (y.v[0] & 1u)) fe_add_portable_nored(yd, y);
            if (op == 8) fe_mul_lz(r, xd, yd);
            else if (op == 9) fe_sqr_lz(r, xd);
            else if (op == 10) fe_add_lz(r, xd, yd);
            else if (op == 11) fe_sub_lz(r, xd, yd);
            else {
                fe_zero(r);
                r.v[0] = fe_is_zero_lz(xd) ? 1u : 2u;
                fe_to_be_bytes(out + e * 32, r);              // raw flag, not a field element
                return;
            }
            break;
        }
#endif
        default: fe_neg(r, x); break;
    }
    fe_from_mont(r, r);
    fe_to_be_bytes(out + e * 32, r);
}

__global__ void k_test_point(int op, const uint8_t *__restrict__ p, const uint8_t *__restrict__ q,
                             const int32_t *__restrict__ v, uint8_t *__restrict__ out, int64_t count) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= count) return;
    pt P, Q, R;
    load_canonical_point(P, p + e * 64);
    if (op == 0) {
        load_canonical_point(Q, q + e * 64);
        pt_add_nl(R, P, Q);
    } else if (op == 1) {
        pt_dbl_nl(R, P);
    } else if (op == 2) {
        pt_mul_small(R, v[e], P);
    } else if (op == 3) {
        uint32_t k[8];
        be32_to_words(q + e * 64, k);
        pt_mul_scalar_win(R, k, P);           // 4-bit windows, Jacobian (the decrypt / encrypt ECSM)
    } else {
        uint32_t k[8];
        be32_to_words(q + e * 64, k);
        pt_mul_scalar(R, k, P);               // binary double-and-add, complete formulas
    }
    store_canonical_point(out + e * 64, R);
}

// ------------------------------------------------------------ launchers
static inline unsigned blocks_for(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

cudaError_t launch_import(const uint8_t *ct, int64_t count, uint32_t *soa, int *status, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    k_import<<<blocks_for(2 * count, 128), 128, 0, s>>>(ct, count, soa, status);
    return cudaGetLastError();
}

cudaError_t launch_plan(const int8_t *A, int m, int n, int w, int is_signed, int N, ColPlan *plans, uint8_t *rank,
                        int *status, cudaStream_t s) {
    k_plan<<<blocks_for((int64_t)n * 32, 128), 128, 0, s>>>(A, m, n, w, is_signed, N, plans, rank, status);
    return cudaGetLastError();
}


static int tables_fast_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("PCMM_TABLES_FAST");
        v = e ? atoi(e) : 1;
    }
    return v;
}

cudaError_t launch_tables(const uint32_t *bsoa, const ColPlan *plans, int n, int l, int N, int slots, int maxup,
                          int is_signed, uint32_t *tables, uint32_t *scratch, cudaStream_t s, int fast, int maxlen,
                          const int *general) {
    // few tables (fewer than two per SM) of >= 16 entries (maxlen = min(m, 2^w - 1)): one CTA per
    // table with block-scan prefix sums (measured: at 8-15 entries the serial thread is faster)
    static int scan_env = -1;                                 // PCMM_TABLES_SCAN: 0 never, 1 auto, 2 always
    if (scan_env < 0) {
        const char *e = getenv("PCMM_TABLES_SCAN");
        scan_env = e ? atoi(e) : 1;
    }
    if (!fast && (scan_env == 2 || (scan_env == 1 && maxlen >= 16 && 2LL * n * l <= 2LL * num_sms()))) {
        k_tables_scan<<<(unsigned)(2LL * n * l), kTScanT, 0, s>>>(bsoa, plans, n, l, N, slots, maxup, tables, scratch);
        return cudaGetLastError();
    }
    static int x_env = -1;                                    // PCMM_TABLES_XYZZ: 0 off, 1 for 2^w >= 128 slots
    if (x_env < 0) {
        const char *e = getenv("PCMM_TABLES_XYZZ");
        x_env = e ? atoi(e) : 1;
    }
    if (x_env && (slots >= 128 || x_env == 2) && N >= 2) {    // w = 8, 256^3: 4.49 -> 4.31 ms; w = 6: 3 % slower
        if (is_signed)
            k_tables_x<true><<<blocks_for(2LL * n * l, 128), 128, 0, s>>>(bsoa, plans, n, l, N, slots, maxup, tables,
                                                                          scratch, fast);
        else
            k_tables_x<false><<<blocks_for(2LL * n * l, 128), 128, 0, s>>>(bsoa, plans, n, l, N, slots, maxup, tables,
                                                                           scratch, fast);
        return cudaGetLastError();
    }
    if (is_signed)
        k_tables<true><<<blocks_for(2LL * n * l, 128), 128, 0, s>>>(bsoa, plans, n, l, N, slots, maxup, tables, scratch,
                                                                    fast, general);
    else
        k_tables<false><<<blocks_for(2LL * n * l, 128), 128, 0, s>>>(bsoa, plans, n, l, N, slots, maxup, tables,
                                                                     scratch, fast, general);
    return cudaGetLastError();
}

int tables_fast_on() { return tables_fast_enabled(); }

int tables_coz_mode() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("PCMM_TABLES_COZ");
        v = e ? atoi(e) : 1;
    }
    return v;
}

cudaError_t launch_tables_fast(const uint32_t *bsoa, const ColPlan *plans, int n, int l, int N, int slots,
                               uint32_t *tables, uint32_t *atables, cudaStream_t s) {
    k_tables_fast<<<blocks_for(2LL * n * l, 128), 128, 0, s>>>(bsoa, plans, n, l, N, slots, tables, atables);
    return cudaGetLastError();
}

cudaError_t launch_reduce_splits(const uint32_t *partial, int ksplit, int64_t count, uint32_t *out, cudaStream_t s,
                                 bool accumulate) {
    k_reduce<<<blocks_for(2 * count, 128), 128, 0, s>>>(partial, ksplit, count, out, accumulate ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_schoolbook(const int8_t *A, int m, int n, int l, int w, int is_signed, const uint32_t *bsoa,
                              uint32_t *out, int *status, cudaStream_t s) {
    // PCMM_SCHOOL_XYZZ=1: the XYZZ schoolbook (school.cu; fewer products, measured slower)
    static int xz = -1;
    if (xz < 0) {
        const char *e = getenv("PCMM_SCHOOL_XYZZ");
        xz = e ? atoi(e) : 0;
    }
    if (xz) return launch_schoolbook_xyzz(A, m, n, l, w, is_signed, bsoa, out, status, s);
    const int64_t blocks = (int64_t)((l + 31) / 32) * ((m + 3) / 4) * 2;
    k_school<<<(unsigned)blocks, 128, 0, s>>>(A, m, n, l, w, is_signed, bsoa, out, status);
    return cudaGetLastError();
}

cudaError_t launch_normalize(const uint32_t *proj, int64_t count, uint8_t *ct, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    // points per thread: up to kBatch (one inversion per batch), fewer when that would
    // leave fewer than ~8 warps per SM (small outputs: the inversion latency is the cost)
    const int64_t batch = std::min<int64_t>(kBatch, std::max<int64_t>(1, 2 * count / ((int64_t)num_sms() * 256)));
    const int64_t threads = (2 * count + batch - 1) / batch;
    k_normalize<<<blocks_for(threads, 128), 128, 0, s>>>(proj, count, ct);
    return cudaGetLastError();
}

cudaError_t launch_encrypt(const uint8_t *pk64, const int32_t *b, const uint8_t *r, int64_t count, uint8_t *ct,
                           cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    Pk64 pk;
    for (int i = 0; i < 64; i++) pk.b[i] = pk64[i];
    k_encrypt<<<blocks_for(count, 64), 64, 0, s>>>(pk, b, r, count, ct);
    return cudaGetLastError();
}

cudaError_t launch_pubkey(const uint32_t x[8], uint8_t *out64_d, cudaStream_t s) {
    k_pubkey<<<1, 1, 0, s>>>(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7], out64_d);
    return cudaGetLastError();
}


cudaError_t launch_test_field(int op, const uint8_t *a, const uint8_t *b, uint8_t *out, int64_t count,
                              cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    k_test_field<<<blocks_for(count, 128), 128, 0, s>>>(op, a, b, out, count);
    return cudaGetLastError();
}

cudaError_t launch_test_point(int op, const uint8_t *p, const uint8_t *q, const int32_t *v, uint8_t *out,
                              int64_t count, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    k_test_point<<<blocks_for(count, 64), 64, 0, s>>>(op, p, q, v, out, count);
    return cudaGetLastError();
}

}  // namespace pcmm
