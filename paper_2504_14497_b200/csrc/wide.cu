// wide.cu -- the wide-plaintext Cussen path (the paper's
// t = 12, 16 grid, Table A9): plaintexts up to 16 bits as int32, a column
// may hold up to min(m, 2^t - 1) distinct nonzero values, so the plan arrays,
// the rank (uint16) and the tables (up to m + 1 slots per (k, j, c)) are sized
// per problem and the tables are built and consumed in chunks of KC inner
// indices k (api.cu).  The steps are those of the byte path (kernels.cu k_plan,
// k_tables; hot.cu k_accum_g): Alg. 2 l.3-12 / Alg. 3 l.3 compression
// (P:344-355), Alg. 3 l.5 ECSMs, l.6 prefix sums and
// l.7-9 accumulation, with readings R1, R3, R6, R7, R10.
#include <limits.h>

#include "ec.cuh"
#include "internal.h"

namespace pcmm {

namespace {

__device__ __forceinline__ void w_soa_load(pt &P, const uint32_t *base, int64_t stride, int64_t idx) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
        P.X.v[i] = base[(0 * 8 + i) * stride + idx];
        P.Y.v[i] = base[(1 * 8 + i) * stride + idx];
        P.Z.v[i] = base[(2 * 8 + i) * stride + idx];
    }
}

__device__ __forceinline__ void w_soa_store(uint32_t *base, int64_t stride, int64_t idx, const pt &P) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
        base[(0 * 8 + i) * stride + idx] = P.X.v[i];
        base[(1 * 8 + i) * stride + idx] = P.Y.v[i];
        base[(2 * 8 + i) * stride + idx] = P.Z.v[i];
    }
}

// Bitonic sort of s[0..P) (P a power of two) by the whole CTA, ascending.
__device__ void cta_sort(int32_t *s, int P) {
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            __syncthreads();
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const int32_t a = s[i], b = s[ixj];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) {
                        s[i] = b;
                        s[ixj] = a;
                    }
                }
            }
        }
    }
    __syncthreads();
}

// first index e in [0, len) with L[e] >= v (L ascending)
__device__ __forceinline__ int lower_bound_i32(const int32_t *L, int len, int32_t v) {
    int lo = 0, hi = len;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (L[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__host__ __device__ inline int pow2_at_least(int x) {
    int p = 2;
    while (p < x) p <<= 1;
    return p;
}

// ------------------------------------------------------------ a1 (wide): one CTA per column k
// Level 1 = sorted distinct nonzero values of A[:,k] (R1); rank[k][i] = 1 + index
// of a_ik in level 1 (0 for a_ik = 0); level w+1 = sorted distinct values of the
// differenced level w (first element kept, R6) with ptr[w-1][e] = index of
// element e of the differenced level w in level w+1 (R3); level N values -> sN.
// Shared memory: sb[P2] (sort buffer), L[cap] (current level), V[cap] (its differences).
__global__ void __launch_bounds__(256) k_plan_wide(const int32_t *__restrict__ A, int m, int n, int w,
                                                   int is_signed, int N, int cap, int P2,
                                                   int32_t *__restrict__ pn, int32_t *__restrict__ psN,
                                                   uint16_t *__restrict__ pptr, uint16_t *__restrict__ rank,
                                                   int *__restrict__ status) {
    extern __shared__ int32_t wsm[];
    int32_t *sb = wsm, *L = wsm + P2, *V = L + cap;
    __shared__ int ns_sh;
    const int k = blockIdx.x;
    const int lo = is_signed ? -(1 << (w - 1)) : 0;
    const int hi = is_signed ? (1 << (w - 1)) - 1 : (1 << w) - 1;
    bool bad = false;
    for (int i = threadIdx.x; i < P2; i += blockDim.x) {
        int32_t v = INT_MAX;
        if (i < m) {
            const int32_t a = A[(int64_t)i * n + k];
            if (a < lo || a > hi) bad = true;
            else if (a != 0) v = a;
        }
        sb[i] = v;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status, kStatusBound);
    cta_sort(sb, P2);
    if (threadIdx.x == 0) {                                          // de-duplicate -> level 1
        int ns = 0;
        for (int i = 0; i < P2 && sb[i] != INT_MAX; i++)
            if (ns == 0 || sb[i] != L[ns - 1]) L[ns++] = sb[i];
        ns_sh = ns;
    }
    __syncthreads();
    int ns = ns_sh;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const int32_t a = A[(int64_t)i * n + k];
        uint16_t r = 0;
        if (a != 0 && a >= lo && a <= hi) r = (uint16_t)(1 + lower_bound_i32(L, ns, a));
        rank[(int64_t)k * m + i] = r;
    }
    for (int lev = 1; lev <= N; lev++) {
        if (threadIdx.x == 0) pn[(int64_t)k * 4 + lev - 1] = ns;
        if (lev == N) {
            for (int e = threadIdx.x; e < ns; e += blockDim.x) psN[(int64_t)k * cap + e] = L[e];
            break;
        }
        // differences of consecutive elements, first kept (Alg. 2 l.6-10); nonzero (distinct values)
        for (int e = threadIdx.x; e < ns; e += blockDim.x) V[e] = e == 0 ? L[0] : L[e] - L[e - 1];
        const int P = pow2_at_least(ns);
        __syncthreads();
        for (int e = threadIdx.x; e < P; e += blockDim.x) sb[e] = e < ns ? V[e] : INT_MAX;
        cta_sort(sb, P);
        if (threadIdx.x == 0) {
            int u = 0;
            for (int e = 0; e < P && sb[e] != INT_MAX; e++)
                if (u == 0 || sb[e] != L[u - 1]) L[u++] = sb[e];
            ns_sh = u;
        }
        __syncthreads();
        const int nn = ns_sh;
        for (int e = threadIdx.x; e < ns; e += blockDim.x)           // R3 tracking pointers
            pptr[((int64_t)k * 3 + (lev - 1)) * cap + e] = (uint16_t)lower_bound_i32(L, nn, V[e]);
        __syncthreads();
        ns = nn;
    }
}

// ------------------------------------------------------------ a2 + a3 (wide): tables of one k-chunk
// Thread per (c, kk, j), j fastest; k = k0 + kk.  Same reconstruction as
// kernels.cu k_tables (levels N-1..2 in a j-innermost global scratch of 2 x cap
// entries per (c, kk, j), level 1 straight to the table); S = cap + 1 slots.
__device__ __forceinline__ void wt_store(uint32_t *block, int slot, const pt &q) {
    uint4 *d = reinterpret_cast<uint4 *>(block + (int64_t)slot * kPtWords);
    d[0] = make_uint4(q.X.v[0], q.X.v[1], q.X.v[2], q.X.v[3]);
    d[1] = make_uint4(q.X.v[4], q.X.v[5], q.X.v[6], q.X.v[7]);
    d[2] = make_uint4(q.Y.v[0], q.Y.v[1], q.Y.v[2], q.Y.v[3]);
    d[3] = make_uint4(q.Y.v[4], q.Y.v[5], q.Y.v[6], q.Y.v[7]);
    d[4] = make_uint4(q.Z.v[0], q.Z.v[1], q.Z.v[2], q.Z.v[3]);
    d[5] = make_uint4(q.Z.v[4], q.Z.v[5], q.Z.v[6], q.Z.v[7]);
}

__device__ __forceinline__ void ws_store(uint32_t *scr, int64_t base, int e, int64_t l, const pt &q) {
    uint32_t *d = scr + (base + (int64_t)e * kPtWords) * l;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        d[(0 * 8 + i) * l] = q.X.v[i];
        d[(1 * 8 + i) * l] = q.Y.v[i];
        d[(2 * 8 + i) * l] = q.Z.v[i];
    }
}

__device__ __forceinline__ void ws_load(pt &q, const uint32_t *scr, int64_t base, int e, int64_t l) {
    const uint32_t *d = scr + (base + (int64_t)e * kPtWords) * l;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        q.X.v[i] = d[(0 * 8 + i) * l];
        q.Y.v[i] = d[(1 * 8 + i) * l];
        q.Z.v[i] = d[(2 * 8 + i) * l];
    }
}

#ifndef PCMM_WIDE_SHARED_DBL
#define PCMM_WIDE_SHARED_DBL 1      // level-N ECSMs of k_tables_wide with shared doublings (0: one binary ECSM per value)
#endif
constexpr bool kWideSharedDbl = PCMM_WIDE_SHARED_DBL != 0;

__global__ void __launch_bounds__(128, 3) k_tables_wide(const uint32_t *__restrict__ bsoa,
                                                        const int32_t *__restrict__ pn,
                                                        const int32_t *__restrict__ psN,
                                                        const uint16_t *__restrict__ pptr, int n, int l, int N,
                                                        int cap, int S, int k0, int kc,
                                                        uint32_t *__restrict__ tables, uint32_t *__restrict__ scr) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2LL * kc * l) return;
    const int j = (int)(t % l);
    const int kk = (int)((t / l) % kc);
    const int c = (int)(t / ((int64_t)l * kc));
    const int k = k0 + kk;
    const int64_t cnt = (int64_t)n * l;
    pt P;
    w_soa_load(P, bsoa + (int64_t)c * kPtWords * cnt, cnt, (int64_t)k * l + j);
    const int32_t *nl = pn + (int64_t)k * 4;
    const int32_t *sN = psN + (int64_t)k * cap;
    const uint16_t *ptr = pptr + (int64_t)k * 3 * cap;
    uint32_t *blk = tables + (((int64_t)c * kc + kk) * l + j) * (int64_t)S * kPtWords;
    uint32_t *sj = scr + j;
    const int64_t sbase = ((int64_t)c * kc + kk) * 2 * cap * kPtWords;
    pt id;
    pt_identity(id);
    wt_store(blk, 0, id);
    const int n1 = nl[0];
    if (n1 == 0) return;                 // all-zero column: its tracking pointers were never written
    if (N == 1) {
        for (int u = 0; u < n1; u++) {
            pt e;
            pt_mul_small_g<MulCall>(e, sN[u], P);                           // Alg. 3 l.5
            wt_store(blk, u + 1, e);
        }
    } else {
        int src = 0;
        const int nN = nl[N - 1];
        // Alg. 3 l.5: the level-N ECSMs s^(N)[u] P all multiply the same point, so the doublings are
        // shared: D[i] = 2^i P once (nb - 1 doublings), then v P = the sum of the D[i] of v's set bits
        // (popcount - 1 complete additions instead of nb - 1 doublings + popcount - 1 additions per value;
        // t = 16, 256 rows: ~250 values per column, 24 -> 8 point operations each)
        unsigned maxmag = 0;
        for (int u = 0; u < nN; u++) {
            const int v = sN[u];
            maxmag = max(maxmag, v < 0 ? (unsigned)(-v) : (unsigned)v);
        }
        int nb = 0;
        while (nb < 32 && (maxmag >> nb)) nb++;
        constexpr int kMaxBits = 20;
        if (kWideSharedDbl && nN >= 3 && nb <= kMaxBits) {
            pt D[kMaxBits];
            D[0] = P;
            for (int i = 1; i < nb; i++) pt_dbl_pair(D[i], D[i - 1]);
            for (int u = 0; u < nN; u++) {
                const int v = sN[u];
                unsigned a = v < 0 ? (unsigned)(-v) : (unsigned)v;
                pt e;
                pt_identity(e);
                bool first = true;
                for (int i = 0; i < nb; i++) {
                    if ((a >> i) & 1u) {
                        if (first) e = D[i];
                        else pt_add_pair(e, e, D[i]);
                        first = false;
                    }
                }
                if (v < 0) pt_neg(e, e);
                ws_store(sj, sbase, src + u, l, e);
            }
        } else {
            for (int u = 0; u < nN; u++) {
                pt e;
                pt_mul_small_g<MulCall>(e, sN[u], P);                       // Alg. 3 l.5
                ws_store(sj, sbase, src + u, l, e);
            }
        }
        for (int lev = N - 1; lev >= 2; lev--) {                            // prefix sums, levels N-1 .. 2
            const int dst = cap - src;
            const int nlv = nl[lev - 1];
            const uint16_t *pl = ptr + (int64_t)(lev - 1) * cap;
            pt run, g;
            ws_load(run, sj, sbase, src + pl[0], l);
            ws_store(sj, sbase, dst, l, run);
            for (int u = 1; u < nlv; u++) {
                ws_load(g, sj, sbase, src + pl[u], l);
                pt_add_pair(run, run, g);
                ws_store(sj, sbase, dst + u, l, run);
            }
            src = dst;
        }
        pt run, g;                                                          // level 1 -> the table
        ws_load(run, sj, sbase, src + ptr[0], l);
        wt_store(blk, 1, run);
        for (int u = 1; u < n1; u++) {
            ws_load(g, sj, sbase, src + ptr[u], l);
            pt_add_pair(run, run, g);
            wt_store(blk, u + 1, run);
        }
    }
    for (int slot = n1 + 1; slot < S; slot++) wt_store(blk, slot, id);
}

// ------------------------------------------------------------ a2 + a3 (wide), few tables: one CTA per table
// For launches with few tables (a single plaintext vector times one or a few
// ciphertexts, Tables A7/A8 P:886-949) the one-thread-per-table kernel above is a
// serial chain of up to cap complete additions per level.  Here a CTA builds one
// table: the level-N ECSMs in parallel, and each level's prefix sum
// b^(w)[u] = sum_{v <= u} b^(w+1)[ptr^(w)[v]] (Alg. 2 l.14-23, any addition order:
// R7) as a block scan: every thread sums its run of consecutive elements, a
// Hillis-Steele scan over the run totals in shared memory, then each run adds its
// exclusive prefix -- latency ~ 2 cap / T + log2 T additions instead of cap.
constexpr int kScanT = 128;

__device__ __forceinline__ void wt_load(pt &q, const uint32_t *block, int slot) {
    const uint4 *d = reinterpret_cast<const uint4 *>(block + (int64_t)slot * kPtWords);
    const uint4 x0 = d[0], x1 = d[1], y0 = d[2], y1 = d[3], z0 = d[4], z1 = d[5];
    q.X = fe{{x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w}};
    q.Y = fe{{y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w}};
    q.Z = fe{{z0.x, z0.y, z0.z, z0.w, z1.x, z1.y, z1.z, z1.w}};
}

__device__ __forceinline__ void sm_store(uint32_t *sm, int i, const pt &q) {
#pragma unroll
    for (int w = 0; w < 8; w++) {
        sm[(0 * 8 + w) * kScanT + i] = q.X.v[w];
        sm[(1 * 8 + w) * kScanT + i] = q.Y.v[w];
        sm[(2 * 8 + w) * kScanT + i] = q.Z.v[w];
    }
}

__device__ __forceinline__ void sm_load(pt &q, const uint32_t *sm, int i) {
#pragma unroll
    for (int w = 0; w < 8; w++) {
        q.X.v[w] = sm[(0 * 8 + w) * kScanT + i];
        q.Y.v[w] = sm[(1 * 8 + w) * kScanT + i];
        q.Z.v[w] = sm[(2 * 8 + w) * kScanT + i];
    }
}

__global__ void __launch_bounds__(kScanT) k_tables_wide_scan(const uint32_t *__restrict__ bsoa,
                                                             const int32_t *__restrict__ pn,
                                                             const int32_t *__restrict__ psN,
                                                             const uint16_t *__restrict__ pptr, int n, int l, int N,
                                                             int cap, int S, int k0, int kc,
                                                             uint32_t *__restrict__ tables,
                                                             uint32_t *__restrict__ scr) {
    __shared__ uint32_t sm[kPtWords * kScanT];
    const int64_t t = blockIdx.x;                                       // table (c, kk, j), j fastest
    const int tid = (int)threadIdx.x;
    const int j = (int)(t % l);
    const int kk = (int)((t / l) % kc);
    const int c = (int)(t / ((int64_t)l * kc));
    const int k = k0 + kk;
    const int64_t cnt = (int64_t)n * l;
    pt P;
    w_soa_load(P, bsoa + (int64_t)c * kPtWords * cnt, cnt, (int64_t)k * l + j);
    const int32_t *nl = pn + (int64_t)k * 4;
    const int32_t *sN = psN + (int64_t)k * cap;
    const uint16_t *ptr = pptr + (int64_t)k * 3 * cap;
    uint32_t *blk = tables + t * (int64_t)S * kPtWords;
    uint32_t *sj = scr + j;
    const int64_t sbase = ((int64_t)c * kc + kk) * 2 * cap * kPtWords;
    pt id;
    pt_identity(id);
    const int n1 = nl[0];
    if (tid == 0) wt_store(blk, 0, id);
    for (int slot = n1 + 1 + tid; slot < S; slot += kScanT) wt_store(blk, slot, id);
    if (N == 1) {
        for (int u = tid; u < n1; u += kScanT) {
            pt e;
            pt_mul_small_g<MulCall>(e, sN[u], P);                           // Alg. 3 l.5
            wt_store(blk, u + 1, e);
        }
        return;
    }
    int src = 0;
    for (int u = tid; u < nl[N - 1]; u += kScanT) {
        pt e;
        pt_mul_small_g<MulCall>(e, sN[u], P);                               // Alg. 3 l.5
        ws_store(sj, sbase, src + u, l, e);
    }
    __syncthreads();
    for (int lev = N - 1; lev >= 1; lev--) {                                // levels N-1 .. 1
        const int nlv = nl[lev - 1];
        const uint16_t *pl = ptr + (int64_t)(lev - 1) * cap;
        const int dst = cap - src;
        const int E = (nlv + kScanT - 1) / kScanT;
        const int u0 = min(tid * E, nlv), u1 = min(u0 + E, nlv);
        pt run = id, g;
        for (int u = u0; u < u1; u++) {                                    // own run, inclusive
            ws_load(g, sj, sbase, src + pl[u], l);
            pt_add_nl(run, run, g);
            if (lev == 1) wt_store(blk, u + 1, run);
            else ws_store(sj, sbase, dst + u, l, run);
        }
        sm_store(sm, tid, run);
        __syncthreads();
        for (int d = 1; d < kScanT; d <<= 1) {                             // Hillis-Steele over run totals
            pt o;
            if (tid >= d) sm_load(o, sm, tid - d);
            __syncthreads();
            if (tid >= d) {
                pt_add_nl(run, run, o);
                sm_store(sm, tid, run);
            }
            __syncthreads();
        }
        pt excl = id;
        if (tid > 0) sm_load(excl, sm, tid - 1);
        if (tid > 0) {
            for (int u = u0; u < u1; u++) {                                // + exclusive prefix
                pt v;
                if (lev == 1) wt_load(v, blk, u + 1);
                else ws_load(v, sj, sbase, dst + u, l);
                pt_add_nl(v, excl, v);
                if (lev == 1) wt_store(blk, u + 1, v);
                else ws_store(sj, sbase, dst + u, l, v);
            }
        }
        __syncthreads();
        src = dst;
    }
}

// ------------------------------------------------------------ s1 (wide): schoolbook with int32 plaintexts
__global__ void __launch_bounds__(128) k_school_wide(const int32_t *__restrict__ A, int m, int n, int l, int w,
                                                     int is_signed, const uint32_t *__restrict__ bsoa,
                                                     uint32_t *__restrict__ out, int *__restrict__ status) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int jb = blockIdx.x, c = blockIdx.z;
    const int i = blockIdx.y * 4 + warp;
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
        int v = A[(int64_t)i * n + k];
        if (v < lo || v > hi) { bad = true; v = 0; }
        if (v == 0) continue;                                  // 0 * ct = (inf, inf), warp-uniform
        w_soa_load(P, bc, cnt, (int64_t)k * l + jj);
        pt_mul_small_pair(T, v, P);                           // one ECSM per term
        pt_add_pair(acc, acc, T);
    }
    if (bad && lane == 0) atomicOr(status, kStatusBound);
    if (j < l) {
        const int64_t oc = (int64_t)m * l;
        w_soa_store(out + (int64_t)c * kPtWords * oc, oc, (int64_t)i * l + j, acc);
    }
}

inline unsigned wblocks(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

}  // namespace

int wide_plan_p2(int m) { return pow2_at_least(m < 2 ? 2 : m); }

size_t wide_plan_smem(int m, int cap) { return (size_t)(wide_plan_p2(m) + 2 * cap) * sizeof(int32_t); }

cudaError_t launch_plan_wide(const int32_t *A, int m, int n, int w, int is_signed, int N, int cap, int32_t *pn,
                             int32_t *psN, uint16_t *pptr, uint16_t *rank, int *status, cudaStream_t s) {
    const size_t smem = wide_plan_smem(m, cap);
    cudaError_t e = cudaFuncSetAttribute(k_plan_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
    k_plan_wide<<<n, 256, smem, s>>>(A, m, n, w, is_signed, N, cap, wide_plan_p2(m), pn, psN, pptr, rank, status);
    return cudaGetLastError();
}

cudaError_t launch_tables_wide(const uint32_t *bsoa, const int32_t *pn, const int32_t *psN, const uint16_t *pptr,
                               int n, int l, int N, int cap, int S, int k0, int kc, uint32_t *tables,
                               uint32_t *scratch, cudaStream_t s) {
    k_tables_wide<<<wblocks(2LL * kc * l, 128), 128, 0, s>>>(bsoa, pn, psN, pptr, n, l, N, cap, S, k0, kc, tables,
                                                            scratch);
    return cudaGetLastError();
}

cudaError_t launch_tables_wide_scan(const uint32_t *bsoa, const int32_t *pn, const int32_t *psN,
                                    const uint16_t *pptr, int n, int l, int N, int cap, int S, int k0, int kc,
                                    uint32_t *tables, uint32_t *scratch, cudaStream_t s) {
    k_tables_wide_scan<<<(unsigned)(2LL * kc * l), kScanT, 0, s>>>(bsoa, pn, psN, pptr, n, l, N, cap, S, k0, kc,
                                                                   tables, scratch);
    return cudaGetLastError();
}

cudaError_t launch_schoolbook_wide(const int32_t *A, int m, int n, int l, int w, int is_signed,
                                   const uint32_t *bsoa, uint32_t *out, int *status, cudaStream_t s) {
    dim3 grid((unsigned)((l + 31) / 32), (unsigned)((m + 3) / 4), 2);
    k_school_wide<<<grid, 128, 0, s>>>(A, m, n, l, w, is_signed, bsoa, out, status);
    return cudaGetLastError();
}

}  // namespace pcmm
