// taff.cu -- steps a2 + a3 + a3' of the Cussen path for consecutive columns in
// one kernel (k_tables_coz): the table entries are computed and converted to
// the affine (x, y) that k_accum reads, with no intermediate table in HBM.
//
// A column whose level-1 set is s^(1) = {1, ..., n1} (every column of the
// unsigned BASELINE configs at m >= 64) has levels 2..N = {1}: Alg. 2's
// reconstruction (Alg. 3 l.5-6) is the prefix sum
// T[u] = T[u-1] + 1 P of the ciphertext component P itself (T[1] = P).  The
// chain runs in co-Z Jacobian coordinates (Meloni 2007; Goundar-Joye-Miyaji
// 2011): every T[u] shares its Z with the running copy of P, so one step
// (ZADDU: T[u+1] = P + T[u] and P re-expressed on the new Z) costs 5M + 2S
// instead of the XYZZ mixed addition's 8M + 2S, and Z_{u+1} = Z_u lambda_u with
// lambda_u = X_P - X_T[u].  The step starts from the co-Z doubling of the affine
// P (DBLU, 2M + 4S).  Because the Z of every entry is a prefix product of the
// lambdas, one inversion of the last Z per table gives all of them backwards
// (1/Z_{u-1} = lambda_{u-1} / Z_u); the tables of a CTA share that inversion
// (Montgomery's trick across lanes, shared.cuh cta_inverse).  Per entry 9M + 3S
// (the step, 1/Z_u, x = X/Z^2, y = Y/Z^3) against 9.1 + 7.6 fp_mul-eq for the
// XYZZ chain plus k_affine's conversion, and one kernel instead of two: (X, Y,
// lambda) of each entry are parked in the (otherwise unused) projective slot of
// the table region and read back by the same thread.
//
// Exceptional cases: ZADDU with X_P = X_T needs T[u] = +-P, i.e. u = +-1 mod q,
// impossible for u >= 2; the doubling needs y != 0 (P-256 has no point of order
// 2).  An identity component makes every entry the identity (handled up
// front).  The result is the same group elements as Alg. 2's prefix sum (the
// additions are exactly T[u] + P in order; only the coordinates differ).
#include <algorithm>

#include "canon.cuh"
#include "ec.cuh"
#include "internal.h"
#include "shared.cuh"

namespace pcmm {

namespace {

__device__ __forceinline__ void ld_x(fe &x, const uint32_t *d) {
    const uint4 *q = reinterpret_cast<const uint4 *>(d);
    const uint4 a = q[0], b = q[1];
    x = fe{{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w}};
}

__device__ __forceinline__ void ld_xy(fe &x, fe &y, const uint32_t *d) {
    const uint4 *q = reinterpret_cast<const uint4 *>(d);
    const uint4 a = q[0], b = q[1], c = q[2], e = q[3];
    x = fe{{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w}};
    y = fe{{c.x, c.y, c.z, c.w, e.x, e.y, e.z, e.w}};
}

__device__ __forceinline__ void st_x(uint32_t *d, const fe &a) {
    uint4 *q = reinterpret_cast<uint4 *>(d);
    q[0] = make_uint4(a.v[0], a.v[1], a.v[2], a.v[3]);
    q[1] = make_uint4(a.v[4], a.v[5], a.v[6], a.v[7]);
}

__device__ __forceinline__ void st_xy(uint32_t *d, const fe &x, const fe &y) {
    st_x(d, x);
    st_x(d + 8, y);
}

// 1 / a for every lane of the warp with one field inversion (all 32 lanes active): inclusive prefix (Q)
// and suffix (S) products by shuffles, the inverse of the warp total (every lane runs it on the same
// value), then 1/a = inv(total) Q(lane - 1) S(lane + 1).  No block barrier, unlike cta_inverse.
__device__ __forceinline__ fe warp_inverse(const fe &a, const fe &one) {
    const int lane = (int)(threadIdx.x & 31);
    fe Q = a, S = a;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const fe q = fe_shfl_up(Q, d), sv = fe_shfl_down(S, d);
        fe qm, sm;
        fe_mul(qm, Q, q);
        fe_mul(sm, S, sv);
        if (lane >= d) Q = qm;
        if (lane + d < 32) S = sm;
    }
    fe tot;
#pragma unroll
    for (int i = 0; i < 8; i++) tot.v[i] = __shfl_sync(0xffffffffu, Q.v[i], 31);
    fe ti;
    fe_inv(ti, tot);
    fe qprev = fe_shfl_up(Q, 1), snext = fe_shfl_down(S, 1);
    if (lane == 0) qprev = one;
    if (lane == 31) snext = one;
    fe r;
    fe_mul(r, ti, qprev);
    fe_mul(r, r, snext);
    return r;
}

}  // namespace

#ifndef PCMM_TCOZ_WARPINV
#define PCMM_TCOZ_WARPINV 0     // 1: one inversion per warp (no block barrier) instead of per CTA
#endif
#ifndef PCMM_TCOZ_DISCARD
#define PCMM_TCOZ_DISCARD 1     // discard.global.L2 the parked entries after the backward pass
#endif
#ifndef PCMM_TCOZ_MINB
#define PCMM_TCOZ_MINB 4
#endif
#ifndef PCMM_TCOZ_PREFETCH
#define PCMM_TCOZ_PREFETCH 1    // 1 (default; 256^3 tables 0.406 -> 0.376 ms): backward pass loads the next parked entry before the current entry's products
#endif

// Slot of the value v of column pl (1 + the number of level-1 values below v), or -1 if v does not
// occur.  Unsigned chain columns: the values are {1..coz}, slot v = v.
__device__ __forceinline__ int coz_slot(const ColPlan &pl, int v) {
    if (!pl.sgn) return v;
    const int b = v + 128;
    if (!((pl.bm1[b >> 5] >> (b & 31)) & 1u)) return -1;
    int r = 0;
    for (int q = 0; q < (b >> 5); q++) r += __popc(pl.bm1[q]);
    return 1 + r + __popc(pl.bm1[b >> 5] & ((1u << (b & 31)) - 1u));
}

// (x, y) -> the slots of +u and -u ((x, -y): DESIGN.md R10b) that the column has
__device__ __forceinline__ void coz_store(const ColPlan &pl, uint32_t *ablk, int u, const fe &x, const fe &y, int S) {
    const int sp = coz_slot(pl, u);
    PCMM_DCHECK(sp < S);
    if (sp >= 1) st_xy(ablk + sp * kAffWords, x, y);
    if (pl.sgn) {
        const int sn = coz_slot(pl, -u);
        PCMM_DCHECK(sn < S);
        if (sn >= 1) {
            fe zero, ny;
            fe_zero(zero);
            fe_sub(ny, zero, y);
            st_xy(ablk + sn * kAffWords, x, ny);
        }
    }
}

// Builds the chain of one table (c, k, j) and returns whether it has entries
// to convert (chain length >= 2, component not the identity), with the Z of its
// last entry.  Writes the affine slots 0, +-1 and the unused ones and parks
// (X, Y, lambda) of the multiples 2..n1 in projective slots 2..n1.  (Running
// the two components' chains in lockstep in one thread halves the thread count
// and measured slower: 256^3 0.47 vs 0.39 ms.)
__device__ __forceinline__ bool coz_chain(const uint32_t *__restrict__ bsoa, const ColPlan *__restrict__ plans,
                                          int n, int l, int N, int S, uint32_t *__restrict__ ptab,
                                          uint32_t *__restrict__ atab, int64_t t, const fe &one, fe &Zf) {
    const int j = (int)(t % l);
    const int k = (int)((t / l) % n);
    const int c = (int)(t / ((int64_t)l * n));
    const ColPlan &pl = plans[k];
    if (!col_consecutive(pl, N)) return false;
    const int n1 = pl.coz;                                              // chain length (multiples 1..n1)
    const int used = pl.n[0];                                           // slots 1..used hold entries
    PCMM_DCHECK(n1 < S && used < S && t < 2LL * n * l);
    uint32_t *ablk = atab + t * (int64_t)(kAffWords * S);              // table index (c n + k) l + j = t
    uint32_t *pblk = ptab + t * (int64_t)(kPtWords * S);
    st_aff_inf(ablk);                                                   // slot 0 = the identity
    for (int u = used + 1; u < S; u++) st_aff_inf(ablk + u * kAffWords);
    const int64_t cnt = (int64_t)n * l;
    pt P;
    soa_load(P, bsoa + (int64_t)c * kPtWords * cnt, cnt, (int64_t)k * l + j);
    if (pt_is_identity(P)) {                                            // every multiple is the identity
        for (int u = 1; u <= used; u++) st_aff_inf(ablk + u * kAffWords);
        return false;
    }
    coz_store(pl, ablk, 1, P.X, P.Y, S);                                // T[+-1] = +-P (Z = 1 after k_import)
    if (n1 < 2) return false;
    // DBLU: 2P on Z = 2y, and P on the same Z: (4 x y^2, 8 y^4)
    fe B, E, L, Sx, M, X2, Y2, t0;
    fe_sqr(E, P.Y);
    fe_sqr(B, P.X);
    fe_sqr(L, E);
    fe_mul(Sx, P.X, E);
    fe_add(Sx, Sx, Sx);
    fe_add(Sx, Sx, Sx);                                                 // S = 4 x y^2
    fe_sub(M, B, one);
    fe_add(t0, M, M);
    fe_add(M, t0, M);                                                   // M = 3 x^2 + a, a = -3
    fe_add(L, L, L);
    fe_add(L, L, L);
    fe_add(L, L, L);                                                    // 8 y^4
    fe_sqr(X2, M);
    fe_add(t0, Sx, Sx);
    fe_sub(X2, X2, t0);                                                 // X = M^2 - 2S
    fe_sub(t0, Sx, X2);
    fe_mul(Y2, M, t0);
    fe_sub(Y2, Y2, L);                                                  // Y = M (S - X) - 8 y^4
    fe Z;
    fe_add(Z, P.Y, P.Y);                                                // Z = 2y
    st_xy(pblk + 2 * kPtWords, X2, Y2);
    fe PX = Sx, PY = L, TX = X2, TY = Y2;
    for (int u = 2; u < n1; u++) {
        // ZADDU: T[u+1] = P + T[u] on Z' = Z lambda, P re-expressed on Z'
        fe lam, C, W1, W2, dy, D, A1, X3, Y3, e;
        fe_sub(lam, PX, TX);
        fe_sqr(C, lam);
        fe_mul(W1, PX, C);
        fe_mul(W2, TX, C);
        fe_sub(dy, PY, TY);
        fe_sqr(D, dy);
        fe_sub(e, W1, W2);
        fe_mul(A1, PY, e);                                              // Y_P' = Y_P lambda^3
        fe_sub(X3, D, W1);
        fe_sub(X3, X3, W2);                                             // X3 = D - W1 - W2
        fe_sub(e, W1, X3);
        fe_mul(Y3, dy, e);
        fe_sub(Y3, Y3, A1);                                             // Y3 = (Y_P - Y_T)(W1 - X3) - A1
        fe_mul(Z, Z, lam);
        uint32_t *q = pblk + (u + 1) * kPtWords;
        st_xy(q, X3, Y3);
        st_x(q + 16, lam);                                              // Z_{u+1} = Z_u lambda
        PX = W1;
        PY = A1;
        TX = X3;
        TY = Y3;
    }
    Zf = Z;
    return true;
}

// One thread per `batch` tables (t, t + T, ...; T = grid size, so a warp takes
// consecutive j and shares k), one inversion per CTA for all of them: the
// thread's product of last-entry Zs goes through cta_inverse, the per-table
// prefix and Z are parked in the table's (unused) projective slot 0.  No thread
// returns before cta_inverse (barriers).
__global__ void __launch_bounds__(128, PCMM_TCOZ_MINB)
    k_tables_coz(const uint32_t *__restrict__ bsoa, const ColPlan *__restrict__ plans, int n, int l, int N, int S,
                 int batch, uint32_t *__restrict__ ptab, uint32_t *__restrict__ atab) {
    __shared__ fe wtot[4], winv[4];
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = 2LL * n * l;
    fe one;
    fe_one_mont(one);
    fe acc = one;
    uint32_t live = 0;                                                  // bit g: table g has entries to convert
    PCMM_DCHECK(batch <= 32);
    for (int g = 0; g < batch; g++) {
        const int64_t t = t0 + g * T;
        if (t >= total) break;
        fe Zf;
        if (coz_chain(bsoa, plans, n, l, N, S, ptab, atab, t, one, Zf)) {
            st_xy(ptab + t * (int64_t)(kPtWords * S), acc, Zf);
            fe_mul(acc, acc, Zf);
            live |= 1u << g;
        }
    }
#if PCMM_TCOZ_WARPINV
    fe inv = warp_inverse(acc, one);                                    // 1 / (product of this thread's Zs)
#else
    fe inv = cta_inverse<false>(acc, wtot, winv);                       // 1 / (product of this thread's Zs)
#endif
    for (int g = batch - 1; g >= 0; g--) {
        if (!((live >> g) & 1u)) continue;
        const int64_t t = t0 + g * T;
        const ColPlan &pl = plans[(int)((t / l) % n)];
        const int n1 = pl.coz;
        uint32_t *pblk = ptab + t * (int64_t)(kPtWords * S);
        uint32_t *ablk = atab + t * (int64_t)(kAffWords * S);
        fe pre, Zf, zinv;
        ld_xy(pre, Zf, pblk);
        fe_mul(zinv, inv, pre);                                         // 1 / Z_{n1}
        fe_mul(inv, inv, Zf);
        // backward: x = X / Z^2, y = Y / Z^3, then 1 / Z_{u-1} = lambda_{u-1} / Z_u
#if PCMM_TCOZ_PREFETCH
        // the next entry's parked (X, Y, lambda) are loaded before this entry's products (the loads'
        // L2 / HBM latency overlaps the arithmetic instead of stalling the chain)
        fe X, Y, lam = one;
        ld_xy(X, Y, pblk + n1 * kPtWords);
        if (n1 >= 3) ld_x(lam, pblk + n1 * kPtWords + 16);
        for (int u = n1; u >= 2; u--) {
            fe Xn, Yn, lamn;
            if (u >= 3) {
                const uint32_t *qn = pblk + (u - 1) * kPtWords;
                ld_xy(Xn, Yn, qn);
                ld_x(lamn, qn + 16);
            }
            fe zi2, zi3, x, y;
            fe_sqr(zi2, zinv);
            fe_mul(x, X, zi2);
            fe_mul(zi3, zi2, zinv);
            fe_mul(y, Y, zi3);
            coz_store(pl, ablk, u, x, y, S);
            if (u >= 3) {
                fe_mul(zinv, zinv, lam);
                X = Xn;
                Y = Yn;
                lam = lamn;
            }
        }
#else
        for (int u = n1; u >= 2; u--) {
            const uint32_t *q = pblk + u * kPtWords;
            fe X, Y, zi2, zi3, x, y;
            ld_xy(X, Y, q);
            fe_sqr(zi2, zinv);
            fe_mul(x, X, zi2);
            fe_mul(zi3, zi2, zinv);
            fe_mul(y, Y, zi3);
            coz_store(pl, ablk, u, x, y, S);
            if (u >= 3) {
                fe lam;
                ld_x(lam, q + 16);
                fe_mul(zinv, zinv, lam);
            }
        }
#endif
#if PCMM_TCOZ_DISCARD
        // the parked (X, Y, lambda) and (prefix, Z) are dead: drop their L2 lines without writing them back
        if ((S * kPtWords * 4) % 128 == 0) {
            const char *base = reinterpret_cast<const char *>(pblk);
            for (int o = 0; o < S * kPtWords * 4; o += 128)
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(base + o) : "memory");
        }
#endif
    }
}

cudaError_t launch_tables_coz(const uint32_t *bsoa, const ColPlan *plans, int n, int l, int N, int slots,
                              uint32_t *tables, uint32_t *atables, cudaStream_t s) {
    const int64_t total = 2LL * n * l;
    // tables per thread: enough to fill one wave of resident CTAs (one inversion per CTA), at most 16
    static int occ = 0;
    if (!occ) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tables_coz, 128, 0) != cudaSuccess || occ <= 0)
            occ = 4;
    }
    static int batch_env = -1;
    if (batch_env < 0) {
        const char *e = getenv("PCMM_TCOZ_BATCH");
        batch_env = e ? atoi(e) : 0;
    }
    const int64_t wave = (int64_t)num_sms() * occ * 128;
    const int batch = batch_env > 0 ? batch_env : (int)std::min<int64_t>(16, std::max<int64_t>(1, (total + wave - 1) / wave));
    const int64_t threads = (total + batch - 1) / batch;
    k_tables_coz<<<(unsigned)((threads + 127) / 128), 128, 0, s>>>(bsoa, plans, n, l, N, slots, batch, tables,
                                                                     atables);
    return cudaGetLastError();
}

}  // namespace pcmm
