// tgz.cu -- steps a2 + a3 + a3' of the Cussen path for GENERAL columns in one kernel
// (k_tables_gz): Alg. 2's reconstruction in its own order (Alg. 3 l.5-6,
// P:440-441) with the level-1 prefix sum in XYZZ coordinates and the conversion to the affine
// (x, y) that k_accum reads fused in, instead of k_tables (complete homogeneous additions, 14
// fp_mul per entry) followed by k_affine (7.6 per entry).
//
//   1. level N: the small ECSMs s^(N)[u] P (Alg. 3 l.5), levels N-1 .. 2: prefix sums by tracking
//      pointer, complete additions (a handful of entries; thread-local arrays);
//   2. the level-2 entries -- the only addends of the level-1 prefix sum -- are made affine with
//      one inversion per CTA (Montgomery's trick over the thread's entries, shared.cuh cta_inverse);
//   3. level 1: T[u] = T[u-1] + D[ptr[u]] as XYZZ + affine mixed additions (madd-2008-s, 8M + 2S).
//      ZZ_u = ZZ_{u-1} f_u and ZZZ_u = ZZZ_{u-1} g_u with (f, g) = (PP, PPP) of the step, so the
//      inverses of every entry's ZZ and ZZZ follow backwards from those of the last entry:
//      (X, Y, f) are parked in the entry's projective slot and g in its affine slot;
//   4. one more inversion per CTA (the last ZZZ of every thread), then backwards per entry
//      x = X / ZZ, y = Y / ZZZ (2M) and the two running inverses times f, g (2M).
// Per entry 12M + 2S against 21.6 fp_mul-equivalents, one kernel instead of two, no homogeneous
// table round trip.
//
// Exceptional cases of the mixed addition inside one table (all entries are multiples v P of one
// point of prime order q, 0 < |v| < q): the sum is never the identity (that would be the value 0,
// which R1 drops from every level), the accumulator is never the identity after the first entry,
// and T[u-1] = D[ptr[u]] (e.g. s^(1) = {1, 2, ..}: T[2] = P + P) is the doubling, done with
// dbl-2008-s-1 (ZZ3 = V ZZ, ZZZ3 = W ZZZ: the same product structure, (f, g) = (V, W)).  An
// identity ciphertext component makes every entry the identity marker.
#include <algorithm>

#include "canon.cuh"
#include "ec.cuh"
#include "internal.h"
#include "shared.cuh"

namespace pcmm {

namespace {

__device__ __forceinline__ void gz_ld_x(fe &x, const uint32_t *d) {
    const uint4 *q = reinterpret_cast<const uint4 *>(d);
    const uint4 a = q[0], b = q[1];
    x = fe{{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w}};
}

__device__ __forceinline__ void gz_st_x(uint32_t *d, const fe &a) {
    uint4 *q = reinterpret_cast<uint4 *>(d);
    q[0] = make_uint4(a.v[0], a.v[1], a.v[2], a.v[3]);
    q[1] = make_uint4(a.v[4], a.v[5], a.v[6], a.v[7]);
}

#ifdef __CUDA_ARCH__
// (c^2, d^2) out of line (the chain step's code must stay within the instruction cache: with every
// product inlined the level-1 loop was ~60 KB of SASS and ran 4x slower)
__device__ __noinline__ fe2 gz_sqr2_call(const fe c, const fe d) {
    fe2 r;
    fe_sqr(r.x, c);
    fe_sqr(r.y, d);
    return r;
}

// XYZZ doubling (dbl-2008-s-1, a = -3) with the factors f = V, g = W of ZZ3 = V ZZ, ZZZ3 = W ZZZ
__device__ __noinline__ void gz_double(fe &X, fe &Y, const fe &ZZ, fe &f, fe &g) {
    fe U, Sv, M, X3, Y3, t0, t1;
    fe_add(U, Y, Y);
    f = fe_mul_call(U, U);                                    // V
    const fe2 ws = fe_mul2_call(U, f, X, f);                  // W, S = X V
    g = ws.x;
    Sv = ws.y;
    fe_sub(t0, X, ZZ);
    fe_add(t1, X, ZZ);
    M = fe_mul_call(t0, t1);
    fe_add(t0, M, M);
    fe_add(M, t0, M);                                         // M = 3 (X^2 - ZZ^2)
    X3 = fe_mul_call(M, M);
    fe_sub(X3, X3, Sv);
    fe_sub(X3, X3, Sv);
    fe_sub(t0, Sv, X3);
    const fe2 yy = fe_mul2_call(M, t0, g, Y);
    fe_sub(Y3, yy.x, yy.y);
    X = X3;
    Y = Y3;
}
#endif

}  // namespace

#ifndef PCMM_TGZ_MINB
#define PCMM_TGZ_MINB 3
#endif

// One thread per table (c, k, j), j fastest.  No thread returns before the two cta_inverse calls.
// skip_chain: chain columns (ColPlan::coz > 0) are left to k_tables_coz.
template <int MAXUP>
__global__ void __launch_bounds__(128, PCMM_TGZ_MINB)
    k_tables_gz(const uint32_t *__restrict__ bsoa, const ColPlan *__restrict__ plans, int n, int l, int N, int S,
                uint32_t *__restrict__ ptab, uint32_t *__restrict__ atab, int skip_chain,
                const int *__restrict__ general) {
#ifdef __CUDA_ARCH__
    __shared__ fe wtot[4], winv[4];
    if (skip_chain && general != nullptr && *general == 0) return;       // every column is a chain column (k_plan)
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = 2LL * n * l;
    bool valid = t < total;
    const int64_t tt = valid ? t : total - 1;
    const int j = (int)(tt % l);
    const int k = (int)((tt / l) % n);
    const int c = (int)(tt / ((int64_t)l * n));
    const ColPlan &pl = plans[k];
    if (skip_chain && col_consecutive(pl, N)) valid = false;
    uint32_t *ablk = atab + tt * (int64_t)(kAffWords * S);
    uint32_t *pblk = ptab + tt * (int64_t)(kPtWords * S);
    const int n1 = pl.n[0];
    PCMM_DCHECK(n1 < S && N >= 2);
    fe one;
    fe_one_mont(one);
    pt up[2 * MAXUP];                                   // levels N .. 2, two ping-pong halves
    fe dx[MAXUP], dy[MAXUP], pre[MAXUP];                // affine level-2 entries; prefix products of their Z
    int src = 0, n2 = 0;
    bool live = false;
    if (valid) {
        st_aff_inf(ablk);                               // slot 0 and the unused slots: the identity
        for (int u = n1 + 1; u < S; u++) st_aff_inf(ablk + u * kAffWords);
        if (n1 > 0) {
            const int64_t cnt = (int64_t)n * l;
            pt P;
            soa_load(P, bsoa + (int64_t)c * kPtWords * cnt, cnt, (int64_t)k * l + j);
            if (pt_is_identity(P)) {                    // every multiple is the identity
                for (int u = 1; u <= n1; u++) st_aff_inf(ablk + u * kAffWords);
            } else {
                live = true;
                const int nN = pl.n[N - 1];
                PCMM_DCHECK(nN <= MAXUP);
                for (int u = 0; u < nN; u++) pt_mul_small_g<MulCall>(up[u], pl.sN[u], P);    // Alg. 3 l.5
                for (int lev = N - 1; lev >= 2; lev--) {                                      // Alg. 2 l.14-23
                    const int dst = MAXUP - src;
                    const int nl = pl.n[lev - 1];
                    PCMM_DCHECK(nl <= MAXUP);
                    pt run = up[src + pl.ptr[lev - 1][0]];
                    up[dst] = run;
                    for (int u = 1; u < nl; u++) {
                        pt_add_pair(run, run, up[src + pl.ptr[lev - 1][u]]);
                        up[dst + u] = run;
                    }
                    src = dst;
                }
                n2 = pl.n[1];
            }
        }
    }
    // ---- level-2 entries -> affine (x = X / Z, y = Y / Z; Z != 0: v P is not the identity)
    fe acc = one;
    for (int u = 0; u < n2; u++) {
        pre[u] = acc;
        acc = fe_mul_call(acc, up[src + u].Z);
    }
    fe inv = cta_inverse<false>(acc, wtot, winv);
    for (int u = n2 - 1; u >= 0; u--) {
        const fe2 zi = fe_mul2_call(inv, pre[u], inv, up[src + u].Z);     // 1 / Z_u, the running inverse
        inv = zi.y;
        const fe2 xy = fe_mul2_call(up[src + u].X, zi.x, up[src + u].Y, zi.x);
        dx[u] = xy.x;
        dy[u] = xy.y;
    }
    // ---- level 1: XYZZ prefix sum, (X, Y, f) and g parked per entry
    fe X, Y, ZZ = one, ZZZ = one;
    if (live) {
        const int e0 = pl.ptr[0][0];
        X = dx[e0];
        Y = dy[e0];
        uint4 *q = reinterpret_cast<uint4 *>(ablk + kAffWords);           // T[s_1] = D[ptr_1]: affine already
        q[0] = make_uint4(X.v[0], X.v[1], X.v[2], X.v[3]);
        q[1] = make_uint4(X.v[4], X.v[5], X.v[6], X.v[7]);
        q[2] = make_uint4(Y.v[0], Y.v[1], Y.v[2], Y.v[3]);
        q[3] = make_uint4(Y.v[4], Y.v[5], Y.v[6], Y.v[7]);
        for (int u = 1; u < n1; u++) {
            const int e = pl.ptr[0][u];
            fe Pd, R, f, g;
            const fe2 us = fe_mul2_call(dx[e], ZZ, dy[e], ZZZ);           // U2, S2
            fe_sub(Pd, us.x, X);
            fe_sub(R, us.y, Y);
            if (fe_is_zero(Pd)) {
                gz_double(X, Y, ZZ, f, g);                                // T[u-1] = D[e]: doubling
                const fe2 zz = fe_mul2_call(ZZ, f, ZZZ, g);
                ZZ = zz.x;
                ZZZ = zz.y;
            } else {
                fe X3, Y3, t0;
                const fe2 sq = gz_sqr2_call(Pd, R);                       // PP, R^2
                f = sq.x;
                const fe3 m3 = fe_mul3_call(Pd, f, X, f, ZZ, f);          // PPP, Q = X PP, ZZ3
                g = m3.x;
                fe_sub(X3, sq.y, g);
                fe_sub(X3, X3, m3.y);
                fe_sub(X3, X3, m3.y);                                     // X3 = R^2 - PPP - 2Q
                fe_sub(t0, m3.y, X3);
                const fe3 n3 = fe_mul3_call(R, t0, Y, g, ZZZ, g);         // R (Q - X3), Y PPP, ZZZ3
                fe_sub(Y3, n3.x, n3.y);
                X = X3;
                Y = Y3;
                ZZ = m3.z;
                ZZZ = n3.z;
            }
            uint32_t *pq = pblk + (u + 1) * kPtWords;
            gz_st_x(pq, X);
            gz_st_x(pq + 8, Y);
            gz_st_x(pq + 16, f);
            gz_st_x(ablk + (u + 1) * kAffWords, g);
        }
    }
    // ---- one inversion per CTA of every thread's last ZZZ, then backwards
    const bool chain = live && n1 >= 2;
    fe izzz = cta_inverse<false>(chain ? ZZZ : one, wtot, winv);
    if (chain) {
        fe iz, izz;
        iz = fe_mul_call(ZZ, izzz);                                       // ZZ / ZZZ = 1 / Z
        izz = fe_mul_call(iz, iz);                                        // 1 / ZZ
        for (int u = n1 - 1; u >= 1; u--) {
            const uint32_t *pq = pblk + (u + 1) * kPtWords;
            uint32_t *aq = ablk + (u + 1) * kAffWords;
            fe Xu, Yu, f, g, x, y;
            gz_ld_x(Xu, pq);
            gz_ld_x(Yu, pq + 8);
            gz_ld_x(f, pq + 16);
            gz_ld_x(g, aq);
            const fe2 xy = fe_mul2_call(Xu, izz, Yu, izzz);
            x = xy.x;
            y = xy.y;
            gz_st_x(aq, x);
            gz_st_x(aq + 8, y);
            if (u >= 2) {
                const fe2 ii = fe_mul2_call(izz, f, izzz, g);
                izz = ii.x;
                izzz = ii.y;
            }
        }
    }
#endif
}

// PCMM_TABLES_GZ: 0 off (k_tables + k_affine), 1 auto (default), 2 always
int tables_gz_mode() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("PCMM_TABLES_GZ");
        v = e ? atoi(e) : 1;
    }
    return v;
}

cudaError_t launch_tables_gz(const uint32_t *bsoa, const ColPlan *plans, int n, int l, int N, int slots, int maxup,
                             uint32_t *tables, uint32_t *atables, int skip_chain, const int *general,
                             cudaStream_t s) {
    const int64_t total = 2LL * n * l;
    const unsigned grid = (unsigned)((total + 127) / 128);
    if (maxup <= 8)
        k_tables_gz<8><<<grid, 128, 0, s>>>(bsoa, plans, n, l, N, slots, tables, atables, skip_chain, general);
    else
        k_tables_gz<32><<<grid, 128, 0, s>>>(bsoa, plans, n, l, N, slots, tables, atables, skip_chain, general);
    return cudaGetLastError();
}

}  // namespace pcmm
