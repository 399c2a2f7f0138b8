// paillier.cu -- SURVEY.md §8(f) NEXT-4: PC-MM over the Paillier scheme
// (Sec. 2.5; extension).
//
// Ciphertexts are residues mod n^2 (L x 32-bit limbs, little-endian, L in
// {16, 32, 64, 96}: n^2 of 512..3072 bits).  The homomorphism of Eq. 6
// turns PC-MM into C_ij = prod_k c_kj^{a_ik} mod n^2
// (PAPER.md:591-606): point addition becomes a modular multiplication and an
// ECSM a modular exponentiation, which the paper computes with the Montgomery
// powering ladder (Alg. 4).  The Cussen path is Alg. 3 with
// those substitutions: the byte path's compression plan (k_plan,
// rank), level-N exponentiations by Alg. 4, prefix PRODUCTS, and the gather +
// multiply accumulation.  Plaintexts are non-negative (R20).
//
// Arithmetic, two families with the same memory layout (choice per kernel in
// run_paillier_L): warp-cooperative products for L >= 32 (paillier_warp.cuh;
// always at 3072 bits and for the key setup, otherwise for launches of few
// products) and the original one thread per modular product, Montgomery CIOS with R = 2^(32L):
// the left operand and the running sum t in registers (inner loops fully
// unrolled over the L limbs), the right operand streamed from memory one limb
// per outer step, the modulus and -n^-1 mod 2^32 in the kernel's parameter
// space (a __grid_constant__ struct: compile-time offsets, so they are constant
// bank operands of the IMADs and every launch carries its own modulus).
#include "internal.h"
#include "paillier_warp.cuh"

namespace pcmm {

namespace {

template <int L>
struct ModN {
    uint32_t n[L];
    uint32_t n0;          // -n^-1 mod 2^32
};

// r = a b R^-1 mod N (a in registers, b in memory; a, b < N); r may alias a
template <int L>
__device__ __forceinline__ void mont_mul(uint32_t r[L], const uint32_t a[L], const uint32_t *b, const ModN<L> &M) {
    uint32_t t[L + 2];
#pragma unroll
    for (int j = 0; j < L + 2; j++) t[j] = 0;
#pragma unroll 1
    for (int i = 0; i < L; i++) {
        const uint32_t bi = b[i];
        uint32_t C = 0;
#pragma unroll
        for (int j = 0; j < L; j++) {
            const uint64_t p = (uint64_t)a[j] * bi + t[j] + C;
            t[j] = (uint32_t)p;
            C = (uint32_t)(p >> 32);
        }
        uint64_t s = (uint64_t)t[L] + C;
        t[L] = (uint32_t)s;
        t[L + 1] = (uint32_t)(s >> 32);
        const uint32_t q = t[0] * M.n0;
        uint64_t p = (uint64_t)q * M.n[0] + t[0];
        C = (uint32_t)(p >> 32);
#pragma unroll
        for (int j = 1; j < L; j++) {
            p = (uint64_t)q * M.n[j] + t[j] + C;
            t[j - 1] = (uint32_t)p;
            C = (uint32_t)(p >> 32);
        }
        s = (uint64_t)t[L] + C;
        t[L - 1] = (uint32_t)s;
        t[L] = t[L + 1] + (uint32_t)(s >> 32);
    }
    // t < 2N: subtract N when t >= N
    uint32_t d[L];
    uint32_t borrow = 0;
#pragma unroll
    for (int j = 0; j < L; j++) {
        const uint64_t x = (uint64_t)t[j] - M.n[j] - borrow;
        d[j] = (uint32_t)x;
        borrow = (uint32_t)(x >> 63);
    }
    const bool ge = t[L] != 0 || borrow == 0;
#pragma unroll
    for (int j = 0; j < L; j++) r[j] = ge ? d[j] : t[j];
}

template <int L>
__device__ __forceinline__ void ld(uint32_t r[L], const uint32_t *p) {
#pragma unroll
    for (int j = 0; j < L; j++) r[j] = p[j];
}

template <int L>
__device__ __forceinline__ void st(uint32_t *p, const uint32_t r[L]) {
#pragma unroll
    for (int j = 0; j < L; j++) p[j] = r[j];
}

// Alg. 4 over t bits of k: r0 <- 1, r1 <- g; per bit b:
// r_{1-b} <- r1 r0, r_b <- r_b^2; returns r0 (all in Montgomery form).
// r0 / r1 live in the caller's scratch (local memory) so that each product
// streams one operand from memory.
template <int L>
__device__ void ladder(uint32_t *out, const uint32_t *g, int k, int t, const uint32_t *one, const ModN<L> &M,
                       uint32_t *r0, uint32_t *r1) {
    uint32_t x[L];
    ld<L>(x, one);
    st<L>(r0, x);
    ld<L>(x, g);
    st<L>(r1, x);
    for (int i = t - 1; i >= 0; i--) {
        const int b = (k >> i) & 1;
        uint32_t *rb = b ? r1 : r0, *rnb = b ? r0 : r1;
        ld<L>(x, r1);
        mont_mul<L>(x, x, r0, M);                 // r_{1-b} <- r1 r0
        uint32_t y[L];
        ld<L>(y, rb);
        mont_mul<L>(y, y, rb, M);                 // r_b <- r_b^2
        st<L>(rnb, x);
        st<L>(rb, y);
    }
    ld<L>(x, r0);
    st<L>(out, x);
}

// key setup (one thread): R mod N = 2^(32L) - kN (at most 4 subtractions: N has
// 32L - 1 or 32L bits), then x = 2^(L/2) R mod N by L/2 modular doublings and
// six Montgomery squarings x <- x^2 R^-1: 2^((L/2) 64) R = R^2 mod N.
template <int L>
__global__ void k_pl_setup(const __grid_constant__ ModN<L> M, uint32_t *__restrict__ one, uint32_t *__restrict__ r2,
                           uint32_t *__restrict__ unit) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int j = 0; j < L; j++) unit[j] = j == 0 ? 1u : 0u;  // plain 1: mont_mul(x, 1) leaves Montgomery form
    uint32_t x[L], top = 1;                                  // x + top 2^(32L) = 2^(32L)
    for (int j = 0; j < L; j++) x[j] = 0;
    for (int rep = 0; rep < 8; rep++) {                      // while (top, x) >= N: subtract N
        uint32_t d[L], borrow = 0;
        for (int j = 0; j < L; j++) {
            const uint64_t v = (uint64_t)x[j] - M.n[j] - borrow;
            d[j] = (uint32_t)v;
            borrow = (uint32_t)(v >> 63);
        }
        if (top < borrow) break;                             // (top, x) < N
        top -= borrow;
        for (int j = 0; j < L; j++) x[j] = d[j];
    }
    for (int j = 0; j < L; j++) one[j] = x[j];
    for (int it = 0; it < L / 2; it++) {                     // x <- 2x mod N
        uint32_t c = 0;
        for (int j = 0; j < L; j++) {
            const uint32_t nx = (x[j] << 1) | c;
            c = x[j] >> 31;
            x[j] = nx;
        }
        uint32_t d[L], borrow = 0;
        for (int j = 0; j < L; j++) {
            const uint64_t v = (uint64_t)x[j] - M.n[j] - borrow;
            d[j] = (uint32_t)v;
            borrow = (uint32_t)(v >> 63);
        }
        if (c || !borrow)
            for (int j = 0; j < L; j++) x[j] = d[j];
    }
    for (int sq = 0; sq < 6; sq++) {
        st<L>(r2, x);
        mont_mul<L>(x, x, r2, M);
    }
    st<L>(r2, x);
}

// normal -> Montgomery form (c R mod N = mont_mul(c, R^2)); status bit if c >= N
template <int L>
__global__ void __launch_bounds__(128) k_pl_import(const __grid_constant__ ModN<L> M, const uint32_t *__restrict__ c,
                                                   int64_t count, const uint32_t *__restrict__ r2,
                                                   uint32_t *__restrict__ out, int *__restrict__ status) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= count) return;
    uint32_t x[L];
    ld<L>(x, c + e * L);
    uint32_t borrow = 0;
#pragma unroll
    for (int j = 0; j < L; j++) {
        const uint64_t v = (uint64_t)x[j] - M.n[j] - borrow;
        borrow = (uint32_t)(v >> 63);
    }
    if (!borrow) atomicOr(status, kStatusCurve);          // c >= n^2: not a residue
    mont_mul<L>(x, x, r2, M);
    st<L>(out + e * L, x);
}

// a2 + a3 (Paillier): thread per (k, j); table [k][j][slot][L], slot 0 = 1 (R mod N)
template <int L>
__global__ void __launch_bounds__(64) k_pl_tables(const __grid_constant__ ModN<L> M, const uint32_t *__restrict__ bm,
                                                  const ColPlan *__restrict__ plans, int n, int l, int N, int S,
                                                  int maxup, int t, const uint32_t *__restrict__ one,
                                                  uint32_t *__restrict__ tables, uint32_t *__restrict__ scr) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= (int64_t)n * l) return;
    const int k = (int)(tid / l);                            // tid = k l + j
    const ColPlan &pl = plans[k];
    const uint32_t *P = bm + tid * L;
    uint32_t *blk = tables + tid * (int64_t)S * L;
    uint32_t *sc = scr + tid * (int64_t)2 * maxup * L;
    uint32_t r0[L], r1[L];                                    // ladder registers (local memory)
    uint32_t x[L];
    ld<L>(x, one);
    st<L>(blk, x);                                            // slot 0: a_ik = 0 -> 1
    const int n1 = pl.n[0];
    if (N == 1) {
        for (int u = 0; u < n1; u++) ladder<L>(blk + (int64_t)(u + 1) * L, P, pl.sN[u], t, one, M, r0, r1);
    } else {
        int src = 0;
        for (int u = 0; u < pl.n[N - 1]; u++) ladder<L>(sc + (int64_t)u * L, P, pl.sN[u], t, one, M, r0, r1);
        for (int lev = N - 1; lev >= 2; lev--) {              // prefix products, levels N-1 .. 2
            const int dst = maxup - src;
            const int nl = pl.n[lev - 1];
            ld<L>(x, sc + (int64_t)(src + pl.ptr[lev - 1][0]) * L);
            st<L>(sc + (int64_t)dst * L, x);
            for (int u = 1; u < nl; u++) {
                mont_mul<L>(x, x, sc + (int64_t)(src + pl.ptr[lev - 1][u]) * L, M);
                st<L>(sc + (int64_t)(dst + u) * L, x);
            }
            src = dst;
        }
        ld<L>(x, sc + (int64_t)(src + pl.ptr[0][0]) * L);       // level 1 -> the table
        st<L>(blk + (int64_t)L, x);
        for (int u = 1; u < n1; u++) {
            mont_mul<L>(x, x, sc + (int64_t)(src + pl.ptr[0][u]) * L, M);
            st<L>(blk + (int64_t)(u + 1) * L, x);
        }
    }
    ld<L>(x, one);
    for (int slot = n1 + 1; slot < S; slot++) st<L>(blk + (int64_t)slot * L, x);
}

// a4 (Paillier): thread per (i, j), i fastest (a warp shares the tables of one j)
template <int L>
__global__ void __launch_bounds__(64) k_pl_accum(const __grid_constant__ ModN<L> M, const uint32_t *__restrict__ tables,
                                                 const uint8_t *__restrict__ rank, int m, int n, int l, int S,
                                                 const uint32_t *__restrict__ one, const uint32_t *__restrict__ unit,
                                                 uint32_t *__restrict__ out) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= (int64_t)m * l) return;
    const int i = (int)(tid % m), j = (int)(tid / m);
    uint32_t acc[L];
    ld<L>(acc, one);
    for (int k = 0; k < n; k++) {
        const int u = rank[(int64_t)k * m + i];
        if (u) mont_mul<L>(acc, acc, tables + (((int64_t)k * l + j) * S + u) * L, M);
    }
    mont_mul<L>(acc, acc, unit, M);                           // out of Montgomery form
    st<L>(out + ((int64_t)i * l + j) * L, acc);
}

// s1 (Paillier): thread per (i, j), j fastest (a_ik warp-uniform): prod_k Alg.4(c_kj, a_ik)
template <int L>
__global__ void __launch_bounds__(64) k_pl_school(const __grid_constant__ ModN<L> M, const uint8_t *__restrict__ A,
                                                  int m, int n, int l, int w, const uint32_t *__restrict__ bm,
                                                  const uint32_t *__restrict__ one, const uint32_t *__restrict__ unit,
                                                  uint32_t *__restrict__ out, int *__restrict__ status) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= (int64_t)m * l) return;
    const int j = (int)(tid % l), i = (int)(tid / l);
    uint32_t acc[L], r0[L], r1[L], e[L];
    ld<L>(acc, one);
    bool bad = false;
    for (int k = 0; k < n; k++) {
        const int a = A[(int64_t)i * n + k];
        if (a >= (1 << w)) { bad = true; continue; }
        if (!a) continue;
        ladder<L>(e, bm + ((int64_t)k * l + j) * L, a, w, one, M, r0, r1);
        mont_mul<L>(acc, acc, e, M);
    }
    if (bad) atomicOr(status, kStatusBound);
    mont_mul<L>(acc, acc, unit, M);
    st<L>(out + ((int64_t)i * l + j) * L, acc);
}

// ------------------------------------------------------------ warp-cooperative kernels (L = 32 NL)
// Same steps as the per-thread kernels above, one warp per residue operation
// (paillier_warp.cuh): no local-memory ladder registers, ~40 registers per lane.
template <int NL>
__device__ __forceinline__ void wmodn(uint32_t n[NL], const ModN<32 * NL> &M, int lane) {
#pragma unroll
    for (int j = 0; j < NL; j++) n[j] = M.n[lane * NL + j];
}

// (v, top) - N when (v, top) >= N; returns the new top
template <int NL>
__device__ __forceinline__ uint32_t wsub_top(uint32_t v[NL], uint32_t top, const uint32_t n[NL], int lane) {
    uint32_t d[NL], b = 0, zero = 0;
#pragma unroll
    for (int j = 0; j < NL; j++) {
        const uint64_t x = (uint64_t)v[j] - n[j] - b;
        d[j] = (uint32_t)x;
        b = (uint32_t)(x >> 63);
        zero |= d[j];
    }
    const uint32_t G = __ballot_sync(pw::kFull, b != 0), Pm = __ballot_sync(pw::kFull, b == 0 && zero == 0);
    uint32_t bout;
    uint32_t bin = pw::lookahead(G, Pm, lane, &bout);
#pragma unroll
    for (int j = 0; j < NL; j++) {
        const uint64_t x = (uint64_t)d[j] - bin;
        d[j] = (uint32_t)x;
        bin = (uint32_t)(x >> 63);
    }
    if (top < bout) return top;                              // (v, top) < N: unchanged
#pragma unroll
    for (int j = 0; j < NL; j++) v[j] = d[j];
    return top - bout;
}

template <int NL>
__global__ void __launch_bounds__(32) k_plw_setup(const __grid_constant__ ModN<32 * NL> M, uint32_t *__restrict__ one,
                                                  uint32_t *__restrict__ r2, uint32_t *__restrict__ unit) {
    constexpr int L = 32 * NL;
    const int lane = (int)threadIdx.x;
    uint32_t n[NL], x[NL];
    wmodn<NL>(n, M, lane);
#pragma unroll
    for (int j = 0; j < NL; j++) {
        x[j] = 0;
        unit[lane * NL + j] = (lane == 0 && j == 0) ? 1u : 0u;  // plain 1: leaves Montgomery form
    }
    uint32_t top = 1;                                        // (x, top) = 2^(32L) = R
    for (int rep = 0; rep < 8; rep++) {
        const uint32_t t2 = wsub_top<NL>(x, top, n, lane);
        if (t2 == top) break;
        top = t2;
    }
    pw::wst<NL>(one, x, lane);                               // R mod N
    for (int it = 0; it < L / 2; it++) {                     // x <- 2x mod N
        const uint32_t below = __shfl_up_sync(pw::kFull, x[NL - 1] >> 31, 1);
        const uint32_t c = __shfl_sync(pw::kFull, x[NL - 1] >> 31, 31);
#pragma unroll
        for (int j = NL - 1; j > 0; j--) x[j] = (x[j] << 1) | (x[j - 1] >> 31);
        x[0] = (x[0] << 1) | (lane == 0 ? 0u : below);
        pw::wsub_cond<NL>(x, c, n, lane);
    }
    for (int sq = 0; sq < 6; sq++) pw::wmont<NL>(x, x, x, n, M.n0, lane);   // 2^(L/2) R -> R^2 (6 squarings)
    pw::wst<NL>(r2, x, lane);
}

template <int NL>
__global__ void __launch_bounds__(128) k_plw_import(const __grid_constant__ ModN<32 * NL> M, const uint32_t *__restrict__ c,
                                                    int64_t count, const uint32_t *__restrict__ r2,
                                                    uint32_t *__restrict__ out, int *__restrict__ status) {
    constexpr int L = 32 * NL;
    const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = (int)(threadIdx.x & 31);
    if (e >= count) return;                                  // warp-uniform
    uint32_t n[NL], x[NL], y[NL], r[NL];
    wmodn<NL>(n, M, lane);
    pw::wld<NL>(x, c + e * L, lane);
#pragma unroll
    for (int j = 0; j < NL; j++) y[j] = x[j];
    wsub_top<NL>(y, 0, n, lane);                             // y = x - N iff x >= N (not a residue)
    uint32_t diff = 0;
#pragma unroll
    for (int j = 0; j < NL; j++) diff |= y[j] ^ x[j];
    if (__any_sync(pw::kFull, diff != 0) && lane == 0) atomicOr(status, kStatusCurve);
    pw::wld<NL>(r, r2, lane);
    pw::wmont<NL>(x, x, r, n, M.n0, lane);
    pw::wst<NL>(out + e * L, x, lane);
}

// a2 + a3 (Paillier, warp per (k, j)): table [k][j][slot][L], slot 0 = 1 (R mod N)
template <int NL>
__global__ void __launch_bounds__(128) k_plw_tables(const __grid_constant__ ModN<32 * NL> M,
                                                    const uint32_t *__restrict__ bm, const ColPlan *__restrict__ plans,
                                                    int n_, int l, int N, int S, int maxup, int t,
                                                    const uint32_t *__restrict__ onep, uint32_t *__restrict__ tables,
                                                    uint32_t *__restrict__ scr) {
    constexpr int L = 32 * NL;
    const int64_t tid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = (int)(threadIdx.x & 31);
    if (tid >= (int64_t)n_ * l) return;
    const int k = (int)(tid / l);
    const ColPlan &pl = plans[k];
    uint32_t n[NL], one[NL], P[NL], x[NL], y[NL];
    wmodn<NL>(n, M, lane);
    pw::wld<NL>(one, onep, lane);
    pw::wld<NL>(P, bm + tid * L, lane);
    uint32_t *blk = tables + tid * (int64_t)S * L;
    uint32_t *sc = scr + tid * (int64_t)2 * maxup * L;
    pw::wst<NL>(blk, one, lane);                             // slot 0: a_ik = 0 -> 1
    const int n1 = pl.n[0];
    if (N == 1) {
        for (int u = 0; u < n1; u++) {
            pw::wladder<NL>(x, P, pl.sN[u], t, one, n, M.n0, lane);
            pw::wst<NL>(blk + (int64_t)(u + 1) * L, x, lane);
        }
    } else {
        int src = 0;
        for (int u = 0; u < pl.n[N - 1]; u++) {
            pw::wladder<NL>(x, P, pl.sN[u], t, one, n, M.n0, lane);
            pw::wst<NL>(sc + (int64_t)u * L, x, lane);
        }
        for (int lev = N - 1; lev >= 2; lev--) {             // prefix products, levels N-1 .. 2
            const int dst = maxup - src;
            const int nl = pl.n[lev - 1];
            pw::wld<NL>(x, sc + (int64_t)(src + pl.ptr[lev - 1][0]) * L, lane);
            pw::wst<NL>(sc + (int64_t)dst * L, x, lane);
            for (int u = 1; u < nl; u++) {
                pw::wld<NL>(y, sc + (int64_t)(src + pl.ptr[lev - 1][u]) * L, lane);
                pw::wmont<NL>(x, x, y, n, M.n0, lane);
                pw::wst<NL>(sc + (int64_t)(dst + u) * L, x, lane);
            }
            src = dst;
        }
        pw::wld<NL>(x, sc + (int64_t)(src + pl.ptr[0][0]) * L, lane);   // level 1 -> the table
        pw::wst<NL>(blk + (int64_t)L, x, lane);
        for (int u = 1; u < n1; u++) {
            pw::wld<NL>(y, sc + (int64_t)(src + pl.ptr[0][u]) * L, lane);
            pw::wmont<NL>(x, x, y, n, M.n0, lane);
            pw::wst<NL>(blk + (int64_t)(u + 1) * L, x, lane);
        }
    }
    for (int slot = n1 + 1; slot < S; slot++) pw::wst<NL>(blk + (int64_t)slot * L, one, lane);
}

// a4 (Paillier, warp per (i, j), i fastest)
template <int NL>
__global__ void __launch_bounds__(128) k_plw_accum(const __grid_constant__ ModN<32 * NL> M,
                                                   const uint32_t *__restrict__ tables, const uint8_t *__restrict__ rank,
                                                   int m, int n_, int l, int S, const uint32_t *__restrict__ onep,
                                                   const uint32_t *__restrict__ unitp, uint32_t *__restrict__ out) {
    constexpr int L = 32 * NL;
    const int64_t tid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = (int)(threadIdx.x & 31);
    if (tid >= (int64_t)m * l) return;
    const int i = (int)(tid % m), j = (int)(tid / m);
    uint32_t n[NL], acc[NL], y[NL];
    wmodn<NL>(n, M, lane);
    pw::wld<NL>(acc, onep, lane);
    for (int k = 0; k < n_; k++) {
        const int u = rank[(int64_t)k * m + i];
        if (!u) continue;
        pw::wld<NL>(y, tables + (((int64_t)k * l + j) * S + u) * L, lane);
        pw::wmont<NL>(acc, acc, y, n, M.n0, lane);
    }
    pw::wld<NL>(y, unitp, lane);
    pw::wmont<NL>(acc, acc, y, n, M.n0, lane);               // out of Montgomery form
    pw::wst<NL>(out + ((int64_t)i * l + j) * L, acc, lane);
}

// s1 (Paillier, warp per (i, j), j fastest): prod_k Alg.4(c_kj, a_ik)
template <int NL>
__global__ void __launch_bounds__(128) k_plw_school(const __grid_constant__ ModN<32 * NL> M,
                                                    const uint8_t *__restrict__ A, int m, int n_, int l, int w,
                                                    const uint32_t *__restrict__ bm, const uint32_t *__restrict__ onep,
                                                    const uint32_t *__restrict__ unitp, uint32_t *__restrict__ out,
                                                    int *__restrict__ status) {
    constexpr int L = 32 * NL;
    const int64_t tid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = (int)(threadIdx.x & 31);
    if (tid >= (int64_t)m * l) return;
    const int j = (int)(tid % l), i = (int)(tid / l);
    uint32_t n[NL], one[NL], acc[NL], g[NL], e[NL];
    wmodn<NL>(n, M, lane);
    pw::wld<NL>(one, onep, lane);
    for (int q = 0; q < NL; q++) acc[q] = one[q];
    bool bad = false;
    for (int k = 0; k < n_; k++) {
        const int a = A[(int64_t)i * n_ + k];
        if (a >= (1 << w)) {
            bad = true;
            continue;
        }
        if (!a) continue;
        pw::wld<NL>(g, bm + ((int64_t)k * l + j) * L, lane);
        pw::wladder<NL>(e, g, a, w, one, n, M.n0, lane);
        pw::wmont<NL>(acc, acc, e, n, M.n0, lane);
    }
    if (bad && lane == 0) atomicOr(status, kStatusBound);
    pw::wld<NL>(e, unitp, lane);
    pw::wmont<NL>(acc, acc, e, n, M.n0, lane);
    pw::wst<NL>(out + ((int64_t)i * l + j) * L, acc, lane);
}

static int paillier_warp_on() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("PCMM_PAILLIER_WARP");          // measurement override: 0 = one thread per product
        v = e ? atoi(e) : 1;
    }
    return v;
}

// warp-cooperative kernels for L >= 32 where they win (measured, tools/paillier_prof.py):
// always at 3072 bits (per-thread L = 96 spills) and for the key setup; at 1024 /
// 2048 bits only in the latency regime of few independent products (fewer than
// 32768 warps' worth), where one thread's 32L-long carry chains are the critical path
inline bool use_warp(int L, int64_t count) {
    return L >= 32 && paillier_warp_on() && (L >= 96 || count < 32768);
}
inline unsigned nbw(int64_t warps) { return (unsigned)((warps + 3) / 4); }

inline unsigned nbp(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

template <int L>
cudaError_t run_paillier_L(int path, const uint8_t *A, int m, int n, int l, int w, int N, const uint32_t *Nh,
                           const uint32_t *ctB, uint32_t *ctC, uint8_t *ws, const size_t *off, int S, int maxup,
                           cudaStream_t s) {
    ModN<L> M;
    for (int j = 0; j < L; j++) M.n[j] = Nh[j];
    uint32_t inv = Nh[0];                                     // Newton: inv = N0^-1 mod 2^32
    for (int it = 0; it < 5; it++) inv *= 2u - Nh[0] * inv;
    M.n0 = 0u - inv;
    int *status = (int *)ws;
    uint32_t *one = (uint32_t *)(ws + off[0]), *r2 = one + L, *unit = r2 + L;
    uint32_t *bm = (uint32_t *)(ws + off[1]);
    cudaError_t e;
    const int64_t nl = (int64_t)n * l, ml = (int64_t)m * l;
    prof_begin("pl_setup", s);
    if constexpr (L >= 32) {
        if (use_warp(L, 1)) k_plw_setup<L / 32><<<1, 32, 0, s>>>(M, one, r2, unit);
        else k_pl_setup<L><<<1, 1, 0, s>>>(M, one, r2, unit);
    } else {
        k_pl_setup<L><<<1, 1, 0, s>>>(M, one, r2, unit);
    }
    prof_end(s);
    if ((e = cudaGetLastError())) return e;
    prof_begin("pl_import", s);
    if constexpr (L >= 32) {
        if (use_warp(L, nl)) k_plw_import<L / 32><<<nbw(nl), 128, 0, s>>>(M, ctB, nl, r2, bm, status);
        else k_pl_import<L><<<nbp(nl, 128), 128, 0, s>>>(M, ctB, nl, r2, bm, status);
    } else {
        k_pl_import<L><<<nbp(nl, 128), 128, 0, s>>>(M, ctB, nl, r2, bm, status);
    }
    prof_end(s);
    if ((e = cudaGetLastError())) return e;
    if (path == 0) {
        prof_begin("pl_school", s);
        if constexpr (L >= 32) {
            if (use_warp(L, ml))
                k_plw_school<L / 32><<<nbw(ml), 128, 0, s>>>(M, A, m, n, l, w, bm, one, unit, ctC, status);
            else
                k_pl_school<L><<<nbp(ml, 64), 64, 0, s>>>(M, A, m, n, l, w, bm, one, unit, ctC, status);
        } else {
            k_pl_school<L><<<nbp(ml, 64), 64, 0, s>>>(M, A, m, n, l, w, bm, one, unit, ctC, status);
        }
        prof_end(s);
        e = cudaGetLastError();
    } else {
        ColPlan *plans = (ColPlan *)(ws + off[2]);
        uint8_t *rank = ws + off[3];
        uint32_t *tables = (uint32_t *)(ws + off[4]), *scr = (uint32_t *)(ws + off[5]);
        prof_begin("plan", s);
        e = launch_plan((const int8_t *)A, m, n, w, 0, N, plans, rank, status, s);
        prof_end(s);
        if (e) return e;
        prof_begin("pl_tables", s);
        if constexpr (L >= 32) {
            if (use_warp(L, nl))
                k_plw_tables<L / 32><<<nbw(nl), 128, 0, s>>>(M, bm, plans, n, l, N, S, maxup, w, one, tables, scr);
            else
                k_pl_tables<L><<<nbp(nl, 64), 64, 0, s>>>(M, bm, plans, n, l, N, S, maxup, w, one, tables, scr);
        } else {
            k_pl_tables<L><<<nbp(nl, 64), 64, 0, s>>>(M, bm, plans, n, l, N, S, maxup, w, one, tables, scr);
        }
        prof_end(s);
        if ((e = cudaGetLastError())) return e;
        prof_begin("pl_accum", s);
        if constexpr (L >= 32) {
            if (use_warp(L, ml))
                k_plw_accum<L / 32><<<nbw(ml), 128, 0, s>>>(M, tables, rank, m, n, l, S, one, unit, ctC);
            else
                k_pl_accum<L><<<nbp(ml, 64), 64, 0, s>>>(M, tables, rank, m, n, l, S, one, unit, ctC);
        } else {
            k_pl_accum<L><<<nbp(ml, 64), 64, 0, s>>>(M, tables, rank, m, n, l, S, one, unit, ctC);
        }
        prof_end(s);
        e = cudaGetLastError();
    }
    return e;
}

}  // namespace

bool paillier_limbs_ok(int L) { return L == 16 || L == 32 || L == 64 || L == 96; }

cudaError_t run_paillier(int path, const uint8_t *A, int m, int n, int l, int w, int N, int L, const uint32_t *Nh,
                         const uint32_t *ctB, uint32_t *ctC, uint8_t *ws, const size_t *off, int S, int maxup,
                         cudaStream_t s) {
    switch (L) {
        case 16: return run_paillier_L<16>(path, A, m, n, l, w, N, Nh, ctB, ctC, ws, off, S, maxup, s);
        case 32: return run_paillier_L<32>(path, A, m, n, l, w, N, Nh, ctB, ctC, ws, off, S, maxup, s);
        case 64: return run_paillier_L<64>(path, A, m, n, l, w, N, Nh, ctB, ctC, ws, off, S, maxup, s);
        case 96: return run_paillier_L<96>(path, A, m, n, l, w, N, Nh, ctB, ctC, ws, off, S, maxup, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace pcmm
