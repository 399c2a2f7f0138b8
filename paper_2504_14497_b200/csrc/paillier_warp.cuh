// paillier_warp.cuh -- warp-cooperative arithmetic mod n^2 for the Paillier PC-MM
// (included by paillier.cu).
//
// One residue of L = 32 NL limbs is spread over a warp: lane l holds limbs
// l NL .. l NL + NL - 1 (little-endian), so a 3072-bit residue is 3 registers
// per lane instead of 96 registers (and local-memory spills) in one thread.
// The Montgomery product is CIOS, word-serial over b's limbs (each limb
// broadcast by a shuffle): every lane multiplies its NL limbs of a and of N,
// carries stay inside the lane and the carry out of a lane's top limb is kept
// pending (ov) until the one-limb shift of the iteration moves the next lane's
// bottom limb into that position.  Carries across lanes are resolved once per
// product with a carry-lookahead over the warp (ballots of generate / propagate
// bits summed as two 32-bit words), and the final conditional subtraction uses
// the same lookahead for its borrows.  Latency of one 3072-bit product: 96
// iterations of a few shuffles + 2 NL multiply-adds, against 96 x 96 dependent
// multiply-adds in one thread.
#pragma once
#include <stdint.h>

namespace pcmm {
namespace pw {

constexpr unsigned kFull = 0xffffffffu;

template <int NL>
__device__ __forceinline__ void wld(uint32_t v[NL], const uint32_t *p, int lane) {
#pragma unroll
    for (int j = 0; j < NL; j++) v[j] = p[lane * NL + j];
}

template <int NL>
__device__ __forceinline__ void wst(uint32_t *p, const uint32_t v[NL], int lane) {
#pragma unroll
    for (int j = 0; j < NL; j++) p[lane * NL + j] = v[j];
}

// carry into each lane from a warp-wide lookahead: G = lanes generating a carry,
// Pm = lanes passing an incoming carry on (disjoint from G).  Returns the carry into
// this lane; *out = carry out of lane 31.
__device__ __forceinline__ uint32_t lookahead(uint32_t G, uint32_t Pm, int lane, uint32_t *out) {
    const uint64_t A = (uint64_t)(G | Pm), B = (uint64_t)G;
    const uint64_t S = A + B;
    const uint32_t cin = (uint32_t)(S ^ A ^ B);          // bit l: carry into position l
    *out = (uint32_t)(S >> 32);
    return (cin >> lane) & 1u;
}

// Resolve pending lane carries: ov of lane l belongs to position (l + 1) NL.  Returns
// the value above the top limb (lane 31's ov plus the final carry).
template <int NL>
__device__ __forceinline__ uint32_t wnorm(uint32_t v[NL], uint64_t ov, int lane) {
    uint32_t in = (uint32_t)__shfl_up_sync(kFull, (unsigned long long)ov, 1);
    const uint64_t top_ov = __shfl_sync(kFull, (unsigned long long)ov, 31);
    if (lane == 0) in = 0;
    // the incoming carry is < 2^33 in principle but only ever <= 3 here; add it as 32 bits
    uint64_t s = (uint64_t)v[0] + in;
    v[0] = (uint32_t)s;
    uint32_t c = (uint32_t)(s >> 32);
#pragma unroll
    for (int j = 1; j < NL; j++) {
        s = (uint64_t)v[j] + c;
        v[j] = (uint32_t)s;
        c = (uint32_t)(s >> 32);
    }
    uint32_t ones = 0xffffffffu;
#pragma unroll
    for (int j = 0; j < NL; j++) ones &= v[j];
    const uint32_t G = __ballot_sync(kFull, c != 0), Pm = __ballot_sync(kFull, c == 0 && ones == 0xffffffffu);
    uint32_t out;
    c = lookahead(G, Pm, lane, &out);
#pragma unroll
    for (int j = 0; j < NL; j++) {
        s = (uint64_t)v[j] + c;
        v[j] = (uint32_t)s;
        c = (uint32_t)(s >> 32);
    }
    return (uint32_t)top_ov + out;
}

// v <- v - N if v + top 2^(32L) >= N (warp-uniform decision)
template <int NL>
__device__ __forceinline__ void wsub_cond(uint32_t v[NL], uint32_t top, const uint32_t n[NL], int lane) {
    uint32_t d[NL], b = 0, zero = 0;
#pragma unroll
    for (int j = 0; j < NL; j++) {
        const uint64_t x = (uint64_t)v[j] - n[j] - b;
        d[j] = (uint32_t)x;
        b = (uint32_t)(x >> 63);
        zero |= d[j];
    }
    // borrow out with borrow-in 1: b | (d == 0)
    const uint32_t G = __ballot_sync(kFull, b != 0), Pm = __ballot_sync(kFull, b == 0 && zero == 0);
    uint32_t bout;
    uint32_t bin = lookahead(G, Pm, lane, &bout);
#pragma unroll
    for (int j = 0; j < NL; j++) {
        const uint64_t x = (uint64_t)d[j] - bin;
        d[j] = (uint32_t)x;
        bin = (uint32_t)(x >> 63);
    }
    const bool ge = top != 0 || bout == 0;
#pragma unroll
    for (int j = 0; j < NL; j++) v[j] = ge ? d[j] : v[j];
}

// r = a b R^-1 mod N (a, b < N, lane-distributed); r may alias a or b
template <int NL>
__device__ __forceinline__ void wmont(uint32_t r[NL], const uint32_t a[NL], const uint32_t b[NL], const uint32_t n[NL],
                                      uint32_t n0, int lane) {
    uint32_t t[NL];
#pragma unroll
    for (int j = 0; j < NL; j++) t[j] = 0;
    uint64_t ov = 0;
    uint32_t bl[NL];
#pragma unroll
    for (int j = 0; j < NL; j++) bl[j] = b[j];
#pragma unroll 1
    for (int src = 0; src < 32; src++) {
#pragma unroll
        for (int jj = 0; jj < NL; jj++) {
            const uint32_t bi = __shfl_sync(kFull, bl[jj], src);   // limb src NL + jj of b
            uint64_t c = 0;
#pragma unroll
            for (int j = 0; j < NL; j++) {
                const uint64_t s = (uint64_t)a[j] * bi + t[j] + c;
                t[j] = (uint32_t)s;
                c = s >> 32;
            }
            ov += c;
            const uint32_t q = __shfl_sync(kFull, t[0] * n0, 0);
            c = 0;
#pragma unroll
            for (int j = 0; j < NL; j++) {
                const uint64_t s = (uint64_t)n[j] * q + t[j] + c;
                t[j] = (uint32_t)s;
                c = s >> 32;
            }
            ov += c;
            // divide by 2^32: the global limb 0 (lane 0's t[0]) is now 0
            uint32_t up = __shfl_down_sync(kFull, t[0], 1);
            if (lane == 31) up = 0;
#pragma unroll
            for (int j = 0; j < NL - 1; j++) t[j] = t[j + 1];
            const uint64_t s = (uint64_t)up + ov;                 // the pending carry lands on the new top limb
            t[NL - 1] = (uint32_t)s;
            ov = s >> 32;
        }
    }
    const uint32_t top = wnorm<NL>(t, ov, lane);
    wsub_cond<NL>(t, top, n, lane);
#pragma unroll
    for (int j = 0; j < NL; j++) r[j] = t[j];
}

// Alg. 4, registers only: r0 <- 1, r1 <- g; per bit b of k (t bits):
// r_{1-b} <- r1 r0, r_b <- r_b^2
template <int NL>
__device__ __forceinline__ void wladder(uint32_t out[NL], const uint32_t g[NL], int k, int t, const uint32_t one[NL],
                                        const uint32_t n[NL], uint32_t n0, int lane) {
    uint32_t r0[NL], r1[NL];
#pragma unroll
    for (int j = 0; j < NL; j++) {
        r0[j] = one[j];
        r1[j] = g[j];
    }
    for (int i = t - 1; i >= 0; i--) {
        const int b = (k >> i) & 1;                               // warp-uniform
        uint32_t x[NL], y[NL];
        wmont<NL>(x, r1, r0, n, n0, lane);
        if (b) {
            wmont<NL>(y, r1, r1, n, n0, lane);
#pragma unroll
            for (int j = 0; j < NL; j++) {
                r0[j] = x[j];
                r1[j] = y[j];
            }
        } else {
            wmont<NL>(y, r0, r0, n, n0, lane);
#pragma unroll
            for (int j = 0; j < NL; j++) {
                r1[j] = x[j];
                r0[j] = y[j];
            }
        }
    }
#pragma unroll
    for (int j = 0; j < NL; j++) out[j] = r0[j];
}

}  // namespace pw
}  // namespace pcmm
