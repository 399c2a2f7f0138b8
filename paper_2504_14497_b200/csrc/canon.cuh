// canon.cuh -- device helpers shared by kernels.cu and next2.cu: the 128-byte
// canonical ciphertext wire format (R13: x || y big-endian per point,
// the identity = 64 zero bytes), SoA point access, the generator, scalars.
#pragma once
#include "ec.cuh"
#include "internal.h"

namespace pcmm {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// 64 canonical bytes (x||y big-endian) -> 16 words as stored little-endian
__device__ __forceinline__ void load64(const uint8_t *p, uint32_t w[16]) {
    const uint4 *q = reinterpret_cast<const uint4 *>(p);
#pragma unroll
    for (int i = 0; i < 4; i++) {
        uint4 t = q[i];
        w[4 * i + 0] = t.x; w[4 * i + 1] = t.y; w[4 * i + 2] = t.z; w[4 * i + 3] = t.w;
    }
}

__device__ __forceinline__ void store64(uint8_t *p, const uint32_t w[16]) {
    uint4 *q = reinterpret_cast<uint4 *>(p);
#pragma unroll
    for (int i = 0; i < 4; i++) q[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
}

// canonical words -> (x, y) limbs (not reduced / not Montgomery); returns any-nonzero
__device__ __forceinline__ uint32_t words_to_xy(const uint32_t w[16], fe &x, fe &y) {
    uint32_t any = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        x.v[i] = bswap32(w[7 - i]);
        y.v[i] = bswap32(w[15 - i]);
        any |= w[i] | w[8 + i];
    }
    return any;
}

__device__ __forceinline__ bool fe_lt_p(const fe &a) {
    uint64_t borrow = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        uint64_t x = (uint64_t)a.v[i] - p_limb(i) - borrow;
        borrow = (x >> 63) & 1;
    }
    return borrow != 0;
}

// canonical 64 bytes -> projective Montgomery point; returns false if invalid
static __device__ bool load_canonical_point(pt &P, const uint8_t *p) {
    uint32_t w[16];
    load64(p, w);
    fe x, y;
    if (words_to_xy(w, x, y) == 0) {
        pt_identity(P);
        return true;
    }
    bool ok = fe_lt_p(x) && fe_lt_p(y);
    fe_to_mont(x, x);
    fe_to_mont(y, y);
    pt_from_affine(P, x, y);
    return ok && affine_on_curve(x, y);
}

// affine (x, y) Montgomery -> canonical 64 bytes
static __device__ void store_canonical_xy(uint8_t *p, const fe &xm, const fe &ym) {
    fe x, y;
    fe_from_mont(x, xm);
    fe_from_mont(y, ym);
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        w[7 - i] = bswap32(x.v[i]);
        w[15 - i] = bswap32(y.v[i]);
    }
    store64(p, w);
}

static __device__ void store_canonical_point(uint8_t *p, const pt &P) {
    if (pt_is_identity(P)) {
        uint32_t w[16] = {0};
        store64(p, w);
        return;
    }
    fe zi, x, y;
    fe_inv(zi, P.Z);
    fe_mul(x, P.X, zi);
    fe_mul(y, P.Y, zi);
    store_canonical_xy(p, x, y);
}

// SoA point access: base -> [coord][limb][stride]
__device__ __forceinline__ void soa_load(pt &P, const uint32_t *base, int64_t stride, int64_t idx) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
        P.X.v[i] = base[(0 * 8 + i) * stride + idx];
        P.Y.v[i] = base[(1 * 8 + i) * stride + idx];
        P.Z.v[i] = base[(2 * 8 + i) * stride + idx];
    }
}

__device__ __forceinline__ void soa_store(uint32_t *base, int64_t stride, int64_t idx, const pt &P) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
        base[(0 * 8 + i) * stride + idx] = P.X.v[i];
        base[(1 * 8 + i) * stride + idx] = P.Y.v[i];
        base[(2 * 8 + i) * stride + idx] = P.Z.v[i];
    }
}

__device__ __forceinline__ void generator_mont(pt &G) {
    G.X.v[0] = 0x18a9143cu; G.X.v[1] = 0x79e730d4u; G.X.v[2] = 0x5fedb601u; G.X.v[3] = 0x75ba95fcu;
    G.X.v[4] = 0x77622510u; G.X.v[5] = 0x79fb732bu; G.X.v[6] = 0xa53755c6u; G.X.v[7] = 0x18905f76u;
    G.Y.v[0] = 0xce95560au; G.Y.v[1] = 0xddf25357u; G.Y.v[2] = 0xba19e45cu; G.Y.v[3] = 0x8b4ab8e4u;
    G.Y.v[4] = 0xdd21f325u; G.Y.v[5] = 0xd2e88688u; G.Y.v[6] = 0x25885d85u; G.Y.v[7] = 0x8571ff18u;
    fe_one_mont(G.Z);
}

__device__ __forceinline__ void be32_to_words(const uint8_t *p, uint32_t k[8]) {
    const uint4 *q = reinterpret_cast<const uint4 *>(p);
    uint4 a = q[0], b = q[1];
    uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 8; i++) k[i] = bswap32(w[7 - i]);
}

}  // namespace pcmm
