// affine.cu -- step a3' of the Cussen path: table entries -> affine (x, y) by
// Montgomery's simultaneous inversion (k_affine), in its own translation unit so
// that it can be compiled with its own ptxas options (build.py: -O1 measured 10 %
// faster for this kernel; the accumulate kernel wants -O3).
#include <algorithm>

#include "ec.cuh"
#include "internal.h"
#include "shared.cuh"

namespace pcmm {

static inline unsigned blocks_for(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

// ------------------------------------------------------------ a3': tables -> affine
// The accumulate loop adds table entries with the XYZZ + affine mixed
// addition (hot.cu), so the tables are converted once to affine (x, y) =
// (X/Z, Y/Z) with Montgomery's simultaneous inversion: each lane takes `batch`
// entries (stride = grid size, so a warp reads consecutive entries), one fe_inv
// per CTA (below), 5 products per entry.  The prefix products are parked in
// the output's y words between the two passes.  Identity entries (Z = 0:
// slot 0 and unused slots) become x = all ones (hot.cu aff_is_inf).
struct AffIn {
    fe z;
    bool ok;        // entry exists and Z != 0
};

__device__ __forceinline__ AffIn aff_load_z(const uint32_t *__restrict__ tab, int64_t e, int64_t entries) {
    AffIn a;
    a.ok = false;
    fe_one_mont(a.z);
    if (e < entries) {
        const uint4 *src = reinterpret_cast<const uint4 *>(tab + e * kPtWords);
        const uint4 z0 = src[4], z1 = src[5];
        if ((z0.x | z0.y | z0.z | z0.w | z1.x | z1.y | z1.z | z1.w) != 0) {
            a.z = fe{{z0.x, z0.y, z0.z, z0.w, z1.x, z1.y, z1.z, z1.w}};
            a.ok = true;
        }
    }
    return a;
}

__device__ __forceinline__ void aff_pass1_store(uint32_t *__restrict__ atab, int64_t e, int64_t entries,
                                                const AffIn &a, const fe &prefix) {
    if (e >= entries) return;
    uint4 *dst = reinterpret_cast<uint4 *>(atab + e * kAffWords);
    if (!a.ok) {
        const uint4 ones = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
        dst[0] = ones;
        dst[1] = ones;
        dst[2] = make_uint4(0, 0, 0, 0);
        dst[3] = make_uint4(0, 0, 0, 0);
    } else {
        dst[2] = make_uint4(prefix.v[0], prefix.v[1], prefix.v[2], prefix.v[3]);
        dst[3] = make_uint4(prefix.v[4], prefix.v[5], prefix.v[6], prefix.v[7]);
    }
}

// Entry kinds for k_affine: homogeneous (X : Y : Z) from k_tables, or, in a
// consecutive column (k_tables_fast), slots 2..n1 hold XYZZ (X, Y, ZZ in the
// projective slot, ZZZ in the x half of the affine slot: 1/ZZZ from the batch,
// 1/Z = ZZ/ZZZ, x = X/Z^2, y = Y/ZZZ) and the other slots are already final.
enum { kAffSkip = 0, kAffProj = 1, kAffXyzz = 2, kAffInf = 3 };   // kAffInf: slot 0 / unused slot of a k_tables column
__device__ __forceinline__ AffIn aff_load_zzz(const uint32_t *__restrict__ atab, int64_t e) {
    AffIn a;
    const uint4 *src = reinterpret_cast<const uint4 *>(atab + e * kAffWords);
    const uint4 z0 = src[0], z1 = src[1];
    a.z = fe{{z0.x, z0.y, z0.z, z0.w, z1.x, z1.y, z1.z, z1.w}};
    a.ok = (z0.x | z0.y | z0.z | z0.w | z1.x | z1.y | z1.z | z1.w) != 0;
    return a;
}

// One table entry's inputs for the second pass, loaded one iteration ahead
struct AffEnt {
    fe X, Y, Z, pre;      // Z: homogeneous Z, or ZZ of an XYZZ entry; pre = prefix product
    fe zz3;               // ZZZ of an XYZZ entry
    int kind;
    bool ok;
};

__device__ __forceinline__ void aff_fetch(AffEnt &a, const uint32_t *__restrict__ tab,
                                          const uint32_t *__restrict__ atab, int64_t e, int kind) {
    a.kind = kind;
    a.ok = false;
    if (kind == kAffSkip || kind == kAffInf) return;
    const uint4 *src = reinterpret_cast<const uint4 *>(tab + e * kPtWords);
    const uint4 x0 = src[0], x1 = src[1], y0 = src[2], y1 = src[3], z0 = src[4], z1 = src[5];
    a.X = fe{{x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w}};
    a.Y = fe{{y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w}};
    a.Z = fe{{z0.x, z0.y, z0.z, z0.w, z1.x, z1.y, z1.z, z1.w}};
    const uint4 *d = reinterpret_cast<const uint4 *>(atab + e * kAffWords);
    const uint4 q0 = d[0], q1 = d[1], p0 = d[2], p1 = d[3];
    a.pre = fe{{p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w}};
    if (kind == kAffXyzz) {
        a.zz3 = fe{{q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w}};
        a.ok = !fe_is_zero(a.zz3) && (q1.w & q1.z) != 0xffffffffu;   // not the pass-1 identity marker
    } else {
        a.ok = !fe_is_zero(a.Z);
    }
}

#ifndef PCMM_AFFINE_MINB
#define PCMM_AFFINE_MINB 4
#endif
template <bool kFermat>
__global__ void __launch_bounds__(128, PCMM_AFFINE_MINB) k_affine(const uint32_t *__restrict__ tab, int64_t entries,
                                                                  int batch, uint32_t *__restrict__ atab,
                                                                  const ColPlan *__restrict__ plans, int n, int l,
                                                                  int S, int N, int fast,
                                                                  const int *__restrict__ general) {
    __shared__ fe wtot[4], winv[4];
    if (fast == 2 && general != nullptr && *general == 0) return;     // every column done by k_tables_coz
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // entry e = ((c n + k) l + j) S + slot, S a power of two; plans != nullptr only on the byte path;
    // 32-bit index arithmetic when entries < 2^32
    const uint32_t sl = (uint32_t)S * (uint32_t)l;
    const bool small = entries < (1LL << 32);
    auto kind = [&](int64_t e) -> int {
        if (e >= entries) return kAffSkip;
        if (plans == nullptr) return kAffProj;
        const uint32_t e32 = (uint32_t)e;
        const ColPlan &pl = plans[small ? (e32 / sl) % (uint32_t)n : (int)((e / ((int64_t)S * l)) % n)];
        const int slot = (int)(e & (int64_t)(S - 1));
        if (fast && col_consecutive(pl, N)) {
            if (fast == 2) return kAffSkip;                                // k_tables_aff: final already
            return (slot >= 2 && slot <= pl.n[0]) ? (PCMM_TFAST_PROJ ? kAffProj : kAffXyzz) : kAffSkip;
        }
        // k_tables leaves slot 0 and the unused slots unwritten: the identity marker is written here
        return (slot >= 1 && slot <= pl.n[0]) ? kAffProj : kAffInf;
    };
    fe one;
    fe_one_mont(one);
    fe acc = one;
    int any = 0;
    for (int r = 0; r < batch; r++) {
        const int64_t e = t + r * T;
        if (e >= entries) break;
        const int kd = kind(e);
        if (kd == kAffSkip) continue;
        if (kd == kAffInf) {
            st_aff_inf(atab + e * kAffWords);
            continue;
        }
        const AffIn a0 = kd == kAffProj ? aff_load_z(tab, e, entries) : aff_load_zzz(atab, e);
        if (kd == kAffProj) {
            aff_pass1_store(atab, e, entries, a0, acc);
        } else if (a0.ok) {
            uint4 *dst = reinterpret_cast<uint4 *>(atab + e * kAffWords);
            dst[2] = make_uint4(acc.v[0], acc.v[1], acc.v[2], acc.v[3]);
            dst[3] = make_uint4(acc.v[4], acc.v[5], acc.v[6], acc.v[7]);
        } else {
            // ZZZ = 0 (an identity ciphertext component): the identity marker is final here, so a
            // CTA with nothing to invert can return before pass 2 (pass 2 sees the marker, aff_fetch)
            st_aff_inf(atab + e * kAffWords);
        }
        if (a0.ok) {
            fe_mul(acc, acc, a0.z);
            any = 1;
        }
    }
    if (!__syncthreads_or(any)) return;                                // nothing to invert in this CTA
    fe inv = cta_inverse<kFermat>(acc, wtot, winv);
    AffEnt cur;
    int r = batch - 1;
    aff_fetch(cur, tab, atab, t + r * T, kind(t + r * T));
    for (; r >= 0; r--) {
        const int64_t e = t + r * T;
        AffEnt nxt;
        nxt.kind = kAffSkip;
        nxt.ok = false;
        if (r > 0) aff_fetch(nxt, tab, atab, e - T, kind(e - T));   // next entry's loads in flight
        if (cur.ok) {
            fe ui, x, y;
            fe_mul(ui, inv, cur.pre);              // 1 / Z (homogeneous) or 1 / ZZZ (XYZZ)
            if (cur.kind == kAffProj) {
                fe_mul(inv, inv, cur.Z);
                fe_mul(x, cur.X, ui);
                fe_mul(y, cur.Y, ui);
            } else {
                fe zi, zi2;
                fe_mul(inv, inv, cur.zz3);
                fe_mul(zi, ui, cur.Z);             // 1 / Z = ZZ / ZZZ
                fe_sqr(zi2, zi);
                fe_mul(x, cur.X, zi2);
                fe_mul(y, cur.Y, ui);
            }
            uint4 *dst = reinterpret_cast<uint4 *>(atab + e * kAffWords);
            dst[0] = make_uint4(x.v[0], x.v[1], x.v[2], x.v[3]);
            dst[1] = make_uint4(x.v[4], x.v[5], x.v[6], x.v[7]);
            dst[2] = make_uint4(y.v[0], y.v[1], y.v[2], y.v[3]);
            dst[3] = make_uint4(y.v[4], y.v[5], y.v[6], y.v[7]);
        } else if (cur.kind == kAffXyzz) {
            st_aff_inf(atab + e * kAffWords);      // ZZZ = 0: the identity
        }
        cur = nxt;
    }
}

cudaError_t launch_affine(const uint32_t *tables, int64_t entries, uint32_t *atables, cudaStream_t s,
                          const ColPlan *plans, int n, int l, int S, int N, int fast, const int *general) {
    if (entries <= 0) return cudaSuccess;
    // up to 32 entries per lane (one inversion per 4096 entries), fewer when that
    // would leave fewer than ~4 warps per SM (256^3: batch 32 0.48 ms, 16 0.55, 8 0.76)
    static int batch_env = -1;
    if (batch_env < 0) {
        const char *e = getenv("PCMM_AFFINE_BATCH");
        batch_env = e ? atoi(e) : 0;
    }
    // fill exactly one wave of resident CTAs (128 lanes each), at most 64 entries per lane (w = 8, 256^3:
    // 64 per lane 2.85 ms vs 32: 3.23)
    static int occ = 0;
    if (!occ) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_affine<true>, 128, 0) != cudaSuccess || occ <= 0)
            occ = 3;
    }
    const int64_t wave = (int64_t)num_sms() * occ * 128;
    const int batch = batch_env > 0 ? batch_env : (int)std::min<int64_t>(64, std::max<int64_t>(1, (entries + wave - 1) / wave));
    const int64_t threads = (entries + batch - 1) / batch;
    // 256^3 (2.1 M entries): Fermat 0.29 ms vs divsteps 0.36; 64^3 (131 K): 0.113 vs 0.084
    static int inv_env = -2;
    if (inv_env == -2) {
        const char *e = getenv("PCMM_AFFINE_FERMAT");         // measurement override: 1 Fermat, 0 divsteps
        inv_env = e ? atoi(e) : -1;
    }
    // with the one-wave batch and 128 registers (PCMM_AFFINE_MINB) divsteps win everywhere:
    // 256^3 0.309 vs 0.324 ms, 512^3 0.299 vs 0.314, ML 0.246 vs 0.261, 64^3 0.091 vs 0.107
    if (inv_env == 1)
        k_affine<true><<<blocks_for(threads, 128), 128, 0, s>>>(tables, entries, batch, atables, plans, n, l, S, N,
                                                                  fast, general);
    else
        k_affine<false><<<blocks_for(threads, 128), 128, 0, s>>>(tables, entries, batch, atables, plans, n, l, S, N,
                                                                   fast, general);
    return cudaGetLastError();
}

}  // namespace pcmm
