// next2.cu -- SURVEY.md §8(f) NEXT-2: GPU-resident steps either side of PC-MM.
//
//  * Fixed-base comb encryption (Sec. 2.4 Encrypt: (rG, rH + phi(b))
//    with phi(b) = bG): per key, tables T_P[i][v] = v 2^(8i) P for
//    P in {G, H}, i < 32 byte windows, v < 256 (affine, 512 KB per base);
//    then rG = sum_i T_G[i][r_i] and rH + bG = sum_i T_H[i][r_i] +- sum_{i<4}
//    T_G[i][|b|_i]: <= 68 Jacobian + affine mixed additions per ciphertext
//    instead of two 256-bit double-and-add ladders.
//  * Baby-step giant-step decryption (phi^-1 is a discrete log
//    that is only feasible for bounded messages): per context a device hash
//    table of the baby steps { jG : 1 <= j < s } (key = x || parity(y) of the
//    affine Montgomery coordinates, so jG and -jG differ), then per ciphertext
//    M = C2 - x C1 - lo G and giant steps M - i s G, i = 0, 1, ..., in batches
//    of 8 sharing one inversion, until the affine point is the identity
//    (j = 0) or hits the table: m = lo + i s + j.
#include "canon.cuh"
#include "jac.cuh"

namespace pcmm {

namespace {

constexpr int kWin = 32, kEnt = 256;                                   // 8-bit windows of 256-bit scalars
constexpr size_t kCombBase = (size_t)kWin * kEnt * kAffWords;          // words per base table
constexpr uint32_t kEncMagic = 0x636f6d62u, kBsgsMagic = 0x62736773u;  // "comb", "bsgs"

struct Pk64n2 {
    uint8_t b[64];
};
struct Sc8 {
    uint32_t k[8];
};

__device__ __forceinline__ void ld_aff(fe &x, fe &y, const uint32_t *e) {
    const uint4 *q = reinterpret_cast<const uint4 *>(e);
    const uint4 a = q[0], b = q[1], c = q[2], d = q[3];
    x = fe{{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w}};
    y = fe{{c.x, c.y, c.z, c.w, d.x, d.y, d.z, d.w}};
}

__device__ __forceinline__ void st_homog(uint32_t *e, const pt &q) {
    uint4 *d = reinterpret_cast<uint4 *>(e);
    d[0] = make_uint4(q.X.v[0], q.X.v[1], q.X.v[2], q.X.v[3]);
    d[1] = make_uint4(q.X.v[4], q.X.v[5], q.X.v[6], q.X.v[7]);
    d[2] = make_uint4(q.Y.v[0], q.Y.v[1], q.Y.v[2], q.Y.v[3]);
    d[3] = make_uint4(q.Y.v[4], q.Y.v[5], q.Y.v[6], q.Y.v[7]);
    d[4] = make_uint4(q.Z.v[0], q.Z.v[1], q.Z.v[2], q.Z.v[3]);
    d[5] = make_uint4(q.Z.v[4], q.Z.v[5], q.Z.v[6], q.Z.v[7]);
}

// ------------------------------------------------------------ comb tables
// thread (b, i): 2^(8i) P_b by 8i doublings (P_0 = G, P_1 = H); header word 1 = 1 if H is valid
__global__ void k_comb_bases(const __grid_constant__ Pk64n2 pk, uint32_t *__restrict__ bases,
                             uint32_t *__restrict__ hdr) {
    const int t = (int)threadIdx.x;
    if (t >= 2 * kWin) return;
    const int b = t / kWin, i = t % kWin;
    pt P;
    if (b == 0) {
        generator_mont(P);
    } else {
        uint8_t pkb[64];
#pragma unroll
        for (int q = 0; q < 64; q++) pkb[q] = pk.b[q];
        const int bad = pt_from_canonical(P, pkb) || pt_is_identity(P);
        if (i == 0) hdr[1] = bad ? 0u : 1u;
    }
    for (int d = 0; d < 8 * i; d++) pt_dbl_nl(P, P);
    st_homog(bases + (size_t)t * kPtWords, P);
}

// thread (b, i, chunk of 16 values): v B_{b,i} for v = 16c .. 16c + 15 (homogeneous; v = 0 -> identity)
__global__ void k_comb_fill(const uint32_t *__restrict__ bases, uint32_t *__restrict__ tmp) {
    const int t = (int)(blockIdx.x * blockDim.x + threadIdx.x);
    if (t >= 2 * kWin * (kEnt / 16)) return;
    const int bi = t / (kEnt / 16), c = t % (kEnt / 16);
    pt B, acc;
    const uint32_t *bp = bases + (size_t)bi * kPtWords;
#pragma unroll
    for (int q = 0; q < 8; q++) {
        B.X.v[q] = bp[q];
        B.Y.v[q] = bp[8 + q];
        B.Z.v[q] = bp[16 + q];
    }
    pt_mul_small(acc, 16 * c, B);
    for (int v = 16 * c; v < 16 * c + 16; v++) {
        st_homog(tmp + ((size_t)bi * kEnt + v) * kPtWords, acc);
        pt_add_nl(acc, acc, B);
    }
}

// ------------------------------------------------------------ comb encryption
__device__ __forceinline__ void jac_to_affine_pair(const jacc &A, const jacc &B, fe &xa, fe &ya, fe &xb, fe &yb) {
    // one inversion for both: 1/(Za Zb); identity handled by the caller
    fe t, inv, za, zb, z2;
    fe_mul(t, A.Z, B.Z);
    fe_inv(inv, t);
    fe_mul(za, inv, B.Z);
    fe_mul(zb, inv, A.Z);
    fe_sqr(z2, za);
    fe_mul(xa, A.X, z2);
    fe_mul(z2, z2, za);
    fe_mul(ya, A.Y, z2);
    fe_sqr(z2, zb);
    fe_mul(xb, B.X, z2);
    fe_mul(z2, z2, zb);
    fe_mul(yb, B.Y, z2);
}

__device__ __forceinline__ void jac_to_affine(const jacc &A, fe &x, fe &y) {
    fe zi, z2;
    fe_inv(zi, A.Z);
    fe_sqr(z2, zi);
    fe_mul(x, A.X, z2);
    fe_mul(z2, z2, zi);
    fe_mul(y, A.Y, z2);
}

__global__ void __launch_bounds__(128) k_encrypt_comb(const uint32_t *__restrict__ ctx, const int32_t *__restrict__ bv,
                                                      const uint8_t *__restrict__ r, int64_t count,
                                                      uint8_t *__restrict__ ct) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= count) return;
    const uint32_t *TG = ctx + 64, *TH = TG + kCombBase;
    uint32_t rk[8];
    be32_to_words(r + e * 32, rk);                      // little-endian 32-bit words of r
    jacc c1, c2;
    jac_init(c1);
    jac_init(c2);
    fe x, y;
    for (int i = 0; i < kWin; i++) {
        const int v = (rk[i >> 2] >> (8 * (i & 3))) & 0xff;
        if (!v) continue;
        ld_aff(x, y, TG + ((size_t)i * kEnt + v) * kAffWords);
        jac_add_aff(c1, x, y);                          // r G
        ld_aff(x, y, TH + ((size_t)i * kEnt + v) * kAffWords);
        jac_add_aff(c2, x, y);                          // r H
    }
    const int32_t b = bv[e];
    const uint32_t ab = b < 0 ? (uint32_t)(-(int64_t)b) : (uint32_t)b;
    for (int i = 0; i < 4; i++) {
        const int v = (ab >> (8 * i)) & 0xff;
        if (!v) continue;
        ld_aff(x, y, TG + ((size_t)i * kEnt + v) * kAffWords);
        if (b < 0) fe_neg(y, y);                        // (q - |b|) G = -|b| G
        jac_add_aff(c2, x, y);                          // + phi(b) = b G
    }
    uint8_t *o = ct + e * 128;
    if (!c1.inf && !c2.inf) {
        fe x1, y1, x2, y2;
        jac_to_affine_pair(c1, c2, x1, y1, x2, y2);
        store_canonical_xy(o, x1, y1);
        store_canonical_xy(o + 64, x2, y2);
    } else {
        uint32_t zero[16] = {0};
        for (int h = 0; h < 2; h++) {
            const jacc &A = h ? c2 : c1;
            if (A.inf) {
                store64(o + 64 * h, zero);
            } else {
                fe xa, ya;
                jac_to_affine(A, xa, ya);
                store_canonical_xy(o + 64 * h, xa, ya);
            }
        }
    }
}

// ------------------------------------------------------------ BSGS
// context: words [0, 64) header {magic, log2s, s, nslots}, words 16..31 = -s G
// affine (Montgomery); then keys u64[nslots], vals u32[nslots].
__device__ __forceinline__ uint64_t bsgs_key(const fe &xm, const fe &ym) {
    uint64_t k = ((((uint64_t)xm.v[1] << 32) | xm.v[0]) & ~1ull) | (ym.v[0] & 1u);
    k ^= 0x8000000000000000ull;
    return k ? k : 1ull;
}

__device__ __forceinline__ uint64_t bsgs_hash(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    return k;
}

constexpr int kBabyRun = 32;

__global__ void __launch_bounds__(128) k_bsgs_fill(uint32_t *__restrict__ ctx, int log2s) {
    const int64_t s = 1LL << log2s;
    const int64_t nslots = 2 * s;
    uint64_t *keys = reinterpret_cast<uint64_t *>(ctx + 64);
    uint32_t *vals = reinterpret_cast<uint32_t *>(keys + nslots);
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t j0 = 1 + t * kBabyRun;
    if (j0 >= s) return;
    const int cnt = (int)(s - j0 < kBabyRun ? s - j0 : kBabyRun);
    pt G, cur;
    generator_mont(G);
    pt_mul_small(cur, (int)j0, G);
    pt pts[kBabyRun];
    fe pre[kBabyRun];
    fe acc;
    fe_one_mont(acc);
    for (int c = 0; c < cnt; c++) {                      // j G for j = j0 .. j0 + cnt - 1 (never the identity)
        pts[c] = cur;
        pre[c] = acc;
        fe_mul(acc, acc, cur.Z);
        pt_add_nl(cur, cur, G);
    }
    fe inv;
    fe_inv(inv, acc);
    for (int c = cnt - 1; c >= 0; c--) {
        fe zi, xm, ym;
        fe_mul(zi, inv, pre[c]);
        fe_mul(inv, inv, pts[c].Z);
        fe_mul(xm, pts[c].X, zi);
        fe_mul(ym, pts[c].Y, zi);
        const uint64_t key = bsgs_key(xm, ym);
        uint64_t slot = bsgs_hash(key) & (uint64_t)(nslots - 1);
        while (true) {
            const unsigned long long prev =
                atomicCAS(reinterpret_cast<unsigned long long *>(keys + slot), 0ull, (unsigned long long)key);
            if (prev == 0ull) {
                vals[slot] = (uint32_t)(j0 + c);
                break;
            }
            slot = (slot + 1) & (uint64_t)(nslots - 1);
        }
    }
}

__global__ void k_bsgs_header(uint32_t *__restrict__ ctx, int log2s) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    pt G, P;
    generator_mont(G);
    uint32_t k[8] = {0};
    k[log2s >> 5] = 1u << (log2s & 31);                  // s = 2^log2s
    pt_mul_scalar(P, k, G);
    pt_neg(P, P);                                         // -s G
    fe zi, x, y;
    fe_inv(zi, P.Z);
    fe_mul(x, P.X, zi);
    fe_mul(y, P.Y, zi);
#pragma unroll
    for (int q = 0; q < 8; q++) {
        ctx[16 + q] = x.v[q];
        ctx[24 + q] = y.v[q];
    }
    ctx[1] = (uint32_t)log2s;
    ctx[2] = 1u << log2s;
    ctx[3] = 2u << log2s;
    ctx[0] = kBsgsMagic;
}

// -lo G (homogeneous) for the decryption of [lo, hi]
__global__ void k_neg_mulG(int64_t lo, uint32_t *__restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    pt G, P;
    generator_mont(G);
    const uint64_t a = lo < 0 ? (uint64_t)(-lo) : (uint64_t)lo;
    uint32_t k[8] = {(uint32_t)a, (uint32_t)(a >> 32), 0, 0, 0, 0, 0, 0};
    pt_mul_scalar(P, k, G);
    if (lo > 0) pt_neg(P, P);
    st_homog(out, P);
}

constexpr int kGiantBatch = 8;

__global__ void __launch_bounds__(64) k_decrypt_bsgs(const __grid_constant__ Sc8 xs, const uint32_t *__restrict__ ctx,
                                                     const uint8_t *__restrict__ ct, int64_t count, int64_t lo,
                                                     int64_t range, const uint32_t *__restrict__ neglo,
                                                     int64_t *__restrict__ mout, int32_t *__restrict__ status) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= count) return;
    const int log2s = (int)ctx[1];
    const int64_t s = 1LL << log2s, nslots = 2 * s;
    const uint64_t *keys = reinterpret_cast<const uint64_t *>(ctx + 64);
    const uint32_t *vals = reinterpret_cast<const uint32_t *>(keys + nslots);
    pt C1, C2, M, L;
    bool ok = load_canonical_point(C1, ct + e * 128);
    ok = load_canonical_point(C2, ct + e * 128 + 64) && ok;
    if (!ok) {
        mout[e] = 0;
        status[e] = -4;
        return;
    }
    uint32_t xk[8];
#pragma unroll
    for (int i = 0; i < 8; i++) xk[i] = xs.k[i];
    pt_mul_scalar_win(M, xk, C1);                         // C1 decoded: Z = 1 or the identity
    pt_neg(M, M);
    pt_add_nl(M, C2, M);                                  // C2 - x C1 = phi(m)
#pragma unroll
    for (int q = 0; q < 8; q++) {
        L.X.v[q] = neglo[q];
        L.Y.v[q] = neglo[8 + q];
        L.Z.v[q] = neglo[16 + q];
    }
    pt_add_nl(M, M, L);                                   // phi(m - lo)
    jacc P;                                               // Jacobian (X Z, Y Z^2, Z)
    jac_init(P);
    if (!fe_is_zero(M.Z)) {
        P.Z = M.Z;
        fe_sqr(P.ZZ, M.Z);
        fe_mul(P.X, M.X, M.Z);
        fe_mul(P.Y, M.Y, P.ZZ);
        P.inf = 0;
    }
    fe gx, gy;                                            // -s G
#pragma unroll
    for (int q = 0; q < 8; q++) {
        gx.v[q] = ctx[16 + q];
        gy.v[q] = ctx[24 + q];
    }
    const int64_t ngiant = (range + s - 1) / s;
    int32_t st = -5;
    int64_t mv = 0;
    for (int64_t i0 = 0; i0 < ngiant && st != 0; i0 += kGiantBatch) {
        jacc Q[kGiantBatch];
        fe pre[kGiantBatch];
        fe acc;
        fe_one_mont(acc);
        const int nb = (int)(ngiant - i0 < kGiantBatch ? ngiant - i0 : kGiantBatch);
        for (int g = 0; g < nb; g++) {
            Q[g] = P;
            pre[g] = acc;
            if (!P.inf) fe_mul(acc, acc, P.Z);
            jac_add_aff(P, gx, gy);                       // next giant step
        }
        fe inv;
        fe_inv(inv, acc);
        int64_t hit = -1;
        for (int g = nb - 1; g >= 0; g--) {               // all lookups; keep the smallest g that hits
            int64_t j = -1;
            if (Q[g].inf) {
                j = 0;
            } else {
                fe zi, z2, xm, ym;
                fe_mul(zi, inv, pre[g]);
                fe_mul(inv, inv, Q[g].Z);
                fe_sqr(z2, zi);
                fe_mul(xm, Q[g].X, z2);
                fe_mul(z2, z2, zi);
                fe_mul(ym, Q[g].Y, z2);
                const uint64_t key = bsgs_key(xm, ym);
                uint64_t slot = bsgs_hash(key) & (uint64_t)(nslots - 1);
                while (true) {
                    const uint64_t k = keys[slot];
                    if (k == 0) break;
                    if (k == key) {
                        j = vals[slot];
                        break;
                    }
                    slot = (slot + 1) & (uint64_t)(nslots - 1);
                }
            }
            if (j >= 0) hit = (i0 + g) * s + j;
        }
        if (hit >= 0) {
            if (hit < range) {
                st = 0;
                mv = lo + hit;
            } else {
                break;                                    // m - lo >= range: outside [lo, hi]
            }
        }
    }
    mout[e] = mv;
    status[e] = st;
}

inline unsigned nb2(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

size_t enc_ctx_bytes() { return 256 + 2 * kCombBase * 4; }

cudaError_t launch_enc_ctx_init(const uint8_t pk[64], uint32_t *ctx, cudaStream_t s) {
    Pk64n2 p;
    for (int i = 0; i < 64; i++) p.b[i] = pk[i];
    uint32_t *tmp = nullptr;
    cudaError_t e = cudaMallocAsync((void **)&tmp, (size_t)2 * kWin * (kEnt + 1) * kPtWords * 4, s);
    if (e) return e;
    uint32_t *bases = tmp + (size_t)2 * kWin * kEnt * kPtWords;
    e = cudaMemsetAsync(ctx, 0, 256, s);
    if (!e) {
        k_comb_bases<<<1, 64, 0, s>>>(p, bases, ctx);
        e = cudaGetLastError();
    }
    if (!e) {
        k_comb_fill<<<nb2(2 * kWin * (kEnt / 16), 64), 64, 0, s>>>(bases, tmp);
        e = cudaGetLastError();
    }
    if (!e) e = launch_affine(tmp, (int64_t)2 * kWin * kEnt, ctx + 64, s);
    if (!e) {
        const uint32_t magic = kEncMagic;
        e = cudaMemcpyAsync(ctx, &magic, 4, cudaMemcpyHostToDevice, s);
        if (!e) e = cudaStreamSynchronize(s);       // `magic` lives on this stack frame
    }
    cudaFreeAsync(tmp, s);
    return e;
}

cudaError_t launch_encrypt_comb(const uint32_t *ctx, const int32_t *b, const uint8_t *r, int64_t count, uint8_t *ct,
                                cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    k_encrypt_comb<<<nb2(count, 128), 128, 0, s>>>(ctx, b, r, count, ct);
    return cudaGetLastError();
}

size_t bsgs_ctx_bytes(int log2s) { return 256 + ((size_t)2 << log2s) * 12; }

cudaError_t launch_bsgs_init(int log2s, uint32_t *ctx, cudaStream_t s) {
    const size_t nslots = (size_t)2 << log2s;
    cudaError_t e = cudaMemsetAsync(ctx, 0, 256 + nslots * 8, s);
    if (e) return e;
    const int64_t runs = (((int64_t)1 << log2s) - 1 + kBabyRun - 1) / kBabyRun;
    k_bsgs_fill<<<nb2(runs, 128), 128, 0, s>>>(ctx, log2s);
    e = cudaGetLastError();
    if (e) return e;
    k_bsgs_header<<<1, 1, 0, s>>>(ctx, log2s);
    return cudaGetLastError();
}

cudaError_t launch_decrypt_bsgs(const uint32_t x[8], const uint32_t *ctx, const uint8_t *ct, int64_t count,
                                int64_t lo, int64_t hi, int64_t *m, int32_t *status, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    uint32_t *neglo = nullptr;
    cudaError_t e = cudaMallocAsync((void **)&neglo, kPtWords * 4, s);
    if (e) return e;
    k_neg_mulG<<<1, 1, 0, s>>>(lo, neglo);
    e = cudaGetLastError();
    if (!e) {
        Sc8 xs;
        for (int i = 0; i < 8; i++) xs.k[i] = x[i];
        k_decrypt_bsgs<<<nb2(count, 64), 64, 0, s>>>(xs, ctx, ct, count, lo, hi - lo + 1, neglo, m, status);
        e = cudaGetLastError();
    }
    cudaFreeAsync(neglo, s);
    return e;
}

}  // namespace pcmm
