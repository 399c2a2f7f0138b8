// stepprobe.cu -- standalone probe of the accumulate step's instruction schedule (run on the GPU box):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2504_14497_b200/csrc -o /tmp/stepprobe tools/stepprobe.cu
// A loop of XYZZ + affine mixed additions on register-resident operands (no memory), in several
// orderings of the ten field products, at the occupancy of k_accum (3 CTAs of 128 threads per SM) and
// others.  Variants:
//   0  the step as jac.cuh xyzz_add_aff_pipe has it (groups {S2, PP} {R^2, PPP, Q, ZZ3} {R D, Y PPP, ZZZ3, U2'})
//   1  the same products as one chain PP, S2, PPP, Q, ZZ3, R^2, Y PPP, ZZZ3, U2', R D, each product's
//      operand rows "tied" (a data dependency through an opaque zero) to the end of the previous
//      product's rows and to the result of the one before it, so that ptxas cannot issue all
//      IMAD.WIDE first and leave the carry-chain tails for the end
//   2  variant 1's order without ties
// Prints G fp_mul-equivalents/s (9.125 per step) and the fraction of the 145.4 G IMAD roofline.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "fp.cuh"

namespace pcmm {

#ifdef __CUDA_ARCH__
// fe_prod_eo with a tie: b.v[0] |= tin (tin = 0 at run time); rows_done = a word written by the last row
__device__ __forceinline__ void fe_prod_eo_tie(uint32_t T[16], const fe &a, const fe &b, uint32_t tin, uint32_t &rows_done) {
    uint32_t E[16], O[16];
    const uint32_t b0 = b.v[0] | tin;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const uint64_t pe = (uint64_t)a.v[2 * j] * b0;
        const uint64_t po = (uint64_t)a.v[2 * j + 1] * b0;
        E[2 * j] = (uint32_t)pe;
        E[2 * j + 1] = (uint32_t)(pe >> 32);
        O[2 * j] = (uint32_t)po;
        O[2 * j + 1] = (uint32_t)(po >> 32);
    }
#pragma unroll
    for (int k = 8; k < 16; k++) {
        E[k] = 0;
        O[k] = 0;
    }
    const uint32_t a0 = a.v[0], a1 = a.v[1], a2 = a.v[2], a3 = a.v[3];
    const uint32_t a4 = a.v[4], a5 = a.v[5], a6 = a.v[6], a7 = a.v[7];
#pragma unroll
    for (int i = 1; i < 8; i++) {
        const uint32_t bi = b.v[i];
        if (i & 1) {
            PCMM_CHAIN4C(O[i - 1], O[i], O[i + 1], O[i + 2], O[i + 3], O[i + 4], O[i + 5], O[i + 6], O[i + 7], a0, a2,
                         a4, a6, bi);
            if (i < 7) {
                PCMM_CHAIN4C(E[i + 1], E[i + 2], E[i + 3], E[i + 4], E[i + 5], E[i + 6], E[i + 7], E[i + 8],
                             E[(i + 9) & 15], a1, a3, a5, a7, bi);
            } else {
                PCMM_CHAIN4(E[8], E[9], E[10], E[11], E[12], E[13], E[14], E[15], a1, a3, a5, a7, bi);
            }
        } else {
            PCMM_CHAIN4C(E[i], E[i + 1], E[i + 2], E[i + 3], E[i + 4], E[i + 5], E[i + 6], E[i + 7], E[i + 8], a0, a2,
                         a4, a6, bi);
            PCMM_CHAIN4C(O[i], O[i + 1], O[i + 2], O[i + 3], O[i + 4], O[i + 5], O[i + 6], O[i + 7], O[i + 8], a1, a3,
                         a5, a7, bi);
        }
    }
    rows_done = E[15] | O[14];
    T[0] = E[0];
    asm("add.cc.u32 %0, %15, %30;\n\t"
        "addc.cc.u32 %1, %16, %31;\n\t"
        "addc.cc.u32 %2, %17, %32;\n\t"
        "addc.cc.u32 %3, %18, %33;\n\t"
        "addc.cc.u32 %4, %19, %34;\n\t"
        "addc.cc.u32 %5, %20, %35;\n\t"
        "addc.cc.u32 %6, %21, %36;\n\t"
        "addc.cc.u32 %7, %22, %37;\n\t"
        "addc.cc.u32 %8, %23, %38;\n\t"
        "addc.cc.u32 %9, %24, %39;\n\t"
        "addc.cc.u32 %10, %25, %40;\n\t"
        "addc.cc.u32 %11, %26, %41;\n\t"
        "addc.cc.u32 %12, %27, %42;\n\t"
        "addc.cc.u32 %13, %28, %43;\n\t"
        "addc.u32 %14, %29, %44;"
        : "=r"(T[1]), "=r"(T[2]), "=r"(T[3]), "=r"(T[4]), "=r"(T[5]), "=r"(T[6]), "=r"(T[7]), "=r"(T[8]),
          "=r"(T[9]), "=r"(T[10]), "=r"(T[11]), "=r"(T[12]), "=r"(T[13]), "=r"(T[14]), "=r"(T[15])
        : "r"(E[1]), "r"(E[2]), "r"(E[3]), "r"(E[4]), "r"(E[5]), "r"(E[6]), "r"(E[7]), "r"(E[8]), "r"(E[9]),
          "r"(E[10]), "r"(E[11]), "r"(E[12]), "r"(E[13]), "r"(E[14]), "r"(E[15]),
          "r"(O[0]), "r"(O[1]), "r"(O[2]), "r"(O[3]), "r"(O[4]), "r"(O[5]), "r"(O[6]), "r"(O[7]), "r"(O[8]),
          "r"(O[9]), "r"(O[10]), "r"(O[11]), "r"(O[12]), "r"(O[13]), "r"(O[14]));
}

// the chain state: rd = rows_done word of the previous product, res = a result word of the one before it
struct tie_t {
    uint32_t z, rd, res, res_prev;
};

template <bool TIE>
__device__ __forceinline__ void mul_t(fe &r, const fe &a, const fe &b, tie_t &t) {
    if (TIE) {
        uint32_t T[16], rd;
        fe_prod_eo_tie(T, a, b, (t.rd | t.res_prev) & t.z, rd);
        fe_redc_fast(r, T);
        t.rd = rd;
        t.res_prev = t.res;
        t.res = r.v[7];
    } else {
        fe_mul_fast(r, a, b);
    }
}

template <bool TIE>
__device__ __forceinline__ void sqr_t(fe &r, const fe &a, tie_t &t) {
    if (TIE) {
        // the tie goes through a0 (row 0 of the cross products)
        fe a2 = a;
        a2.v[0] |= (t.rd | t.res_prev) & t.z;
        fe_sqr_fast(r, a2);
        t.rd = r.v[0];                 // no access to the rows: the result stands in
        t.res_prev = t.res;
        t.res = r.v[7];
    } else {
        fe_sqr_fast(r, a);
    }
}

__device__ __noinline__ void slow_path(fe &X, fe &Y) {
    fe_add(X, X, Y);
}
#endif

template <int V, int MB>
__global__ void __launch_bounds__(128, MB) k_step(int iters, uint32_t z, uint32_t *__restrict__ out) {
#ifdef __CUDA_ARCH__
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    fe X, Y, ZZ, ZZZ, x2, y2, xn, U2;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        X.v[i] = (t * 2654435761u + i * 40503u) & 0x7fffffffu;
        Y.v[i] = (t * 97u + i * 131u + 7u) & 0x7fffffffu;
        ZZ.v[i] = (t * 31u + i * 17u + 3u) & 0x7fffffffu;
        ZZZ.v[i] = (t * 131u + i * 1031u + 5u) & 0x7fffffffu;
        x2.v[i] = (t * 7u + i * 3u + 11u) & 0x7fffffffu;
        y2.v[i] = (t * 13u + i * 5u + 1u) & 0x7fffffffu;
    }
    xn = x2;
    fe_mul(U2, x2, ZZ);
    tie_t tie{z, 0, 0, 0};
    for (int it = 0; it < iters; it++) {
        fe P, R;
        fe_sub(P, U2, X);
        if (fe_is_zero(P)) {
            slow_path(X, Y);
            continue;
        }
        if (V == 0) {
            fe S2, PP, R2, PPP, Q, ZZ3, RD, YP, ZZZ3, U2n;
            fe_mul_fast(S2, y2, ZZZ);
            fe_sqr_fast(PP, P);
            fe_sub(R, S2, Y);
            fe_sqr_fast(R2, R);
            fe_mul_fast(PPP, P, PP);
            fe_mul_fast(Q, X, PP);
            fe_mul_fast(ZZ3, ZZ, PP);
            fe X3, Q2, D;
            fe_add(Q2, Q, Q);
            fe_sub(X3, R2, PPP);
            fe_sub(X3, X3, Q2);
            fe_sub(D, Q, X3);
            fe_mul_fast(RD, R, D);
            fe_mul_fast(YP, Y, PPP);
            fe_mul_fast(ZZZ3, ZZZ, PPP);
            fe_mul_fast(U2n, xn, ZZ3);
            fe_sub(Y, RD, YP);
            X = X3;
            ZZ = ZZ3;
            ZZZ = ZZZ3;
            U2 = U2n;
        } else {
            constexpr bool TIE = (V == 1);
            fe S2, PP, R2, PPP, Q, ZZ3, RD, YP, ZZZ3, U2n;
            sqr_t<TIE>(PP, P, tie);
            mul_t<TIE>(S2, y2, ZZZ, tie);
            mul_t<TIE>(PPP, P, PP, tie);
            mul_t<TIE>(Q, X, PP, tie);
            fe_sub(R, S2, Y);
            mul_t<TIE>(ZZ3, ZZ, PP, tie);
            sqr_t<TIE>(R2, R, tie);
            mul_t<TIE>(YP, Y, PPP, tie);
            mul_t<TIE>(ZZZ3, ZZZ, PPP, tie);
            fe X3, Q2, D;
            fe_add(Q2, Q, Q);
            fe_sub(X3, R2, PPP);
            fe_sub(X3, X3, Q2);
            fe_sub(D, Q, X3);
            mul_t<TIE>(U2n, xn, ZZ3, tie);
            mul_t<TIE>(RD, R, D, tie);
            fe_sub(Y, RD, YP);
            X = X3;
            ZZ = ZZ3;
            ZZZ = ZZZ3;
            U2 = U2n;
        }
        // rotate the entry so that successive steps differ
        fe tmp = x2;
        x2 = y2;
        y2 = tmp;
        xn = x2;
    }
#pragma unroll
    for (int i = 0; i < 8; i++) out[t * 8 + i] = X.v[i] ^ Y.v[i] ^ ZZ.v[i] ^ ZZZ.v[i] ^ U2.v[i];
#endif
}

}  // namespace pcmm

template <int V, int MB>
static void run(const char *name, int iters) {
    const int ctas_per_sm = MB;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * ctas_per_sm;
    uint32_t *out;
    cudaMalloc(&out, (size_t)blocks * 128 * 8 * 4);
    // dynamic shared memory limits the residency to ctas_per_sm
    const int smem = (200 * 1024) / ctas_per_sm - 2048;
    cudaFuncSetAttribute(pcmm::k_step<V, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pcmm::k_step<V, MB>, 128, smem);
    pcmm::k_step<V, MB><<<blocks, 128, smem>>>(16, 0, out);
    cudaDeviceSynchronize();
    cudaEvent_t s, e;
    cudaEventCreate(&s);
    cudaEventCreate(&e);
    float best = 1e30f;
    for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(s);
        pcmm::k_step<V, MB><<<blocks, 128, smem>>>(iters, 0, out);
        cudaEventRecord(e);
        cudaEventSynchronize(e);
        float ms;
        cudaEventElapsedTime(&ms, s, e);
        if (ms < best) best = ms;
    }
    const double steps = (double)blocks * 128 * iters;
    const double g = steps * 9.125 / best / 1e6;
    printf("%-28s ctas/SM %d (occ %d)  %8.3f ms  %7.2f G fp_mul-eq/s  frac %.3f  err %s\n", name, ctas_per_sm, occ, best,
           g, g / 145.41, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main(int argc, char **argv) {
    const int iters = argc > 1 ? atoi(argv[1]) : 2000;
    run<0, 2>("v0 groups (as k_accum)", iters);
    run<2, 2>("v2 chain order, no ties", iters);
    run<1, 2>("v1 chain order + ties", iters);
    run<0, 3>("v0 groups (as k_accum)", iters);
    run<2, 3>("v2 chain order, no ties", iters);
    run<1, 3>("v1 chain order + ties", iters);
    run<0, 4>("v0 groups (as k_accum)", iters);
    run<2, 4>("v2 chain order, no ties", iters);
    run<1, 4>("v1 chain order + ties", iters);
    return 0;
}
