// K12: throughput of the exact SASS forms the field product uses (run on the GPU box):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/k12 tools/k12_chain_probe.cu && /tmp/k12
// K11 (k11_imad_probe.cu) measured IMAD.WIDE.U32 with an RZ addend at 32 / clk / SM; its "with
// addend" and "+ IADD3" modes were rewritten by ptxas (adds moved onto the FMA pipe as IMAD.IADD),
// so they do not isolate what fe_prod_eo issues.  Modes here (8 or more independent accumulator
// sets per thread, accumulators live across iterations, multiplicands loop-invariant):
//   0  IMAD.WIDE.U32 R, R, R, R      64-bit register addend, no carry          (mad.wide.u32)
//   1  carry chains of 4: IMAD.WIDE.U32, 3 x IMAD.WIDE.U32.X, IADD3.X  (mad.lo.cc / madc.hi.cc: fe_prod_eo's rows)
//   2  mode 1 without the closing addc (pure IMAD.WIDE(.X))
//   3  mode 1 + 6 IADD3.X-chain ALU instructions per chain (the product's ALU : IMAD.WIDE ratio of 1.5)
//   4  add.cc / addc.cc chains of 8 alone (IADD3 / IADD3.X)
//   5  mode 0 + 6 ALU chain instructions per 4 IMAD.WIDE
// Prints IMAD.WIDE per clk per SM and total warp-instructions per clk per SMSP.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CHAIN4C(d0, d1, d2, d3, d4, d5, d6, d7, c, x0, x1, x2, x3, y)                              \
    asm volatile("mad.lo.cc.u32 %0, %9, %13, %0;\n\t"                                              \
                 "madc.hi.cc.u32 %1, %9, %13, %1;\n\t"                                             \
                 "madc.lo.cc.u32 %2, %10, %13, %2;\n\t"                                            \
                 "madc.hi.cc.u32 %3, %10, %13, %3;\n\t"                                            \
                 "madc.lo.cc.u32 %4, %11, %13, %4;\n\t"                                            \
                 "madc.hi.cc.u32 %5, %11, %13, %5;\n\t"                                            \
                 "madc.lo.cc.u32 %6, %12, %13, %6;\n\t"                                            \
                 "madc.hi.cc.u32 %7, %12, %13, %7;\n\t"                                            \
                 "addc.u32 %8, %8, 0;"                                                              \
                 : "+r"(d0), "+r"(d1), "+r"(d2), "+r"(d3), "+r"(d4), "+r"(d5), "+r"(d6), "+r"(d7), "+r"(c) \
                 : "r"(x0), "r"(x1), "r"(x2), "r"(x3), "r"(y))
#define CHAIN4(d0, d1, d2, d3, d4, d5, d6, d7, x0, x1, x2, x3, y)                                  \
    asm volatile("mad.lo.cc.u32 %0, %8, %12, %0;\n\t"                                              \
                 "madc.hi.cc.u32 %1, %8, %12, %1;\n\t"                                             \
                 "madc.lo.cc.u32 %2, %9, %12, %2;\n\t"                                             \
                 "madc.hi.cc.u32 %3, %9, %12, %3;\n\t"                                             \
                 "madc.lo.cc.u32 %4, %10, %12, %4;\n\t"                                            \
                 "madc.hi.cc.u32 %5, %10, %12, %5;\n\t"                                            \
                 "madc.lo.cc.u32 %6, %11, %12, %6;\n\t"                                            \
                 "madc.hi.u32 %7, %11, %12, %7;"                                                   \
                 : "+r"(d0), "+r"(d1), "+r"(d2), "+r"(d3), "+r"(d4), "+r"(d5), "+r"(d6), "+r"(d7)  \
                 : "r"(x0), "r"(x1), "r"(x2), "r"(x3), "r"(y))
#define ALU6(e0, e1, e2, e3, e4, e5, f)                                                            \
    asm volatile("add.cc.u32 %0, %0, %6;\n\t"                                                      \
                 "addc.cc.u32 %1, %1, %0;\n\t"                                                     \
                 "addc.cc.u32 %2, %2, %1;\n\t"                                                     \
                 "addc.cc.u32 %3, %3, %2;\n\t"                                                     \
                 "addc.cc.u32 %4, %4, %3;\n\t"                                                     \
                 "addc.u32 %5, %5, %4;"                                                            \
                 : "+r"(e0), "+r"(e1), "+r"(e2), "+r"(e3), "+r"(e4), "+r"(e5)                      \
                 : "r"(f))

// six independent (no carry, no mutual dependency) ALU instructions: 3-input adds / logic ops
#define IADD6(e0, e1, e2, e3, e4, e5, f)                                                           \
    asm volatile("add.u32 %0, %0, %6;\n\tadd.u32 %1, %1, %6;\n\tadd.u32 %2, %2, %6;\n\t"            \
                 "add.u32 %3, %3, %6;\n\tadd.u32 %4, %4, %6;\n\tadd.u32 %5, %5, %6;"                 \
                 : "+r"(e0), "+r"(e1), "+r"(e2), "+r"(e3), "+r"(e4), "+r"(e5)                      \
                 : "r"(f))
#define LOP6(e0, e1, e2, e3, e4, e5, f)                                                            \
    asm volatile("lop3.b32 %0, %0, %6, %1, 0x96;\n\tlop3.b32 %1, %1, %6, %2, 0x96;\n\t"             \
                 "lop3.b32 %2, %2, %6, %3, 0x96;\n\tlop3.b32 %3, %3, %6, %4, 0x96;\n\t"             \
                 "lop3.b32 %4, %4, %6, %5, 0x96;\n\tlop3.b32 %5, %5, %6, %0, 0x96;"                  \
                 : "+r"(e0), "+r"(e1), "+r"(e2), "+r"(e3), "+r"(e4), "+r"(e5)                      \
                 : "r"(f))

constexpr int ITERS = 512;
#ifndef K12_NC
#define K12_NC 4
#endif
constexpr int NC = K12_NC;     // accumulator sets per thread

template <int MODE, int MB = 2>
__global__ void __launch_bounds__(256, MB) probe(uint32_t *out, long long *cyc, uint32_t seed) {
    uint32_t d[NC][9], e[NC][6];
    uint64_t w[NC][4];
    const uint32_t t = threadIdx.x + seed;
    uint32_t x0 = t * 2654435761u | 1u, x1 = t * 40503u + 7u, x2 = t * 97u + 3u, x3 = t * 131u + 9u, y = t * 31u + 5u;
#pragma unroll
    for (int k = 0; k < NC; k++) {
#pragma unroll
        for (int i = 0; i < 9; i++) d[k][i] = t + k * 17 + i;
#pragma unroll
        for (int i = 0; i < 6; i++) e[k][i] = t * 3 + k * 5 + i;
#pragma unroll
        for (int i = 0; i < 4; i++) w[k][i] = ((uint64_t)t << 32) + k * 4 + i;
    }
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < ITERS; it++) {
        y += 0x9e3779b9u;          // the multiplier changes every iteration: the products cannot be hoisted
#pragma unroll
        for (int k = 0; k < NC; k++) {
            if (MODE == 0 || MODE == 5) {
                // the multiplicand is another set's low word: nothing to hoist or share
#pragma unroll
                for (int i = 0; i < 4; i++)
                    asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[k][i]) : "r"((uint32_t)w[(k + 1) % NC][(i + 1) & 3]), "r"(y));
                if (MODE == 5) ALU6(e[k][0], e[k][1], e[k][2], e[k][3], e[k][4], e[k][5], y);
            } else if (MODE == 1 || MODE == 3) {
                CHAIN4C(d[k][0], d[k][1], d[k][2], d[k][3], d[k][4], d[k][5], d[k][6], d[k][7], d[k][8], x0, x1, x2, x3, y);
                if (MODE == 3) ALU6(e[k][0], e[k][1], e[k][2], e[k][3], e[k][4], e[k][5], y);
            } else if (MODE == 2) {
                CHAIN4(d[k][0], d[k][1], d[k][2], d[k][3], d[k][4], d[k][5], d[k][6], d[k][7], x0, x1, x2, x3, y);
            } else if (MODE == 4) {
                ALU6(e[k][0], e[k][1], e[k][2], e[k][3], e[k][4], e[k][5], y);
            } else if (MODE == 6) {
                CHAIN4(d[k][0], d[k][1], d[k][2], d[k][3], d[k][4], d[k][5], d[k][6], d[k][7], x0, x1, x2, x3, y);
                IADD6(e[k][0], e[k][1], e[k][2], e[k][3], e[k][4], e[k][5], y);
            } else if (MODE == 7) {
                CHAIN4(d[k][0], d[k][1], d[k][2], d[k][3], d[k][4], d[k][5], d[k][6], d[k][7], x0, x1, x2, x3, y);
                LOP6(e[k][0], e[k][1], e[k][2], e[k][3], e[k][4], e[k][5], y);
            } else if (MODE == 8) {
                IADD6(e[k][0], e[k][1], e[k][2], e[k][3], e[k][4], e[k][5], y);
            } else if (MODE == 9) {
                LOP6(e[k][0], e[k][1], e[k][2], e[k][3], e[k][4], e[k][5], y);
            } else if (MODE == 10) {
                // independent IMAD.WIDE.U32 R, R, R, RZ with distinct source registers
                asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w[k][0]) : "r"(d[k][0]), "r"(y));
                asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w[k][1]) : "r"(d[k][1]), "r"(y));
                asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w[k][2]) : "r"(d[k][2]), "r"(y));
                asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w[k][3]) : "r"(d[k][3]), "r"(y));
                d[k][0] ^= (uint32_t)w[k][3]; d[k][1] ^= (uint32_t)(w[k][0] >> 32);
                d[k][2] ^= (uint32_t)w[k][1]; d[k][3] ^= (uint32_t)(w[k][2] >> 32);
            }
        }
    }
    const long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < NC; k++) {
#pragma unroll
        for (int i = 0; i < 9; i++) acc ^= d[k][i];
#pragma unroll
        for (int i = 0; i < 6; i++) acc ^= e[k][i];
#pragma unroll
        for (int i = 0; i < 4; i++) acc ^= (uint32_t)w[k][i] ^ (uint32_t)(w[k][i] >> 32);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE, int MB = 2>
static void run(const char *name, double wide_per_set, double instr_per_set, int nsm, uint32_t *d_out, long long *d_cyc) {
    const int blocks = nsm * MB;
    probe<MODE, MB><<<blocks, 256>>>(d_out, d_cyc, 1);
    cudaDeviceSynchronize();
    probe<MODE, MB><<<blocks, 256>>>(d_out, d_cyc, 2);
    cudaDeviceSynchronize();
    static long long h[4096];
    cudaMemcpy(h, d_cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < blocks; i++) mean += h[i];
    mean /= blocks;
    // MB CTAs of 256 threads per SM run concurrently over `mean` cycles
    const double sets = 256.0 * MB * ITERS * NC;
    printf("%-44s IMAD.WIDE/clk/SM = %6.2f   warp-instr/clk/SMSP = %.3f   (cycles %.0f)  %s\n", name,
           sets * wide_per_set / mean, sets * instr_per_set / mean / 128.0, mean, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int nsm = p.multiProcessorCount;
    uint32_t *d_out;
    long long *d_cyc;
    cudaMalloc(&d_out, sizeof(uint32_t) * nsm * 8 * 256);
    cudaMalloc(&d_cyc, sizeof(long long) * nsm * 8);
    run<0>("0 IMAD.WIDE R,R,R,R (64-bit addend)", 4, 4, nsm, d_out, d_cyc);
    run<1>("1 chain4 + addc (fe_prod_eo row)", 4, 5, nsm, d_out, d_cyc);
    run<2>("2 chain4 (IMAD.WIDE + 3 IMAD.WIDE.X)", 4, 4, nsm, d_out, d_cyc);
    run<3>("3 chain4 + addc + 6 IADD3.X", 4, 11, nsm, d_out, d_cyc);
    run<4>("4 6 IADD3(.X) chain alone", 0, 6, nsm, d_out, d_cyc);
    run<5>("5 4 IMAD.WIDE (addend) + 6 IADD3.X", 4, 10, nsm, d_out, d_cyc);
    run<6>("6 chain4 + 6 independent IADD", 4, 10, nsm, d_out, d_cyc);
    run<7>("7 chain4 + 6 LOP3", 4, 10, nsm, d_out, d_cyc);
    run<8>("8 6 independent IADD alone", 0, 6, nsm, d_out, d_cyc);
    run<9>("9 6 LOP3 alone", 0, 6, nsm, d_out, d_cyc);
    run<10>("10 4 IMAD.WIDE RZ + 4 LOP3", 4, 8, nsm, d_out, d_cyc);
    run<2, 4>("2 chain4, 32 warps/SM", 4, 4, nsm, d_out, d_cyc);
    run<1, 4>("1 chain4 + addc, 32 warps/SM", 4, 5, nsm, d_out, d_cyc);
    run<3, 4>("3 chain4 + addc + 6 IADD3.X, 32 warps/SM", 4, 11, nsm, d_out, d_cyc);
    run<4, 4>("4 6 IADD3(.X) chain alone, 32 warps/SM", 0, 6, nsm, d_out, d_cyc);
    run<2, 1>("2 chain4, 8 warps/SM", 4, 4, nsm, d_out, d_cyc);
#if K12_NC <= 2
    run<2, 6>("2 chain4, 48 warps/SM", 4, 4, nsm, d_out, d_cyc);
    run<2, 8>("2 chain4, 64 warps/SM", 4, 4, nsm, d_out, d_cyc);
    run<1, 8>("1 chain4 + addc, 64 warps/SM", 4, 5, nsm, d_out, d_cyc);
#endif
    return 0;
}
