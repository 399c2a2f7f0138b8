// K11: IMAD-pipe microbenchmark (roofline denominator P_prod).
// Measures, per SM per clock, the sustained thread-level rate of:
//   IMAD (mad.lo.u32), IMAD.HI (mad.hi.u32), IMAD.WIDE.U32 (mad.wide.u32),
//   IADD3 (add.u32 3-input), and mixes (IMAD.WIDE + IADD3, IMAD + IADD3).
// One CTA of 1024 threads per SM (grid = #SMs), 8 independent chains per thread,
// cycles from clock64() around the timed loop.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o k11 tools/k11_imad_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 2048
#define CH 8

template <int MODE>
__global__ void __launch_bounds__(1024, 1) probe(uint32_t *out, long long *cyc, uint32_t seed) {
    uint32_t a[CH], b = seed * 2654435761u + threadIdx.x, c = seed ^ 0x9e3779b9u;
    uint64_t w[CH];
#pragma unroll
    for (int k = 0; k < CH; k++) { a[k] = threadIdx.x * (k + 3) + seed; w[k] = a[k]; }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int k = 0; k < CH; k++) {
            if (MODE == 0) {        // IMAD
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
            } else if (MODE == 1) { // IMAD.HI
                asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
            } else if (MODE == 2) { // IMAD.WIDE.U32
                asm volatile("{.reg .u32 t; cvt.u32.u64 t, %0; mad.wide.u32 %0, t, %1, %0;}" : "+l"(w[k]) : "r"(b));
            } else if (MODE == 3) { // IADD3
                uint32_t lo = (uint32_t)w[k], hi = (uint32_t)(w[k] >> 32);
                asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %1, %1, %0;" : "+r"(lo), "+r"(hi));
                w[k] = ((uint64_t)hi << 32) | lo;
            } else if (MODE == 4) { // IMAD.WIDE + IADD3 (independent)
                asm volatile("{.reg .u32 t; cvt.u32.u64 t, %0; mad.wide.u32 %0, t, %1, %0;}" : "+l"(w[k]) : "r"(b));
                asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %1, %1, %0;" : "+r"(a[k]), "+r"(c));
            } else if (MODE == 5) { // IMAD + IADD3
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
                uint32_t lo = (uint32_t)w[k], hi = (uint32_t)(w[k] >> 32);
                asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %1, %1, %0;" : "+r"(lo), "+r"(hi));
                w[k] = ((uint64_t)hi << 32) | lo;
            } else if (MODE == 6) { // add.cc / addc chain (IADD3 + IADD3.X)
                asm volatile("add.cc.u32 %0, %0, %1;\n\taddc.u32 %2, %2, %3;"
                             : "+r"(a[k]), "+r"(b) : "r"(c), "r"(c));
            } else if (MODE == 8) { // pure IMAD.WIDE.U32 (mul.wide chains, RZ addend)
                asm volatile("{.reg .u32 t, u; mov.b64 {t, u}, %0; mul.wide.u32 %0, t, u;}" : "+l"(w[k]));
            } else if (MODE == 9) { // IMAD.WIDE + independent IMAD (lo) chain
                asm volatile("{.reg .u32 t, u; mov.b64 {t, u}, %0; mul.wide.u32 %0, t, u;}" : "+l"(w[k]));
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
            } else if (MODE == 10) { // IMAD.WIDE + independent IADD3 pair
                asm volatile("{.reg .u32 t, u; mov.b64 {t, u}, %0; mul.wide.u32 %0, t, u;}" : "+l"(w[k]));
                asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %1, %1, %0;" : "+r"(a[k]), "+r"(c));
            } else if (MODE == 7) { // madc.lo.cc / madc.hi.cc chain
                asm volatile("mad.lo.cc.u32 %0, %0, %1, %2;\n\tmadc.hi.u32 %3, %0, %1, %3;"
                             : "+r"(a[k]), "+r"(b), "+r"(c), "+r"(*(uint32_t *)&w[k]));
            }
        }
    }
    long long t1 = clock64();
    uint32_t acc = b ^ c;
#pragma unroll
    for (int k = 0; k < CH; k++) acc ^= a[k] ^ (uint32_t)w[k] ^ (uint32_t)(w[k] >> 32);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char *name, double instr_per_chain_iter, int nsm, uint32_t *d_out, long long *d_cyc) {
    probe<MODE><<<nsm, 1024>>>(d_out, d_cyc, 1);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<MODE><<<nsm, 1024>>>(d_out, d_cyc, 2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long h[1024]; cudaMemcpy(h, d_cyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost);
    double mean = 0; long long mx = 0;
    for (int i = 0; i < nsm; i++) { mean += h[i]; if (h[i] > mx) mx = h[i]; }
    mean /= nsm;
    double thread_instr = 1024.0 * ITERS * CH * instr_per_chain_iter;
    double per_clk = thread_instr / mean;
    double ghz = (double)mx / (ms * 1e6);
    printf("%-28s thread-instr/clk/SM = %7.2f   (warp-instr/clk/SMSP = %.3f)  cycles=%.0f  ms=%.3f  eff_clk=%.3f GHz\n",
           name, per_clk, per_clk / 128.0, mean, ms, ghz);
}

int main() {
    int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
    int nsm = p.multiProcessorCount;
    printf("device %s  SMs=%d  cc=%d.%d\n", p.name, nsm, p.major, p.minor);
    uint32_t *d_out; long long *d_cyc;
    cudaMalloc(&d_out, sizeof(uint32_t) * nsm * 1024);
    cudaMalloc(&d_cyc, sizeof(long long) * nsm);
    run<0>("IMAD (mad.lo)", 1, nsm, d_out, d_cyc);
    run<1>("IMAD.HI (mad.hi)", 1, nsm, d_out, d_cyc);
    run<2>("IMAD.WIDE.U32 (mad.wide)", 1, nsm, d_out, d_cyc);
    run<3>("IADD3 (2x add.u32)", 2, nsm, d_out, d_cyc);
    run<4>("WIDE + 2 IADD (total instr)", 3, nsm, d_out, d_cyc);
    run<5>("IMAD + 2 IADD (total instr)", 3, nsm, d_out, d_cyc);
    run<6>("add.cc+addc (total instr)", 2, nsm, d_out, d_cyc);
    run<7>("mad.lo.cc+madc.hi (ptx)", 2, nsm, d_out, d_cyc);
    run<8>("IMAD.WIDE pure (mul.wide)", 1, nsm, d_out, d_cyc);
    run<9>("WIDE + IMAD (total instr)", 2, nsm, d_out, d_cyc);
    run<10>("WIDE + 2 IADD3 (total instr)", 3, nsm, d_out, d_cyc);
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
