// internal.h -- shared declarations between kernels.cu and api.cu (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace pcmm {

// Per-column compression plan of Alg. 2 for w <= 8, N <= 4.
// n[w-1] = |a^(w)| (sorted distinct nonzero values at level w, DESIGN R1);
// sN = the level-N values (the multipliers of Alg. 3 line 5; |v| < 640);
// ptr[w-1][e] = index in a^(w+1) of element e of the differenced level-w vector
// (the tracking pointer used by the un-sort / re-insert of level w+1 -> w).
constexpr int kPlanCap = 256;         // |a^(1)| <= 255 for int8 plaintexts
// coz > 0: the column's table is the chain P, 2P, ..., coz P (k_tables_coz): unsigned columns with
// a^(1) = {1..coz} (levels 2..N = {1}), or, sgn = 1, signed columns whose magnitudes are {1..coz}
// (each in either sign; R10b: the entry of -v is the negated entry of v).  bm1 = the level-1
// presence bitmap (bit v + 128), from which k_tables_coz finds the slot of +-v.
struct ColPlan {
    int16_t n[4];
    int16_t coz, sgn;
    int16_t sN[kPlanCap];
    uint8_t ptr[3][kPlanCap];
    uint32_t bm1[12];
};
constexpr int kPtWords = 24;          // X, Y, Z x 8 limbs
constexpr int kAffWords = 16;         // affine table entry: x, y x 8 limbs (identity: x = all ones)
// table slots per (k, j, c) = 2^w (slot 0 = infinity, slots 1..|a^(1)| = entries)
inline int table_slots(int w) { return 1 << (w < 1 ? 1 : w); }

// status word bits (workspace offset 0)
constexpr int kStatusBound = 1;
constexpr int kStatusCurve = 2;

struct Launch {
    cudaStream_t stream;
};

// profiling (api.cu)
void prof_begin(const char *name, cudaStream_t s);
void prof_end(cudaStream_t s);

// kernels.cu launchers; each returns cudaGetLastError()
cudaError_t launch_import(const uint8_t *ct, int64_t count, uint32_t *soa, int *status, cudaStream_t s);
cudaError_t launch_plan(const int8_t *A, int m, int n, int w, int is_signed, int N, ColPlan *plans, uint8_t *rank,
                        int *status, cudaStream_t s);
cudaError_t launch_tables(const uint32_t *bsoa, const ColPlan *plans, int n, int l, int N, int slots, int maxup,
                          int is_signed, uint32_t *tables, uint32_t *scratch, cudaStream_t s,
                          int skip_fast = 0,    // skip_fast: consecutive columns left to k_tables_fast
                          int maxlen = 0,       // min(m, 2^w - 1): long tables of few launches -> block scan
                          const int *general = nullptr);   // k_plan's flag: no general column -> k_tables exits
// homogeneous tables [c][k][j][slot][24] -> affine tables [c][k][j][slot][16] (batch inversion)
// plans != nullptr: entries of consecutive columns (built by k_tables_fast) are skipped
// plans != nullptr (byte path): per-column entry kinds (slot 0 / unused slots -> identity markers without
// reading the tables; fast != 0: consecutive columns come from k_tables_fast)
// general != nullptr with fast = 2: device flag written by k_plan (some column is not consecutive); 0 -> no work
cudaError_t launch_affine(const uint32_t *tables, int64_t entries, uint32_t *atables, cudaStream_t s,
                          const ColPlan *plans = nullptr, int n = 0, int l = 0, int S = 0, int N = 0, int fast = 0,
                          const int *general = nullptr);
// consecutive columns (s^(1) = {1..n1}): XYZZ prefix sums + fused affine conversion
// (k_tables_fast); k_tables skips them when tables_fast_on()
int tables_fast_on();
cudaError_t launch_tables_fast(const uint32_t *bsoa, const ColPlan *plans, int n, int l, int N, int slots,
                               uint32_t *tables, uint32_t *atables, cudaStream_t s);
// consecutive columns, tables and affine conversion in one kernel (taff.cu k_tables_coz: co-Z
// prefix chain, one CTA-shared inversion); k_affine then skips those columns (fast = 2).
// tables: the projective table region (per-entry X, Y, lambda parked there)
cudaError_t launch_tables_coz(const uint32_t *bsoa, const ColPlan *plans, int n, int l, int N, int slots,
                              uint32_t *tables, uint32_t *atables, cudaStream_t s);
int tables_coz_mode();   // PCMM_TABLES_COZ: 0 off, 1 auto (default), 2 always
// general columns, tables and affine conversion in one kernel (tgz.cu k_tables_gz); skip_chain:
// chain columns are left to k_tables_coz.  tables: the projective region (X, Y, f parked per entry)
cudaError_t launch_tables_gz(const uint32_t *bsoa, const ColPlan *plans, int n, int l, int N, int slots, int maxup,
                             uint32_t *tables, uint32_t *atables, int skip_chain, const int *general,
                             cudaStream_t s);
int tables_gz_mode();    // PCMM_TABLES_GZ: 0 off (k_tables + k_affine), 1 auto (default), 2 always
// upper-level reconstruction scratch per (c, k, j): two ping-pong levels of
// kMaxUpper entries (levels >= 2 have <= 7 entries for w <= 4, <= 28 for w <= 8)
inline int max_upper(int w) { return w <= 4 ? 8 : 32; }
// acc_in (ksplit = 1 only): start each accumulator from the running output in `out` (k-chunked byte path)
cudaError_t launch_accum_global(const uint32_t *tables, const uint8_t *rank, int m, int n, int l, int slots,
                                int ksplit, uint32_t *out, int64_t out_stride_split, cudaStream_t s, int acc_in = 0);
int accum_global_ctas_per_sm();
// rows of every 128-row block sorted by nonzero count per k-split (perm: ksplit x ceil(m/128) x 128 ints),
// and the gather accumulate kernel that takes its rows from that permutation (hot.cu k_rowperm, k_accum_g2)
cudaError_t launch_rowperm(const uint8_t *rank, int m, int n, int ksplit, int *perm, cudaStream_t s);
cudaError_t launch_accum_sorted(const uint32_t *tables, const uint8_t *rank, int m, int n, int l, int slots,
                                int ksplit, uint32_t *out, int64_t out_stride_split, cudaStream_t s, int acc_in,
                                const int *perm, int pipe);
cudaError_t launch_accum(const uint32_t *tables, const uint8_t *rank, int m, int n, int l, int slots, int ksplit,
                         uint32_t *out, int64_t out_stride_split, cudaStream_t s, int acc_in = 0);
// out = sum of the ksplit partial sums (+ out itself when accumulate: the byte path's k-chunks)
cudaError_t launch_reduce_splits(const uint32_t *partial, int ksplit, int64_t count, uint32_t *out, cudaStream_t s,
                                 bool accumulate = false);
cudaError_t launch_schoolbook(const int8_t *A, int m, int n, int l, int w, int is_signed, const uint32_t *bsoa,
                              uint32_t *out, int *status, cudaStream_t s);
// the XYZZ schoolbook (school.cu k_school_xyzz), launch_schoolbook with PCMM_SCHOOL_XYZZ=1
cudaError_t launch_schoolbook_xyzz(const int8_t *A, int m, int n, int l, int w, int is_signed, const uint32_t *bsoa,
                                   uint32_t *out, int *status, cudaStream_t s);
cudaError_t launch_normalize(const uint32_t *proj, int64_t count, uint8_t *ct, cudaStream_t s);
cudaError_t launch_encrypt(const uint8_t *pk64, const int32_t *b, const uint8_t *r, int64_t count, uint8_t *ct,
                           cudaStream_t s);
cudaError_t launch_pubkey(const uint32_t x[8], uint8_t *out64_d, cudaStream_t s);
cudaError_t launch_test_field(int op, const uint8_t *a, const uint8_t *b, uint8_t *out, int64_t count,
                              cudaStream_t s);
cudaError_t launch_test_point(int op, const uint8_t *p, const uint8_t *q, const int32_t *v, uint8_t *out,
                              int64_t count, cudaStream_t s);
cudaError_t launch_bench_fp_mul(int variant, int blocks, int threads, int iters, uint32_t *out, cudaStream_t s);
int num_sms();
cudaError_t run_strassen(const void *A, int a_is_i32, int m, int n, int l, int w, int is_signed,
                         const uint32_t *bsoa, int leaf, uint32_t *out, int *status, cudaStream_t s);
int accum_ctas_per_sm(int slots, int rows);   // resident k_accum CTAs per SM (rows per CTA: accum_rows(m))
// NEXT-4 (paillier.cu): PC-MM mod n^2, L 32-bit limbs; off[] = workspace offsets
// {consts (one, R^2, unit: 3L words), Montgomery ciphertexts, plans, rank, tables, scratch}
bool paillier_limbs_ok(int L);
cudaError_t run_paillier(int path, const uint8_t *A, int m, int n, int l, int w, int N, int L, const uint32_t *Nh,
                         const uint32_t *ctB, uint32_t *ctC, uint8_t *ws, const size_t *off, int S, int maxup,
                         cudaStream_t s);
// NEXT-2 (next2.cu): fixed-base comb encryption context, BSGS decryption context
size_t enc_ctx_bytes();
cudaError_t launch_enc_ctx_init(const uint8_t pk[64], uint32_t *ctx, cudaStream_t s);   // synchronises s
cudaError_t launch_encrypt_comb(const uint32_t *ctx, const int32_t *b, const uint8_t *r, int64_t count, uint8_t *ct,
                                cudaStream_t s);
size_t bsgs_ctx_bytes(int log2s);
cudaError_t launch_bsgs_init(int log2s, uint32_t *ctx, cudaStream_t s);
cudaError_t launch_decrypt_bsgs(const uint32_t x[8], const uint32_t *ctx, const uint8_t *ct, int64_t count,
                                int64_t lo, int64_t hi, int64_t *m, int32_t *status, cudaStream_t s);
// wide-plaintext path (wide.cu, hot.cu k_accum_gw): t <= 16, int32 A, uint16 rank, k-chunked tables
int wide_plan_p2(int m);
size_t wide_plan_smem(int m, int cap);
cudaError_t launch_plan_wide(const int32_t *A, int m, int n, int w, int is_signed, int N, int cap, int32_t *pn,
                             int32_t *psN, uint16_t *pptr, uint16_t *rank, int *status, cudaStream_t s);
cudaError_t launch_tables_wide(const uint32_t *bsoa, const int32_t *pn, const int32_t *psN, const uint16_t *pptr,
                               int n, int l, int N, int cap, int S, int k0, int kc, uint32_t *tables,
                               uint32_t *scratch, cudaStream_t s);
// few tables (2 kc l small): one CTA per table, block-scan prefix sums (latency)
cudaError_t launch_tables_wide_scan(const uint32_t *bsoa, const int32_t *pn, const int32_t *psN,
                                    const uint16_t *pptr, int n, int l, int N, int cap, int S, int k0, int kc,
                                    uint32_t *tables, uint32_t *scratch, cudaStream_t s);
cudaError_t launch_accum_wide(const uint32_t *atables, const uint16_t *rank, int m, int l, int S, int k0, int kc,
                              int first, uint32_t *out, cudaStream_t s);
cudaError_t launch_schoolbook_wide(const int32_t *A, int m, int n, int l, int w, int is_signed,
                                   const uint32_t *bsoa, uint32_t *out, int *status, cudaStream_t s);
int accum_rows(int m);   // rows of A per k_accum CTA (128; 64 for m <= 64)
int accum_chunk(int slots);   // k per shared-memory table chunk of k_accum (2^w <= 16 slots)

}  // namespace pcmm

// ---------------------------------------------------------------- checked build
// PCMM_CHECKED=1 (build.py build(checked=True) -> libpcmm_checked.so; pcmm.py loads it when
// PCMM_LIB_VARIANT=checked): device-side bounds checks on the shared-memory staging and scans and on
// the table / plan indices, standing in for compute-sanitizer (not available on the GPU pool).
// A failed check prints its site and traps (the launch fails loudly: PCMM_ECUDA).
#ifndef PCMM_CHECKED
#define PCMM_CHECKED 0
#endif
#if PCMM_CHECKED
#include <cstdio>
#define PCMM_DCHECK(...)                                                                           \
    do {                                                                                           \
        if (!(__VA_ARGS__)) {                                                                      \
            printf("PCMM_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #__VA_ARGS__, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                             \
            __trap();                                                                              \
        }                                                                                          \
    } while (0)
#else
#define PCMM_DCHECK(...) \
    do {                 \
    } while (0)
#endif
