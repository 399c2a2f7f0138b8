/*
 * pcmm.h -- C ABI of libpcmm.so: plaintext-ciphertext matrix multiplication
 * (PC-MM) C = A . Enc(B) over EC-ElGamal on NIST P-256, on one NVIDIA B200
 * (sm_100a), computed by Cussen's compression-reconstruction algorithm
 * (schoolbook PC-MM as the comparison path).
 *
 * Source of every operation: arXiv 2504.14497 ("PAPER.md" line numbers):
 *   KeyGen / Encrypt / Decrypt .......... Sec. 2.4
 *   homomorphism (Eq. 5) ................ PAPER.md:186-193
 *   schoolbook PC-MM .................... Sec. 3.1
 *   Cussen vector-scalar (Alg. 2) ....... Sec. 3.2
 *   proposed PC-MM (Alg. 3) ............. Sec. 3.3
 *   curve P-256 ......................... Sec. 4.1
 * Readings of the paper where it is silent (zero handling, pointer layout,
 * signed plaintexts, wire format, ...) are listed in DESIGN.md (R1-R17).
 *
 * Conventions (all functions):
 *   - Return an int status: PCMM_OK (0) or a negative PCMM_E* code; no C++
 *     exception ever crosses the ABI.  pcmm_last_error() gives a message
 *     (thread-local, valid until the next call on the same thread).
 *   - Suffix _h = HOST pointer, _d = DEVICE pointer.  The caller allocates and
 *     owns every buffer; the library never frees caller memory and never
 *     retains a pointer after a call returns.
 *   - Device work is enqueued on the given CUDA stream (a cudaStream_t passed
 *     as void*; NULL = the legacy default stream) and is ASYNCHRONOUS unless a
 *     function says otherwise.  Errors detected on the device (a plaintext out
 *     of its w-bit range, an input point not on the curve) are recorded in the
 *     workspace and returned by pcmm_status(), which synchronises the stream.
 *   - Canonical ciphertext = 128 bytes C1 || C2; a point = 64 bytes x || y,
 *     each coordinate 32-byte big-endian; the point at infinity is 64 zero
 *     bytes ((0,0) is not on P-256).  Scalars are 32-byte big-endian.
 *   - Matrices are row-major: A is m x n bytes (a_ik at A[i*n + k]), read as
 *     int8 when is_signed and as uint8 otherwise (so unsigned w = 8 reaches 255); Enc(B)
 *     is n x l canonical ciphertexts (b_kj at index k*l + j); outputs are
 *     m x l (c_ij at index i*l + j).
 *   - Signed plaintexts (is_signed = 1): a in [-2^(w-1), 2^(w-1)); a negative
 *     a multiplies by the group element (q - |a|), i.e. -(|a| P) (DESIGN R10).
 *     Unsigned: a in [0, 2^w).
 *   - "Projective" outputs (ctC_proj_d) use an opaque-but-documented layout:
 *     uint32 words [c in {C1,C2}][coord in {X,Y,Z}][limb 0..7][idx], count
 *     = m*l points per component, Montgomery form (x*2^256 mod p),
 *     homogeneous projective (x = X/Z, y = Y/Z, infinity <=> Z = 0).
 *     Size in bytes: pcmm_proj_bytes(count) = 192 * count.
 */
#ifndef PCMM_H
#define PCMM_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PCMM_API __attribute__((visibility("default")))
#else
#define PCMM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define PCMM_OK 0
#define PCMM_EINVAL (-1)       /* null pointer or invalid argument */
#define PCMM_EDIM (-2)         /* a dimension <= 0, or too large */
#define PCMM_EBOUND (-3)       /* a plaintext entry outside its w-bit range */
#define PCMM_ENOTONCURVE (-4)  /* an input point not on P-256 / not reduced */
#define PCMM_EDECODE (-5)      /* (per element) no message in [lo, hi] */
#define PCMM_ECUDA (-6)        /* a CUDA runtime error */
#define PCMM_ENOMEM (-7)       /* workspace too small / allocation failed */
#define PCMM_ENOTSUP (-8)      /* parameters valid but not supported by this build */

#define PCMM_PATH_SCHOOLBOOK 0
#define PCMM_PATH_CUSSEN 1
#define PCMM_PATH_STRASSEN 2

/* Message for the last error on this thread ("" if none). */
PCMM_API const char *pcmm_last_error(void);

/* Library version string. */
PCMM_API const char *pcmm_version(void);

/* Bytes of a projective output buffer for `count` ciphertexts (192 * count). */
PCMM_API size_t pcmm_proj_bytes(int64_t count);

/* KeyGen: x uniform in [1, q-1], H = x G.  x is drawn from
 * SplitMix64(seed): 4 consecutive 64-bit draws concatenated big-endian,
 * redrawn until in [1, q-1] (R12).  Writes sk_h = x (32 B BE) and
 * pk_h = H (64 B canonical point).  SYNCHRONOUS (runs one small kernel on the
 * current device's default stream and waits).  Errors: EINVAL, ECUDA.      */
PCMM_API int pcmm_keygen(uint64_t seed, uint8_t sk_h[32], uint8_t pk_h[64]);

/* Encrypt: ct[e] = (r_e G, r_e H + b_e G) for e < count.
 *   pk_h : H, 64-byte canonical point (host; copied into the launch).
 *   b_d  : int32[count] plaintexts (negative b means scalar q - |b|).
 *   r_d  : uint8[count][32] big-endian randomness, each in [1, q-1] (caller's
 *          responsibility; values are used as given).
 *   ct_d : uint8[count][128] canonical ciphertexts (output).
 * Checks (host, before any launch): pk is the canonical encoding of a P-256
 *   point (x, y < p, y^2 = x^3 - 3x + b; the identity is rejected), r_d and
 *   ct_d are 16-byte aligned.
 * Errors: EINVAL (null / count < 0 / misaligned), ENOTONCURVE (pk not on the
 *   curve or not reduced), ECUDA.  Async.                                   */
PCMM_API int pcmm_encrypt(const uint8_t pk_h[64], const int32_t *b_d, const uint8_t *r_d, int64_t count, uint8_t *ct_d,
                 void *stream);

/* Workspace bytes needed by pcmm_mul_schoolbook (path 0) / pcmm_mul_cussen
 * (path 1) / pcmm_mul_strassen (path 2) / pcmm_normalize (path -1) for these
 * dimensions.  Returns 0 for invalid arguments.  The workspace must be device
 * memory, 256-byte aligned, and must not be used concurrently by two calls. */
PCMM_API size_t pcmm_workspace_bytes(int m, int n, int l, int w, int path);

/* Schoolbook PC-MM: for every (i, j),
 *   Enc(c_ij) = sum_k a_ik * Enc(b_kj)
 * with one small-scalar multiplication (binary double-and-add) per term and
 * complete projective additions.  Output: projective ctC_proj_d (m*l points
 * per component, layout above).  w in [1, 8].  Async.
 * Errors: EINVAL, EDIM, ENOMEM (ws_bytes too small), ECUDA; device-side
 * EBOUND / ENOTONCURVE via pcmm_status(ws_d).                              */
PCMM_API int pcmm_mul_schoolbook(const int8_t *A_d, int m, int n, int l, int w, int is_signed, const uint8_t *ctB_d,
                        void *ctC_proj_d, void *ws_d, size_t ws_bytes, void *stream);

/* Cussen PC-MM (Alg. 3) with `iters` = N iterations of
 * compression / reconstruction (the paper uses N = 4; 1 <= N <= 4 here):
 *   a1  every column A[:,k] is compressed on the device (Alg. 2 lines 3-12):
 *       sorted distinct nonzero values per level, differences, tracking
 *       pointers, and the rank of each a_ik in level 1;
 *   a2  per (k, j) the level-N values are multiplied by the ciphertext
 *       (2 n_N small ECSMs, Alg. 3 line 5);
 *   a3  reconstruction prefix sums (Alg. 2 lines 14-23) build the table
 *       T_kj[v] = v * Enc(b_kj) for the distinct values v of A[:,k];
 *   a4  un-sort / re-insert + accumulation (Alg. 3 lines 6-9): every output
 *       gathers C_ij += T_kj[a_ik] from the affine tables (L1/L2-resident;
 *       m <= 64 and w <= 4: from table chunks staged in shared memory).
 * Output identical (after pcmm_normalize) to pcmm_mul_schoolbook.
 * w in [1, 8] (tables of <= 2^w - 1 entries per (k, j)).  Signed A: a column
 * whose magnitudes are {1..M} gets the entry of -v as the negation of the
 * entry of v (R10b); the outputs do not depend on it.  Async.
 * Errors as pcmm_mul_schoolbook; ENOTSUP for iters outside [1, 4].        */
PCMM_API int pcmm_mul_cussen(const int8_t *A_d, int m, int n, int l, int w, int is_signed, int iters, const uint8_t *ctB_d,
                    void *ctC_proj_d, void *ws_d, size_t ws_bytes, void *stream);

/* Strassen PC-MM, the paper's second comparison path (Sec. 3.1,
 * PAPER.md:253-300): 7 half-size block PC-MMs per level (M1..M7), 5 plaintext
 * block sums / differences (int32 internally: entries grow one bit per level)
 * and 13 ciphertext block additions / subtractions; recursion while m, n, l are
 * even and their halves >= `leaf`, then schoolbook on the blocks.  Output and
 * errors as pcmm_mul_schoolbook (workspace: path 2).  Temporary blocks are
 * allocated stream-ordered on `stream` (cudaMallocAsync).  Async.          */
PCMM_API int pcmm_mul_strassen(const int8_t *A_d, int m, int n, int l, int w, int is_signed, int leaf,
                               const uint8_t *ctB_d, void *ctC_proj_d, void *ws_d, size_t ws_bytes, void *stream);

/* Wide-plaintext PC-MM (the paper's t = 12, 16 grid,
 * PAPER.md:61, Table A9): the same products as pcmm_mul_schoolbook /
 * pcmm_mul_cussen for plaintexts of up to 16 bits.
 *   A_d : int32[m][n] row-major (4-byte aligned); entries in [0, 2^w)
 *         (unsigned) or [-2^(w-1), 2^(w-1)) (is_signed), w in [1, 16];
 *         m <= 16384 (a column is sorted in shared memory).
 * Cussen (Alg. 3): per column up to min(m, 2^w - 1) distinct values, so the
 * compression plan, the uint16 rank and the tables (min(m, 2^w - 1) + 1 slots
 * per (k, j, c)) are sized per problem; the tables are built, converted to
 * affine and accumulated in chunks of inner indices k chosen so that one
 * chunk's tables fit a 2 GiB budget (env PCMM_WIDE_BUDGET_MB overrides).
 * Output, status and errors as pcmm_mul_cussen / pcmm_mul_schoolbook, with
 * the workspace sized by pcmm_workspace_bytes_wide (path 0 schoolbook,
 * 1 Cussen, 2 Strassen; returns 0 for invalid arguments).  Async.
 * pcmm_mul_strassen_wide: pcmm_mul_strassen for int32 plaintexts, w <= 16
 * (the recursion's int32 block sums gain one bit per level).               */
PCMM_API size_t pcmm_workspace_bytes_wide(int m, int n, int l, int w, int path);
PCMM_API int pcmm_mul_cussen_wide(const int32_t *A_d, int m, int n, int l, int w, int is_signed, int iters,
                                  const uint8_t *ctB_d, void *ctC_proj_d, void *ws_d, size_t ws_bytes,
                                  void *stream);
PCMM_API int pcmm_mul_schoolbook_wide(const int32_t *A_d, int m, int n, int l, int w, int is_signed,
                                      const uint8_t *ctB_d, void *ctC_proj_d, void *ws_d, size_t ws_bytes,
                                      void *stream);
PCMM_API int pcmm_mul_strassen_wide(const int32_t *A_d, int m, int n, int l, int w, int is_signed, int leaf,
                                    const uint8_t *ctB_d, void *ctC_proj_d, void *ws_d, size_t ws_bytes,
                                    void *stream);

/* Normalise `count` projective ciphertexts (layout above, as written by
 * pcmm_mul_*) to canonical affine bytes ctC_d[count][128] (x = X/Z, y = Y/Z,
 * out of Montgomery form, big-endian; infinity -> 64 zero bytes), by
 * Montgomery batch inversion.  Async.  Errors: EINVAL, ENOMEM, ECUDA.      */
PCMM_API int pcmm_normalize(const void *ctC_proj_d, int64_t count, uint8_t *ctC_d, void *ws_d, size_t ws_bytes,
                   void *stream);

/* ---- NEXT-4: PC-MM over the Paillier scheme -----------
 * Sec. 2.5 and the extension of PAPER.md:585-626: with
 * Eq. 6 the product is C_ij = prod_k c_kj^{a_ik} mod n^2;
 * path 0 = schoolbook (one Alg. 4 Montgomery powering ladder of w steps per
 * term), path 1 = Cussen (Alg. 3 with point additions ->
 * modular multiplications and ECSMs -> Alg. 4 exponentiations, `iters` = N).
 *   A_d   : uint8[m][n], non-negative plaintexts < 2^w, w in [1, 8]
 *           (negative scalars would need c^-1 mod n^2; R20);
 *   N2_h  : HOST pointer to the modulus n^2, nbits_n2 / 32 little-endian
 *           32-bit words, odd; nbits_n2 in {512, 1024, 2048, 3072};
 *   ctB_d : uint32[n*l][nbits_n2/32] ciphertexts (residues < n^2, words
 *           little-endian, (k, j) row-major);
 *   ctC_d : uint32[m*l][nbits_n2/32] output residues, (i, j) row-major.
 * Workspace: pcmm_paillier_workspace_bytes (0 for invalid arguments).
 * Async.  Device-side status via pcmm_status(ws_d): EBOUND (a_ik >= 2^w),
 * ENOTONCURVE (a ciphertext >= n^2).  Errors: EINVAL, EDIM, ENOMEM,
 * ENOTSUP (modulus size / iters), ECUDA.                                    */
PCMM_API size_t pcmm_paillier_workspace_bytes(int m, int n, int l, int w, int nbits_n2, int path);
PCMM_API int pcmm_paillier_mul(int path, const uint8_t *A_d, int m, int n, int l, int w, int iters,
                               const uint32_t *N2_h, int nbits_n2, const uint32_t *ctB_d, uint32_t *ctC_d,
                               void *ws_d, size_t ws_bytes, void *stream);

/* ---- NEXT-2: fixed-base comb encryption ---------------
 * Encrypt with per-key precomputed tables: a context holds
 * T_P[i][v] = v 2^(8i) P for P in {G, H = pk}, 32 byte windows i, v < 256,
 * affine Montgomery (1 MiB + 256 B, pcmm_enc_ctx_bytes()); then
 *   C1 = r G = sum_i T_G[i][r_i],  C2 = r H + b G = sum_i T_H[i][r_i] +- sum_{i<4} T_G[i][|b|_i]
 * (Jacobian + affine mixed additions with a complete fallback, one inversion
 * per ciphertext).  Output bytes are identical to pcmm_encrypt.
 *   pcmm_enc_ctx_init: ctx_d caller-owned device memory (256-byte aligned,
 *     pcmm_enc_ctx_bytes() bytes); builds the tables on `stream` and
 *     SYNCHRONISES it.  ENOTONCURVE if pk is not a P-256 point (or is 0).
 *   pcmm_encrypt_ctx: as pcmm_encrypt (b_d int32, r_d count x 32 B BE in
 *     [1, q-1], ct_d count x 128 B; r_d / ct_d 16-byte aligned).  Async.   */
PCMM_API size_t pcmm_enc_ctx_bytes(void);
PCMM_API int pcmm_enc_ctx_init(const uint8_t pk_h[64], void *ctx_d, void *stream);
PCMM_API int pcmm_encrypt_ctx(const void *ctx_d, const int32_t *b_d, const uint8_t *r_d, int64_t count,
                              uint8_t *ct_d, void *stream);

/* ---- NEXT-2: baby-step giant-step decryption ----------------------------
 * Decrypt for messages in [lo, hi] with a device hash
 * table of the baby steps { j G : 1 <= j < s = 2^log2_baby } (open addressing,
 * 2s slots, key = affine x with the parity of y, so jG and -jG differ):
 *   pcmm_bsgs_ctx_bytes(log2_baby) = 256 + 24 s bytes (0 if log2_baby is
 *     outside [1, 28]);
 *   pcmm_bsgs_init: builds the table into ctx_d (256-byte aligned). Async.
 *   pcmm_decrypt_bsgs: per ciphertext M = C2 - x C1 - lo G, giant steps
 *     M - i s G (batches of 8 sharing one inversion) until the identity (j = 0)
 *     or a table hit j: m = lo + i s + j.  (hi - lo + 1) / s <= 2^24 and
 *     |lo|, |hi| < 2^62.  m_d / status_d as pcmm_decrypt_small (status 0,
 *     PCMM_EDECODE if m is not in [lo, hi], PCMM_ENOTONCURVE for a bad input).
 *     Async.  Errors: EINVAL, ECUDA.                                         */
PCMM_API size_t pcmm_bsgs_ctx_bytes(int log2_baby);
PCMM_API int pcmm_bsgs_init(int log2_baby, void *ctx_d, void *stream);
PCMM_API int pcmm_decrypt_bsgs(const uint8_t sk_h[32], const void *ctx_d, int log2_baby, const uint8_t *ct_d,
                               int64_t count, int64_t lo, int64_t hi, int64_t *m_d, int32_t *status_d,
                               void *stream);

/* Decrypt: m_e = phi^-1(C2 - x C1), the unique m in
 * [lo, hi] with m G = C2 - x C1 (hi - lo < 2^26, |lo|, |hi| < 2^30), found by
 * baby-step giant-step with a baby-step table of 2^b points built for this
 * call (2^(2b) ~ count (hi - lo + 1); the kernels of pcmm_decrypt_bsgs).
 * sk_h = x (32 B BE).
 * m_d[e] receives the message, status_d[e] = 0 or PCMM_EDECODE if no m in
 * [lo, hi] matches (m_d[e] = 0 then) or PCMM_ENOTONCURVE for a bad input.
 * Async (allocates its table stream-ordered on `stream`).
 * Errors: EINVAL, ENOMEM, ECUDA.                                            */
PCMM_API int pcmm_decrypt_small(const uint8_t sk_h[32], const uint8_t *ct_d, int64_t count, int64_t lo, int64_t hi,
                       int64_t *m_d, int32_t *status_d, void *stream);

/* Synchronise `stream` and return the device-side status recorded in the
 * workspace by the last pcmm_mul_* / pcmm_normalize call that used it:
 * PCMM_OK, PCMM_EBOUND or PCMM_ENOTONCURVE (or ECUDA).                      */
PCMM_API int pcmm_status(const void *ws_d, void *stream);

/* ---- measurement hooks (used by bench.py; not needed for normal use) ---- */
/* Enable (1) / disable (0) per-kernel CUDA-event timing of every launch made
 * by the library; enabling clears the record.                              */
PCMM_API int pcmm_profile_enable(int on);
/* Synchronise the recorded events and copy out up to `max` records: kernel
 * name (NUL-separated into names_h, 48 bytes per record) and duration in ms.
 * Returns the number of records (or a negative status).                    */
PCMM_API int pcmm_profile_read(char *names_h, float *ms_h, int max);

/* ---- test hooks (unit parity tests of single steps) ---------------------- */
/* Batched field ops on 32-byte big-endian values (reduced mod p):
 * op 0 a+b, 1 a-b, 2 a*b, 3 a^-1 (divsteps), 4 -a, 5 a^2 (dedicated
 * squaring), 6 a*b (the alternate product form), 7 a^-1 (Fermat chain)
 * (all mod p); the accumulate loop's almost-reduced forms on operands whose
 * odd Montgomery forms below 2^256 - p are first replaced by form + p:
 * 8 a*b, 9 a^2, 10 a+b, 11 a-b (results reduced mod p), 12 the zero test
 * (out = 1 if a = 0 mod p else 2, as a plain 32-byte integer).
 * out_d[count][32].                                                        */
PCMM_API int pcmm_test_field(int op, const uint8_t *a_d, const uint8_t *b_d, uint8_t *out_d, int64_t count, void *stream);
/* Batched group ops on 64-byte canonical points: op 0 P+Q, 1 2P, 2 v*P
 * (v_d[e], |v| < 2^15), 3 k*P (k = 32-byte BE scalar in q_d[e][0..31]; 4-bit
 * windows, Jacobian: the encrypt / decrypt ECSM), 4 k*P (binary double-and-
 * add with the complete formulas).  out_d[count][64].                        */
PCMM_API int pcmm_test_point(int op, const uint8_t *p_d, const uint8_t *q_d, const int32_t *v_d, uint8_t *out_d,
                    int64_t count, void *stream);
/* The device compression plan of Alg. 2 (step a1) for every column of A:
 * levels_d[n][4] = |a^(1)|..|a^(N)| (0 beyond N), sN_d[n][256] (int16) =
 * values of the last level, rank_d[n][m] = 1 + index of a_ik in a^(1) (0 for
 * a_ik = 0).  w in [1, 8].  Synchronises `stream`; EBOUND on a bad entry.  */
PCMM_API int pcmm_test_plan(const int8_t *A_d, int m, int n, int w, int is_signed, int iters, int32_t *levels_d,
                   int16_t *sN_d, uint8_t *rank_d, void *stream);
/* fp_mul throughput probe: `blocks` x `threads` threads each run `iters`
 * dependent-chain field multiplications on 4 independent chains; variant
 * selects the fe_mul implementation (0 = library default).  Writes a
 * checksum to out_d[blocks*threads][8].  Async.                             */
PCMM_API int pcmm_bench_fp_mul(int variant, int blocks, int threads, int iters, uint32_t *out_d, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* PCMM_H */
