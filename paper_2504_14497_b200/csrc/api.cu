// api.cu -- the C ABI of libpcmm.so (declared and documented in include/pcmm.h).
// Host code only: argument validation, workspace carving, launch ordering on
// the caller's stream, status reporting.  Every step of the PC-MM path runs in
// the kernels of kernels.cu; nothing here computes on the host except keygen's
// SplitMix64 draw of the secret scalar (R12) and pcmm_encrypt's
// on-curve check of the public key (argument validation).
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pcmm.h"
#include "internal.h"

using namespace pcmm;

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, const char *extra = nullptr) {
    char buf[512];
    snprintf(buf, sizeof buf, fmt, extra ? extra : "");
    g_err = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char *where) {
    char buf[512];
    snprintf(buf, sizeof buf, "%s: %s", where, cudaGetErrorString(e));
    g_err = buf;
    return PCMM_ECUDA;
}

#define CK(call, where)                                   \
    do {                                                  \
        cudaError_t _e = (call);                          \
        if (_e != cudaSuccess) return cuda_fail(_e, where); \
    } while (0)

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// ---------------------------------------------------------------- profiling
struct ProfRec {
    const char *name;
    cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;

// ---------------------------------------------------------------- workspace
struct Layout {
    size_t status = 0, bsoa = 0, plans = 0, rank = 0, perm = 0, tables = 0, scratch = 0, partial = 0, bsoa_c = 0, total = 0;
    int rows = 128, ksplit = 1, slots = 16, maxup = 8;
    int kc = 0;                            // inner indices per table chunk (= n: one chunk)
};

// split-k factor of k_accum for an (m, n, l) accumulation: minimise the quantised
// wave count per unit of work, ceil(base*ks / resident) / ks, plus a small charge
// per extra split (the k_reduce additions and per-CTA chunk overheads).
static int choose_ksplit(int m, int n, int l, int w) {
    const int rows = w <= 4 ? accum_rows(m) : 128;
    const int rowblocks = (m + rows - 1) / rows;
    const int64_t base = (int64_t)l * 2 * rowblocks;
    const int slots = table_slots(w);
    const double resident = (double)num_sms() * (w <= 4 ? accum_ctas_per_sm(slots, rows) : accum_global_ctas_per_sm());
    // On the shared-memory path only splits whose k-range is a whole number of table chunks
    // are considered when there are any besides 1 (measured: 256^3 2 splits 4.306 ms vs 3 ragged
    // ones 4.323, 512^3 4 splits 24.50 vs 3: 24.88, ML 16 splits 2.88 vs 10: 2.92).
    const int kch = w <= 4 ? accum_chunk(slots) : 0;
    bool any_aligned = false;
    for (int cand = 2; cand <= 16 && cand <= n && kch && n >= 4 * kch; cand++)   // (64^3: latency regime)
        if (n % (cand * kch) == 0) any_aligned = true;
    int ks = 1;
    double best = 1e30;
    for (int cand = 1; cand <= 16 && cand <= n; cand++) {
        if (any_aligned && cand > 1 && n % (cand * kch) != 0) continue;
        const double waves = std::ceil((double)base * cand / resident);
        const double cost = waves / cand * (1.0 + 0.01 * (cand - 1)) + (n / cand < 8 ? 1.0 : 0.0);
        if (cost < best - 1e-9) { best = cost; ks = cand; }
    }
    if (const char *e = getenv("PCMM_KSPLIT")) {         // measurement override (tools/)
        const int v = atoi(e);
        if (v >= 1 && v <= n) ks = v;
    }
    return ks;
}

// Table memory of the byte path (tables + k_tables scratch / affine tables) per inner index k;
// above the budget (PCMM_BYTE_BUDGET_MB, default 2048) the Cussen path builds and consumes the
// tables in chunks of kc inner indices (the imported rows of the chunk copied to their own
// buffer, each chunk's accumulation added into the running output).
static size_t byte_table_bytes_per_k(int l, int w) {
    const size_t S = (size_t)table_slots(w), mu = (size_t)max_upper(w);
    return 2 * (size_t)l * (S * kPtWords * 4 + std::max(2 * mu * kPtWords * 4, S * kAffWords * 4));
}

static size_t byte_budget() {
    size_t budget = (size_t)2 << 30;
    if (const char *e = getenv("PCMM_BYTE_BUDGET_MB")) budget = (size_t)atoll(e) << 20;
    return budget;
}

Layout layout(int m, int n, int l, int w, int path) {
    Layout L;
    size_t off = 256;                      // status word(s)
    const size_t cnt = (size_t)n * l;
    L.bsoa = off;
    off = align256(off + cnt * 2 * kPtWords * 4);
    if (path == PCMM_PATH_CUSSEN) {
        L.rows = accum_rows(m);
        L.slots = table_slots(w);
        L.maxup = max_upper(w);
        // the whole workspace within the budget when it can be: tables of all n inner indices if they fit
        // beside the fixed parts (imported B, plans, rank, split-k partials), else chunks of kc with at most
        // kChunkSplits partial sums and the chunk's imported rows
        const size_t per_k = byte_table_bytes_per_k(l, w);
        const size_t slot = 2 * (size_t)kPtWords * 4 * (size_t)m * l;     // one set of partial sums
        const size_t fixed0 = off + align256((size_t)n * sizeof(ColPlan)) + align256((size_t)n * m) +
                              align256((size_t)16 * ((m + 127) / 128) * 128 * 4) + 4096;
        const int ks_full = choose_ksplit(m, n, l, w);
        int kc = n;
        if (fixed0 + (ks_full > 1 ? ks_full * slot : 0) + (size_t)n * per_k > byte_budget()) {
            constexpr int kChunkSplits = 4;
            const size_t fixed = fixed0 + kChunkSplits * slot;
            const size_t per_kc = per_k + (size_t)l * 2 * kPtWords * 4;
            kc = (int)std::min<size_t>(n, std::max<size_t>(1, fixed < byte_budget() ? (byte_budget() - fixed) / per_kc : 1));
            const int kch = w <= 4 ? accum_chunk(L.slots) : 0;        // whole k_accum table chunks
            if (kch && kc > kch) kc -= kc % kch;
            L.ksplit = std::min(kChunkSplits, choose_ksplit(m, kc, l, w));
        } else {
            L.ksplit = ks_full;
        }
        L.kc = kc;
        L.plans = off;
        off = align256(off + (size_t)n * sizeof(ColPlan));
        L.rank = off;
        off = align256(off + (size_t)n * m);
        L.perm = off;                      // k_rowperm: up to 16 splits x 128-row blocks x 128 ints
        off = align256(off + (size_t)16 * ((m + 127) / 128) * 128 * 4);
        const size_t ccnt = (size_t)kc * l;
        L.tables = off;
        off = align256(off + ccnt * 2 * (size_t)kPtWords * L.slots * 4);
        // upper-level scratch of k_tables, then (reused) the affine tables of k_affine
        L.scratch = off;
        off = align256(off + std::max(ccnt * 2 * (size_t)kPtWords * 2 * L.maxup * 4,
                                      ccnt * 2 * (size_t)kAffWords * L.slots * 4));
        if (L.ksplit > 1 || kc < n) {
            L.partial = off;
            off = align256(off + (size_t)L.ksplit * 2 * kPtWords * 4 * (size_t)m * l);
        }
        if (kc < n) {
            L.bsoa_c = off;                // the chunk's imported rows
            off = align256(off + ccnt * 2 * kPtWords * 4);
        }
    }
    L.total = off;
    return L;
}

// ---------------------------------------------------------------- wide-plaintext workspace
struct LayoutW {
    size_t bsoa = 0, pn = 0, psN = 0, pptr = 0, rank = 0, tables = 0, scratch = 0, total = 0;
    int cap = 0, S = 0, KC = 0;
};

constexpr int kWideMaxM = 16384;        // k_plan_wide sorts a column in shared memory

LayoutW layout_wide(int m, int n, int l, int w, int path) {
    LayoutW L;
    size_t off = 256;
    const size_t cnt = (size_t)n * l;
    L.bsoa = off;
    off = align256(off + cnt * 2 * kPtWords * 4);
    if (path == PCMM_PATH_CUSSEN) {
        L.cap = (int)std::min<int64_t>(m, (1LL << w) - 1);
        L.S = L.cap + 1;
        // chunk of inner indices k whose tables (+ scratch / affine tables) fit the budget
        size_t budget = (size_t)2 << 30;
        if (const char *e = getenv("PCMM_WIDE_BUDGET_MB")) budget = (size_t)atoll(e) << 20;
        const size_t per_k = 2 * (size_t)l *
                             ((size_t)L.S * kPtWords * 4 +
                              std::max((size_t)2 * L.cap * kPtWords * 4, (size_t)L.S * kAffWords * 4));
        int kc = (int)std::max<size_t>(1, std::min<size_t>((size_t)n, budget / per_k));
        const int chunks = (n + kc - 1) / kc;
        L.KC = (n + chunks - 1) / chunks;
        L.pn = off;
        off = align256(off + (size_t)n * 4 * 4);
        L.psN = off;
        off = align256(off + (size_t)n * L.cap * 4);
        L.pptr = off;
        off = align256(off + (size_t)n * 3 * L.cap * 2);
        L.rank = off;
        off = align256(off + (size_t)n * m * 2);
        L.tables = off;
        off = align256(off + (size_t)L.KC * 2 * l * L.S * kPtWords * 4);
        L.scratch = off;
        off = align256(off + (size_t)L.KC * 2 * l *
                                 std::max((size_t)2 * L.cap * kPtWords * 4, (size_t)L.S * kAffWords * 4));
    }
    L.total = off;
    return L;
}

int check_dims(int m, int n, int l) {
    if (m <= 0 || n <= 0 || l <= 0) return fail(PCMM_EDIM, "dimensions must be positive");
    if ((int64_t)m * l > (1LL << 30) || (int64_t)n * l > (1LL << 30) || (int64_t)m * n > (1LL << 31))
        return fail(PCMM_EDIM, "dimensions too large");
    return PCMM_OK;
}

// SplitMix64 (Steele, Lea, Flood 2014) -- the counter-based generator of DESIGN.md R12
struct SplitMix64 {
    uint64_t s;
    uint64_t next() {
        s += 0x9E3779B97F4A7C15ULL;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
};

// group order q, big-endian 64-bit words
const uint64_t kQ[4] = {0xffffffff00000000ULL, 0xffffffffffffffffULL, 0xbce6faada7179e84ULL, 0xf3b9cac2fc632551ULL};

bool in_range_1_qm1(const uint64_t w[4]) {   // 1 <= w <= q - 1, w big-endian words
    bool zero = (w[0] | w[1] | w[2] | w[3]) == 0;
    if (zero) return false;
    for (int i = 0; i < 4; i++) {
        if (w[i] < kQ[i]) return true;
        if (w[i] > kQ[i]) return false;
    }
    return false;                              // == q
}

// ---- host-side public-key check for pcmm_encrypt (argument validation only; the
// encryption itself runs on the device).  Plain 4 x 64-bit little-endian limbs,
// 512-bit products reduced mod p by shift-and-subtract: slow and obviously right.
typedef unsigned __int128 u128;
const uint64_t kP[4] = {0xffffffffffffffffULL, 0x00000000ffffffffULL, 0x0000000000000000ULL,
                        0xffffffff00000001ULL};       // p = 2^256 - 2^224 + 2^192 + 2^96 - 1 (little-endian limbs)
const uint64_t kB[4] = {0x3bce3c3e27d2604bULL, 0x651d06b0cc53b0f6ULL, 0xb3ebbd55769886bcULL,
                        0x5ac635d8aa3a93e7ULL};       // curve coefficient b (SEC 2)

int cmp4(const uint64_t *a, const uint64_t *b) {
    for (int i = 3; i >= 0; i--) {
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    }
    return 0;
}

void sub4(uint64_t *a, const uint64_t *b) {   // a -= b (a >= b)
    uint64_t br = 0;
    for (int i = 0; i < 4; i++) {
        const u128 d = (u128)a[i] - b[i] - br;
        a[i] = (uint64_t)d;
        br = (uint64_t)(d >> 64) & 1;
    }
}

void mulmod4(uint64_t *r, const uint64_t *a, const uint64_t *b) {   // r = a b mod p (a, b < p)
    uint64_t t[8] = {0};
    for (int i = 0; i < 4; i++) {
        uint64_t c = 0;
        for (int j = 0; j < 4; j++) {
            const u128 s = (u128)a[i] * b[j] + t[i + j] + c;
            t[i + j] = (uint64_t)s;
            c = (uint64_t)(s >> 64);
        }
        t[i + 4] = c;
    }
    uint64_t acc[4] = {0, 0, 0, 0};             // Horner over the 512 bits, msb first: acc = 2 acc + bit
    for (int bit = 511; bit >= 0; bit--) {
        const uint64_t top = acc[3] >> 63;
        for (int i = 3; i > 0; i--) acc[i] = (acc[i] << 1) | (acc[i - 1] >> 63);
        acc[0] = (acc[0] << 1) | ((t[bit >> 6] >> (bit & 63)) & 1);
        if (top || cmp4(acc, kP) >= 0) sub4(acc, kP);   // 2 acc + 1 < 2p: one subtraction (mod 2^256 if top)
    }
    for (int i = 0; i < 4; i++) r[i] = acc[i];
}

void addmod4(uint64_t *r, const uint64_t *a, const uint64_t *b) {
    uint64_t c = 0;
    uint64_t s[4];
    for (int i = 0; i < 4; i++) {
        const u128 x = (u128)a[i] + b[i] + c;
        s[i] = (uint64_t)x;
        c = (uint64_t)(x >> 64);
    }
    if (c || cmp4(s, kP) >= 0) sub4(s, kP);
    for (int i = 0; i < 4; i++) r[i] = s[i];
}

// canonical 64-byte point (x || y, big-endian) on P-256: x, y < p and y^2 = x^3 - 3x + b
bool pk_on_curve_host(const uint8_t pk[64]) {
    uint64_t x[4] = {0}, y[4] = {0};
    for (int i = 0; i < 32; i++) {
        x[3 - i / 8] = (x[3 - i / 8] << 8) | pk[i];
        y[3 - i / 8] = (y[3 - i / 8] << 8) | pk[32 + i];
    }
    if (cmp4(x, kP) >= 0 || cmp4(y, kP) >= 0) return false;
    uint64_t lhs[4], rhs[4], x3[4], neg3x[4], three_x[4];
    mulmod4(lhs, y, y);
    mulmod4(x3, x, x);
    mulmod4(x3, x3, x);
    addmod4(three_x, x, x);
    addmod4(three_x, three_x, x);
    uint64_t zero[4] = {0, 0, 0, 0};
    if (cmp4(three_x, zero) == 0) {
        for (int i = 0; i < 4; i++) neg3x[i] = 0;
    } else {
        for (int i = 0; i < 4; i++) neg3x[i] = kP[i];
        sub4(neg3x, three_x);                    // p - 3x
    }
    addmod4(rhs, x3, neg3x);
    addmod4(rhs, rhs, kB);
    return cmp4(lhs, rhs) == 0;
}

}  // namespace

namespace pcmm {

void prof_begin(const char *name, cudaStream_t s) {
    if (!g_prof_on) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    ProfRec r;
    r.name = name;
    cudaEventCreate(&r.a);
    cudaEventCreate(&r.b);
    cudaEventRecord(r.a, s);
    g_prof.push_back(r);
}

void prof_end(cudaStream_t s) {
    if (!g_prof_on) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (!g_prof.empty()) cudaEventRecord(g_prof.back().b, s);
}

}  // namespace pcmm

#define LAUNCH(name, stream, call)                          \
    do {                                                    \
        prof_begin(name, stream);                           \
        cudaError_t _e = (call);                            \
        prof_end(stream);                                   \
        if (_e != cudaSuccess) return cuda_fail(_e, name);  \
    } while (0)

extern "C" {

const char *pcmm_last_error(void) { return g_err.c_str(); }

const char *pcmm_version(void) { return "pcmm-b200 0.1 (sm_100a)"; }

size_t pcmm_proj_bytes(int64_t count) { return count < 0 ? 0 : (size_t)count * 2 * kPtWords * 4; }

size_t pcmm_workspace_bytes(int m, int n, int l, int w, int path) {
    if (path == -1) return 256;
    if (m <= 0 || n <= 0 || l <= 0 || w < 1 || w > 8) return 0;
    if (path != PCMM_PATH_SCHOOLBOOK && path != PCMM_PATH_CUSSEN && path != PCMM_PATH_STRASSEN) return 0;
    return layout(m, n, l, w, path).total;
}

int pcmm_keygen(uint64_t seed, uint8_t sk_h[32], uint8_t pk_h[64]) {
    g_err.clear();
    if (!sk_h || !pk_h) return fail(PCMM_EINVAL, "null pointer");
    SplitMix64 g{seed};
    uint64_t w[4];
    do {
        for (int i = 0; i < 4; i++) w[i] = g.next();
    } while (!in_range_1_qm1(w));
    for (int i = 0; i < 4; i++)
        for (int b = 0; b < 8; b++) sk_h[8 * i + b] = (uint8_t)(w[i] >> (56 - 8 * b));
    uint32_t x[8];
    for (int i = 0; i < 8; i++) {          // little-endian 32-bit words
        const uint64_t word = w[3 - i / 2];
        x[i] = (uint32_t)(i % 2 ? word >> 32 : word);
    }
    uint8_t *d = nullptr;
    CK(cudaMalloc(&d, 64), "cudaMalloc");
    cudaError_t e = launch_pubkey(x, d, 0);
    if (e == cudaSuccess) e = cudaMemcpy(pk_h, d, 64, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return cuda_fail(e, "keygen");
    return PCMM_OK;
}

int pcmm_encrypt(const uint8_t pk_h[64], const int32_t *b_d, const uint8_t *r_d, int64_t count, uint8_t *ct_d,
                 void *stream) {
    g_err.clear();
    if (count < 0) return fail(PCMM_EINVAL, "count < 0");
    if (count == 0) return PCMM_OK;
    if (!pk_h || !b_d || !r_d || !ct_d) return fail(PCMM_EINVAL, "null pointer");
    bool zero = true;
    for (int i = 0; i < 64; i++) zero = zero && pk_h[i] == 0;
    if (zero) return fail(PCMM_ENOTONCURVE, "public key is the point at infinity");
    if (!pk_on_curve_host(pk_h))
        return fail(PCMM_ENOTONCURVE, "public key is not a point of P-256 (or a coordinate is not reduced)");
    if (((uintptr_t)r_d & 15) || ((uintptr_t)ct_d & 15))
        return fail(PCMM_EINVAL, "misaligned buffer (r / ct 16 B)");
    cudaStream_t s = (cudaStream_t)stream;
    LAUNCH("encrypt", s, launch_encrypt(pk_h, b_d, r_d, count, ct_d, s));
    return PCMM_OK;
}

static int mul_common(int path, const int8_t *A_d, int m, int n, int l, int w, int is_signed, int iters,
                      const uint8_t *ctB_d, void *ctC_proj_d, void *ws_d, size_t ws_bytes, cudaStream_t s) {
    g_err.clear();
    int rc = check_dims(m, n, l);
    if (rc) return rc;
    if (!A_d || !ctB_d || !ctC_proj_d || !ws_d) return fail(PCMM_EINVAL, "null pointer");
    if (((uintptr_t)ctB_d & 15) || ((uintptr_t)ws_d & 255) || ((uintptr_t)ctC_proj_d & 15))
        return fail(PCMM_EINVAL, "misaligned buffer (ctB/ctC 16 B, workspace 256 B)");
    if (w < 1 || w > 8) return fail(PCMM_EINVAL, "w must be in [1, 8]");
    if (path == PCMM_PATH_CUSSEN) {
        if (iters < 1 || iters > 4) return fail(PCMM_ENOTSUP, "iters must be in [1, 4]");
    }
    const Layout L = layout(m, n, l, w, path);
    if (ws_bytes < L.total) return fail(PCMM_ENOMEM, "workspace too small (see pcmm_workspace_bytes)");
    uint8_t *ws = (uint8_t *)ws_d;
    int *status = (int *)ws;
    uint32_t *bsoa = (uint32_t *)(ws + L.bsoa);
    uint32_t *out = (uint32_t *)ctC_proj_d;
    CK(cudaMemsetAsync(status, 0, 8, s), "memset status");      // [0] error bits, [1] k_plan's general-column flag
    LAUNCH("import", s, launch_import(ctB_d, (int64_t)n * l, bsoa, status, s));
    if (path == PCMM_PATH_SCHOOLBOOK) {
        LAUNCH("schoolbook", s, launch_schoolbook(A_d, m, n, l, w, is_signed, bsoa, out, status, s));
        return PCMM_OK;
    }
    ColPlan *plans = (ColPlan *)(ws + L.plans);
    uint8_t *rank = ws + L.rank;
    uint32_t *tables = (uint32_t *)(ws + L.tables);
    LAUNCH("plan", s, launch_plan(A_d, m, n, w, is_signed, iters, plans, rank, status, s));
    const int64_t cnt = (int64_t)m * l;
    const bool chunked = L.kc < n;
    for (int k0 = 0; k0 < n; k0 += L.kc) {
        // the chunk k0 .. k0 + nc - 1 as a sub-problem (m, nc, l): its plans, rank rows and imported rows
        const int nc = std::min(L.kc, n - k0);
        const ColPlan *pc = plans + k0;
        const uint8_t *rc_ = rank + (size_t)k0 * m;
        const uint32_t *bc = bsoa;
        if (chunked) {
            uint32_t *dst = (uint32_t *)(ws + L.bsoa_c);
            CK(cudaMemcpy2DAsync(dst, (size_t)nc * l * 4, bsoa + (size_t)k0 * l, (size_t)n * l * 4, (size_t)nc * l * 4,
                                 2 * kPtWords, cudaMemcpyDeviceToDevice, s),
               "chunk rows");
            bc = dst;
        }
        // consecutive-column tables (k_tables_fast): unsigned A, launches that fill the GPU
        // (64^3: the general kernel runs anyway for the rest and the extra launch costs more)
        // (k_tables_coz, default: the same columns, tables and affine conversion in one kernel; k_affine skips them)
        const int amode = tables_coz_mode();
        // (signed A: columns whose magnitudes are {1..M}, R10b; the others take k_tables + k_affine)
        const int aff = iters >= 2 && (amode == 2 || (amode == 1 && 2LL * nc * l >= 65536));
        const int fast = aff ? 2 : (tables_fast_on() && !is_signed && 2LL * nc * l >= 65536);
        uint32_t *atables = (uint32_t *)(ws + L.scratch);
        // general columns, fused (k_tables_gz: Alg. 2's reconstruction with an XYZZ level-1 prefix sum and
        // the affine conversion in one kernel; no upper-level scratch): launches with enough tables to
        // hide its two CTA-wide inversions (PCMM_TABLES_GZ: 0 never, 1 auto, 2 always; measured: 8,192 tables
        // of w = 4 0.151 -> 0.197 ms, of w = 8 equal, 32,768 of w = 6 0.68 -> 0.61, 131,072 of w = 8 8.2 -> 6.0)
        const int gmode = tables_gz_mode();
        const int gz = iters >= 2 && (fast == 0 || fast == 2) &&
                       (gmode == 2 || (gmode == 1 && 2LL * nc * l >= (L.slots >= 64 ? 8192 : 32768)));
        if (gz) {
            LAUNCH("tables_gz", s, launch_tables_gz(bc, pc, nc, l, iters, L.slots, L.maxup, tables, atables,
                                                    fast == 2, status + 1, s));
            if (fast == 2)
                LAUNCH("tables_coz", s, launch_tables_coz(bc, pc, nc, l, iters, L.slots, tables, atables, s));
        } else {
        LAUNCH("tables", s, launch_tables(bc, pc, nc, l, iters, L.slots, L.maxup, is_signed, tables,
                                          (uint32_t *)(ws + L.scratch), s, fast != 0, std::min(m, L.slots - 1),
                                          status + 1));
        // after k_tables: the affine tables share the region of k_tables' upper-level scratch
        if (fast == 2) {
            LAUNCH("tables_coz", s, launch_tables_coz(bc, pc, nc, l, iters, L.slots, tables, atables, s));
        } else if (fast) {
            LAUNCH("tables_fast", s, launch_tables_fast(bc, pc, nc, l, iters, L.slots, tables, atables, s));
        }
        LAUNCH("affine", s, launch_affine(tables, 2LL * nc * l * L.slots, atables, s, pc, nc, l, L.slots, iters, fast,
                                          status + 1));
        }
        // chunked: when one chunk's accumulation alone fills the GPU (>= 2 waves of CTAs), no split-k --
        // each chunk adds straight into the running output (the accumulators start from it: 3 + 3
        // products per output and chunk instead of a k_reduce pass with a complete addition per split)
        int ks = L.ksplit;
        if (chunked) {
            const int rows = w <= 4 ? accum_rows(m) : 128;
            const double ctas = (double)l * 2 * ((m + rows - 1) / rows);
            const double resident =
                (double)num_sms() * (w <= 4 ? accum_ctas_per_sm(L.slots, rows) : accum_global_ctas_per_sm());
            ks = ctas >= 2 * resident ? 1 : std::min(choose_ksplit(m, nc, l, w), L.ksplit);   // <= partial slots
        }
        const bool direct = ks == 1;                  // the accumulate writes (and in chunks, adds into) `out`
        uint32_t *acc_out = direct ? out : (uint32_t *)(ws + L.partial);
        const int64_t split_stride = direct ? 0 : 2LL * kPtWords * cnt;
        const int acc_in = direct && chunked && k0 > 0;
        // PCMM_ACC_MODE: 0 = k_accum (tables staged in shared memory, w <= 4) / k_accum_g (w > 4);
        // 1 = k_accum_g (gather) for every w; 2 = k_rowperm + k_accum_g2 (gather, rows sorted by nonzero
        // count, 4-group step); 3 (default) = the same with the software-pipelined step.  m <= 64 keeps mode 0.
        static int acc_mode = -1;
        if (acc_mode < 0) {
            const char *e = getenv("PCMM_ACC_MODE");
            acc_mode = e ? atoi(e) : 3;       // measured (256^3 / 512^3 / ML step): mode 0 4.157 / 24.23 / 2.230 ms,
                                              // 1: 4.185 / 25.13 / 2.270, 2: 4.131 / 24.05 / 2.227, 3: 3.979 / 23.14 / 2.152
        }
        if (acc_mode >= 2 && ks <= 16 && m > 64) {
            int *perm = (int *)(ws + L.perm);
            LAUNCH("rowperm", s, launch_rowperm(rc_, m, nc, ks, perm, s));
            LAUNCH("accum", s, launch_accum_sorted(atables, rc_, m, nc, l, L.slots, ks, acc_out, split_stride, s, acc_in,
                                                   perm, acc_mode == 3));
        } else if (w <= 4 && (acc_mode == 0 || (acc_mode >= 2 && m <= 64))) {      // m <= 64: 64-row k_accum CTAs
            LAUNCH("accum", s, launch_accum(atables, rc_, m, nc, l, L.slots, ks, acc_out, split_stride, s, acc_in));
        } else {
            LAUNCH("accum", s,
                   launch_accum_global(atables, rc_, m, nc, l, L.slots, ks, acc_out, split_stride, s, acc_in));
        }
        if (!direct) {
            uint32_t *partial = (uint32_t *)(ws + L.partial);
            LAUNCH("reduce", s, launch_reduce_splits(partial, ks, cnt, out, s, chunked && k0 > 0));
        }
    }
    return PCMM_OK;
}

int pcmm_mul_schoolbook(const int8_t *A_d, int m, int n, int l, int w, int is_signed, const uint8_t *ctB_d,
                        void *ctC_proj_d, void *ws_d, size_t ws_bytes, void *stream) {
    return mul_common(PCMM_PATH_SCHOOLBOOK, A_d, m, n, l, w, is_signed, 0, ctB_d, ctC_proj_d, ws_d, ws_bytes,
                      (cudaStream_t)stream);
}

static int mul_strassen(const void *A_d, int a_is_i32, int m, int n, int l, int w, int is_signed, int leaf,
                        const uint8_t *ctB_d, void *ctC_proj_d, void *ws_d, size_t ws_bytes, cudaStream_t s) {
    g_err.clear();
    int rc = check_dims(m, n, l);
    if (rc) return rc;
    if (!A_d || !ctB_d || !ctC_proj_d || !ws_d) return fail(PCMM_EINVAL, "null pointer");
    if (((uintptr_t)ctB_d & 15) || ((uintptr_t)ws_d & 255) || ((uintptr_t)ctC_proj_d & 15) ||
        (a_is_i32 && ((uintptr_t)A_d & 3)))
        return fail(PCMM_EINVAL, "misaligned buffer (A 4 B if int32, ctB/ctC 16 B, workspace 256 B)");
    if (w < 1 || w > (a_is_i32 ? 16 : 8)) return fail(PCMM_EINVAL, "w out of range (8 for int8 A, 16 for int32 A)");
    if (leaf < 1) return fail(PCMM_EINVAL, "leaf must be >= 1");
    const Layout L = layout(m, n, l, 1, PCMM_PATH_STRASSEN);
    if (ws_bytes < L.total) return fail(PCMM_ENOMEM, "workspace too small (see pcmm_workspace_bytes)");
    uint8_t *ws = (uint8_t *)ws_d;
    int *status = (int *)ws;
    uint32_t *bsoa = (uint32_t *)(ws + L.bsoa);
    CK(cudaMemsetAsync(status, 0, 4, s), "memset status");
    LAUNCH("import", s, launch_import(ctB_d, (int64_t)n * l, bsoa, status, s));
    LAUNCH("strassen", s,
           run_strassen(A_d, a_is_i32, m, n, l, w, is_signed, bsoa, leaf, (uint32_t *)ctC_proj_d, status, s));
    return PCMM_OK;
}

int pcmm_mul_strassen(const int8_t *A_d, int m, int n, int l, int w, int is_signed, int leaf, const uint8_t *ctB_d,
                      void *ctC_proj_d, void *ws_d, size_t ws_bytes, void *stream) {
    return mul_strassen(A_d, 0, m, n, l, w, is_signed, leaf, ctB_d, ctC_proj_d, ws_d, ws_bytes, (cudaStream_t)stream);
}

int pcmm_mul_strassen_wide(const int32_t *A_d, int m, int n, int l, int w, int is_signed, int leaf,
                           const uint8_t *ctB_d, void *ctC_proj_d, void *ws_d, size_t ws_bytes, void *stream) {
    return mul_strassen(A_d, 1, m, n, l, w, is_signed, leaf, ctB_d, ctC_proj_d, ws_d, ws_bytes, (cudaStream_t)stream);
}

int pcmm_mul_cussen(const int8_t *A_d, int m, int n, int l, int w, int is_signed, int iters, const uint8_t *ctB_d,
                    void *ctC_proj_d, void *ws_d, size_t ws_bytes, void *stream) {
    return mul_common(PCMM_PATH_CUSSEN, A_d, m, n, l, w, is_signed, iters, ctB_d, ctC_proj_d, ws_d, ws_bytes,
                      (cudaStream_t)stream);
}

size_t pcmm_workspace_bytes_wide(int m, int n, int l, int w, int path) {
    if (m <= 0 || n <= 0 || l <= 0 || w < 1 || w > 16) return 0;
    if (path == PCMM_PATH_STRASSEN) return layout(m, n, l, 1, PCMM_PATH_STRASSEN).total;
    if (m > kWideMaxM) return 0;
    if (path != PCMM_PATH_SCHOOLBOOK && path != PCMM_PATH_CUSSEN) return 0;
    return layout_wide(m, n, l, w, path).total;
}

static int mul_wide(int path, const int32_t *A_d, int m, int n, int l, int w, int is_signed, int iters,
                    const uint8_t *ctB_d, void *ctC_proj_d, void *ws_d, size_t ws_bytes, cudaStream_t s) {
    g_err.clear();
    int rc = check_dims(m, n, l);
    if (rc) return rc;
    if (m > kWideMaxM) return fail(PCMM_EDIM, "wide path: m must be <= 16384");
    if (!A_d || !ctB_d || !ctC_proj_d || !ws_d) return fail(PCMM_EINVAL, "null pointer");
    if (((uintptr_t)A_d & 3) || ((uintptr_t)ctB_d & 15) || ((uintptr_t)ws_d & 255) || ((uintptr_t)ctC_proj_d & 15))
        return fail(PCMM_EINVAL, "misaligned buffer (A 4 B, ctB/ctC 16 B, workspace 256 B)");
    if (w < 1 || w > 16) return fail(PCMM_EINVAL, "w must be in [1, 16]");
    if (path == PCMM_PATH_CUSSEN && (iters < 1 || iters > 4)) return fail(PCMM_ENOTSUP, "iters must be in [1, 4]");
    const LayoutW L = layout_wide(m, n, l, w, path);
    if (ws_bytes < L.total) return fail(PCMM_ENOMEM, "workspace too small (see pcmm_workspace_bytes_wide)");
    uint8_t *ws = (uint8_t *)ws_d;
    int *status = (int *)ws;
    uint32_t *bsoa = (uint32_t *)(ws + L.bsoa);
    uint32_t *out = (uint32_t *)ctC_proj_d;
    CK(cudaMemsetAsync(status, 0, 8, s), "memset status");      // [0] error bits, [1] k_plan's general-column flag
    LAUNCH("import", s, launch_import(ctB_d, (int64_t)n * l, bsoa, status, s));
    if (path == PCMM_PATH_SCHOOLBOOK) {
        LAUNCH("schoolbook", s, launch_schoolbook_wide(A_d, m, n, l, w, is_signed, bsoa, out, status, s));
        return PCMM_OK;
    }
    int32_t *pn = (int32_t *)(ws + L.pn), *psN = (int32_t *)(ws + L.psN);
    uint16_t *pptr = (uint16_t *)(ws + L.pptr), *rank = (uint16_t *)(ws + L.rank);
    uint32_t *tables = (uint32_t *)(ws + L.tables), *scratch = (uint32_t *)(ws + L.scratch);
    LAUNCH("plan", s, launch_plan_wide(A_d, m, n, w, is_signed, iters, L.cap, pn, psN, pptr, rank, status, s));
    for (int k0 = 0; k0 < n; k0 += L.KC) {
        const int kc = std::min(L.KC, n - k0);
        // few tables (fewer than two per SM): one CTA per table with block-scan prefix sums
        static int scan_env = -1;                             // PCMM_WIDE_SCAN: 0 never, 1 auto, 2 always
        if (scan_env < 0) {
            const char *e = getenv("PCMM_WIDE_SCAN");
            scan_env = e ? atoi(e) : 1;
        }
        const bool scan = scan_env == 2 || (scan_env == 1 && 2LL * kc * l <= 2LL * num_sms());   // t >= 12: the level-N ECSMs alone are long serial chains
        if (scan)
            LAUNCH("tables", s, launch_tables_wide_scan(bsoa, pn, psN, pptr, n, l, iters, L.cap, L.S, k0, kc, tables,
                                                        scratch, s));
        else
            LAUNCH("tables", s, launch_tables_wide(bsoa, pn, psN, pptr, n, l, iters, L.cap, L.S, k0, kc, tables,
                                                   scratch, s));
        LAUNCH("affine", s, launch_affine(tables, 2LL * kc * l * L.S, scratch, s));
        LAUNCH("accum", s, launch_accum_wide(scratch, rank, m, l, L.S, k0, kc, k0 == 0, out, s));
    }
    return PCMM_OK;
}

int pcmm_mul_cussen_wide(const int32_t *A_d, int m, int n, int l, int w, int is_signed, int iters,
                         const uint8_t *ctB_d, void *ctC_proj_d, void *ws_d, size_t ws_bytes, void *stream) {
    return mul_wide(PCMM_PATH_CUSSEN, A_d, m, n, l, w, is_signed, iters, ctB_d, ctC_proj_d, ws_d, ws_bytes,
                    (cudaStream_t)stream);
}

int pcmm_mul_schoolbook_wide(const int32_t *A_d, int m, int n, int l, int w, int is_signed, const uint8_t *ctB_d,
                             void *ctC_proj_d, void *ws_d, size_t ws_bytes, void *stream) {
    return mul_wide(PCMM_PATH_SCHOOLBOOK, A_d, m, n, l, w, is_signed, 0, ctB_d, ctC_proj_d, ws_d, ws_bytes,
                    (cudaStream_t)stream);
}

int pcmm_normalize(const void *ctC_proj_d, int64_t count, uint8_t *ctC_d, void *ws_d, size_t ws_bytes, void *stream) {
    g_err.clear();
    if (count < 0) return fail(PCMM_EINVAL, "count < 0");
    if (count == 0) return PCMM_OK;
    if (!ctC_proj_d || !ctC_d) return fail(PCMM_EINVAL, "null pointer");
    if (((uintptr_t)ctC_d & 15)) return fail(PCMM_EINVAL, "misaligned output (16 B)");
    (void)ws_d;
    (void)ws_bytes;
    cudaStream_t s = (cudaStream_t)stream;
    LAUNCH("normalize", s, launch_normalize((const uint32_t *)ctC_proj_d, count, ctC_d, s));
    return PCMM_OK;
}

int pcmm_decrypt_small(const uint8_t sk_h[32], const uint8_t *ct_d, int64_t count, int64_t lo, int64_t hi,
                       int64_t *m_d, int32_t *status_d, void *stream) {
    g_err.clear();
    if (count < 0 || hi < lo) return fail(PCMM_EINVAL, "count < 0 or hi < lo");
    if (hi - lo >= (1LL << 26) || lo <= -(1LL << 30) || hi >= (1LL << 30))
        return fail(PCMM_EINVAL, "range too large (hi - lo < 2^26, |lo|, |hi| < 2^30)");
    if (count == 0) return PCMM_OK;
    if (!sk_h || !ct_d || !m_d || !status_d) return fail(PCMM_EINVAL, "null pointer");
    if ((uintptr_t)ct_d & 15) return fail(PCMM_EINVAL, "misaligned buffer (ct 16 B)");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t tc = hi - lo + 1;
    uint32_t x[8];
    for (int i = 0; i < 8; i++) {
        const uint8_t *p = sk_h + 28 - 4 * i;
        x[i] = ((uint32_t)p[0] << 24) | ((uint32_t)p[1] << 16) | ((uint32_t)p[2] << 8) | p[3];
    }
    // baby-step giant-step (next2.cu) with a baby-step table sized for this call: s ~ sqrt(count x range)
    // balances the table build (s points) against the giant steps (range / s per ciphertext)
    const uint64_t range = (uint64_t)tc;
    int lb = 4;
    while (lb < 22 && ((uint64_t)1 << (2 * lb)) < range * (uint64_t)std::min<int64_t>(count, 1 << 20)) lb++;
    while ((range >> lb) > (1ULL << 24)) lb++;
    uint8_t *ctx = nullptr;
    CK(cudaMallocAsync((void **)&ctx, bsgs_ctx_bytes(lb), s), "cudaMallocAsync");
    int rc = PCMM_OK;
    do {
        prof_begin("bsgs_init", s);
        cudaError_t e = launch_bsgs_init(lb, (uint32_t *)ctx, s);
        prof_end(s);
        if (e) { rc = cuda_fail(e, "bsgs_init"); break; }
        prof_begin("decrypt", s);
        e = launch_decrypt_bsgs(x, (const uint32_t *)ctx, ct_d, count, lo, hi, m_d, status_d, s);
        prof_end(s);
        if (e) { rc = cuda_fail(e, "decrypt"); break; }
    } while (0);
    cudaFreeAsync(ctx, s);
    return rc;
}

// ---------------------------------------------------------------- NEXT-4: Paillier
static bool paillier_layout(int m, int n, int l, int w, int nbits, int path, size_t off[6], size_t *total, int *S,
                            int *maxup) {
    if (m <= 0 || n <= 0 || l <= 0 || w < 1 || w > 8 || (nbits % 32) != 0) return false;
    const int L = nbits / 32;
    if (!paillier_limbs_ok(L) || (path != 0 && path != 1)) return false;
    if ((int64_t)m * l > (1LL << 30) || (int64_t)n * l > (1LL << 30)) return false;
    *S = table_slots(w);
    *maxup = max_upper(w);
    size_t o = 256;
    off[0] = o;
    o = align256(o + (size_t)3 * L * 4);
    off[1] = o;
    o = align256(o + (size_t)n * l * L * 4);
    off[2] = off[3] = off[4] = off[5] = o;
    if (path == 1) {
        off[2] = o;
        o = align256(o + (size_t)n * sizeof(ColPlan));
        off[3] = o;
        o = align256(o + (size_t)n * m);
        off[4] = o;
        o = align256(o + (size_t)n * l * (*S) * L * 4);
        off[5] = o;
        o = align256(o + (size_t)n * l * 2 * (*maxup) * L * 4);
    }
    *total = o;
    return true;
}

size_t pcmm_paillier_workspace_bytes(int m, int n, int l, int w, int nbits_n2, int path) {
    size_t off[6], total = 0;
    int S, maxup;
    return paillier_layout(m, n, l, w, nbits_n2, path, off, &total, &S, &maxup) ? total : 0;
}

int pcmm_paillier_mul(int path, const uint8_t *A_d, int m, int n, int l, int w, int iters, const uint32_t *N2_h,
                      int nbits_n2, const uint32_t *ctB_d, uint32_t *ctC_d, void *ws_d, size_t ws_bytes,
                      void *stream) {
    g_err.clear();
    int rc = check_dims(m, n, l);
    if (rc) return rc;
    if (!A_d || !N2_h || !ctB_d || !ctC_d || !ws_d) return fail(PCMM_EINVAL, "null pointer");
    if (((uintptr_t)ws_d & 255) || ((uintptr_t)ctB_d & 3) || ((uintptr_t)ctC_d & 3))
        return fail(PCMM_EINVAL, "misaligned buffer (workspace 256 B, ciphertexts 4 B)");
    if (path != 0 && path != 1) return fail(PCMM_EINVAL, "path must be 0 (schoolbook) or 1 (Cussen)");
    if (w < 1 || w > 8) return fail(PCMM_EINVAL, "w must be in [1, 8]");
    if (path == 1 && (iters < 1 || iters > 4)) return fail(PCMM_ENOTSUP, "iters must be in [1, 4]");
    if (nbits_n2 % 32 || !paillier_limbs_ok(nbits_n2 / 32))
        return fail(PCMM_ENOTSUP, "n^2 must have 512, 1024, 2048 or 3072 bits");
    if (!(N2_h[0] & 1u)) return fail(PCMM_EINVAL, "n^2 must be odd");
    size_t off[6], total = 0;
    int S, maxup;
    if (!paillier_layout(m, n, l, w, nbits_n2, path, off, &total, &S, &maxup))
        return fail(PCMM_EDIM, "dimensions too large");
    if (ws_bytes < total) return fail(PCMM_ENOMEM, "workspace too small (see pcmm_paillier_workspace_bytes)");
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t *ws = (uint8_t *)ws_d;
    CK(cudaMemsetAsync(ws, 0, 4, s), "memset status");
    CK(run_paillier(path, A_d, m, n, l, w, iters, nbits_n2 / 32, N2_h, ctB_d, ctC_d, ws, off, S, maxup, s),
       "paillier");
    return PCMM_OK;
}

// ---------------------------------------------------------------- NEXT-2
size_t pcmm_enc_ctx_bytes(void) { return enc_ctx_bytes(); }

int pcmm_enc_ctx_init(const uint8_t pk_h[64], void *ctx_d, void *stream) {
    g_err.clear();
    if (!pk_h || !ctx_d) return fail(PCMM_EINVAL, "null pointer");
    if ((uintptr_t)ctx_d & 255) return fail(PCMM_EINVAL, "context must be 256-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    LAUNCH("enc_ctx_init", s, launch_enc_ctx_init(pk_h, (uint32_t *)ctx_d, s));
    uint32_t hdr[2] = {0, 0};
    CK(cudaMemcpyAsync(hdr, ctx_d, 8, cudaMemcpyDeviceToHost, s), "header copy");
    CK(cudaStreamSynchronize(s), "stream sync");
    if (hdr[1] != 1) {
        CK(cudaMemsetAsync(ctx_d, 0, 4, s), "clear magic");
        return fail(PCMM_ENOTONCURVE, "public key is not a point of P-256 (or is the identity)");
    }
    return PCMM_OK;
}

int pcmm_encrypt_ctx(const void *ctx_d, const int32_t *b_d, const uint8_t *r_d, int64_t count, uint8_t *ct_d,
                     void *stream) {
    g_err.clear();
    if (count < 0) return fail(PCMM_EINVAL, "count < 0");
    if (count == 0) return PCMM_OK;
    if (!ctx_d || !b_d || !r_d || !ct_d) return fail(PCMM_EINVAL, "null pointer");
    if (((uintptr_t)r_d & 15) || ((uintptr_t)ct_d & 15) || ((uintptr_t)ctx_d & 255))
        return fail(PCMM_EINVAL, "misaligned buffer (r / ct 16 B, context 256 B)");
    cudaStream_t s = (cudaStream_t)stream;
    LAUNCH("encrypt_comb", s, launch_encrypt_comb((const uint32_t *)ctx_d, b_d, r_d, count, ct_d, s));
    return PCMM_OK;
}

size_t pcmm_bsgs_ctx_bytes(int log2_baby) {
    if (log2_baby < 1 || log2_baby > 28) return 0;
    return bsgs_ctx_bytes(log2_baby);
}

int pcmm_bsgs_init(int log2_baby, void *ctx_d, void *stream) {
    g_err.clear();
    if (log2_baby < 1 || log2_baby > 28) return fail(PCMM_EINVAL, "log2_baby must be in [1, 28]");
    if (!ctx_d) return fail(PCMM_EINVAL, "null pointer");
    if ((uintptr_t)ctx_d & 255) return fail(PCMM_EINVAL, "context must be 256-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    LAUNCH("bsgs_init", s, launch_bsgs_init(log2_baby, (uint32_t *)ctx_d, s));
    return PCMM_OK;
}

int pcmm_decrypt_bsgs(const uint8_t sk_h[32], const void *ctx_d, int log2_baby, const uint8_t *ct_d, int64_t count,
                      int64_t lo, int64_t hi, int64_t *m_d, int32_t *status_d, void *stream) {
    g_err.clear();
    if (count < 0 || hi < lo) return fail(PCMM_EINVAL, "count < 0 or hi < lo");
    if (log2_baby < 1 || log2_baby > 28) return fail(PCMM_EINVAL, "log2_baby must be in [1, 28]");
    if (lo <= -(1LL << 62) || hi >= (1LL << 62)) return fail(PCMM_EINVAL, "|lo|, |hi| must be < 2^62");
    const uint64_t range = (uint64_t)(hi - lo) + 1;
    if ((range >> log2_baby) > (1ULL << 24)) return fail(PCMM_EINVAL, "range > 2^24 giant steps of 2^log2_baby");
    if (count == 0) return PCMM_OK;
    if (!sk_h || !ctx_d || !ct_d || !m_d || !status_d) return fail(PCMM_EINVAL, "null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t x[8];
    for (int i = 0; i < 8; i++) {
        const uint8_t *p = sk_h + 28 - 4 * i;
        x[i] = ((uint32_t)p[0] << 24) | ((uint32_t)p[1] << 16) | ((uint32_t)p[2] << 8) | p[3];
    }
    LAUNCH("decrypt_bsgs", s, launch_decrypt_bsgs(x, (const uint32_t *)ctx_d, ct_d, count, lo, hi, m_d, status_d, s));
    return PCMM_OK;
}

int pcmm_status(const void *ws_d, void *stream) {
    g_err.clear();
    if (!ws_d) return fail(PCMM_EINVAL, "null workspace");
    cudaStream_t s = (cudaStream_t)stream;
    int st = 0;
    CK(cudaMemcpyAsync(&st, ws_d, 4, cudaMemcpyDeviceToHost, s), "status copy");
    CK(cudaStreamSynchronize(s), "stream sync");
    if (st & kStatusCurve) return fail(PCMM_ENOTONCURVE, "an input point is not on P-256 (or not reduced)");
    if (st & kStatusBound) return fail(PCMM_EBOUND, "a plaintext entry is outside its w-bit range");
    return PCMM_OK;
}

int pcmm_profile_enable(int on) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto &r : g_prof) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    g_prof.clear();
    g_prof_on = on != 0;
    return PCMM_OK;
}

int pcmm_profile_read(char *names_h, float *ms_h, int max) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    int n = 0;
    for (auto &r : g_prof) {
        if (n >= max) break;
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e != cudaSuccess) return cuda_fail(e, "profile sync");
        float ms = 0;
        cudaEventElapsedTime(&ms, r.a, r.b);
        if (names_h) {
            strncpy(names_h + 48 * n, r.name, 47);
            names_h[48 * n + 47] = 0;
        }
        if (ms_h) ms_h[n] = ms;
        n++;
    }
    return n;
}

int pcmm_test_field(int op, const uint8_t *a_d, const uint8_t *b_d, uint8_t *out_d, int64_t count, void *stream) {
    g_err.clear();
    if (count < 0 || op < 0 || op > 12) return fail(PCMM_EINVAL, "bad op / count");
    if (count && (!a_d || !b_d || !out_d)) return fail(PCMM_EINVAL, "null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    LAUNCH("test_field", s, launch_test_field(op, a_d, b_d, out_d, count, s));
    return PCMM_OK;
}

int pcmm_test_point(int op, const uint8_t *p_d, const uint8_t *q_d, const int32_t *v_d, uint8_t *out_d,
                    int64_t count, void *stream) {
    g_err.clear();
    if (count < 0 || op < 0 || op > 4) return fail(PCMM_EINVAL, "bad op / count");
    if (count && (!p_d || !out_d || ((op == 0 || op == 3) && !q_d) || (op == 2 && !v_d)))
        return fail(PCMM_EINVAL, "null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    LAUNCH("test_point", s, launch_test_point(op, p_d, q_d, v_d, out_d, count, s));
    return PCMM_OK;
}

int pcmm_test_plan(const int8_t *A_d, int m, int n, int w, int is_signed, int iters, int32_t *levels_d,
                   int16_t *sN_d, uint8_t *rank_d, void *stream) {
    g_err.clear();
    int rc = check_dims(m, n, 1);
    if (rc) return rc;
    if (w < 1 || w > 8 || iters < 1 || iters > 4) return fail(PCMM_ENOTSUP, "w in [1,8], iters in [1,4]");
    if (!A_d || !levels_d || !sN_d || !rank_d) return fail(PCMM_EINVAL, "null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    ColPlan *plans = nullptr;
    int *status = nullptr;
    const size_t status_off = align256((size_t)n * sizeof(ColPlan));
    CK(cudaMallocAsync((void **)&plans, status_off + 256, s), "alloc");
    status = (int *)((uint8_t *)plans + status_off);
    cudaMemsetAsync(status, 0, 4, s);
    cudaError_t e = launch_plan(A_d, m, n, w, is_signed, iters, plans, rank_d, status, s);
    std::vector<ColPlan> hp(n);
    int st = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(hp.data(), plans, (size_t)n * sizeof(ColPlan), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&st, status, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFreeAsync(plans, s);
    if (e != cudaSuccess) return cuda_fail(e, "test_plan");
    std::vector<int32_t> lev((size_t)n * 4);
    std::vector<int16_t> sn((size_t)n * kPlanCap);
    for (int k = 0; k < n; k++) {
        for (int q = 0; q < 4; q++) lev[(size_t)k * 4 + q] = hp[k].n[q];
        for (int q = 0; q < kPlanCap; q++) sn[(size_t)k * kPlanCap + q] = q < hp[k].n[iters - 1] ? hp[k].sN[q] : 0;
    }
    CK(cudaMemcpy(levels_d, lev.data(), lev.size() * 4, cudaMemcpyHostToDevice), "copy levels");
    CK(cudaMemcpy(sN_d, sn.data(), sn.size() * 2, cudaMemcpyHostToDevice), "copy sN");
    if (st & kStatusBound) return fail(PCMM_EBOUND, "a plaintext entry is outside its w-bit range");
    return PCMM_OK;
}

int pcmm_bench_fp_mul(int variant, int blocks, int threads, int iters, uint32_t *out_d, void *stream) {
    g_err.clear();
    if (blocks <= 0 || threads <= 0 || threads > 128 || iters < 0 || !out_d) return fail(PCMM_EINVAL, "bad args");
    cudaStream_t s = (cudaStream_t)stream;
    LAUNCH("bench_fp_mul", s, launch_bench_fp_mul(variant, blocks, threads, iters, out_d, s));
    return PCMM_OK;
}

}  // extern "C"
