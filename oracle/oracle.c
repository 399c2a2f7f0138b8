/*
 * oracle.c -- plain, slow, CPU oracle for plaintext-ciphertext matrix
 * multiplication (PC-MM) over EC-ElGamal on NIST P-256.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant generator with the CUDA path in
 * paper_2504_14497_b200/ (which must never load it).
 *
 * Everything follows arXiv 2504.14497 ("PAPER.md" line numbers, P:L):
 *   - prime field / curve:        P:496 (p = 2^256 - 2^224 + 2^192 + 2^96 - 1,
 *                                 y^2 = x^3 - 3x + b, prime order q)
 *   - group law, ECSM:            P:150-155, Alg. 1 (Montgomery ladder) P:159-172
 *   - EC-ElGamal:                 P:179-183 (KeyGen / Encrypt / Decrypt)
 *   - homomorphism (Eq. 5):
 *   - schoolbook PC-MM:
 *   - Cussen compression /
 *     reconstruction (Alg. 2):
 *   - proposed PC-MM (Alg. 3):
 * with the readings R1-R17 listed in DESIGN.md.
 *
 * Implementation choices (deliberately different from the GPU path):
 *   - 4 x 64-bit little-endian limbs, unsigned __int128 products;
 *   - values are kept in NORMAL (non-Montgomery) form; a modular product is
 *     two textbook CIOS Montgomery multiplications (HAC Alg. 14.36):
 *     mont(mont(a, b), R^2 mod M) = a*b mod M, for any odd modulus M;
 *   - R^2 mod M is built by 512 modular doublings of 1, -M^-1 mod 2^64 by
 *     Newton iteration, inversion by Fermat (a^(M-2));
 *   - Jacobian coordinates with EXPLICIT special cases (infinity, P == Q,
 *     P == -Q), textbook formulas (Hankerson-Menezes-Vanstone, Guide to ECC,
 *     Sec. 3.2.2), affine only for the final normalisation;
 *   - scalar multiplication by small plaintexts uses the paper's Montgomery
 *     ladder (Alg. 1) with the declared bit width t, so that operation counts
 *     follow the paper's cost model.
 *
 * Canonical encodings (R13): a point is 64 bytes x||y, each 32-byte
 * big-endian; infinity is 64 zero bytes ((0,0) is not on the curve since
 * b != 0).  A ciphertext is 128 bytes C1||C2.  Scalars are 32-byte big-endian.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

typedef unsigned __int128 u128;
typedef struct { uint64_t v[4]; } big;          /* little-endian 64-bit limbs */

typedef struct {
    big M;          /* odd modulus */
    big R2;         /* 2^512 mod M */
    uint64_t minv;  /* -M^-1 mod 2^64 */
} modctx;

/* ---- constants of NIST P-256 (SEC 2 v2 Sec. 2.4.2) ---------------- */
static const char *HEX_P  = "ffffffff00000001000000000000000000000000ffffffffffffffffffffffff";
static const char *HEX_Q  = "ffffffff00000000ffffffffffffffffbce6faada7179e84f3b9cac2fc632551";
static const char *HEX_B  = "5ac635d8aa3a93e7b3ebbd55769886bc651d06b0cc53b0f63bce3c3e27d2604b";
static const char *HEX_GX = "6b17d1f2e12c4247f8bce6e563a440f277037d812deb33a0f4a13945d898c296";
static const char *HEX_GY = "4fe342e2fe1a7f9b8ee7eb4a7c0f9e162bce33576b315ececbb6406837bf51f5";

static modctx FP, FQ;
static big CURVE_B, CURVE_A;   /* a = -3 mod p */
static big GX, GY;
static int g_inited = 0;

/* ---------------------------------------------------------------- bignum -- */
static int hexval(char c) {
    if (c >= '0' && c <= '9') return c - '0';
    if (c >= 'a' && c <= 'f') return c - 'a' + 10;
    if (c >= 'A' && c <= 'F') return c - 'A' + 10;
    return -1;
}

static big big_from_hex(const char *h) {
    big r; memset(&r, 0, sizeof r);
    size_t len = strlen(h);
    for (size_t i = 0; i < len; i++) {
        int d = hexval(h[len - 1 - i]);
        r.v[i / 16] |= (uint64_t)d << (4 * (i % 16));
    }
    return r;
}

static big big_from_be(const uint8_t *b) {
    big r;
    for (int i = 0; i < 4; i++) {
        uint64_t w = 0;
        for (int j = 0; j < 8; j++) w = (w << 8) | b[(3 - i) * 8 + j];
        r.v[i] = w;
    }
    return r;
}

static void big_to_be(const big *a, uint8_t *b) {
    for (int i = 0; i < 4; i++)
        for (int j = 0; j < 8; j++)
            b[(3 - i) * 8 + j] = (uint8_t)(a->v[i] >> (56 - 8 * j));
}

static big big_u64(uint64_t x) { big r = {{x, 0, 0, 0}}; return r; }

static int big_is_zero(const big *a) { return (a->v[0] | a->v[1] | a->v[2] | a->v[3]) == 0; }

static int big_cmp(const big *a, const big *b) {
    for (int i = 3; i >= 0; i--) {
        if (a->v[i] > b->v[i]) return 1;
        if (a->v[i] < b->v[i]) return -1;
    }
    return 0;
}

static uint64_t big_add(big *r, const big *a, const big *b) {
    u128 c = 0;
    for (int i = 0; i < 4; i++) {
        c += (u128)a->v[i] + b->v[i];
        r->v[i] = (uint64_t)c;
        c >>= 64;
    }
    return (uint64_t)c;
}

static uint64_t big_sub(big *r, const big *a, const big *b) {
    uint64_t borrow = 0;
    for (int i = 0; i < 4; i++) {
        uint64_t ai = a->v[i], bi = b->v[i];
        uint64_t d = ai - bi - borrow;
        borrow = (ai < bi) || (ai == bi && borrow) ? 1 : 0;
        r->v[i] = d;
    }
    return borrow;
}

static int big_bit(const big *a, int i) { return (int)((a->v[i / 64] >> (i % 64)) & 1); }

static int big_bitlen(const big *a) {
    for (int i = 255; i >= 0; i--) if (big_bit(a, i)) return i + 1;
    return 0;
}

/* ------------------------------------------------------- modular arithmetic */
/* r = a + b mod M, for a, b < M */
static big mod_add(const modctx *c, big a, big b) {
    big r; uint64_t carry = big_add(&r, &a, &b);
    if (carry || big_cmp(&r, &c->M) >= 0) big_sub(&r, &r, &c->M);
    return r;
}

/* r = a - b mod M, for a, b < M */
static big mod_sub(const modctx *c, big a, big b) {
    big r; uint64_t borrow = big_sub(&r, &a, &b);
    if (borrow) big_add(&r, &r, &c->M);
    return r;
}

/* HAC Alg. 14.36 (CIOS Montgomery multiplication): a*b*2^-256 mod M, a,b < M */
static big mont_mul(const modctx *c, const big *a, const big *b) {
    uint64_t t[6] = {0, 0, 0, 0, 0, 0};
    for (int i = 0; i < 4; i++) {
        u128 carry = 0;
        for (int j = 0; j < 4; j++) {
            carry += (u128)a->v[i] * b->v[j] + t[j];
            t[j] = (uint64_t)carry;
            carry >>= 64;
        }
        carry += t[4];
        t[4] = (uint64_t)carry;
        t[5] = (uint64_t)(carry >> 64);
        uint64_t u = t[0] * c->minv;
        carry = (u128)u * c->M.v[0] + t[0];
        carry >>= 64;
        for (int j = 1; j < 4; j++) {
            carry += (u128)u * c->M.v[j] + t[j];
            t[j - 1] = (uint64_t)carry;
            carry >>= 64;
        }
        carry += t[4];
        t[3] = (uint64_t)carry;
        t[4] = t[5] + (uint64_t)(carry >> 64);
    }
    big r = {{t[0], t[1], t[2], t[3]}};
    if (t[4] || big_cmp(&r, &c->M) >= 0) big_sub(&r, &r, &c->M);
    return r;
}

/* a*b mod M (normal representation in and out) */
static big mod_mul(const modctx *c, big a, big b) {
    big t = mont_mul(c, &a, &b);
    return mont_mul(c, &t, &c->R2);
}

static big mod_pow(const modctx *c, big a, const big *e) {
    big r = big_u64(1);
    for (int i = 255; i >= 0; i--) {
        r = mod_mul(c, r, r);
        if (big_bit(e, i)) r = mod_mul(c, r, a);
    }
    return r;
}

/* Fermat inversion: a^(M-2) mod M, M prime; inverse of 0 is returned as 0. */
static big mod_inv(const modctx *c, big a) {
    big e, two = big_u64(2);
    big_sub(&e, &c->M, &two);
    return mod_pow(c, a, &e);
}

/* reduce an arbitrary 256-bit value mod M (M > 2^255 for p and q) */
static big mod_reduce(const modctx *c, big a) {
    while (big_cmp(&a, &c->M) >= 0) big_sub(&a, &a, &c->M);
    return a;
}

static void modctx_init(modctx *c, const big *M) {
    c->M = *M;
    uint64_t inv = 1;                         /* Newton: inv <- inv (2 - M0 inv) */
    for (int i = 0; i < 7; i++) inv *= 2 - M->v[0] * inv;
    c->minv = (uint64_t)0 - inv;
    big r = big_u64(1);                       /* 2^512 mod M by doubling */
    for (int i = 0; i < 512; i++) r = mod_add(c, r, r);
    c->R2 = r;
}

static void oracle_init_once(void) {
    if (g_inited) return;
    big p = big_from_hex(HEX_P), q = big_from_hex(HEX_Q);
    modctx_init(&FP, &p);
    modctx_init(&FQ, &q);
    CURVE_B = big_from_hex(HEX_B);
    big three = big_u64(3);
    big_sub(&CURVE_A, &p, &three);
    GX = big_from_hex(HEX_GX);
    GY = big_from_hex(HEX_GY);
    g_inited = 1;
}

/* ------------------------------------------------------------- the curve -- */
typedef struct { big X, Y, Z; } jac;  /* (X/Z^2, Y/Z^3); Z == 0 <=> infinity */

typedef struct {
    uint64_t adds;      /* executed point additions (incl. those with infinity) */
    uint64_t dbls;      /* executed point doublings */
    uint64_t ecsm;      /* small-scalar multiplications (ladders) */
    uint64_t ecsm_bits; /* sum of declared ladder widths */
} counters;

static jac jac_inf(void) { jac r; memset(&r, 0, sizeof r); r.X = big_u64(1); r.Y = big_u64(1); return r; }
static int jac_is_inf(const jac *P) { return big_is_zero(&P->Z); }

static jac jac_from_affine(const big *x, const big *y) {
    jac r; r.X = *x; r.Y = *y; r.Z = big_u64(1); return r;
}

/* y^2 == x^3 + a x + b */
static int on_curve(const big *x, const big *y) {
    if (big_cmp(x, &FP.M) >= 0 || big_cmp(y, &FP.M) >= 0) return 0;
    big y2 = mod_mul(&FP, *y, *y);
    big x3 = mod_mul(&FP, mod_mul(&FP, *x, *x), *x);
    big ax = mod_mul(&FP, CURVE_A, *x);
    big rhs = mod_add(&FP, mod_add(&FP, x3, ax), CURVE_B);
    return big_cmp(&y2, &rhs) == 0;
}

/* Doubling in Jacobian coordinates, a = -3 (HMV Alg. 3.21 / standard formula):
 *   M = 3 (X - Z^2)(X + Z^2),  S = 4 X Y^2,
 *   X3 = M^2 - 2S,  Y3 = M (S - X3) - 8 Y^4,  Z3 = 2 Y Z.                    */
static jac jac_dbl(const jac *P, counters *cnt) {
    if (cnt) cnt->dbls++;
    if (jac_is_inf(P) || big_is_zero(&P->Y)) return jac_inf();
    const modctx *f = &FP;
    big Z2 = mod_mul(f, P->Z, P->Z);
    big M = mod_mul(f, mod_sub(f, P->X, Z2), mod_add(f, P->X, Z2));
    M = mod_add(f, mod_add(f, M, M), M);
    big Y2 = mod_mul(f, P->Y, P->Y);
    big S = mod_mul(f, P->X, Y2);
    S = mod_add(f, S, S); S = mod_add(f, S, S);
    big X3 = mod_sub(f, mod_mul(f, M, M), mod_add(f, S, S));
    big Y4 = mod_mul(f, Y2, Y2);
    big Y4_8 = mod_add(f, Y4, Y4); Y4_8 = mod_add(f, Y4_8, Y4_8); Y4_8 = mod_add(f, Y4_8, Y4_8);
    big Y3 = mod_sub(f, mod_mul(f, M, mod_sub(f, S, X3)), Y4_8);
    big YZ = mod_mul(f, P->Y, P->Z);
    jac r; r.X = X3; r.Y = Y3; r.Z = mod_add(f, YZ, YZ);
    return r;
}

/* General addition in Jacobian coordinates with explicit special cases:
 *   U1 = X1 Z2^2, U2 = X2 Z1^2, S1 = Y1 Z2^3, S2 = Y2 Z1^3, H = U2-U1, R = S2-S1
 *   H == 0: R == 0 -> 2P, else -> infinity
 *   X3 = R^2 - H^3 - 2 U1 H^2, Y3 = R (U1 H^2 - X3) - S1 H^3, Z3 = H Z1 Z2    */
static jac jac_add(const jac *P, const jac *Q, counters *cnt) {
    if (jac_is_inf(P)) { if (cnt) cnt->adds++; return *Q; }
    if (jac_is_inf(Q)) { if (cnt) cnt->adds++; return *P; }
    const modctx *f = &FP;
    big Z1s = mod_mul(f, P->Z, P->Z), Z2s = mod_mul(f, Q->Z, Q->Z);
    big U1 = mod_mul(f, P->X, Z2s), U2 = mod_mul(f, Q->X, Z1s);
    big S1 = mod_mul(f, P->Y, mod_mul(f, Z2s, Q->Z));
    big S2 = mod_mul(f, Q->Y, mod_mul(f, Z1s, P->Z));
    big H = mod_sub(f, U2, U1), R = mod_sub(f, S2, S1);
    if (big_is_zero(&H)) {
        if (big_is_zero(&R)) return jac_dbl(P, cnt);   /* counted as a doubling */
        if (cnt) cnt->adds++;
        return jac_inf();
    }
    if (cnt) cnt->adds++;
    big H2 = mod_mul(f, H, H), H3 = mod_mul(f, H2, H);
    big U1H2 = mod_mul(f, U1, H2);
    big X3 = mod_sub(f, mod_sub(f, mod_mul(f, R, R), H3), mod_add(f, U1H2, U1H2));
    big Y3 = mod_sub(f, mod_mul(f, R, mod_sub(f, U1H2, X3)), mod_mul(f, S1, H3));
    jac r; r.X = X3; r.Y = Y3; r.Z = mod_mul(f, H, mod_mul(f, P->Z, Q->Z));
    return r;
}

static jac jac_neg(const jac *P) {
    jac r = *P;
    if (!jac_is_inf(P)) r.Y = mod_sub(&FP, big_u64(0), P->Y);
    return r;
}

/* affine normalisation: x = X/Z^2, y = Y/Z^3 (infinity -> flag) */
static void jac_to_affine(const jac *P, big *x, big *y, int *inf) {
    if (jac_is_inf(P)) { *inf = 1; *x = big_u64(0); *y = big_u64(0); return; }
    big zi = mod_inv(&FP, P->Z);
    big zi2 = mod_mul(&FP, zi, zi);
    *x = mod_mul(&FP, P->X, zi2);
    *y = mod_mul(&FP, P->Y, mod_mul(&FP, zi2, zi));
    *inf = 0;
}

/* k*P for an arbitrary 256-bit k, MSB-first double-and-add */
static jac scalar_mul(const big *k, const jac *P) {
    jac R = jac_inf();
    for (int i = 255; i >= 0; i--) {
        R = jac_dbl(&R, NULL);
        if (big_bit(k, i)) R = jac_add(&R, P, NULL);
    }
    return R;
}

/* Alg. 1: Montgomery ladder for a t-bit k >= 0:
 *   R0 <- inf, R1 <- P; for i = t-1 .. 0: b <- k_i; R_{1-b} <- R1 + R0; R_b <- 2 R_b
 * exactly t additions and t doublings.                                       */
static jac ladder_mul(uint64_t k, int t, const jac *P, counters *cnt) {
    jac R[2]; R[0] = jac_inf(); R[1] = *P;
    for (int i = t - 1; i >= 0; i--) {
        int b = (int)((k >> i) & 1);
        jac sum = jac_add(&R[1], &R[0], cnt);
        jac dbl = jac_dbl(&R[b], cnt);
        R[1 - b] = sum;
        R[b] = dbl;
    }
    if (cnt) { cnt->ecsm++; cnt->ecsm_bits += (uint64_t)t; }
    return R[0];
}

static int bits_needed(uint64_t v) { int t = 0; while (v) { t++; v >>= 1; } return t; }

/* v*P for a small signed plaintext v (R10: v < 0 -> -(|v| P), which is
 * the same group element as (q - |v|) P).  Width t = max(declared width, bits). */
static jac small_mul(int64_t v, int t, const jac *P, counters *cnt) {
    uint64_t a = v < 0 ? (uint64_t)(-v) : (uint64_t)v;
    int need = bits_needed(a);
    if (need > t) t = need;
    if (t == 0) t = 1;
    jac r = ladder_mul(a, t, P, cnt);
    return v < 0 ? jac_neg(&r) : r;
}

/* ------------------------------------------------------ canonical encodings */
static void point_to_bytes(const jac *P, uint8_t *out64) {
    big x, y; int inf;
    jac_to_affine(P, &x, &y, &inf);
    if (inf) { memset(out64, 0, 64); return; }
    big_to_be(&x, out64);
    big_to_be(&y, out64 + 32);
}

/* returns 0 ok, -4 not on curve */
static int point_from_bytes(const uint8_t *in64, jac *P) {
    int zero = 1;
    for (int i = 0; i < 64; i++) if (in64[i]) { zero = 0; break; }
    if (zero) { *P = jac_inf(); return 0; }
    big x = big_from_be(in64), y = big_from_be(in64 + 32);
    if (!on_curve(&x, &y)) return -4;
    *P = jac_from_affine(&x, &y);
    return 0;
}

static big scalar_from_i64(int64_t v) {
    if (v >= 0) return big_u64((uint64_t)v);
    big a = big_u64((uint64_t)(-v)), r;
    big_sub(&r, &FQ.M, &a);
    return r;
}

/* ========================================================= exported API === */
#define EXPORT __attribute__((visibility("default")))

EXPORT void oracle_init(void) { oracle_init_once(); }

/* --- raw field / scalar arithmetic (pinned against Python ints, P2) ------- */
/* which: 0 -> mod p, 1 -> mod q.  op: 0 add, 1 sub, 2 mul, 3 inv, 4 pow     */
EXPORT int oracle_modop(int which, int op, const uint8_t *a_be, const uint8_t *b_be, uint8_t *out_be) {
    oracle_init_once();
    const modctx *c = which ? &FQ : &FP;
    big a = mod_reduce(c, big_from_be(a_be));
    big b = b_be ? big_from_be(b_be) : big_u64(0);
    big r;
    switch (op) {
        case 0: r = mod_add(c, a, mod_reduce(c, b)); break;
        case 1: r = mod_sub(c, a, mod_reduce(c, b)); break;
        case 2: r = mod_mul(c, a, mod_reduce(c, b)); break;
        case 3: r = mod_inv(c, a); break;
        case 4: r = mod_pow(c, a, &b); break;
        default: return -1;
    }
    big_to_be(&r, out_be);
    return 0;
}

/* --- group operations on canonical 64-byte points ------------------------- */
EXPORT int oracle_point_on_curve(const uint8_t *pt64) {
    oracle_init_once();
    jac P; return point_from_bytes(pt64, &P) == 0 ? 1 : 0;
}

EXPORT int oracle_point_add(const uint8_t *p64, const uint8_t *q64, uint8_t *out64) {
    oracle_init_once();
    jac P, Q;
    if (point_from_bytes(p64, &P) || point_from_bytes(q64, &Q)) return -4;
    jac R = jac_add(&P, &Q, NULL);
    point_to_bytes(&R, out64);
    return 0;
}

EXPORT int oracle_point_dbl(const uint8_t *p64, uint8_t *out64) {
    oracle_init_once();
    jac P;
    if (point_from_bytes(p64, &P)) return -4;
    jac R = jac_dbl(&P, NULL);
    point_to_bytes(&R, out64);
    return 0;
}

EXPORT int oracle_point_neg(const uint8_t *p64, uint8_t *out64) {
    oracle_init_once();
    jac P;
    if (point_from_bytes(p64, &P)) return -4;
    jac R = jac_neg(&P);
    point_to_bytes(&R, out64);
    return 0;
}

/* k*P, k a 32-byte big-endian scalar (any value; reduced by the group law) */
EXPORT int oracle_scalar_mul(const uint8_t *k_be, const uint8_t *p64, uint8_t *out64) {
    oracle_init_once();
    jac P;
    if (point_from_bytes(p64, &P)) return -4;
    big k = big_from_be(k_be);
    jac R = scalar_mul(&k, &P);
    point_to_bytes(&R, out64);
    return 0;
}

/* k*G */
EXPORT int oracle_scalar_mul_base(const uint8_t *k_be, uint8_t *out64) {
    oracle_init_once();
    jac G = jac_from_affine(&GX, &GY);
    big k = big_from_be(k_be);
    jac R = scalar_mul(&k, &G);
    point_to_bytes(&R, out64);
    return 0;
}

/* Alg. 1 ladder k*P with width t; counts returned in cnt_out[4] = adds, dbls, ecsm, bits */
EXPORT int oracle_ladder_mul(uint64_t k, int t, const uint8_t *p64, uint8_t *out64, uint64_t *cnt_out) {
    oracle_init_once();
    jac P;
    if (point_from_bytes(p64, &P)) return -4;
    counters c = {0, 0, 0, 0};
    jac R = ladder_mul(k, t, &P, &c);
    point_to_bytes(&R, out64);
    if (cnt_out) { cnt_out[0] = c.adds; cnt_out[1] = c.dbls; cnt_out[2] = c.ecsm; cnt_out[3] = c.ecsm_bits; }
    return 0;
}

EXPORT void oracle_generator(uint8_t *out64) {
    oracle_init_once();
    big_to_be(&GX, out64); big_to_be(&GY, out64 + 32);
}

/* --- EC-ElGamal ------------------------------------------------ */
/* KeyGen given x: H = x G */
EXPORT int oracle_pubkey(const uint8_t *x_be, uint8_t *H64) {
    return oracle_scalar_mul_base(x_be, H64);
}

/* Encrypt: (r G, r H + phi(b)), phi(b) = b G; b may be negative.
 * Elements are independent; they are split over `nthreads` pthreads.          */
typedef struct { jac H; int64_t e0, e1; const int64_t *b; const uint8_t *r_be; uint8_t *ct; } enc_job;

static void *enc_worker(void *arg) {
    enc_job *J = (enc_job *)arg;
    jac G = jac_from_affine(&GX, &GY);
    for (int64_t e = J->e0; e < J->e1; e++) {
        big r = big_from_be(J->r_be + 32 * e);
        big bs = scalar_from_i64(J->b[e]);
        jac C1 = scalar_mul(&r, &G);
        jac rH = scalar_mul(&r, &J->H);
        jac bG = scalar_mul(&bs, &G);
        jac C2 = jac_add(&rH, &bG, NULL);
        point_to_bytes(&C1, J->ct + 128 * e);
        point_to_bytes(&C2, J->ct + 128 * e + 64);
    }
    return NULL;
}

EXPORT int oracle_encrypt(const uint8_t *H64, int64_t count, const int64_t *b, const uint8_t *r_be,
                          uint8_t *ct128, int nthreads) {
    oracle_init_once();
    jac H;
    if (point_from_bytes(H64, &H)) return -4;
    if (nthreads < 1) nthreads = 1;
    if (count < nthreads) nthreads = count > 0 ? (int)count : 1;
    enc_job *jobs = (enc_job *)calloc((size_t)nthreads, sizeof(enc_job));
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int w = 0; w < nthreads; w++) {
        jobs[w].H = H; jobs[w].b = b; jobs[w].r_be = r_be; jobs[w].ct = ct128;
        jobs[w].e0 = count * w / nthreads; jobs[w].e1 = count * (w + 1) / nthreads;
        pthread_create(&th[w], NULL, enc_worker, &jobs[w]);
    }
    for (int w = 0; w < nthreads; w++) pthread_join(th[w], NULL);
    free(jobs); free(th);
    return 0;
}

/* Eq. 5 closed form of one output of PC-MM, straight from the
 * plaintext inputs: with R = sum_k a_k r_k mod q and c = sum_k a_k b_k,
 *   Enc(c) = ( R G , (x R + c) G ).
 * Inputs: x (32 B BE), a[n] (int32), b[n] (int64), r[n] (32 B BE each).         */
EXPORT int oracle_closed_form(const uint8_t *x_be, int n, const int32_t *a, const int64_t *b, const uint8_t *r_be,
                              uint8_t *out128) {
    oracle_init_once();
    big R = big_u64(0), c = big_u64(0);
    for (int k = 0; k < n; k++) {
        big ak = scalar_from_i64(a[k]);
        big rk = mod_reduce(&FQ, big_from_be(r_be + 32 * (size_t)k));
        R = mod_add(&FQ, R, mod_mul(&FQ, ak, rk));
        c = mod_add(&FQ, c, mod_mul(&FQ, ak, scalar_from_i64(b[k])));
    }
    big x = mod_reduce(&FQ, big_from_be(x_be));
    big s2 = mod_add(&FQ, mod_mul(&FQ, x, R), c);
    jac G = jac_from_affine(&GX, &GY);
    jac C1 = scalar_mul(&R, &G), C2 = scalar_mul(&s2, &G);
    point_to_bytes(&C1, out128);
    point_to_bytes(&C2, out128 + 64);
    return 0;
}

typedef struct { uint8_t key[64]; int64_t m; } dlog_entry;

static int dlog_cmp(const void *a, const void *b) {
    return memcmp(((const dlog_entry *)a)->key, ((const dlog_entry *)b)->key, 64);
}

/* Decrypt: m = phi^{-1}(C2 - x C1) by exhaustive table over [lo, hi].
 * status[e] = 0 on success, -5 (PCMM_EDECODE) when no m in [lo, hi] matches.  */
EXPORT int oracle_decrypt(const uint8_t *x_be, int64_t count, const uint8_t *ct128, int64_t lo, int64_t hi,
                          int64_t *m_out, int32_t *status) {
    oracle_init_once();
    if (hi < lo) return -1;
    int64_t span = hi - lo + 1;
    dlog_entry *tab = (dlog_entry *)malloc(sizeof(dlog_entry) * (size_t)span);
    if (!tab) return -7;
    jac G = jac_from_affine(&GX, &GY);
    big los = scalar_from_i64(lo);
    jac cur = scalar_mul(&los, &G);
    for (int64_t i = 0; i < span; i++) {
        point_to_bytes(&cur, tab[i].key);
        tab[i].m = lo + i;
        cur = jac_add(&cur, &G, NULL);
    }
    qsort(tab, (size_t)span, sizeof(dlog_entry), dlog_cmp);
    big x = big_from_be(x_be);
    for (int64_t e = 0; e < count; e++) {
        jac C1, C2;
        if (point_from_bytes(ct128 + 128 * e, &C1) || point_from_bytes(ct128 + 128 * e + 64, &C2)) {
            status[e] = -4; m_out[e] = 0; continue;
        }
        jac xC1 = scalar_mul(&x, &C1);
        jac nx = jac_neg(&xC1);
        jac M = jac_add(&C2, &nx, NULL);
        dlog_entry probe; point_to_bytes(&M, probe.key);
        dlog_entry *hit = (dlog_entry *)bsearch(&probe, tab, (size_t)span, sizeof(dlog_entry), dlog_cmp);
        if (hit) { m_out[e] = hit->m; status[e] = 0; }
        else { m_out[e] = 0; status[e] = -5; }
    }
    free(tab);
    return 0;
}

/* ================================================ Cussen's algorithm ======= */
#define MAXLEV 16

typedef struct {
    int N;                  /* iterations of compression / reconstruction */
    int len0;               /* n_0 = length of the input vector */
    int n[MAXLEV + 1];      /* n[w] = length of a^(w), w = 1..N */
    int64_t *s[MAXLEV + 1]; /* a^(w): sorted distinct (nonzero) values, BEFORE differencing */
    int *ptr[MAXLEV + 1];   /* ptr[w][e], e < n[w-1]: index of a^(w-1)[e] in a^(w); -1 if zero */
} colplan;

static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* Alg. 2 compression phase, with reading R1 (value 0 is dropped:
 * 0 * ct = infinity costs nothing; it is the only reading that reproduces
 * Tables A1/A2) and R3 (tracking pointer of element e of level w-1 = index of
 * its value in the sorted, de-duplicated level w).                            */
static int cussen_compress(const int64_t *a, int len, int N, colplan *pl) {
    memset(pl, 0, sizeof *pl);
    if (N < 1 || N > MAXLEV) return -1;
    pl->N = N; pl->len0 = len;
    int64_t *v = (int64_t *)malloc(sizeof(int64_t) * (size_t)(len > 0 ? len : 1));
    int vlen = len;
    memcpy(v, a, sizeof(int64_t) * (size_t)len);
    for (int w = 1; w <= N; w++) {
        /* line 5: sort a^(w-1), eliminate duplicates (and zeros, R1) */
        int64_t *s = (int64_t *)malloc(sizeof(int64_t) * (size_t)(vlen > 0 ? vlen : 1));
        int ns = 0;
        for (int e = 0; e < vlen; e++) if (v[e] != 0) s[ns++] = v[e];
        qsort(s, (size_t)ns, sizeof(int64_t), cmp_i64);
        int u = 0;
        for (int e = 0; e < ns; e++) if (u == 0 || s[e] != s[u - 1]) s[u++] = s[e];
        ns = u;
        /* "store pointers to track sorting order" */
        int *ptr = (int *)malloc(sizeof(int) * (size_t)(vlen > 0 ? vlen : 1));
        for (int e = 0; e < vlen; e++) {
            if (v[e] == 0) { ptr[e] = -1; continue; }
            int lo = 0, hi = ns - 1;
            while (lo < hi) { int mid = (lo + hi) / 2; if (s[mid] < v[e]) lo = mid + 1; else hi = mid; }
            ptr[e] = lo;
        }
        pl->n[w] = ns; pl->s[w] = s; pl->ptr[w] = ptr;
        /* lines 6-10: differences of consecutive elements, i = n_w .. 2 */
        free(v);
        v = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ns > 0 ? ns : 1));
        for (int e = 0; e < ns; e++) v[e] = s[e];
        if (w != N) for (int i = ns - 1; i >= 1; i--) v[i] = v[i] - v[i - 1];
        vlen = ns;
        /* the next level sorts the differenced vector */
    }
    free(v);
    return 0;
}

static void colplan_free(colplan *pl) {
    for (int w = 1; w <= pl->N; w++) { free(pl->s[w]); free(pl->ptr[w]); }
    memset(pl, 0, sizeof *pl);
}

/* value of element u of the (possibly differenced) vector at level w: the
 * vector that level w+1 sorts and the reconstruction multiplies / prefix-sums */
static int64_t level_value(const colplan *pl, int w, int u) {
    if (w == pl->N || u == 0) return pl->s[w][u];
    return pl->s[w][u] - pl->s[w][u - 1];
}

/* counts of one compressed column:
 *   mults     = n_N                         (Table A1 quantity)
 *   adds_pm   = sum_{w<N} n_w               (paper-model adds, reading R2; Table A2)
 *   adds_exec = sum_{w<N} max(n_w - 1, 0)   (additions actually executed)       */
EXPORT int oracle_cussen_counts(const int64_t *a, int len, int N, int64_t *out3, int *levels_out) {
    colplan pl;
    if (cussen_compress(a, len, N, &pl)) return -1;
    int64_t adds_pm = 0, adds_ex = 0;
    for (int w = 1; w < N; w++) { adds_pm += pl.n[w]; adds_ex += pl.n[w] > 0 ? pl.n[w] - 1 : 0; }
    out3[0] = pl.n[N]; out3[1] = adds_pm; out3[2] = adds_ex;
    if (levels_out) for (int w = 1; w <= N; w++) levels_out[w - 1] = pl.n[w];
    colplan_free(&pl);
    return 0;
}

/* The compressed levels of one column (for tests): s_out[w-1][u] (row stride len),
 * ptr_out[w-1][e] (row stride len).                                           */
EXPORT int oracle_cussen_plan(const int64_t *a, int len, int N, int *n_out, int64_t *s_out, int *ptr_out) {
    colplan pl;
    if (cussen_compress(a, len, N, &pl)) return -1;
    for (int w = 1; w <= N; w++) {
        n_out[w - 1] = pl.n[w];
        for (int u = 0; u < pl.n[w]; u++) s_out[(size_t)(w - 1) * len + u] = pl.s[w][u];
        int prev = w == 1 ? len : pl.n[w - 1];
        for (int e = 0; e < prev; e++) ptr_out[(size_t)(w - 1) * len + e] = pl.ptr[w][e];
    }
    colplan_free(&pl);
    return 0;
}

/* Alg. 2 end to end on plaintext integers: b = C * a. */
EXPORT int oracle_cussen_vs_mul_plain(const int64_t *a, int len, int64_t C, int N, int64_t *b_out) {
    colplan pl;
    if (cussen_compress(a, len, N, &pl)) return -1;
    /* line 13: b^(N) = C * a^(N) */
    int64_t *b = (int64_t *)malloc(sizeof(int64_t) * (size_t)(pl.n[N] > 0 ? pl.n[N] : 1));
    for (int u = 0; u < pl.n[N]; u++) b[u] = C * level_value(&pl, N, u);
    for (int w = N; w >= 1; w--) {
        if (w != N) for (int i = 0; i + 1 < pl.n[w]; i++) b[i + 1] = b[i + 1] + b[i];   /* lines 16-19 */
        int prev = w == 1 ? len : pl.n[w - 1];                                      /* line 21 */
        int64_t *nb = (int64_t *)malloc(sizeof(int64_t) * (size_t)(prev > 0 ? prev : 1));
        for (int e = 0; e < prev; e++) nb[e] = pl.ptr[w][e] < 0 ? 0 : b[pl.ptr[w][e]];
        free(b); b = nb;
    }
    memcpy(b_out, b, sizeof(int64_t) * (size_t)len);
    free(b);
    colplan_free(&pl);
    return 0;
}

/* Encrypted vector-scalar reconstruction (Alg. 3 lines 5-6) of one
 * column plan with one point P: out[i] = a_i * P (infinity for a_i = 0).
 * `t` is the declared plaintext width used by the ladder (cost model).        */
static void cussen_reconstruct(const colplan *pl, int t, const jac *P, jac *out, counters *cnt) {
    int N = pl->N;
    jac *b = (jac *)malloc(sizeof(jac) * (size_t)(pl->n[N] > 0 ? pl->n[N] : 1));
    for (int u = 0; u < pl->n[N]; u++) b[u] = small_mul(level_value(pl, N, u), t, P, cnt);  /* line 5 */
    for (int w = N; w >= 1; w--) {
        if (w != N) for (int i = 0; i + 1 < pl->n[w]; i++) b[i + 1] = jac_add(&b[i + 1], &b[i], cnt);
        int prev = w == 1 ? pl->len0 : pl->n[w - 1];
        jac *nb = (jac *)malloc(sizeof(jac) * (size_t)(prev > 0 ? prev : 1));
        for (int e = 0; e < prev; e++) nb[e] = pl->ptr[w][e] < 0 ? jac_inf() : b[pl->ptr[w][e]];
        free(b); b = nb;
    }
    memcpy(out, b, sizeof(jac) * (size_t)pl->len0);
    free(b);
}

EXPORT int oracle_cussen_vs_mul_encrypted(const int64_t *a, int len, int t, int N, const uint8_t *ct128,
                                          uint8_t *out128, uint64_t *cnt_out) {
    oracle_init_once();
    colplan pl;
    if (cussen_compress(a, len, N, &pl)) return -1;
    jac C1, C2;
    if (point_from_bytes(ct128, &C1) || point_from_bytes(ct128 + 64, &C2)) { colplan_free(&pl); return -4; }
    jac *o1 = (jac *)malloc(sizeof(jac) * (size_t)len), *o2 = (jac *)malloc(sizeof(jac) * (size_t)len);
    counters c = {0, 0, 0, 0};
    cussen_reconstruct(&pl, t, &C1, o1, &c);
    cussen_reconstruct(&pl, t, &C2, o2, &c);
    for (int i = 0; i < len; i++) { point_to_bytes(&o1[i], out128 + 128 * i); point_to_bytes(&o2[i], out128 + 128 * i + 64); }
    if (cnt_out) { cnt_out[0] = c.adds; cnt_out[1] = c.dbls; cnt_out[2] = c.ecsm; cnt_out[3] = c.ecsm_bits; }
    free(o1); free(o2); colplan_free(&pl);
    return 0;
}

/* ================================================ PC-MM engines ============ */
typedef struct {
    int m, n, l, t, N, path;
    const int32_t *A;
    const jac *B;              /* [n*l*2] parsed ciphertext points, (k, j, c) */
    const colplan *plans;      /* [n] (Cussen) */
    uint8_t *out;              /* [m*l*128] */
    int j0, j1;
    counters cnt;
} job;

/* Schoolbook PC-MM: Enc(c_ij) = sum_k a_ik * Enc(b_kj);
 * each term is 2 ECSMs (Alg. 1 ladder of width t), accumulated from infinity. */
static void *school_worker(void *arg) {
    job *J = (job *)arg;
    for (int j = J->j0; j < J->j1; j++)
        for (int i = 0; i < J->m; i++) {
            jac acc[2] = {jac_inf(), jac_inf()};
            for (int k = 0; k < J->n; k++) {
                int64_t a = J->A[(size_t)i * J->n + k];
                for (int c = 0; c < 2; c++) {
                    jac term = small_mul(a, J->t, &J->B[((size_t)k * J->l + j) * 2 + c], &J->cnt);
                    acc[c] = jac_add(&acc[c], &term, &J->cnt);
                }
            }
            uint8_t *o = J->out + ((size_t)i * J->l + j) * 128;
            point_to_bytes(&acc[0], o);
            point_to_bytes(&acc[1], o + 64);
        }
    return NULL;
}

/* Alg. 3: C <- inf; for k: compress A[:,k] (line 3, amortised over
 * j, computed once before the workers start); for j: 2 m' ECSMs (line 5) and
 * reconstruction by point additions (line 6); for i: C_ij += a_ik B_kj (line 8).
 * Workers own disjoint sets of output columns j; per output the k order is
 * ascending exactly as in Alg. 3.                                             */
static void *cussen_worker(void *arg) {
    job *J = (job *)arg;
    jac *acc = (jac *)malloc(sizeof(jac) * (size_t)J->m * 2);
    jac *col = (jac *)malloc(sizeof(jac) * (size_t)J->m);
    for (int j = J->j0; j < J->j1; j++) {
        for (int i = 0; i < 2 * J->m; i++) acc[i] = jac_inf();
        for (int k = 0; k < J->n; k++)
            for (int c = 0; c < 2; c++) {
                cussen_reconstruct(&J->plans[k], J->t, &J->B[((size_t)k * J->l + j) * 2 + c], col, &J->cnt);
                for (int i = 0; i < J->m; i++) acc[2 * i + c] = jac_add(&acc[2 * i + c], &col[i], &J->cnt);
            }
        for (int i = 0; i < J->m; i++) {
            uint8_t *o = J->out + ((size_t)i * J->l + j) * 128;
            point_to_bytes(&acc[2 * i], o);
            point_to_bytes(&acc[2 * i + 1], o + 64);
        }
    }
    free(acc); free(col);
    return NULL;
}

/* path: 0 = schoolbook, 1 = Cussen (Alg. 3).  t: declared plaintext width (ladder
 * width, cost model).  N: Cussen iterations (the paper uses 4).  ct: n*l
 * canonical ciphertexts (k, j) row-major.  out: m*l canonical ciphertexts.
 * cnt_out[4] = executed adds, doublings, ECSMs, ECSM bits.                    */
EXPORT int oracle_pcmm(int path, int m, int n, int l, int t, int N, const int32_t *A, const uint8_t *ct,
                       uint8_t *out, int nthreads, uint64_t *cnt_out) {
    oracle_init_once();
    if (m <= 0 || n <= 0 || l <= 0) return -2;
    jac *B = (jac *)malloc(sizeof(jac) * (size_t)n * l * 2);
    for (size_t e = 0; e < (size_t)n * l * 2; e++)
        if (point_from_bytes(ct + 64 * e, &B[e])) { free(B); return -4; }
    colplan *plans = NULL;
    if (path == 1) {
        plans = (colplan *)calloc((size_t)n, sizeof(colplan));
        int64_t *colv = (int64_t *)malloc(sizeof(int64_t) * (size_t)m);
        for (int k = 0; k < n; k++) {
            for (int i = 0; i < m; i++) colv[i] = A[(size_t)i * n + k];
            cussen_compress(colv, m, N, &plans[k]);
        }
        free(colv);
    }
    if (nthreads < 1) nthreads = 1;
    if (nthreads > l) nthreads = l;
    job *jobs = (job *)calloc((size_t)nthreads, sizeof(job));
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int w = 0; w < nthreads; w++) {
        job *J = &jobs[w];
        J->m = m; J->n = n; J->l = l; J->t = t; J->N = N; J->path = path;
        J->A = A; J->B = B; J->plans = plans; J->out = out;
        J->j0 = (int)((int64_t)l * w / nthreads); J->j1 = (int)((int64_t)l * (w + 1) / nthreads);
        pthread_create(&th[w], NULL, path == 1 ? cussen_worker : school_worker, J);
    }
    counters tot = {0, 0, 0, 0};
    for (int w = 0; w < nthreads; w++) {
        pthread_join(th[w], NULL);
        tot.adds += jobs[w].cnt.adds; tot.dbls += jobs[w].cnt.dbls;
        tot.ecsm += jobs[w].cnt.ecsm; tot.ecsm_bits += jobs[w].cnt.ecsm_bits;
    }
    if (cnt_out) { cnt_out[0] = tot.adds; cnt_out[1] = tot.dbls; cnt_out[2] = tot.ecsm; cnt_out[3] = tot.ecsm_bits; }
    if (plans) { for (int k = 0; k < n; k++) colplan_free(&plans[k]); free(plans); }
    free(jobs); free(th); free(B);
    return 0;
}

/* One output ciphertext C_ij of the schoolbook definition (for sampled parity
 * at full sizes): row a[0..n-1] against the column ct[k] (n canonical cts).    */
EXPORT int oracle_inner_product(int n, const int32_t *a, const uint8_t *ct_col, uint8_t *out128) {
    oracle_init_once();
    jac acc[2] = {jac_inf(), jac_inf()};
    for (int k = 0; k < n; k++)
        for (int c = 0; c < 2; c++) {
            jac P;
            if (point_from_bytes(ct_col + 128 * (size_t)k + 64 * c, &P)) return -4;
            big s = scalar_from_i64(a[k]);
            jac term = scalar_mul(&s, &P);
            acc[c] = jac_add(&acc[c], &term, NULL);
        }
    point_to_bytes(&acc[0], out128);
    point_to_bytes(&acc[1], out128 + 64);
    return 0;
}
