// Host build of the CUDA path's portable field / curve code (csrc/fp.cuh,
// csrc/ec.cuh) for CPU unit tests of its ALGORITHMS (reduction, inversion
// chain, RCB formulas, encodings).  Test infrastructure only: the product
// library never runs this on the host; the GPU tests check the device build.
#include <stdint.h>
#include <string.h>
#include "../../paper_2504_14497_b200/csrc/ec.cuh"

using namespace pcmm;

extern "C" {

// op: 0 add, 1 sub, 2 mul (plain a*b mod p via Montgomery), 3 inv (divsteps), 4 neg,
//     5 inv (Fermat chain)
int hfp_op(int op, const uint8_t *a_be, const uint8_t *b_be, uint8_t *out_be) {
    fe a, b, r;
    fe_from_be_bytes(a, a_be);
    fe_from_be_bytes(b, b_be);
    fe_to_mont(a, a);
    fe_to_mont(b, b);
    switch (op) {
        case 0: fe_add(r, a, b); break;
        case 1: fe_sub(r, a, b); break;
        case 2: fe_mul(r, a, b); break;
        case 3: fe_inv(r, a); break;
        case 4: fe_neg(r, a); break;
        case 5: fe_inv_fermat(r, a); break;
        case 6: fe_inv_var(r, a); break;
        default: return -1;
    }
    fe_from_mont(r, r);
    fe_to_be_bytes(out_be, r);
    return 0;
}

// plain x^-1 mod p by the divsteps inversions (ct: constant-time half-delta, else variable-time)
int hfp_inv_plain(int ct, const uint8_t *a_be, uint8_t *out_be) {
    fe a, r;
    fe_from_be_bytes(a, a_be);
    if (ct) fe_inv_plain_divsteps(r, a);
    else fe_inv_plain_divsteps_var(r, a);
    fe_to_be_bytes(out_be, r);
    return 0;
}

// raw Montgomery product of two (possibly unreduced < p) limb vectors
int hfp_mont_mul_raw(const uint8_t *a_be, const uint8_t *b_be, uint8_t *out_be) {
    fe a, b, r;
    fe_from_be_bytes(a, a_be);
    fe_from_be_bytes(b, b_be);
    fe_mul(r, a, b);
    fe_to_be_bytes(out_be, r);
    return 0;
}

int hpt_add(const uint8_t *p64, const uint8_t *q64, uint8_t *out64) {
    pt P, Q, R;
    if (pt_from_canonical(P, p64) || pt_from_canonical(Q, q64)) return -4;
    pt_add(R, P, Q);
    pt_to_canonical(out64, R);
    return 0;
}

int hpt_dbl(const uint8_t *p64, uint8_t *out64) {
    pt P, R;
    if (pt_from_canonical(P, p64)) return -4;
    pt_dbl(R, P);
    pt_to_canonical(out64, R);
    return 0;
}

int hpt_mul_small(int v, const uint8_t *p64, uint8_t *out64) {
    pt P, R;
    if (pt_from_canonical(P, p64)) return -4;
    pt_mul_small(R, v, P);
    pt_to_canonical(out64, R);
    return 0;
}

int hpt_mul_scalar(const uint8_t *k_be, const uint8_t *p64, uint8_t *out64) {
    pt P, R;
    if (pt_from_canonical(P, p64)) return -4;
    uint32_t k[8];
    for (int i = 0; i < 8; i++) {
        const uint8_t *w = k_be + 28 - 4 * i;
        k[i] = ((uint32_t)w[0] << 24) | ((uint32_t)w[1] << 16) | ((uint32_t)w[2] << 8) | w[3];
    }
    pt_mul_scalar(R, k, P);
    pt_to_canonical(out64, R);
    return 0;
}

int hpt_on_curve(const uint8_t *p64) {
    pt P;
    return pt_from_canonical(P, p64) == 0 ? 1 : 0;
}

}
