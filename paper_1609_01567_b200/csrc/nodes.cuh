// nodes.cuh -- one thread = one node of one codeword: the check and variable updates of
// the on-chip (onchip.cu) and grid (grid.cu) schedules, exact fp64.
//
// Same arithmetic as the streaming register kernels (serial.py:63-133, one rounding per
// operation, left-to-right products, the division fast path of common.cuh); only the
// storage differs, so it is abstracted by an accessor ACC with
//     double *slot(int s)        the message slot s (check order)
//     double prior_of(int var)   p of variable `var`
// and the code tables (canonical CSR of both sides).  Degrees <= 16 gather their d
// inputs into registers first (independent loads overlap their latency); higher
// degrees take the generic serial loop.
#pragma once
#include "common.cuh"

namespace ldpc {

struct NodeTables {
    const int32_t *chk_off, *chk_var;  // check CSR over slots; variable of each slot
    const int32_t *var_off, *var_pos;  // variable CSR over canonical edges; slot of each edge
};

// check-node update of check `c` (serial.py:92-112); prior-fed pre-pass when FROM_PRIOR
template <bool FROM_PRIOR, class ACC>
__device__ __forceinline__ void check_update(const ACC &acc, const NodeTables &t, int c) {
    const int s0 = __ldg(t.chk_off + c), d = __ldg(t.chk_off + c + 1) - s0;
    auto bval = [&](int i) {
        const double q = FROM_PRIOR ? acc.prior_of(__ldg(t.chk_var + s0 + i)) : *acc.slot(s0 + i);
        return __dsub_rn(1.0, __dmul_rn(2.0, q));
    };
    double pre = 1.0;
    for (int k = 0; k < d; k++) {
        double acc_k = pre;
        for (int i = k + 1; i < d; i++) acc_k = __dmul_rn(acc_k, bval(i));
        pre = __dmul_rn(pre, bval(k));  // slot k's q is read before r_k overwrites it
        *acc.slot(s0 + k) = __dsub_rn(1.0, __dadd_rn(0.5, __dmul_rn(0.5, acc_k)));
    }
}

// variable-node update + estimate of variable v (serial.py:63-89, 115-133); returns the hard decision
template <class ACC>
__device__ __forceinline__ uint8_t var_update(const ACC &acc, const NodeTables &t, int v, bool write_q, double pj) {
    const int e0 = __ldg(t.var_off + v), d = __ldg(t.var_off + v + 1) - e0;
    double pre0 = __dsub_rn(1.0, pj), pre1 = pj;
    for (int k = 0; k < d; k++) {
        double *sk = acc.slot(__ldg(t.var_pos + e0 + k));
        const double rk = *sk;
        if (write_q) {
            double q0 = pre0, q1 = pre1;
            for (int i = k + 1; i < d; i++) {
                const double ri = *acc.slot(__ldg(t.var_pos + e0 + i));
                q0 = __dmul_rn(q0, __dsub_rn(1.0, ri));
                q1 = __dmul_rn(q1, ri);
            }
            pre0 = __dmul_rn(pre0, __dsub_rn(1.0, rk));
            pre1 = __dmul_rn(pre1, rk);
            const double den = __dadd_rn(q0, q1);
            bool ok;
            double q = ddiv_fast(q1, den, ok);
            if (!ok) q = (den == 0.0) ? 0.5 : __ddiv_rn(q1, den);
            *sk = q;  // r_k was read into the prefix first
        } else {
            pre0 = __dmul_rn(pre0, __dsub_rn(1.0, rk));
            pre1 = __dmul_rn(pre1, rk);
        }
    }
    return (pre0 > pre1) ? 0 : 1;
}

// Degree-specialised forms: inputs gathered into registers, then the register kernels'
// arithmetic; outputs go back through the same pointers (each slot is read before any
// output of the node is stored).
template <int D, bool FROM_PRIOR, class ACC>
__device__ __forceinline__ void check_update_d(const ACC &acc, const NodeTables &t, int s0) {
    double *ptr[D];
    double b[D];
#pragma unroll
    for (int i = 0; i < D; i++) {
        ptr[i] = acc.slot(s0 + i);
        const double q = FROM_PRIOR ? acc.prior_of(__ldg(t.chk_var + s0 + i)) : *ptr[i];
        b[i] = __dsub_rn(1.0, __dmul_rn(2.0, q));
    }
    double pre = 1.0;
#pragma unroll
    for (int k = 0; k < D; k++) {
        double acc_k = pre;
#pragma unroll
        for (int i = k + 1; i < D; i++) acc_k = __dmul_rn(acc_k, b[i]);
        *ptr[k] = __dsub_rn(1.0, __dadd_rn(0.5, __dmul_rn(0.5, acc_k)));
        if (k + 1 < D) pre = __dmul_rn(pre, b[k]);
    }
}

template <int D, class ACC>
__device__ __forceinline__ uint8_t var_update_d(const ACC &acc, const NodeTables &t, int e0, bool write_q, double pj) {
    double *ptr[D];
    double r[D], om[D];
#pragma unroll
    for (int i = 0; i < D; i++) {
        ptr[i] = acc.slot(__ldg(t.var_pos + e0 + i));
        r[i] = *ptr[i];
        om[i] = __dsub_rn(1.0, r[i]);
    }
    double p0 = __dsub_rn(1.0, pj), p1 = pj;
#pragma unroll
    for (int k = 0; k < D; k++) {
        if (write_q) {
            double q0 = p0, q1 = p1;
#pragma unroll
            for (int i = k + 1; i < D; i++) {
                q0 = __dmul_rn(q0, om[i]);
                q1 = __dmul_rn(q1, r[i]);
            }
            const double den = __dadd_rn(q0, q1);
            bool ok;
            double q = ddiv_fast(q1, den, ok);
            if (!ok) q = (den == 0.0) ? 0.5 : __ddiv_rn(q1, den);
            *ptr[k] = q;
        }
        p0 = __dmul_rn(p0, om[k]);
        p1 = __dmul_rn(p1, r[k]);
    }
    return (p0 > p1) ? 0 : 1;
}

template <bool FROM_PRIOR, class ACC>
__device__ __forceinline__ void check_node(const ACC &acc, const NodeTables &t, int c) {
    const int s0 = __ldg(t.chk_off + c), d = __ldg(t.chk_off + c + 1) - s0;
    switch (d) {
#define CASE(D) \
    case D: check_update_d<D, FROM_PRIOR>(acc, t, s0); return;
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
        CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
        default: check_update<FROM_PRIOR>(acc, t, c);
    }
}

template <class ACC>
__device__ __forceinline__ uint8_t var_node(const ACC &acc, const NodeTables &t, int v, bool write_q, double pj) {
    const int e0 = __ldg(t.var_off + v), d = __ldg(t.var_off + v + 1) - e0;
    switch (d) {
#define CASE(D) \
    case D: return var_update_d<D>(acc, t, e0, write_q, pj);
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
        CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
        default: return var_update(acc, t, v, write_q, pj);
    }
}

}  // namespace ldpc
