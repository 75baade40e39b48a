// kernels_var.cu -- G3: variable-node update fused with the estimate, exact fp64.
//
// Reference arithmetic, variable j of degree d with canonical edges g0..g0+d-1
// (rows descending, tables.py:66-77) and prior p:
//   V-phase (serial.py:63-89): for edge k,
//       q0 = (1-p) * (1-r_0) * ... (skip k) ... * (1-r_{d-1})      left to right
//       q1 =   p   *    r_0  * ... (skip k) ... *    r_{d-1}
//       q_k = 0.5 if q0 + q1 == 0.0 else q1 / (q0 + q1)
//   estimate (serial.py:115-133): Q0, Q1 over ALL edges; c_hat = 0 iff Q0 > Q1.
// The prefix products (1-p)(1-r_0)...(1-r_{k-1}) are shared by all k, and the
// full product is exactly the estimate's Q0/Q1, so the estimate of round t-1
// comes for free with the V-phase of round t (one pass over r instead of two).
//
// Work mapping as in kernels_check.cu: warp = variable x 32*V codewords; the
// d incoming messages are gathered from their check-ordered slots
// (var_pos), each gather one contiguous 256*V-byte run.  Hard decisions are
// bit-sliced with __ballot_sync: one 32-bit word per (variable, 32 codewords).
// In early-stop mode, bits of codewords that already stopped are kept frozen
// (serial.py:169-177 returns the estimate of the round that succeeded).
#include "common.cuh"

namespace ldpc {
namespace {

template <int V>
__device__ __forceinline__ void load_v(const double *p, double (&o)[V]) {
    if constexpr (V == 2) {
        double2 t = ld_msg(reinterpret_cast<const double2 *>(p));
        o[0] = t.x;
        o[1] = t.y;
    } else {
        o[0] = ld_msg(p);
    }
}

template <int V>
__device__ __forceinline__ void load_prior(const double *p, double (&o)[V]) {
    if constexpr (V == 2) {
        double2 t = __ldg(reinterpret_cast<const double2 *>(p));
        o[0] = t.x;
        o[1] = t.y;
    } else {
        o[0] = __ldg(p);
    }
}

template <int V>
__device__ __forceinline__ void store_v(double *p, const double (&o)[V]) {
    if constexpr (V == 2) {
        st_msg(reinterpret_cast<double2 *>(p), make_double2(o[0], o[1]));
    } else {
        st_msg(p, o[0]);
    }
}

// Merge new estimate bits into chat[node][w], keeping bits of stopped codewords.
__device__ __forceinline__ void put_bits(uint32_t *dst, uint32_t bits, const uint32_t *done, int w) {
    if (done != nullptr) {
        uint32_t dm = done[w];
        if (dm) bits = (bits & ~dm) | (*dst & dm);
    }
    *dst = bits;
}

template <int D, int V, bool WRITE_Q>
__global__ void __launch_bounds__(kThreads, (D <= 2 && V == 2) ? 5 : 1) k_var_reg(NodeLaunch a) {
    const int lane = threadIdx.x & 31;
    // grid (node blocks, codeword chunks), dispatched x-fastest: chunk-major sweep
    const int ch = blockIdx.y;
    const int ni = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (ni >= a.node_count) return;
    if (a.done != nullptr) {
        bool all;
        if constexpr (V == 2) {
            uint2 d = *reinterpret_cast<const uint2 *>(a.done + 2 * ch);
            all = (d.x & d.y) == 0xffffffffu;
        } else {
            all = a.done[ch] == 0xffffffffu;
        }
        if (all) return;
    }
    const int cw0 = ch * 32 * V;
    double *mb = chunk_base(a.msg, a.msg_rows, cw0) + lane * V;
    // one round of independent index loads (bucket-ordered flat tables)
    const int node = __ldg(a.order + a.node_begin + ni);
    const int32_t base = a.edge_begin + ni * D;
    int pos[D];
#pragma unroll
    for (int i = 0; i < D; i++) pos[i] = __ldg(a.slot_ord + base + i);

    double pj[V];
    load_prior<V>(chunk_base(a.P, a.p_rows, cw0) + lane * V + row_off(node), pj);
    double r[D][V];
#pragma unroll
    for (int i = 0; i < D; i++) load_v<V>(mb + row_off(pos[i]), r[i]);
    double om[D][V];  // 1 - r_i
#pragma unroll
    for (int i = 0; i < D; i++)
#pragma unroll
        for (int v = 0; v < V; v++) om[i][v] = __dsub_rn(1.0, r[i][v]);

    double pre0[V], pre1[V];
#pragma unroll
    for (int v = 0; v < V; v++) {
        pre0[v] = __dsub_rn(1.0, pj[v]);
        pre1[v] = pj[v];
    }
    uint32_t slow = 0;  // outputs whose division needs the library slow path (or den == 0)
#pragma unroll
    for (int k = 0; k < D; k++) {
        if constexpr (WRITE_Q) {
            double out[V];
            bool all_ok = true;
#pragma unroll
            for (int v = 0; v < V; v++) {
                double q0 = pre0[v], q1 = pre1[v];
#pragma unroll
                for (int i = k + 1; i < D; i++) {
                    q0 = __dmul_rn(q0, om[i][v]);
                    q1 = __dmul_rn(q1, r[i][v]);
                }
                bool ok;
                out[v] = ddiv_fast(q1, __dadd_rn(q0, q1), ok);  // den == 0 -> !ok
                all_ok = all_ok && ok;
            }
            if (all_ok) store_v<V>(mb + row_off(pos[k]), out);
            else slow |= 1u << k;
        }
#pragma unroll
        for (int v = 0; v < V; v++) {
            pre0[v] = __dmul_rn(pre0[v], om[k][v]);
            pre1[v] = __dmul_rn(pre1[v], r[k][v]);
        }
    }
    if constexpr (WRITE_Q) {
        if (slow) {  // rare: tiny/zero denominators; recompute in reference order, divide via the library
            for (int k = 0; k < D; k++) {
                if (!((slow >> k) & 1u)) continue;
                double out[V];
#pragma unroll
                for (int v = 0; v < V; v++) {
                    double q0 = __dsub_rn(1.0, pj[v]), q1 = pj[v];
                    for (int i = 0; i < D; i++) {
                        if (i == k) continue;
                        q0 = __dmul_rn(q0, om[i][v]);
                        q1 = __dmul_rn(q1, r[i][v]);
                    }
                    const double den = __dadd_rn(q0, q1);
                    out[v] = (den == 0.0) ? 0.5 : __ddiv_rn(q1, den);
                }
                store_v<V>(mb + row_off(pos[k]), out);
            }
        }
    }
    // estimate: c_hat = 0 iff Q0 > Q1 (ties -> 1), serial.py:132
    uint32_t *row = a.chat + (size_t)node * a.NW;
    if constexpr (V == 2) {
        const uint32_t even = __ballot_sync(0xffffffffu, !(pre0[0] > pre1[0]));
        const uint32_t odd = __ballot_sync(0xffffffffu, !(pre0[1] > pre1[1]));
        if (lane == 0) {
            const uint32_t lo = part1by1(even) | (part1by1(odd) << 1);
            const uint32_t hi = part1by1(even >> 16) | (part1by1(odd >> 16) << 1);
            put_bits(row + 2 * ch, lo, a.done, 2 * ch);
            put_bits(row + 2 * ch + 1, hi, a.done, 2 * ch + 1);
        }
    } else {
        const uint32_t bits = __ballot_sync(0xffffffffu, !(pre0[0] > pre1[0]));
        if (lane == 0) put_bits(row + ch, bits, a.done, ch);
    }
}

// ---- wide path: one block per (variable, tile of TW codewords) -------------
template <bool WRITE_Q>
__global__ void __launch_bounds__(kThreads) k_var_wide(NodeLaunch a, int TW, int max_deg) {
    extern __shared__ double sm[];
    double *r = sm;                                  // [max_deg][TW]
    double *pre0 = r + (size_t)max_deg * TW;         // [max_deg+1][TW]
    double *pre1 = pre0 + (size_t)(max_deg + 1) * TW; // [max_deg+1][TW]
    int *spos = reinterpret_cast<int *>(pre1 + (size_t)(max_deg + 1) * TW);  // [max_deg]
    const int tile = blockIdx.x / a.node_count;  // tile-major: all nodes of tile 0 first
    const int ni = blockIdx.x - tile * a.node_count;
    const int c = threadIdx.x % TW;
    const int worker = threadIdx.x / TW;
    const int nwk = blockDim.x / TW;
    const int cw = tile * TW + c;
    const int w = (tile * TW) >> 5;
    const uint32_t tmask = (TW >= 32) ? 0xffffffffu : (((1u << TW) - 1u) << ((tile * TW) & 31));
    if (a.done != nullptr && (a.done[w] & tmask) == tmask) return;
    const int node = __ldg(a.order + a.node_begin + ni);
    const int e0 = __ldg(a.off + node);
    const int d = __ldg(a.off + node + 1) - e0;
    for (int i = threadIdx.x; i < d; i += blockDim.x) spos[i] = a.slot ? __ldg(a.slot + e0 + i) : e0 + i;
    __syncthreads();
    for (int i = worker; i < d; i += nwk) r[i * TW + c] = ld_msg(a.msg + cofs(a.msg_rows, spos[i], cw));
    __syncthreads();
    if (worker == 0) {
        const double p = __ldg(a.P + cofs(a.p_rows, node, cw));
        double x0 = __dsub_rn(1.0, p), x1 = p;
        for (int i = 0; i < d; i++) {
            pre0[i * TW + c] = x0;
            pre1[i * TW + c] = x1;
            const double ri = r[i * TW + c];
            x0 = __dmul_rn(x0, __dsub_rn(1.0, ri));
            x1 = __dmul_rn(x1, ri);
        }
        pre0[d * TW + c] = x0;
        pre1[d * TW + c] = x1;
    }
    __syncthreads();
    if (WRITE_Q) {
        for (int j = worker; j < d; j += nwk) {
            const int k = (j & 1) ? (d - 1 - (j >> 1)) : (j >> 1);
            double q0 = pre0[k * TW + c], q1 = pre1[k * TW + c];
            for (int i = k + 1; i < d; i++) {
                const double ri = r[i * TW + c];
                q0 = __dmul_rn(q0, __dsub_rn(1.0, ri));
                q1 = __dmul_rn(q1, ri);
            }
            const double den = __dadd_rn(q0, q1);
            bool ok;
            double q = ddiv_fast(q1, den, ok);
            if (!ok) q = (den == 0.0) ? 0.5 : __ddiv_rn(q1, den);
            st_msg(a.msg + cofs(a.msg_rows, spos[k], cw), q);
        }
    }
    if (worker == 0) {
        // bits of this tile's codewords; tiles smaller than a word share it -> atomics
        const bool one = !(pre0[d * TW + c] > pre1[d * TW + c]);
        const uint32_t keep = a.done ? a.done[w] : 0u;
        uint32_t bits = 0;
        if (TW >= 32) {
            bits = __ballot_sync(0xffffffffu, one);
            if (c == 0) {
                uint32_t *dst = a.chat + (size_t)node * a.NW + w;
                *dst = keep ? ((bits & ~keep) | (*dst & keep)) : bits;
            }
        } else {
            // TW < 32: the worker-0 threads are lanes 0..TW-1 of warp 0
            const uint32_t sub = __ballot_sync((TW == 32) ? 0xffffffffu : ((1u << TW) - 1u), one);
            if (c == 0) {
                const int sh = (tile * TW) & 31;
                const uint32_t upd = tmask & ~keep;
                uint32_t *dst = a.chat + (size_t)node * a.NW + w;
                atomicAnd(dst, ~upd);
                atomicOr(dst, (sub << sh) & upd);
            }
        }
    }
}

int vpolicy_var(int deg) {
    static int forced = [] {
        const char *e = getenv("LDPC_VAR_V");
        return e ? atoi(e) : 0;
    }();
    if (forced == 1 || forced == 2) return forced;
    return deg <= 6 ? 2 : 1;
}

template <int D, int V, bool WQ>
int launch_one(const NodeLaunch &a, cudaStream_t s) {
    const dim3 grid((a.node_count + kWarpsPerBlock - 1) / kWarpsPerBlock, a.Bp / (32 * V));
    if (a.node_count == 0) return LDPC_OK;
    LDPC_ARG_CHECK(grid.y <= 65535u, "batch too large for one launch (%d codewords)", a.Bp);
    k_var_reg<D, V, WQ><<<grid, kThreads, 0, s>>>(a);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

template <int D>
int launch_deg(const NodeLaunch &a, bool wq, cudaStream_t s) {
    const int V = (a.Bp % 64) ? 1 : vpolicy_var(D);  // tile views of 32 codewords take V=1
    if (V == 2) return wq ? launch_one<D, 2, true>(a, s) : launch_one<D, 2, false>(a, s);
    return wq ? launch_one<D, 1, true>(a, s) : launch_one<D, 1, false>(a, s);
}

}  // namespace

int launch_var_bucket(const NodeLaunch &a, int deg, bool write_q, cudaStream_t s) {
    switch (deg) {
#define CASE(D) \
    case D: return launch_deg<D>(a, write_q, s);
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
        CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
        default:
            set_error("register-path variable degree %d out of range", deg);
            return LDPC_EINVAL;
    }
}

int launch_var_wide(const NodeLaunch &a, int max_deg, bool write_q, cudaStream_t s) {
    if (a.node_count == 0) return LDPC_OK;
    const size_t budget = 200 * 1024;
    auto bytes = [&](int TW) {
        return ((size_t)max_deg + 2 * ((size_t)max_deg + 1)) * TW * sizeof(double) + (size_t)max_deg * sizeof(int);
    };
    int TW = 32;
    while (TW > 1 && bytes(TW) > budget) TW >>= 1;
    if (bytes(TW) > budget) {
        set_error("variable degree %d exceeds the shared-memory staging limit", max_deg);
        return LDPC_EINVAL;
    }
    const size_t smem = bytes(TW);
    auto kern = write_q ? k_var_wide<true> : k_var_wide<false>;
    LDPC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t blocks = (int64_t)a.node_count * (a.Bp / TW);
    kern<<<(unsigned)blocks, kThreads, smem, s>>>(a, TW, max_deg);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

}  // namespace ldpc
