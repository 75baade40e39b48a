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
    const int nch = active_chunks(a, (int)gridDim.y, 32 * V);
    if ((int)blockIdx.y >= nch) return;
    const int ch = a.reverse ? nch - 1 - (int)blockIdx.y : (int)blockIdx.y;
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

// ---- high-degree path: chains of outputs over shared-memory r / 1-r -----------
// Same structure as k_check_chains (kernels_check.cu): one block of up to 1024 threads per
// (variable, tile of TW codewords), degrees past 16; r and 1 - r staged in shared memory
// (or the workspace scratch past the shared-memory budget); outputs in
// groups of R = 8 with CPT = R*TW/32 chains per thread, each chain the pair
// (q0, q1) of serial.py:77-88; W warps take groups w, 2W-1-w, 2W+w, ... ascending so a
// running prefix pair ((1-p)*prod(1-r_i), p*prod(r_i)) is carried across groups.
// Warp 0 part 0 carries its prefix to the end: the estimate's (Q0, Q1).
constexpr int kChainR = 8;
constexpr int kChainThreads = 1024;

__device__ __forceinline__ int var_chains_group(int w, int t, int nw) {  // t-th group of warp w (of nw)
    const int band = t >> 1;
    return band * 2 * nw + ((t & 1) ? 2 * nw - 1 - w : w);
}

template <int TW, bool WRITE_Q, bool GS>  // GS: staging in global scratch (degrees past the smem budget)
__global__ void __launch_bounds__(kChainThreads) k_var_chains(NodeLaunch a, int max_deg) {
    constexpr int CPT = kChainR * TW / 32;
    static_assert(CPT >= 1, "TW must be >= 4");
    extern __shared__ double smem_rs[];
    double *sm = GS ? a.scratch + (size_t)blockIdx.x * max_deg * TW * 2 : smem_rs;
    int ni, tile;
    lpt_block(blockIdx.x, a.node_count, a.Bp / TW, ni, tile);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int c = lane % TW, h = lane / TW;
    const int cw = tile * TW + c;
    const int w = (tile * TW) >> 5;
    const uint32_t tmask = (TW >= 32) ? 0xffffffffu : (((1u << TW) - 1u) << ((tile * TW) & 31));
    if (a.done != nullptr && (a.done[w] & tmask) == tmask) return;
    const int node = __ldg(a.order + a.node_begin + ni);
    const int e0 = __ldg(a.off + node);
    const int d = __ldg(a.off + node + 1) - e0;
    const int G = (d + kChainR - 1) / kChainR;
    double *rs = sm;                    // [d][TW] r_i
    double *os = sm + (size_t)d * TW;   // [d][TW] 1 - r_i
    const double pj = __ldg(a.P + cofs(a.p_rows, node, cw));
    if constexpr (!GS) {
        // the tile's d row segments all in flight at once (cp.async), then 1 - r
        constexpr int PPR = TW / 2;  // 16-byte pieces per row segment
        for (int e = threadIdx.x; e < d * PPR; e += blockDim.x) {
            const int i = e / PPR, pc = e - i * PPR;
            cp_async16(rs + i * TW + 2 * pc,
                       a.msg + cofs(a.msg_rows, a.slot ? __ldg(a.slot + e0 + i) : e0 + i, tile * TW + 2 * pc));
        }
        cp_commit();
        cp_wait<0>();
        __syncthreads();
        for (int e = threadIdx.x; e < d * TW; e += blockDim.x) os[e] = __dsub_rn(1.0, rs[e]);
    } else {
        for (int e = threadIdx.x; e < d * TW; e += blockDim.x) {
            const int i = e / TW, cc = e - i * TW;
            const double r = ld_msg(a.msg + cofs(a.msg_rows, a.slot ? __ldg(a.slot + e0 + i) : e0 + i, tile * TW + cc));
            rs[e] = r;
            os[e] = __dsub_rn(1.0, r);
        }
    }
    __syncthreads();
    const double *rc = rs + c, *oc = os + c;
    double pre0 = __dsub_rn(1.0, pj), pre1 = pj;  // running prefix pair over positions < at
    int at = 0;
    auto step = [&](int i) {
        if (i < d) {
            pre0 = __dmul_rn(pre0, oc[i * TW]);
            pre1 = __dmul_rn(pre1, rc[i * TW]);
        }
    };
    if constexpr (WRITE_Q) {
        const int j0 = h * CPT;
        for (int t = 0;; t++) {
            const int g = var_chains_group(warp, t, nw);
            if (g >= G) break;
            const int kb = g * kChainR + j0;
            const int next = var_chains_group(warp, t + 1, nw) * kChainR + j0;
            for (; at < kb; at++) step(at);
            double a0[CPT], a1[CPT];
            double p0 = pre0, p1 = pre1;
#pragma unroll
            for (int j = 0; j < CPT; j++) {
                a0[j] = p0;
                a1[j] = p1;
                if (j + 1 < CPT && kb + j < d) {
                    p0 = __dmul_rn(p0, oc[(kb + j) * TW]);
                    p1 = __dmul_rn(p1, rc[(kb + j) * TW]);
                }
            }
#pragma unroll
            for (int j = 1; j < CPT; j++) {
                if (kb + j < d) {
                    const double x0 = oc[(kb + j) * TW], x1 = rc[(kb + j) * TW];
#pragma unroll
                    for (int jj = 0; jj < j; jj++) {
                        a0[jj] = __dmul_rn(a0[jj], x0);
                        a1[jj] = __dmul_rn(a1[jj], x1);
                    }
                }
            }
            for (; at < kb + CPT && at < next; at++) step(at);
            int i = kb + CPT;
            const int stop_carry = min(next, d);
            for (; i < stop_carry; i++) {
                const double x0 = oc[i * TW], x1 = rc[i * TW];
#pragma unroll
                for (int j = 0; j < CPT; j++) {
                    a0[j] = __dmul_rn(a0[j], x0);
                    a1[j] = __dmul_rn(a1[j], x1);
                }
                pre0 = __dmul_rn(pre0, x0);
                pre1 = __dmul_rn(pre1, x1);
            }
            if (i > at) at = i;
#pragma unroll 4
            for (; i < d; i++) {
                const double x0 = oc[i * TW], x1 = rc[i * TW];
#pragma unroll
                for (int j = 0; j < CPT; j++) {
                    a0[j] = __dmul_rn(a0[j], x0);
                    a1[j] = __dmul_rn(a1[j], x1);
                }
            }
#pragma unroll
            for (int j = 0; j < CPT; j++) {
                const int k = kb + j;
                if (k < d) {
                    const double den = __dadd_rn(a0[j], a1[j]);
                    bool ok;
                    double q = ddiv_fast(a1[j], den, ok);
                    if (!ok) q = (den == 0.0) ? 0.5 : __ddiv_rn(a1[j], den);
                    st_msg(a.msg + cofs(a.msg_rows, a.slot ? __ldg(a.slot + e0 + k) : e0 + k, cw), q);
                }
            }
        }
    }
    // estimate (serial.py:125-132): warp 0, part 0 holds or completes the full products
    if (warp == 0) {
        if (h == 0)
            for (; at < d; at++) step(at);
        const bool one = !(pre0 > pre1);
        const uint32_t keep = a.done ? a.done[w] : 0u;
        const uint32_t sub = __ballot_sync(0xffffffffu, h == 0 && one);  // bit c of lanes 0..TW-1
        if (lane == 0) {
            uint32_t *dst = a.chat + (size_t)node * a.NW + w;
            if (TW >= 32) {
                *dst = keep ? ((sub & ~keep) | (*dst & keep)) : sub;
            } else {  // tiles smaller than a word share it -> atomics
                const int sh = (tile * TW) & 31;
                const uint32_t upd = tmask & ~keep;
                atomicAnd(dst, ~upd);
                atomicOr(dst, (sub << sh) & upd);
            }
        }
    }
}

template <int TW, bool GS>
int launch_var_chains(const NodeLaunch &a, int max_deg, size_t smem, bool write_q, cudaStream_t s) {
    auto kern = write_q ? k_var_chains<TW, true, GS> : k_var_chains<TW, false, GS>;
    // the cap (not this launch's size): launches of one instantiation with different tiles may be issued
    // from several threads or side streams
    if (smem) LDPC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kChainSmemBudget));
    const int64_t blocks = (int64_t)a.node_count * (a.Bp / TW);
    // warps: two groups each (balanced band pairs), up to 32
    const int nw = std::max(1, std::min(32, ((max_deg + kChainR - 1) / kChainR + 1) / 2));
    kern<<<(unsigned)blocks, 32 * nw, smem, s>>>(a, max_deg);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
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
    // the widest tile whose r and 1-r fit in shared memory; past that, 16-codeword tiles
    // staged in the workspace scratch.  LDPC_WIDE_TW=4|8|16 forces a tile.
    static const int forced = [] {
        const char *e = getenv("LDPC_WIDE_TW");
        return e ? atoi(e) : 0;
    }();
    auto smem = [&](int tw) { return (size_t)2 * max_deg * tw * sizeof(double); };
    if ((forced == 0 || forced == 16) && smem(16) <= kChainSmemBudget) return launch_var_chains<16, false>(a, max_deg, smem(16), write_q, s);
    if ((forced == 0 || forced == 8) && smem(8) <= kChainSmemBudget) return launch_var_chains<8, false>(a, max_deg, smem(8), write_q, s);
    if ((forced == 0 || forced == 4) && smem(4) <= kChainSmemBudget) return launch_var_chains<4, false>(a, max_deg, smem(4), write_q, s);
    LDPC_ARG_CHECK(a.scratch != nullptr, "variable degree %d needs the workspace scratch", max_deg);
    return launch_var_chains<kChainTW, true>(a, max_deg, 0, write_q, s);
}

}  // namespace ldpc
