// kernels_check.cu -- G2: check-node update (the C-phase), exact fp64.
//
// Reference arithmetic (serial.py:92-112, engine.py:124-129), per check group
// of degree d with slots h0..h0+d-1 in ascending variable order:
//     prod_k = 1.0 * b_0 * ... * b_{k-1} * b_{k+1} * ... * b_{d-1}   (left to right)
//     b_i    = 1.0 - 2.0 * q_i
//     r_k    = 1.0 - (0.5 + 0.5 * prod_k)
// The shared prefix 1.0*b_0*...*b_{k-1} is the same sequence of roundings for
// every k, so it is carried once; the suffix is applied per k (d(d-1)/2
// multiplies per node).  Every operation is an explicit round-to-nearest
// intrinsic, so nothing is contracted into an FMA: results are bit-identical
// to the CPython reference.
//
// Work mapping: one warp = one check node x 32*V codewords (lane = V adjacent
// codewords, V = 2 -> 16-byte loads).  Messages are chunk-major
// (msg[c/64][slot][c%64], common.cuh): a warp's access per edge is one
// contiguous 256*V-byte run, a check's d slots are adjacent, and the grid
// sweeps all nodes of one codeword chunk before the next so the concurrently
// touched window stays small.  The update is in place (q read, r written to
// the same slots): each slot belongs to exactly one check.
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
__device__ __forceinline__ void load_v_cached(const double *p, double (&o)[V]) {
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

// true when every codeword of this warp's chunk has stopped (early-stop mode)
template <int V>
__device__ __forceinline__ bool chunk_done(const uint32_t *done, int chunk) {
    if (done == nullptr) return false;
    if constexpr (V == 2) {
        uint2 d = *reinterpret_cast<const uint2 *>(done + 2 * chunk);
        return (d.x & d.y) == 0xffffffffu;
    } else {
        return done[chunk] == 0xffffffffu;
    }
}

template <int D, int V, bool FROM_PRIOR>
__global__ void __launch_bounds__(kThreads) k_check_reg(NodeLaunch a) {
    const int lane = threadIdx.x & 31;
    // grid (node blocks, codeword chunks): blocks are dispatched x-fastest, so
    // the grid sweeps all nodes of chunk 0, then chunk 1, ... (chunk-major)
    const int nch = active_chunks(a, (int)gridDim.y, 32 * V);
    if ((int)blockIdx.y >= nch) return;
    const int ch = a.reverse ? nch - 1 - (int)blockIdx.y : (int)blockIdx.y;
    const int ni = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (ni >= a.node_count) return;
    if (chunk_done<V>(a.done, ch)) return;
    const int cw0 = ch * 32 * V;
    double *mb = chunk_base(a.msg, a.msg_rows, cw0) + lane * V;
    // one round of independent index loads (bucket-ordered flat tables)
    const int32_t base = a.edge_begin + ni * D;
    int slot[D];
#pragma unroll
    for (int i = 0; i < D; i++) slot[i] = __ldg(a.slot_ord + base + i);

    double b[D][V];
#pragma unroll
    for (int i = 0; i < D; i++) {
        double q[V];
        if constexpr (FROM_PRIOR) {
            // pre-pass (serial.py:58,166): q = p[v-bar] straight from the priors
            const double *pb = chunk_base(a.P, a.p_rows, cw0) + lane * V;
            load_v_cached<V>(pb + row_off(__ldg(a.var_ord + base + i)), q);
        } else {
            load_v<V>(mb + row_off(slot[i]), q);
        }
#pragma unroll
        for (int v = 0; v < V; v++) b[i][v] = __dsub_rn(1.0, __dmul_rn(2.0, q[v]));
    }
    double pre[V];
#pragma unroll
    for (int v = 0; v < V; v++) pre[v] = 1.0;
#pragma unroll
    for (int k = 0; k < D; k++) {
        double out[V];
#pragma unroll
        for (int v = 0; v < V; v++) {
            double acc = pre[v];
#pragma unroll
            for (int i = k + 1; i < D; i++) acc = __dmul_rn(acc, b[i][v]);
            out[v] = __dsub_rn(1.0, __dadd_rn(0.5, __dmul_rn(0.5, acc)));
        }
        store_v<V>(mb + row_off(slot[k]), out);
        if (k + 1 < D) {
#pragma unroll
            for (int v = 0; v < V; v++) pre[v] = __dmul_rn(pre[v], b[k][v]);
        }
    }
}

// ---- high-degree path: chains of outputs over shared-memory b ------------------
// One block per (check, tile of TW codewords), 1024 threads; degrees past kMaxRegCheckDegree.  The d outputs need
// d(d-1)/2 ordered multiplies per codeword (exactness forbids a suffix-product
// shortcut), so the work is fp64-bound for d >> 16 and is spread as:
//   * b_i = 1 - 2 q_i of the tile staged in shared memory ([d][TW]), or in the
//     workspace scratch when d is past the shared-memory budget; after that barrier
//     the in-place slot writes cannot race a read;
//   * outputs in groups of R = 8; lane = (codeword c = lane % TW, part h = lane / TW)
//     and each thread carries CPT = R*TW/32 output chains of its group, so one
//     shared load feeds CPT independent multiplies, and the TW lanes reading a row
//     form a conflict-free wavefront (the 32/TW parts read the same row: broadcast);
//   * a block has W = min(32, ceil(G/2)) warps for G groups (mid degrees get small
//     blocks, many per SM);
//   * warp w takes groups w, 2W-1-w, 2W+w, 4W-1-w, ... : ascending (so one running
//     prefix 1*b_0*...*b_{k-1} carried across its groups replaces a sequential
//     prefix pass), and balanced (each band of 64 pairs a long suffix with a short
//     one).  The carry rides in the body loop as one more chain.
constexpr int kWideR = 8;
constexpr int kWideThreads = 1024;

__device__ __forceinline__ int chains_group(int w, int t, int nw) {  // t-th group of warp w (of nw)
    const int band = t >> 1;
    return band * 2 * nw + ((t & 1) ? 2 * nw - 1 - w : w);
}

// R: outputs per group (R*TW/32 chains per thread)
template <int TW, bool FROM_PRIOR, bool GS, int R = kWideR>  // GS: staging in global scratch (degrees past the smem budget)
__global__ void __launch_bounds__(kWideThreads) k_check_chains(NodeLaunch a, int max_deg) {
    constexpr int CPT = R * TW / 32;   // chains per thread
    static_assert(CPT >= 1 && kWideThreads == 1024, "TW must be >= 4; up to 32 warps");
    extern __shared__ double smem_b[];
    double *b = GS ? a.scratch + (size_t)blockIdx.x * max_deg * TW : smem_b;  // [d][TW]
    int ni, tile;
    lpt_block(blockIdx.x, a.node_count, a.Bp / TW, ni, tile);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int c = lane % TW, h = lane / TW;
    const int cw = tile * TW + c;
    if (a.done != nullptr) {
        const int w0 = (tile * TW) >> 5;
        const uint32_t mask = (TW >= 32) ? 0xffffffffu : (((1u << TW) - 1u) << ((tile * TW) & 31));
        if ((a.done[w0] & mask) == mask) return;
    }
    const int node = __ldg(a.order + a.node_begin + ni);
    const int pos0 = __ldg(a.off + node);
    const int d = __ldg(a.off + node + 1) - pos0;
    const int G = (d + R - 1) / R;
    if constexpr (!GS) {
        // the tile's d row segments (TW codewords, 16-byte pieces) all in flight at once
        // (cp.async, no register round trip), then b = 1 - 2q in place
        constexpr int PPR = TW / 2;  // pieces per row segment
        for (int e = threadIdx.x; e < d * PPR; e += blockDim.x) {
            const int i = e / PPR, pc = e - i * PPR;
            const int cwe = tile * TW + 2 * pc;
            const double *src = FROM_PRIOR ? a.P + cofs(a.p_rows, __ldg(a.idx + pos0 + i), cwe)
                                           : a.msg + cofs(a.msg_rows, a.slot ? __ldg(a.slot + pos0 + i) : pos0 + i, cwe);
            cp_async16(b + i * TW + 2 * pc, src);
        }
        cp_commit();
        cp_wait<0>();
        __syncthreads();
        for (int e = threadIdx.x; e < d * TW; e += blockDim.x) b[e] = __dsub_rn(1.0, __dmul_rn(2.0, b[e]));
    } else {
        for (int e = threadIdx.x; e < d * TW; e += blockDim.x) {
            const int i = e / TW, cc = e - i * TW;
            const int cwe = tile * TW + cc;
            const double q = FROM_PRIOR ? __ldg(a.P + cofs(a.p_rows, __ldg(a.idx + pos0 + i), cwe))
                                        : ld_msg(a.msg + cofs(a.msg_rows, a.slot ? __ldg(a.slot + pos0 + i) : pos0 + i, cwe));
            b[e] = __dsub_rn(1.0, __dmul_rn(2.0, q));
        }
    }
    __syncthreads();
    const double *bc = b + c;
    auto B = [&](int i) { return bc[i * TW]; };
    const int j0 = h * CPT;  // this thread's outputs in a group: k0 + j0 .. k0 + j0 + CPT - 1
    // running prefix: pre = 1*b_0*...*b_{at-1}, left to right from 1.0 (serial.py:105-110 order)
    double pre = 1.0;
    int at = 0;
    for (int t = 0;; t++) {
        const int g = chains_group(warp, t, nw);
        if (g >= G) break;
        const int k0 = g * R, kb = k0 + j0;            // first output of this thread
        const int gn = chains_group(warp, t + 1, nw);
        const int next = gn * R + j0;                  // where the carry must stop (next group's kb)
        for (; at < kb; at++) pre = __dmul_rn(pre, at < d ? B(at) : 1.0);
        double acc[CPT];
        double p = pre;
#pragma unroll
        for (int j = 0; j < CPT; j++) {
            acc[j] = p;
            if (j + 1 < CPT) p = __dmul_rn(p, kb + j < d ? B(kb + j) : 1.0);
        }
        // head: position kb + j multiplies the chains whose output is below it
#pragma unroll
        for (int j = 1; j < CPT; j++) {
            if (kb + j < d) {
                const double x = B(kb + j);
#pragma unroll
                for (int jj = 0; jj < j; jj++) acc[jj] = __dmul_rn(acc[jj], x);
            }
        }
        // body with the carry: positions kb .. next-1 also extend the running prefix
        for (; at < kb + CPT && at < next; at++) pre = __dmul_rn(pre, at < d ? B(at) : 1.0);
        int i = kb + CPT;
        const int stop_carry = min(next, d);
        for (; i < stop_carry; i++) {
            const double x = B(i);
#pragma unroll
            for (int j = 0; j < CPT; j++) acc[j] = __dmul_rn(acc[j], x);
            pre = __dmul_rn(pre, x);
        }
        if (i > at) at = i;
        for (; i + 1 < d; i += 2) {
            const double x0 = B(i), x1 = B(i + 1);
#pragma unroll
            for (int j = 0; j < CPT; j++) acc[j] = __dmul_rn(__dmul_rn(acc[j], x0), x1);
        }
        if (i < d) {
            const double x = B(i);
#pragma unroll
            for (int j = 0; j < CPT; j++) acc[j] = __dmul_rn(acc[j], x);
        }
        // r_k = 1 - (0.5 + 0.5 * prod_k)
#pragma unroll
        for (int j = 0; j < CPT; j++) {
            const int k = kb + j;
            if (k < d)
                st_msg(a.msg + cofs(a.msg_rows, a.slot ? __ldg(a.slot + pos0 + k) : pos0 + k, cw),
                       __dsub_rn(1.0, __dadd_rn(0.5, __dmul_rn(0.5, acc[j]))));
        }
    }
}

// ---- dispatch -----------------------------------------------------------------
int vpolicy_check(int deg) {
    static int forced = [] {
        const char *e = getenv("LDPC_CHECK_V");
        return e ? atoi(e) : 0;
    }();
    if (forced == 1 || forced == 2) return forced;
    return deg <= 8 ? 2 : 1;
}

template <int D, int V, bool FP>
int launch_one(const NodeLaunch &a, cudaStream_t s) {
    const dim3 grid((a.node_count + kWarpsPerBlock - 1) / kWarpsPerBlock, a.Bp / (32 * V));
    if (a.node_count == 0) return LDPC_OK;
    LDPC_ARG_CHECK(grid.y <= 65535u, "batch too large for one launch (%d codewords)", a.Bp);
    k_check_reg<D, V, FP><<<grid, kThreads, 0, s>>>(a);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

template <int D>
int launch_deg(const NodeLaunch &a, bool fp, cudaStream_t s) {
    // tile views of 32 codewords take V=1; so do degrees past 16 (D*V values in registers)
    if constexpr (D > kMaxRegDegree) {
        return fp ? launch_one<D, 1, true>(a, s) : launch_one<D, 1, false>(a, s);
    } else {
        const int V = (a.Bp % 64) ? 1 : vpolicy_check(D);
        if (V == 2) return fp ? launch_one<D, 2, true>(a, s) : launch_one<D, 2, false>(a, s);
        return fp ? launch_one<D, 1, true>(a, s) : launch_one<D, 1, false>(a, s);
    }
}

}  // namespace

int launch_check_bucket(const NodeLaunch &a, int deg, bool from_prior, cudaStream_t s) {
    switch (deg) {
#define CASE(D) \
    case D: return launch_deg<D>(a, from_prior, s);
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
        CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
        CASE(17) CASE(18) CASE(19) CASE(20) CASE(21) CASE(22) CASE(23) CASE(24)
        CASE(25) CASE(26) CASE(27) CASE(28) CASE(29) CASE(30) CASE(31) CASE(32)
#undef CASE
        default:
            set_error("register-path check degree %d out of range", deg);
            return LDPC_EINVAL;
    }
}

// warps per block: enough for two groups each (a band pairs a long suffix with a short one), up to 32
inline int chain_warps(int max_deg, int R) {
    const int G = (max_deg + R - 1) / R;
    return std::max(1, std::min(32, (G + 1) / 2));
}

template <int TW, bool GS>
int launch_chains(const NodeLaunch &a, int max_deg, size_t smem, bool from_prior, cudaStream_t s) {
    // groups of 16 outputs (8 chains per thread at TW = 16) when they still fill the 32 warps'
    // bands; else 8.  LDPC_CHAIN_R=8|16 forces one.
    static const int r_env = [] {
        const char *e = getenv("LDPC_CHAIN_R");
        return e ? atoi(e) : 0;
    }();
    const bool r16 = r_env ? r_env == 16 : (max_deg + 15) / 16 >= 48;
    auto kern = from_prior ? k_check_chains<TW, true, GS> : k_check_chains<TW, false, GS>;
    if (r16) kern = from_prior ? k_check_chains<TW, true, GS, 16> : k_check_chains<TW, false, GS, 16>;
    // the cap (not this launch's size): launches of one instantiation with different tiles may be issued
    // from several threads or side streams
    if (smem) LDPC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kChainSmemBudget));
    const int64_t blocks = (int64_t)a.node_count * (a.Bp / TW);
    kern<<<(unsigned)blocks, 32 * chain_warps(max_deg, r16 ? 16 : kWideR), smem, s>>>(a, max_deg);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

int launch_check_wide(const NodeLaunch &a, int max_deg, bool from_prior, cudaStream_t s) {
    if (a.node_count == 0) return LDPC_OK;
    // the widest tile (more chains per thread) whose b fits in shared memory; past that,
    // 16-codeword tiles staged in the workspace scratch.  LDPC_WIDE_TW=4|8|16 forces a tile.
    static const int forced = [] {
        const char *e = getenv("LDPC_WIDE_TW");
        return e ? atoi(e) : 0;
    }();
    auto smem = [&](int tw) { return (size_t)max_deg * tw * sizeof(double); };
    if ((forced == 0 || forced == 16) && smem(16) <= kChainSmemBudget) return launch_chains<16, false>(a, max_deg, smem(16), from_prior, s);
    if ((forced == 0 || forced == 8) && smem(8) <= kChainSmemBudget) return launch_chains<8, false>(a, max_deg, smem(8), from_prior, s);
    if ((forced == 0 || forced == 4) && smem(4) <= kChainSmemBudget) return launch_chains<4, false>(a, max_deg, smem(4), from_prior, s);
    LDPC_ARG_CHECK(a.scratch != nullptr, "check degree %d needs the workspace scratch (workspace too old?)", max_deg);
    return launch_chains<kChainTW, true>(a, max_deg, 0, from_prior, s);
}

}  // namespace ldpc
