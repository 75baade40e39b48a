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
    const int ch = blockIdx.y;
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

// ---- wide path: one block per (node, tile of TW codewords) -----------------
// Shared memory holds b_i and the prefix products for the tile; worker w of
// the block produces outputs k = w, w + NWK, ... (NWK = 256 / TW workers).
template <bool FROM_PRIOR>
__global__ void __launch_bounds__(kThreads) k_check_wide(NodeLaunch a, int TW, int max_deg) {
    extern __shared__ double sm[];
    double *b = sm;                         // [max_deg][TW]
    double *pre = sm + (size_t)max_deg * TW; // [max_deg][TW]
    const int tile = blockIdx.x / a.node_count;  // tile-major: all nodes of tile 0 first
    const int ni = blockIdx.x - tile * a.node_count;
    const int c = threadIdx.x % TW;
    const int worker = threadIdx.x / TW;
    const int nwk = blockDim.x / TW;
    const int cw = tile * TW + c;
    if (a.done != nullptr) {
        const int w0 = (tile * TW) >> 5;
        const uint32_t mask = (TW >= 32) ? 0xffffffffu : (((1u << TW) - 1u) << ((tile * TW) & 31));
        bool all = true;
        for (int w = w0; w < w0 + (TW + 31) / 32; w++) all = all && ((a.done[w] & mask) == mask);
        if (all) return;
    }
    const int node = __ldg(a.order + a.node_begin + ni);
    const int pos0 = __ldg(a.off + node);
    const int d = __ldg(a.off + node + 1) - pos0;
    for (int i = worker; i < d; i += nwk) {
        double q = FROM_PRIOR ? __ldg(a.P + cofs(a.p_rows, __ldg(a.idx + pos0 + i), cw))
                              : ld_msg(a.msg + cofs(a.msg_rows, a.slot ? __ldg(a.slot + pos0 + i) : pos0 + i, cw));
        b[i * TW + c] = __dsub_rn(1.0, __dmul_rn(2.0, q));
    }
    __syncthreads();
    if (worker == 0) {
        double p = 1.0;
        for (int i = 0; i < d; i++) {
            pre[i * TW + c] = p;
            p = __dmul_rn(p, b[i * TW + c]);
        }
    }
    __syncthreads();
    // fold outputs so each worker gets a mix of long and short suffix chains
    for (int j = worker; j < d; j += nwk) {
        const int k = (j & 1) ? (d - 1 - (j >> 1)) : (j >> 1);
        double acc = pre[k * TW + c];
        for (int i = k + 1; i < d; i++) acc = __dmul_rn(acc, b[i * TW + c]);
        st_msg(a.msg + cofs(a.msg_rows, a.slot ? __ldg(a.slot + pos0 + k) : pos0 + k, cw), __dsub_rn(1.0, __dadd_rn(0.5, __dmul_rn(0.5, acc))));
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
    const int V = (a.Bp % 64) ? 1 : vpolicy_check(D);  // tile views of 32 codewords take V=1
    if (V == 2) return fp ? launch_one<D, 2, true>(a, s) : launch_one<D, 2, false>(a, s);
    return fp ? launch_one<D, 1, true>(a, s) : launch_one<D, 1, false>(a, s);
}

}  // namespace

int launch_check_bucket(const NodeLaunch &a, int deg, bool from_prior, cudaStream_t s) {
    switch (deg) {
#define CASE(D) \
    case D: return launch_deg<D>(a, from_prior, s);
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
        CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
        default:
            set_error("register-path check degree %d out of range", deg);
            return LDPC_EINVAL;
    }
}

int launch_check_wide(const NodeLaunch &a, int max_deg, bool from_prior, cudaStream_t s) {
    if (a.node_count == 0) return LDPC_OK;
    const size_t budget = 200 * 1024;
    int TW = 32;
    while (TW > 1 && (size_t)2 * max_deg * TW * sizeof(double) > budget) TW >>= 1;
    const size_t smem = (size_t)2 * max_deg * TW * sizeof(double);
    if (smem > budget) {
        set_error("check degree %d exceeds the shared-memory staging limit", max_deg);
        return LDPC_EINVAL;
    }
    auto kern = from_prior ? k_check_wide<true> : k_check_wide<false>;
    LDPC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t blocks = (int64_t)a.node_count * (a.Bp / TW);
    kern<<<(unsigned)blocks, kThreads, smem, s>>>(a, TW, max_deg);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

}  // namespace ldpc
