// grid.cu -- the whole decode of a few codewords in ONE cooperative launch (grid schedule).
//
// The streaming schedule pads a batch to 64 codewords and makes each of its ~5 launches
// per iteration move the padded chunk through HBM: a single C3 frame costs what 64 do
// (2.9 ms at 16 iterations).  For B <= kGridMaxB codewords of a code too large for the
// on-chip schedule, one cooperative grid (every SM, all blocks resident) instead keeps
// the B codewords' messages in a workspace (B * E * 8 bytes: 1.8 MB per C3
// codeword, L2-resident) and runs Algorithm 2 with grid-wide barriers, one thread per
// (node, codeword) item (codeword-minor layout, node-major items: a warp's accesses to a message
// row are one contiguous run):
//   init:   priors (or observations -> priors, priors.cuh), zeroed outputs and flags
//   pre:    C-phase from the priors (serial.py:166)
//   round t (serial.py:165-178), two barriers, as the on-chip kernel:
//     VE: chat_t = Est(r_t) and, unless t = max, q_{t+1} = V(p, r_t)
//     SC: z_t = Syn(chat_t) -> unsat bit of the codeword, and, unless t = max, r_{t+1} = C(q_{t+1})
//     a codeword whose syndrome is zero stops (early stop): its items are skipped from then
//     on, so its estimate and syndrome stay those of round t.
//   final:  packed estimate / syndrome rows, success, iterations.
// Node arithmetic: nodes.cuh (= the register kernels, operation for operation).
#include <cooperative_groups.h>

#include <mutex>

#include "common.cuh"
#include "nodes.cuh"
#include "priors.cuh"

namespace cg = cooperative_groups;

namespace ldpc {
namespace {

constexpr int kGridThreads = 256;

struct GridArgs {
    int32_t n, m, B, max_iter, early, RWn, RWm;
    const double *in;      // [B][n] priors, or observations when sig2 != nullptr
    const double *sig2;    // [B] or nullptr
    NodeTables tb;
    double *msg;           // [B][E]
    double *pr;            // [B][n]
    uint8_t *chat;         // [B][n]
    unsigned long long *unsat;  // [2]: bit cw = codeword cw unsatisfied, by round parity
    uint32_t *est;         // [B][RWn]
    uint8_t *succ;         // [B]
    int32_t *iters;        // [B]
    uint32_t *syn;         // [B][RWm] or nullptr
    int64_t E;
};

// Layout: codeword-minor -- msg[E][B], pr[n][B], chat[n][B] -- and items ordered node-major
// (item k = node k / B, codeword k % B), so the 32 lanes of a warp are consecutive codewords of one
// node (or a few nodes when B < 32) and each message row a warp touches is one contiguous run.
struct GridAcc {  // nodes.cuh accessor for codeword cw
    double *msg;        // &msg[0][cw]
    const double *pr;   // &pr[0][cw]
    int32_t B;
    __device__ __forceinline__ double *slot(int s) const { return msg + (size_t)s * B; }
    __device__ __forceinline__ double prior_of(int v) const { return pr[(size_t)v * B]; }
};

__global__ void __launch_bounds__(kGridThreads) k_grid(const __grid_constant__ GridArgs a) {
    cg::grid_group grid = cg::this_grid();
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    const int64_t nB = (int64_t)a.n * a.B, mB = (int64_t)a.m * a.B;
    using Mask = unsigned long long;  // one bit per codeword (B <= 64)
    const Mask all = (a.B >= 64) ? ~0ull : ((1ull << a.B) - 1ull);
    auto acc = [&](int cw) { return GridAcc{a.msg + cw, a.pr + cw, a.B}; };

    // init: [B][n] input -> pr[n][B]
    for (int64_t k = tid; k < nB; k += T) {
        const int v = (int)(k / a.B), cw = (int)(k - (int64_t)v * a.B);
        const double x = __ldg(a.in + (size_t)cw * a.n + v);
        a.pr[k] = a.sig2 ? awgn_prior(x, __ldg(a.sig2 + cw)) : x;
    }
    for (int64_t k = tid; k < (int64_t)a.B * a.RWn; k += T) a.est[k] = 0u;
    if (a.syn)
        for (int64_t k = tid; k < (int64_t)a.B * a.RWm; k += T) a.syn[k] = 0u;
    if (tid < 2) a.unsat[tid] = 0ull;
    grid.sync();
    // pre-pass C-phase from the priors
    for (int64_t k = tid; k < mB; k += T) {
        const int c = (int)(k / a.B), cw = (int)(k - (int64_t)c * a.B);
        check_node<true>(acc(cw), a.tb, c);
    }
    grid.sync();
    Mask done = 0;  // identical in every thread: derived from the same flags after a barrier
    int t = 0;
    for (;; t++) {
        const bool more = t < a.max_iter;
        // VE
        for (int64_t k = tid; k < nB; k += T) {
            const int v = (int)(k / a.B), cw = (int)(k - (int64_t)v * a.B);
            if ((done >> cw) & 1u) continue;
            a.chat[k] = var_node(acc(cw), a.tb, v, more, a.pr[k]);
        }
        grid.sync();
        // SC; the other parity's flag was last read before the VE barrier: reset it for round t+1
        if (tid == 0) a.unsat[(t + 1) & 1] = 0ull;
        Mask unsat = 0;
        for (int64_t k = tid; k < mB; k += T) {
            const int c = (int)(k / a.B), cw = (int)(k - (int64_t)c * a.B);
            if ((done >> cw) & 1u) continue;
            const int s0 = __ldg(a.tb.chk_off + c), d = __ldg(a.tb.chk_off + c + 1) - s0;
            const uint8_t *ch = a.chat + cw;
            int z = 0;
            for (int i = 0; i < d; i++) z ^= ch[(size_t)__ldg(a.tb.chk_var + s0 + i) * a.B];
            if (z) unsat |= 1ull << cw;
            if (more) check_node<false>(acc(cw), a.tb, c);
        }
        // one atomic per warp
        for (int o = 16; o > 0; o >>= 1) unsat |= __shfl_xor_sync(0xffffffffu, unsat, o);
        if ((threadIdx.x & 31) == 0 && unsat) atomicOr(a.unsat + (t & 1), unsat);
        grid.sync();
        const Mask u = *((volatile Mask *)a.unsat + (t & 1));
        const Mask newly = all & ~done & ~u;  // zero syndrome at round t
        if (tid < a.B && ((newly >> tid) & 1u) && a.early) {
            a.succ[tid] = 1;
            a.iters[tid] = t;
        }
        if (a.early) done |= newly;
        if (done == all || !more) break;
    }
    // codewords still running: ran out of rounds (early stop) or fixed iterations
    if (tid < a.B && !((done >> tid) & 1u)) {
        const Mask u = *((volatile Mask *)a.unsat + (t & 1));
        a.succ[tid] = ((u >> tid) & 1u) ? 0 : 1;
        a.iters[tid] = a.max_iter;
    }
    // packed estimate and syndrome rows of the final state
    for (int64_t k = tid; k < nB; k += T) {
        if (!a.chat[k]) continue;
        const int v = (int)(k / a.B), cw = (int)(k - (int64_t)v * a.B);
        atomicOr(a.est + (size_t)cw * a.RWn + (v >> 5), 1u << (v & 31));
    }
    if (a.syn)
        for (int64_t k = tid; k < mB; k += T) {
            const int c = (int)(k / a.B), cw = (int)(k - (int64_t)c * a.B);
            const int s0 = __ldg(a.tb.chk_off + c), d = __ldg(a.tb.chk_off + c + 1) - s0;
            const uint8_t *ch = a.chat + cw;
            int z = 0;
            for (int i = 0; i < d; i++) z ^= ch[(size_t)__ldg(a.tb.chk_var + s0 + i) * a.B];
            if (z) atomicOr(a.syn + (size_t)cw * a.RWm + (c >> 5), 1u << (c & 31));
        }
}

std::mutex g_grid_mu;
int g_grid_blocks[64] = {};  // resident blocks per SM, per device

}  // namespace

size_t grid_workspace_bytes(const ldpc_graph *g, int32_t B) {
    return (size_t)B * ((size_t)g->E * 8 + (size_t)g->n * 8 + (size_t)g->n) + 256;
}

bool grid_suitable(const ldpc_graph *g, int32_t B) {
    return B >= 1 && B <= kGridMaxB && g->max_dv <= kMaxRegDegree && g->max_dc <= kMaxRegDegree;
}

int launch_grid(const ldpc_graph *g, const double *in, const double *sig2, int32_t B, int32_t max_iter, bool early,
                uint32_t *est, uint8_t *succ, int32_t *iters, uint32_t *syn, void *ws, size_t ws_bytes,
                cudaStream_t s) {
    LDPC_ARG_CHECK(B >= 1 && B <= kGridMaxB, "grid schedule takes 1..%d codewords", kGridMaxB);
    LDPC_ARG_CHECK(ws_bytes >= grid_workspace_bytes(g, B), "workspace too small for the grid schedule");
    int dev = 0;
    LDPC_CUDA_TRY(cudaGetDevice(&dev));
    LDPC_ARG_CHECK(dev >= 0 && dev < 64, "device ordinal %d out of range", dev);
    int per_sm, sms;
    {
        std::lock_guard<std::mutex> lock(g_grid_mu);
        if (g_grid_blocks[dev] == 0) {
            int b = 0;
            LDPC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_grid, kGridThreads, 0));
            LDPC_ARG_CHECK(b >= 1, "grid kernel does not fit on an SM");
            g_grid_blocks[dev] = b;
        }
        per_sm = g_grid_blocks[dev];
    }
    LDPC_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    GridArgs a{};
    a.n = g->n;
    a.m = g->m;
    a.B = B;
    a.max_iter = max_iter;
    a.early = early ? 1 : 0;
    a.RWn = (g->n + 31) / 32;
    a.RWm = (g->m + 31) / 32;
    a.in = in;
    a.sig2 = sig2;
    a.tb = NodeTables{g->chk_off, g->chk_var, g->var_off, g->var_pos};
    a.E = g->E;
    auto *base = static_cast<unsigned char *>(ws);
    a.msg = reinterpret_cast<double *>(base);
    a.pr = a.msg + (size_t)B * g->E;
    a.unsat = reinterpret_cast<unsigned long long *>(a.pr + (size_t)B * g->n);
    a.chat = reinterpret_cast<uint8_t *>(a.unsat + 16);
    a.est = est;
    a.succ = succ;
    a.iters = iters;
    a.syn = syn;
    // enough threads for one item each, capped at what is resident (cooperative launch)
    const int64_t items = (int64_t)std::max(g->n, g->m) * B;
    const int64_t want = (items + kGridThreads - 1) / kGridThreads;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)per_sm * sms));
    void *args[] = {&a};
    LDPC_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)k_grid, dim3(blocks), dim3(kGridThreads), args, 0, s));
    count_launch();
    return LDPC_OK;
}

}  // namespace ldpc
