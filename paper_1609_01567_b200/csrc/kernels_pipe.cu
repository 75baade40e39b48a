// kernels_pipe.cu -- node updates fed by asynchronous bulk copies (the default path
// for node degrees <= kMaxRegDegree).
//
// Same arithmetic as kernels_check.cu / kernels_var.cu (serial.py:63-133,
// exact fp64, explicit round-to-nearest intrinsics), different data movement:
// each warp runs its own S-stage ring in shared memory.  For a task
// (node, 64-codeword chunk) lanes 0..ROWS-1 each issue one 512-byte
// `cp.async.bulk` (UBLKCP) global->shared copy -- one message row per edge,
// plus the prior row for variables -- completing on the stage's mbarrier.
// While the warp computes task i from shared memory, the rows of tasks
// i+1 .. i+S-1 are already in flight, so the gathers of the variable phase
// (scattered slots) no longer stall on DRAM latency with registers tied up in
// outstanding loads.  Outputs are written straight to global (one coalesced
// 512-byte run per edge).  The grid is persistent: warp w of W handles tasks
// w, w+W, ... in chunk-major order, so the concurrently touched rows stay
// inside one codeword chunk's message window.
#include <algorithm>
#include <mutex>

#include "common.cuh"

namespace ldpc {
namespace {

constexpr int kRowBytes = 64 * sizeof(double);  // one slot x 64 codewords

// ring depth: up to 4 stages while a warp's ring stays within 24 KB
constexpr int stages_for(int rows) {
    return rows * kRowBytes * 4 <= 24576 ? 4 : (rows * kRowBytes * 3 <= 24576 ? 3 : 2);
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void st_cs2(double *p, double x, double y) {
    __stcs(reinterpret_cast<double2 *>(p), make_double2(x, y));
}

// Per-warp shared-memory carve: [S] mbarriers | [S][ROWS] slot ids | [S] skip flags | rows
template <int ROWS>
struct WarpRing {
    static constexpr int kStages = stages_for(ROWS);
    // barriers + ids + flags, then 128B-aligned rows
    static constexpr size_t kHeader = ((size_t)8 * kStages + 4 * kStages * ROWS + 4 * kStages + 127) / 128 * 128;
    static constexpr size_t kBytes = kHeader + (size_t)kStages * ROWS * kRowBytes;
    uint64_t *bar;
    int32_t *ids;
    int32_t *skip;
    double *rows;
    __device__ WarpRing(unsigned char *base) {
        bar = reinterpret_cast<uint64_t *>(base);
        ids = reinterpret_cast<int32_t *>(base + 8 * kStages);
        skip = ids + kStages * ROWS;
        rows = reinterpret_cast<double *>(base + kHeader);
    }
    __device__ double *row(int s, int r) const { return rows + ((size_t)s * ROWS + r) * 64; }
};

__device__ __forceinline__ bool chunk64_done(const uint32_t *done, int ch) {
    if (done == nullptr) return false;
    const uint2 d = *reinterpret_cast<const uint2 *>(done + 2 * ch);
    return (d.x & d.y) == 0xffffffffu;
}

// Issue the copies of task t into stage s (all lanes call; lanes < ROWS copy).
template <int D, bool IS_VAR, bool FROM_PRIOR>
__device__ __forceinline__ void issue_task(const NodeLaunch &a, const WarpRing<D + (IS_VAR ? 1 : 0)> &ring,
                                           int s, int64_t t, int lane) {
    constexpr int ROWS = D + (IS_VAR ? 1 : 0);
    const int ch = (int)(t / a.node_count);
    const int ni = (int)(t - (int64_t)ch * a.node_count);
    const bool skip = chunk64_done(a.done, ch);
    const int32_t base = a.edge_begin + ni * D;  // bucket-ordered flat edge tables
    const double *src = nullptr;
    int id = -1;
    if (lane < D) {
        id = __ldg(a.slot_ord + base + lane);
        if constexpr (IS_VAR) {
            src = a.msg + cofs(a.msg_rows, id, ch * 64);
        } else {
            src = FROM_PRIOR ? a.P + cofs(a.p_rows, __ldg(a.var_ord + base + lane), ch * 64)
                             : a.msg + cofs(a.msg_rows, id, ch * 64);
        }
    } else if (IS_VAR && lane == D) {
        id = __ldg(a.order + a.node_begin + ni);
        src = a.P + cofs(a.p_rows, id, ch * 64);
    }
    if (lane < ROWS) ring.ids[s * ROWS + lane] = id;
    if (lane == 0) {
        ring.skip[s] = skip ? 1 : 0;
        if (!skip) mbar_arrive_expect_tx(&ring.bar[s], ROWS * kRowBytes);
        else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&ring.bar[s])) : "memory");
    }
    __syncwarp();
    if (!skip && lane < ROWS) bulk_g2s(ring.row(s, lane), src, kRowBytes, &ring.bar[s]);
}

template <int D, bool FROM_PRIOR>
__device__ __forceinline__ void compute_check(const NodeLaunch &a, const WarpRing<D> &ring, int s, int ch, int lane) {
    double b[D][2];
#pragma unroll
    for (int i = 0; i < D; i++) {
        const double2 q = *reinterpret_cast<const double2 *>(ring.row(s, i) + 2 * lane);
        b[i][0] = __dsub_rn(1.0, __dmul_rn(2.0, q.x));
        b[i][1] = __dsub_rn(1.0, __dmul_rn(2.0, q.y));
    }
    double pre0 = 1.0, pre1 = 1.0;
#pragma unroll
    for (int k = 0; k < D; k++) {
        double acc0 = pre0, acc1 = pre1;
#pragma unroll
        for (int i = k + 1; i < D; i++) {
            acc0 = __dmul_rn(acc0, b[i][0]);
            acc1 = __dmul_rn(acc1, b[i][1]);
        }
        st_cs2(a.msg + cofs(a.msg_rows, ring.ids[s * D + k], ch * 64 + 2 * lane),
               __dsub_rn(1.0, __dadd_rn(0.5, __dmul_rn(0.5, acc0))),
               __dsub_rn(1.0, __dadd_rn(0.5, __dmul_rn(0.5, acc1))));
        if (k + 1 < D) {
            pre0 = __dmul_rn(pre0, b[k][0]);
            pre1 = __dmul_rn(pre1, b[k][1]);
        }
    }
}

template <int D, bool WRITE_Q>
__device__ __forceinline__ void compute_var(const NodeLaunch &a, const WarpRing<D + 1> &ring, int s, int ch, int lane) {
    double r[D][2], om[D][2];
#pragma unroll
    for (int i = 0; i < D; i++) {
        const double2 x = *reinterpret_cast<const double2 *>(ring.row(s, i) + 2 * lane);
        r[i][0] = x.x;
        r[i][1] = x.y;
        om[i][0] = __dsub_rn(1.0, x.x);
        om[i][1] = __dsub_rn(1.0, x.y);
    }
    const double2 pj = *reinterpret_cast<const double2 *>(ring.row(s, D) + 2 * lane);
    double p0[2] = {__dsub_rn(1.0, pj.x), __dsub_rn(1.0, pj.y)};
    double p1[2] = {pj.x, pj.y};
#pragma unroll
    for (int k = 0; k < D; k++) {
        if constexpr (WRITE_Q) {
            double out[2];
#pragma unroll
            for (int v = 0; v < 2; v++) {
                double q0 = p0[v], q1 = p1[v];
#pragma unroll
                for (int i = k + 1; i < D; i++) {
                    q0 = __dmul_rn(q0, om[i][v]);
                    q1 = __dmul_rn(q1, r[i][v]);
                }
                const double den = __dadd_rn(q0, q1);
                bool ok;
                out[v] = ddiv_fast(q1, den, ok);
                if (!ok) out[v] = (den == 0.0) ? 0.5 : __ddiv_rn(q1, den);
            }
            st_cs2(a.msg + cofs(a.msg_rows, ring.ids[s * (D + 1) + k], ch * 64 + 2 * lane), out[0], out[1]);
        }
#pragma unroll
        for (int v = 0; v < 2; v++) {
            p0[v] = __dmul_rn(p0[v], om[k][v]);
            p1[v] = __dmul_rn(p1[v], r[k][v]);
        }
    }
    // estimate (serial.py:132): bit = !(Q0 > Q1); ballots -> natural codeword order
    const uint32_t even = __ballot_sync(0xffffffffu, !(p0[0] > p1[0]));
    const uint32_t odd = __ballot_sync(0xffffffffu, !(p0[1] > p1[1]));
    if (lane == 0) {
        const int node = ring.ids[s * (D + 1) + D];
        uint32_t lo = part1by1(even) | (part1by1(odd) << 1);
        uint32_t hi = part1by1(even >> 16) | (part1by1(odd >> 16) << 1);
        uint32_t *dst = a.chat + (size_t)node * a.NW + 2 * ch;
        if (a.done != nullptr) {
            const uint32_t d0 = a.done[2 * ch], d1 = a.done[2 * ch + 1];
            if (d0) lo = (lo & ~d0) | (dst[0] & d0);
            if (d1) hi = (hi & ~d1) | (dst[1] & d1);
        }
        *reinterpret_cast<uint2 *>(dst) = make_uint2(lo, hi);
    }
}

template <int D, bool IS_VAR, bool FLAG>  // FLAG = FROM_PRIOR (checks) / WRITE_Q (variables)
__global__ void __launch_bounds__(kThreads) k_node_pipe(NodeLaunch a, int64_t ntasks) {
    constexpr int ROWS = D + (IS_VAR ? 1 : 0);
    constexpr int kStages = WarpRing<ROWS>::kStages;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    WarpRing<ROWS> ring(smem + (size_t)warp * WarpRing<ROWS>::kBytes);
    if (lane == 0) {
        for (int s = 0; s < kStages; s++) mbar_init(&ring.bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int64_t W = (int64_t)gridDim.x * kWarpsPerBlock;
    const int64_t first = (int64_t)blockIdx.x * kWarpsPerBlock + warp;
    for (int s = 0; s < kStages; s++) {
        const int64_t t = first + s * W;
        if (t < ntasks) issue_task<D, IS_VAR, IS_VAR ? false : FLAG>(a, ring, s, t, lane);
    }
    int it = 0;
    for (int64_t t = first; t < ntasks; t += W, it++) {
        const int s = it % kStages;
        mbar_wait(&ring.bar[s], (it / kStages) & 1);
        const int ch = (int)(t / a.node_count);
        if (!ring.skip[s]) {
            if constexpr (IS_VAR) compute_var<D, FLAG>(a, ring, s, ch, lane);
            else compute_check<D, FLAG>(a, ring, s, ch, lane);
        }
        __syncwarp();  // everyone is done reading stage s before it is refilled
        const int64_t tn = t + kStages * W;
        if (tn < ntasks) issue_task<D, IS_VAR, IS_VAR ? false : FLAG>(a, ring, s, tn, lane);
    }
}

template <int D, bool IS_VAR, bool FLAG>
int launch_pipe(const NodeLaunch &a, cudaStream_t st) {
    constexpr int ROWS = D + (IS_VAR ? 1 : 0);
    const size_t smem = (size_t)kWarpsPerBlock * WarpRing<ROWS>::kBytes;
    auto kern = k_node_pipe<D, IS_VAR, FLAG>;
    static int per_sm = -1;
    static int sms = 0;
    static std::mutex mu;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (per_sm < 0) {
            LDPC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            int dev = 0;
            LDPC_CUDA_TRY(cudaGetDevice(&dev));
            LDPC_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            LDPC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem));
            if (per_sm < 1) {
                set_error("pipelined node kernel (degree %d) does not fit on an SM", D);
                per_sm = -1;
                return LDPC_ECUDA;
            }
        }
    }
    const int64_t ntasks = (int64_t)a.node_count * (a.Bp / 64);
    if (ntasks == 0) return LDPC_OK;
    const int64_t need = (ntasks + kWarpsPerBlock - 1) / kWarpsPerBlock;
    const int64_t blocks = std::min<int64_t>(need, (int64_t)per_sm * sms);
    kern<<<(unsigned)blocks, kThreads, smem, st>>>(a, ntasks);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

}  // namespace

int launch_check_pipe(const NodeLaunch &a, int deg, bool from_prior, cudaStream_t s) {
    switch (deg) {
#define CASE(D) \
    case D: return from_prior ? launch_pipe<D, false, true>(a, s) : launch_pipe<D, false, false>(a, s);
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
        CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
        default:
            set_error("pipelined check degree %d out of range", deg);
            return LDPC_EINVAL;
    }
}

int launch_var_pipe(const NodeLaunch &a, int deg, bool write_q, cudaStream_t s) {
    switch (deg) {
#define CASE(D) \
    case D: return write_q ? launch_pipe<D, true, true>(a, s) : launch_pipe<D, true, false>(a, s);
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
        CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
        default:
            set_error("pipelined variable degree %d out of range", deg);
            return LDPC_EINVAL;
    }
}

}  // namespace ldpc
