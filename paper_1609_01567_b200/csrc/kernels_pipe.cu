// kernels_pipe.cu -- node updates fed by an asynchronous per-warp copy ring.
//
// Same arithmetic as kernels_check.cu / kernels_var.cu (serial.py:63-133,
// exact fp64, explicit round-to-nearest operations), different data movement.
//
// Why: the register-load kernels keep a warp's message rows in registers
// while they are in flight, so the bytes in flight per SM are capped by the
// register file; ncu shows DRAM efficiency tracking exactly that (check
// kernel ~84 KB in flight -> 84 % of peak, variable kernels ~42 KB -> 60 %).
// Here every lane copies its 16-byte piece of each row with `cp.async.cg`
// (LDGSTS: global -> shared, no register destination) into an S-stage ring
// owned by the warp, so S-1 tasks per warp are in flight while the warp
// computes the oldest one from shared memory.  Each lane reads back only the
// bytes it copied itself, so the lane-local cp.async.wait_group is the only
// synchronisation the data needs.  The row ids of a task are loaded one ring
// step before its copies are issued, so index latency is off the critical path.
//
// A task is (node, 64-codeword chunk); lane l owns codewords 2l, 2l+1 of the
// chunk (16 bytes of each 512-byte row).  The grid is persistent: warp w of W
// takes tasks w, w+W, ... in chunk-major order.
#include <algorithm>
#include <mutex>

#include "common.cuh"

namespace ldpc {
namespace {

constexpr int kRow = 64;  // doubles per row (one slot x 64 codewords)

// ring depth: ~13 KB of ring per warp (two 8-warp blocks per SM)
constexpr int ring_stages(int rows) {
    const int s = (13 * 1024) / (rows * kRow * 8);
    return s < 2 ? 2 : (s > 8 ? 8 : s);
}

template <int ROWS>
struct Ring {
    static constexpr int S = ring_stages(ROWS);
    static constexpr size_t kIdsBytes = (size_t)S * 32 * sizeof(int);  // row ids per stage, one per lane
    static constexpr size_t kBytes = kIdsBytes + (size_t)S * ROWS * kRow * sizeof(double);
};

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void st_cs2(double *p, double x, double y) {
    __stcs(reinterpret_cast<double2 *>(p), make_double2(x, y));
}

__device__ __forceinline__ bool chunk64_done(const uint32_t *done, int ch) {
    if (done == nullptr) return false;
    const uint2 d = *reinterpret_cast<const uint2 *>(done + 2 * ch);
    return (d.x & d.y) == 0xffffffffu;
}

// Row ids of a task, one per lane:
//   lanes 0..D-1: message slots of the node's edges (outputs; inputs unless FROM_PRIOR)
//   variables: lane D = the variable (its prior row and c_hat row)
//   checks FROM_PRIOR: lanes 16..16+D-1 = variables whose prior rows are the inputs
template <int D, bool IS_VAR, bool FROM_PRIOR>
__device__ __forceinline__ int load_id(const NodeLaunch &a, int64_t t, int lane) {
    const int ni = (int)(t % a.node_count);
    const int32_t base = a.edge_begin + ni * D;
    if (lane < D) return __ldg(a.slot_ord + base + lane);
    if (IS_VAR && lane == D) return __ldg(a.order + a.node_begin + ni);
    if (!IS_VAR && FROM_PRIOR && lane >= 16 && lane < 16 + D) return __ldg(a.var_ord + base + lane - 16);
    return 0;
}

template <int D, bool IS_VAR, bool FROM_PRIOR>
__device__ __forceinline__ void issue(const NodeLaunch &a, double *rows, int *ids_s, int64_t t, int id, int lane) {
    constexpr int ROWS = D + (IS_VAR ? 1 : 0);
    const int ch = (int)(t / a.node_count);
    ids_s[lane] = id;
    if (chunk64_done(a.done, ch)) return;  // nothing to fetch; compute skips it too
#pragma unroll
    for (int r = 0; r < ROWS; r++) {
        const double *src;
        if (IS_VAR && r == D) src = a.P + cofs(a.p_rows, __shfl_sync(0xffffffffu, id, D), ch * 64);
        else if (!IS_VAR && FROM_PRIOR) src = a.P + cofs(a.p_rows, __shfl_sync(0xffffffffu, id, 16 + r), ch * 64);
        else src = a.msg + cofs(a.msg_rows, __shfl_sync(0xffffffffu, id, r), ch * 64);
        cp_async16(rows + r * kRow + 2 * lane, src + 2 * lane);
    }
}

template <int D>
__device__ __forceinline__ void compute_check(const NodeLaunch &a, const double *rows, const int *ids, int ch,
                                              int lane) {
    double b[D][2];
#pragma unroll
    for (int i = 0; i < D; i++) {
        const double2 q = *reinterpret_cast<const double2 *>(rows + i * kRow + 2 * lane);
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
        st_cs2(a.msg + cofs(a.msg_rows, ids[k], ch * 64 + 2 * lane), __dsub_rn(1.0, __dadd_rn(0.5, __dmul_rn(0.5, acc0))),
               __dsub_rn(1.0, __dadd_rn(0.5, __dmul_rn(0.5, acc1))));
        if (k + 1 < D) {
            pre0 = __dmul_rn(pre0, b[k][0]);
            pre1 = __dmul_rn(pre1, b[k][1]);
        }
    }
}

template <int D, bool WRITE_Q>
__device__ __forceinline__ void compute_var(const NodeLaunch &a, const double *rows, const int *ids, int ch,
                                            int lane) {
    double r[D][2], om[D][2];
#pragma unroll
    for (int i = 0; i < D; i++) {
        const double2 x = *reinterpret_cast<const double2 *>(rows + i * kRow + 2 * lane);
        r[i][0] = x.x;
        r[i][1] = x.y;
        om[i][0] = __dsub_rn(1.0, x.x);
        om[i][1] = __dsub_rn(1.0, x.y);
    }
    const double2 pj = *reinterpret_cast<const double2 *>(rows + D * kRow + 2 * lane);
    double p0[2] = {__dsub_rn(1.0, pj.x), __dsub_rn(1.0, pj.y)};
    double p1[2] = {pj.x, pj.y};
    uint32_t slow = 0;
#pragma unroll
    for (int k = 0; k < D; k++) {
        if constexpr (WRITE_Q) {
            double out[2];
            bool all_ok = true;
#pragma unroll
            for (int v = 0; v < 2; v++) {
                double q0 = p0[v], q1 = p1[v];
#pragma unroll
                for (int i = k + 1; i < D; i++) {
                    q0 = __dmul_rn(q0, om[i][v]);
                    q1 = __dmul_rn(q1, r[i][v]);
                }
                bool ok;
                out[v] = ddiv_fast(q1, __dadd_rn(q0, q1), ok);  // den == 0 -> !ok
                all_ok = all_ok && ok;
            }
            if (all_ok) st_cs2(a.msg + cofs(a.msg_rows, ids[k], ch * 64 + 2 * lane), out[0], out[1]);
            else slow |= 1u << k;
        }
#pragma unroll
        for (int v = 0; v < 2; v++) {
            p0[v] = __dmul_rn(p0[v], om[k][v]);
            p1[v] = __dmul_rn(p1[v], r[k][v]);
        }
    }
    if constexpr (WRITE_Q) {
        if (slow) {  // rare: tiny or zero denominators -> reference-order recompute, library division
            const double pv[2] = {pj.x, pj.y};
#pragma unroll
            for (int k = 0; k < D; k++) {
                if (!((slow >> k) & 1u)) continue;
                double out[2];
#pragma unroll
                for (int v = 0; v < 2; v++) {
                    double q0 = __dsub_rn(1.0, pv[v]), q1 = pv[v];
#pragma unroll
                    for (int i = 0; i < D; i++) {
                        if (i == k) continue;
                        q0 = __dmul_rn(q0, om[i][v]);
                        q1 = __dmul_rn(q1, r[i][v]);
                    }
                    const double den = __dadd_rn(q0, q1);
                    out[v] = (den == 0.0) ? 0.5 : __ddiv_rn(q1, den);
                }
                st_cs2(a.msg + cofs(a.msg_rows, ids[k], ch * 64 + 2 * lane), out[0], out[1]);
            }
        }
    }
    // estimate (serial.py:132): bit = !(Q0 > Q1); two ballots -> natural codeword order
    const uint32_t even = __ballot_sync(0xffffffffu, !(p0[0] > p1[0]));
    const uint32_t odd = __ballot_sync(0xffffffffu, !(p0[1] > p1[1]));
    if (lane == 0) {
        uint32_t lo = part1by1(even) | (part1by1(odd) << 1);
        uint32_t hi = part1by1(even >> 16) | (part1by1(odd >> 16) << 1);
        uint32_t *dst = a.chat + (size_t)ids[D] * a.NW + 2 * ch;
        if (a.done != nullptr) {
            const uint32_t d0 = a.done[2 * ch], d1 = a.done[2 * ch + 1];
            if (d0) lo = (lo & ~d0) | (dst[0] & d0);
            if (d1) hi = (hi & ~d1) | (dst[1] & d1);
        }
        *reinterpret_cast<uint2 *>(dst) = make_uint2(lo, hi);
    }
}

template <int D, bool IS_VAR, bool FLAG>  // FLAG: FROM_PRIOR for checks, WRITE_Q for variables
__global__ void __launch_bounds__(kThreads, 2) k_node_ring(NodeLaunch a, int64_t ntasks) {
    constexpr int ROWS = D + (IS_VAR ? 1 : 0);
    constexpr bool FP = !IS_VAR && FLAG;
    using R = Ring<ROWS>;
    constexpr int S = R::S;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int *ids = reinterpret_cast<int *>(smem + (size_t)warp * R::kBytes);  // [S][32]
    double *rows = reinterpret_cast<double *>(smem + (size_t)warp * R::kBytes + R::kIdsBytes);  // [S][ROWS][64]
    const int64_t W = (int64_t)gridDim.x * kWarpsPerBlock;
    const int64_t first = (int64_t)blockIdx.x * kWarpsPerBlock + warp;

    // prologue: ids of the first task, then copies of tasks 0..S-2 (one commit group per task)
    int nid = first < ntasks ? load_id<D, IS_VAR, FP>(a, first, lane) : 0;
    for (int s = 0; s < S - 1; s++) {
        const int64_t t = first + s * W;
        const int id = nid;
        if (t + W < ntasks) nid = load_id<D, IS_VAR, FP>(a, t + W, lane);
        if (t < ntasks) issue<D, IS_VAR, FP>(a, rows + (size_t)s * ROWS * kRow, ids + s * 32, t, id, lane);
        cp_commit();
    }
    int it = 0;
    for (int64_t t = first; t < ntasks; t += W, it++) {
        // keep S-1 tasks in flight: issue task t + (S-1) W into the stage freed last iteration
        const int64_t tn = t + (int64_t)(S - 1) * W;
        const int sn = (it + S - 1) % S;
        const int id = nid;
        if (tn + W < ntasks) nid = load_id<D, IS_VAR, FP>(a, tn + W, lane);
        if (tn < ntasks) issue<D, IS_VAR, FP>(a, rows + (size_t)sn * ROWS * kRow, ids + sn * 32, tn, id, lane);
        cp_commit();
        cp_wait<S - 1>();  // this lane's copies of task t have landed
        __syncwarp();      // row ids of task t (written by their lanes) are visible
        const int s = it % S;
        const int ch = (int)(t / a.node_count);
        if (!chunk64_done(a.done, ch)) {
            if constexpr (IS_VAR) compute_var<D, FLAG>(a, rows + (size_t)s * ROWS * kRow, ids + s * 32, ch, lane);
            else compute_check<D>(a, rows + (size_t)s * ROWS * kRow, ids + s * 32, ch, lane);
        }
        __syncwarp();  // stage s is reused by the issue of the next iteration
    }
    cp_wait<0>();
}

template <int D, bool IS_VAR, bool FLAG>
int launch_ring(const NodeLaunch &a, cudaStream_t st) {
    constexpr int ROWS = D + (IS_VAR ? 1 : 0);
    const size_t smem = (size_t)kWarpsPerBlock * Ring<ROWS>::kBytes;
    auto kern = k_node_ring<D, IS_VAR, FLAG>;
    static int per_sm = -1, sms = 0;
    static std::mutex mu;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (per_sm < 0) {
            LDPC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            int dev = 0;
            LDPC_CUDA_TRY(cudaGetDevice(&dev));
            LDPC_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            int b = 0;
            LDPC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kThreads, smem));
            if (b < 1) {
                set_error("ring node kernel (degree %d) does not fit on an SM", D);
                return LDPC_ECUDA;
            }
            per_sm = b;
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
    case D: return from_prior ? launch_ring<D, false, true>(a, s) : launch_ring<D, false, false>(a, s);
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
        CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
        default:
            set_error("ring check degree %d out of range", deg);
            return LDPC_EINVAL;
    }
}

int launch_var_pipe(const NodeLaunch &a, int deg, bool write_q, cudaStream_t s) {
    switch (deg) {
#define CASE(D) \
    case D: return write_q ? launch_ring<D, true, true>(a, s) : launch_ring<D, true, false>(a, s);
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
        CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
        default:
            set_error("ring variable degree %d out of range", deg);
            return LDPC_EINVAL;
    }
}

}  // namespace ldpc
