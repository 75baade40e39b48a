// kernels_varmid.cu -- variable nodes of degree 17..64 (e.g. the heavy columns of 5G-NR-like
// codes) and check nodes of degree 33..64: the register kernels' data movement with the
// arithmetic read from shared memory.
//
// Past degree 16, holding r and 1-r of every edge in registers (the register / ring kernels)
// needs ~255 registers, and the block-per-(node, tile) chains kernels are issue-bound at these
// degrees.  Here a warp takes (variable, 32 codewords), lane = codeword, as the register
// kernels do: its d message rows (256 bytes each) are copied with cp.async into the warp's
// shared memory (all in flight at once, no register destination), then each lane computes
// its codeword's d outputs in groups of G from its shared-memory column:
//   output k = k0 + j of group k0: (1-p) (1-r_0)...(1-r_{k-1}) [running prefix]
//              * (1-r_{k+1}) ... (1-r_{k0+G-1})                  [head, inside the group]
//              * (1-r_{k0+G}) ... (1-r_{d-1})                     [body, shared loads]
// (and the same with p, r_i), i.e. the reference's left-to-right products skipping edge k
// (serial.py:77-88), one rounding per operation; q = q1 / (q0 + q1) by the exact division of
// common.cuh, 0.5 when the denominator is zero.  The full prefix is the estimate's
// (Q0, Q1) (serial.py:125-132).
#include "common.cuh"

namespace ldpc {
namespace {

constexpr int kMidG = 8;    // outputs per group (chains per lane), variables
constexpr int kMidGC = 16;  // checks (one chain per output: twice the outputs for the same registers)
// per-warp stage of MAXD rows x 256 bytes; 8 warps per block up to degree 32 (64 KB), 4 past it
template <int MAXD>
constexpr int mid_warps() { return MAXD <= 32 ? 8 : 4; }

template <bool WRITE_Q, bool EARLY, int MAXD>
__global__ void __launch_bounds__(32 * mid_warps<MAXD>()) k_var_mid(NodeLaunch a, int D) {
    constexpr int kMidWarps = mid_warps<MAXD>();
    extern __shared__ __align__(16) double mid_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nch = active_chunks(a, (int)gridDim.y, 32);
    if ((int)blockIdx.y >= nch) return;
    const int ch = a.reverse ? nch - 1 - (int)blockIdx.y : (int)blockIdx.y;
    const int ni = blockIdx.x * kMidWarps + warp;
    if (ni >= a.node_count) return;
    uint32_t dmask = 0;
    if constexpr (EARLY) {
        dmask = a.done[ch];
        if (dmask == 0xffffffffu) return;
    }
    double *rows = mid_smem + (size_t)warp * MAXD * 32;  // [D][32]: row i, column = codeword
    const int cw0 = ch * 32;
    const int node = __ldg(a.order + a.node_begin + ni);
    // slot of edge i: lane i (< 32) holds id0, lane i - 32 holds id1 (degrees past 32)
    const int32_t *sl = a.slot_ord + a.edge_begin + ni * D;
    const int id0 = lane < D ? __ldg(sl + lane) : 0;
    const int id1 = (MAXD > 32 && lane + 32 < D) ? __ldg(sl + lane + 32) : 0;
    auto slot_of = [&](int i) {  // every lane calls it (shuffles); i may differ per lane
        const int x0 = __shfl_sync(0xffffffffu, id0, i & 31);
        if constexpr (MAXD <= 32) return x0;
        const int x1 = __shfl_sync(0xffffffffu, id1, i & 31);
        return i < 32 ? x0 : x1;
    };
    const double *mb_src = chunk_base(a.msg, a.msg_rows, cw0);
    // row i (32 doubles = 256 bytes) is 16 pieces of 16 bytes: lanes 0-15 copy row 2j, 16-31 row 2j+1
    const int sub = lane >> 4, piece = lane & 15;
    for (int j = 0; j < (D + 1) / 2; j++) {
        const int r = 2 * j + sub;
        const int src = slot_of(r < D ? r : D - 1);
        if (r < D) cp_async16(rows + r * 32 + 2 * piece, mb_src + row_off(src) + 2 * piece);
    }
    cp_commit();
    const double pj = __ldg(chunk_base(a.P, a.p_rows, cw0) + lane + row_off(node));
    cp_wait<0>();
    __syncwarp();
    const double *col = rows + lane;
    double *mb = chunk_base(a.msg, a.msg_rows, cw0) + lane;
    double p0 = __dsub_rn(1.0, pj), p1 = pj;  // running prefix over positions < k0
    for (int k0 = 0; k0 < D; k0 += kMidG) {
        double a0[kMidG], a1[kMidG];
        double q0 = p0, q1 = p1;
#pragma unroll
        for (int j = 0; j < kMidG; j++) {
            a0[j] = q0;
            a1[j] = q1;
            if (k0 + j < D) {
                const double r = col[(k0 + j) * 32];
                q0 = __dmul_rn(q0, __dsub_rn(1.0, r));
                q1 = __dmul_rn(q1, r);
            }
        }
        p0 = q0;  // prefix through the group (the estimate's products at the end)
        p1 = q1;
        if (!WRITE_Q) continue;
#pragma unroll
        for (int jj = 1; jj < kMidG; jj++) {  // head: positions inside the group after each output
            if (k0 + jj < D) {
                const double r = col[(k0 + jj) * 32], om = __dsub_rn(1.0, r);
#pragma unroll
                for (int j = 0; j < jj; j++) {
                    a0[j] = __dmul_rn(a0[j], om);
                    a1[j] = __dmul_rn(a1[j], r);
                }
            }
        }
#pragma unroll 4
        for (int i = k0 + kMidG; i < D; i++) {  // body
            const double r = col[i * 32], om = __dsub_rn(1.0, r);
#pragma unroll
            for (int j = 0; j < kMidG; j++) {
                a0[j] = __dmul_rn(a0[j], om);
                a1[j] = __dmul_rn(a1[j], r);
            }
        }
#pragma unroll
        for (int j = 0; j < kMidG; j++) {
            const int k = k0 + j;
            const int slot = slot_of(k < D ? k : 0);
            if (k < D) {
                const double den = __dadd_rn(a0[j], a1[j]);
                bool ok;
                double q = ddiv_fast(a1[j], den, ok);
                if (!ok) q = (den == 0.0) ? 0.5 : __ddiv_rn(a1[j], den);
                st_msg(mb + row_off(slot), q);
            }
        }
    }
    // estimate (serial.py:132): bit = !(Q0 > Q1); bits of stopped codewords stay frozen
    uint32_t bits = __ballot_sync(0xffffffffu, !(p0 > p1));
    if (lane == 0) {
        uint32_t *dst = a.chat + (size_t)node * a.NW + ch;
        if (EARLY && dmask) bits = (bits & ~dmask) | (*dst & dmask);
        *dst = bits;
    }
}

// Checks of degree 33..64, same scheme (serial.py:92-112): b_i = 1 - 2 q_i staged per warp, then
// prod_k = 1 * b_0 ... b_{k-1} * b_{k+1} ... b_{d-1} in groups of G from shared memory and
// r_k = 1 - (0.5 + 0.5 prod_k) written back in place (every input is in shared memory first).
template <bool FROM_PRIOR, bool EARLY>
__global__ void __launch_bounds__(128) k_check_mid(NodeLaunch a, int D) {
    constexpr int MAXD = 64, kW = 4;
    extern __shared__ __align__(16) double mid_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nch = active_chunks(a, (int)gridDim.y, 32);
    if ((int)blockIdx.y >= nch) return;
    const int ch = a.reverse ? nch - 1 - (int)blockIdx.y : (int)blockIdx.y;
    const int ni = blockIdx.x * kW + warp;
    if (ni >= a.node_count) return;
    if (EARLY && a.done[ch] == 0xffffffffu) return;
    double *rows = mid_smem + (size_t)warp * MAXD * 32;
    const int cw0 = ch * 32;
    const int32_t *sl = a.slot_ord + a.edge_begin + ni * D;
    const int32_t *vr = a.var_ord + a.edge_begin + ni * D;
    const int id0 = lane < D ? __ldg(sl + lane) : 0, id1 = lane + 32 < D ? __ldg(sl + lane + 32) : 0;
    int src0 = 0, src1 = 0;  // input row ids: the message slots, or (pre-pass) the variables' prior rows
    if (FROM_PRIOR) {
        src0 = lane < D ? __ldg(vr + lane) : 0;
        src1 = lane + 32 < D ? __ldg(vr + lane + 32) : 0;
    }
    auto pick = [&](int x0, int x1, int i) {  // value of lane (i & 31) of x0 (i < 32) or x1
        const int v0 = __shfl_sync(0xffffffffu, x0, i & 31), v1 = __shfl_sync(0xffffffffu, x1, i & 31);
        return i < 32 ? v0 : v1;
    };
    const double *base = FROM_PRIOR ? chunk_base(a.P, a.p_rows, cw0) : chunk_base(a.msg, a.msg_rows, cw0);
    const int sub = lane >> 4, piece = lane & 15;
    for (int j = 0; j < (D + 1) / 2; j++) {
        const int r = 2 * j + sub, rr = r < D ? r : D - 1;
        const int src = FROM_PRIOR ? pick(src0, src1, rr) : pick(id0, id1, rr);
        if (r < D) cp_async16(rows + r * 32 + 2 * piece, base + row_off(src) + 2 * piece);
    }
    cp_commit();
    cp_wait<0>();
    __syncwarp();
    double *col = rows + lane;
    for (int i = 0; i < D; i++) col[i * 32] = __dsub_rn(1.0, __dmul_rn(2.0, col[i * 32]));
    double *mb = chunk_base(a.msg, a.msg_rows, cw0) + lane;
    double pre = 1.0;
    for (int k0 = 0; k0 < D; k0 += kMidGC) {
        double acc[kMidGC];
        double q = pre;
#pragma unroll
        for (int j = 0; j < kMidGC; j++) {
            acc[j] = q;
            if (k0 + j < D) q = __dmul_rn(q, col[(k0 + j) * 32]);
        }
        pre = q;
#pragma unroll
        for (int jj = 1; jj < kMidGC; jj++) {
            if (k0 + jj < D) {
                const double x = col[(k0 + jj) * 32];
#pragma unroll
                for (int j = 0; j < jj; j++) acc[j] = __dmul_rn(acc[j], x);
            }
        }
#pragma unroll 4
        for (int i = k0 + kMidGC; i < D; i++) {
            const double x = col[i * 32];
#pragma unroll
            for (int j = 0; j < kMidGC; j++) acc[j] = __dmul_rn(acc[j], x);
        }
#pragma unroll
        for (int j = 0; j < kMidGC; j++) {
            const int k = k0 + j;
            const int slot = pick(id0, id1, k < D ? k : 0);
            if (k < D) st_msg(mb + row_off(slot), __dsub_rn(1.0, __dadd_rn(0.5, __dmul_rn(0.5, acc[j]))));
        }
    }
}

template <bool FP, bool EARLY>
int launch_cmid(const NodeLaunch &a, int deg, cudaStream_t s) {
    const size_t smem = (size_t)4 * 64 * 32 * sizeof(double);
    auto kern = k_check_mid<FP, EARLY>;
    static bool attr[64] = {};
    int dev = 0;
    LDPC_CUDA_TRY(cudaGetDevice(&dev));
    LDPC_ARG_CHECK(dev >= 0 && dev < 64, "device ordinal %d out of range", dev);
    if (!attr[dev]) {
        LDPC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr[dev] = true;
    }
    const dim3 grid((a.node_count + 3) / 4, a.Bp / 32);
    LDPC_ARG_CHECK(grid.y <= 65535u, "batch too large for one launch (%d codewords)", a.Bp);
    kern<<<grid, 128, smem, s>>>(a, deg);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

template <bool WQ, bool EARLY, int MAXD>
int launch_mid(const NodeLaunch &a, int deg, cudaStream_t s) {
    constexpr int kMidWarps = mid_warps<MAXD>();
    const size_t smem = (size_t)kMidWarps * MAXD * 32 * sizeof(double);
    auto kern = k_var_mid<WQ, EARLY, MAXD>;
    static bool attr[64] = {};  // the shared-memory attribute is per device
    int dev = 0;
    LDPC_CUDA_TRY(cudaGetDevice(&dev));
    LDPC_ARG_CHECK(dev >= 0 && dev < 64, "device ordinal %d out of range", dev);
    if (!attr[dev]) {
        LDPC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr[dev] = true;
    }
    const dim3 grid((a.node_count + kMidWarps - 1) / kMidWarps, a.Bp / 32);
    LDPC_ARG_CHECK(grid.y <= 65535u, "batch too large for one launch (%d codewords)", a.Bp);
    kern<<<grid, 32 * kMidWarps, smem, s>>>(a, deg);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

}  // namespace

template <int MAXD>
int launch_mid_d(const NodeLaunch &a, int deg, bool write_q, cudaStream_t s) {
    if (a.done != nullptr)
        return write_q ? launch_mid<true, true, MAXD>(a, deg, s) : launch_mid<false, true, MAXD>(a, deg, s);
    return write_q ? launch_mid<true, false, MAXD>(a, deg, s) : launch_mid<false, false, MAXD>(a, deg, s);
}

int launch_check_mid(const NodeLaunch &a, int deg, bool from_prior, cudaStream_t s) {
    LDPC_ARG_CHECK(deg > 0 && deg <= kMaxMidCheckDegree, "mid-degree check kernel takes degrees up to %d",
                   kMaxMidCheckDegree);
    if (a.node_count == 0) return LDPC_OK;
    if (a.done != nullptr) return from_prior ? launch_cmid<true, true>(a, deg, s) : launch_cmid<false, true>(a, deg, s);
    return from_prior ? launch_cmid<true, false>(a, deg, s) : launch_cmid<false, false>(a, deg, s);
}

int launch_var_mid(const NodeLaunch &a, int deg, bool write_q, cudaStream_t s) {
    LDPC_ARG_CHECK(deg > 0 && deg <= kMaxMidVarDegree, "mid-degree variable kernel takes degrees up to %d",
                   kMaxMidVarDegree);
    if (a.node_count == 0) return LDPC_OK;
    return deg <= 32 ? launch_mid_d<32>(a, deg, write_q, s) : launch_mid_d<64>(a, deg, write_q, s);
}

}  // namespace ldpc
