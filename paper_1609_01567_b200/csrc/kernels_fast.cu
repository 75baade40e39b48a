// kernels_fast.cu -- f4: fp32 fast mode.
//
// The same algorithm as the exact kernels -- probability-domain messages, the
// reference's left-to-right product order (serial.py:63-133), prefix sharing,
// the den == 0 -> 1/2 and tie -> 1 rules -- evaluated in IEEE fp32 (round to
// nearest, no FMA contraction; the division is the 2-ulp approximate one for normal
// denominators).  Messages take 4 bytes, so the HBM roofline doubles.  Results are NOT bit-identical to the fp64 reference:
// the tolerance (message LLR error and hard-decision agreement) is measured in
// tests/test_fast_gpu.py and stated in DESIGN.md.
//
// Layout: msg32[Bp/64][E][64] and P32[Bp/64][n][64] fp32 (chunk-major like the
// exact path); a warp handles one node x 64 codewords, lane = 2 codewords
// (8-byte float2 accesses, one contiguous 256-byte run per edge).
#include "common.cuh"

namespace ldpc {
namespace {

// fp32 mode keeps evict-first hints and a forward sweep (measured faster than default caching
// with the alternating sweep the fp64 kernels use: 7.9 vs 7.7-7.8 Gbit/s)
__device__ __forceinline__ float2 ld2(const float *p) { return __ldcs(reinterpret_cast<const float2 *>(p)); }
__device__ __forceinline__ void st2(float *p, float x, float y) {
    __stcs(reinterpret_cast<float2 *>(p), make_float2(x, y));
}

// q = q1 / den in the fast mode: the approximate division (2 ulp) for normal denominators; the
// IEEE division (with its slow path) only for subnormal ones; den == 0 -> 1/2 (serial.py:86-88)
__device__ __forceinline__ float fdiv_msg(float q1, float den) {
    if (den >= 1.17549435e-38f) return __fdividef(q1, den);
    return den == 0.0f ? 0.5f : __fdiv_rn(q1, den);
}

template <int D, bool FROM_PRIOR>
__global__ void __launch_bounds__(kThreads) k_check_f32(NodeLaunch a, float *msg, const float *P) {
    const int lane = threadIdx.x & 31;
    // grid (node blocks, codeword chunks), dispatched x-fastest: chunk-major sweep
    const int nch = active_chunks(a, (int)gridDim.y, 64);
    if ((int)blockIdx.y >= nch) return;
    const int ch = a.reverse ? nch - 1 - (int)blockIdx.y : (int)blockIdx.y;
    const int ni = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (ni >= a.node_count) return;
    if (a.done != nullptr) {
        const uint2 d = *reinterpret_cast<const uint2 *>(a.done + 2 * ch);
        if ((d.x & d.y) == 0xffffffffu) return;
    }
    float *mb = chunk_base(msg, a.msg_rows, ch * 64) + 2 * lane;
    const float *pb = chunk_base(P, a.p_rows, ch * 64) + 2 * lane;
    const int32_t base = a.edge_begin + ni * D;
    int slot[D];
#pragma unroll
    for (int i = 0; i < D; i++) slot[i] = __ldg(a.slot_ord + base + i);
    float b[D][2];
#pragma unroll
    for (int i = 0; i < D; i++) {
        const float2 q = FROM_PRIOR ? *reinterpret_cast<const float2 *>(pb + row_off(__ldg(a.var_ord + base + i)))
                                    : ld2(mb + row_off(slot[i]));
        b[i][0] = __fsub_rn(1.0f, __fmul_rn(2.0f, q.x));
        b[i][1] = __fsub_rn(1.0f, __fmul_rn(2.0f, q.y));
    }
    float pre0 = 1.0f, pre1 = 1.0f;
#pragma unroll
    for (int k = 0; k < D; k++) {
        float a0 = pre0, a1 = pre1;
#pragma unroll
        for (int i = k + 1; i < D; i++) {
            a0 = __fmul_rn(a0, b[i][0]);
            a1 = __fmul_rn(a1, b[i][1]);
        }
        st2(mb + row_off(slot[k]), __fsub_rn(1.0f, __fadd_rn(0.5f, __fmul_rn(0.5f, a0))),
            __fsub_rn(1.0f, __fadd_rn(0.5f, __fmul_rn(0.5f, a1))));
        if (k + 1 < D) {
            pre0 = __fmul_rn(pre0, b[k][0]);
            pre1 = __fmul_rn(pre1, b[k][1]);
        }
    }
}

template <int D, bool WRITE_Q>
__global__ void __launch_bounds__(kThreads) k_var_f32(NodeLaunch a, float *msg, const float *P) {
    const int lane = threadIdx.x & 31;
    // grid (node blocks, codeword chunks), dispatched x-fastest: chunk-major sweep
    const int nch = active_chunks(a, (int)gridDim.y, 64);
    if ((int)blockIdx.y >= nch) return;
    const int ch = a.reverse ? nch - 1 - (int)blockIdx.y : (int)blockIdx.y;
    const int ni = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (ni >= a.node_count) return;
    if (a.done != nullptr) {
        const uint2 d = *reinterpret_cast<const uint2 *>(a.done + 2 * ch);
        if ((d.x & d.y) == 0xffffffffu) return;
    }
    float *mb = chunk_base(msg, a.msg_rows, ch * 64) + 2 * lane;
    const float *pb = chunk_base(P, a.p_rows, ch * 64) + 2 * lane;
    const int node = __ldg(a.order + a.node_begin + ni);
    const int32_t base = a.edge_begin + ni * D;
    int pos[D];
#pragma unroll
    for (int i = 0; i < D; i++) pos[i] = __ldg(a.slot_ord + base + i);
    const float2 pj = *reinterpret_cast<const float2 *>(pb + row_off(node));
    float r[D][2], om[D][2];
#pragma unroll
    for (int i = 0; i < D; i++) {
        const float2 x = ld2(mb + row_off(pos[i]));
        r[i][0] = x.x;
        r[i][1] = x.y;
        om[i][0] = __fsub_rn(1.0f, x.x);
        om[i][1] = __fsub_rn(1.0f, x.y);
    }
    float p0[2] = {__fsub_rn(1.0f, pj.x), __fsub_rn(1.0f, pj.y)};
    float p1[2] = {pj.x, pj.y};
#pragma unroll
    for (int k = 0; k < D; k++) {
        if constexpr (WRITE_Q) {
            float out[2];
#pragma unroll
            for (int v = 0; v < 2; v++) {
                float q0 = p0[v], q1 = p1[v];
#pragma unroll
                for (int i = k + 1; i < D; i++) {
                    q0 = __fmul_rn(q0, om[i][v]);
                    q1 = __fmul_rn(q1, r[i][v]);
                }
                out[v] = fdiv_msg(q1, __fadd_rn(q0, q1));
            }
            st2(mb + row_off(pos[k]), out[0], out[1]);
        }
#pragma unroll
        for (int v = 0; v < 2; v++) {
            p0[v] = __fmul_rn(p0[v], om[k][v]);
            p1[v] = __fmul_rn(p1[v], r[k][v]);
        }
    }
    const uint32_t even = __ballot_sync(0xffffffffu, !(p0[0] > p1[0]));
    const uint32_t odd = __ballot_sync(0xffffffffu, !(p0[1] > p1[1]));
    if (lane == 0) {
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

// fp64 priors [Bp/64][n][64] -> fp32 [Bp/64][n][64] (round to nearest)
__global__ void k_priors_to_f32(const double *P, float *P32, size_t count) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < count; k += (size_t)gridDim.x * blockDim.x)
        P32[k] = __double2float_rn(P[k]);
}

__global__ void k_canon_to_slots_f32(const int32_t *var_slot, int64_t E, const double *src, int32_t B, float *msg,
                                     int32_t Bp) {
    const int64_t total = E * Bp;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = k / Bp;
        const int c = (int)(k - e * Bp);
        const int32_t slot = var_slot ? var_slot[e] : (int32_t)e;
        msg[cofs((int32_t)E, slot, c)] = (c < B) ? __double2float_rn(src[(size_t)c * E + e]) : 0.5f;
    }
}

__global__ void k_slots_to_canon_f32(const int32_t *var_slot, int64_t E, const float *msg, int32_t Bp, double *dst,
                                     int32_t B) {
    const int64_t total = E * B;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(k / E);
        const int64_t e = k - (int64_t)c * E;
        const int32_t slot = var_slot ? var_slot[e] : (int32_t)e;
        dst[k] = (double)msg[cofs((int32_t)E, slot, c)];
    }
}

unsigned grid_of(int64_t work) {
    int64_t b = (work + 255) / 256;
    return (unsigned)(b < 1 ? 1 : (b > 148 * 64 ? 148 * 64 : b));
}

template <int D, bool FLAG, bool IS_VAR>
int launch_f32(const NodeLaunch &a, float *msg, const float *P, cudaStream_t s) {
    if (a.node_count == 0) return LDPC_OK;
    const dim3 grid((a.node_count + kWarpsPerBlock - 1) / kWarpsPerBlock, a.Bp / 64);
    LDPC_ARG_CHECK(grid.y <= 65535u, "batch too large for one launch (%d codewords)", a.Bp);
    if constexpr (IS_VAR) k_var_f32<D, FLAG><<<grid, kThreads, 0, s>>>(a, msg, P);
    else k_check_f32<D, FLAG><<<grid, kThreads, 0, s>>>(a, msg, P);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

}  // namespace

int launch_check_f32(const NodeLaunch &a, int deg, bool from_prior, float *msg, const float *P, cudaStream_t s) {
    switch (deg) {
#define CASE(D) \
    case D: return from_prior ? launch_f32<D, true, false>(a, msg, P, s) : launch_f32<D, false, false>(a, msg, P, s);
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
        CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
        default:
            set_error("fp32 fast mode supports node degrees up to %d (check degree %d)", kMaxRegDegree, deg);
            return LDPC_EINVAL;
    }
}

int launch_var_f32(const NodeLaunch &a, int deg, bool write_q, float *msg, const float *P, cudaStream_t s) {
    switch (deg) {
#define CASE(D) \
    case D: return write_q ? launch_f32<D, true, true>(a, msg, P, s) : launch_f32<D, false, true>(a, msg, P, s);
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
        CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
        default:
            set_error("fp32 fast mode supports node degrees up to %d (variable degree %d)", kMaxRegDegree, deg);
            return LDPC_EINVAL;
    }
}

int launch_canon_to_slots_f32(const ldpc_graph *g, const double *src, int32_t B, float *msg, int32_t Bp,
                              cudaStream_t s) {
    k_canon_to_slots_f32<<<grid_of(g->E * Bp), 256, 0, s>>>(g->var_slot, g->E, src, B, msg, Bp);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

int launch_slots_to_canon_f32(const ldpc_graph *g, const float *msg, int32_t Bp, double *dst, int32_t B,
                              cudaStream_t s) {
    k_slots_to_canon_f32<<<grid_of(g->E * B), 256, 0, s>>>(g->var_slot, g->E, msg, Bp, dst, B);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

int launch_priors_to_f32(const double *P, float *P32, size_t count, cudaStream_t s) {
    size_t blocks = (count + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    k_priors_to_f32<<<(unsigned)blocks, 256, 0, s>>>(P, P32, count);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

}  // namespace ldpc
