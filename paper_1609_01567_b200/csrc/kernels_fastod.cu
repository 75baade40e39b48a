// kernels_fastod.cu -- f4 fast mode, O(d) per node for ANY degree.
//
// The exact kernels carry the reference's ordered products (serial.py:63-112):
// d(d-1)/2 multiplies per node and codeword, which at degree 1000 is the whole
// cost of a decode.  The fast mode drops the order and the fp64 width:
//
//   check (serial.py:92-112 restated):  b_i = 1 - 2 q_i   (= -tanh(L_i / 2))
//       prod_k = (prefix product of b before k) * (suffix product after k)
//       r_k    = 1 - (0.5 + 0.5 * prod_k)                 (the reference's formula, fp32)
//   variable (serial.py:63-89 / 115-133 restated in the log domain):
//       l_i = log2 r_i - log2 (1 - r_i),   Lp = log2 p - log2 (1 - p)
//       L   = Lp + sum_i l_i;  q_k = 1 / (1 + 2^-(L - l_k));  c_hat = (L >= 0)  (tie -> 1)
//
// so a node costs O(d) and no degree is special.  Products are prefix x suffix
// (no division, so a zero factor is harmless); the variable side sums logarithms
// (no underflow at any degree, where fp32 products of 200 factors < 1 would
// vanish); the log-ratios are clamped to +-kL2Clamp so saturated messages (r = 0
// or 1 exactly) stay finite.  NOT bit-exact: tolerance vs the oracle is stated in
// DESIGN.md and tested in tests/test_fast_gpu.py.
//
// Work mapping: one block per task (node, tile of 32 codewords), lane = codeword
// (one 128-byte line per row and warp), warp w = a segment of <= kOdSeg rows held
// in registers.  A block of W warps covers kOdSeg*W rows per pass; the segment
// totals are exchanged through shared memory (exclusive prefix/suffix across
// warps), then each thread walks its segment backward (suffixes) and forward
// (outputs).  Nodes longer than one pass (d > 512) take two passes over their
// rows: pass A stores the pass totals in a per-block scratch slice (checks) or
// accumulates the log-sum (variables), pass B writes the outputs.
// Layout: fp32 messages msg32[Bp/64][E][64], priors P32[Bp/64][n][64] (kernels_fast.cu).
#include <algorithm>

#include "common.cuh"

namespace ldpc {
namespace {

constexpr int kOdSeg = 16;                       // rows per thread and pass (registers)
constexpr int kOdMaxWarps = 32;
constexpr int kOdPass = kOdSeg * kOdMaxWarps;    // rows per block pass at 32 warps
constexpr float kL2Clamp = 1000.0f;              // |log2 ratio| cap (2^-1000: certainty)

__device__ __forceinline__ float lg2(float x) {
    float y;
    asm("lg2.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float log_ratio(float r) {  // log2(r / (1 - r)), clamped
    const float l = __fsub_rn(lg2(r), lg2(__fsub_rn(1.0f, r)));
    return fminf(fmaxf(l, -kL2Clamp), kL2Clamp);        // (NaN only for NaN input)
}

// row address of position k of the node (slot map or identity)
__device__ __forceinline__ uint32_t slot_of(const NodeLaunch &a, int pos) {
    return row_off(a.slot ? __ldg(a.slot + pos) : pos);
}

// Task t of a side's launch: largest degree first, all tiles of a node together (lpt_block)
struct OdTask {
    int tile, ni;
};
__device__ __forceinline__ OdTask od_task(int64_t t, int node_count, int tiles) {
    OdTask o;
    lpt_block((int)t, node_count, tiles, o.ni, o.tile);
    return o;
}

// Rows [lo, hi) of one pass, split over W warps: warp w owns [lo + w*seg, ...)
struct Seg {
    int r0, cnt;
};
__device__ __forceinline__ Seg seg_of(int lo, int hi, int W, int w) {
    const int seg = (hi - lo + W - 1) / W;
    Seg s;
    s.r0 = lo + w * seg;
    s.cnt = max(0, min(seg, hi - s.r0));
    return s;
}

template <bool FROM_PRIOR>
__device__ __forceinline__ float check_input(const NodeLaunch &a, const float *mb, const float *pb, int pos) {
    // b = 1 - 2q; the pre-pass reads q = p[v-bar] (serial.py:58,166)
    const float q = FROM_PRIOR ? __ldg(pb + row_off(__ldg(a.idx + pos))) : __ldcs(mb + slot_of(a, pos));
    return __fsub_rn(1.0f, __fmul_rn(2.0f, q));
}

// products of the W warp totals before / after warp w (fixed order: deterministic)
__device__ __forceinline__ void cross_warp_products(const float *tot, int W, int w, int lane, float &before,
                                                    float &after, float &all) {
    before = 1.0f;
    after = 1.0f;
    for (int x = 0; x < W; x++) {
        const float t = tot[x * 32 + lane];
        if (x < w) before = __fmul_rn(before, t);
        if (x > w) after = __fmul_rn(after, t);
    }
    all = __fmul_rn(__fmul_rn(before, tot[w * 32 + lane]), after);
}

template <bool FROM_PRIOR>
__global__ void __launch_bounds__(1024) k_check_f32_od(NodeLaunch a, float *msg, const float *P, float *scratch,
                                                       int scratch_stride, int64_t ntasks) {
    __shared__ float tot[kOdMaxWarps * 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
    float *sc = scratch ? scratch + (size_t)blockIdx.x * scratch_stride : nullptr;  // [J][32] pass totals
    for (int64_t t = blockIdx.x; t < ntasks; t += gridDim.x) {
        const OdTask tk = od_task(t, a.node_count, a.Bp / 32);
        if (a.done != nullptr && a.done[tk.tile] == 0xffffffffu) continue;  // uniform per block
        const int node = __ldg(a.order + a.node_begin + tk.ni);
        const int pos0 = __ldg(a.off + node), d = __ldg(a.off + node + 1) - pos0;
        float *mb = chunk_base(msg, a.msg_rows, tk.tile * 32) + lane;
        const float *pb = chunk_base(P, a.p_rows, tk.tile * 32) + lane;
        const int pass_rows = kOdSeg * W;
        const int J = (d + pass_rows - 1) / pass_rows;
        if (J > 1) {
            // pass A: the product of every pass, then (warp 0) suffix products over passes in place
            for (int j = 0; j < J; j++) {
                const Seg s = seg_of(j * pass_rows, min(d, (j + 1) * pass_rows), W, w);
                float p = 1.0f;
                for (int i = 0; i < s.cnt; i++) p = __fmul_rn(p, check_input<FROM_PRIOR>(a, mb, pb, pos0 + s.r0 + i));
                tot[w * 32 + lane] = p;
                __syncthreads();
                if (w == 0) {
                    float all = 1.0f;
                    for (int x = 0; x < W; x++) all = __fmul_rn(all, tot[x * 32 + lane]);
                    sc[j * 32 + lane] = all;
                }
                __syncthreads();
            }
            if (w == 0) {
                float run = 1.0f;
                for (int j = J - 1; j >= 0; j--) {
                    const float x = sc[j * 32 + lane];
                    sc[j * 32 + lane] = run;  // product of the passes after j
                    run = __fmul_rn(run, x);
                }
            }
            __syncthreads();
        }
        float carry = 1.0f;  // product of the passes before j
        for (int j = 0; j < J; j++) {
            const Seg s = seg_of(j * pass_rows, min(d, (j + 1) * pass_rows), W, w);
            float b[kOdSeg];
#pragma unroll
            for (int i = 0; i < kOdSeg; i++)
                b[i] = i < s.cnt ? check_input<FROM_PRIOR>(a, mb, pb, pos0 + s.r0 + i) : 1.0f;
            float p = 1.0f;
#pragma unroll
            for (int i = 0; i < kOdSeg; i++) p = __fmul_rn(p, b[i]);
            tot[w * 32 + lane] = p;
            __syncthreads();
            float before, after, all;
            cross_warp_products(tot, W, w, lane, before, after, all);
            const float F = J > 1 ? __fmul_rn(after, sc[j * 32 + lane]) : after;
            float suf[kOdSeg];
            float run = F;
#pragma unroll
            for (int i = kOdSeg - 1; i >= 0; i--) {
                suf[i] = run;
                run = __fmul_rn(run, b[i]);
            }
            float pre = __fmul_rn(carry, before);
#pragma unroll
            for (int i = 0; i < kOdSeg; i++) {
                if (i < s.cnt) {
                    const float prod = __fmul_rn(pre, suf[i]);
                    __stcs(mb + slot_of(a, pos0 + s.r0 + i), __fsub_rn(1.0f, __fadd_rn(0.5f, __fmul_rn(0.5f, prod))));
                }
                pre = __fmul_rn(pre, b[i]);
            }
            carry = __fmul_rn(carry, all);
            __syncthreads();  // tot is rewritten by the next pass / task
        }
    }
}

template <bool WRITE_Q>
__global__ void __launch_bounds__(1024) k_var_f32_od(NodeLaunch a, float *msg, int64_t ntasks) {
    __shared__ float tot[kOdMaxWarps * 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
    for (int64_t t = blockIdx.x; t < ntasks; t += gridDim.x) {
        const OdTask tk = od_task(t, a.node_count, a.Bp / 32);
        const uint32_t done = a.done != nullptr ? a.done[tk.tile] : 0u;
        if (done == 0xffffffffu) continue;
        const int node = __ldg(a.order + a.node_begin + tk.ni);
        const int pos0 = __ldg(a.off + node), d = __ldg(a.off + node + 1) - pos0;
        float *mb = chunk_base(msg, a.msg_rows, tk.tile * 32) + lane;
        // prior log-ratio from the fp64 prior (one per node and codeword)
        const double pj = __ldg(chunk_base(a.P, a.p_rows, tk.tile * 32) + lane + row_off(node));
        const float Lp = fminf(fmaxf((float)(log2(pj) - log2(1.0 - pj)), -kL2Clamp), kL2Clamp);
        const int pass_rows = kOdSeg * W;
        const int J = (d + pass_rows - 1) / pass_rows;
        float part = 0.0f;  // this thread's log-ratio sum over all passes
        float l[kOdSeg];
        for (int j = 0; j < J; j++) {
            const Seg s = seg_of(j * pass_rows, min(d, (j + 1) * pass_rows), W, w);
#pragma unroll
            for (int i = 0; i < kOdSeg; i++) {
                l[i] = i < s.cnt ? log_ratio(__ldcs(mb + slot_of(a, pos0 + s.r0 + i))) : 0.0f;
                part = __fadd_rn(part, l[i]);
            }
        }
        tot[w * 32 + lane] = part;
        __syncthreads();
        float L = Lp;
        for (int x = 0; x < W; x++) L = __fadd_rn(L, tot[x * 32 + lane]);
        if (w == 0) {
            // estimate (serial.py:132): c = !(Q0 > Q1)  <=>  log2(Q1/Q0) = L >= 0
            uint32_t bits = __ballot_sync(0xffffffffu, L >= 0.0f);
            if (lane == 0) {
                uint32_t *dst = a.chat + (size_t)node * a.NW + tk.tile;
                if (done) bits = (bits & ~done) | (*dst & done);  // stopped codewords keep their bits
                *dst = bits;
            }
        }
        if constexpr (WRITE_Q) {
            for (int j = J - 1; j >= 0; j--) {  // the last pass's log-ratios are still in registers
                const Seg s = seg_of(j * pass_rows, min(d, (j + 1) * pass_rows), W, w);
                if (j != J - 1) {
#pragma unroll
                    for (int i = 0; i < kOdSeg; i++)
                        l[i] = i < s.cnt ? log_ratio(__ldcs(mb + slot_of(a, pos0 + s.r0 + i))) : 0.0f;
                }
#pragma unroll
                for (int i = 0; i < kOdSeg; i++) {
                    if (i < s.cnt) {
                        const float x = __fsub_rn(L, l[i]);
                        __stcs(mb + slot_of(a, pos0 + s.r0 + i), __fdividef(1.0f, __fadd_rn(1.0f, ex2(-x))));
                    }
                }
            }
        }
        __syncthreads();  // tot is rewritten by the next task
    }
}

// warps per block for a bucket range whose largest degree is dmax: enough for kOdSeg rows per
// warp in one pass, rounded up to a power of two (<= 2x idle), capped at 32 (then 2+ passes)
int od_warps(int dmax) {
    const int need = (std::min(dmax, kOdPass) + kOdSeg - 1) / kOdSeg;
    int W = 1;
    while (W < need) W <<= 1;
    return W;
}

}  // namespace

int fast_od_scratch_stride(const ldpc_graph *g) {
    const int J = (g->max_dc + kOdPass - 1) / kOdPass;
    return J > 1 ? J * 32 : 0;
}

// The buckets of degree >= min_deg grouped into launches by warps per block (buckets are sorted by
// degree, so a class is a contiguous node range).
std::vector<OdClass> fast_od_classes(const std::vector<Bucket> &buckets, int min_deg) {
    std::vector<OdClass> out;
    size_t i = 0;
    while (i < buckets.size()) {
        if (buckets[i].deg < min_deg || buckets[i].node_count == 0) {
            i++;
            continue;
        }
        const int W = od_warps(buckets[i].deg);
        OdClass c{buckets[i].node_begin, 0, W, 0, 0};
        size_t k = i;
        while (k < buckets.size() && od_warps(buckets[k].deg) == W) {
            c.dmax = std::max(c.dmax, buckets[k].deg);
            c.edges += (int64_t)buckets[k].node_count * buckets[k].deg;
            k++;
        }
        c.node_count = buckets[k - 1].node_begin + buckets[k - 1].node_count - c.node_begin;
        out.push_back(c);
        i = k;
    }
    return out;
}

// One class.  Checks longer than one pass keep their pass totals in scratch: scratch_blocks slices
// of scratch_stride floats (fast_od_scratch_stride), one per resident block of the launch.
int launch_fast_od_class(const NodeLaunch &base, const OdClass &c, bool var_side, bool flag, float *msg,
                         const float *P, float *scratch, int scratch_stride, int scratch_blocks, cudaStream_t s) {
    NodeLaunch a = base;
    a.node_begin = c.node_begin;
    a.node_count = c.node_count;
    const int W = c.warps;
    const int64_t ntasks = (int64_t)a.node_count * (base.Bp / 32);
    if (ntasks == 0) return LDPC_OK;
    const bool multi = c.dmax > kOdSeg * W;  // some node needs two passes
    int64_t grid = std::min<int64_t>(ntasks, 148LL * 64);
    if (var_side) {
        if (flag) k_var_f32_od<true><<<(unsigned)grid, 32 * W, 0, s>>>(a, msg, ntasks);
        else k_var_f32_od<false><<<(unsigned)grid, 32 * W, 0, s>>>(a, msg, ntasks);
    } else {
        if (multi) {
            LDPC_ARG_CHECK(scratch != nullptr && scratch_blocks > 0 &&
                               scratch_stride >= (c.dmax + kOdSeg * W - 1) / (kOdSeg * W) * 32,
                           "fast mode: check degree %d needs the workspace scratch", c.dmax);
            grid = std::min<int64_t>(grid, scratch_blocks);
        }
        float *sc = multi ? scratch : nullptr;
        if (flag) k_check_f32_od<true><<<(unsigned)grid, 32 * W, 0, s>>>(a, msg, P, sc, scratch_stride, ntasks);
        else k_check_f32_od<false><<<(unsigned)grid, 32 * W, 0, s>>>(a, msg, P, sc, scratch_stride, ntasks);
    }
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

}  // namespace ldpc
