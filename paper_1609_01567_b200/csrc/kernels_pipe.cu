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
// computes the oldest one from shared memory (cp.async.wait_group, then a
// __syncwarp because with V=1 a lane reads pieces other lanes copied).  The
// row ids of a task are loaded one ring step before its copies are issued, so
// index latency is off the critical path.
//
// A task is (node, 32*V codewords), lane l owns codewords V*l .. V*l+V-1.  V=2
// (16-byte rows pieces, 2 blocks/SM) suits low degrees; V=1 halves the
// registers per lane so 3 blocks (24 warps) fit per SM, which the high-degree
// variable buckets need to hide their fp64 dependency chains.  The grid is
// persistent: warp w of W takes tasks w, w+W, ... in chunk-major order.
#include <algorithm>
#include <mutex>
#include <string>

#include <cuda.h>

#include "common.cuh"

namespace ldpc {
namespace {

// V = codewords per lane (1 or 2): a task is (node, 32*V codewords), a row is
// 32*V doubles (256*V bytes).  Copies are always 16 bytes per lane, so a V=1
// warp moves two rows per cp.async instruction.
// ring depth from a per-warp shared-memory budget at MINB resident blocks (8 warps each) per SM:
// ~13 KB at 2 blocks, ~9 KB at 3, ~6.5 KB at 4
template <int V, int MINB>
constexpr int ring_stages(int rows) {
    const int budget = MINB <= 2 ? 13 * 1024 : (MINB == 3 ? 9 * 1024 : 6656);
    const int s = budget / (rows * 32 * V * 8);
    return s < 2 ? 2 : (s > 8 ? 8 : s);
}

// Per stage: 32 row ids (one per lane), the task's codeword chunk at [32], its skip flag at [33]
// and its done-mask words at [34..35] (early stop: read with the ids, two issues ahead).
constexpr int kIdsStride = 36;
template <int ROWS, int V, int MINB, bool TMA = false>
struct Ring {
    static constexpr int S = ring_stages<V, MINB>(ROWS);
    // TMA: one mbarrier per stage after the ids, and stages 128-byte aligned (bulk-tensor destinations)
    static constexpr size_t kBarOff = (size_t)S * kIdsStride * sizeof(int);
    static constexpr size_t kIdsBytes = TMA ? (kBarOff + S * sizeof(uint64_t) + 127) / 128 * 128 : kBarOff;
    static constexpr size_t kBytes = kIdsBytes + (size_t)S * ROWS * 32 * V * sizeof(double);
};

// ---- TMA (bulk tensor) data movement for the variable ring --------------------
// The message and prior arrays as 2-D tensors: [Bp/64 * rows][64] fp64 (a 64-codeword chunk row is
// 512 contiguous bytes); box = one row of a task (32 * V doubles).  One elected lane fetches a task's
// rows with tile::gather4 (4 rows, given by their indices, per instruction) plus single-row tile
// loads, completing on the stage's mbarrier (complete_tx), instead of 32 lanes issuing LDGSTS.
struct __align__(64) TMap {
    uint64_t v[16];  // CUtensorMap (opaque, 128 bytes)
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void tma_gather4(void *dst, const TMap *map, int c0, int r0, int r1, int r2, int r3,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_row(void *dst, const TMap *map, int c0, int r, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(r), "r"(smem_u32(bar))
        : "memory");
}


template <int V>
__device__ __forceinline__ void st_v(double *p, const double (&o)[V]) {
    if constexpr (V == 2) st_msg(reinterpret_cast<double2 *>(p), make_double2(o[0], o[1]));
    else st_msg(p, o[0]);
}

template <int V>
__device__ __forceinline__ void ld_smem(const double *p, double (&o)[V]) {
    if constexpr (V == 2) {
        const double2 x = *reinterpret_cast<const double2 *>(p);
        o[0] = x.x;
        o[1] = x.y;
    } else {
        o[0] = *p;
    }
}


// all codewords of warp-chunk ch (32*V codewords) have stopped
template <int V>
__device__ __forceinline__ bool wchunk_done(const uint32_t *done, int ch) {
    if (done == nullptr) return false;
    if constexpr (V == 2) {
        const uint2 d = *reinterpret_cast<const uint2 *>(done + 2 * ch);
        return (d.x & d.y) == 0xffffffffu;
    } else {
        return done[ch] == 0xffffffffu;
    }
}

// done-mask words of warp-chunk ch (0 when not in early-stop mode), read ahead of the task
struct DoneMask {
    uint32_t w0 = 0, w1 = 0;
};
template <int V>
__device__ __forceinline__ DoneMask load_done(const uint32_t *done, int ch) {
    DoneMask m;
    if (done == nullptr) return m;
    if constexpr (V == 2) {
        const uint2 d = *reinterpret_cast<const uint2 *>(done + 2 * ch);
        m.w0 = d.x;
        m.w1 = d.y;
    } else {
        m.w0 = done[ch];
    }
    return m;
}
template <int V>
__device__ __forceinline__ bool all_done(const DoneMask &m) {
    return V == 2 ? (m.w0 & m.w1) == 0xffffffffu : m.w0 == 0xffffffffu;
}

// Row ids of a task, one per lane:
//   lanes 0..D-1: message slots of the node's edges (outputs; inputs unless FROM_PRIOR)
//   variables: lane D = the variable (its prior row and c_hat row)
//   checks FROM_PRIOR: lanes 16..16+D-1 = variables whose prior rows are the inputs
// NPT nodes per task (low-degree variables): lanes u*(D+1) .. u*(D+1)+D hold node u's D slots and
// its variable; a missing last node gets variable -1 (skipped) and slot 0 (a harmless fetch)
template <int D, int NPT>
__device__ __forceinline__ int load_id_npt(const NodeLaunch &a, int ni, int lane) {
    const int u = lane / (D + 1), j = lane - u * (D + 1);
    const int node = ni * NPT + u;
    if (u >= NPT) return 0;
    if (node >= a.node_count) return j == D ? -1 : 0;
    if (j < D) return __ldg(a.slot_ord + a.edge_begin + node * D + j);
    return __ldg(a.order + a.node_begin + node);
}

template <int D, bool IS_VAR, bool FROM_PRIOR>
__device__ __forceinline__ int load_id(const NodeLaunch &a, int ni, int lane) {
    const int32_t base = a.edge_begin + ni * D;
    if (lane < D) return __ldg(a.slot_ord + base + lane);
    if (IS_VAR && lane == D) return __ldg(a.order + a.node_begin + ni);
    if (!IS_VAR && FROM_PRIOR && lane >= 16 && lane < 16 + D) return __ldg(a.var_ord + base + lane - 16);
    return 0;
}

// Variables of degree >= kPriorRegDeg fetch their prior row into registers one
// iteration ahead (their iterations are long enough to hide the latency, and the
// smaller ring gains a stage); lower degrees stage the prior row in the ring.
#ifndef LDPC_PRIOR_REG_DEG
#define LDPC_PRIOR_REG_DEG 6
#endif
constexpr int kPriorRegDeg = LDPC_PRIOR_REG_DEG;
template <int D, bool IS_VAR>
constexpr bool prior_in_ring() { return IS_VAR && D < kPriorRegDeg; }
template <int D, bool IS_VAR>
constexpr int ring_rows() { return D + (prior_in_ring<D, IS_VAR>() ? 1 : 0); }

template <int D, int V, bool EARLY, int NPT>
__device__ __forceinline__ void issue_npt(const NodeLaunch &a, double *rows, int *ids_s, int ch, int id,
                                          const DoneMask &dm, int lane) {
    static_assert(prior_in_ring<D, true>(), "NPT > 1 needs the prior row in the ring");
    constexpr int ROWS = ring_rows<D, true>();  // per node: D message rows + the prior row
    constexpr int ROW = 32 * V;
    constexpr int RPI = V == 2 ? 1 : 2;
    const bool skip = EARLY && all_done<V>(dm);
    ids_s[lane] = id;
    if (lane == 0) {
        ids_s[32] = ch;
        if constexpr (EARLY) {
            ids_s[33] = skip ? 1 : 0;
            ids_s[34] = (int)dm.w0;
            ids_s[35] = (int)dm.w1;
        }
    }
    if (skip) return;
    const int cw0 = ch * 32 * V;
    const int sub = V == 2 ? 0 : (lane >> 4);
    const int piece = V == 2 ? lane : (lane & 15);
    const double *mb = chunk_base(a.msg, a.msg_rows, cw0) + 2 * piece;
    const double *pb = chunk_base(a.P, a.p_rows, cw0) + 2 * piece;
    double *dst = rows + 2 * piece;
#pragma unroll
    for (int j = 0; j < (NPT * ROWS + RPI - 1) / RPI; j++) {
        const int r = j * RPI + sub;
        const int rr = r < NPT * ROWS ? r : NPT * ROWS - 1;
        const int u = rr / ROWS, k = rr - u * ROWS;  // node u of the task, its row k (k == D: prior)
        const int src_id = max(0, __shfl_sync(0xffffffffu, id, u * (D + 1) + k));
        const double *src = (k == D ? pb : mb) + row_off(src_id);
        if (r < NPT * ROWS) cp_async16(dst + r * ROW, src);
    }
}

template <int D, int V, bool IS_VAR, bool FROM_PRIOR, bool EARLY>
__device__ __forceinline__ void issue(const NodeLaunch &a, double *rows, int *ids_s, int ch, int id,
                                      const DoneMask &dm, int lane) {
    constexpr int ROWS = ring_rows<D, IS_VAR>();
    constexpr int ROW = 32 * V;                 // doubles per row
    constexpr int RPI = V == 2 ? 1 : 2;         // rows per copy instruction
    const bool skip = EARLY && all_done<V>(dm);
    ids_s[lane] = id;
    if (lane == 0) {
        ids_s[32] = ch;
        if constexpr (EARLY) {
            ids_s[33] = skip ? 1 : 0;
            ids_s[34] = (int)dm.w0;
            ids_s[35] = (int)dm.w1;
        }
    }
    if (skip) return;  // every codeword of the chunk has stopped: nothing to fetch; compute skips it too
    if constexpr (!EARLY) {
        if (wchunk_done<V>(a.done, ch)) return;  // (a.done is null here: the fixed-iteration kernel's code)
    }
    const int cw0 = ch * 32 * V;
    const int sub = V == 2 ? 0 : (lane >> 4);  // which row of the instruction's pair this lane copies
    const int piece = V == 2 ? lane : (lane & 15);
    const double *mb = chunk_base(a.msg, a.msg_rows, cw0) + 2 * piece;
    const double *pb = chunk_base(a.P, a.p_rows, cw0) + 2 * piece;
    double *dst = rows + 2 * piece;
#pragma unroll
    for (int j = 0; j < (ROWS + RPI - 1) / RPI; j++) {
        const int r = j * RPI + sub;
        // every lane takes part in the shuffles; lanes past the last row skip the copy
        const int rr = r < ROWS ? r : ROWS - 1;
        const bool prior_row = (prior_in_ring<D, IS_VAR>() && rr == D) || (!IS_VAR && FROM_PRIOR);
        const int src_id = __shfl_sync(0xffffffffu, id, (!IS_VAR && FROM_PRIOR) ? 16 + rr : rr);
        const double *src = (prior_row ? pb : mb) + row_off(src_id);
        if (r < ROWS) cp_async16(dst + r * ROW, src);
    }
}

// Variables only: the task's D message rows (gather4 in fours, then single rows) and, for low
// degrees, its prior row, all by lane 0, completing on the stage's mbarrier.
template <int D, int V, bool EARLY>
__device__ __forceinline__ void issue_tma(const NodeLaunch &a, double *rows, int *ids_s, uint64_t *bar, int ch,
                                          int id, const DoneMask &dm, int lane, const TMap *tm_msg,
                                          const TMap *tm_p) {
    constexpr int ROWS = ring_rows<D, true>();
    constexpr int ROW = 32 * V;
    const bool skip = EARLY && all_done<V>(dm);
    ids_s[lane] = id;
    if (lane == 0) {
        ids_s[32] = ch;
        if constexpr (EARLY) {
            ids_s[33] = skip ? 1 : 0;
            ids_s[34] = (int)dm.w0;
            ids_s[35] = (int)dm.w1;
        }
    }
    __syncwarp();  // lane 0 reads every lane's row id
    if (lane != 0) return;
    if (skip) {  // nothing to fetch: complete the stage's phase without a transaction
        mbar_arrive(bar);
        return;
    }
    const int c64 = V == 2 ? ch : (ch >> 1);         // 64-codeword chunk of the task
    const int c0 = V == 2 ? 0 : (ch & 1) * 32;       // its first codeword within the chunk row
    const int rm = c64 * a.msg_rows, rp = c64 * a.p_rows;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the stage's earlier generic reads
    mbar_arrive_tx(bar, ROWS * ROW * (uint32_t)sizeof(double));
    int r = 0;
#pragma unroll
    for (; r + 4 <= D; r += 4)
        tma_gather4(rows + r * ROW, tm_msg, c0, rm + ids_s[r], rm + ids_s[r + 1], rm + ids_s[r + 2], rm + ids_s[r + 3],
                    bar);
#pragma unroll
    for (; r < D; r++) tma_row(rows + r * ROW, tm_msg, c0, rm + ids_s[r], bar);
    if constexpr (prior_in_ring<D, true>()) tma_row(rows + D * ROW, tm_p, c0, rp + ids_s[D], bar);
}

template <int D, int V>
__device__ __forceinline__ void compute_check(const NodeLaunch &a, const double *rows, const int *ids, int ch,
                                              int lane) {
    constexpr int ROW = 32 * V;
    double *mb = chunk_base(a.msg, a.msg_rows, ch * 32 * V) + lane * V;
    double b[D][V];
#pragma unroll
    for (int i = 0; i < D; i++) {
        double q[V];
        ld_smem<V>(rows + i * ROW + V * lane, q);
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
        st_v<V>(mb + row_off(ids[k]), out);
        if (k + 1 < D) {
#pragma unroll
            for (int v = 0; v < V; v++) pre[v] = __dmul_rn(pre[v], b[k][v]);
        }
    }
}

template <int D, int V, bool WRITE_Q, bool EARLY>
__device__ __forceinline__ void compute_var(const NodeLaunch &a, const double *rows, const int *ids, int ch,
                                            int lane, const double (&pj)[V], const int *masks) {
    constexpr int ROW = 32 * V;
    double *mb = chunk_base(a.msg, a.msg_rows, ch * 32 * V) + lane * V;
    double r[D][V], om[D][V];
#pragma unroll
    for (int i = 0; i < D; i++) {
        ld_smem<V>(rows + i * ROW + V * lane, r[i]);
#pragma unroll
        for (int v = 0; v < V; v++) om[i][v] = __dsub_rn(1.0, r[i][v]);
    }
    double p0[V], p1[V];
#pragma unroll
    for (int v = 0; v < V; v++) {
        p0[v] = __dsub_rn(1.0, pj[v]);
        p1[v] = pj[v];
    }
    uint32_t slow = 0;
#pragma unroll
    for (int k = 0; k < D; k++) {
        if constexpr (WRITE_Q) {
            double out[V];
            bool all_ok = true;
#pragma unroll
            for (int v = 0; v < V; v++) {
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
            // stored unconditionally (no branch per output); the rare inexact ones are
            // recomputed and overwritten below, later in this thread's program order
            st_v<V>(mb + row_off(ids[k]), out);
            if (!all_ok) slow |= 1u << k;
        }
#pragma unroll
        for (int v = 0; v < V; v++) {
            p0[v] = __dmul_rn(p0[v], om[k][v]);
            p1[v] = __dmul_rn(p1[v], r[k][v]);
        }
    }
    if constexpr (WRITE_Q) {
        if (slow) {  // rare: tiny or zero denominators -> reference-order recompute, library division
#pragma unroll
            for (int k = 0; k < D; k++) {
                if (!((slow >> k) & 1u)) continue;
                double out[V];
#pragma unroll
                for (int v = 0; v < V; v++) {
                    double q0 = __dsub_rn(1.0, pj[v]), q1 = pj[v];
#pragma unroll
                    for (int i = 0; i < D; i++) {
                        if (i == k) continue;
                        q0 = __dmul_rn(q0, om[i][v]);
                        q1 = __dmul_rn(q1, r[i][v]);
                    }
                    const double den = __dadd_rn(q0, q1);
                    out[v] = (den == 0.0) ? 0.5 : __ddiv_rn(q1, den);
                }
                st_v<V>(mb + row_off(ids[k]), out);
            }
        }
    }
    // estimate (serial.py:132): bit = !(Q0 > Q1)
    uint32_t *row = a.chat + (size_t)ids[D] * a.NW;
    if constexpr (V == 2) {
        const uint32_t even = __ballot_sync(0xffffffffu, !(p0[0] > p1[0]));
        const uint32_t odd = __ballot_sync(0xffffffffu, !(p0[1] > p1[1]));
        if (lane == 0) {
            uint32_t lo = part1by1(even) | (part1by1(odd) << 1);
            uint32_t hi = part1by1(even >> 16) | (part1by1(odd >> 16) << 1);
            uint32_t *dst = row + 2 * ch;
            if constexpr (EARLY) {
                const uint32_t d0 = (uint32_t)masks[0], d1 = (uint32_t)masks[1];  // prefetched done mask
                if (d0) lo = (lo & ~d0) | (dst[0] & d0);
                if (d1) hi = (hi & ~d1) | (dst[1] & d1);
            }
            *reinterpret_cast<uint2 *>(dst) = make_uint2(lo, hi);
        }
    } else {
        uint32_t bits = __ballot_sync(0xffffffffu, !(p0[0] > p1[0]));
        if (lane == 0) {
            if constexpr (EARLY) {
                const uint32_t d0 = (uint32_t)masks[0];  // prefetched done mask
                if (d0) bits = (bits & ~d0) | (row[ch] & d0);
            }
            row[ch] = bits;
        }
    }
}

// a variable's prior row (V doubles per lane) straight into registers
template <int V>
__device__ __forceinline__ void load_prior(const NodeLaunch &a, int node, int ch, int lane, double (&o)[V]) {
    const double *p = chunk_base(a.P, a.p_rows, ch * 32 * V) + V * lane + row_off(node);
    if constexpr (V == 2) {
        const double2 x = __ldg(reinterpret_cast<const double2 *>(p));
        o[0] = x.x;
        o[1] = x.y;
    } else {
        o[0] = __ldg(p);
    }
}

// EARLY: early-stop mode (a.done != nullptr): per-task chunk-done masks, read ahead with the ids
template <int D, int V, bool IS_VAR, bool FLAG, int MINB, bool EARLY, bool TMA = false, int NPT = 1>  // FLAG: FROM_PRIOR / WRITE_Q
__device__ __forceinline__ void ring_loop(const NodeLaunch &a, int64_t ntasks, int64_t first, int64_t W,
                                          unsigned char *wsm, const TMap *tm_msg = nullptr,
                                          const TMap *tm_p = nullptr) {
    // one warp's persistent task loop: tasks first, first + W, ... of a side's bucket,
    // its ring (ids + stages) at wsm; a task is NPT nodes (NPT > 1: low-degree variables)
    static_assert(!TMA || IS_VAR, "the TMA ring serves the variable side");
    static_assert(NPT == 1 || (IS_VAR && !TMA && NPT * (D + 1) <= 32), "NPT > 1: variables, ids in one warp");
    constexpr int ROWS = NPT * ring_rows<D, IS_VAR>();  // rows per stage
    constexpr int NROWS = ring_rows<D, IS_VAR>();       // rows per node
    constexpr bool PREG = IS_VAR && !prior_in_ring<D, IS_VAR>();  // prior via registers
    constexpr int ROW = 32 * V;
    constexpr bool FP = !IS_VAR && FLAG;
    using R = Ring<ROWS, V, MINB, TMA>;
    constexpr int S = R::S;
    const int lane = threadIdx.x & 31;
    int *ids = reinterpret_cast<int *>(wsm);                          // [S][kIdsStride]
    double *rows = reinterpret_cast<double *>(wsm + R::kIdsBytes);    // [S][ROWS][ROW]
    uint64_t *bars = reinterpret_cast<uint64_t *>(wsm + R::kBarOff);  // [S] (TMA)
    if constexpr (TMA) {
        if (lane == 0) {
            for (int k = 0; k < S; k++) mbar_init(bars + k, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }
    // early-stop compaction: only the active chunks' tasks (chunk-major, so a prefix of the tasks)
    const int wchunks = active_chunks(a, a.Bp / (32 * V), 32 * V);
    const int ncs = (a.node_count + NPT - 1) / NPT;  // tasks per chunk
    ntasks = min(ntasks, (int64_t)ncs * wchunks);
    if (first >= ntasks) return;
    const int ntask = (int)((ntasks - first + W - 1) / W);  // this warp's tasks: first, first + W, ...
    auto load_ids = [&](int ni) {
        if constexpr (NPT > 1) return load_id_npt<D, NPT>(a, ni, lane);
        else return load_id<D, IS_VAR, FP>(a, ni, lane);
    };

    // The row ids of task j are loaded two issues ahead (while task j - 2 is
    // issued), so the index loads' L2 latency is off the critical path; the
    // cursor runs two tasks ahead of the issue.
    TaskCursor cur(first, W, ncs);
    const int chunks_m1 = wchunks - 1;  // reverse sweep: chunk c -> chunks-1-c
    auto chunk_of = [&](int c) { return a.reverse ? chunks_m1 - c : c; };
    int nid0 = load_ids(cur.ni), nch0 = chunk_of(cur.ch);
    DoneMask nd0 = EARLY ? load_done<V>(a.done, nch0) : DoneMask{};
    cur.next();
    int nid1 = 0, nch1 = 0;
    DoneMask nd1;
    if (ntask > 1) {
        nid1 = load_ids(cur.ni);
        nch1 = chunk_of(cur.ch);
        if (EARLY) nd1 = load_done<V>(a.done, nch1);
        cur.next();
    }
    auto issue_next = [&](int j) {  // issue task j (j < ntask) into stage j % S
        const int id = nid0, ich = nch0;
        const DoneMask idone = nd0;
        nid0 = nid1;
        nch0 = nch1;
        nd0 = nd1;
        if (j + 2 < ntask) {
            nid1 = load_ids(cur.ni);
            nch1 = chunk_of(cur.ch);
            if (EARLY) nd1 = load_done<V>(a.done, nch1);
            cur.next();
        }
        const int sj = j % S;
        if constexpr (TMA)
            issue_tma<D, V, EARLY>(a, rows + (size_t)sj * ROWS * ROW, ids + sj * kIdsStride, bars + sj, ich, id, idone,
                                   lane, tm_msg, tm_p);
        else if constexpr (NPT > 1)
            issue_npt<D, V, EARLY, NPT>(a, rows + (size_t)sj * ROWS * ROW, ids + sj * kIdsStride, ich, id, idone, lane);
        else
            issue<D, V, IS_VAR, FP, EARLY>(a, rows + (size_t)sj * ROWS * ROW, ids + sj * kIdsStride, ich, id, idone,
                                           lane);
    };
    // prologue: copies of tasks 0..S-2 (one commit group per task)
    for (int j = 0; j < S - 1; j++) {
        if (j < ntask) issue_next(j);
        cp_commit();
    }
    // Variables of high degree: the prior row of a task is loaded into registers
    // PD iterations before it is computed (its ids were issued S-1 >= PD
    // iterations ahead, so they are in smem); one iteration did not cover the
    // DRAM latency (ncu: the first use of the prior was the top stall).
    constexpr int PD = S >= 3 ? 2 : 1;
    double pq[PD][V] = {};
    if (PREG) {
        __syncwarp();  // row ids written at issue (plain shared stores) are visible
#pragma unroll
        for (int d = 0; d < PD; d++)
            if (d < ntask) load_prior<V>(a, ids[d * kIdsStride + D], ids[d * kIdsStride + 32], lane, pq[d]);
    }
    for (int it = 0; it < ntask; it++) {
        // keep S-1 tasks in flight: issue task it + S-1 into the stage freed last iteration
        if (it + S - 1 < ntask) issue_next(it + S - 1);
        const int s = it % S;
        if constexpr (TMA) {
            mbar_wait(bars + s, (uint32_t)(it / S) & 1u);  // the stage's bytes (and lane 0's ids) landed
            __syncwarp();
        } else {
            cp_commit();
            cp_wait<S - 1>();  // this lane's copies of task it have landed
            __syncwarp();      // ... and every other lane's (V=1 lanes read pieces copied by other lanes)
        }
        const int *ids_s = ids + s * kIdsStride;
        const int ch = ids_s[32];
        double pj[V];
        if constexpr (PREG) {
#pragma unroll
            for (int v = 0; v < V; v++) pj[v] = pq[0][v];
#pragma unroll
            for (int d = 0; d + 1 < PD; d++)
#pragma unroll
                for (int v = 0; v < V; v++) pq[d][v] = pq[d + 1][v];
            if (it + PD < ntask) {
                const int *idsn = ids + ((it + PD) % S) * kIdsStride;
                load_prior<V>(a, idsn[D], idsn[32], lane, pq[PD - 1]);
            }
        } else if constexpr (IS_VAR && NPT == 1) {
            ld_smem<V>(rows + (size_t)s * ROWS * ROW + D * ROW + V * lane, pj);
        }
        if (EARLY ? !ids_s[33] : !wchunk_done<V>(a.done, ch)) {
            if constexpr (NPT > 1) {
#pragma unroll
                for (int u = 0; u < NPT; u++) {
                    if (ids_s[u * (D + 1) + D] < 0) break;  // a missing last node (warp-uniform)
                    const double *nrows = rows + (size_t)s * ROWS * ROW + (size_t)u * NROWS * ROW;
                    ld_smem<V>(nrows + D * ROW + V * lane, pj);
                    compute_var<D, V, FLAG, EARLY>(a, nrows, ids_s + u * (D + 1), ch, lane, pj, ids_s + 34);
                }
            } else if constexpr (IS_VAR) {
                compute_var<D, V, FLAG, EARLY>(a, rows + (size_t)s * ROWS * ROW, ids_s, ch, lane, pj, ids_s + 34);
            } else {
                compute_check<D, V>(a, rows + (size_t)s * ROWS * ROW, ids_s, ch, lane);
            }
        }
        __syncwarp();  // stage s is reused by the issue of the next iteration
    }
    if constexpr (!TMA) cp_wait<0>();
}

template <int D, int V, bool IS_VAR, bool FLAG, int MINB, bool EARLY, int NPT = 1>  // FLAG: FROM_PRIOR / WRITE_Q
__global__ void __launch_bounds__(kThreads, MINB) k_node_ring(NodeLaunch a, int64_t ntasks) {
    using R = Ring<NPT * ring_rows<D, IS_VAR>(), V, MINB>;
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5;
    ring_loop<D, V, IS_VAR, FLAG, MINB, EARLY, false, NPT>(a, ntasks, (int64_t)blockIdx.x * kWarpsPerBlock + warp,
                                                          (int64_t)gridDim.x * kWarpsPerBlock,
                                                          smem + (size_t)warp * R::kBytes);
}

template <int D, int V, bool WRITE_Q, int MINB, bool EARLY>
__global__ void __launch_bounds__(kThreads, MINB)
    k_var_ring_tma(NodeLaunch a, int64_t ntasks, const __grid_constant__ TMap tm_msg, const __grid_constant__ TMap tm_p) {
    using R = Ring<ring_rows<D, true>(), V, MINB, true>;
    extern __shared__ __align__(128) unsigned char smem_t[];
    const int warp = threadIdx.x >> 5;
    ring_loop<D, V, true, WRITE_Q, MINB, EARLY, true>(a, ntasks, (int64_t)blockIdx.x * kWarpsPerBlock + warp,
                                                     (int64_t)gridDim.x * kWarpsPerBlock,
                                                     smem_t + (size_t)warp * R::kBytes, &tm_msg, &tm_p);
}

// Codewords per lane: V=1 (3 blocks/SM, more warps to hide the fp64 chains) for
// variables of degree >= 3, V=2 (16-byte rows pieces per lane) for degree 2 and
// checks (profiles/r1_kernel_choice.md).  LDPC_RING_V=1|2 forces one.
int ring_v(bool var_side, int deg) {
    static const int forced = [] {
        const char *e = getenv("LDPC_RING_V");
        return e ? atoi(e) : 0;
    }();
    if (forced == 1 || forced == 2) return forced;
    return var_side && deg >= 3 ? 1 : 2;
}

template <int D, int V, bool IS_VAR, bool FLAG, int MINB, bool EARLY, int NPT = 1>
int launch_ring_ve(const NodeLaunch &a, cudaStream_t st) {
    constexpr int ROWS = NPT * ring_rows<D, IS_VAR>();
    const size_t smem = (size_t)kWarpsPerBlock * Ring<ROWS, V, MINB>::kBytes;
    auto kern = k_node_ring<D, V, IS_VAR, FLAG, MINB, EARLY, NPT>;
    // the shared-memory attribute is per device: set it (and size the grid) once per device
    constexpr int kMaxDevices = 64;
    static int per_sm_of[kMaxDevices] = {}, sms_of[kMaxDevices] = {};
    static std::mutex mu;
    int dev = 0;
    LDPC_CUDA_TRY(cudaGetDevice(&dev));
    LDPC_ARG_CHECK(dev >= 0 && dev < kMaxDevices, "device ordinal %d out of range", dev);
    int per_sm, sms;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (per_sm_of[dev] == 0) {
            LDPC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            LDPC_CUDA_TRY(cudaDeviceGetAttribute(&sms_of[dev], cudaDevAttrMultiProcessorCount, dev));
            int b = 0;
            LDPC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kThreads, smem));
            if (b < 1) {
                set_error("ring node kernel (degree %d) does not fit on an SM", D);
                return LDPC_ECUDA;
            }
            per_sm_of[dev] = b;
        }
        per_sm = per_sm_of[dev];
        sms = sms_of[dev];
    }
    const int64_t ntasks = (int64_t)((a.node_count + NPT - 1) / NPT) * (a.Bp / (32 * V));
    if (ntasks == 0) return LDPC_OK;
    const int64_t need = (ntasks + kWarpsPerBlock - 1) / kWarpsPerBlock;
    const int64_t blocks = std::min<int64_t>(need, (int64_t)per_sm * sms);
    kern<<<(unsigned)blocks, kThreads, smem, st>>>(a, ntasks);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

// ---- host: tensor maps for the TMA ring ----
using EncodeTiled = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                 const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// [Bp/64 * rows][64] fp64 chunk-major array as a 2-D tensor, box = one task row (32 * V doubles)
int make_row_map(const double *base, int32_t rows, int32_t Bp, int V, TMap *out) {
    static EncodeTiled encode = [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<EncodeTiled>(fn);
    }();
    if (encode == nullptr) {
        set_error("cuTensorMapEncodeTiled is not available from the driver");
        return LDPC_ECUDA;
    }
    const uint64_t total_rows = (uint64_t)(Bp / 64) * (uint64_t)rows;
    LDPC_ARG_CHECK(total_rows < (1ull << 31), "TMA ring: %llu rows exceed 32-bit coordinates",
                   (unsigned long long)total_rows);
    static_assert(sizeof(TMap) == sizeof(CUtensorMap), "TMap must hold a CUtensorMap");
    const cuuint64_t dims[2] = {64, total_rows};
    const cuuint64_t strides[1] = {64 * sizeof(double)};
    const cuuint32_t box[2] = {(cuuint32_t)(32 * V), 1};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode(reinterpret_cast<CUtensorMap *>(out), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                              const_cast<double *>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
        return LDPC_ECUDA;
    }
    return LDPC_OK;
}

template <int D, int V, bool WRITE_Q, int MINB, bool EARLY>
int launch_var_tma_ve(const NodeLaunch &a, cudaStream_t st) {
    constexpr int ROWS = ring_rows<D, true>();
    const size_t smem = (size_t)kWarpsPerBlock * Ring<ROWS, V, MINB, true>::kBytes;
    auto kern = k_var_ring_tma<D, V, WRITE_Q, MINB, EARLY>;
    constexpr int kMaxDevices = 64;
    static int per_sm_of[kMaxDevices] = {}, sms_of[kMaxDevices] = {};
    static std::mutex mu;
    int dev = 0;
    LDPC_CUDA_TRY(cudaGetDevice(&dev));
    LDPC_ARG_CHECK(dev >= 0 && dev < kMaxDevices, "device ordinal %d out of range", dev);
    int per_sm, sms;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (per_sm_of[dev] == 0) {
            LDPC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            LDPC_CUDA_TRY(cudaDeviceGetAttribute(&sms_of[dev], cudaDevAttrMultiProcessorCount, dev));
            int b = 0;
            LDPC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kThreads, smem));
            if (b < 1) {
                set_error("TMA ring kernel (degree %d) does not fit on an SM", D);
                return LDPC_ECUDA;
            }
            per_sm_of[dev] = b;
        }
        per_sm = per_sm_of[dev];
        sms = sms_of[dev];
    }
    const int64_t ntasks = (int64_t)a.node_count * (a.Bp / (32 * V));
    if (ntasks == 0) return LDPC_OK;
    TMap tm_msg, tm_p;
    int rc = make_row_map(a.msg, a.msg_rows, a.Bp, V, &tm_msg);
    if (rc == LDPC_OK) rc = make_row_map(a.P, a.p_rows, a.Bp, V, &tm_p);
    if (rc) return rc;
    const int64_t need = (ntasks + kWarpsPerBlock - 1) / kWarpsPerBlock;
    const int64_t blocks = std::min<int64_t>(need, (int64_t)per_sm * sms);
    kern<<<(unsigned)blocks, kThreads, smem, st>>>(a, ntasks, tm_msg, tm_p);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

// LDPC_KERNEL=tma: variable buckets of the ring path through the TMA ring (A/B of the data mover)
bool use_tma_ring() {
    static const bool on = [] {
        const char *e = getenv("LDPC_KERNEL");
        return e && std::string(e) == "tma";
    }();
    return on;
}

// variables get a fixed-iteration instantiation without the early-stop bookkeeping; checks
// (ring only on request) keep the one that handles both modes
// Nodes per ring task for the shortest variable tasks: two for degree 2 and for the final estimate
// pass (no q writes) of degree 3, halving their per-task overhead; measured per launch (ncu, C3):
// deg 2 226.3 -> 224.8 us, deg-2 estimate 145.1 -> 134.2, deg-3 estimate 113.6 -> 96.7, but deg 3
// with q writes 195.9 -> 198.2 (kept at one).  LDPC_RING_NPT=1|2 forces one choice for degrees <= 3.
int ring_npt(int deg, bool write_q) {
    static const int forced = [] {
        const char *e = getenv("LDPC_RING_NPT");
        return e ? atoi(e) : 0;
    }();
    if (forced == 1 || forced == 2) return forced;
    return (deg == 2 || (deg == 3 && !write_q)) ? 2 : 1;
}

template <int D, int V, bool IS_VAR, bool FLAG, int MINB>
int launch_ring_v(const NodeLaunch &a, cudaStream_t st) {
    if constexpr (IS_VAR) {
        if (use_tma_ring() && a.Bp % 64 == 0)
            return a.done == nullptr ? launch_var_tma_ve<D, V, FLAG, MINB, false>(a, st)
                                     : launch_var_tma_ve<D, V, FLAG, MINB, true>(a, st);
        if constexpr (D <= 3) {
            if (ring_npt(D, FLAG) == 2)
                return a.done == nullptr ? launch_ring_ve<D, V, IS_VAR, FLAG, MINB, false, 2>(a, st)
                                         : launch_ring_ve<D, V, IS_VAR, FLAG, MINB, true, 2>(a, st);
        }
        if (a.done == nullptr) return launch_ring_ve<D, V, IS_VAR, FLAG, MINB, false>(a, st);
    }
    return launch_ring_ve<D, V, IS_VAR, FLAG, MINB, true>(a, st);
}

// Resident blocks per SM (sets the ring depth): 2 for V=2, 3 for V=1 by default;
// LDPC_RING_MINB=3 (V=2) / 4 (V=1) trades ring depth for warps on the variable side.
int ring_minb(bool var_side, int V) {
    static const int forced = [] {
        const char *e = getenv("LDPC_RING_MINB");
        return e ? atoi(e) : 0;
    }();
    if (var_side && forced == (V == 2 ? 3 : 4)) return forced;
    return V == 2 ? 2 : 3;
}

template <int D, bool IS_VAR, bool FLAG>
int launch_ring(const NodeLaunch &a, cudaStream_t st) {
    if (a.Bp % 64 || ring_v(IS_VAR, D) == 1) {
        if (IS_VAR && ring_minb(IS_VAR, 1) == 4) return launch_ring_v<D, 1, IS_VAR, FLAG, 4>(a, st);
        return launch_ring_v<D, 1, IS_VAR, FLAG, 3>(a, st);
    }
    if (IS_VAR && ring_minb(IS_VAR, 2) == 3) return launch_ring_v<D, 2, IS_VAR, FLAG, 3>(a, st);
    return launch_ring_v<D, 2, IS_VAR, FLAG, 2>(a, st);
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
