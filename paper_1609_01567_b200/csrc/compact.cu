// compact.cu -- per-codeword early stop: live codewords compacted into dense chunks.
//
// The reference stops each frame at its first all-zero syndrome and does no
// further work on it (serial.py:169-177, engine.py:341-347).  The node kernels
// skip work per 32/64-codeword warp chunk (done masks), so without compaction a
// chunk runs until its slowest codeword stops.  Here, after the early-stop
// update of a round, a one-block plan kernel counts the live codewords L; when
// the active chunks would shrink enough (ceil(L/64) <= a fraction of them) it
//   * retires every stopped codeword of the active region: its estimate bits
//     (bit-sliced chat -> the caller's packed rows, through the position ->
//     codeword map), success = 1, iterations, an all-zero syndrome row;
//   * moves the live codewords' state (messages and priors, the only state
//     that crosses a round) into positions 0..L-1, in place.  Default (fill):
//     the live codewords at positions >= L move into the stopped positions
//     below L, i-th source into i-th hole -- only those move, and sources and
//     destinations are disjoint.  LDPC_COMPACT_MODE=stable: all live codewords
//     shift down in order; one warp per row walks the output chunks upward, so
//     every source it still has to read lies above everything it wrote;
//   * rewrites the maps and done masks (positions >= L become padding, done).
// Codewords are independent and each keeps its own arithmetic, so results are
// bit-identical to the uncompacted decode.  Everything stays on the device
// (the decision is data dependent, so every kernel is launched every round and
// the row move / retire exit at once when the plan says "no").
#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"

namespace ldpc {
namespace {

constexpr int kPlanThreads = 1024;

// ctl[0] = active 64-codeword chunks, ctl[1] = compact this round, ctl[2] = L (live codewords),
// ctl[3] = first output chunk whose contents change, ctl[4] = active chunks before this round's plan
// The plan also does the early-stop update of round `round` first (k_update_done's work,
// serial.py:169-177: codewords whose syndrome is all-zero stop now with iterations_used = round).
__global__ void __launch_bounds__(kPlanThreads) k_compact_plan(uint32_t *done, uint32_t *unsat, int32_t *iters,
                                                               int32_t NW, int32_t round, int32_t *orig,
                                                               int32_t *ret_orig, int32_t *perm, uint32_t *ret_sel,
                                                               int32_t *ctl, int frac_pct, int fill) {
    __shared__ int warp_tot[kPlanThreads / 32];
    __shared__ int first_moved, live_below_L;
    const int t = threadIdx.x;
    for (int w = t; w < NW; w += kPlanThreads) {
        const uint32_t d = done[w], newly = ~d & ~unsat[w];
        for (uint32_t x = newly; x; x &= x - 1) iters[32 * w + __ffs(x) - 1] = round;
        done[w] = d | newly;
        unsat[w] = 0;
    }
    __syncthreads();
    const int act = ctl[0];
    const int NWa = 2 * act;  // active done words
    const int per = (NWa + kPlanThreads - 1) / kPlanThreads;
    const int w0 = min(NWa, t * per), w1 = min(NWa, w0 + per);
    int live = 0;
    for (int w = w0; w < w1; w++) live += __popc(~done[w]);
    // exclusive scan of the live counts: shuffles within warps, then over the 32 warp totals
    const int lane = t & 31;
    int incl = live;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
    }
    if (lane == 31) warp_tot[t >> 5] = incl;
    if (t == 0) first_moved = INT32_MAX;
    __syncthreads();
    int wt = lane < kPlanThreads / 32 ? warp_tot[lane] : 0, wincl = wt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, wincl, o);
        if (lane >= o) wincl += x;
    }
    const int L = __shfl_sync(0xffffffffu, wincl, 31);
    const int base = __shfl_sync(0xffffffffu, wincl - wt, t >> 5) + incl - live;
    const int new_act = (L + 63) / 64;
    const bool go = new_act < act && (int64_t)new_act * 100 <= (int64_t)act * frac_pct;
    __syncthreads();  // every thread has read ctl[0] and the scan before ctl changes
    if (!go) {
        if (t == 0) ctl[1] = 0;
        return;
    }
    if (t == 0) ctl[4] = act;
    if (fill) {
        // hole filling: the live codewords at positions >= L move into the stopped positions below L,
        // the i-th such source into the i-th hole (perm[i] = hole, perm[half + i] = source)
        if (32 * w0 <= L && L < 32 * w1) {
            int c = base;
            for (int w = w0; 32 * (w + 1) <= L; w++) c += __popc(~done[w]);
            if (L & 31) c += __popc(~done[L >> 5] & ((1u << (L & 31)) - 1u));
            live_below_L = c;
        }
        if (t == 0 && L >= 32 * NWa) live_below_L = L;
        __syncthreads();
        const int K = L - live_below_L, half = 16 * NW, src0 = L - K;
        int k = base;
        for (int w = w0; w < w1; w++) {
            const uint32_t d = done[w];
            ret_sel[w] = d;
            for (int b = 0; b < 32; b++) {
                const int p = 32 * w + b;
                const bool lv = !((d >> b) & 1u);
                if (p < L && !lv) perm[p - k] = p;
                if (p >= L && lv) perm[half + k - src0] = p;
                k += lv;
            }
        }
        for (int p = t; p < 64 * act; p += kPlanThreads) ret_orig[p] = orig[p];
        __syncthreads();
        for (int p = L + t; p < 64 * act; p += kPlanThreads) orig[p] = -1;
        for (int i = t; i < K; i += kPlanThreads) orig[perm[i]] = ret_orig[perm[half + i]];
        if (t == 0) ctl[3] = K;
    } else {
        // stable: the live positions in order (perm[new] = old), everything from the first change moves
        int k = base;
        for (int w = w0; w < w1; w++) {
            const uint32_t d = done[w];
            ret_sel[w] = d;
            for (uint32_t x = ~d; x; x &= x - 1) {
                const int p = 32 * w + __ffs(x) - 1;
                perm[k] = p;
                if (p != k) atomicMin(&first_moved, k);
                k++;
            }
        }
        for (int p = t; p < 64 * act; p += kPlanThreads) ret_orig[p] = orig[p];
        __syncthreads();
        for (int p = t; p < 64 * act; p += kPlanThreads) orig[p] = p < L ? ret_orig[perm[p]] : -1;
        if (t == 0) ctl[3] = first_moved == INT32_MAX ? new_act : first_moved / 64;
    }
    // the new done words (positions >= L: padding, stopped)
    for (int w = t; w < NWa; w += kPlanThreads) {
        const int lo = 32 * w;
        done[w] = lo >= L ? 0xffffffffu : (L - lo >= 32 ? 0u : ~((1u << (L - lo)) - 1u));
    }
    if (t == 0) {
        ctl[0] = new_act;
        ctl[1] = 1;
        ctl[2] = L;
    }
}

// The arrays whose rows move (chunk-major [Bp/64][rows][64], 4- or 8-byte elements)
struct MoveArrays {
    void *p[3];
    int32_t rows[3];
    int32_t elem[3];
    int count;
};

constexpr int kMoveBatch = 4;  // output chunks per load/store round of a row warp

// In-place row compaction of one row: new position k takes old position perm[k] (perm[k] >= k).
// Output chunks ascending, kMoveBatch at a time: all loads of a batch, a __syncwarp (a lane may read
// a position another lane of the batch overwrites), then the stores; sources of later batches lie
// at or above their own positions, so above everything stored so far.
template <typename T>
__device__ __forceinline__ void move_row(T *a, int32_t rows, int32_t r, const int32_t *__restrict__ perm, int L,
                                         int oc0, int new_act, int lane) {
    for (int oc = oc0; oc < new_act; oc += kMoveBatch) {
        T v[kMoveBatch][2];
#pragma unroll
        for (int u = 0; u < kMoveBatch; u++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int k = (oc + u) * 64 + 32 * h + lane;
                if (oc + u < new_act && k < L) v[u][h] = a[cofs(rows, r, __ldg(perm + k))];
            }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < kMoveBatch; u++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int k = (oc + u) * 64 + 32 * h + lane;
                if (oc + u < new_act && k < L) a[cofs(rows, r, k)] = v[u][h];
            }
    }
}

// Hole filling of one row: position perm[i] (< L, stopped) takes position perm[half + i] (>= L, live).
// Sources and destinations are disjoint, so no ordering is needed.
template <typename T>
__device__ __forceinline__ void move_fill(T *a, int32_t rows, int32_t r, const int32_t *__restrict__ perm, int half,
                                          int K, int lane) {
    constexpr int U = 4;
    for (int i0 = 0; i0 < K; i0 += 32 * U) {
        T v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int i = i0 + 32 * u + lane;
            if (i < K) v[u] = a[cofs(rows, r, __ldg(perm + half + i))];
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int i = i0 + 32 * u + lane;
            if (i < K) a[cofs(rows, r, __ldg(perm + i))] = v[u];
        }
    }
}

// Everything a compaction point does after its plan, in one launch (exits at once when the plan
// said "no"): warps over
//   [0, T0)        retire estimate bits, one (row block, word) tile each: a 32x32 ballot transpose
//                  of the stopped codewords' bits (as k_pack_rows) into the caller's packed rows
//   [T0, T0 + T1)  retire success / iterations / an all-zero syndrome row, one done word each
//   the rest       move the rows of the state arrays
__global__ void k_compact_apply(const uint32_t *__restrict__ chat, int32_t n, int32_t NWs,
                                const uint32_t *__restrict__ ret_sel, const int32_t *__restrict__ ret_orig,
                                const int32_t *__restrict__ iters_ws, const int32_t *__restrict__ ctl, DecodeOut out,
                                int32_t RWm, int32_t B, const int32_t *__restrict__ perm, MoveArrays arr,
                                int retire, int fill, int half) {
    if (ctl[1] == 0) return;
    const int lane = threadIdx.x & 31;
    const int NWa = 2 * ctl[4];  // the words active before the plan: ret_sel / ret_orig cover exactly those
    const int L = ctl[2], oc0 = ctl[3], new_act = ctl[0];  // oc0: first moved chunk, or the hole count (fill)
    const int RWn = (n + 31) / 32;
    const int64_t T0 = retire ? (int64_t)RWn * NWa : 0, T1 = retire ? NWa : 0;
    int64_t total = T0 + T1;
    for (int i = 0; i < arr.count; i++) total += arr.rows[i];
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < total; g += nwarps) {
        if (g < T0) {
            const int w = (int)(g % NWa), rb = (int)(g / NWa);
            const uint32_t sel = ret_sel[w];
            if (sel == 0) continue;  // warp-uniform
            const int row = rb * 32 + lane;
            const uint32_t x = (row < n) ? chat[(size_t)row * NWs + w] : 0u;
            uint32_t mine = 0;
#pragma unroll
            for (int c = 0; c < 32; c++) {
                const uint32_t y = __ballot_sync(0xffffffffu, (x >> c) & 1u);
                if (lane == c) mine = y;
            }
            if ((sel >> lane) & 1u) {
                const int o = ret_orig[32 * w + lane];
                if (o >= 0 && o < B) out.est[(size_t)o * RWn + rb] = mine;
            }
        } else if (g < T0 + T1) {
            const int w = (int)(g - T0), p = 32 * w + lane;
            if (!((ret_sel[w] >> lane) & 1u)) continue;
            const int o = ret_orig[p];
            if (o < 0 || o >= B) continue;
            out.success[o] = 1;  // stopped <=> all-zero syndrome (serial.py:169,176)
            out.iters[o] = iters_ws[p];
            if (out.syn)
                for (int r = 0; r < RWm; r++) out.syn[(size_t)o * RWm + r] = 0u;
        } else {
            int64_t r = g - T0 - T1;
            int i = 0;
            while (r >= arr.rows[i]) r -= arr.rows[i++];
            if (fill) {  // oc0 = the number of holes filled
                if (arr.elem[i] == 8)
                    move_fill(static_cast<double *>(arr.p[i]), arr.rows[i], (int32_t)r, perm, half, oc0, lane);
                else
                    move_fill(static_cast<float *>(arr.p[i]), arr.rows[i], (int32_t)r, perm, half, oc0, lane);
            } else if (arr.elem[i] == 8) {
                move_row(static_cast<double *>(arr.p[i]), arr.rows[i], (int32_t)r, perm, L, oc0, new_act, lane);
            } else {
                move_row(static_cast<float *>(arr.p[i]), arr.rows[i], (int32_t)r, perm, L, oc0, new_act, lane);
            }
        }
    }
}

// Final outputs through the map: every position that still holds a codeword (orig >= 0).
__global__ void k_pack_rows_mapped(const uint32_t *__restrict__ src, int32_t rows, int32_t NW,
                                   const int32_t *__restrict__ orig, int32_t B, uint32_t *__restrict__ dst) {
    const int lane = threadIdx.x & 31;
    const int RW = (rows + 31) / 32;
    const int64_t tiles = (int64_t)RW * NW;
    for (int64_t t = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); t < tiles;
         t += (int64_t)gridDim.x * (blockDim.x / 32)) {
        const int w = (int)(t % NW), rb = (int)(t / NW);
        const int row = rb * 32 + lane;
        const uint32_t x = (row < rows) ? src[(size_t)row * NW + w] : 0u;
        uint32_t mine = 0;
#pragma unroll
        for (int c = 0; c < 32; c++) {
            const uint32_t y = __ballot_sync(0xffffffffu, (x >> c) & 1u);
            if (lane == c) mine = y;
        }
        const int o = orig[32 * w + lane];
        if (o >= 0 && o < B) dst[(size_t)o * RW + rb] = mine;
    }
}

__global__ void k_finalize_mapped(const uint32_t *done, const int32_t *iters_ws, const int32_t *orig, int32_t Bp,
                                  int32_t B, uint8_t *success, int32_t *iters) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < Bp; p += gridDim.x * blockDim.x) {
        const int o = orig[p];
        if (o < 0 || o >= B) continue;
        success[o] = (done[p >> 5] >> (p & 31)) & 1u;
        iters[o] = iters_ws[p];
    }
}

__global__ void k_compact_init(int32_t *orig, int32_t B, int32_t Bp, int32_t *ctl) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < Bp; p += gridDim.x * blockDim.x) orig[p] = p < B ? p : -1;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctl[0] = Bp / 64;
        ctl[1] = 0;
        ctl[2] = B;
        ctl[3] = 0;
        ctl[4] = Bp / 64;
    }
}

unsigned blocks_of(int64_t work, int threads, int64_t cap = 148 * 16) {
    int64_t b = (work + threads - 1) / threads;
    return (unsigned)std::max<int64_t>(1, std::min(b, cap));
}

// k_compact_apply runs every round and exits at once on most of them, where each block of its grid
// costs dispatch time: one resident wave (SMs x blocks per SM) and a grid-stride loop.
int64_t apply_wave() {
    static const int64_t wave = [] {
        int dev = 0, sms = 148, per = 4;
        if (cudaGetDevice(&dev) == cudaSuccess) {
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_compact_apply, 256, 0);
        }
        cudaGetLastError();
        return (int64_t)std::max(sms, 1) * std::max(per, 1);
    }();
    return wave;
}

// LDPC_COMPACT_MODE=fill|stable: how the live codewords move (default fill)
int compact_fill() {
    static const int v = [] {
        const char *e = getenv("LDPC_COMPACT_MODE");
        return (e && std::string(e) == "stable") ? 0 : 1;
    }();
    return v;
}

}  // namespace

int launch_compact_init(const Workspace &w, cudaStream_t s) {
    k_compact_init<<<blocks_of(w.Bp, 256), 256, 0, s>>>(w.orig, w.B, w.Bp, w.ctl);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

// One compaction point (after the syndrome of a round): the early-stop update and the plan on `s`;
// then the message rows move on `s` (the next check phase reads them) while the retiring of the
// stopped codewords and the other state arrays (priors, read by the next variable phase) move on
// `side` when given (the caller joins it back before that variable phase), else on `s`.
int launch_compact(const ldpc_graph *g, const Workspace &w, int32_t round, int frac_pct, const DecodeOut &out,
                   const CompactArray *arrays, int count, cudaStream_t s, cudaStream_t side,
                   cudaEvent_t fork) {
    LDPC_ARG_CHECK(count >= 1 && count <= 3, "compaction moves 1..3 arrays");
    const int fill = compact_fill();
    k_compact_plan<<<1, kPlanThreads, 0, s>>>(w.done, w.unsat, w.iters, w.NW, round, w.orig, w.ret_orig, w.perm,
                                              w.ret_sel, w.ctl, frac_pct, fill);
    LDPC_CHECK_LAUNCH();
    MoveArrays first{}, rest{};
    first.p[0] = arrays[0].p;
    first.rows[0] = arrays[0].rows;
    first.elem[0] = arrays[0].elem_bytes;
    first.count = 1;
    int64_t rows_rest = 0;
    for (int i = 1; i < count; i++) {
        rest.p[i - 1] = arrays[i].p;
        rest.rows[i - 1] = arrays[i].rows;
        rest.elem[i - 1] = arrays[i].elem_bytes;
        rows_rest += arrays[i].rows;
    }
    rest.count = count - 1;
    cudaStream_t s2 = s;
    if (side != nullptr) {
        LDPC_CUDA_TRY(cudaEventRecord(fork, s));
        LDPC_CUDA_TRY(cudaStreamWaitEvent(side, fork, 0));
        s2 = side;
    }
    const int64_t tiles = (int64_t)((g->n + 31) / 32) * w.NW;
    k_compact_apply<<<blocks_of(32 * std::max<int64_t>(rows_rest, tiles), 256, apply_wave()), 256, 0, s2>>>(
        w.chat, g->n, w.NWs, w.ret_sel, w.ret_orig, w.iters, w.ctl, out, (g->m + 31) / 32, w.B, w.perm, rest, 1, fill, 16 * w.NW);
    LDPC_CHECK_LAUNCH();
    k_compact_apply<<<blocks_of(32 * (int64_t)arrays[0].rows, 256, apply_wave()), 256, 0, s>>>(
        w.chat, g->n, w.NWs, w.ret_sel, w.ret_orig, w.iters, w.ctl, out, (g->m + 31) / 32, w.B, w.perm, first, 0, fill, 16 * w.NW);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

// Final outputs of a compacted decode: estimate and syndrome rows and success / iterations of the
// codewords still mapped to positions.
int launch_compact_finish(const ldpc_graph *g, const Workspace &w, const DecodeOut &out, cudaStream_t s) {
    const int64_t tn = (int64_t)((g->n + 31) / 32) * w.NW;
    k_pack_rows_mapped<<<blocks_of(tn * 32, 256, 148 * 8), 256, 0, s>>>(w.chat, g->n, w.NW, w.orig, w.B, out.est);
    LDPC_CHECK_LAUNCH();
    if (out.syn) {
        const int64_t tm = (int64_t)((g->m + 31) / 32) * w.NW;
        k_pack_rows_mapped<<<blocks_of(tm * 32, 256, 148 * 8), 256, 0, s>>>(w.zb, g->m, w.NW, w.orig, w.B, out.syn);
        LDPC_CHECK_LAUNCH();
    }
    k_finalize_mapped<<<blocks_of(w.Bp, 256), 256, 0, s>>>(w.done, w.iters, w.orig, w.Bp, w.B, out.success, out.iters);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

}  // namespace ldpc
