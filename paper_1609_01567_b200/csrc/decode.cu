// decode.cu -- G5: batched decode driver, single-phase entry points, and the
// host-buffer decoder (the C-ABI the Python ParallelDecoder mirror calls).
//
// Phase order (serial.py:150-178 / engine.py:311-347, paper Algorithm 2):
//     r = C(p[v]);  c = Est(p, r);  z = Syn(c);  stop if z == 0      (round 0)
//     for t in 1..I:  q = V(p, r);  r = C(q);  c = Est(p, r);  z = Syn(c);  stop if z == 0
// Kernel sequence used here (Est(t-1) is fused into V(t) because both read the
// same r and p; the final estimate is a V pass without the q write):
//     C0   VE1 [S0 U0]  C1   VE2 [S1 U1]  C2  ...  VE_I [S_{I-1} U_{I-1}]  C_I   E_I  S_I [U_I]
// where S = syndrome + OR-reduced unsatisfied flags and U = early-stop update
// ([..] only in early-stop mode).  A codeword that stops at round t keeps its
// round-t estimate (frozen bits) and iteration count; its later message
// updates are wasted but harmless, and warps whose 32*V codewords have all
// stopped skip their work.  All control stays on the device: no host sync
// between rounds.
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <map>

#include <sched.h>
#include <mutex>
#include <thread>

#include "common.cuh"

namespace ldpc {


namespace {
size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
}  // namespace

// LDPC_GRAPHS=0 disables CUDA-graph replay of decode sequences
bool graphs_enabled() {
    static const bool on = [] {
        const char *e = getenv("LDPC_GRAPHS");
        return !(e && std::string(e) == "0");
    }();
    return on;
}

// Kernel family per (side, degree) for the register-path degrees (<= kMaxRegDegree):
// the cp.async ring (kernels_pipe.cu) or register loads (kernels_check/var.cu).
// Measured on B200 (profiles/r1_kernel_choice.md): the ring wins for every
// variable bucket, register loads for checks (their slots are contiguous).
// LDPC_KERNEL=reg|pipe forces one family (A/B runs).
bool use_ring(bool var_side, int deg) {
    static const int forced = [] {
        const char *e = getenv("LDPC_KERNEL");
        if (e && std::string(e) == "reg") return 1;
        if (e && std::string(e) == "pipe") return 2;
        return 0;
    }();
    if (forced) return forced == 2;
    return var_side && deg >= 2;
}

size_t chain_scratch_doubles(const ldpc_graph *g, int32_t Bp) {
    // per phase: every wide node of the side x its tile x the side's max degree (x2 for r and 1-r)
    size_t wide_c = 0, wide_v = 0;
    for (const Bucket &b : g->chk_buckets)
        if (b.deg > kMaxMidCheckDegree) wide_c += (size_t)b.node_count;
    for (const Bucket &b : g->var_buckets)
        if (b.deg > kMaxMidVarDegree) wide_v += (size_t)b.node_count;
    size_t need = 0;
    if ((size_t)g->max_dc * kChainTW * sizeof(double) > kChainSmemBudget)
        need = std::max(need, wide_c * (size_t)g->max_dc * (size_t)Bp);
    if ((size_t)2 * g->max_dv * kChainTW * sizeof(double) > kChainSmemBudget)
        need = std::max(need, wide_v * (size_t)g->max_dv * 2 * (size_t)Bp);
    return need;
}

size_t workspace_bytes(const ldpc_graph *g, int32_t B) {
    const size_t Bp = (size_t)padded_batch(B), NW = Bp / 32;
    size_t b = 0;
    b += align256(sizeof(double) * chain_scratch_doubles(g, (int32_t)Bp));
    b += align256(sizeof(double) * (size_t)g->E * Bp);
    b += align256(sizeof(double) * (size_t)g->n * Bp);
    b += align256(sizeof(uint32_t) * (size_t)g->n * NW);
    b += align256(sizeof(uint32_t) * (size_t)g->m * NW);
    b += align256(sizeof(uint32_t) * NW) * 2;
    b += align256(sizeof(int32_t) * Bp);
    b += align256(sizeof(float) * (size_t)kOdScratchBlocks * fast_od_scratch_stride(g));
    b += align256(sizeof(int32_t) * Bp) * 3 + align256(sizeof(uint32_t) * NW) + align256(sizeof(int32_t) * 8);
    // the same workspace serves the grid schedule for small batches (codeword-minor, B bytes per variable
    // for the hard decisions)
    if (B <= kGridMaxB) b = std::max(b, grid_workspace_bytes(g, B));
    return b;
}

int carve_workspace(const ldpc_graph *g, int32_t B, void *ws, size_t bytes, Workspace *w) {
    LDPC_ARG_CHECK(B >= 1, "batch must be at least 1");
    const size_t need = workspace_bytes(g, B);
    LDPC_ARG_CHECK(ws != nullptr && bytes >= need, "workspace too small: %zu < %zu bytes", bytes, need);
    LDPC_ARG_CHECK(((uintptr_t)ws & 255) == 0, "workspace must be 256-byte aligned");
    LDPC_ARG_CHECK((uint64_t)g->E * 64 < (1ull << 32) && (uint64_t)g->n * 64 < (1ull << 32),
                   "graph too large: %lld edges (32-bit row offsets need E < 2^26)", (long long)g->E);
    w->B = B;
    w->Bp = padded_batch(B);
    w->NW = w->Bp / 32;
    w->NWs = w->NW;
    char *p = (char *)ws;
    auto take = [&](size_t sz) {
        char *r = p;
        p += align256(sz);
        return r;
    };
    const size_t scratch = chain_scratch_doubles(g, w->Bp);
    w->scratch = scratch ? (double *)take(sizeof(double) * scratch) : nullptr;
    w->msg = (double *)take(sizeof(double) * (size_t)g->E * w->Bp);
    w->P = (double *)take(sizeof(double) * (size_t)g->n * w->Bp);
    w->chat = (uint32_t *)take(sizeof(uint32_t) * (size_t)g->n * w->NW);
    w->zb = (uint32_t *)take(sizeof(uint32_t) * (size_t)g->m * w->NW);
    w->done = (uint32_t *)take(sizeof(uint32_t) * w->NW);
    w->unsat = (uint32_t *)take(sizeof(uint32_t) * w->NW);
    w->iters = (int32_t *)take(sizeof(int32_t) * w->Bp);
    w->od_stride = fast_od_scratch_stride(g);
    w->od_scratch = w->od_stride ? (float *)take(sizeof(float) * (size_t)kOdScratchBlocks * w->od_stride) : nullptr;
    w->orig = (int32_t *)take(sizeof(int32_t) * w->Bp);
    w->ret_orig = (int32_t *)take(sizeof(int32_t) * w->Bp);
    w->perm = (int32_t *)take(sizeof(int32_t) * w->Bp);
    w->ret_sel = (uint32_t *)take(sizeof(uint32_t) * w->NW);
    w->ctl = (int32_t *)take(sizeof(int32_t) * 8);
    return LDPC_OK;
}

Workspace tile_view(const ldpc_graph *g, const Workspace &w, int32_t group0, int32_t groups) {
    // groups of 32 codewords; a multi-group view must start on a 64-codeword chunk so the
    // chunk arithmetic of the kernels (relative to the view base) stays valid
    Workspace v = w;
    const size_t chunk = (size_t)(group0 >> 1), half = (size_t)(group0 & 1) * 32;
    v.msg = w.msg + chunk * (size_t)g->E * 64 + half;
    v.P = w.P + chunk * (size_t)g->n * 64 + half;
    v.chat = w.chat + group0;
    v.zb = w.zb + group0;
    v.done = w.done + group0;
    v.unsat = w.unsat + group0;
    v.iters = w.iters + 32 * (size_t)group0;
    v.Bp = 32 * groups;
    v.B = std::max(0, std::min(w.B - 32 * group0, v.Bp));
    v.NW = groups;
    v.NWs = w.NWs;
    return v;
}

namespace {

constexpr size_t kMaxGraphKeys = 256;  // distinct (pointers, sizes, flags, stream) keys cached per code

// ---- per-kernel-class event timing ------------------------------------------
struct Prof {
    ldpc_profile *out = nullptr;
    cudaStream_t s = nullptr;
    struct Mark {
        int cls;
        cudaEvent_t a, b;
        int64_t bytes;
    };
    std::vector<Mark> marks;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    cudaEvent_t get() {
        if (used == pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            pool.push_back(e);
        }
        return pool[used++];
    }
    cudaEvent_t begin() {
        if (!out) return nullptr;
        cudaEvent_t e = get();
        cudaEventRecord(e, s);
        return e;
    }
    void end(int cls, cudaEvent_t a, int64_t bytes) {
        if (!out) return;
        cudaEvent_t e = get();
        cudaEventRecord(e, s);
        marks.push_back(Mark{cls, a, e, bytes});
    }
    int flush() {
        if (!out || marks.empty()) return LDPC_OK;
        LDPC_CUDA_TRY(cudaEventSynchronize(marks.back().b));
        for (auto &m : marks) {
            float ms = 0.f;
            LDPC_CUDA_TRY(cudaEventElapsedTime(&ms, m.a, m.b));
            out->ms[m.cls] += ms;
            out->launches[m.cls] += 1;
            out->bytes[m.cls] += m.bytes;
        }
        marks.clear();
        used = 0;
        return LDPC_OK;
    }
    ~Prof() {
        for (auto e : pool) cudaEventDestroy(e);
    }
};

#define RUN(cls, bytes, call)                     \
    do {                                          \
        cudaEvent_t _a = prof.begin();            \
        int _rc = (call);                         \
        if (_rc != LDPC_OK) return _rc;           \
        prof.end((cls), _a, (int64_t)(bytes));    \
    } while (0)

NodeLaunch check_args(const ldpc_graph *g, const Workspace &w, const uint32_t *done) {
    return NodeLaunch{g->chk_off, g->chk_var, g->chk_order, 0, 0, w.msg, w.P, nullptr, done, w.Bp, w.NWs,
                      (int32_t)g->E, g->n, g->chk_slot, g->chk_slot_ord, g->chk_var_ord, 0, w.scratch, 0, w.act};
}

NodeLaunch var_args(const ldpc_graph *g, const Workspace &w, const uint32_t *done) {
    return NodeLaunch{g->var_off, nullptr, g->var_order, 0, 0, w.msg, w.P, w.chat, done, w.Bp, w.NWs,
                      (int32_t)g->E, g->n, g->var_slot, g->var_slot_ord, nullptr, 0, w.scratch, 0, w.act};
}

// fp32 fast mode (LDPC_FLAG_FP32): fp32 messages and priors live in the fp64 message buffer
float *msg32(const ldpc_graph *g, const Workspace &w) { return reinterpret_cast<float *>(w.msg); }
float *prior32(const ldpc_graph *g, const Workspace &w) { return reinterpret_cast<float *>(w.msg) + (size_t)g->E * w.Bp; }

// Alternating sweep direction: each node kernel sweeps the codeword chunks opposite to the
// kernel before it, so it starts on the chunk whose rows the previous kernel touched last and
// finds part of them in L2 (C3 step 14.16 -> 14.02 ms with default-caching hints;
// profiles/r1_kernel_choice.md).  LDPC_ALT_SWEEP=0 disables it.
// fp32 fast mode: nodes of degree <= kMaxRegDegree take the fp32 register kernels (the reference's
// product order, kernels_fast.cu); from this degree on the O(d) kernels (kernels_fastod.cu).
// LDPC_FAST_OD=1 sends every degree to the O(d) kernels.
static int fast_od_min_degree() {
    static const int v = [] {
        const char *e = getenv("LDPC_FAST_OD");
        return (e && e[0] == '1') ? 1 : kMaxRegDegree + 1;
    }();
    return v;
}

static bool alt_sweep() {
    static const bool on = [] {
        const char *e = getenv("LDPC_ALT_SWEEP");
        return !(e && e[0] == '0');
    }();
    return on;
}
static thread_local int g_sweep = 0;  // direction of the next node-kernel launch

// ---- launches of one phase: big buckets in order on the calling stream, small ones beside them ----
// A phase is one launch per degree bucket (plus one for the high-degree range).  Memory-bound
// launches of the big buckets stay in order on the calling stream (run side by side they only
// split the bandwidth: profiles/r1_kernel_choice.md); launches of buckets holding less than
// 1/kSmallShare of the edges (latency-bound, a few blocks per SM) and every launch of the mid- and
// high-degree kernels (compute-bound: O(d^2) ordered fp64 products) go to side streams forked from
// and joined back into the calling stream, so they overlap each other and the big ones.  Buckets write disjoint slots and c_hat rows, so the
// order is free.  Also inside CUDA-graph capture (the side streams join the capture through the
// fork event).  LDPC_FORK=0 keeps every launch on the calling stream.
constexpr int kSideStreams = 3;
constexpr int64_t kSmallShare = 8;

struct ForkSet {
    cudaStream_t side[kSideStreams] = {};
    cudaEvent_t fork = nullptr, join[kSideStreams] = {};
};

static bool fork_enabled() {
    static const bool on = [] {
        const char *e = getenv("LDPC_FORK");
        return !(e && e[0] == '0');
    }();
    return on;
}

// the side streams of (device, calling stream), created on first use (never during a capture: the
// first call of a decode sequence runs eagerly); nullptr when unavailable (then sequential)
static ForkSet *fork_set(cudaStream_t s) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, ForkSet> sets;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_pair(dev, s);
    auto it = sets.find(key);
    if (it != sets.end()) return &it->second;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (sets.size() >= 64 || cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
        return nullptr;
    ForkSet f;
    bool ok = cudaEventCreateWithFlags(&f.fork, cudaEventDisableTiming) == cudaSuccess;
    for (int k = 0; k < kSideStreams && ok; k++)
        ok = cudaStreamCreateWithFlags(&f.side[k], cudaStreamNonBlocking) == cudaSuccess &&
             cudaEventCreateWithFlags(&f.join[k], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        return nullptr;
    }
    return &sets.emplace(key, f).first->second;
}

struct PhaseLaunch {
    std::function<int(cudaStream_t)> run;
    bool small;
};

static int run_phase(const std::vector<PhaseLaunch> &L, cudaStream_t s) {
    int n_small = 0;
    for (const auto &x : L) n_small += x.small ? 1 : 0;
    ForkSet *f = (fork_enabled() && n_small > 0 && L.size() > 1) ? fork_set(s) : nullptr;
    if (f == nullptr) {
        for (const auto &x : L)
            if (int rc = x.run(s)) return rc;
        return LDPC_OK;
    }
    LDPC_CUDA_TRY(cudaEventRecord(f->fork, s));
    const int used = std::min(n_small, kSideStreams);
    for (int k = 0; k < used; k++) LDPC_CUDA_TRY(cudaStreamWaitEvent(f->side[k], f->fork, 0));
    int next = 0, rc = LDPC_OK;
    for (const auto &x : L) {  // small ones first, so they start beside the first big launch
        if (!x.small) continue;
        if ((rc = x.run(f->side[next]))) break;
        next = (next + 1) % used;
    }
    for (const auto &x : L) {
        if (rc) break;
        if (!x.small) rc = x.run(s);
    }
    for (int k = 0; k < used; k++) {  // join even after an error, so no stream is left forked
        cudaEventRecord(f->join[k], f->side[k]);
        cudaStreamWaitEvent(s, f->join[k], 0);
    }
    return rc;
}

int check_phase(const ldpc_graph *g, const Workspace &w, bool from_prior, const uint32_t *done, cudaStream_t s,
                bool fast = false) {
    const NodeLaunch a0 = check_args(g, w, done);
    std::vector<PhaseLaunch> L;
    auto small = [&](int64_t edges) { return edges * kSmallShare < g->E; };
    if (fast) {
        for (const Bucket &b : g->chk_buckets) {
            if (b.deg >= fast_od_min_degree()) break;  // buckets are sorted by degree
            NodeLaunch a = a0;
            a.node_begin = b.node_begin;
            a.node_count = b.node_count;
            a.edge_begin = b.edge_begin;
            const int deg = b.deg;
            L.push_back({[=](cudaStream_t st) {
                             return launch_check_f32(a, deg, from_prior, msg32(g, w), prior32(g, w), st);
                         },
                         small((int64_t)b.node_count * b.deg)});
        }
        for (const OdClass &c : fast_od_classes(g->chk_buckets, fast_od_min_degree()))
            L.push_back({[=](cudaStream_t st) {
                             return launch_fast_od_class(a0, c, false, from_prior, msg32(g, w), prior32(g, w),
                                                         w.od_scratch, w.od_stride, kOdScratchBlocks, st);
                         },
                         true});  // O(d) classes: few blocks per SM, latency-bound
        return run_phase(L, s);
    }
    int wide_begin = -1, wide_end = 0, wide_max = 0;
    for (const Bucket &b : g->chk_buckets) {
        if (b.deg <= kMaxMidCheckDegree) {
            NodeLaunch a = a0;
            a.node_begin = b.node_begin;
            a.node_count = b.node_count;
            a.edge_begin = b.edge_begin;
            a.reverse = alt_sweep() ? ((g_sweep ^= 1) ^ 1) : 0;
            const int deg = b.deg;
            L.push_back({[=](cudaStream_t st) {
                             return deg > kMaxRegCheckDegree ? launch_check_mid(a, deg, from_prior, st)
                                    : use_ring(false, deg)    ? launch_check_pipe(a, deg, from_prior, st)
                                                              : launch_check_bucket(a, deg, from_prior, st);
                         },
                         small((int64_t)b.node_count * b.deg) || deg > kMaxRegCheckDegree});
        } else {
            if (wide_begin < 0) wide_begin = b.node_begin;
            wide_end = b.node_begin + b.node_count;
            wide_max = std::max(wide_max, b.deg);
        }
    }
    if (wide_begin >= 0) {  // compute-bound (O(d^2) fp64): beside the memory-bound buckets
        NodeLaunch a = a0;
        a.node_begin = wide_begin;
        a.node_count = wide_end - wide_begin;
        L.push_back({[=](cudaStream_t st) { return launch_check_wide(a, wide_max, from_prior, st); }, true});
    }
    return run_phase(L, s);
}

int var_phase(const ldpc_graph *g, const Workspace &w, bool write_q, const uint32_t *done, cudaStream_t s,
              bool fast = false) {
    const NodeLaunch a0 = var_args(g, w, done);
    std::vector<PhaseLaunch> L;
    auto small = [&](int64_t edges) { return edges * kSmallShare < g->E; };
    if (fast) {
        for (const Bucket &b : g->var_buckets) {
            if (b.deg >= fast_od_min_degree()) break;  // buckets are sorted by degree
            NodeLaunch a = a0;
            a.node_begin = b.node_begin;
            a.node_count = b.node_count;
            a.edge_begin = b.edge_begin;
            const int deg = b.deg;
            L.push_back({[=](cudaStream_t st) {
                             return launch_var_f32(a, deg, write_q, msg32(g, w), prior32(g, w), st);
                         },
                         small((int64_t)b.node_count * b.deg)});
        }
        for (const OdClass &c : fast_od_classes(g->var_buckets, fast_od_min_degree()))
            L.push_back({[=](cudaStream_t st) {
                             return launch_fast_od_class(a0, c, true, write_q, msg32(g, w), nullptr, nullptr, 0, 0,
                                                         st);
                         },
                         true});  // O(d) classes: few blocks per SM, latency-bound
        return run_phase(L, s);
    }
    int wide_begin = -1, wide_end = 0, wide_max = 0;
    for (const Bucket &b : g->var_buckets) {
        if (b.deg <= kMaxMidVarDegree) {
            NodeLaunch a = a0;
            a.node_begin = b.node_begin;
            a.node_count = b.node_count;
            a.edge_begin = b.edge_begin;
            a.reverse = alt_sweep() ? ((g_sweep ^= 1) ^ 1) : 0;
            const int deg = b.deg;
            L.push_back({[=](cudaStream_t st) {
                             return deg > kMaxRegDegree   ? launch_var_mid(a, deg, write_q, st)
                                    : use_ring(true, deg) ? launch_var_pipe(a, deg, write_q, st)
                                                          : launch_var_bucket(a, deg, write_q, st);
                         },
                         small((int64_t)b.node_count * b.deg) || deg > kMaxRegDegree});
        } else {
            if (wide_begin < 0) wide_begin = b.node_begin;
            wide_end = b.node_begin + b.node_count;
            wide_max = std::max(wide_max, b.deg);
        }
    }
    if (wide_begin >= 0) {  // compute-bound (O(d^2) fp64): beside the memory-bound buckets
        NodeLaunch a = a0;
        a.node_begin = wide_begin;
        a.node_count = wide_end - wide_begin;
        L.push_back({[=](cudaStream_t st) { return launch_var_wide(a, wide_max, write_q, st); }, true});
    }
    return run_phase(L, s);
}

// done bits of padded codewords (>= B) are set from the start in early-stop mode
int init_flags(const Workspace &w, bool early, cudaStream_t s, int32_t chat_rows = 0, bool wide_vars = false) {
    LDPC_CUDA_TRY(cudaMemsetAsync(w.unsat, 0, sizeof(uint32_t) * w.NW, s));
    LDPC_CUDA_TRY(cudaMemsetAsync(w.done, 0, sizeof(uint32_t) * w.NW, s));
    if (early) {
        LDPC_CUDA_TRY(cudaMemsetAsync(w.iters, 0, sizeof(int32_t) * w.Bp, s));
        const int full = w.B / 32;
        if (w.B % 32) {
            int rc = launch_fill_u32(w.done + full, ~((1u << (w.B % 32)) - 1u), 1, s);
            if (rc) return rc;
        }
        const int first_pad_word = (w.B + 31) / 32;
        int rc = launch_fill_u32(w.done + first_pad_word, 0xffffffffu, (size_t)(w.NW - first_pad_word), s);
        if (rc) return rc;
    }
    // Estimate words whose old bits are read back get a defined value first (compute-sanitizer
    // initcheck): the bits of stopped codewords are kept (padding codewords are stopped from the
    // start), and high-degree tiles narrower than a word update their bits with atomics.
    if (chat_rows > 0 && ((early && w.B != w.Bp) || wide_vars))
        LDPC_CUDA_TRY(cudaMemsetAsync(w.chat, 0, sizeof(uint32_t) * (size_t)chat_rows * w.NWs, s));
    return LDPC_OK;
}

}  // namespace

// The compaction's side stream of (device, calling stream): its own stream and events, apart from the
// phase side streams (created eagerly like those; nullptr during a capture that has none yet)
struct CompactFork {
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
static CompactFork *compact_fork(cudaStream_t s) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, CompactFork> sets;
    if (!fork_enabled()) return nullptr;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_pair(dev, s);
    auto it = sets.find(key);
    if (it != sets.end()) return &it->second;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (sets.size() >= 64 || cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
        return nullptr;
    CompactFork f;
    if (cudaStreamCreateWithFlags(&f.side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&f.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&f.join, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return &sets.emplace(key, f).first->second;
}

// Early-stop compaction (compact.cu): compact when the live codewords fit in at most this percent
// of the active chunks; LDPC_COMPACT=0 disables it, LDPC_COMPACT=<pct> sets the threshold.
static int compact_pct() {
    static const int v = [] {
        const char *e = getenv("LDPC_COMPACT");
        return e ? std::max(0, std::min(100, atoi(e))) : 80;
    }();
    return v;
}

// Algorithm 2 (serial.py:165-178) on one view of the workspace: the whole batch
// (streaming schedule) or one tile (tiled schedule).  `out` != nullptr: early stop with
// compaction, retired codewords' results written to the caller's outputs as they stop.
static int decode_view(const ldpc_graph *g, const Workspace &w, int32_t max_iter, bool early, cudaStream_t s,
                       Prof &prof, bool fast, const DecodeOut *out = nullptr) {
    g_sweep = 0;  // every decode (and so every captured graph) uses the same direction sequence
    const int64_t B = w.B, E = g->E, n = g->n, m = g->m;
    const int64_t wb = fast ? 4 : 8;                         // message / prior width in bytes
    const int64_t c_bytes = 2 * wb * E * B;                  // read q (or p-gather) + write r
    const int64_t ve_bytes = (2 * wb * E + wb * n + n / 8) * B; // read r, p; write q, c_hat bits
    const int64_t e_bytes = (wb * E + wb * n + n / 8) * B;   // read r, p; write c_hat bits
    const int64_t s_bytes = (n / 8) * B;                     // read c_hat bits
    const uint32_t *done = early ? w.done : nullptr;
    CompactFork *cf = nullptr;
    RUN(LDPC_KCLASS_CHECK, c_bytes, check_phase(g, w, true, nullptr, s, fast));
    for (int32_t t = 1; t <= max_iter; t++) {
        RUN(LDPC_KCLASS_VARIABLE, ve_bytes, var_phase(g, w, true, done, s, fast));
        if (early) {
            RUN(LDPC_KCLASS_SYNDROME, s_bytes, launch_syndrome(g, w, false, true, s));
            if (out == nullptr) RUN(LDPC_KCLASS_SYNDROME, 0, launch_update_done(w, t - 1, false, s));
        }
        if (out != nullptr) {  // (the compaction plan does the early-stop update of round t - 1 first)
            // the state that crosses into round t: q (messages) and the priors
            // (the fp32 fast mode moves its fp32 messages and priors, and the fp64 priors its O(d)
            // variable kernels read)
            const CompactArray exact[2] = {{w.msg, (int32_t)E, 8}, {w.P, (int32_t)n, 8}};
            const CompactArray f32[3] = {{msg32(g, w), (int32_t)E, 4}, {prior32(g, w), (int32_t)n, 4}, {w.P, (int32_t)n, 8}};
            // the priors move and the stopped codewords retire beside the check phase (joined before
            // the next variable phase, which reads both); eager profiling keeps one stream
            cf = prof.out == nullptr ? compact_fork(s) : nullptr;
            if (cf == nullptr) {
                RUN(LDPC_KCLASS_LAYOUT, 0, launch_compact(g, w, t - 1, compact_pct(), *out, fast ? f32 : exact,
                                                          fast ? 3 : 2, s));
            } else {
                // (no profiling here: prof is inactive whenever the side stream is used)
                int rc = launch_compact(g, w, t - 1, compact_pct(), *out, fast ? f32 : exact, fast ? 3 : 2, s,
                                        cf->side, cf->fork);
                if (rc == LDPC_OK) rc = check_phase(g, w, false, done, s, fast);
                // join even after an error, so no stream is left forked (a capture could not end)
                const cudaError_t e1 = cudaEventRecord(cf->join, cf->side);
                const cudaError_t e2 = cudaStreamWaitEvent(s, cf->join, 0);
                cf = nullptr;
                if (rc) return rc;
                LDPC_CUDA_TRY(e1);
                LDPC_CUDA_TRY(e2);
                continue;
            }
        }
        RUN(LDPC_KCLASS_CHECK, c_bytes, check_phase(g, w, false, done, s, fast));
    }
    RUN(LDPC_KCLASS_ESTIMATE, e_bytes, var_phase(g, w, false, done, s, fast));
    RUN(LDPC_KCLASS_SYNDROME, s_bytes + (m / 8) * B, launch_syndrome(g, w, true, early, s));
    if (early) RUN(LDPC_KCLASS_SYNDROME, 0, launch_update_done(w, max_iter, true, s));
    return LDPC_OK;
}

// Tiled (L2-resident) schedule, OFF by default: instead of sweeping every phase
// over the whole batch (each half-iteration one HBM round trip of the 1.86 GB
// message array at C3), run ALL iterations of one tile of codewords before the
// next, the tile's messages + priors sized to stay in the 126 MB L2.  Codewords
// are independent, so results are bit-identical to the streaming schedule.
// Measured on B200 (profiles/r1_kernel_choice.md): pure data movement gains
// 1.33x in this pattern, but the node kernels become issue-bound on a 32-codeword
// tile (the deg-8 variable kernel needs ~4.8 us of instruction issue per tile at
// IPC 1 vs 6.3 us of L2 traffic), so C3 runs at 18.8 ms tiled vs 14.2 ms
// streaming.  Kept as an experiment switch: LDPC_TILE=k runs tiles of k
// 32-codeword groups (even when >= 2 so views stay chunk-aligned).
static int32_t tile_groups(const ldpc_graph *g, const Workspace &w, bool fast) {
    static const int forced = [] {
        const char *e = getenv("LDPC_TILE");
        return e ? atoi(e) : 0;
    }();
    (void)g;
    if (fast || forced <= 0) return 0;
    const int32_t groups = (w.B + 31) / 32;
    int32_t T = forced;
    if (T >= 2) T &= ~1;
    return std::min(T, groups);
}

// The decode proper on a carved workspace whose P is filled, then the caller's outputs.
int run_decode(const ldpc_graph *g, const Workspace &w, int32_t max_iter, bool early, cudaStream_t s, Prof &prof,
               bool fast, const DecodeOut &out) {
    int rc = init_flags(w, early, s, g->n, g->max_dv > kMaxMidVarDegree);
    if (rc) return rc;
    if (fast) {
        rc = launch_priors_to_f32(w.P, prior32(g, w), (size_t)g->n * w.Bp, s);
        if (rc) return rc;
    }
    const int32_t T = tile_groups(g, w, fast);
    const int64_t n = g->n, m = g->m, B = w.B;
    if (T == 0 && early && compact_pct() > 0 && w.Bp > kBatchAlign) {
        RUN(LDPC_KCLASS_LAYOUT, 0, launch_compact_init(w, s));
        Workspace wc = w;
        wc.act = w.ctl;  // node kernels cover the active chunks only
        if ((rc = decode_view(g, wc, max_iter, early, s, prof, fast, &out))) return rc;
        RUN(LDPC_KCLASS_LAYOUT, (n / 8) * 2 * B + (out.syn ? (m / 8) * 2 * B : 0), launch_compact_finish(g, w, out, s));
        return LDPC_OK;
    }
    if (T == 0) {
        rc = decode_view(g, w, max_iter, early, s, prof, fast);
    } else {
        const int32_t groups = (w.B + 31) / 32;
        for (int32_t g0 = 0; g0 < groups && rc == LDPC_OK; g0 += T)
            rc = decode_view(g, tile_view(g, w, g0, std::min(T, groups - g0)), max_iter, early, s, prof, fast);
    }
    if (rc) return rc;
    RUN(LDPC_KCLASS_LAYOUT, (n / 8) * 2 * B, launch_pack_rows(w.chat, g->n, w.NW, w.B, out.est, s));
    if (out.syn) RUN(LDPC_KCLASS_LAYOUT, (m / 8) * 2 * B, launch_pack_rows(w.zb, g->m, w.NW, w.B, out.syn, s));
    RUN(LDPC_KCLASS_LAYOUT, 0, launch_finalize(w, early, max_iter, out.success, out.iters, s));
    return LDPC_OK;
}

}  // namespace ldpc

using namespace ldpc;

extern "C" size_t ldpc_workspace_bytes(const ldpc_graph *g, int32_t B) {
    if (!g || B < 1) return 0;
    return workspace_bytes(g, B);
}

// grid schedule by default for B <= kGridMaxB while its working set stays well inside the L2
// (LDPC_GRID=0 disables the automatic choice)
// grid vs stream, device time per decode (tools/grid_vs_stream.py, 2 dB, early stop, 50 rounds):
// C3 B = 16 1.45 vs 4.15 ms, B = 32 2.67 vs 4.16 ms (75 MB working set); C2 B = 32 0.35 vs 1.46 ms
constexpr size_t kGridAutoBytes = 96ull << 20;
static bool grid_auto() {
    static const bool on = [] {
        const char *e = getenv("LDPC_GRID");
        return !(e && e[0] == '0');
    }();
    return on;
}

// p_dev: priors [B][n]; or, with sig2 != nullptr, observations y [B][n] whose priors are
// formed inside the layout transpose (priors.cuh).
static int decode_impl(const ldpc_graph *g, const double *p_dev, const double *sig2, int32_t B, int32_t max_iterations,
                       uint32_t flags, uint32_t *est_bits_dev, uint8_t *success_dev, int32_t *iters_dev,
                       uint32_t *syn_bits_dev, void *workspace_dev, size_t workspace_bytes_, void *stream,
                       ldpc_profile *prof_host) {
    LDPC_ARG_CHECK(g != nullptr, "NULL graph");
    DeviceGuard dg(g->device);
    LDPC_ARG_CHECK(max_iterations >= 0, "max_iterations must be non-negative");
    LDPC_ARG_CHECK(p_dev && est_bits_dev && success_dev && iters_dev, "NULL output/input pointer");
    LDPC_ARG_CHECK((flags & ~(LDPC_FLAG_FIXED_ITERS | LDPC_FLAG_FP32 | LDPC_FLAG_STREAMING | LDPC_FLAG_ONCHIP |
                              LDPC_FLAG_GRID)) == 0,
                   "unknown flags 0x%x", flags);
    const bool fast = (flags & LDPC_FLAG_FP32) != 0;
    LDPC_ARG_CHECK(__builtin_popcount(flags & (LDPC_FLAG_STREAMING | LDPC_FLAG_ONCHIP | LDPC_FLAG_GRID)) <= 1,
                   "at most one schedule flag");
    cudaStream_t s = (cudaStream_t)stream;
    const bool early = !(flags & LDPC_FLAG_FIXED_ITERS);
    // a few codewords of a code too large for the on-chip schedule: one cooperative launch (grid.cu)
    const bool want_grid = (flags & LDPC_FLAG_GRID) != 0;
    LDPC_ARG_CHECK(!want_grid || (!fast && grid_suitable(g, B)),
                   "the grid schedule takes 1..%d codewords of a code with node degrees <= %d (fp64)", kGridMaxB,
                   kMaxRegDegree);
    // small codes: the whole decode on chip (onchip.cu), unless the caller forces streaming
    const bool want_onchip = (flags & LDPC_FLAG_ONCHIP) != 0;
    const int cs = (fast || (flags & (LDPC_FLAG_STREAMING | LDPC_FLAG_GRID))) ? 0
                   : want_onchip ? onchip_cluster_size(g, true) : (onchip_auto(g, B) ? 1 : 0);
    LDPC_ARG_CHECK(!(flags & LDPC_FLAG_ONCHIP) || (cs > 0 && !(flags & LDPC_FLAG_STREAMING)),
                   "the on-chip schedule needs a code whose messages fit 8 CTAs' shared memory (fp64)");
    if (cs > 0 && prof_host == nullptr) {
        LDPC_ARG_CHECK(B >= 1, "batch must be at least 1");
        return launch_onchip(g, cs, p_dev, sig2, B, max_iterations, early, est_bits_dev, success_dev, iters_dev,
                             syn_bits_dev, s);
    }
    if (prof_host == nullptr && !fast && !(flags & (LDPC_FLAG_STREAMING | LDPC_FLAG_ONCHIP)) &&
        (want_grid || (grid_auto() && grid_suitable(g, B) && grid_workspace_bytes(g, B) <= kGridAutoBytes))) {
        LDPC_ARG_CHECK(workspace_dev != nullptr, "NULL workspace");
        return launch_grid(g, p_dev, sig2, B, max_iterations, early, est_bits_dev, success_dev, iters_dev,
                           syn_bits_dev, workspace_dev, workspace_bytes_, s);
    }
    Workspace w;
    int rc = carve_workspace(g, B, workspace_dev, workspace_bytes_, &w);
    if (rc) return rc;
    auto sequence = [&](Prof &prof) -> int {
        const int64_t n = g->n, m = g->m;
        RUN(LDPC_KCLASS_LAYOUT, 16 * n * B, launch_transpose_priors(p_dev, sig2, B, g->n, w.P, w.Bp, s));
        return run_decode(g, w, max_iterations, early, s, prof, fast,
                          DecodeOut{est_bits_dev, success_dev, iters_dev, syn_bits_dev});
    };
    Prof prof;
    prof.out = prof_host;
    prof.s = s;
    if (prof_host == nullptr && s != nullptr && graphs_enabled()) {
        // Replay the whole sequence (~50 dependent launches at C3) as one CUDA
        // graph: captured on the second call with the same pointers and sizes
        // (the first call runs eagerly and initialises every launcher), then
        // launched from the cache.
        auto *gg = const_cast<ldpc_graph *>(g);
        const ldpc_graph::GraphKey key{p_dev, sig2, B, max_iterations, flags, est_bits_dev, success_dev, iters_dev,
                                       syn_bits_dev, workspace_dev, stream};
        std::shared_ptr<ldpc_graph::GraphEntry> entry;
        bool capture = false;
        cudaGraphExec_t exec_now = nullptr;
        long long exec_kernels = 0;
        {
            std::lock_guard<std::mutex> lock(gg->graphs_mu);
            auto it = gg->graphs.find(key);
            if (it == gg->graphs.end()) {
                if (gg->graphs.size() >= kMaxGraphKeys) {
                    // bounded: drop keys that never repeated, then the least recently used captured
                    // ones (an evicted entry a caller still holds lives on through its shared_ptr)
                    for (auto e = gg->graphs.begin(); e != gg->graphs.end();)
                        e = (e->second->exec == nullptr && !e->second->capturing) ? gg->graphs.erase(e) : std::next(e);
                    while (gg->graphs.size() >= kMaxGraphKeys) {
                        auto lru = gg->graphs.end();
                        for (auto e = gg->graphs.begin(); e != gg->graphs.end(); ++e)
                            if (!e->second->capturing && (lru == gg->graphs.end() ||
                                                          e->second->last_use < lru->second->last_use))
                                lru = e;
                        if (lru == gg->graphs.end()) break;
                        gg->graphs.erase(lru);
                    }
                }
                it = gg->graphs.emplace(key, std::make_shared<ldpc_graph::GraphEntry>()).first;
            }
            entry = it->second;
            entry->uses++;
            entry->last_use = ++gg->graph_clock;
            if (entry->exec == nullptr && !entry->capturing && entry->uses >= 2) capture = entry->capturing = true;
            exec_now = entry->exec;
            exec_kernels = entry->kernels;
        }
        if (capture) {
            cudaGraph_t graph = nullptr;
            const long long k0 = ldpc_kernel_launches();
            cudaError_t ce = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
            int r = LDPC_OK;
            if (ce == cudaSuccess) {
                r = sequence(prof);
                ce = cudaStreamEndCapture(s, &graph);
            }
            const long long kernels = ldpc_kernel_launches() - k0;
            count_launches(-kernels);  // captured, not executed
            cudaGraphExec_t exec = nullptr;
            if (r == LDPC_OK && ce == cudaSuccess && graph != nullptr) ce = cudaGraphInstantiate(&exec, graph, 0);
            if (graph) cudaGraphDestroy(graph);
            {
                std::lock_guard<std::mutex> lock(gg->graphs_mu);
                entry->capturing = false;
                if (exec) {
                    entry->exec = exec;
                    entry->kernels = kernels;
                }
            }
            if (r != LDPC_OK) return r;
            if (exec == nullptr) {
                cudaGetLastError();
                set_error("graph capture: %s", cudaGetErrorString(ce));
                return LDPC_ECUDA;
            }
            exec_now = exec;
            exec_kernels = kernels;
        }
        if (exec_now != nullptr) {  // entry (held above) keeps exec_now alive through the launch
            LDPC_CUDA_TRY(cudaGraphLaunch(exec_now, s));
            count_launches(exec_kernels);
            return LDPC_OK;
        }
    }
    rc = sequence(prof);
    if (rc) return rc;
    return prof.flush();
}

extern "C" int ldpc_decode(const ldpc_graph *g, const double *p_dev, int32_t B, int32_t max_iterations,
                           uint32_t flags, uint32_t *est_bits_dev, uint8_t *success_dev, int32_t *iters_dev,
                           uint32_t *syn_bits_dev, void *workspace_dev, size_t workspace_bytes_, void *stream,
                           ldpc_profile *prof_host) {
    return decode_impl(g, p_dev, nullptr, B, max_iterations, flags, est_bits_dev, success_dev, iters_dev,
                       syn_bits_dev, workspace_dev, workspace_bytes_, stream, prof_host);
}

extern "C" int ldpc_decode_awgn(const ldpc_graph *g, const double *y_dev, const double *sigma2_dev, int32_t B,
                                int32_t max_iterations, uint32_t flags, uint32_t *est_bits_dev, uint8_t *success_dev,
                                int32_t *iters_dev, uint32_t *syn_bits_dev, void *workspace_dev,
                                size_t workspace_bytes_, void *stream, ldpc_profile *prof_host) {
    LDPC_ARG_CHECK(sigma2_dev != nullptr, "NULL sigma2");
    return decode_impl(g, y_dev, sigma2_dev, B, max_iterations, flags, est_bits_dev, success_dev, iters_dev,
                       syn_bits_dev, workspace_dev, workspace_bytes_, stream, prof_host);
}

// f1: channel prologue on the device (noise + priors), then the same decode sequence
extern "C" int ldpc_decode_channel(const ldpc_graph *g, uint64_t seed, uint64_t point, uint64_t frame0, int32_t B,
                                   double sigma2, int32_t max_iterations, uint32_t flags, uint32_t *est_bits_dev,
                                   uint8_t *success_dev, int32_t *iters_dev, uint32_t *syn_bits_dev,
                                   void *workspace_dev, size_t workspace_bytes_, void *stream) {
    LDPC_ARG_CHECK(g != nullptr, "NULL graph");
    DeviceGuard dg(g->device);
    LDPC_ARG_CHECK(max_iterations >= 0, "max_iterations must be non-negative");
    LDPC_ARG_CHECK(sigma2 > 0.0, "sigma2 must be positive");
    LDPC_ARG_CHECK(est_bits_dev && success_dev && iters_dev, "NULL output pointer");
    LDPC_ARG_CHECK((flags & ~(LDPC_FLAG_FIXED_ITERS | LDPC_FLAG_FP32 | LDPC_FLAG_STREAMING | LDPC_FLAG_ONCHIP)) == 0,
                   "unknown flags 0x%x", flags);
    const bool fast = (flags & LDPC_FLAG_FP32) != 0;
    cudaStream_t s = (cudaStream_t)stream;
    const bool early = !(flags & LDPC_FLAG_FIXED_ITERS);
    // (device-generated priors land chunk-major, so this path always streams)
    LDPC_ARG_CHECK(!(flags & LDPC_FLAG_ONCHIP), "decode_channel runs the streaming schedule");
    Workspace w;
    int rc = carve_workspace(g, B, workspace_dev, workspace_bytes_, &w);
    if (rc) return rc;
    Prof prof;
    if ((rc = launch_channel_priors(seed, point, frame0, B, g->n, sigma2, w.P, w.Bp, s))) return rc;
    return run_decode(g, w, max_iterations, early, s, prof, fast,
                      DecodeOut{est_bits_dev, success_dev, iters_dev, syn_bits_dev});
}

extern "C" int ldpc_count_errors(const ldpc_graph *g, const uint32_t *est_bits_dev, const uint8_t *success_dev,
                                 const int32_t *iters_dev, int32_t B, int64_t *counts_dev, void *stream) {
    LDPC_ARG_CHECK(g && est_bits_dev && success_dev && iters_dev && counts_dev, "NULL argument");
    DeviceGuard dg(g->device);
    LDPC_ARG_CHECK(B >= 1, "batch must be at least 1");
    return launch_count_errors(est_bits_dev, (g->n + 31) / 32, success_dev, iters_dev, B, counts_dev,
                               (cudaStream_t)stream);
}

// ---- single phases -----------------------------------------------------------
extern "C" int ldpc_phase_to_variable(const ldpc_graph *g, const double *q_dev, double *r_dev, int32_t B,
                                      void *ws, size_t ws_bytes, void *stream) {
    LDPC_ARG_CHECK(g && q_dev && r_dev, "NULL argument");
    DeviceGuard dg(g->device);
    Workspace w;
    int rc = carve_workspace(g, B, ws, ws_bytes, &w);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    if ((rc = launch_canon_to_slots(g, q_dev, B, w.msg, w.Bp, s))) return rc;
    if ((rc = check_phase(g, w, false, nullptr, s))) return rc;
    return launch_slots_to_canon(g, w.msg, w.Bp, r_dev, B, s);
}

extern "C" int ldpc_phase_to_check(const ldpc_graph *g, const double *p_dev, const double *r_dev, double *q_dev,
                                   int32_t B, void *ws, size_t ws_bytes, void *stream) {
    LDPC_ARG_CHECK(g && p_dev && r_dev && q_dev, "NULL argument");
    DeviceGuard dg(g->device);
    Workspace w;
    int rc = carve_workspace(g, B, ws, ws_bytes, &w);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    if ((rc = launch_transpose_priors(p_dev, nullptr, B, g->n, w.P, w.Bp, s))) return rc;
    if ((rc = launch_canon_to_slots(g, r_dev, B, w.msg, w.Bp, s))) return rc;
    if ((rc = var_phase(g, w, true, nullptr, s))) return rc;
    return launch_slots_to_canon(g, w.msg, w.Bp, q_dev, B, s);
}

extern "C" int ldpc_phase_estimate(const ldpc_graph *g, const double *p_dev, const double *r_dev,
                                   uint8_t *chat_dev, int32_t B, void *ws, size_t ws_bytes, void *stream) {
    LDPC_ARG_CHECK(g && p_dev && r_dev && chat_dev, "NULL argument");
    DeviceGuard dg(g->device);
    Workspace w;
    int rc = carve_workspace(g, B, ws, ws_bytes, &w);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    if ((rc = launch_transpose_priors(p_dev, nullptr, B, g->n, w.P, w.Bp, s))) return rc;
    if ((rc = launch_canon_to_slots(g, r_dev, B, w.msg, w.Bp, s))) return rc;
    if ((rc = var_phase(g, w, false, nullptr, s))) return rc;
    return launch_bits_to_bytes(w.chat, g->n, w.NW, B, chat_dev, s);
}

extern "C" int ldpc_phase_syndrome(const ldpc_graph *g, const uint8_t *chat_dev, uint8_t *z_dev, int32_t B,
                                   void *ws, size_t ws_bytes, void *stream) {
    LDPC_ARG_CHECK(g && chat_dev && z_dev, "NULL argument");
    DeviceGuard dg(g->device);
    Workspace w;
    int rc = carve_workspace(g, B, ws, ws_bytes, &w);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    if ((rc = launch_bytes_to_bits(chat_dev, B, g->n, w.chat, w.NW, s))) return rc;
    LDPC_CUDA_TRY(cudaMemsetAsync(w.unsat, 0, sizeof(uint32_t) * w.NW, s));
    if ((rc = launch_syndrome(g, w, true, false, s))) return rc;
    return launch_bits_to_bytes(w.zb, g->m, w.NW, B, z_dev, s);
}

// fp32 fast-mode single phases (message tolerance tests): inputs/outputs fp64 canonical order
extern "C" int ldpc_phase_f32(const ldpc_graph *g, int phase, const double *p_dev, const double *in_dev,
                              double *out_dev, int32_t B, void *ws, size_t ws_bytes, void *stream) {
    LDPC_ARG_CHECK(g && in_dev && out_dev && (phase == 1 || p_dev), "NULL argument");
    DeviceGuard dg(g->device);
    LDPC_ARG_CHECK(phase == 0 || phase == 1, "phase must be 0 (to check) or 1 (to variable)");
    Workspace w;
    int rc = carve_workspace(g, B, ws, ws_bytes, &w);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    if (phase == 0) {
        if ((rc = launch_transpose_priors(p_dev, nullptr, B, g->n, w.P, w.Bp, s))) return rc;
        if ((rc = launch_priors_to_f32(w.P, prior32(g, w), (size_t)g->n * w.Bp, s))) return rc;
    }
    if ((rc = launch_canon_to_slots_f32(g, in_dev, B, msg32(g, w), w.Bp, s))) return rc;
    rc = phase == 0 ? var_phase(g, w, true, nullptr, s, true) : check_phase(g, w, false, nullptr, s, true);
    if (rc) return rc;
    return launch_slots_to_canon_f32(g, msg32(g, w), w.Bp, out_dev, B, s);
}

// ---- host-buffer decoder: pipelined H2D / decode / D2H ------------------------
// Device input and output buffers cover the whole max_batch, so every
// sub-batch's H2D copy is enqueued up front on the copy stream (one event per
// sub-batch) before the host spends time enqueuing decode launches; each
// sub-batch waits for its own copy and the output stream returns its packed
// results as soon as it is decoded.  Sub-batches grow geometrically (64, 96,
// 144, ... up to `sub`) so the pipeline fill -- the first H2D, which nothing
// overlaps -- stays short.  Consecutive sub-batches alternate between two
// compute streams with their own workspaces, so a small sub-batch's kernel
// tails are filled by the next one instead of idling SMs (a lone 64-codeword
// decode runs ~20% below the full-batch rate).
namespace {
constexpr int kMaxChunks = 64;
constexpr int kLanes = 4;         // compute streams available
constexpr int kDefaultLanes = 2;  // used by default (LDPC_E2E_LANES=1..4 overrides)
int e2e_lanes() {
    static const int v = [] {
        const char *e = getenv("LDPC_E2E_LANES");
        const int x = e ? atoi(e) : kDefaultLanes;
        return x < 1 ? 1 : (x > kLanes ? kLanes : x);
    }();
    return v;
}
}

// Host threads that copy between pageable (user) and pinned (staging) memory in parallel slices;
// the calling thread copies the first slice itself.
struct CopyPool {
    std::vector<std::thread> th;
    std::mutex mu;
    std::condition_variable go, fin;
    char *dst = nullptr;
    const char *src = nullptr;
    size_t bytes = 0;
    uint64_t gen = 0;
    int pending = 0;
    bool stop = false;

    int parts() const { return (int)th.size() + 1; }
    void slice(int i, char *d, const char *s, size_t n) const {
        const size_t per = (n / parts() + 4095) & ~(size_t)4095;
        const size_t lo = std::min(n, per * i), hi = std::min(n, lo + per);
        if (hi > lo) memcpy(d + lo, s + lo, hi - lo);
    }
    void start(int workers) {
        for (int i = 1; i <= workers; i++)
            th.emplace_back([this, i] {
                uint64_t seen = 0;
                for (;;) {
                    std::unique_lock<std::mutex> lk(mu);
                    go.wait(lk, [&] { return stop || gen != seen; });
                    if (stop) return;
                    seen = gen;
                    char *d = dst;
                    const char *s = src;
                    const size_t n = bytes;
                    lk.unlock();
                    slice(i, d, s, n);
                    lk.lock();
                    if (--pending == 0) fin.notify_one();
                }
            });
    }
    void copy(void *d, const void *s, size_t n) {
        if (th.empty() || n < (1u << 20)) {
            memcpy(d, s, n);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(mu);
            dst = static_cast<char *>(d);
            src = static_cast<const char *>(s);
            bytes = n;
            pending = (int)th.size();
            gen++;
        }
        go.notify_all();
        slice(0, static_cast<char *>(d), static_cast<const char *>(s), n);
        std::unique_lock<std::mutex> lk(mu);
        fin.wait(lk, [&] { return pending == 0; });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu);
            stop = true;
        }
        go.notify_all();
        for (auto &t : th) t.join();
    }
};

struct ldpc_decoder {
    // pageable host buffers (plain numpy arrays): inputs staged through pinned slots by the copy
    // pool, overlapped with the H2D DMA of the previous slot; results land in pinned buffers and
    // are copied out at the end (allocated on first pageable use)
    static constexpr int kStages = 3;
    static constexpr size_t kStageBytes = 16u << 20;
    void *stage[kStages] = {};
    cudaEvent_t stage_free[kStages] = {};
    int stage_next = 0;
    uint32_t *est_pin = nullptr, *syn_pin = nullptr;
    uint8_t *succ_pin = nullptr;
    int32_t *its_pin = nullptr;
    CopyPool pool;
    const ldpc_graph *g = nullptr;
    int32_t max_batch = 0, sub = 0;
    cudaStream_t s_in = nullptr, s_out = nullptr;
    cudaStream_t s_comp[kLanes] = {};  // sub-batch i decodes on s_comp[i % lanes] ...
    void *ws[kLanes] = {};             // ... in workspace ws[i % lanes]
    int lanes = 1;
    size_t ws_bytes = 0;
    double *p = nullptr;      // [max_batch][n] priors or observations
    double *s2 = nullptr;     // [max_batch] noise variances (observation input)
    uint32_t *est = nullptr;  // [max_batch][RWn]
    uint32_t *syn = nullptr;  // [max_batch][RWm]
    uint8_t *succ = nullptr;  // [max_batch]
    int32_t *its = nullptr;   // [max_batch]
    cudaEvent_t in_ready[kMaxChunks] = {}, decoded[kMaxChunks] = {};
    // streaming slots (ldpc_decoder_submit / wait), allocated on first use
    struct Slot {
        double *p = nullptr, *s2 = nullptr;
        uint32_t *est = nullptr, *syn = nullptr;
        uint8_t *succ = nullptr;
        int32_t *its = nullptr;
        cudaEvent_t in_done = nullptr, dec_done = nullptr, out_done = nullptr;
        int64_t ticket = -1;  // in flight when >= 0
    } slots[2];
    void *ws_full = nullptr;  // workspace for a whole max_batch decode
    size_t ws_full_bytes = 0;
    int64_t next_ticket = 0;
    bool poisoned = false;
    std::mutex mu;
};

static void decoder_free(ldpc_decoder *d) {
    if (!d) return;
    DeviceGuard dg(d->g->device);
    for (cudaStream_t s : {d->s_in, d->s_comp[0], d->s_comp[1], d->s_comp[2], d->s_comp[3], d->s_out})
        if (s) cudaStreamSynchronize(s);
    for (void *w : d->ws) cudaFree(w);
    cudaFree(d->ws_full);
    for (auto &sl : d->slots) {
        cudaFree(sl.p);
        cudaFree(sl.s2);
        cudaFree(sl.est);
        cudaFree(sl.syn);
        cudaFree(sl.succ);
        cudaFree(sl.its);
        for (cudaEvent_t e : {sl.in_done, sl.dec_done, sl.out_done})
            if (e) cudaEventDestroy(e);
    }
    cudaFree(d->p);
    cudaFree(d->s2);
    cudaFree(d->est);
    cudaFree(d->syn);
    cudaFree(d->succ);
    cudaFree(d->its);
    for (int i = 0; i < kMaxChunks; i++)
        for (cudaEvent_t e : {d->in_ready[i], d->decoded[i]})
            if (e) cudaEventDestroy(e);
    for (int k = 0; k < ldpc_decoder::kStages; k++) {
        if (d->stage[k]) cudaFreeHost(d->stage[k]);
        if (d->stage_free[k]) cudaEventDestroy(d->stage_free[k]);
    }
    for (void *h : {(void *)d->est_pin, (void *)d->syn_pin, (void *)d->succ_pin, (void *)d->its_pin})
        if (h) cudaFreeHost(h);
    for (cudaStream_t s : {d->s_in, d->s_comp[0], d->s_comp[1], d->s_comp[2], d->s_comp[3], d->s_out})
        if (s) cudaStreamDestroy(s);
    delete d;
}

// Sub-batch sizes for a batch of B: multiples of 64 codewords (the kernels pad a
// batch to a multiple of 64, so e.g. 96 would cost the work of 128), growing
// geometrically from 64 (LDPC_E2E_GROWTH, x100, default 150), capped at `sub`; a
// remainder smaller than the sub-batch before it is merged into that one, since
// the last decode is exposed after the last copy.
static std::vector<int32_t> chunk_plan(int32_t B, int32_t sub, bool taper = false) {
    static const int growth = [] {
        const char *e = getenv("LDPC_E2E_GROWTH");
        return e ? std::max(101, atoi(e)) : 150;
    }();
    // experiment hook: LDPC_E2E_PLAN="64,64,128,..." (sizes in order; the last one repeats)
    static const std::vector<int32_t> fixed = [] {
        std::vector<int32_t> f;
        if (const char *e = getenv("LDPC_E2E_PLAN"))
            for (const char *q = e; *q;) {
                const int x = atoi(q);
                if (x > 0) f.push_back(x);
                while (*q && *q != ',') q++;
                if (*q == ',') q++;
            }
        return f;
    }();
    std::vector<int32_t> v;
    if (!fixed.empty()) {
        for (int32_t c0 = 0, i = 0; c0 < B; i++) {
            int32_t take = std::min<int32_t>(fixed[std::min<size_t>(i, fixed.size() - 1)], B - c0);
            if ((int)v.size() == kMaxChunks - 1) take = B - c0;
            v.push_back(take);
            c0 += take;
        }
        return v;
    }
    const int32_t cap = std::max<int32_t>(64, sub / 64 * 64);
    int32_t b = std::min<int32_t>(cap, 64);
    for (int32_t c0 = 0; c0 < B;) {
        int32_t take = std::min(b, B - c0);
        if ((int)v.size() == kMaxChunks - 1) take = B - c0;  // keep within the event budget
        v.push_back(take);
        c0 += take;
        b = std::min<int32_t>(cap, std::max<int32_t>(b + 64, (b * growth / 100) / 64 * 64));
    }
    if (v.size() >= 2 && v.back() < v[v.size() - 2]) {
        v[v.size() - 2] += v.back();
        v.pop_back();
    }
    // taper (pageable input, whose host staging runs slower than the DMA): the last sub-batch's
    // decode is exposed after its input lands, so end on a small one (C3 B = 1024: 64, 128, 192,
    // 256, 384 -> ..., 256, 128: 18.3 -> 16.1 ms per call; tools/pageable_probe.py)
    constexpr int32_t kTail = 128;
    if (taper && v.back() > kTail && (int)v.size() < kMaxChunks) {
        v.back() -= kTail;
        v.push_back(kTail);
    }
    return v;
}

extern "C" int ldpc_decoder_create(const ldpc_graph *g, int32_t max_batch, int32_t sub_batch, ldpc_decoder **out) {
    LDPC_ARG_CHECK(g && out, "NULL argument");
    DeviceGuard dg(g->device);
    LDPC_ARG_CHECK(max_batch >= 1, "max_batch must be at least 1");
    *out = nullptr;
    ldpc_decoder *d = new ldpc_decoder();
    d->g = g;
    d->max_batch = max_batch;
    d->sub = sub_batch > 0 ? std::min(sub_batch, max_batch) : std::min(max_batch, 512);
    // the largest sub-batch the plan produces for ANY batch the decoder accepts: a smaller batch
    // can merge its remainder into a larger last chunk than max_batch's plan has (e.g. B = 800 with
    // sub = 512: 64, 128, 192, 416), so take the maximum over every b <= max_batch
    int32_t biggest = 0;
    for (int32_t b = max_batch; b >= 1 && biggest < max_batch; b--)
        for (bool taper : {false, true})
            for (int32_t x : chunk_plan(b, d->sub, taper)) biggest = std::max(biggest, x);
    d->ws_bytes = workspace_bytes(g, biggest);
    const size_t RWn = (g->n + 31) / 32, RWm = (g->m + 31) / 32, MB = (size_t)max_batch;
    cudaError_t e = cudaSuccess;
    d->lanes = chunk_plan(max_batch, d->sub).size() > 1 ? e2e_lanes() : 1;
    for (cudaStream_t *s : {&d->s_in, &d->s_out})
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
    for (int l = 0; l < d->lanes && e == cudaSuccess; l++) {
        e = cudaStreamCreateWithFlags(&d->s_comp[l], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaMalloc(&d->ws[l], d->ws_bytes);
    }
    if (e == cudaSuccess) e = cudaMalloc((void **)&d->p, sizeof(double) * (size_t)g->n * MB);
    if (e == cudaSuccess) e = cudaMalloc((void **)&d->s2, sizeof(double) * MB);
    if (e == cudaSuccess) e = cudaMalloc((void **)&d->est, sizeof(uint32_t) * RWn * MB);
    if (e == cudaSuccess) e = cudaMalloc((void **)&d->syn, sizeof(uint32_t) * RWm * MB);
    if (e == cudaSuccess) e = cudaMalloc((void **)&d->succ, MB);
    if (e == cudaSuccess) e = cudaMalloc((void **)&d->its, sizeof(int32_t) * MB);
    for (int i = 0; i < kMaxChunks && e == cudaSuccess; i++)
        for (cudaEvent_t *ev : {&d->in_ready[i], &d->decoded[i]})
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        set_error("decoder allocation: %s", cudaGetErrorString(e));
        decoder_free(d);
        return e == cudaErrorMemoryAllocation ? LDPC_ENOMEM : LDPC_ECUDA;
    }
    *out = d;
    return LDPC_OK;
}

static bool host_pinned(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

static int staging_alloc(ldpc_decoder *d) {
    // complete or nothing: a failed allocation is retried by the next pageable call (whatever was
    // allocated stays owned by the decoder and is freed with it)
    bool done = d->its_pin != nullptr;
    for (int k = 0; k < ldpc_decoder::kStages; k++) done = done && d->stage[k] && d->stage_free[k];
    if (done) return LDPC_OK;
    const size_t MB = (size_t)d->max_batch, RWn = (d->g->n + 31) / 32, RWm = (d->g->m + 31) / 32;
    for (int k = 0; k < ldpc_decoder::kStages; k++) {
        if (!d->stage[k]) LDPC_CUDA_TRY(cudaHostAlloc(&d->stage[k], ldpc_decoder::kStageBytes, cudaHostAllocDefault));
        if (!d->stage_free[k]) LDPC_CUDA_TRY(cudaEventCreateWithFlags(&d->stage_free[k], cudaEventDisableTiming));
    }
    if (!d->est_pin) LDPC_CUDA_TRY(cudaHostAlloc((void **)&d->est_pin, sizeof(uint32_t) * RWn * MB, cudaHostAllocDefault));
    if (!d->syn_pin) LDPC_CUDA_TRY(cudaHostAlloc((void **)&d->syn_pin, sizeof(uint32_t) * RWm * MB, cudaHostAllocDefault));
    if (!d->succ_pin) LDPC_CUDA_TRY(cudaHostAlloc((void **)&d->succ_pin, MB, cudaHostAllocDefault));
    if (!d->its_pin) LDPC_CUDA_TRY(cudaHostAlloc((void **)&d->its_pin, sizeof(int32_t) * MB, cudaHostAllocDefault));
    if (!d->pool.th.empty()) return LDPC_OK;
    // copy threads: every CPU this process may run on (the rank's NUMA-local set when bound), capped
    // at 16; LDPC_COPY_THREADS overrides
    cpu_set_t cs;
    int ncpu = (sched_getaffinity(0, sizeof(cs), &cs) == 0) ? CPU_COUNT(&cs) : (int)std::thread::hardware_concurrency();
    if (const char *e = getenv("LDPC_COPY_THREADS")) ncpu = atoi(e);
    d->pool.start(std::max(0, std::min(16, ncpu) - 1));  // + the calling thread
    return LDPC_OK;
}

// pageable host -> device through the pinned slots: copy a slot's piece on the host threads once its
// previous DMA is done, then its DMA on the copy stream (the next piece's host copy overlaps it)
static cudaError_t stage_in(ldpc_decoder *d, void *dst_dev, const void *src_host, size_t bytes) {
    for (size_t off = 0; off < bytes; off += ldpc_decoder::kStageBytes) {
        const size_t len = std::min(ldpc_decoder::kStageBytes, bytes - off);
        const int k = d->stage_next;
        d->stage_next = (k + 1) % ldpc_decoder::kStages;
        cudaError_t e = cudaEventSynchronize(d->stage_free[k]);
        if (e != cudaSuccess) return e;
        d->pool.copy(d->stage[k], static_cast<const char *>(src_host) + off, len);
        e = cudaMemcpyAsync(static_cast<char *>(dst_dev) + off, d->stage[k], len, cudaMemcpyHostToDevice, d->s_in);
        if (e == cudaSuccess) e = cudaEventRecord(d->stage_free[k], d->s_in);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

static int decoder_run(ldpc_decoder *d, const double *p_host, const double *s2_host, int32_t B,
                       int32_t max_iterations, uint32_t flags, uint32_t *est_bits_host, uint8_t *success_host,
                       int32_t *iters_host, uint32_t *syn_bits_host) {
    if (d == nullptr) {
        set_error("decoder is closed");
        return LDPC_ECLOSED;
    }
    std::lock_guard<std::mutex> lock(d->mu);
    DeviceGuard dg(d->g->device);
    if (d->poisoned) {
        set_error("decoder is closed after a device fault");
        return LDPC_ECLOSED;
    }
    LDPC_ARG_CHECK(p_host && est_bits_host && success_host && iters_host, "NULL argument");
    LDPC_ARG_CHECK(B >= 1 && B <= d->max_batch, "batch %d outside 1..%d", B, d->max_batch);
    LDPC_ARG_CHECK(max_iterations >= 0, "max_iterations must be non-negative");
    const ldpc_graph *g = d->g;
    const size_t n = g->n, RWn = (g->n + 31) / 32, RWm = (g->m + 31) / 32;
    // Plain (pageable) host arrays, as the reference API's callers pass them (engine.py:363-372), go
    // through pinned staging: a pageable cudaMemcpyAsync would be staged by the driver one
    // synchronous piece at a time.
    const bool in_pinned = host_pinned(p_host);  // (sigma2, B doubles, is copied as it is)
    const std::vector<int32_t> plan = chunk_plan(B, d->sub, !in_pinned);
    int rc = LDPC_OK;
    cudaError_t e = cudaSuccess;
    auto cuda = [&](cudaError_t x, const char *what) {
        if (x != cudaSuccess && e == cudaSuccess) {
            e = x;
            set_error("%s: %s", what, cudaGetErrorString(x));
        }
    };
    const bool out_pinned = host_pinned(est_bits_host) && host_pinned(success_host) && host_pinned(iters_host) &&
                            (syn_bits_host == nullptr || host_pinned(syn_bits_host));
    if (!in_pinned || !out_pinned) {
        rc = staging_alloc(d);
        if (rc) return rc;
    }
    uint32_t *est_dst = out_pinned ? est_bits_host : d->est_pin;
    uint8_t *succ_dst = out_pinned ? success_host : d->succ_pin;
    int32_t *its_dst = out_pinned ? iters_host : d->its_pin;
    uint32_t *syn_dst = (out_pinned || syn_bits_host == nullptr) ? syn_bits_host : d->syn_pin;
    // 1. pinned input: every H2D copy, back to back on the copy stream
    if (s2_host)
        cuda(cudaMemcpyAsync(d->s2, s2_host, sizeof(double) * B, cudaMemcpyHostToDevice, d->s_in), "H2D sigma2");
    if (in_pinned)
        for (size_t i = 0, c0 = 0; i < plan.size(); c0 += plan[i], i++) {
            cuda(cudaMemcpyAsync(d->p + c0 * n, p_host + c0 * n, sizeof(double) * n * plan[i], cudaMemcpyHostToDevice,
                                 d->s_in), s2_host ? "H2D observations" : "H2D priors");
            cuda(cudaEventRecord(d->in_ready[i], d->s_in), "record");
        }
    // 2. decodes in order, each results copy right behind its decode (pageable input: each
    //    sub-batch staged just before its decode is enqueued)
    for (size_t i = 0, c0 = 0; i < plan.size() && rc == LDPC_OK && e == cudaSuccess; c0 += plan[i], i++) {
        const int32_t b = plan[i];
        const int l = (int)(i % d->lanes);
        if (!in_pinned) {
            cuda(stage_in(d, d->p + c0 * n, p_host + c0 * n, sizeof(double) * n * b), "H2D (staged)");
            cuda(cudaEventRecord(d->in_ready[i], d->s_in), "record");
        }
        cuda(cudaStreamWaitEvent(d->s_comp[l], d->in_ready[i], 0), "wait input");
        if (e != cudaSuccess) break;
        rc = decode_impl(g, d->p + c0 * n, s2_host ? d->s2 + c0 : nullptr, b, max_iterations, flags,
                         d->est + c0 * RWn, d->succ + c0, d->its + c0, syn_bits_host ? d->syn + c0 * RWm : nullptr,
                         d->ws[l], d->ws_bytes, d->s_comp[l], nullptr);
        if (rc) break;
        cuda(cudaEventRecord(d->decoded[i], d->s_comp[l]), "record");
        cuda(cudaStreamWaitEvent(d->s_out, d->decoded[i], 0), "wait decode");
        cuda(cudaMemcpyAsync(est_dst + c0 * RWn, d->est + c0 * RWn, sizeof(uint32_t) * RWn * b,
                             cudaMemcpyDeviceToHost, d->s_out), "D2H estimate");
        cuda(cudaMemcpyAsync(succ_dst + c0, d->succ + c0, b, cudaMemcpyDeviceToHost, d->s_out), "D2H success");
        cuda(cudaMemcpyAsync(its_dst + c0, d->its + c0, sizeof(int32_t) * b, cudaMemcpyDeviceToHost, d->s_out),
             "D2H iterations");
        if (syn_bits_host)
            cuda(cudaMemcpyAsync(syn_dst + c0 * RWm, d->syn + c0 * RWm, sizeof(uint32_t) * RWm * b,
                                 cudaMemcpyDeviceToHost, d->s_out), "D2H syndrome");
    }
    for (cudaStream_t s : {d->s_in, d->s_comp[0], d->s_comp[1], d->s_comp[2], d->s_comp[3], d->s_out})
        if (s) cuda(cudaStreamSynchronize(s), "decode");
    if (!out_pinned && rc == LDPC_OK && e == cudaSuccess) {
        d->pool.copy(est_bits_host, est_dst, sizeof(uint32_t) * RWn * B);
        memcpy(success_host, succ_dst, (size_t)B);
        memcpy(iters_host, its_dst, sizeof(int32_t) * B);
        if (syn_bits_host) d->pool.copy(syn_bits_host, syn_dst, sizeof(uint32_t) * RWm * B);
    }
    if (rc == LDPC_OK && e != cudaSuccess) rc = LDPC_ECUDA;
    if (rc == LDPC_ECUDA) d->poisoned = true;  // mirrors engine.py:389-392: refuse further use
    return rc;
}

extern "C" int ldpc_decoder_decode_host(ldpc_decoder *d, const double *p_host, int32_t B, int32_t max_iterations,
                                        uint32_t flags, uint32_t *est_bits_host, uint8_t *success_host,
                                        int32_t *iters_host, uint32_t *syn_bits_host) {
    return decoder_run(d, p_host, nullptr, B, max_iterations, flags, est_bits_host, success_host, iters_host,
                       syn_bits_host);
}

extern "C" int ldpc_decoder_decode_awgn_host(ldpc_decoder *d, const double *y_host, const double *sigma2_host,
                                             int32_t B, int32_t max_iterations, uint32_t flags,
                                             uint32_t *est_bits_host, uint8_t *success_host, int32_t *iters_host,
                                             uint32_t *syn_bits_host) {
    LDPC_ARG_CHECK(sigma2_host != nullptr, "NULL sigma2");
    return decoder_run(d, y_host, sigma2_host, B, max_iterations, flags, est_bits_host, success_host, iters_host,
                       syn_bits_host);
}

// ---- streaming: submit / wait ---------------------------------------------------
static int slot_finish(ldpc_decoder *d, ldpc_decoder::Slot &sl) {
    if (sl.ticket < 0) return LDPC_OK;
    const cudaError_t e = cudaEventSynchronize(sl.out_done);
    sl.ticket = -1;
    if (e != cudaSuccess) {
        set_error("decode: %s", cudaGetErrorString(e));
        d->poisoned = true;
        return LDPC_ECUDA;
    }
    return LDPC_OK;
}

static int slots_alloc(ldpc_decoder *d) {
    if (d->slots[0].p != nullptr) return LDPC_OK;
    const ldpc_graph *g = d->g;
    const size_t RWn = (g->n + 31) / 32, RWm = (g->m + 31) / 32, MB = (size_t)d->max_batch;
    cudaError_t e = cudaSuccess;
    d->ws_full_bytes = workspace_bytes(g, d->max_batch);
    e = cudaMalloc(&d->ws_full, d->ws_full_bytes);
    for (auto &sl : d->slots) {
        if (e == cudaSuccess) e = cudaMalloc((void **)&sl.p, sizeof(double) * (size_t)g->n * MB);
        if (e == cudaSuccess) e = cudaMalloc((void **)&sl.s2, sizeof(double) * MB);
        if (e == cudaSuccess) e = cudaMalloc((void **)&sl.est, sizeof(uint32_t) * RWn * MB);
        if (e == cudaSuccess) e = cudaMalloc((void **)&sl.syn, sizeof(uint32_t) * RWm * MB);
        if (e == cudaSuccess) e = cudaMalloc((void **)&sl.succ, MB);
        if (e == cudaSuccess) e = cudaMalloc((void **)&sl.its, sizeof(int32_t) * MB);
        for (cudaEvent_t *ev : {&sl.in_done, &sl.dec_done, &sl.out_done})
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        set_error("streaming slots: %s", cudaGetErrorString(e));
        cudaGetLastError();
        return e == cudaErrorMemoryAllocation ? LDPC_ENOMEM : LDPC_ECUDA;
    }
    return LDPC_OK;
}

static int decoder_submit(ldpc_decoder *d, const double *p_host, const double *s2_host, int32_t B,
                          int32_t max_iterations, uint32_t flags, uint32_t *est_bits_host, uint8_t *success_host,
                          int32_t *iters_host, uint32_t *syn_bits_host, int64_t *ticket) {
    if (d == nullptr) {
        set_error("decoder is closed");
        return LDPC_ECLOSED;
    }
    std::lock_guard<std::mutex> lock(d->mu);
    DeviceGuard dg(d->g->device);
    if (d->poisoned) {
        set_error("decoder is closed after a device fault");
        return LDPC_ECLOSED;
    }
    LDPC_ARG_CHECK(p_host && est_bits_host && success_host && iters_host && ticket, "NULL argument");
    LDPC_ARG_CHECK(B >= 1 && B <= d->max_batch, "batch %d outside 1..%d", B, d->max_batch);
    LDPC_ARG_CHECK(max_iterations >= 0, "max_iterations must be non-negative");
    int rc = slots_alloc(d);
    if (rc) return rc;
    const int64_t k = d->next_ticket;
    auto &sl = d->slots[k & 1];
    if ((rc = slot_finish(d, sl))) return rc;  // the slot's previous batch (ticket k - 2) is home
    const ldpc_graph *g = d->g;
    const size_t n = g->n, RWn = (g->n + 31) / 32, RWm = (g->m + 31) / 32;
    cudaStream_t sc = d->s_comp[0];
    cudaError_t e = cudaSuccess;
    auto cuda = [&](cudaError_t x, const char *what) {
        if (x != cudaSuccess && e == cudaSuccess) {
            e = x;
            set_error("%s: %s", what, cudaGetErrorString(x));
        }
    };
    if (s2_host) cuda(cudaMemcpyAsync(sl.s2, s2_host, sizeof(double) * B, cudaMemcpyHostToDevice, d->s_in), "H2D sigma2");
    cuda(cudaMemcpyAsync(sl.p, p_host, sizeof(double) * n * B, cudaMemcpyHostToDevice, d->s_in), "H2D input");
    cuda(cudaEventRecord(sl.in_done, d->s_in), "record");
    cuda(cudaStreamWaitEvent(sc, sl.in_done, 0), "wait input");
    if (e == cudaSuccess)
        rc = decode_impl(g, sl.p, s2_host ? sl.s2 : nullptr, B, max_iterations, flags, sl.est, sl.succ, sl.its,
                         syn_bits_host ? sl.syn : nullptr, d->ws_full, d->ws_full_bytes, sc, nullptr);
    if (rc == LDPC_OK && e == cudaSuccess) {
        cuda(cudaEventRecord(sl.dec_done, sc), "record");
        cuda(cudaStreamWaitEvent(d->s_out, sl.dec_done, 0), "wait decode");
        cuda(cudaMemcpyAsync(est_bits_host, sl.est, sizeof(uint32_t) * RWn * B, cudaMemcpyDeviceToHost, d->s_out),
             "D2H estimate");
        cuda(cudaMemcpyAsync(success_host, sl.succ, B, cudaMemcpyDeviceToHost, d->s_out), "D2H success");
        cuda(cudaMemcpyAsync(iters_host, sl.its, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, d->s_out),
             "D2H iterations");
        if (syn_bits_host)
            cuda(cudaMemcpyAsync(syn_bits_host, sl.syn, sizeof(uint32_t) * RWm * B, cudaMemcpyDeviceToHost,
                                 d->s_out), "D2H syndrome");
        cuda(cudaEventRecord(sl.out_done, d->s_out), "record");
    }
    if (rc == LDPC_OK && e != cudaSuccess) rc = LDPC_ECUDA;
    if (rc == LDPC_ECUDA) {
        d->poisoned = true;
        return rc;
    }
    if (rc) return rc;
    sl.ticket = k;
    d->next_ticket = k + 1;
    *ticket = k;
    return LDPC_OK;
}

extern "C" int ldpc_decoder_submit(ldpc_decoder *d, const double *p_host, int32_t B, int32_t max_iterations,
                                   uint32_t flags, uint32_t *est_bits_host, uint8_t *success_host,
                                   int32_t *iters_host, uint32_t *syn_bits_host, int64_t *ticket) {
    return decoder_submit(d, p_host, nullptr, B, max_iterations, flags, est_bits_host, success_host, iters_host,
                          syn_bits_host, ticket);
}

extern "C" int ldpc_decoder_submit_awgn(ldpc_decoder *d, const double *y_host, const double *sigma2_host, int32_t B,
                                        int32_t max_iterations, uint32_t flags, uint32_t *est_bits_host,
                                        uint8_t *success_host, int32_t *iters_host, uint32_t *syn_bits_host,
                                        int64_t *ticket) {
    LDPC_ARG_CHECK(sigma2_host != nullptr, "NULL sigma2");
    return decoder_submit(d, y_host, sigma2_host, B, max_iterations, flags, est_bits_host, success_host, iters_host,
                          syn_bits_host, ticket);
}

extern "C" int ldpc_decoder_wait(ldpc_decoder *d, int64_t ticket) {
    if (d == nullptr) {
        set_error("decoder is closed");
        return LDPC_ECLOSED;
    }
    std::lock_guard<std::mutex> lock(d->mu);
    DeviceGuard dg(d->g->device);
    LDPC_ARG_CHECK(ticket >= 0 && ticket < d->next_ticket, "unknown ticket %lld", (long long)ticket);
    auto &sl = d->slots[ticket & 1];
    if (sl.ticket != ticket) return d->poisoned ? LDPC_ECLOSED : LDPC_OK;  // already collected
    return slot_finish(d, sl);
}

extern "C" void ldpc_decoder_destroy(ldpc_decoder *d) { decoder_free(d); }
