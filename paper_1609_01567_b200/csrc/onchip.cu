// onchip.cu -- whole-decode-on-chip path for codes whose messages fit in the
// shared memory of one CTA or of a thread-block cluster (DSMEM).
//
// The streaming kernels make one HBM round trip of the message array per
// half-iteration.  For small codes (C1: E = 3,584; C2: E = 28,672) one
// codeword's messages (8 B per edge), priors and hard decisions fit in
// 1 / 2 / 4 / 8 CTAs' shared memory, so a cluster of CS CTAs keeps a codeword
// on chip for ALL its iterations: HBM sees the priors once and the packed
// results once.  Clusters take codewords cw, cw + nclusters, ...
//
// Arithmetic is the reference's, operation for operation (serial.py:63-178;
// same as kernels_check.cu / kernels_var.cu): left-to-right products skipping
// the output's own edge, IEEE division (ddiv_fast + __ddiv_rn fallback),
// estimate tie -> 1, syndrome XOR, early stop with exact iteration counts.
//
// Layout across the cluster (rank r of CS):
//   * checks [cb[r], cb[r+1]) by id, so their message slots [sb[r], sb[r+1])
//     (check-order slots) are contiguous: rank r's smem `msg`;
//   * variables at positions [vb[r], vb[r+1]) of var_order (degree-sorted, so a
//     warp's nodes share a degree): rank r's smem `p` (priors) and `chat`;
//   * a slot or variable of another rank is read / written through DSMEM.
// In-place updates never race: a node reads each of its slots' old value
// before overwriting that slot (the prefix is advanced past slot k before r_k
// / q_k is stored there), and a slot belongs to exactly one check and one
// variable.
//
// Per iteration (serial.py:165-178, two cluster barriers; flags and syndrome rows alternate by parity):
//   VE: chat_t = Est(r_t) and, unless t = max, q_{t+1} = V(p, r_t)  (same pass over r_t)
//   SC: z_t = Syn(chat_t) -> unsat flag, and, unless t = max, r_{t+1} = C(q_{t+1})
//   stop when no rank saw an unsatisfied check (early stop) or t = max.
// r_{t+1} is wasted work when t stops, but it is not an output.
#include <cooperative_groups.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "nodes.cuh"
#include "priors.cuh"

namespace cg = cooperative_groups;

namespace ldpc {

constexpr int kOnchipThreads = 512;   // 128 registers: degree-16 nodes gather into registers without spills
constexpr int kOnchipMaxCS = 8;
constexpr size_t kOnchipSmemBudget = 200 * 1024;

struct OnchipArgs {
    int32_t n, m, B, max_iter, early, RWn, RWm;
    int32_t sb[kOnchipMaxCS + 1];  // slot boundaries per rank
    int32_t cb[kOnchipMaxCS + 1];  // check-id boundaries per rank
    int32_t vb[kOnchipMaxCS + 1];  // var_order position boundaries per rank
    const double *P;               // [B][n] priors (host layout), or observations y when sig2 != nullptr
    const double *sig2;            // [B] noise variances: priors formed on chip (priors.cuh)
    const int32_t *var_off, *var_pos, *var_order, *inv_pos;  // canonical var CSR; slot of edge; order; position of var
    const int32_t *chk_off, *chk_var, *chk_list;              // check CSR over slots; var of slot; checks per rank by degree
    uint32_t *est;      // [B][RWn]
    uint8_t *succ;      // [B]
    int32_t *iters;     // [B]
    uint32_t *syn;      // [B][RWm] or nullptr
};

namespace {

template <int CS>
struct Cl {
    // per rank r (shared-memory tables, so a computed rank index does not spill to local memory)
    double **msg;        // slot sb[r] at msg[r][0]
    double **p;          // position vb[r] at p[r][0]
    uint8_t **chat;
    int **flag;          // [2]: unsat flag by iteration parity
    const OnchipArgs *a;
    __device__ __forceinline__ int slot_rank(int s) const {
        int r = 0;
#pragma unroll
        for (int k = 1; k < CS; k++) r += (s >= a->sb[k]);
        return r;
    }
    __device__ __forceinline__ double *slot(int s) const {
        if (CS == 1) return msg[0] + s;
        const int r = slot_rank(s);
        return msg[r] + (s - a->sb[r]);
    }
    __device__ __forceinline__ int pos_rank(int v) const {
        int r = 0;
#pragma unroll
        for (int k = 1; k < CS; k++) r += (v >= a->vb[k]);
        return r;
    }
    __device__ __forceinline__ double prior_of(int var) const {
        const int pos = __ldg(a->inv_pos + var);
        if (CS == 1) return p[0][pos];
        const int r = pos_rank(pos);
        return p[r][pos - a->vb[r]];
    }
    __device__ __forceinline__ uint8_t chat_of(int var) const {
        const int pos = __ldg(a->inv_pos + var);
        if (CS == 1) return chat[0][pos];
        const int r = pos_rank(pos);
        return chat[r][pos - a->vb[r]];
    }
};

template <int CS>
__device__ __forceinline__ void cluster_barrier() {
    if constexpr (CS == 1) {
        __syncthreads();
    } else {
        cg::this_cluster().sync();
    }
}

// shared-memory layout of a rank: [erow RWn u32][zrow 2 x RWm u32][flag 4 int] (a fixed-size header,
// so rank 0's output rows sit at the same offset in every rank's view) | msg | p | chat
__host__ __device__ __forceinline__ size_t onchip_header(int RWn, int RWm) {
    return ((size_t)(RWn + 2 * RWm + 4) * 4 + 15) & ~(size_t)15;
}

template <int CS>
__global__ void __launch_bounds__(kOnchipThreads) k_onchip(const __grid_constant__ OnchipArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    int rank = 0;
    if constexpr (CS > 1) rank = (int)cg::this_cluster().block_rank();
    const int nclusters = gridDim.x / CS;
    const int cid = blockIdx.x / CS;
    const size_t hdr = onchip_header(a.RWn, a.RWm);
    const int nslots = a.sb[rank + 1] - a.sb[rank];
    const int nvars = a.vb[rank + 1] - a.vb[rank];
    uint32_t *erow = reinterpret_cast<uint32_t *>(sm);  // [RWn] (used on rank 0)
    uint32_t *zrow = erow + a.RWn;                      // [2][RWm] by iteration parity (used on rank 0)
    int *flag = reinterpret_cast<int *>(zrow + 2 * a.RWm);  // [2] unsat flag by iteration parity
    double *msg = reinterpret_cast<double *>(sm + hdr);
    double *pl = msg + nslots;
    uint8_t *chat = reinterpret_cast<uint8_t *>(pl + nvars);
    __shared__ double *t_msg[CS], *t_p[CS];
    __shared__ uint8_t *t_chat[CS];
    __shared__ int *t_flag[CS];
    Cl<CS> cl;
    cl.a = &a;
    cl.msg = t_msg;
    cl.p = t_p;
    cl.chat = t_chat;
    cl.flag = t_flag;
    uint32_t *erow0 = erow, *zrow0 = zrow;  // rank 0's output rows (DSMEM for the other ranks)
    if constexpr (CS == 1) {
        if (threadIdx.x == 0) {
            t_msg[0] = msg;
            t_p[0] = pl;
            t_chat[0] = chat;
            t_flag[0] = flag;
        }
    } else {
        cg::cluster_group clu = cg::this_cluster();
        if (threadIdx.x < CS) {  // rank r's offsets from rank r's sizes
            const int r = threadIdx.x;
            const int ns = a.sb[r + 1] - a.sb[r], nv = a.vb[r + 1] - a.vb[r];
            unsigned char *base = clu.map_shared_rank(sm, r);
            t_flag[r] = reinterpret_cast<int *>(base) + a.RWn + 2 * a.RWm;
            t_msg[r] = reinterpret_cast<double *>(base + hdr);
            t_p[r] = t_msg[r] + ns;
            t_chat[r] = reinterpret_cast<uint8_t *>(t_p[r] + nv);
        }
        erow0 = clu.map_shared_rank(erow, 0);
        zrow0 = clu.map_shared_rank(zrow, 0);
    }
    __syncthreads();
    const int c0 = a.cb[rank], c1 = a.cb[rank + 1];
    const int v0 = a.vb[rank];
    const NodeTables tb{a.chk_off, a.chk_var, a.var_off, a.var_pos};

    for (int cw = cid; cw < a.B; cw += nclusters) {
        // priors of this rank's variables (serial.py:58: q = p[v] feeds the pre-pass)
        const double *Pc = a.P + (size_t)cw * a.n;
        if (a.sig2 == nullptr) {
            for (int i = threadIdx.x; i < nvars; i += blockDim.x) pl[i] = __ldg(Pc + __ldg(a.var_order + v0 + i));
        } else {
            const double s2 = __ldg(a.sig2 + cw);
            for (int i = threadIdx.x; i < nvars; i += blockDim.x)
                pl[i] = awgn_prior(__ldg(Pc + __ldg(a.var_order + v0 + i)), s2);
        }
        if (threadIdx.x < 2) flag[threadIdx.x] = 0;
        if (rank == 0) {
            for (int i = threadIdx.x; i < a.RWn; i += blockDim.x) erow[i] = 0u;
            for (int i = threadIdx.x; i < 2 * a.RWm; i += blockDim.x) zrow[i] = 0u;
        }
        cluster_barrier<CS>();
        // pre-pass C-phase from the priors (serial.py:166)
        for (int i = c0 + threadIdx.x; i < c1; i += blockDim.x) check_node<true>(cl, tb, __ldg(a.chk_list + i));
        cluster_barrier<CS>();
        int t = 0;
        bool success = false;
        for (;; t++) {
            const bool more = t < a.max_iter;
            // VE: estimate of round t and, unless this is the last round, q for round t+1
            for (int i = threadIdx.x; i < nvars; i += blockDim.x)
                chat[i] = var_node(cl, tb, __ldg(a.var_order + v0 + i), more, pl[i]);
            cluster_barrier<CS>();
            // SC: syndrome of round t (+ its bits) and r for round t+1.  The other parity's flag and
            // syndrome row were last read / written before the VE barrier: reset them for round t+1.
            if (threadIdx.x == 0) flag[(t + 1) & 1] = 0;
            if (rank == 0)
                for (int i = threadIdx.x; i < a.RWm; i += blockDim.x) zrow[((t + 1) & 1) * a.RWm + i] = 0u;
            uint32_t *zr = zrow0 + (t & 1) * a.RWm;
            int unsat = 0;
            for (int i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
                const int c = __ldg(a.chk_list + i);
                const int s0 = __ldg(a.chk_off + c), d = __ldg(a.chk_off + c + 1) - s0;
                int z = 0;
                for (int k = 0; k < d; k++) z ^= cl.chat_of(__ldg(a.chk_var + s0 + k));
                unsat |= z;
                if (z && a.syn) atomicOr(zr + (c >> 5), 1u << (c & 31));
                if (more) check_node<false>(cl, tb, c);
            }
            if (__syncthreads_or(unsat) && threadIdx.x == 0) flag[t & 1] = 1;
            cluster_barrier<CS>();
            int any = 0;
#pragma unroll
            for (int r = 0; r < CS; r++) any |= cl.flag[r][t & 1];
            success = !any;
            if ((a.early && success) || !more) break;
        }
        // results (serial.py:169-178): estimate bits of round t, syndrome bits, success, rounds used
        for (int i = threadIdx.x; i < nvars; i += blockDim.x)
            if (chat[i]) {
                const int v = __ldg(a.var_order + v0 + i);
                atomicOr(erow0 + (v >> 5), 1u << (v & 31));
            }
        cluster_barrier<CS>();
        if (rank == 0) {
            for (int i = threadIdx.x; i < a.RWn; i += blockDim.x) a.est[(size_t)cw * a.RWn + i] = erow[i];
            if (a.syn)
                for (int i = threadIdx.x; i < a.RWm; i += blockDim.x) a.syn[(size_t)cw * a.RWm + i] = zrow[(t & 1) * a.RWm + i];
            if (threadIdx.x == 0) {
                a.succ[cw] = success ? 1 : 0;
                a.iters[cw] = (a.early && success) ? t : a.max_iter;
            }
        }
        cluster_barrier<CS>();  // rank 0's rows and every rank's smem are reused by the next codeword
    }
}

// per-(graph, CS) plan: boundaries + check lists, built once on the host from the device tables
struct Plan {
    int CS = 0;
    int32_t sb[kOnchipMaxCS + 1], cb[kOnchipMaxCS + 1], vb[kOnchipMaxCS + 1];
    int32_t *inv_pos = nullptr, *chk_list = nullptr;
    size_t smem = 0;
};
std::mutex g_plan_mu;
std::map<std::pair<const ldpc_graph *, int>, Plan> g_plans;

size_t rank_smem(int nslots, int nvars, int RWn, int RWm) {
    return onchip_header(RWn, RWm) + (size_t)nslots * 8 + (size_t)nvars * 8 + (size_t)nvars;
}

int build_plan(const ldpc_graph *g, int CS, Plan *pl) {
    const int n = g->n, m = g->m;
    std::vector<int32_t> chk_off(m + 1), var_order(n), chk_order(m);
    LDPC_CUDA_TRY(cudaMemcpy(chk_off.data(), g->chk_off, sizeof(int32_t) * (m + 1), cudaMemcpyDeviceToHost));
    LDPC_CUDA_TRY(cudaMemcpy(var_order.data(), g->var_order, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    LDPC_CUDA_TRY(cudaMemcpy(chk_order.data(), g->chk_order, sizeof(int32_t) * m, cudaMemcpyDeviceToHost));
    pl->CS = CS;
    // checks split by id into CS contiguous ranges of ~E/CS slots; variables into CS ranges of var_order
    pl->cb[0] = 0;
    pl->sb[0] = 0;
    for (int r = 1; r < CS; r++) {
        const int64_t target = g->E * r / CS;
        int c = (int)(std::lower_bound(chk_off.begin(), chk_off.end(), (int32_t)target) - chk_off.begin());
        c = std::min(std::max(c, pl->cb[r - 1]), m);
        pl->cb[r] = c;
        pl->sb[r] = chk_off[c];
    }
    pl->cb[CS] = m;
    pl->sb[CS] = (int32_t)g->E;
    for (int r = 0; r <= CS; r++) pl->vb[r] = (int32_t)((int64_t)n * r / CS);
    // each rank's checks in degree order (chk_order is sorted by (degree, id))
    std::vector<int32_t> list;
    list.reserve(m);
    for (int r = 0; r < CS; r++)
        for (int32_t c : chk_order)
            if (c >= pl->cb[r] && c < pl->cb[r + 1]) list.push_back(c);
    std::vector<int32_t> inv(n);
    for (int i = 0; i < n; i++) inv[var_order[i]] = i;
    LDPC_CUDA_TRY(cudaMalloc(&pl->inv_pos, sizeof(int32_t) * n));
    LDPC_CUDA_TRY(cudaMalloc(&pl->chk_list, sizeof(int32_t) * m));
    LDPC_CUDA_TRY(cudaMemcpy(pl->inv_pos, inv.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
    LDPC_CUDA_TRY(cudaMemcpy(pl->chk_list, list.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice));
    const int RWn = (n + 31) / 32, RWm = (m + 31) / 32;
    size_t mx = 0;
    for (int r = 0; r < CS; r++)
        mx = std::max(mx, rank_smem(pl->sb[r + 1] - pl->sb[r], pl->vb[r + 1] - pl->vb[r], RWn, RWm));
    pl->smem = mx;
    return LDPC_OK;
}

}  // namespace

// Smallest cluster size whose per-rank shared memory fits, 0 if none (or the graph
// uses variable-major slots); LDPC_ONCHIP=0 disables the path, =1/2/4/8 forces CS.
// `required`: the caller asked for the on-chip schedule (any degree).
int onchip_cluster_size(const ldpc_graph *g, bool required) {
    static const int forced = [] {
        const char *e = getenv("LDPC_ONCHIP");
        return e ? atoi(e) : -1;
    }();
    if (forced == 0 || g->var_major) return 0;
    // one thread per node with d(d-1)/2 ordered products: chosen automatically only for
    // degrees the streaming register kernels also take (high degrees stream to the chains kernels)
    if (!required && (g->max_dv > kMaxRegDegree || g->max_dc > kMaxRegDegree)) return 0;
    const int RWn = (g->n + 31) / 32, RWm = (g->m + 31) / 32;
    for (int cs : {1, 2, 4, 8}) {
        if (forced > 0 && cs != forced) continue;
        // estimate with even splits plus one max-degree check of slack per rank
        const size_t s = rank_smem((int)(g->E / cs + g->max_dc), (g->n + cs - 1) / cs, RWn, RWm);
        if (s <= kOnchipSmemBudget) return cs;
    }
    return 0;
}

// Automatic choice (measured on B200, profiles/r1_kernel_choice.md): a single CTA per
// codeword beats the streaming schedule up to ~1500 codewords of C1 (0.32 vs 1.08 ms
// for one frame, 50 iterations); clusters lose to streaming (DSMEM latency), so the
// auto schedule takes the on-chip path only at cluster size 1 and B <= 2x the
// resident CTAs.
static int resident_ctas(const ldpc_graph *g) {
    const int RWn = (g->n + 31) / 32, RWm = (g->m + 31) / 32;
    const size_t smem = rank_smem((int)g->E, g->n, RWn, RWm);
    int dev = 0, sms = 0, per_sm = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev))
        return 0;
    cudaFuncSetAttribute(k_onchip<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_onchip<1>, kOnchipThreads, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return sms * per_sm;
}

static std::mutex g_res_mu;
static std::map<const ldpc_graph *, int> g_resident;  // per graph; dropped by onchip_forget

bool onchip_auto(const ldpc_graph *g, int32_t B) {
    if (onchip_cluster_size(g) != 1) return false;
    int res;
    {
        std::lock_guard<std::mutex> lock(g_res_mu);
        auto it = g_resident.find(g);
        if (it == g_resident.end()) it = g_resident.emplace(g, resident_ctas(g)).first;
        res = it->second;
    }
    return B <= 2 * res;
}

int launch_onchip(const ldpc_graph *g, int CS, const double *p_dev, const double *sig2, int32_t B, int32_t max_iter,
                  bool early, uint32_t *est, uint8_t *succ, int32_t *iters, uint32_t *syn, cudaStream_t s) {
    Plan *pl;
    {
        std::lock_guard<std::mutex> lock(g_plan_mu);
        Plan &p = g_plans[{g, CS}];
        if (p.CS == 0) {
            int rc = build_plan(g, CS, &p);
            if (rc) {
                g_plans.erase({g, CS});
                return rc;
            }
        }
        pl = &p;
    }
    LDPC_ARG_CHECK(pl->smem <= kOnchipSmemBudget + 16 * 1024, "on-chip plan needs %zu bytes per CTA", pl->smem);
    OnchipArgs a{};
    a.n = g->n;
    a.m = g->m;
    a.B = B;
    a.max_iter = max_iter;
    a.early = early ? 1 : 0;
    a.RWn = (g->n + 31) / 32;
    a.RWm = (g->m + 31) / 32;
    for (int r = 0; r <= CS; r++) {
        a.sb[r] = pl->sb[r];
        a.cb[r] = pl->cb[r];
        a.vb[r] = pl->vb[r];
    }
    a.P = p_dev;
    a.sig2 = sig2;
    a.var_off = g->var_off;
    a.var_pos = g->var_pos;
    a.var_order = g->var_order;
    a.inv_pos = pl->inv_pos;
    a.chk_off = g->chk_off;
    a.chk_var = g->chk_var;
    a.chk_list = pl->chk_list;
    a.est = est;
    a.succ = succ;
    a.iters = iters;
    a.syn = syn;
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        LDPC_CUDA_TRY(cudaGetDevice(&dev));
        LDPC_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    void (*kern)(const OnchipArgs) = CS == 1 ? k_onchip<1> : CS == 2 ? k_onchip<2> : CS == 4 ? k_onchip<4> : k_onchip<8>;
    LDPC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl->smem));
    int per_sm = 1;
    LDPC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kOnchipThreads, pl->smem));
    per_sm = std::max(per_sm, 1);
    const int clusters = std::max(1, std::min<int>(B, sms * per_sm / CS));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(clusters * CS));
    cfg.blockDim = dim3(kOnchipThreads);
    cfg.dynamicSmemBytes = pl->smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    LDPC_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a));
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

void onchip_forget(const ldpc_graph *g) {
    {
        std::lock_guard<std::mutex> lock(g_res_mu);
        g_resident.erase(g);
    }
    std::lock_guard<std::mutex> lock(g_plan_mu);
    for (auto it = g_plans.begin(); it != g_plans.end();) {
        if (it->first.first == g) {
            cudaFree(it->second.inv_pos);
            cudaFree(it->second.chk_list);
            it = g_plans.erase(it);
        } else {
            ++it;
        }
    }
}

}  // namespace ldpc
