// graph.cu -- G1: device builder of the edge tables and degree buckets.
//
// Replaces the reference's table construction (tables.py:50-116) and matrix
// validation (codes.py:42-61).  Both edge orders are produced by sorting
// unique 64-bit keys on the device:
//   canonical (variable) order: key = col << 32 | (m-1-row)  -> columns ascending,
//                               rows DESCENDING inside a column (tables.py:66-77)
//   check order:                key = row << 32 | col        -> rows ascending,
//                               canonical index ascending inside a row, which is
//                               the stable argsort of tables.py:88 (within one row
//                               the canonical index grows with the column).
// Degrees come from atomic counts, offsets from an exclusive scan, the slot of
// every canonical edge from a binary search in its column, and the degree
// buckets from a sort of (degree << 32 | node).  Keys are unique, so the
// (non-stable) bitonic sort yields one deterministic result.
#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <atomic>

#include "common.cuh"

namespace ldpc {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void count_launches(long long k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

void set_error(const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
}

namespace {

// ---- bitonic sort of uint64 keys (N a power of two) ------------------------
constexpr int kLocal = 2048;  // elements sorted per block in shared memory

__device__ __forceinline__ void cmp_swap(uint64_t &a, uint64_t &b, bool ascending) {
    if ((a > b) == ascending) {
        uint64_t t = a;
        a = b;
        b = t;
    }
}

// Full bitonic sort of each L-element chunk (stages k = 2..L), directions from the
// global index so the chunks form the input of the global merge stages.
__global__ void k_bitonic_local_sort(uint64_t *keys, int L) {
    extern __shared__ uint64_t s[];
    const size_t base = (size_t)blockIdx.x * L;
    for (int i = threadIdx.x; i < L; i += blockDim.x) s[i] = keys[base + i];
    __syncthreads();
    for (int k = 2; k <= L; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int t = threadIdx.x; t < L / 2; t += blockDim.x) {
                int i = 2 * t - (t & (j - 1));
                bool asc = (((base + i) & (size_t)k) == 0);
                cmp_swap(s[i], s[i + j], asc);
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < L; i += blockDim.x) keys[base + i] = s[i];
}

// Stages j = L/2 .. 1 of merge level k, chunk-local.
__global__ void k_bitonic_local_merge(uint64_t *keys, size_t k, int L) {
    extern __shared__ uint64_t s[];
    const size_t base = (size_t)blockIdx.x * L;
    for (int i = threadIdx.x; i < L; i += blockDim.x) s[i] = keys[base + i];
    __syncthreads();
    const bool asc = ((base & k) == 0);  // whole chunk shares the direction (k > L)
    for (int j = L >> 1; j > 0; j >>= 1) {
        for (int t = threadIdx.x; t < L / 2; t += blockDim.x) {
            int i = 2 * t - (t & (j - 1));
            cmp_swap(s[i], s[i + j], asc);
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < L; i += blockDim.x) keys[base + i] = s[i];
}

__global__ void k_bitonic_global_step(uint64_t *keys, size_t half, size_t j, size_t k) {
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < half; t += (size_t)gridDim.x * blockDim.x) {
        size_t i = 2 * t - (t & (j - 1));
        uint64_t a = keys[i], b = keys[i + j];
        bool asc = ((i & k) == 0);
        if ((a > b) == asc) {
            keys[i] = b;
            keys[i + j] = a;
        }
    }
}

int sort_u64(uint64_t *keys, size_t N, cudaStream_t s) {
    if (N < 2) return LDPC_OK;
    const int L = (int)std::min<size_t>(N, kLocal);
    const int threads = std::min(L / 2, 1024);
    k_bitonic_local_sort<<<(unsigned)(N / L), threads, L * sizeof(uint64_t), s>>>(keys, L);
    LDPC_CHECK_LAUNCH();
    for (size_t k = 2 * (size_t)L; k <= N; k <<= 1) {
        for (size_t j = k >> 1; j >= (size_t)L; j >>= 1) {
            size_t half = N / 2;
            unsigned blocks = (unsigned)std::min<size_t>((half + 255) / 256, 148 * 16);
            k_bitonic_global_step<<<blocks, 256, 0, s>>>(keys, half, j, k);
            LDPC_CHECK_LAUNCH();
        }
        k_bitonic_local_merge<<<(unsigned)(N / L), threads, L * sizeof(uint64_t), s>>>(keys, k, L);
        LDPC_CHECK_LAUNCH();
    }
    return LDPC_OK;
}

// ---- exclusive scan of int32 counts (out has count+1 entries) ---------------
constexpr int kScanBlock = 1024;

__global__ void k_scan_blocks(const int32_t *in, int32_t *out, int32_t *block_sums, int64_t count) {
    __shared__ int32_t s[kScanBlock];
    int64_t i = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
    int32_t v = (i < count) ? in[i] : 0;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < kScanBlock; off <<= 1) {  // Hillis-Steele inclusive scan
        int32_t t = (threadIdx.x >= (unsigned)off) ? s[threadIdx.x - off] : 0;
        __syncthreads();
        s[threadIdx.x] += t;
        __syncthreads();
    }
    if (i < count) out[i] = s[threadIdx.x] - v;  // exclusive
    if (threadIdx.x == kScanBlock - 1) block_sums[blockIdx.x] = s[threadIdx.x];
}

__global__ void k_scan_sums(int32_t *block_sums, int64_t nblocks, int32_t *out_total) {
    // single block: exclusive scan of block sums in place, sequential over chunks
    __shared__ int32_t s[kScanBlock];
    __shared__ int32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < nblocks; base += kScanBlock) {
        int64_t i = base + threadIdx.x;
        int32_t v = (i < nblocks) ? block_sums[i] : 0;
        s[threadIdx.x] = v;
        __syncthreads();
        for (int off = 1; off < kScanBlock; off <<= 1) {
            int32_t t = (threadIdx.x >= (unsigned)off) ? s[threadIdx.x - off] : 0;
            __syncthreads();
            s[threadIdx.x] += t;
            __syncthreads();
        }
        if (i < nblocks) block_sums[i] = carry + s[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == kScanBlock - 1) carry += s[threadIdx.x];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out_total = carry;
}

__global__ void k_scan_add(int32_t *out, const int32_t *block_sums, int64_t count) {
    int64_t i = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
    if (i < count) out[i] += block_sums[blockIdx.x];
}

int exclusive_scan(const int32_t *in, int32_t *out, int64_t count, int32_t *tmp, cudaStream_t s) {
    int64_t nblocks = (count + kScanBlock - 1) / kScanBlock;
    if (nblocks == 0) nblocks = 1;
    k_scan_blocks<<<(unsigned)nblocks, kScanBlock, 0, s>>>(in, out, tmp, count);
    LDPC_CHECK_LAUNCH();
    k_scan_sums<<<1, kScanBlock, 0, s>>>(tmp, nblocks, out + count);
    LDPC_CHECK_LAUNCH();
    k_scan_add<<<(unsigned)nblocks, kScanBlock, 0, s>>>(out, tmp, count);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

// ---- builder kernels ----------------------------------------------------------
enum : uint32_t { kErrRange = 1, kErrDup = 2, kErrEmptyRow = 4, kErrEmptyCol = 8 };

__global__ void k_make_keys(const int32_t *rows, const int32_t *cols, int64_t E, size_t N, int32_t n, int32_t m,
                            uint64_t *var_key, uint64_t *chk_key, uint32_t *err) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < N; k += (size_t)gridDim.x * blockDim.x) {
        if (k < (size_t)E) {
            int32_t r = rows[k], c = cols[k];
            if (r < 0 || r >= m || c < 0 || c >= n) {
                atomicOr(err, kErrRange);
                r = 0;
                c = 0;
            }
            var_key[k] = ((uint64_t)(uint32_t)c << 32) | (uint32_t)(m - 1 - r);
            chk_key[k] = ((uint64_t)(uint32_t)r << 32) | (uint32_t)c;
        } else {
            var_key[k] = ~0ull;
            chk_key[k] = ~0ull;
        }
    }
}

__global__ void k_degrees(const uint64_t *var_key, const uint64_t *chk_key, int64_t E, int32_t *var_deg,
                          int32_t *chk_deg, uint32_t *err) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < E; k += (int64_t)gridDim.x * blockDim.x) {
        atomicAdd(&var_deg[var_key[k] >> 32], 1);
        atomicAdd(&chk_deg[chk_key[k] >> 32], 1);
        if (k > 0 && chk_key[k] == chk_key[k - 1]) atomicOr(err, kErrDup);
    }
}

__global__ void k_empty(const int32_t *var_deg, int32_t n, const int32_t *chk_deg, int32_t m, uint32_t *err,
                        int32_t *max_deg) {
    int64_t tot = (int64_t)n + m;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < tot; k += (int64_t)gridDim.x * blockDim.x) {
        if (k < n) {
            if (var_deg[k] == 0) atomicOr(err, kErrEmptyCol);
            atomicMax(&max_deg[0], var_deg[k]);
        } else {
            if (chk_deg[k - n] == 0) atomicOr(err, kErrEmptyRow);
            atomicMax(&max_deg[1], chk_deg[k - n]);
        }
    }
}

__global__ void k_fill_var(const uint64_t *var_key, int64_t E, int32_t m, int32_t *var_chk) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < E; k += (int64_t)gridDim.x * blockDim.x)
        var_chk[k] = m - 1 - (int32_t)(uint32_t)(var_key[k] & 0xffffffffu);
}

// Slot (check order) -> canonical edge via binary search in the column's
// descending row list; also the inverse map canonical edge -> slot.
__global__ void k_fill_chk(const uint64_t *chk_key, int64_t E, const int32_t *var_off, const int32_t *var_chk,
                           int32_t *chk_var, int32_t *chk_edge, int32_t *var_pos) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < E; p += (int64_t)gridDim.x * blockDim.x) {
        int32_t row = (int32_t)(chk_key[p] >> 32);
        int32_t col = (int32_t)(chk_key[p] & 0xffffffffu);
        int32_t lo = var_off[col], hi = var_off[col + 1] - 1;  // var_chk descending on [lo, hi]
        while (lo < hi) {
            int32_t mid = (lo + hi) >> 1;
            if (var_chk[mid] > row) lo = mid + 1;
            else hi = mid;
        }
        chk_var[p] = col;
        chk_edge[p] = lo;
        var_pos[lo] = (int32_t)p;
    }
}

__global__ void k_bucket_keys(const int32_t *deg, int32_t count, size_t N, uint64_t *keys) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < N; k += (size_t)gridDim.x * blockDim.x)
        keys[k] = (k < (size_t)count) ? (((uint64_t)(uint32_t)deg[k] << 32) | (uint32_t)k) : ~0ull;
}

__global__ void k_low32(const uint64_t *keys, int32_t count, int32_t *out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x)
        out[k] = (int32_t)(keys[k] & 0xffffffffu);
}

size_t next_pow2(size_t x) {
    size_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

unsigned grid_for(int64_t work, int threads = 256) {
    int64_t b = (work + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > 148 * 32) b = 148 * 32;
    return (unsigned)b;
}

template <typename T>
int dalloc(T **p, size_t count) {
    cudaError_t e = cudaMalloc((void **)p, std::max<size_t>(count, 1) * sizeof(T));
    if (e != cudaSuccess) {
        set_error("cudaMalloc(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
        *p = nullptr;
        return LDPC_ENOMEM;
    }
    return LDPC_OK;
}

int build_buckets(const int32_t *deg_dev, int32_t count, int32_t *order_dev, std::vector<Bucket> *buckets,
                  cudaStream_t s) {
    size_t N = next_pow2((size_t)count);
    uint64_t *keys = nullptr;
    int rc = dalloc(&keys, N);
    if (rc) return rc;
    k_bucket_keys<<<grid_for((int64_t)N), 256, 0, s>>>(deg_dev, count, N, keys);
    rc = cudaGetLastError() == cudaSuccess ? LDPC_OK : LDPC_ECUDA;
    if (!rc) rc = sort_u64(keys, N, s);
    if (!rc) {
        k_low32<<<grid_for(count), 256, 0, s>>>(keys, count, order_dev);
        if (cudaGetLastError() != cudaSuccess) rc = LDPC_ECUDA;
    }
    std::vector<uint64_t> host(count);
    if (!rc && cudaMemcpyAsync(host.data(), keys, count * sizeof(uint64_t), cudaMemcpyDeviceToHost, s) != cudaSuccess)
        rc = LDPC_ECUDA;
    if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = LDPC_ECUDA;
    cudaFree(keys);
    if (rc) {
        if (g_last_error.empty()) set_error("bucket build failed: %s", cudaGetErrorString(cudaGetLastError()));
        return rc;
    }
    buckets->clear();
    for (int32_t i = 0; i < count;) {
        int32_t d = (int32_t)(host[i] >> 32);
        int32_t j = i;
        while (j < count && (int32_t)(host[j] >> 32) == d) j++;
        const int32_t eb = buckets->empty() ? 0 : buckets->back().edge_begin + buckets->back().deg * buckets->back().node_count;
        buckets->push_back(Bucket{d, i, j - i, eb});
        i = j;
    }
    return LDPC_OK;
}

__global__ void k_deg_by_order(const int32_t *order, const int32_t *off, int32_t count, int32_t *deg_ord) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t node = order[k];
        deg_ord[k] = off[node + 1] - off[node];
    }
}

__global__ void k_fill_ord(const int32_t *order, const int32_t *off, int32_t count, const int32_t *ord_off,
                           const int32_t *slot, const int32_t *aux, int32_t *slot_ord, int32_t *aux_ord) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t node = order[k];
        const int32_t a = off[node], d = off[node + 1] - a, o = ord_off[k];
        for (int32_t i = 0; i < d; i++) {
            slot_ord[o + i] = slot ? slot[a + i] : a + i;
            if (aux_ord) aux_ord[o + i] = aux[a + i];
        }
    }
}

// Flat bucket-ordered edge tables of one side (see ldpc_graph::*_ord).
int build_ord(const int32_t *order, int32_t count, const int32_t *off, const int32_t *slot, const int32_t *aux,
              int64_t E, int32_t *tmp, int32_t **slot_ord, int32_t **aux_ord, cudaStream_t s) {
    int32_t *deg_ord = nullptr, *ord_off = nullptr;
    int rc = dalloc(&deg_ord, count);
    if (!rc) rc = dalloc(&ord_off, (size_t)count + 1);
    if (!rc) rc = dalloc(slot_ord, E);
    if (!rc && aux_ord) rc = dalloc(aux_ord, E);
    if (!rc) {
        k_deg_by_order<<<grid_for(count), 256, 0, s>>>(order, off, count, deg_ord);
        rc = cudaGetLastError() == cudaSuccess ? LDPC_OK : LDPC_ECUDA;
    }
    if (!rc) rc = exclusive_scan(deg_ord, ord_off, count, tmp, s);
    if (!rc) {
        k_fill_ord<<<grid_for(count), 256, 0, s>>>(order, off, count, ord_off, slot, aux, *slot_ord,
                                                   aux_ord ? *aux_ord : nullptr);
        rc = cudaGetLastError() == cudaSuccess ? LDPC_OK : LDPC_ECUDA;
    }
    if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = LDPC_ECUDA;
    if (rc == LDPC_ECUDA) set_error("flat edge tables: %s", cudaGetErrorString(cudaGetLastError()));
    cudaFree(deg_ord);
    cudaFree(ord_off);
    return rc;
}

void free_graph(ldpc_graph *g) {
    if (!g) return;
    DeviceGuard dg(g->device);
    onchip_forget(g);
    g->graphs.clear();  // GraphEntry destructors release the executable graphs
    cudaFree(g->var_slot_ord);
    cudaFree(g->chk_slot_ord);
    cudaFree(g->chk_var_ord);
    cudaFree(g->var_off);
    cudaFree(g->var_pos);
    cudaFree(g->var_chk);
    cudaFree(g->chk_off);
    cudaFree(g->chk_var);
    cudaFree(g->chk_edge);
    cudaFree(g->var_order);
    cudaFree(g->chk_order);
    delete g;
}

}  // namespace

// ---- t, s, u of one orientation from CSR offsets (for table export) ---------
__global__ void k_group_arrays(const int32_t *owner_of_pos, const int32_t *off, int64_t E, int64_t *t, int64_t *s,
                               int64_t *u) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < E; k += (int64_t)gridDim.x * blockDim.x) {
        int32_t node = owner_of_pos[k];
        int32_t a = off[node], b = off[node + 1];
        t[k] = b - a;
        s[k] = a;
        u[k] = k - a;
    }
}

}  // namespace ldpc

using namespace ldpc;

extern "C" const char *ldpc_last_error(void) { return g_last_error.c_str(); }
extern "C" int ldpc_abi_version(void) { return LDPC_B200_ABI_VERSION; }
extern "C" int64_t ldpc_kernel_launches(void) { return (int64_t)g_launches.load(); }

extern "C" int ldpc_graph_create(int32_t n, int32_t m, int64_t nnz, const int32_t *rows_host,
                                 const int32_t *cols_host, void *stream, ldpc_graph **out) {
    g_last_error.clear();
    LDPC_ARG_CHECK(out != nullptr, "out must not be NULL");
    *out = nullptr;
    LDPC_ARG_CHECK(n >= 1 && m >= 1, "matrix dimensions must be positive");
    LDPC_ARG_CHECK(nnz >= 1 && nnz < (int64_t)INT32_MAX, "edge count %lld out of range", (long long)nnz);
    LDPC_ARG_CHECK(rows_host && cols_host, "rows/cols must not be NULL");
    cudaStream_t s = (cudaStream_t)stream;
    ldpc_graph *g = new ldpc_graph();
    LDPC_CUDA_TRY(cudaGetDevice(&g->device));
    g->n = n;
    g->m = m;
    g->E = nnz;
    const size_t N = next_pow2((size_t)nnz);
    int32_t *d_rows = nullptr, *d_cols = nullptr, *var_deg = nullptr, *chk_deg = nullptr, *tmp = nullptr;
    int32_t *d_max = nullptr;
    uint64_t *var_key = nullptr, *chk_key = nullptr;
    uint32_t *d_err = nullptr;
    int rc = LDPC_OK;
    auto fail = [&](int code) {
        cudaFree(d_rows); cudaFree(d_cols); cudaFree(var_deg); cudaFree(chk_deg); cudaFree(tmp);
        cudaFree(d_max); cudaFree(var_key); cudaFree(chk_key); cudaFree(d_err);
        if (code != LDPC_OK) free_graph(g);
        return code;
    };
#define G1_TRY(x)                                  \
    do {                                           \
        int _rc = (x);                             \
        if (_rc != LDPC_OK) return fail(_rc);      \
    } while (0)
#define G1_CUDA(x)                                                                       \
    do {                                                                                 \
        cudaError_t _e = (x);                                                            \
        if (_e != cudaSuccess) {                                                         \
            set_error("%s:%d: %s: %s", __FILE__, __LINE__, #x, cudaGetErrorString(_e));  \
            return fail(LDPC_ECUDA);                                                     \
        }                                                                                \
    } while (0)
    G1_TRY(dalloc(&d_rows, nnz));
    G1_TRY(dalloc(&d_cols, nnz));
    G1_TRY(dalloc(&var_key, N));
    G1_TRY(dalloc(&chk_key, N));
    G1_TRY(dalloc(&var_deg, n));
    G1_TRY(dalloc(&chk_deg, m));
    G1_TRY(dalloc(&tmp, (std::max<int64_t>(n, m) + kScanBlock - 1) / kScanBlock + 1));
    G1_TRY(dalloc(&d_max, 2));
    G1_TRY(dalloc(&d_err, 1));
    G1_TRY(dalloc(&g->var_off, (size_t)n + 1));
    G1_TRY(dalloc(&g->chk_off, (size_t)m + 1));
    G1_TRY(dalloc(&g->var_pos, nnz));
    G1_TRY(dalloc(&g->var_chk, nnz));
    G1_TRY(dalloc(&g->chk_var, nnz));
    G1_TRY(dalloc(&g->chk_edge, nnz));
    G1_TRY(dalloc(&g->var_order, n));
    G1_TRY(dalloc(&g->chk_order, m));
    G1_CUDA(cudaMemcpyAsync(d_rows, rows_host, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    G1_CUDA(cudaMemcpyAsync(d_cols, cols_host, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    G1_CUDA(cudaMemsetAsync(var_deg, 0, n * sizeof(int32_t), s));
    G1_CUDA(cudaMemsetAsync(chk_deg, 0, m * sizeof(int32_t), s));
    G1_CUDA(cudaMemsetAsync(d_max, 0, 2 * sizeof(int32_t), s));
    G1_CUDA(cudaMemsetAsync(d_err, 0, sizeof(uint32_t), s));
    k_make_keys<<<grid_for((int64_t)N), 256, 0, s>>>(d_rows, d_cols, nnz, N, n, m, var_key, chk_key, d_err);
    G1_CUDA(cudaGetLastError());
    G1_TRY(sort_u64(var_key, N, s));
    G1_TRY(sort_u64(chk_key, N, s));
    k_degrees<<<grid_for(nnz), 256, 0, s>>>(var_key, chk_key, nnz, var_deg, chk_deg, d_err);
    G1_CUDA(cudaGetLastError());
    k_empty<<<grid_for((int64_t)n + m), 256, 0, s>>>(var_deg, n, chk_deg, m, d_err, d_max);
    G1_CUDA(cudaGetLastError());
    uint32_t err = 0;
    int32_t maxd[2] = {0, 0};
    G1_CUDA(cudaMemcpyAsync(&err, d_err, sizeof(err), cudaMemcpyDeviceToHost, s));
    G1_CUDA(cudaMemcpyAsync(maxd, d_max, sizeof(maxd), cudaMemcpyDeviceToHost, s));
    G1_CUDA(cudaStreamSynchronize(s));
    // codes.py:42-61 raise order: range, duplicate, empty row, empty column
    if (err & kErrRange) { set_error("entry outside a %dx%d matrix", m, n); return fail(LDPC_EINVAL); }
    if (err & kErrDup) { set_error("duplicate entry"); return fail(LDPC_EINVAL); }
    if (err & kErrEmptyRow) { set_error("a row has no entries"); return fail(LDPC_EINVAL); }
    if (err & kErrEmptyCol) { set_error("a column has no entries"); return fail(LDPC_EINVAL); }
    g->max_dv = maxd[0];
    g->max_dc = maxd[1];
    G1_TRY(exclusive_scan(var_deg, g->var_off, n, tmp, s));
    G1_TRY(exclusive_scan(chk_deg, g->chk_off, m, tmp, s));
    k_fill_var<<<grid_for(nnz), 256, 0, s>>>(var_key, nnz, m, g->var_chk);
    G1_CUDA(cudaGetLastError());
    k_fill_chk<<<grid_for(nnz), 256, 0, s>>>(chk_key, nnz, g->var_off, g->var_chk, g->chk_var, g->chk_edge,
                                             g->var_pos);
    G1_CUDA(cudaGetLastError());
    G1_TRY(build_buckets(var_deg, n, g->var_order, &g->var_buckets, s));
    G1_TRY(build_buckets(chk_deg, m, g->chk_order, &g->chk_buckets, s));
    G1_CUDA(cudaStreamSynchronize(s));
    {
        // LDPC_SLOTS=var: variable-major message slots (A/B layout experiments); default check-major
        const char *lay = getenv("LDPC_SLOTS");
        g->var_major = lay && std::string(lay) == "var";
        g->chk_slot = g->var_major ? g->chk_edge : nullptr;
        g->var_slot = g->var_major ? nullptr : g->var_pos;
    }
    G1_TRY(build_ord(g->var_order, n, g->var_off, g->var_slot, nullptr, nnz, tmp, &g->var_slot_ord, nullptr, s));
    G1_TRY(build_ord(g->chk_order, m, g->chk_off, g->chk_slot, g->chk_var, nnz, tmp, &g->chk_slot_ord,
                     &g->chk_var_ord, s));
#undef G1_TRY
#undef G1_CUDA
    fail(LDPC_OK);  // frees the temporaries only
    *out = g;
    return LDPC_OK;
}

extern "C" void ldpc_graph_destroy(ldpc_graph *g) { free_graph(g); }

extern "C" int ldpc_graph_info(const ldpc_graph *g, int64_t *info) {
    LDPC_ARG_CHECK(g && info, "NULL argument");
    info[0] = g->n;
    info[1] = g->m;
    info[2] = g->E;
    info[3] = g->max_dv;
    info[4] = g->max_dc;
    info[5] = (int64_t)g->var_buckets.size();
    info[6] = (int64_t)g->chk_buckets.size();
    info[7] = g->device;
    return LDPC_OK;
}

extern "C" int ldpc_graph_get_buckets(const ldpc_graph *g, int side, int32_t *deg, int32_t *count, int32_t cap) {
    LDPC_ARG_CHECK(g != nullptr, "NULL graph");
    const auto &b = side == LDPC_VARIABLE ? g->var_buckets : g->chk_buckets;
    for (int32_t i = 0; i < (int32_t)b.size() && i < cap; i++) {
        if (deg) deg[i] = b[i].deg;
        if (count) count[i] = b[i].node_count;
    }
    return (int)b.size();
}

extern "C" int ldpc_graph_get_tables(const ldpc_graph *g, int orientation, int64_t *e, int64_t *v, int64_t *c,
                                     int64_t *t, int64_t *s, int64_t *u) {
    LDPC_ARG_CHECK(g && e && v && c && t && s && u, "NULL argument");
    LDPC_ARG_CHECK(orientation == LDPC_VARIABLE || orientation == LDPC_CHECK, "bad orientation");
    const int64_t E = g->E;
    std::vector<int32_t> a(E), b(E), pos(E);
    int64_t *dt = nullptr, *ds = nullptr, *du = nullptr;
    int32_t *owner = nullptr;
    if (dalloc(&dt, E) || dalloc(&ds, E) || dalloc(&du, E) || dalloc(&owner, E)) {
        cudaFree(dt); cudaFree(ds); cudaFree(du); cudaFree(owner);
        return LDPC_ENOMEM;
    }
    int rc = LDPC_OK;
    auto cuda = [&](cudaError_t x) {
        if (x != cudaSuccess && rc == LDPC_OK) {
            set_error("get_tables: %s", cudaGetErrorString(x));
            rc = LDPC_ECUDA;
        }
    };
    if (orientation == LDPC_VARIABLE) {
        // e identity, v = owner, c = var_chk
        cuda(cudaMemcpy(b.data(), g->var_chk, E * sizeof(int32_t), cudaMemcpyDeviceToHost));
        std::vector<int32_t> off(g->n + 1);
        cuda(cudaMemcpy(off.data(), g->var_off, (g->n + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost));
        for (int32_t j = 0; j < g->n; j++)
            for (int32_t k = off[j]; k < off[j + 1]; k++) a[k] = j;
        cuda(cudaMemcpy(owner, a.data(), E * sizeof(int32_t), cudaMemcpyHostToDevice));
        k_group_arrays<<<grid_for(E), 256>>>(owner, g->var_off, E, dt, ds, du);
        cuda(cudaGetLastError());
        for (int64_t k = 0; k < E; k++) {
            e[k] = k;
            v[k] = a[k];
            c[k] = b[k];
        }
    } else {
        // e-bar = chk_edge, v-bar = chk_var, c-bar = owner check
        cuda(cudaMemcpy(pos.data(), g->chk_edge, E * sizeof(int32_t), cudaMemcpyDeviceToHost));
        cuda(cudaMemcpy(b.data(), g->chk_var, E * sizeof(int32_t), cudaMemcpyDeviceToHost));
        std::vector<int32_t> off(g->m + 1);
        cuda(cudaMemcpy(off.data(), g->chk_off, (g->m + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost));
        for (int32_t i = 0; i < g->m; i++)
            for (int32_t k = off[i]; k < off[i + 1]; k++) a[k] = i;
        cuda(cudaMemcpy(owner, a.data(), E * sizeof(int32_t), cudaMemcpyHostToDevice));
        k_group_arrays<<<grid_for(E), 256>>>(owner, g->chk_off, E, dt, ds, du);
        cuda(cudaGetLastError());
        for (int64_t k = 0; k < E; k++) {
            e[k] = pos[k];
            v[k] = b[k];
            c[k] = a[k];
        }
    }
    cuda(cudaMemcpy(t, dt, E * sizeof(int64_t), cudaMemcpyDeviceToHost));
    cuda(cudaMemcpy(s, ds, E * sizeof(int64_t), cudaMemcpyDeviceToHost));
    cuda(cudaMemcpy(u, du, E * sizeof(int64_t), cudaMemcpyDeviceToHost));
    cudaFree(dt); cudaFree(ds); cudaFree(du); cudaFree(owner);
    return rc;
}

extern "C" int ldpc_graph_get_var_groups(const ldpc_graph *g, int64_t *start, int64_t *size) {
    LDPC_ARG_CHECK(g && start && size, "NULL argument");
    std::vector<int32_t> off(g->n + 1);
    LDPC_CUDA_TRY(cudaMemcpy(off.data(), g->var_off, (g->n + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost));
    for (int32_t j = 0; j < g->n; j++) {
        start[j] = off[j];
        size[j] = off[j + 1] - off[j];
    }
    return LDPC_OK;
}
