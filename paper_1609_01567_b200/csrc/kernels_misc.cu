// kernels_misc.cu -- G4 syndrome / early-stop flags, layout and output kernels.
//
// Syndrome (serial.py:136-147, engine.py:144-149, paper Algorithm 7): with the
// estimate bit-sliced 32 codewords per word, z for 32 codewords of check i is
// the XOR of the words of its variables -- one 32-bit XOR per edge instead of
// 32 byte XORs.  The all-zero test (serial.py:169/176; serial per round in the
// reference, engine.py:324-326, "about 34% of decode time" in the paper) is an
// OR-reduction of z over checks: per thread in registers, per block in shared
// memory, then one atomicOr per word per block.
#include <algorithm>

#include "common.cuh"
#include "priors.cuh"

namespace ldpc {
namespace {

unsigned blocks_for(int64_t work, int threads, int64_t cap = 148 * 64) {
    int64_t b = (work + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return (unsigned)b;
}

// P_in [B][n] -> P [Bp/64][n][64] (chunk-major); padded codewords get p = 0.5 (no information).
// AWGN: the input is observations y and the prior 1/(1+exp(-2y/sigma2[c])) is formed on the way
// (priors.cuh, bit-identical to the reference's numpy expression).
template <bool AWGN>
__global__ void k_transpose_priors(const double *__restrict__ in, const double *__restrict__ sig2, int32_t B,
                                   int32_t n, double *__restrict__ P, int32_t Bp) {
    __shared__ double tile[32][33];
    const int j0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    // blockDim (32, 8): 4 rows per thread, loads issued before any prior arithmetic
    double v[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int c = c0 + threadIdx.y + 8 * k, j = j0 + threadIdx.x;
        v[k] = (c < B && j < n) ? __ldcs(in + (size_t)c * n + j) : 0.5;
    }
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int c = c0 + threadIdx.y + 8 * k;
        if (AWGN && c < B && j0 + (int)threadIdx.x < n) v[k] = awgn_prior(v[k], __ldg(sig2 + c));
        tile[threadIdx.y + 8 * k][threadIdx.x] = v[k];
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int j = j0 + y, c = c0 + threadIdx.x;
        if (j < n && c < Bp) P[cofs(n, j, c)] = tile[threadIdx.x][y];
    }
}

constexpr int kLongSyndrome = 64;  // checks of higher degree: one block per (check, word), k_syndrome_long

// blockDim (32, 8): x -> word, y -> check; grid (check slabs, word groups)
__global__ void k_syndrome(const int32_t *__restrict__ chk_off, const int32_t *__restrict__ chk_var, int32_t m,
                           const uint32_t *__restrict__ chat, int32_t NW, int32_t NWs, uint32_t *__restrict__ zb,
                           uint32_t *__restrict__ unsat, const uint32_t *__restrict__ done, int skip_long) {
    __shared__ uint32_t red[8][32];
    const int w = blockIdx.y * 32 + threadIdx.x;
    uint32_t acc = 0;
    const bool live = (w < NW) && !(done != nullptr && done[w] == 0xffffffffu);
    if (live) {
        for (int i = blockIdx.x * 8 + threadIdx.y; i < m; i += gridDim.x * 8) {
            const int a = __ldg(chk_off + i), b = __ldg(chk_off + i + 1);
            if (skip_long && b - a > kLongSyndrome) continue;  // k_syndrome_long
            uint32_t z = 0;
            // 8 independent loads in flight per step (a long check would otherwise pay one
            // dependent L2 round trip per variable)
            for (int p = a; p < b; p += 8) {
                uint32_t x[8];
#pragma unroll
                for (int u = 0; u < 8; u++) x[u] = (p + u < b) ? chat[(size_t)__ldg(chk_var + p + u) * NWs + w] : 0u;
#pragma unroll
                for (int u = 0; u < 8; u++) z ^= x[u];
            }
            if (zb != nullptr) zb[(size_t)i * NWs + w] = z;
            acc |= z;
        }
    } else if (w < NW && zb != nullptr) {
        for (int i = blockIdx.x * 8 + threadIdx.y; i < m; i += gridDim.x * 8) zb[(size_t)i * NWs + w] = 0;
    }
    red[threadIdx.y][threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.y == 0 && w < NW) {
        uint32_t o = 0;
#pragma unroll
        for (int y = 0; y < 8; y++) o |= red[y][threadIdx.x];
        if (o & ~unsat[w]) atomicOr(unsat + w, o);
    }
}

// Syndrome words of the long checks chk_order[first ..]: block (check, word), 256 threads over
// the check's variables, XOR-reduced through shuffles and shared memory (one round trip
// instead of one per variable).
__global__ void k_syndrome_long(const int32_t *__restrict__ chk_off, const int32_t *__restrict__ chk_var,
                                const int32_t *__restrict__ chk_order, int32_t first, const uint32_t *__restrict__ chat,
                                int32_t NWs, uint32_t *__restrict__ zb, uint32_t *__restrict__ unsat,
                                const uint32_t *__restrict__ done) {
    __shared__ uint32_t red[8];
    const int c = __ldg(chk_order + first + blockIdx.x);
    const int w = blockIdx.y;
    const bool live = !(done != nullptr && done[w] == 0xffffffffu);
    uint32_t z = 0;
    if (live) {
        const int a = __ldg(chk_off + c), b = __ldg(chk_off + c + 1);
        for (int p = a + threadIdx.x; p < b; p += blockDim.x) z ^= chat[(size_t)__ldg(chk_var + p) * NWs + w];
        for (int o = 16; o > 0; o >>= 1) z ^= __shfl_xor_sync(0xffffffffu, z, o);
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = z;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); k++) t ^= red[k];
        if (zb != nullptr) zb[(size_t)c * NWs + w] = t;
        if (t & ~unsat[w]) atomicOr(unsat + w, t);
    }
}

// Early-stop bookkeeping after the syndrome of round t (serial.py:169-177):
// codewords with an all-zero syndrome stop now with iterations_used = t.
__global__ void k_update_done(uint32_t *done, uint32_t *unsat, int32_t *iters, int32_t NW, int32_t t, int final_round) {
    for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < NW; w += gridDim.x * blockDim.x) {
        const uint32_t d = done[w], u = unsat[w];
        const uint32_t newly = ~d & ~u;
        uint32_t set = newly;
        if (final_round) set = ~d;  // stopped now, or ran out of rounds (serial.py:178)
        for (uint32_t x = set; x; x &= x - 1) iters[32 * w + __ffs(x) - 1] = t;
        done[w] = d | newly;
        unsat[w] = 0;
    }
}

// src [rows][NW] bit-sliced (bit b of word w = codeword 32w+b) ->
// dst [B][RW] per-codeword packed rows (bit b of word r = row 32r+b), RW = ceil(rows/32).
// One warp per 32x32 bit tile, transposed with 32 ballots.
__global__ void k_pack_rows(const uint32_t *__restrict__ src, int32_t rows, int32_t NW, int32_t B,
                            uint32_t *__restrict__ dst) {
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
        const int cw = w * 32 + lane;
        if (cw < B) dst[(size_t)cw * RW + rb] = mine;
    }
}

__global__ void k_finalize(const uint32_t *done, const uint32_t *unsat, const int32_t *iters_ws, int32_t B,
                           int early_stop, int32_t max_iter, uint8_t *success, int32_t *iters) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < B; c += gridDim.x * blockDim.x) {
        const uint32_t bit = 1u << (c & 31);
        if (early_stop) {
            success[c] = (done[c >> 5] & bit) ? 1 : 0;
            iters[c] = iters_ws[c];
        } else {
            success[c] = (unsat[c >> 5] & bit) ? 0 : 1;
            iters[c] = max_iter;
        }
    }
}

__global__ void k_count_errors(const uint32_t *est, int32_t RW, const uint8_t *success, const int32_t *iters,
                               int32_t B, unsigned long long *counts) {
    __shared__ unsigned long long s[3];
    if (threadIdx.x < 3) s[threadIdx.x] = 0;
    __syncthreads();
    unsigned long long bits = 0, fail = 0, its = 0;
    const int64_t total = (int64_t)B * RW;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x)
        bits += __popc(est[k]);
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < B; c += gridDim.x * blockDim.x) {
        fail += success[c] ? 0 : 1;
        its += (unsigned long long)iters[c];
    }
    for (int o = 16; o > 0; o >>= 1) {
        bits += __shfl_xor_sync(0xffffffffu, bits, o);
        fail += __shfl_xor_sync(0xffffffffu, fail, o);
        its += __shfl_xor_sync(0xffffffffu, its, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&s[0], bits);
        atomicAdd(&s[1], fail);
        atomicAdd(&s[2], its);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd(&counts[0], s[0]);
        atomicAdd(&counts[1], s[1]);
        atomicAdd(&counts[2], s[2]);
        if (blockIdx.x == 0) atomicAdd(&counts[3], (unsigned long long)B);
    }
}

// phase-API converters (not on the decode path) ------------------------------
__global__ void k_canon_to_slots(const int32_t *var_slot, int64_t E, const double *src, int32_t B, double *msg,
                                 int32_t Bp) {
    const int64_t total = E * Bp;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = k / Bp;
        const int c = (int)(k - e * Bp);
        const int32_t slot = var_slot ? var_slot[e] : (int32_t)e;
        msg[cofs((int32_t)E, slot, c)] = (c < B) ? src[(size_t)c * E + e] : 0.5;
    }
}

__global__ void k_slots_to_canon(const int32_t *var_slot, int64_t E, const double *msg, int32_t Bp, double *dst,
                                 int32_t B) {
    const int64_t total = E * B;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(k / E);
        const int64_t e = k - (int64_t)c * E;
        const int32_t slot = var_slot ? var_slot[e] : (int32_t)e;
        dst[k] = msg[cofs((int32_t)E, slot, c)];
    }
}

__global__ void k_bytes_to_bits(const uint8_t *src, int32_t B, int32_t rows, uint32_t *dst, int32_t NW) {
    const int64_t total = (int64_t)rows * NW;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = k / NW;
        const int w = (int)(k - row * NW);
        uint32_t x = 0;
        for (int b = 0; b < 32; b++) {
            const int c = w * 32 + b;
            if (c < B && (src[(size_t)c * rows + row] & 1)) x |= 1u << b;
        }
        dst[k] = x;
    }
}

__global__ void k_bits_to_bytes(const uint32_t *src, int32_t rows, int32_t NW, int32_t B, uint8_t *dst) {
    const int64_t total = (int64_t)rows * B;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(k / rows);
        const int64_t row = k - (int64_t)c * rows;
        dst[k] = (uint8_t)((src[row * NW + (c >> 5)] >> (c & 31)) & 1u);
    }
}

__global__ void k_fill_u32(uint32_t *dst, uint32_t value, size_t count) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < count; k += (size_t)gridDim.x * blockDim.x)
        dst[k] = value;
}

}  // namespace

int launch_transpose_priors(const double *p_in, const double *sig2, int32_t B, int32_t n, double *P, int32_t Bp,
                            cudaStream_t s) {
    dim3 grid((n + 31) / 32, (Bp + 31) / 32);
    if (sig2)
        k_transpose_priors<true><<<grid, dim3(32, 8), 0, s>>>(p_in, sig2, B, n, P, Bp);
    else
        k_transpose_priors<false><<<grid, dim3(32, 8), 0, s>>>(p_in, nullptr, B, n, P, Bp);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

int launch_syndrome(const ldpc_graph *g, const Workspace &w, bool write_z, bool use_done, cudaStream_t s) {
    // checks past kLongSyndrome: a suffix of chk_order (sorted by degree), one block per (check, word)
    int32_t first_long = g->m;
    for (const Bucket &b : g->chk_buckets)
        if (b.deg > kLongSyndrome) first_long = std::min(first_long, b.node_begin);
    const unsigned gx = blocks_for(g->m, 8, 148 * 8);
    dim3 grid(gx, (w.NW + 31) / 32);
    k_syndrome<<<grid, dim3(32, 8), 0, s>>>(g->chk_off, g->chk_var, g->m, w.chat, w.NW, w.NWs, write_z ? w.zb : nullptr,
                                             w.unsat, use_done ? w.done : nullptr, first_long < g->m ? 1 : 0);
    LDPC_CHECK_LAUNCH();
    if (first_long < g->m) {
        k_syndrome_long<<<dim3(g->m - first_long, w.NW), 256, 0, s>>>(
            g->chk_off, g->chk_var, g->chk_order, first_long, w.chat, w.NWs, write_z ? w.zb : nullptr, w.unsat,
            use_done ? w.done : nullptr);
        LDPC_CHECK_LAUNCH();
    }
    return LDPC_OK;
}

int launch_update_done(const Workspace &w, int32_t round, bool final_round, cudaStream_t s) {
    k_update_done<<<blocks_for(w.NW, 256), 256, 0, s>>>(w.done, w.unsat, w.iters, w.NW, round, final_round ? 1 : 0);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

int launch_pack_rows(const uint32_t *src, int32_t rows, int32_t NW, int32_t B, uint32_t *dst, cudaStream_t s) {
    const int64_t tiles = (int64_t)((rows + 31) / 32) * NW;
    k_pack_rows<<<blocks_for(tiles * 32, 256), 256, 0, s>>>(src, rows, NW, B, dst);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

int launch_finalize(const Workspace &w, bool early_stop, int32_t max_iter, uint8_t *success, int32_t *iters,
                    cudaStream_t s) {
    k_finalize<<<blocks_for(w.B, 256), 256, 0, s>>>(w.done, w.unsat, w.iters, w.B, early_stop ? 1 : 0, max_iter,
                                                     success, iters);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

int launch_count_errors(const uint32_t *est_bits, int32_t words_per_row, const uint8_t *success,
                        const int32_t *iters, int32_t B, int64_t *counts, cudaStream_t s) {
    k_count_errors<<<blocks_for((int64_t)B * words_per_row, 256, 148 * 4), 256, 0, s>>>(
        est_bits, words_per_row, success, iters, B, reinterpret_cast<unsigned long long *>(counts));
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

int launch_canon_to_slots(const ldpc_graph *g, const double *src, int32_t B, double *msg, int32_t Bp,
                          cudaStream_t s) {
    k_canon_to_slots<<<blocks_for(g->E * Bp, 256), 256, 0, s>>>(g->var_slot, g->E, src, B, msg, Bp);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

int launch_slots_to_canon(const ldpc_graph *g, const double *msg, int32_t Bp, double *dst, int32_t B,
                          cudaStream_t s) {
    k_slots_to_canon<<<blocks_for(g->E * B, 256), 256, 0, s>>>(g->var_slot, g->E, msg, Bp, dst, B);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

int launch_bytes_to_bits(const uint8_t *src, int32_t B, int32_t rows, uint32_t *dst, int32_t NW, cudaStream_t s) {
    k_bytes_to_bits<<<blocks_for((int64_t)rows * NW, 256), 256, 0, s>>>(src, B, rows, dst, NW);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

int launch_bits_to_bytes(const uint32_t *src, int32_t rows, int32_t NW, int32_t B, uint8_t *dst, cudaStream_t s) {
    k_bits_to_bytes<<<blocks_for((int64_t)rows * B, 256), 256, 0, s>>>(src, rows, NW, B, dst);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

int launch_fill_u32(uint32_t *dst, uint32_t value, size_t count, cudaStream_t s) {
    if (count == 0) return LDPC_OK;
    k_fill_u32<<<blocks_for((int64_t)count, 256), 256, 0, s>>>(dst, value, count);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

}  // namespace ldpc

// ---- self-test: ddiv_fast (when its test passes) == __ddiv_rn, bitwise ---------
namespace ldpc {
namespace {
__device__ __forceinline__ uint64_t xs64(uint64_t &s) {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    return s;
}

__global__ void k_selftest_ddiv(uint64_t seed, int64_t count, unsigned long long *out) {
    uint64_t s = seed ^ (0x9E3779B97F4A7C15ull * (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x + 1));
    unsigned long long bad = 0, fast = 0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t u = xs64(s), v = xs64(s), w = xs64(s);
        double a, b;
        switch (w & 3) {
            case 0: {  // decoder-like: q1 in [0,1], den = q0 + q1 in (0, 2]
                a = (u >> 11) * 0x1.0p-53;
                b = __dadd_rn(a, (v >> 11) * 0x1.0p-53);
                break;
            }
            case 1: {  // products of messages: random exponents down to the subnormal range
                a = __longlong_as_double((long long)((u & 0x000FFFFFFFFFFFFFull) | ((uint64_t)((w >> 8) % 1030) << 52)));
                b = __dadd_rn(a, __longlong_as_double((long long)((v & 0x000FFFFFFFFFFFFFull) |
                                                                  ((uint64_t)((w >> 20) % 1030) << 52))));
                break;
            }
            case 2: {  // arbitrary positive finite bit patterns
                a = __longlong_as_double((long long)(u & 0x7FEFFFFFFFFFFFFFull));
                b = __longlong_as_double((long long)(v & 0x7FEFFFFFFFFFFFFFull));
                break;
            }
            default: {  // mantissas near all-ones / powers of two
                a = __longlong_as_double((long long)(0x3FE0000000000000ull | (u & 0xFull) | ((u >> 4 & 1) ? 0x000FFFFFFFFFFFF0ull : 0)));
                b = __longlong_as_double((long long)(0x3FF0000000000000ull | (v & 0xFull) | ((v >> 4 & 1) ? 0x000FFFFFFFFFFFF0ull : 0)));
                break;
            }
        }
        bool ok;
        const double q = ddiv_fast(a, b, ok);
        if (ok) {
            fast++;
            if (__double_as_longlong(q) != __double_as_longlong(__ddiv_rn(a, b))) bad++;
        }
    }
    atomicAdd(&out[0], bad);
    atomicAdd(&out[1], fast);
}
}  // namespace
}  // namespace ldpc

extern "C" int ldpc_selftest_division(uint64_t seed, int64_t count, int64_t *result_host) {
    using namespace ldpc;
    LDPC_ARG_CHECK(result_host != nullptr && count > 0, "bad argument");
    unsigned long long *d = nullptr;
    LDPC_CUDA_TRY(cudaMalloc(&d, 2 * sizeof(unsigned long long)));
    cudaMemset(d, 0, 2 * sizeof(unsigned long long));
    k_selftest_ddiv<<<148 * 8, 256>>>(seed, count, d);
    count_launch();
    cudaError_t e = cudaGetLastError();
    unsigned long long h[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) {
        set_error("selftest: %s", cudaGetErrorString(e));
        return LDPC_ECUDA;
    }
    result_host[0] = (int64_t)h[0];
    result_host[1] = (int64_t)h[1];
    return LDPC_OK;
}
