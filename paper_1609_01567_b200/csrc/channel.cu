// channel.cu -- f1: device channel prologue for GPU-speed Monte Carlo.
//
// Per frame f of Eb/N0 point `point`, the reference draws its noise from
// xorshift128+ (rng.py:34-41) seeded by derive_state(seed, point, f)
// (rng.py:59-80, channel.py:112), maps 64-bit words to (0,1] (rng.py:44-50),
// turns pairs of uniforms into normals with Box-Muller (channel.py:31-37) and
// sends the all-zero codeword as y = -1 + sigma z (channel.py:47-67).  Here the
// integer part (seeding, the stream, the uniforms) is bit-exact; Box-Muller
// uses the device's fp64 log/sqrt/sincos, which are not bit-identical to
// glibc's, so y -- and parity with the reference -- is statistical
// (tests/test_channel_gpu.py bounds the difference of y and compares BER
// points).  The prior p = 1/(1+exp(-2y/s2)) of that y (serial.py:39-50) is
// numpy's, bit for bit (priors.cuh).
//
// Parallelism: xorshift128+ is linear over GF(2)^128, so the state after s*L
// draws is (M^L)^s times the seed state.  A host-built table of those 128x128
// bit matrices lets thread (frame f, segment s) jump straight to draw s*L of
// frame f's stream and produce its L draws -- the same integers as the
// sequential stream (tests pin this) -- with the grid covering
// frames x segments.  Lanes of a warp are consecutive frames of one segment,
// so the chunk-major priors P[f/64][j][f%64] are written coalesced.
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "priors.cuh"

namespace ldpc {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

// rng.py:67-80 derive_state(seed, point, frame)
__device__ __forceinline__ void derive_state3(uint64_t a, uint64_t b, uint64_t c, uint64_t &s0, uint64_t &s1) {
    uint64_t acc = 0;
    acc = mix64(acc + kGolden + a);
    acc = mix64(acc + kGolden + b);
    acc = mix64(acc + kGolden + c);
    s0 = mix64(acc + kGolden);
    s1 = mix64(acc + 2 * kGolden);
    if (s0 == 0 && s1 == 0) s1 = kGolden;
}

// rng.py:34-56: one xorshift128+ step -> u01 in (0, 1]
__device__ __forceinline__ double next_u01(uint64_t &s0, uint64_t &s1) {
    uint64_t x = s0;
    const uint64_t y = s1;
    x ^= x << 23;
    x ^= x >> 18;
    x ^= y ^ (y >> 5);
    s0 = y;
    s1 = x;
    return (double)(((x + y) >> 11) + 1) * 0x1.0p-53;
}

constexpr int kSegDraws = 256;  // draws per segment (even: Box-Muller pairs never straddle segments)

// state <- J * state over GF(2); J is 128 rows x (2 x u64), row i = output bit i (0..63 s0, 64..127 s1)
__device__ __forceinline__ void jump(const uint64_t *J, uint64_t &s0, uint64_t &s1) {
    uint64_t r0 = 0, r1 = 0;
#pragma unroll 8
    for (int i = 0; i < 64; i++) {
        const uint64_t b = (uint64_t)(__popcll((J[2 * i] & s0) ^ (J[2 * i + 1] & s1)) & 1);
        r0 |= b << i;
    }
#pragma unroll 8
    for (int i = 0; i < 64; i++) {
        const uint64_t b = (uint64_t)(__popcll((J[128 + 2 * i] & s0) ^ (J[128 + 2 * i + 1] & s1)) & 1);
        r1 |= b << i;
    }
    s0 = r0;
    s1 = r1;
}

// MODE 0: y row-major [B][n] (test hook); MODE 1: priors chunk-major [Bp/64][n][64]
// grid: x = frames (blockDim.x per block), y = segments of kSegDraws draws
template <int MODE>
__global__ void k_channel(uint64_t seed, uint64_t point, uint64_t frame0, int32_t B, int32_t n, double sigma2,
                          double *out, int32_t Bp, const uint64_t *jumps) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    const int seg = blockIdx.y;
    const int j0 = seg * kSegDraws, j1 = min(n, j0 + kSegDraws);
    if (f >= Bp) return;
    if (f >= B) {  // padded codewords: no information
        if (MODE == 1)
            for (int j = j0; j < j1; j++) out[cofs(n, j, f)] = 0.5;
        return;
    }
    uint64_t s0, s1;
    derive_state3(seed, point, frame0 + (uint64_t)f, s0, s1);
    if (seg > 0) jump(jumps + (size_t)seg * 256, s0, s1);
    const double sigma = sqrt(sigma2);
    const double two_pi = 2.0 * 3.141592653589793;
    for (int j = j0; j < j1; j += 2) {
        const double u1 = next_u01(s0, s1);
        const double u2 = next_u01(s0, s1);
        const double radius = sqrt(-2.0 * log(u1));
        double sn, cs;
        sincos(two_pi * u2, &sn, &cs);
        const double y0 = -1.0 + sigma * (radius * cs);
        const double y1 = -1.0 + sigma * (radius * sn);
        if (MODE == 0) {
            out[(size_t)f * n + j] = y0;
            if (j + 1 < n) out[(size_t)f * n + j + 1] = y1;
        } else {
            out[cofs(n, j, f)] = awgn_prior(y0, sigma2);
            if (j + 1 < n) out[cofs(n, j + 1, f)] = awgn_prior(y1, sigma2);
        }
    }
}

}  // namespace

// ---- host: jump tables (M^(kSegDraws))^s, s = 0..segs-1, per device -----------
namespace {
typedef std::vector<uint64_t> Mat;  // 128 rows x 2 words; bit c of row r = M[r][c]

Mat step_matrix() {  // one xorshift128+ step, state (s0, s1) -> (s1, x)
    Mat M(256, 0);
    for (int c = 0; c < 128; c++) {
        uint64_t s0 = c < 64 ? (1ull << c) : 0, s1 = c >= 64 ? (1ull << (c - 64)) : 0;
        uint64_t x = s0;
        const uint64_t y = s1;
        x ^= x << 23;
        x ^= x >> 18;
        x ^= y ^ (y >> 5);
        const uint64_t n0 = y, n1 = x;
        for (int r = 0; r < 128; r++) {
            const uint64_t bit = r < 64 ? (n0 >> r) & 1 : (n1 >> (r - 64)) & 1;
            if (bit) M[2 * r + (c >= 64)] |= 1ull << (c & 63);
        }
    }
    return M;
}

Mat mul(const Mat &A, const Mat &B) {  // (A B)[r][c] = xor_k A[r][k] B[k][c]
    Mat C(256, 0);
    for (int r = 0; r < 128; r++)
        for (int k = 0; k < 128; k++)
            if ((A[2 * r + (k >= 64)] >> (k & 63)) & 1) {
                C[2 * r] ^= B[2 * k];
                C[2 * r + 1] ^= B[2 * k + 1];
            }
    return C;
}

std::mutex g_jump_mu;
std::map<int, std::pair<uint64_t *, int>> g_jumps;  // device -> (table, segments)

int jump_table(int segs, const uint64_t **out) {
    int dev = 0;
    LDPC_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_jump_mu);
    auto it = g_jumps.find(dev);
    if (it != g_jumps.end() && it->second.second >= segs) {
        *out = it->second.first;
        return LDPC_OK;
    }
    Mat L = step_matrix();
    for (int k = 0; (1 << k) < kSegDraws; k++) L = mul(L, L);  // M^kSegDraws (power of two)
    std::vector<uint64_t> host((size_t)segs * 256, 0);
    Mat P(256, 0);
    for (int r = 0; r < 128; r++) P[2 * r + (r >= 64)] = 1ull << (r & 63);  // identity
    for (int s = 0; s < segs; s++) {
        std::copy(P.begin(), P.end(), host.begin() + (size_t)s * 256);
        P = mul(L, P);
    }
    uint64_t *d = nullptr;
    LDPC_CUDA_TRY(cudaMalloc(&d, host.size() * sizeof(uint64_t)));
    LDPC_CUDA_TRY(cudaMemcpy(d, host.data(), host.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
    if (it != g_jumps.end()) cudaFree(it->second.first);
    g_jumps[dev] = {d, segs};
    *out = d;
    return LDPC_OK;
}
}  // namespace

template <int MODE>
int launch_channel(uint64_t seed, uint64_t point, uint64_t frame0, int32_t B, int32_t n, double sigma2, double *out,
                   int32_t Bp, cudaStream_t s) {
    const int segs = (n + kSegDraws - 1) / kSegDraws;
    const uint64_t *J = nullptr;
    int rc = jump_table(segs, &J);
    if (rc) return rc;
    dim3 grid((Bp + 127) / 128, segs);
    k_channel<MODE><<<grid, 128, 0, s>>>(seed, point, frame0, B, n, sigma2, out, Bp, J);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

int launch_channel_priors(uint64_t seed, uint64_t point, uint64_t frame0, int32_t B, int32_t n, double sigma2,
                          double *P, int32_t Bp, cudaStream_t s) {
    return launch_channel<1>(seed, point, frame0, B, n, sigma2, P, Bp, s);
}

}  // namespace ldpc

using namespace ldpc;

extern "C" int ldpc_channel_awgn(uint64_t seed, uint64_t point, uint64_t frame0, int32_t B, int32_t n,
                                 double sigma2, double *y_dev, void *stream) {
    LDPC_ARG_CHECK(y_dev && B >= 1 && n >= 1, "bad argument");
    LDPC_ARG_CHECK(sigma2 > 0.0, "sigma2 must be positive");
    return launch_channel<0>(seed, point, frame0, B, n, sigma2, y_dev, B, (cudaStream_t)stream);
}
