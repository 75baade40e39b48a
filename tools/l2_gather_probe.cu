// l2_gather_probe.cu -- can an L2-resident codeword tile beat HBM streaming? (throwaway tool)
// One tile of C codewords (layout [E][C] doubles, priors [n][C]); the stream (check-like) and
// gather (variable-like) movement kernels run back to back on the same tile, as one
// half-iteration each.  Reports the effective GB/s of the moved bytes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_gather_probe tools/l2_gather_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

template <int C>
struct Row {  // one lane's share of a C-codeword row
    static constexpr int K = C / 32;
};

template <int C>
__global__ void k_stream(double *msg, int m, int dc) {
    const int lane = threadIdx.x & 31;
    const int ni = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (ni >= m) return;
    double v[8];
    double *base = msg + (size_t)ni * dc * C + lane * (C / 32);
#pragma unroll
    for (int i = 0; i < 7; i++) v[i] = base[i * C];
#pragma unroll
    for (int i = 0; i < 7; i++) base[i * C] = v[i] + 1.0;
}

template <int C, int D>
__global__ void k_gather(double *msg, const double *P, const int *slots, int cnt, int node0) {
    const int lane = threadIdx.x & 31;
    const int ni = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (ni >= cnt) return;
    int s[D];
#pragma unroll
    for (int i = 0; i < D; i++) s[i] = __ldg(slots + (size_t)ni * D + i);
    const double p = P[(size_t)(node0 + ni) * C + lane * (C / 32)];
    double v[D];
#pragma unroll
    for (int i = 0; i < D; i++) v[i] = msg[(size_t)s[i] * C + lane * (C / 32)];
#pragma unroll
    for (int i = 0; i < D; i++) msg[(size_t)s[i] * C + lane * (C / 32)] = v[i] + p;
}

int main(int argc, char **argv) {
    const int tiles = argc > 1 ? atoi(argv[1]) : 1;  // tiles of 32 codewords, run one after another
    constexpr int C = 32;
    const int n8 = 12960, n3 = 19440, n2 = 32400, n = n8 + n3 + n2, m = 32400, dc = 7;
    const int E = m * dc;
    std::vector<int> perm(E);
    for (int i = 0; i < E; i++) perm[i] = i;
    std::shuffle(perm.begin(), perm.end(), std::mt19937(1));
    double *msg, *P;
    int *slots;
    cudaMalloc(&msg, (size_t)E * C * 8 * tiles);
    cudaMalloc(&P, (size_t)n * C * 8 * tiles);
    cudaMalloc(&slots, (size_t)E * 4);
    cudaMemset(msg, 0, (size_t)E * C * 8 * tiles);
    cudaMemset(P, 0, (size_t)n * C * 8 * tiles);
    cudaMemcpy(slots, perm.data(), (size_t)E * 4, cudaMemcpyHostToDevice);
    const int *s8 = slots, *s3 = slots + (size_t)n8 * 8, *s2 = s3 + (size_t)n3 * 3;
    cudaStream_t st;
    cudaStreamCreate(&st);
    auto half_iters = [&](int t, int iters) {
        double *mm = msg + (size_t)t * E * C;
        double *pp = P + (size_t)t * n * C;
        for (int it = 0; it < iters; it++) {
            k_stream<C><<<(m + 7) / 8, 256, 0, st>>>(mm, m, dc);
            k_gather<C, 8><<<(n8 + 7) / 8, 256, 0, st>>>(mm, pp, s8, n8, 0);
            k_gather<C, 3><<<(n3 + 7) / 8, 256, 0, st>>>(mm, pp, s3, n3, n8);
            k_gather<C, 2><<<(n2 + 7) / 8, 256, 0, st>>>(mm, pp, s2, n2, n8 + n3);
        }
    };
    const int iters = 10;
    // capture: tile-major (all iterations of a tile, then the next) vs iteration-major
    for (int order = 0; order < 2; order++) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        if (order == 0) {
            for (int t = 0; t < tiles; t++) half_iters(t, iters);
        } else {
            for (int it = 0; it < iters; it++)
                for (int t = 0; t < tiles; t++) half_iters(t, 1);
        }
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st);
        cudaStreamSynchronize(st);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, st);
        const int R = 5;
        for (int r = 0; r < R; r++) cudaGraphLaunch(ge, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= R;
        const double bytes = (double)tiles * iters * C * 8.0 * (2.0 * E + 2.0 * E + n);
        printf("tiles=%d (%.0f MB/tile) %s: %.3f ms per pass, %.1f GB/s effective, %.2f us/codeword-iteration\n",
               tiles, (E + n) * C * 8.0 / 1e6, order == 0 ? "tile-major (L2-resident)" : "iteration-major (streaming)",
               ms, bytes / (ms * 1e-3) / 1e9, ms * 1e3 / (tiles * C * iters));
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
