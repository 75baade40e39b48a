// gather_probe.cu -- HBM access-pattern probe for the variable phase (throwaway tool).
//
// Moves the same bytes as one C3 half-iteration with no arithmetic:
//   stream:  warp = (check, 64-codeword chunk), reads its 7 adjacent 512-byte rows, writes them back
//   gather:  warp = (variable, chunk), reads its d rows at random slots (+ prior row), writes d rows back
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe tools/gather_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

constexpr int C = 64;  // codewords per chunk

__global__ void k_stream(double *msg, int E, int m, int dc) {
    const int lane = threadIdx.x & 31;
    const int ch = blockIdx.y;
    const int ni = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (ni >= m) return;
    double2 *base = reinterpret_cast<double2 *>(msg + (size_t)ch * E * C) + lane;
    double2 v[8];
#pragma unroll
    for (int i = 0; i < 7; i++) v[i] = __ldcs(base + (size_t)(ni * dc + i) * (C / 2));
#pragma unroll
    for (int i = 0; i < 7; i++) {
        v[i].x += 1.0;
        __stcs(base + (size_t)(ni * dc + i) * (C / 2), v[i]);
    }
}

// split layout: read D contiguous rows (own slots ni*D+i) of `src`, write them to scattered slots of `dst`
template <int D>
__global__ void k_split(const double *src, double *dst, const double *P, const int *slots, int E, int n, int cnt,
                        int node0, int base) {
    const int lane = threadIdx.x & 31;
    const int ch = blockIdx.y;
    const int ni = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (ni >= cnt) return;
    const double2 *sb = reinterpret_cast<const double2 *>(src + (size_t)ch * E * C) + lane;
    double2 *db = reinterpret_cast<double2 *>(dst + (size_t)ch * E * C) + lane;
    const double2 *pb = reinterpret_cast<const double2 *>(P + (size_t)ch * n * C) + lane;
    int s[D];
#pragma unroll
    for (int i = 0; i < D; i++) s[i] = __ldg(slots + (size_t)ni * D + i);
    double2 p = __ldg(pb + (size_t)(node0 + ni) * (C / 2));
    double2 v[D];
#pragma unroll
    for (int i = 0; i < D; i++) v[i] = __ldcs(sb + (size_t)(base + ni * D + i) * (C / 2));
#pragma unroll
    for (int i = 0; i < D; i++) {
        v[i].x += p.x;
        __stcs(db + (size_t)s[i] * (C / 2), v[i]);
    }
}

template <int D>
__global__ void k_gather(double *msg, const double *P, const int *slots, int E, int n, int cnt, int node0) {
    const int lane = threadIdx.x & 31;
    const int ch = blockIdx.y;
    const int ni = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (ni >= cnt) return;
    double2 *base = reinterpret_cast<double2 *>(msg + (size_t)ch * E * C) + lane;
    const double2 *pb = reinterpret_cast<const double2 *>(P + (size_t)ch * n * C) + lane;
    int s[D];
#pragma unroll
    for (int i = 0; i < D; i++) s[i] = __ldg(slots + (size_t)ni * D + i);
    double2 p = __ldg(pb + (size_t)(node0 + ni) * (C / 2));
    double2 v[D];
#pragma unroll
    for (int i = 0; i < D; i++) v[i] = __ldcs(base + (size_t)s[i] * (C / 2));
#pragma unroll
    for (int i = 0; i < D; i++) {
        v[i].x += p.x;
        __stcs(base + (size_t)s[i] * (C / 2), v[i]);
    }
}

int main(int argc, char **argv) {
    const int B = 1024, chunks = B / C;
    const int n8 = 12960, n3 = 19440, n2 = 32400, n = n8 + n3 + n2, m = 32400, dc = 7;
    const int E = m * dc;
    const int mode = argc > 1 ? atoi(argv[1]) : 0;  // 0 random slots, 1 sorted-per-variable (contiguous)
    std::vector<int> perm(E);
    for (int i = 0; i < E; i++) perm[i] = i;
    if (mode == 0) std::shuffle(perm.begin(), perm.end(), std::mt19937(1));
    double *msg, *P;
    int *slots;
    cudaMalloc(&msg, (size_t)E * B * 8);
    cudaMalloc(&P, (size_t)n * B * 8);
    cudaMalloc(&slots, (size_t)E * 4);
    cudaMemset(msg, 0, (size_t)E * B * 8);
    cudaMemset(P, 0, (size_t)n * B * 8);
    cudaMemcpy(slots, perm.data(), (size_t)E * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char *name, double bytes, auto launch) {
        for (int i = 0; i < 3; i++) launch();
        cudaEventRecord(a);
        const int R = 20;
        for (int i = 0; i < R; i++) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-28s %8.1f us  %7.1f GB/s\n", name, 1e3 * ms / R, bytes / (ms / R * 1e-3) / 1e9);
    };
    const double row = C * 8.0;
    run("stream check deg7", 2.0 * E * row * chunks, [&] {
        k_stream<<<dim3((m + 7) / 8, chunks), 256>>>(msg, E, m, dc);
    });
    const int *s8 = slots, *s3 = slots + (size_t)n8 * 8, *s2 = s3 + (size_t)n3 * 3;
    run("gather var deg8", (2.0 * n8 * 8 + n8) * row * chunks, [&] {
        k_gather<8><<<dim3((n8 + 7) / 8, chunks), 256>>>(msg, P, s8, E, n, n8, 0);
    });
    run("gather var deg3", (2.0 * n3 * 3 + n3) * row * chunks, [&] {
        k_gather<3><<<dim3((n3 + 7) / 8, chunks), 256>>>(msg, P, s3, E, n, n3, n8);
    });
    run("gather var deg2", (2.0 * n2 * 2 + n2) * row * chunks, [&] {
        k_gather<2><<<dim3((n2 + 7) / 8, chunks), 256>>>(msg, P, s2, E, n, n2, n8 + n3);
    });
    double *msg2;
    cudaMalloc(&msg2, (size_t)E * B * 8);
    cudaMemset(msg2, 0, (size_t)E * B * 8);
    run("split var deg8 (rd contig, wr scat)", (2.0 * n8 * 8 + n8) * row * chunks, [&] {
        k_split<8><<<dim3((n8 + 7) / 8, chunks), 256>>>(msg, msg2, P, s8, E, n, n8, 0, 0);
    });
    run("split var deg3", (2.0 * n3 * 3 + n3) * row * chunks, [&] {
        k_split<3><<<dim3((n3 + 7) / 8, chunks), 256>>>(msg, msg2, P, s3, E, n, n3, n8, n8 * 8);
    });
    run("split var deg2", (2.0 * n2 * 2 + n2) * row * chunks, [&] {
        k_split<2><<<dim3((n2 + 7) / 8, chunks), 256>>>(msg, msg2, P, s2, E, n, n2, n8 + n3, n8 * 8 + n3 * 3);
    });
    // check-like with scattered writes: read 7 contiguous rows, write them to a random permutation
    run("split check deg7 (rd contig, wr scat)", 2.0 * E * row * chunks, [&] {
        k_split<7><<<dim3((m + 7) / 8, chunks), 256>>>(msg, msg2, P, slots, E, n, m, 0, 0);
    });
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
