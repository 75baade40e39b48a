// tile_persist_probe.cu -- could a persistent, L2-resident tiled schedule beat streaming? (throwaway tool)
//
// Pure data movement of a C3 decode (10 rounds + pre-pass + final estimate, no arithmetic) in two
// schedules over the same chunk-major message layout [B/64][E][64] the decoder uses:
//   streaming: one launch per phase over the whole batch (check: warp = check x 64 codewords,
//              adjacent rows; variable: warp = variable x 64 codewords, random rows + prior row)
//   persistent tiled: ONE cooperative launch; 32-codeword tiles one after another, all 21 phases of
//              a tile with grid-wide barriers between them (warp = node x 32 codewords), so a tile's
//              58 MB of messages + 16.6 MB of priors stay in the 126 MB L2 across its phases.
// Reports ms per 1024-codeword decode.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tile_persist_probe tools/tile_persist_probe.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

namespace cg = cooperative_groups;

constexpr int C = 64;
constexpr int n8 = 12960, n3 = 19440, n2 = 32400, n = n8 + n3 + n2, m = 32400, dc = 7;
constexpr int E = m * dc;
constexpr int B = 1024;

struct Tabs {
    const int *slot8, *slot3, *slot2;  // variable -> its message slots (random check positions)
};

// ---- streaming (one launch per phase) ----
__global__ void k_stream_check(double *msg) {
    const int lane = threadIdx.x & 31, ch = blockIdx.y;
    const int ni = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (ni >= m) return;
    double2 *base = reinterpret_cast<double2 *>(msg + (size_t)ch * E * C) + lane;
    double2 v[dc];
#pragma unroll
    for (int i = 0; i < dc; i++) v[i] = base[(size_t)(ni * dc + i) * (C / 2)];
#pragma unroll
    for (int i = 0; i < dc; i++) {
        v[i].x += 1.0;
        base[(size_t)(ni * dc + i) * (C / 2)] = v[i];
    }
}
template <int D>
__global__ void k_stream_var(double *msg, const double *P, const int *slots, int cnt, int node0) {
    const int lane = threadIdx.x & 31, ch = blockIdx.y;
    const int ni = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (ni >= cnt) return;
    double2 *mb = reinterpret_cast<double2 *>(msg + (size_t)ch * E * C) + lane;
    const double2 *pb = reinterpret_cast<const double2 *>(P + (size_t)ch * n * C) + lane;
    int s[D];
#pragma unroll
    for (int i = 0; i < D; i++) s[i] = __ldg(slots + (size_t)ni * D + i);
    const double2 p = pb[(size_t)(node0 + ni) * (C / 2)];
    double2 v[D];
#pragma unroll
    for (int i = 0; i < D; i++) v[i] = mb[(size_t)s[i] * (C / 2)];
#pragma unroll
    for (int i = 0; i < D; i++) {
        v[i].x += p.x;
        mb[(size_t)s[i] * (C / 2)] = v[i];
    }
}

// ---- persistent tiled: warp = node x 32 codewords of the current tile (lane = codeword) ----
template <int D>
__device__ __forceinline__ void var_task(double *mb, const double *pb, const int *slots, int ni, int node) {
    int s[D];
#pragma unroll
    for (int i = 0; i < D; i++) s[i] = __ldg(slots + (size_t)ni * D + i);
    const double p = pb[(size_t)node * C];
    double v[D];
#pragma unroll
    for (int i = 0; i < D; i++) v[i] = mb[(size_t)s[i] * C];
#pragma unroll
    for (int i = 0; i < D; i++) mb[(size_t)s[i] * C] = v[i] + p;
}

__global__ void __launch_bounds__(256) k_persist(double *msg, const double *P, Tabs t, int rounds) {
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int GW = (gridDim.x * blockDim.x) >> 5;
    for (int tile = 0; tile < B / 32; tile++) {
        const int ch = tile >> 1, half = (tile & 1) * 32;
        double *mb = msg + (size_t)ch * E * C + half + lane;
        const double *pb = P + (size_t)ch * n * C + half + lane;
        for (int ph = 0; ph < 2 * rounds + 2; ph++) {
            if ((ph & 1) == 0) {  // check phase: adjacent rows
                for (int ni = gw; ni < m; ni += GW) {
                    double v[dc];
#pragma unroll
                    for (int i = 0; i < dc; i++) v[i] = mb[(size_t)(ni * dc + i) * C];
#pragma unroll
                    for (int i = 0; i < dc; i++) mb[(size_t)(ni * dc + i) * C] = v[i] + 1.0;
                }
            } else {  // variable phase: all buckets in one task space
                for (int k = gw; k < n; k += GW) {
                    if (k < n8) var_task<8>(mb, pb, t.slot8, k, k);
                    else if (k < n8 + n3) var_task<3>(mb, pb, t.slot3, k - n8, k);
                    else var_task<2>(mb, pb, t.slot2, k - n8 - n3, k);
                }
            }
            grid.sync();
        }
    }
}

int main() {
    std::mt19937 rng(7);
    std::vector<int> slots(E);
    for (int i = 0; i < E; i++) slots[i] = i;
    std::shuffle(slots.begin(), slots.end(), rng);
    int *d_slots;
    cudaMalloc(&d_slots, sizeof(int) * E);
    cudaMemcpy(d_slots, slots.data(), sizeof(int) * E, cudaMemcpyHostToDevice);
    Tabs t{d_slots, d_slots + n8 * 8, d_slots + n8 * 8 + n3 * 3};
    double *msg, *P;
    cudaMalloc(&msg, sizeof(double) * (size_t)E * B);
    cudaMalloc(&P, sizeof(double) * (size_t)n * B);
    cudaMemset(msg, 0, sizeof(double) * (size_t)E * B);
    cudaMemset(P, 0, sizeof(double) * (size_t)n * B);
    const int rounds = 10;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto stream_decode = [&]() {
        const dim3 gc((m + 7) / 8, B / C);
        for (int ph = 0; ph < 2 * rounds + 2; ph++) {
            if ((ph & 1) == 0) {
                k_stream_check<<<gc, 256>>>(msg);
            } else {
                k_stream_var<8><<<dim3((n8 + 7) / 8, B / C), 256>>>(msg, P, t.slot8, n8, 0);
                k_stream_var<3><<<dim3((n3 + 7) / 8, B / C), 256>>>(msg, P, t.slot3, n3, n8);
                k_stream_var<2><<<dim3((n2 + 7) / 8, B / C), 256>>>(msg, P, t.slot2, n2, n8 + n3);
            }
        }
    };
    for (int w = 0; w < 2; w++) stream_decode();
    cudaEventRecord(e0);
    for (int r = 0; r < 3; r++) stream_decode();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("streaming (launch per phase): %.3f ms per decode\n", ms / 3);
    int dev = 0, sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_persist, 256, 0);
    for (int bps : {1, 2, 4, per}) {
        if (bps > per) continue;
        const int blocks = sms * bps;
        void *args[] = {&msg, &P, &t, (void *)&rounds};
        cudaLaunchCooperativeKernel((void *)k_persist, blocks, 256, args);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; r++) cudaLaunchCooperativeKernel((void *)k_persist, blocks, 256, args);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("persistent tiled (%d blocks/SM, %d warps): %.3f ms per decode (%s)\n", bps, blocks * 8, ms / 3,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
