// row_probe.cu -- pure data movement of one C3 half-iteration with 512-byte vs 448-byte message rows
// (448 B = 64 codewords x 7 bytes: 56-bit packed messages).  Throwaway tool.
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

template <int RB>  // row bytes (multiple of 16)
__global__ void k_stream(uint4 *msg, int E, int m, int dc) {
    constexpr int P = RB / 16;  // 16-byte pieces per row
    const int lane = threadIdx.x & 31;
    const int ch = blockIdx.y;
    const int ni = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (ni >= m || lane >= P) return;
    uint4 *base = msg + (size_t)ch * E * P + lane;
    uint4 v[7];
#pragma unroll
    for (int i = 0; i < 7; i++) v[i] = __ldcg(base + (size_t)(ni * dc + i) * P);
#pragma unroll
    for (int i = 0; i < 7; i++) {
        v[i].x += 1;
        __stcg(base + (size_t)(ni * dc + i) * P, v[i]);
    }
}

template <int RB, int D>
__global__ void k_gather(uint4 *msg, const uint4 *Pr, const int *slots, int E, int n, int cnt, int node0) {
    constexpr int P = RB / 16;
    const int lane = threadIdx.x & 31;
    const int ch = blockIdx.y;
    const int ni = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (ni >= cnt) return;
    int s[D];
#pragma unroll
    for (int i = 0; i < D; i++) s[i] = __ldg(slots + (size_t)ni * D + i);
    const uint4 p = __ldg(Pr + ((size_t)ch * n + node0 + ni) * 32 + lane);  // prior row: 512 B fp64
    if (lane >= P) return;
    uint4 *base = msg + (size_t)ch * E * P + lane;
    uint4 v[D];
#pragma unroll
    for (int i = 0; i < D; i++) v[i] = __ldcg(base + (size_t)s[i] * P);
#pragma unroll
    for (int i = 0; i < D; i++) {
        v[i].x += p.x;
        __stcg(base + (size_t)s[i] * P, v[i]);
    }
}

// rows of RB >= 512 bytes: each lane moves RB/512 pieces of 16 B per row
template <int RB, int D>
__global__ void k_gather_wide(uint4 *msg, const uint4 *Pr, const int *slots, int E, int n, int cnt, int node0, int cw_per_row) {
    constexpr int P = RB / 16, PL = P / 32;
    const int lane = threadIdx.x & 31;
    const int ch = blockIdx.y;
    const int ni = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (ni >= cnt) return;
    int s[D];
#pragma unroll
    for (int i = 0; i < D; i++) s[i] = __ldg(slots + (size_t)ni * D + i);
    uint4 p[PL];
#pragma unroll
    for (int k = 0; k < PL; k++) p[k] = __ldg(Pr + ((size_t)ch * n + node0 + ni) * P + lane + 32 * k);
    uint4 *base = msg + (size_t)ch * E * P + lane;
    uint4 v[D][PL];
#pragma unroll
    for (int i = 0; i < D; i++)
#pragma unroll
        for (int k = 0; k < PL; k++) v[i][k] = __ldcg(base + (size_t)s[i] * P + 32 * k);
#pragma unroll
    for (int i = 0; i < D; i++)
#pragma unroll
        for (int k = 0; k < PL; k++) {
            v[i][k].x += p[k].x;
            __stcg(base + (size_t)s[i] * P + 32 * k, v[i][k]);
        }
}

template <int RB>
void run_wide(uint4 *msg, uint4 *Pr, int *slots) {
    const int B = 1024, chunks = B / (RB / 8);
    const int n8 = 12960, n3 = 19440, n2 = 32400, n = n8 + n3 + n2;
    const int m = 32400, E = m * 7;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char *name, auto launch) {
        for (int i = 0; i < 3; i++) launch();
        cudaEventRecord(a);
        for (int i = 0; i < 20; i++) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("rows %4d B  %-18s %8.1f us\n", RB, name, 1e3 * ms / 20);
    };
    const int *s8 = slots, *s3 = slots + (size_t)n8 * 8, *s2 = s3 + (size_t)n3 * 3;
    run("gather var d8", [&] { k_gather_wide<RB, 8><<<dim3((n8 + 7) / 8, chunks), 256>>>(msg, Pr, s8, E, n, n8, 0, RB / 8); });
    run("gather var d3", [&] { k_gather_wide<RB, 3><<<dim3((n3 + 7) / 8, chunks), 256>>>(msg, Pr, s3, E, n, n3, n8, RB / 8); });
    run("gather var d2", [&] { k_gather_wide<RB, 2><<<dim3((n2 + 7) / 8, chunks), 256>>>(msg, Pr, s2, E, n, n2, n8 + n3, RB / 8); });
}

template <int RB>
void run_all(uint4 *msg, uint4 *Pr, int *slots) {
    const int B = 1024, chunks = B / 64;
    const int n8 = 12960, n3 = 19440, n2 = 32400, n = n8 + n3 + n2, m = 32400, dc = 7, E = m * dc;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char *name, auto launch) {
        for (int i = 0; i < 3; i++) launch();
        cudaEventRecord(a);
        for (int i = 0; i < 20; i++) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("rows %3d B  %-18s %8.1f us\n", RB, name, 1e3 * ms / 20);
    };
    run("stream check d7", [&] { k_stream<RB><<<dim3((m + 7) / 8, chunks), 256>>>(msg, E, m, dc); });
    const int *s8 = slots, *s3 = slots + (size_t)n8 * 8, *s2 = s3 + (size_t)n3 * 3;
    run("gather var d8", [&] { k_gather<RB, 8><<<dim3((n8 + 7) / 8, chunks), 256>>>(msg, Pr, s8, E, n, n8, 0); });
    run("gather var d3", [&] { k_gather<RB, 3><<<dim3((n3 + 7) / 8, chunks), 256>>>(msg, Pr, s3, E, n, n3, n8); });
    run("gather var d2", [&] { k_gather<RB, 2><<<dim3((n2 + 7) / 8, chunks), 256>>>(msg, Pr, s2, E, n, n2, n8 + n3); });
}

int main() {
    const int n = 64800, m = 32400, E = m * 7, B = 1024;
    std::vector<int> perm(E);
    for (int i = 0; i < E; i++) perm[i] = i;
    std::shuffle(perm.begin(), perm.end(), std::mt19937(1));
    uint4 *msg, *Pr;
    int *slots;
    cudaMalloc(&msg, (size_t)E * B * 8);
    cudaMalloc(&Pr, (size_t)n * B * 8);
    cudaMalloc(&slots, (size_t)E * 4);
    cudaMemset(msg, 0, (size_t)E * B * 8);
    cudaMemset(Pr, 0, (size_t)n * B * 8);
    cudaMemcpy(slots, perm.data(), (size_t)E * 4, cudaMemcpyHostToDevice);
    run_all<512>(msg, Pr, slots);
    run_all<448>(msg, Pr, slots);
    run_all<256>(msg, Pr, slots);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
