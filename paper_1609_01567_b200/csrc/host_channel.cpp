// host_channel.cpp -- the reference's AWGN channel on the host, bit for bit, at C speed.
//
// transmit_all_zero (edgeldpc channel.py:47-67) draws, per frame, xorshift128+ uniforms
// (rng.py:34-50) from derive_state(seed, point, frame) (rng.py:59-80, channel.py:112)
// and turns pairs into normals with Box-Muller (channel.py:31-37) using Python's math
// module, i.e. this host's libm log / cos / sin and IEEE sqrt.  This file makes the same
// calls in the same order with the same roundings (built with -ffp-contract=off and no
// sin/cos -> sincos fusion), so y equals the reference's on the same machine -- the
// device channel (channel.cu) cannot promise that, since CUDA's log/sin/cos are other
// implementations.  Frames are independent streams, so they are spread over threads.
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "../../include/ldpc_b200.h"

namespace ldpc {
void set_error(const char *fmt, ...);  // common.cuh
}

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

struct Rng {
    uint64_t s0, s1;
    // rng.py:67-80 with keys (seed, point, frame)
    Rng(uint64_t seed, uint64_t point, uint64_t frame) {
        uint64_t acc = 0;
        for (uint64_t k : {seed, point, frame}) acc = mix64(acc + kGolden + k);
        s0 = mix64(acc + kGolden);
        s1 = mix64(acc + 2 * kGolden);
        if (s0 == 0 && s1 == 0) s1 = kGolden;
    }
    // rng.py:34-41 (23/18/5) and rng.py:44-50: ((x >> 11) + 1) * 2^-53, in (0, 1]
    double uniform01() {
        uint64_t x = s0;
        const uint64_t y = s1;
        x ^= x << 23;
        x ^= x >> 18;
        x ^= y ^ (y >> 5);
        s0 = y;
        s1 = x;
        return (double)(((x + y) >> 11) + 1) * 0x1p-53;
    }
};

// volatile function pointers: keep the separate libm calls of math.cos / math.sin (no sincos)
double (*volatile p_log)(double) = std::log;
double (*volatile p_cos)(double) = std::cos;
double (*volatile p_sin)(double) = std::sin;

void frames(uint64_t seed, uint64_t point, uint64_t frame0, int32_t f0, int32_t f1, int32_t n, double sigma,
            double *y) {
    const double two_pi = 2.0 * M_PI;  // channel.py:35: 2.0 * math.pi * u2, evaluated left to right
    for (int32_t f = f0; f < f1; f++) {
        Rng rng(seed, point, frame0 + (uint64_t)f);
        double *row = y + (size_t)f * n;
        for (int32_t i = 0; i < n; i += 2) {
            const double u1 = rng.uniform01();
            const double u2 = rng.uniform01();
            const double radius = std::sqrt(-2.0 * p_log(u1));
            const double angle = two_pi * u2;
            row[i] = -1.0 + sigma * (radius * p_cos(angle));
            if (i + 1 < n) row[i + 1] = -1.0 + sigma * (radius * p_sin(angle));
        }
    }
}

}  // namespace

extern "C" int ldpc_channel_awgn_host(uint64_t seed, uint64_t point, uint64_t frame0, int32_t B, int32_t n,
                                      double sigma2, double *y_host, int32_t threads) {
    if (y_host == nullptr || B < 0 || n < 0) {
        ldpc::set_error("bad argument");
        return LDPC_EINVAL;
    }
    if (!(sigma2 > 0.0)) {
        ldpc::set_error("sigma2 must be positive");
        return LDPC_EINVAL;
    }
    const double sigma = std::sqrt(sigma2);  // channel.py:59
    int T = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
    if (T < 1) T = 1;
    if (T > B) T = B > 0 ? B : 1;
    if (T == 1) {
        frames(seed, point, frame0, 0, B, n, sigma, y_host);
        return LDPC_OK;
    }
    std::vector<std::thread> pool;
    for (int t = 0; t < T; t++)
        pool.emplace_back(frames, seed, point, frame0, (int32_t)((int64_t)B * t / T), (int32_t)((int64_t)B * (t + 1) / T),
                          n, sigma, y_host);
    for (auto &th : pool) th.join();
    return LDPC_OK;
}
