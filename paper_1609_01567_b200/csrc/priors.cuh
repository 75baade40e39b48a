// priors.cuh -- the reference's AWGN prior p = 1/(1 + exp(-2y/sigma2)) on the device,
// bit-identical to the numpy expression it evaluates (serial.py:49-50).
//
// numpy's float64 exp is not correctly rounded and is machine dependent: on
// AVX512_SKX hosts numpy 2.x hands contiguous arrays to Intel SVML's
// __svml_exp8_ha.  np_exp below runs that algorithm -- same operation order,
// same rounding modes (the first fma rounds toward zero), same constants and
// tables -- with explicit IEEE intrinsics, so it reproduces numpy's results
// bit for bit (oracle/npexp.c restates it on the CPU; tests/test_priors.py
// pins both against np.exp).  Whether the host's numpy runs this algorithm is
// checked at run time by the Python layer (decoder.device_priors_exact) before
// observations are decoded with device priors.
//
// Main path, |x| < 0x1.61da04cbafe44p+9 (or NaN): 16-entry table,
//   s = fma_rz(x, 1/ln2, 1.5*2^48 + 1023); k = s - shifter; j = low 4 bits of s
//   r = fma(-k, ln2_hi, x); r = fma(-k, ln2_lo, r)
//   P = r^2 (r^2 (a6 r + a5) + (a4 r + a3)) + (a2 r + a1)
//   e = T2[j] (P r + T1[j]) + T2[j];  exp(x) = e 2^floor(k)
// Rare path (|x| beyond that, +-inf): SVML's scalar 64-entry-table routine.
//
// Attribution: the algorithm, its constants and both tables are Intel's SVML exp (__svml_exp8_ha,
// __svml_dexp_ha_cout_rare_internal) as vendored in numpy under the BSD-3-Clause license
// (Copyright (c) Intel Corporation; numpy/_core/src/umath/svml/LICENSE); restated here.
#pragma once
#include <cstdint>

#include "common.cuh"

namespace ldpc {

static __device__ __forceinline__ double bits_d(uint64_t u) { return __longlong_as_double((long long)u); }

__device__ const uint64_t kExpT2[16] = {
    0x3ff0000000000000ull, 0x3ff0b5586cf9890full, 0x3ff172b83c7d517bull, 0x3ff2387a6e756238ull,
    0x3ff306fe0a31b715ull, 0x3ff3dea64c123422ull, 0x3ff4bfdad5362a27ull, 0x3ff5ab07dd485429ull,
    0x3ff6a09e667f3bcdull, 0x3ff7a11473eb0187ull, 0x3ff8ace5422aa0dbull, 0x3ff9c49182a3f090ull,
    0x3ffae89f995ad3adull, 0x3ffc199bdd85529cull, 0x3ffd5818dcfba487ull, 0x3ffea4afa2a490daull};
__device__ const uint64_t kExpT1[16] = {
    0x0000000000000000ull, 0x3c979aa65d837b6dull, 0xbc801b15eaa59348ull, 0x3c968efde3a8a894ull,
    0x3c834d754db0abb6ull, 0x3c859f48a72a4c6dull, 0x3c7690cebb7aafb0ull, 0x3c9063e1e21c5409ull,
    0xbc93b3efbf5e2228ull, 0xbc7b32dcb94da51dull, 0x3c8db72fc1f0eab4ull, 0x3c71affc2b91ce27ull,
    0x3c8c1a7792cb3387ull, 0x3c736eae30af0cb3ull, 0x3c74a385a63d07a7ull, 0xbc8ff7128fd391f0ull};
__device__ const uint64_t kExpRare[128] = {  // pairs (2^(j/64) hi, lo)
    0x3ff0000000000000ull, 0x0000000000000000ull, 0x3ff02c9a3e778061ull, 0xbc7160139cd8dc5dull,
    0x3ff059b0d3158574ull, 0x3c8cd2523567f613ull, 0x3ff0874518759bc8ull, 0x3c60f74e61e6c861ull,
    0x3ff0b5586cf9890full, 0x3c979aa65d837b6dull, 0x3ff0e3ec32d3d1a2ull, 0x3c3ebe3d702f9cd1ull,
    0x3ff11301d0125b51ull, 0xbc9556522a2fbd0eull, 0x3ff1429aaea92de0ull, 0xbc91c923b9d5f416ull,
    0x3ff172b83c7d517bull, 0xbc801b15eaa59348ull, 0x3ff1a35beb6fcb75ull, 0x3c8b898c3f1353bfull,
    0x3ff1d4873168b9aaull, 0x3c9aecf73e3a2f60ull, 0x3ff2063b88628cd6ull, 0x3c8a6f4144a6c38dull,
    0x3ff2387a6e756238ull, 0x3c968efde3a8a894ull, 0x3ff26b4565e27cddull, 0x3c80472b981fe7f2ull,
    0x3ff29e9df51fdee1ull, 0x3c82f7e16d09ab31ull, 0x3ff2d285a6e4030bull, 0x3c8b3782720c0ab4ull,
    0x3ff306fe0a31b715ull, 0x3c834d754db0abb6ull, 0x3ff33c08b26416ffull, 0x3c8fdd395dd3f84aull,
    0x3ff371a7373aa9cbull, 0xbc924aedcc4b5068ull, 0x3ff3a7db34e59ff7ull, 0xbc71d1e83e9436d2ull,
    0x3ff3dea64c123422ull, 0x3c859f48a72a4c6dull, 0x3ff4160a21f72e2aull, 0xbc58a78f4817895bull,
    0x3ff44e086061892dull, 0x3c4363ed60c2ac11ull, 0x3ff486a2b5c13cd0ull, 0x3c6ecce1daa10379ull,
    0x3ff4bfdad5362a27ull, 0x3c7690cebb7aafb0ull, 0x3ff4f9b2769d2ca7ull, 0xbc8f94340071a38eull,
    0x3ff5342b569d4f82ull, 0xbc78dec6bd0f385full, 0x3ff56f4736b527daull, 0x3c93350518fdd78eull,
    0x3ff5ab07dd485429ull, 0x3c9063e1e21c5409ull, 0x3ff5e76f15ad2148ull, 0x3c9432e62b64c035ull,
    0x3ff6247eb03a5585ull, 0xbc8c33c53bef4da8ull, 0x3ff6623882552225ull, 0xbc93cedd78565858ull,
    0x3ff6a09e667f3bcdull, 0xbc93b3efbf5e2228ull, 0x3ff6dfb23c651a2full, 0xbc6367efb86da9eeull,
    0x3ff71f75e8ec5f74ull, 0xbc781f647e5a3ecfull, 0x3ff75feb564267c9ull, 0xbc8619321e55e68aull,
    0x3ff7a11473eb0187ull, 0xbc7b32dcb94da51dull, 0x3ff7e2f336cf4e62ull, 0x3c65ebe1abd66c55ull,
    0x3ff82589994cce13ull, 0xbc9369b6f13b3734ull, 0x3ff868d99b4492edull, 0xbc94d450d872576eull,
    0x3ff8ace5422aa0dbull, 0x3c8db72fc1f0eab4ull, 0x3ff8f1ae99157736ull, 0x3c7bf68359f35f44ull,
    0x3ff93737b0cdc5e5ull, 0xbc5da9b88b6c1e29ull, 0x3ff97d829fde4e50ull, 0xbc92434322f4f9aaull,
    0x3ff9c49182a3f090ull, 0x3c71affc2b91ce27ull, 0x3ffa0c667b5de565ull, 0xbc87c50422622263ull,
    0x3ffa5503b23e255dull, 0xbc91bbd1d3bcbb15ull, 0x3ffa9e6b5579fdbfull, 0x3c8469846e735ab3ull,
    0x3ffae89f995ad3adull, 0x3c8c1a7792cb3387ull, 0x3ffb33a2b84f15fbull, 0xbc55c3d956dcaebaull,
    0x3ffb7f76f2fb5e47ull, 0xbc68d6f438ad9334ull, 0x3ffbcc1e904bc1d2ull, 0x3c74ffd70a5fddcdull,
    0x3ffc199bdd85529cull, 0x3c736eae30af0cb3ull, 0x3ffc67f12e57d14bull, 0x3c84e08fd10959acull,
    0x3ffcb720dcef9069ull, 0x3c676b2c6c921968ull, 0x3ffd072d4a07897cull, 0xbc8fad5d3ffffa6full,
    0x3ffd5818dcfba487ull, 0x3c74a385a63d07a7ull, 0x3ffda9e603db3285ull, 0x3c8e5a50d5c192acull,
    0x3ffdfc97337b9b5full, 0xbc82d52107b43e1full, 0x3ffe502ee78b3ff6ull, 0x3c74b604603a88d3ull,
    0x3ffea4afa2a490daull, 0xbc8ff7128fd391f0ull, 0x3ffefa1bee615a27ull, 0x3c8ec3bc41aa2008ull,
    0x3fff50765b6e4540ull, 0x3c8a64a931d185eeull, 0x3fffa7c1819e90d8ull, 0x3c77893b4d91cd9dull};

// SVML's scalar routine for |x| >= 0x1.61da04cbafe44p+9 and +-inf (no fma: SSE2 code)
static __device__ __noinline__ double np_exp_rare(double x) {
    const uint64_t u = (uint64_t)__double_as_longlong(x);
    const int ex = (int)((u >> 52) & 0x7ff);
    if (ex == 0x7ff) return (u == 0xfff0000000000000ull) ? 0.0 : __dmul_rn(x, x);
    if (ex <= 0x3ca) return __dadd_rn(1.0, x);
    if (x > bits_d(0x40862e42fefa39efull)) return __longlong_as_double(0x7ff0000000000000ll);  // max*max
    if (x < bits_d(0xc0874910d52d3051ull)) return 0.0;                                         // tiny*tiny
    const double shift = bits_d(0x4338000000000000ull);
    const double sv = __dadd_rn(__dmul_rn(x, bits_d(0x40571547652b82feull)), shift);
    const uint32_t k = (uint32_t)__double_as_longlong(sv);
    const int j = (int)(k & 0x3f);
    const double kd = __dsub_rn(sv, shift);
    const double r = __dsub_rn(__dsub_rn(x, __dmul_rn(kd, bits_d(0x3f862e42fefa0000ull))),
                               __dmul_rn(kd, bits_d(0x3d1cf79abc9e3b3aull)));
    double p = __dadd_rn(__dmul_rn(bits_d(0x3f56c16a1c2a3ffdull), r), bits_d(0x3f8111123aaf20d3ull));
    p = __dadd_rn(__dmul_rn(p, r), bits_d(0x3fa5555555558fccull));
    p = __dadd_rn(__dmul_rn(p, r), bits_d(0x3fc55555555548f8ull));
    p = __dadd_rn(__dmul_rn(p, r), 0.5);
    p = __dadd_rn(__dmul_rn(__dmul_rn(p, r), r), r);
    const double hi = bits_d(__ldg(kExpRare + 2 * j));
    p = __dmul_rn(__dadd_rn(p, bits_d(__ldg(kExpRare + 2 * j + 1))), hi);
    const int e = (int)(((k >> 6) + 0x3ff) & 0x7ff);
    if (!(x < bits_d(0xc086232bdd7abcd2ull))) {
        p = __dadd_rn(p, hi);
        if (e <= 0x7fe) return __dmul_rn(p, bits_d((uint64_t)e << 52));
        return __dmul_rn(__dmul_rn(p, bits_d((uint64_t)(e - 1) << 52)), 2.0);
    }
    const int e60 = (int)(((k >> 6) + 0x43b) & 0x7ff);  // subnormal result: scale by 2^60, round once
    const double sc = bits_d((uint64_t)e60 << 52);
    const double lo = __dmul_rn(p, sc), h1 = __dmul_rn(hi, sc), sum = __dadd_rn(h1, lo);
    const double tiny = bits_d(0x3c30000000000000ull);
    if (e60 <= 0x32) return __dmul_rn(sum, tiny);
    double lo2 = __dadd_rn(__dsub_rn(h1, sum), lo);
    const double t = __dmul_rn(sum, bits_d(0x41f8000000000000ull));
    const double v = __dsub_rn(__dadd_rn(sum, t), t);
    lo2 = __dadd_rn(lo2, __dsub_rn(sum, v));
    return __dadd_rn(__dmul_rn(v, tiny), __dmul_rn(lo2, tiny));
}

static __device__ __forceinline__ double np_exp(double x) {
    if (fabs(x) >= bits_d(0x40861da04cbafe44ull)) return np_exp_rare(x);
    const double shifter = bits_d(0x42f8000000003ff0ull);
    const double s = __fma_rz(x, bits_d(0x3ff71547652b82feull), shifter);
    const double k = __dsub_rn(s, shifter);
    const int j = (int)(__double_as_longlong(s) & 15);
    double r = __fma_rn(-k, bits_d(0x3fe62e42fefa39efull), x);
    r = __fma_rn(-bits_d(0x3c7abc9e3b39803full), k, r);
    r = __longlong_as_double(__double_as_longlong(r) & 0xbfffffffffffffffll);
    const double r2 = __dmul_rn(r, r);
    double a = __fma_rn(bits_d(0x3f57411836940c04ull), r, bits_d(0x3f81101cbbc265c0ull));
    const double b = __fma_rn(bits_d(0x3fa55557242d68feull), r, bits_d(0x3fc5555553939732ull));
    const double c = __fma_rn(bits_d(0x3fe000000000d008ull), r, bits_d(0x3fefffffffffff70ull));
    a = __fma_rn(r2, a, b);
    a = __fma_rn(r2, a, c);
    const double t2 = bits_d(__ldg(kExpT2 + j));
    double e = __fma_rn(a, r, bits_d(__ldg(kExpT1 + j)));
    e = __fma_rn(t2, e, t2);
    if (k != k) return k;  // NaN
    // |k| < 1021 here: 2^floor(k) is a normal double and the scaling is exact
    return __dmul_rn(e, bits_d((uint64_t)((int)floor(k) + 1023) << 52));
}

// IEEE division, = __ddiv_rn bit for bit (common.cuh ddiv_fast, slow path only when needed)
static __device__ __forceinline__ double ddiv_exact(double a, double b) {
    bool ok;
    const double q = ddiv_fast(a, b, ok);
    return ok ? q : __ddiv_rn(a, b);
}

// serial.py:49-50: 1.0 / (1.0 + np.exp(-2.0 * y / sigma2)), one rounding per operation
static __device__ __forceinline__ double awgn_prior(double y, double sigma2) {
    const double t = ddiv_exact(__dmul_rn(-2.0, y), sigma2);
    return ddiv_exact(1.0, __dadd_rn(1.0, np_exp(t)));
}

}  // namespace ldpc
