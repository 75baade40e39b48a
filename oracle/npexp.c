/*
 * TEST INFRASTRUCTURE (oracle): restatement of the float64 exp that numpy
 * 2.3 evaluates on AVX512_SKX hosts, i.e. the exp inside the reference's
 * prior expression 1/(1+np.exp(-2y/sigma2)) (edgeldpc serial.py:49-50).
 * numpy is a third-party dependency of the reference (pyproject: numpy 2.x);
 * on hosts with AVX512_SKX its DOUBLE_exp loop hands contiguous,
 * non-overlapping arrays to Intel SVML's __svml_exp8_ha (numpy/_core/src/
 * umath/loops_umath_fp.dispatch.c.src; SVML sources vendored by numpy under
 * BSD-3).  That exp is not correctly rounded (about 4.6% of results differ
 * from glibc's), so device-computed priors are bit-identical to the
 * reference's only if they run the same algorithm.  The operation order,
 * rounding modes and constants below were read from numpy's own
 * _multiarray_umath binary (objdump of __svml_exp8_ha and
 * __svml_dexp_ha_cout_rare_internal; tables __svml_dexp_ha_data_internal_
 * avx512 and _imldExpHATab); tests/test_priors.py pins this file against
 * np.exp on the host, and csrc/priors.cu against this file.
 *
 * Main path (|x| < 0x1.61da04cbafe44p+9 or NaN), 16-entry table:
 *   s  = fma_rz(x, 1/ln2, 1.5*2^48 + 1023)     k = s - shifter = floor(16 x/ln2)/16
 *   j  = low 4 bits of s;  r = fma(-k, ln2_hi, x);  r = fma(-k, ln2_lo, r)
 *   P  = r^2 (r^2 (a6 r + a5) + (a4 r + a3)) + (a2 r + a1)     (fused)
 *   e  = T2[j] * (P r + T1[j]) + T2[j]                           (fused)
 *   exp(x) = e * 2^floor(k)
 * Rare path (|x| >= that bound, +-inf), scalar, 64-entry table, no fma.
 */
#include <fenv.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

static double bits(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
static uint64_t ubits(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
static double pow2(int e) { return bits((uint64_t)(e + 1023) << 52); }   /* normal range only */

static const uint64_t T2[16] = {   /* 2^(j/16) */
    0x3ff0000000000000, 0x3ff0b5586cf9890f, 0x3ff172b83c7d517b, 0x3ff2387a6e756238,
    0x3ff306fe0a31b715, 0x3ff3dea64c123422, 0x3ff4bfdad5362a27, 0x3ff5ab07dd485429,
    0x3ff6a09e667f3bcd, 0x3ff7a11473eb0187, 0x3ff8ace5422aa0db, 0x3ff9c49182a3f090,
    0x3ffae89f995ad3ad, 0x3ffc199bdd85529c, 0x3ffd5818dcfba487, 0x3ffea4afa2a490da,
};
static const uint64_t T1[16] = {   /* tails */
    0x0000000000000000, 0x3c979aa65d837b6d, 0xbc801b15eaa59348, 0x3c968efde3a8a894,
    0x3c834d754db0abb6, 0x3c859f48a72a4c6d, 0x3c7690cebb7aafb0, 0x3c9063e1e21c5409,
    0xbc93b3efbf5e2228, 0xbc7b32dcb94da51d, 0x3c8db72fc1f0eab4, 0x3c71affc2b91ce27,
    0x3c8c1a7792cb3387, 0x3c736eae30af0cb3, 0x3c74a385a63d07a7, 0xbc8ff7128fd391f0,
};
static const uint64_t RARE[128] = {   /* pairs (2^(j/64) hi, lo) */
    0x3ff0000000000000, 0x0000000000000000, 0x3ff02c9a3e778061, 0xbc7160139cd8dc5d,
    0x3ff059b0d3158574, 0x3c8cd2523567f613, 0x3ff0874518759bc8, 0x3c60f74e61e6c861,
    0x3ff0b5586cf9890f, 0x3c979aa65d837b6d, 0x3ff0e3ec32d3d1a2, 0x3c3ebe3d702f9cd1,
    0x3ff11301d0125b51, 0xbc9556522a2fbd0e, 0x3ff1429aaea92de0, 0xbc91c923b9d5f416,
    0x3ff172b83c7d517b, 0xbc801b15eaa59348, 0x3ff1a35beb6fcb75, 0x3c8b898c3f1353bf,
    0x3ff1d4873168b9aa, 0x3c9aecf73e3a2f60, 0x3ff2063b88628cd6, 0x3c8a6f4144a6c38d,
    0x3ff2387a6e756238, 0x3c968efde3a8a894, 0x3ff26b4565e27cdd, 0x3c80472b981fe7f2,
    0x3ff29e9df51fdee1, 0x3c82f7e16d09ab31, 0x3ff2d285a6e4030b, 0x3c8b3782720c0ab4,
    0x3ff306fe0a31b715, 0x3c834d754db0abb6, 0x3ff33c08b26416ff, 0x3c8fdd395dd3f84a,
    0x3ff371a7373aa9cb, 0xbc924aedcc4b5068, 0x3ff3a7db34e59ff7, 0xbc71d1e83e9436d2,
    0x3ff3dea64c123422, 0x3c859f48a72a4c6d, 0x3ff4160a21f72e2a, 0xbc58a78f4817895b,
    0x3ff44e086061892d, 0x3c4363ed60c2ac11, 0x3ff486a2b5c13cd0, 0x3c6ecce1daa10379,
    0x3ff4bfdad5362a27, 0x3c7690cebb7aafb0, 0x3ff4f9b2769d2ca7, 0xbc8f94340071a38e,
    0x3ff5342b569d4f82, 0xbc78dec6bd0f385f, 0x3ff56f4736b527da, 0x3c93350518fdd78e,
    0x3ff5ab07dd485429, 0x3c9063e1e21c5409, 0x3ff5e76f15ad2148, 0x3c9432e62b64c035,
    0x3ff6247eb03a5585, 0xbc8c33c53bef4da8, 0x3ff6623882552225, 0xbc93cedd78565858,
    0x3ff6a09e667f3bcd, 0xbc93b3efbf5e2228, 0x3ff6dfb23c651a2f, 0xbc6367efb86da9ee,
    0x3ff71f75e8ec5f74, 0xbc781f647e5a3ecf, 0x3ff75feb564267c9, 0xbc8619321e55e68a,
    0x3ff7a11473eb0187, 0xbc7b32dcb94da51d, 0x3ff7e2f336cf4e62, 0x3c65ebe1abd66c55,
    0x3ff82589994cce13, 0xbc9369b6f13b3734, 0x3ff868d99b4492ed, 0xbc94d450d872576e,
    0x3ff8ace5422aa0db, 0x3c8db72fc1f0eab4, 0x3ff8f1ae99157736, 0x3c7bf68359f35f44,
    0x3ff93737b0cdc5e5, 0xbc5da9b88b6c1e29, 0x3ff97d829fde4e50, 0xbc92434322f4f9aa,
    0x3ff9c49182a3f090, 0x3c71affc2b91ce27, 0x3ffa0c667b5de565, 0xbc87c50422622263,
    0x3ffa5503b23e255d, 0xbc91bbd1d3bcbb15, 0x3ffa9e6b5579fdbf, 0x3c8469846e735ab3,
    0x3ffae89f995ad3ad, 0x3c8c1a7792cb3387, 0x3ffb33a2b84f15fb, 0xbc55c3d956dcaeba,
    0x3ffb7f76f2fb5e47, 0xbc68d6f438ad9334, 0x3ffbcc1e904bc1d2, 0x3c74ffd70a5fddcd,
    0x3ffc199bdd85529c, 0x3c736eae30af0cb3, 0x3ffc67f12e57d14b, 0x3c84e08fd10959ac,
    0x3ffcb720dcef9069, 0x3c676b2c6c921968, 0x3ffd072d4a07897c, 0xbc8fad5d3ffffa6f,
    0x3ffd5818dcfba487, 0x3c74a385a63d07a7, 0x3ffda9e603db3285, 0x3c8e5a50d5c192ac,
    0x3ffdfc97337b9b5f, 0xbc82d52107b43e1f, 0x3ffe502ee78b3ff6, 0x3c74b604603a88d3,
    0x3ffea4afa2a490da, 0xbc8ff7128fd391f0, 0x3ffefa1bee615a27, 0x3c8ec3bc41aa2008,
    0x3fff50765b6e4540, 0x3c8a64a931d185ee, 0x3fffa7c1819e90d8, 0x3c77893b4d91cd9d,
};

static double fma_rz(double a, double b, double c)
{
    int mode = fegetround();
    fesetround(FE_TOWARDZERO);
    volatile double r = fma(a, b, c);
    fesetround(mode);
    return r;
}

static double rare(double x)
{
    uint64_t u = ubits(x);
    int ex = (int)((u >> 52) & 0x7ff);
    if (ex == 0x7ff) return (u == 0xfff0000000000000ull) ? 0.0 : x * x;
    if (ex <= 0x3ca) return 1.0 + x;
    if (x > bits(0x40862e42fefa39ef)) { volatile double h = bits(0x7fefffffffffffff); return h * h; }
    if (x < bits(0xc0874910d52d3051)) { volatile double t = bits(0x0010000000000001); return t * t; }
    double s = x * bits(0x40571547652b82fe) + bits(0x4338000000000000);
    uint32_t k = (uint32_t)ubits(s);
    int j = (int)(k & 0x3f);
    double kd = s - bits(0x4338000000000000);
    double r = (x - kd * bits(0x3f862e42fefa0000)) - kd * bits(0x3d1cf79abc9e3b3a);
    double p = bits(0x3f56c16a1c2a3ffd) * r + bits(0x3f8111123aaf20d3);
    p = p * r + bits(0x3fa5555555558fcc);
    p = p * r + bits(0x3fc55555555548f8);
    p = p * r + 0.5;
    p = p * r * r + r;
    double hi = bits(RARE[2 * j]);
    p = (p + bits(RARE[2 * j + 1])) * hi;
    int e = (int)(((k >> 6) + 0x3ff) & 0x7ff);
    if (!(x < bits(0xc086232bdd7abcd2))) {
        p = p + hi;
        if (e <= 0x7fe) return p * bits((uint64_t)e << 52);
        return p * bits((uint64_t)(e - 1) << 52) * 2.0;
    }
    /* the result is subnormal: scale by 2^60 first, round once at the end */
    int e60 = (int)(((k >> 6) + 0x43b) & 0x7ff);
    double sc = bits((uint64_t)e60 << 52);
    double lo = p * sc, h1 = hi * sc, sum = h1 + lo;
    const double tiny = bits(0x3c30000000000000);
    if (e60 <= 0x32) return sum * tiny;
    double lo2 = (h1 - sum) + lo;
    double t = sum * bits(0x41f8000000000000);
    double v = (sum + t) - t;
    double w = sum - v;
    lo2 = lo2 + w;
    return v * tiny + lo2 * tiny;
}

double oracle_npexp(double x)
{
    if (fabs(x) >= bits(0x40861da04cbafe44)) return rare(x);
    const double shifter = bits(0x42f8000000003ff0);
    double s = fma_rz(x, bits(0x3ff71547652b82fe), shifter);
    double k = s - shifter;
    int j = (int)(ubits(s) & 15);
    double r = fma(-k, bits(0x3fe62e42fefa39ef), x);
    r = fma(-bits(0x3c7abc9e3b39803f), k, r);
    r = bits(ubits(r) & 0xbfffffffffffffffull);
    double r2 = r * r;
    double a = fma(bits(0x3f57411836940c04), r, bits(0x3f81101cbbc265c0));
    double b = fma(bits(0x3fa55557242d68fe), r, bits(0x3fc5555553939732));
    double c = fma(bits(0x3fe000000000d008), r, bits(0x3fefffffffffff70));
    a = fma(r2, a, b);
    a = fma(r2, a, c);
    double e = fma(a, r, bits(T1[j]));
    e = fma(bits(T2[j]), e, bits(T2[j]));
    if (k != k) return k;                                    /* NaN: scalef returns it */
    return e * pow2((int)floor(k));                          /* |k| < 1021: exact */
}

/* The reference prior expression, 1/(1 + exp(-2 y / sigma2)), one rounding per operation. */
void oracle_priors_awgn(const double *y, long n, double sigma2, double *out)
{
    for (long i = 0; i < n; ++i) {
        double t = (-2.0 * y[i]) / sigma2;
        out[i] = 1.0 / (1.0 + oracle_npexp(t));
    }
}

void oracle_npexp_array(const double *x, long n, double *out)
{
    for (long i = 0; i < n; ++i) out[i] = oracle_npexp(x[i]);
}
