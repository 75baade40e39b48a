// priors.cu -- AWGN priors from channel observations on the device (serial.py:39-50),
// bit-identical to the reference's numpy expression (priors.cuh).  The decode path
// fuses the prior into the layout transpose (kernels_misc.cu k_transpose_priors);
// these entry points are the standalone forms (tests, callers that keep priors).
#include "common.cuh"
#include "priors.cuh"

namespace ldpc {
namespace {

// y [B][n] -> p [B][n]; sigma2 per codeword.  Grid-stride over rows x columns.
__global__ void k_priors_awgn(const double *__restrict__ y, const double *__restrict__ sig2, int32_t B, int32_t n,
                              double *__restrict__ p) {
    const int64_t total = (int64_t)B * n;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(k / n);
        p[k] = awgn_prior(__ldcs(y + k), __ldg(sig2 + c));
    }
}

__global__ void k_npexp(const double *__restrict__ x, int64_t count, double *__restrict__ out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x)
        out[k] = np_exp(x[k]);
}

unsigned grid_for(int64_t work) {
    int64_t b = (work + 255) / 256;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}

}  // namespace
}  // namespace ldpc

using namespace ldpc;

extern "C" int ldpc_priors_awgn(const double *y_dev, const double *sigma2_dev, int32_t B, int32_t n, double *p_dev,
                                void *stream) {
    LDPC_ARG_CHECK(y_dev && sigma2_dev && p_dev, "NULL argument");
    LDPC_ARG_CHECK(B >= 0 && n >= 0, "negative size");
    if ((int64_t)B * n == 0) return LDPC_OK;
    k_priors_awgn<<<grid_for((int64_t)B * n), 256, 0, (cudaStream_t)stream>>>(y_dev, sigma2_dev, B, n, p_dev);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}

extern "C" int ldpc_npexp(const double *x_dev, int64_t count, double *out_dev, void *stream) {
    LDPC_ARG_CHECK(x_dev && out_dev && count >= 0, "bad argument");
    if (count == 0) return LDPC_OK;
    k_npexp<<<grid_for(count), 256, 0, (cudaStream_t)stream>>>(x_dev, count, out_dev);
    LDPC_CHECK_LAUNCH();
    return LDPC_OK;
}
