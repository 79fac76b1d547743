// harness_capi.cu -- C entries of the bench harness library
// (include/mersenne_b200_harness.h): seeded workload generators and the
// microbenchmarks that measure the roofline denominators.  Kept out of the
// product library so the drop-in ABI (include/mersenne_b200.h) is only the
// reference's surface.  Errors go through the product's last-error message.
#include <cuda_runtime.h>

#include <cmath>

#include "../../include/mersenne_b200_harness.h"
#include "../csrc/mb200_capi_util.h"
#include "harness_internal.h"

using namespace mb200;

extern "C" {

// ---------------------------------------------------------------- generators
int mb200_gen_u32_keys(uint64_t seed, uint64_t start, uint64_t n, uint32_t* d_out, void* stream) {
    cudaError_t e = launch_gen_u32(seed, start, n, d_out, (cudaStream_t)stream);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "gen");
}
int mb200_gen_u64_keys(uint64_t seed, uint64_t start, uint64_t n, uint64_t* d_out, void* stream) {
    cudaError_t e = launch_gen_u64(seed, start, n, d_out, (cudaStream_t)stream);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "gen");
}
int mb200_gen_below_p61(uint64_t seed, uint64_t start, uint64_t n, uint64_t* d_out, uint64_t* d_bad, void* stream) {
    cudaError_t e = launch_gen_below_p61(seed, start, n, d_out, (unsigned long long*)d_bad, (cudaStream_t)stream);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "gen");
}
int mb200_gen_pm_inputs(uint64_t seed, uint64_t c, uint64_t start, uint64_t n, uint64_t* d_out, uint64_t* d_bad,
                        void* stream) {
    cudaError_t e = launch_gen_pm_inputs(seed, c, start, n, d_out, (unsigned long long*)d_bad, (cudaStream_t)stream);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "gen");
}

int mb200_zipf_table(double alpha, uint32_t T, double universe, uint64_t* h_cdf, double* tail_c1) {
    if (alpha != 1.2) return fail(MB200_UNSUPPORTED, "zipf generator implements alpha = 1.2 (tail exponent 5)");
    if (T < 2 || !h_cdf || !tail_c1) return fail(MB200_INVALID_ARGUMENT, "bad zipf table arguments");
    double head = 0;
    for (uint32_t r = 1; r <= T; ++r) head += std::pow((double)r, -alpha);
    const double tail = (std::pow(T + 0.5, 1 - alpha) - std::pow(universe + 0.5, 1 - alpha)) / (alpha - 1);
    const double total = head + tail;
    double acc = 0;
    for (uint32_t r = 1; r <= T; ++r) {
        acc += std::pow((double)r, -alpha);
        const double sc = (acc / total) * 18446744073709551616.0;
        h_cdf[r - 1] = sc >= 18446744073709551615.0 ? ~0ull : (sc <= 0 ? 0 : (uint64_t)sc);
    }
    *tail_c1 = 1.0 - std::pow((universe + 0.5) / (T + 0.5), 1 - alpha);
    return MB200_OK;
}

int mb200_gen_zipf_items(uint64_t master_seed, const uint64_t* d_cdf, uint32_t T, double tail_c1, double universe,
                         uint64_t start, uint64_t n, uint32_t* d_keys, int32_t* d_weights, void* stream) {
    cudaError_t e = launch_gen_zipf(master_seed, d_cdf, T, tail_c1, universe, start, n, d_keys, d_weights,
                                    (cudaStream_t)stream);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "gen");
}

int mb200_probe_imad(int blocks, int threads, int iters, uint64_t* d_sink, void* stream) {
    cudaError_t e = launch_probe_imad(blocks, threads, iters, d_sink, (cudaStream_t)stream);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "probe");
}
int mb200_probe_atomics(int mode, int blocks, int threads, int iters, uint64_t* d_buf, uint64_t span, void* stream) {
    cudaError_t e = launch_probe_atomics(mode, blocks, threads, iters, d_buf, span, (cudaStream_t)stream);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "probe");
}

int mb200_probe_dsmem(int cluster, int mode, int blocks, int threads, int iters, uint32_t words, uint64_t* d_out,
                      void* stream) {
    cudaError_t e = launch_probe_dsmem(cluster, mode, blocks, threads, iters, words, d_out, (cudaStream_t)stream);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "probe");
}

}  // extern "C"
