// harness_internal.h -- launchers of the bench harness library
// (libmersenne_b200_harness.so): workload generators and roofline probes.
// Not part of the product boundary; see include/mersenne_b200_harness.h.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../csrc/mb200_internal.h"  // sm_count(), device_id() of the product library

namespace mb200 {

// workload generators (kernels_gen.cu)
cudaError_t launch_gen_u32(uint64_t seed, uint64_t start, uint64_t n, uint32_t* out, cudaStream_t s);
cudaError_t launch_gen_u64(uint64_t seed, uint64_t start, uint64_t n, uint64_t* out, cudaStream_t s);
cudaError_t launch_gen_below_p61(uint64_t seed, uint64_t start, uint64_t n, uint64_t* out,
                                 unsigned long long* d_bad, cudaStream_t s);
cudaError_t launch_gen_pm_inputs(uint64_t seed, uint64_t c, uint64_t start, uint64_t n, uint64_t* out,
                                 unsigned long long* d_bad, cudaStream_t s);
cudaError_t launch_gen_zipf(uint64_t master, const uint64_t* cdf, uint32_t T, double c1,
                            double universe, uint64_t start, uint64_t n, uint32_t* keys,
                            int32_t* weights, cudaStream_t s);

// probes (kernels_probe.cu)
cudaError_t launch_probe_imad(int blocks, int threads, int iters, uint64_t* sink, cudaStream_t s);
cudaError_t launch_probe_atomics(int mode, int blocks, int threads, int iters, uint64_t* buf,
                                 uint64_t span, cudaStream_t s);
cudaError_t launch_probe_dsmem(int cluster, int mode, int blocks, int threads, int iters, uint32_t words,
                               uint64_t* out, cudaStream_t s);

}  // namespace mb200
