// mb200_capi_util.h -- helpers shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <functional>
#include <string>

#include "../../include/mersenne_b200.h"
#include "mb200_internal.h"

namespace mb200 {

extern thread_local std::string g_last_error;
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
bool prime_exponent(unsigned b);
int build_sketch_params(const mb200_sketch_desc* d, SketchParams& sp);
int check_keys(const void* d_keys, int key_width, uint64_t n, unsigned key_bits, cudaStream_t s);
// mb200_cs_update without the data-dependent key check (caller validated)
int cs_update_nocheck(const mb200_sketch_desc* desc, const void* d_keys, int key_width, const void* d_weights,
                      int weight_kind, uint64_t n, int64_t* d_counters, void* stream);
int count_on_device(const std::function<cudaError_t(unsigned long long*, cudaStream_t)>& launch, cudaStream_t s,
                    unsigned long long* out);

}  // namespace mb200
