// Stand-alone driver of cs_private89_kernel for A/B timing of source variants
// (tools/kvariants/c4_variants.py compiles it once per -D flag set).
#include "mb200_sketch_dev.cuh"
namespace mb200 {
__device__ unsigned long long g_hot_stats[8];
}
#include "mb200_private89.cuh"

using namespace mb200;

extern "C" float c4_run(const uint64_t* keys, uint64_t n, const uint32_t* coef12, int reps, void* scratch,
                        int64_t* table, const uint32_t* go) {
    Coef89 c;
    for (int j = 0; j < 4; ++j)
        for (int l = 0; l < 3; ++l) c.a[j][l] = coef12[3 * j + l];
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto fp = cs_private89_kernel<16, false>;
    cudaFuncSetAttribute(fp, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 << 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        fp<<<sms, kP89Threads, 2 << 16>>>(c, reinterpret_cast<const ulonglong2*>(keys), n / 2, nullptr,
                                          reinterpret_cast<uint4*>(scratch), reinterpret_cast<uint64_t*>(table), go);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    return cudaGetLastError() == cudaSuccess ? best : -1.0f;
}
