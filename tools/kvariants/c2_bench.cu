// Stand-alone config-2 hash kernel variants (degree k-1 mod 2^61-1, u64 keys in
// [0, p)) for A/B timing (tools/kvariants/c2_variants.py).  LOCK = 1: the KU
// Horner chains of a thread advance in lockstep (step outer, keys inner).
#include <cstdint>

#include "mb200_device.cuh"

using namespace mb200;

#ifndef KU
#define KU 8
#endif
#ifndef LOCK
#define LOCK 1
#endif
#ifndef NT
#define NT 256
#endif

template <int K>
__global__ void __launch_bounds__(NT) c2_kernel(const u64* __restrict__ keys, uint64_t n, const u64* __restrict__ cg,
                                                u64* __restrict__ out) {
    u64 a[K];
#pragma unroll
    for (int i = 0; i < K; ++i) a[i] = cg[i];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; base + 1 < n;
         base += stride * 2 * (KU / 2)) {
        u64 x[KU], y[KU];
#pragma unroll
        for (int u = 0; u < KU / 2; ++u) {
            const uint64_t j = base + (uint64_t)u * stride * 2;
            if (j + 1 < n) {
                const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2*>(keys + j));
                x[2 * u] = h61_key64(v.x);
                x[2 * u + 1] = h61_key64(v.y);
            } else {
                x[2 * u] = x[2 * u + 1] = 0;
            }
        }
#if LOCK
#pragma unroll
        for (int u = 0; u < KU; ++u) y[u] = a[K - 1];
#pragma unroll
        for (int i = K - 2; i >= 0; --i) {
#pragma unroll
            for (int u = 0; u < KU; ++u) {
                if ((K - 2 - i) > 0 && (K - 2 - i) % kLazySteps == 0) y[u] = h61_fold(y[u]);
                y[u] = h61_step64(y[u], x[u], a[i]);
            }
        }
#else
#pragma unroll
        for (int u = 0; u < KU; ++u) y[u] = h61_eval64<K>(a, x[u]);
#endif
#pragma unroll
        for (int u = 0; u < KU / 2; ++u) {
            const uint64_t j = base + (uint64_t)u * stride * 2;
            if (j + 1 < n) {
                ulonglong2 h;
                h.x = h61_finish(y[2 * u]);
                h.y = h61_finish(y[2 * u + 1]);
                __stcs(reinterpret_cast<ulonglong2*>(out + j), h);
            }
        }
    }
}

// Preconditioned degree-7 evaluation (Knuth 4.6.4, adapted coefficients):
// u(x) = a7 (x + s) U(x) + r0 with the monic sextic U = (w + z + al4) w + al5,
// w = (x + al2) z + al3, z = (x + al0) x + al1: five modular products instead of
// Horner's seven.  plan = {al0..al5, s, a7, r0}.
template <bool SHIFT>
__global__ void __launch_bounds__(NT) c2_pre_kernel(const u64* __restrict__ keys, uint64_t n, const u64* __restrict__ pg,
                                                    u64* __restrict__ out) {
    u64 al[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) al[i] = pg[i];
    const u64 s = pg[6], a7 = pg[7], r0 = pg[8];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; base + 1 < n;
         base += stride * 2 * (KU / 2)) {
        u64 x[KU], y[KU];
#pragma unroll
        for (int u = 0; u < KU / 2; ++u) {
            const uint64_t j = base + (uint64_t)u * stride * 2;
            if (j + 1 < n) {
                const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2*>(keys + j));
                x[2 * u] = h61_key64(v.x);
                x[2 * u + 1] = h61_key64(v.y);
            } else {
                x[2 * u] = x[2 * u + 1] = 0;
            }
        }
#pragma unroll
        for (int u = 0; u < KU; ++u) {
            const u64 x0 = x[u];
            const u64 z = h61_fold(h61_step64(x0 + al[0], x0, al[1]));
            const u64 w = h61_fold(h61_step64(x0 + al[2], z, al[3]));
            u64 U = h61_step64(w + z + al[4], w, al[5]);
            u64 V;
            if (SHIFT) V = h61_step64(h61_fold(U), x0 + s, 0);
            else V = h61_step64(U, x0, 0);
            y[u] = h61_step64(h61_fold(V), a7, r0);
        }
#pragma unroll
        for (int u = 0; u < KU / 2; ++u) {
            const uint64_t j = base + (uint64_t)u * stride * 2;
            if (j + 1 < n) {
                ulonglong2 h;
                h.x = h61_finish(y[2 * u]);
                h.y = h61_finish(y[2 * u + 1]);
                __stcs(reinterpret_cast<ulonglong2*>(out + j), h);
            }
        }
    }
}

extern "C" float c2_run_pre(const uint64_t* keys, uint64_t n, const uint64_t* d_plan, int shift, int reps, uint64_t* out) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int per = 0;
    auto fn = shift ? c2_pre_kernel<true> : c2_pre_kernel<false>;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, NT, 0);
    const unsigned grid = (unsigned)(sms * (per > 0 ? per : 1));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        fn<<<grid, NT>>>(keys, n, d_plan, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    return cudaGetLastError() == cudaSuccess ? best : -1.0f;
}

extern "C" float c2_run(const uint64_t* keys, uint64_t n, const uint64_t* d_coeffs, int k, int reps, uint64_t* out) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int per = 0;
    auto fn = k == 8 ? c2_kernel<8> : c2_kernel<4>;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, NT, 0);
    const unsigned grid = (unsigned)(sms * (per > 0 ? per : 1));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        fn<<<grid, NT>>>(keys, n, d_coeffs, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    return cudaGetLastError() == cudaSuccess ? best : -1.0f;
}
