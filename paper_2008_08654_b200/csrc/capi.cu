// capi.cu -- device-array entries of the C-ABI boundary (include/mersenne_b200.h):
// argument validation with the reference's exception classes and messages,
// data-dependent domain checks, and kernel dispatch.  No CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mersenne_b200.h"
#include "mb200_capi_util.h"
#include "mb200_internal.h"

using namespace mb200;

namespace mb200 {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    return fail(MB200_CUDA_ERROR, std::string(where) + ": " + cudaGetErrorString(e));
}

bool prime_exponent(unsigned b) {
    static const unsigned kPrimes[] = {2, 3, 5, 7, 13, 17, 19, 31, 61, 89, 107, 127};  // field.cpp:12
    for (unsigned p : kPrimes)
        if (p == b) return true;
    return false;
}

// Synchronous device counter read used by the all-or-nothing domain checks.
int count_on_device(const std::function<cudaError_t(unsigned long long*, cudaStream_t)>& launch,
                    cudaStream_t s, unsigned long long* out) {
    unsigned long long* d = nullptr;
    cudaError_t e = cudaMallocAsync(&d, sizeof(*d), s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
    e = cudaMemsetAsync(d, 0, sizeof(*d), s);
    if (e == cudaSuccess) e = launch(d, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, sizeof(*d), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(d, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "domain check");
    return MB200_OK;
}

int check_keys(const void* d_keys, int key_width, uint64_t n, unsigned key_bits, cudaStream_t s) {
    if (key_bits >= (unsigned)key_width || n == 0) return MB200_OK;
    unsigned long long bad = 0;
    int rc = count_on_device(
        [&](unsigned long long* d, cudaStream_t st) {
            return launch_count_out_of_domain(d_keys, key_width, n, key_bits, d, st);
        },
        s, &bad);
    if (rc) return rc;
    if (bad) return fail(MB200_DOMAIN_ERROR, "key outside domain");  // polyhash.cpp:60
    return MB200_OK;
}

int build_sketch_params(const mb200_sketch_desc* d, SketchParams& sp) {
    if (!d) return fail(MB200_INVALID_ARGUMENT, "null sketch descriptor");
    if (d->rows == 0) return fail(MB200_INVALID_ARGUMENT, "need at least one row");  // sketch.cpp:71
    if (d->rows > (unsigned)kMaxFamilies) return fail(MB200_UNSUPPORTED, "GPU path supports at most 16 rows");
    if (d->k == 0) return fail(MB200_INVALID_ARGUMENT, "independence degree must be at least 1");
    if (d->k > (unsigned)kMaxK) return fail(MB200_UNSUPPORTED, "GPU path supports independence <= 16");
    if (d->b < 2 || d->b > 127) return fail(MB200_INVALID_ARGUMENT, "exponent must be in [2, 127]");
    if (d->width < 2) return fail(MB200_INVALID_ARGUMENT, "width must be at least 2");  // sketch.cpp:99
    const bool pow2 = (d->width & (d->width - 1)) == 0;
    switch (d->splitter) {
        case MB200_SPLIT_POW2:
        case MB200_SPLIT_TWO_FOR_ONE:
            // sketch.cpp:101-107 (b >= 64 always admits a 64-bit width)
            if (!pow2 || (d->b < 64 && d->width >= (1ull << d->b)))
                return fail(MB200_INVALID_ARGUMENT, "width must be a power of two strictly inside the hash range");
            break;
        case MB200_SPLIT_UNIFORM_ARB:
        case MB200_SPLIT_MERSENNE_ARB:
            if (d->b < 64 && d->width > (1ull << (d->b - 1)))
                return fail(MB200_INVALID_ARGUMENT, "width exceeds half the hash range");  // sketch.cpp:109-113
            break;
        default:
            return fail(MB200_INVALID_ARGUMENT, "unknown splitter");
    }
    if ((unsigned __int128)d->rows * d->width > ((unsigned __int128)1 << 34))
        return fail(MB200_INVALID_ARGUMENT, "sketch dimensions too large");  // sketch.cpp:116-118
    // key domain: polyhash.cpp:48-57 (p >= 2u - 1); b == 61 also admits full 64-bit keys
    if (d->key_bits > 64) return fail(MB200_UNSUPPORTED, "keys wider than 64 bits");
    if (d->b != 61 && d->b <= 64 && d->key_bits > d->b - 1)
        return fail(MB200_INVALID_ARGUMENT, "modulus too small for key domain");
    const unsigned lw = (unsigned)__builtin_ctzll(d->width);
    const unsigned families = d->splitter == MB200_SPLIT_TWO_FOR_ONE ? (d->rows + 1) / 2 : d->rows;
    if (d->splitter == MB200_SPLIT_TWO_FOR_ONE) {
        // row j uses index bits [l j, l j + l) and sign bit b-1-j (disjoint, in the low word)
        if (2 * lw + 2 > d->b || 2 * lw > 64)
            return fail(MB200_INVALID_ARGUMENT, "two-for-one split needs 2 log2(width) + 2 <= b");
    }
    if (families * d->k > (unsigned)kMaxCoeffs) return fail(MB200_UNSUPPORTED, "too many coefficients");
    if (!d->coeffs_lo) return fail(MB200_INVALID_ARGUMENT, "null coefficients");
    std::memset(&sp, 0, sizeof(sp));
    sp.rows = d->rows;
    sp.families = families;
    sp.k = d->k;
    sp.b = d->b;
    sp.lw = lw;
    sp.splitter = (uint32_t)d->splitter;
    sp.width = d->width;
    sp.p = d->b < 64 ? (1ull << d->b) - 1 : ~0ull;
    for (unsigned i = 0; i < families * d->k; ++i) {
        sp.lo[i] = d->coeffs_lo[i];
        sp.hi[i] = d->coeffs_hi ? d->coeffs_hi[i] : 0;
        const bool reduced = d->b < 64 ? sp.lo[i] < sp.p && sp.hi[i] == 0
                                       : (sp.hi[i] < (1ull << (d->b - 64)) - 1) ||
                                             (sp.hi[i] == (1ull << (d->b - 64)) - 1 && sp.lo[i] != ~0ull);
        if (!reduced) return fail(MB200_INVALID_ARGUMENT, "coefficient not reduced");  // polyhash.cpp:43
    }
    return MB200_OK;
}

int cs_update_nocheck(const mb200_sketch_desc* desc, const void* d_keys, int key_width, const void* d_weights,
                      int weight_kind, uint64_t n, int64_t* d_counters, void* stream) {
    SketchParams sp;
    if (int rc = build_sketch_params(desc, sp)) return rc;
    if (n == 0) return MB200_OK;
    cudaError_t e = launch_cs_update(sp, d_keys, key_width, d_weights, weight_kind, n, d_counters, (cudaStream_t)stream);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "mb200_cs_update");
}

}  // namespace mb200

extern "C" {

const char* mb200_last_error(void) { return g_last_error.c_str(); }
int mb200_abi_version(void) { return MB200_ABI_VERSION; }

int mb200_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int good = 0;
    for (int d = 0; d < n; ++d) {
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, d) == cudaSuccess && prop.major == 10) ++good;
    }
    return good;
}

int mb200_mersenne_modulus_check(unsigned b, int require_prime) {
    if (b < 2 || b > 127) return fail(MB200_INVALID_ARGUMENT, "exponent must be in [2, 127]");
    if (require_prime && !prime_exponent(b))
        return fail(MB200_INVALID_ARGUMENT, "2^b - 1 is not prime for this exponent");
    return MB200_OK;
}

int mb200_hash61(const void* d_keys, int key_width, uint64_t n, unsigned b, const uint64_t* coeffs, unsigned k,
                 unsigned key_bits, uint64_t* d_out, void* stream) {
    if (b < 2 || b > 61) return fail(MB200_INVALID_ARGUMENT, "mb200_hash61 needs 2 <= b <= 61");
    if (k == 0) return fail(MB200_INVALID_ARGUMENT, "independence degree must be at least 1");
    if (k > (unsigned)kMaxK) return fail(MB200_UNSUPPORTED, "GPU path supports independence <= 16");
    if (key_width != 32 && key_width != 64) return fail(MB200_INVALID_ARGUMENT, "key width must be 32 or 64");
    if (key_bits > 64) return fail(MB200_INVALID_ARGUMENT, "key domain exceeds 64 bits");
    if (b != 61 && key_bits > b - 1) return fail(MB200_INVALID_ARGUMENT, "modulus too small for key domain");
    if (!coeffs) return fail(MB200_INVALID_ARGUMENT, "null coefficients");
    HashParams hp;
    std::memset(&hp, 0, sizeof(hp));
    hp.b = b;
    hp.k = k;
    hp.p = (1ull << b) - 1;
    for (unsigned i = 0; i < k; ++i) {
        if (coeffs[i] >= hp.p) return fail(MB200_INVALID_ARGUMENT, "coefficient not reduced");
        hp.lo[i] = coeffs[i];
    }
    if (n == 0) return MB200_OK;
    if (!d_keys || !d_out) return fail(MB200_INVALID_ARGUMENT, "null buffer");
    cudaStream_t s = (cudaStream_t)stream;
    if (int rc = check_keys(d_keys, key_width, n, key_bits, s)) return rc;
    cudaError_t e;
    if (b == 61 && key_width == 64 && k == 8) {
        // degree 7: five modular products per key with adapted coefficients instead
        // of Horner's seven (same value; host/precond61.cpp)
        // (a family's plan is kept: the adaptation takes tens of microseconds on the host)
        thread_local uint64_t cached_coeffs[8], cached_plan[9];
        thread_local int cached_rc = -1;
        if (cached_rc < 0 || std::memcmp(cached_coeffs, coeffs, sizeof(cached_coeffs)) != 0) {
            std::memcpy(cached_coeffs, coeffs, sizeof(cached_coeffs));
            cached_rc = mb200_precondition61(coeffs, cached_plan);
        }
        if (cached_rc == MB200_OK) {
            for (int i = 0; i < 9; ++i) hp.hi[i] = cached_plan[i];
            hp.pre = cached_plan[6] ? 2 : 1;
        }
    }
    if (b == 61 && key_width == 32) e = launch_hash61_key32((const uint32_t*)d_keys, n, hp, d_out, s);
    else if (b == 61) e = launch_hash61_key64((const uint64_t*)d_keys, n, hp, d_out, s);
    else e = launch_hash_generic(d_keys, key_width, n, hp, d_out, s);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "mb200_hash61");
}

int mb200_hash89(const uint64_t* d_keys, uint64_t n, const uint64_t* coeffs_lo, const uint64_t* coeffs_hi,
                 unsigned k, unsigned key_bits, uint64_t* d_out_lo, uint64_t* d_out_hi, void* stream) {
    if (k == 0) return fail(MB200_INVALID_ARGUMENT, "independence degree must be at least 1");
    if (k > (unsigned)kMaxK) return fail(MB200_UNSUPPORTED, "GPU path supports independence <= 16");
    if (key_bits > 64) return fail(MB200_UNSUPPORTED, "keys wider than 64 bits");
    if (!coeffs_lo || !coeffs_hi) return fail(MB200_INVALID_ARGUMENT, "null coefficients");
    HashParams hp;
    std::memset(&hp, 0, sizeof(hp));
    hp.b = 89;
    hp.k = k;
    for (unsigned i = 0; i < k; ++i) {
        const bool reduced = coeffs_hi[i] < (1ull << 25) - 1 || (coeffs_hi[i] == (1ull << 25) - 1 && coeffs_lo[i] != ~0ull);
        if (!reduced) return fail(MB200_INVALID_ARGUMENT, "coefficient not reduced");
        hp.lo[i] = coeffs_lo[i];
        hp.hi[i] = coeffs_hi[i];
    }
    if (n == 0) return MB200_OK;
    if (!d_keys || !d_out_lo || !d_out_hi) return fail(MB200_INVALID_ARGUMENT, "null buffer");
    cudaStream_t s = (cudaStream_t)stream;
    if (int rc = check_keys(d_keys, 64, n, key_bits, s)) return rc;
    cudaError_t e = launch_hash89(d_keys, n, hp, d_out_lo, d_out_hi, s);
    if (e == cudaErrorMisalignedAddress) return fail(MB200_INVALID_ARGUMENT, "mb200_hash89 needs 16-byte aligned buffers");
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "mb200_hash89");
}

int mb200_hash_wide(const uint64_t* d_keys, uint64_t n, unsigned b, const uint64_t* coeffs_lo,
                    const uint64_t* coeffs_hi, unsigned k, unsigned key_bits, uint64_t* d_out_lo, uint64_t* d_out_hi,
                    void* stream) {
    if (b < 62 || b > 127) return fail(MB200_INVALID_ARGUMENT, "mb200_hash_wide needs 62 <= b <= 127");
    if (k == 0) return fail(MB200_INVALID_ARGUMENT, "independence degree must be at least 1");
    if (k > (unsigned)kMaxK) return fail(MB200_UNSUPPORTED, "GPU path supports independence <= 16");
    if (key_bits > 64) return fail(MB200_UNSUPPORTED, "keys wider than 64 bits");
    if (b <= 64 && key_bits > b - 1) return fail(MB200_INVALID_ARGUMENT, "modulus too small for key domain");
    if (!coeffs_lo || !coeffs_hi) return fail(MB200_INVALID_ARGUMENT, "null coefficients");
    HashParams hp;
    std::memset(&hp, 0, sizeof(hp));
    hp.b = b;
    hp.k = k;
    for (unsigned i = 0; i < k; ++i) {  // coefficient < p = 2^b - 1 (polyhash.cpp:43)
        const unsigned __int128 a = ((unsigned __int128)coeffs_hi[i] << 64) | coeffs_lo[i];
        const unsigned __int128 p = (((unsigned __int128)1) << b) - 1;
        if (a >= p) return fail(MB200_INVALID_ARGUMENT, "coefficient not reduced");
        hp.lo[i] = coeffs_lo[i];
        hp.hi[i] = coeffs_hi[i];
    }
    if (n == 0) return MB200_OK;
    if (!d_keys || !d_out_lo || !d_out_hi) return fail(MB200_INVALID_ARGUMENT, "null buffer");
    cudaStream_t s = (cudaStream_t)stream;
    if (int rc = check_keys(d_keys, 64, n, key_bits, s)) return rc;
    cudaError_t e = launch_hash_wide(d_keys, n, hp, d_out_lo, d_out_hi, s);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "mb200_hash_wide");
}

int mb200_pm_divmod(const uint64_t* d_v, uint64_t n, unsigned b, uint64_t c, unsigned m_iters, uint64_t* d_q,
                    uint64_t* d_r, uint64_t* d_overflow, void* stream) {
    if (b < 2 || b > 64) {
        if (b >= 2 && b <= 127) return fail(MB200_UNSUPPORTED, "GPU division supports b <= 64");
        return fail(MB200_INVALID_ARGUMENT, "width must be in [2, 127]");
    }
    unsigned m = 0;
    uint64_t max_input[4];
    if (int rc = mb200_pm_modulus(b, c, 0, m_iters, &m, max_input)) return rc;
    if (n == 0) return MB200_OK;
    if (!d_v || !d_q) return fail(MB200_INVALID_ARGUMENT, "null buffer");  // d_r null: quotient only
    cudaStream_t s = (cudaStream_t)stream;
    if (max_input[2] == 0 && max_input[3] == 0) {  // domain narrower than u128: check
        unsigned long long bad = 0;
        int rc = count_on_device(
            [&](unsigned long long* d, cudaStream_t st) {
                return launch_count_above(d_v, n, max_input[0], max_input[1], d, st);
            },
            s, &bad);
        if (rc) return rc;
        if (bad) return fail(MB200_DOMAIN_ERROR, "input exceeds division domain for m iterations");  // field.cpp:262
    }
    unsigned long long* flags = reinterpret_cast<unsigned long long*>(d_overflow);
    unsigned long long* scratch = nullptr;
    cudaError_t e = cudaSuccess;
    if (!flags) {
        e = cudaMallocAsync(&scratch, sizeof(*scratch), s);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
        flags = scratch;
    }
    e = launch_pm_divmod(d_v, n, b, c, m, d_q, d_r, flags, s);
    if (scratch) cudaFreeAsync(scratch, s);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "mb200_pm_divmod");
}

int mb200_pm_div(const uint64_t* d_v, uint64_t n, unsigned b, uint64_t c, unsigned m_iters, uint64_t* d_q,
                 uint64_t* d_overflow, void* stream) {
    if (!d_q && n) return fail(MB200_INVALID_ARGUMENT, "null buffer");
    return mb200_pm_divmod(d_v, n, b, c, m_iters, d_q, nullptr, d_overflow, stream);
}

int mb200_pm_mod(const uint64_t* d_v, const uint64_t* d_z, uint64_t n, unsigned b, uint64_t c, uint64_t* d_r,
                 void* stream) {
    if (b < 2 || b > 64) {
        if (b >= 2 && b <= 127) return fail(MB200_UNSUPPORTED, "GPU division supports b <= 64");
        return fail(MB200_INVALID_ARGUMENT, "width must be in [2, 127]");
    }
    if (int rc = mb200_pm_modulus(b, c, 0, 1, nullptr, nullptr)) return rc;  // validates (b, c) only
    if (n == 0) return MB200_OK;
    if (!d_v || !d_z || !d_r) return fail(MB200_INVALID_ARGUMENT, "null buffer");
    cudaError_t e = launch_pm_mod(d_v, d_z, n, b, c, d_r, (cudaStream_t)stream);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "mb200_pm_mod");
}

int mb200_mersenne_divmod(const uint64_t* d_v, uint64_t n, unsigned b, uint64_t* d_q, uint64_t* d_r,
                          void* stream) {
    if (b < 2 || b > 127) return fail(MB200_INVALID_ARGUMENT, "exponent must be in [2, 127]");  // field.cpp:198
    if (b > 63) return fail(MB200_UNSUPPORTED, "GPU Mersenne divmod supports b <= 63");
    if (n == 0) return MB200_OK;
    if (!d_v || !d_q || !d_r) return fail(MB200_INVALID_ARGUMENT, "null buffer");
    cudaStream_t s = (cudaStream_t)stream;
    // v < 2^(2b), else domain_error (field.cpp:209-210); checked before any output
    const uint64_t max_lo = b >= 32 ? ~0ull : (1ull << (2 * b)) - 1;
    const uint64_t max_hi = b >= 32 ? (b == 64 ? ~0ull : (1ull << (2 * b - 64)) - 1) : 0;
    unsigned long long bad = 0;
    int rc = count_on_device(
        [&](unsigned long long* d, cudaStream_t st) { return launch_count_above(d_v, n, max_lo, max_hi, d, st); }, s,
        &bad);
    if (rc) return rc;
    if (bad) return fail(MB200_DOMAIN_ERROR, "input exceeds 2^(2b)");
    // Alg 3 is Alg 4 + 5 at c = 1, m = 2: z = ((v+1) >> b + v + 1) >> b, y = (v + z) & p
    unsigned long long* flags = nullptr;
    cudaError_t e = cudaMallocAsync(&flags, sizeof(*flags), s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
    e = launch_pm_divmod(d_v, n, b, 1, 2, d_q, d_r, flags, s);
    cudaFreeAsync(flags, s);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "mb200_mersenne_divmod");
}

int mb200_split_batch(int splitter, const uint64_t* d_h, uint64_t n, unsigned b, uint64_t l_or_r, uint64_t* d_index,
                      int32_t* d_sign, uint64_t* d_out_of_domain, void* stream) {
    if (b < 2 || b > 127) return fail(MB200_INVALID_ARGUMENT, "exponent must be in [2, 127]");
    if (b > 64) return fail(MB200_UNSUPPORTED, "GPU splitters take hash values of b <= 64 bits");
    SketchParams sp{};
    sp.b = b;
    sp.splitter = (uint32_t)splitter;
    sp.families = sp.rows = 1;
    if (splitter == MB200_SPLIT_POW2) {  // sketch.cpp:14: l < b
        if (l_or_r >= b) return fail(MB200_INVALID_ARGUMENT, "split_pow2 needs l < b");
        sp.lw = (uint32_t)l_or_r;
        sp.width = 1ull << l_or_r;
    } else if (splitter == MB200_SPLIT_UNIFORM_ARB || splitter == MB200_SPLIT_MERSENNE_ARB) {
        if (l_or_r < 1 || l_or_r > (1ull << (b - 1)))  // sketch.cpp:24
            return fail(MB200_INVALID_ARGUMENT, "bucket count must be in [1, 2^(b-1)]");
        sp.width = l_or_r;
    } else {
        return fail(MB200_INVALID_ARGUMENT, "unknown splitter");
    }
    if (n == 0) return MB200_OK;
    if (!d_h || !d_index || !d_sign) return fail(MB200_INVALID_ARGUMENT, "null buffer");
    cudaStream_t s = (cudaStream_t)stream;
    if (d_out_of_domain) {
        cudaError_t e = launch_split_batch(sp, d_h, n, d_index, d_sign,
                                           reinterpret_cast<unsigned long long*>(d_out_of_domain), s);
        return e == cudaSuccess ? MB200_OK : cuda_fail(e, "mb200_split_batch");
    }
    unsigned long long bad = 0;
    int rc = count_on_device(
        [&](unsigned long long* d, cudaStream_t st) { return launch_split_batch(sp, d_h, n, d_index, d_sign, d, st); },
        s, &bad);
    if (rc) return rc;
    if (bad) return fail(MB200_DOMAIN_ERROR, "hash value outside the splitter's domain");
    return MB200_OK;
}

int mb200_bucket_map(int kind, const uint64_t* d_v, uint64_t n, unsigned b, uint64_t c, uint64_t r,
                     uint64_t* d_out, uint64_t* d_out_of_domain, void* stream) {
    if (kind != MB200_MAP_POW2 && kind != MB200_MAP_MERSENNE && kind != MB200_MAP_EXACT_DIV)
        return fail(MB200_INVALID_ARGUMENT, "unknown bucket map");
    unsigned m = 0;
    uint64_t bound = 0;  // values must be < bound (0: all of u64)
    if (kind == MB200_MAP_EXACT_DIV) {
        if (int rc = mb200_exact_division_iterations(b, c, r, &m)) return rc;
        if (b > 64) return fail(MB200_UNSUPPORTED, "GPU bucket maps support b <= 64");
        bound = b == 64 ? (uint64_t)0 - c : (1ull << b) - c;
    } else {
        if (b < 1 + (kind == MB200_MAP_MERSENNE) || b > 127)  // bucketing.cpp:62, :69
            return fail(MB200_INVALID_ARGUMENT, "width must be in [1, 127] (map_pow2) / [2, 127] (map_mersenne)");
        if (b > 64) return fail(MB200_UNSUPPORTED, "GPU bucket maps support b <= 64");
        const uint64_t top = b == 64 ? ~0ull : (1ull << b) - (kind == MB200_MAP_MERSENNE);  // largest r
        if (r == 0 || r > top) return fail(MB200_INVALID_ARGUMENT, "bucket count out of range for the map");
        bound = kind == MB200_MAP_POW2 ? (b == 64 ? 0 : 1ull << b) : (b == 64 ? ~0ull : (1ull << b) - 1);
    }
    if (n == 0) return MB200_OK;
    if (!d_v || !d_out) return fail(MB200_INVALID_ARGUMENT, "null buffer");
    cudaStream_t s = (cudaStream_t)stream;
    if (d_out_of_domain) {
        cudaError_t e = launch_bucket_map(kind, d_v, n, b, c, m, r, bound, d_out,
                                          reinterpret_cast<unsigned long long*>(d_out_of_domain), s);
        return e == cudaSuccess ? MB200_OK : cuda_fail(e, "mb200_bucket_map");
    }
    unsigned long long bad = 0;
    int rc = count_on_device(
        [&](unsigned long long* d, cudaStream_t st) {
            return launch_bucket_map(kind, d_v, n, b, c, m, r, bound, d_out, d, st);
        },
        s, &bad);
    if (rc) return rc;
    if (bad) return fail(MB200_DOMAIN_ERROR, "value outside the map's domain");
    return MB200_OK;
}

int mb200_enum_moment_sums(unsigned b, uint64_t key_domain, uint64_t buckets, int splitter, const uint64_t* keys,
                           const int64_t* deltas, uint64_t n, uint64_t out[5], void* stream) {
    // validate_moment_spec (verify.cpp:480-503)
    if (b < 2 || b > 31) return fail(MB200_INVALID_ARGUMENT, "width must be in [2, 31]");
    if (splitter != MB200_SPLIT_POW2 && splitter != MB200_SPLIT_UNIFORM_ARB && splitter != MB200_SPLIT_MERSENNE_ARB)
        return fail(MB200_INVALID_ARGUMENT, "unknown splitter");
    // validate_splitter_width (verify.cpp:401-409)
    if (buckets < 1) return fail(MB200_INVALID_ARGUMENT, "bucket count must be at least 1");
    if (splitter == MB200_SPLIT_POW2 && (buckets & (buckets - 1)) != 0)
        return fail(MB200_INVALID_ARGUMENT, "bucket count must be a power of two for this splitter");
    if (buckets > (1ull << (b - 1))) return fail(MB200_INVALID_ARGUMENT, "bucket count exceeds half the hash range");
    const uint64_t p = (1ull << b) - 1;
    if (key_domain < 1 || key_domain > p) return fail(MB200_INVALID_ARGUMENT, "modulus too small for key domain");
    if (n == 0) return fail(MB200_INVALID_ARGUMENT, "stream must not be empty");
    if (!keys || !deltas || !out) return fail(MB200_INVALID_ARGUMENT, "null buffer");
    uint64_t weight = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (keys[i] >= key_domain) return fail(MB200_INVALID_ARGUMENT, "key outside domain");
        weight += deltas[i] < 0 ? 0ull - (uint64_t)deltas[i] : (uint64_t)deltas[i];
        if (weight > 1024) return fail(MB200_INVALID_ARGUMENT, "stream weights too large for exact enumeration");
    }
    {
        std::vector<uint64_t> res(n);
        for (uint64_t i = 0; i < n; ++i) res[i] = keys[i] % p;
        std::sort(res.begin(), res.end());
        if (std::adjacent_find(res.begin(), res.end()) != res.end())
            return fail(MB200_INVALID_ARGUMENT, "stream keys must be distinct modulo the modulus");
    }
    // exact_family_count (verify.cpp:566-573)
    if (b > 15) return fail(MB200_INVALID_ARGUMENT, "width must be in [2, 15] to enumerate exactly");
    // entries with delta = 0 never move a counter
    std::vector<uint32_t> xs;
    std::vector<int32_t> ws;
    uint32_t w2 = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (deltas[i] == 0) continue;
        ws.push_back((int32_t)deltas[i]);
        w2 += (uint32_t)(deltas[i] * deltas[i]);
    }
    const uint32_t m = (uint32_t)ws.size();
    if (m > 64) return fail(MB200_UNSUPPORTED, "GPU enumeration supports at most 64 non-zero stream entries");
    xs.resize(3 * (size_t)m);
    for (uint64_t i = 0, j = 0; i < n; ++i) {
        if (deltas[i] == 0) continue;
        const uint64_t x = keys[i] % p, x2 = x * x % p;
        xs[j] = (uint32_t)x;
        xs[m + j] = (uint32_t)x2;
        xs[2 * m + j] = (uint32_t)(x2 * x % p);
        ++j;
    }
    SketchParams sp;
    std::memset(&sp, 0, sizeof(sp));
    sp.rows = sp.families = 1;
    sp.b = b;
    sp.p = p;
    sp.splitter = (uint32_t)splitter;
    sp.width = buckets;
    sp.lw = (unsigned)__builtin_ctzll(buckets);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t xs_bytes = 3 * (size_t)m * 4 + 16, ws_bytes = (size_t)m * 4 + 16, tab_bytes = (size_t)p * 2 + 16;
    unsigned char* ws_dev = nullptr;
    cudaError_t e = cudaMallocAsync(&ws_dev, 32 + xs_bytes + ws_bytes + tab_bytes, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
    unsigned long long* d_out = reinterpret_cast<unsigned long long*>(ws_dev);
    uint32_t* d_xs = reinterpret_cast<uint32_t*>(ws_dev + 32);
    int32_t* d_ws = reinterpret_cast<int32_t*>(ws_dev + 32 + xs_bytes);
    uint16_t* d_tab = reinterpret_cast<uint16_t*>(ws_dev + 32 + xs_bytes + ws_bytes);
    uint64_t host[4] = {0, 0, 0, 0};
    e = cudaMemsetAsync(d_out, 0, 32, s);
    if (e == cudaSuccess && m) e = cudaMemcpyAsync(d_xs, xs.data(), 3 * (size_t)m * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && m) e = cudaMemcpyAsync(d_ws, ws.data(), (size_t)m * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = launch_enum_moments(sp, m, w2, d_xs, d_ws, d_tab, d_out, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(host, d_out, 32, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(ws_dev, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "mb200_enum_moment_sums");
    for (int i = 0; i < 4; ++i) out[i] = host[i];
    out[4] = p * p * p * p;
    return MB200_OK;
}

int mb200_cs_update(const mb200_sketch_desc* desc, const void* d_keys, int key_width, const void* d_weights,
                    int weight_kind, uint64_t n, int64_t* d_counters, void* stream) {
    SketchParams sp;
    if (int rc = build_sketch_params(desc, sp)) return rc;
    if (key_width != 32 && key_width != 64) return fail(MB200_INVALID_ARGUMENT, "key width must be 32 or 64");
    if (weight_kind != MB200_W_NONE && weight_kind != MB200_W_I32 && weight_kind != MB200_W_I64)
        return fail(MB200_INVALID_ARGUMENT, "unknown weight kind");
    if (n == 0) return MB200_OK;  // an empty batch touches nothing (empty tensors may be null)
    if (weight_kind != MB200_W_NONE && !d_weights) return fail(MB200_INVALID_ARGUMENT, "null weights");
    if (!d_keys || !d_counters) return fail(MB200_INVALID_ARGUMENT, "null buffer");
    cudaStream_t s = (cudaStream_t)stream;
    if (int rc = check_keys(d_keys, key_width, n, desc->key_bits, s)) return rc;
    cudaError_t e = launch_cs_update(sp, d_keys, key_width, d_weights, weight_kind, n, d_counters, s);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "mb200_cs_update");
}

int mb200_cs_moments(const int64_t* d_counters, unsigned rows, uint64_t width, uint64_t* d_out, void* stream) {
    if (!d_counters || !d_out) return fail(MB200_INVALID_ARGUMENT, "null buffer");
    cudaError_t e = launch_cs_moments(d_counters, rows, width, d_out, (cudaStream_t)stream);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "mb200_cs_moments");
}

int mb200_cs_merge(int64_t* d_dst, const int64_t* d_src, uint64_t count, void* stream) {
    if (count && (!d_dst || !d_src)) return fail(MB200_INVALID_ARGUMENT, "null buffer");
    cudaError_t e = launch_cs_merge(d_dst, d_src, count, (cudaStream_t)stream);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "mb200_cs_merge");
}

int mb200_cs_point_query(const mb200_sketch_desc* desc, const int64_t* d_counters, const void* d_keys, int key_width,
                         uint64_t n, int64_t* d_out, void* stream) {
    SketchParams sp;
    if (int rc = build_sketch_params(desc, sp)) return rc;
    if (key_width != 32 && key_width != 64) return fail(MB200_INVALID_ARGUMENT, "key width must be 32 or 64");
    if (n == 0) return MB200_OK;
    if (!d_keys || !d_counters || !d_out) return fail(MB200_INVALID_ARGUMENT, "null buffer");
    cudaStream_t s = (cudaStream_t)stream;
    if (int rc = check_keys(d_keys, key_width, n, desc->key_bits, s)) return rc;
    cudaError_t e = launch_cs_point_query(sp, d_counters, d_keys, key_width, n, d_out, s);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "mb200_cs_point_query");
}

int mb200_kernel_timer(int enable) {
    kernel_timer(enable != 0);
    return MB200_OK;
}

int mb200_kernel_timer_read(double* total_ms, uint64_t* launches) {
    cudaError_t e = kernel_timer_read(total_ms, launches);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "mb200_kernel_timer_read");
}

int mb200_hot_stats(uint64_t out[8], int reset) {
    cudaError_t e = hot_stats(out, reset != 0);
    return e == cudaSuccess ? MB200_OK : cuda_fail(e, "mb200_hot_stats");
}

int mb200_set_large_table_strategy(int strategy, int* previous) {
    const int old = set_large_table_strategy(strategy);
    if (old < 0) return fail(MB200_INVALID_ARGUMENT, "unknown large-table strategy");
    if (previous) *previous = old;
    return MB200_OK;
}

}  // extern "C"
