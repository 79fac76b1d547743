// handles.cpp -- object entries of the C-ABI (mb200_sketch_*): the C++
// CountSketch (mersenne_b200.hpp) behind an opaque handle, with exceptions
// mapped back to status codes + the reference's messages.
#include <cuda_runtime.h>

#include <cstring>
#include <stdexcept>

#include "../../include/mersenne_b200.h"
#include "../../include/mersenne_b200/mersenne_b200.hpp"
#include "../csrc/mb200_capi_util.h"

using mersenne::b200::CountSketch;
using mersenne::b200::MersenneModulus;
using mersenne::b200::PolyHashFamily;
using mersenne::b200::Splitter;
using mersenne::b200::u128;

struct mb200_sketch {
    CountSketch sk;
};

namespace {

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return MB200_OK;
    } catch (const std::invalid_argument& e) {
        return mb200::fail(MB200_INVALID_ARGUMENT, e.what());
    } catch (const std::domain_error& e) {
        return mb200::fail(MB200_DOMAIN_ERROR, e.what());
    } catch (const std::logic_error& e) {
        return mb200::fail(MB200_LOGIC_ERROR, e.what());
    } catch (const std::exception& e) {
        return mb200::fail(MB200_CUDA_ERROR, e.what());
    }
}

u128 domain_of(unsigned key_bits) { return u128(1) << key_bits; }

}  // namespace

extern "C" {

int mb200_sketch_create(unsigned rows, uint64_t width, unsigned b, unsigned key_bits, int splitter, uint64_t seed,
                        unsigned independence, mb200_sketch** out) {
    if (!out) return mb200::fail(MB200_INVALID_ARGUMENT, "null output handle");
    *out = nullptr;
    if (key_bits > 126) return mb200::fail(MB200_INVALID_ARGUMENT, "key domain too wide");
    return guarded([&] {
        *out = new mb200_sketch{CountSketch(rows, width, MersenneModulus(b, true), domain_of(key_bits),
                                            Splitter(splitter), seed, independence)};
    });
}

int mb200_sketch_create_families(uint64_t width, int splitter, unsigned b, unsigned key_bits, unsigned families,
                                 unsigned k, const uint64_t* coeffs_lo, const uint64_t* coeffs_hi, unsigned rows,
                                 mb200_sketch** out) {
    if (!out || !coeffs_lo) return mb200::fail(MB200_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    return guarded([&] {
        MersenneModulus mod(b, true);
        std::vector<PolyHashFamily> fams;
        for (unsigned f = 0; f < families; ++f) {
            std::vector<u128> c(k);
            for (unsigned i = 0; i < k; ++i)
                c[i] = (u128(coeffs_hi ? coeffs_hi[f * k + i] : 0) << 64) | coeffs_lo[f * k + i];
            fams.emplace_back(mod, std::move(c), domain_of(key_bits));
        }
        *out = new mb200_sketch{CountSketch(width, Splitter(splitter), std::move(fams), rows)};
    });
}

void mb200_sketch_destroy(mb200_sketch* s) { delete s; }

int mb200_sketch_process(mb200_sketch* s, const void* h_keys, int key_width, const void* h_weights, int weight_kind,
                         uint64_t n) {
    if (!s) return mb200::fail(MB200_INVALID_ARGUMENT, "null sketch");
    return guarded([&] { s->sk.process_batch(h_keys, key_width, h_weights, weight_kind, n); });
}

void mb200_set_host_threads(int n) { mersenne::b200::set_host_threads(n); }
int mb200_host_threads(void) { return mersenne::b200::get_host_threads(); }

int mb200_sketch_h2d_bytes(const mb200_sketch* s, uint64_t* out) {
    if (!s || !out) return mb200::fail(MB200_INVALID_ARGUMENT, "null argument");
    *out = s->sk.h2d_bytes();
    return MB200_OK;
}

int mb200_sketch_process_device(mb200_sketch* s, const void* d_keys, int key_width, const void* d_weights,
                                int weight_kind, uint64_t n, void* stream) {
    if (!s) return mb200::fail(MB200_INVALID_ARGUMENT, "null sketch");
    return guarded([&] { s->sk.process_device(d_keys, key_width, d_weights, weight_kind, n, stream); });
}

int mb200_sketch_row_second_moment(mb200_sketch* s, unsigned row, uint64_t* lo, uint64_t* hi, int* saturated) {
    if (!s) return mb200::fail(MB200_INVALID_ARGUMENT, "null sketch");
    return guarded([&] {
        auto m = s->sk.row_second_moment(row);
        *lo = uint64_t(m.value);
        *hi = uint64_t(m.value >> 64);
        *saturated = m.saturated;
    });
}

int mb200_sketch_second_moment(mb200_sketch* s, int median_rows, uint64_t* lo, uint64_t* hi, int* saturated) {
    if (!s) return mb200::fail(MB200_INVALID_ARGUMENT, "null sketch");
    return guarded([&] {
        auto m = s->sk.second_moment(median_rows != 0);
        *lo = uint64_t(m.value);
        *hi = uint64_t(m.value >> 64);
        *saturated = m.saturated;
    });
}

int mb200_sketch_point_query(mb200_sketch* s, const void* h_keys, int key_width, uint64_t n, int64_t* h_out) {
    if (!s) return mb200::fail(MB200_INVALID_ARGUMENT, "null sketch");
    return guarded([&] {
        auto v = s->sk.point_query_batch(h_keys, key_width, n);
        std::memcpy(h_out, v.data(), v.size() * sizeof(int64_t));
    });
}

int mb200_sketch_merge(mb200_sketch* dst, const mb200_sketch* src) {
    if (!dst || !src) return mb200::fail(MB200_INVALID_ARGUMENT, "null sketch");
    return guarded([&] { dst->sk.merge(src->sk); });
}

int mb200_sketch_allreduce(mb200_sketch* s, void* nccl_comm) {
    if (!s) return mb200::fail(MB200_INVALID_ARGUMENT, "null sketch");
    return guarded([&] { s->sk.allreduce(nccl_comm); });
}

int mb200_sketch_counters(mb200_sketch* s, int64_t* h_out) {
    if (!s) return mb200::fail(MB200_INVALID_ARGUMENT, "null sketch");
    return guarded([&] {
        auto v = s->sk.counters();
        std::memcpy(h_out, v.data(), v.size() * sizeof(int64_t));
    });
}

int mb200_sketch_set_counters(mb200_sketch* s, const int64_t* h_in) {
    if (!s) return mb200::fail(MB200_INVALID_ARGUMENT, "null sketch");
    return guarded([&] {
        std::vector<int64_t> v(h_in, h_in + size_t(s->sk.rows()) * s->sk.width());
        s->sk.set_counters(v);
    });
}

int64_t* mb200_sketch_device_counters(mb200_sketch* s) { return s ? s->sk.device_counters() : nullptr; }

int mb200_sketch_info(const mb200_sketch* s, unsigned* rows, uint64_t* width, unsigned* b, unsigned* k,
                      unsigned* key_bits, int* splitter) {
    if (!s) return mb200::fail(MB200_INVALID_ARGUMENT, "null sketch");
    if (rows) *rows = s->sk.rows();
    if (width) *width = s->sk.width();
    if (b) *b = s->sk.modulus().b();
    if (k) *k = s->sk.independence();
    if (key_bits) *key_bits = s->sk.families().front().key_bits();
    if (splitter) *splitter = int(s->sk.splitter());
    return MB200_OK;
}

int mb200_sketch_seeds(const mb200_sketch* s, uint64_t* out) {
    if (!s) return mb200::fail(MB200_INVALID_ARGUMENT, "null sketch");
    if (s->sk.seeds().empty()) return mb200::fail(MB200_LOGIC_ERROR, "sketch with injected families has no seeds");
    std::memcpy(out, s->sk.seeds().data(), s->sk.seeds().size() * sizeof(uint64_t));
    return MB200_OK;
}

int mb200_sketch_serialize(mb200_sketch* s, uint8_t* out, uint64_t cap, uint64_t* len) {
    if (!s || !len) return mb200::fail(MB200_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        const std::vector<uint8_t> bytes = s->sk.serialize();
        *len = bytes.size();
        if (out && cap >= bytes.size()) std::memcpy(out, bytes.data(), bytes.size());
    });
}

int mb200_sketch_deserialize(const uint8_t* bytes, uint64_t len, mb200_sketch** out) {
    if (!out || (!bytes && len)) return mb200::fail(MB200_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    return guarded([&] {
        std::vector<uint8_t> v(bytes, bytes + len);
        *out = new mb200_sketch{CountSketch::deserialize(v)};
    });
}

int mb200_sketch_coeffs(const mb200_sketch* s, uint64_t* lo, uint64_t* hi) {
    if (!s) return mb200::fail(MB200_INVALID_ARGUMENT, "null sketch");
    size_t i = 0;
    for (const auto& f : s->sk.families())
        for (u128 a : f.coefficients()) {
            if (lo) lo[i] = uint64_t(a);
            if (hi) hi[i] = uint64_t(a >> 64);
            ++i;
        }
    return MB200_OK;
}

}  // extern "C"
