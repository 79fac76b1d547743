// mersenne_b200.cpp -- the reference's C++ API (field / polyhash / sketch)
// re-hosted on the GPU path.  Every per-key computation goes through the
// C-ABI kernels; this file only validates, owns device memory and streams,
// pipelines host<->device copies and applies the host-side median.
#include "../../include/mersenne_b200/mersenne_b200.hpp"

#include <cuda_runtime.h>

#include <sched.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>

#include "../csrc/mb200_capi_util.h"

namespace mersenne::b200 {

void throw_status(int status) {
    if (status == MB200_OK) return;
    const std::string msg = mb200_last_error();
    switch (status) {
        case MB200_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case MB200_DOMAIN_ERROR: throw std::domain_error(msg);
        case MB200_LOGIC_ERROR: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}

namespace {

void cuda_check(cudaError_t e, const char* where) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(where) + ": " + cudaGetErrorString(e));
}

unsigned log2_pow2(u128 v) {
    const u64 hi = u64(v >> 64);
    if (hi) return 64 + unsigned(__builtin_ctzll(hi));
    return unsigned(__builtin_ctzll(u64(v)));
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    explicit DevBuf(size_t n) { cuda_check(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc"); }
    ~DevBuf() { cudaFree(p); }
};

}  // namespace

// ------------------------------------------------------------------ field --
MersenneModulus::MersenneModulus(unsigned b, bool require_prime) : b_(b) {
    throw_status(mb200_mersenne_modulus_check(b, 0));
    prime_ = mb200_mersenne_modulus_check(b, 1) == MB200_OK;
    if (require_prime && !prime_) throw std::invalid_argument("2^b - 1 is not prime for this exponent");
}

PseudoMersenneModulus::PseudoMersenneModulus(unsigned b, u128 c, unsigned m_iters, Engine engine)
    : b_(b), c_(c), engine_(engine) {
    unsigned m = 0;
    std::array<u64, 4> mx{};
    throw_status(mb200_pm_modulus(b, u64(c), u64(c >> 64), m_iters, &m, mx.data()));  // field.cpp:225-228, 242-243
    switch (engine) {  // field.cpp:229-241
        case Engine::Auto: engine_ = b <= 61 ? Engine::Native : Engine::Generic; break;
        case Engine::Native:
            if (b > 61) throw std::invalid_argument("native engine requires b <= 61");
            break;
        case Engine::Generic: break;
    }
    m_ = m;
    max_input_.limb = mx;
}

namespace {
// the GPU division path covers b <= 64 (then c < 2^63)
void require_gpu_division(const PseudoMersenneModulus& mod) {
    if (mod.b() > 64) throw_status(mb200_pm_div(nullptr, 0, mod.b(), 0, 0, nullptr, nullptr, nullptr));
}
}  // namespace

void PseudoMersenneModulus::divmod_device(const u64* d_v, u64 n, u64* d_q, u64* d_r, void* stream) const {
    require_gpu_division(*this);
    DevBuf<u64> ovf(1);
    cuda_check(cudaMemsetAsync(ovf.p, 0, sizeof(u64), (cudaStream_t)stream), "memset");
    throw_status(mb200_pm_divmod(d_v, n, b_, u64(c_), m_, d_q, d_r, ovf.p, stream));
    u64 o = 0;
    cuda_check(cudaMemcpyAsync(&o, ovf.p, sizeof(u64), cudaMemcpyDeviceToHost, (cudaStream_t)stream), "copy");
    cuda_check(cudaStreamSynchronize((cudaStream_t)stream), "sync");
    if (o) throw std::domain_error("quotient exceeds 64 bits");
}

void mersenne_divmod_device(const u64* d_v, u64 n, const MersenneModulus& mod, u64* d_q, u64* d_r, void* stream) {
    throw_status(mb200_mersenne_divmod(d_v, n, mod.b(), d_q, d_r, stream));
}

void pseudo_mersenne_div_device(const u64* d_v, u64 n, const PseudoMersenneModulus& mod, u64* d_q, void* stream) {
    mod.divmod_device(d_v, n, d_q, nullptr, stream);
}

void pseudo_mersenne_mod_device(const u64* d_v, const u64* d_z, u64 n, const PseudoMersenneModulus& mod, u64* d_r,
                                void* stream) {
    require_gpu_division(mod);
    throw_status(mb200_pm_mod(d_v, d_z, n, mod.b(), u64(mod.c()), d_r, stream));
}

namespace {
bool wide_greater(const UWide& a, const UWide& b) {
    for (int i = 3; i >= 0; --i)
        if (a.limb[i] != b.limb[i]) return a.limb[i] > b.limb[i];
    return false;
}
// one u128 value to the device as a (lo, hi) pair, `outs` u64 results back
template <typename F>
std::vector<u64> one_value(const UWide& v, int outs, F&& launch) {
    DevBuf<u64> d(2 + 2 * size_t(outs));
    const u64 in[2] = {v.limb[0], v.limb[1]};
    cuda_check(cudaMemcpy(d.p, in, sizeof in, cudaMemcpyHostToDevice), "H2D");
    launch(d.p, d.p + 2);
    std::vector<u64> out(static_cast<size_t>(outs));
    cuda_check(cudaMemcpy(out.data(), d.p + 2, out.size() * sizeof(u64), cudaMemcpyDeviceToHost), "D2H");
    return out;
}
}  // namespace

DivMod mersenne_divmod(const UWide& v, const MersenneModulus& mod) {  // field.cpp:208-222
    const unsigned b = mod.b();
    const bool fits = v.fits_u128() && (2 * b >= 128 || (v.low_u128() >> (2 * b)) == 0);
    if (!fits) throw std::domain_error("input exceeds 2^(2b)");
    const auto qr = one_value(v, 2, [&](const u64* dv, u64* out) { mersenne_divmod_device(dv, 1, mod, out, out + 1); });
    return {UWide(qr[0]), UWide(qr[1])};
}

UWide pseudo_mersenne_div(const UWide& v, const PseudoMersenneModulus& mod) {  // field.cpp:260-265
    if (wide_greater(v, mod.max_input())) throw std::domain_error("input exceeds division domain for m iterations");
    require_gpu_division(mod);
    if (!v.fits_u128()) throw std::runtime_error("GPU division takes dividends below 2^128");
    const auto q = one_value(v, 1, [&](const u64* dv, u64* out) { pseudo_mersenne_div_device(dv, 1, mod, out); });
    return UWide(q[0]);
}

UWide pseudo_mersenne_mod(const UWide& v, const UWide& z, const PseudoMersenneModulus& mod) {  // field.cpp:267-273
    require_gpu_division(mod);
    // (v + z c) mod 2^b with b <= 64 depends on the low words only
    DevBuf<u64> d(4);
    const u64 in[3] = {v.limb[0], v.limb[1], z.limb[0]};
    cuda_check(cudaMemcpy(d.p, in, sizeof in, cudaMemcpyHostToDevice), "H2D");
    pseudo_mersenne_mod_device(d.p, d.p + 2, 1, mod, d.p + 3);
    u64 r = 0;
    cuda_check(cudaMemcpy(&r, d.p + 3, sizeof r, cudaMemcpyDeviceToHost), "D2H");
    return UWide(r);
}

void PseudoMersenneModulus::divmod(const u64* h_v, u64 n, u64* h_q, u64* h_r) const {
    if (n == 0) return;
    DevBuf<u64> v(2 * n), q(n), r(n);
    cuda_check(cudaMemcpy(v.p, h_v, 2 * n * sizeof(u64), cudaMemcpyHostToDevice), "H2D");
    divmod_device(v.p, n, q.p, r.p, nullptr);
    cuda_check(cudaMemcpy(h_q, q.p, n * sizeof(u64), cudaMemcpyDeviceToHost), "D2H");
    cuda_check(cudaMemcpy(h_r, r.p, n * sizeof(u64), cudaMemcpyDeviceToHost), "D2H");
}

// -------------------------------------------------------------- bucketing --
void map_pow2_device(const u64* d_v, u64 n, unsigned b, u64 r, u64* d_out, void* stream) {
    throw_status(mb200_bucket_map(MB200_MAP_POW2, d_v, n, b, 0, r, d_out, nullptr, stream));
}

void map_mersenne_device(const u64* d_v, u64 n, unsigned b, u64 r, u64* d_out, void* stream) {
    throw_status(mb200_bucket_map(MB200_MAP_MERSENNE, d_v, n, b, 0, r, d_out, nullptr, stream));
}

namespace {
PseudoMersenneModulus exact_divider(const PseudoMersenneModulus& mod, u64 r) {
    unsigned m = 0;
    if (mod.b() > 64) throw_status(mb200_bucket_map(MB200_MAP_EXACT_DIV, nullptr, 0, mod.b(), 0, r, nullptr, nullptr, nullptr));
    throw_status(mb200_exact_division_iterations(mod.b(), u64(mod.c()), r, &m));
    return PseudoMersenneModulus(mod.b(), mod.c(), m);
}
}  // namespace

ExactDivisionMap::ExactDivisionMap(const PseudoMersenneModulus& mod, u64 r)
    : divider_(exact_divider(mod, r)), r_(r) {}

void ExactDivisionMap::map_device(const u64* d_v, u64 n, u64* d_out, void* stream) const {
    throw_status(mb200_bucket_map(MB200_MAP_EXACT_DIV, d_v, n, divider_.b(), u64(divider_.c()), r_, d_out, nullptr,
                                  stream));
}

u64 ExactDivisionMap::operator()(u64 v) const {
    DevBuf<u64> d(2);
    cuda_check(cudaMemcpy(d.p, &v, sizeof(u64), cudaMemcpyHostToDevice), "H2D");
    map_device(d.p, 1, d.p + 1, nullptr);
    u64 out = 0;
    cuda_check(cudaMemcpy(&out, d.p + 1, sizeof(u64), cudaMemcpyDeviceToHost), "D2H");
    return out;
}

// --------------------------------------------------------------- polyhash --
PolyHashFamily::PolyHashFamily(const MersenneModulus& modulus, unsigned k, u128 key_domain, u64 seed,
                               HashFinish finish)
    : modulus_(modulus), key_domain_(key_domain), finish_(finish) {
    if (k == 0) throw std::invalid_argument("independence degree must be at least 1");
    std::vector<u64> lo(k), hi(k);
    throw_status(mb200_draw_coeffs(modulus.b(), k, seed, lo.data(), hi.data()));
    coeffs_.resize(k);
    for (unsigned i = 0; i < k; ++i) coeffs_[i] = (u128(hi[i]) << 64) | lo[i];
    validate();
}

PolyHashFamily::PolyHashFamily(const MersenneModulus& modulus, std::vector<u128> coefficients, u128 key_domain,
                               HashFinish finish)
    : modulus_(modulus), coeffs_(std::move(coefficients)), key_domain_(key_domain), finish_(finish) {
    if (coeffs_.empty()) throw std::invalid_argument("independence degree must be at least 1");
    for (u128 a : coeffs_)
        if (a >= modulus_.p()) throw std::invalid_argument("coefficient not reduced");  // polyhash.cpp:43
    validate();
}

void PolyHashFamily::validate() const {  // polyhash.cpp:48-57
    if (key_domain_ == 0 || (key_domain_ & (key_domain_ - 1)) != 0)
        throw std::invalid_argument("key domain must be a power of two");
    if (modulus_.p() < 2 * key_domain_ - 1) throw std::invalid_argument("modulus too small for key domain");
}

unsigned PolyHashFamily::key_bits() const { return log2_pow2(key_domain_); }

void PolyHashFamily::hash_device(const void* d_keys, int key_width, u64 n, u64* d_out_lo, u64* d_out_hi,
                                 void* stream) const {
    const unsigned b = modulus_.b();
    const unsigned k = independence();
    std::vector<u64> lo(k), hi(k);
    for (unsigned i = 0; i < k; ++i) {
        lo[i] = u64(coeffs_[i]);
        hi[i] = u64(coeffs_[i] >> 64);
    }
    const unsigned kb = std::min(key_bits(), 64u);
    if (b <= 61) {
        throw_status(mb200_hash61(d_keys, key_width, n, b, lo.data(), k, kb, d_out_lo, stream));
    } else if (b == 89) {
        if (key_width != 64) throw std::invalid_argument("the 89-bit path takes u64 keys");
        if (!d_out_hi) throw std::invalid_argument("b > 64 needs a high-word output");
        throw_status(mb200_hash89((const u64*)d_keys, n, lo.data(), hi.data(), k, kb, d_out_lo, d_out_hi, stream));
    } else {  // 62 <= b <= 127: the generic four-limb path
        if (key_width != 64) throw std::invalid_argument("the b > 61 paths take u64 keys");
        if (!d_out_hi) throw std::invalid_argument("b > 64 needs a high-word output");
        throw_status(
            mb200_hash_wide((const u64*)d_keys, n, b, lo.data(), hi.data(), k, kb, d_out_lo, d_out_hi, stream));
    }
}

std::vector<u128> PolyHashFamily::hash(const std::vector<u64>& keys) const {
    const u64 n = keys.size();
    std::vector<u128> out(n);
    if (n == 0) return out;
    for (u64 x : keys)
        if (key_bits() < 64 && x >= (u64(1) << key_bits())) throw std::domain_error("key outside domain");
    DevBuf<u64> dk(n), dlo(n), dhi(n);
    cuda_check(cudaMemcpy(dk.p, keys.data(), n * sizeof(u64), cudaMemcpyHostToDevice), "H2D");
    hash_device(dk.p, 64, n, dlo.p, dhi.p, nullptr);
    std::vector<u64> lo(n), hi(n, 0);
    cuda_check(cudaMemcpy(lo.data(), dlo.p, n * sizeof(u64), cudaMemcpyDeviceToHost), "D2H");
    if (modulus_.b() > 64) cuda_check(cudaMemcpy(hi.data(), dhi.p, n * sizeof(u64), cudaMemcpyDeviceToHost), "D2H");
    for (u64 i = 0; i < n; ++i) out[i] = (u128(hi[i]) << 64) | lo[i];
    return out;
}

u128 PolyHashFamily::operator()(u128 x) const {
    if (x >= key_domain_) throw std::domain_error("key outside domain");  // polyhash.cpp:60
    return hash(std::vector<u64>{u64(x)})[0];
}

SignIndexPair split_pow2(u128 h, unsigned b, unsigned l) {
    const u128 i = h & ((u128(1) << l) - 1);
    const int a = int(h >> (b - 1));
    return {i, 1 - 2 * a};
}

namespace {
// floor(j r / 2^s) for j, r < 2^127 (map_pow2, bucketing.cpp:61-66): the 254-bit
// product from four 64 x 64 partial products
u128 mul_shift(u128 j, u128 r, unsigned s) {
    const u64 j0 = u64(j), j1 = u64(j >> 64), r0 = u64(r), r1 = u64(r >> 64);
    const u128 p00 = u128(j0) * r0, p01 = u128(j0) * r1, p10 = u128(j1) * r0, p11 = u128(j1) * r1;
    const u128 mid = (p00 >> 64) + u64(p01) + u64(p10);
    const u128 lo = (mid << 64) | u64(p00);
    const u128 hi = p11 + (p01 >> 64) + (p10 >> 64) + (mid >> 64);
    if (s == 0) return lo;
    if (s >= 128) return hi >> (s - 128);
    return (hi << (128 - s)) | (lo >> s);
}
}  // namespace

SignIndexPair split_arb_uniform(u128 h, unsigned b, u128 r) {
    const unsigned s = b - 1;
    const u128 j = h & ((u128(1) << s) - 1);  // low b-1 bits
    const int a = int(h >> s);                // top bit: set -> +1
    return {mul_shift(j, r, s), 2 * a - 1};
}

SignIndexPair split_arb_mersenne(u128 h, unsigned b, u128 r) { return split_arb_uniform(h + 1, b, r); }

void split_device(Splitter splitter, const u64* d_h, u64 n, unsigned b, u64 l_or_r, u64* d_index, int32_t* d_sign,
                  void* stream) {
    throw_status(mb200_split_batch(int(splitter), d_h, n, b, l_or_r, d_index, d_sign, nullptr, stream));
}

// ----------------------------------------------------------------- sketch --
struct CountSketch::Staging {
    cudaStream_t copy = nullptr;
    cudaEvent_t ready[2] = {nullptr, nullptr};
    cudaEvent_t freed[2] = {nullptr, nullptr};
    cudaEvent_t shipped[2] = {nullptr, nullptr};  // narrowed deltas of the slot have left host memory
    void* d_keys[2] = {nullptr, nullptr};
    void* d_w[2] = {nullptr, nullptr};
    void* d_wn[2] = {nullptr, nullptr};  // narrowed deltas as they arrive
    void* h_wn[2] = {nullptr, nullptr};  // pinned host staging of the narrowed deltas
    void* h_kn[2] = {nullptr, nullptr};  // pinned host staging of u64 keys narrowed to u32
    u64 chunk = 0;
    int narrow_bits = 8;  // width tried first for the next chunk
    u64 h2d_bytes = 0;    // bytes process_batch moved host -> device
    ~Staging() {
        for (int i = 0; i < 2; ++i) {
            cudaFree(d_keys[i]);
            cudaFree(d_w[i]);
            cudaFree(d_wn[i]);
            cudaFreeHost(h_wn[i]);
            cudaFreeHost(h_kn[i]);
            if (ready[i]) cudaEventDestroy(ready[i]);
            if (freed[i]) cudaEventDestroy(freed[i]);
            if (shipped[i]) cudaEventDestroy(shipped[i]);
        }
        if (copy) cudaStreamDestroy(copy);
    }
};

namespace {
// Host threads for the transport packing and the domain check: set by
// mb200_set_host_threads, else the CPUs in this process's affinity mask shared
// among the ranks a launcher started on this node (LOCAL_WORLD_SIZE, which
// torchrun sets), one left free from 8 on, at most 8.  OMP_NUM_THREADS is not consulted:
// torchrun forces it to 1.  Packing loops are scheduled dynamically in 2^15-item
// blocks so a descheduled thread does not stall the chunk.
std::atomic<int> g_host_threads{0};
constexpr int kMaxAutoThreads = 8;
int auto_host_threads() {
    static const int t = [] {
        int n = 0;
        cpu_set_t set;
        if (sched_getaffinity(0, sizeof set, &set) == 0) n = CPU_COUNT(&set);
        if (n <= 0) n = int(std::thread::hardware_concurrency());
        int local = 1;
        if (const char* e = std::getenv("LOCAL_WORLD_SIZE")) local = std::max(1, std::atoi(e));
        n /= local;
        // one core left to the caller's other threads; 8 already outrun PCIe
        return std::max(1, std::min(n >= 8 ? n - 1 : n, kMaxAutoThreads));
    }();
    return t;
}
int host_threads() {
    const int t = g_host_threads.load(std::memory_order_relaxed);
    return t > 0 ? t : auto_host_threads();
}
// Narrowing pays only when packing a chunk outruns the PCIe time it saves
// (about 6 cores against ~55 GB/s at i32 -> i8); fewer threads ship as given.
constexpr int kNarrowMinThreads = 6;

// Copies src[0, m) into dst as Dst while checking that every value fits Dst;
// false if one does not (dst is then garbage).  Parallel over the host cores.
template <typename Dst, typename Src>
bool pack_narrow(const Src* src, Dst* dst, u64 m) {
    constexpr Src lo = std::numeric_limits<Dst>::min(), hi = std::numeric_limits<Dst>::max();
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 1 << 15) reduction(| : bad) num_threads(host_threads()) if (m >= (u64(1) << 16))
    for (long long i = 0; i < (long long)m; ++i) {
        const Src v = src[i];
        bad |= (v < lo) | (v > hi);
        dst[i] = Dst(v);
    }
    return !bad;
}

// Narrowest of {i8, i16} holding every delta of the chunk, starting at `first`
// (the width the previous chunk needed); 0 = ship the deltas as they are.
template <typename Src>
int narrow_chunk(const Src* src, void* dst, u64 m, int first) {
    if (first <= 8 && pack_narrow<int8_t>(src, (int8_t*)dst, m)) return 8;
    if (first <= 16 && pack_narrow<int16_t>(src, (int16_t*)dst, m)) return 16;
    return 0;
}
}  // namespace

CountSketch::CountSketch(unsigned rows, u64 width, const MersenneModulus& modulus, u128 key_domain,
                         Splitter splitter, u64 seed, unsigned independence)
    : rows_(rows), width_(width), splitter_(splitter) {
    if (rows == 0) throw std::invalid_argument("need at least one row");  // sketch.cpp:71
    const unsigned fams = splitter == Splitter::TwoForOne ? (rows + 1) / 2 : rows;
    seeds_.resize(fams);
    throw_status(mb200_row_seeds(seed, fams, seeds_.data()));  // sketch.cpp:72-77
    for (unsigned f = 0; f < fams; ++f) families_.emplace_back(modulus, independence, key_domain, seeds_[f]);
    validate();
    init_device();
}

CountSketch::CountSketch(u64 width, Splitter splitter, std::vector<PolyHashFamily> families, unsigned rows)
    : width_(width), splitter_(splitter), families_(std::move(families)) {
    if (families_.empty()) throw std::invalid_argument("need at least one row");
    for (const PolyHashFamily& f : families_) {
        if (f.modulus().b() != families_.front().modulus().b() || f.key_domain() != families_.front().key_domain())
            throw std::invalid_argument("rows must share modulus and key domain");
        if (f.independence() != families_.front().independence())
            throw std::invalid_argument("GPU path needs equal independence across rows");
    }
    rows_ = rows ? rows : (splitter == Splitter::TwoForOne ? 2 * unsigned(families_.size()) : unsigned(families_.size()));
    validate();
    init_device();
}

CountSketch::CountSketch(CountSketch&& o) noexcept
    : rows_(o.rows_), width_(o.width_), splitter_(o.splitter_), families_(std::move(o.families_)),
      seeds_(std::move(o.seeds_)), clo_(std::move(o.clo_)), chi_(std::move(o.chi_)), d_counters_(o.d_counters_),
      stream_(o.stream_), staging_(std::move(o.staging_)) {
    o.d_counters_ = nullptr;
    o.stream_ = nullptr;
}

CountSketch::CountSketch(const CountSketch& o)
    : rows_(o.rows_), width_(o.width_), splitter_(o.splitter_), families_(o.families_), seeds_(o.seeds_) {
    init_device();
    o.synchronize();
    cuda_check(cudaMemcpyAsync(d_counters_, o.d_counters_, size_t(rows_) * width_ * sizeof(i64),
                               cudaMemcpyDeviceToDevice, (cudaStream_t)stream_),
               "D2D");
    synchronize();
}

CountSketch& CountSketch::operator=(const CountSketch& o) {
    if (this != &o) {
        CountSketch tmp(o);
        std::swap(rows_, tmp.rows_);
        std::swap(width_, tmp.width_);
        std::swap(splitter_, tmp.splitter_);
        std::swap(families_, tmp.families_);
        std::swap(seeds_, tmp.seeds_);
        std::swap(d_counters_, tmp.d_counters_);
        std::swap(stream_, tmp.stream_);
        std::swap(staging_, tmp.staging_);
    }
    return *this;
}

i64 CountSketch::counter(unsigned row, u64 index) const {
    if (row >= rows_ || index >= width_) throw std::out_of_range("counter index out of range");
    i64 v = 0;
    cudaStream_t s = (cudaStream_t)stream_;
    cuda_check(cudaMemcpyAsync(&v, d_counters_ + size_t(row) * width_ + index, sizeof v, cudaMemcpyDeviceToHost, s),
               "D2H");
    cuda_check(cudaStreamSynchronize(s), "sync");
    return v;
}

bool operator==(const CountSketch& a, const CountSketch& b) {  // sketch.hpp:78-82
    return a.width_ == b.width_ && a.splitter_ == b.splitter_ && a.seeds_ == b.seeds_ && a.rows_ == b.rows_ &&
           a.modulus().b() == b.modulus().b() && a.key_domain() == b.key_domain() &&
           a.independence() == b.independence() && a.counters() == b.counters();
}

CountSketch::~CountSketch() {
    staging_.reset();
    if (d_counters_) cudaFree(d_counters_);
    if (stream_) cudaStreamDestroy((cudaStream_t)stream_);
}

void CountSketch::validate() const {
    mb200_sketch_desc d = desc();
    // reuse the C-ABI validation (sketch.cpp:97-119 + GPU coverage) with a dry run
    int64_t dummy = 0;
    throw_status(mb200_cs_update(&d, &dummy, 64, nullptr, MB200_W_NONE, 0, &dummy, nullptr));
}

mb200_sketch_desc CountSketch::desc() const {
    clo_.clear();
    chi_.clear();
    for (const PolyHashFamily& f : families_)
        for (u128 a : f.coefficients()) {
            clo_.push_back(u64(a));
            chi_.push_back(u64(a >> 64));
        }
    mb200_sketch_desc d;
    d.rows = rows_;
    d.width = width_;
    d.b = families_.front().modulus().b();
    d.k = families_.front().independence();
    d.key_bits = std::min(families_.front().key_bits(), 64u);
    d.splitter = int(splitter_);
    d.coeffs_lo = clo_.data();
    d.coeffs_hi = chi_.data();
    return d;
}

void CountSketch::init_device() {
    cudaStream_t s;
    cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    stream_ = s;
    const size_t bytes = size_t(rows_) * width_ * sizeof(i64);
    // the counters, then the estimator's 4 x rows u64 words (row_moments reuses
    // them: no allocation -- and no device-synchronising cudaFree -- per call)
    cuda_check(cudaMalloc(&d_counters_, bytes + 4 * size_t(rows_) * sizeof(u64)), "cudaMalloc counters");
    cuda_check(cudaMemsetAsync(d_counters_, 0, bytes, s), "memset");
    cuda_check(cudaStreamSynchronize(s), "sync");
}

void CountSketch::synchronize() const { cuda_check(cudaStreamSynchronize((cudaStream_t)stream_), "sync"); }

void CountSketch::process_device(const void* d_keys, int key_width, const void* d_weights, int weight_kind, u64 n,
                                 void* stream) {
    mb200_sketch_desc d = desc();
    throw_status(mb200_cs_update(&d, d_keys, key_width, d_weights, weight_kind, n, d_counters_,
                                 stream ? stream : stream_));
}

void CountSketch::process_batch(const void* h_keys, int key_width, const void* h_weights, int weight_kind, u64 n) {
    if (n == 0) return;
    if (key_width != 32 && key_width != 64) throw std::invalid_argument("key width must be 32 or 64");
    const unsigned kb = families_.front().key_bits();
    if (kb < unsigned(key_width)) {  // all-or-nothing domain check before any update (polyhash.cpp:60)
        const u64 lim = u64(1) << kb;
        int bad = 0;
        if (key_width == 32) {
            const uint32_t* k = (const uint32_t*)h_keys;
#pragma omp parallel for schedule(static) reduction(| : bad) num_threads(host_threads()) if (n >= (u64(1) << 16))
            for (long long i = 0; i < (long long)n; ++i) bad |= k[i] >= lim;
        } else {
            const u64* k = (const u64*)h_keys;
#pragma omp parallel for schedule(static) reduction(| : bad) num_threads(host_threads()) if (n >= (u64(1) << 16))
            for (long long i = 0; i < (long long)n; ++i) bad |= k[i] >= lim;
        }
        if (bad) throw std::domain_error("key outside domain");
    }
    // 64-bit keys of a <= 32-bit domain (checked above) cross PCIe as u32: the
    // kernels hash the key's value, whatever width it arrives in
    const bool narrow = host_threads() >= kNarrowMinThreads;
    const bool narrow_keys = narrow && key_width == 64 && kb <= 32;
    const int kw_dev = narrow_keys ? 32 : key_width;
    const size_t kbytes = key_width / 8;
    const size_t wbytes = weight_kind == MB200_W_NONE ? 0 : size_t(weight_kind) / 8;
    if (!staging_) staging_ = std::make_unique<Staging>();
    Staging& st = *staging_;
    const u64 want = std::min<u64>(n, u64(1) << 24);
    if (st.chunk < want) {
        // the previous call's copies and kernels have completed (it synchronised)
        for (int i = 0; i < 2; ++i) {
            cudaFree(st.d_keys[i]);
            cudaFree(st.d_w[i]);
            cudaFree(st.d_wn[i]);
            cudaFreeHost(st.h_wn[i]);
            cudaFreeHost(st.h_kn[i]);
            st.d_keys[i] = st.d_w[i] = st.d_wn[i] = st.h_wn[i] = st.h_kn[i] = nullptr;
            cuda_check(cudaMalloc(&st.d_keys[i], want * 8), "cudaMalloc staging");
            cuda_check(cudaMalloc(&st.d_w[i], want * 8), "cudaMalloc staging");
            cuda_check(cudaMalloc(&st.d_wn[i], want * 2), "cudaMalloc staging");
            cuda_check(cudaHostAlloc(&st.h_wn[i], want * 2, cudaHostAllocDefault), "cudaHostAlloc staging");
            cuda_check(cudaHostAlloc(&st.h_kn[i], want * 4, cudaHostAllocDefault), "cudaHostAlloc staging");
        }
        st.chunk = want;
    }
    if (!st.copy) {
        cuda_check(cudaStreamCreateWithFlags(&st.copy, cudaStreamNonBlocking), "stream");
        for (int i = 0; i < 2; ++i) {
            cuda_check(cudaEventCreateWithFlags(&st.ready[i], cudaEventDisableTiming), "event");
            cuda_check(cudaEventCreateWithFlags(&st.freed[i], cudaEventDisableTiming), "event");
            // the host sleeps on this one (it waits while the packing threads idle)
            cuda_check(cudaEventCreateWithFlags(&st.shipped[i], cudaEventDisableTiming | cudaEventBlockingSync),
                       "event");
        }
    }
    const mb200_sketch_desc d = desc();
    cudaStream_t cs = (cudaStream_t)stream_;
    const u64 chunks = (n + st.chunk - 1) / st.chunk;
    st.narrow_bits = 8;
    // A throw mid-loop (CUDA error, status) must not leave copies in flight from
    // the staging slots the next call repacks: drain both streams first.
    struct Drain {
        cudaStream_t a, b;
        ~Drain() {
            if (std::uncaught_exceptions()) {
                cudaStreamSynchronize(a);
                cudaStreamSynchronize(b);
            }
        }
    } drain{st.copy, cs};
    // MB200_TRACE_PROCESS=1: per-chunk copy / kernel event times and host-side
    // waits to stderr (diagnosis of slow host-buffer calls; off by default)
    static const bool trace = std::getenv("MB200_TRACE_PROCESS") != nullptr;
    std::vector<cudaEvent_t> tev;
    std::vector<double> t_pack, t_wait;
    const auto t_call = std::chrono::steady_clock::now();
    auto tevent = [&](cudaStream_t on) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, on);
        tev.push_back(e);
    };
    for (u64 c = 0; c < chunks; ++c) {
        const int slot = int(c & 1);
        const auto t0 = std::chrono::steady_clock::now();
        const u64 off = c * st.chunk;
        const u64 m = std::min<u64>(st.chunk, n - off);
        // Deltas cross PCIe in the narrowest of i8 / i16 that holds the whole
        // chunk (packed here on the host cores while the previous chunk is in
        // flight, sign-extended back on the device): PCIe is the bound of this
        // call, and config 5's |delta| <= 100 ship 5 instead of 8 bytes per item.
        // Updates are bit-identical; a chunk that fits neither ships as is.
        if (c >= 2 && narrow) cuda_check(cudaEventSynchronize(st.shipped[slot]), "sync staging");
        const auto t1 = std::chrono::steady_clock::now();
        int nbits = 0;
        if (wbytes && narrow) {
            const char* src = (const char*)h_weights + off * wbytes;
            nbits = weight_kind == MB200_W_I32 ? narrow_chunk((const int32_t*)src, st.h_wn[slot], m, st.narrow_bits)
                                               : narrow_chunk((const int64_t*)src, st.h_wn[slot], m, st.narrow_bits);
            st.narrow_bits = nbits ? nbits : 64;
        }
        if (narrow_keys) {
            const u64* src = (const u64*)h_keys + off;
            uint32_t* dst = (uint32_t*)st.h_kn[slot];
#pragma omp parallel for schedule(dynamic, 1 << 15) num_threads(host_threads()) if (m >= (u64(1) << 16))
            for (long long i = 0; i < (long long)m; ++i) dst[i] = uint32_t(src[i]);
        }
        if (c >= 2) cuda_check(cudaStreamWaitEvent(st.copy, st.freed[slot], 0), "wait");
        if (trace) {
            const auto t2 = std::chrono::steady_clock::now();
            t_wait.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
            t_pack.push_back(std::chrono::duration<double, std::milli>(t2 - t1).count());
            tevent(st.copy);
        }
        if (narrow_keys)
            cuda_check(cudaMemcpyAsync(st.d_keys[slot], st.h_kn[slot], m * 4, cudaMemcpyHostToDevice, st.copy),
                       "H2D keys");
        else
            cuda_check(cudaMemcpyAsync(st.d_keys[slot], (const char*)h_keys + off * kbytes, m * kbytes,
                                       cudaMemcpyHostToDevice, st.copy),
                       "H2D keys");
        st.h2d_bytes += m * (narrow_keys ? 4 : kbytes);
        if (nbits) {
            cuda_check(cudaMemcpyAsync(st.d_wn[slot], st.h_wn[slot], m * (nbits / 8), cudaMemcpyHostToDevice, st.copy),
                       "H2D weights");
            st.h2d_bytes += m * (nbits / 8);
        } else if (wbytes) {
            cuda_check(cudaMemcpyAsync(st.d_w[slot], (const char*)h_weights + off * wbytes, m * wbytes,
                                       cudaMemcpyHostToDevice, st.copy),
                       "H2D weights");
            st.h2d_bytes += m * wbytes;
        }
        cuda_check(cudaEventRecord(st.shipped[slot], st.copy), "record");
        cuda_check(cudaEventRecord(st.ready[slot], st.copy), "record");
        if (trace) tevent(st.copy);
        cuda_check(cudaStreamWaitEvent(cs, st.ready[slot], 0), "wait");
        if (trace) tevent(cs);
        if (nbits) cuda_check(mb200::launch_widen_deltas(st.d_wn[slot], nbits, st.d_w[slot], weight_kind, m, cs), "widen");
        // keys were validated on the host above: skip the per-chunk device check
        throw_status(mb200::cs_update_nocheck(&d, st.d_keys[slot], kw_dev, wbytes ? st.d_w[slot] : nullptr, weight_kind,
                                     m, d_counters_, cs));
        cuda_check(cudaEventRecord(st.freed[slot], cs), "record");
        if (trace) tevent(cs);
    }
    cuda_check(cudaStreamSynchronize(cs), "sync");
    if (trace && !tev.empty()) {
        double copy = 0, cmax = 0, kern = 0, kmax = 0, span = 0;
        for (size_t c = 0; c + 3 < tev.size(); c += 4) {
            float a = 0, b = 0;
            cudaEventElapsedTime(&a, tev[c], tev[c + 1]);
            cudaEventElapsedTime(&b, tev[c + 2], tev[c + 3]);
            copy += a, cmax = std::max(cmax, (double)a), kern += b, kmax = std::max(kmax, (double)b);
        }
        float sp = 0;
        cudaEventElapsedTime(&sp, tev.front(), tev.back());
        span = sp;
        double pk = 0, pmax = 0, wt = 0, wmax = 0;
        for (double v : t_pack) pk += v, pmax = std::max(pmax, v);
        for (double v : t_wait) wt += v, wmax = std::max(wmax, v);
        const double wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_call).count();
        std::fprintf(stderr,
                     "[mb200 process] n=%llu chunks=%llu wall %.1f ms | device span %.1f | copies %.1f (max %.2f) | "
                     "kernels %.1f (max %.2f) | host pack %.1f (max %.2f) | host waits %.1f (max %.2f)\n",
                     (unsigned long long)n, (unsigned long long)chunks, wall, span, copy, cmax, kern, kmax, pk, pmax, wt,
                     wmax);
        for (cudaEvent_t e : tev) cudaEventDestroy(e);
    }
}

u64 CountSketch::h2d_bytes() const { return staging_ ? staging_->h2d_bytes : 0; }

void set_host_threads(int n) { g_host_threads.store(n > 0 ? n : 0, std::memory_order_relaxed); }
int get_host_threads() { return host_threads(); }

void CountSketch::process(u128 x, i64 delta) {
    if (x >= key_domain()) throw std::domain_error("key outside domain");
    const u64 k = u64(x);
    process_batch(&k, 64, &delta, MB200_W_I64, 1);
}

std::vector<CountSketch::Moment> CountSketch::row_moments() const {
    u64* out = reinterpret_cast<u64*>(d_counters_ + size_t(rows_) * width_);  // init_device's moment words
    cudaStream_t s = (cudaStream_t)stream_;
    throw_status(mb200_cs_moments(d_counters_, rows_, width_, out, s));
    std::vector<u64> h(4 * size_t(rows_));
    cuda_check(cudaMemcpyAsync(h.data(), out, h.size() * sizeof(u64), cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaStreamSynchronize(s), "sync");
    std::vector<Moment> m(rows_);
    for (unsigned r = 0; r < rows_; ++r) m[r] = {(u128(h[4 * r + 1]) << 64) | h[4 * r], h[4 * r + 2] != 0};
    return m;
}

CountSketch::Moment CountSketch::row_second_moment(unsigned row) const {
    if (row >= rows_) throw std::invalid_argument("row out of range");
    return row_moments()[row];
}

CountSketch::Moment CountSketch::second_moment(bool median_rows) const {  // sketch.cpp:160-168
    std::vector<Moment> all = row_moments();
    if (!median_rows || rows_ == 1) return all[0];
    std::sort(all.begin(), all.end(), [](const Moment& a, const Moment& b) { return a.value < b.value; });
    return all[(all.size() - 1) / 2];
}

std::vector<i64> CountSketch::point_query_batch(const void* h_keys, int key_width, u64 n) const {
    std::vector<i64> out(n);
    if (n == 0) return out;
    const size_t kbytes = key_width / 8;
    DevBuf<unsigned char> dk(n * kbytes);
    DevBuf<i64> dout(n);
    cudaStream_t s = (cudaStream_t)stream_;
    cuda_check(cudaMemcpyAsync(dk.p, h_keys, n * kbytes, cudaMemcpyHostToDevice, s), "H2D");
    mb200_sketch_desc d = desc();
    throw_status(mb200_cs_point_query(&d, d_counters_, dk.p, key_width, n, dout.p, s));
    cuda_check(cudaMemcpyAsync(out.data(), dout.p, n * sizeof(i64), cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaStreamSynchronize(s), "sync");
    return out;
}

i64 CountSketch::point_query(u128 x) const {
    if (x >= key_domain()) throw std::domain_error("key outside domain");
    const u64 k = u64(x);
    return point_query_batch(&k, 64, 1)[0];
}

CountSketch& CountSketch::merge(const CountSketch& other) {  // sketch.cpp:182-193
    if (width_ != other.width_ || splitter_ != other.splitter_ || rows_ != other.rows_ ||
        families_.size() != other.families_.size() || seeds_ != other.seeds_ ||
        modulus().b() != other.modulus().b() || key_domain() != other.key_domain() ||
        independence() != other.independence() || seeds_.empty()) {
        throw std::invalid_argument("sketches differ in geometry or seeds");
    }
    other.synchronize();
    throw_status(mb200_cs_merge(d_counters_, other.d_counters_, u64(rows_) * width_, stream_));
    synchronize();
    return *this;
}

CountSketch& CountSketch::allreduce(void* nccl_comm) {
    cudaStream_t s = (cudaStream_t)stream_;
    throw_status(mb200_cs_allreduce(d_counters_, u64(rows_) * width_, nccl_comm, s));
    synchronize();
    return *this;
}

NcclCommunicator::Id NcclCommunicator::unique_id() {
    Id id{};
    throw_status(mb200_nccl_unique_id(id.data()));
    return id;
}

NcclCommunicator::NcclCommunicator(int nranks, const Id& id, int rank) : nranks_(nranks), rank_(rank) {
    throw_status(mb200_nccl_comm_init(nranks, id.data(), rank, &comm_));
}

NcclCommunicator::~NcclCommunicator() { mb200_nccl_comm_destroy(comm_); }

namespace {
void put_u32(std::vector<uint8_t>& out, uint32_t v) {
    for (int i = 0; i < 4; ++i) out.push_back(uint8_t(v >> (8 * i)));
}
void put_u64(std::vector<uint8_t>& out, uint64_t v) {
    for (int i = 0; i < 8; ++i) out.push_back(uint8_t(v >> (8 * i)));
}
uint32_t get_u32(const uint8_t* p) {
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= uint32_t(p[i]) << (8 * i);
    return v;
}
uint64_t get_u64(const uint8_t* p) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= uint64_t(p[i]) << (8 * i);
    return v;
}
constexpr char kMagic[5] = {'M', 'C', 'S', 'K', '1'};
}  // namespace

std::vector<uint8_t> CountSketch::serialize() const {  // sketch.cpp:195-211
    if (seeds_.empty()) throw std::logic_error("sketch with injected families cannot serialize");
    if (splitter_ == Splitter::TwoForOne)
        throw std::logic_error("two-for-one sketches have no MCSK1 form");  // not a reference splitter
    const std::vector<i64> c = counters();
    std::vector<uint8_t> out;
    out.reserve(33 + 8 * seeds_.size() + 8 * c.size());
    out.insert(out.end(), std::begin(kMagic), std::end(kMagic));
    put_u32(out, modulus().b());
    put_u32(out, rows_);
    put_u64(out, width_);
    put_u32(out, independence());
    put_u32(out, uint32_t(splitter_));
    put_u32(out, families_.front().key_bits());
    for (u64 s : seeds_) put_u64(out, s);
    for (i64 v : c) put_u64(out, u64(v));
    return out;
}

CountSketch CountSketch::deserialize(const std::vector<uint8_t>& bytes) {  // sketch.cpp:213-244
    if (bytes.size() < 33 || !std::equal(std::begin(kMagic), std::end(kMagic), bytes.begin()))
        throw std::invalid_argument("malformed sketch payload");
    const uint8_t* p = bytes.data() + 5;
    const uint32_t b = get_u32(p), d = get_u32(p + 4);
    const uint64_t r = get_u64(p + 8);
    const uint32_t k = get_u32(p + 16), splitter = get_u32(p + 20), key_bits = get_u32(p + 24);
    if (b < 2 || b > 127 || d == 0 || splitter > 2 || key_bits > 126 || k == 0)
        throw std::invalid_argument("malformed sketch payload");
    const u128 expect = 33 + u128(8) * d + u128(8) * d * r;
    if (u128(bytes.size()) != expect) throw std::invalid_argument("malformed sketch payload");
    MersenneModulus modulus(b);
    const u128 key_domain = u128(1) << key_bits;
    const uint8_t* q = bytes.data() + 33;
    std::vector<u64> seeds(d);
    std::vector<PolyHashFamily> families;
    for (uint32_t row = 0; row < d; ++row, q += 8) {
        seeds[row] = get_u64(q);
        families.emplace_back(modulus, k, key_domain, seeds[row]);  // re-derived from the seeds
    }
    CountSketch sk(r, Splitter(splitter), std::move(families));
    sk.seeds_ = std::move(seeds);
    std::vector<i64> c(size_t(d) * r);
    for (size_t i = 0; i < c.size(); ++i, q += 8) c[i] = i64(get_u64(q));
    sk.set_counters(c);
    return sk;
}

std::vector<i64> CountSketch::counters() const {
    std::vector<i64> h(size_t(rows_) * width_);
    cudaStream_t s = (cudaStream_t)stream_;
    cuda_check(cudaMemcpyAsync(h.data(), d_counters_, h.size() * sizeof(i64), cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaStreamSynchronize(s), "sync");
    return h;
}

void CountSketch::set_counters(const std::vector<i64>& c) {
    if (c.size() != size_t(rows_) * width_) throw std::invalid_argument("counter count mismatch");
    cudaStream_t s = (cudaStream_t)stream_;
    cuda_check(cudaMemcpyAsync(d_counters_, c.data(), c.size() * sizeof(i64), cudaMemcpyHostToDevice, s), "H2D");
    cuda_check(cudaStreamSynchronize(s), "sync");
}

}  // namespace mersenne::b200
