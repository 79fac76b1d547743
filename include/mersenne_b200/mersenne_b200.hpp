// mersenne_b200.hpp -- C++ host API of the B200 path, keeping the reference
// library's names and semantics (/root/reference/proj/include/mersenne/
// {field,polyhash,sketch}.hpp) and adding batched device methods.  It reaches
// the GPU only through the C-ABI in <mersenne_b200.h>.
//
// Error behaviour mirrors the reference: std::invalid_argument at
// construction, std::domain_error at call (all-or-nothing for batches),
// std::logic_error for serializing injected families; CUDA failures raise
// std::runtime_error.  There is no CPU fallback.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <vector>

#include "../mersenne_b200.h"

namespace mersenne::b200 {

using u64 = std::uint64_t;
using i64 = std::int64_t;
using u128 = unsigned __int128;

// throws the reference exception class for an mb200 status code
void throw_status(int status);

// field.hpp:20-33
class MersenneModulus {
public:
    explicit MersenneModulus(unsigned b, bool require_prime = false);
    unsigned b() const { return b_; }
    u128 p() const { return (u128(1) << b_) - 1; }
    bool prime_exponent() const { return prime_; }

private:
    unsigned b_;
    bool prime_;
};

// field.hpp:11: arithmetic backend.  On the GPU every engine computes the same
// values (the kernels are fixed-limb); the choice is validated and kept for parity.
enum class Engine { Auto, Native, Generic };

// 256-bit little-endian value: the role of the reference's UWide (uwide.hpp) at
// this API's single-value entries.  The GPU batches take u128 (lo, hi) pairs.
struct UWide {
    std::array<u64, 4> limb{};
    UWide() = default;
    explicit UWide(u64 v) : limb{v, 0, 0, 0} {}
    static UWide of_u128(u128 v) {
        UWide w;
        w.limb = {u64(v), u64(v >> 64), 0, 0};
        return w;
    }
    u128 low_u128() const { return (u128(limb[1]) << 64) | limb[0]; }
    bool fits_u128() const { return limb[2] == 0 && limb[3] == 0; }
    u64 operator[](size_t i) const { return limb[i]; }
    friend bool operator==(const UWide&, const UWide&) = default;
};

struct DivMod {  // field.hpp:13-16
    UWide quotient;
    UWide remainder;
};

// field.hpp:38-63: modulus 2^b - c, iteration count and admissible maximum
// computed on the host for any u128 c (field.cpp:224-244).  The GPU batches
// divide for b <= 64 (c < 2^(b-1) < 2^64); wider moduli are validated and
// described here but their division raises runtime_error (MB200_UNSUPPORTED).
class PseudoMersenneModulus {
public:
    PseudoMersenneModulus(unsigned b, u128 c, unsigned m_iters = 0, Engine engine = Engine::Auto);
    unsigned b() const { return b_; }
    u128 c() const { return c_; }
    u128 p() const { return (u128(1) << b_) - c_; }
    unsigned iterations() const { return m_; }
    Engine engine() const { return engine_; }
    const UWide& max_input() const { return max_input_; }

    // pseudo_mersenne_div + pseudo_mersenne_mod over device arrays (field.cpp:260-273):
    // d_v holds n u128 as (lo, hi) pairs; d_q, d_r receive n u64 each (d_r may be null).
    void divmod_device(const u64* d_v, u64 n, u64* d_q, u64* d_r, void* stream = nullptr) const;
    // host-buffer convenience: copies in, divides, copies out
    void divmod(const u64* h_v, u64 n, u64* h_q, u64* h_r) const;

private:
    unsigned b_;
    u128 c_;
    unsigned m_;
    Engine engine_;
    UWide max_input_;
};

// field.hpp:76-82 -- the reference's free functions.  Single values launch a
// one-element GPU batch (API parity); the *_device forms are the batch path.
DivMod mersenne_divmod(const UWide& v, const MersenneModulus& mod);            // Alg 3, b <= 63
UWide pseudo_mersenne_div(const UWide& v, const PseudoMersenneModulus& mod);   // Alg 4
UWide pseudo_mersenne_mod(const UWide& v, const UWide& z, const PseudoMersenneModulus& mod);  // Alg 5
void mersenne_divmod_device(const u64* d_v, u64 n, const MersenneModulus& mod, u64* d_q, u64* d_r,
                            void* stream = nullptr);
void pseudo_mersenne_div_device(const u64* d_v, u64 n, const PseudoMersenneModulus& mod, u64* d_q,
                                void* stream = nullptr);
void pseudo_mersenne_mod_device(const u64* d_v, const u64* d_z, u64 n, const PseudoMersenneModulus& mod,
                                u64* d_r, void* stream = nullptr);

// bucketing.hpp:31-58 -- bucket maps over device u64 arrays (b <= 64)
// map_pow2: floor(v r / 2^b), v < 2^b;  map_mersenne: floor((v+1) r / 2^b), v < 2^b - 1
void map_pow2_device(const u64* d_v, u64 n, unsigned b, u64 r, u64* d_out, void* stream = nullptr);
void map_mersenne_device(const u64* d_v, u64 n, unsigned b, u64 r, u64* d_out, void* stream = nullptr);

// bucketing.hpp:43-58: floor(v r / p) on [0, p) by Alg 4, the divider's iteration
// count grown at construction until (p-1) r is admissible (bucketing.cpp:75-89)
class ExactDivisionMap {
public:
    ExactDivisionMap(const PseudoMersenneModulus& mod, u64 r);
    u64 operator()(u64 v) const;  // one value (API parity; launches a one-element batch)
    void map_device(const u64* d_v, u64 n, u64* d_out, void* stream = nullptr) const;
    const PseudoMersenneModulus& divider() const { return divider_; }
    u64 buckets() const { return r_; }

private:
    PseudoMersenneModulus divider_;
    u64 r_;
};

enum class HashFinish { ConditionalSubtract, BranchFree };  // polyhash.hpp:10-13 (same values)

// polyhash.hpp:18-43
class PolyHashFamily {
public:
    PolyHashFamily(const MersenneModulus& modulus, unsigned k, u128 key_domain, u64 seed,
                   HashFinish finish = HashFinish::ConditionalSubtract);
    PolyHashFamily(const MersenneModulus& modulus, std::vector<u128> coefficients, u128 key_domain,
                   HashFinish finish = HashFinish::ConditionalSubtract);

    // one key (API parity; launches a one-element batch)
    u128 operator()(u128 x) const;
    // batch over device keys (u32 or u64): out_lo gets the low 64 bits, out_hi (b > 64 only) the rest
    void hash_device(const void* d_keys, int key_width, u64 n, u64* d_out_lo, u64* d_out_hi = nullptr,
                     void* stream = nullptr) const;
    // batch over host keys
    std::vector<u128> hash(const std::vector<u64>& keys) const;

    const MersenneModulus& modulus() const { return modulus_; }
    const std::vector<u128>& coefficients() const { return coeffs_; }
    unsigned independence() const { return unsigned(coeffs_.size()); }
    u128 key_domain() const { return key_domain_; }
    unsigned key_bits() const;
    HashFinish finish() const { return finish_; }

private:
    void validate() const;
    MersenneModulus modulus_;
    std::vector<u128> coeffs_;
    u128 key_domain_;
    HashFinish finish_;
};

enum class Splitter : uint32_t { Pow2 = 0, UniformArb = 1, MersenneArb = 2, TwoForOne = 3 };

struct SignIndexPair {
    u128 index;
    int sign;
    friend bool operator==(const SignIndexPair&, const SignIndexPair&) = default;
};
// sketch.hpp:17-30 (host helpers; the kernels apply the same rules in registers)
SignIndexPair split_pow2(u128 h, unsigned b, unsigned l);            // sketch.cpp:13-19
SignIndexPair split_arb_uniform(u128 h, unsigned b, u128 r);         // sketch.cpp:21-29
SignIndexPair split_arb_mersenne(u128 h, unsigned b, u128 r);        // sketch.cpp:31-34
// the same three rules over a device batch of u64 hash values (b <= 64):
// l_or_r = l for Pow2, r for the arbitrary-width splitters; d_sign gets +1 / -1
void split_device(Splitter splitter, const u64* d_h, u64 n, unsigned b, u64 l_or_r, u64* d_index, int32_t* d_sign,
                  void* stream = nullptr);

// sketch.hpp:40-92 with counters resident in HBM of the current device
class CountSketch {
public:
    CountSketch(unsigned rows, u64 width, const MersenneModulus& modulus, u128 key_domain, Splitter splitter,
                u64 seed, unsigned independence = 4);
    // Injected families: one per row (or one per two rows for Splitter::TwoForOne).
    CountSketch(u64 width, Splitter splitter, std::vector<PolyHashFamily> families, unsigned rows = 0);
    CountSketch(const CountSketch& other);             // value semantics: own HBM table, copied D2D
    CountSketch& operator=(const CountSketch& other);
    CountSketch(CountSketch&&) noexcept;
    ~CountSketch();

    void process(u128 x, i64 delta);  // API parity (one-item batch)
    // host batch: key_width 32/64, weight_kind MB200_W_* (h_weights may be null = +1)
    void process_batch(const void* h_keys, int key_width, const void* h_weights, int weight_kind, u64 n);
    // bytes process_batch has moved host -> device over this sketch's lifetime
    u64 h2d_bytes() const;
    // device batch, asynchronous on `stream`
    void process_device(const void* d_keys, int key_width, const void* d_weights, int weight_kind, u64 n,
                        void* stream = nullptr);

    struct Moment {
        u128 value;
        bool saturated;
        friend bool operator==(const Moment&, const Moment&) = default;
    };
    Moment row_second_moment(unsigned row) const;
    Moment second_moment(bool median_rows = false) const;
    std::vector<Moment> row_moments() const;

    i64 point_query(u128 x) const;
    std::vector<i64> point_query_batch(const void* h_keys, int key_width, u64 n) const;

    CountSketch& merge(const CountSketch& other);  // requires identical seeds (sketch.cpp:182-193)
    // merge() across GPUs: the tables of this sketch's replicas on every rank of
    // `nccl_comm` (an ncclComm_t, e.g. NcclCommunicator::get()) are summed in place
    // by one NCCL allreduce; every rank ends with the merged table.
    CountSketch& allreduce(void* nccl_comm);

    // MCSK1 wire format (sketch.cpp:195-244), byte-identical to the reference:
    // "MCSK1", u32 b, u32 rows, u64 width, u32 k, u32 splitter, u32 log2(u),
    // rows x u64 seeds, rows x width x u64 counters, little endian.
    std::vector<uint8_t> serialize() const;
    static CountSketch deserialize(const std::vector<uint8_t>& bytes);

    unsigned rows() const { return rows_; }
    u64 width() const { return width_; }
    Splitter splitter() const { return splitter_; }
    const MersenneModulus& modulus() const { return families_.front().modulus(); }
    u128 key_domain() const { return families_.front().key_domain(); }
    unsigned independence() const { return families_.front().independence(); }
    const std::vector<u64>& seeds() const { return seeds_; }
    const std::vector<PolyHashFamily>& families() const { return families_; }
    std::vector<i64> counters() const;         // D2H copy (row-major, sketch.hpp:75)
    i64 counter(unsigned row, u64 index) const;  // sketch.hpp:76 (one D2H read)
    // sketch.hpp:78-82: geometry, seeds and counters
    friend bool operator==(const CountSketch& a, const CountSketch& b);
    void set_counters(const std::vector<i64>& c);
    i64* device_counters() { return d_counters_; }
    const i64* device_counters() const { return d_counters_; }
    void synchronize() const;

private:
    void validate() const;
    void init_device();
    mb200_sketch_desc desc() const;

    unsigned rows_;
    u64 width_;
    Splitter splitter_;
    std::vector<PolyHashFamily> families_;
    std::vector<u64> seeds_;
    mutable std::vector<u64> clo_, chi_;  // coefficient cache for the C-ABI descriptor
    i64* d_counters_ = nullptr;
    void* stream_ = nullptr;  // cudaStream_t owned by the sketch
    struct Staging;
    std::unique_ptr<Staging> staging_;
};

// One NCCL communicator over the ranks of a job (one GPU per rank), for
// CountSketch::allreduce.  Rank 0 draws unique_id() and ships its bytes to the
// other ranks by any side channel; every rank then constructs with them.
class NcclCommunicator {
public:
    using Id = std::array<uint8_t, MB200_NCCL_UNIQUE_ID_BYTES>;
    static Id unique_id();
    NcclCommunicator(int nranks, const Id& id, int rank);  // current device; collective
    NcclCommunicator(const NcclCommunicator&) = delete;
    NcclCommunicator& operator=(const NcclCommunicator&) = delete;
    ~NcclCommunicator();
    void* get() const { return comm_; }
    int size() const { return nranks_; }
    int rank() const { return rank_; }

private:
    void* comm_ = nullptr;
    int nranks_, rank_;
};

// Host threads CountSketch::process_batch uses to pack and check its inputs
// (0 = automatic: this process's CPUs / LOCAL_WORLD_SIZE); below 6 the
// deltas and keys ship unnarrowed.
void set_host_threads(int n);
int get_host_threads();

}  // namespace mersenne::b200
