// mb200_internal.h -- launchers shared between the kernel translation units
// and the C-ABI layer (capi.cu).  Not part of the public boundary.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace mb200 {

constexpr int kMaxK = 16;        // coefficients per family
constexpr int kMaxFamilies = 16; // hash families per sketch
constexpr int kMaxCoeffs = 128;  // families x k

enum KeyWidth { KEY32 = 32, KEY64 = 64 };
enum WeightKind { W_NONE = 0, W_I32 = 32, W_I64 = 64 };
enum SplitKind { SPLIT_POW2 = 0, SPLIT_UNIFORM_ARB = 1, SPLIT_MERSENNE_ARB = 2, SPLIT_TWO_FOR_ONE = 3 };

struct HashParams {
    uint32_t b, k;
    uint64_t p;
    uint64_t lo[kMaxK];
    uint64_t hi[kMaxK];
    // b = 61, k = 8, 64-bit keys: 1 = hi[0..8] hold the adapted coefficients
    // (mb200_precondition61) with shift 0, 2 = with a shift; 0 = Horner
    uint32_t pre;
};

struct SketchParams {
    uint32_t rows;       // counter rows t
    uint32_t families;   // hash families (rows, or ceil(rows/2) for two-for-one)
    uint32_t k;          // coefficients per family
    uint32_t b;          // Mersenne exponent
    uint32_t lw;         // log2 width (Pow2 / two-for-one)
    uint32_t splitter;   // SplitKind
    uint64_t width;      // counters per row
    uint64_t p;
    uint64_t lo[kMaxCoeffs];
    uint64_t hi[kMaxCoeffs];
};

// hashing (kernels_hash.cu)
cudaError_t launch_hash61_key32(const uint32_t* keys, uint64_t n, const HashParams& hp, uint64_t* out,
                                cudaStream_t s);
cudaError_t launch_hash61_key64(const uint64_t* keys, uint64_t n, const HashParams& hp, uint64_t* out,
                                cudaStream_t s);
cudaError_t launch_hash_generic(const void* keys, int key_width, uint64_t n, const HashParams& hp,
                                uint64_t* out, cudaStream_t s);
cudaError_t launch_hash89(const uint64_t* keys, uint64_t n, const HashParams& hp, uint64_t* out_lo,
                          uint64_t* out_hi, cudaStream_t s);
// 62 <= b <= 127: generic four-limb Horner, outputs low 64 / high bits
cudaError_t launch_hash_wide(const uint64_t* keys, uint64_t n, const HashParams& hp, uint64_t* out_lo,
                             uint64_t* out_hi, cudaStream_t s);
// domain validation: counts keys >= 2^key_bits into *d_count (pre-zeroed)
cudaError_t launch_count_out_of_domain(const void* keys, int key_width, uint64_t n, uint32_t key_bits,
                                       unsigned long long* d_count, cudaStream_t s);

// sketch (kernels_sketch.cu)
// Sign-extend host-narrowed deltas (i8 or i16, see CountSketch::process_batch)
// back to the API's weight kind (i32 or i64) in device memory.
cudaError_t launch_widen_deltas(const void* src, int src_bits, void* dst, int dst_bits, uint64_t n,
                                cudaStream_t s);
cudaError_t launch_cs_update(const SketchParams& sp, const void* keys, int key_width, const void* w,
                             int w_kind, uint64_t n, int64_t* table, cudaStream_t s);
// heavy-hitter pipeline for tables larger than shared memory (kernels_hot.cu);
// requires |delta| < 2^31 (w_kind W_NONE or W_I32)
cudaError_t launch_cs_hot(const SketchParams& sp, const void* keys, int key_width, const void* w, int w_kind,
                          uint64_t n, int64_t* table, cudaStream_t s);
cudaError_t hot_stats(uint64_t out[8], bool reset);
// bench hook: events around the dominant scatter kernel of each launch_cs_hot call
void kernel_timer(bool enable);
cudaError_t kernel_timer_read(double* total_ms, uint64_t* launches);
enum LargeTableStrategy { STRAT_DIRECT = 0, STRAT_BINNED = 1, STRAT_ROWS = 2 };
int set_large_table_strategy(int s);  // returns the previous strategy, -1 if invalid
cudaError_t launch_cs_moments(const int64_t* table, uint32_t rows, uint64_t width, uint64_t* out,
                              cudaStream_t s);
cudaError_t launch_cs_merge(int64_t* dst, const int64_t* src, uint64_t count, cudaStream_t s);
// split_pow2 / split_arb_uniform / split_arb_mersenne (sketch.cpp:13-34) of u64 hash
// values (sp carries b, splitter and width = 2^l or r); hashes outside the
// splitter's domain are counted into *d_flags
cudaError_t launch_split_batch(const SketchParams& sp, const uint64_t* h, uint64_t n, uint64_t* index,
                               int32_t* sign, unsigned long long* d_flags, cudaStream_t s);
cudaError_t launch_cs_point_query(const SketchParams& sp, const int64_t* table, const void* keys,
                                  int key_width, uint64_t n, int64_t* out, cudaStream_t s);

// division (kernels_divmod.cu)
cudaError_t launch_pm_divmod(const uint64_t* v, uint64_t n, uint32_t b, uint64_t c, uint32_t iters,
                             uint64_t* q, uint64_t* r, unsigned long long* d_flags, cudaStream_t s);
// Alg 5 from given quotients z (u64): r = (v + z c) mod 2^b
cudaError_t launch_pm_mod(const uint64_t* v, const uint64_t* z, uint64_t n, uint32_t b, uint64_t c, uint64_t* r,
                          cudaStream_t s);
cudaError_t launch_count_above(const uint64_t* v, uint64_t n, uint64_t max_lo, uint64_t max_hi,
                               unsigned long long* d_count, cudaStream_t s);
// bucket maps: kind 0 map_pow2, 1 map_mersenne, 2 exact division (m iterations);
// values >= bound (0 = no bound) are counted into *d_flags
cudaError_t launch_bucket_map(int kind, const uint64_t* v, uint64_t n, uint32_t b, uint64_t c, uint32_t m,
                              uint64_t r, uint64_t bound, uint64_t* out, unsigned long long* d_flags,
                              cudaStream_t s);

// exhaustive moment enumeration (kernels_enum.cu): sp carries b, p, splitter, width
cudaError_t launch_enum_moments(const SketchParams& sp, uint32_t n, uint32_t w2, const uint32_t* xs,
                                const int32_t* ws, uint16_t* tab, unsigned long long* out, cudaStream_t s);

int sm_count();
int device_id();

}  // namespace mb200
