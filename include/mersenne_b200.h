/*
 * mersenne_b200.h -- C-ABI drop-in boundary of the B200 hashing / sketching path.
 *
 * The reference (/root/reference/proj) exposes this path only as C++ classes of
 * a static library.  This header is the flat C boundary a binding
 * (ctypes, cgo, JNI, N-API, or the reference's own C++ classes) binds to.  Each
 * entry cites the reference interface it replaces.  Plain pointers and sizes
 * only; CUDA streams travel as `void*` (a cudaStream_t, NULL = legacy default).
 *
 * Two layers:
 *   1. device-array entries (mb200_hash61, mb200_cs_update, ...): inputs and
 *      outputs are device pointers; the call is asynchronous on `stream` unless
 *      a data-dependent domain check is required (see each entry).
 *   2. object entries (mb200_sketch_*): the reference's CountSketch API on
 *      host buffers; host<->device copies are inside the call.
 *
 * Errors: every entry returns a status code; the code names the reference
 * exception class it stands for and mb200_last_error() returns the
 * reference's message (thread-local).  There is no CPU fallback: when no
 * sm_100 device is present every device entry returns MB200_CUDA_ERROR.
 */
#ifndef MERSENNE_B200_H
#define MERSENNE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MB200_ABI_VERSION 2

#define MB200_OK 0
#define MB200_INVALID_ARGUMENT 1 /* std::invalid_argument (construction-time checks) */
#define MB200_DOMAIN_ERROR 2     /* std::domain_error (polyhash.cpp:60, field.cpp:210, :262) */
#define MB200_LOGIC_ERROR 3      /* std::logic_error (sketch.cpp:197) */
#define MB200_CUDA_ERROR 4       /* CUDA runtime failure / no usable device */
#define MB200_UNSUPPORTED 5      /* valid for the reference, not implemented on the GPU path */

/* key widths */
#define MB200_KEY_U32 32
#define MB200_KEY_U64 64
/* weight kinds (NULL weights = every delta is +1) */
#define MB200_W_NONE 0
#define MB200_W_I32 32
#define MB200_W_I64 64
/* splitters: sketch.hpp:33-37, plus the config-4 two-for-one row layout */
#define MB200_SPLIT_POW2 0         /* split_pow2, sketch.cpp:13-19 */
#define MB200_SPLIT_UNIFORM_ARB 1  /* split_arb_uniform, sketch.cpp:21-29 */
#define MB200_SPLIT_MERSENNE_ARB 2 /* split_arb_mersenne, sketch.cpp:31-34 */
#define MB200_SPLIT_TWO_FOR_ONE 3  /* one hash -> two rows */

const char* mb200_last_error(void);
int mb200_abi_version(void);
/* number of visible sm_100 devices (0 when none) */
int mb200_device_count(void);

/* ---------------------------------------------------------------- field --- */
/* MersenneModulus(b, require_prime) validation: field.cpp:197-206 */
int mb200_mersenne_modulus_check(unsigned b, int require_prime);
/* PseudoMersenneModulus(b, c, m_iters) ctor: field.cpp:224-244 (default
 * iteration count field.cpp:156-171, domain threshold :173-193) for any u128
 * c = (c_hi << 64) | c_lo; max_input receives the 256-bit admissible maximum. */
int mb200_pm_modulus(unsigned b, uint64_t c_lo, uint64_t c_hi, unsigned m_iters, unsigned* iterations,
                     uint64_t max_input[4]);

/* ------------------------------------------------------------- hashing --- */
/* PolyHashFamily(modulus, k, u, seed) coefficient draw: polyhash.cpp:12-35.
 * lo/hi receive a_0..a_{k-1} (hi only for b > 64; may be NULL otherwise). */
int mb200_draw_coeffs(unsigned b, unsigned k, uint64_t seed, uint64_t* lo, uint64_t* hi);
/* Adapted coefficients of a degree-7 polynomial over Z_p, p = 2^61 - 1 (the k = 8
 * family of PolyHashFamily::operator(), polyhash.cpp:64-76): plan = {al0..al5, s,
 * a7, r0} with  u(x) = a7 (x + s) U(x) + r0,  U = (w + z + al4) w + al5,
 * w = (x + al2) z + al3,  z = (x + al0) x + al1  -- five modular products per
 * key instead of Horner's seven, same value.  mb200_hash61 calls this itself
 * for k = 8 and 64-bit keys; exported for tests.  MB200_UNSUPPORTED when
 * coeffs[7] = 0 (Horner is used then).  No reference counterpart. */
int mb200_precondition61(const uint64_t coeffs[8], uint64_t plan[9]);
/* CountSketch row seeds: successive SplitMix64(master).next(), sketch.cpp:72-77 */
int mb200_row_seeds(uint64_t master, unsigned rows, uint64_t* out);

/* K1 -- Alg 1 for p = 2^b - 1, b <= 61: replaces PolyHashFamily::operator()
 * native path (polyhash.cpp:59-76) over a batch.  coeffs: host array a_0..a_{k-1}
 * (k <= 16, each < p).  Keys must lie in [0, 2^key_bits) (domain_error otherwise,
 * all-or-nothing: checked before any output is written; the check synchronizes
 * `stream` and only runs when key_bits < key_width).  For b == 61 any
 * key_bits <= 64 is accepted (keys beyond the reference's u <= 2^60 are reduced
 * exactly); for b < 61 the reference domain p >= 2u - 1 applies.  d_out: n u64. */
int mb200_hash61(const void* d_keys, int key_width, uint64_t n, unsigned b, const uint64_t* coeffs,
                 unsigned k, unsigned key_bits, uint64_t* d_out, void* stream);

/* K2 -- Alg 1 for p = 2^89 - 1: replaces the generic path (polyhash.cpp:78-88 with
 * wide_mul uwide.hpp:148-163 and mersenne_reduce_partial field.hpp:66-73).
 * u64 keys; outputs split into low 64 bits and high 25 bits (two dense arrays). */
int mb200_hash89(const uint64_t* d_keys, uint64_t n, const uint64_t* coeffs_lo,
                 const uint64_t* coeffs_hi, unsigned k, unsigned key_bits, uint64_t* d_out_lo,
                 uint64_t* d_out_hi, void* stream);
/* Generic Horner for 62 <= b <= 127 (polyhash.cpp:78-88: UWide products,
 * mersenne_reduce_partial field.hpp:66-73, branch-free finish), u64 keys in
 * [0, 2^key_bits) (key_bits <= b - 1 for b <= 64); coefficients as (lo, hi)
 * 64-bit halves, lowest first; outputs split into low and high 64 bits. */
int mb200_hash_wide(const uint64_t* d_keys, uint64_t n, unsigned b, const uint64_t* coeffs_lo,
                    const uint64_t* coeffs_hi, unsigned k, unsigned key_bits, uint64_t* d_out_lo,
                    uint64_t* d_out_hi, void* stream);

/* ------------------------------------------------------------ division --- */
/* K6 -- Alg 4 + Alg 5 for p = 2^b - c (2 <= b <= 64, 1 <= c < 2^(b-1)):
 * replaces pseudo_mersenne_div (field.cpp:260-265) + pseudo_mersenne_mod
 * (:267-273).  d_v: n u128 as interleaved (lo, hi) u64 pairs; d_q, d_r: n u64.
 * m_iters = 0 picks the reference default.  Inputs above max_input raise
 * domain_error (checked, synchronizing, only when max_input < 2^128).
 * d_overflow (nullable, device u64, accumulated): number of warps that met a
 * quotient >= 2^64 (possible only for v >= 2^64 p). */
int mb200_pm_divmod(const uint64_t* d_v, uint64_t n, unsigned b, uint64_t c, unsigned m_iters,
                    uint64_t* d_q, uint64_t* d_r, uint64_t* d_overflow, void* stream);

/* pseudo_mersenne_div alone (field.cpp:260-265): quotients only (same rules as
 * mb200_pm_divmod, which also accepts d_r == NULL) */
int mb200_pm_div(const uint64_t* d_v, uint64_t n, unsigned b, uint64_t c, unsigned m_iters,
                 uint64_t* d_q, uint64_t* d_overflow, void* stream);
/* pseudo_mersenne_mod alone (field.cpp:267-273): r = (v + z c) & (2^b - 1) for
 * given quotients z (u64); b <= 64 */
int mb200_pm_mod(const uint64_t* d_v, const uint64_t* d_z, uint64_t n, unsigned b, uint64_t c,
                 uint64_t* d_r, void* stream);
/* mersenne_divmod, Alg 3 (field.cpp:208-222) for p = 2^b - 1, 2 <= b <= 63:
 * branch-free quotient and remainder of every v < 2^(2b) (u128 (lo, hi) pairs);
 * any larger input raises domain_error "input exceeds 2^(2b)" before any output
 * is written (synchronizes `stream`).  b in [64, 127]: MB200_UNSUPPORTED. */
int mb200_mersenne_divmod(const uint64_t* d_v, uint64_t n, unsigned b, uint64_t* d_q, uint64_t* d_r,
                          void* stream);

/* ------------------------------------------------------------- bucketing --- */
/* Bucket maps of bucketing.hpp:31-58 on device u64 arrays (b <= 64):
 *   MB200_MAP_POW2      map_pow2(v, b, r)      = floor(v r / 2^b)       bucketing.cpp:61-66
 *                       v < 2^b, 1 <= r <= 2^b (r < 2^64)
 *   MB200_MAP_MERSENNE  map_mersenne(v, b, r)  = floor((v+1) r / 2^b)   bucketing.cpp:68-73
 *                       v < 2^b - 1, 1 <= r <= 2^b - 1
 *   MB200_MAP_EXACT_DIV ExactDivisionMap(PseudoMersenneModulus(b, c), r)(v)
 *                       = floor(v r / p), p = 2^b - c, by Alg 4     bucketing.cpp:75-95
 *                       v < p, 1 <= r <= p; c is ignored by the other kinds. */
#define MB200_MAP_POW2 0
#define MB200_MAP_MERSENNE 1
#define MB200_MAP_EXACT_DIV 2
/* ExactDivisionMap ctor (bucketing.cpp:75-89): the divider's iteration count,
 * the smallest m >= 1 with (p-1) r <= max_input(b, c, m).  r outside [1, p]:
 * MB200_INVALID_ARGUMENT "bucket count must be in [1, p]".  b <= 127. */
int mb200_exact_division_iterations(unsigned b, uint64_t c, uint64_t r, unsigned* iterations);
/* The reference asserts the value domain; here values outside it are counted:
 * into *d_out_of_domain (nullable device u64, accumulated, asynchronous), or,
 * when d_out_of_domain is NULL, by a synchronizing read-back that returns
 * MB200_DOMAIN_ERROR "value outside the map's domain" (outputs for in-domain
 * values are written either way). */
int mb200_bucket_map(int kind, const uint64_t* d_v, uint64_t n, unsigned b, uint64_t c, uint64_t r,
                     uint64_t* d_out, uint64_t* d_out_of_domain, void* stream);

/* ------------------------------------------------ moment enumeration --- */
/* enum_moment_sums_serial / _parallel (verify.hpp:123-145, verify.cpp:505-603):
 * over all p^4 degree-3 coefficient vectors (p = 2^b - 1) build the one-row
 * sketch of the stream (keys[i], deltas[i]) with `buckets` counters and the
 * given splitter (MB200_SPLIT_POW2 / _UNIFORM_ARB / _MERSENNE_ARB), and sum
 * X = sum_i C_i^2 and X^2 exactly.  out[0..1] = sum_x (lo, hi), out[2..3] =
 * sum_x_sq (lo, hi), out[4] = families (p^4).  Validation and messages follow
 * validate_moment_spec (verify.cpp:480-503) and exact_family_count (:566-573):
 * 2 <= b <= 15, keys < key_domain <= p, distinct modulo p, sum |delta| <= 1024.
 * The GPU kernel takes at most 64 non-zero-weight entries (MB200_UNSUPPORTED
 * beyond).  Synchronizes `stream`. */
int mb200_enum_moment_sums(unsigned b, uint64_t key_domain, uint64_t buckets, int splitter,
                           const uint64_t* keys, const int64_t* deltas, uint64_t n, uint64_t out[5],
                           void* stream);

/* ------------------------------------------------------------ splitters --- */
/* The two-for-one bucket/sign split on a batch of u64 hash values (b <= 64):
 *   MB200_SPLIT_POW2         split_pow2(h, b, l)          sketch.cpp:13-19   (l_or_r = l < b)
 *   MB200_SPLIT_UNIFORM_ARB  split_arb_uniform(h, b, r)   sketch.cpp:21-29   (1 <= r <= 2^(b-1))
 *   MB200_SPLIT_MERSENNE_ARB split_arb_mersenne(h, b, r)  sketch.cpp:31-34
 * d_index: u64 index, d_sign: +1 / -1.  Hash values outside the splitter's domain
 * (h >= 2^b; h >= 2^b - 1 for the Mersenne splitter; the reference asserts) are
 * counted into *d_out_of_domain (nullable, accumulated), or, when it is NULL, by a
 * synchronizing read-back returning MB200_DOMAIN_ERROR. */
int mb200_split_batch(int splitter, const uint64_t* d_h, uint64_t n, unsigned b, uint64_t l_or_r,
                      uint64_t* d_index, int32_t* d_sign, uint64_t* d_out_of_domain, void* stream);

/* --------------------------------------------------------- count sketch --- */
typedef struct {
    unsigned rows;             /* counter rows t (<= 16) */
    uint64_t width;            /* counters per row */
    unsigned b;                /* Mersenne exponent: <= 61 or 89 */
    unsigned k;                /* coefficients per family (independence, <= 16) */
    unsigned key_bits;         /* key domain is [0, 2^key_bits) */
    int splitter;              /* MB200_SPLIT_* */
    const uint64_t* coeffs_lo; /* host, families x k (families = rows, or ceil(rows/2) for TWO_FOR_ONE) */
    const uint64_t* coeffs_hi; /* host, families x k, b > 64 only (else NULL) */
} mb200_sketch_desc;

/* K3+K4 -- fused hash -> split -> scatter-add: replaces CountSketch::process
 * (sketch.cpp:133-140) over a batch.  d_counters: rows x width i64, row-major
 * (sketch.hpp:75 layout), accumulated in place with wrapping adds.  Keys are
 * domain-checked all-or-nothing (see mb200_hash61). */
int mb200_cs_update(const mb200_sketch_desc* desc, const void* d_keys, int key_width,
                    const void* d_weights, int weight_kind, uint64_t n, int64_t* d_counters,
                    void* stream);
/* K5 -- row_second_moment for every row (sketch.cpp:142-158): d_out receives
 * rows x 4 u64 = (value lo, value hi, saturated, 0).  The lower median over rows
 * (second_moment(true), sketch.cpp:160-168) is taken on the host. */
int mb200_cs_moments(const int64_t* d_counters, unsigned rows, uint64_t width, uint64_t* d_out,
                     void* stream);
/* CountSketch::merge counter sum (sketch.cpp:182-193), wrapping */
int mb200_cs_merge(int64_t* d_dst, const int64_t* d_src, uint64_t count, void* stream);
/* CountSketch::point_query (sketch.cpp:170-180) over a batch of keys */
int mb200_cs_point_query(const mb200_sketch_desc* desc, const int64_t* d_counters,
                         const void* d_keys, int key_width, uint64_t n, int64_t* d_out,
                         void* stream);

/* ---------------------------------------------- sketch object (host API) --- */
typedef struct mb200_sketch mb200_sketch;
/* CountSketch(rows, width, MersenneModulus(b, true), 2^key_bits, splitter, seed,
 * independence): sketch.cpp:68-82.  Counters live in HBM on the current device. */
int mb200_sketch_create(unsigned rows, uint64_t width, unsigned b, unsigned key_bits, int splitter,
                        uint64_t seed, unsigned independence, mb200_sketch** out);
/* CountSketch(width, splitter, families): sketch.cpp:84-95 (families x k coefficients) */
int mb200_sketch_create_families(uint64_t width, int splitter, unsigned b, unsigned key_bits,
                                 unsigned families, unsigned k, const uint64_t* coeffs_lo,
                                 const uint64_t* coeffs_hi, unsigned rows, mb200_sketch** out);
void mb200_sketch_destroy(mb200_sketch* s);
/* process(key, delta) for every item of a HOST batch: copies are pipelined in
 * chunks against the scatter kernel; returns after the batch is applied. */
int mb200_sketch_process(mb200_sketch* s, const void* h_keys, int key_width, const void* h_weights,
                         int weight_kind, uint64_t n);
/* bytes mb200_sketch_process has moved host -> device for this sketch (keys
 * plus deltas; deltas travel narrowed to i8 / i16 when a chunk fits).  A
 * transport statistic with no reference counterpart. */
int mb200_sketch_h2d_bytes(const mb200_sketch* s, uint64_t* out);
/* host threads mb200_sketch_process packs and checks with (0 = automatic:
 * this process's CPUs divided by LOCAL_WORLD_SIZE); with fewer than 6 the
 * inputs ship unnarrowed.  No reference counterpart. */
void mb200_set_host_threads(int n);
int mb200_host_threads(void);
/* same on DEVICE arrays, asynchronous on `stream` */
int mb200_sketch_process_device(mb200_sketch* s, const void* d_keys, int key_width,
                                const void* d_weights, int weight_kind, uint64_t n, void* stream);
int mb200_sketch_row_second_moment(mb200_sketch* s, unsigned row, uint64_t* lo, uint64_t* hi,
                                   int* saturated);
int mb200_sketch_second_moment(mb200_sketch* s, int median_rows, uint64_t* lo, uint64_t* hi,
                               int* saturated);
int mb200_sketch_point_query(mb200_sketch* s, const void* h_keys, int key_width, uint64_t n,
                             int64_t* h_out);
int mb200_sketch_merge(mb200_sketch* dst, const mb200_sketch* src);
int mb200_sketch_counters(mb200_sketch* s, int64_t* h_out);
int mb200_sketch_set_counters(mb200_sketch* s, const int64_t* h_in);
int64_t* mb200_sketch_device_counters(mb200_sketch* s);
int mb200_sketch_info(const mb200_sketch* s, unsigned* rows, uint64_t* width, unsigned* b,
                      unsigned* k, unsigned* key_bits, int* splitter);
/* seeds() (sketch.hpp:73): logic_error for injected families */
int mb200_sketch_seeds(const mb200_sketch* s, uint64_t* out);
/* families x k coefficients actually used on the device */
int mb200_sketch_coeffs(const mb200_sketch* s, uint64_t* lo, uint64_t* hi);
/* CountSketch::serialize (sketch.cpp:195-211): MCSK1 bytes, byte-identical to the
 * reference.  *len receives the size; bytes are written only when cap >= *len.
 * logic_error for injected families (and for the two-for-one splitter). */
int mb200_sketch_serialize(mb200_sketch* s, uint8_t* out, uint64_t cap, uint64_t* len);
/* CountSketch::deserialize (sketch.cpp:213-244): families re-derived from the
 * stored seeds, counters uploaded to HBM; invalid_argument on malformed payloads */
int mb200_sketch_deserialize(const uint8_t* bytes, uint64_t len, mb200_sketch** out);

/* ------------------------------------------------------ multi-GPU merge --- */
/* SURVEY 8b entry 6 / 8e: the per-GPU tables of one logical sketch (item stream
 * sharded over the ranks) are summed by ONE in-place NCCL allreduce -- the
 * distributed CountSketch::merge (sketch.cpp:182-193, wrapping u64 add).
 * NCCL is bound at run time (dlopen "libnccl.so.2"; inside a process that
 * already loaded NCCL, e.g. PyTorch, that copy is used): every entry returns
 * MB200_UNSUPPORTED when no NCCL can be loaded.  A communicator is an
 * ncclComm_t passed as void*: one made here, or any ncclComm_t of the same
 * NCCL library the caller already owns. */
#define MB200_NCCL_UNIQUE_ID_BYTES 128
int mb200_nccl_version(int* version);
/* ncclGetUniqueId: rank 0 calls it and ships the bytes to the other ranks */
int mb200_nccl_unique_id(uint8_t out[MB200_NCCL_UNIQUE_ID_BYTES]);
/* ncclCommInitRank on the CURRENT device (collective: every rank calls it) */
int mb200_nccl_comm_init(int nranks, const uint8_t id[MB200_NCCL_UNIQUE_ID_BYTES], int rank,
                         void** comm);
int mb200_nccl_comm_destroy(void* comm);
int mb200_nccl_comm_size(void* comm, int* nranks);
/* In-place sum over the communicator's ranks of `count` counters (t x m of a
 * sketch), asynchronous on `stream`: every rank ends with the merged table.
 * Collective: every rank calls it with the same count. */
int mb200_cs_allreduce(int64_t* d_counters, uint64_t count, void* nccl_comm, void* stream);
/* the same on a sketch object's HBM table (its own stream; returns when the
 * merged table is in place) -- CountSketch::allreduce */
int mb200_sketch_allreduce(mb200_sketch* s, void* nccl_comm);

/* ------------------------------------------------------------- diagnostics --- */
/* Counters of the heavy-hitter Count Sketch kernels since the last reset (device-
 * wide, synchronizes the device): [0] items, [1] items that missed the shared-
 * memory hot set, [2] hot keys applied (each once per call), [3] hot keys placed in
 * the shared table, [4] row updates written to HBM bins, [5] row updates
 * that took the direct red.global path, [6] red.global merges of bin tables,
 * [7] batches binned from the raw stream (no hot pass).  L2 reductions issued =
 * rows x [2] + [5] + [6]. */
int mb200_hot_stats(uint64_t out[8], int reset);
/* Bench hook: while enabled, every large-table Count Sketch call records CUDA
 * events around its dominant scatter kernel (cs_hot / cs_private /
 * cs_private89) on the stream it runs on; _read synchronizes on them, returns
 * the summed kernel time and the number of launches, and starts a new period.
 * Enabling also starts a new period. */
int mb200_kernel_timer(int enable);
int mb200_kernel_timer_read(double* total_ms, uint64_t* launches);
/* Strategy for Count Sketch tables larger than shared memory (all exact):
 * MB200_LARGE_DIRECT (default) sends hot-set misses straight to L2 reductions;
 * MB200_LARGE_BINNED routes them through HBM bins summed in shared memory;
 * MB200_LARGE_ROWS leaves them in an HBM miss buffer that row passes (one CTA =
 * one whole row of <= 2^16 cells in shared memory) sum per row.
 * *previous (if not NULL) receives the strategy in force before the call.
 * MB200_INVALID_ARGUMENT for an unknown strategy. */
#define MB200_LARGE_DIRECT 0
#define MB200_LARGE_BINNED 1
#define MB200_LARGE_ROWS 2
int mb200_set_large_table_strategy(int strategy, int* previous);
#ifdef __cplusplus
}
#endif
#endif
