/*
 * oracle.h -- CPU restatement of the reference hashing / sketching path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2008_08654_b200/)
 * links, loads or calls this library.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may use it, and only as
 * the checker or the timed CPU baseline, never as the thing measured on GPU.
 *
 * Parity pin: every function below restates a reference routine (file:line
 * under /root/reference/proj) and is checked in tests/test_oracle.py against
 * (a) the known-answer values frozen in the reference's own unit tests and
 * (b) the JSON fixtures in tests/golden/, produced by executing the reference itself
 * (oracle/_ref/libmersenne_ref.so, built from the reference sources by
 * oracle/Makefile; generator: tests/golden/make_golden.py).
 *
 * Conventions: u128 values cross the ABI as (lo, hi) u64 pairs.
 */
#ifndef MERSENNE_ORACLE_H
#define MERSENNE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- prng.hpp:10-38 ---------------------------------------------------- */
uint64_t orc_splitmix_next(uint64_t* state);
uint64_t orc_splitmix_below(uint64_t* state, uint64_t bound);
/* value of the i-th next() (0-based) of SplitMix64(seed): counter form */
uint64_t orc_splitmix_at(uint64_t seed, uint64_t i);

/* ---- polyhash.cpp:12-35 (draw_residue + seeded ctor) ------------------- */
/* k coefficients a_0..a_{k-1} of PolyHashFamily(MersenneModulus(b), k, u, seed) */
void orc_draw_coeffs(unsigned b, unsigned k, uint64_t seed, uint64_t* lo, uint64_t* hi);
/* sketch.cpp:72-77: row seeds are successive next() of SplitMix64(master) */
void orc_row_seeds(uint64_t master, unsigned rows, uint64_t* out);

/* ---- polyhash.cpp:59-89 (Alg 1) ---------------------------------------- */
/* returns 0 on success, 1 if the key is outside [0, 2^key_bits) (domain_error),
 * 2 if the Horner invariant y < 2p (polyhash.cpp:71,87 asserts) fails.
 * finish: 0 = ConditionalSubtract, 1 = BranchFree. b in [2,127]. */
int orc_hash(unsigned b, const uint64_t* clo, const uint64_t* chi, unsigned k, unsigned key_bits,
             uint64_t x_lo, uint64_t x_hi, int finish, uint64_t* out_lo, uint64_t* out_hi);
/* batched native/generic Alg 1 over u64 keys (x < 2^key_bits); OpenMP.
 * returns number of keys rejected (outputs for them are left 0). */
uint64_t orc_hash_batch(unsigned b, const uint64_t* clo, const uint64_t* chi, unsigned k,
                        unsigned key_bits, const uint64_t* keys, uint64_t n, uint64_t* out_lo,
                        uint64_t* out_hi);
/* config-2 restatement: Horner over keys in [0, 2^64) for b <= 61 with a
 * FULL reduction per step through Alg 3 (mersenne_divmod, field.cpp:208-222).  Keys are
 * first reduced mod p through Alg 3 as well.  OpenMP. */
void orc_hash_full_batch(unsigned b, const uint64_t* coeffs, unsigned k, const uint64_t* keys,
                         uint64_t n, uint64_t* out);

/* ---- field.cpp:208-222 (Alg 3) ----------------------------------------- */
/* returns 0, or 1 if v >= 2^(2b) (domain_error).  b <= 64 (v fits u128). */
int orc_mersenne_divmod(unsigned b, uint64_t v_lo, uint64_t v_hi, uint64_t* q_lo, uint64_t* q_hi,
                        uint64_t* r_lo, uint64_t* r_hi);
/* field.hpp:66-73: (y & p) + (y >> b) */
void orc_mersenne_reduce_partial(unsigned b, uint64_t y_lo, uint64_t y_hi, uint64_t* lo,
                                 uint64_t* hi);

/* ---- field.cpp:158-193, 224-273 (Alg 4 / Alg 5) ------------------------ */
/* PseudoMersenneModulus(b, c, m_iters): returns chosen m, max_input as 4 limbs.
 * returns 0 on error (invalid_argument). c < 2^64 here. */
unsigned orc_pm_setup(unsigned b, uint64_t c, unsigned m_iters, uint64_t max_input[4]);
/* pseudo_mersenne_div + pseudo_mersenne_mod for u128 inputs; returns 1 if
 * v > max_input (domain_error).  q, r as u128 pairs. */
int orc_pm_divmod(unsigned b, uint64_t c, unsigned m, const uint64_t max_input[4], uint64_t v_lo,
                  uint64_t v_hi, uint64_t* q_lo, uint64_t* q_hi, uint64_t* r_lo, uint64_t* r_hi);
/* div_unchecked with an explicit iteration count (field.cpp:246-258) */
void orc_pm_div_iters(unsigned b, uint64_t c, unsigned iters, uint64_t v_lo, uint64_t v_hi,
                      uint64_t* q_lo, uint64_t* q_hi);
/* batch over interleaved (lo,hi) inputs, b <= 64 so q and r fit u64; OpenMP.
 * returns number of domain rejections. */
uint64_t orc_pm_divmod_batch(unsigned b, uint64_t c, unsigned m, const uint64_t max_input[4],
                             const uint64_t* v, uint64_t n, uint64_t* q, uint64_t* r);
/* field.cpp:275-311 (Alg 8, cascade baseline) for u128 inputs */
void orc_cch_divmod(unsigned b, uint64_t c, uint64_t v_lo, uint64_t v_hi, uint64_t* q_lo,
                    uint64_t* q_hi, uint64_t* r_lo, uint64_t* r_hi);

/* ---- sketch.cpp:13-34 (Alg 2 and the arbitrary-width splitters) -------- */
void orc_split_pow2(uint64_t h_lo, uint64_t h_hi, unsigned b, unsigned l, uint64_t* index,
                    int* sign);
void orc_split_arb_uniform(uint64_t h_lo, uint64_t h_hi, unsigned b, uint64_t r, uint64_t* index,
                           int* sign);
void orc_split_arb_mersenne(uint64_t h_lo, uint64_t h_hi, unsigned b, uint64_t r,
                            uint64_t* index, int* sign);

/* ---- bucketing.cpp:61-95 (bucket maps) ---------------------------------- */
/* ExactDivisionMap ctor: smallest m with (p-1) r <= max_input(b, c, m); 0 if r not in [1, p] */
unsigned orc_exact_div_iterations(unsigned b, uint64_t c, uint64_t r);
/* kind 0 map_pow2, 1 map_mersenne, 2 ExactDivisionMap (c, m used only by kind 2) */
uint64_t orc_bucket_map(int kind, unsigned b, uint64_t c, unsigned m, uint64_t r, uint64_t v);
void orc_bucket_map_batch(int kind, unsigned b, uint64_t c, unsigned m, uint64_t r,
                          const uint64_t* v, uint64_t n, uint64_t* out);

/* ---- sketch.cpp:133-168, 182-193 (Count Sketch) ------------------------ */
/* splitter: 0 Pow2, 1 UniformArb, 2 MersenneArb, 3 TwoForOne (one family per two rows,
 * SURVEY 7.4 bit layout: row j takes index bits [l j, l j + l) and sign bit b-1-j).
 * coeffs: rows_families x k (lo/hi).  keys < 2^key_bits (returns rejected count, all-
 * or-nothing: on rejection nothing is applied).  weights: NULL (+1), i32 or i64.
 * Counters row-major [row*width+index], wrapping u64 adds.  OpenMP sharded + merged. */
uint64_t orc_cs_process(unsigned rows, uint64_t width, unsigned b, unsigned k,
                        const uint64_t* clo, const uint64_t* chi, unsigned key_bits,
                        int splitter, const uint64_t* keys64, const uint32_t* keys32,
                        const int32_t* w32, const int64_t* w64, uint64_t n, int64_t* counters);
/* row_second_moment: u128 sum of squares + saturation flag */
void orc_cs_row_moment(const int64_t* counters, uint64_t width, uint64_t* lo, uint64_t* hi,
                       int* saturated);
/* second_moment(median_rows): lower median over rows (sketch.cpp:160-168) */
void orc_cs_second_moment(const int64_t* counters, unsigned rows, uint64_t width, int median,
                          uint64_t* lo, uint64_t* hi, int* saturated);
/* point_query (sketch.cpp:170-180) for a batch of keys */
uint64_t orc_cs_point_query(unsigned rows, uint64_t width, unsigned b, unsigned k,
                            const uint64_t* clo, const uint64_t* chi, unsigned key_bits,
                            int splitter, const int64_t* counters, const uint64_t* keys,
                            uint64_t n, int64_t* out);
/* merge: dst += src, wrapping */
void orc_cs_merge(int64_t* dst, const int64_t* src, uint64_t count);
/* exact enumeration over all p^k coefficient vectors of a one-row sketch
 * (width <= 64): sum of F2 estimates and of point-query estimates at qkey
 * (test_sketch.cpp:119-178) */
void orc_enum_sums(unsigned b, unsigned k, unsigned key_bits, uint64_t width, int splitter,
                   const uint64_t* keys, const int64_t* deltas, uint64_t n, uint64_t qkey,
                   uint64_t* sum_f2, int64_t* sum_pq);
/* verify.cpp:505-603 enum_moment_sums: sum over Z_p^4 (p = 2^b - 1) of X = sum c^2
 * and X^2 for a one-row sketch (splitter 0 Pow2 with l = log2 r, 1 UniformArb,
 * 2 MersenneArb).  out: sum_x lo/hi, sum_x_sq lo/hi. */
void orc_enum_moment_sums(unsigned b, uint64_t buckets, int splitter, const uint64_t* keys,
                          const int64_t* deltas, uint64_t n, uint64_t out[4]);

/* ---- synthetic workload generators ---------------- */
void orc_gen_u32_keys(uint64_t key_seed, uint64_t start, uint64_t n, uint32_t* out);
void orc_gen_u64_keys(uint64_t key_seed, uint64_t start, uint64_t n, uint64_t* out);
/* below(p) stream for p = 2^61-1: next()>>3; returns count of rejections seen (must be 0) */
uint64_t orc_gen_below_p61(uint64_t key_seed, uint64_t start, uint64_t n, uint64_t* out);
/* u128 uniform in [0, p^2) for p = 2^64 - c: hi = next_{2i}, lo = next_{2i+1};
 * returns count of values >= p^2 (must be 0); out interleaved (lo,hi). */
uint64_t orc_gen_pm_inputs(uint64_t key_seed, uint64_t c, uint64_t start, uint64_t n,
                           uint64_t* out);
/* Zipf head table: cdf[r-1] for ranks r = 1..T over a 2^64 fixed-point scale, plus the
 * tail constant; alpha must be 1.2 (tail exponent 1/(alpha-1) = 5). */
void orc_zipf_table(double alpha, uint32_t T, double universe, uint64_t* cdf, double* tail_c1);
void orc_gen_zipf_items(uint64_t master_seed, const uint64_t* cdf, uint32_t T, double tail_c1,
                        double universe, uint64_t start, uint64_t n, uint32_t* keys,
                        int32_t* weights);
uint32_t orc_feistel32(uint64_t key, uint32_t x);

#ifdef __cplusplus
}
#endif
#endif
