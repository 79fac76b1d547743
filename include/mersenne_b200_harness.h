/*
 * mersenne_b200_harness.h -- bench / test harness of the B200 path
 * (libmersenne_b200_harness.so).  NOT part of the drop-in boundary: the
 * reference has no counterpart to these entries.  They generate the seeded
 * synthetic inputs of BASELINE.json's configs directly in HBM (DESIGN.md
 * "Inputs") and measure the roofline denominators MEASURED_PEAKS.json lacks.
 * Status codes and the error message (mb200_last_error) are those of
 * <mersenne_b200.h>.
 */
#ifndef MERSENNE_B200_HARNESS_H
#define MERSENNE_B200_HARNESS_H

#include "mersenne_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------- workload generators (counter-form SplitMix64) --- */
/* i-th output of SplitMix64(seed) (prng.hpp:14-19) for i in [start, start+n) */
int mb200_gen_u32_keys(uint64_t seed, uint64_t start, uint64_t n, uint32_t* d_out, void* stream);
int mb200_gen_u64_keys(uint64_t seed, uint64_t start, uint64_t n, uint64_t* d_out, void* stream);
/* config 2 keys: below(p) for p = 2^61 - 1; rejections counted into *d_bad */
int mb200_gen_below_p61(uint64_t seed, uint64_t start, uint64_t n, uint64_t* d_out,
                        uint64_t* d_bad, void* stream);
/* config 3 inputs: u128 uniform in [0, (2^64-c)^2) as (lo, hi) pairs */
int mb200_gen_pm_inputs(uint64_t seed, uint64_t c, uint64_t start, uint64_t n, uint64_t* d_out,
                        uint64_t* d_bad, void* stream);
/* config 5 stream: Zipf(1.2) head CDF (host) and items (keys + i32 deltas) */
int mb200_zipf_table(double alpha, uint32_t T, double universe, uint64_t* h_cdf, double* tail_c1);
int mb200_gen_zipf_items(uint64_t master_seed, const uint64_t* d_cdf, uint32_t T, double tail_c1,
                         double universe, uint64_t start, uint64_t n, uint32_t* d_keys,
                         int32_t* d_weights, void* stream);

/* ------------------------------------------------------------- probes --- */
/* blocks x threads threads each issue 8 x iters independent mad.wide.u32 */
int mb200_probe_imad(int blocks, int threads, int iters, uint64_t* d_sink, void* stream);
int mb200_probe_atomics(int mode, int blocks, int threads, int iters, uint64_t* d_buf,
                        uint64_t span, void* stream);
/* cluster-of-`cluster` CTAs each owning `words` u32 cells in shared memory:
 * mode 0 random remote-or-local red.shared::cluster, 1 local only, 2 one hot cell */
int mb200_probe_dsmem(int cluster, int mode, int blocks, int threads, int iters, uint32_t words,
                      uint64_t* d_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif
