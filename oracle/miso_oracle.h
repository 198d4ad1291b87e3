/*
 * miso_oracle.h -- CPU restatement of the MISO decision core (TEST INFRASTRUCTURE ONLY).
 *
 * This is the parity checker for the CUDA path, not part of the product. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load it.
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj/include/miso/). Parity is pinned by tests/golden/ fixtures that were
 * produced by the reference itself (oracle/_ref, built from the reference headers by
 * oracle/Makefile) and by the reference's own known-answer tests.
 *
 * Build: gcc -O2 -ffp-contract=off (no FMA contraction: the reference is plain SSE2 FP64).
 */
#ifndef MISO_ORACLE_H
#define MISO_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- common.hpp:70-119 -------------------------------------------------- */
typedef struct {
  uint64_t mt[312];
  int mti;
} orc_rng;

uint64_t orc_splitmix64(uint64_t x);                         /* common.hpp:70-75 */
uint64_t orc_mix_seed(uint64_t seed, uint64_t tag);          /* common.hpp:77-79 */
void orc_rng_seed(orc_rng* r, uint64_t seed);                /* std::mt19937_64(seed) */
uint64_t orc_rng_raw(orc_rng* r);                            /* eng_() */
double orc_uniform01(orc_rng* r);                            /* common.hpp:90 */
double orc_uniform(orc_rng* r, double lo, double hi);        /* common.hpp:93 */
double orc_exponential(orc_rng* r, double mean);             /* common.hpp:96-99 */
double orc_normal01(orc_rng* r);                             /* common.hpp:103-108 */
double orc_lognormal(orc_rng* r, double mu, double sigma);   /* common.hpp:110 */
int orc_index(orc_rng* r, int n);                            /* common.hpp:113 */

/* ---- topology.hpp ------------------------------------------------------- */
#define ORC_KINDS 5
#define ORC_MAX_ENTRIES 36
#define ORC_MAX_CANDS 111

typedef struct {
  int n_entries;
  uint8_t counts[ORC_MAX_ENTRIES][ORC_KINDS]; /* catalog_order-sorted (topology.hpp:178-180) */
} orc_catalog;

/* Candidate = (entry, distinct permutation). Sorted by (m, OptKey rank). */
typedef struct {
  int n;
  int base[9];                          /* candidates of size m: [base[m], base[m+1]) */
  uint8_t entry[ORC_MAX_CANDS];         /* index into the default catalog */
  uint8_t m[ORC_MAX_CANDS];
  uint8_t place[ORC_MAX_CANDS][7];      /* slice kind index per job */
} orc_candidates;

extern const int orc_gpc[ORC_KINDS];      /* topology.hpp:39-45 */
extern const int orc_mem_gb[ORC_KINDS];
extern const int orc_units[ORC_KINDS];
extern const int orc_max_count[ORC_KINDS];

int orc_violation(const uint8_t counts[ORC_KINDS]);           /* topology.hpp:84-101, 0 = ok */
void orc_build_catalog(orc_catalog* cat);                      /* topology.hpp:189-202 */
void orc_build_candidates(orc_candidates* out);                /* optimizer.hpp:46-51 ranks */
int orc_min_slice_for(int mem_gb, int qos_min_gpc);            /* topology.hpp:68-72, -1 none */
int orc_max_spare_slice_for(const orc_catalog* cat, const int* min_kinds, int m); /* :227-252 */
/* LUT over sorted multisets of <=6 min kinds (462 keys). key = orc_spare_key(). */
int orc_spare_key(const int* min_kinds, int m);
void orc_build_spare_lut(const orc_catalog* cat, int8_t lut[462]);

/* ---- optimizer.hpp:62-115 ------------------------------------------------ */
/* speeds: m rows x 5 (kind order 1g..7g). Returns 1 feasible / 0 infeasible / -1 bad m.
 * entry = index in `cat`, place[m] = kind per job, *obj = objective. */
int orc_optimize(const orc_catalog* cat, const double* speeds, int m, int* entry, uint8_t* place,
                 double* obj);
void orc_optimize_batch(const orc_catalog* cat, const double* speeds, const uint32_t* offsets,
                        size_t n, int16_t* entry, uint8_t* place, double* obj);

/* ---- profiles.hpp -------------------------------------------------------- */
double orc_effective_speed(double speed, int kind, int mem_gb, int qos_kind); /* :60-65 */
double orc_perturb_speed(double truth, double target_mae, uint64_t entry_seed); /* :193-205 */
/* One real column of predict_mig_speeds (:214-253): in truth f7,f4,f3 -> out f7,f4,f3. */
void orc_predict_column(const double truth3[3], int col, uint64_t rng_seed, uint64_t nonce,
                        int noisy, double target_mae, double out3[3]);
/* extrapolate_small_slices (:370-384): f7,f4,f3 -> f2,f1 */
void orc_extrapolate(const double w2[4], const double w1[4], const double f[3], double* f2,
                     double* f1);
/* Full chain for a batch of columns (C3 layout): column j is column j%cpg of group j/cpg,
 * nonce = first_nonce + j/cpg. out: 5 speeds per column, kind order 1g..7g. */
void orc_predict_batch(const double* truth3, size_t ncols, int cols_per_group,
                       uint64_t first_nonce, uint64_t rng_seed, int noisy, double target_mae,
                       const double w2[4], const double w1[4], double* out5);

/* make_synthetic_profile (:443-465). speeds5 kind order 1g..7g. */
void orc_synthetic_profile(orc_rng* r, double speeds5[5], int* mem_gb, double mps3[3]);
/* fit_small_slice_model(make_training_corpus(n, seed)) (:340-361, :469-475) */
void orc_default_model(double w2[4], double w1[4]);

/* ---- generators used by the configs ------------------------------------- */
/* acceptance_test.cpp:66-85: m = 1+index(7); f4~U(.2,1) ... f1 = 0 w.p. .25 */
size_t orc_gen_mixes(uint64_t seed, size_t n, double* speeds, uint32_t* offsets,
                     size_t max_jobs);
/* C3 stream: DetRng(mix_seed(seed, 0x50)); truth3 = f7,f4,f3 per profile */
void orc_gen_profiles(uint64_t seed, size_t n, double* truth3, double* small2);

#ifdef __cplusplus
}
#endif
#endif
