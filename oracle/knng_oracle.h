/* TEST INFRASTRUCTURE ONLY — the CPU checker, never linked into the product.
 *
 * Plain-C restatement of the reference NN-Descent path
 * (the headers under /root/reference/proj/include/knng/).  Every entry point mirrors the
 * extern "C" harness of the reference itself (oracle/ref_harness.cpp,
 * prefix ref_) with the same signature, so tests can run both on the same
 * inputs and demand bit-identical results.  Parity is PINNED: see
 * tests/test_oracle_pins.py (restatement == reference harness, bit for bit,
 * on whole runs, single join steps, selection, init, reorder, brute force)
 * and tests/golden/ (fixtures written by the reference harness).
 *
 * Return codes: 0 ok, 1 invalid argument (the reference's
 * std::invalid_argument), 2 other failure; message via oracle_last_error().
 */
#ifndef KNNG_ORACLE_H
#define KNNG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* oracle_last_error(void);

int oracle_run(const float* data, uint32_t n, uint32_t d, uint32_t k, uint32_t cap,
               double delta, uint32_t max_iterations, int reorder, uint32_t reorder_after,
               uint64_t seed, uint32_t* out_ids, float* out_dists, uint8_t* out_flags,
               uint64_t* iter_evals, uint64_t* iter_changes, double* iter_wall,
               uint32_t* n_rows, double* total_wall, uint32_t* sigma);

int oracle_capture_step(const float* data, uint32_t n, uint32_t d, uint32_t k, uint32_t cap,
                        uint64_t seed, uint32_t t, uint32_t* in_ids, float* in_dists,
                        uint8_t* in_flags, uint32_t* in_rev_deg, uint32_t* cand_ids,
                        uint32_t* new_counts, uint32_t* old_counts, uint32_t* out_ids,
                        float* out_dists, uint8_t* out_flags, uint32_t* out_rev_deg,
                        uint64_t* changes, uint64_t* evals);

int oracle_compute_step(const float* data, uint32_t n, uint32_t d, uint32_t k, uint32_t cap,
                        const uint32_t* in_ids, const float* in_dists, const uint8_t* in_flags,
                        const uint32_t* cand_ids, const uint32_t* new_counts,
                        const uint32_t* old_counts, int flat, uint32_t* out_ids,
                        float* out_dists, uint8_t* out_flags, uint32_t* out_rev_deg,
                        uint64_t* changes, uint64_t* evals);

int oracle_init_random(const float* data, uint32_t n, uint32_t d, uint32_t k, uint64_t seed,
                       uint32_t* out_ids, float* out_dists, uint8_t* out_flags,
                       uint32_t* out_rev_deg, uint64_t* evals);

int oracle_select_turbo(uint32_t n, uint32_t k, uint32_t cap, const uint32_t* in_ids,
                        const float* in_dists, const uint8_t* in_flags, uint64_t seed,
                        uint32_t* cand_ids, uint32_t* new_counts, uint32_t* old_counts,
                        uint8_t* out_flags_after_consume);

int oracle_brute_force(const float* data, uint32_t n, uint32_t d, uint32_t k,
                       uint32_t* out_ids, double* out_dists);

int oracle_recall(uint32_t n, uint32_t k, const uint32_t* approx_ids, const float* approx_dists,
                  const uint32_t* exact_ids, double* out);

int oracle_greedy_cluster(uint32_t n, uint32_t k, const uint32_t* ids, const float* dists,
                          const uint8_t* flags, uint32_t* sigma, uint32_t* sigma_inv);

float oracle_l2_sq(const float* a, const float* b, uint32_t d);
int oracle_block_l2_sq(const float* rows_a, uint32_t na, const float* rows_b, uint32_t nb,
                       uint32_t d, float* out);
int oracle_mutual_block(const float* rows, uint32_t m, uint32_t d, float* out_matrix,
                        uint32_t* visit_pairs, uint64_t* n_visits);

void oracle_mt64_stream(uint64_t seed, uint64_t* out, uint32_t count);

#ifdef __cplusplus
}
#endif
#endif
