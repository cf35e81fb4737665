/* TEST INFRASTRUCTURE ONLY — the CPU checker for the GPU engine.
 *
 * Plain-C restatement of the reference's iterative-Shor hot path
 * (/root/reference/proj/src/statevector.cpp:285-412 and the helpers it calls),
 * using the compressed N-amplitude representation of SURVEY.md F3 /
 * Appendix A. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library, and only as the checker. The
 * product (paper_2308_05047_b200/) never links or calls it.
 *
 * Parity pin: tests/test_oracle.py checks every function here against the
 * reference library itself (oracle/_ref, built from /root/reference by
 * oracle/Makefile) and against the golden fixtures in tests/golden/.
 *
 * Status codes are those of include/shorsim_b200.h.
 */
#ifndef SHOR_ORACLE_H
#define SHOR_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t kind; /* ErrorKind order of proj/include/shorsim/noise.hpp:13-20 */
    double delta, px, py, pz;
    int32_t has_pauli;
} so_error;

/* rng: proj/include/shorsim/rng.hpp:16-83 */
void so_philox_block(uint64_t key, const uint32_t ctr[4], uint32_t out[4]);
uint64_t so_rng_u64(uint64_t seed, uint32_t a, uint32_t b, uint32_t domain, uint32_t index);
double so_rng_double(uint64_t seed, uint32_t a, uint32_t b, uint32_t domain, uint32_t index);

/* number theory: proj/include/shorsim/int128.hpp:28-30, proj/src/numtheory.cpp:25-46 */
uint64_t so_mulmod(uint64_t a, uint64_t b, uint64_t m);
int so_mod_inverse(uint64_t a, uint64_t n, uint64_t* inv, uint64_t* gcd);
unsigned so_recommended_t(uint64_t n);
unsigned so_bit_length(uint64_t n);
/* gather[z] = a_inv * z mod N for z in [first, first+count): proj/src/statevector.cpp:148-152 */
int so_index_map(uint64_t a_pow, uint64_t n, uint64_t first, uint64_t count, uint64_t* out);

/* noise hooks: proj/src/noise.cpp:13-151 */
int so_error_validate(const so_error* e);
void so_reinit_state(const so_error* e, double out[4]);
double so_stage_phase(unsigned cbit, uint64_t prefix_lo, uint64_t prefix_hi);
/* out = {sampled_bit, observed_bit, error_branch, classical_flip} */
void so_sample_measurement(double p1, uint64_t seed, uint32_t idx, uint32_t stage, const so_error* e,
                           int32_t out[4]);
void so_bitflip(uint64_t j[2], unsigned t, double delta, uint64_t seed, uint32_t idx);

/* proj/src/statevector.cpp:32-40 */
double so_combine_blocks(const double* blocks, uint64_t count);
/* correctly rounded (nearest-even) exact sum of non-negative doubles */
double so_exact_sum(const double* values, uint64_t count);

/* engine: compressed restatement of IterativeShorEngine (Appendix A) */
typedef struct so_engine so_engine;
int so_engine_create(uint64_t N, uint64_t a, unsigned L, unsigned t, const so_error* e,
                     unsigned shard_count, unsigned qubit_ceiling, int check_norms,
                     so_engine** out);
void so_engine_destroy(so_engine* e);
int so_engine_multipliers(const so_engine* e, uint64_t* out);
/* combine_mode 0 = Kahan over blocks (reference), 1 = exact correctly-rounded sum
 * trace: p1[t]; ints[4*t] = sampled, observed, classical_flip, quantum_error_branch */
int so_engine_run(so_engine* e, uint64_t seed, uint64_t idx, int combine_mode, uint64_t j[2],
                  uint64_t js[2], double* p1, int32_t* ints);

/* step/measure API (forced sequences). State after init: e_1, inv = 1. */
int so_state_init(so_engine* e);
int so_stage_probs(so_engine* e, unsigned s, uint64_t prefix_lo, uint64_t prefix_hi,
                   int combine_mode, double* p0, double* p1);
/* post-Hadamard amplitudes of group x at the pending stage, y in [first, first+count) */
int so_stage_read(so_engine* e, int x, uint64_t first, uint64_t count, double* out);
int so_stage_collapse(so_engine* e, int src_group, double p_src);
/* materialised reference state g_x[y] = w_x * (sel[y] * inv) after a collapse/init */
int so_state_read(so_engine* e, int x, uint64_t first, uint64_t count, double* out);
/* block partial sums of the pending stage: out[0..nb) = S0, out[nb..2nb) = S1 */
int so_stage_block_sums(so_engine* e, double* out);
uint64_t so_num_blocks(const so_engine* e);

/* sparse-support engine: the same recipe on the support of the state only
 * (N beyond the dense restatement's reach, e.g. config 4). Bit-identical p0/p1
 * (both combine modes) and amplitudes to so_engine on the same forced sequence. */
typedef struct so_sparse so_sparse;
int so_sparse_create(uint64_t N, uint64_t a, unsigned L, unsigned t, const so_error* e,
                     int check_norms, so_sparse** out);
void so_sparse_destroy(so_sparse* g);
int so_sparse_init(so_sparse* g);
int so_sparse_stage_probs(so_sparse* g, unsigned s, uint64_t prefix_lo, uint64_t prefix_hi,
                          int combine_mode, double* p0, double* p1);
int so_sparse_stage_collapse(so_sparse* g, int src_group, double p_src);
uint64_t so_sparse_size(const so_sparse* g);
/* z_out[size] = sorted support (may be NULL); out[2*size] = g_x there (may be NULL) */
int so_sparse_state(const so_sparse* g, int x, uint64_t* z_out, double* out);

#ifdef __cplusplus
}
#endif
#endif
