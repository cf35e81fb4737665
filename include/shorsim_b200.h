/* shorsim_b200 — B200-native iterative-Shor engine, C ABI (the drop-in boundary).
 *
 * Replaces the reference's C++ class API for the hot path:
 *   shorsim::IterativeShorEngine      /root/reference/proj/include/shorsim/statevector.hpp:169-191
 *   shorsim::run_iterative_shor       .../statevector.hpp:164-165
 *   per-gate step/measure API         .../statevector.hpp:68-133 (init_state, apply_oracle,
 *                                     apply_phase, apply_hadamard_top, measure_top, reset_top)
 *   build_permutation_plan (gather)   .../statevector.hpp:88, proj/src/statevector.cpp:133-154
 * The C++ wrapper include/shorsim_b200.hpp re-exposes these with the reference's
 * names and exception types; INTEGRATION.md shows how the reference's callers
 * (proj/src/harness.cpp:121-133, :504-506) bind to it.
 *
 * Conventions: plain pointers and sizes only; no callbacks; no allocation
 * crosses the boundary (caller owns every output buffer); u128 bit strings
 * travel as two u64 words {lo, hi}. An engine is not thread-safe (as the
 * reference's is not: its buffers are mutable); use one engine per thread.
 *
 * Status codes (mirror proj/include/shorsim/errors.hpp:8-43):
 *   0 ok                    1 Error (norm drift > 1e-9, statevector.cpp:374-375)
 *   2 ConfigError           3 CeilingExceededError (statevector.cpp:291-294)
 *   4 DegenerateBranchError 5 BudgetExceededError
 *   6 NotInvertibleError    (the gcd is reported in shs_last_error())
 *   7 std::invalid_argument (layout / argument validation, statevector.cpp:65-72)
 *   8 CUDA error / no device (the engine never falls back to the CPU)
 *   9 FactorizationTimeoutError (Pollard rho budget, numtheory.cpp:137, 149)
 */
#ifndef SHORSIM_B200_H
#define SHORSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SHS_OK 0
#define SHS_ERROR 1
#define SHS_CONFIG_ERROR 2
#define SHS_CEILING_EXCEEDED 3
#define SHS_DEGENERATE_BRANCH 4
#define SHS_BUDGET_EXCEEDED 5
#define SHS_NOT_INVERTIBLE 6
#define SHS_INVALID_ARGUMENT 7
#define SHS_CUDA_ERROR 8
#define SHS_FACTORIZATION_TIMEOUT 9 /* FactorizationTimeoutError (numtheory.cpp:137, 149) */

/* ErrorKind order of proj/include/shorsim/noise.hpp:13-20 */
#define SHS_ERR_NONE 0
#define SHS_ERR_AMPLITUDE_INIT 1
#define SHS_ERR_PHASE_INIT 2
#define SHS_ERR_CLASSICAL_MEASURE 3
#define SHS_ERR_QUANTUM_MEASURE 4
#define SHS_ERR_BITFLIP 5

/* How p0/p1 are combined from the fixed 256-amplitude block partials
 * (proj/src/statevector.cpp:16-40). KAHAN reproduces the reference's
 * sequential compensated sum bit-for-bit; EXACT is the correctly rounded sum
 * of the same partials (deterministic, shard-count independent, within 1 ulp
 * of KAHAN). AUTO = KAHAN while the block count is small, EXACT beyond. */
#define SHS_COMBINE_AUTO 0
#define SHS_COMBINE_KAHAN 1
#define SHS_COMBINE_EXACT 2

/* Permutation kernel selection. AUTO tiles every non-identity stage whose
 * multiplier admits balanced rows once N >= 2^20; FORCE tiles whenever a plan
 * exists (tests use it at small N); OFF always uses the direct gather. */
#define SHS_TILING_AUTO 0
#define SHS_TILING_FORCE 1
#define SHS_TILING_OFF 2

/* FactoringProblem, proj/include/shorsim/problems.hpp:15-25 (p, q ride along
 * for verification only and are not needed by the engine) */
typedef struct {
    uint64_t N;
    uint64_t a;
    uint32_t L; /* bit length of N; the engine keeps y < min(N, 2^L) */
    uint32_t t; /* stages / classical bits */
    uint64_t seed;
} shs_problem;

/* ErrorConfig, proj/include/shorsim/noise.hpp:29-37 */
typedef struct {
    int32_t kind;
    double delta;
    double px, py, pz;
    int32_t has_pauli; /* PauliProbs present (quantum_measure only) */
} shs_error;

/* SimulatorOptions, proj/include/shorsim/statevector.hpp:154-159, plus the
 * device-side knobs. shard_count / workers are validated exactly as the
 * reference validates them but do not change results (as in the reference). */
typedef struct {
    uint32_t shard_count;   /* reference default 4 */
    uint32_t workers;       /* reference default 1 (unused: the GPU grid replaces threads) */
    uint32_t qubit_ceiling; /* reference default 26 */
    int32_t check_norms;    /* reference default true */
    int32_t device;         /* CUDA device ordinal */
    int32_t combine;        /* SHS_COMBINE_* */
    int32_t tiling;         /* SHS_TILING_*: sorted-residue tiles for the permutation */
    /* Multi-GPU: 0 = one device (`device`); >= 2 = the state is
     * block-sharded over devices[0..n_devices) (NULL: device, device+1, ...; a
     * device may repeat: virtual shards); < 0 = AUTO: one device while the state
     * (32 B per amplitude) fits it, else as many as needed (the SHS_DEVICES
     * environment variable, e.g. "0,1,2,3", overrides AUTO). `combine` applies
     * to the global block partials exactly as on one device. */
    int32_t n_devices;
    const int32_t* devices;
} shs_options;

/* StageTrace, proj/include/shorsim/statevector.hpp:135-141 */
typedef struct {
    uint32_t cbit;
    double p1;
    int32_t sampled_bit;
    int32_t observed_bit;
    uint8_t classical_flip;
    uint8_t quantum_error_branch;
} shs_stage_trace;

typedef struct shs_engine shs_engine;

/* Library defaults (SimulatorOptions{4, 1, 26, true} on device 0, AUTO, AUTO, one device). */
void shs_default_options(shs_options* out);

/* IterativeShorEngine::IterativeShorEngine, statevector.cpp:285-321. */
int shs_engine_create(const shs_problem* problem, const shs_error* error,
                      const shs_options* options, shs_engine** out);
void shs_engine_destroy(shs_engine* engine);

/* IterativeShorEngine::run, statevector.cpp:323-412. j / j_sampled = {lo, hi};
 * trace may be NULL, else t entries. */
int shs_engine_run(shs_engine* engine, uint64_t seed, uint64_t bitstring_index, uint64_t j[2],
                   uint64_t j_sampled[2], shs_stage_trace* trace);

/* count consecutive runs idx0 .. idx0+count-1; j receives 2*count words. Small
 * problems (N <= 4096, t <= 20: configs 1-2) run whole runs on the device, one
 * CTA per run (batch.cuh); mid-size ones (N <= 2^22) advance the shots stage by
 * stage together (lockstep.cuh); larger ones run one after another. Identical
 * results. */
int shs_engine_run_batch(shs_engine* engine, uint64_t seed, uint64_t idx0, uint32_t count,
                         uint64_t* j);
/* as run_batch, with optional per-run outputs (NULL to skip): j_sampled [2*count],
 * p1 [count*t], bits [count*t*4] = sampled, observed, classical_flip, error_branch */
int shs_engine_run_many(shs_engine* engine, uint64_t seed, uint64_t idx0, uint32_t count,
                        uint64_t* j, uint64_t* j_sampled, double* p1, int32_t* bits);
/* 1 when run_batch / run_many use the whole-run device kernel for this problem,
 * 2 when they advance the shots in lockstep, 0 otherwise */
int shs_engine_batched(const shs_engine* engine);
/* the same runs forced through the per-stage path (for comparisons) */
int shs_engine_run_sequential(shs_engine* engine, uint64_t seed, uint64_t idx0, uint32_t count,
                              uint64_t* j);

/* IterativeShorEngine::stage_multipliers: a^(2^(t-1-s)) mod N, t entries. */
int shs_engine_stage_multipliers(const shs_engine* engine, uint64_t* out);
/* sparse prefix of runs: the first stages computed on the support of the
 * state (2^(s+1) amplitudes after stage s), bit-identical p0/p1 and bit
 * strings; on by default where it applies (N >= 2^21, support <= N / 16, the
 * orbit does not wrap). shs_engine_sparse_stages = stages it covers (0: none). */
int shs_engine_set_sparse(shs_engine* engine, int32_t enable);
uint32_t shs_engine_sparse_stages(const shs_engine* engine);
uint32_t shs_engine_stages(const shs_engine* engine);
/* orbit-compressed stages: the work register's support is always inside the
 * orbit <a> (r = ord_N(a) <= N / 2 for a semiprime), so stages with whole-band
 * tile plans can store and sweep only its r members (both measurement groups
 * written by the probs pass, no collapse pass); bit-identical p0/p1, states and
 * bit strings. On by default from N >= 2^21 (SHS_ORBIT=0 or
 * shs_engine_set_orbit(0): dense stages); toggling resets the state. shs_engine_orbit_info:
 * out[0] = r (0: off), out[1] = stages run compressed, out[2] = the first. */
int shs_engine_set_orbit(shs_engine* engine, int32_t enable);
int shs_engine_orbit_info(const shs_engine* engine, uint64_t out[3]);
/* out[s] = 1 when stage s runs compressed (t entries) */
int shs_engine_orbit_stages(const shs_engine* engine, uint8_t* out);

/* ---- step/measure API (forced measurement sequences, amplitude parity) ----
 * The engine holds the state as in the reference after init_state / reset_top:
 * g_x[y] = w_x * (sel[y] * inv), y < N (zero for N <= y < 2^L). */

/* init_state, statevector.cpp:126-131 */
int shs_state_init(shs_engine* engine);
/* Stage s gates: apply_oracle(a_pow[s]) + apply_phase(s, prefix) +
 * apply_hadamard_top + the |psi|^2 reduction (statevector.cpp:339-375).
 * Returns the group masses p0, p1 (the reference's measure_top p1). */
int shs_stage_probs(shs_engine* engine, uint32_t s, uint64_t prefix_lo, uint64_t prefix_hi,
                    double* p0, double* p1);
/* reset_top(src_group, reinit, p_source), statevector.cpp:263-283 / 384-401 */
int shs_stage_collapse(shs_engine* engine, int32_t src_group, double p_source);
/* post-Hadamard amplitudes of group x of the pending stage, y in [first, first+count),
 * interleaved (re, im) */
int shs_stage_read(shs_engine* engine, int32_t x, uint64_t first, uint64_t count,
                   double* interleaved);
/* current (post-init / post-reset) amplitudes g_x[y], interleaved (re, im) */
int shs_state_read(shs_engine* engine, int32_t x, uint64_t first, uint64_t count,
                   double* interleaved);
/* shs_state_read at arbitrary y: out[i] = g_x[idx[i]] (0 for idx[i] >= N); the
 * ShardedState::amp_xy(x, y) accessor, statevector.hpp:44, batched */
int shs_state_gather(shs_engine* engine, int32_t x, const uint64_t* idx, uint64_t count,
                     double* interleaved);
/* 256-amplitude block partials of the pending stage: out[0..nb) S0, out[nb..2nb) S1 */
int shs_stage_block_sums(shs_engine* engine, double* out);
uint64_t shs_num_blocks(const shs_engine* engine);

/* ExchangePlan::gather computed on the device: src[z] = a_inv(s) * z mod N for
 * z in [first, first+count) (identity for a_pow = 1). */
int shs_index_map(shs_engine* engine, uint32_t s, uint64_t first, uint64_t count,
                  uint64_t* src_out);

/* sample_measurement, statevector.cpp:236-256 (host-side, exported for tests):
 * out = {sampled_bit, observed_bit, error_branch, classical_flip} */
int shs_sample_measurement(double p1, uint64_t seed, uint32_t idx, uint32_t stage,
                           const shs_error* error, int32_t out[4]);

/* bitflip_bitstring with RngStream(seed, idx, 0, bitflip), statevector.cpp:404-409
 * (host-side; used by drivers that assemble runs themselves, e.g. the sharded one):
 * j = {lo, hi} updated in place */
int shs_bitflip(uint64_t j[2], uint32_t t, double delta, uint64_t seed, uint32_t idx);

/* ---- instrumentation (bench / profiling) ---- */
/* Per-kernel CUDA-event timing on the engine's stream. kind: 0 probs, 1 combine,
 * 2 collapse. Returns accumulated milliseconds and launch counts since enable. */
int shs_engine_set_timing(shs_engine* engine, int32_t enable);
int shs_engine_kernel_times(const shs_engine* engine, double ms[3], uint64_t launches[3]);
/* Tile plan of stage s: out = {tiled, H, u, v, du, dv}; tiled = 0 means the
 * stage runs the direct-gather kernels (identity, first stage, small N, or a
 * multiplier without balanced rows). */
int shs_stage_tile_plan(const shs_engine* engine, uint32_t s, uint64_t out[6]);
/* cudaStream_t the engine launches on (as void*) */
void* shs_engine_stream(const shs_engine* engine);
/* total kernels launched by this engine since creation */
uint64_t shs_engine_launch_count(const shs_engine* engine);
/* bytes of device memory the engine holds */
uint64_t shs_engine_device_bytes(const shs_engine* engine);
/* devices the engine's state lives on (several when sharded): writes up to max
 * ordinals, returns their count */
int shs_engine_devices(const shs_engine* engine, int32_t* out, int32_t max);

/* ---- sharded engine (one shard of the state per GPU; §8e) ----------------
 * Shard q of G owns global amplitude indices [q*S, min(N, (q+1)*S)), S a
 * multiple of 256. Each shard holds two buffers (sel and the exchange buffer P,
 * swapping roles every stage) and needs every other shard's buffers: attach
 * them as device pointers valid in this process (same process) or as CUDA IPC
 * handles (one process per GPU). Per stage the driver runs, on every shard:
 *   if shs_shard_needs_exchange(s): shs_shard_exchange(s); sync; barrier
 *   shs_shard_probs(s, prefix, digits); allreduce-sum digits over shards;
 *   shs_digits_to_probs(total) -> p0, p1; norm check; sample (same on all)
 *   if s + 1 < t: shs_shard_collapse(bit, p_src); sync; barrier
 * (paper_2308_05047_b200/sharded.py implements this driver for virtual shards
 * in one process and for torch.distributed ranks). Results are bit-identical
 * to the single engine with SHS_COMBINE_EXACT for every shard count. */
typedef struct shs_shard shs_shard;
#define SHS_MAX_SHARDS 16
#define SHS_DIGITS 80 /* 2 groups x 40 x 32-bit digits (in uint64 words) */
#define SHS_SHARD_IPC_BYTES 1088 /* shs_shard_ipc_handles blob */

int shs_shard_create(const shs_problem* problem, const shs_error* error,
                     const shs_options* options, uint32_t rank, uint32_t nshards,
                     shs_shard** out);
void shs_shard_destroy(shs_shard* shard);
/* out = {lo, hi, S} */
int shs_shard_range(const shs_shard* shard, uint64_t out[3]);
/* this shard's two device buffers (allocated at create) */
int shs_shard_buffers(const shs_shard* shard, void* out[2]);
/* CUDA IPC handles of this shard's buffers, stage digits and ordering events:
 * out receives SHS_SHARD_IPC_BYTES; a peer process passes them to
 * shs_shard_attach_ipc */
int shs_shard_ipc_handles(const shs_shard* shard, void* out);
/* peer buffers only (enough for the per-stage driver); cross-device pointers
 * get peer access enabled, or an error when the devices cannot reach each other */
int shs_shard_attach(shs_shard* shard, uint32_t peer, void* const bufs[2]);
int shs_shard_attach_ipc(shs_shard* shard, uint32_t peer, const void* handles);
/* a peer shard object of this process (buffers, digits, events) */
int shs_shard_attach_local(shs_shard* shard, shs_shard* peer);
/* host barrier of a one-process-per-GPU run: a POSIX shared-memory segment
 * name ("/..."), the same on every rank of the run (all ranks on one node) */
int shs_shard_set_barrier(shs_shard* shard, const char* shm_name);
/* IterativeShorEngine::run over the shards, device-resident (collective: the
 * shards of this process; with count < G every process calls it with its own
 * shards and the barrier set). Per stage: exchange, probs, the exact digit sum
 * and the measurement on every device (no host round trip), collapse; stage
 * ordering across shards by (IPC) events. trace: t entries or NULL. */
int shs_shards_run(shs_shard* const* shards, uint32_t count, uint64_t seed, uint64_t idx,
                   uint64_t j[2], uint64_t j_sampled[2], shs_stage_trace* trace);
uint64_t shs_shard_device_bytes(const shs_shard* shard);
/* the node-local host barrier shs_shard_set_barrier installs (a sense-reversing
 * counter in POSIX shared memory; it orders enqueues, never GPU work), on its
 * own: every one of `parties` processes opens the same name and arrives */
typedef struct shs_node_barrier shs_node_barrier;
int shs_node_barrier_open(const char* shm_name, uint32_t parties, int32_t unlink_at_close,
                          shs_node_barrier** out);
int shs_node_barrier_arrive(shs_node_barrier* barrier);
void shs_node_barrier_close(shs_node_barrier* barrier);
int shs_shard_init(shs_shard* shard);
int shs_shard_needs_exchange(const shs_shard* shard, uint32_t s);
int shs_shard_exchange(shs_shard* shard, uint32_t s);
int shs_shard_probs(shs_shard* shard, uint32_t s, uint64_t prefix_lo, uint64_t prefix_hi,
                    uint64_t digits[SHS_DIGITS]);
int shs_shard_collapse(shs_shard* shard, int32_t src_group, double p_source);
int shs_shard_sync(shs_shard* shard);
/* amplitudes (global indices; zero outside this shard), as shs_state_read / shs_stage_read */
int shs_shard_state_read(shs_shard* shard, int32_t x, uint64_t first, uint64_t count,
                         double* interleaved);
int shs_shard_stage_read(shs_shard* shard, int32_t x, uint64_t first, uint64_t count,
                         double* interleaved);
/* 1 when the shards combine p0/p1 like the reference (sequential Kahan over the
 * global block partials: combine = KAHAN, or AUTO with <= 1024 blocks); then,
 * once every shard's probs of the stage is done, shs_shard_kahan_probs runs that
 * combine on this shard's device over all shards' partials (peer pointers) */
int shs_shard_kahan(const shs_shard* shard);
/* sparse prefix of device-resident sharded runs (on by default where it applies,
 * as shs_engine_set_sparse): every shard runs the first stages on the support
 * redundantly and scatters its own range; results identical */
int shs_shard_set_sparse(shs_shard* shard, int32_t enable);
uint32_t shs_shard_sparse_stages(const shs_shard* shard);
int shs_shard_kahan_probs(shs_shard* shard, double* p0, double* p1);
/* correctly rounded p0, p1 from summed exact digits (host-side, no device) */
int shs_digits_to_probs(const uint64_t digits[SHS_DIGITS], double* p0, double* p1);
/* per-kernel CUDA-event times like shs_engine_kernel_times (each timed launch
 * synchronises its stream): kind 0 probs, 1 exchange (v1), 2 collapse,
 * 3 pack and 4 unpack (exchange v2, device-resident runs) */
int shs_shard_set_timing(shs_shard* shard, int32_t enable);
int shs_shard_kernel_times(const shs_shard* shard, double ms[5], uint64_t launches[5]);
uint64_t shs_shard_launch_count(const shs_shard* shard);
/* launch timeline of the next device-resident runs (no per-launch sync): after a
 * run, out[3 i .. 3 i + 2] = {kind (as shs_shard_kernel_times), start ms, end ms}
 * relative to the run's start on this shard's main stream; returns the entry
 * count (entries beyond max_entries are counted, not written) */
int shs_shard_set_timeline(shs_shard* shard, int32_t enable);
int64_t shs_shard_timeline(shs_shard* shard, double* out, uint64_t max_entries);
void* shs_shard_stream(const shs_shard* shard);

/* ---- the per-gate API on a device-resident state ----
 * shs_sv = ShardedState (statevector.hpp:33-65): 2^n complex amplitudes in
 * device memory, the top index bit selects the group (x = 0: [0, 2^(n-1)),
 * x = 1: [2^(n-1), 2^n)), global indices as the reference's amp()/set_amp().
 * Gates reproduce the reference's arithmetic bit for bit. */
typedef struct shs_sv shs_sv;
/* ShardedState(n, shard_count) zeroed: make_shard_layout's validation and
 * messages (statevector.cpp:65-72, invalid_argument) */
int shs_sv_create(uint32_t n, uint32_t shard_count, int32_t device, shs_sv** out);
int shs_sv_clone(const shs_sv* state, shs_sv** out); /* value copy (device to device) */
void shs_sv_destroy(shs_sv* state);
int shs_sv_layout(const shs_sv* state, uint32_t out[2]); /* {n, g}: shard_count = 2^g */
/* amp / set_amp over [first, first+count), interleaved (re, im) */
int shs_sv_read(const shs_sv* state, uint64_t first, uint64_t count, double* interleaved);
int shs_sv_write(shs_sv* state, uint64_t first, uint64_t count, const double* interleaved);
/* init_state (statevector.cpp:126-131) on this state: zero, then amp(1) = a0,
 * amp(2^(n-1) + 1) = a1; pair = {a0.re, a0.im, a1.re, a1.im} */
int shs_sv_init_state(shs_sv* state, const double pair[4]);
/* apply_oracle (statevector.cpp:223-244): group 1 gathered through
 * src[y] = a_inv y mod N for y < min(N, 2^(n-1)); NotInvertibleError as the reference */
int shs_sv_apply_oracle(shs_sv* state, uint64_t a_pow, uint64_t N);
/* apply_phase (statevector.cpp:246-253): group 1 *= e^{i pi prefix 2^-cbit}, skipped at phi = 0 */
int shs_sv_apply_phase(shs_sv* state, uint32_t cbit, uint64_t prefix_lo, uint64_t prefix_hi);
/* apply_hadamard_top (statevector.cpp:255-270) */
int shs_sv_apply_hadamard_top(shs_sv* state);
/* {group_norm_squared(0), group_norm_squared(1)} (statevector.cpp:95-117):
 * fixed 256-blocks, sequential Kahan over the non-zero blocks */
int shs_sv_group_norms(const shs_sv* state, double out[2]);
/* reset_top(bit, branch, reinit, p_source) (statevector.cpp:263-283);
 * DegenerateBranchError below 1e-300 */
int shs_sv_reset_top(shs_sv* state, int32_t bit, int32_t error_branch, const double reinit[4],
                     double p_source);
uint64_t shs_sv_launch_count(const shs_sv* state);

/* build_permutation_plan (statevector.cpp:133-154) on the device: a_inv,
 * identity, y_limit = min(N, 2^(n-1)); gather[y_limit] (NULL to skip) and
 * pair_counts[(2^(g-1))^2] row-major [src_xrank][dst_xrank] (NULL to skip) */
int shs_plan_build(uint64_t a_pow, uint64_t N, uint32_t n, uint32_t shard_count, int32_t device,
                   uint64_t* a_inv, int32_t* identity, uint64_t* y_limit, uint64_t* gather,
                   uint64_t* pair_counts);
/* plan_receive_lists (send = 0) / plan_send_lists (send = 1) for group shard
 * xrank (statevector.cpp:156-181): counts[2^(g-1)] per peer, indices = the
 * local indices grouped by ascending peer, each group in the reference's
 * order (indices needs 2^(n-g) entries) */
int shs_plan_lists(uint64_t a_pow, uint64_t N, uint32_t n, uint32_t shard_count, uint32_t xrank,
                   int32_t send, int32_t device, uint64_t* counts, uint64_t* indices);

/* ---- exhaustive_joint_distribution (statevector.hpp:193-198, statevector.cpp:533-579) ----
 * Exact distribution over the 2^t observed bit strings by enumerating every
 * measurement path on the device, error branches marginalised; out receives
 * 2^t doubles. Same limits and errors as the reference (t <= 14 and n <= 12,
 * else SHS_BUDGET_EXCEEDED; node budget, default 2^22) and bit-identical output. */
int shs_exhaustive_distribution(const shs_problem* problem, const shs_error* error,
                                uint64_t node_budget, int32_t device, double* out);

/* ---- Shor standard post-processing on the device (proj/src/postprocess.cpp:55-89) ----
 * shor_standard_procedure(j, t, N, a, known_order) for a batch of bit strings
 * (u128 j as {lo, hi} pairs), one device thread each. classification follows
 * shorsim::Classification (postprocess.hpp:12); order_match: 0/1, or 2 when no
 * known order is given (std::nullopt). Errors as the reference: t >= 128 or
 * j >= 2^t -> SHS_INVALID_ARGUMENT (numtheory.cpp:237-239). */
enum { SHS_CLASS_SUCCESS = 0, SHS_CLASS_LUCKY_NE = 1, SHS_CLASS_LUCKY_NO = 2,
       SHS_CLASS_LUCKY_OO = 3, SHS_CLASS_FAIL = 4 };
typedef struct {
    int32_t classification;
    uint8_t r_even, a_r_is_one, a_half_not_minus_one, order_match;
    uint64_t k[2], r[2];        /* the convergent k / r used (u128 as {lo, hi}) */
    uint32_t n_factors;         /* nontrivial divisors found, ascending */
    uint32_t pad;
    uint64_t factors[4];
} shs_shor_outcome;
int shs_shor_postprocess(const uint64_t* j, uint32_t count, uint32_t t, uint64_t N, uint64_t a,
                         uint64_t known_order, int32_t has_known_order, int32_t device,
                         shs_shor_outcome* out);

/* ---- Ekerå post-processing on the device (proj/src/postprocess.cpp:92-171) ----
 * ekera_postprocess(j, t, N, a, params, RngStream(seed, idx0 + i, 1, postprocess),
 * known_order) for a batch of bit strings; params as EkeraParams
 * (postprocess.hpp:43-53; for_problem(L, t) = {B = L, c = 1, k = 100,
 * varsigma = 1, m = L, ell = t - L}). */
typedef struct {
    uint64_t B, c;
    uint32_t k, varsigma, m, ell;
    uint64_t rho_budget; /* factorize()'s Pollard-rho step budget in recover_order
                            (0: the reference's default 10^7) */
} shs_ekera_params;
typedef struct {
    int32_t classification;     /* SHS_CLASS_SUCCESS or SHS_CLASS_FAIL */
    uint8_t order_match;        /* 0/1, 2 = no known order */
    uint8_t has_recovered_order, has_offset;
    uint8_t timeout;            /* recover_order's factorize ran out of its rho budget */
    uint64_t k[2], r[2];        /* extract_denominator(j) */
    uint64_t recovered_order;
    int64_t candidate_offset;   /* the j' = j + offset that factored N */
    uint32_t n_factors, pad2;
    uint64_t factors[4];
} shs_ekera_outcome;
int shs_ekera_postprocess(const uint64_t* j, uint32_t count, uint32_t t, uint64_t N, uint64_t a,
                          const shs_ekera_params* params, uint64_t seed, uint64_t idx0,
                          uint64_t known_order, int32_t has_known_order, int32_t device,
                          shs_ekera_outcome* out);

/* factorize (numtheory.cpp:170-187) on the device: sorted prime powers of n
 * (primes / exponents need 64 entries); SHS_FACTORIZATION_TIMEOUT when the
 * Pollard-rho steps exceed rho_budget (0: 10^7), as the reference throws */
int shs_factorize(uint64_t n, uint64_t rho_budget, int32_t device, uint64_t* primes,
                  uint32_t* exponents, uint32_t* count);

/* thread-local message of the last failing call */
const char* shs_last_error(void);
/* library build string (arch, flags) */
const char* shs_build_info(void);

#ifdef __cplusplus
}
#endif
#endif
