// TEST INFRASTRUCTURE ONLY — never part of the product path.
//
// C shim over the UNMODIFIED reference library (/root/reference/proj/src/*.cpp,
// compiled out-of-tree by oracle/Makefile into oracle/_ref/libshorsim_ref.so).
// It exposes the reference's own entry points to ctypes so that tests/ and
// bench.py's reference arm can call the real reference:
//   IterativeShorEngine        proj/include/shorsim/statevector.hpp:169-191
//   per-gate step/measure API   proj/include/shorsim/statevector.hpp:68-133
//   build_permutation_plan      proj/src/statevector.cpp:133-154
//   exhaustive_joint_distribution proj/src/statevector.cpp:533-579
//   philox::block               proj/include/shorsim/rng.hpp:16-31
//   shor_standard_procedure     proj/src/postprocess.cpp:55-89
//   run_problem                 proj/src/harness.cpp:109-148
//   ekera_postprocess           proj/src/postprocess.cpp:138-171
//   multiplicative_order        proj/src/numtheory.cpp:207-234
// Nothing here re-implements reference logic; it only marshals arguments.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "shorsim/harness.hpp"
#include "shorsim/noise.hpp"
#include "shorsim/postprocess.hpp"
#include "shorsim/numtheory.hpp"
#include "shorsim/problems.hpp"
#include "shorsim/statevector.hpp"

using namespace shorsim;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

// status codes mirror include/shorsim_b200.h
template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const CeilingExceededError& e) {
        return fail(e, 3);
    } catch (const DegenerateBranchError& e) {
        return fail(e, 4);
    } catch (const BudgetExceededError& e) {
        return fail(e, 5);
    } catch (const NotInvertibleError& e) {
        return fail(e, 6);
    } catch (const ConfigError& e) {
        return fail(e, 2);
    } catch (const FactorizationTimeoutError& e) {
        return fail(e, 9);
    } catch (const Error& e) {
        return fail(e, 1);
    } catch (const std::invalid_argument& e) {
        return fail(e, 7);
    } catch (const std::exception& e) {
        return fail(e, 9);
    }
}

ErrorConfig make_error(int kind, double delta, double px, double py, double pz, int has_pauli) {
    ErrorConfig e;
    e.kind = static_cast<ErrorKind>(kind);
    e.delta = delta;
    if (has_pauli) e.pauli = PauliProbs{px, py, pz};
    return e;
}

FactoringProblem make_problem(uint64_t N, uint64_t a, unsigned L, unsigned t) {
    FactoringProblem p;
    p.N = N;
    p.a = a;
    p.L = L;
    p.t = t;
    return p;
}

struct RefEngine {
    IterativeShorEngine engine;
    unsigned t;
};

struct RefState {
    ShardedState state;
};

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_philox_block(uint64_t key, const uint32_t ctr[4], uint32_t out[4]) {
    auto r = philox::block(key, {ctr[0], ctr[1], ctr[2], ctr[3]});
    for (int i = 0; i < 4; ++i) out[i] = r[i];
}

uint64_t ref_rng_u64(uint64_t seed, uint32_t a, uint32_t b, uint32_t domain, uint32_t index) {
    RngStream s(seed, a, b, static_cast<RngDomain>(domain));
    return s.at(index);
}

unsigned ref_recommended_t(uint64_t n) { return recommended_t(n); }
unsigned ref_bit_length(uint64_t n) { return bit_length_u64(n); }

int ref_mod_inverse(uint64_t a, uint64_t n, uint64_t* out) {
    return guarded([&] { *out = mod_inverse(a, n); });
}

int ref_reinit_state(int kind, double delta, double out[4]) {
    return guarded([&] {
        ErrorConfig e = make_error(kind, delta, 0, 0, 0, 0);
        QubitPair q = reinit_state(e);
        out[0] = q.a0.real();
        out[1] = q.a0.imag();
        out[2] = q.a1.real();
        out[3] = q.a1.imag();
    });
}

double ref_stage_phase(unsigned cbit, uint64_t prefix_lo, uint64_t prefix_hi) {
    return stage_phase(cbit, (u128{prefix_hi} << 64) | prefix_lo);
}

// ExchangePlan gather table (u32, as the reference stores it) and pair counts.
int ref_permutation_plan(uint64_t a_pow, uint64_t N, unsigned n, unsigned shards, uint32_t* gather,
                         uint64_t* pair_counts, uint64_t* a_inv, int* identity) {
    return guarded([&] {
        ShardLayout layout = make_shard_layout(n, shards);
        ExchangePlan plan = build_permutation_plan(a_pow, N, layout);
        if (gather) std::memcpy(gather, plan.gather.data(), plan.gather.size() * sizeof(uint32_t));
        if (pair_counts) {
            unsigned gs = layout.group_shards();
            for (unsigned s = 0; s < gs; ++s)
                for (unsigned d = 0; d < gs; ++d) pair_counts[s * gs + d] = plan.pair_counts[s][d];
        }
        if (a_inv) *a_inv = plan.a_inv;
        if (identity) *identity = plan.identity ? 1 : 0;
    });
}

int ref_engine_create(uint64_t N, uint64_t a, unsigned L, unsigned t, int kind, double delta,
                      double px, double py, double pz, int has_pauli, unsigned shard_count,
                      unsigned workers, unsigned qubit_ceiling, int check_norms, void** out) {
    return guarded([&] {
        SimulatorOptions o;
        o.shard_count = shard_count;
        o.workers = workers;
        o.qubit_ceiling = qubit_ceiling;
        o.check_norms = check_norms != 0;
        auto* e = new RefEngine{IterativeShorEngine(make_problem(N, a, L, t),
                                                    make_error(kind, delta, px, py, pz, has_pauli), o),
                                t};
        *out = e;
    });
}

void ref_engine_destroy(void* h) { delete static_cast<RefEngine*>(h); }

int ref_engine_multipliers(void* h, uint64_t* out) {
    auto* e = static_cast<RefEngine*>(h);
    const auto& m = e->engine.stage_multipliers();
    for (size_t i = 0; i < m.size(); ++i) out[i] = m[i];
    return 0;
}

// trace layout per stage: p1 (double) in p1[s]; ints[s*4 + {0,1,2,3}] =
// sampled_bit, observed_bit, classical_flip, quantum_error_branch.
int ref_engine_run(void* h, uint64_t seed, uint64_t idx, uint64_t j[2], uint64_t js[2], double* p1,
                   int32_t* ints) {
    auto* e = static_cast<RefEngine*>(h);
    return guarded([&] {
        RunResult r = e->engine.run(seed, idx);
        j[0] = static_cast<uint64_t>(r.bits.j);
        j[1] = static_cast<uint64_t>(r.bits.j >> 64);
        js[0] = static_cast<uint64_t>(r.j_sampled);
        js[1] = static_cast<uint64_t>(r.j_sampled >> 64);
        for (size_t s = 0; s < r.trace.size(); ++s) {
            if (p1) p1[s] = r.trace[s].p1;
            if (ints) {
                ints[s * 4 + 0] = r.trace[s].sampled_bit;
                ints[s * 4 + 1] = r.trace[s].observed_bit;
                ints[s * 4 + 2] = r.trace[s].event.classical_flip ? 1 : 0;
                ints[s * 4 + 3] = r.trace[s].event.quantum_error_branch ? 1 : 0;
            }
        }
    });
}

// Wall time of `count` engine.run calls (steady_clock), for the CPU baseline.
int ref_engine_time_runs(void* h, uint64_t seed, uint64_t idx0, unsigned count, double* seconds,
                         uint64_t* last_j) {
    auto* e = static_cast<RefEngine*>(h);
    return guarded([&] {
        auto t0 = std::chrono::steady_clock::now();
        u128 j = 0;
        for (unsigned i = 0; i < count; ++i) j = e->engine.run(seed, idx0 + i).bits.j;
        auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
        if (last_j) *last_j = static_cast<uint64_t>(j);
    });
}

// ----- per-gate ("step/measure") API: proj/src/statevector.cpp:126-283 -----

int ref_state_create(unsigned n, int kind, double delta, unsigned shards, void** out) {
    return guarded([&] {
        QubitPair q = reinit_state(make_error(kind, delta, 0, 0, 0, 0));
        *out = new RefState{init_state(n, q, shards)};
    });
}

void ref_state_destroy(void* h) { delete static_cast<RefState*>(h); }

int ref_state_set_amp(void* h, uint64_t global, double re, double im) {
    return guarded([&] { static_cast<RefState*>(h)->state.set_amp(global, cplx{re, im}); });
}

int ref_apply_oracle(void* h, uint64_t a_pow, uint64_t N) {
    return guarded([&] { apply_oracle(static_cast<RefState*>(h)->state, a_pow, N); });
}

int ref_apply_phase(void* h, unsigned cbit, uint64_t prefix_lo, uint64_t prefix_hi) {
    return guarded([&] {
        apply_phase(static_cast<RefState*>(h)->state, cbit, (u128{prefix_hi} << 64) | prefix_lo);
    });
}

int ref_apply_hadamard(void* h) {
    return guarded([&] { apply_hadamard_top(static_cast<RefState*>(h)->state); });
}

double ref_group_norm(void* h, int x) {
    return static_cast<RefState*>(h)->state.group_norm_squared(x);
}

int ref_reset_top(void* h, int bit, int error_branch, int kind, double delta, double p_source) {
    return guarded([&] {
        QubitPair q = reinit_state(make_error(kind, delta, 0, 0, 0, 0));
        reset_top(static_cast<RefState*>(h)->state, bit,
                  error_branch ? MeasureBranch::error : MeasureBranch::correct, q, p_source);
    });
}

// interleaved (re, im) of global amplitudes [first, first + count)
int ref_state_read(void* h, uint64_t first, uint64_t count, double* out) {
    return guarded([&] {
        auto& st = static_cast<RefState*>(h)->state;
        for (uint64_t i = 0; i < count; ++i) {
            cplx v = st.amp(first + i);
            out[2 * i] = v.real();
            out[2 * i + 1] = v.imag();
        }
    });
}

// sample_measurement (proj/src/statevector.cpp:236-256) for a given p1
int ref_sample_measurement(double p1, uint64_t seed, uint32_t idx, uint32_t stage, int kind,
                           double delta, double px, double py, double pz, int has_pauli,
                           int32_t out[4]) {
    return guarded([&] {
        RngStream rng(seed, idx, stage, RngDomain::measurement);
        MeasureResult m = sample_measurement(p1, rng, make_error(kind, delta, px, py, pz, has_pauli));
        out[0] = m.sampled_bit;
        out[1] = m.observed_bit;
        out[2] = m.branch == MeasureBranch::error ? 1 : 0;
        out[3] = m.event.classical_flip ? 1 : 0;
    });
}

int ref_exhaustive(uint64_t N, uint64_t a, unsigned L, unsigned t, int kind, double delta, double px,
                   double py, double pz, int has_pauli, double* out /* 2^t */) {
    return guarded([&] {
        auto d = exhaustive_joint_distribution(make_problem(N, a, L, t),
                                               make_error(kind, delta, px, py, pz, has_pauli));
        std::memcpy(out, d.data(), d.size() * sizeof(double));
    });
}

// shor_standard_procedure: ints = {classification, r_even, a_r_is_one,
// a_half_not_minus_one, order_match (0/1, 2 = none), n_factors}; kr = {k_lo,
// k_hi, r_lo, r_hi}; factors[4].
int ref_shor_standard_procedure(uint64_t j_lo, uint64_t j_hi, unsigned t, uint64_t N, uint64_t a,
                                uint64_t known_order, int has_order, int32_t ints[6],
                                uint64_t kr[4], uint64_t factors[4]) {
    return guarded([&] {
        u128 j = (u128{j_hi} << 64) | j_lo;
        std::optional<u64> ko;
        if (has_order) ko = known_order;
        PostProcessOutcome o = shor_standard_procedure(j, t, N, a, ko);
        ints[0] = static_cast<int32_t>(o.classification);
        ints[1] = o.checks.r_even;
        ints[2] = o.checks.a_r_is_one;
        ints[3] = o.checks.a_half_not_minus_one;
        ints[4] = o.order_match ? (*o.order_match ? 1 : 0) : 2;
        ints[5] = static_cast<int32_t>(o.factors.size());
        kr[0] = static_cast<uint64_t>(o.convergent.k);
        kr[1] = static_cast<uint64_t>(o.convergent.k >> 64);
        kr[2] = static_cast<uint64_t>(o.convergent.r);
        kr[3] = static_cast<uint64_t>(o.convergent.r >> 64);
        for (size_t i = 0; i < 4; ++i) factors[i] = i < o.factors.size() ? o.factors[i] : 0;
    });
}

// factorize (numtheory.cpp:170-187) with an explicit rho budget
int ref_factorize(uint64_t n, uint64_t budget, uint64_t* primes, uint32_t* exps, uint32_t* count) {
    return guarded([&] {
        auto f = factorize(n, budget);
        *count = static_cast<uint32_t>(f.size());
        for (size_t i = 0; i < f.size(); ++i) {
            primes[i] = f[i].prime;
            exps[i] = f[i].exponent;
        }
    });
}

int ref_multiplicative_order(uint64_t a, uint64_t N, uint64_t p, uint64_t q, uint64_t* out) {
    return guarded([&] {
        std::optional<std::pair<u64, u64>> kf;
        if (p && q) kf = std::make_pair(p, q);
        *out = multiplicative_order(a, N, kf).value;
    });
}

// run_problem (simulator backend, Shor post-processing) on the reference engine:
// counts = {order, success, lucky_ne, lucky_no, lucky_oo, fail, first_factor_index
// (0 = none), first_order_index (0 = none), r_overflow, r_other, r_total_lucky,
// order_solvable, n_reciprocal}; recip = {D, count} pairs (up to cap).
int ref_run_problem(uint64_t N, uint64_t a, uint64_t p, uint64_t q, unsigned L, unsigned t,
                    uint64_t seed, unsigned M, int kind, double delta, double px, double py,
                    double pz, int has_pauli, unsigned qubit_ceiling, uint64_t counts[13],
                    uint64_t* recip, unsigned cap, int post_ekera) {
    return guarded([&] {
        FactoringProblem prob = make_problem(N, a, L, t);
        prob.p = p;
        prob.q = q;
        prob.seed = seed;
        CampaignSpec spec;
        spec.M = M;
        spec.error = make_error(kind, delta, px, py, pz, has_pauli);
        spec.sim.qubit_ceiling = qubit_ceiling;
        spec.post_mode = post_ekera ? PostMode::ekera : PostMode::shor;
        ProblemResult r = run_problem(prob, spec);
        counts[0] = r.order;
        counts[1] = r.success;
        counts[2] = r.lucky_ne;
        counts[3] = r.lucky_no;
        counts[4] = r.lucky_oo;
        counts[5] = r.fail;
        counts[6] = r.first_factor_index ? *r.first_factor_index : 0;
        counts[7] = r.first_order_index ? *r.first_order_index : 0;
        counts[8] = r.r_ratio.overflow;
        counts[9] = r.r_ratio.other;
        counts[10] = r.r_ratio.total_lucky;
        counts[11] = r.order_solvable ? 1 : 0;
        counts[12] = r.r_ratio.reciprocal.size();
        unsigned i = 0;
        for (const auto& [D, c] : r.r_ratio.reciprocal) {
            if (i >= cap) break;
            recip[2 * i] = D;
            recip[2 * i + 1] = c;
            ++i;
        }
    });
}

// ekera_postprocess with RngStream(seed, idx, 1, postprocess) as run_problem uses it:
// ints = {classification, order_match (0/1, 2 = none), has_recovered_order,
// has_offset, n_factors}; u64s = {k_lo, k_hi, r_lo, r_hi, recovered_order,
// offset (two's complement)}; factors[4].
int ref_ekera_postprocess(uint64_t j_lo, uint64_t j_hi, unsigned t, uint64_t N, uint64_t a,
                          uint64_t B, uint64_t c, unsigned k, unsigned varsigma, unsigned m,
                          unsigned ell, uint64_t seed, uint32_t idx, uint64_t known_order,
                          int has_order, int32_t ints[5], uint64_t u64s[6], uint64_t factors[4]) {
    return guarded([&] {
        u128 j = (u128{j_hi} << 64) | j_lo;
        EkeraParams prm;
        prm.B = B;
        prm.c = c;
        prm.k = k;
        prm.varsigma = varsigma;
        prm.m = m;
        prm.ell = ell;
        RngStream rng(seed, idx, 1, RngDomain::postprocess);
        std::optional<u64> ko;
        if (has_order) ko = known_order;
        PostProcessOutcome o = ekera_postprocess(j, t, N, a, prm, rng, ko);
        ints[0] = static_cast<int32_t>(o.classification);
        ints[1] = o.order_match ? (*o.order_match ? 1 : 0) : 2;
        ints[2] = o.recovered_order ? 1 : 0;
        ints[3] = o.candidate_offset ? 1 : 0;
        ints[4] = static_cast<int32_t>(o.factors.size());
        u64s[0] = static_cast<uint64_t>(o.convergent.k);
        u64s[1] = static_cast<uint64_t>(o.convergent.k >> 64);
        u64s[2] = static_cast<uint64_t>(o.convergent.r);
        u64s[3] = static_cast<uint64_t>(o.convergent.r >> 64);
        u64s[4] = o.recovered_order ? *o.recovered_order : 0;
        u64s[5] = o.candidate_offset ? static_cast<uint64_t>(static_cast<int64_t>(*o.candidate_offset)) : 0;
        for (size_t i = 0; i < 4; ++i) factors[i] = i < o.factors.size() ? o.factors[i] : 0;
    });
}

} // extern "C"
