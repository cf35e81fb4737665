// Drop-in replacement for the reference's "shorsim/statevector.hpp"
// (/root/reference/proj/include/shorsim/statevector.hpp): the same declarations
// in namespace shorsim, backed by the B200 engine through the C ABI
// (include/shorsim_b200.h). Put -I<repo>/include/dropin -I<repo>/include ahead
// of the reference's include directory, drop proj/src/statevector.cpp from
// the build and link -lshorsim_b200: the reference's callers (harness.cpp,
// the acceptance driver, tests/test_statevector.cpp) compile unchanged.
//
//   ShardLayout / make_shard_layout   statevector.hpp:20-31, statevector.cpp:65-72
//   ShardedState                      :33-65 — amplitudes in device memory (value
//                                     type: copies are device-to-device clones);
//                                     amp / set_amp / amp_xy / group_base /
//                                     norm_squared / group_norm_squared. The
//                                     host views shards() / group_spans() of the
//                                     CPU layout have no device counterpart.
//   init_state, apply_oracle, apply_phase, stage_phase, apply_hadamard_top,
//   measure_top, sample_measurement, reset_top              :68-133
//   ExchangePlan, build_permutation_plan, plan_receive_lists,
//   plan_send_lists                   :75-97 (computed on the device)
//   StageTrace, BitString, RunResult, SimulatorOptions      :135-159
//   IterativeShorEngine, run_iterative_shor                 :161-191 (GPU engine;
//                                     sharded over devices when the state
//                                     outgrows one, SHS_DEVICES to choose)
//   exhaustive_joint_distribution     :193-198 (device enumerator)
// Device: SHS_DEVICE (default 0).
#pragma once

#include <cmath>
#include <complex>
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <utility>
#include <vector>

#include "shorsim/errors.hpp"
#include "shorsim/int128.hpp"
#include "shorsim/noise.hpp"
#include "shorsim/problems.hpp"
#include "shorsim/rng.hpp"
#include "shorsim_b200.h"

namespace shorsim {

using cplx = std::complex<double>;

struct ShardLayout {
    unsigned n = 2;
    unsigned g = 1;  // shard count S = 2^g
    unsigned shard_count() const { return 1u << g; }
    u64 shard_size() const { return u64{1} << (n - g); }
    u64 group_size() const { return u64{1} << (n - 1); }
    unsigned group_shards() const { return 1u << (g - 1); }
    unsigned shard_of(u64 global) const { return static_cast<unsigned>(global >> (n - g)); }
    u64 offset_of(u64 global) const { return global & (shard_size() - 1); }
};

struct ErrorEvent {
    bool classical_flip = false;
    bool quantum_error_branch = false;
};

struct MeasureResult {
    int sampled_bit;
    int observed_bit;
    double p1;
    MeasureBranch branch = MeasureBranch::correct;
    ErrorEvent event;
};

struct StageTrace {
    unsigned cbit;
    double p1;
    int sampled_bit;
    int observed_bit;
    ErrorEvent event;
};

struct BitString {
    unsigned t = 0;
    u128 j = 0;
};

struct RunResult {
    BitString bits;
    u128 j_sampled = 0;
    std::vector<StageTrace> trace;
};

struct SimulatorOptions {
    unsigned shard_count = 4;
    unsigned workers = 1;
    unsigned qubit_ceiling = 26;
    bool check_norms = true;
};

}  // namespace shorsim

#include "shorsim_b200.hpp"

namespace shorsim {

namespace b200 {
inline int device_from_env() { return default_device(); }
inline shs_sv* clone_sv(const shs_sv* h) {
    shs_sv* c = nullptr;
    if (h) throw_status(shs_sv_clone(h, &c));
    return c;
}
}  // namespace b200

inline ShardLayout make_shard_layout(unsigned n, unsigned shard_count) {
    if (n < 2 || n > 33) throw std::invalid_argument("shard layout: need 2 <= n <= 33");
    if (shard_count < 2 || (shard_count & (shard_count - 1)) != 0)
        throw std::invalid_argument("shard layout: shard count must be a power of two >= 2");
    unsigned g = 0;
    while ((1u << g) < shard_count) ++g;
    if (g > n - 1) throw std::invalid_argument("shard layout: more shards than group states");
    return ShardLayout{n, g};
}

class ShardedState {
public:
    ShardedState() = default;
    ShardedState(unsigned n, unsigned shard_count) : layout_(make_shard_layout(n, shard_count)) {
        b200::throw_status(shs_sv_create(n, shard_count, b200::device_from_env(), &h_));
    }
    ShardedState(const ShardedState& o) : layout_(o.layout_), h_(b200::clone_sv(o.h_)) {}
    ShardedState(ShardedState&& o) noexcept : layout_(o.layout_), h_(std::exchange(o.h_, nullptr)) {}
    ShardedState& operator=(ShardedState o) noexcept {
        std::swap(layout_, o.layout_);
        std::swap(h_, o.h_);
        return *this;
    }
    ~ShardedState() {
        if (h_) shs_sv_destroy(h_);
    }

    const ShardLayout& layout() const { return layout_; }
    unsigned qubits() const { return layout_.n; }

    cplx amp(u64 global) const {
        double v[2];
        b200::throw_status(shs_sv_read(h_, global, 1, v));
        return {v[0], v[1]};
    }
    void set_amp(u64 global, cplx v) {
        const double w[2] = {v.real(), v.imag()};
        b200::throw_status(shs_sv_write(h_, global, 1, w));
    }
    cplx amp_xy(int x, u64 y) const { return amp(group_base(x) + y); }
    u64 group_base(int x) const { return x == 0 ? 0 : layout_.group_size(); }

    // deterministic fixed-block compensated sums, statevector.cpp:95-124
    double group_norm_squared(int x) const {
        double p[2];
        b200::throw_status(shs_sv_group_norms(h_, p));
        return p[x];
    }
    double norm_squared() const {
        double p[2];
        b200::throw_status(shs_sv_group_norms(h_, p));
        return p[0] + p[1];
    }

    shs_sv* handle() const { return h_; }

private:
    ShardLayout layout_;
    shs_sv* h_ = nullptr;
};

inline ShardedState init_state(unsigned n, QubitPair top_qubit_state, unsigned shard_count) {
    ShardedState state(n, shard_count);
    const double pair[4] = {top_qubit_state.a0.real(), top_qubit_state.a0.imag(),
                            top_qubit_state.a1.real(), top_qubit_state.a1.imag()};
    b200::throw_status(shs_sv_init_state(state.handle(), pair));
    return state;
}

struct ExchangePlan {
    u64 modulus = 1;
    u64 a_pow = 1;
    u64 a_inv = 1;
    u64 y_limit = 0;
    ShardLayout layout;
    std::vector<u32> gather;
    bool identity = false;
    std::vector<std::vector<u64>> pair_counts;
};

inline ExchangePlan build_permutation_plan(u64 a_pow, u64 n_modulus, const ShardLayout& layout) {
    if (n_modulus < 2) throw std::invalid_argument("permutation plan: modulus >= 2");
    ExchangePlan plan;
    std::uint64_t inv = 0, ylim = 0;
    std::int32_t ident = 0;
    const int dev = b200::device_from_env();
    b200::throw_status(shs_plan_build(a_pow, n_modulus, layout.n, layout.shard_count(), dev, &inv,
                                      &ident, &ylim, nullptr, nullptr));
    const unsigned gs = layout.group_shards();
    std::vector<std::uint64_t> gather(ylim ? ylim : 1), counts(std::size_t(gs) * gs);
    b200::throw_status(shs_plan_build(a_pow, n_modulus, layout.n, layout.shard_count(), dev,
                                      nullptr, nullptr, nullptr, gather.data(), counts.data()));
    plan.modulus = n_modulus;
    plan.a_pow = a_pow % n_modulus;
    plan.a_inv = inv;
    plan.layout = layout;
    plan.y_limit = ylim;
    plan.identity = ident != 0;
    plan.gather.assign(gather.begin(), gather.begin() + ylim);  // u32, as the reference's
    plan.pair_counts.assign(gs, std::vector<u64>(gs, 0));
    for (unsigned s = 0; s < gs; ++s)
        for (unsigned d = 0; d < gs; ++d) plan.pair_counts[s][d] = counts[std::size_t(s) * gs + d];
    return plan;
}

struct ShardIndexList {
    unsigned xrank;
    std::vector<u64> local_index;
};

namespace b200 {
inline std::vector<ShardIndexList> plan_lists(const ExchangePlan& plan, unsigned xrank, int send) {
    const unsigned gs = plan.layout.group_shards();
    std::vector<std::uint64_t> counts(gs), idx(plan.layout.shard_size());
    throw_status(shs_plan_lists(plan.a_pow, plan.modulus, plan.layout.n, plan.layout.shard_count(),
                                xrank, send, device_from_env(), counts.data(), idx.data()));
    std::vector<ShardIndexList> out;
    std::size_t k = 0;
    for (unsigned p = 0; p < gs; ++p) {
        if (counts[p])
            out.push_back(ShardIndexList{p, std::vector<u64>(idx.begin() + k,
                                                             idx.begin() + k + counts[p])});
        k += counts[p];
    }
    return out;
}
}  // namespace b200

inline std::vector<ShardIndexList> plan_receive_lists(const ExchangePlan& plan, unsigned dst_xrank) {
    return b200::plan_lists(plan, dst_xrank, 0);
}
inline std::vector<ShardIndexList> plan_send_lists(const ExchangePlan& plan, unsigned src_xrank) {
    return b200::plan_lists(plan, src_xrank, 1);
}

inline void apply_oracle(ShardedState& state, u64 a_pow, u64 n_modulus) {
    if (n_modulus < 2) throw std::invalid_argument("permutation plan: modulus >= 2");
    b200::throw_status(shs_sv_apply_oracle(state.handle(), a_pow, n_modulus));
}

inline double stage_phase(unsigned cbit, u128 measured_bits_so_far) {
    if (cbit == 0) return 0.0;
    return 3.14159265358979323846 * static_cast<double>(measured_bits_so_far) *
           std::exp2(-static_cast<double>(cbit));
}

inline void apply_phase(ShardedState& state, unsigned cbit, u128 measured_bits_so_far) {
    b200::throw_status(shs_sv_apply_phase(state.handle(), cbit,
                                          static_cast<std::uint64_t>(measured_bits_so_far),
                                          static_cast<std::uint64_t>(measured_bits_so_far >> 64)));
}

inline void apply_hadamard_top(ShardedState& state) {
    b200::throw_status(shs_sv_apply_hadamard_top(state.handle()));
}

// The host-side draw of statevector.cpp:236-256 from the caller's stream: the
// depolarizing channel decides bit and branch; otherwise R < p1, then the
// classical misreading of the observed bit.
inline MeasureResult sample_measurement(double p1, RngStream& stage_rng, const ErrorConfig& error) {
    MeasureResult m;
    m.p1 = p1;
    if (error.kind == ErrorKind::quantum_measure) {
        const DepolarizingOutcome d = depolarizing_measure_branch(p1, *error.pauli, stage_rng);
        m.sampled_bit = m.observed_bit = d.bit;
        m.branch = d.branch;
        m.event.quantum_error_branch = d.branch == MeasureBranch::error;
        return m;
    }
    m.sampled_bit = stage_rng.next_double() < p1 ? 1 : 0;
    m.observed_bit = m.sampled_bit;
    if (error.kind == ErrorKind::classical_measure) {
        const FlipResult f = classical_flip(m.sampled_bit, error.delta, stage_rng);
        m.observed_bit = f.observed;
        m.event.classical_flip = f.flipped;
    }
    return m;
}

inline MeasureResult measure_top(const ShardedState& state, RngStream& stage_rng,
                                 const ErrorConfig& error) {
    return sample_measurement(state.group_norm_squared(1), stage_rng, error);
}

inline void reset_top(ShardedState& state, int bit, MeasureBranch branch, QubitPair reinit,
                      double p_source) {
    const double pair[4] = {reinit.a0.real(), reinit.a0.imag(), reinit.a1.real(), reinit.a1.imag()};
    b200::throw_status(shs_sv_reset_top(state.handle(), bit,
                                        branch == MeasureBranch::error ? 1 : 0, pair, p_source));
}

using IterativeShorEngine = b200::IterativeShorEngine;

inline RunResult run_iterative_shor(const FactoringProblem& problem, const ErrorConfig& error,
                                    u64 seed, u64 bitstring_index, const SimulatorOptions& options) {
    IterativeShorEngine engine(problem, error, options, b200::device_from_env());
    return engine.run(seed, bitstring_index);
}

inline std::vector<double> exhaustive_joint_distribution(const FactoringProblem& problem,
                                                         const ErrorConfig& error,
                                                         u64 node_budget = u64{1} << 22) {
    return b200::exhaustive_joint_distribution(problem, error, node_budget, b200::device_from_env());
}

}  // namespace shorsim
