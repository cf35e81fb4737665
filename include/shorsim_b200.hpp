// shorsim_b200.hpp — C++ drop-in for the reference's engine API, over the C ABI.
//
// Include AFTER the reference's "shorsim/statevector.hpp" (it supplies
// FactoringProblem, ErrorConfig, SimulatorOptions, RunResult and the exception
// types of proj/include/shorsim/errors.hpp). Provides, in namespace
// shorsim::b200, the reference's entry points with the same signatures and
// exception behaviour:
//   class IterativeShorEngine   — proj/include/shorsim/statevector.hpp:169-191
//   run_iterative_shor          — statevector.hpp:164-165
//   StepEngine (per-gate path)  — statevector.hpp:68-133 on the compressed state
//   exhaustive_joint_distribution — statevector.hpp:193-198 (on the device)
// A state larger than one GPU is block-sharded over as many devices as it needs
// (shs_options.n_devices = AUTO; SHS_DEVICES="0,1,..." picks them explicitly),
// behind the same class: the reference's callers reach the multi-GPU engine
// unchanged.
// A caller switches with one alias:
//   namespace shorsim { using IterativeShorEngine = b200::IterativeShorEngine; }
#pragma once

#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "shorsim_b200.h"

namespace shorsim::b200 {

// CUDA device of engines created without an explicit one: SHS_DEVICE (default 0)
inline int default_device() {
    const char* d = std::getenv("SHS_DEVICE");
    return d ? std::atoi(d) : 0;
}

// Map a status code to the reference's exception types (errors.hpp:8-43).
inline void throw_status(int rc) {
    if (rc == SHS_OK) return;
    std::string msg = shs_last_error();
    switch (rc) {
        case SHS_CONFIG_ERROR: throw ConfigError(msg);
        case SHS_CEILING_EXCEEDED: throw CeilingExceededError(msg);
        case SHS_DEGENERATE_BRANCH: throw DegenerateBranchError(msg);
        case SHS_BUDGET_EXCEEDED: throw BudgetExceededError(msg);
        case SHS_FACTORIZATION_TIMEOUT: throw FactorizationTimeoutError(msg);
        case SHS_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case SHS_NOT_INVERTIBLE: {
            // "not invertible: gcd(a, n) = g"
            std::uint64_t a = 0, n = 0, g = 0;
            auto p = msg.find("gcd(");
            if (p != std::string::npos) {
                a = std::stoull(msg.substr(p + 4));
                n = std::stoull(msg.substr(msg.find(", ", p) + 2));
                g = std::stoull(msg.substr(msg.rfind("= ") + 2));
            }
            throw NotInvertibleError(a, n, g);
        }
        default: throw Error(msg);  // SHS_ERROR (norm drift) and CUDA failures
    }
}

inline shs_error to_c(const ErrorConfig& e) {
    shs_error c{};
    c.kind = static_cast<int32_t>(e.kind);
    c.delta = e.delta;
    if (e.pauli) {
        c.px = e.pauli->px;
        c.py = e.pauli->py;
        c.pz = e.pauli->pz;
        c.has_pauli = 1;
    }
    return c;
}

// p1 is combined like the reference (sequential Kahan, bit-identical) up to 1024
// blocks (N <= 2^18) and exactly above that (combine = SHS_COMBINE_AUTO; within
// 1 ulp of the reference's Kahan, include/shorsim_b200.h); pass
// SHS_COMBINE_KAHAN to keep the reference's combine at every size (slower:
// sequential over N/256 partials per stage).
inline shs_options to_c(const SimulatorOptions& o, int device, int combine = SHS_COMBINE_AUTO) {
    shs_options c;
    shs_default_options(&c);
    c.shard_count = o.shard_count;
    c.workers = o.workers;
    c.qubit_ceiling = o.qubit_ceiling;
    c.check_norms = o.check_norms ? 1 : 0;
    c.device = device;
    c.combine = combine;
    c.n_devices = -1;  // AUTO: shard over devices when the state outgrows one
    return c;
}

class IterativeShorEngine {
public:
    IterativeShorEngine(const FactoringProblem& problem, const ErrorConfig& error,
                        const SimulatorOptions& options, int device = default_device(),
                        int combine = SHS_COMBINE_AUTO)
        : t_(problem.t) {
        shs_problem p{problem.N, problem.a, problem.L, problem.t, problem.seed};
        shs_error e = to_c(error);
        shs_options o = to_c(options, device, combine);
        throw_status(shs_engine_create(&p, &e, &o, &h_));
        a_pows_.resize(t_);
        throw_status(shs_engine_stage_multipliers(h_, a_pows_.data()));
        trace_.resize(t_);
        batch_mode_ = shs_engine_batched(h_);
        batched_ = batch_mode_ != 0;
    }
    ~IterativeShorEngine() {
        if (h_) shs_engine_destroy(h_);
    }
    IterativeShorEngine(const IterativeShorEngine&) = delete;
    IterativeShorEngine& operator=(const IterativeShorEngine&) = delete;
    IterativeShorEngine(IterativeShorEngine&& o) noexcept
        : h_(std::exchange(o.h_, nullptr)), t_(o.t_), a_pows_(std::move(o.a_pows_)),
          trace_(std::move(o.trace_)), batched_(o.batched_), batch_mode_(o.batch_mode_),
          next_fetch_(o.next_fetch_), cache_seed_(o.cache_seed_),
          cache_lo_(o.cache_lo_), cache_n_(o.cache_n_), have_last_(o.have_last_),
          last_seed_(o.last_seed_), last_idx_(o.last_idx_), nobatch_seed_(o.nobatch_seed_),
          nobatch_lo_(o.nobatch_lo_), nobatch_hi_(o.nobatch_hi_), c_j_(std::move(o.c_j_)),
          c_js_(std::move(o.c_js_)), c_p1_(std::move(o.c_p1_)), c_bits_(std::move(o.c_bits_)) {}

    // IterativeShorEngine::run, statevector.cpp:323-412. A run is a pure function
    // of (seed, bitstring_index), so for problems the batched paths cover
    // (shs_engine_batched: 1 = whole runs per CTA, N <= 4096; 2 = lockstep
    // shots, mid-size N) a shot loop is served from batches: the reference's
    // loops (run_problem, simulate_to_jsonl) call run(seed, m) for consecutive
    // m. A first call runs alone (run_iterative_shor's one run costs one run);
    // a miss that continues the previous index fetches the next indices in one
    // call — 256 runs (a campaign's M), doubling on consecutive misses up to
    // 4096. A batch that fails on a model error (degenerate branch, norm drift)
    // is served run by run inside its window, so exactly the failing index
    // throws; batching resumes past it. CUDA errors propagate.
    RunResult run(u64 seed, u64 bitstring_index) {
        if (batched_) {
            bool hit = cache_seed_ == seed && bitstring_index >= cache_lo_ &&
                       bitstring_index < cache_lo_ + cache_n_;
            const bool consecutive = have_last_ && seed == last_seed_ &&
                                     bitstring_index == last_idx_ + 1;
            const bool in_failed = seed == nobatch_seed_ && bitstring_index >= nobatch_lo_ &&
                                   bitstring_index < nobatch_hi_;
            have_last_ = true;
            last_seed_ = seed;
            last_idx_ = bitstring_index;
            // a first call (or a jump) fetches just this run, through the same
            // batched path (pooled buffers: no per-engine allocation); a call that
            // continues the previous index fetches the next window
            if (!hit && !in_failed) hit = prefetch(seed, bitstring_index, consecutive);
            if (hit) return unpack(bitstring_index - cache_lo_);
        }
        std::uint64_t j[2], js[2];
        throw_status(shs_engine_run(h_, seed, bitstring_index, j, js, trace_.data()));
        RunResult r;
        r.bits = BitString{t_, (u128{j[1]} << 64) | j[0]};
        r.j_sampled = (u128{js[1]} << 64) | js[0];
        r.trace.reserve(t_);
        for (const auto& s : trace_)
            r.trace.push_back(StageTrace{s.cbit, s.p1, s.sampled_bit, s.observed_bit,
                                         ErrorEvent{s.classical_flip != 0,
                                                    s.quantum_error_branch != 0}});
        return r;
    }

    const std::vector<u64>& stage_multipliers() const { return a_pows_; }
    shs_engine* handle() const { return h_; }

private:
    static constexpr std::uint32_t kFetchFirst = 256;     // first fetch ...
    static constexpr std::uint32_t kFetchMax = 4096;      // ... doubling up to this

    // true when [idx0, idx0 + n) is now cached; window = false: n = 1
    bool prefetch(u64 seed, u64 idx0, bool window) {
        const bool next = cache_n_ && cache_seed_ == seed && idx0 == cache_lo_ + cache_n_;
        if (window) next_fetch_ = next && next_fetch_ ? std::min(2 * next_fetch_, kFetchMax) : kFetchFirst;
        const std::uint32_t n = window ? next_fetch_ : 1;
        c_j_.resize(2 * std::size_t(n));
        c_js_.resize(2 * std::size_t(n));
        c_p1_.resize(std::size_t(n) * t_);
        c_bits_.resize(std::size_t(n) * t_ * 4);
        cache_n_ = 0;
        const int rc = shs_engine_run_many(h_, seed, idx0, n, c_j_.data(), c_js_.data(),
                                           c_p1_.data(), c_bits_.data());
        if (rc == SHS_CUDA_ERROR || rc == SHS_INVALID_ARGUMENT) throw_status(rc);
        if (rc != SHS_OK) {  // a model error inside the window: serve it run by run
            nobatch_seed_ = seed;
            nobatch_lo_ = idx0;
            nobatch_hi_ = idx0 + n;
            next_fetch_ = 0;
            return false;
        }
        cache_seed_ = seed;
        cache_lo_ = idx0;
        cache_n_ = n;
        return true;
    }

    RunResult unpack(u64 k) const {
        RunResult r;
        r.bits = BitString{t_, (u128{c_j_[2 * k + 1]} << 64) | c_j_[2 * k]};
        r.j_sampled = (u128{c_js_[2 * k + 1]} << 64) | c_js_[2 * k];
        r.trace.reserve(t_);
        for (unsigned s = 0; s < t_; ++s) {
            const std::int32_t* b = &c_bits_[(k * t_ + s) * 4];
            r.trace.push_back(StageTrace{s, c_p1_[k * t_ + s], b[0], b[1],
                                         ErrorEvent{b[2] != 0, b[3] != 0}});
        }
        return r;
    }

    shs_engine* h_ = nullptr;
    unsigned t_;
    std::vector<u64> a_pows_;
    std::vector<shs_stage_trace> trace_;
    bool batched_ = false;
    int batch_mode_ = 0;
    std::uint32_t next_fetch_ = 0;
    u64 cache_seed_ = 0, cache_lo_ = 0, cache_n_ = 0;
    bool have_last_ = false;
    u64 last_seed_ = 0, last_idx_ = 0;
    u64 nobatch_seed_ = 0, nobatch_lo_ = 0, nobatch_hi_ = 0;
    std::vector<std::uint64_t> c_j_, c_js_;
    std::vector<double> c_p1_;
    std::vector<std::int32_t> c_bits_;
};

inline RunResult run_iterative_shor(const FactoringProblem& problem, const ErrorConfig& error,
                                    u64 seed, u64 bitstring_index,
                                    const SimulatorOptions& options) {
    IterativeShorEngine engine(problem, error, options);
    return engine.run(seed, bitstring_index);
}

// exhaustive_joint_distribution, statevector.hpp:193-198 / statevector.cpp:533-579:
// every measurement path enumerated on the device (csrc/exhaustive.cu), error
// branches marginalised; bit-identical to the reference, same limits and
// BudgetExceededError.
inline std::vector<double> exhaustive_joint_distribution(const FactoringProblem& problem,
                                                         const ErrorConfig& error,
                                                         u64 node_budget = u64{1} << 22,
                                                         int device = 0) {
    shs_problem p{problem.N, problem.a, problem.L, problem.t, problem.seed};
    shs_error e = to_c(error);
    if (problem.t > 14 || problem.L + 1 > 12) {  // checked before sizing the output
        throw_status(shs_exhaustive_distribution(&p, &e, node_budget, device, nullptr));
    }
    std::vector<double> out(std::size_t{1} << problem.t);
    throw_status(shs_exhaustive_distribution(&p, &e, node_budget, device, out.data()));
    return out;
}

// The per-gate ("step/measure") path for forced measurement sequences:
// stage_probs = apply_oracle + apply_phase + apply_hadamard_top + the two group
// norms; collapse = reset_top(src_group, reinit, p_source).
class StepEngine {
public:
    explicit StepEngine(IterativeShorEngine& e) : h_(e.handle()) { throw_status(shs_state_init(h_)); }
    std::pair<double, double> stage_probs(unsigned s, u128 prefix) {
        double p0 = 0, p1 = 0;
        throw_status(shs_stage_probs(h_, s, static_cast<std::uint64_t>(prefix),
                                     static_cast<std::uint64_t>(prefix >> 64), &p0, &p1));
        return {p0, p1};
    }
    void collapse(int src_group, double p_source) {
        throw_status(shs_stage_collapse(h_, src_group, p_source));
    }
    std::vector<double> state(int x, u64 first, u64 count) {
        std::vector<double> out(2 * count);
        throw_status(shs_state_read(h_, x, first, count, out.data()));
        return out;
    }

private:
    shs_engine* h_;
};

}  // namespace shorsim::b200
