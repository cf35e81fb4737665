// Link-level drop-in (TEST INFRASTRUCTURE): definitions of the reference's
// shorsim::IterativeShorEngine constructor and run(), and of
// exhaustive_joint_distribution, on top of the B200 engine's
// C ABI, so the reference's OWN callers — proj/src/harness.cpp (run_problem,
// simulate_to_jsonl) and proj/tests/acceptance/acceptance_main.cpp — compile
// UNCHANGED and run on the GPU. oracle/Makefile compiles the reference's
// statevector.cpp with -DIterativeShorEngine=IterativeShorEngine_reference so
// its engine symbols do not clash with these (likewise
// -Dexhaustive_joint_distribution=exhaustive_joint_distribution_reference).
//
// The reference class's layout (proj/include/shorsim/statevector.hpp:177-190) is
// fixed by its header; the engine handle therefore lives in a registry keyed by
// the object's address (the implicit destructor cannot release it; a handle is
// released when its address is reused and at exit).
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>

#include "shorsim/statevector.hpp"
#include "shorsim_b200.hpp"

namespace {

// The reference object cannot own the B200 engine (its layout is fixed and its
// destructor implicit), so engines live here keyed by the object's address.
// At most kLive engines are kept: the least recently used one is released and
// re-created from its stored arguments if its object runs again (a harness
// creates one engine per problem; without a bound every problem's engine —
// and its device buffers — would live until exit).
struct Entry {
    shorsim::FactoringProblem problem;
    shorsim::ErrorConfig error;
    shorsim::SimulatorOptions options;
    std::shared_ptr<shorsim::b200::IterativeShorEngine> engine;
    std::uint64_t last_use = 0;
};

struct Registry {
    std::mutex mu;
    std::map<const void*, Entry> entries;
    std::uint64_t clock = 0;
    std::size_t live = 0;
};

constexpr std::size_t kLive = 32;

Registry& registry() {
    static Registry r;
    return r;
}

int device_from_env() {
    const char* d = std::getenv("SHS_DEVICE");
    return d ? std::atoi(d) : 0;
}

// caller holds r.mu
void evict_if_full(Registry& r) {
    while (r.live >= kLive) {
        Entry* lru = nullptr;
        for (auto& kv : r.entries)
            if (kv.second.engine && (!lru || kv.second.last_use < lru->last_use)) lru = &kv.second;
        if (!lru) return;
        lru->engine.reset();  // a run in flight keeps its own reference
        --r.live;
    }
}

}  // namespace

namespace shorsim {

IterativeShorEngine::IterativeShorEngine(const FactoringProblem& problem, const ErrorConfig& error,
                                         const SimulatorOptions& options)
    : problem_(problem), error_(error), options_(options) {
    // constructed eagerly: validation errors surface here, as in the reference
    auto engine = std::make_shared<b200::IterativeShorEngine>(problem, error, options,
                                                              device_from_env());
    a_pows_ = engine->stage_multipliers();  // stage_multipliers() is inline in the header
    n_ = problem.L + 1;
    y_limit_ = problem.N;
    auto& r = registry();
    std::lock_guard<std::mutex> lock(r.mu);
    Entry& e = r.entries[this];
    if (e.engine) --r.live;  // a dead object's address reused
    e.engine.reset();
    evict_if_full(r);
    e = Entry{problem, error, options, std::move(engine), ++r.clock};
    ++r.live;
}

// exhaustive_joint_distribution (statevector.cpp:533-579) on the device enumerator
std::vector<double> exhaustive_joint_distribution(const FactoringProblem& problem,
                                                  const ErrorConfig& error, u64 node_budget) {
    return b200::exhaustive_joint_distribution(problem, error, node_budget, device_from_env());
}

RunResult IterativeShorEngine::run(u64 seed, u64 bitstring_index) {
    std::shared_ptr<b200::IterativeShorEngine> engine;
    {
        auto& r = registry();
        std::lock_guard<std::mutex> lock(r.mu);
        Entry& e = r.entries.at(this);
        if (!e.engine) {
            evict_if_full(r);
            e.engine = std::make_shared<b200::IterativeShorEngine>(e.problem, e.error, e.options,
                                                                   device_from_env());
            ++r.live;
        }
        e.last_use = ++r.clock;
        engine = e.engine;
    }
    return engine->run(seed, bitstring_index);
}

}  // namespace shorsim
