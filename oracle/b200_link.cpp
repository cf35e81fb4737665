// Link-level drop-in (TEST INFRASTRUCTURE): definitions of the reference's
// shorsim::IterativeShorEngine constructor and run() on top of the B200 engine's
// C ABI, so the reference's OWN callers — proj/src/harness.cpp (run_problem,
// simulate_to_jsonl) and proj/tests/acceptance/acceptance_main.cpp — compile
// UNCHANGED and run on the GPU. oracle/Makefile compiles the reference's
// statevector.cpp with -DIterativeShorEngine=IterativeShorEngine_reference so
// its engine symbols do not clash with these.
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

struct Registry {
    std::mutex mu;
    std::map<const void*, std::unique_ptr<shorsim::b200::IterativeShorEngine>> engines;
};

Registry& registry() {
    static Registry r;
    return r;
}

int device_from_env() {
    const char* d = std::getenv("SHS_DEVICE");
    return d ? std::atoi(d) : 0;
}

}  // namespace

namespace shorsim {

IterativeShorEngine::IterativeShorEngine(const FactoringProblem& problem, const ErrorConfig& error,
                                         const SimulatorOptions& options)
    : problem_(problem), error_(error), options_(options) {
    auto engine = std::make_unique<b200::IterativeShorEngine>(problem, error, options,
                                                              device_from_env());
    a_pows_ = engine->stage_multipliers();  // stage_multipliers() is inline in the header
    n_ = problem.L + 1;
    y_limit_ = problem.N;
    auto& r = registry();
    std::lock_guard<std::mutex> lock(r.mu);
    r.engines[this] = std::move(engine);
}

RunResult IterativeShorEngine::run(u64 seed, u64 bitstring_index) {
    b200::IterativeShorEngine* engine;
    {
        auto& r = registry();
        std::lock_guard<std::mutex> lock(r.mu);
        engine = r.engines.at(this).get();
    }
    return engine->run(seed, bitstring_index);
}

}  // namespace shorsim
