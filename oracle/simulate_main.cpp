// TEST INFRASTRUCTURE: calls the reference's own shorsim::simulate_to_jsonl
// (proj/src/harness.cpp:494-529) and prints the JSONL. Linked twice by
// oracle/Makefile — against the reference engine (simulate_ref) and against the
// B200 engine via b200_link.cpp (simulate_b200) — so the outputs can be compared
// byte for byte. Usage: simulate N a t shots seed [shards] [error-spec]
#include <cstdlib>
#include <iostream>
#include <string>

#include "shorsim/harness.hpp"
#include "shorsim/noise.hpp"

int main(int argc, char** argv) {
    if (argc < 6) {
        std::cerr << "usage: simulate N a t shots seed [shards] [error]\n";
        return 2;
    }
    shorsim::FactoringProblem p;
    p.N = std::stoull(argv[1]);
    p.a = std::stoull(argv[2]);
    p.L = shorsim::bit_length_u64(p.N);
    p.t = static_cast<unsigned>(std::stoul(argv[3]));
    unsigned shots = static_cast<unsigned>(std::stoul(argv[4]));
    shorsim::u64 seed = std::stoull(argv[5]);
    shorsim::SimulatorOptions o;
    o.qubit_ceiling = 33;
    if (argc > 6) o.shard_count = static_cast<unsigned>(std::stoul(argv[6]));
    shorsim::ErrorConfig e;
    if (argc > 7) e = shorsim::parse_error_config(argv[7]);
    try {
        std::cout << shorsim::simulate_to_jsonl(p, e, shots, seed, o);
    } catch (const std::exception& ex) {
        std::cerr << "error: " << ex.what() << "\n";
        return 1;
    }
    return 0;
}
