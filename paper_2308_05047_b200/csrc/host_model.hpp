// Host-side scalar model of the engine: Philox streams, number theory, noise
// hooks, stage phase and measurement sampling. These are the reference's
// per-stage scalar steps,
// restated for the B200 engine's host driver. Compiled with
// -ffp-contract=off so every scalar rounds as the reference's does.
#pragma once

#include <cstdint>
#include <string>

#include "../../include/shorsim_b200.h"

namespace shs {

using u32 = std::uint32_t;
using u64 = std::uint64_t;
using u128 = unsigned __int128;

// proj/include/shorsim/rng.hpp:16-31 (Philox4x32-10)
void philox_block(u64 key, const u32 in[4], u32 out[4]);
// RngStream(seed, a, b, domain).at(index) / at_double(index), rng.hpp:70-74
u64 rng_u64(u64 seed, u32 a, u32 b, u32 domain, u32 index);
double rng_double(u64 seed, u32 a, u32 b, u32 domain, u32 index);

constexpr u32 kDomainMeasurement = 0;  // rng.hpp:43
constexpr u32 kDomainBitflip = 1;      // rng.hpp:44

// int128.hpp:28-30
inline u64 mulmod(u64 a, u64 b, u64 m) { return static_cast<u64>((u128{a} * b) % m); }
// numtheory.cpp:25-46; returns 0 on success, SHS_NOT_INVERTIBLE with *gcd set
int mod_inverse(u64 a, u64 n, u64* inv, u64* gcd);
// floor(m * 2^64 / n), the Shoup companion of multiplier m (m < n < 2^63)
inline u64 shoup(u64 m, u64 n) { return static_cast<u64>((u128{m} << 64) / n); }

// noise.cpp:13-25; returns 0 or SHS_CONFIG_ERROR with *why set
int validate_error(const shs_error& e, std::string* why);
// noise.cpp:81-95: {w0r, w0i, w1r, w1i}
void reinit_state(const shs_error& e, double w[4]);
// statevector.cpp:201-206
double stage_phase(unsigned cbit, u128 prefix);

struct Measurement {
    int sampled_bit;
    int observed_bit;
    bool error_branch;     // MeasureBranch::error (quantum model)
    bool classical_flip;
};
// sample_measurement, statevector.cpp:236-256 (+ noise.cpp:128-145)
Measurement sample_measurement(double p1, u64 seed, u32 idx, u32 stage, const shs_error& e);
// bitflip_bitstring with RngStream(seed, idx, 0, bitflip), statevector.cpp:406-409
u128 bitflip_bitstring(u128 j, unsigned t, double delta, u64 seed, u32 idx);

// thread-local last error shared by every C-ABI entry point (shs_last_error)
int set_error(int code, const std::string& msg);
const char* last_error();

// IterativeShorEngine construction checks in the reference's order
// (statevector.cpp:289-295, :65-72), plus this engine's own limits
int validate_engine_config(const shs_problem& pr, const shs_error& er, const shs_options& o);

// correctly rounded (nearest-even) value of an exact 40-digit accumulator
// (value = F * 2^-1088, 32-bit digits in uint64 words); normalises in place
double digits_to_double_host(std::uint64_t* digits);

}  // namespace shs
