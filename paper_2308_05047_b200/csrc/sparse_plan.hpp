// Planning of the sparse prefix of a run (sparse.cuh), shared by the single
// engine (engine.cu) and the sharded engine (shard.cu): host-side only.
#pragma once

#include <cstdint>
#include <unordered_map>
#include <vector>

#include "host_model.hpp"

namespace shs {

// Smallest j in [1, M) with A^j = 1 (mod N), or 0 when there is none
// (baby-step giant-step, O(sqrt M) multiplications). A is a unit mod N.
inline uint64_t small_order(uint64_t A, uint64_t N, uint64_t M) {
    if (A % N == 1) return 1;
    uint64_t m = 1;
    while (m * m < M) ++m;
    std::unordered_map<uint64_t, uint64_t> baby;
    baby.reserve(2 * m);
    uint64_t x = 1;
    for (uint64_t i = 0; i < m; ++i) {
        if (i > 0 && x == 1) return i < M ? i : 0;
        baby.emplace(x, i);
        x = mulmod(x, A, N);
    }
    uint64_t ginv = 0, g = 0;  // x = A^m
    if (mod_inverse(x, N, &ginv, &g) != SHS_OK) return 0;
    uint64_t y = 1;
    for (uint64_t q = 1; q <= m; ++q) {
        y = mulmod(y, ginv, N);  // A^(-q m)
        auto it = baby.find(y);
        if (it != baby.end()) {
            const uint64_t j = q * m + it->second;
            return j < M ? j : 0;
        }
    }
    return 0;
}

constexpr uint64_t kSparseMinN = 1ull << 22;  // sparse prefix from 64 MB of state
constexpr uint64_t kSparseDensity = 16;       // support <= N / 16 (A/B: 64 / 32 / 16 / 8 -> config 4 2345 / 2299 / 2269 / 2290 ms per run)

// Stages run on the support: the largest n <= t - 1 with 2^n <= cap whose last
// multiplier A_{n-1} has order >= 2^n (then every earlier stage's has too:
// ord(A_s) >= ord(A_{n-1}) / 2^(n-1-s)), so the orbit never wraps. 0 below
// kSparseMinN.
inline uint32_t sparse_prefix_stages(uint64_t N, uint32_t t, const std::vector<u64>& a_pows,
                                     uint64_t cap) {
    if (N < kSparseMinN) return 0;
    uint32_t n = 0;
    while (n + 1 <= t - 1 && (uint64_t(1) << (n + 1)) <= cap) ++n;
    if (n == 0) return 0;
    const uint64_t ord = small_order(a_pows[n - 1], N, uint64_t(1) << n);
    if (ord == 0) return n;
    // ord(A_{n-1}) < 2^n: the largest s with ord(A_s) >= 2^(s+1)
    for (uint32_t m = n; m > 0; --m) {
        uint64_t o = ord;
        for (uint32_t k = 0; k < n - m && o % 2 == 0; ++k) o /= 2;  // ord(A_{m-1})
        if (o >= (uint64_t(1) << m)) return m;
    }
    return 0;
}

}  // namespace shs
