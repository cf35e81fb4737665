// See host_model.hpp. Each function cites the reference lines it restates.
#include "host_model.hpp"

#include <cmath>
#include <string>

namespace shs {

namespace {
constexpr double kPi = 3.14159265358979323846;          // statevector.cpp:15
constexpr double kInvSqrt2 = 0.70710678118654752440;    // noise.cpp:10
using i128 = __int128;
}  // namespace

void philox_block(u64 key, const u32 in[4], u32 out[4]) {
    u32 c0 = in[0], c1 = in[1], c2 = in[2], c3 = in[3];
    u32 k0 = static_cast<u32>(key), k1 = static_cast<u32>(key >> 32);
    for (int round = 0; round < 10; ++round) {
        u64 p0 = u64{0xD2511F53u} * c0;
        u64 p1 = u64{0xCD9E8D57u} * c2;
        u32 n0 = static_cast<u32>(p1 >> 32) ^ c1 ^ k0;
        u32 n1 = static_cast<u32>(p1);
        u32 n2 = static_cast<u32>(p0 >> 32) ^ c3 ^ k1;
        u32 n3 = static_cast<u32>(p0);
        c0 = n0;
        c1 = n1;
        c2 = n2;
        c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

u64 rng_u64(u64 seed, u32 a, u32 b, u32 domain, u32 index) {
    u32 ctr[4] = {index, a, b, domain}, out[4];
    philox_block(seed, ctr, out);
    return (u64{out[0]} << 32) | out[1];
}

double rng_double(u64 seed, u32 a, u32 b, u32 domain, u32 index) {
    return static_cast<double>(rng_u64(seed, a, b, domain, index) >> 11) * 0x1.0p-53;
}

int mod_inverse(u64 a, u64 n, u64* inv, u64* gcd) {
    i128 old_r = static_cast<i128>(a % n), r = static_cast<i128>(n), old_x = 1, x = 0;
    while (r != 0) {
        i128 q = old_r / r, tmp;
        tmp = old_r - q * r;
        old_r = r;
        r = tmp;
        tmp = old_x - q * x;
        old_x = x;
        x = tmp;
    }
    if (gcd) *gcd = static_cast<u64>(old_r);
    if (old_r != 1) return SHS_NOT_INVERTIBLE;
    i128 v = old_x % static_cast<i128>(n);
    if (v < 0) v += n;
    *inv = static_cast<u64>(v);
    return SHS_OK;
}

int validate_error(const shs_error& e, std::string* why) {
    auto bad = [&](const char* m) {
        if (why) *why = m;
        return SHS_CONFIG_ERROR;
    };
    if (e.delta < 0.0 || e.delta > 1.0) return bad("error config: delta outside [0, 1]");
    if (e.kind < SHS_ERR_NONE || e.kind > SHS_ERR_BITFLIP) return bad("unknown error kind");
    if (e.kind == SHS_ERR_QUANTUM_MEASURE) {
        if (!e.has_pauli) return bad("quantum_measure requires px/py(/pz)");
        if (e.px < 0 || e.py < 0 || e.pz < 0 || e.px + e.py + e.pz > 1.0)
            return bad("error config: invalid Pauli probabilities");
        double d = e.px + e.py;
        if (std::abs(d - e.delta) > 1e-12) return bad("quantum_measure: delta != px + py");
    } else if (e.has_pauli) {
        return bad("error config: pauli probabilities only apply to quantum_measure");
    }
    return SHS_OK;
}

void reinit_state(const shs_error& e, double w[4]) {
    if (e.kind == SHS_ERR_AMPLITUDE_INIT) {  // plus_state_amplitude_error, noise.cpp:81-83
        w[0] = std::sqrt((1.0 + e.delta) / 2.0);
        w[1] = 0.0;
        w[2] = std::sqrt((1.0 - e.delta) / 2.0);
        w[3] = 0.0;
    } else if (e.kind == SHS_ERR_PHASE_INIT) {  // std::polar(kInvSqrt2, pi delta), :85-87
        double th = kPi * e.delta;
        w[0] = kInvSqrt2;
        w[1] = 0.0;
        w[2] = kInvSqrt2 * std::cos(th);
        w[3] = kInvSqrt2 * std::sin(th);
    } else {
        w[0] = kInvSqrt2;
        w[1] = 0.0;
        w[2] = kInvSqrt2;
        w[3] = 0.0;
    }
}

double stage_phase(unsigned cbit, u128 prefix) {
    if (cbit == 0) return 0.0;
    return kPi * static_cast<double>(prefix) * std::exp2(-static_cast<double>(cbit));
}

Measurement sample_measurement(double p1, u64 seed, u32 idx, u32 stage, const shs_error& e) {
    u32 draw = 0;
    auto next = [&] { return rng_double(seed, idx, stage, kDomainMeasurement, draw++); };
    Measurement m{0, 0, false, false};
    if (e.kind == SHS_ERR_QUANTUM_MEASURE) {  // depolarizing_measure_branch, noise.cpp:133-145
        double dxy = e.px + e.py;
        double p1_prime = (1.0 - dxy) * p1 + dxy * (1.0 - p1);
        int bit = next() < p1_prime ? 1 : 0;
        double p_bit = bit == 1 ? p1 : 1.0 - p1;
        double p_other = 1.0 - p_bit;
        double p_bit_prime = bit == 1 ? p1_prime : 1.0 - p1_prime;
        double p_error = p_bit_prime > 0.0 ? dxy * p_other / p_bit_prime : 0.0;
        m.sampled_bit = bit;
        m.observed_bit = bit;
        m.error_branch = next() < p_error;
        return m;
    }
    double r = next();
    m.sampled_bit = r < p1 ? 1 : 0;
    m.observed_bit = m.sampled_bit;
    if (e.kind == SHS_ERR_CLASSICAL_MEASURE) {  // classical_flip, noise.cpp:128-131
        bool flip = next() < e.delta;
        m.observed_bit = flip ? 1 - m.sampled_bit : m.sampled_bit;
        m.classical_flip = flip;
    }
    return m;
}

namespace {
thread_local std::string g_last_error;
}  // namespace

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

const char* last_error() { return g_last_error.c_str(); }

int validate_engine_config(const shs_problem& pr, const shs_error& er, const shs_options& o) {
    std::string why;
    if (validate_error(er, &why)) return set_error(SHS_CONFIG_ERROR, why);  // :289
    unsigned n = pr.L + 1;
    if (n > o.qubit_ceiling)  // statevector.cpp:291-294
        return set_error(SHS_CEILING_EXCEEDED, "simulator: n = " + std::to_string(n) +
                                                   " exceeds qubit ceiling " +
                                                   std::to_string(o.qubit_ceiling));
    // make_shard_layout (statevector.cpp:65-72); the n <= 33 cap of the u32
    // reference layout is lifted (indices are u64 here, N < 2^63).
    if (n < 2) return set_error(SHS_INVALID_ARGUMENT, "shard layout: need 2 <= n");
    if (o.shard_count < 2 || (o.shard_count & (o.shard_count - 1)) != 0)
        return set_error(SHS_INVALID_ARGUMENT,
                         "shard layout: shard count must be a power of two >= 2");
    if (static_cast<unsigned>(__builtin_ctz(o.shard_count)) > n - 1)
        return set_error(SHS_INVALID_ARGUMENT, "shard layout: more shards than group states");
    if (pr.N < 2) return set_error(SHS_INVALID_ARGUMENT, "modulus must be >= 2");
    if (pr.L > 62) return set_error(SHS_INVALID_ARGUMENT, "L > 62 unsupported (N < 2^63)");
    if (pr.N > (u64{1} << pr.L))
        return set_error(SHS_INVALID_ARGUMENT, "N exceeds 2^L: L must be at least bit_length(N)");
    if (pr.t < 1 || pr.t > 127) return set_error(SHS_INVALID_ARGUMENT, "t must be in [1, 127]");
    if (o.combine < SHS_COMBINE_AUTO || o.combine > SHS_COMBINE_EXACT)
        return set_error(SHS_INVALID_ARGUMENT, "unknown combine mode");
    if (o.tiling < SHS_TILING_AUTO || o.tiling > SHS_TILING_OFF)
        return set_error(SHS_INVALID_ARGUMENT, "unknown tiling mode");
    return SHS_OK;
}


double digits_to_double_host(std::uint64_t* acc) {
    constexpr int kDigitsN = 40, kAnchorBits = 1088;
    std::uint64_t carry = 0;
    for (int i = 0; i < kDigitsN; ++i) {
        std::uint64_t v = acc[i] + carry;
        acc[i] = v & 0xffffffffull;
        carry = v >> 32;
    }
    int top = -1;
    for (int i = kDigitsN - 1; i >= 0 && top < 0; --i)
        if (acc[i]) top = i * 32 + 63 - __builtin_clzll(acc[i]);
    if (top < 0) return 0.0;
    auto bit = [&](int p) -> int {
        return p >= 0 ? static_cast<int>((acc[p >> 5] >> (p & 31)) & 1ull) : 0;
    };
    int lsb = top - 52;
    if (lsb < kAnchorBits - 1074) lsb = kAnchorBits - 1074;
    std::uint64_t mant = 0;
    for (int p = top; p >= lsb; --p) mant = (mant << 1) | static_cast<std::uint64_t>(bit(p));
    const int round = bit(lsb - 1);
    int sticky = 0;
    for (int p = lsb - 2; p >= 0 && !sticky; --p) sticky = bit(p);
    if (round && (sticky || (mant & 1ull))) ++mant;
    return std::ldexp(static_cast<double>(mant), lsb - kAnchorBits);
}

u128 bitflip_bitstring(u128 j, unsigned t, double delta, u64 seed, u32 idx) {
    for (unsigned i = 0; i < t; ++i)
        if (rng_double(seed, idx, 0, kDomainBitflip, i) < delta) j ^= u128{1} << i;
    return j;
}

}  // namespace shs
