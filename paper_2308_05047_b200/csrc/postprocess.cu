// Shor's standard post-processing on the device (§8 f4): the step right after
// the path. Every measured bit string j of a batch (the batched engine's shots,
// proj/src/harness.cpp:128-147) goes through shor_standard_procedure
// (proj/src/postprocess.cpp:55-89) in its own thread:
//   extract_denominator   continued fraction of j / 2^t, last convergent with
//                         r < N (proj/src/numtheory.cpp:236-270), u128 Euclid
//   checks                r even, a^r = 1, a^floor(r/2) != -1 (mod N)
//   factors               gcd(a^floor(r/2) -/+ 1, N) through add_nontrivial_factor
//                         (postprocess.cpp:24-32), sorted ascending
//   classification        classify_lucky with the known order (postprocess.cpp:48-53),
//                         else the algorithm-only labels (postprocess.cpp:79-86)
// Integer-only: the outcome is identical to the reference's by construction and
// checked field by field against it (tests/test_gpu_postprocess.py).
#include <cuda_runtime.h>

#include <string>

#include "../../include/shorsim_b200.h"
#include "host_model.hpp"
#include "measure.cuh"

using namespace shs;

namespace {

typedef unsigned __int128 u128d;

__device__ __forceinline__ uint64_t pp_mulmod(uint64_t a, uint64_t b, uint64_t n) {
    return static_cast<uint64_t>((u128d(a) * b) % n);  // mulmod_u64, int128.hpp:28-30
}

__device__ uint64_t pp_mod_pow(uint64_t base, uint64_t e, uint64_t n) {  // numtheory.cpp:48-59
    if (n == 1) return 0;
    uint64_t r = 1, b = base % n;
    while (e) {
        if (e & 1) r = pp_mulmod(r, b, n);
        b = pp_mulmod(b, b, n);
        e >>= 1;
    }
    return r;
}

__device__ uint64_t pp_gcd(uint64_t a, uint64_t b) {  // std::gcd
    while (b) {
        const uint64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

struct Factors {
    uint64_t v[4];
    uint32_t n;
};

__device__ bool has(const Factors& f, uint64_t g) {
    for (uint32_t i = 0; i < f.n; ++i)
        if (f.v[i] == g) return true;
    return false;
}

__device__ void add_nontrivial_factor(Factors& f, uint64_t g, uint64_t n) {  // postprocess.cpp:24-32
    if (g <= 1 || g >= n) return;
    if (!has(f, g)) f.v[f.n++] = g;
    const uint64_t cof = n / g;
    if (g * cof == n && cof > 1 && cof < n && !has(f, cof)) f.v[f.n++] = cof;
}

__global__ void k_shor_postprocess(const uint64_t* __restrict__ j, uint32_t count, uint32_t t,
                                   uint64_t N, uint64_t a, uint64_t order, int has_order,
                                   shs_shor_outcome* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const u128d jj = (u128d(j[2 * i + 1]) << 64) | j[2 * i];
    // extract_denominator(j, t, N): convergents of j / 2^t in order, keep the
    // last with r < N (denominators never decrease)
    u128d bk = 0, br = 1;  // Convergent{0, 1}
    if (jj != 0) {
        u128d p2 = 1, q2 = 0, p1 = 0, q1 = 1;
        u128d num = u128d(1) << t, den = jj;
        while (den != 0) {
            const u128d aq = num / den, rem = num % den;
            const u128d p = aq * p1 + p2, q = aq * q1 + q2;
            if (q < u128d(N)) {
                bk = p;
                br = q;
            } else {
                break;
            }
            p2 = p1;
            p1 = p;
            q2 = q1;
            q1 = q;
            num = den;
            den = rem;
        }
    }
    shs_shor_outcome o{};
    o.classification = SHS_CLASS_FAIL;
    o.k[0] = static_cast<uint64_t>(bk);
    o.k[1] = static_cast<uint64_t>(bk >> 64);
    o.r[0] = static_cast<uint64_t>(br);
    o.r[1] = static_cast<uint64_t>(br >> 64);
    const uint64_t r = static_cast<uint64_t>(br);
    o.order_match = has_order ? (r == order ? 1 : 0) : 2;
    if (r >= 2) {  // no gcd attempt for r in {0, 1}
        o.r_even = (r % 2 == 0) ? 1 : 0;
        o.a_r_is_one = pp_mod_pow(a, r, N) == 1 ? 1 : 0;
        const uint64_t x = pp_mod_pow(a, r / 2, N);
        o.a_half_not_minus_one = x != N - 1 ? 1 : 0;
        Factors f{{0, 0, 0, 0}, 0};
        add_nontrivial_factor(f, pp_gcd((x + N - 1) % N, N), N);
        add_nontrivial_factor(f, pp_gcd((x + 1) % N, N), N);
        for (uint32_t u = 1; u < f.n; ++u)  // std::sort, ascending
            for (uint32_t v = u; v > 0 && f.v[v - 1] > f.v[v]; --v) {
                const uint64_t tmp = f.v[v];
                f.v[v] = f.v[v - 1];
                f.v[v - 1] = tmp;
            }
        o.n_factors = f.n;
        for (uint32_t u = 0; u < 4; ++u) o.factors[u] = u < f.n ? f.v[u] : 0;
        const bool all = o.r_even && o.a_r_is_one && o.a_half_not_minus_one;
        if (has_order) {  // classify_lucky
            if (f.n == 0) o.classification = SHS_CLASS_FAIL;
            else if (r == order) o.classification = (r % 2 == 0 && all) ? SHS_CLASS_SUCCESS
                                                                        : SHS_CLASS_LUCKY_OO;
            else o.classification = r % 2 == 0 ? SHS_CLASS_LUCKY_NE : SHS_CLASS_LUCKY_NO;
        } else if (f.n == 0) {
            o.classification = SHS_CLASS_FAIL;
        } else if (all) {
            o.classification = SHS_CLASS_SUCCESS;
        } else {
            o.classification = o.r_even ? SHS_CLASS_LUCKY_NE : SHS_CLASS_LUCKY_NO;
        }
    }
    out[i] = o;
}

// ------------------------------------------------------------ Ekerå
// ekera_postprocess (postprocess.cpp:138-171) per bit string: the ±B sweep of
// j' = j + offset, each through extract_denominator, recover_order (the
// smooth lift, postprocess.cpp:102-134) and factor_from_order
// (postprocess.cpp:136-164) with the shot's RngStream (seed, m, 1, postprocess).
//
// recover_order returns ord(a) exactly when a^R = 1 for R = r * prod_{q <= cm}
// q^floor(log_q 2^m) (every prime of R is stripped, in any order), else
// nothing; here R is kept as an exponent vector over its primes (the q <= cm
// and the primes of r, found by Miller-Rabin with the 12 bases that are exact
// for 64-bit n, and Brent's rho), a^R by successive powering and ord(a) by
// per-prime valuation: no big integers, the same result.

__device__ uint64_t pp_mod_pow_u(uint64_t b, uint64_t e, uint64_t n) { return pp_mod_pow(b, e, n); }

__device__ bool pp_mr_witness(uint64_t n, uint64_t a, uint64_t d, unsigned s) {
    uint64_t x = pp_mod_pow(a % n, d, n);
    if (x == 1 || x == n - 1) return false;
    for (unsigned i = 1; i < s; ++i) {
        x = pp_mulmod(x, x, n);
        if (x == n - 1) return false;
    }
    return true;
}

__device__ bool pp_is_prime(uint64_t n) {  // is_probable_prime, numtheory.cpp:95-116
    if (n < 2) return false;
    const uint64_t bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (uint64_t p : bases) {
        if (n == p) return true;
        if (n % p == 0) return false;
    }
    uint64_t d = n - 1;
    unsigned s = 0;
    while ((d & 1) == 0) {
        d >>= 1;
        ++s;
    }
    for (uint64_t a : bases)
        if (pp_mr_witness(n, a, d, s)) return false;
    return true;
}

// Brent's rho with the reference's batch of 128 and its step budget
// (numtheory.cpp:120-157): the budget counts rho steps over one factorize()
// call; running out sets *timeout (FactorizationTimeoutError there). The same
// batch, restart and backtracking order gives the same divisor, hence the same
// recursion and the same budget use as the reference.
__device__ uint64_t pp_rho(uint64_t n, uint64_t* budget, bool* timeout) {
    if ((n & 1) == 0) return 2;
    for (uint64_t c = 1;; ++c) {
        uint64_t x = 2, y = 2, d = 1, q = 1, ys = 0, r = 1;
        constexpr uint64_t kBatch = 128;
        auto step = [&](uint64_t v) { return (pp_mulmod(v, v, n) + c) % n; };
        while (d == 1) {
            x = y;
            for (uint64_t i = 0; i < r; ++i) y = step(y);
            for (uint64_t k = 0; k < r && d == 1; k += kBatch) {
                ys = y;
                const uint64_t lim = r - k < kBatch ? r - k : kBatch;
                for (uint64_t i = 0; i < lim; ++i) {
                    y = step(y);
                    q = pp_mulmod(q, x > y ? x - y : y - x, n);
                }
                if (*budget < lim) {
                    *timeout = true;
                    return 0;
                }
                *budget -= lim;
                d = pp_gcd(q, n);
            }
            r *= 2;
        }
        if (d == n) {  // backtrack one by one from the last saved point
            d = 1;
            while (d == 1) {
                ys = step(ys);
                d = pp_gcd(x > ys ? x - ys : ys - x, n);
                if (*budget == 0) {
                    *timeout = true;
                    return 0;
                }
                --*budget;
            }
        }
        if (d != n) return d;
    }
}

constexpr int kMaxPrimes = 32;
constexpr uint64_t kRhoBudget = 10000000;  // factorize()'s default, numtheory.hpp:53

// factorize (numtheory.cpp:170-187): trial division by the primes below 100,
// then factor_rec's depth-first splits (d first). Primes with multiplicity are
// appended to p[*np] in discovery order; false on a budget timeout.
__device__ bool pp_factorize(uint64_t n, uint64_t budget, uint64_t* p, int* np, int cap) {
    const uint8_t small[25] = {2,  3,  5,  7,  11, 13, 17, 19, 23, 29, 31, 37, 41,
                               43, 47, 53, 59, 61, 67, 71, 73, 79, 83, 89, 97};
    for (int i = 0; i < 25; ++i)
        while (n % small[i] == 0) {
            if (*np < cap) p[(*np)++] = small[i];
            n /= small[i];
        }
    uint64_t stack[64];
    int top = 0;
    if (n > 1) stack[top++] = n;
    bool timeout = false;
    while (top) {  // LIFO: push n / d, then d, so d is factored first
        const uint64_t m = stack[--top];
        if (m == 1) continue;
        if (pp_is_prime(m)) {
            if (*np < cap) p[(*np)++] = m;
            continue;
        }
        const uint64_t d = pp_rho(m, &budget, &timeout);
        if (timeout) return false;
        stack[top++] = m / d;
        stack[top++] = d;
    }
    return true;
}

// distinct primes of n (unsorted) appended to p[*np]; false on a budget timeout
__device__ bool pp_prime_factors(uint64_t n, uint64_t* p, int* np, uint64_t budget) {
    uint64_t all[64];
    int na = 0;
    if (!pp_factorize(n, budget, all, &na, 64)) return false;
    for (int i = 0; i < na; ++i) {
        bool seen = false;
        for (int k = 0; k < *np; ++k) seen |= p[k] == all[i];
        if (!seen && *np < kMaxPrimes) p[(*np)++] = all[i];
    }
    return true;
}

// recover_order: ord(a) when a^R = 1, else 0
__device__ uint64_t pp_recover_order(uint64_t r, uint64_t a, uint64_t N, uint64_t c, uint64_t m,
                                     uint64_t budget, bool* timeout) {
    if (r == 0) r = 1;
    uint64_t pr[kMaxPrimes], ex[kMaxPrimes];
    int np = 0;
    const uint64_t cm = c * m;
    const unsigned __int128 cap = static_cast<unsigned __int128>(1) << m;
    for (uint64_t q = 2; q <= cm; ++q) {  // primes <= cm: their lift exponent
        bool prime = true;
        for (uint64_t d = 2; d * d <= q; ++d) prime &= (q % d) != 0;
        if (!prime) continue;
        unsigned __int128 pw = q;
        uint64_t e = 1;
        while (pw * q <= cap) {
            pw *= q;
            ++e;
        }
        pr[np] = q;
        ex[np] = e;
        ++np;
    }
    const int nlift = np;
    uint64_t rp[kMaxPrimes];
    int nr = 0;
    if (!pp_prime_factors(r, rp, &nr, budget)) {  // factorize(r_candidate), postprocess.cpp:113
        *timeout = true;
        return 0;
    }
    for (int i = 0; i < nr; ++i) {
        uint64_t v = 0, x = r;
        while (x % rp[i] == 0) {
            x /= rp[i];
            ++v;
        }
        int at = -1;
        for (int k = 0; k < nlift; ++k)
            if (pr[k] == rp[i]) at = k;
        if (at >= 0) {
            ex[at] += v;
        } else if (np < kMaxPrimes) {
            pr[np] = rp[i];
            ex[np] = v;
            ++np;
        }
    }
    auto pow_all = [&](int skip) {  // a^(R / q_skip^e_skip)
        uint64_t x = a % N;
        for (int k = 0; k < np; ++k) {
            if (k == skip) continue;
            for (uint64_t e = 0; e < ex[k]; ++e) x = pp_mod_pow(x, pr[k], N);
        }
        return x;
    };
    if (pow_all(-1) != 1) return 0;
    uint64_t ord = 1;
    for (int k = 0; k < np; ++k) {  // v_q(ord): smallest f with y^(q^f) = 1
        uint64_t y = pow_all(k), f = 0;
        while (y != 1) {
            y = pp_mod_pow(y, pr[k], N);
            ++f;
        }
        for (uint64_t i = 0; i < f; ++i) ord *= pr[k];
    }
    return ord;
}

struct PostRng {  // RngStream(seed, m, 1, postprocess), rng.hpp:52-83
    uint64_t seed;
    uint32_t a, b, index;
    __device__ uint64_t next() {
        uint32_t cc[4] = {index++, a, b, 5u};
        philox_dev(seed, cc);
        return (uint64_t(cc[0]) << 32) | cc[1];
    }
    __device__ uint64_t below(uint64_t n) {
        const uint64_t limit = ~uint64_t(0) - ~uint64_t(0) % n;
        uint64_t x;
        do {
            x = next();
        } while (x >= limit);
        return x % n;
    }
};

__device__ void pp_sort(Factors& f) {
    for (uint32_t u = 1; u < f.n; ++u)
        for (uint32_t v = u; v > 0 && f.v[v - 1] > f.v[v]; --v) {
            const uint64_t tmp = f.v[v];
            f.v[v] = f.v[v - 1];
            f.v[v - 1] = tmp;
        }
}

// factor_from_order (postprocess.cpp:136-164)
__device__ void pp_factor_from_order(uint64_t N, uint64_t order, PostRng& rng, uint32_t k_trials,
                                     uint32_t varsigma, Factors& f) {
    f.n = 0;
    uint64_t odd = order;
    unsigned d2 = 0;
    while ((odd & 1) == 0) {
        odd >>= 1;
        ++d2;
    }
    const unsigned levels = d2 + 1 + (varsigma > 1 ? varsigma : 1);
    for (uint32_t trial = 0; trial < k_trials; ++trial) {
        const uint64_t x = 2 + rng.below(N - 2);
        const uint64_t g = pp_gcd(x, N);
        if (g != 1) {
            add_nontrivial_factor(f, g, N);
            pp_sort(f);
            return;
        }
        uint64_t y = pp_mod_pow(x, odd, N);
        for (unsigned level = 0; level < levels; ++level) {
            if (y == 1) break;
            add_nontrivial_factor(f, pp_gcd((y + N - 1) % N, N), N);
            add_nontrivial_factor(f, pp_gcd((y + 1) % N, N), N);
            if (f.n) {
                pp_sort(f);
                return;
            }
            y = pp_mulmod(y, y, N);
        }
    }
}

__device__ void pp_extract(u128d jj, uint32_t t, uint64_t N, u128d& bk, u128d& br) {
    bk = 0;
    br = 1;
    if (jj == 0) return;
    u128d p2 = 1, q2 = 0, p1 = 0, q1 = 1;
    u128d num = u128d(1) << t, den = jj;
    while (den != 0) {
        const u128d aq = num / den, rem = num % den;
        const u128d p = aq * p1 + p2, q = aq * q1 + q2;
        if (q >= u128d(N)) break;
        bk = p;
        br = q;
        p2 = p1;
        p1 = p;
        q2 = q1;
        q1 = q;
        num = den;
        den = rem;
    }
}

__global__ void k_ekera_postprocess(const uint64_t* __restrict__ j, uint32_t count, uint32_t t,
                                    uint64_t N, uint64_t a, shs_ekera_params prm, uint64_t seed,
                                    uint64_t idx0, uint64_t order, int has_order,
                                    shs_ekera_outcome* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const u128d jj = (u128d(j[2 * i + 1]) << 64) | j[2 * i];
    shs_ekera_outcome o{};
    u128d bk, br;
    pp_extract(jj, t, N, bk, br);
    o.k[0] = static_cast<uint64_t>(bk);
    o.k[1] = static_cast<uint64_t>(bk >> 64);
    o.r[0] = static_cast<uint64_t>(br);
    o.r[1] = static_cast<uint64_t>(br >> 64);
    o.classification = SHS_CLASS_FAIL;
    PostRng rng{seed, static_cast<uint32_t>(idx0 + i), 1u, 0u};
    const u128d mask = t >= 128 ? ~u128d(0) : ((u128d(1) << t) - 1);
    uint64_t rec = 0;
    const uint64_t budget = prm.rho_budget ? prm.rho_budget : kRhoBudget;
    for (uint64_t step = 0; step <= prm.B; ++step) {
        for (int sgn = -1; sgn <= 1; sgn += 2) {
            if (step == 0 && sgn == 1) continue;  // offset 0 once
            const u128d jp = (sgn < 0 ? jj - u128d(step) : jj + u128d(step)) & mask;
            u128d ck, cr;
            pp_extract(jp, t, N, ck, cr);
            bool timeout = false;
            const uint64_t ordr =
                pp_recover_order(static_cast<uint64_t>(cr), a, N, prm.c, prm.m, budget, &timeout);
            if (timeout) {  // FactorizationTimeoutError out of ekera_postprocess
                o.timeout = 1;
                out[i] = o;
                return;
            }
            if (!ordr) continue;
            if (!rec) rec = ordr;
            Factors f{{0, 0, 0, 0}, 0};
            pp_factor_from_order(N, ordr, rng, prm.k, prm.varsigma, f);
            if (f.n) {
                o.n_factors = f.n;
                for (uint32_t u = 0; u < 4; ++u) o.factors[u] = u < f.n ? f.v[u] : 0;
                o.has_recovered_order = 1;
                o.recovered_order = ordr;
                o.has_offset = 1;
                o.candidate_offset = sgn < 0 ? -static_cast<int64_t>(step) : static_cast<int64_t>(step);
                o.classification = SHS_CLASS_SUCCESS;
                o.order_match = has_order ? (ordr == order ? 1 : 0) : 2;
                out[i] = o;
                return;
            }
        }
    }
    o.has_recovered_order = rec ? 1 : 0;
    o.recovered_order = rec;
    o.order_match = has_order ? ((rec && rec == order) ? 1 : 0) : 2;
    out[i] = o;
}

__global__ void k_factorize(uint64_t n, uint64_t budget, uint64_t* out, int* count, int* ok) {
    uint64_t p[64];
    int np = 0;
    *ok = pp_factorize(n, budget, p, &np, 64) ? 1 : 0;
    for (int u = 1; u < np; ++u)  // sorted ascending, as factorize() returns them
        for (int v = u; v > 0 && p[v - 1] > p[v]; --v) {
            const uint64_t tmp = p[v];
            p[v] = p[v - 1];
            p[v - 1] = tmp;
        }
    for (int i = 0; i < np; ++i) out[i] = p[i];
    *count = np;
}

}  // namespace

extern "C" int shs_factorize(uint64_t n, uint64_t rho_budget, int32_t device, uint64_t* primes,
                             uint32_t* exponents, uint32_t* count) {
    if (!primes || !exponents || !count) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    if (n == 0) return set_error(SHS_INVALID_ARGUMENT, "factorize(0)");
    cudaError_t ce = cudaSetDevice(device);
    if (ce != cudaSuccess) return set_error(SHS_CUDA_ERROR, cudaGetErrorString(ce));
    struct Out {
        uint64_t p[64];
        int count, ok;
    };
    Out* d = nullptr;
    if ((ce = cudaMalloc(&d, sizeof(Out))) != cudaSuccess)
        return set_error(SHS_CUDA_ERROR, cudaGetErrorString(ce));
    k_factorize<<<1, 1>>>(n, rho_budget ? rho_budget : kRhoBudget, d->p, &d->count, &d->ok);
    Out h;
    ce = cudaGetLastError();
    if (ce == cudaSuccess) ce = cudaMemcpy(&h, d, sizeof(Out), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (ce != cudaSuccess) return set_error(SHS_CUDA_ERROR, cudaGetErrorString(ce));
    if (!h.ok) return set_error(SHS_FACTORIZATION_TIMEOUT, "pollard rho budget exhausted");
    uint32_t k = 0;
    for (int i = 0; i < h.count; ++i) {  // prime powers, numtheory.cpp:180-185
        if (k && primes[k - 1] == h.p[i]) {
            ++exponents[k - 1];
        } else {
            primes[k] = h.p[i];
            exponents[k] = 1;
            ++k;
        }
    }
    *count = k;
    return SHS_OK;
}

extern "C" int shs_shor_postprocess(const uint64_t* j, uint32_t count, uint32_t t, uint64_t N,
                                    uint64_t a, uint64_t known_order, int32_t has_known_order,
                                    int32_t device, shs_shor_outcome* out) {
    if ((!j || !out) && count) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    if (t >= 128) return set_error(SHS_INVALID_ARGUMENT, "convergents: t must be < 128");
    if (N < 2) return set_error(SHS_INVALID_ARGUMENT, "modulus must be >= 2");
    for (uint32_t i = 0; i < count; ++i)  // convergents(): j < 2^t
        if ((t < 64 && (j[2 * i + 1] != 0 || (j[2 * i] >> t) != 0)) ||
            (t >= 64 && (j[2 * i + 1] >> (t - 64)) != 0))
            return set_error(SHS_INVALID_ARGUMENT, "convergents: j >= 2^t");
    if (!count) return SHS_OK;
    cudaError_t ce = cudaSetDevice(device);
    if (ce != cudaSuccess) return set_error(SHS_CUDA_ERROR, cudaGetErrorString(ce));
    uint64_t* dj = nullptr;
    shs_shor_outcome* dout = nullptr;
    auto fail = [&](cudaError_t e) {
        cudaFree(dj);
        cudaFree(dout);
        return set_error(SHS_CUDA_ERROR, std::string("postprocess: ") + cudaGetErrorString(e));
    };
    if ((ce = cudaMalloc(&dj, sizeof(uint64_t) * 2 * count)) != cudaSuccess) return fail(ce);
    if ((ce = cudaMalloc(&dout, sizeof(shs_shor_outcome) * count)) != cudaSuccess) return fail(ce);
    if ((ce = cudaMemcpy(dj, j, sizeof(uint64_t) * 2 * count, cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail(ce);
    const int threads = 128;
    k_shor_postprocess<<<(count + threads - 1) / threads, threads>>>(
        dj, count, t, N, a, known_order, has_known_order ? 1 : 0, dout);
    if ((ce = cudaGetLastError()) != cudaSuccess) return fail(ce);
    if ((ce = cudaMemcpy(out, dout, sizeof(shs_shor_outcome) * count, cudaMemcpyDeviceToHost)) !=
        cudaSuccess)
        return fail(ce);
    cudaFree(dj);
    cudaFree(dout);
    return SHS_OK;
}

extern "C" int shs_ekera_postprocess(const uint64_t* j, uint32_t count, uint32_t t, uint64_t N,
                                     uint64_t a, const shs_ekera_params* params, uint64_t seed,
                                     uint64_t idx0, uint64_t known_order, int32_t has_known_order,
                                     int32_t device, shs_ekera_outcome* out) {
    if ((!j || !out || !params) && count) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    if (t >= 128) return set_error(SHS_INVALID_ARGUMENT, "convergents: t must be < 128");
    if (N < 3) return set_error(SHS_INVALID_ARGUMENT, "modulus must be >= 3");
    if (params->m > 63) return set_error(SHS_INVALID_ARGUMENT, "recover_order: m <= 63");
    if (params->k == 0 || params->B > (uint64_t(1) << 20))
        return set_error(SHS_INVALID_ARGUMENT, "ekera: k >= 1 and B <= 2^20");
    for (uint32_t i = 0; i < count; ++i)
        if ((t < 64 && (j[2 * i + 1] != 0 || (j[2 * i] >> t) != 0)) ||
            (t >= 64 && (j[2 * i + 1] >> (t - 64)) != 0))
            return set_error(SHS_INVALID_ARGUMENT, "convergents: j >= 2^t");
    if (!count) return SHS_OK;
    cudaError_t ce = cudaSetDevice(device);
    if (ce != cudaSuccess) return set_error(SHS_CUDA_ERROR, cudaGetErrorString(ce));
    uint64_t* dj = nullptr;
    shs_ekera_outcome* dout = nullptr;
    auto fail = [&](cudaError_t e) {
        cudaFree(dj);
        cudaFree(dout);
        return set_error(SHS_CUDA_ERROR, std::string("ekera: ") + cudaGetErrorString(e));
    };
    if ((ce = cudaMalloc(&dj, sizeof(uint64_t) * 2 * count)) != cudaSuccess) return fail(ce);
    if ((ce = cudaMalloc(&dout, sizeof(shs_ekera_outcome) * count)) != cudaSuccess) return fail(ce);
    if ((ce = cudaMemcpy(dj, j, sizeof(uint64_t) * 2 * count, cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail(ce);
    const int threads = 64;
    k_ekera_postprocess<<<(count + threads - 1) / threads, threads>>>(
        dj, count, t, N, a, *params, seed, idx0, known_order, has_known_order ? 1 : 0, dout);
    if ((ce = cudaGetLastError()) != cudaSuccess) return fail(ce);
    if ((ce = cudaMemcpy(out, dout, sizeof(shs_ekera_outcome) * count, cudaMemcpyDeviceToHost)) !=
        cudaSuccess)
        return fail(ce);
    cudaFree(dj);
    cudaFree(dout);
    for (uint32_t i = 0; i < count; ++i)  // the reference throws out of the first such shot
        if (out[i].timeout)
            return set_error(SHS_FACTORIZATION_TIMEOUT,
                             "pollard rho budget exhausted (bit string " + std::to_string(i) + ")");
    return SHS_OK;
}
