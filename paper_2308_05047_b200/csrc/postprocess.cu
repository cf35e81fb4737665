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

}  // namespace

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
