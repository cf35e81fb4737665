// Orbit-compressed state storage.
//
// The reference's work register starts at |1> (statevector.cpp:326-328) and every
// stage only gathers it through z -> z * a^(-2^k) mod N (:341-345), so the
// support of g0 / g1 is always inside the orbit <a> = {a^x mod N}, of size
// r = ord_N(a). For a semiprime N = p q, r | lcm(p - 1, q - 1) <= N / 2: at least
// half of the N amplitudes the reference sweeps every stage are identically
// zero (config 4: r = 2147417454 = N / 2 - 28; config 3: r <= N / 6).
//
// The compressed layout stores the r orbit members in z order: member z lives at
// its rank rank(z) = #{orbit members < z}. A record per 64-index word of Z_N
// holds the word's membership bits and the rank of its first index:
//   rec[w] = {bits of z in [64 w, 64 w + 64), rank(64 w)}   (16 B per 64 z)
// so rank and membership of any z cost one 16 B read, and a 32-index window
// (a tile row / column run) costs two consecutive records.
//
// Exactness: non-members carry +-0 in the reference; their |h|^2 = +0.0 adds
// nothing to the in-order block sums (a non-negative running sum s + 0.0 = s),
// so every block partial, p0 / p1, measurement and kept amplitude is unchanged
// (tests: test_gpu_orbit.py, the config-4 parity suite).
#pragma once

#include "device_math.cuh"
#include "stage_kernels.cuh"

namespace shs {

// from 2^21 (config 3, N = 16777207: a run 9.0 -> 6.4 ms; N = 4186067: 4.75 ->
// 4.21 ms); below 2^21 the stages have no tile plans (AUTO tiling), so nothing
// would run compressed
constexpr uint64_t kOrbitMinN = uint64_t(1) << 21;
constexpr int kOrbThreads = 256;

__device__ __forceinline__ uint64_t lowmask64(unsigned o) { return o ? (~0ull >> (64 - o)) : 0ull; }

// membership and rank of z (rec has nwords + 2 entries, zero bits past N)
__device__ __forceinline__ bool orb_lookup(const ulonglong2* __restrict__ rec, uint64_t z,
                                           uint64_t& rank) {
    const ulonglong2 R = __ldg(rec + (z >> 6));
    const unsigned o = static_cast<unsigned>(z & 63);
    rank = R.y + __popcll(R.x & lowmask64(o));
    return (R.x >> o) & 1ull;
}

// ------------------------------------------------------------------ index build
// thread k marks a^x for x in [k B, min((k + 1) B, r)), starting from starts[k] = a^(k B)
static __global__ void k_orb_mark(const uint64_t* __restrict__ starts, uint64_t nthreads,
                                  uint64_t B, uint64_t r, uint64_t a, uint64_t a_sh, uint64_t N,
                                  unsigned int* __restrict__ bits) {
    const uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (k >= nthreads) return;
    uint64_t z = starts[k];
    const uint64_t x1 = (k + 1) * B < r ? (k + 1) * B : r;
    for (uint64_t x = k * B; x < x1; ++x) {
        atomicOr(bits + (z >> 5), 1u << (z & 31));
        z = mulmod_shoup(z, a, a_sh, N);
    }
}

static __global__ void k_orb_counts(const unsigned int* __restrict__ bits, uint64_t nw,
                                    unsigned long long* __restrict__ counts) {
    for (uint64_t w = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; w < nw;
         w += uint64_t(gridDim.x) * blockDim.x)
        counts[w] = __popc(bits[2 * w]) + __popc(bits[2 * w + 1]);
}

static __global__ void k_orb_records(const unsigned int* __restrict__ bits,
                                     const unsigned long long* __restrict__ base, uint64_t nw,
                                     uint64_t r, ulonglong2* __restrict__ rec) {
    for (uint64_t w = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; w < nw + 2;
         w += uint64_t(gridDim.x) * blockDim.x) {
        if (w < nw)
            rec[w] = make_ulonglong2(uint64_t(bits[2 * w]) | (uint64_t(bits[2 * w + 1]) << 32), base[w]);
        else
            rec[w] = make_ulonglong2(0ull, r);
    }
}

// ------------------------------------------------------------------ conversions
// the compressed state of a device-resident run: slot 0 or 1 of a pair, picked
// by the previous stage's collapse group (dev slot) or by the host
struct OrbSrc {
    const double2* c0;
    const double2* c1;
    const DevStage* prev;  // non-null: prev->sel picks the slot
    int sel;               // otherwise
    __device__ __forceinline__ const double2* get() const {
        return (prev ? prev->sel : sel) ? c1 : c0;
    }
};

// dense D[z] (every z of Z_N) from the compressed state (zeros off the orbit)
static __global__ void k_orb_expand(OrbSrc src, const ulonglong2* __restrict__ rec, uint64_t N,
                                    double2* __restrict__ D) {
    const double2* C = src.get();
    for (uint64_t z = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; z < N;
         z += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t k;
        D[z] = orb_lookup(rec, z, k) ? C[k] : make_double2(0.0, 0.0);
    }
}

// compressed C from a dense state D
static __global__ void k_orb_compress(const double2* __restrict__ D,
                                      const ulonglong2* __restrict__ rec, uint64_t N,
                                      double2* __restrict__ C) {
    for (uint64_t z = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; z < N;
         z += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t k;
        if (orb_lookup(rec, z, k)) C[k] = D[z];
    }
}

// compressed C (zeroed beforehand) from the sparse prefix's support points
static __global__ void k_orb_scatter(const uint64_t* __restrict__ Z, const double2* __restrict__ V,
                                     uint64_t K, const ulonglong2* __restrict__ rec,
                                     double2* __restrict__ C) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < K;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t k;
        if (orb_lookup(rec, Z[i], k)) C[k] = V[i];
    }
}

// amplitude at global z of a compressed state
__device__ __forceinline__ double2 orb_amp(const double2* __restrict__ C,
                                           const ulonglong2* __restrict__ rec, uint64_t z) {
    uint64_t k;
    return orb_lookup(rec, z, k) ? C[k] : make_double2(0.0, 0.0);
}

// k_state_read / k_state_gather on a compressed state: w_x * (sel[y] * inv) at
// idx ? idx[i] : first + i
static __global__ void k_orb_state_read(OrbSrc src, const ulonglong2* __restrict__ rec, uint64_t N,
                                        double wr, double wi, double inv,
                                        const uint64_t* __restrict__ idx, uint64_t first,
                                        uint64_t count, double2* __restrict__ out) {
    const double2* C = src.get();
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t z = idx ? idx[i] : first + i;
        if (z >= N) {
            out[i] = make_double2(0.0, 0.0);
            continue;
        }
        const double2 v = orb_amp(C, rec, z);
        double re, im;
        cmul(wr, wi, __dmul_rn(v.x, inv), __dmul_rn(v.y, inv), re, im);
        out[i] = make_double2(re, im);
    }
}

// k_stage_read on a compressed state (post-Hadamard amplitudes of group x)
static __global__ void k_orb_stage_read(StageParams p, OrbSrc src, const ulonglong2* __restrict__ rec,
                                        int x, int gather, uint64_t first, uint64_t count,
                                        double2* __restrict__ out) {
    const double2* C = src.get();
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t z = first + i;
        if (z >= p.N) {
            out[i] = make_double2(0.0, 0.0);
            continue;
        }
        const double2 xa = orb_amp(C, rec, z);
        const double2 xs = gather ? orb_amp(C, rec, mulmod_shoup(z, p.m, p.m_sh, p.N)) : xa;
        double h0r, h0i, h1r, h1i;
        stage_pair(p.sc, xa, xs, h0r, h0i, h1r, h1i);
        out[i] = x ? make_double2(h1r, h1i) : make_double2(h0r, h0i);
    }
}

}  // namespace shs
