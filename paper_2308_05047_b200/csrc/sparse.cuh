// Sparse prefix of a run: the first stages on the support of the state only.
//
// From the run start e_1, stage s can only make amplitudes at z and at
// A_s z nonzero, so the state entering stage s (s >= 1) lives on
//     supp_s = { A_{s-1}^k mod N : k < 2^s }      (A_{s-1} = A_s^2)
// and stage s maps orbit index k to the two new indices 2k (z = A_{s-1}^k: the
// direct term, the gathered term is outside the support) and 2k+1
// (z = A_{s-1}^k A_s: the gathered term, the direct term is outside). The
// engine keeps (z, value) pairs in orbit order while 2^(s+1) <= N / 16 and the
// orbit does not wrap (the host proves ord(A) >= 2^(s+1) once per engine by a
// baby-step giant-step search), then scatters them into the dense buffer.
//
// Exactness: every amplitude outside the support is exactly zero, its |h|^2
// is +0.0 and adding +0.0 leaves the reference's in-order 256-block sums
// unchanged, so each block partial is the in-z-order fold of the support
// norms that fall in it (the pairs are sorted by z, CUB radix sort) and p0/p1
// (the exact sum of the partials) are bit-identical to the dense passes'. The
// only difference is invisible to every output: a stored zero that the dense
// pass would have written as -0.0 is +0.0 here.
#pragma once

#include <cub/cub.cuh>

#include "device_math.cuh"
#include "measure.cuh"
#include "stage_kernels.cuh"

namespace shs {

constexpr int kSparseThreads = 256;

struct SparseParams {
    const uint64_t* Zo;   // [Ko] support entering the stage (orbit order)
    const double2* Vo;    // [Ko] its amplitudes (sel)
    uint64_t Ko;
    uint64_t A, A_sh, N;  // stage multiplier (z -> A z is the gathered image)
    StageScalars sc;      // host scalars (stage 0) ...
    const DevStage* dev;  // ... or the device slot (later stages)
    uint64_t* Zn;         // [2 Ko] support after the stage (orbit order)
    double2* Vn;          // [2 Ko] collapse output
    double2* nrm;         // [2 Ko] (|h0|^2, |h1|^2) per new index (the sort payload)
};

__device__ __forceinline__ StageScalars sparse_scalars(const SparseParams& p) {
    return p.dev ? p.dev->sc : p.sc;
}

// run start: supp = {1}, value 1 (the implicit e_1 with inv = 1)
static __global__ void k_sparse_init(uint64_t* Z, double2* V) {
    Z[0] = 1;
    V[0] = make_double2(1.0, 0.0);
}

// probs side: the new support (orbit order), the sort payload and both norms
static __global__ void __launch_bounds__(kSparseThreads) k_sparse_expand(SparseParams p) {
    const StageScalars sc = sparse_scalars(p);
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < p.Ko;
         k += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t z0 = p.Zo[k];
        const double2 v = p.Vo[k], zero = make_double2(0.0, 0.0);
        double h0r, h0i, h1r, h1i;
        stage_pair(sc, v, zero, h0r, h0i, h1r, h1i);  // z0: direct term only
        p.nrm[2 * k] = make_double2(cnorm(h0r, h0i), cnorm(h1r, h1i));
        stage_pair(sc, zero, v, h0r, h0i, h1r, h1i);  // A z0: gathered term only
        p.nrm[2 * k + 1] = make_double2(cnorm(h0r, h0i), cnorm(h1r, h1i));
        p.Zn[2 * k] = z0;
        p.Zn[2 * k + 1] = mulmod_shoup(z0, p.A, p.A_sh, p.N);
    }
}

// Block partials over the z-sorted support (norm pairs sorted along): the
// first element of every 256-block run folds the run in order (0.0 + x + ...);
// exact per-CTA digits.
static __global__ void __launch_bounds__(kSparseThreads)
    k_sparse_fold(const uint64_t* __restrict__ zs, const double2* __restrict__ nrm, uint64_t Kn,
                  unsigned long long* partials) {
    __shared__ unsigned long long digits[2][kDigits];
    const int tid = threadIdx.x;
    for (int i = tid; i < 2 * kDigits; i += blockDim.x) (&digits[0][0])[i] = 0ull;
    __syncthreads();
    DigitWindow w0, w1;
    window_reset(w0);
    window_reset(w1);
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + tid; i < Kn;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t b = zs[i] >> 8;
        if (i > 0 && (zs[i - 1] >> 8) == b) continue;  // not the first of its block
        double s0 = 0.0, s1 = 0.0;
        for (uint64_t j = i; j < Kn && (zs[j] >> 8) == b; ++j) {
            const double2 n = nrm[j];
            s0 = __dadd_rn(s0, n.x);
            s1 = __dadd_rn(s1, n.y);
        }
        window_add(w0, s0, digits[0]);
        window_add(w1, s1, digits[1]);
    }
    window_flush(w0, digits[0]);
    window_flush(w1, digits[1]);
    __syncthreads();
    write_cta_digits(digits, partials + uint64_t(blockIdx.x) * 2 * kDigits, tid);
}

// collapse side: the kept group's amplitudes in orbit order
static __global__ void __launch_bounds__(kSparseThreads) k_sparse_collapse(SparseParams p, int sel_host) {
    const StageScalars sc = sparse_scalars(p);
    const int sel = p.dev ? p.dev->sel : sel_host;
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < p.Ko;
         k += uint64_t(gridDim.x) * blockDim.x) {
        const double2 v = p.Vo[k], zero = make_double2(0.0, 0.0);
        double h0r, h0i, h1r, h1i;
        stage_pair(sc, v, zero, h0r, h0i, h1r, h1i);
        p.Vn[2 * k] = sel ? make_double2(h1r, h1i) : make_double2(h0r, h0i);
        stage_pair(sc, zero, v, h0r, h0i, h1r, h1i);
        p.Vn[2 * k + 1] = sel ? make_double2(h1r, h1i) : make_double2(h0r, h0i);
    }
}

// the dense state (zeroed beforehand) from the support
static __global__ void k_sparse_scatter(const uint64_t* __restrict__ Z,
                                        const double2* __restrict__ V, uint64_t K,
                                        double2* __restrict__ X) {
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < K;
         k += uint64_t(gridDim.x) * blockDim.x)
        X[Z[k]] = V[k];
}

// one shard's dense sel (zeroed beforehand) from the support: the points in
// [lo, hi), at local index z - lo (the sharded engine's materialisation)
static __global__ void k_sparse_scatter_range(const uint64_t* __restrict__ Z,
                                              const double2* __restrict__ V, uint64_t K,
                                              uint64_t lo, uint64_t hi, double2* __restrict__ X) {
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < K;
         k += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t z = Z[k];
        if (z >= lo && z < hi) X[z - lo] = V[k];
    }
}

}  // namespace shs
