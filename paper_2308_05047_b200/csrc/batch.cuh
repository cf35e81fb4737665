// Batched small-N engine (§8 f1): whole iterative-Shor runs on the device, one
// CTA per (seed, bitstring index), for the campaign regime of configs 1-2
// (N = 15 ... a few thousand; thousands of shots per problem, e.g. acceptance
// criterion 2's 100 000 runs of N = 15 and run_problem's M shots per base,
// proj/src/harness.cpp:109-148). The whole state lives in shared memory; the
// host is not involved between stages.
//
// Bit-exactness with the per-stage engine (and so with the reference):
//   * the stage arithmetic is the same stage_pair();
//   * block partials are the in-order 256-block folds, combined by the
//     reference's sequential Kahan (statevector.cpp:32-40) — N is small;
//   * Philox4x32-10 and the measurement rules are restated on the device with
//     explicitly rounded fp64 ops (rng.hpp:16-83, statevector.cpp:236-256,
//     noise.cpp:128-151);
//   * the phase e^{i pi prefix 2^-s} is NOT evaluated on the device (CUDA's
//     cos/sin are not glibc's): the host tabulates std::polar(1, stage_phase)
//     for every (s, observed prefix) once per engine (t <= kBatchMaxT).
#pragma once

#include "device_math.cuh"
#include "measure.cuh"

namespace shs {

constexpr uint32_t kBatchMaxT = 20;      // phase table of 2^t entries (16 MB at t = 20)
constexpr uint64_t kBatchMaxN = 4096;    // 64 KB of shared state per CTA
constexpr int kBatchThreads = 128;  // CTA size cap; small N use one warp per run

struct BatchParams {
    uint64_t N;
    uint32_t t;
    uint64_t seed;
    uint64_t idx0;
    uint32_t count;
    const uint64_t* a_pows;   // [t]
    const uint64_t* a_invs;   // [t]
    const uint64_t* a_invsh;  // [t] Shoup companions
    const double2* phase;     // [2^t - 1]: (cos, sin) of stage s, prefix p at (1 << s) - 1 + p
    double w0r, w0i, w1r, w1i;
    int kind;                 // SHS_ERR_*
    double delta, px, py;
    int check_norms;
    uint64_t* j_out;          // [count][2]
    uint64_t* js_out;         // [count][2]
    double* p1_out;           // [count][t] or null
    int32_t* bits_out;        // [count][t][4] or null: sampled, observed, flip, error branch
    int32_t* status;          // [count]: 0 ok, SHS_ERROR, SHS_DEGENERATE_BRANCH
};

__device__ __forceinline__ double kahan_blocks(const double* x, int n) {
    double s = 0, c = 0;
    for (int i = 0; i < n; ++i) {
        if (x[i] != 0.0) {
            const double y = __dsub_rn(x[i], c);
            const double t = __dadd_rn(s, y);
            c = __dsub_rn(__dsub_rn(t, s), y);
            s = t;
        }
    }
    return s;
}

static __global__ void __launch_bounds__(kBatchThreads) k_batch_runs(BatchParams bp) {
    // blockDim.x = batch_threads(N): 32..128
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint64_t N = bp.N;
    const int nb = static_cast<int>((N + kBlock - 1) / kBlock);
    double2* X = reinterpret_cast<double2*>(smem_raw);
    double2* Y = X + N;
    double* nrm = reinterpret_cast<double*>(Y + N);  // [2][nb * kBlock] (zero-padded)
    double* bsum = nrm + 2 * nb * kBlock;             // [2][nb]
    __shared__ double sh_p0, sh_p1, sh_inv_next;
    __shared__ int sh_sel, sh_stop;
    const int tid = threadIdx.x;

    for (uint32_t run = blockIdx.x; run < bp.count; run += gridDim.x) {
        const uint64_t idx = bp.idx0 + run;
        const uint32_t idx32 = static_cast<uint32_t>(idx);  // statevector.cpp:377
        bool e1 = true;
        double inv = 1.0;
        unsigned __int128 observed = 0, sampled = 0;
        for (uint64_t i = tid; i < 2 * uint64_t(nb) * kBlock; i += blockDim.x) nrm[i] = 0.0;
        if (tid == 0) sh_stop = 0;
        __syncthreads();
        for (uint32_t s = 0; s < bp.t; ++s) {
            const uint64_t A = bp.a_pows[s];
            const bool gather = A != 1;
            const uint64_t prefix = static_cast<uint64_t>(observed);
            const double2 ph = s == 0 ? make_double2(1.0, 0.0)
                                      : bp.phase[((uint64_t(1) << s) - 1) + prefix];
            StageScalars sc;
            sc.w0r = bp.w0r;
            sc.w0i = bp.w0i;
            sc.w1r = bp.w1r;
            sc.w1i = bp.w1i;
            sc.phr = ph.x;
            sc.phi = ph.y;
            sc.inv = inv;
            const bool phi_nonzero = s != 0 && prefix != 0;  // stage_phase(s, p) == 0 iff p == 0
            sc.phase_mul = (gather || phi_nonzero) ? 1 : 0;
            const uint64_t m = bp.a_invs[s], msh = bp.a_invsh[s];
            // pass 1: |h0|^2, |h1|^2 of every z
            for (uint64_t z = tid; z < N; z += blockDim.x) {
                const uint64_t src = gather ? mulmod_shoup(z, m, msh, N) : z;
                const double2 xa = e1 ? make_double2(z == 1 ? 1.0 : 0.0, 0.0) : X[z];
                const double2 xs = e1 ? make_double2(src == 1 ? 1.0 : 0.0, 0.0) : X[src];
                double h0r, h0i, h1r, h1i;
                stage_pair(sc, xa, xs, h0r, h0i, h1r, h1i);
                nrm[z] = cnorm(h0r, h0i);
                nrm[nb * kBlock + z] = cnorm(h1r, h1i);
            }
            __syncthreads();
            // in-order 256-block folds over the live amplitudes (statevector.cpp:354-370)
            if (tid < 2 * nb) {
                const int g = tid / nb, b = tid % nb;
                const double* row = nrm + g * nb * kBlock + b * kBlock;
                const int live = static_cast<int>(min(uint64_t(kBlock), N - uint64_t(b) * kBlock));
                double acc = 0.0;
                for (int i = 0; i < live; ++i) acc = __dadd_rn(acc, row[i]);
                bsum[g * nb + b] = acc;
            }
            __syncthreads();
            if (tid == 0) {
                const double p0 = kahan_blocks(bsum, nb);
                const double p1 = kahan_blocks(bsum + nb, nb);
                sh_p0 = p0;
                sh_p1 = p1;
                MeasureCfg mc{bp.seed, idx32, bp.kind, bp.delta, bp.px, bp.py, bp.check_norms};
                const DevMeasure mr = measure_dev(p0, p1, mc, s, s + 1 < bp.t);
                const int sbit = mr.sbit, obit = mr.obit, flip = mr.flip, ebranch = mr.ebranch;
                const int status = mr.status;
                if (bp.p1_out) bp.p1_out[uint64_t(run) * bp.t + s] = p1;
                if (bp.bits_out) {
                    int32_t* o = bp.bits_out + (uint64_t(run) * bp.t + s) * 4;
                    o[0] = sbit;
                    o[1] = obit;
                    o[2] = flip;
                    o[3] = ebranch;
                }
                observed |= static_cast<unsigned __int128>(obit) << s;
                sampled |= static_cast<unsigned __int128>(sbit) << s;
                sh_sel = mr.src_group;
                sh_inv_next = __ddiv_rn(1.0, __dsqrt_rn(mr.p_src));
                if (status) {
                    bp.status[run] = status;
                    sh_stop = 1;
                }
            }
            __syncthreads();
            // every thread keeps the same prefix bits: broadcast through shared memory
            {
                __shared__ unsigned long long sh_obs[2], sh_smp[2];
                if (tid == 0) {
                    sh_obs[0] = static_cast<unsigned long long>(observed);
                    sh_obs[1] = static_cast<unsigned long long>(observed >> 64);
                    sh_smp[0] = static_cast<unsigned long long>(sampled);
                    sh_smp[1] = static_cast<unsigned long long>(sampled >> 64);
                }
                __syncthreads();
                observed = (static_cast<unsigned __int128>(sh_obs[1]) << 64) | sh_obs[0];
                sampled = (static_cast<unsigned __int128>(sh_smp[1]) << 64) | sh_smp[0];
            }
            if (sh_stop) break;
            if (s + 1 < bp.t) {
                // collapse (statevector.cpp:384-401): Y = h_sel, then swap
                const int sel = sh_sel;
                for (uint64_t z = tid; z < N; z += blockDim.x) {
                    const uint64_t src = gather ? mulmod_shoup(z, m, msh, N) : z;
                    const double2 xa = e1 ? make_double2(z == 1 ? 1.0 : 0.0, 0.0) : X[z];
                    const double2 xs = e1 ? make_double2(src == 1 ? 1.0 : 0.0, 0.0) : X[src];
                    double h0r, h0i, h1r, h1i;
                    stage_pair(sc, xa, xs, h0r, h0i, h1r, h1i);
                    Y[z] = sel ? make_double2(h1r, h1i) : make_double2(h0r, h0i);
                }
                __syncthreads();
                double2* tmp = X;
                X = Y;
                Y = tmp;
                e1 = false;
                inv = sh_inv_next;
            }
        }
        if (tid == 0) {
            if (!sh_stop) {
                unsigned __int128 j = observed;
                if (bp.kind == SHS_ERR_BITFLIP)  // noise.cpp:147-151, stream (seed, idx, 0, bitflip)
                    for (uint32_t i = 0; i < bp.t; ++i)
                        if (rng_double_dev(bp.seed, idx32, 0, 1, i) < bp.delta)
                            j ^= static_cast<unsigned __int128>(1) << i;
                bp.j_out[2 * uint64_t(run)] = static_cast<uint64_t>(j);
                bp.j_out[2 * uint64_t(run) + 1] = static_cast<uint64_t>(j >> 64);
                if (bp.js_out) {
                    bp.js_out[2 * uint64_t(run)] = static_cast<uint64_t>(sampled);
                    bp.js_out[2 * uint64_t(run) + 1] = static_cast<uint64_t>(sampled >> 64);
                }
                bp.status[run] = 0;
            }
            sh_stop = 0;
        }
        // X/Y may have been swapped an odd number of times: restore the base layout
        X = reinterpret_cast<double2*>(smem_raw);
        Y = X + N;
        __syncthreads();
    }
}

inline int batch_threads(uint64_t N) {
    return N <= 64 ? 32 : (N <= 256 ? 64 : kBatchThreads);
}

inline size_t batch_smem_bytes(uint64_t N) {
    const uint64_t nb = (N + kBlock - 1) / kBlock;
    return 2 * N * sizeof(double2) + 2 * nb * kBlock * sizeof(double) + 2 * nb * sizeof(double);
}

}  // namespace shs
