// The reference's per-gate ("step/measure") API on a device-resident state
// (SURVEY §8a rows A5, A6): ShardedState, init_state, apply_oracle,
// apply_phase, apply_hadamard_top, group_norm_squared, reset_top
// (/root/reference/proj/include/shorsim/statevector.hpp:20-133,
// proj/src/statevector.cpp:65-283) and the ExchangePlan views
// build_permutation_plan / plan_receive_lists / plan_send_lists
// (statevector.cpp:133-181), computed on the device.
//
// Unlike the engine (engine.cu), which keeps the compressed state of SURVEY F3,
// an shs_sv holds the full 2^n amplitudes, group x = top index bit, exactly as
// ShardedState does; the shard split only matters for the plan's views (the
// reference's shards are a layout of one address space, and so is ours: one
// contiguous device array). Every gate reproduces the reference's operation
// order with explicitly rounded fp64 (--fmad=false): amplitudes are
// bit-identical to the reference's after every gate.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/shorsim_b200.h"
#include "device_math.cuh"
#include "host_model.hpp"
#include "stage_kernels.cuh"

using namespace shs;

struct shs_sv {
    uint32_t n = 2, g = 1;
    uint64_t size = 0, group = 0;  // 2^n, 2^(n-1)
    int dev = 0;
    cudaStream_t stream = nullptr;
    double2* amp = nullptr;        // [2^n]: group 0 then group 1
    double2* scratch = nullptr;    // [2^(n-1)] apply_oracle snapshot (on first use)
    double* S = nullptr;           // [2][nb] block norms (on first use)
    double* d_out = nullptr;       // [2]
    uint64_t launches = 0;
};

namespace {

#define SV_CUDA(call)                                                                   \
    do {                                                                                \
        cudaError_t _e = (call);                                                        \
        if (_e != cudaSuccess)                                                          \
            return set_error(SHS_CUDA_ERROR, std::string(#call) + ": " +                \
                                                 cudaGetErrorString(_e));               \
    } while (0)

constexpr double kDegenerateMass = 1e-300;  // statevector.cpp:19

// make_shard_layout, statevector.cpp:65-72 (same messages)
int shard_layout(uint32_t n, uint32_t shard_count, uint32_t* g) {
    if (n < 2 || n > 33) return set_error(SHS_INVALID_ARGUMENT, "shard layout: need 2 <= n <= 33");
    if (shard_count < 2 || (shard_count & (shard_count - 1)) != 0)
        return set_error(SHS_INVALID_ARGUMENT,
                         "shard layout: shard count must be a power of two >= 2");
    uint32_t gg = 0;
    while ((1u << gg) < shard_count) ++gg;
    if (gg > n - 1)
        return set_error(SHS_INVALID_ARGUMENT, "shard layout: more shards than group states");
    *g = gg;
    return SHS_OK;
}

template <typename F>
int sv_guard(const shs_sv* sv, F&& f) {
    if (!sv) return set_error(SHS_INVALID_ARGUMENT, "null state");
    cudaError_t e = cudaSetDevice(sv->dev);
    if (e != cudaSuccess) return set_error(SHS_CUDA_ERROR, cudaGetErrorString(e));
    return f();
}

int grid_for(uint64_t n) { return static_cast<int>(std::min<uint64_t>((n + 255) / 256, 8192)); }

int launched(shs_sv* sv) {
    sv->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(SHS_CUDA_ERROR, std::string("launch: ") + cudaGetErrorString(e));
    return SHS_OK;
}

// apply_oracle's gather, statevector.cpp:231-244: out[y] = g1[a_inv y mod N], y < y_limit
__global__ void k_sv_gather(const double2* __restrict__ g1, double2* __restrict__ out,
                            uint64_t y_limit, uint64_t m, uint64_t m_sh, uint64_t N) {
    for (uint64_t y = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; y < y_limit;
         y += uint64_t(gridDim.x) * blockDim.x)
        out[y] = g1[mulmod_shoup(y, m, m_sh, N)];
}

// apply_phase, statevector.cpp:246-253: group 1 *= ph
__global__ void k_sv_phase(double2* __restrict__ g1, uint64_t count, double phr, double phi) {
    for (uint64_t y = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; y < count;
         y += uint64_t(gridDim.x) * blockDim.x) {
        double2 v = g1[y];
        double r, i;
        cmul(v.x, v.y, phr, phi, r, i);
        g1[y] = make_double2(r, i);
    }
}

// apply_hadamard_top, statevector.cpp:255-270
__global__ void k_sv_hadamard(double2* __restrict__ g0, double2* __restrict__ g1, uint64_t count) {
    for (uint64_t y = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; y < count;
         y += uint64_t(gridDim.x) * blockDim.x) {
        const double2 u = g0[y], v = g1[y];
        g0[y] = make_double2(__dmul_rn(__dadd_rn(u.x, v.x), kInvSqrt2),
                             __dmul_rn(__dadd_rn(u.y, v.y), kInvSqrt2));
        g1[y] = make_double2(__dmul_rn(__dsub_rn(u.x, v.x), kInvSqrt2),
                             __dmul_rn(__dsub_rn(u.y, v.y), kInvSqrt2));
    }
}

// group_norm_squared's fixed 256-blocks, statevector.cpp:95-117: S[x * nb + b]
// = sequential sum of std::norm over block b of group x (one thread per block,
// in index order)
__global__ void k_sv_block_norms(const double2* __restrict__ amp, uint64_t group, uint64_t nb,
                                 double* __restrict__ S) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < 2 * nb;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t x = i / nb, b = i - x * nb;
        const double2* p = amp + x * group + b * kBlock;
        const uint64_t rest = group - b * kBlock, len = rest < kBlock ? rest : kBlock;
        double s = 0.0;
        for (uint64_t k = 0; k < len; ++k) s = __dadd_rn(s, cnorm(p[k].x, p[k].y));
        S[i] = s;
    }
}

// reset_top, statevector.cpp:263-283: v = g_src * inv; g0 = a0 v; g1 = a1 v
__global__ void k_sv_reset(double2* __restrict__ g0, double2* __restrict__ g1, uint64_t count,
                           int src, double inv, double a0r, double a0i, double a1r, double a1i) {
    for (uint64_t y = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; y < count;
         y += uint64_t(gridDim.x) * blockDim.x) {
        const double2 s = src ? g1[y] : g0[y];
        const double vr = __dmul_rn(s.x, inv), vi = __dmul_rn(s.y, inv);
        double r0, i0, r1, i1;
        cmul(a0r, a0i, vr, vi, r0, i0);
        cmul(a1r, a1i, vr, vi, r1, i1);
        g0[y] = make_double2(r0, i0);
        g1[y] = make_double2(r1, i1);
    }
}

// ---- ExchangePlan on the device (statevector.cpp:133-181)

__global__ void k_plan_gather(uint64_t first, uint64_t count, uint64_t m, uint64_t m_sh,
                              uint64_t N, uint64_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = mulmod_shoup(first + i, m, m_sh, N);
}

// pair_counts[src_xrank][dst_xrank] += 1 for z < y_limit (statevector.cpp:149-152);
// a per-CTA shared histogram when the matrix is small
__global__ void k_plan_pair_counts(uint64_t y_limit, uint64_t m, uint64_t m_sh, uint64_t N,
                                   uint32_t xshift, uint32_t gs,
                                   unsigned long long* __restrict__ counts) {
    extern __shared__ unsigned long long hist[];
    const bool local = gs * gs <= 4096;
    if (local)
        for (uint32_t k = threadIdx.x; k < gs * gs; k += blockDim.x) hist[k] = 0;
    __syncthreads();
    for (uint64_t z = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; z < y_limit;
         z += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t src = mulmod_shoup(z, m, m_sh, N);
        const uint64_t cell = (src >> xshift) * gs + (z >> xshift);
        if (local) atomicAdd(&hist[cell], 1ull);
        else atomicAdd(&counts[cell], 1ull);
    }
    __syncthreads();
    if (local)
        for (uint32_t k = threadIdx.x; k < gs * gs; k += blockDim.x)
            if (hist[k]) atomicAdd(&counts[k], hist[k]);
}

// keys/values of one shard's lists: receive (dst_xrank fixed, z in its range):
// key = src shard, value = z - z_begin; send (src_xrank fixed, all z): flag =
// src in that shard, key = dst shard, value = src - src_xrank * shard_size
__global__ void k_plan_list_kv(uint64_t z0, uint64_t count, uint64_t m, uint64_t m_sh, uint64_t N,
                               uint32_t xshift, uint64_t shard_size, uint32_t xrank, int send,
                               uint32_t* __restrict__ keys, uint64_t* __restrict__ vals,
                               uint8_t* __restrict__ flags) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t z = z0 + i;
        const uint64_t src = mulmod_shoup(z, m, m_sh, N);
        if (send) {
            flags[i] = (src >> xshift) == xrank ? 1 : 0;
            keys[i] = static_cast<uint32_t>(z >> xshift);
            vals[i] = src - uint64_t(xrank) * shard_size;
        } else {
            flags[i] = 1;
            keys[i] = static_cast<uint32_t>(src >> xshift);
            vals[i] = i;
        }
    }
}

struct PlanArgs {
    uint64_t N, a_pow, a_inv, m_sh, y_limit;
    uint32_t n, g, xshift, gs;
    uint64_t shard_size;
    bool identity;
};

int plan_args(uint64_t a_pow, uint64_t N, uint32_t n, uint32_t shard_count, PlanArgs* pa) {
    uint32_t g = 0;
    int rc = shard_layout(n, shard_count, &g);
    if (rc) return rc;
    if (N < 2) return set_error(SHS_INVALID_ARGUMENT, "permutation plan: modulus >= 2");
    pa->N = N;
    pa->a_pow = a_pow % N;
    u64 inv = 0, gcd = 0;
    if (mod_inverse(pa->a_pow, N, &inv, &gcd) != SHS_OK)  // statevector.cpp:137 (throws)
        return set_error(SHS_NOT_INVERTIBLE, "not invertible: gcd(" + std::to_string(pa->a_pow) +
                                                 ", " + std::to_string(N) + ") = " +
                                                 std::to_string(gcd));
    pa->a_inv = inv;
    pa->m_sh = shoup(inv, N);
    pa->n = n;
    pa->g = g;
    pa->xshift = n - g;
    pa->gs = 1u << (g - 1);
    pa->shard_size = uint64_t(1) << (n - g);
    pa->y_limit = std::min<uint64_t>(N, uint64_t(1) << (n - 1));
    pa->identity = pa->a_pow == 1;
    return SHS_OK;
}

}  // namespace

extern "C" {

int shs_sv_create(uint32_t n, uint32_t shard_count, int32_t device, shs_sv** out) {
    if (!out) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    uint32_t g = 0;
    int rc = shard_layout(n, shard_count, &g);
    if (rc) return rc;
    auto* sv = new shs_sv;
    sv->n = n;
    sv->g = g;
    sv->size = uint64_t(1) << n;
    sv->group = sv->size >> 1;
    sv->dev = device;
    auto fail = [&](cudaError_t e, const char* what) {
        std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
        shs_sv_destroy(sv);
        return set_error(SHS_CUDA_ERROR, msg);
    };
    cudaError_t e;
    if ((e = cudaSetDevice(device)) != cudaSuccess) return fail(e, "cudaSetDevice");
    if ((e = cudaStreamCreateWithFlags(&sv->stream, cudaStreamNonBlocking)) != cudaSuccess)
        return fail(e, "cudaStreamCreate");
    if ((e = cudaMalloc(&sv->amp, sizeof(double2) * sv->size)) != cudaSuccess)
        return fail(e, "cudaMalloc(state)");
    if ((e = cudaMalloc(&sv->d_out, 2 * sizeof(double))) != cudaSuccess)
        return fail(e, "cudaMalloc");
    if ((e = cudaMemsetAsync(sv->amp, 0, sizeof(double2) * sv->size, sv->stream)) != cudaSuccess)
        return fail(e, "cudaMemset");
    if ((e = cudaStreamSynchronize(sv->stream)) != cudaSuccess) return fail(e, "sync");
    *out = sv;
    return SHS_OK;
}

void shs_sv_destroy(shs_sv* sv) {
    if (!sv) return;
    cudaSetDevice(sv->dev);
    if (sv->stream) cudaStreamSynchronize(sv->stream);
    cudaFree(sv->amp);
    cudaFree(sv->scratch);
    cudaFree(sv->S);
    cudaFree(sv->d_out);
    if (sv->stream) cudaStreamDestroy(sv->stream);
    delete sv;
}

int shs_sv_clone(const shs_sv* src, shs_sv** out) {
    return sv_guard(src, [&]() -> int {
        shs_sv* sv = nullptr;
        int rc = shs_sv_create(src->n, 1u << src->g, src->dev, &sv);
        if (rc) return rc;
        SV_CUDA(cudaStreamSynchronize(src->stream));
        cudaError_t e = cudaMemcpyAsync(sv->amp, src->amp, sizeof(double2) * src->size,
                                        cudaMemcpyDeviceToDevice, sv->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(sv->stream);
        if (e != cudaSuccess) {
            shs_sv_destroy(sv);
            return set_error(SHS_CUDA_ERROR, std::string("clone: ") + cudaGetErrorString(e));
        }
        *out = sv;
        return SHS_OK;
    });
}

int shs_sv_layout(const shs_sv* sv, uint32_t out[2]) {
    if (!sv || !out) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    out[0] = sv->n;
    out[1] = sv->g;
    return SHS_OK;
}

int shs_sv_read(const shs_sv* sv, uint64_t first, uint64_t count, double* host) {
    return sv_guard(sv, [&]() -> int {
        if (first > sv->size || count > sv->size - first)
            return set_error(SHS_INVALID_ARGUMENT, "amplitude index out of range");
        if (!count) return SHS_OK;
        SV_CUDA(cudaMemcpyAsync(host, sv->amp + first, sizeof(double2) * count,
                                cudaMemcpyDeviceToHost, sv->stream));
        SV_CUDA(cudaStreamSynchronize(sv->stream));
        return SHS_OK;
    });
}

int shs_sv_write(shs_sv* sv, uint64_t first, uint64_t count, const double* host) {
    return sv_guard(sv, [&]() -> int {
        if (first > sv->size || count > sv->size - first)
            return set_error(SHS_INVALID_ARGUMENT, "amplitude index out of range");
        if (!count) return SHS_OK;
        SV_CUDA(cudaMemcpyAsync(sv->amp + first, host, sizeof(double2) * count,
                                cudaMemcpyHostToDevice, sv->stream));
        SV_CUDA(cudaStreamSynchronize(sv->stream));
        return SHS_OK;
    });
}

// init_state, statevector.cpp:126-131 (on an existing state: zeroed first)
int shs_sv_init_state(shs_sv* sv, const double pair[4]) {
    return sv_guard(sv, [&]() -> int {
        if (!pair) return set_error(SHS_INVALID_ARGUMENT, "null argument");
        SV_CUDA(cudaMemsetAsync(sv->amp, 0, sizeof(double2) * sv->size, sv->stream));
        SV_CUDA(cudaMemcpyAsync(sv->amp + 1, pair, sizeof(double2), cudaMemcpyHostToDevice,
                                sv->stream));
        SV_CUDA(cudaMemcpyAsync(sv->amp + sv->group + 1, pair + 2, sizeof(double2),
                                cudaMemcpyHostToDevice, sv->stream));
        SV_CUDA(cudaStreamSynchronize(sv->stream));
        return SHS_OK;
    });
}

int shs_sv_apply_oracle(shs_sv* sv, uint64_t a_pow, uint64_t N) {
    return sv_guard(sv, [&]() -> int {
        PlanArgs pa{};
        int rc = plan_args(a_pow, N, sv->n, 1u << sv->g, &pa);
        if (rc) return rc;
        if (pa.identity) return SHS_OK;  // statevector.cpp:226
        if (N > sv->group)  // the reference's snapshot has 2^(n-1) entries (statevector.cpp:229)
            return set_error(SHS_INVALID_ARGUMENT, "apply_oracle: modulus exceeds the group size");
        if (!sv->scratch) SV_CUDA(cudaMalloc(&sv->scratch, sizeof(double2) * sv->group));
        double2* g1 = sv->amp + sv->group;
        k_sv_gather<<<grid_for(pa.y_limit), 256, 0, sv->stream>>>(g1, sv->scratch, pa.y_limit,
                                                                 pa.a_inv, pa.m_sh, N);
        if ((rc = launched(sv))) return rc;
        SV_CUDA(cudaMemcpyAsync(g1, sv->scratch, sizeof(double2) * pa.y_limit,
                                cudaMemcpyDeviceToDevice, sv->stream));
        SV_CUDA(cudaStreamSynchronize(sv->stream));
        return SHS_OK;
    });
}

int shs_sv_apply_phase(shs_sv* sv, uint32_t cbit, uint64_t lo, uint64_t hi) {
    return sv_guard(sv, [&]() -> int {
        const double phi = stage_phase(cbit, (u128{hi} << 64) | lo);
        if (phi == 0.0) return SHS_OK;  // statevector.cpp:248
        const double phr = 1.0 * std::cos(phi), phs = 1.0 * std::sin(phi);  // std::polar
        k_sv_phase<<<grid_for(sv->group), 256, 0, sv->stream>>>(sv->amp + sv->group, sv->group,
                                                               phr, phs);
        int rc = launched(sv);
        if (rc) return rc;
        SV_CUDA(cudaStreamSynchronize(sv->stream));
        return SHS_OK;
    });
}

int shs_sv_apply_hadamard_top(shs_sv* sv) {
    return sv_guard(sv, [&]() -> int {
        k_sv_hadamard<<<grid_for(sv->group), 256, 0, sv->stream>>>(sv->amp, sv->amp + sv->group,
                                                                  sv->group);
        int rc = launched(sv);
        if (rc) return rc;
        SV_CUDA(cudaStreamSynchronize(sv->stream));
        return SHS_OK;
    });
}

// out[0] = group_norm_squared(0), out[1] = group_norm_squared(1): fixed
// 256-blocks, then the reference's sequential Kahan over the non-zero blocks
// (combine_blocks, statevector.cpp:32-40), bit-identical
int shs_sv_group_norms(const shs_sv* csv, double out[2]) {
    auto* sv = const_cast<shs_sv*>(csv);
    return sv_guard(sv, [&]() -> int {
        if (!out) return set_error(SHS_INVALID_ARGUMENT, "null argument");
        const uint64_t nb = (sv->group + kBlock - 1) / kBlock;
        if (!sv->S) SV_CUDA(cudaMalloc(&sv->S, sizeof(double) * 2 * nb));
        k_sv_block_norms<<<grid_for(2 * nb), 256, 0, sv->stream>>>(sv->amp, sv->group, nb, sv->S);
        int rc = launched(sv);
        if (rc) return rc;
        k_finalize<<<1, kFinalizeThreads, 0, sv->stream>>>(nullptr, 0, sv->S, nb, 1, sv->d_out);
        if ((rc = launched(sv))) return rc;
        SV_CUDA(cudaMemcpyAsync(out, sv->d_out, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                                sv->stream));
        SV_CUDA(cudaStreamSynchronize(sv->stream));
        return SHS_OK;
    });
}

int shs_sv_reset_top(shs_sv* sv, int32_t bit, int32_t error_branch, const double reinit[4],
                     double p_source) {
    return sv_guard(sv, [&]() -> int {
        if (!reinit) return set_error(SHS_INVALID_ARGUMENT, "null argument");
        if (p_source < kDegenerateMass)  // statevector.cpp:265-266
            return set_error(SHS_DEGENERATE_BRANCH,
                             "reset_top: selected branch has no probability mass");
        const int src = error_branch ? 1 - bit : bit;
        const double inv = 1.0 / std::sqrt(p_source);
        k_sv_reset<<<grid_for(sv->group), 256, 0, sv->stream>>>(
            sv->amp, sv->amp + sv->group, sv->group, src, inv, reinit[0], reinit[1], reinit[2],
            reinit[3]);
        int rc = launched(sv);
        if (rc) return rc;
        SV_CUDA(cudaStreamSynchronize(sv->stream));
        return SHS_OK;
    });
}

uint64_t shs_sv_launch_count(const shs_sv* sv) { return sv ? sv->launches : 0; }

// ---- ExchangePlan (statevector.cpp:133-181), on the device

int shs_plan_build(uint64_t a_pow, uint64_t N, uint32_t n, uint32_t shard_count, int32_t device,
                   uint64_t* a_inv, int32_t* identity, uint64_t* y_limit, uint64_t* gather,
                   uint64_t* pair_counts) {
    PlanArgs pa{};
    int rc = plan_args(a_pow, N, n, shard_count, &pa);
    if (rc) return rc;
    if (pa.gs > 4096) return set_error(SHS_INVALID_ARGUMENT, "permutation plan: > 4096 group shards");
    if (a_inv) *a_inv = pa.a_inv;
    if (identity) *identity = pa.identity ? 1 : 0;
    if (y_limit) *y_limit = pa.y_limit;
    if (!gather && !pair_counts) return SHS_OK;
    if (cudaSetDevice(device) != cudaSuccess) return set_error(SHS_CUDA_ERROR, "cudaSetDevice");
    cudaStream_t st = nullptr;
    SV_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    uint64_t* dg = nullptr;
    unsigned long long* dc = nullptr;
    const size_t cells = size_t(pa.gs) * pa.gs;
    auto done = [&](int code) {
        if (dg) cudaFreeAsync(dg, st);
        if (dc) cudaFreeAsync(dc, st);
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
        return code;
    };
    if (gather) {
        if (cudaMallocAsync(&dg, sizeof(uint64_t) * std::max<uint64_t>(pa.y_limit, 1), st) != cudaSuccess)
            return done(set_error(SHS_CUDA_ERROR, "cudaMalloc(gather)"));
        k_plan_gather<<<grid_for(pa.y_limit), 256, 0, st>>>(0, pa.y_limit, pa.a_inv, pa.m_sh, N, dg);
        cudaMemcpyAsync(gather, dg, sizeof(uint64_t) * pa.y_limit, cudaMemcpyDeviceToHost, st);
    }
    if (pair_counts) {
        if (cudaMallocAsync(&dc, sizeof(unsigned long long) * cells, st) != cudaSuccess)
            return done(set_error(SHS_CUDA_ERROR, "cudaMalloc(pair counts)"));
        cudaMemsetAsync(dc, 0, sizeof(unsigned long long) * cells, st);
        const size_t sm = cells <= 4096 ? cells * sizeof(unsigned long long) : 0;
        k_plan_pair_counts<<<grid_for(pa.y_limit), 256, sm, st>>>(pa.y_limit, pa.a_inv, pa.m_sh, N,
                                                                 pa.xshift, pa.gs, dc);
        cudaMemcpyAsync(pair_counts, dc, sizeof(unsigned long long) * cells, cudaMemcpyDeviceToHost,
                        st);
    }
    cudaError_t e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return done(set_error(SHS_CUDA_ERROR, cudaGetErrorString(e)));
    return done(SHS_OK);
}

// plan_receive_lists (send = 0) / plan_send_lists (send = 1) for group shard
// xrank: counts[peer] (group_shards entries) and the local indices grouped by
// peer in ascending peer order, each group in the reference's z order (a
// stable radix sort by peer on the device). indices needs shard_size entries.
int shs_plan_lists(uint64_t a_pow, uint64_t N, uint32_t n, uint32_t shard_count, uint32_t xrank,
                   int32_t send, int32_t device, uint64_t* counts, uint64_t* indices) {
    PlanArgs pa{};
    int rc = plan_args(a_pow, N, n, shard_count, &pa);
    if (rc) return rc;
    if (xrank >= pa.gs) return set_error(SHS_INVALID_ARGUMENT, "plan lists: shard out of range");
    if (!counts || !indices) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    std::fill(counts, counts + pa.gs, 0);
    uint64_t z0 = 0, cnt = pa.y_limit;
    if (!send) {  // the receiver's z range (statevector.cpp:160-163)
        z0 = uint64_t(xrank) * pa.shard_size;
        const uint64_t z1 = std::min(pa.y_limit, z0 + pa.shard_size);
        cnt = z0 < z1 ? z1 - z0 : 0;
    }
    if (!cnt) return SHS_OK;
    if (cudaSetDevice(device) != cudaSuccess) return set_error(SHS_CUDA_ERROR, "cudaSetDevice");
    cudaStream_t st = nullptr;
    SV_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    uint32_t *k0 = nullptr, *k1 = nullptr, *k2 = nullptr;
    uint64_t *v0 = nullptr, *v1 = nullptr, *v2 = nullptr;
    uint8_t* fl = nullptr;
    int* nsel = nullptr;
    void* tmp = nullptr;
    std::vector<void*> owned;
    auto alloc = [&](void** p, size_t bytes) {
        if (cudaMallocAsync(p, std::max<size_t>(bytes, 8), st) != cudaSuccess) return false;
        owned.push_back(*p);
        return true;
    };
    auto done = [&](int code) {
        for (void* p : owned) cudaFreeAsync(p, st);
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
        return code;
    };
    if (!alloc((void**)&k0, 4 * cnt) || !alloc((void**)&k1, 4 * cnt) || !alloc((void**)&k2, 4 * cnt) ||
        !alloc((void**)&v0, 8 * cnt) || !alloc((void**)&v1, 8 * cnt) || !alloc((void**)&v2, 8 * cnt) ||
        !alloc((void**)&fl, cnt) || !alloc((void**)&nsel, sizeof(int)))
        return done(set_error(SHS_CUDA_ERROR, "cudaMalloc(plan lists)"));
    k_plan_list_kv<<<grid_for(cnt), 256, 0, st>>>(z0, cnt, pa.a_inv % N, shoup(pa.a_inv % N, N), N,
                                                  pa.xshift, pa.shard_size, xrank, send, k0, v0, fl);
    // keep the flagged entries in z order, then a stable sort by peer shard
    size_t b1 = 0, b2 = 0, b3 = 0;
    const int ic = static_cast<int>(cnt);
    cub::DeviceSelect::Flagged(nullptr, b1, k0, fl, k1, nsel, ic, st);
    cub::DeviceSelect::Flagged(nullptr, b2, v0, fl, v1, nsel, ic, st);
    int bits = 1;
    while ((1u << bits) < pa.gs) ++bits;
    cub::DeviceRadixSort::SortPairs(nullptr, b3, k1, k2, v1, v2, ic, 0, bits, st);
    if (!alloc(&tmp, std::max(b1, std::max(b2, b3))))
        return done(set_error(SHS_CUDA_ERROR, "cudaMalloc(cub scratch)"));
    size_t tb = std::max(b1, std::max(b2, b3));
    cub::DeviceSelect::Flagged(tmp, tb, k0, fl, k1, nsel, ic, st);
    tb = std::max(b1, std::max(b2, b3));
    cub::DeviceSelect::Flagged(tmp, tb, v0, fl, v1, nsel, ic, st);
    int hsel = 0;
    cudaMemcpyAsync(&hsel, nsel, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return done(set_error(SHS_CUDA_ERROR, cudaGetErrorString(e)));
    tb = std::max(b1, std::max(b2, b3));
    cub::DeviceRadixSort::SortPairs(tmp, tb, k1, k2, v1, v2, hsel, 0, bits, st);
    std::vector<uint32_t> hk(hsel);
    cudaMemcpyAsync(hk.data(), k2, 4 * size_t(hsel), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(indices, v2, 8 * size_t(hsel), cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return done(set_error(SHS_CUDA_ERROR, cudaGetErrorString(e)));
    for (uint32_t k : hk) counts[k]++;
    return done(SHS_OK);
}

}  // extern "C"
