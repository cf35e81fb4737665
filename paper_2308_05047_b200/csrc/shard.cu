// Sharded engine (§8e): one shard of the iterative-Shor state per GPU.
//
// Shard q of G owns global indices [q*S, min(N, (q+1)*S)) of `sel`, S a
// multiple of 256 (so the reference's 256-blocks, and with them the block
// partials and the exact accumulator, are shard-local). A non-identity stage is
//   exchange  P = sel o src over all shards (exchange.cuh: tiled pull/push over
//             peer pointers, or a direct pull without a tile plan)
//   probs     shard-local h0/h1 from (sel, P), block partials, exact digits
//             -> the driver allreduces the 80 integer digits (exact and
//             order-independent: identical p0/p1 for every G)
//   collapse  shard-local, in place over P, which becomes the next sel.
// Identity stages and the first stage (implicit |1>) need no exchange.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/shorsim_b200.h"
#include "device_math.cuh"
#include "exchange.cuh"
#include "host_model.hpp"
#include "stage_kernels.cuh"
#include "tile_plan.hpp"
#include "tiled.cuh"

using namespace shs;

struct shs_shard {
    shs_problem prob{};
    shs_error err{};
    shs_options opt{};
    uint64_t N = 0, S = 0, lo = 0, hi = 0, nloc = 0, nb = 0, nchunks = 0;
    uint32_t t = 0, rank = 0, G = 1;
    std::vector<u64> a_pows, a_invs;
    std::vector<TilePlanHost> plans;
    double w[4] = {0, 0, 0, 0};
    int dev = 0, num_sms = 148, grid_cap = 0;
    cudaStream_t stream = nullptr;
    double2* buf[2] = {nullptr, nullptr};
    double2* peer[kMaxShards][2] = {};
    bool peer_ipc[kMaxShards] = {};
    int parity = 0;  // sel = buf[parity], P = buf[parity ^ 1] (same on every shard)
    double* Sb = nullptr;
    unsigned long long* partials = nullptr;
    unsigned long long* d_digits = nullptr;
    unsigned long long* h_digits = nullptr;
    bool e1 = true;
    double inv = 1.0;
    bool pending = false;
    int exchanged = -1;  // stage whose exchange was issued
    uint32_t ps = 0;
    StageScalars sc{};
    // instrumentation
    bool timing = false;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    double kms[3] = {0, 0, 0};
    uint64_t klaunch[3] = {0, 0, 0};
    uint64_t launches = 0;
};

namespace {

#define SHD_CUDA(call)                                                                  \
    do {                                                                                \
        cudaError_t _e = (call);                                                        \
        if (_e != cudaSuccess)                                                          \
            return set_error(SHS_CUDA_ERROR, std::string(#call) + ": " +                \
                                                 cudaGetErrorString(_e));               \
    } while (0)

constexpr double kNormTolerance = 1e-9;

template <typename F>
int shard_guard(shs_shard* sh, F&& f) {
    if (!sh) return set_error(SHS_INVALID_ARGUMENT, "null shard");
    cudaError_t err = cudaSetDevice(sh->dev);
    if (err != cudaSuccess) return set_error(SHS_CUDA_ERROR, cudaGetErrorString(err));
    return f();
}

template <typename F>
int shard_launch(shs_shard* sh, int kind, F&& f) {
    static const char* kNames[3] = {"shs shard probs", "shs shard exchange", "shs shard collapse"};
    nvtxRangePushA(kNames[kind]);
    struct Pop {
        ~Pop() { nvtxRangePop(); }
    } pop;
    if (sh->timing) cudaEventRecord(sh->ev[0], sh->stream);
    f();
    cudaError_t err = cudaGetLastError();
    if (sh->timing) {
        cudaEventRecord(sh->ev[1], sh->stream);
        cudaEventSynchronize(sh->ev[1]);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, sh->ev[0], sh->ev[1]);
        sh->kms[kind] += ms;
        sh->klaunch[kind] += 1;
    }
    sh->launches++;
    if (err != cudaSuccess)
        return set_error(SHS_CUDA_ERROR, std::string("kernel launch: ") + cudaGetErrorString(err));
    return SHS_OK;
}

StageParams local_params(const shs_shard* sh, uint32_t s, bool use_p) {
    StageParams p{};
    p.X = sh->buf[sh->parity];
    p.Xs = use_p ? sh->buf[sh->parity ^ 1] : nullptr;
    p.Y = sh->buf[sh->parity ^ 1];
    p.N = sh->N;
    p.z0 = sh->lo;
    p.zend = sh->hi;
    p.m = sh->a_invs[s];
    p.m_sh = sh->a_pows[s] != 1 ? shoup(p.m, sh->N) : 0;
    p.m_step = sh->a_pows[s] != 1 ? mulmod(p.m, kBlock, sh->N) : 0;
    p.sc = sh->sc;
    p.S = sh->Sb;
    p.nb = sh->nb;
    p.partials = sh->partials;
    p.nchunks = sh->nchunks;
    return p;
}

ShardMap shard_map(const shs_shard* sh) {
    ShardMap m{};
    m.S = sh->S;
    m.S_inv = ~uint64_t(0) / sh->S;
    m.G = static_cast<int>(sh->G);
    for (uint32_t q = 0; q < sh->G; ++q) {
        m.src[q] = sh->peer[q][sh->parity];
        m.dst[q] = sh->peer[q][sh->parity ^ 1];
    }
    return m;
}

int grid(const shs_shard* sh) {
    return static_cast<int>(std::min<uint64_t>(sh->nchunks, static_cast<uint64_t>(sh->grid_cap)));
}

void release(shs_shard* sh) {
    if (!sh) return;
    cudaSetDevice(sh->dev);
    if (sh->stream) cudaStreamSynchronize(sh->stream);
    for (uint32_t q = 0; q < sh->G; ++q)
        if (sh->peer_ipc[q])
            for (int b = 0; b < 2; ++b)
                if (sh->peer[q][b]) cudaIpcCloseMemHandle(sh->peer[q][b]);
    cudaFree(sh->buf[0]);
    cudaFree(sh->buf[1]);
    cudaFree(sh->Sb);
    cudaFree(sh->partials);
    cudaFree(sh->d_digits);
    if (sh->h_digits) cudaFreeHost(sh->h_digits);
    for (auto& e : sh->ev)
        if (e) cudaEventDestroy(e);
    if (sh->stream) cudaStreamDestroy(sh->stream);
    delete sh;
}

bool stage_needs_exchange(const shs_shard* sh, uint32_t s) {
    return !sh->e1 && sh->a_pows[s] != 1;
}

}  // namespace

extern "C" {

int shs_shard_create(const shs_problem* problem, const shs_error* error,
                     const shs_options* options, uint32_t rank, uint32_t nshards,
                     shs_shard** out) {
    if (!problem || !error || !out) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    shs_options o;
    if (options) o = *options;
    else shs_default_options(&o);
    int rc = validate_engine_config(*problem, *error, o);
    if (rc) return rc;
    if (nshards < 1 || nshards > kMaxShards)
        return set_error(SHS_INVALID_ARGUMENT, "shard count must be in [1, 16]");
    if (rank >= nshards) return set_error(SHS_INVALID_ARGUMENT, "shard rank out of range");
    auto* sh = new shs_shard;
    sh->prob = *problem;
    sh->err = *error;
    sh->opt = o;
    sh->N = problem->N;
    sh->t = problem->t;
    sh->rank = rank;
    sh->G = nshards;
    sh->dev = o.device;
    const uint64_t per = (sh->N + nshards - 1) / nshards;
    sh->S = (per + kBlock - 1) / kBlock * kBlock;
    sh->lo = uint64_t(rank) * sh->S;
    sh->hi = std::min(sh->N, sh->lo + sh->S);
    if (sh->lo >= sh->hi) {
        delete sh;
        return set_error(SHS_INVALID_ARGUMENT, "more shards than 256-amplitude blocks");
    }
    sh->nloc = sh->hi - sh->lo;
    sh->nb = (sh->nloc + kBlock - 1) / kBlock;
    sh->nchunks = (sh->nloc + kChunk - 1) / kChunk;
    reinit_state(sh->err, sh->w);
    sh->a_pows.assign(sh->t, 0);
    sh->a_invs.assign(sh->t, 1);
    sh->a_pows[sh->t - 1] = problem->a % problem->N;
    for (uint32_t s = sh->t - 1; s > 0; --s)
        sh->a_pows[s - 1] = mulmod(sh->a_pows[s], sh->a_pows[s], sh->N);
    sh->plans.assign(sh->t, TilePlanHost{});
    std::vector<std::pair<uint64_t, TilePlanHost>> cache;
    for (uint32_t s = 0; s < sh->t; ++s) {
        if (sh->a_pows[s] == 1) continue;
        u64 g = 0;
        if (mod_inverse(sh->a_pows[s], sh->N, &sh->a_invs[s], &g) != SHS_OK) {
            std::string msg = "not invertible: gcd(" + std::to_string(sh->a_pows[s]) + ", " +
                              std::to_string(sh->N) + ") = " + std::to_string(g);
            delete sh;
            return set_error(SHS_NOT_INVERTIBLE, msg);
        }
        if (s == 0) continue;
        auto it = std::find_if(cache.begin(), cache.end(),
                               [&](const auto& kv) { return kv.first == sh->a_pows[s]; });
        if (it == cache.end()) {
            cache.emplace_back(sh->a_pows[s],
                               make_tile_plan(sh->a_pows[s], sh->a_invs[s], sh->N, o.tiling));
            it = cache.end() - 1;
        }
        sh->plans[s] = it->second;
    }
    auto fail = [&](cudaError_t err, const char* what) {
        std::string msg = std::string(what) + ": " + cudaGetErrorString(err);
        release(sh);
        return set_error(SHS_CUDA_ERROR, msg);
    };
    cudaError_t ce = cudaSetDevice(sh->dev);
    if (ce != cudaSuccess) return fail(ce, "cudaSetDevice");
    cudaDeviceProp prop;
    if ((ce = cudaGetDeviceProperties(&prop, sh->dev)) != cudaSuccess)
        return fail(ce, "cudaGetDeviceProperties");
    if (prop.major < 10) {
        release(sh);
        return set_error(SHS_CUDA_ERROR, "device is not sm_100-class (B200 required)");
    }
    sh->num_sms = prop.multiProcessorCount;
    int occ = 0;
    ce = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stage_probs<kSrcBuffer, false, false>,
                                                       kThreads, 0);
    if (ce != cudaSuccess) return fail(ce, "occupancy");
    sh->grid_cap = std::max(1, occ) * sh->num_sms;
    ce = cudaFuncSetAttribute(k_exchange, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(exchange_smem_bytes()));
    if (ce != cudaSuccess) return fail(ce, "cudaFuncSetAttribute(k_exchange)");
    if ((ce = cudaStreamCreateWithFlags(&sh->stream, cudaStreamNonBlocking)) != cudaSuccess)
        return fail(ce, "cudaStreamCreate");
    for (int b = 0; b < 2; ++b)
        if ((ce = cudaMalloc(&sh->buf[b], sizeof(double2) * sh->nloc)) != cudaSuccess)
            return fail(ce, "cudaMalloc(shard buffer)");
    if ((ce = cudaMalloc(&sh->Sb, sizeof(double) * 2 * sh->nb)) != cudaSuccess)
        return fail(ce, "cudaMalloc(block sums)");
    if ((ce = cudaMalloc(&sh->partials, sizeof(unsigned long long) * 2 * kDigits * sh->grid_cap)) !=
        cudaSuccess)
        return fail(ce, "cudaMalloc(partials)");
    if ((ce = cudaMalloc(&sh->d_digits, sizeof(unsigned long long) * 2 * kDigits)) != cudaSuccess)
        return fail(ce, "cudaMalloc(digits)");
    if ((ce = cudaHostAlloc(&sh->h_digits, sizeof(unsigned long long) * 2 * kDigits,
                            cudaHostAllocDefault)) != cudaSuccess)
        return fail(ce, "cudaHostAlloc");
    for (auto& e : sh->ev)
        if ((ce = cudaEventCreate(&e)) != cudaSuccess) return fail(ce, "cudaEventCreate");
    sh->peer[rank][0] = sh->buf[0];
    sh->peer[rank][1] = sh->buf[1];
    *out = sh;
    return SHS_OK;
}

void shs_shard_destroy(shs_shard* sh) { release(sh); }

int shs_shard_range(const shs_shard* sh, uint64_t out[3]) {
    if (!sh || !out) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    out[0] = sh->lo;
    out[1] = sh->hi;
    out[2] = sh->S;
    return SHS_OK;
}

int shs_shard_buffers(const shs_shard* sh, void* out[2]) {
    if (!sh || !out) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    out[0] = sh->buf[0];
    out[1] = sh->buf[1];
    return SHS_OK;
}

int shs_shard_ipc_handles(const shs_shard* csh, void* out) {
    auto* sh = const_cast<shs_shard*>(csh);
    return shard_guard(sh, [&]() -> int {
        cudaIpcMemHandle_t h[2];
        for (int b = 0; b < 2; ++b) SHD_CUDA(cudaIpcGetMemHandle(&h[b], sh->buf[b]));
        std::memcpy(out, h, sizeof(h));
        return SHS_OK;
    });
}

int shs_shard_attach(shs_shard* sh, uint32_t peer, void* const bufs[2]) {
    if (!sh || !bufs || peer >= sh->G) return set_error(SHS_INVALID_ARGUMENT, "bad attach");
    sh->peer[peer][0] = static_cast<double2*>(bufs[0]);
    sh->peer[peer][1] = static_cast<double2*>(bufs[1]);
    sh->peer_ipc[peer] = false;
    return SHS_OK;
}

int shs_shard_attach_ipc(shs_shard* sh, uint32_t peer, const void* handles) {
    return shard_guard(sh, [&]() -> int {
        if (!handles || peer >= sh->G) return set_error(SHS_INVALID_ARGUMENT, "bad attach");
        if (peer == sh->rank) return SHS_OK;
        cudaIpcMemHandle_t h[2];
        std::memcpy(h, handles, sizeof(h));
        for (int b = 0; b < 2; ++b) {
            void* p = nullptr;
            SHD_CUDA(cudaIpcOpenMemHandle(&p, h[b], cudaIpcMemLazyEnablePeerAccess));
            sh->peer[peer][b] = static_cast<double2*>(p);
        }
        sh->peer_ipc[peer] = true;
        return SHS_OK;
    });
}

int shs_shard_init(shs_shard* sh) {
    if (!sh) return set_error(SHS_INVALID_ARGUMENT, "null shard");
    sh->e1 = true;
    sh->inv = 1.0;
    sh->parity = 0;
    sh->pending = false;
    sh->exchanged = -1;
    return SHS_OK;
}

int shs_shard_needs_exchange(const shs_shard* sh, uint32_t s) {
    if (!sh || s >= sh->t) return 0;
    return stage_needs_exchange(sh, s) ? 1 : 0;
}

int shs_shard_exchange(shs_shard* sh, uint32_t s) {
    return shard_guard(sh, [&]() -> int {
        if (s >= sh->t) return set_error(SHS_INVALID_ARGUMENT, "stage index out of range");
        if (!stage_needs_exchange(sh, s)) {
            sh->exchanged = static_cast<int>(s);
            return SHS_OK;
        }
        for (uint32_t q = 0; q < sh->G; ++q)
            if (!sh->peer[q][0] || !sh->peer[q][1])
                return set_error(SHS_INVALID_ARGUMENT, "shard " + std::to_string(q) + " not attached");
        const ShardMap map = shard_map(sh);
        const TilePlanHost& pl = sh->plans[s];
        int rc;
        if (pl.tiled) {
            TileParams tp{};
            tp.N = sh->N;
            tp.A = pl.A;
            tp.A_sh = pl.A_sh;
            tp.m = pl.m;
            tp.m_sh = pl.m_sh;
            tp.m_chunk = mulmod(pl.m, kCols, sh->N);
            tp.H = pl.H;
            tp.u = pl.u;
            tp.v = pl.v;
            tp.du = pl.du;
            tp.dv = pl.dv;
            tp.ntiles = pl.ntiles;
            const uint64_t mine = (pl.ntiles + sh->G - 1 - sh->rank) / sh->G;
            const int g = static_cast<int>(std::min<uint64_t>(std::max<uint64_t>(mine, 1), sh->num_sms));
            rc = shard_launch(sh, 1, [&] {
                k_exchange<<<g, kExchangeThreads, exchange_smem_bytes(), sh->stream>>>(
                    tp, map, sh->rank, sh->G);
            });
        } else {
            StageParams p = local_params(sh, s, false);
            rc = shard_launch(sh, 1, [&] {
                k_exchange_direct<<<grid(sh), kThreads, 0, sh->stream>>>(p, map,
                                                                        sh->buf[sh->parity ^ 1]);
            });
        }
        if (rc) return rc;
        sh->exchanged = static_cast<int>(s);
        return SHS_OK;
    });
}

int shs_shard_probs(shs_shard* sh, uint32_t s, uint64_t lo, uint64_t hi,
                    uint64_t digits[SHS_DIGITS]) {
    return shard_guard(sh, [&]() -> int {
        if (s >= sh->t) return set_error(SHS_INVALID_ARGUMENT, "stage index out of range");
        const bool ex = stage_needs_exchange(sh, s);
        if (ex && sh->exchanged != static_cast<int>(s))
            return set_error(SHS_INVALID_ARGUMENT, "probs before this stage's exchange");
        const double phi = stage_phase(s, (u128{hi} << 64) | lo);
        const bool gather = sh->a_pows[s] != 1;
        sh->sc.w0r = sh->w[0];
        sh->sc.w0i = sh->w[1];
        sh->sc.w1r = sh->w[2];
        sh->sc.w1i = sh->w[3];
        sh->sc.phr = 1.0 * std::cos(phi);  // std::polar(1.0, phi), statevector.cpp:338
        sh->sc.phi = 1.0 * std::sin(phi);
        sh->sc.inv = sh->inv;
        sh->sc.phase_mul = (gather || phi != 0.0) ? 1 : 0;
        sh->ps = s;
        StageParams p = local_params(sh, s, ex);
        const int g = grid(sh);
        int rc = shard_launch(sh, 0, [&] {
            if (sh->e1) {
                if (gather) k_stage_probs<kSrcGather, true, false><<<g, kThreads, 0, sh->stream>>>(p);
                else k_stage_probs<kSrcDirect, true, false><<<g, kThreads, 0, sh->stream>>>(p);
            } else if (ex) {
                k_stage_probs<kSrcBuffer, false, false><<<g, kThreads, 0, sh->stream>>>(p);
            } else {
                k_stage_probs<kSrcDirect, false, false><<<g, kThreads, 0, sh->stream>>>(p);
            }
            k_sum_partials<<<1, kFinalizeThreads, 0, sh->stream>>>(sh->partials, g, sh->d_digits);
        });
        if (rc) return rc;
        SHD_CUDA(cudaMemcpyAsync(sh->h_digits, sh->d_digits, sizeof(unsigned long long) * 2 * kDigits,
                                 cudaMemcpyDeviceToHost, sh->stream));
        SHD_CUDA(cudaStreamSynchronize(sh->stream));
        for (int i = 0; i < 2 * kDigits; ++i) digits[i] = sh->h_digits[i];
        sh->pending = true;
        return SHS_OK;
    });
}

int shs_shard_collapse(shs_shard* sh, int32_t src_group, double p_src) {
    return shard_guard(sh, [&]() -> int {
        if (!sh->pending) return set_error(SHS_INVALID_ARGUMENT, "collapse without a pending stage");
        if (src_group != 0 && src_group != 1)
            return set_error(SHS_INVALID_ARGUMENT, "src_group must be 0 or 1");
        if (p_src < kDegenerateMass)
            return set_error(SHS_DEGENERATE_BRANCH,
                             "impossible measurement branch at stage " + std::to_string(sh->ps));
        const uint32_t s = sh->ps;
        const bool ex = stage_needs_exchange(sh, s);
        const bool gather = sh->a_pows[s] != 1;
        StageParams p = local_params(sh, s, ex);
        p.sel = src_group;
        const int g = grid(sh);
        int rc = shard_launch(sh, 2, [&] {
            if (sh->e1) {
                if (gather) k_stage_collapse<kSrcGather, true, false><<<g, kThreads, 0, sh->stream>>>(p);
                else k_stage_collapse<kSrcDirect, true, false><<<g, kThreads, 0, sh->stream>>>(p);
            } else if (ex) {  // in place over P
                k_stage_collapse<kSrcBuffer, false, false><<<g, kThreads, 0, sh->stream>>>(p);
            } else {
                k_stage_collapse<kSrcDirect, false, false><<<g, kThreads, 0, sh->stream>>>(p);
            }
        });
        if (rc) return rc;
        sh->parity ^= 1;
        sh->e1 = false;
        sh->inv = 1.0 / std::sqrt(p_src);
        sh->pending = false;
        sh->exchanged = -1;
        return SHS_OK;
    });
}

int shs_shard_sync(shs_shard* sh) {
    return shard_guard(sh, [&]() -> int {
        SHD_CUDA(cudaStreamSynchronize(sh->stream));
        return SHS_OK;
    });
}

int shs_shard_state_read(shs_shard* sh, int32_t x, uint64_t first, uint64_t count, double* host) {
    return shard_guard(sh, [&]() -> int {
        if (x != 0 && x != 1) return set_error(SHS_INVALID_ARGUMENT, "group must be 0 or 1");
        if (count == 0) return SHS_OK;
        double2* d = nullptr;
        SHD_CUDA(cudaMallocAsync(&d, sizeof(double2) * count, sh->stream));
        const int g = static_cast<int>(std::min<uint64_t>((count + 255) / 256, 4096));
        const double wr = sh->w[2 * x], wi = sh->w[2 * x + 1];
        const double2* X = sh->buf[sh->parity];
        if (sh->e1) k_state_read<true><<<g, 256, 0, sh->stream>>>(X, sh->lo, sh->hi, wr, wi, sh->inv, first, count, d);
        else k_state_read<false><<<g, 256, 0, sh->stream>>>(X, sh->lo, sh->hi, wr, wi, sh->inv, first, count, d);
        SHD_CUDA(cudaGetLastError());
        SHD_CUDA(cudaMemcpyAsync(host, d, sizeof(double2) * count, cudaMemcpyDeviceToHost, sh->stream));
        SHD_CUDA(cudaFreeAsync(d, sh->stream));
        SHD_CUDA(cudaStreamSynchronize(sh->stream));
        return SHS_OK;
    });
}

int shs_shard_stage_read(shs_shard* sh, int32_t x, uint64_t first, uint64_t count, double* host) {
    return shard_guard(sh, [&]() -> int {
        if (!sh->pending) return set_error(SHS_INVALID_ARGUMENT, "no pending stage");
        if (count == 0) return SHS_OK;
        const uint32_t s = sh->ps;
        const bool ex = stage_needs_exchange(sh, s);
        const bool gather = sh->a_pows[s] != 1;
        StageParams p = local_params(sh, s, ex);
        double2* d = nullptr;
        SHD_CUDA(cudaMallocAsync(&d, sizeof(double2) * count, sh->stream));
        const int g = static_cast<int>(std::min<uint64_t>((count + 255) / 256, 4096));
        if (sh->e1) {
            if (gather) k_stage_read<kSrcGather, true><<<g, 256, 0, sh->stream>>>(p, x, first, count, d);
            else k_stage_read<kSrcDirect, true><<<g, 256, 0, sh->stream>>>(p, x, first, count, d);
        } else if (ex) {
            k_stage_read<kSrcBuffer, false><<<g, 256, 0, sh->stream>>>(p, x, first, count, d);
        } else {
            k_stage_read<kSrcDirect, false><<<g, 256, 0, sh->stream>>>(p, x, first, count, d);
        }
        SHD_CUDA(cudaGetLastError());
        SHD_CUDA(cudaMemcpyAsync(host, d, sizeof(double2) * count, cudaMemcpyDeviceToHost, sh->stream));
        SHD_CUDA(cudaFreeAsync(d, sh->stream));
        SHD_CUDA(cudaStreamSynchronize(sh->stream));
        return SHS_OK;
    });
}

int shs_digits_to_probs(const uint64_t digits[SHS_DIGITS], double* p0, double* p1) {
    if (!digits || !p0 || !p1) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    uint64_t acc[2 * kDigits];
    std::memcpy(acc, digits, sizeof(acc));
    *p0 = digits_to_double_host(acc);
    *p1 = digits_to_double_host(acc + kDigits);
    return SHS_OK;
}

int shs_shard_set_timing(shs_shard* sh, int32_t enable) {
    if (!sh) return set_error(SHS_INVALID_ARGUMENT, "null shard");
    sh->timing = enable != 0;
    for (int k = 0; k < 3; ++k) {
        sh->kms[k] = 0;
        sh->klaunch[k] = 0;
    }
    return SHS_OK;
}

int shs_shard_kernel_times(const shs_shard* sh, double ms[3], uint64_t launches[3]) {
    if (!sh) return set_error(SHS_INVALID_ARGUMENT, "null shard");
    for (int k = 0; k < 3; ++k) {
        if (ms) ms[k] = sh->kms[k];
        if (launches) launches[k] = sh->klaunch[k];
    }
    return SHS_OK;
}

uint64_t shs_shard_launch_count(const shs_shard* sh) { return sh ? sh->launches : 0; }

void* shs_shard_stream(const shs_shard* sh) { return sh ? static_cast<void*>(sh->stream) : nullptr; }

}  // extern "C"
