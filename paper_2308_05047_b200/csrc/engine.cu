// shorsim_b200 engine: sm_100a kernels for the iterative-Shor stage loop and the
// host driver behind the C ABI of include/shorsim_b200.h.
//
// State: after every reset the reference's 2 x 2^L state is the
// product (w0|0> + w1|1>) (x) |v> with v = sel * inv (statevector.cpp:391-400),
// so the engine keeps ONE fp64 complex buffer `sel` of N amplitudes in HBM plus
// the scalar inv, and recomputes g0/g1 on the fly, bit-exactly. A stage is two
// HBM passes over N amplitudes:
//   k_stage_probs    read sel[z], sel[src z]; h0/h1 of every z; sequential
//                    256-block |h|^2 partials (bit-identical to the reference's
//                    block sums, statevector.cpp:353-371) folded into an exact
//                    integer accumulator per CTA                     32 B/amp
//   k_finalize       p0/p1 from the per-CTA accumulators (exact, correctly
//                    rounded) or by sequential Kahan (bit-identical) over the
//                    block partials when there are few blocks       ~0 B/amp
//   k_stage_collapse read sel[z], sel[src z]; write sel'[z] = h_bit  48 B/amp
// with src z = a_inv * z mod N computed by Shoup multiplication once per thread
// and add/conditional-subtract afterwards (no index tables: 0 B/amp).
// Non-identity stages of large states run the same two passes as sorted-residue
// tiles (tiled.cuh, k_tiled<true|false> + k_tile_fixup) so both the direct and
// the gathered side of the permutation are coalesced.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/shorsim_b200.h"
#include "device_math.cuh"
#include "host_model.hpp"
#include "stage_kernels.cuh"
#include "tile_plan.hpp"
#include "tiled.cuh"
#include "batch.cuh"
#include "sparse.cuh"
#include "lockstep.cuh"
#include "shard_group.hpp"
#include "sparse_plan.hpp"

using namespace shs;

namespace {


#define SHS_CUDA(call)                                                                  \
    do {                                                                                \
        cudaError_t _e = (call);                                                        \
        if (_e != cudaSuccess)                                                          \
            return set_error(SHS_CUDA_ERROR, std::string(#call) + ": " +                \
                                                 cudaGetErrorString(_e));               \
    } while (0)

constexpr double kNormTolerance = 1e-9;     // statevector.cpp:18

}  // namespace

// ---------------------------------------------------------------------------
struct shs_engine {
    shs_problem prob{};
    shs_error err{};
    shs_options opt{};
    uint64_t N = 0;
    uint32_t t = 0;
    std::vector<u64> a_pows, a_invs;
    double w[4] = {0, 0, 0, 0};
    int dev = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    double2* X = nullptr;
    double2* Y = nullptr;
    double* S = nullptr;
    unsigned long long* partials = nullptr;
    double* d_out = nullptr;
    double* h_out = nullptr;
    uint64_t nb = 0, nchunks = 0;
    int grid_cap = 0;        // CTAs of the persistent stage kernels
    int tiled_cap = 0;       // CTAs of the persistent tiled kernels
    int fixup_cap = 0;       // CTAs of k_tile_fixup
    std::vector<TilePlanHost> plans;  // per stage
    uint64_t max_rows = 0;   // largest H over the stages' plans
    double* head = nullptr;  // [max_rows][2][256]
    double* tail = nullptr;  // [max_rows][2]
    uint2* split = nullptr;  // [t][tiled_cap + 1] CTA range starts of the tiled stages
    unsigned long long* band_ctr = nullptr;  // k_tiled<., false> dynamic band counter
    uint64_t band_issued = 0;                // its value before the next launch
    bool spec_on = true;                     // speculative group-0 writes (SHS_SPEC=0: off)
    int64_t spec_stage = -1;                 // Y holds h0 of this stage's tiled probs pass
    bool kahan = false;      // resolved combine mode
    bool lock_ws = true;     // lockstep probs: warp-specialized k_lock_probs_ws
    // state
    bool e1 = true;
    double inv = 1.0;
    bool pending = false;
    uint32_t ps = 0;
    StageScalars sc{};
    double p0 = 0, p1 = 0;
    // instrumentation
    bool timing = false;
    struct Mark {
        int kind;
        cudaEvent_t a, b;
    };
    std::vector<Mark> marks;
    std::vector<cudaEvent_t> pool;
    double kms[3] = {0, 0, 0};
    uint64_t klaunch[3] = {0, 0, 0};
    uint64_t launches = 0;
    uint64_t device_bytes = 0;
    // batched small-N runs (batch.cuh), allocated on first use
    uint64_t* d_apows = nullptr;
    uint64_t* d_ainvs = nullptr;
    uint64_t* d_ainvsh = nullptr;
    double2* d_phase = nullptr;
    void* d_batch_out = nullptr;
    size_t batch_out_bytes = 0;
    int batch_grid = 0;
    // device-resident runs (engine_run_device), allocated on first use
    DevStage* d_slots = nullptr;   // [2] stage scalars + collapse group
    StageRec* h_rec = nullptr;     // [t] host-mapped per-stage records
    StageRec* d_rec = nullptr;     // its device alias
    cudaEvent_t meas_ev[2] = {nullptr, nullptr};
    bool host_measure = false;     // SHS_HOST_MEASURE=1: the host-driven loop (A/B)
    bool lockstep = true;          // SHS_LOCKSTEP=0: run_many runs shot by shot (A/B)
    // sparse prefix of device-resident runs (sparse.cuh): stages 0 .. sparse_n-1
    // on the support, carved out of Y (unused until the first dense stage)
    uint32_t sparse_n = 0;
    bool sparse_on = true;         // shs_engine_set_sparse
    uint64_t* sZ[2] = {nullptr, nullptr};
    double2* sV[2] = {nullptr, nullptr};
    uint64_t* sKeys = nullptr;
    double2* sNrm = nullptr;       // norm pairs in orbit order (sort input)
    double2* sNrm2 = nullptr;      // ... sorted by z
    void* sTemp = nullptr;
    size_t sTempBytes = 0;
    // multi-device engine (options.n_devices): the state is block-sharded over a
    // shard group driven by this engine (shard.cu); every run / step call below
    // is forwarded to it
    ShardGroup* group = nullptr;
    // orbit-compressed stages (orbit.cuh): the state holds only the r members of
    // <a>, in z order. Stages with orb_use[s] run k_tiled<true, false, true>
    // (both groups written, no collapse pass); each N-amplitude buffer holds a
    // pair of compressed slots (stride orb_pad), the current pair in X
    bool orb_want = true;          // SHS_ORBIT=0 / shs_engine_set_orbit(0): dense only
    bool pdl = true;               // SHS_PDL=0: orbit stages launched without programmatic dependent launch
    bool orb_ready = false;        // rank records built
    uint64_t orb_r = 0, orb_pad = 0;
    std::vector<uint8_t> orb_use;  // per stage
    ulonglong2* orb_rec = nullptr; // [ceil(N / 64) + 2]
    bool rep_orb = false;          // the current state is compressed (pair in X)
    int orb_sel = 0;               // its slot when the host knows it ...
    const DevStage* orb_prev = nullptr;  // ... else the device slot whose sel picks it
    int64_t orb_stage = -1;        // the stage whose probs pass ran compressed (pending collapse)
};

namespace {

cudaEvent_t take_event(shs_engine* e) {
    if (!e->pool.empty()) {
        cudaEvent_t ev = e->pool.back();
        e->pool.pop_back();
        return ev;
    }
    cudaEvent_t ev;
    cudaEventCreate(&ev);
    return ev;
}

// Resolve recorded kernel intervals after the stream has been synchronised.
void resolve_marks(shs_engine* e) {
    for (auto& m : e->marks) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, m.a, m.b) == cudaSuccess) {
            e->kms[m.kind] += ms;
            e->klaunch[m.kind] += 1;
        }
        e->pool.push_back(m.a);
        e->pool.push_back(m.b);
    }
    e->marks.clear();
}

template <typename F>
int launch(shs_engine* e, int kind, F&& f) {
    // an error left by an earlier runtime call is reported as such, not as this launch's
    const cudaError_t stale = cudaGetLastError();
    if (stale != cudaSuccess)
        return set_error(SHS_CUDA_ERROR, std::string("pending CUDA error before a launch: ") +
                                             cudaGetErrorString(stale));
    cudaEvent_t a = nullptr, b = nullptr;
    const bool timed = e->timing && kind >= 0;
    if (timed) {
        a = take_event(e);
        b = take_event(e);
        cudaEventRecord(a, e->stream);
    }
    f();
    cudaError_t err = cudaGetLastError();
    if (timed) {
        cudaEventRecord(b, e->stream);
        e->marks.push_back({kind, a, b});
    }
    e->launches++;
    if (err != cudaSuccess)
        return set_error(SHS_CUDA_ERROR, std::string("kernel launch: ") + cudaGetErrorString(err));
    return SHS_OK;
}

int sync(shs_engine* e) {
    cudaError_t err = cudaStreamSynchronize(e->stream);
    if (err != cudaSuccess)
        return set_error(SHS_CUDA_ERROR, std::string("stream sync: ") + cudaGetErrorString(err));
    if (e->timing) resolve_marks(e);
    return SHS_OK;
}

// Direct-kernel stages with a small multiplier stage their A gathered runs
// through shared memory (stage_kernels.cuh kSrcStreams) from 16 MB of state on:
// always in the collapse pass; in the probs pass, whose in-order block folds
// stall the staged CTAs, only from A = kStreamsProbsMinA (config 4, B200:
// A = 625 probs 92 -> 51 ms, collapse 119 -> 46 ms; A = 25 collapse 65 -> 36 ms,
// probs 40 either way; A = 5 probs 32 ms gathered vs 41 ms staged).
// Head scratch a small-multiplier tile plan may use (tile_plan.hpp
// make_small_a_plan): up to half a state buffer (config 4, A = 625: 28 GB
// beside the 137 GB state on a 180 GB B200).
uint64_t small_a_scratch(uint64_t N) { return N * sizeof(double2) / 2; }

constexpr uint32_t kStreamsProbsMinA = 64;
bool streams_stage(const shs_engine* e, uint32_t s) {
    return e->a_pows[s] != 1 && e->a_pows[s] <= kStreamsMaxA && e->N >= kTileAutoMinN &&
           e->opt.tiling != SHS_TILING_OFF;
}

size_t streams_smem(const StageParams& p) { return sizeof(double2) * p.A * p.W; }

StageParams params_for(const shs_engine* e, uint32_t s) {
    StageParams p{};
    p.X = e->X;
    p.Xs = nullptr;
    p.Y = e->Y;
    p.N = e->N;
    p.z0 = 0;
    p.zend = e->N;
    p.m = e->a_invs[s];
    p.m_sh = e->a_pows[s] != 1 ? shoup(p.m, e->N) : 0;
    p.m_step = e->a_pows[s] != 1 ? mulmod(p.m, kBlock, e->N) : 0;
    p.sc = e->sc;
    p.S = e->S;
    p.nb = e->nb;
    p.partials = e->partials;
    p.nchunks = e->nchunks;
    if (streams_stage(e, s)) {
        p.A = static_cast<uint32_t>(e->a_pows[s]);
        p.W = (kChunk + 2 * p.A - 1) / p.A | 1u;  // ceil((A - 1 + kChunk) / A), odd
        p.invA = 1.0f / static_cast<float>(p.A);
        p.invW = 1.0f / static_cast<float>(p.W);
    }
    return p;
}

TileParams tile_params_for(const shs_engine* e, uint32_t s) {
    const TilePlanHost& pl = e->plans[s];
    TileParams p{};
    p.X = e->X;
    p.Y = e->Y;
    p.N = e->N;
    p.A = pl.A;
    p.A_sh = pl.A_sh;
    p.m = pl.m;
    p.m_sh = pl.m_sh;
    p.m_chunk = mulmod(pl.m, kCols, e->N);
    p.H = pl.H;
    p.u = pl.u;
    p.v = pl.v;
    p.du = pl.du;
    p.dv = pl.dv;
    p.ntiles = pl.ntiles;
    p.split = e->split + uint64_t(s) * (e->tiled_cap + 1);
    p.bulk_rounds = pl.bulk_rounds;
    p.band_ctr = e->band_ctr;
    p.band_base = e->band_issued;
    p.sc = e->sc;
    p.S = e->S;
    p.nb = e->nb;
    p.partials = e->partials;
    p.head = e->head;
    p.tail = e->tail;
    return p;
}

int grid_for(const shs_engine* e) {
    return static_cast<int>(std::min<uint64_t>(e->nchunks, static_cast<uint64_t>(e->grid_cap)));
}

template <bool G, bool E1, bool D>
void launch_probs_v(shs_engine* e, const StageParams& p) {
    if (G && p.A >= kStreamsProbsMinA)
        k_stage_probs<kSrcStreams, E1, D><<<grid_for(e), kThreads, streams_smem(p), e->stream>>>(p);
    else
        k_stage_probs<G ? kSrcGather : kSrcDirect, E1, D><<<grid_for(e), kThreads, 0, e->stream>>>(p);
}

// stage 0 (E1) always runs on host scalars (inv = 1, phi = 0)
template <bool G, bool E1>
void launch_probs(shs_engine* e, const StageParams& p) {
    if (!E1 && p.dev) launch_probs_v<G, false, true>(e, p);
    else launch_probs_v<G, E1, false>(e, p);
}

template <bool G, bool E1, bool D>
void launch_collapse_v(shs_engine* e, const StageParams& p) {
    if (G && p.A)
        k_stage_collapse<kSrcStreams, E1, D><<<grid_for(e), kThreads, streams_smem(p), e->stream>>>(p);
    else
        k_stage_collapse<G ? kSrcGather : kSrcDirect, E1, D><<<grid_for(e), kThreads, 0, e->stream>>>(p);
}

// stage 0's collapse (E1) reads the slot too in a device-resident run (its group
// is measured on the device)
template <bool G, bool E1>
void launch_collapse(shs_engine* e, const StageParams& p) {
    if (p.dev) launch_collapse_v<G, E1, true>(e, p);
    else launch_collapse_v<G, E1, false>(e, p);
}

// Lockstep multi-shot buffers (lockstep.cuh), pooled per process: the campaign
// harness creates one engine per problem, and cudaMalloc/cudaFree of a batch's
// states plus the pinned host records cost as much as the batch's kernels at
// N = 2^18 (and more after large allocations). A call checks a set out (any
// engine, same device, large enough), returns it after; the pool keeps at most
// kLockPoolBytes of device memory. Engines on different threads take different sets.
struct LockBufs {
    int dev = -1;
    size_t state_bytes = 0, s_bytes = 0, parts_bytes = 0, shots = 0, rec_bytes = 0;
    double2* X = nullptr;
    double2* Y = nullptr;
    double* S = nullptr;
    unsigned long long* parts = nullptr;
    DevStage* slots = nullptr;
    NextPhase* d_nph = nullptr;
    NextPhase* h_nph = nullptr;
    StageRec* h_rec = nullptr;
    StageRec* d_rec = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    size_t device_bytes() const { return 2 * state_bytes + s_bytes + parts_bytes; }
};

void free_lock_buffers(LockBufs& L) {
    cudaFree(L.X);
    cudaFree(L.Y);
    cudaFree(L.S);
    cudaFree(L.parts);
    cudaFree(L.slots);
    cudaFree(L.d_nph);
    if (L.h_nph) cudaFreeHost(L.h_nph);
    if (L.h_rec) cudaFreeHost(L.h_rec);
    for (auto v : L.ev)
        if (v) cudaEventDestroy(v);
    L = LockBufs{};
}

constexpr size_t kLockPoolBytes = size_t(4) << 30;
std::mutex g_lock_pool_mu;
std::vector<LockBufs> g_lock_pool;  // never freed at exit (CUDA may be torn down first)

// A set with at least the given sizes on `dev`: from the pool, else allocated.
cudaError_t lock_checkout(int dev, size_t state_bytes, size_t s_bytes, size_t parts_bytes,
                          size_t shots, size_t rec_bytes, LockBufs& out) {
    {
        std::lock_guard<std::mutex> g(g_lock_pool_mu);
        for (size_t i = 0; i < g_lock_pool.size(); ++i) {
            const LockBufs& c = g_lock_pool[i];
            if (c.dev == dev && c.state_bytes >= state_bytes && c.s_bytes >= s_bytes &&
                c.parts_bytes >= parts_bytes && c.shots >= shots && c.rec_bytes >= rec_bytes) {
                out = c;
                g_lock_pool.erase(g_lock_pool.begin() + static_cast<std::ptrdiff_t>(i));
                return cudaSuccess;
            }
        }
    }
    LockBufs L;
    L.dev = dev;
    L.state_bytes = state_bytes;
    L.s_bytes = s_bytes;
    L.parts_bytes = parts_bytes;
    L.shots = shots;
    L.rec_bytes = rec_bytes;
    cudaError_t ce;
    if ((ce = cudaMalloc(&L.X, state_bytes)) != cudaSuccess ||
        (ce = cudaMalloc(&L.Y, state_bytes)) != cudaSuccess ||
        (ce = cudaMalloc(&L.S, s_bytes)) != cudaSuccess ||
        (ce = cudaMalloc(&L.parts, parts_bytes)) != cudaSuccess ||
        (ce = cudaMalloc(&L.slots, sizeof(DevStage) * 2 * shots)) != cudaSuccess ||
        (ce = cudaMalloc(&L.d_nph, sizeof(NextPhase) * 2 * shots)) != cudaSuccess ||
        (ce = cudaHostAlloc(&L.h_nph, sizeof(NextPhase) * 2 * shots, cudaHostAllocDefault)) != cudaSuccess ||
        (ce = cudaHostAlloc(&L.h_rec, rec_bytes, cudaHostAllocMapped)) != cudaSuccess ||
        (ce = cudaHostGetDevicePointer(reinterpret_cast<void**>(&L.d_rec), L.h_rec, 0)) != cudaSuccess ||
        (ce = cudaEventCreateWithFlags(&L.ev[0], cudaEventDisableTiming)) != cudaSuccess ||
        (ce = cudaEventCreateWithFlags(&L.ev[1], cudaEventDisableTiming)) != cudaSuccess) {
        free_lock_buffers(L);
        return ce;
    }
    out = L;
    return cudaSuccess;
}

// Back to the pool (its work on the caller's stream already synchronised);
// sets that would push the pool past kLockPoolBytes evict the oldest first.
void lock_return(LockBufs& L) {
    if (L.device_bytes() > kLockPoolBytes) {
        free_lock_buffers(L);
        return;
    }
    std::vector<LockBufs> evicted;
    {
        std::lock_guard<std::mutex> g(g_lock_pool_mu);
        size_t total = L.device_bytes();
        for (const auto& c : g_lock_pool) total += c.device_bytes();
        while (total > kLockPoolBytes && !g_lock_pool.empty()) {
            total -= g_lock_pool.front().device_bytes();
            evicted.push_back(g_lock_pool.front());
            g_lock_pool.erase(g_lock_pool.begin());
        }
        g_lock_pool.push_back(L);
    }
    for (auto& c : evicted) free_lock_buffers(c);
    L = LockBufs{};
}

void release(shs_engine* e) {
    if (!e) return;
    group_destroy(e->group);
    e->group = nullptr;
    cudaSetDevice(e->dev);
    if (e->stream) cudaStreamSynchronize(e->stream);
    for (auto& m : e->marks) {
        cudaEventDestroy(m.a);
        cudaEventDestroy(m.b);
    }
    for (auto ev : e->pool) cudaEventDestroy(ev);
    cudaFree(e->X);
    cudaFree(e->Y);
    cudaFree(e->S);
    cudaFree(e->partials);
    cudaFree(e->head);
    cudaFree(e->tail);
    cudaFree(e->split);
    cudaFree(e->band_ctr);
    cudaFree(e->d_apows);
    cudaFree(e->d_ainvs);
    cudaFree(e->d_ainvsh);
    cudaFree(e->d_phase);
    cudaFree(e->d_batch_out);
    cudaFree(e->d_out);
    if (e->h_out) cudaFreeHost(e->h_out);
    cudaFree(e->d_slots);
    cudaFree(e->orb_rec);
    if (e->h_rec) cudaFreeHost(e->h_rec);
    for (auto ev : e->meas_ev)
        if (ev) cudaEventDestroy(ev);
    if (e->stream) cudaStreamDestroy(e->stream);
    delete e;
}

// The two N-amplitude buffers (sel and its successor) and the block partials
// are allocated on first use, so engines used only for validation or index
// maps never reserve 2 x 16 N bytes of HBM.
// Stages run on the support (sparse_plan.hpp): the largest n <= t - 1 with
// 2^n <= N / 16 whose orbit does not wrap.
uint32_t plan_sparse_prefix(const shs_engine* e) {
    if (e->kahan) return 0;
    uint64_t density = kSparseDensity;
    if (const char* d = std::getenv("SHS_SPARSE_DENSITY"))  // A/B hook (>= 8: buffers fit Y)
        density = std::max<uint64_t>(8, std::strtoull(d, nullptr, 10));
    return sparse_prefix_stages(e->N, e->t, e->a_pows, e->N / density);
}

// Sparse buffers inside the current Y (free until the first dense collapse of a
// run; carved again at every run start since X / Y swap): Z0 Z1 (u64), V0 V1
// (double2), sorted keys (u64), norm pairs and their sorted copy (double2) per
// support element, then the radix sort's scratch.
int carve_sparse(shs_engine* e) {
    const uint64_t K = uint64_t(1) << e->sparse_n;
    char* p = reinterpret_cast<char*>(e->Y);
    auto take = [&](size_t bytes) {
        char* q = p;
        p += (bytes + 255) & ~size_t(255);
        return q;
    };
    e->sZ[0] = reinterpret_cast<uint64_t*>(take(8 * K));
    e->sZ[1] = reinterpret_cast<uint64_t*>(take(8 * K));
    e->sV[0] = reinterpret_cast<double2*>(take(16 * K));
    e->sV[1] = reinterpret_cast<double2*>(take(16 * K));
    e->sKeys = reinterpret_cast<uint64_t*>(take(8 * K));
    e->sNrm = reinterpret_cast<double2*>(take(16 * K));
    e->sNrm2 = reinterpret_cast<double2*>(take(16 * K));
    if (!e->sTempBytes) {
        SHS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, e->sTempBytes, e->sZ[0], e->sKeys,
                                                 e->sNrm, e->sNrm2, static_cast<int>(K), 0, 64,
                                                 e->stream));
    }
    e->sTemp = take(e->sTempBytes);
    if (static_cast<size_t>(p - reinterpret_cast<char*>(e->Y)) > sizeof(double2) * e->N)
        return set_error(SHS_CUDA_ERROR, "sparse prefix buffers exceed the state buffer");
    return SHS_OK;
}

// All-or-nothing: a failed allocation frees what this call allocated, so a
// retry starts clean (and no kernel ever runs with a half-allocated engine).
int ensure_buffers_once(shs_engine* e);
int orb_build(shs_engine* e);
int ensure_buffers(shs_engine* e) {
    if (e->X) return SHS_OK;
    const uint64_t bytes0 = e->device_bytes;
    int rc = ensure_buffers_once(e);
    if (rc) {
        for (void* p : {static_cast<void*>(e->X), static_cast<void*>(e->Y), static_cast<void*>(e->S),
                        static_cast<void*>(e->head), static_cast<void*>(e->tail),
                        static_cast<void*>(e->split)})
            cudaFree(p);
        e->X = e->Y = nullptr;
        e->S = nullptr;
        e->head = e->tail = nullptr;
        e->split = nullptr;
        e->device_bytes = bytes0;
        cudaGetLastError();  // the failed cudaMalloc is reported through rc
    }
    return rc;
}

int ensure_buffers_once(shs_engine* e) {
    const size_t amp_bytes = sizeof(double2) * e->N;
    SHS_CUDA(cudaMalloc(&e->X, amp_bytes));
    SHS_CUDA(cudaMalloc(&e->Y, amp_bytes));
    SHS_CUDA(cudaMalloc(&e->S, sizeof(double) * 2 * e->nb));
    e->device_bytes += 2 * amp_bytes + sizeof(double) * 2 * e->nb;
    if (e->max_rows) {
        SHS_CUDA(cudaMalloc(&e->head, sizeof(double) * 2 * 256 * e->max_rows));
        SHS_CUDA(cudaMalloc(&e->tail, sizeof(double) * 2 * e->max_rows));
        e->device_bytes += sizeof(double) * 2 * 257 * e->max_rows;
        // the tiled stages' CTA range tables (tile_plan.hpp make_tile_split)
        const size_t per = static_cast<size_t>(e->tiled_cap) + 1;
        std::vector<uint32_t> tab(2 * per * e->t, 0);
        for (uint32_t s = 0; s < e->t; ++s)
            if (e->plans[s].tiled)
                std::copy(e->plans[s].split.begin(), e->plans[s].split.end(),
                          tab.begin() + 2 * per * s);
        SHS_CUDA(cudaMalloc(&e->split, sizeof(uint32_t) * tab.size()));
        SHS_CUDA(cudaMemcpy(e->split, tab.data(), sizeof(uint32_t) * tab.size(),
                            cudaMemcpyHostToDevice));
        e->device_bytes += sizeof(uint32_t) * tab.size();
    }
    if (e->orb_want && e->orb_r) return orb_build(e);
    return SHS_OK;
}

// Rank records of the orbit <a> (orbit.cuh), built once per engine with Y as
// scratch (called only while Y holds no state): membership bits by
// enumerating a^x for x < r (r from a baby-step giant-step order search at
// create), word popcounts, an exclusive scan, the records.
int orb_build(shs_engine* e) {
    if (e->orb_ready || !e->orb_r || !e->Y) return SHS_OK;
    const uint64_t N = e->N, r = e->orb_r, nw = (N + 63) / 64;
    // the compressed stages need the rank records beside the state: without
    // room for them (plus 1 GB of slack) the engine runs every stage dense, with
    // identical results
    {
        const size_t need = sizeof(ulonglong2) * (nw + 2) + (size_t(1) << 30);
        size_t free_b = 0, total_b = 0;
        if (!e->orb_rec && (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess || free_b < need)) {
            cudaGetLastError();
            e->orb_want = false;
            e->orb_r = 0;
            return SHS_OK;
        }
    }
    const uint64_t a = e->prob.a % N;
    char* scratch = reinterpret_cast<char*>(e->Y);
    auto* bits = reinterpret_cast<unsigned int*>(scratch);
    scratch += ((8 * nw + 255) / 256) * 256;
    auto* counts = reinterpret_cast<unsigned long long*>(scratch);
    scratch += ((8 * nw + 255) / 256) * 256;
    auto* bases = reinterpret_cast<unsigned long long*>(scratch);
    scratch += ((8 * nw + 255) / 256) * 256;
    const uint64_t T = std::min<uint64_t>(r, uint64_t(e->num_sms) * 2048);
    const uint64_t B = (r + T - 1) / T;
    auto* starts = reinterpret_cast<uint64_t*>(scratch);
    scratch += ((8 * T + 255) / 256) * 256;
    size_t temp_bytes = 0;
    SHS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, counts, bases, static_cast<int64_t>(nw),
                                           e->stream));
    if (static_cast<uint64_t>(scratch - reinterpret_cast<char*>(e->Y)) + temp_bytes > sizeof(double2) * N)
        return set_error(SHS_CUDA_ERROR, "orbit index scratch exceeds the state buffer");
    std::vector<uint64_t> h(T);
    {
        uint64_t step = 1, base = a, ex = B;  // a^B
        while (ex) {
            if (ex & 1) step = mulmod(step, base, N);
            base = mulmod(base, base, N);
            ex >>= 1;
        }
        uint64_t v = 1;
        for (uint64_t k = 0; k < T; ++k) {
            h[k] = v;
            v = mulmod(v, step, N);
        }
    }
    if (!e->orb_rec) {
        SHS_CUDA(cudaMalloc(&e->orb_rec, sizeof(ulonglong2) * (nw + 2)));
        e->device_bytes += sizeof(ulonglong2) * (nw + 2);
    }
    SHS_CUDA(cudaMemcpyAsync(starts, h.data(), 8 * T, cudaMemcpyHostToDevice, e->stream));
    SHS_CUDA(cudaMemsetAsync(bits, 0, 8 * nw, e->stream));
    const int grid = static_cast<int>(std::min<uint64_t>((nw + 255) / 256, uint64_t(e->num_sms) * 16));
    int rc = launch(e, -1, [&] {
        k_orb_mark<<<static_cast<int>((T + 255) / 256), 256, 0, e->stream>>>(starts, T, B, r, a,
                                                                            shoup(a, N), N, bits);
        k_orb_counts<<<grid, 256, 0, e->stream>>>(bits, nw, counts);
        size_t tb = temp_bytes;
        cub::DeviceScan::ExclusiveSum(scratch, tb, counts, bases, static_cast<int64_t>(nw), e->stream);
        k_orb_records<<<grid, 256, 0, e->stream>>>(bits, bases, nw, r, e->orb_rec);
    });
    if (rc) return rc;
    unsigned long long last[2] = {0, 0};
    SHS_CUDA(cudaMemcpyAsync(&last[0], bases + nw - 1, 8, cudaMemcpyDeviceToHost, e->stream));
    SHS_CUDA(cudaMemcpyAsync(&last[1], counts + nw - 1, 8, cudaMemcpyDeviceToHost, e->stream));
    if ((rc = sync(e))) return rc;
    if (last[0] + last[1] != r)
        return set_error(SHS_ERROR, "orbit index: " + std::to_string(last[0] + last[1]) +
                                        " members marked, order " + std::to_string(r));
    e->orb_ready = true;
    return SHS_OK;
}

bool orb_stage_on(const shs_engine* e, uint32_t s) {
    return e->orb_want && e->orb_ready && e->orb_use[s] && !e->e1;
}

int orb_grid(const shs_engine* e) { return e->num_sms * 8; }

// dense X -> compressed slot 0 of Y's pair, then swap: the pair is in X
int orb_enter(shs_engine* e) {
    int rc = launch(e, -1, [&] {
        k_orb_compress<<<orb_grid(e), kOrbThreads, 0, e->stream>>>(e->X, e->orb_rec, e->N, e->Y);
    });
    if (rc) return rc;
    std::swap(e->X, e->Y);
    e->rep_orb = true;
    e->orb_sel = 0;
    e->orb_prev = nullptr;
    return SHS_OK;
}

OrbSrc orb_src(const shs_engine* e) {
    return OrbSrc{e->X, e->X + e->orb_pad, e->orb_prev, e->orb_sel};
}

// compressed pair in X -> dense Y, then swap: the dense state is in X
int orb_leave(shs_engine* e) {
    int rc = launch(e, -1, [&] {
        k_orb_expand<<<orb_grid(e), kOrbThreads, 0, e->stream>>>(orb_src(e), e->orb_rec, e->N, e->Y);
    });
    if (rc) return rc;
    std::swap(e->X, e->Y);
    e->rep_orb = false;
    e->orb_prev = nullptr;
    return SHS_OK;
}

int state_init(shs_engine* e) {
    e->rep_orb = false;
    e->orb_prev = nullptr;
    e->orb_sel = 0;
    e->orb_stage = -1;
    if (e->orb_want && !e->orb_ready && e->orb_r && e->X) {
        int rc = orb_build(e);
        if (rc) return rc;
    }
    e->spec_stage = -1;
    e->e1 = true;  // sel = e_1 implicitly: no memset of the N-amplitude buffer
    e->inv = 1.0;
    e->pending = false;
    return SHS_OK;
}

// NVTX range for the lifetime of a scope (visible in nsys / ncu timelines)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// Host-side scalars of stage s for the observed prefix (statevector.cpp:338-349).
StageScalars host_scalars(const shs_engine* e, uint32_t s, u128 prefix, double inv) {
    const double phi = stage_phase(s, prefix);
    const bool gather = e->a_pows[s] != 1;
    StageScalars sc{};
    sc.w0r = e->w[0];
    sc.w0i = e->w[1];
    sc.w1r = e->w[2];
    sc.w1i = e->w[3];
    sc.phr = 1.0 * std::cos(phi);  // std::polar(1.0, phi), statevector.cpp:338
    sc.phi = 1.0 * std::sin(phi);
    sc.inv = inv;
    sc.phase_mul = (gather || phi != 0.0) ? 1 : 0;
    return sc;
}

// k_tile_fixup's grid: one warp per 32 items (k_tile_fixup1) when every such
// warp fits on the GPU at once, else 8-warp CTAs up to fixup_cap
int fixup_grid(const shs_engine* e, const TileParams& tp) {
    const uint64_t w = (2 * tp.H + 31) / 32;
    if (w <= uint64_t(kFix1Ctas) * e->num_sms && !std::getenv("SHS_FIXUP8")) return static_cast<int>(w);
    return static_cast<int>(
        std::min<uint64_t>((2 * tp.H + 32 * kFixWarps - 1) / (32 * kFixWarps), static_cast<uint64_t>(e->fixup_cap)));
}
void launch_fixup(shs_engine* e, const TileParams& tp, int g1, int g2) {
    unsigned long long* slots = e->partials + uint64_t(g1) * 2 * kDigits;
    if ((2 * tp.H + 31) / 32 <= uint64_t(kFix1Ctas) * e->num_sms && !std::getenv("SHS_FIXUP8")) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(g2);
        cfg.blockDim = dim3(32);
        cfg.dynamicSmemBytes = kFix1Smem;
        cfg.stream = e->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = e->pdl ? 1 : 0;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_tile_fixup1, tp, slots);
    } else {
        k_tile_fixup<<<g2, 32 * kFixWarps, kFixSmem, e->stream>>>(tp, slots);
    }
}

// Probs pass of stage s on the current sel (tiled or direct kernels, plus the
// tiled fixup). Scalars: e->sc, or the device slot `dev` when non-null.
// *nparts = the exact-accumulator slots it filled.
int launch_probs_pass(shs_engine* e, uint32_t s, const DevStage* dev, int* nparts) {
    const bool gather = e->a_pows[s] != 1;
    int rc;
    *nparts = grid_for(e);
    e->orb_stage = -1;
    const bool orb = orb_stage_on(e, s);
    if (orb && !e->rep_orb && (rc = orb_enter(e))) return rc;
    if (!orb && e->rep_orb && (rc = orb_leave(e))) return rc;
    if (orb) {
        // compressed: h0 and h1 of every member into Y's pair (no collapse pass)
        TileParams tp = tile_params_for(e, s);
        tp.dev = dev;
        tp.spec = 0;
        tp.X1 = e->X + e->orb_pad;
        tp.prev = e->orb_prev;
        tp.prev_sel = e->orb_sel;
        tp.Y1 = e->Y + e->orb_pad;
        tp.orb = e->orb_rec;
        tp.write = s + 1 < e->t ? 1 : 0;
        const TilePlanHost& pl = e->plans[s];
        // whole bands from the dynamic counter, unless the plan has too few bands
        // for it to balance; then the split plan's static work items (row spans
        // cut at 256-block boundaries). Config 4's long-row plans (>= 4 bands per
        // SM) measured 1% faster whole, n30's few-band ones 6% faster per run split.
        const bool split = pl.split_tail && pl.ntiles < 4 * static_cast<uint64_t>(e->num_sms);
        const int g1 = split ? pl.grid : static_cast<int>(std::min<uint64_t>(pl.ntiles, e->tiled_cap));
        const int g2 = fixup_grid(e, tp);
        rc = launch(e, 0, [&] {
            // programmatic dependent launch: the plan warps overlap the previous
            // stage's finalize (k_tiled's griddepcontrol.wait guards the rest)
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(g1);
            cfg.dynamicSmemBytes = tile_smem_bytes<true, true>();
            cfg.stream = e->stream;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = e->pdl ? 1 : 0;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            if (split) {
                cfg.blockDim = dim3(tile_threads<true, true, true>());
                cudaLaunchKernelEx(&cfg, k_tiled<true, true, true>, tp);
            } else {
                cfg.blockDim = dim3(tile_threads<true, false, true>());
                cudaLaunchKernelEx(&cfg, k_tiled<true, false, true>, tp);
                e->band_issued += pl.ntiles;
            }
            launch_fixup(e, tp, g1, g2);
        });
        e->launches++;  // k_tiled + k_tile_fixup in one launch group
        *nparts = g1 + g2;
        e->spec_stage = -1;
        e->orb_stage = s;
        return rc;
    }
    if (e->plans[s].tiled && !e->e1) {
        TileParams tp = tile_params_for(e, s);
        tp.dev = dev;
        tp.spec = e->spec_on && s + 1 < e->t ? 1 : 0;
        const TilePlanHost& pl = e->plans[s];
        const int g1 = pl.split_tail ? pl.grid
                                     : static_cast<int>(std::min<uint64_t>(pl.ntiles, e->tiled_cap));
        const int g2 = fixup_grid(e, tp);
        rc = launch(e, 0, [&] {
            if (pl.split_tail) {
                k_tiled<true, true><<<g1, tile_threads<true, true>(), tile_smem_bytes<true>(), e->stream>>>(tp);
            } else {
                k_tiled<true, false><<<g1, tile_threads<true, false>(), tile_smem_bytes<true>(), e->stream>>>(tp);
                e->band_issued += pl.ntiles;
            }
            launch_fixup(e, tp, g1, g2);
        });
        e->launches++;  // k_tiled + k_tile_fixup: two kernels in one launch group
        *nparts = g1 + g2;
        e->spec_stage = tp.spec ? static_cast<int64_t>(s) : -1;
    } else if (e->e1) {
        e->spec_stage = -1;
        // stage 0 from the implicit e_1: two live amplitudes (k_stage_probs_e1)
        StageParams p = params_for(e, s);
        rc = launch(e, 0, [&] {
            cudaMemsetAsync(e->S, 0, sizeof(double) * 2 * e->nb, e->stream);
            k_stage_probs_e1<<<1, 32, 0, e->stream>>>(p, e->a_pows[s]);
        });
        *nparts = 1;
    } else {
        StageParams p = params_for(e, s);
        p.dev = dev;
        p.spec = e->spec_on && s + 1 < e->t ? 1 : 0;
        e->spec_stage = p.spec ? static_cast<int64_t>(s) : -1;
        rc = launch(e, 0, [&] {
            if (gather) launch_probs<true, false>(e, p);
            else launch_probs<false, false>(e, p);
        });
    }
    return rc;
}

// Collapse pass of stage s into the successor buffer (then swapped in).
int launch_collapse_pass(shs_engine* e, uint32_t s, int src_group, const DevStage* dev) {
    const bool gather = e->a_pows[s] != 1;
    int rc;
    if (e->orb_stage == static_cast<int64_t>(s)) {
        // the compressed probs pass wrote both groups into Y's pair: keep one
        e->orb_stage = -1;
        std::swap(e->X, e->Y);
        e->orb_prev = dev;
        e->orb_sel = dev ? 0 : src_group;
        e->e1 = false;
        return SHS_OK;
    }
    if (e->plans[s].tiled && !e->e1) {
        TileParams tp = tile_params_for(e, s);
        tp.sel = src_group;
        tp.dev = dev;
        tp.spec = e->spec_stage == static_cast<int64_t>(s) ? 1 : 0;
        const TilePlanHost& pl = e->plans[s];
        const int g1 = pl.split_tail ? pl.grid
                                     : static_cast<int>(std::min<uint64_t>(pl.ntiles, e->tiled_cap));
        const bool skip = tp.spec && !dev && src_group == 0;  // Y already holds h0
        if (skip) {
            e->spec_stage = -1;
            std::swap(e->X, e->Y);
            e->e1 = false;
            return SHS_OK;
        }
        rc = launch(e, 2, [&] {
            if (pl.split_tail) {
                k_tiled<false, true><<<g1, tile_threads<false, true>(), tile_smem_bytes<false>(), e->stream>>>(tp);
            } else {
                k_tiled<false, false><<<g1, tile_threads<false, false>(), tile_smem_bytes<false>(), e->stream>>>(tp);
                e->band_issued += pl.ntiles;
            }
        });
    } else {
        StageParams p = params_for(e, s);
        p.sel = src_group;
        p.dev = dev;
        p.spec = e->spec_stage == static_cast<int64_t>(s) ? 1 : 0;
        if (p.spec && !dev && src_group == 0) {  // Y already holds h0
            e->spec_stage = -1;
            std::swap(e->X, e->Y);
            e->e1 = false;
            return SHS_OK;
        }
        rc = launch(e, 2, [&] {
            if (gather) {
                if (e->e1) launch_collapse<true, true>(e, p);
                else launch_collapse<true, false>(e, p);
            } else {
                if (e->e1) launch_collapse<false, true>(e, p);
                else launch_collapse<false, false>(e, p);
            }
        });
    }
    if (rc) return rc;
    e->spec_stage = -1;
    std::swap(e->X, e->Y);
    e->e1 = false;
    return SHS_OK;
}

int stage_probs(shs_engine* e, uint32_t s, u128 prefix, double* p0, double* p1) {
    if (s >= e->t) return set_error(SHS_INVALID_ARGUMENT, "stage index out of range");
    NvtxRange nvtx("shs stage probs");
    int rc = ensure_buffers(e);
    if (rc) return rc;
    e->sc = host_scalars(e, s, prefix, e->inv);
    e->ps = s;
    int nparts = 0;
    rc = launch_probs_pass(e, s, nullptr, &nparts);
    if (rc) return rc;
    rc = launch(e, 1, [&] {
        k_finalize<<<1, kFinalizeThreads, 0, e->stream>>>(e->partials, nparts, e->S, e->nb, e->kahan ? 1 : 0,
                                             e->d_out);
    });
    if (rc) return rc;
    SHS_CUDA(cudaMemcpyAsync(e->h_out, e->d_out, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                             e->stream));
    rc = sync(e);
    if (rc) return rc;
    e->p0 = e->h_out[0];
    e->p1 = e->h_out[1];
    e->pending = true;
    if (p0) *p0 = e->p0;
    if (p1) *p1 = e->p1;
    if (e->opt.check_norms && std::abs(e->p0 + e->p1 - 1.0) > kNormTolerance)  // :374-375
        return set_error(SHS_ERROR, "statevector norm drifted beyond 1e-9 at stage " +
                                        std::to_string(s));
    return SHS_OK;
}

int stage_collapse(shs_engine* e, int src_group, double p_src, bool wait) {
    if (!e->pending) return set_error(SHS_INVALID_ARGUMENT, "collapse without a pending stage");
    if (src_group != 0 && src_group != 1)
        return set_error(SHS_INVALID_ARGUMENT, "src_group must be 0 or 1");
    NvtxRange nvtx("shs stage collapse");
    if (p_src < kDegenerateMass)  // statevector.cpp:388-390 / 265-266
        return set_error(SHS_DEGENERATE_BRANCH,
                         "impossible measurement branch at stage " + std::to_string(e->ps));
    int rc = launch_collapse_pass(e, e->ps, src_group, nullptr);
    if (rc) return rc;
    e->inv = 1.0 / std::sqrt(p_src);  // statevector.cpp:391
    e->pending = false;
    if (wait) return sync(e);
    return SHS_OK;
}

// Sparse prefix stage s (sparse.cuh) on the support of 2^s elements:
// expand (both norms per new orbit index) -> radix sort by z -> in-order block
// folds into exact digit slots. *nparts = the fold's CTAs.
SparseParams sparse_params(shs_engine* e, uint32_t s, const DevStage* dev) {
    SparseParams p{};
    p.Zo = e->sZ[s & 1];
    p.Vo = e->sV[s & 1];
    p.Ko = uint64_t(1) << s;
    p.A = e->a_pows[s];
    p.A_sh = shoup(p.A, e->N);
    p.N = e->N;
    p.sc = e->sc;
    p.dev = dev;
    p.Zn = e->sZ[(s + 1) & 1];
    p.Vn = e->sV[(s + 1) & 1];
    p.nrm = e->sNrm;
    return p;
}

int sparse_grid(const shs_engine* e, uint64_t n) {
    return static_cast<int>(std::max<uint64_t>(
        1, std::min<uint64_t>((n + kSparseThreads - 1) / kSparseThreads, e->grid_cap)));
}

int launch_sparse_probs(shs_engine* e, uint32_t s, const DevStage* dev, int* nparts) {
    SparseParams p = sparse_params(e, s, dev);
    const uint64_t Kn = 2 * p.Ko;
    int end_bit = 1;
    while (end_bit < 64 && (e->N - 1) >> end_bit) ++end_bit;
    const int gf = sparse_grid(e, Kn);
    cudaError_t sort_err = cudaSuccess;
    int rc = launch(e, 0, [&] {
        if (s == 0) k_sparse_init<<<1, 1, 0, e->stream>>>(e->sZ[0], e->sV[0]);
        k_sparse_expand<<<sparse_grid(e, p.Ko), kSparseThreads, 0, e->stream>>>(p);
        size_t bytes = e->sTempBytes;
        sort_err = cub::DeviceRadixSort::SortPairs(e->sTemp, bytes, p.Zn, e->sKeys, e->sNrm,
                                                   e->sNrm2, static_cast<int>(Kn), 0, end_bit,
                                                   e->stream);
        k_sparse_fold<<<gf, kSparseThreads, 0, e->stream>>>(e->sKeys, e->sNrm2, Kn, e->partials);
    });
    if (rc) return rc;
    if (sort_err != cudaSuccess)
        return set_error(SHS_CUDA_ERROR, std::string("sparse sort: ") + cudaGetErrorString(sort_err));
    e->launches += 2;  // expand + fold (and the sort's own kernels) beside the counted one
    *nparts = gf;
    return SHS_OK;
}

int launch_sparse_collapse(shs_engine* e, uint32_t s, const DevStage* dev) {
    SparseParams p = sparse_params(e, s, dev);
    return launch(e, 2, [&] {
        k_sparse_collapse<<<sparse_grid(e, p.Ko), kSparseThreads, 0, e->stream>>>(p, 0);
    });
}

// the dense sel (X) from the support entering stage s (compressed when stage s
// runs compressed)
int materialize_sparse(shs_engine* e, uint32_t s) {
    const uint64_t K = uint64_t(1) << s;
    if (e->orb_want && e->orb_ready && e->orb_use[s]) {
        SHS_CUDA(cudaMemsetAsync(e->X, 0, sizeof(double2) * e->orb_r, e->stream));
        int rc = launch(e, -1, [&] {
            k_orb_scatter<<<sparse_grid(e, K), kSparseThreads, 0, e->stream>>>(
                e->sZ[s & 1], e->sV[s & 1], K, e->orb_rec, e->X);
        });
        e->e1 = false;
        e->rep_orb = true;
        e->orb_sel = 0;
        e->orb_prev = nullptr;
        return rc;
    }
    SHS_CUDA(cudaMemsetAsync(e->X, 0, sizeof(double2) * e->N, e->stream));
    int rc = launch(e, -1, [&] {
        k_sparse_scatter<<<sparse_grid(e, K), kSparseThreads, 0, e->stream>>>(e->sZ[s & 1],
                                                                           e->sV[s & 1], K, e->X);
    });
    e->e1 = false;
    return rc;
}

// Device-resident run (the default for engine_run): per stage the host queues
//   probs(s) -> k_finalize_measure(s) -> collapse(s)
// and the device measures and collapses without a host round trip. The host
// stays one stage behind: before queueing stage s's measurement it waits for
// stage s-1's record (the GPU is then running collapse(s-1) with probs(s)
// queued) to learn the observed prefix, from which it computes both candidate
// phases of stage s+1 with glibc (statevector.cpp:338). Results, errors and
// the final engine state equal the host-driven loop's (engine_run_host).
int ensure_device_run(shs_engine* e) {
    if (e->d_slots) return SHS_OK;
    SHS_CUDA(cudaMalloc(&e->d_slots, 2 * sizeof(DevStage)));
    SHS_CUDA(cudaHostAlloc(&e->h_rec, sizeof(StageRec) * e->t, cudaHostAllocMapped));
    SHS_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->d_rec), e->h_rec, 0));
    for (auto& ev : e->meas_ev) SHS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    e->device_bytes += 2 * sizeof(DevStage);
    return SHS_OK;
}

int engine_run_device(shs_engine* e, u64 seed, u64 idx, u128* j_out, u128* js_out,
                      shs_stage_trace* trace) {
    NvtxRange nvtx("shs run (device-resident)");
    int rc = ensure_buffers(e);
    if (rc) return rc;
    if ((rc = ensure_device_run(e))) return rc;
    state_init(e);
    std::memset(e->h_rec, 0, sizeof(StageRec) * e->t);
    MeasureCfg mc{seed, static_cast<u32>(idx), e->err.kind, e->err.delta, e->err.px, e->err.py,
                  e->opt.check_norms};
    u128 observed = 0, sampled = 0;
    double inv = 1.0;                        // host mirror of stage s's inv
    StageScalars sc = host_scalars(e, 0, 0, 1.0);
    // read stage r's record (its measure kernel has completed) and fold it in
    auto absorb = [&](uint32_t r) -> int {
        cudaError_t ce = cudaEventSynchronize(e->meas_ev[r & 1]);
        if (ce != cudaSuccess)
            return set_error(SHS_CUDA_ERROR, std::string("event sync: ") + cudaGetErrorString(ce));
        StageRec rec;  // written by the device; complete once its event has
        std::memcpy(&rec, e->h_rec + r, sizeof(rec));
        if (!rec.done) return set_error(SHS_CUDA_ERROR, "stage record missing");
        if (trace) {
            trace[r].cbit = r;
            trace[r].p1 = rec.p1;
            trace[r].sampled_bit = rec.sbit;
            trace[r].observed_bit = rec.obit;
            trace[r].classical_flip = static_cast<uint8_t>(rec.flip);
            trace[r].quantum_error_branch = static_cast<uint8_t>(rec.ebranch);
        }
        e->p0 = rec.p0;
        e->p1 = rec.p1;
        if (rec.status == SHS_ERROR)
            return set_error(SHS_ERROR, "statevector norm drifted beyond 1e-9 at stage " +
                                            std::to_string(r));
        if (rec.status == SHS_DEGENERATE_BRANCH)
            return set_error(SHS_DEGENERATE_BRANCH,
                             "impossible measurement branch at stage " + std::to_string(r));
        observed |= u128{static_cast<unsigned>(rec.obit)} << r;
        sampled |= u128{static_cast<unsigned>(rec.sbit)} << r;
        if (r + 1 < e->t) {
            const int src_group = rec.ebranch ? 1 - rec.sbit : rec.sbit;
            inv = 1.0 / std::sqrt(src_group == 1 ? rec.p1 : rec.p0);  // statevector.cpp:391
            sc = host_scalars(e, r + 1, observed, inv);
        }
        return SHS_OK;
    };
    auto fail = [&](int code) {
        cudaStreamSynchronize(e->stream);  // queued stages fold zeros (inv = 0): drain them
        if (e->timing) resolve_marks(e);
        e->pending = false;
        return code;
    };
    const uint32_t nsp = e->sparse_on ? e->sparse_n : 0;  // stages on the support
    if (nsp && (rc = carve_sparse(e))) return rc;
    for (uint32_t s = 0; s < e->t; ++s) {
        DevStage* cur = e->d_slots + (s & 1);
        DevStage* nxt = e->d_slots + ((s + 1) & 1);
        int nparts = 0;
        e->sc = sc;  // stage 0's kernel arguments (later stages read the slot)
        if (s < nsp) {
            if ((rc = launch_sparse_probs(e, s, s == 0 ? nullptr : cur, &nparts))) return fail(rc);
        } else {
            if (s == nsp && nsp && (rc = materialize_sparse(e, s))) return fail(rc);
            if ((rc = launch_probs_pass(e, s, s == 0 ? nullptr : cur, &nparts))) return fail(rc);
        }
        // the observed prefix through stage s-1
        if (s > 0 && (rc = absorb(s - 1))) return fail(rc);
        MeasureStep ms{};
        ms.cfg = mc;
        ms.s = s;
        ms.collapse = s + 1 < e->t ? 1 : 0;
        ms.init_cur = s == 0 ? 1 : 0;
        ms.sc0 = sc;
        ms.cur = cur;
        ms.next = nxt;
        if (s + 1 < e->t) {
            for (int bit = 0; bit < 2; ++bit) {
                const StageScalars c =
                    host_scalars(e, s + 1, observed | (u128{static_cast<unsigned>(bit)} << s), 0.0);
                ms.nph.phr[bit] = c.phr;
                ms.nph.phi[bit] = c.phi;
                ms.nph.phase_mul[bit] = c.phase_mul;
            }
        }
        ms.rec = e->d_rec;
        rc = launch(e, 1, [&] {
            // programmatic dependent of the probs pass's last kernel (k_tile_fixup1
            // triggers at its start; the others at their end): its first
            // instruction waits for them
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(1);
            cfg.blockDim = dim3(kFinalizeThreads);
            cfg.stream = e->stream;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = e->pdl ? 1 : 0;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k_finalize_measure, static_cast<const unsigned long long*>(e->partials),
                               nparts, static_cast<const double*>(e->S), e->nb, e->kahan ? 1 : 0, ms);
        });
        if (rc) return fail(rc);
        if (cudaEventRecord(e->meas_ev[s & 1], e->stream) != cudaSuccess)
            return fail(set_error(SHS_CUDA_ERROR, "event record"));
        if (s + 1 < e->t) {
            rc = s < nsp ? launch_sparse_collapse(e, s, cur) : launch_collapse_pass(e, s, 0, cur);
            if (rc) return fail(rc);
        }
    }
    if ((rc = absorb(e->t - 1))) return fail(rc);
    if ((rc = sync(e))) return rc;
    // engine state as the host-driven loop leaves it: stage t-1 pending
    e->ps = e->t - 1;
    e->inv = inv;
    e->sc = sc;
    e->pending = true;
    u128 j = observed;
    if (e->err.kind == SHS_ERR_BITFLIP)
        j = bitflip_bitstring(j, e->t, e->err.delta, seed, static_cast<u32>(idx));
    *j_out = j;
    if (js_out) *js_out = sampled;
    return SHS_OK;
}

int engine_run_host(shs_engine* e, u64 seed, u64 idx, u128* j_out, u128* js_out,
                    shs_stage_trace* trace) {
    NvtxRange nvtx("shs run (host-driven)");
    state_init(e);
    u128 observed = 0, sampled = 0;
    for (uint32_t s = 0; s < e->t; ++s) {
        double p0, p1;
        int rc = stage_probs(e, s, observed, &p0, &p1);
        if (rc) return rc;
        Measurement mr = sample_measurement(p1, seed, static_cast<u32>(idx), s, e->err);
        if (trace) {
            trace[s].cbit = s;
            trace[s].p1 = p1;
            trace[s].sampled_bit = mr.sampled_bit;
            trace[s].observed_bit = mr.observed_bit;
            trace[s].classical_flip = mr.classical_flip ? 1 : 0;
            trace[s].quantum_error_branch = mr.error_branch ? 1 : 0;
        }
        observed |= u128{static_cast<unsigned>(mr.observed_bit)} << s;
        sampled |= u128{static_cast<unsigned>(mr.sampled_bit)} << s;
        if (s + 1 < e->t) {
            const int src_group = mr.error_branch ? 1 - mr.sampled_bit : mr.sampled_bit;
            const double p_src = src_group == 1 ? p1 : p0;
            rc = stage_collapse(e, src_group, p_src, false);
            if (rc) return rc;
        }
    }
    u128 j = observed;
    if (e->err.kind == SHS_ERR_BITFLIP)
        j = bitflip_bitstring(j, e->t, e->err.delta, seed, static_cast<u32>(idx));
    *j_out = j;
    if (js_out) *js_out = sampled;
    return SHS_OK;
}

int engine_run(shs_engine* e, u64 seed, u64 idx, u128* j_out, u128* js_out,
               shs_stage_trace* trace) {
    if (e->group) return group_run(e->group, seed, idx, j_out, js_out, trace);
    return e->host_measure ? engine_run_host(e, seed, idx, j_out, js_out, trace)
                           : engine_run_device(e, seed, idx, j_out, js_out, trace);
}

bool batchable(const shs_engine* e) {
    return !e->group && e->N <= kBatchMaxN && e->t <= kBatchMaxT;
}

// Device tables for whole-run batches: multipliers, inverses (+ Shoup) and the
// phase table std::polar(1, stage_phase(s, p)) for every (s, prefix) computed
// here with glibc, exactly as the per-stage driver computes each phase.
int ensure_batch_tables(shs_engine* e) {
    if (e->d_phase) return SHS_OK;
    std::vector<uint64_t> invsh(e->t, 0);
    for (uint32_t s = 0; s < e->t; ++s)
        if (e->a_pows[s] != 1) invsh[s] = shoup(e->a_invs[s], e->N);
    const uint64_t entries = (uint64_t(1) << e->t) - 1;
    std::vector<double2> phase(std::max<uint64_t>(entries, 1));
    for (uint32_t s = 0; s < e->t; ++s)
        for (uint64_t pfx = 0; pfx < (uint64_t(1) << s); ++pfx) {
            const double phi = stage_phase(s, pfx);
            phase[((uint64_t(1) << s) - 1) + pfx] = make_double2(1.0 * std::cos(phi), 1.0 * std::sin(phi));
        }
    SHS_CUDA(cudaMalloc(&e->d_apows, sizeof(uint64_t) * e->t));
    SHS_CUDA(cudaMalloc(&e->d_ainvs, sizeof(uint64_t) * e->t));
    SHS_CUDA(cudaMalloc(&e->d_ainvsh, sizeof(uint64_t) * e->t));
    SHS_CUDA(cudaMalloc(&e->d_phase, sizeof(double2) * phase.size()));
    SHS_CUDA(cudaMemcpy(e->d_apows, e->a_pows.data(), sizeof(uint64_t) * e->t, cudaMemcpyHostToDevice));
    SHS_CUDA(cudaMemcpy(e->d_ainvs, e->a_invs.data(), sizeof(uint64_t) * e->t, cudaMemcpyHostToDevice));
    SHS_CUDA(cudaMemcpy(e->d_ainvsh, invsh.data(), sizeof(uint64_t) * e->t, cudaMemcpyHostToDevice));
    SHS_CUDA(cudaMemcpy(e->d_phase, phase.data(), sizeof(double2) * phase.size(), cudaMemcpyHostToDevice));
    const size_t smem = batch_smem_bytes(e->N);
    {  // the attribute is process-wide: set it once per device to the largest size any
       // engine needs (per-engine values raced between harness threads: a launch of a
       // larger problem failed with "invalid argument" after another thread lowered it)
        static std::mutex mu;
        static std::vector<int> done;
        std::lock_guard<std::mutex> g(mu);
        if (std::find(done.begin(), done.end(), e->dev) == done.end()) {
            SHS_CUDA(cudaFuncSetAttribute(k_batch_runs, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(batch_smem_bytes(kBatchMaxN))));
            done.push_back(e->dev);
        }
    }
    int occ = 0;
    SHS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_batch_runs, batch_threads(e->N), smem));
    e->batch_grid = std::max(1, occ) * e->num_sms;
    e->device_bytes += sizeof(uint64_t) * 3 * e->t + sizeof(double2) * phase.size();
    return SHS_OK;
}

// `count` whole runs idx0 .. idx0+count-1 in one launch (one CTA per run).
// Lockstep multi-shot runs (lockstep.cuh) for mid-size N: up to `cap` shots at
// a time advance stage by stage together; the host stays one stage behind,
// computing both candidate phases of every shot's next stage with glibc.
constexpr uint64_t kLockMaxN = uint64_t(1) << 22;           // beyond: engine_run per shot
constexpr uint64_t kLockBudget = uint64_t(16) << 30;         // HBM for the batch's states
constexpr uint64_t kLockMinShots = 64;

bool lockstep_ok(const shs_engine* e, uint32_t count) {
    return count >= 1 && !e->group && !batchable(e) && e->N <= kLockMaxN;
}

int run_many_lockstep(shs_engine* e, u64 seed, u64 idx0, uint32_t count, uint64_t* j,
                      uint64_t* js, double* p1, int32_t* bits) {
    const uint64_t N = e->N, nb = e->nb, t = e->t;
    const uint64_t per_shot = 2 * sizeof(double2) * N + 2 * sizeof(double) * nb;
    // shots per batch: 2^24 / N (all of a campaign problem's M shots while N is
    // small), at least 64 (measured at N = 2^18: 8 / 16 / 32 / 64 / 256 shots per
    // batch -> 205 / 129 / 155 / 116 / 146 ms for 256 shots), at most kLockBudget
    uint64_t want = std::max<uint64_t>(kLockMinShots, (uint64_t(1) << 24) / N);
    if (const char* v = std::getenv("SHS_LOCK_BATCH")) want = std::max(1ull, std::strtoull(v, nullptr, 10));
    const uint32_t B = static_cast<uint32_t>(std::max<uint64_t>(
        1, std::min<uint64_t>({uint64_t(count), want, kLockBudget / per_shot})));
    // one chunk per CTA: the grid runs shot-major (blockIdx.x fastest), so only
    // the ~(resident CTAs / nchunks) shots in flight share the L2 and their
    // gathered reads hit it (N = 2^18: a shot is 4.2 MB; 64 shots at once at
    // ~10 CTAs each thrashed it, probs + collapse at 1.6 / 2.4 TB/s)
    const int G = static_cast<int>(std::max<uint64_t>(1, e->nchunks));
    // the warp-specialized probs pass walks kLockWsChunks chunks per CTA
    const int Gp = e->lock_ws ? static_cast<int>((e->nchunks + kLockWsChunks - 1) / kLockWsChunks) : G;
    LockBufs L;
    auto cleanup = [&] {
        cudaStreamSynchronize(e->stream);
        lock_return(L);
    };
    cudaError_t ce = lock_checkout(
        e->dev, sizeof(double2) * N * B, sizeof(double) * 2 * nb * B,
        sizeof(unsigned long long) * 2 * kDigits * G * B, B, sizeof(StageRec) * t * B, L);
    if (ce != cudaSuccess)
        return set_error(SHS_CUDA_ERROR, std::string("lockstep buffers: ") + cudaGetErrorString(ce));
    double2 *X = L.X, *Y = L.Y;
    double* S = L.S;
    unsigned long long* parts = L.parts;
    DevStage* slots = L.slots;
    NextPhase* d_nph = L.d_nph;
    NextPhase* h_nph = L.h_nph;
    StageRec* h_rec = L.h_rec;
    StageRec* d_rec = L.d_rec;
    cudaEvent_t* ev = L.ev;
    std::vector<u128> observed(B), sampled(B);
    for (uint32_t b0 = 0; b0 < count; b0 += B) {
        const uint32_t nbat = std::min<uint32_t>(B, count - b0);
        std::memset(h_rec, 0, sizeof(StageRec) * t * B);
        std::fill(observed.begin(), observed.end(), u128{0});
        std::fill(sampled.begin(), sampled.end(), u128{0});
        LockParams lp{};
        lp.X = X;
        lp.Y = Y;
        lp.N = N;
        lp.nb = nb;
        lp.nchunks = e->nchunks;
        lp.sc0 = host_scalars(e, 0, 0, 1.0);
        lp.slots = slots;
        lp.S = S;
        lp.partials = parts;
        const dim3 grid(G, nbat);
        // stage r's records, then every shot's candidates for stage r + 2
        auto absorb = [&](uint32_t r) -> int {
            if ((ce = cudaEventSynchronize(ev[r & 1])) != cudaSuccess)
                return set_error(SHS_CUDA_ERROR, std::string("event sync: ") + cudaGetErrorString(ce));
            for (uint32_t i = 0; i < nbat; ++i) {
                StageRec rec;
                std::memcpy(&rec, h_rec + uint64_t(i) * t + r, sizeof(rec));
                if (!rec.done) return set_error(SHS_CUDA_ERROR, "stage record missing");
                if (rec.status == SHS_ERROR)
                    return set_error(SHS_ERROR, "statevector norm drifted beyond 1e-9 at stage " +
                                                    std::to_string(r));
                if (rec.status == SHS_DEGENERATE_BRANCH)
                    return set_error(SHS_DEGENERATE_BRANCH,
                                     "impossible measurement branch at stage " + std::to_string(r));
                observed[i] |= u128{static_cast<unsigned>(rec.obit)} << r;
                sampled[i] |= u128{static_cast<unsigned>(rec.sbit)} << r;
            }
            return SHS_OK;
        };
        int rc = SHS_OK;
        for (uint32_t s = 0; s < t && rc == SHS_OK; ++s) {
            const bool gather = e->a_pows[s] != 1;
            lp.m = e->a_invs[s];
            lp.m_sh = gather ? shoup(lp.m, N) : 0;
            lp.m_step = gather ? mulmod(lp.m, kBlock, N) : 0;
            lp.gather = gather ? 1 : 0;
            lp.e1 = s == 0 ? 1 : 0;
            lp.cur = static_cast<int>(s & 1);
            lp.spec = e->lock_ws && e->spec_on && s + 1 < t ? 1 : 0;  // probs and collapse of stage s
            if (e->lock_ws)
                rc = launch(e, 0, [&] {
                    k_lock_probs_ws<<<dim3(Gp, nbat), kLockWsThreads, kLockWsSmem, e->stream>>>(lp);
                });
            else
                rc = launch(e, 0, [&] { k_lock_probs<<<grid, kThreads, 0, e->stream>>>(lp); });
            if (rc) break;
            if (s > 0 && (rc = absorb(s - 1))) break;
            NextPhase* hn = h_nph + (s & 1) * B;
            if (s + 1 < t) {
                for (uint32_t i = 0; i < nbat; ++i)
                    for (int bit = 0; bit < 2; ++bit) {
                        const StageScalars c = host_scalars(
                            e, s + 1, observed[i] | (u128{static_cast<unsigned>(bit)} << s), 0.0);
                        hn[i].phr[bit] = c.phr;
                        hn[i].phi[bit] = c.phi;
                        hn[i].phase_mul[bit] = c.phase_mul;
                    }
            }
            NextPhase* dn = d_nph + (s & 1) * B;
            if ((ce = cudaMemcpyAsync(dn, hn, sizeof(NextPhase) * nbat, cudaMemcpyHostToDevice,
                                      e->stream)) != cudaSuccess) {
                rc = set_error(SHS_CUDA_ERROR, std::string("candidates: ") + cudaGetErrorString(ce));
                break;
            }
            LockMeasure q{};
            q.seed = seed;
            q.idx0 = idx0 + b0;
            q.kind = e->err.kind;
            q.delta = e->err.delta;
            q.px = e->err.px;
            q.py = e->err.py;
            q.check_norms = e->opt.check_norms;
            q.s = s;
            q.t = static_cast<uint32_t>(t);
            q.collapse = s + 1 < t ? 1 : 0;
            q.kahan = e->kahan ? 1 : 0;
            q.nparts = Gp;
            q.nph = dn;
            q.rec = d_rec;
            rc = launch(e, 1, [&] { k_lock_measure<<<nbat, kFinalizeThreads, 0, e->stream>>>(lp, q); });
            if (rc) break;
            if ((ce = cudaEventRecord(ev[s & 1], e->stream)) != cudaSuccess) {
                rc = set_error(SHS_CUDA_ERROR, "event record");
                break;
            }
            if (s + 1 < t) {
                rc = launch(e, 2, [&] { k_lock_collapse<<<grid, kThreads, 0, e->stream>>>(lp); });
                std::swap(lp.X, lp.Y);
            }
        }
        if (rc == SHS_OK) rc = absorb(static_cast<uint32_t>(t - 1));
        if (rc) {
            cleanup();
            return rc;
        }
        for (uint32_t i = 0; i < nbat; ++i) {
            const uint64_t o = b0 + i;
            u128 jj = observed[i];
            if (e->err.kind == SHS_ERR_BITFLIP)
                jj = bitflip_bitstring(jj, static_cast<unsigned>(t), e->err.delta, seed,
                                       static_cast<u32>(idx0 + o));
            j[2 * o] = static_cast<uint64_t>(jj);
            j[2 * o + 1] = static_cast<uint64_t>(jj >> 64);
            if (js) {
                js[2 * o] = static_cast<uint64_t>(sampled[i]);
                js[2 * o + 1] = static_cast<uint64_t>(sampled[i] >> 64);
            }
            for (uint64_t s = 0; s < t; ++s) {
                const StageRec& rec = h_rec[uint64_t(i) * t + s];
                if (p1) p1[o * t + s] = rec.p1;
                if (bits) {
                    int32_t* b = bits + (o * t + s) * 4;
                    b[0] = rec.sbit;
                    b[1] = rec.obit;
                    b[2] = rec.flip;
                    b[3] = rec.ebranch;
                }
            }
        }
    }
    cleanup();
    if (e->timing) resolve_marks(e);
    state_init(e);  // the engine's own buffers were not touched
    return SHS_OK;
}

int run_many_batched(shs_engine* e, u64 seed, u64 idx0, uint32_t count, uint64_t* j,
                     uint64_t* js, double* p1, int32_t* bits) {
    int rc = ensure_batch_tables(e);
    if (rc) return rc;
    const size_t jb = sizeof(uint64_t) * 2 * count;
    const size_t pb = p1 ? sizeof(double) * count * e->t : 0;
    const size_t bb = bits ? sizeof(int32_t) * 4 * count * e->t : 0;
    const size_t sb = sizeof(int32_t) * count;
    const size_t need = 2 * jb + pb + bb + sb + 64;
    if (need > e->batch_out_bytes) {
        cudaFree(e->d_batch_out);
        e->d_batch_out = nullptr;
        SHS_CUDA(cudaMalloc(&e->d_batch_out, need));
        e->batch_out_bytes = need;
    }
    char* base = static_cast<char*>(e->d_batch_out);
    BatchParams bp{};
    bp.N = e->N;
    bp.t = e->t;
    bp.seed = seed;
    bp.idx0 = idx0;
    bp.count = count;
    bp.a_pows = e->d_apows;
    bp.a_invs = e->d_ainvs;
    bp.a_invsh = e->d_ainvsh;
    bp.phase = e->d_phase;
    bp.w0r = e->w[0];
    bp.w0i = e->w[1];
    bp.w1r = e->w[2];
    bp.w1i = e->w[3];
    bp.kind = e->err.kind;
    bp.delta = e->err.delta;
    bp.px = e->err.px;
    bp.py = e->err.py;
    bp.check_norms = e->opt.check_norms;
    bp.j_out = reinterpret_cast<uint64_t*>(base);
    bp.js_out = reinterpret_cast<uint64_t*>(base + jb);
    bp.p1_out = p1 ? reinterpret_cast<double*>(base + 2 * jb) : nullptr;
    bp.bits_out = bits ? reinterpret_cast<int32_t*>(base + 2 * jb + pb) : nullptr;
    bp.status = reinterpret_cast<int32_t*>(base + 2 * jb + pb + bb);
    const int g = static_cast<int>(std::min<uint64_t>(count, static_cast<uint64_t>(e->batch_grid)));
    rc = launch(e, -1, [&] {
        k_batch_runs<<<g, batch_threads(e->N), batch_smem_bytes(e->N), e->stream>>>(bp);
    });
    if (rc) return rc;
    std::vector<int32_t> status(count);
    SHS_CUDA(cudaMemcpyAsync(status.data(), bp.status, sb, cudaMemcpyDeviceToHost, e->stream));
    SHS_CUDA(cudaMemcpyAsync(j, bp.j_out, jb, cudaMemcpyDeviceToHost, e->stream));
    if (js) SHS_CUDA(cudaMemcpyAsync(js, bp.js_out, jb, cudaMemcpyDeviceToHost, e->stream));
    if (p1) SHS_CUDA(cudaMemcpyAsync(p1, bp.p1_out, pb, cudaMemcpyDeviceToHost, e->stream));
    if (bits) SHS_CUDA(cudaMemcpyAsync(bits, bp.bits_out, bb, cudaMemcpyDeviceToHost, e->stream));
    rc = sync(e);
    if (rc) return rc;
    for (uint32_t i = 0; i < count; ++i) {
        if (status[i] == SHS_ERROR)
            return set_error(SHS_ERROR, "statevector norm drifted beyond 1e-9 (run " +
                                            std::to_string(idx0 + i) + ")");
        if (status[i] == SHS_DEGENERATE_BRANCH)
            return set_error(SHS_DEGENERATE_BRANCH,
                             "impossible measurement branch (run " + std::to_string(idx0 + i) + ")");
    }
    return SHS_OK;
}

template <typename F>
int guarded(shs_engine* e, F&& f) {
    if (!e) return set_error(SHS_INVALID_ARGUMENT, "null engine");
    cudaError_t err = cudaSetDevice(e->dev);
    if (err != cudaSuccess) return set_error(SHS_CUDA_ERROR, cudaGetErrorString(err));
    return f();
}

}  // namespace

// ---------------------------------------------------------------------------
extern "C" {

void shs_default_options(shs_options* o) {
    o->shard_count = 4;
    o->workers = 1;
    o->qubit_ceiling = 26;
    o->check_norms = 1;
    o->device = 0;
    o->combine = SHS_COMBINE_AUTO;
    o->tiling = SHS_TILING_AUTO;
    o->n_devices = 0;
    o->devices = nullptr;
}

const char* shs_last_error(void) { return last_error(); }

const char* shs_build_info(void) {
    return "shorsim_b200: sm_100a, fp64 no-FMA (--fmad=false), nvcc " SHS_NVCC_VERSION;
}

// Which stages run compressed (orbit.cuh): maximal runs of >= 2 consecutive
// stages with whole-band tile plans (k_tiled<., false>), on a single-device
// engine from kOrbitMinN, when the orbit fills at most half of Z_N (2 slots per
// buffer). The order r comes from a baby-step giant-step search (sparse_plan.hpp).
namespace {
void plan_orbit(shs_engine* e) {
    e->orb_use.assign(e->t, 0);
    e->orb_r = 0;
    const char* env = std::getenv("SHS_ORBIT");  // SHS_ORBIT=0: dense stages only
    e->orb_want = !(env && env[0] == '0');
    uint64_t min_n = kOrbitMinN;
    if (const char* mn = std::getenv("SHS_ORBIT_MIN_LOG2"))  // A/B hook
        min_n = uint64_t(1) << std::min(62, std::atoi(mn));
    if (e->group || e->N < min_n) return;
    std::vector<uint8_t> cap(e->t, 0);
    for (uint32_t s = 1; s < e->t; ++s)
        cap[s] = e->a_pows[s] != 1 && e->plans[s].tiled;
    bool any = false;
    for (uint32_t s = 1; s < e->t;) {
        uint32_t s1 = s;
        while (s1 < e->t && cap[s1]) ++s1;
        if (s1 - s >= 2) {
            for (uint32_t k = s; k < s1; ++k) e->orb_use[k] = 1;
            any = true;
        }
        s = s1 + 1;
    }
    if (!any) return;
    const uint64_t r = small_order(e->prob.a % e->N, e->N, e->N);
    const uint64_t pad = (r + 63) / 64 * 64;
    if (r == 0 || 2 * pad > e->N) {
        e->orb_use.assign(e->t, 0);
        return;
    }
    e->orb_r = r;
    e->orb_pad = pad;
}
}  // namespace

int shs_engine_create(const shs_problem* problem, const shs_error* error,
                      const shs_options* options, shs_engine** out) {
    if (!problem || !error || !out) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    shs_options o;
    if (options) o = *options;
    else shs_default_options(&o);
    int rc = validate_engine_config(*problem, *error, o);
    if (rc) return rc;
    auto* e = new shs_engine;
    e->prob = *problem;
    e->err = *error;
    e->opt = o;
    e->N = problem->N;
    e->t = problem->t;
    e->dev = o.device;
    reinit_state(e->err, e->w);
    // stage multipliers by backward squaring, statevector.cpp:302-306
    e->a_pows.assign(e->t, 0);
    e->a_invs.assign(e->t, 1);
    e->a_pows[e->t - 1] = problem->a % problem->N;
    for (uint32_t s = e->t - 1; s > 0; --s)
        e->a_pows[s - 1] = mulmod(e->a_pows[s], e->a_pows[s], e->N);
    for (uint32_t s = 0; s < e->t; ++s) {  // statevector.cpp:308-320 (no tables kept)
        if (e->a_pows[s] == 1) continue;
        u64 g = 0;
        if (mod_inverse(e->a_pows[s], e->N, &e->a_invs[s], &g) != SHS_OK) {
            std::string msg = "not invertible: gcd(" + std::to_string(e->a_pows[s]) + ", " +
                              std::to_string(e->N) + ") = " + std::to_string(g);
            delete e;
            return set_error(SHS_NOT_INVERTIBLE, msg);
        }
    }
    {
        std::vector<std::pair<uint64_t, TilePlanHost>> cache;  // per distinct multiplier
        e->plans.assign(e->t, TilePlanHost{});
        for (uint32_t s = 1; s < e->t; ++s) {  // stage 0 always starts from |1> (direct kernels)
            if (e->a_pows[s] == 1) continue;
            auto it = std::find_if(cache.begin(), cache.end(),
                                   [&](const auto& kv) { return kv.first == e->a_pows[s]; });
            if (it == cache.end()) {
                cache.emplace_back(e->a_pows[s],
                                   make_tile_plan(e->a_pows[s], e->a_invs[s], e->N, o.tiling,
                                                  small_a_scratch(e->N)));
                it = cache.end() - 1;
            }
            e->plans[s] = it->second;
            if (it->second.tiled) e->max_rows = std::max(e->max_rows, it->second.H);
        }
    }
    e->nb = (e->N + kBlock - 1) / kBlock;
    e->nchunks = (e->N + kChunk - 1) / kChunk;
    e->kahan = o.combine == SHS_COMBINE_KAHAN ||
               (o.combine == SHS_COMBINE_AUTO && e->nb <= kKahanMaxBlocks);

    auto fail = [&](cudaError_t err, const char* what) {
        std::string msg = std::string(what) + ": " + cudaGetErrorString(err);
        release(e);
        return set_error(SHS_CUDA_ERROR, msg);
    };
    cudaError_t ce = cudaSetDevice(e->dev);
    if (ce != cudaSuccess) return fail(ce, "cudaSetDevice");
    // two attributes, not cudaGetDeviceProperties (which queries every field:
    // milliseconds per engine, and the campaign harness creates one per problem)
    int major = 0, sms = 0;
    if ((ce = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, e->dev)) != cudaSuccess ||
        (ce = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, e->dev)) != cudaSuccess)
        return fail(ce, "cudaDeviceGetAttribute");
    if (major < 10) {
        release(e);
        return set_error(SHS_CUDA_ERROR, "device is not sm_100-class (B200 required)");
    }
    e->num_sms = sms;
    e->tiled_cap = e->num_sms;
    e->max_rows = 0;
    // test hook: SHS_TILE_SPLIT=0 / 1 forces the tiled kernels' work-split variant
    const char* force_split = std::getenv("SHS_TILE_SPLIT");
    for (auto& pl : e->plans) {
        if (!pl.tiled) continue;
        make_tile_split(pl, e->tiled_cap);
        if (force_split && (force_split[0] == '0' || force_split[0] == '1'))
            pl.split_tail = force_split[0] == '1';
        if (o.tiling == SHS_TILING_AUTO &&
            pl.chunks < kTileMinChunksPerCTA * static_cast<uint64_t>(e->tiled_cap))
            pl.tiled = false;
        if (pl.tiled) e->max_rows = std::max(e->max_rows, pl.H);
    }
    int occ = 0;
    ce = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stage_probs<kSrcGather, false, false>, kThreads, 0);
    if (ce != cudaSuccess) return fail(ce, "occupancy");
    e->grid_cap = std::max(1, occ) * e->num_sms;
    // one persistent TMA-pipelined CTA per SM for the tiled passes
    // kSrcStreams: up to kStreamsMaxA * 5 staged amplitudes (80 KB) of dynamic smem
    for (auto fn : {k_stage_probs<kSrcStreams, false, false>, k_stage_probs<kSrcStreams, true, false>,
                    k_stage_probs<kSrcStreams, false, true>,
                    k_stage_collapse<kSrcStreams, false, false>, k_stage_collapse<kSrcStreams, true, false>,
                    k_stage_collapse<kSrcStreams, false, true>, k_stage_collapse<kSrcStreams, true, true>}) {
        ce = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sizeof(double2) * kStreamsMaxA * 5));
        if (ce != cudaSuccess) return fail(ce, "cudaFuncSetAttribute(streams)");
    }
    for (auto fn : {k_tiled<true, false>, k_tiled<true, true>}) {
        ce = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(tile_smem_bytes<true>()));
        if (ce != cudaSuccess) return fail(ce, "cudaFuncSetAttribute(k_tiled<probs>)");
    }
    for (auto fn : {k_tiled<true, false, true>, k_tiled<true, true, true>}) {
        ce = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(tile_smem_bytes<true, true>()));
        if (ce != cudaSuccess) return fail(ce, "cudaFuncSetAttribute(k_tiled<orbit>)");
    }
    for (auto fn : {k_tiled<false, false>, k_tiled<false, true>}) {
        ce = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(tile_smem_bytes<false>()));
        if (ce != cudaSuccess) return fail(ce, "cudaFuncSetAttribute(k_tiled<collapse>)");
    }
    ce = cudaFuncSetAttribute(k_tile_fixup, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(kFixSmem));
    if (ce != cudaSuccess) return fail(ce, "cudaFuncSetAttribute(k_tile_fixup)");
    ce = cudaFuncSetAttribute(k_tile_fixup1, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(kFix1Smem));
    if (ce != cudaSuccess) return fail(ce, "cudaFuncSetAttribute(k_tile_fixup1)");
    ce = cudaFuncSetAttribute(k_lock_probs_ws, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(kLockWsSmem));
    if (ce != cudaSuccess) return fail(ce, "cudaFuncSetAttribute(k_lock_probs_ws)");
    e->fixup_cap = 3 * e->num_sms;  // 3 x 68 KB of transposed head slabs per SM
    {
        const char* hm = std::getenv("SHS_HOST_MEASURE");
        e->host_measure = hm && hm[0] == '1';
        const char* ls = std::getenv("SHS_LOCKSTEP");
        e->lockstep = !(ls && ls[0] == '0');
        const char* lw = std::getenv("SHS_LOCK_WS");  // A/B: 0 = k_lock_probs
        e->lock_ws = !(lw && lw[0] == '0');
        const char* sp = std::getenv("SHS_SPEC");  // A/B: 0 = every collapse runs
        e->spec_on = !(sp && sp[0] == '0');
        const char* pd = std::getenv("SHS_PDL");  // A/B: 0 = plain launches
        e->pdl = !(pd && pd[0] == '0');
    }
    ce = cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking);
    if (ce != cudaSuccess) return fail(ce, "cudaStreamCreate");
    const size_t part_bytes = sizeof(unsigned long long) * 2 * kDigits *
                              std::max(e->grid_cap, e->tiled_cap + e->fixup_cap);
    if ((ce = cudaMalloc(&e->partials, part_bytes)) != cudaSuccess)
        return fail(ce, "cudaMalloc(partials)");
    if ((ce = cudaMalloc(&e->d_out, 4 * sizeof(double))) != cudaSuccess)
        return fail(ce, "cudaMalloc(out)");
    if ((ce = cudaMalloc(&e->band_ctr, sizeof(unsigned long long))) != cudaSuccess ||
        (ce = cudaMemset(e->band_ctr, 0, sizeof(unsigned long long))) != cudaSuccess)
        return fail(ce, "cudaMalloc(band_ctr)");
    if ((ce = cudaHostAlloc(&e->h_out, 4 * sizeof(double), cudaHostAllocDefault)) != cudaSuccess)
        return fail(ce, "cudaHostAlloc");
    e->device_bytes = part_bytes + 32;  // the N-amplitude buffers come with the first stage
    e->sparse_n = plan_sparse_prefix(e);
    state_init(e);
    {  // multi-device: options.n_devices, AUTO by the state's size
        std::vector<int> devs;
        if (o.n_devices >= 2) {
            if (o.n_devices > SHS_MAX_SHARDS) {
                release(e);
                return set_error(SHS_INVALID_ARGUMENT, "n_devices must be <= 16");
            }
            for (int q = 0; q < o.n_devices; ++q) devs.push_back(o.devices ? o.devices[q] : o.device + q);
        } else if (o.n_devices < 0) {
            if ((rc = plan_devices(e->N, o.device, &devs))) {
                release(e);
                return rc;
            }
        }
        if (devs.size() >= 2) {
            if ((rc = group_create(*problem, *error, o, devs, &e->group))) {
                release(e);
                return rc;
            }
            e->sparse_n = 0;  // the group runs every stage dense
        }
    }
    plan_orbit(e);
    *out = e;
    return SHS_OK;
}

void shs_engine_destroy(shs_engine* e) { release(e); }

int shs_engine_set_orbit(shs_engine* e, int32_t enable) {
    if (!e) return set_error(SHS_INVALID_ARGUMENT, "null engine");
    if (e->rep_orb || e->pending) state_init(e);  // takes effect from a fresh state
    e->orb_want = enable != 0;
    return SHS_OK;
}

int shs_engine_orbit_stages(const shs_engine* e, uint8_t* out) {
    if (!e || !out) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    for (uint32_t s = 0; s < e->t; ++s) out[s] = e->orb_want && e->orb_r && e->orb_use[s] ? 1 : 0;
    return SHS_OK;
}

int shs_engine_orbit_info(const shs_engine* e, uint64_t out[3]) {
    if (!e || !out) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    out[0] = e->orb_want ? e->orb_r : 0;
    out[1] = 0;
    out[2] = 0;
    if (!out[0]) return SHS_OK;
    for (uint32_t s = e->t; s-- > 0;)
        if (e->orb_use[s]) {
            out[1] += 1;
            out[2] = s;
        }
    return SHS_OK;
}

uint32_t shs_engine_stages(const shs_engine* e) { return e ? e->t : 0; }

int shs_engine_set_sparse(shs_engine* e, int32_t enable) {
    if (!e) return set_error(SHS_INVALID_ARGUMENT, "null engine");
    e->sparse_on = enable != 0;
    if (e->group) group_set_sparse(e->group, enable != 0);
    return SHS_OK;
}

uint32_t shs_engine_sparse_stages(const shs_engine* e) {
    if (e && e->group) return group_sparse_stages(e->group);
    return e && e->sparse_on ? e->sparse_n : 0;
}

int shs_engine_stage_multipliers(const shs_engine* e, uint64_t* out) {
    if (!e || !out) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    std::memcpy(out, e->a_pows.data(), sizeof(uint64_t) * e->t);
    return SHS_OK;
}

int shs_engine_run(shs_engine* e, uint64_t seed, uint64_t idx, uint64_t j[2],
                   uint64_t j_sampled[2], shs_stage_trace* trace) {
    return guarded(e, [&] {
        u128 jj = 0, js = 0;
        int rc = engine_run(e, seed, idx, &jj, &js, trace);
        if (rc) return rc;
        if (j) {
            j[0] = static_cast<uint64_t>(jj);
            j[1] = static_cast<uint64_t>(jj >> 64);
        }
        if (j_sampled) {
            j_sampled[0] = static_cast<uint64_t>(js);
            j_sampled[1] = static_cast<uint64_t>(js >> 64);
        }
        return SHS_OK;
    });
}

int shs_engine_run_many(shs_engine* e, uint64_t seed, uint64_t idx0, uint32_t count,
                        uint64_t* j, uint64_t* j_sampled, double* p1, int32_t* bits) {
    return guarded(e, [&]() -> int {
        if (!j) return set_error(SHS_INVALID_ARGUMENT, "null output");
        if (count == 0) return SHS_OK;
        if (batchable(e)) return run_many_batched(e, seed, idx0, count, j, j_sampled, p1, bits);
        if (lockstep_ok(e, count) && e->lockstep)
            return run_many_lockstep(e, seed, idx0, count, j, j_sampled, p1, bits);
        std::vector<shs_stage_trace> tr(e->t);
        for (uint32_t i = 0; i < count; ++i) {
            u128 jj = 0, js = 0;
            int rc = engine_run(e, seed, idx0 + i, &jj, &js, tr.data());
            if (rc) return rc;
            j[2 * i] = static_cast<uint64_t>(jj);
            j[2 * i + 1] = static_cast<uint64_t>(jj >> 64);
            if (j_sampled) {
                j_sampled[2 * i] = static_cast<uint64_t>(js);
                j_sampled[2 * i + 1] = static_cast<uint64_t>(js >> 64);
            }
            for (uint32_t s = 0; s < e->t; ++s) {
                if (p1) p1[uint64_t(i) * e->t + s] = tr[s].p1;
                if (bits) {
                    int32_t* o = bits + (uint64_t(i) * e->t + s) * 4;
                    o[0] = tr[s].sampled_bit;
                    o[1] = tr[s].observed_bit;
                    o[2] = tr[s].classical_flip;
                    o[3] = tr[s].quantum_error_branch;
                }
            }
        }
        return SHS_OK;
    });
}

int shs_engine_batched(const shs_engine* e) {
    if (!e) return 0;
    if (batchable(e)) return 1;
    return lockstep_ok(e, 2) && e->lockstep ? 2 : 0;
}

int shs_engine_run_batch(shs_engine* e, uint64_t seed, uint64_t idx0, uint32_t count,
                         uint64_t* j) {
    return shs_engine_run_many(e, seed, idx0, count, j, nullptr, nullptr, nullptr);
}

int shs_engine_run_sequential(shs_engine* e, uint64_t seed, uint64_t idx0, uint32_t count,
                              uint64_t* j) {
    return guarded(e, [&] {
        for (uint32_t i = 0; i < count; ++i) {
            u128 jj = 0;
            int rc = engine_run(e, seed, idx0 + i, &jj, nullptr, nullptr);
            if (rc) return rc;
            j[2 * i] = static_cast<uint64_t>(jj);
            j[2 * i + 1] = static_cast<uint64_t>(jj >> 64);
        }
        return SHS_OK;
    });
}

int shs_state_init(shs_engine* e) {
    return guarded(e, [&] { return e->group ? group_state_init(e->group) : state_init(e); });
}

int shs_stage_probs(shs_engine* e, uint32_t s, uint64_t lo, uint64_t hi, double* p0, double* p1) {
    return guarded(e, [&] {
        if (e->group) {
            if (s >= e->t) return set_error(SHS_INVALID_ARGUMENT, "stage index out of range");
            return group_stage_probs(e->group, s, (u128{hi} << 64) | lo, p0, p1);
        }
        return stage_probs(e, s, (u128{hi} << 64) | lo, p0, p1);
    });
}

int shs_stage_collapse(shs_engine* e, int32_t src_group, double p_source) {
    return guarded(e, [&] {
        if (e->group) return group_stage_collapse(e->group, src_group, p_source);
        return stage_collapse(e, src_group, p_source, true);
    });
}

int shs_stage_read(shs_engine* e, int32_t x, uint64_t first, uint64_t count, double* host) {
    return guarded(e, [&]() -> int {
        if (e->group) return group_stage_read(e->group, x, first, count, host);
        if (!e->pending) return set_error(SHS_INVALID_ARGUMENT, "no pending stage");
        if (count == 0) return SHS_OK;
        double2* d = nullptr;
        SHS_CUDA(cudaMallocAsync(&d, sizeof(double2) * count, e->stream));
        StageParams p = params_for(e, e->ps);
        const bool gather = e->a_pows[e->ps] != 1;
        const int grid = static_cast<int>(std::min<uint64_t>((count + 255) / 256, 4096));
        // a compressed probs pass has already swapped nothing: its input pair is X
        int rc = e->rep_orb ? launch(e, -1, [&] {
            k_orb_stage_read<<<grid, 256, 0, e->stream>>>(p, orb_src(e), e->orb_rec, x, gather ? 1 : 0,
                                                          first, count, d);
        }) : launch(e, -1, [&] {
            if (gather) {
                if (e->e1) k_stage_read<kSrcGather, true><<<grid, 256, 0, e->stream>>>(p, x, first, count, d);
                else k_stage_read<kSrcGather, false><<<grid, 256, 0, e->stream>>>(p, x, first, count, d);
            } else {
                if (e->e1) k_stage_read<kSrcDirect, true><<<grid, 256, 0, e->stream>>>(p, x, first, count, d);
                else k_stage_read<kSrcDirect, false><<<grid, 256, 0, e->stream>>>(p, x, first, count, d);
            }
        });
        if (rc) return rc;
        SHS_CUDA(cudaMemcpyAsync(host, d, sizeof(double2) * count, cudaMemcpyDeviceToHost,
                                 e->stream));
        SHS_CUDA(cudaFreeAsync(d, e->stream));
        return sync(e);
    });
}

int shs_state_read(shs_engine* e, int32_t x, uint64_t first, uint64_t count, double* host) {
    return guarded(e, [&]() -> int {
        if (x != 0 && x != 1) return set_error(SHS_INVALID_ARGUMENT, "group must be 0 or 1");
        if (e->group) return group_state_read(e->group, x, first, count, host);
        if (!e->e1 && !e->X) return set_error(SHS_INVALID_ARGUMENT, "no state");
        if (count == 0) return SHS_OK;
        double2* d = nullptr;
        SHS_CUDA(cudaMallocAsync(&d, sizeof(double2) * count, e->stream));
        const int grid = static_cast<int>(std::min<uint64_t>((count + 255) / 256, 4096));
        const double wr = e->w[2 * x], wi = e->w[2 * x + 1];
        int rc = e->rep_orb ? launch(e, -1, [&] {
            k_orb_state_read<<<grid, 256, 0, e->stream>>>(orb_src(e), e->orb_rec, e->N, wr, wi, e->inv,
                                                          nullptr, first, count, d);
        }) : launch(e, -1, [&] {
            if (e->e1) k_state_read<true><<<grid, 256, 0, e->stream>>>(e->X, 0, e->N, wr, wi, e->inv, first, count, d);
            else k_state_read<false><<<grid, 256, 0, e->stream>>>(e->X, 0, e->N, wr, wi, e->inv, first, count, d);
        });
        if (rc) return rc;
        SHS_CUDA(cudaMemcpyAsync(host, d, sizeof(double2) * count, cudaMemcpyDeviceToHost,
                                 e->stream));
        SHS_CUDA(cudaFreeAsync(d, e->stream));
        return sync(e);
    });
}

int shs_state_gather(shs_engine* e, int32_t x, const uint64_t* idx, uint64_t count,
                     double* host) {
    return guarded(e, [&]() -> int {
        if (x != 0 && x != 1) return set_error(SHS_INVALID_ARGUMENT, "group must be 0 or 1");
        if (!e->e1 && !e->X) return set_error(SHS_INVALID_ARGUMENT, "no state");
        if (count == 0) return SHS_OK;
        if (!idx || !host) return set_error(SHS_INVALID_ARGUMENT, "null argument");
        if (e->group) return group_state_gather(e->group, x, idx, count, host);
        uint64_t* di = nullptr;
        double2* d = nullptr;
        SHS_CUDA(cudaMallocAsync(&di, sizeof(uint64_t) * count, e->stream));
        SHS_CUDA(cudaMallocAsync(&d, sizeof(double2) * count, e->stream));
        SHS_CUDA(cudaMemcpyAsync(di, idx, sizeof(uint64_t) * count, cudaMemcpyHostToDevice,
                                 e->stream));
        const int grid = static_cast<int>(std::min<uint64_t>((count + 255) / 256, 4096));
        const double wr = e->w[2 * x], wi = e->w[2 * x + 1];
        int rc = e->rep_orb ? launch(e, -1, [&] {
            k_orb_state_read<<<grid, 256, 0, e->stream>>>(orb_src(e), e->orb_rec, e->N, wr, wi, e->inv,
                                                          di, 0, count, d);
        }) : launch(e, -1, [&] {
            if (e->e1) k_state_gather<true><<<grid, 256, 0, e->stream>>>(e->X, 0, e->N, wr, wi, e->inv, di, count, d);
            else k_state_gather<false><<<grid, 256, 0, e->stream>>>(e->X, 0, e->N, wr, wi, e->inv, di, count, d);
        });
        if (rc) return rc;
        SHS_CUDA(cudaMemcpyAsync(host, d, sizeof(double2) * count, cudaMemcpyDeviceToHost,
                                 e->stream));
        SHS_CUDA(cudaFreeAsync(d, e->stream));
        SHS_CUDA(cudaFreeAsync(di, e->stream));
        return sync(e);
    });
}

uint64_t shs_num_blocks(const shs_engine* e) { return e ? e->nb : 0; }

int shs_stage_tile_plan(const shs_engine* e, uint32_t s, uint64_t out[6]) {
    if (!e || !out) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    if (s >= e->t) return set_error(SHS_INVALID_ARGUMENT, "stage index out of range");
    const TilePlanHost& pl = e->plans[s];
    out[0] = pl.tiled ? 1 : 0;
    out[1] = pl.H;
    out[2] = pl.u;
    out[3] = pl.v;
    out[4] = pl.du;
    out[5] = pl.dv;
    return SHS_OK;
}

int shs_stage_block_sums(shs_engine* e, double* out) {
    return guarded(e, [&]() -> int {
        if (e->group) return set_error(SHS_INVALID_ARGUMENT, "block sums of a sharded engine live on its shards");
        if (!e->pending) return set_error(SHS_INVALID_ARGUMENT, "no pending stage");
        SHS_CUDA(cudaMemcpyAsync(out, e->S, sizeof(double) * 2 * e->nb, cudaMemcpyDeviceToHost,
                                 e->stream));
        return sync(e);
    });
}

int shs_index_map(shs_engine* e, uint32_t s, uint64_t first, uint64_t count, uint64_t* host) {
    return guarded(e, [&]() -> int {
        if (s >= e->t) return set_error(SHS_INVALID_ARGUMENT, "stage index out of range");
        if (first >= e->N || count > e->N - first)
            return set_error(SHS_INVALID_ARGUMENT, "index range outside [0, N)");
        if (count == 0) return SHS_OK;
        uint64_t* d = nullptr;
        SHS_CUDA(cudaMallocAsync(&d, sizeof(uint64_t) * count, e->stream));
        int rc;
        if (e->a_pows[s] == 1) {  // identity permutation (ExchangePlan::identity)
            const int grid = static_cast<int>(std::min<uint64_t>((count + 255) / 256, 4096));
            rc = launch(e, -1, [&] { k_fill_identity<<<grid, 256, 0, e->stream>>>(first, count, d); });
        } else {
            StageParams p = params_for(e, s);
            const uint64_t c0 = first / kChunk, c1 = (first + count - 1) / kChunk + 1;
            const int grid = static_cast<int>(std::min<uint64_t>(c1 - c0, 4096));
            rc = launch(e, -1, [&] {
                k_index_map<<<grid, kThreads, 0, e->stream>>>(p, c0, c1 - c0, first, count, d);
            });
        }
        if (rc) return rc;
        SHS_CUDA(cudaMemcpyAsync(host, d, sizeof(uint64_t) * count, cudaMemcpyDeviceToHost,
                                 e->stream));
        SHS_CUDA(cudaFreeAsync(d, e->stream));
        return sync(e);
    });
}

int shs_sample_measurement(double p1, uint64_t seed, uint32_t idx, uint32_t stage,
                           const shs_error* error, int32_t out[4]) {
    if (!error || !out) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    Measurement m = sample_measurement(p1, seed, idx, stage, *error);
    out[0] = m.sampled_bit;
    out[1] = m.observed_bit;
    out[2] = m.error_branch ? 1 : 0;
    out[3] = m.classical_flip ? 1 : 0;
    return SHS_OK;
}

int shs_bitflip(uint64_t j[2], uint32_t t, double delta, uint64_t seed, uint32_t idx) {
    if (!j) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    u128 v = bitflip_bitstring((u128{j[1]} << 64) | j[0], t, delta, seed, idx);
    j[0] = static_cast<uint64_t>(v);
    j[1] = static_cast<uint64_t>(v >> 64);
    return SHS_OK;
}

int shs_engine_set_timing(shs_engine* e, int32_t enable) {
    return guarded(e, [&]() -> int {
        int rc = sync(e);
        if (rc) return rc;
        e->timing = enable != 0;
        for (int k = 0; k < 3; ++k) {
            e->kms[k] = 0;
            e->klaunch[k] = 0;
        }
        return SHS_OK;
    });
}

int shs_engine_kernel_times(const shs_engine* e, double ms[3], uint64_t launches[3]) {
    if (!e) return set_error(SHS_INVALID_ARGUMENT, "null engine");
    for (int k = 0; k < 3; ++k) {
        if (ms) ms[k] = e->kms[k];
        if (launches) launches[k] = e->klaunch[k];
    }
    return SHS_OK;
}

void* shs_engine_stream(const shs_engine* e) { return e ? static_cast<void*>(e->stream) : nullptr; }

uint64_t shs_engine_launch_count(const shs_engine* e) {
    return e ? e->launches + (e->group ? group_launches(e->group) : 0) : 0;
}

uint64_t shs_engine_device_bytes(const shs_engine* e) {
    return e ? e->device_bytes + (e->group ? group_device_bytes(e->group) : 0) : 0;
}

int shs_engine_devices(const shs_engine* e, int32_t* out, int32_t max) {
    if (!e) return 0;
    if (!e->group) {
        if (out && max > 0) out[0] = e->dev;
        return 1;
    }
    const int n = static_cast<int>(e->group->shards.size());
    for (int q = 0; q < n && out && q < max; ++q) out[q] = shard_device(e->group->shards[q]);
    return n;
}

}  // extern "C"
