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
#include <fcntl.h>
#include <nvtx3/nvToolsExt.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/shorsim_b200.h"
#include "device_math.cuh"
#include "exchange.cuh"
#include "exchange2.cuh"
#include "sparse.cuh"
#include "sparse_plan.hpp"
#include <cub/cub.cuh>
#include "host_model.hpp"
#include "stage_kernels.cuh"
#include "tile_plan.hpp"
#include "tiled.cuh"
#include "shard_group.hpp"

using namespace shs;

// Shards of one in-process group that share a device (virtual shards): set by
// group_create while it creates them, so each sizes its receive slots for its
// share of the device (1 outside group_create).
static thread_local uint32_t g_coresident = 1;

// Host barrier for one-process-per-GPU sharded runs: a sense-reversing counter
// in a POSIX shared-memory segment (every rank of a run lives on one node: the
// NVLink domain). It orders ENQUEUES, never GPU work: a rank records its event
// for stage s before the barrier, its peers enqueue their waits on that event
// after it (cudaStreamWaitEvent waits on the record enqueued before the call).
struct ShmBarrier {
    struct Seg {
        std::atomic<uint32_t> count;
        std::atomic<uint32_t> gen;
    };
    Seg* seg = nullptr;
    std::string name;
    uint32_t n = 1;
    bool owner = false;
    ~ShmBarrier() {
        if (seg) munmap(seg, sizeof(Seg));
        if (owner) shm_unlink(name.c_str());
    }
    int open(const char* nm, uint32_t parties, bool unlink_at_close) {
        name = nm;
        n = parties;
        owner = unlink_at_close;
        const int fd = shm_open(nm, O_CREAT | O_RDWR, 0600);
        if (fd < 0) return set_error(SHS_INVALID_ARGUMENT, std::string("shm_open ") + nm);
        if (ftruncate(fd, sizeof(Seg)) != 0) {  // zero-filled on first creation
            ::close(fd);
            return set_error(SHS_INVALID_ARGUMENT, std::string("ftruncate ") + nm);
        }
        void* p = mmap(nullptr, sizeof(Seg), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        ::close(fd);
        if (p == MAP_FAILED) return set_error(SHS_INVALID_ARGUMENT, std::string("mmap ") + nm);
        seg = static_cast<Seg*>(p);
        return SHS_OK;
    }
    // every party calls arrive(); returns when all n have arrived
    int arrive() {
        const uint32_t g = seg->gen.load(std::memory_order_acquire);
        if (seg->count.fetch_add(1, std::memory_order_acq_rel) + 1 == n) {
            seg->count.store(0, std::memory_order_relaxed);
            seg->gen.fetch_add(1, std::memory_order_acq_rel);
            return SHS_OK;
        }
        const auto t0 = std::chrono::steady_clock::now();
        for (uint64_t k = 0; seg->gen.load(std::memory_order_acquire) == g; ++k) {
            if (k > 1024) sched_yield();
            if ((k & 0xffff) == 0 &&
                std::chrono::steady_clock::now() - t0 > std::chrono::seconds(600))
                return set_error(SHS_CUDA_ERROR, "sharded run: peer rank did not reach the barrier "
                                                 "within 600 s");
        }
        return SHS_OK;
    }
};

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
    // timeline (shs_shard_set_timeline): start / end events of every launch, on
    // the stream it ran on, resolved against tl0 after the run (no sync per launch)
    struct TLRec {
        int kind;
        cudaEvent_t a, b;
    };
    bool tl_on = false;
    std::vector<TLRec> tl;
    cudaEvent_t tl0 = nullptr;
    double kms[5] = {0, 0, 0, 0, 0};  // probs, exchange v1, collapse, pack, unpack
    uint64_t klaunch[5] = {0, 0, 0, 0, 0};
    uint64_t launches = 0;
    // device-resident runs (shard_run): stage slots and host-mapped records as
    // the single engine's, this shard's exact digits per stage parity (read by
    // every peer's finalize), and the cross-shard ordering events per parity:
    // X = exchange pushes done, D = digits written, C = collapse done (all
    // interprocess-capable), M = measurement record written (host only).
    DevStage* d_slots = nullptr;
    StageRec* h_rec = nullptr;
    StageRec* d_rec = nullptr;
    unsigned long long* d_dig2 = nullptr;  // [2 parities][2 groups][kDigits]
    const unsigned long long* peer_dig[kMaxShards] = {};
    bool peer_dig_ipc[kMaxShards] = {};
    cudaEvent_t evx[2] = {}, evd[2] = {}, evc[2] = {}, evm[2] = {};
    cudaEvent_t pevx[kMaxShards][2] = {}, pevd[kMaxShards][2] = {}, pevc[kMaxShards][2] = {};
    bool peer_ev_ipc[kMaxShards] = {};
    ShmBarrier* barrier = nullptr;
    uint64_t device_bytes = 0;
    // p0/p1 like the reference (sequential Kahan over the global block partials,
    // statevector.cpp:32-40) for small N under AUTO, or always under KAHAN: then
    // Sb holds two stage parities and every finalize gathers the G shards'
    // partials through peer pointers; otherwise the exact digit sum.
    bool kahan = false;
    const double* peer_S[kMaxShards] = {};
    bool peer_S_ipc[kMaxShards] = {};
    double* Scat = nullptr;   // kahan: [2][nb_total] gathered partials
    double* d_p = nullptr;    // kahan step API: p0, p1
    // exchange v2 (exchange2.cuh) in device-resident runs: two receive slots of
    // x2_slot elements (peers write their streams into them), the per-stage
    // stream offsets (data-independent, prepared once per shard set), the
    // region base of every sender in this shard's slot per (stage, round)
    // (exported: senders read them once), pack on its own stream
    bool x2_on = true;                     // SHS_EXCHANGE=1: v1 in runs too
    uint32_t x2_K = 1;                     // rounds per exchange stage
    uint64_t x2_slot = 0;                  // elements per receive slot
    double2* x2_recv = nullptr;            // [2][x2_slot]
    double2* peer_recv[kMaxShards] = {};
    bool peer_recv_ipc[kMaxShards] = {};
    unsigned long long* x2_bases = nullptr;  // [t][x2_K][G]: base of sender q's region, per round
    const unsigned long long* peer_bases[kMaxShards] = {};
    bool peer_bases_ipc[kMaxShards] = {};
    bool x2_ready = false;                 // offsets / bases prepared
    std::vector<uint8_t> x2_stage;         // stage uses v2
    std::vector<unsigned long long*> x2_soff, x2_roff;  // per stage: [G][nbands+1]
    std::vector<uint64_t> x2_dst;          // [t][x2_K][G]: my region base in receiver r's slot
    std::vector<uint64_t> x2_rbase;        // [t][x2_K][G]: sender q's region base in my slot
    std::vector<std::vector<uint64_t>> x2_bounds;  // [t][x2_K + 1]: first band of each round
    uint64_t x2_round = 0;                 // global round counter (event / slot parity)
    cudaStream_t xstream = nullptr;
    cudaEvent_t evp[2] = {}, evu[2] = {};  // pack / unpack of a round done (interprocess)
    cudaEvent_t pevp[kMaxShards][2] = {}, pevu[kMaxShards][2] = {};
    double x2_ms[2] = {0, 0};              // instrumentation: pack, unpack
    // sparse prefix of device-resident runs (sparse.cuh): every shard runs the
    // first stages on the support redundantly (identical results, no peer
    // traffic), its buffers carved out of its P, then scatters the points of
    // its own range into its sel
    uint32_t sparse_n = 0;
    bool sparse_on = true;
    uint64_t* sZ[2] = {nullptr, nullptr};
    double2* sV[2] = {nullptr, nullptr};
    uint64_t* sKeys = nullptr;
    double2* sNrm = nullptr;
    double2* sNrm2 = nullptr;
    void* sTemp = nullptr;
    size_t sTempBytes = 0;
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
int shard_launch(shs_shard* sh, int kind, F&& f, cudaStream_t st = nullptr) {
    static const char* kNames[5] = {"shs shard probs", "shs shard exchange", "shs shard collapse",
                                    "shs shard pack", "shs shard unpack"};
    nvtxRangePushA(kNames[kind]);
    struct Pop {
        ~Pop() { nvtxRangePop(); }
    } pop;
    if (!st) st = sh->stream;
    if (sh->timing) cudaEventRecord(sh->ev[0], st);
    shs_shard::TLRec tr{kind, nullptr, nullptr};
    if (sh->tl_on) {
        cudaEventCreate(&tr.a);
        cudaEventCreate(&tr.b);
        cudaEventRecord(tr.a, st);
    }
    f();
    cudaError_t err = cudaGetLastError();
    if (sh->tl_on) {
        cudaEventRecord(tr.b, st);
        sh->tl.push_back(tr);
    }
    if (sh->timing) {
        cudaEventRecord(sh->ev[1], st);
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
    p.S = sh->Sb;  // (a kahan run selects the stage parity: launch_run_probs)
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
    for (uint32_t q = 0; q < sh->G; ++q) {
        if (sh->peer_dig_ipc[q] && sh->peer_dig[q])
            cudaIpcCloseMemHandle(const_cast<unsigned long long*>(sh->peer_dig[q]));
        if (sh->peer_ev_ipc[q])
            for (int k = 0; k < 2; ++k) {  // opened IPC events are released like events
                if (sh->pevx[q][k]) cudaEventDestroy(sh->pevx[q][k]);
                if (sh->pevd[q][k]) cudaEventDestroy(sh->pevd[q][k]);
                if (sh->pevc[q][k]) cudaEventDestroy(sh->pevc[q][k]);
            }
    }
    for (int k = 0; k < 2; ++k)
        for (cudaEvent_t e : {sh->evx[k], sh->evd[k], sh->evc[k], sh->evm[k]})
            if (e) cudaEventDestroy(e);
    cudaFree(sh->d_slots);
    if (sh->h_rec) cudaFreeHost(sh->h_rec);
    cudaFree(sh->d_dig2);
    cudaFree(sh->Scat);
    cudaFree(sh->d_p);
    for (auto* x : sh->x2_soff) cudaFree(x);
    for (auto* x : sh->x2_roff) cudaFree(x);
    cudaFree(sh->x2_recv);
    cudaFree(sh->x2_bases);
    for (uint32_t q = 0; q < sh->G; ++q) {
        if (sh->peer_recv_ipc[q] && sh->peer_recv[q]) cudaIpcCloseMemHandle(sh->peer_recv[q]);
        if (sh->peer_bases_ipc[q] && sh->peer_bases[q])
            cudaIpcCloseMemHandle(const_cast<unsigned long long*>(sh->peer_bases[q]));
        if (sh->peer_ev_ipc[q])
            for (int k = 0; k < 2; ++k) {
                if (sh->pevp[q][k]) cudaEventDestroy(sh->pevp[q][k]);
                if (sh->pevu[q][k]) cudaEventDestroy(sh->pevu[q][k]);
            }
    }
    for (int k = 0; k < 2; ++k)
        for (cudaEvent_t e : {sh->evp[k], sh->evu[k]})
            if (e) cudaEventDestroy(e);
    if (sh->xstream) cudaStreamDestroy(sh->xstream);
    for (auto& r : sh->tl) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    if (sh->tl0) cudaEventDestroy(sh->tl0);
    for (uint32_t q = 0; q < sh->G; ++q)
        if (sh->peer_S_ipc[q] && sh->peer_S[q])
            cudaIpcCloseMemHandle(const_cast<double*>(sh->peer_S[q]));
    delete sh->barrier;
    if (sh->stream) cudaStreamDestroy(sh->stream);
    delete sh;
}

bool stage_needs_exchange(const shs_shard* sh, uint32_t s) {
    return !sh->e1 && sh->a_pows[s] != 1;
}


// The exchange of stage s (exchange.cuh): this rank's round-robin share of the
// tiles, or the owner-addressed direct pull for stages without a tile plan.
int launch_exchange(shs_shard* sh, uint32_t s) {
    const ShardMap map = shard_map(sh);
    const TilePlanHost& pl = sh->plans[s];
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
        return shard_launch(sh, 1, [&] {
            k_exchange<<<g, kExchangeThreads, exchange_smem_bytes(), sh->stream>>>(tp, map, sh->rank,
                                                                                  sh->G);
        });
    }
    StageParams p = local_params(sh, s, false);
    return shard_launch(sh, 1, [&] {
        k_exchange_direct<<<grid(sh), kThreads, 0, sh->stream>>>(p, map, sh->buf[sh->parity ^ 1]);
    });
}


// ---- exchange v2 (exchange2.cuh)

TileParams plan_tile_params(const shs_shard* sh, uint32_t s) {
    const TilePlanHost& pl = sh->plans[s];
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
    return tp;
}

X2Params x2_params(const shs_shard* sh, uint32_t s) {
    X2Params p{};
    p.tp = plan_tile_params(sh, s);
    p.S = sh->S;
    p.S_inv = ~uint64_t(0) / sh->S;
    p.N = sh->N;
    p.G = static_cast<int>(sh->G);
    p.me = static_cast<int>(sh->rank);
    p.sel = sh->buf[sh->parity];
    p.P = sh->buf[sh->parity ^ 1];
    for (uint64_t c = 0; c <= 32; ++c) p.mstep[c] = mulmod(p.tp.m, c, sh->N);
    return p;
}

// a stage runs exchange v2 when it has a tile plan whose rows fit a shard
bool x2_eligible(const shs_shard* sh, uint32_t s) {
    const TilePlanHost& pl = sh->plans[s];
    return sh->x2_on && sh->x2_recv && s > 0 && sh->a_pows[s] != 1 && pl.tiled &&
           pl.du + pl.dv <= sh->S;
}

// Round boundaries of stage s: bands cut where the cumulative element count
// (row lengths du, dv, du + dv by the three-distance classes) crosses k N / K,
// so every round moves about N / K elements (a band-count split does not: the
// length classes are contiguous in j).
std::vector<uint64_t> x2_round_bounds(const TilePlanHost& pl, uint64_t N, uint32_t K) {
    std::vector<uint64_t> b(K + 1, pl.ntiles);
    b[0] = 0;
    auto len = [&](uint64_t j) -> uint64_t {
        if (j >= pl.H) return 0;
        if (j + pl.u < pl.H) return pl.du;
        if (j >= pl.v) return pl.dv;
        return pl.du + pl.dv;
    };
    uint64_t cum = 0;
    uint32_t k = 1;
    for (uint64_t band = 0; band < pl.ntiles && k < K; ++band) {
        while (k < K && cum >= (static_cast<unsigned __int128>(N) * k) / K) b[k++] = band;
        for (uint64_t j = band * kRows; j < (band + 1) * kRows; ++j) cum += len(j);
    }
    return b;
}

uint64_t x2_band(const shs_shard* sh, uint32_t s, uint32_t k) { return sh->x2_bounds[s][k]; }

int x2_grid(const shs_shard* sh, uint64_t bands) {  // one band per warp
    const uint64_t ctas = (bands + kX2Warps - 1) / kX2Warps;
    return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(ctas, 12ull * sh->num_sms)));
}

// round k of stage s, global round g: this shard's pack (its pack stream)
int launch_x2_pack(shs_shard* sh, uint32_t s, uint32_t k, uint64_t g) {
    const TilePlanHost& pl = sh->plans[s];
    X2Params p = x2_params(sh, s);
    p.b0 = x2_band(sh, s, k);
    p.b1 = x2_band(sh, s, k + 1);
    p.off = sh->x2_soff[s];
    for (uint32_t r = 0; r < sh->G; ++r)
        p.dst[r] = sh->peer_recv[r] + (g & 1) * sh->x2_slot +
                   sh->x2_dst[(uint64_t(s) * sh->x2_K + k) * sh->G + r];
    if (p.b0 == p.b1) return SHS_OK;
    return shard_launch(sh, 3, [&] {
        k_x2_pack<<<x2_grid(sh, p.b1 - p.b0), kX2Threads, 0, sh->xstream>>>(p);
    }, sh->xstream);
}

// ... and its unpack (main stream), into P
int launch_x2_unpack(shs_shard* sh, uint32_t s, uint32_t k, uint64_t g) {
    const std::vector<uint64_t>& rbase = sh->x2_rbase;
    const TilePlanHost& pl = sh->plans[s];
    X2Params p = x2_params(sh, s);
    p.b0 = x2_band(sh, s, k);
    p.b1 = x2_band(sh, s, k + 1);
    p.off = sh->x2_roff[s];
    for (uint32_t q = 0; q < sh->G; ++q)
        p.src[q] = sh->x2_recv + (g & 1) * sh->x2_slot +
                   rbase[(uint64_t(s) * sh->x2_K + k) * sh->G + q];
    if (p.b0 == p.b1) return SHS_OK;
    return shard_launch(sh, 4, [&] {
        k_x2_unpack<<<x2_grid(sh, p.b1 - p.b0), kX2Threads, 0, sh->stream>>>(p);
    });
}


// ---- sparse prefix (sparse.cuh) on a shard

int shard_sparse_grid(const shs_shard* sh, uint64_t n) {
    return static_cast<int>(std::max<uint64_t>(
        1, std::min<uint64_t>((n + kSparseThreads - 1) / kSparseThreads, sh->grid_cap)));
}

// the support buffers in this shard's P (free until the first dense stage)
int shard_carve_sparse(shs_shard* sh) {
    const uint64_t K = uint64_t(1) << sh->sparse_n;
    char* p = reinterpret_cast<char*>(sh->buf[sh->parity ^ 1]);
    char* const base = p;
    auto take = [&](size_t bytes) {
        char* q = p;
        p += (bytes + 255) & ~size_t(255);
        return q;
    };
    sh->sZ[0] = reinterpret_cast<uint64_t*>(take(8 * K));
    sh->sZ[1] = reinterpret_cast<uint64_t*>(take(8 * K));
    sh->sV[0] = reinterpret_cast<double2*>(take(16 * K));
    sh->sV[1] = reinterpret_cast<double2*>(take(16 * K));
    sh->sKeys = reinterpret_cast<uint64_t*>(take(8 * K));
    sh->sNrm = reinterpret_cast<double2*>(take(16 * K));
    sh->sNrm2 = reinterpret_cast<double2*>(take(16 * K));
    if (!sh->sTempBytes) {
        cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, sh->sTempBytes, sh->sZ[0],
                                                        sh->sKeys, sh->sNrm, sh->sNrm2,
                                                        static_cast<int>(K), 0, 64, sh->stream);
        if (e != cudaSuccess) return set_error(SHS_CUDA_ERROR, cudaGetErrorString(e));
    }
    sh->sTemp = take(sh->sTempBytes);
    if (static_cast<size_t>(p - base) > sizeof(double2) * sh->nloc)
        return set_error(SHS_CUDA_ERROR, "sparse prefix buffers exceed the shard's P");
    return SHS_OK;
}

SparseParams shard_sparse_params(const shs_shard* sh, uint32_t s, const DevStage* dev) {
    SparseParams p{};
    p.Zo = sh->sZ[s & 1];
    p.Vo = sh->sV[s & 1];
    p.Ko = uint64_t(1) << s;
    p.A = sh->a_pows[s];
    p.A_sh = shoup(p.A, sh->N);
    p.N = sh->N;
    p.sc = sh->sc;
    p.dev = dev;
    p.Zn = sh->sZ[(s + 1) & 1];
    p.Vn = sh->sV[(s + 1) & 1];
    p.nrm = sh->sNrm;
    return p;
}

// probs of sparse stage s: expand, sort by z, in-order block folds (exact digits)
int launch_shard_sparse_probs(shs_shard* sh, uint32_t s, const DevStage* dev, int* nparts) {
    SparseParams p = shard_sparse_params(sh, s, dev);
    const uint64_t Kn = 2 * p.Ko;
    int end_bit = 1;
    while (end_bit < 64 && (sh->N - 1) >> end_bit) ++end_bit;
    const int gf = shard_sparse_grid(sh, Kn);
    cudaError_t sort_err = cudaSuccess;
    int rc = shard_launch(sh, 0, [&] {
        if (s == 0) k_sparse_init<<<1, 1, 0, sh->stream>>>(sh->sZ[0], sh->sV[0]);
        k_sparse_expand<<<shard_sparse_grid(sh, p.Ko), kSparseThreads, 0, sh->stream>>>(p);
        size_t bytes = sh->sTempBytes;
        sort_err = cub::DeviceRadixSort::SortPairs(sh->sTemp, bytes, p.Zn, sh->sKeys, sh->sNrm,
                                                   sh->sNrm2, static_cast<int>(Kn), 0, end_bit,
                                                   sh->stream);
        k_sparse_fold<<<gf, kSparseThreads, 0, sh->stream>>>(sh->sKeys, sh->sNrm2, Kn, sh->partials);
    });
    if (rc) return rc;
    if (sort_err != cudaSuccess)
        return set_error(SHS_CUDA_ERROR, std::string("sparse sort: ") + cudaGetErrorString(sort_err));
    *nparts = gf;
    return SHS_OK;
}

int launch_shard_sparse_collapse(shs_shard* sh, uint32_t s, const DevStage* dev) {
    SparseParams p = shard_sparse_params(sh, s, dev);
    return shard_launch(sh, 2, [&] {
        k_sparse_collapse<<<shard_sparse_grid(sh, p.Ko), kSparseThreads, 0, sh->stream>>>(p, 0);
    });
}

// the shard's dense sel from the support entering stage s (its own range only)
int shard_materialize_sparse(shs_shard* sh, uint32_t s) {
    const uint64_t K = uint64_t(1) << s;
    double2* X = sh->buf[sh->parity];
    SHD_CUDA(cudaMemsetAsync(X, 0, sizeof(double2) * sh->nloc, sh->stream));
    int rc = shard_launch(sh, 0, [&] {  // (timed with the probs passes)
        k_sparse_scatter_range<<<shard_sparse_grid(sh, K), kSparseThreads, 0, sh->stream>>>(
            sh->sZ[s & 1], sh->sV[s & 1], K, sh->lo, sh->hi, X);
    });
    sh->e1 = false;
    return rc;
}

// Host scalars of stage s for the observed prefix (statevector.cpp:338-349).
StageScalars shard_scalars(const shs_shard* sh, uint32_t s, u128 prefix, double inv) {
    const double phi = stage_phase(s, prefix);
    StageScalars sc{};
    sc.w0r = sh->w[0];
    sc.w0i = sh->w[1];
    sc.w1r = sh->w[2];
    sc.w1i = sh->w[3];
    sc.phr = 1.0 * std::cos(phi);  // std::polar(1.0, phi), statevector.cpp:338
    sc.phi = 1.0 * std::sin(phi);
    sc.inv = inv;
    sc.phase_mul = (sh->a_pows[s] != 1 || phi != 0.0) ? 1 : 0;
    return sc;
}

// probs(s) of a device-resident run: scalars from slot `dev` (stage 0: the
// host's, run start e_1), then this shard's exact digits into parity s & 1.
int launch_run_probs(shs_shard* sh, uint32_t s, const DevStage* dev) {
    const bool ex = stage_needs_exchange(sh, s);
    const bool gather = sh->a_pows[s] != 1;
    StageParams p = local_params(sh, s, ex);
    p.dev = dev;
    if (sh->kahan) p.S = sh->Sb + (s & 1) * 2 * sh->nb;  // peers read it in their finalize
    const int g = grid(sh);
    unsigned long long* out = sh->d_dig2 + (s & 1) * 2 * kDigits;
    return shard_launch(sh, 0, [&] {
        if (sh->e1) {
            if (gather) k_stage_probs<kSrcGather, true, false><<<g, kThreads, 0, sh->stream>>>(p);
            else k_stage_probs<kSrcDirect, true, false><<<g, kThreads, 0, sh->stream>>>(p);
        } else if (ex) {
            k_stage_probs<kSrcBuffer, false, true><<<g, kThreads, 0, sh->stream>>>(p);
        } else {
            k_stage_probs<kSrcDirect, false, true><<<g, kThreads, 0, sh->stream>>>(p);
        }
        k_sum_partials<<<1, kFinalizeThreads, 0, sh->stream>>>(sh->partials, g, out);
    });
}

// collapse(s) of a device-resident run: group and scalars from slot `dev`
int launch_run_collapse(shs_shard* sh, uint32_t s, const DevStage* dev) {
    const bool ex = stage_needs_exchange(sh, s);
    const bool gather = sh->a_pows[s] != 1;
    StageParams p = local_params(sh, s, ex);
    p.dev = dev;
    const int g = grid(sh);
    int rc = shard_launch(sh, 2, [&] {
        if (sh->e1) {
            if (gather) k_stage_collapse<kSrcGather, true, true><<<g, kThreads, 0, sh->stream>>>(p);
            else k_stage_collapse<kSrcDirect, true, true><<<g, kThreads, 0, sh->stream>>>(p);
        } else if (ex) {  // in place over P
            k_stage_collapse<kSrcBuffer, false, true><<<g, kThreads, 0, sh->stream>>>(p);
        } else {
            k_stage_collapse<kSrcDirect, false, true><<<g, kThreads, 0, sh->stream>>>(p);
        }
    });
    if (rc) return rc;
    sh->parity ^= 1;
    sh->e1 = false;
    return SHS_OK;
}

// the G shards' block partials of stage parity k (kahan combine)
ShardPartials shard_partials(const shs_shard* sh, int k) {
    ShardPartials sp{};
    sp.G = static_cast<int>(sh->G);
    uint64_t off = 0;
    for (uint32_t q = 0; q < sh->G; ++q) {
        const uint64_t lo = uint64_t(q) * sh->S, hi = std::min(sh->N, lo + sh->S);
        const uint64_t nbq = (hi - lo + kBlock - 1) / kBlock;
        sp.off[q] = off;
        sp.S[q] = sh->peer_S[q] + k * 2 * nbq;
        off += nbq;
    }
    sp.off[sh->G] = off;
    return sp;
}

#define RUN_CUDA(call)                                                                     \
    do {                                                                                   \
        cudaError_t _e = (call);                                                           \
        if (_e != cudaSuccess)                                                             \
            return set_error(SHS_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

}  // namespace


// Offsets of exchange v2 for every eligible stage (collective over the shard
// set; once): per stage, count(b, me, r) and count(b, q, me) per band on the
// device, their exclusive scans over bands, the region base of every sender in
// this shard's receive slot per round (x2_bases, exported), then every
// sender's own base in each receiver's slot read back from the peers.
int x2_prepare(const std::vector<shs_shard*>& L, ShmBarrier* bar) {
    const uint32_t t = L[0]->t, G = L[0]->G, K = L[0]->x2_K;
    for (size_t li = 0; li < L.size(); ++li) {
        shs_shard* q = L[li];
        q->x2_rbase.assign(size_t(t) * K * G + t, 0);
        RUN_CUDA(cudaSetDevice(q->dev));
        q->x2_stage.assign(t, 0);
        q->x2_bounds.assign(t, {});
        q->x2_soff.assign(t, nullptr);
        q->x2_roff.assign(t, nullptr);
        std::vector<uint64_t>& hb = q->x2_rbase;
        unsigned long long* cnt = nullptr;
        uint64_t cnt_cap = 0;
        void* tmp = nullptr;
        size_t tmp_bytes = 0;
        for (uint32_t s = 0; s < t; ++s) {
            if (!x2_eligible(q, s)) continue;
            const TilePlanHost& pl = q->plans[s];
            const uint64_t nb1 = pl.ntiles + 1;
            q->x2_bounds[s] = x2_round_bounds(pl, q->N, K);
            RUN_CUDA(cudaMalloc(&q->x2_soff[s], sizeof(unsigned long long) * G * nb1));
            RUN_CUDA(cudaMalloc(&q->x2_roff[s], sizeof(unsigned long long) * G * nb1));
            if (nb1 > cnt_cap) {
                cudaFree(cnt);
                RUN_CUDA(cudaMalloc(&cnt, sizeof(unsigned long long) * G * nb1 * 2));
                cnt_cap = nb1;
            }
            X2Params p = x2_params(q, s);
            RUN_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * G * nb1 * 2, q->stream));
            const int grid = x2_grid(q, pl.ntiles);
            k_x2_count<true><<<grid, kX2Threads, 0, q->stream>>>(p, cnt);
            k_x2_count<false><<<grid, kX2Threads, 0, q->stream>>>(p, cnt + G * nb1);
            RUN_CUDA(cudaGetLastError());
            size_t need = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, need, cnt, q->x2_soff[s], static_cast<int>(nb1),
                                          q->stream);
            if (need > tmp_bytes) {
                cudaFree(tmp);
                RUN_CUDA(cudaMalloc(&tmp, need));
                tmp_bytes = need;
            }
            for (uint32_t g = 0; g < G; ++g) {
                size_t tb = tmp_bytes;
                cub::DeviceScan::ExclusiveSum(tmp, tb, cnt + g * nb1, q->x2_soff[s] + g * nb1,
                                              static_cast<int>(nb1), q->stream);
                tb = tmp_bytes;
                cub::DeviceScan::ExclusiveSum(tmp, tb, cnt + G * nb1 + g * nb1,
                                              q->x2_roff[s] + g * nb1, static_cast<int>(nb1),
                                              q->stream);
            }
            // receive offsets at the round boundaries -> this shard's region bases
            std::vector<unsigned long long> at(size_t(G) * (K + 1));
            for (uint32_t g = 0; g < G; ++g)
                for (uint32_t k = 0; k <= K; ++k)
                    RUN_CUDA(cudaMemcpyAsync(&at[g * (K + 1) + k],
                                             q->x2_roff[s] + g * nb1 + q->x2_bounds[s][k],
                                             sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                             q->stream));
            RUN_CUDA(cudaStreamSynchronize(q->stream));
            bool fits = true;
            for (uint32_t k = 0; k < K; ++k) {
                uint64_t base = 0;
                for (uint32_t g = 0; g < G; ++g) {
                    hb[(uint64_t(s) * K + k) * G + g] = base;
                    base += at[g * (K + 1) + k + 1] - at[g * (K + 1) + k];
                }
                fits = fits && base <= q->x2_slot;
            }
            // a stage whose rounds overflow some rank's slot (few, lumpy rows at
            // small N) runs exchange v1: decided with every rank's flag below
            hb[uint64_t(t) * K * G + s] = fits ? 1 : 0;
            q->x2_stage[s] = 1;
        }
        RUN_CUDA(cudaMemcpyAsync(q->x2_bases, hb.data(), sizeof(uint64_t) * hb.size(),
                                 cudaMemcpyHostToDevice, q->stream));
        RUN_CUDA(cudaStreamSynchronize(q->stream));
        cudaFree(cnt);
        cudaFree(tmp);
    }
    if (bar) {
        int rc = bar->arrive();
        if (rc) return rc;
    }
    std::vector<uint64_t> pb(size_t(t) * K * G + t);
    for (shs_shard* q : L) {
        RUN_CUDA(cudaSetDevice(q->dev));
        q->x2_dst.assign(size_t(t) * K * G, 0);
        for (uint32_t r = 0; r < G; ++r) {
            RUN_CUDA(cudaMemcpy(pb.data(), q->peer_bases[r], sizeof(uint64_t) * pb.size(),
                                cudaMemcpyDefault));
            for (uint64_t sk = 0; sk < uint64_t(t) * K; ++sk)
                q->x2_dst[sk * G + r] = pb[sk * G + q->rank];
            for (uint32_t s = 0; s < t; ++s)  // the same decision on every rank
                if (!pb[uint64_t(t) * K * G + s]) q->x2_stage[s] = 0;
        }
        q->x2_ready = true;
    }
    if (bar) return bar->arrive();  // nobody packs before every peer read the bases
    return SHS_OK;
}

// ---------------------------------------------------------------------------
// Device-resident sharded run (IterativeShorEngine::run, statevector.cpp:323-412,
// over G block shards). `L` = the shards THIS host thread drives: all G of them
// (one process drives several devices, or virtual shards on one device), or
// one (one process per GPU, `bar` = the node-local host barrier). Per stage s
// every shard q enqueues, with no host wait on the GPU:
//   [exchange stages] wait C_r[s-1] of every peer r (its collapse wrote the sel
//       q pulls from, and freed the P q pushes into); k_exchange; record X_q[s]
//   [barrier]  wait X_r[s] (every push into q's P landed)
//   probs(s) -> k_sum_partials -> digits_q[s & 1]; record D_q[s]
//   [barrier]  (host) read stage s-1's record: the observed prefix, from which
//       both candidate phases of stage s+1 are computed with glibc
//   wait D_r[s]; k_shard_finalize_measure: p0/p1 from the G digit arrays (exact,
//       so identical on every shard), the measurement, the next scalars;
//       record M_q[s]; collapse(s); record C_q[s]
//   [barrier]
// Barriers order enqueues only (a wait must be enqueued after the record it
// waits on); events carry two parities, so a record for stage s+2 can never
// overtake a peer's wait for stage s (the peer passed stage s+1's barriers).
// Results equal the single engine with SHS_COMBINE_EXACT for every G.
int shards_run(const std::vector<shs_shard*>& L, ShmBarrier* bar, u64 seed, u64 idx, u128* j_out,
               u128* js_out, shs_stage_trace* trace) {
    nvtxRangePushA("shs sharded run (device-resident)");
    struct Pop {
        ~Pop() { nvtxRangePop(); }
    } pop;
    shs_shard* s0 = L.front();
    const uint32_t t = s0->t, G = s0->G;
    for (shs_shard* q : L) {
        if (q->tl_on) {  // time zero of this run's timeline
            RUN_CUDA(cudaSetDevice(q->dev));
            if (!q->tl0) RUN_CUDA(cudaEventCreate(&q->tl0));
            for (auto& r : q->tl) {
                cudaEventDestroy(r.a);
                cudaEventDestroy(r.b);
            }
            q->tl.clear();
            RUN_CUDA(cudaEventRecord(q->tl0, q->stream));
        }
        for (uint32_t r = 0; r < G; ++r)
            if (!q->peer[r][0] || !q->peer_dig[r] || !q->pevd[r][0])
                return set_error(SHS_INVALID_ARGUMENT, "sharded run: shard " + std::to_string(r) +
                                                           " not attached to " + std::to_string(q->rank));
        RUN_CUDA(cudaSetDevice(q->dev));
        shs_shard_init(q);
        std::memset(q->h_rec, 0, sizeof(StageRec) * t);
    }
    auto barrier = [&]() -> int { return bar ? bar->arrive() : SHS_OK; };
    auto wait_peers = [&](shs_shard* q, cudaEvent_t (*ev)[2], int k) -> int {
        for (uint32_t r = 0; r < G; ++r)
            if (r != q->rank) RUN_CUDA(cudaStreamWaitEvent(q->stream, ev[r][k], 0));
        return SHS_OK;
    };
    MeasureCfg mc{seed, static_cast<u32>(idx), s0->err.kind, s0->err.delta, s0->err.px,
                  s0->err.py, s0->opt.check_norms};
    u128 observed = 0, sampled = 0;
    double inv = 1.0;
    StageScalars sc = shard_scalars(s0, 0, 0, 1.0);
    int status = SHS_OK;
    if (G > 1 && s0->x2_on && s0->x2_recv && !s0->x2_ready) {
        for (shs_shard* q : L)
            for (uint32_t r = 0; r < G; ++r)
                if (!q->peer_recv[r] || !q->peer_bases[r] || !q->pevp[r][0])
                    return set_error(SHS_INVALID_ARGUMENT, "sharded run: exchange buffers of shard " +
                                                               std::to_string(r) + " not attached");
        if ((status = x2_prepare(L, bar))) return status;
    }
    auto absorb = [&](uint32_t r) -> int {
        RUN_CUDA(cudaSetDevice(s0->dev));
        RUN_CUDA(cudaEventSynchronize(s0->evm[r & 1]));
        StageRec rec;
        std::memcpy(&rec, s0->h_rec + r, sizeof(rec));
        if (!rec.done) return set_error(SHS_CUDA_ERROR, "stage record missing");
        if (trace) {
            trace[r].cbit = r;
            trace[r].p1 = rec.p1;
            trace[r].sampled_bit = rec.sbit;
            trace[r].observed_bit = rec.obit;
            trace[r].classical_flip = static_cast<uint8_t>(rec.flip);
            trace[r].quantum_error_branch = static_cast<uint8_t>(rec.ebranch);
        }
        if (rec.status == SHS_ERROR)
            return set_error(SHS_ERROR, "statevector norm drifted beyond 1e-9 at stage " +
                                            std::to_string(r));
        if (rec.status == SHS_DEGENERATE_BRANCH)
            return set_error(SHS_DEGENERATE_BRANCH,
                             "impossible measurement branch at stage " + std::to_string(r));
        observed |= u128{static_cast<unsigned>(rec.obit)} << r;
        sampled |= u128{static_cast<unsigned>(rec.sbit)} << r;
        if (r + 1 < t) {
            const int src_group = rec.ebranch ? 1 - rec.sbit : rec.sbit;
            inv = 1.0 / std::sqrt(src_group == 1 ? rec.p1 : rec.p0);  // statevector.cpp:391
            sc = shard_scalars(s0, r + 1, observed, inv);
        }
        return SHS_OK;
    };
    auto drain = [&](int code) {
        for (shs_shard* q : L) {
            cudaSetDevice(q->dev);
            cudaStreamSynchronize(q->stream);  // queued stages fold zeros (inv = 0)
            q->pending = false;
        }
        return code;
    };
    // sparse prefix: every shard runs stages 0 .. nsp-1 on the support on its own
    // device (identical results, no peer traffic), then scatters its range
    const uint32_t nsp = s0->sparse_on ? s0->sparse_n : 0;
    if (nsp)
        for (shs_shard* q : L) {
            RUN_CUDA(cudaSetDevice(q->dev));
            if ((status = shard_carve_sparse(q))) return status;
        }
    for (uint32_t s = 0; s < nsp; ++s) {
        const int k = s & 1;
        int nparts = 0;
        for (shs_shard* q : L) {
            RUN_CUDA(cudaSetDevice(q->dev));
            q->sc = sc;
            q->ps = s;
            if ((status = launch_shard_sparse_probs(q, s, s == 0 ? nullptr : q->d_slots + k,
                                                    &nparts)))
                return drain(status);
        }
        if (s > 0 && (status = absorb(s - 1))) return drain(status);
        MeasureStep ms{};
        ms.cfg = mc;
        ms.s = s;
        ms.collapse = s + 1 < t ? 1 : 0;
        ms.init_cur = s == 0 ? 1 : 0;
        ms.sc0 = sc;
        for (int bit = 0; bit < 2; ++bit) {
            const StageScalars c =
                shard_scalars(s0, s + 1, observed | (u128{static_cast<unsigned>(bit)} << s), 0.0);
            ms.nph.phr[bit] = c.phr;
            ms.nph.phi[bit] = c.phi;
            ms.nph.phase_mul[bit] = c.phase_mul;
        }
        for (shs_shard* q : L) {
            RUN_CUDA(cudaSetDevice(q->dev));
            ms.cur = q->d_slots + k;
            ms.next = q->d_slots + (k ^ 1);
            ms.rec = q->d_rec;
            k_finalize_measure<<<1, kFinalizeThreads, 0, q->stream>>>(q->partials, nparts, nullptr,
                                                                    0, 0, ms);
            q->launches++;
            RUN_CUDA(cudaGetLastError());
            RUN_CUDA(cudaEventRecord(q->evm[k], q->stream));
            if ((status = launch_shard_sparse_collapse(q, s, q->d_slots + k))) return drain(status);
        }
    }
    if (nsp) {  // the dense state entering stage nsp, each shard its own range
        for (shs_shard* q : L) {
            RUN_CUDA(cudaSetDevice(q->dev));
            if ((status = shard_materialize_sparse(q, nsp))) return drain(status);
            RUN_CUDA(cudaEventRecord(q->evc[(nsp - 1) & 1], q->stream));
        }
        if ((status = barrier())) return drain(status);
    }
    for (uint32_t s = nsp; s < t; ++s) {
        const int k = s & 1;
        const bool ex = stage_needs_exchange(s0, s);
        if (ex && s0->x2_ready && s0->x2_stage[s]) {
            // exchange v2: K rounds of pack (pack streams) -> unpack (main streams);
            // pack of round g+1 overlaps unpack of round g
            for (uint32_t kr = 0; kr < s0->x2_K; ++kr) {
                const uint64_t g = s0->x2_round;
                for (shs_shard* q : L) {
                    RUN_CUDA(cudaSetDevice(q->dev));
                    if (kr == 0)  // own sel written by the previous collapse
                        RUN_CUDA(cudaStreamWaitEvent(q->xstream, q->evc[(s - 1) & 1], 0));
                    if (g >= 2)  // every receiver unpacked round g-2 out of slot g & 1
                        for (uint32_t r = 0; r < G; ++r)
                            RUN_CUDA(cudaStreamWaitEvent(q->xstream, q->pevu[r][g & 1], 0));
                    if ((status = launch_x2_pack(q, s, kr, g))) return drain(status);
                    RUN_CUDA(cudaEventRecord(q->evp[g & 1], q->xstream));
                }
                if ((status = barrier())) return drain(status);
                for (shs_shard* q : L) {
                    RUN_CUDA(cudaSetDevice(q->dev));
                    for (uint32_t r = 0; r < G; ++r)  // every sender's round g landed
                        RUN_CUDA(cudaStreamWaitEvent(q->stream, q->pevp[r][g & 1], 0));
                    if ((status = launch_x2_unpack(q, s, kr, g))) return drain(status);
                    RUN_CUDA(cudaEventRecord(q->evu[g & 1], q->stream));
                }
                if ((status = barrier())) return drain(status);
                for (shs_shard* q : L) q->x2_round++;
            }
        } else if (ex) {
            for (shs_shard* q : L) {
                RUN_CUDA(cudaSetDevice(q->dev));
                if (s > 0 && (status = wait_peers(q, q->pevc, (s - 1) & 1))) return drain(status);
                if ((status = launch_exchange(q, s))) return drain(status);
                RUN_CUDA(cudaEventRecord(q->evx[k], q->stream));
            }
            if ((status = barrier())) return drain(status);
            for (shs_shard* q : L) {
                RUN_CUDA(cudaSetDevice(q->dev));
                if ((status = wait_peers(q, q->pevx, k))) return drain(status);
            }
        }
        for (shs_shard* q : L) {
            RUN_CUDA(cudaSetDevice(q->dev));
            q->sc = sc;  // stage 0's kernel arguments (later stages read the slot)
            q->ps = s;
            if ((status = launch_run_probs(q, s, s == 0 ? nullptr : q->d_slots + k)))
                return drain(status);
            RUN_CUDA(cudaEventRecord(q->evd[k], q->stream));
        }
        if ((status = barrier())) return drain(status);
        if (s > 0 && (status = absorb(s - 1))) return drain(status);
        MeasureStep ms{};
        ms.cfg = mc;
        ms.s = s;
        ms.collapse = s + 1 < t ? 1 : 0;
        ms.init_cur = s == 0 ? 1 : 0;
        ms.sc0 = sc;
        if (s + 1 < t)
            for (int bit = 0; bit < 2; ++bit) {
                const StageScalars c =
                    shard_scalars(s0, s + 1, observed | (u128{static_cast<unsigned>(bit)} << s), 0.0);
                ms.nph.phr[bit] = c.phr;
                ms.nph.phi[bit] = c.phi;
                ms.nph.phase_mul[bit] = c.phase_mul;
            }
        for (shs_shard* q : L) {
            RUN_CUDA(cudaSetDevice(q->dev));
            if ((status = wait_peers(q, q->pevd, k))) return drain(status);
            ms.cur = q->d_slots + k;
            ms.next = q->d_slots + (k ^ 1);
            ms.rec = q->d_rec;
            if (q->kahan) {  // the reference's sequential Kahan over all G shards' partials
                const ShardPartials sp = shard_partials(q, k);
                const uint64_t nbt = sp.off[G];
                const int gg = static_cast<int>(std::min<uint64_t>((2 * nbt + 255) / 256, 1024));
                k_shard_gather_partials<<<gg, 256, 0, q->stream>>>(sp, q->Scat);
                k_finalize_measure<<<1, kFinalizeThreads, 0, q->stream>>>(nullptr, 0, q->Scat, nbt, 1, ms);
                q->launches += 2;
            } else {
                ShardDigits sd{};
                sd.G = static_cast<int>(G);
                for (uint32_t r = 0; r < G; ++r) sd.d[r] = q->peer_dig[r] + k * 2 * kDigits;
                k_shard_finalize_measure<<<1, 2 * kDigits, 0, q->stream>>>(sd, ms);
                q->launches++;
            }
            RUN_CUDA(cudaGetLastError());
            RUN_CUDA(cudaEventRecord(q->evm[k], q->stream));
            if (s + 1 < t) {
                if ((status = launch_run_collapse(q, s, q->d_slots + k))) return drain(status);
                RUN_CUDA(cudaEventRecord(q->evc[k], q->stream));
            }
        }
        if ((status = barrier())) return drain(status);
    }
    if ((status = absorb(t - 1))) return drain(status);
    for (shs_shard* q : L) {
        RUN_CUDA(cudaSetDevice(q->dev));
        RUN_CUDA(cudaStreamSynchronize(q->stream));
        // shard state as the host-driven loop leaves it: stage t-1 pending
        q->ps = t - 1;
        q->inv = inv;
        q->sc = sc;
        q->pending = true;
        q->exchanged = stage_needs_exchange(q, t - 1) ? static_cast<int>(t - 1) : -1;
    }
    // the collapses advanced parity / e1; the pending stage t-1 read its sel from
    // the parity before the last (absent) collapse, i.e. the current one
    u128 j = observed;
    if (s0->err.kind == SHS_ERR_BITFLIP)
        j = bitflip_bitstring(j, t, s0->err.delta, seed, static_cast<u32>(idx));
    *j_out = j;
    if (js_out) *js_out = sampled;
    return SHS_OK;
}

namespace {
}  // namespace


// ---------------------------------------------------------------------------
// In-process groups (shard_group.hpp)

int plan_devices(uint64_t N, int first_device, std::vector<int>* devices) {
    devices->clear();
    if (const char* env = std::getenv("SHS_DEVICES")) {  // e.g. "0,1" or "0,0" (virtual shards)
        std::string v(env);
        size_t pos = 0;
        while (pos <= v.size()) {
            size_t e = v.find(',', pos);
            if (e == std::string::npos) e = v.size();
            if (e > pos) devices->push_back(std::atoi(v.substr(pos, e - pos).c_str()));
            pos = e + 1;
        }
        if (devices->empty()) return set_error(SHS_INVALID_ARGUMENT, "SHS_DEVICES is empty");
        return SHS_OK;
    }
    const double need = 32.0 * static_cast<double>(N);  // sel + successor (or P) per amplitude
    const double slack = 2.0e9;                         // partials, plans, scratch
    if (need + slack <= 16.0e9) {  // fits any B200: no device query per engine
        devices->push_back(first_device);
        return SHS_OK;
    }
    int ndev = 0;
    RUN_CUDA(cudaGetDeviceCount(&ndev));
    size_t fr = 0, tot = 0;
    RUN_CUDA(cudaSetDevice(first_device));
    RUN_CUDA(cudaMemGetInfo(&fr, &tot));
    if (need + slack <= static_cast<double>(fr)) {
        devices->push_back(first_device);
        return SHS_OK;
    }
    for (int G = 2; G <= std::min(ndev, kMaxShards); ++G)
        if (need / G + slack <= static_cast<double>(fr)) {
            for (int q = 0; q < G; ++q) devices->push_back((first_device + q) % ndev);
            return SHS_OK;
        }
    return set_error(SHS_CUDA_ERROR, "the state (" + std::to_string(need / 1e9) +
                                         " GB) does not fit the " + std::to_string(ndev) +
                                         " visible device(s)");
}

void group_destroy(ShardGroup* g) {
    if (!g) return;
    for (shs_shard* q : g->shards) release(q);
    delete g;
}

int group_create(const shs_problem& problem, const shs_error& error, const shs_options& options,
                 const std::vector<int>& devices, ShardGroup** out) {
    auto* g = new ShardGroup;
    const uint32_t G = static_cast<uint32_t>(devices.size());
    for (uint32_t q = 0; q < G; ++q) {
        // the group's shards on this device (this one included)
        g_coresident = static_cast<uint32_t>(std::count(devices.begin(), devices.end(), devices[q]));
        shs_options o = options;
        o.device = devices[q];
        o.n_devices = 0;
        o.devices = nullptr;
        shs_shard* sh = nullptr;
        int rc = shs_shard_create(&problem, &error, &o, q, G, &sh);
        g_coresident = 1;
        if (rc) {
            group_destroy(g);
            return rc;
        }
        g->shards.push_back(sh);
    }
    for (shs_shard* a : g->shards)
        for (shs_shard* b : g->shards)
            if (a != b) {
                int rc = shs_shard_attach_local(a, b);
                if (rc) {
                    group_destroy(g);
                    return rc;
                }
            }
    g->N = problem.N;
    g->S = g->shards[0]->S;
    g->t = problem.t;
    *out = g;
    return SHS_OK;
}

int group_run(ShardGroup* g, u64 seed, u64 idx, u128* j, u128* js, shs_stage_trace* trace) {
    int rc = shards_run(g->shards, nullptr, seed, idx, j, js, trace);
    g->pending = rc == SHS_OK;
    return rc;
}

int group_state_init(ShardGroup* g) {
    for (shs_shard* q : g->shards) shs_shard_init(q);
    g->pending = false;
    return SHS_OK;
}

// the per-gate path over the group: exchange on every shard, then probs and the
// exact digit sum (what the device-resident run does on the device)
int group_stage_probs(ShardGroup* g, uint32_t s, u128 prefix, double* p0, double* p1) {
    int rc;
    for (shs_shard* q : g->shards)
        if ((rc = shs_shard_exchange(q, s))) return rc;
    for (shs_shard* q : g->shards)
        if ((rc = shs_shard_sync(q))) return rc;
    uint64_t total[SHS_DIGITS] = {}, d[SHS_DIGITS];
    for (shs_shard* q : g->shards) {
        if ((rc = shs_shard_probs(q, s, static_cast<uint64_t>(prefix),
                                  static_cast<uint64_t>(prefix >> 64), d)))
            return rc;
        for (int i = 0; i < SHS_DIGITS; ++i) total[i] += d[i];
    }
    shs_digits_to_probs(total, &g->p0, &g->p1);
    if (g->shards[0]->kahan && (rc = shs_shard_kahan_probs(g->shards[0], &g->p0, &g->p1)))
        return rc;
    *p0 = g->p0;
    *p1 = g->p1;
    g->pending = true;
    if (g->shards[0]->opt.check_norms && std::fabs(g->p0 + g->p1 - 1.0) > kNormTolerance)
        return set_error(SHS_ERROR, "statevector norm drifted beyond 1e-9 at stage " +
                                        std::to_string(s));
    return SHS_OK;
}

int group_stage_collapse(ShardGroup* g, int src_group, double p_src) {
    int rc;
    for (shs_shard* q : g->shards)
        if ((rc = shs_shard_collapse(q, src_group, p_src))) return rc;
    for (shs_shard* q : g->shards)
        if ((rc = shs_shard_sync(q))) return rc;
    g->pending = false;
    return SHS_OK;
}

template <typename F>
int group_read_ranges(ShardGroup* g, uint64_t first, uint64_t count, double* host, F&& read) {
    std::fill(host, host + 2 * count, 0.0);
    for (shs_shard* q : g->shards) {
        const uint64_t a = std::max(first, q->lo), b = std::min(first + count, q->hi);
        if (a >= b) continue;
        int rc = read(q, a, b - a, host + 2 * (a - first));
        if (rc) return rc;
    }
    return SHS_OK;
}

int group_state_read(ShardGroup* g, int x, uint64_t first, uint64_t count, double* host) {
    return group_read_ranges(g, first, count, host, [&](shs_shard* q, uint64_t a, uint64_t n,
                                                        double* out) {
        return shs_shard_state_read(q, x, a, n, out);
    });
}

int group_stage_read(ShardGroup* g, int x, uint64_t first, uint64_t count, double* host) {
    return group_read_ranges(g, first, count, host, [&](shs_shard* q, uint64_t a, uint64_t n,
                                                        double* out) {
        return shs_shard_stage_read(q, x, a, n, out);
    });
}

int group_state_gather(ShardGroup* g, int x, const uint64_t* idx, uint64_t count, double* host) {
    // one contiguous read per index (the parity checks gather a few thousand points)
    for (uint64_t i = 0; i < count; ++i) {
        double v[2] = {0.0, 0.0};
        if (idx[i] < g->N) {
            shs_shard* q = g->shards[std::min<uint64_t>(idx[i] / g->S, g->shards.size() - 1)];
            int rc = shs_shard_state_read(q, x, idx[i], 1, v);
            if (rc) return rc;
        }
        host[2 * i] = v[0];
        host[2 * i + 1] = v[1];
    }
    return SHS_OK;
}

int group_set_sparse(ShardGroup* g, bool on) {
    for (shs_shard* q : g->shards) shs_shard_set_sparse(q, on ? 1 : 0);
    return SHS_OK;
}

uint32_t group_sparse_stages(const ShardGroup* g) { return shs_shard_sparse_stages(g->shards[0]); }

uint64_t group_launches(const ShardGroup* g) {
    uint64_t n = 0;
    for (const shs_shard* q : g->shards) n += q->launches;
    return n;
}

int shard_device(const shs_shard* sh) { return sh->dev; }

uint64_t group_device_bytes(const ShardGroup* g) {
    uint64_t n = 0;
    for (const shs_shard* q : g->shards) n += q->device_bytes;
    return n;
}

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
            // shards keep no per-row head scratch (the single engine's reason for
            // the 2^18-row cap): rows of ~8192 at every size, so the exchanges
            // have as many bands (warps / tiles) as the state has rows
            cache.emplace_back(sh->a_pows[s],
                               make_tile_plan(sh->a_pows[s], sh->a_invs[s], sh->N, o.tiling, 0,
                                              uint64_t(1) << 22));
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
    const uint64_t nb_total = (sh->N + kBlock - 1) / kBlock;
    sh->kahan = o.combine == SHS_COMBINE_KAHAN ||
                (o.combine == SHS_COMBINE_AUTO && nb_total <= kKahanMaxBlocks);
    if ((ce = cudaMalloc(&sh->Sb, sizeof(double) * 2 * sh->nb * (sh->kahan ? 2 : 1))) != cudaSuccess)
        return fail(ce, "cudaMalloc(block sums)");
    if (sh->kahan) {
        if ((ce = cudaMalloc(&sh->Scat, sizeof(double) * 2 * nb_total)) != cudaSuccess ||
            (ce = cudaMalloc(&sh->d_p, sizeof(double) * 2)) != cudaSuccess)
            return fail(ce, "cudaMalloc(kahan scratch)");
    }
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
    // device-resident run state (shard_run)
    if ((ce = cudaMalloc(&sh->d_slots, 2 * sizeof(DevStage))) != cudaSuccess)
        return fail(ce, "cudaMalloc(slots)");
    if ((ce = cudaHostAlloc(&sh->h_rec, sizeof(StageRec) * sh->t, cudaHostAllocMapped)) != cudaSuccess)
        return fail(ce, "cudaHostAlloc(records)");
    if ((ce = cudaHostGetDevicePointer(reinterpret_cast<void**>(&sh->d_rec), sh->h_rec, 0)) !=
        cudaSuccess)
        return fail(ce, "cudaHostGetDevicePointer");
    if ((ce = cudaMalloc(&sh->d_dig2, sizeof(unsigned long long) * 4 * kDigits)) != cudaSuccess)
        return fail(ce, "cudaMalloc(stage digits)");
    if ((ce = cudaMemset(sh->d_dig2, 0, sizeof(unsigned long long) * 4 * kDigits)) != cudaSuccess)
        return fail(ce, "cudaMemset");
    for (int k = 0; k < 2; ++k) {
        const unsigned ipc = cudaEventDisableTiming | cudaEventInterprocess;
        if ((ce = cudaEventCreateWithFlags(&sh->evx[k], ipc)) != cudaSuccess ||
            (ce = cudaEventCreateWithFlags(&sh->evd[k], ipc)) != cudaSuccess ||
            (ce = cudaEventCreateWithFlags(&sh->evc[k], ipc)) != cudaSuccess ||
            (ce = cudaEventCreateWithFlags(&sh->evm[k], cudaEventDisableTiming)) != cudaSuccess)
            return fail(ce, "cudaEventCreate(run events)");
        sh->pevx[rank][k] = sh->evx[k];
        sh->pevd[rank][k] = sh->evd[k];
        sh->pevc[rank][k] = sh->evc[k];
    }
    if (nshards >= 2) {  // exchange v2: receive slots, round count, bases, pack stream
        const char* xe = std::getenv("SHS_EXCHANGE");
        sh->x2_on = !(xe && xe[0] == '1');
        size_t fr = 0, tot = 0;
        if ((ce = cudaMemGetInfo(&fr, &tot)) != cudaSuccess) return fail(ce, "cudaMemGetInfo");
        // a round receives ~S/K elements (more where few rows make the z-spread
        // lumpy): slots of c S / K with c = 2 when memory allows, down to 1.25,
        // then more rounds. K is collective (every rank must cut the same rounds):
        // a function of the device's TOTAL memory and S only, identical on
        // identical GPUs; peers' K are checked when they attach. The device is
        // shared by the group's g_coresident shards placed on it.
        const double reserve = 6.0e9;  // contexts, partials, plans, scratch
        const double state = 2.0 * sizeof(double2) * static_cast<double>(sh->S);
        const double avail = (static_cast<double>(tot) - reserve) / g_coresident - state;
        const double slot_cap = std::max(0.0, avail) / (2 * sizeof(double2));
        const double Sd = static_cast<double>(sh->S);
        uint32_t K = 1;
        double c = 2.0;
        while (c * Sd / K + 65536.0 > slot_cap) {
            if (c > 1.25) c = std::max(1.25, c - 0.25);
            else if (K < 256) ++K;
            else break;
        }
        if (const char* kr = std::getenv("SHS_X2_ROUNDS")) K = std::max(1, std::atoi(kr));
        sh->x2_K = K;
        sh->x2_slot = static_cast<uint64_t>(c * Sd / K) + 65536;
        if ((ce = cudaMalloc(&sh->x2_recv, 2 * sizeof(double2) * sh->x2_slot)) != cudaSuccess)
            return fail(ce, "cudaMalloc(exchange receive slots)");
        // [t][K][G] region bases, then [t] "every round of the stage fits my slot"
        if ((ce = cudaMalloc(&sh->x2_bases,
                             sizeof(unsigned long long) * sh->t * (uint64_t(K) * nshards + 1))) !=
            cudaSuccess)
            return fail(ce, "cudaMalloc(exchange bases)");
        if ((ce = cudaStreamCreateWithFlags(&sh->xstream, cudaStreamNonBlocking)) != cudaSuccess)
            return fail(ce, "cudaStreamCreate(pack)");
        for (int k = 0; k < 2; ++k) {
            const unsigned ipc = cudaEventDisableTiming | cudaEventInterprocess;
            if ((ce = cudaEventCreateWithFlags(&sh->evp[k], ipc)) != cudaSuccess ||
                (ce = cudaEventCreateWithFlags(&sh->evu[k], ipc)) != cudaSuccess)
                return fail(ce, "cudaEventCreate(exchange events)");
            sh->pevp[rank][k] = sh->evp[k];
            sh->pevu[rank][k] = sh->evu[k];
        }
        sh->peer_recv[rank] = sh->x2_recv;
        sh->peer_bases[rank] = sh->x2_bases;
        sh->device_bytes += 2 * sizeof(double2) * sh->x2_slot;
    }
    sh->peer_dig[rank] = sh->d_dig2;
    sh->peer_S[rank] = sh->Sb;
    sh->peer[rank][0] = sh->buf[0];
    sh->peer[rank][1] = sh->buf[1];
    if (!sh->kahan) {  // support points fit every shard's P (the last shard is the smallest)
        const uint64_t smallest = sh->N - uint64_t(nshards - 1) * sh->S;
        const uint64_t bytes = sizeof(double2) * std::min(smallest, sh->S);
        // 88 B of carved arrays + the radix sort's ~24 B per point, 1 MB of slack
        const uint64_t kcap = bytes > (1ull << 20) ? (bytes - (1ull << 20)) / 128 : 0;
        sh->sparse_n = sparse_prefix_stages(sh->N, sh->t, sh->a_pows,
                                            std::min<uint64_t>(sh->N / kSparseDensity, kcap));
    }
    sh->device_bytes = 2 * sizeof(double2) * sh->nloc + sizeof(double) * 2 * sh->nb +
                       sizeof(unsigned long long) * (2 * kDigits * sh->grid_cap + 6 * kDigits);
    *out = sh;
    return SHS_OK;
}

void shs_shard_destroy(shs_shard* sh) { release(sh); }

int shs_shard_attach_local(shs_shard* sh, shs_shard* peer) {
    if (!sh || !peer || peer->G != sh->G || peer->rank >= sh->G)
        return set_error(SHS_INVALID_ARGUMENT, "bad local attach");
    if (peer == sh) return SHS_OK;
    if (peer->x2_K != sh->x2_K)
        return set_error(SHS_INVALID_ARGUMENT, "exchange rounds differ between shards");
    void* bufs[2] = {peer->buf[0], peer->buf[1]};
    int rc = shs_shard_attach(sh, peer->rank, bufs);
    if (rc) return rc;
    sh->peer_dig[peer->rank] = peer->d_dig2;
    sh->peer_S[peer->rank] = peer->Sb;
    sh->peer_recv[peer->rank] = peer->x2_recv;
    sh->peer_bases[peer->rank] = peer->x2_bases;
    for (int k = 0; k < 2; ++k) {
        sh->pevp[peer->rank][k] = peer->evp[k];
        sh->pevu[peer->rank][k] = peer->evu[k];
    }
    for (int k = 0; k < 2; ++k) {  // cross-device stream waits on events work in-process
        sh->pevx[peer->rank][k] = peer->evx[k];
        sh->pevd[peer->rank][k] = peer->evd[k];
        sh->pevc[peer->rank][k] = peer->evc[k];
    }
    sh->peer_ev_ipc[peer->rank] = false;
    return SHS_OK;
}

int shs_shards_run(shs_shard* const* shards, uint32_t count, uint64_t seed, uint64_t idx,
                   uint64_t j[2], uint64_t j_sampled[2], shs_stage_trace* trace) {
    if (!shards || count == 0 || !j) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    std::vector<shs_shard*> L(shards, shards + count);
    const uint32_t G = L[0]->G;
    ShmBarrier* bar = nullptr;
    if (count < G) {
        bar = L[0]->barrier;
        if (!bar)
            return set_error(SHS_INVALID_ARGUMENT,
                             "sharded run over processes needs shs_shard_set_barrier");
    }
    u128 jj = 0, js = 0;
    int rc = shards_run(L, bar, seed, idx, &jj, &js, trace);
    if (rc) return rc;
    j[0] = static_cast<uint64_t>(jj);
    j[1] = static_cast<uint64_t>(jj >> 64);
    if (j_sampled) {
        j_sampled[0] = static_cast<uint64_t>(js);
        j_sampled[1] = static_cast<uint64_t>(js >> 64);
    }
    return SHS_OK;
}

uint64_t shs_shard_device_bytes(const shs_shard* sh) { return sh ? sh->device_bytes : 0; }
// The node-local host barrier of multi-process runs, exposed on its own (no
// device involved) so the host side of the protocol is testable without a GPU.
struct shs_node_barrier {
    ShmBarrier bar;
};

int shs_node_barrier_open(const char* name, uint32_t parties, int32_t unlink_at_close,
                          shs_node_barrier** out) {
    if (!name || name[0] != '/' || parties < 1 || !out)
        return set_error(SHS_INVALID_ARGUMENT, "barrier: name must start with '/', parties >= 1");
    auto* b = new shs_node_barrier;
    int rc = b->bar.open(name, parties, unlink_at_close != 0);
    if (rc) {
        delete b;
        return rc;
    }
    *out = b;
    return SHS_OK;
}

int shs_node_barrier_arrive(shs_node_barrier* b) {
    if (!b) return set_error(SHS_INVALID_ARGUMENT, "null barrier");
    return b->bar.arrive();
}

void shs_node_barrier_close(shs_node_barrier* b) { delete b; }


int shs_shard_kahan(const shs_shard* sh) { return sh && sh->kahan ? 1 : 0; }

int shs_shard_set_timeline(shs_shard* sh, int32_t enable) {
    if (!sh) return set_error(SHS_INVALID_ARGUMENT, "null shard");
    sh->tl_on = enable != 0;
    return SHS_OK;
}

int64_t shs_shard_timeline(shs_shard* sh, double* out, uint64_t max_entries) {
    if (!sh || !sh->tl0) return 0;
    if (cudaSetDevice(sh->dev) != cudaSuccess) return -1;
    cudaDeviceSynchronize();
    uint64_t n = 0;
    for (const auto& r : sh->tl) {
        if (n < max_entries && out) {
            float a = 0.f, b = 0.f;
            cudaEventElapsedTime(&a, sh->tl0, r.a);
            cudaEventElapsedTime(&b, sh->tl0, r.b);
            out[3 * n] = r.kind;
            out[3 * n + 1] = a;
            out[3 * n + 2] = b;
        }
        ++n;
    }
    return static_cast<int64_t>(n);
}

int shs_shard_set_sparse(shs_shard* sh, int32_t enable) {
    if (!sh) return set_error(SHS_INVALID_ARGUMENT, "null shard");
    sh->sparse_on = enable != 0;
    return SHS_OK;
}

uint32_t shs_shard_sparse_stages(const shs_shard* sh) {
    return sh && sh->sparse_on ? sh->sparse_n : 0;
}

int shs_shard_kahan_probs(shs_shard* sh, double* p0, double* p1) {
    return shard_guard(sh, [&]() -> int {
        if (!sh->kahan) return set_error(SHS_INVALID_ARGUMENT, "shard combines exactly (digits)");
        if (!p0 || !p1) return set_error(SHS_INVALID_ARGUMENT, "null argument");
        for (uint32_t r = 0; r < sh->G; ++r)
            if (!sh->peer_S[r]) return set_error(SHS_INVALID_ARGUMENT, "peer partials not attached");
        const ShardPartials sp = shard_partials(sh, 0);
        const uint64_t nbt = sp.off[sh->G];
        const int gg = static_cast<int>(std::min<uint64_t>((2 * nbt + 255) / 256, 1024));
        k_shard_gather_partials<<<gg, 256, 0, sh->stream>>>(sp, sh->Scat);
        k_finalize<<<1, kFinalizeThreads, 0, sh->stream>>>(nullptr, 0, sh->Scat, nbt, 1, sh->d_p);
        sh->launches += 2;
        SHD_CUDA(cudaGetLastError());
        double pp[2];
        SHD_CUDA(cudaMemcpyAsync(pp, sh->d_p, sizeof(pp), cudaMemcpyDeviceToHost, sh->stream));
        SHD_CUDA(cudaStreamSynchronize(sh->stream));
        *p0 = pp[0];
        *p1 = pp[1];
        return SHS_OK;
    });
}



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

// What a peer process needs to reach this shard: its two state buffers, its
// per-stage digits and its three ordering events per parity.
struct ShardIpcBlob {
    cudaIpcMemHandle_t buf[2];
    cudaIpcMemHandle_t dig;
    cudaIpcMemHandle_t sb;
    cudaIpcEventHandle_t evx[2], evd[2], evc[2];
    cudaIpcMemHandle_t recv, bases;  // exchange v2
    cudaIpcEventHandle_t evp[2], evu[2];
    int32_t has_x2;
    uint32_t x2_K;
};
static_assert(sizeof(ShardIpcBlob) <= SHS_SHARD_IPC_BYTES, "SHS_SHARD_IPC_BYTES too small");

int shs_shard_ipc_handles(const shs_shard* csh, void* out) {
    auto* sh = const_cast<shs_shard*>(csh);
    return shard_guard(sh, [&]() -> int {
        if (!out) return set_error(SHS_INVALID_ARGUMENT, "null argument");
        ShardIpcBlob b;
        for (int k = 0; k < 2; ++k) SHD_CUDA(cudaIpcGetMemHandle(&b.buf[k], sh->buf[k]));
        SHD_CUDA(cudaIpcGetMemHandle(&b.dig, sh->d_dig2));
        SHD_CUDA(cudaIpcGetMemHandle(&b.sb, sh->Sb));
        b.has_x2 = sh->x2_recv ? 1 : 0;
        b.x2_K = sh->x2_K;
        if (b.has_x2) {
            SHD_CUDA(cudaIpcGetMemHandle(&b.recv, sh->x2_recv));
            SHD_CUDA(cudaIpcGetMemHandle(&b.bases, sh->x2_bases));
            for (int k = 0; k < 2; ++k) {
                SHD_CUDA(cudaIpcGetEventHandle(&b.evp[k], sh->evp[k]));
                SHD_CUDA(cudaIpcGetEventHandle(&b.evu[k], sh->evu[k]));
            }
        }
        for (int k = 0; k < 2; ++k) {
            SHD_CUDA(cudaIpcGetEventHandle(&b.evx[k], sh->evx[k]));
            SHD_CUDA(cudaIpcGetEventHandle(&b.evd[k], sh->evd[k]));
            SHD_CUDA(cudaIpcGetEventHandle(&b.evc[k], sh->evc[k]));
        }
        std::memset(out, 0, SHS_SHARD_IPC_BYTES);
        std::memcpy(out, &b, sizeof(b));
        return SHS_OK;
    });
}

// Raw device pointers of a peer's buffers, valid in this process. A buffer on
// another device is reached over NVLink: peer access is enabled here (an
// explicit error when the devices cannot access each other).
int shs_shard_attach(shs_shard* sh, uint32_t peer, void* const bufs[2]) {
    return shard_guard(sh, [&]() -> int {
        if (!bufs || peer >= sh->G) return set_error(SHS_INVALID_ARGUMENT, "bad attach");
        for (int b = 0; b < 2; ++b) {
            cudaPointerAttributes at{};
            SHD_CUDA(cudaPointerGetAttributes(&at, bufs[b]));
            if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
                return set_error(SHS_INVALID_ARGUMENT, "attach: not a device pointer");
            if (at.device != sh->dev) {
                int can = 0;
                SHD_CUDA(cudaDeviceCanAccessPeer(&can, sh->dev, at.device));
                if (!can)
                    return set_error(SHS_INVALID_ARGUMENT,
                                     "attach: device " + std::to_string(sh->dev) +
                                         " cannot access device " + std::to_string(at.device));
                cudaError_t pe = cudaDeviceEnablePeerAccess(at.device, 0);
                if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else if (pe != cudaSuccess)
                    return set_error(SHS_CUDA_ERROR, std::string("cudaDeviceEnablePeerAccess: ") +
                                                         cudaGetErrorString(pe));
            }
        }
        sh->peer[peer][0] = static_cast<double2*>(bufs[0]);
        sh->peer[peer][1] = static_cast<double2*>(bufs[1]);
        sh->peer_ipc[peer] = false;
        return SHS_OK;
    });
}

int shs_shard_attach_ipc(shs_shard* sh, uint32_t peer, const void* handles) {
    return shard_guard(sh, [&]() -> int {
        if (!handles || peer >= sh->G) return set_error(SHS_INVALID_ARGUMENT, "bad attach");
        if (peer == sh->rank) return SHS_OK;
        ShardIpcBlob b;
        std::memcpy(&b, handles, sizeof(b));
        for (int k = 0; k < 2; ++k) {
            void* p = nullptr;
            SHD_CUDA(cudaIpcOpenMemHandle(&p, b.buf[k], cudaIpcMemLazyEnablePeerAccess));
            sh->peer[peer][k] = static_cast<double2*>(p);
        }
        sh->peer_ipc[peer] = true;
        void* d = nullptr;
        SHD_CUDA(cudaIpcOpenMemHandle(&d, b.dig, cudaIpcMemLazyEnablePeerAccess));
        sh->peer_dig[peer] = static_cast<const unsigned long long*>(d);
        sh->peer_dig_ipc[peer] = true;
        void* sp = nullptr;
        SHD_CUDA(cudaIpcOpenMemHandle(&sp, b.sb, cudaIpcMemLazyEnablePeerAccess));
        sh->peer_S[peer] = static_cast<const double*>(sp);
        sh->peer_S_ipc[peer] = true;
        if (b.has_x2 && sh->x2_recv) {
            if (b.x2_K != sh->x2_K)
                return set_error(SHS_INVALID_ARGUMENT,
                                 "exchange rounds differ between shards (" + std::to_string(b.x2_K) +
                                     " vs " + std::to_string(sh->x2_K) + "): set SHS_X2_ROUNDS");
            void* rp = nullptr;
            SHD_CUDA(cudaIpcOpenMemHandle(&rp, b.recv, cudaIpcMemLazyEnablePeerAccess));
            sh->peer_recv[peer] = static_cast<double2*>(rp);
            sh->peer_recv_ipc[peer] = true;
            void* bp = nullptr;
            SHD_CUDA(cudaIpcOpenMemHandle(&bp, b.bases, cudaIpcMemLazyEnablePeerAccess));
            sh->peer_bases[peer] = static_cast<const unsigned long long*>(bp);
            sh->peer_bases_ipc[peer] = true;
            for (int k = 0; k < 2; ++k) {
                SHD_CUDA(cudaIpcOpenEventHandle(&sh->pevp[peer][k], b.evp[k]));
                SHD_CUDA(cudaIpcOpenEventHandle(&sh->pevu[peer][k], b.evu[k]));
            }
        }
        for (int k = 0; k < 2; ++k) {
            SHD_CUDA(cudaIpcOpenEventHandle(&sh->pevx[peer][k], b.evx[k]));
            SHD_CUDA(cudaIpcOpenEventHandle(&sh->pevd[peer][k], b.evd[k]));
            SHD_CUDA(cudaIpcOpenEventHandle(&sh->pevc[peer][k], b.evc[k]));
        }
        sh->peer_ev_ipc[peer] = true;
        return SHS_OK;
    });
}

int shs_shard_set_barrier(shs_shard* sh, const char* name) {
    if (!sh || !name || name[0] != '/')
        return set_error(SHS_INVALID_ARGUMENT, "barrier name must start with '/'");
    delete sh->barrier;
    sh->barrier = new ShmBarrier;
    int rc = sh->barrier->open(name, sh->G, sh->rank == 0);
    if (rc) {
        delete sh->barrier;
        sh->barrier = nullptr;
    }
    return rc;
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
        int rc = launch_exchange(sh, s);
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
    for (int k = 0; k < 5; ++k) {
        sh->kms[k] = 0;
        sh->klaunch[k] = 0;
    }
    return SHS_OK;
}

int shs_shard_kernel_times(const shs_shard* sh, double ms[5], uint64_t launches[5]) {
    if (!sh) return set_error(SHS_INVALID_ARGUMENT, "null shard");
    for (int k = 0; k < 5; ++k) {
        if (ms) ms[k] = sh->kms[k];
        if (launches) launches[k] = sh->klaunch[k];
    }
    return SHS_OK;
}

uint64_t shs_shard_launch_count(const shs_shard* sh) { return sh ? sh->launches : 0; }

void* shs_shard_stream(const shs_shard* sh) { return sh ? static_cast<void*>(sh->stream) : nullptr; }

}  // extern "C"
