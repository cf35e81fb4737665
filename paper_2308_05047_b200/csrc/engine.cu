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

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/shorsim_b200.h"
#include "device_math.cuh"
#include "host_model.hpp"
#include "tiled.cuh"

using namespace shs;

namespace {

thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

#define SHS_CUDA(call)                                                                  \
    do {                                                                                \
        cudaError_t _e = (call);                                                        \
        if (_e != cudaSuccess)                                                          \
            return set_error(SHS_CUDA_ERROR, std::string(#call) + ": " +                \
                                                 cudaGetErrorString(_e));               \
    } while (0)

constexpr double kNormTolerance = 1e-9;     // statevector.cpp:18
constexpr double kDegenerateMass = 1e-300;  // statevector.cpp:19
constexpr uint64_t kKahanMaxBlocks = 1024;  // AUTO: sequential Kahan up to 2^18 amplitudes
constexpr uint64_t kTileAutoMinN = 1ull << 20;  // AUTO tiling from 16 MB of state
constexpr uint64_t kTileMinRow = 512;           // every 256-block touches <= 2 rows
constexpr uint64_t kTileMaxRows = 1ull << 18;   // head scratch <= 1 GB
constexpr uint64_t kTileMinRowsPlan = 256;      // >= 16 tiles of kRows rows

// Host side of a stage's sorted-residue tiling (see tiled.cuh).
struct TilePlanHost {
    bool tiled = false;
    uint64_t H = 0, u = 0, v = 0, du = 0, dv = 0;
    uint64_t A = 0, A_sh = 0, m = 0, m_sh = 0, ntiles = 0;
};

// Pick the largest row count H (powers of two and 3 * 2^k up to N/1024) whose
// three gap lengths are all >= kTileMinRow and at most 3x the mean row: one
// O(H) scan of j*A mod N with running argmin / argmax gives u(H), v(H) for
// every candidate. Multipliers without such an H (tiny A, or A/N with a huge
// partial quotient) keep the direct gather, whose warps then read a few long
// runs anyway.
TilePlanHost make_tile_plan(uint64_t A, uint64_t m, uint64_t N, int tiling) {
    TilePlanHost pl;
    if (tiling == SHS_TILING_OFF || A == 1) return pl;
    if (tiling == SHS_TILING_AUTO && N < kTileAutoMinN) return pl;
    const uint64_t hmax = std::min<uint64_t>(N / 1024, kTileMaxRows);
    std::vector<uint64_t> cands;
    for (uint64_t h = 2; h <= hmax; h *= 2) {
        cands.push_back(h);
        if (h >= 4 && h / 2 * 3 <= hmax) cands.push_back(h / 2 * 3);
    }
    std::sort(cands.begin(), cands.end());
    uint64_t j = 1, r = 0, umin = N, uj = 0, vmax = 0, vj = 0;
    for (uint64_t H : cands) {
        for (; j < H; ++j) {
            r += A;
            if (r >= N) r -= N;
            if (r < umin) { umin = r; uj = j; }
            if (r > vmax) { vmax = r; vj = j; }
        }
        const uint64_t du = umin, dv = N - vmax;
        // rows must be long enough (each 256-block touches <= 2 rows) and balanced
        // (the longest row, du + dv, within 3x the mean N / H), else a tile idles SMs
        if (H >= kTileMinRowsPlan && du >= kTileMinRow && dv >= kTileMinRow &&
            du + dv <= 3 * (N / H + 1)) {
            pl.tiled = true;
            pl.H = H;
            pl.u = uj;
            pl.v = vj;
            pl.du = du;
            pl.dv = dv;
        }
    }
    if (pl.tiled) {
        pl.A = A;
        pl.A_sh = shoup(A, N);
        pl.m = m;
        pl.m_sh = shoup(m, N);
        pl.ntiles = (pl.H + kRows - 1) / kRows;
    }
    return pl;
}

struct StageParams {
    const double2* X;
    double2* Y;
    uint64_t N;
    uint64_t m;       // a_inv of the stage
    uint64_t m_sh;    // Shoup companion of m
    uint64_t m_step;  // kBlock * m mod N: source advance per thread element
    StageScalars sc;
    double* S;        // block partials: S0 [0, nb), S1 [nb, 2 nb)
    uint64_t nb;
    unsigned long long* partials;  // [gridDim.x][2][kDigits]
    uint64_t nchunks;
    int sel;          // collapse: group kept
};

template <bool kE1>
__device__ __forceinline__ double2 load_amp(const double2* __restrict__ X, uint64_t z) {
    if (kE1) return make_double2(z == 1 ? 1.0 : 0.0, 0.0);  // run start: sel = e_1, inv = 1
    return __ldg(X + z);
}

// Amplitude pairs (sel[z], sel[src z]) for the kPer elements z0 + e*kBlock of one thread.
template <bool kGather, bool kE1>
__device__ __forceinline__ void load_pairs(const StageParams& p, uint64_t z0, double2 (&xa)[kPer],
                                           double2 (&xs)[kPer]) {
    uint64_t src = kGather ? mulmod_shoup(z0, p.m, p.m_sh, p.N) : 0;
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
        const uint64_t z = z0 + uint64_t(e) * kBlock;
        if (z < p.N) {
            xa[e] = load_amp<kE1>(p.X, z);
            xs[e] = kGather ? load_amp<kE1>(p.X, src) : xa[e];
        } else {
            xa[e] = make_double2(0.0, 0.0);
            xs[e] = xa[e];
        }
        if (kGather) src = addmod(src, p.m_step, p.N);
    }
}

template <bool kGather, bool kE1>
__global__ void __launch_bounds__(kThreads) k_stage_probs(StageParams p) {
    __shared__ double nrm[2 * kPer][kBlock + 1];  // +1: conflict-free column walks
    __shared__ unsigned long long digits[2][kDigits];
    const int tid = threadIdx.x;
    for (int i = tid; i < 2 * kDigits; i += kThreads) (&digits[0][0])[i] = 0ull;
    DigitWindow win;
    window_reset(win);
    __syncthreads();

    for (uint64_t c = blockIdx.x; c < p.nchunks; c += gridDim.x) {
        const uint64_t z0 = c * kChunk + tid;
        double2 xa[kPer], xs[kPer];
        load_pairs<kGather, kE1>(p, z0, xa, xs);
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            double h0r, h0i, h1r, h1i;
            stage_pair(p.sc, xa[e], xs[e], h0r, h0i, h1r, h1i);
            const bool live = z0 + uint64_t(e) * kBlock < p.N;
            nrm[e][tid] = live ? cnorm(h0r, h0i) : 0.0;
            nrm[kPer + e][tid] = live ? cnorm(h1r, h1i) : 0.0;
        }
        __syncthreads();
        if (tid < 2 * kPer) {
            // one lane per (block, group): the reference's in-order block sum
            double s = 0.0;
#pragma unroll 16
            for (int i = 0; i < kBlock; ++i) s = __dadd_rn(s, nrm[tid][i]);
            const uint64_t b = c * kPer + (tid & (kPer - 1));
            const int g = tid / kPer;
            if (b < p.nb) {
                p.S[g * p.nb + b] = s;
                window_add(win, s, digits[g]);
            }
        }
        __syncthreads();
    }
    if (tid < 2 * kPer) window_flush(win, digits[tid / kPer]);
    __syncthreads();
    if (tid < 2) {
        unsigned long long carry = 0;
        unsigned long long* out = p.partials + (uint64_t(blockIdx.x) * 2 + tid) * kDigits;
        for (int i = 0; i < kDigits; ++i) {
            unsigned long long v = digits[tid][i] + carry;
            out[i] = v & 0xffffffffull;
            carry = v >> 32;
        }
    }
}

// p0/p1 from the stage. kahan: reference combine_blocks (statevector.cpp:32-40),
// two interleaved sequential chains, zeros skipped; else exact sum of partials.
__global__ void k_finalize(const unsigned long long* __restrict__ partials, int nparts,
                           const double* __restrict__ S, uint64_t nb, int kahan,
                           double* __restrict__ out) {
    __shared__ unsigned long long acc[2][kDigits];
    if (kahan) {
        if (threadIdx.x == 0) {
            double s0 = 0, c0 = 0, s1 = 0, c1 = 0;
            for (uint64_t b = 0; b < nb; ++b) {
                const double x0 = S[b], x1 = S[nb + b];
                if (x0 != 0.0) {
                    double y = __dsub_rn(x0, c0);
                    double t = __dadd_rn(s0, y);
                    c0 = __dsub_rn(__dsub_rn(t, s0), y);
                    s0 = t;
                }
                if (x1 != 0.0) {
                    double y = __dsub_rn(x1, c1);
                    double t = __dadd_rn(s1, y);
                    c1 = __dsub_rn(__dsub_rn(t, s1), y);
                    s1 = t;
                }
            }
            out[0] = s0;
            out[1] = s1;
        }
        return;
    }
    for (int i = threadIdx.x; i < 2 * kDigits; i += blockDim.x) {
        unsigned long long s = 0;
        for (int c = 0; c < nparts; ++c) s += partials[uint64_t(c) * 2 * kDigits + i];
        (&acc[0][0])[i] = s;
    }
    __syncthreads();
    if (threadIdx.x < 2) out[threadIdx.x] = digits_to_double(acc[threadIdx.x]);
}

template <bool kGather, bool kE1>
__global__ void __launch_bounds__(kThreads) k_stage_collapse(StageParams p) {
    const int tid = threadIdx.x;
    for (uint64_t c = blockIdx.x; c < p.nchunks; c += gridDim.x) {
        const uint64_t z0 = c * kChunk + tid;
        double2 xa[kPer], xs[kPer];
        load_pairs<kGather, kE1>(p, z0, xa, xs);
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const uint64_t z = z0 + uint64_t(e) * kBlock;
            double h0r, h0i, h1r, h1i;
            stage_pair(p.sc, xa[e], xs[e], h0r, h0i, h1r, h1i);
            if (z < p.N) p.Y[z] = p.sel ? make_double2(h1r, h1i) : make_double2(h0r, h0i);
        }
    }
}

// Post-Hadamard amplitudes of group x for y in [first, first + count).
template <bool kGather, bool kE1>
__global__ void k_stage_read(StageParams p, int x, uint64_t first, uint64_t count,
                             double2* __restrict__ out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t z = first + i;
        if (z >= p.N) {
            out[i] = make_double2(0.0, 0.0);
            continue;
        }
        const uint64_t src = kGather ? mulmod_shoup(z, p.m, p.m_sh, p.N) : z;
        double2 xa = load_amp<kE1>(p.X, z), xs = load_amp<kE1>(p.X, src);
        double h0r, h0i, h1r, h1i;
        stage_pair(p.sc, xa, xs, h0r, h0i, h1r, h1i);
        out[i] = x ? make_double2(h1r, h1i) : make_double2(h0r, h0i);
    }
}

// g_x[y] = w_x * (sel[y] * inv), the reference state after init / reset_top.
template <bool kE1>
__global__ void k_state_read(const double2* __restrict__ X, uint64_t N, double wr, double wi,
                             double inv, uint64_t first, uint64_t count,
                             double2* __restrict__ out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t z = first + i;
        if (z >= N) {
            out[i] = make_double2(0.0, 0.0);
            continue;
        }
        double2 v = load_amp<kE1>(X, z);
        double r, im;
        cmul(wr, wi, __dmul_rn(v.x, inv), __dmul_rn(v.y, inv), r, im);
        out[i] = make_double2(r, im);
    }
}

// The index map exactly as the stage kernels walk it (Shoup per thread, then
// incremental), written out for the bit-exact index-map parity check.
__global__ void k_index_map(StageParams p, uint64_t chunk0, uint64_t nchunk, uint64_t first,
                            uint64_t count, uint64_t* __restrict__ out) {
    for (uint64_t c = chunk0 + blockIdx.x; c < chunk0 + nchunk; c += gridDim.x) {
        const uint64_t z0 = c * kChunk + threadIdx.x;
        uint64_t src = mulmod_shoup(z0, p.m, p.m_sh, p.N);
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const uint64_t z = z0 + uint64_t(e) * kBlock;
            if (z >= first && z < first + count && z < p.N) out[z - first] = src;
            src = addmod(src, p.m_step, p.N);
        }
    }
}

__global__ void k_fill_identity(uint64_t first, uint64_t count, uint64_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = first + i;
}

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
    bool kahan = false;      // resolved combine mode
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

StageParams params_for(const shs_engine* e, uint32_t s) {
    StageParams p{};
    p.X = e->X;
    p.Y = e->Y;
    p.N = e->N;
    p.m = e->a_invs[s];
    p.m_sh = e->a_pows[s] != 1 ? shoup(p.m, e->N) : 0;
    p.m_step = e->a_pows[s] != 1 ? mulmod(p.m, kBlock, e->N) : 0;
    p.sc = e->sc;
    p.S = e->S;
    p.nb = e->nb;
    p.partials = e->partials;
    p.nchunks = e->nchunks;
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

template <bool G, bool E1>
void launch_probs(shs_engine* e, const StageParams& p) {
    k_stage_probs<G, E1><<<grid_for(e), kThreads, 0, e->stream>>>(p);
}

template <bool G, bool E1>
void launch_collapse(shs_engine* e, const StageParams& p) {
    k_stage_collapse<G, E1><<<grid_for(e), kThreads, 0, e->stream>>>(p);
}

int engine_validate(const shs_problem& pr, const shs_error& er, const shs_options& o) {
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

void release(shs_engine* e) {
    if (!e) return;
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
    cudaFree(e->d_out);
    if (e->h_out) cudaFreeHost(e->h_out);
    if (e->stream) cudaStreamDestroy(e->stream);
    delete e;
}

// The two N-amplitude buffers (sel and its successor) and the block partials
// are allocated on first use, so engines used only for validation or index
// maps never reserve 2 x 16 N bytes of HBM.
int ensure_buffers(shs_engine* e) {
    if (e->X) return SHS_OK;
    const size_t amp_bytes = sizeof(double2) * e->N;
    SHS_CUDA(cudaMalloc(&e->X, amp_bytes));
    SHS_CUDA(cudaMalloc(&e->Y, amp_bytes));
    SHS_CUDA(cudaMalloc(&e->S, sizeof(double) * 2 * e->nb));
    e->device_bytes += 2 * amp_bytes + sizeof(double) * 2 * e->nb;
    if (e->max_rows) {
        SHS_CUDA(cudaMalloc(&e->head, sizeof(double) * 2 * 256 * e->max_rows));
        SHS_CUDA(cudaMalloc(&e->tail, sizeof(double) * 2 * e->max_rows));
        e->device_bytes += sizeof(double) * 2 * 257 * e->max_rows;
    }
    return SHS_OK;
}

int state_init(shs_engine* e) {
    e->e1 = true;  // sel = e_1 implicitly: no memset of the N-amplitude buffer
    e->inv = 1.0;
    e->pending = false;
    return SHS_OK;
}

int stage_probs(shs_engine* e, uint32_t s, u128 prefix, double* p0, double* p1) {
    if (s >= e->t) return set_error(SHS_INVALID_ARGUMENT, "stage index out of range");
    int rc = ensure_buffers(e);
    if (rc) return rc;
    const double phi = stage_phase(s, prefix);
    const bool gather = e->a_pows[s] != 1;
    e->sc.w0r = e->w[0];
    e->sc.w0i = e->w[1];
    e->sc.w1r = e->w[2];
    e->sc.w1i = e->w[3];
    e->sc.phr = 1.0 * std::cos(phi);  // std::polar(1.0, phi), statevector.cpp:338
    e->sc.phi = 1.0 * std::sin(phi);
    e->sc.inv = e->inv;
    e->sc.phase_mul = (gather || phi != 0.0) ? 1 : 0;
    e->ps = s;
    int nparts = grid_for(e);
    if (e->plans[s].tiled && !e->e1) {
        TileParams tp = tile_params_for(e, s);
        const int g1 = static_cast<int>(std::min<uint64_t>(tp.ntiles, e->tiled_cap));
        const int g2 = static_cast<int>(
            std::min<uint64_t>((2 * tp.H + 255) / 256, static_cast<uint64_t>(e->fixup_cap)));
        rc = launch(e, 0, [&] {
            k_tiled<true><<<g1, tile_threads<true>(), tile_smem_bytes<true>(), e->stream>>>(tp);
            k_tile_fixup<<<g2, 256, 0, e->stream>>>(tp, e->partials + uint64_t(g1) * 2 * kDigits);
        });
        nparts = g1 + g2;
    } else {
        StageParams p = params_for(e, s);
        rc = launch(e, 0, [&] {
            if (gather) {
                if (e->e1) launch_probs<true, true>(e, p);
                else launch_probs<true, false>(e, p);
            } else {
                if (e->e1) launch_probs<false, true>(e, p);
                else launch_probs<false, false>(e, p);
            }
        });
    }
    if (rc) return rc;
    rc = launch(e, 1, [&] {
        k_finalize<<<1, 128, 0, e->stream>>>(e->partials, nparts, e->S, e->nb, e->kahan ? 1 : 0,
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
    if (p_src < kDegenerateMass)  // statevector.cpp:388-390 / 265-266
        return set_error(SHS_DEGENERATE_BRANCH,
                         "impossible measurement branch at stage " + std::to_string(e->ps));
    const bool gather = e->a_pows[e->ps] != 1;
    int rc;
    if (e->plans[e->ps].tiled && !e->e1) {
        TileParams tp = tile_params_for(e, e->ps);
        tp.sel = src_group;
        const int g1 = static_cast<int>(std::min<uint64_t>(tp.ntiles, e->tiled_cap));
        rc = launch(e, 2, [&] {
            k_tiled<false><<<g1, tile_threads<false>(), tile_smem_bytes<false>(), e->stream>>>(tp);
        });
    } else {
        StageParams p = params_for(e, e->ps);
        p.sel = src_group;
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
    std::swap(e->X, e->Y);
    e->e1 = false;
    e->inv = 1.0 / std::sqrt(p_src);  // statevector.cpp:391
    e->pending = false;
    if (wait) return sync(e);
    return SHS_OK;
}

int engine_run(shs_engine* e, u64 seed, u64 idx, u128* j_out, u128* js_out,
               shs_stage_trace* trace) {
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
}

const char* shs_last_error(void) { return g_last_error.c_str(); }

const char* shs_build_info(void) {
    return "shorsim_b200: sm_100a, fp64 no-FMA (--fmad=false), nvcc " SHS_NVCC_VERSION;
}

int shs_engine_create(const shs_problem* problem, const shs_error* error,
                      const shs_options* options, shs_engine** out) {
    if (!problem || !error || !out) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    shs_options o;
    if (options) o = *options;
    else shs_default_options(&o);
    int rc = engine_validate(*problem, *error, o);
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
                                   make_tile_plan(e->a_pows[s], e->a_invs[s], e->N, o.tiling));
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
    cudaDeviceProp prop;
    ce = cudaGetDeviceProperties(&prop, e->dev);
    if (ce != cudaSuccess) return fail(ce, "cudaGetDeviceProperties");
    if (prop.major < 10) {
        release(e);
        return set_error(SHS_CUDA_ERROR, "device is not sm_100-class (B200 required)");
    }
    e->num_sms = prop.multiProcessorCount;
    int occ = 0;
    ce = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stage_probs<true, false>, kThreads, 0);
    if (ce != cudaSuccess) return fail(ce, "occupancy");
    e->grid_cap = std::max(1, occ) * e->num_sms;
    // one persistent TMA-pipelined CTA per SM for the tiled passes
    ce = cudaFuncSetAttribute(k_tiled<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(tile_smem_bytes<true>()));
    if (ce != cudaSuccess) return fail(ce, "cudaFuncSetAttribute(k_tiled<probs>)");
    ce = cudaFuncSetAttribute(k_tiled<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(tile_smem_bytes<false>()));
    if (ce != cudaSuccess) return fail(ce, "cudaFuncSetAttribute(k_tiled<collapse>)");
    e->tiled_cap = e->num_sms;
    e->fixup_cap = 2 * e->num_sms;
    ce = cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking);
    if (ce != cudaSuccess) return fail(ce, "cudaStreamCreate");
    const size_t part_bytes = sizeof(unsigned long long) * 2 * kDigits *
                              std::max(e->grid_cap, e->tiled_cap + e->fixup_cap);
    if ((ce = cudaMalloc(&e->partials, part_bytes)) != cudaSuccess)
        return fail(ce, "cudaMalloc(partials)");
    if ((ce = cudaMalloc(&e->d_out, 4 * sizeof(double))) != cudaSuccess)
        return fail(ce, "cudaMalloc(out)");
    if ((ce = cudaHostAlloc(&e->h_out, 4 * sizeof(double), cudaHostAllocDefault)) != cudaSuccess)
        return fail(ce, "cudaHostAlloc");
    e->device_bytes = part_bytes + 32;  // the N-amplitude buffers come with the first stage
    state_init(e);
    *out = e;
    return SHS_OK;
}

void shs_engine_destroy(shs_engine* e) { release(e); }

uint32_t shs_engine_stages(const shs_engine* e) { return e ? e->t : 0; }

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

int shs_engine_run_batch(shs_engine* e, uint64_t seed, uint64_t idx0, uint32_t count,
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
    return guarded(e, [&] { return state_init(e); });
}

int shs_stage_probs(shs_engine* e, uint32_t s, uint64_t lo, uint64_t hi, double* p0, double* p1) {
    return guarded(e, [&] { return stage_probs(e, s, (u128{hi} << 64) | lo, p0, p1); });
}

int shs_stage_collapse(shs_engine* e, int32_t src_group, double p_source) {
    return guarded(e, [&] { return stage_collapse(e, src_group, p_source, true); });
}

int shs_stage_read(shs_engine* e, int32_t x, uint64_t first, uint64_t count, double* host) {
    return guarded(e, [&]() -> int {
        if (!e->pending) return set_error(SHS_INVALID_ARGUMENT, "no pending stage");
        if (count == 0) return SHS_OK;
        double2* d = nullptr;
        SHS_CUDA(cudaMallocAsync(&d, sizeof(double2) * count, e->stream));
        StageParams p = params_for(e, e->ps);
        const bool gather = e->a_pows[e->ps] != 1;
        const int grid = static_cast<int>(std::min<uint64_t>((count + 255) / 256, 4096));
        int rc = launch(e, -1, [&] {
            if (gather) {
                if (e->e1) k_stage_read<true, true><<<grid, 256, 0, e->stream>>>(p, x, first, count, d);
                else k_stage_read<true, false><<<grid, 256, 0, e->stream>>>(p, x, first, count, d);
            } else {
                if (e->e1) k_stage_read<false, true><<<grid, 256, 0, e->stream>>>(p, x, first, count, d);
                else k_stage_read<false, false><<<grid, 256, 0, e->stream>>>(p, x, first, count, d);
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
        if (!e->e1 && !e->X) return set_error(SHS_INVALID_ARGUMENT, "no state");
        if (count == 0) return SHS_OK;
        double2* d = nullptr;
        SHS_CUDA(cudaMallocAsync(&d, sizeof(double2) * count, e->stream));
        const int grid = static_cast<int>(std::min<uint64_t>((count + 255) / 256, 4096));
        const double wr = e->w[2 * x], wi = e->w[2 * x + 1];
        int rc = launch(e, -1, [&] {
            if (e->e1) k_state_read<true><<<grid, 256, 0, e->stream>>>(e->X, e->N, wr, wi, e->inv, first, count, d);
            else k_state_read<false><<<grid, 256, 0, e->stream>>>(e->X, e->N, wr, wi, e->inv, first, count, d);
        });
        if (rc) return rc;
        SHS_CUDA(cudaMemcpyAsync(host, d, sizeof(double2) * count, cudaMemcpyDeviceToHost,
                                 e->stream));
        SHS_CUDA(cudaFreeAsync(d, e->stream));
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

uint64_t shs_engine_launch_count(const shs_engine* e) { return e ? e->launches : 0; }

uint64_t shs_engine_device_bytes(const shs_engine* e) { return e ? e->device_bytes : 0; }

}  // extern "C"
