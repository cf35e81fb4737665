// Lockstep multi-shot runs for mid-size N (§8 f1 beyond the shared-memory
// batch engine): the shots of run_problem (harness.cpp:128-147) advance stage
// by stage together, one state per shot in HBM, blockIdx.y = shot. Per stage:
//   k_lock_probs     |h|^2 of every z of every shot, in-order 256-block sums
//                    (the reference's, statevector.cpp:353-371), exact digits
//   k_lock_measure   p0/p1 per shot (sequential Kahan or exact, as the single
//                    engine), the shot's measurement on the device (measure.cuh),
//                    its collapse group and next-stage scalars (the phase picked
//                    from the host's two candidates by the observed bit)
//   k_lock_collapse  the kept group of every shot
// Arithmetic, block partials and combine are the single engine's, so every
// shot's bits and p1 trace equal engine.run(seed, idx) for that shot; the host
// is one stage behind, supplying 2 candidate phases per shot (glibc cos/sin).
#pragma once

#include "device_math.cuh"
#include "measure.cuh"
#include "stage_kernels.cuh"

namespace shs {

struct LockParams {
    double2* X;          // [B][N] sel of each shot
    double2* Y;          // [B][N] collapse output
    uint64_t N, nb, nchunks;
    uint64_t m, m_sh, m_step;  // stage multiplier's inverse (gather) and Shoup companion
    int gather;          // A != 1
    int e1;              // stage 0: the implicit e_1 (sc0 for every shot)
    StageScalars sc0;
    DevStage* slots;     // [B][2]
    int cur;             // slot s & 1
    double* S;           // [B][2][nb] block partials
    unsigned long long* partials;  // [B][gridDim.x][2][kDigits]
    int spec;            // k_lock_probs_ws also stores h0 into Y; the collapse of a
                         // shot that keeps group 0 then has nothing to write
};

__device__ __forceinline__ StageScalars lock_scalars(const LockParams& p, uint32_t shot) {
    return p.e1 ? p.sc0 : p.slots[2 * shot + p.cur].sc;
}

// (sel[z], sel[src z]) of the thread's kPer elements zg + e*kBlock, all 2 kPer
// loads issued before any is used (one round trip per chunk instead of kPer:
// collapse 128 -> 122 us per N = 2^18 stage of 64 shots; the probs pass keeps
// its per-element loads — batched, its 120 registers cost occupancy and it ran
// 168 -> 182-199 us). Stage 0 synthesises e_1. Zero beyond N.
__device__ __forceinline__ void lock_load(const LockParams& p, const double2* __restrict__ X,
                                          uint64_t zg, double2 (&xa)[kPer], double2 (&xs)[kPer]) {
    uint64_t src[kPer];
    src[0] = p.gather ? mulmod_shoup(zg, p.m, p.m_sh, p.N) : zg;
#pragma unroll
    for (int e = 1; e < kPer; ++e)
        src[e] = p.gather ? addmod(src[e - 1], p.m_step, p.N) : src[e - 1] + kBlock;
    if (p.e1) {
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const uint64_t z = zg + uint64_t(e) * kBlock;
            xa[e] = make_double2(z < p.N && z == 1 ? 1.0 : 0.0, 0.0);
            xs[e] = make_double2(z < p.N && src[e] == 1 ? 1.0 : 0.0, 0.0);
        }
        return;
    }
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
        const uint64_t z = zg + uint64_t(e) * kBlock;
        const bool in = z < p.N;
        xa[e] = in ? __ldg(X + z) : make_double2(0.0, 0.0);
        xs[e] = in ? __ldg(X + src[e]) : make_double2(0.0, 0.0);
    }
}

static __global__ void __launch_bounds__(kThreads) k_lock_probs(LockParams p) {
    __shared__ double nrm[2 * kPer][kBlock + 1];
    __shared__ unsigned long long digits[2][kDigits];
    const uint32_t shot = blockIdx.y;
    const int tid = threadIdx.x;
    const double2* X = p.X + uint64_t(shot) * p.N;
    double* S = p.S + uint64_t(shot) * 2 * p.nb;
    const StageScalars sc = lock_scalars(p, shot);
    for (int i = tid; i < 2 * kDigits; i += kThreads) (&digits[0][0])[i] = 0ull;
    DigitWindow win;
    window_reset(win);
    __syncthreads();
    for (uint64_t c = blockIdx.x; c < p.nchunks; c += gridDim.x) {
        const uint64_t zg = c * kChunk + tid;
        uint64_t src = p.gather ? mulmod_shoup(zg, p.m, p.m_sh, p.N) : zg;
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const uint64_t z = zg + uint64_t(e) * kBlock;
            double2 xa = make_double2(0.0, 0.0), xs = xa;
            if (z < p.N) {
                if (p.e1) {
                    xa = make_double2(z == 1 ? 1.0 : 0.0, 0.0);
                    xs = make_double2(src == 1 ? 1.0 : 0.0, 0.0);
                } else {
                    xa = X[z];
                    xs = X[src];
                }
            }
            double h0r, h0i, h1r, h1i;
            stage_pair(sc, xa, xs, h0r, h0i, h1r, h1i);
            nrm[e][tid] = z < p.N ? cnorm(h0r, h0i) : 0.0;
            nrm[kPer + e][tid] = z < p.N ? cnorm(h1r, h1i) : 0.0;
            if (p.gather) src = addmod(src, p.m_step, p.N);
            else src += kBlock;
        }
        __syncthreads();
        if (tid < 2 * kPer) {  // one lane per (block, group): in-order block sum
            double s = 0.0;
#pragma unroll 16
            for (int i = 0; i < kBlock; ++i) s = __dadd_rn(s, nrm[tid][i]);
            const uint64_t b = c * kPer + (tid & (kPer - 1));
            const int g = tid / kPer;
            if (b < p.nb) {
                S[g * p.nb + b] = s;
                window_add(win, s, digits[g]);
            }
        }
        __syncthreads();
    }
    if (tid < 2 * kPer) window_flush(win, digits[tid / kPer]);
    __syncthreads();
    write_cta_digits(digits,
                     p.partials + (uint64_t(shot) * gridDim.x + blockIdx.x) * 2 * kDigits, tid);
}

// k_lock_probs, warp-specialized: 8 load warps produce a chunk's |h|^2 into one
// of two norm buffers while the chain warp folds the previous chunk's 16
// in-order block sums (the 256 dependent DADDs per block no longer stall the
// loads; in k_lock_probs every warp waits for them at the CTA barrier). Same
// arithmetic and fold order, so S and the digits are identical. Each CTA walks
// kLockWsChunks chunks of one shot (blockIdx.x + k gridDim.x), so the grid stays
// shot-major. Dynamic shared memory: kLockWsSmem.
constexpr int kLockWsLoadThreads = kThreads;                  // 8 load warps
constexpr int kLockWsThreads = kLockWsLoadThreads + 32;       // + the chain warp
constexpr int kLockWsChunks = 4;                              // chunks per CTA
constexpr size_t kLockWsSmem = sizeof(double) * 2 * (2 * kPer) * (kBlock + 1);
constexpr int kLockFull0 = 1, kLockEmpty0 = 3;                // named barriers (+ buffer)

__device__ __forceinline__ void lock_bar_sync(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kLockWsThreads) : "memory");
}
__device__ __forceinline__ void lock_bar_arrive(int id) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(kLockWsThreads) : "memory");
}

static __global__ void __launch_bounds__(kLockWsThreads, 2) k_lock_probs_ws(LockParams p) {
    extern __shared__ double lock_nrm[];  // [2][2 kPer][kBlock + 1]
    __shared__ unsigned long long digits[2][kDigits];
    const uint32_t shot = blockIdx.y;
    const int tid = threadIdx.x;
    const double2* X = p.X + uint64_t(shot) * p.N;
    double2* Ys = p.Y + uint64_t(shot) * p.N;
    for (int i = tid; i < 2 * kDigits; i += kLockWsThreads) (&digits[0][0])[i] = 0ull;
    __syncthreads();
    constexpr int kRow = kBlock + 1, kBuf = 2 * kPer * kRow;
    if (tid < kLockWsLoadThreads) {
        const StageScalars sc = lock_scalars(p, shot);
        int i = 0;
        for (uint64_t c = blockIdx.x; c < p.nchunks; c += gridDim.x, ++i) {
            const int buf = i & 1;
            double* nrm = lock_nrm + buf * kBuf;
            const uint64_t zg = c * kChunk + tid;
            double n0[kPer], n1[kPer];
            {
                double2 xa[kPer], xs[kPer];
                lock_load(p, X, zg, xa, xs);
#pragma unroll
                for (int e = 0; e < kPer; ++e) {
                    const uint64_t z = zg + uint64_t(e) * kBlock;
                    double h0r, h0i, h1r, h1i;
                    stage_pair(sc, xa[e], xs[e], h0r, h0i, h1r, h1i);
                    n0[e] = z < p.N ? cnorm(h0r, h0i) : 0.0;
                    n1[e] = z < p.N ? cnorm(h1r, h1i) : 0.0;
                    if (p.spec && z < p.N) Ys[z] = make_double2(h0r, h0i);
                }
            }
            if (i >= 2) lock_bar_sync(kLockEmpty0 + buf);  // the chain warp is done with it
#pragma unroll
            for (int e = 0; e < kPer; ++e) {
                nrm[e * kRow + tid] = n0[e];
                nrm[(kPer + e) * kRow + tid] = n1[e];
            }
            lock_bar_arrive(kLockFull0 + buf);
        }
    } else {
        const int lane = tid - kLockWsLoadThreads;
        double* S = p.S + uint64_t(shot) * 2 * p.nb;
        DigitWindow win;
        window_reset(win);
        int i = 0;
        for (uint64_t c = blockIdx.x; c < p.nchunks; c += gridDim.x, ++i) {
            const int buf = i & 1;
            lock_bar_sync(kLockFull0 + buf);
            if (lane < 2 * kPer) {  // one lane per (block, group): in-order block sum
                const double* row = lock_nrm + buf * kBuf + lane * kRow;
                double s = 0.0;
#pragma unroll 16
                for (int k = 0; k < kBlock; ++k) s = __dadd_rn(s, row[k]);
                const uint64_t b = c * kPer + (lane & (kPer - 1));
                const int g = lane / kPer;
                if (b < p.nb) {
                    S[g * p.nb + b] = s;
                    window_add(win, s, digits[g]);
                }
            }
            __syncwarp();
            // release the buffer only if the load warps will wait for it
            if (c + 2 * uint64_t(gridDim.x) < p.nchunks) lock_bar_arrive(kLockEmpty0 + buf);
        }
        if (lane < 2 * kPer) window_flush(win, digits[lane / kPer]);
    }
    __syncthreads();
    write_cta_digits(digits,
                     p.partials + (uint64_t(shot) * gridDim.x + blockIdx.x) * 2 * kDigits, tid);
}

struct LockMeasure {
    uint64_t seed, idx0;
    int kind;
    double delta, px, py;
    int check_norms;
    uint32_t s, t;
    int collapse;        // s + 1 < t
    int kahan;
    int nparts;          // CTAs per shot of k_lock_probs
    const NextPhase* nph;  // [B] candidates of stage s + 1
    StageRec* rec;       // [B][t] (host-mapped)
};

static __global__ void __launch_bounds__(kFinalizeThreads) k_lock_measure(LockParams p, LockMeasure q) {
    __shared__ unsigned long long acc[2][kDigits];
    __shared__ double pp[2];
    const uint32_t shot = blockIdx.x;
    const double* S = p.S + uint64_t(shot) * 2 * p.nb;
    if (q.kahan) {
        kahan_combine(S, p.nb, pp);  // combine_blocks, statevector.cpp:32-40
    } else {
        sum_slots(p.partials + uint64_t(shot) * q.nparts * 2 * kDigits, q.nparts, acc);
        if (threadIdx.x < 2) pp[threadIdx.x] = digits_to_double(acc[threadIdx.x]);
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const double p0 = pp[0], p1 = pp[1];
    MeasureCfg mc{q.seed, static_cast<uint32_t>(q.idx0 + shot), q.kind, q.delta, q.px, q.py,
                  q.check_norms};
    const DevMeasure mr = measure_dev(p0, p1, mc, q.s, q.collapse != 0);
    DevStage* cur = p.slots + 2 * shot + p.cur;
    DevStage* nxt = p.slots + 2 * shot + (p.cur ^ 1);
    StageScalars n = p.e1 ? p.sc0 : cur->sc;
    if (p.e1) cur->sc = p.sc0;
    cur->sel = mr.src_group;
    const NextPhase& ph = q.nph[shot];
    n.phr = ph.phr[mr.obit];
    n.phi = ph.phi[mr.obit];
    n.phase_mul = ph.phase_mul[mr.obit];
    n.inv = mr.status ? 0.0 : __ddiv_rn(1.0, __dsqrt_rn(mr.p_src));
    nxt->sc = n;
    StageRec r;
    r.p0 = p0;
    r.p1 = p1;
    r.sbit = mr.sbit;
    r.obit = mr.obit;
    r.flip = mr.flip;
    r.ebranch = mr.ebranch;
    r.status = mr.status;
    r.done = 1;
    q.rec[uint64_t(shot) * q.t + q.s] = r;
}

static __global__ void __launch_bounds__(kThreads) k_lock_collapse(LockParams p) {
    const uint32_t shot = blockIdx.y;
    const double2* X = p.X + uint64_t(shot) * p.N;
    double2* Y = p.Y + uint64_t(shot) * p.N;
    const DevStage* cur = p.slots + 2 * shot + p.cur;
    const StageScalars sc = cur->sc;  // stage 0: k_lock_measure stored sc0 there
    const int sel = cur->sel;
    if (p.spec && sel == 0) return;  // Y already holds this shot's h0
    for (uint64_t c = blockIdx.x; c < p.nchunks; c += gridDim.x) {
        const uint64_t zg = c * kChunk + threadIdx.x;
        double2 xa[kPer], xs[kPer];
        lock_load(p, X, zg, xa, xs);
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const uint64_t z = zg + uint64_t(e) * kBlock;
            if (z < p.N) {
                double h0r, h0i, h1r, h1i;
                stage_pair(sc, xa[e], xs[e], h0r, h0i, h1r, h1i);
                Y[z] = sel ? make_double2(h1r, h1i) : make_double2(h0r, h0i);
            }
        }
    }
}

}  // namespace shs
