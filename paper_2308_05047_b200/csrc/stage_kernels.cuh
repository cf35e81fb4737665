// Direct (untiled) stage kernels, shared by the single-GPU engine (engine.cu)
// and the sharded engine (shard.cu).
//
// Each kernel walks amplitude indices z in [z0, zend) — the whole of Z_N for the
// single engine, one shard for the sharded engine — in chunks of kChunk (8
// reduction blocks), with local buffer offsets z - z0 (z0 is a multiple of 256,
// so the reference's fixed 256-blocks never straddle a shard). The gathered
// side of the permutation comes from one of three sources:
//   kSrcGather  sel[src z], src z = a_inv * z mod N (Shoup once per thread, then
//               add / conditional subtract) — single engine only (z0 = 0)
//   kSrcDirect  sel[z] itself (identity stage: a_pow = 1)
//   kSrcBuffer  P[z - z0], the value a separate exchange already gathered
//   kSrcStreams small multipliers A (the last stages: a, a^2, a^4 ...): with
//               z = A q + r, src z = q + r a_inv mod N, so a chunk's gathered
//               side is A contiguous runs (one per residue r); they are staged
//               through shared memory with coalesced loads instead of one
//               scattered 16 B request per amplitude — single engine only
// and kE1 replaces sel by the implicit run start e_1 (no memory traffic).
#pragma once

#include "device_math.cuh"
#include "measure.cuh"

namespace shs {

enum SrcMode : int { kSrcGather = 0, kSrcDirect = 1, kSrcBuffer = 2, kSrcStreams = 3 };

constexpr uint32_t kStreamsMaxA = 1024;  // kSrcStreams: A <= this (<= 80 KB staged per CTA)

struct StageParams {
    const double2* X;   // sel over [z0, zend), local index z - z0
    const double2* Xs;  // kSrcBuffer: gathered values, local index z - z0
    double2* Y;         // collapse output, local index z - z0 (may alias Xs)
    uint64_t N, z0, zend;
    uint64_t m;       // a_inv of the stage
    uint64_t m_sh;    // Shoup companion of m
    uint64_t m_step;  // kBlock * m mod N: source advance per thread element
    StageScalars sc;
    double* S;        // local block partials: S0 [0, nb), S1 [nb, 2 nb)
    uint64_t nb;
    unsigned long long* partials;  // [gridDim.x][2][kDigits]
    uint64_t nchunks;
    int sel;          // collapse: group kept
    // kSrcStreams: the stage multiplier A, the staged run stride W (odd: the
    // residue-major reads are bank-conflict free), 1/A and 1/W for small divisions
    uint32_t A, W;
    float invA, invW;
    const DevStage* dev;  // device-resident run: sc / sel from this slot instead
    int spec;             // single engine: the probs pass also stores h0 into Y, and
                          // the collapse that keeps group 0 has nothing to write
};

// floor(d / D) for d < 2^20, D <= 2^11, from a float reciprocal and one correction
__device__ __forceinline__ uint32_t small_div(uint32_t d, uint32_t D, float invD) {
    uint32_t q = __float2uint_rz(__fmul_rn(__uint2float_rn(d) + 0.5f, invD));
    if (q * D > d) --q;
    else if ((q + 1) * D <= d) ++q;
    return q;
}


// amplitude at GLOBAL index z; under kE1 the run-start state e_1 (inv = 1)
template <bool kE1>
__device__ __forceinline__ double2 load_amp(const double2* __restrict__ X, uint64_t z,
                                            uint64_t z0) {
    if (kE1) return make_double2(z == 1 ? 1.0 : 0.0, 0.0);
    return __ldg(X + (z - z0));
}

// kSrcStreams: stage the gathered side of chunk c, buf[r * W + w] = sel[src z]
// for z = A (q_lo + w) + r in the chunk (q_lo = floor(chunk start / A)).
// Returns rho = chunk start mod A once this thread's copies have landed; callers
// fence buf with __syncthreads().
template <bool kE1>
__device__ __forceinline__ uint32_t stage_streams(const StageParams& p, uint64_t c,
                                                  double2* __restrict__ buf) {
    const uint64_t zc = c * kChunk;
    const uint64_t q_lo = zc / p.A;
    const uint32_t rho = static_cast<uint32_t>(zc - q_lo * p.A);
    const uint32_t nf = p.A * p.W;
    for (uint32_t f = threadIdx.x; f < nf; f += kThreads) {
        const uint32_t r = small_div(f, p.W, p.invW);
        const uint32_t w = f - r * p.W;
        const uint32_t d = w * p.A + r;  // z - zc + rho
        if (d >= rho && d - rho < kChunk && zc + (d - rho) < p.zend) {
            uint64_t src = mulmod_shoup(r, p.m, p.m_sh, p.N) + q_lo + w;
            if (src >= p.N) src -= p.N;
            if (kE1) {
                buf[f] = load_amp<kE1>(p.X, src, 0);
            } else {  // asynchronous 16 B copy (LDGSTS): the loop never waits on DRAM
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                 static_cast<uint32_t>(__cvta_generic_to_shared(buf + f))),
                             "l"(p.X + src)
                             : "memory");
            }
        }
    }
    if (!kE1) asm volatile("cp.async.wait_all;" ::: "memory");
    return rho;
}

// (sel[z], gathered[z]) for the kPer elements zg + e*kBlock of one thread
template <int kMode, bool kE1>
__device__ __forceinline__ void load_pairs(const StageParams& p, uint64_t zg, double2 (&xa)[kPer],
                                           double2 (&xs)[kPer]) {
    uint64_t src = kMode == kSrcGather ? mulmod_shoup(zg, p.m, p.m_sh, p.N) : 0;
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
        const uint64_t z = zg + uint64_t(e) * kBlock;
        if (z < p.zend) {
            xa[e] = load_amp<kE1>(p.X, z, p.z0);
            if (kMode == kSrcGather) xs[e] = load_amp<kE1>(p.X, src, p.z0);
            else if (kMode == kSrcBuffer) xs[e] = p.Xs[z - p.z0];
            else if (kMode == kSrcStreams) xs[e] = xa[e];  // replaced from the staged runs
            else xs[e] = xa[e];
        } else {
            xa[e] = make_double2(0.0, 0.0);
            xs[e] = xa[e];
        }
        if (kMode == kSrcGather) src = addmod(src, p.m_step, p.N);
    }
}

// kSrcStreams: the gathered values of this thread's kPer elements from the staged runs
__device__ __forceinline__ void read_streams(const StageParams& p, uint32_t rho,
                                             const double2* __restrict__ buf,
                                             double2 (&xs)[kPer]) {
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
        const uint32_t d = rho + threadIdx.x + e * kBlock;
        const uint32_t w = small_div(d, p.A, p.invA);
        const uint32_t r = d - w * p.A;
        xs[e] = buf[r * p.W + w];
    }
}

__device__ __forceinline__ void write_cta_digits(unsigned long long (*digits)[kDigits],
                                                 unsigned long long* out_slot, int tid) {
    if (tid < 2) {
        unsigned long long carry = 0;
        unsigned long long* out = out_slot + tid * kDigits;
        for (int i = 0; i < kDigits; ++i) {
            unsigned long long v = digits[tid][i] + carry;
            out[i] = v & 0xffffffffull;
            carry = v >> 32;
        }
    }
}

// kDev: the stage scalars come from p.dev (device-resident runs), staged in
// shared memory and read at every use (volatile); otherwise they are the kernel
// arguments p.sc, read as constant-bank operands. (Holding device-loaded
// scalars in registers makes ptxas give up the batching of the 2 kPer loads
// for occupancy: +25% on the gather stages.)
template <int kMode, bool kE1, bool kDev>
__global__ void __launch_bounds__(kThreads) k_stage_probs(StageParams p) {
    extern __shared__ double2 streams_buf[];      // kSrcStreams: [A][W]
    __shared__ double nrm[2 * kPer][kBlock + 1];  // +1: conflict-free column walks
    __shared__ unsigned long long digits[2][kDigits];
    __shared__ StageScalars s_sc;
    const int tid = threadIdx.x;
    for (int i = tid; i < 2 * kDigits; i += kThreads) (&digits[0][0])[i] = 0ull;
    if (kDev && tid == 0) s_sc = p.dev->sc;
    const volatile StageScalars& dsc = s_sc;
    DigitWindow win;
    window_reset(win);
    __syncthreads();

    for (uint64_t c = blockIdx.x; c < p.nchunks; c += gridDim.x) {
        const uint64_t zg = p.z0 + c * kChunk + tid;
        double2 xa[kPer], xs[kPer];
        uint32_t rho = 0;
        if (kMode == kSrcStreams) rho = stage_streams<kE1>(p, c, streams_buf);
        load_pairs<kMode, kE1>(p, zg, xa, xs);
        if (kMode == kSrcStreams) {
            __syncthreads();  // staged runs complete (the previous chunk's reads ended
                              // before its fold barrier)
            read_streams(p, rho, streams_buf, xs);
        }
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            double h0r, h0i, h1r, h1i;
            if (kDev) stage_pair(dsc, xa[e], xs[e], h0r, h0i, h1r, h1i);
            else stage_pair(p.sc, xa[e], xs[e], h0r, h0i, h1r, h1i);
            const bool live = zg + uint64_t(e) * kBlock < p.zend;
            nrm[e][tid] = live ? cnorm(h0r, h0i) : 0.0;
            nrm[kPer + e][tid] = live ? cnorm(h1r, h1i) : 0.0;
            if (p.spec && live) p.Y[zg + uint64_t(e) * kBlock - p.z0] = make_double2(h0r, h0i);
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
    write_cta_digits(digits, p.partials + uint64_t(blockIdx.x) * 2 * kDigits, tid);
}

// Probs pass of stage 0, whose state is the run start e_1 (inv = 1): only
// z = 1 and z = A (src A = 1) carry amplitude, every other |h|^2 is +0.0, and
// adding +0.0 leaves the reference's in-order block sums unchanged. So the two
// live norms (and their sum when both fall in one 256-block, z = 1 first) are
// the block partials; the host zeroes S beforehand. One thread, one digit slot
// (slot 0): the 2 N amplitude-stages of work of the general kernel become O(1).
static __global__ void k_stage_probs_e1(StageParams p, uint64_t A) {
    __shared__ unsigned long long digits[2][kDigits];
    const int tid = threadIdx.x;
    for (int i = tid; i < 2 * kDigits; i += blockDim.x) (&digits[0][0])[i] = 0ull;
    __syncthreads();
    if (tid == 0) {
        const bool gather = A != 1;
        const uint64_t zs[2] = {1, A};
        const int nz = gather ? 2 : 1;  // z = 1 < z = A
        double nrm[2][2];
        for (int q = 0; q < nz; ++q) {
            const uint64_t z = zs[q];
            const uint64_t src = gather ? mulmod_shoup(z, p.m, p.m_sh, p.N) : z;
            const double2 xa = make_double2(z == 1 ? 1.0 : 0.0, 0.0);
            const double2 xs = make_double2(src == 1 ? 1.0 : 0.0, 0.0);
            double h0r, h0i, h1r, h1i;
            stage_pair(p.sc, xa, xs, h0r, h0i, h1r, h1i);
            nrm[q][0] = cnorm(h0r, h0i);
            nrm[q][1] = cnorm(h1r, h1i);
        }
        DigitWindow w0, w1;
        window_reset(w0);
        window_reset(w1);
        for (int g = 0; g < 2; ++g) {
            DigitWindow& w = g ? w1 : w0;
            const uint64_t b1 = zs[0] >> 8;
            if (nz == 2 && (zs[1] >> 8) == b1) {
                const double s = __dadd_rn(__dadd_rn(0.0, nrm[0][g]), nrm[1][g]);
                p.S[g * p.nb + b1] = s;
                window_add(w, s, digits[g]);
            } else {
                for (int q = 0; q < nz; ++q) {
                    const double s = __dadd_rn(0.0, nrm[q][g]);
                    p.S[g * p.nb + (zs[q] >> 8)] = s;
                    window_add(w, s, digits[g]);
                }
            }
            window_flush(w, digits[g]);
        }
    }
    __syncthreads();
    write_cta_digits(digits, p.partials, tid);
}

// p0/p1 from the stage. kahan: reference combine_blocks (statevector.cpp:32-40),
// two interleaved sequential chains, zeros skipped; else exact sum of partials.
constexpr int kFinalizeSlices = 12;
constexpr int kFinalizeThreads = 2 * kDigits * kFinalizeSlices;  // 960

// acc = the sum of the nparts per-CTA digit slots (carry-save). kFinalizeSlices x
// 80 threads: slice l sums slots l, l + kFinalizeSlices, ... (coalesced 640 B
// rows), then one thread per digit adds the slices. Ends with __syncthreads().
__device__ __forceinline__ void sum_slots(const unsigned long long* __restrict__ partials,
                                          int nparts, unsigned long long (*acc)[kDigits]) {
    __shared__ unsigned long long red[kFinalizeSlices][2 * kDigits];
    const int i = threadIdx.x % (2 * kDigits), l = threadIdx.x / (2 * kDigits);
    if (l < kFinalizeSlices) {
        unsigned long long s = 0;
#pragma unroll 8
        for (int c = l; c < nparts; c += kFinalizeSlices) s += partials[uint64_t(c) * 2 * kDigits + i];
        red[l][i] = s;
    }
    __syncthreads();
    if (threadIdx.x < 2 * kDigits) {
        unsigned long long s = 0;
        for (int k = 0; k < kFinalizeSlices; ++k) s += red[k][threadIdx.x];
        (&acc[0][0])[threadIdx.x] = s;
    }
    __syncthreads();
}

// combine_blocks (statevector.cpp:32-40) for both groups: sequential Kahan over
// the non-zero block partials in block order, bit-identical to the reference.
// Called by every thread of the CTA (>= 3 warps). Warps 2.. stage tiles of S
// into shared memory (coalesced, one tile ahead); lane 0 of warp g folds group
// g's chain from shared memory, so the two 4-DADD chains run side by side and
// no fold waits on a global load. pp[0] = p0, pp[1] = p1 on return (synced).
constexpr int kKahanTile = 512;
__device__ __forceinline__ void kahan_combine(const double* __restrict__ S, uint64_t nb,
                                              double* pp) {
    __shared__ double tile[2][2][kKahanTile];  // [buffer][group][block]
    const int g = threadIdx.x >> 5;
    const bool folder = g < 2 && (threadIdx.x & 31) == 0;
    const uint64_t ntiles = (nb + kKahanTile - 1) / kKahanTile;
    auto load = [&](uint64_t k) {
        if (threadIdx.x < 64) return;
        const uint64_t b0 = k * kKahanTile;
        for (int i = threadIdx.x - 64; i < 2 * kKahanTile; i += blockDim.x - 64) {
            const int gg = i / kKahanTile, j = i % kKahanTile;
            tile[k & 1][gg][j] = b0 + j < nb ? S[gg * nb + b0 + j] : 0.0;
        }
    };
    double s = 0.0, c = 0.0;
    load(0);
    __syncthreads();
    for (uint64_t k = 0; k < ntiles; ++k) {
        if (k + 1 < ntiles) load(k + 1);
        if (folder) {
            const double2* x = reinterpret_cast<const double2*>(tile[k & 1][g]);
            double2 cur[4], nxt[4];  // 8 partials in registers, the next 8 in flight
#pragma unroll
            for (int u = 0; u < 4; ++u) cur[u] = x[u];
#pragma unroll 1
            for (int i = 0; i < kKahanTile / 2; i += 4) {
#pragma unroll
                for (int u = 0; u < 4; ++u) nxt[u] = x[(i + 4 + u) % (kKahanTile / 2)];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const double v = (u & 1) ? cur[u >> 1].y : cur[u >> 1].x;
                    if (v != 0.0) {  // zero partials skipped (tile padding included)
                        const double y = __dsub_rn(v, c);
                        const double t = __dadd_rn(s, y);
                        c = __dsub_rn(__dsub_rn(t, s), y);
                        s = t;
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) cur[u] = nxt[u];
            }
        }
        __syncthreads();
    }
    if (folder) pp[g] = s;
    __syncthreads();
}

static __global__ void __launch_bounds__(kFinalizeThreads) k_finalize(const unsigned long long* __restrict__ partials, int nparts,
                           const double* __restrict__ S, uint64_t nb, int kahan,
                           double* __restrict__ out) {
    __shared__ unsigned long long acc[2][kDigits];
    if (kahan) {
        __shared__ double pp[2];
        kahan_combine(S, nb, pp);
        if (threadIdx.x < 2) out[threadIdx.x] = pp[threadIdx.x];
        return;
    }
    sum_slots(partials, nparts, acc);
    if (threadIdx.x < 2) out[threadIdx.x] = digits_to_double(acc[threadIdx.x]);
}

// Stage s of a device-resident run (engine.cu engine_run_device): p0/p1 as
// k_finalize, then the measurement on the device (measure.cuh), the collapse
// group into slot s & 1 and the next stage's scalars into slot (s + 1) & 1 —
// its phase picked from the host's two candidates by the observed bit, its inv
// = 1/sqrt(p_src) correctly rounded like the host's 1.0 / std::sqrt
// (statevector.cpp:391). A failed stage (norm drift, degenerate branch) zeroes
// the next inv so the stages the host already queued fold zeros until it
// reads the status one stage later and stops.
struct MeasureStep {
    MeasureCfg cfg;
    uint32_t s;
    int collapse;        // s + 1 < t
    int init_cur;        // stage 0: slot s & 1 takes sc0 (its probs pass used kernel args)
    StageScalars sc0;
    DevStage* cur;       // slot s & 1
    DevStage* next;      // slot (s + 1) & 1
    NextPhase nph;
    StageRec* rec;       // [t], host-mapped
};

// thread 0 of a finalize kernel, once p0/p1 are known
__device__ __forceinline__ void measure_step(double p0, double p1, const MeasureStep& ms) {
    const DevMeasure mr = measure_dev(p0, p1, ms.cfg, ms.s, ms.collapse != 0);
    StageScalars n = ms.init_cur ? ms.sc0 : ms.cur->sc;
    if (ms.init_cur) ms.cur->sc = ms.sc0;
    ms.cur->sel = mr.src_group;
    n.phr = ms.nph.phr[mr.obit];
    n.phi = ms.nph.phi[mr.obit];
    n.phase_mul = ms.nph.phase_mul[mr.obit];
    n.inv = mr.status ? 0.0 : __ddiv_rn(1.0, __dsqrt_rn(mr.p_src));
    ms.next->sc = n;
    StageRec r;
    r.p0 = p0;
    r.p1 = p1;
    r.sbit = mr.sbit;
    r.obit = mr.obit;
    r.flip = mr.flip;
    r.ebranch = mr.ebranch;
    r.status = mr.status;
    r.done = 1;
    ms.rec[ms.s] = r;
}

static __global__ void __launch_bounds__(kFinalizeThreads)
    k_finalize_measure(const unsigned long long* __restrict__ partials, int nparts,
                       const double* __restrict__ S, uint64_t nb, int kahan, MeasureStep ms) {
    __shared__ unsigned long long acc[2][kDigits];
    __shared__ double pp[2];
    // launched as a programmatic dependent of the fixup: wait for the partials;
    // the next stage's orbit kernel may be scheduled now (its plan warps start,
    // everything else in it waits for this grid: griddepcontrol.wait)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    if (kahan) {
        kahan_combine(S, nb, pp);
    } else {
        sum_slots(partials, nparts, acc);
        if (threadIdx.x < 2) pp[threadIdx.x] = digits_to_double(acc[threadIdx.x]);
    }
    __syncthreads();
    if (threadIdx.x == 0) measure_step(pp[0], pp[1], ms);
}

// Stage s of a device-resident SHARDED run (shard.cu): every shard's finalize
// sums the G shards' exact digit arrays (integers: order-independent, so every
// shard computes the same p0/p1 and the same measurement) read through peer
// pointers, then proceeds as k_finalize_measure for its own slots.
struct ShardDigits {
    const unsigned long long* d[16];  // shard q's carry-normalised digits [2][kDigits]
    int G;
};

// The G shards' block partials (each [2][nb_q], in shard = block order) copied
// into one [2][nb_total] array for the reference's sequential Kahan combine
// (kahan_combine) when a sharded engine combines like the reference (small N).
struct ShardPartials {
    const double* S[16];
    uint64_t off[17];  // first global block of shard q; off[G] = nb_total
    int G;
};

static __global__ void k_shard_gather_partials(ShardPartials sp, double* __restrict__ out) {
    const uint64_t nbt = sp.off[sp.G];
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < 2 * nbt;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t g = i / nbt, b = i - g * nbt;
        int q = 0;
        while (q + 1 < sp.G && sp.off[q + 1] <= b) ++q;
        const uint64_t nbq = sp.off[q + 1] - sp.off[q];
        out[i] = sp.S[q][g * nbq + (b - sp.off[q])];
    }
}

static __global__ void __launch_bounds__(2 * kDigits)
    k_shard_finalize_measure(ShardDigits sd, MeasureStep ms) {
    __shared__ unsigned long long acc[2][kDigits];
    __shared__ double pp[2];
    unsigned long long s = 0;
    for (int q = 0; q < sd.G; ++q) s += sd.d[q][threadIdx.x];
    (&acc[0][0])[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x < 2) pp[threadIdx.x] = digits_to_double(acc[threadIdx.x]);
    __syncthreads();
    if (threadIdx.x == 0) measure_step(pp[0], pp[1], ms);
}

// The exact digits of this engine's (or shard's) partial masses: sum of the
// per-CTA digit slots, carry-normalised to 32-bit digits (for an allreduce).
static __global__ void __launch_bounds__(kFinalizeThreads) k_sum_partials(const unsigned long long* __restrict__ partials, int nparts,
                               unsigned long long* __restrict__ out) {
    __shared__ unsigned long long acc[2][kDigits];
    sum_slots(partials, nparts, acc);
    if (threadIdx.x < 2) {
        unsigned long long carry = 0;
        for (int i = 0; i < kDigits; ++i) {
            unsigned long long v = acc[threadIdx.x][i] + carry;
            out[threadIdx.x * kDigits + i] = v & 0xffffffffull;
            carry = v >> 32;
        }
    }
}

template <int kMode, bool kE1, bool kDev>
__global__ void __launch_bounds__(kThreads) k_stage_collapse(StageParams p) {
    extern __shared__ double2 streams_buf[];  // kSrcStreams: [A][W]
    __shared__ StageScalars s_sc;             // kDev: as k_stage_probs
    __shared__ int s_sel;
    const int tid = threadIdx.x;
    if (kDev && tid == 0) {
        s_sc = p.dev->sc;
        s_sel = p.dev->sel;
    }
    if (kDev) __syncthreads();
    const volatile StageScalars& dsc = s_sc;
    const int sel = kDev ? s_sel : p.sel;
    if (p.spec && sel == 0) return;  // Y already holds h0 (speculative probs pass)
    for (uint64_t c = blockIdx.x; c < p.nchunks; c += gridDim.x) {
        const uint64_t zg = p.z0 + c * kChunk + tid;
        double2 xa[kPer], xs[kPer];
        uint32_t rho = 0;
        if (kMode == kSrcStreams) {
            __syncthreads();  // the previous chunk's reads of the staged runs ended
            rho = stage_streams<kE1>(p, c, streams_buf);
        }
        load_pairs<kMode, kE1>(p, zg, xa, xs);
        if (kMode == kSrcStreams) {
            __syncthreads();
            read_streams(p, rho, streams_buf, xs);
        }
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const uint64_t z = zg + uint64_t(e) * kBlock;
            double h0r, h0i, h1r, h1i;
            // stage 0 (kE1): the scalars are the host's even in a device-resident run
            if (kDev && !kE1) stage_pair(dsc, xa[e], xs[e], h0r, h0i, h1r, h1i);
            else stage_pair(p.sc, xa[e], xs[e], h0r, h0i, h1r, h1i);
            if (z < p.zend)
                p.Y[z - p.z0] = sel ? make_double2(h1r, h1i) : make_double2(h0r, h0i);
        }
    }
}

// Post-Hadamard amplitudes of group x for global y in [first, first + count).
template <int kMode, bool kE1>
__global__ void k_stage_read(StageParams p, int x, uint64_t first, uint64_t count,
                             double2* __restrict__ out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t z = first + i;
        if (z >= p.zend || z < p.z0) {
            out[i] = make_double2(0.0, 0.0);
            continue;
        }
        double2 xa = load_amp<kE1>(p.X, z, p.z0), xs;
        if (kMode == kSrcGather) xs = load_amp<kE1>(p.X, mulmod_shoup(z, p.m, p.m_sh, p.N), p.z0);
        else if (kMode == kSrcBuffer) xs = p.Xs[z - p.z0];
        else xs = xa;
        double h0r, h0i, h1r, h1i;
        stage_pair(p.sc, xa, xs, h0r, h0i, h1r, h1i);
        out[i] = x ? make_double2(h1r, h1i) : make_double2(h0r, h0i);
    }
}

// g_x[y] = w_x * (sel[y] * inv), the reference state after init / reset_top,
// for global y in [first, first + count) (zero outside [z0, zend)).
template <bool kE1>
__global__ void k_state_read(const double2* __restrict__ X, uint64_t z0, uint64_t zend, double wr,
                             double wi, double inv, uint64_t first, uint64_t count,
                             double2* __restrict__ out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t z = first + i;
        if (z >= zend || z < z0) {
            out[i] = make_double2(0.0, 0.0);
            continue;
        }
        double2 v = load_amp<kE1>(X, z, z0);
        double r, im;
        cmul(wr, wi, __dmul_rn(v.x, inv), __dmul_rn(v.y, inv), r, im);
        out[i] = make_double2(r, im);
    }
}

// k_state_read at arbitrary global indices idx[i] (the sparse-support parity
// check reads the 2^(s+1) support points of a dense state this way).
template <bool kE1>
__global__ void k_state_gather(const double2* __restrict__ X, uint64_t z0, uint64_t zend,
                               double wr, double wi, double inv,
                               const uint64_t* __restrict__ idx, uint64_t count,
                               double2* __restrict__ out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t z = idx[i];
        if (z >= zend || z < z0) {
            out[i] = make_double2(0.0, 0.0);
            continue;
        }
        double2 v = load_amp<kE1>(X, z, z0);
        double r, im;
        cmul(wr, wi, __dmul_rn(v.x, inv), __dmul_rn(v.y, inv), r, im);
        out[i] = make_double2(r, im);
    }
}

// The index map exactly as the gather kernels walk it (Shoup per thread, then
// incremental), written out for the bit-exact index-map parity check.
static __global__ void k_index_map(StageParams p, uint64_t chunk0, uint64_t nchunk, uint64_t first,
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

static __global__ void k_fill_identity(uint64_t first, uint64_t count, uint64_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = first + i;
}

}  // namespace shs
