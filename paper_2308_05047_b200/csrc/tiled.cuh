// Sorted-residue tiles for the modular-multiplication permutation,
// fed by asynchronous global->shared copies through an mbarrier ring.
//
// For the stage multiplier A (m = A^-1 mod N) and a row count H, the residues
// z_j = j*A mod N (j < H) split Z_N into H rows [z_j, z_j + g_j) and
//                      src(z_j + i) = (j + i*m) mod N.
// A chunk of kRows consecutive rows j and kCols consecutive columns i therefore
// reads the gathered side as kCols runs of kRows amplitudes and the direct side
// / output as kRows runs of kCols amplitudes: both HBM sides are whole-line and
// coalesced; the transpose happens in shared memory. 32 x 32 chunks (512 B
// runs on both sides) measured best on B200 (profiles/r01/README.md: 16 x 64,
// i.e. 256 B gathered runs, was 10% slower). By the three-distance theorem a row's length and its successor in z
// order need no sort: with u = argmin_{0<j<H} (jA mod N), v = argmax (jA mod N),
//   j + u < H : length du = uA mod N,       successor j + u
//   j >= v    : length dv = N - (vA mod N),  successor j - v
//   otherwise : length du + dv,              successor j + u - v.
//
// Work split (CtaWork): whole bands round-robin, then the remaining bands' chunks
// (kRows rows x kCols columns, band-major) cut into one contiguous range per CTA
// (host table `split`, balanced to within a chunk). Where a cut falls inside a
// band at column i, each row r is
// cut at its first 256-block boundary e_r >= i (or its end): the earlier CTA
// runs the row's columns [.., e_r), the later one [e_r, ..). So no block is
// folded by two CTAs except at row boundaries (k_tile_fixup), and any plan,
// even one with fewer bands than SMs, keeps every SM busy.
//
// CTA roles (one persistent CTA per SM):
//   producer warps     — 16-byte cp.async (LDGSTS) copies of the chunk's 64
//                        source-column runs and 16 row runs into a kStages-deep
//                        ring; each producer thread's copies complete on
//                        full[stage] via cp.async.mbarrier.arrive.noinc. (1D TMA
//                        bulk copies were measured slower here: ~80 requests of
//                        256 B - 1 KB per 32 KB chunk are TMA-issue bound.)
//   warps 0..7         — consumers: h0/h1 of 4 amplitudes per thread from shared
//                        memory; the probs pass writes |h|^2 to a double-buffered
//                        norm tile, the collapse pass stores sel'[z] (coalesced)
//   warp kChainWarp    — probs pass only: one lane per (row, group) folds the
//                        norms in z order into the fixed 256-block partials,
//                        bit-identical to proj/src/statevector.cpp:353-371, and
//                        into the CTA's exact accumulator; the block straddling
//                        two rows is finished by k_tile_fixup from the
//                        predecessor's tail partial and the row's stored head.
#pragma once

#include <type_traits>


#include "device_math.cuh"
#include "stage_kernels.cuh"
#include "orbit.cuh"

namespace shs {

#ifndef SHS_TILE_ROWS
#define SHS_TILE_ROWS 32
#endif
#ifndef SHS_TILE_COLS
#define SHS_TILE_COLS 32
#endif
#ifndef SHS_RING_STAGES
#define SHS_RING_STAGES 4
#endif
constexpr int kRows = SHS_TILE_ROWS;    // rows per tile (gathered-side run length)
constexpr int kCols = SHS_TILE_COLS;    // columns per chunk (direct-side run length)
constexpr int kStages = SHS_RING_STAGES;  // copy ring depth
constexpr int kConsumerWarps = 8;  // exchange kernels and the split tiled variant
constexpr int kConsumers = 32 * kConsumerWarps;
constexpr int kProducerWarps = 4;
constexpr int kProducers = 32 * kProducerWarps;
constexpr int kProducerWarp = kConsumerWarps;                   // warps 8..11
constexpr int kChainWarp = kConsumerWarps + kProducerWarps;     // first chain warp (probs only)
constexpr int kChainWarps = (2 * kRows + 31) / 32;              // one lane per (row, group)
constexpr int kCopiesPerProducer = kRows * kCols / kProducers;  // copies per side per chunk
constexpr int kDstRowStep = kProducers / kCols;                 // rows between a thread's copies
constexpr int kRowsPerConsumer = kRows * kCols / kConsumers;    // rows a consumer thread owns
constexpr int kNormSync = kConsumers + 32 * kChainWarps;        // named-barrier thread count
static_assert(kRows <= 64 && (kRows & (kRows - 1)) == 0, "kRows: power of two <= 64");
constexpr int kRowsPerLane = kRows > 32 ? kRows / 32 : 1;       // row bookkeeping per lane
static_assert(kCols <= 256 && kProducers % kCols == 0 && kConsumers % kCols == 0, "kCols");
// Consumer warps of k_tiled<., kSplit>: 16 for the round-robin whole-band
// variant (config 4: -2.3% per stage vs 8; more warps hide the shared-memory
// and FP64 latencies of the per-element math), 8 for the split variant (16 spill
// there and cost 15% at config 3).
#ifndef SHS_RR_CONSUMER_WARPS
#define SHS_RR_CONSUMER_WARPS 16
#endif
// The orbit variant (kOrb) runs 14 consumer warps (members only, each found by a
// search of its slot's row offsets).
#ifndef SHS_NORM_BUFS
#define SHS_NORM_BUFS 4
#endif
#ifndef SHS_ORB_PLAN_WARPS
#define SHS_ORB_PLAN_WARPS 2
#endif
#ifndef SHS_ORB_SLOTS
#define SHS_ORB_SLOTS 5
#endif
#ifndef SHS_ORB_NORM_BUFS
#define SHS_ORB_NORM_BUFS 2
#endif
#ifndef SHS_ORB_PRODUCER_WARPS
#define SHS_ORB_PRODUCER_WARPS 8
#endif
#ifndef SHS_ORB_CONSUMER_WARPS
#define SHS_ORB_CONSUMER_WARPS 6
#endif
template <bool kSplit, bool kOrb = false>
struct TileCfg {
    static constexpr int kCW = kOrb ? SHS_ORB_CONSUMER_WARPS : kSplit ? kConsumerWarps : SHS_RR_CONSUMER_WARPS;
    static constexpr int kCons = 32 * kCW;
    static constexpr int kPW = kOrb ? SHS_ORB_PRODUCER_WARPS : kProducerWarps;  // producer warps
    static_assert(kRows % kPW == 0 && kCols % kPW == 0, "producer warps split the rows / columns");
    static constexpr int kProds = 32 * kPW;
    static constexpr int kCopies = kRows * kCols / kProds;  // copies per side per producer
    static constexpr int kColStep = kProds / kRows;         // columns between a thread's copies
    static constexpr int kRowStep = kProds / kCols;         // rows between a thread's copies
    // orbit: 5 slots and 2 norm tiles (a compact norm tile holds a slot's norms;
    // the slots are what keeps bytes in flight)
    static constexpr int kST = kOrb ? SHS_ORB_SLOTS : kStages;
    static constexpr int kNB = kOrb ? SHS_ORB_NORM_BUFS : SHS_NORM_BUFS;
    static constexpr int kProdWarp = kCW;                   // first producer warp
    static constexpr int kChainWarp0 = kCW + kPW;           // first chain warp (probs only)
    static constexpr int kRowsPerCons = kRows * kCols / kCons;
    static constexpr int kNSync = kCons + 32 * kChainWarps;   // norm named-barrier thread count
    static_assert(kCons % kCols == 0 && kRowsPerCons >= 1, "consumer layout");
};
constexpr int kNormBufs = SHS_NORM_BUFS;           // norm tiles in flight (chain slack)
constexpr int kNormFull0 = 1, kNormEmpty0 = 1 + kNormBufs;  // named barrier ids
constexpr int kNrmStride = kCols + 2;              // 16 B-aligned rows, conflict-free LDS.128

struct TileParams {
    const double2* X;
    double2* Y;
    uint64_t N;
    uint64_t A, A_sh;   // z_j = j * A mod N
    uint64_t m, m_sh;   // src = j + i * m mod N
    uint64_t m_chunk;   // kCols * m mod N: source advance per chunk
    uint64_t H, u, v, du, dv;
    uint64_t ntiles;    // bands of kRows rows
    uint64_t bulk_rounds;  // whole bands per CTA, round-robin (CtaWork)
    unsigned long long* band_ctr;  // CtaWork<false>: bands handed out (monotonic over launches)
    uint64_t band_base;            // band_ctr at this launch
    const uint2* split;    // [gridDim.x + 1] (band, chunk): each CTA's remainder range
    StageScalars sc;
    double* S;          // block partials, S0 [0, nb), S1 [nb, 2nb)
    uint64_t nb;
    unsigned long long* partials;  // exact-accumulator slots, [slot][2][kDigits]
    double* head;       // [H][2][256] head norms of each row (before its first boundary)
    double* tail;       // [H][2]      predecessor's tail partial, indexed by successor row
    int sel;            // collapse: group kept
    // speculative group-0 write: the probs pass also stores h0 into Y (the
    // collapse of group 0 would write exactly those values), and the collapse
    // of a stage whose probs pass did so returns at once when group 0 is kept
    int spec;
    const DevStage* dev;  // device-resident run: sc / sel from this slot instead
    // orbit-compressed state (orbit.cuh, k_tiled<true, false, true>): the source
    // is slot X or X1 of a pair, picked by prev->sel (device-resident run) or
    // prev_sel; both groups are written, h0 to Y and h1 to Y1, at the members'
    // ranks unless `write` is 0 (the run's last stage); rec: the rank records
    const double2* X1;
    double2* Y1;
    const ulonglong2* orb;
    const DevStage* prev;
    int prev_sel;
    int write;
};

__device__ __forceinline__ uint64_t tile_row_len(uint64_t j, const TileParams& p) {
    if (j >= p.H) return 0;
    if (j + p.u < p.H) return p.du;
    if (j >= p.v) return p.dv;
    return p.du + p.dv;
}

__device__ __forceinline__ uint64_t tile_row_succ(uint64_t j, const TileParams& p) {
    if (j + p.u < p.H) return j + p.u;
    if (j >= p.v) return j - p.v;
    return j + p.u - p.v;
}

// ---------------------------------------------------------------- PTX glue
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// 16-byte asynchronous copy global -> shared (LDGSTS), L1 bypassed
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void orb_window(const ulonglong2* __restrict__ rec, uint64_t s,
                                           uint32_t& bits, uint64_t& rank) {
    const ulonglong2 R0 = __ldg(rec + (s >> 6)), R1 = __ldg(rec + (s >> 6) + 1);
    const unsigned o = static_cast<unsigned>(s & 63);
    bits = static_cast<uint32_t>(o ? (R0.x >> o) | (R1.x << (64 - o)) : R0.x);
    rank = R0.y + __popcll(R0.x & lowmask64(o));
}

// predicated 16-byte cp.async (no branch around it). No "memory" clobber: the
// producers never read the slot they fill, and their barrier arrives order the
// copies; without it the compiler can batch the plan reads ahead of the copies.
__device__ __forceinline__ void cp_async16_if(bool pred, void* dst, const void* src) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t@p cp.async.cg.shared.global [%0], [%1], 16;\n}" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(static_cast<uint32_t>(pred)));
}
// arrive on bar once all of this thread's prior cp.async copies have landed
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void write_partials(unsigned long long (*digits)[kDigits],
                                               unsigned long long* out_slot, int tid) {
    write_cta_digits(digits, out_slot, tid);
}

// One ring slot: the chunk's gathered columns (transposed, +1 padding against
// bank conflicts), its direct rows, and the row table the consumers need.
struct __align__(16) TileStage {
    double2 src[kCols][kRows + 1];
    double2 dst[kRows][kCols];
    uint64_t row_z[kRows];
    uint32_t row_lo[kRows];  // the CTA's columns of each row: [row_lo, row_lo + row_n)
    uint32_t row_n[kRows];   // (rows are < 2^32 long: make_tile_plan)
    uint64_t i0;
    uint64_t last;  // 1 on the last chunk of the CTA's sequence
};

// Orbit variant (kOrb). Plan warps turn the rank records into one OrbPlan per
// band and 32-column sub-chunk (the rank base and membership window of each
// gathered column run and of each row run) in a shared-memory ring ahead of the
// producers, so no record lookup sits on their path; the producers pack the
// members of up to kOrbSub consecutive sub-chunks of a band into one compact
// slot (up to kOrbCap members per side: a slot holds as many live amplitudes as
// a dense 32 x 32 chunk would, so as many bytes are in flight per SM).
struct OrbPlan {
    uint64_t crank[kCols];  // rank of column run c's first source; bit 63: the run wraps past N - 1
    uint64_t rrank[kRows];  // rank of row r's first index of the sub-chunk
    uint32_t cbits[kCols];  // membership of the run's kRows sources
    uint32_t rbits[kRows];  // membership of the row's kCols indices (0 past the row's end)
};
#ifndef SHS_ORB_GROUPS
#define SHS_ORB_GROUPS 1
#endif
constexpr int kOrbGroups = SHS_ORB_GROUPS;  // producer groups filling alternate slots
static_assert(kOrbGroups == 1, "the packing is computed once per slot by producer warp 0");
#ifndef SHS_ORB_CAP
#define SHS_ORB_CAP 1088
#endif
constexpr int kOrbCap = SHS_ORB_CAP;  // members per slot (one compact norm tile per group)
#ifndef SHS_ORB_SUB
#define SHS_ORB_SUB 4
#endif
constexpr int kOrbSub = SHS_ORB_SUB;  // sub-chunks per slot at most
constexpr int kOrbPlanRing = 8;
constexpr uint64_t kOrbWrap = 1ull << 63;

// A slot: the members of nsub consecutive sub-chunks of one band, row-major over
// the slot's columns (row r's members, all its sub-chunks, in z order, are
// rank-contiguous), so the consumers store them as runs and the chains fold them
// from a compact norm tile.
struct __align__(16) OrbSlot {
    double2 src[kOrbCap];            // gathered values of the slot's members (member order)
    double2 dst[kOrbCap];            // direct values
    uint64_t rrank[kRows];           // rank of row r's first position in the slot
    uint32_t rbits[kOrbSub][kRows];  // row r's members among sub-chunk j's 32 columns
    uint16_t soff[kRows + 1];        // row r's first member in the slot; soff[32] = members
    uint16_t nsub;
    uint32_t i0, last;               // (i0: band column of the slot's first sub-chunk)
};
// what the chains need of a slot, kept with its norm tile (the slot itself is
// recycled as soon as the consumers are done)
struct OrbMeta {
    uint32_t rbits[kOrbSub][kRows];
    uint16_t soff[kRows];
    uint16_t nsub;
};

template <bool kProbs, bool kOrb = false>
struct TileSmem {
    static constexpr int kST = kOrb ? SHS_ORB_SLOTS : kStages;
    static constexpr int kNB = kOrb ? SHS_ORB_NORM_BUFS : kNormBufs;
    std::conditional_t<kOrb, OrbSlot, TileStage> stage[kST];
    double nrm[kProbs && !kOrb ? kNB : 1][2][kOrb ? 1 : kRows][kOrb ? 1 : kNrmStride];  // [buffer][group][row][col]
    double onrm[kOrb ? kNB : 1][2][kOrb ? kOrbCap : 1];  // orbit: [buffer][group][member]
    uint64_t full[kST], empty[kST];
    unsigned long long digits[2][kDigits];
    uint32_t bandq[16 + 1];  // CtaWork<false>: the CTA's k-th band in bandq[k % 16];
                             // bandq[16]: how many entries P0 has published
    OrbMeta meta[kOrb ? kNB : 1];  // orbit: the slot of each norm tile
    uint64_t planfull[kOrb ? kOrbPlanRing : 1], planempty[kOrb ? kOrbPlanRing : 1];
    alignas(128) OrbPlan plan[kOrb ? kOrbPlanRing : 1];  // bulk-copy destinations: 16 B aligned at least
};

static_assert(sizeof(TileSmem<true, true>) <= 232448, "orbit variant: shared memory per CTA");

constexpr int kOrbPlanWarps = SHS_ORB_PLAN_WARPS;
template <bool kProbs, bool kSplit, bool kOrb = false>
constexpr int tile_threads() {  // (+ the orbit variant's plan warps)
    return 32 * (TileCfg<kSplit, kOrb>::kCW + TileCfg<kSplit, kOrb>::kPW + (kProbs ? kChainWarps : 0) +
                 (kOrb ? kOrbPlanWarps : 0));
}

template <bool kProbs, bool kOrb = false>
constexpr size_t tile_smem_bytes() {
    return sizeof(TileSmem<kProbs, kOrb>);
}



// The tile's row table, spread over a warp: lane l holds rows l + 32 h
// (h < kRowsPerLane), or row l & (kRows - 1) when kRows < 32. Returns the tile
// length (longest row).
struct LaneRows {
    uint64_t z[kRowsPerLane], len[kRowsPerLane];
    uint64_t lo[kRowsPerLane], hi[kRowsPerLane];  // this CTA's columns of the row
};

// where a row starting at z, of length len, is cut for a band cut at column i:
// its first 256-block boundary at or after i, or its end
__device__ __forceinline__ uint64_t row_cut(uint64_t z, uint64_t len, uint64_t i) {
    const uint64_t e = i + ((256 - ((z + i) & 255)) & 255);
    return e < len ? e : len;
}

__device__ __forceinline__ uint64_t tile_rows(const TileParams& p, uint64_t j0, int lane,
                                              LaneRows& lr) {
    uint64_t mx = 0;
#pragma unroll
    for (int h = 0; h < kRowsPerLane; ++h) {
        const int r = kRows >= 32 ? lane + 32 * h : (lane & (kRows - 1));
        const uint64_t j = j0 + r;
        lr.len[h] = tile_row_len(j, p);
        lr.z[h] = lr.len[h] ? mulmod_shoup(j, p.A, p.A_sh, p.N) : 0;
        mx = lr.len[h] > mx ? lr.len[h] : mx;
    }
#pragma unroll
    for (int o = (kRows >= 32 ? 16 : kRows / 2); o > 0; o >>= 1) {
        const uint64_t other = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = other > mx ? other : mx;
    }
    return mx;
}

// Rows of band j0 / kRows for a CTA whose range covers the band's columns from
// lo_col (0: the band's start) to hi_col (~0: its end). Returns the largest hi.
__device__ __forceinline__ uint64_t tile_rows_split(const TileParams& p, uint64_t j0, int lane,
                                                    LaneRows& lr, uint64_t lo_col,
                                                    uint64_t hi_col) {
    tile_rows(p, j0, lane, lr);
    uint64_t mx = 0;
#pragma unroll
    for (int h = 0; h < kRowsPerLane; ++h) {
        lr.lo[h] = lo_col ? row_cut(lr.z[h], lr.len[h], lo_col) : 0;
        lr.hi[h] = hi_col != ~0ull ? row_cut(lr.z[h], lr.len[h], hi_col) : lr.len[h];
        mx = lr.hi[h] > mx ? lr.hi[h] : mx;
    }
#pragma unroll
    for (int o = (kRows >= 32 ? 16 : kRows / 2); o > 0; o >>= 1) {
        const uint64_t other = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = other > mx ? other : mx;
    }
    return mx;
}

// A CTA's work items, each a band and a column range [lo_col, hi_col) (lo_col 0:
// the band's start; hi_col ~0: its end), walked identically by producers and
// chain warps: first bulk_rounds whole bands round-robin (band g + k * grid), so
// the CTAs in flight work on neighbouring bands and their gathered runs are
// adjacent in HBM (DRAM pages used whole: 8-14% faster than scattered ranges at
// config 4); then one contiguous, balanced chunk range of the remaining bands
// (host table `split`, so the leftover nbands mod grid bands, or a plan with
// fewer bands than SMs, still keeps every SM busy). CtaWork<false>: whole bands
// round-robin only (plans with >= kTileRoundRobinBands bands per CTA, where the
// imbalance of one band is small): no cut columns, and no span arithmetic left
// in the inner loops once lo = 0 / hi = len fold at compile time.
template <bool kSplit>
struct CtaWork;

// CtaWork<false> hands out whole bands dynamically: CTA g starts with band g,
// then its producer thread P0 takes the next band from a global counter, two
// bands ahead, into the shared queue bandq (so a band's successor and hence its
// "last" flag are known before its chunks are issued). Stragglers (SMs that get
// less DRAM bandwidth) no longer set the kernel time: with static round-robin
// bands the slowest CTA of a config-4 collapse ended 15% after the median.
// Results do not depend on the order (block partials land in fixed slots; the
// exact accumulator is order-independent). The counter advances by exactly
// ntiles - gridDim.x + gridDim.x = ntiles per launch (bands gridDim.x ..
// ntiles - 1 plus one terminal fetch per CTA), so the host keeps band_base
// without resetting it. The chain warps read bandq[k] only after consuming band
// k - 1, whose chunks P0 issued after writing it (mbarrier release -> consumer
// acquire -> named barrier).
constexpr int kBandQ = 16;  // > kStages + kNormBufs: the chain lags <= 8 chunks (bands)
constexpr int kProducerBar = 1 + 2 * kNormBufs;  // named barrier of the producer warps
constexpr int kConsumerBar = kProducerBar + 1;   // orbit variant: consumers released together

template <>
struct CtaWork<false> {
    uint32_t* q;
    uint64_t b, nt, k;
    bool producer, p0;
    int nprod;  // producer threads (named barrier count)
    __device__ __forceinline__ uint64_t fetch(const TileParams& p) const {
        return gridDim.x + (atomicAdd(p.band_ctr, 1ull) - p.band_base);
    }
    __device__ __forceinline__ CtaWork(const TileParams& p, uint32_t* queue, bool is_producer,
                                       int prod_warp0 = TileCfg<false>::kProdWarp,
                                       int nprod_ = kProducers)
        : q(queue), b(blockIdx.x), nt(p.ntiles), k(0), producer(is_producer), nprod(nprod_) {
        p0 = producer && threadIdx.x == 32 * prod_warp0;
        if (p0) {
            q[0] = static_cast<uint32_t>(b);
            const uint64_t b1 = fetch(p);
            q[1] = static_cast<uint32_t>(b1 < nt ? b1 : nt);
            publish(2);
        }
        if (producer) named_sync(kProducerBar, nprod);
    }
    // Readers outside the producer barrier (the orbit plan warps run up to a
    // plan ring ahead of the producers, so a band of <= 8 sub-chunks could end
    // before P0 wrote its successor) wait for P0's count of written entries.
    __device__ __forceinline__ void publish(uint32_t n) {
        __threadfence_block();
        reinterpret_cast<volatile uint32_t*>(q)[kBandQ] = n;
    }
    __device__ __forceinline__ void await(uint64_t n) const {
        while (reinterpret_cast<volatile uint32_t*>(q)[kBandQ] < n) __nanosleep(64);
        __threadfence_block();
    }
    __device__ __forceinline__ bool valid() const { return b < nt; }
    __device__ __forceinline__ void next(const TileParams& p) {
        if (p0) {
            const uint64_t b1 = q[(k + 1) % kBandQ];
            if (b1 < nt) {
                const uint64_t b2 = fetch(p);
                q[(k + 2) % kBandQ] = static_cast<uint32_t>(b2 < nt ? b2 : nt);
            }
            publish(static_cast<uint32_t>(k + 3));
        }
        if (producer) named_sync(kProducerBar, nprod);
        else await(k + 2);
        ++k;
        b = q[k % kBandQ];
    }
    __device__ __forceinline__ bool last() const { return q[(k + 1) % kBandQ] >= nt; }
    __device__ __forceinline__ uint64_t band() const { return b; }
    __device__ __forceinline__ uint64_t lo() const { return 0; }
    __device__ __forceinline__ uint64_t hi() const { return ~0ull; }
};

template <>
struct CtaWork<true> {
    uint64_t k, K, b, b_first, b_last, lo_col, hi_col, nt;
    bool bulk, tail_empty;
    __device__ __forceinline__ CtaWork(const TileParams& p, uint32_t*, bool, int = 0, int = 0) {
        const uint2 s0 = p.split[blockIdx.x], s1 = p.split[blockIdx.x + 1];
        b_first = s0.x;
        lo_col = uint64_t(s0.y) * kCols;
        b_last = s1.y ? s1.x : uint64_t(s1.x) - 1;
        hi_col = uint64_t(s1.y) * kCols;
        tail_empty = s0.x == s1.x && s0.y == s1.y;
        K = p.bulk_rounds;
        nt = p.ntiles;
        k = 0;
        bulk = K > 0 && blockIdx.x < nt;
        b = bulk ? blockIdx.x : b_first;
    }
    __device__ __forceinline__ bool valid() const { return bulk || (!tail_empty && b <= b_last); }
    __device__ __forceinline__ void next(const TileParams&) {
        if (bulk) {
            if (++k < K && b + gridDim.x < nt) {
                b += gridDim.x;
            } else {
                bulk = false;
                b = b_first;
            }
        } else {
            ++b;
        }
    }
    __device__ __forceinline__ bool last() const {
        return bulk ? ((k + 1 == K || b + gridDim.x >= nt) && tail_empty) : b == b_last;
    }
    __device__ __forceinline__ uint64_t band() const { return b; }
    __device__ __forceinline__ uint64_t lo() const { return (!bulk && b == b_first) ? lo_col : 0; }
    __device__ __forceinline__ uint64_t hi() const {
        return (!bulk && b == b_last && hi_col) ? hi_col : ~0ull;
    }
};

// (z, lo, hi) of tile row r from the warp's LaneRows (all lanes must call)
__device__ __forceinline__ void row_span_from_lanes(const LaneRows& lr, int r, uint64_t& z,
                                                    uint64_t& lo, uint64_t& hi) {
    const int src_lane = r & 31;
    const int h = kRowsPerLane > 1 ? (r >> 5) : 0;
    z = lo = hi = 0;
#pragma unroll
    for (int hh = 0; hh < kRowsPerLane; ++hh) {
        const uint64_t zz = __shfl_sync(0xffffffffu, lr.z[hh], src_lane);
        const uint64_t ll = __shfl_sync(0xffffffffu, lr.lo[hh], src_lane);
        const uint64_t uu = __shfl_sync(0xffffffffu, lr.hi[hh], src_lane);
        if (hh == h) {
            z = zz;
            lo = ll;
            hi = uu;
        }
    }
}

// write the band's row spans into a ring slot (lanes of one warp)
__device__ __forceinline__ void store_row_spans(const LaneRows& lr, int lane, uint64_t* row_z,
                                                uint32_t* row_lo, uint32_t* row_n) {
#pragma unroll
    for (int h = 0; h < kRowsPerLane; ++h) {
        const int r = lane + 32 * h;
        if (kRows >= 32 || lane < kRows) {
            row_z[r] = lr.z[h];
            row_lo[r] = static_cast<uint32_t>(lr.lo[h]);
            row_n[r] = static_cast<uint32_t>(lr.hi[h] > lr.lo[h] ? lr.hi[h] - lr.lo[h] : 0);
        }
    }
}

// (z, len) of tile row r from the warp's LaneRows (all lanes must call)
__device__ __forceinline__ void row_from_lanes(const LaneRows& lr, int r, uint64_t& z,
                                               uint64_t& len) {
    const int src_lane = r & 31;
    const int h = kRowsPerLane > 1 ? (r >> 5) : 0;
    z = 0;
    len = 0;
#pragma unroll
    for (int hh = 0; hh < kRowsPerLane; ++hh) {
        const uint64_t zz = __shfl_sync(0xffffffffu, lr.z[hh], src_lane);
        const uint64_t ll = __shfl_sync(0xffffffffu, lr.len[hh], src_lane);
        if (hh == h) {
            z = zz;
            len = ll;
        }
    }
}

// write the tile's row table into a ring slot (lanes of one warp)
__device__ __forceinline__ void store_rows(const LaneRows& lr, int lane, uint64_t* row_z,
                                           uint64_t* row_l) {
#pragma unroll
    for (int h = 0; h < kRowsPerLane; ++h) {
        const int r = lane + 32 * h;
        if (kRows >= 32 || lane < kRows) {
            row_z[r] = lr.z[h];
            row_l[r] = lr.len[h];
        }
    }
}

template <bool kProbs, bool kSplit, bool kOrb = false>
__global__ void __launch_bounds__((tile_threads<kProbs, kSplit, kOrb>()), 1) k_tiled(TileParams p) {
    static_assert(!kOrb || (kProbs && kRows == 32 && kCols == 32),
                  "orbit variant: probs pass, 32 x 32 chunks");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    TileSmem<kProbs, kOrb>& sm = *reinterpret_cast<TileSmem<kProbs, kOrb>*>(smem_raw);
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    using Cfg = TileCfg<kSplit, kOrb>;
    constexpr int kStages = Cfg::kST, kNormBufs = Cfg::kNB;
    constexpr int kConsumerWarps = Cfg::kCW, kConsumers = Cfg::kCons;
    constexpr int kProducerWarp = Cfg::kProdWarp, kChainWarp = Cfg::kChainWarp0;
    constexpr int kRowsPerConsumer = Cfg::kRowsPerCons, kNormSync = Cfg::kNSync;
    (void)kConsumers;
    // the orbit variant may start under programmatic dependent launch while the
    // previous stage's finalize still runs: its scalars are read after the wait
    StageScalars sc = p.sc;
    int sel = p.sel;
    if (!kOrb && p.dev) {
        sc = p.dev->sc;
        sel = p.dev->sel;
    }
    if (!kProbs && p.spec && sel == 0) {
        // Y already holds h0 (raw, like every collapse output); the dynamic band
        // counter still advances by the ntiles fetches a full launch makes
        if (!kSplit && blockIdx.x == 0 && tid == 0) atomicAdd(p.band_ctr, p.ntiles);
        return;
    }
    const bool spec = kProbs && p.spec;
#ifdef SHS_CTA_TRACE
    uint64_t trace_t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(trace_t0));
#endif

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            // copies of every producer + header
            mbar_init(&sm.full[s], Cfg::kProds / (kOrb ? kOrbGroups : 1) + 1);
            mbar_init(&sm.empty[s], kConsumerWarps);
        }
        if constexpr (kOrb)
            for (int s = 0; s < kOrbPlanRing; ++s) {
                mbar_init(&sm.planfull[s], 1);
                mbar_init(&sm.planempty[s], Cfg::kPW);
            }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (kProbs)
        for (int i = tid; i < 2 * kDigits; i += blockDim.x) (&sm.digits[0][0])[i] = 0ull;
    if (tid == 0) sm.bandq[kBandQ] = 0;  // CtaWork<false>: nothing published yet
    __syncthreads();
    if constexpr (kOrb) {
        // k_tile_fixup1 may be scheduled on SMs this grid leaves (it waits for
        // the whole grid before reading anything)
        asm volatile("griddepcontrol.launch_dependents;");
        // every role but the plan warps (records and the plan only) waits for the
        // previous kernels' writes before it reads or writes global state
        const bool plan_warp = !(warp >= kProducerWarp && warp < kProducerWarp + Cfg::kPW) &&
                               warp >= kConsumerWarps && warp >= kChainWarp + kChainWarps;
        if (!plan_warp) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            if (p.dev) {
                sc = p.dev->sc;
                sel = p.dev->sel;
            }
        }
    }

    if (warp >= kProducerWarp && warp < kProducerWarp + Cfg::kPW) {
        // ------------------------------------------------------------ producers
        // gathered side: element e = pt + kProducers * k is (column e / kRows,
        // row e % kRows = pt % kRows): kRows consecutive threads copy one
        // column's run. Direct side: element e is (row e / kCols = pt / kCols +
        // kDstRowStep k, column e % kCols = pt % kCols): kCols threads per row run. The row
        // table lives in every producer warp's lanes (tile_rows_split) and is
        // fetched by shuffles.
        const int pt = tid - 32 * kProducerWarp;
        const int r_src = pt & (kRows - 1);
        const int src_c0 = pt / kRows;
        const int dst_r0 = pt / kCols, dst_c = pt % kCols;
        int stage = 0;
        uint32_t phase = 0;
        if constexpr (kOrb) {
            // Orbit variant. Element (row r, column c) of a sub-chunk is an orbit
            // member on the direct side (z_j + c) iff its gathered source (j + c m)
            // is one (m is a power of a); members are copied into the slot in
            // row-major member order, each side from its rank. Warp w copies the
            // gathered columns w + 4k (lanes = rows) and the direct rows w + 4k
            // (lanes = columns). Every warp evaluates the same packing decision
            // from the same plan; warp 0 also writes the slot's tables. The plan
            // entries come from the plan warp (below).
            // The producer warps form kOrbGroups groups that fill alternate slots
            // (a slot's copies are a long dependent chain per warp: one group at a
            // time left the slot period set by it); every group evaluates every
            // slot's packing, so all agree on where each slot starts.
            constexpr int kGW = Cfg::kPW / kOrbGroups;  // warps per group
            const int grp = (warp - kProducerWarp) / kGW;
            const int pw = (warp - kProducerWarp) % kGW;  // warp within the group
            const double2* Xs = (p.prev ? p.prev->sel : p.prev_sel) ? p.X1 : p.X;
            const uint32_t lt_lane = (1u << lane) - 1u;
            constexpr uint32_t kOrbWarpCols = [] {  // columns 0, kGW, 2 kGW, ...
                uint32_t m = 0;
                for (int c = 0; c < kCols; c += kGW) m |= 1u << c;
                return m;
            }();
            uint64_t qs = 0;  // slots of this CTA so far (slot qs goes to group qs % kOrbGroups)
            uint64_t gc = 0;  // plan entries consumed
            for (CtaWork<kSplit> wk(p, sm.bandq, true, kProducerWarp, Cfg::kProds); wk.valid(); wk.next(p)) {
                const uint64_t j0 = wk.band() * kRows;
                const uint64_t lo_col = wk.lo();  // split plans: this CTA's columns of the band
                LaneRows lr;
                const uint64_t tend = tile_rows_split(p, j0, lane, lr, lo_col, wk.hi());
                const uint64_t iend = tend > lo_col ? tend : lo_col + 1;  // >= 1 sub-chunk per item
                const uint64_t nch = (iend - lo_col + kCols - 1) / kCols;
                uint64_t n = 0;
                while (n < nch) {
                    const bool mine = static_cast<int>(qs % kOrbGroups) == grp;
                    OrbSlot& st = sm.stage[stage];
                    // pass 1 (warp 0 of the group): how many sub-chunks fit, the row
                    // offsets; published in the slot for the other producer warps
                    uint32_t rbj[kOrbSub], cntj[kOrbSub];
                    int K = 0;
                    uint32_t M = 0;
                    if (mine && pw == 0) {
                        mbar_wait(&sm.empty[stage], phase ^ 1);
                        bool stop = false;
#pragma unroll
                        for (int jj = 0; jj < kOrbSub; ++jj) {
                            rbj[jj] = cntj[jj] = 0;
                            if (!stop && n + jj < nch) {
                                const uint64_t g = gc + jj;
                                const int ps = static_cast<int>(g % kOrbPlanRing);
                                mbar_wait(&sm.planfull[ps], static_cast<uint32_t>((g / kOrbPlanRing) & 1));
                                const uint32_t rb = sm.plan[ps].rbits[lane];  // row `lane`
                                const uint32_t c = __popc(rb);
                                const uint32_t tot = __reduce_add_sync(0xffffffffu, c);
                                if (jj > 0 && M + tot > kOrbCap) {
                                    stop = true;
                                } else {
                                    rbj[jj] = rb;
                                    cntj[jj] = c;
                                    M += tot;
                                    K = jj + 1;
                                }
                            }
                        }
                        uint32_t rc = 0;
#pragma unroll
                        for (int jj = 0; jj < kOrbSub; ++jj) rc += cntj[jj];
                        uint32_t inc = rc;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
                            if (lane >= o) inc += v;
                        }
#pragma unroll
                        for (int jj = 0; jj < kOrbSub; ++jj)
                            if (jj < K) st.rbits[jj][lane] = rbj[jj];
                        st.soff[lane] = static_cast<uint16_t>(inc - rc);
                        if (lane == 31) st.soff[kRows] = static_cast<uint16_t>(inc);
                        if (lane == 0) st.nsub = static_cast<uint16_t>(K);
                    }
                    if (kOrbGroups == 1) named_sync(kProducerBar, Cfg::kProds);
                    if (mine && pw != 0) {
                        K = st.nsub;
                        M = st.soff[kRows];
#pragma unroll
                        for (int jj = 0; jj < kOrbSub; ++jj) {
                            rbj[jj] = jj < K ? st.rbits[jj][lane] : 0u;
                            cntj[jj] = __popc(rbj[jj]);
                        }
                    }
                    if (!mine) {  // the other group's slot (kOrbGroups > 1): where it ends
                        bool stop = false;
#pragma unroll
                        for (int jj = 0; jj < kOrbSub; ++jj) {
                            rbj[jj] = cntj[jj] = 0;
                            if (!stop && n + jj < nch) {
                                const uint64_t g = gc + jj;
                                const int ps = static_cast<int>(g % kOrbPlanRing);
                                mbar_wait(&sm.planfull[ps], static_cast<uint32_t>((g / kOrbPlanRing) & 1));
                                const uint32_t tot = __reduce_add_sync(0xffffffffu, __popc(sm.plan[ps].rbits[lane]));
                                if (jj > 0 && M + tot > kOrbCap) stop = true;
                                else { M += tot; K = jj + 1; }
                            }
                        }
                    }
                    uint32_t rowc = 0;
#pragma unroll
                    for (int jj = 0; jj < kOrbSub; ++jj) rowc += cntj[jj];
                    uint32_t base = mine ? st.soff[lane] : 0u;  // this row's next member slot index
                    uint32_t rowc_before[kOrbSub];  // this row's members in the slot's earlier sub-chunks
#pragma unroll
                    for (int jj = 0, acc = 0; jj < kOrbSub; ++jj) {
                        rowc_before[jj] = acc;
                        acc += cntj[jj];
                    }
                    // (one bulk copy per row for the direct side measured slower:
                    // 13.1 vs 11.8 ms at n30, TMA-issue bound)
                    // pass 2: copies, sub-chunk by sub-chunk
#pragma unroll
                    for (int jj = 0; jj < kOrbSub; ++jj) {
                        if (jj >= K) break;
                        const uint64_t g = gc + jj;
                        const int ps = static_cast<int>(g % kOrbPlanRing);
                        if (!mine) {  // the other group's slot: release the entry only
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&sm.planempty[ps]);
                            continue;
                        }
                        const OrbPlan& E = sm.plan[ps];
                        const uint32_t rb = rbj[jj];
                        const uint64_t i0 = lo_col + (n + jj) * kCols;
                        const uint32_t wrapc = __ballot_sync(0xffffffffu, (E.crank[lane] & kOrbWrap) != 0) &
                                               (kOrbWarpCols << pw);
                        constexpr int kG = kCols / kGW, kD = kRows / kGW;
#pragma unroll
                        for (int k = 0; k < kG; ++k) {  // gathered: column pw + kGW k, row `lane`
                            const int cc = pw + kGW * k;
                            const uint64_t rank = (E.crank[cc] & ~kOrbWrap) + __popc(E.cbits[cc] & lt_lane);
                            cp_async16_if(((rb & ~wrapc) >> cc) & 1u,
                                          &st.src[base + __popc(rb & ((1u << cc) - 1u))], Xs + rank);
                        }
#pragma unroll
                        for (int k = 0; k < kD; ++k) {  // direct: row pw + kGW k, column `lane`
                            const int rr = pw + kGW * k;
                            const uint32_t rbr = __shfl_sync(0xffffffffu, rb, rr);
                            const uint32_t brr = __shfl_sync(0xffffffffu, base, rr);
                            const uint32_t below = __popc(rbr & lt_lane);
                            cp_async16_if((rbr >> lane) & 1u, &st.dst[brr + below], Xs + (E.rrank[rr] + below));
                        }
                        if (wrapc) {  // wrapped columns: every element by lookup
                            for (uint32_t wm = wrapc; wm; wm &= wm - 1) {
                                const int cc = __ffs(wm) - 1;
                                const uint64_t cs = addmod(j0, mulmod_shoup(i0 + cc, p.m, p.m_sh, p.N), p.N);
                                const uint64_t src = cs + lane >= p.N ? cs + lane - p.N : cs + lane;
                                uint64_t rank;
                                orb_lookup(p.orb, src, rank);
                                if ((rb >> cc) & 1u)
                                    cp_async16(&st.src[base + __popc(rb & ((1u << cc) - 1u))], Xs + rank);
                            }
                        }
                        if (pw == 0) {
                            // the row's first members in the slot: the rank of its
                            // first included position (spans of split plans start mid-row)
                            const uint32_t before = jj ? rowc_before[jj] : 0u;
                            if (rb && before == 0) st.rrank[lane] = E.rrank[lane];
                        }
                        base += cntj[jj];
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&sm.planempty[ps]);
                    }
                    if (mine && pw == 0 && lane == 0) st.i0 = static_cast<uint32_t>(lo_col + n * kCols);
                    gc += K;
                    n += K;
                    ++qs;
                    if (mine) {
                        if (pw == 0 && lane == 0) st.last = (wk.last() && n == nch) ? 1u : 0u;
                        cp_async_arrive(&sm.full[stage]);
                        if (pw == 0) {
                            __syncwarp();  // slot tables ordered before lane 0's release
                            if (lane == 0) mbar_arrive(&sm.full[stage]);
                        }
                    }
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        } else
        for (CtaWork<kSplit> wk(p, sm.bandq, true); wk.valid(); wk.next(p)) {
            const uint64_t j0 = wk.band() * kRows;
            const uint64_t lo_col = wk.lo();
            LaneRows lr;
            const uint64_t tend = tile_rows_split(p, j0, lane, lr, lo_col, wk.hi());
            const uint64_t iend = tend > lo_col ? tend : lo_col + 1;  // >= 1 chunk per item
            // this thread's source row r_src = lane + 32 * (warp-uniform h)
            const int hs = kRowsPerLane > 1 ? (r_src >> 5) : 0;
            // spans as (lo, n), 32-bit: pos in [lo, lo + n) <=> pos - lo < n (unsigned)
            const uint32_t rlo = static_cast<uint32_t>(lr.lo[hs]);
            const uint32_t rn = static_cast<uint32_t>(lr.hi[hs] > lr.lo[hs] ? lr.hi[hs] - lr.lo[hs] : 0);
            // source index of this thread's copies, advanced by kCols*m per chunk
            uint64_t sidx[kCopiesPerProducer];
            const double2* dptr[kCopiesPerProducer];
            uint32_t dlo[kCopiesPerProducer], dn[kCopiesPerProducer];
#pragma unroll
            for (int k = 0; k < kCopiesPerProducer; ++k) {
                const uint64_t c = lo_col + src_c0 + (kProducers / kRows) * k;
                sidx[k] = addmod(j0 + r_src, mulmod_shoup(c, p.m, p.m_sh, p.N), p.N);
                uint64_t dz, l, h;
                row_span_from_lanes(lr, dst_r0 + kDstRowStep * k, dz, l, h);
                dlo[k] = static_cast<uint32_t>(l);
                dn[k] = static_cast<uint32_t>(h > l ? h - l : 0);
                dptr[k] = p.X + dz + lo_col + dst_c;
            }
            for (uint64_t i0 = lo_col; i0 < iend; i0 += kCols) {
                mbar_wait(&sm.empty[stage], phase ^ 1);
                TileStage& st = sm.stage[stage];
#pragma unroll
                for (int k = 0; k < kCopiesPerProducer; ++k) {
                    const uint32_t pos =
                        static_cast<uint32_t>(i0) + src_c0 + (kProducers / kRows) * k;
                    if (pos - rlo < rn)
                        cp_async16(&st.src[src_c0 + (kProducers / kRows) * k][r_src],
                                   p.X + sidx[k]);
                    sidx[k] = addmod(sidx[k], p.m_chunk, p.N);
                }
#pragma unroll
                for (int k = 0; k < kCopiesPerProducer; ++k) {
                    const uint32_t pos = static_cast<uint32_t>(i0) + dst_c;
                    if (pos - dlo[k] < dn[k])
                        cp_async16(&st.dst[dst_r0 + kDstRowStep * k][dst_c], dptr[k]);
                    dptr[k] += kCols;
                }
                cp_async_arrive(&sm.full[stage]);
                if (warp == kProducerWarp) {
                    store_row_spans(lr, lane, st.row_z, st.row_lo, st.row_n);
                    __syncwarp();  // row table stores ordered before lane 0's release
                    if (lane == 0) {
                        st.i0 = i0;
                        st.last = (wk.last() && i0 + kCols >= iend) ? 1 : 0;
                        mbar_arrive(&sm.full[stage]);
                    }
                }
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp < kConsumerWarps) {
        // ------------------------------------------------------------ consumers
        int stage = 0;
        uint32_t phase = 0;
        uint64_t k = 0;  // chunk counter (norm buffer parity)
        const int c = tid & (kCols - 1);
        const int rg = tid / kCols;  // row group: rows rg * kRowsPerConsumer + q
        // collapse with 32-column chunks: a warp owns whole row segments; a row that
        // starts at an odd index stores its segment shifted by one element (the last
        // one is carried into the next chunk) so every store covers whole 32 B sectors
        constexpr bool kSectorShift = !kProbs && kCols == 32;
        // speculative h0 stores: plain (the sector-shifted stores measured 2% slower
        // per config-4 stage, profiles/r01/README.md v15); -DSHS_SPEC_SHIFT for A/B
#ifdef SHS_SPEC_SHIFT
        constexpr bool kSpecShift = kProbs && kCols == 32;
#else
        constexpr bool kSpecShift = false;
#endif
        double2 carry[kRowsPerConsumer];
#pragma unroll
        for (int q = 0; q < kRowsPerConsumer; ++q) carry[q] = make_double2(0.0, 0.0);
        bool more = true;  // every CTA has >= 1 item, every item >= 1 chunk
        while (more) {
            if constexpr (kOrb) {
                // one warp polls the slot's barrier, the others sleep on a named
                // barrier (14 spinning warps took issue slots from the producers)
                if (warp == 0) mbar_wait(&sm.full[stage], phase);
                named_sync(kConsumerBar, kConsumers);
            } else {
                mbar_wait(&sm.full[stage], phase);
            }
            auto& st = sm.stage[stage];
            const uint32_t i0 = static_cast<uint32_t>(st.i0);
            const uint32_t pos = i0 + c;
            more = st.last == 0;
            if constexpr (kOrb) {
                // the slot's members -> one compact norm tile (member order) and
                // both groups' stores: warp w takes rows w, w + kCW, ...; lane i
                // the row's members i, i + 32, ... (consecutive smem and ranks)
                const int b = static_cast<int>(k % kNormBufs);
                if (k >= kNormBufs) named_sync(kNormEmpty0 + b, kNormSync);
                double* n0 = &sm.onrm[b][0][0];
                double* n1 = &sm.onrm[b][1][0];
                const int K = st.nsub;
                for (int r = warp; r < kRows; r += kConsumerWarps) {
                    const uint32_t e0 = st.soff[r], e1 = st.soff[r + 1];
                    const uint64_t rk = st.rrank[r];
                    // the chains' copy of this row's slot table
                    if (lane < K) sm.meta[b].rbits[lane][r] = st.rbits[lane][r];
                    if (lane == 31) sm.meta[b].soff[r] = static_cast<uint16_t>(e0);
                    for (uint32_t e = e0 + lane; e < e1; e += 32) {
                        double h0r, h0i, h1r, h1i;
                        stage_pair(sc, st.dst[e], st.src[e], h0r, h0i, h1r, h1i);
                        n0[e] = cnorm(h0r, h0i);
                        n1[e] = cnorm(h1r, h1i);
                        if (p.write) {  // both groups at the member's rank
                            const uint64_t at = rk + (e - e0);
                            p.Y[at] = make_double2(h0r, h0i);
                            p.Y1[at] = make_double2(h1r, h1i);
                        }
                    }
                }
                if (tid == 0) sm.meta[b].nsub = static_cast<uint16_t>(K);
                named_arrive(kNormFull0 + b, kNormSync);
                ++k;
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.empty[stage]);
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            } else {
            const int b = static_cast<int>(k % kNormBufs);
            if (kProbs && k >= kNormBufs) named_sync(kNormEmpty0 + b, kNormSync);
#pragma unroll
            for (int q = 0; q < kRowsPerConsumer; ++q) {
                const int r = rg * kRowsPerConsumer + q;
                const uint32_t rlo = kSplit ? st.row_lo[r] : 0u, rn = st.row_n[r];
                const bool live = pos - rlo < rn;
                double h0r, h0i, h1r, h1i;
                stage_pair(sc, st.dst[r][c], st.src[c][r], h0r, h0i, h1r, h1i);
                // row segment store of this warp's 32 columns (collapse output, or
                // the probs pass's speculative h0): a row that starts at an odd
                // index stores shifted by one element so every store covers whole
                // 32 B sectors (the last element is carried into the next chunk)
                auto store_seg = [&](const double2 hv) {
                    const uint64_t rz = st.row_z[r];
                    if ((rz & 1) == 0) {
                        if (live) p.Y[rz + pos] = hv;
                    } else {
                        // lane c stores column c - 1; lane 0 the previous chunk's column 31
                        // (carried: i0 - 1 >= row_lo means that chunk was this CTA's)
                        const double2 up = make_double2(__shfl_up_sync(0xffffffffu, hv.x, 1),
                                                        __shfl_up_sync(0xffffffffu, hv.y, 1));
                        const double2 last = make_double2(__shfl_sync(0xffffffffu, hv.x, 31),
                                                          __shfl_sync(0xffffffffu, hv.y, 31));
                        if (c > 0) {
                            if (pos - 1 - rlo < rn) p.Y[rz + pos - 1] = up;
                        } else if (i0 - 1 - rlo < rn) {  // (i0 = 0 wraps: never below 2^32 - 1 - lo)
                            p.Y[rz + i0 - 1] = carry[q];
                        }
                        // the span's final element when it falls in column 31 of its last chunk
                        if (c == kCols - 1 && live && pos + 1 == rlo + rn) p.Y[rz + pos] = hv;
                        carry[q] = last;
                    }
                };
                if (kProbs) {
                    sm.nrm[b][0][r][c] = live ? cnorm(h0r, h0i) : 0.0;
                    sm.nrm[b][1][r][c] = live ? cnorm(h1r, h1i) : 0.0;
                    if (spec) {
                        if (kSpecShift) store_seg(make_double2(h0r, h0i));
                        else if (live) p.Y[st.row_z[r] + pos] = make_double2(h0r, h0i);
                    }
                } else if (kSectorShift) {
                    store_seg(sel ? make_double2(h1r, h1i) : make_double2(h0r, h0i));
                } else if (live) {
                    p.Y[st.row_z[r] + pos] =
                        sel ? make_double2(h1r, h1i) : make_double2(h0r, h0i);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[stage]);
            if (kProbs) named_arrive(kNormFull0 + b, kNormSync);
            ++k;
            if (++stage == kStages) {
                stage = 0;
                phase ^= 1;
            }
            }  // dense slot
        }
        if (kProbs) {  // match the chain's releases of the last kNormBufs norm tiles
            for (uint64_t q = (k > kNormBufs ? k - kNormBufs : 0); q < k; ++q)
                named_sync(kNormEmpty0 + static_cast<int>(q % kNormBufs), kNormSync);
        }
    } else if (kOrb && warp >= kChainWarp + kChainWarps) {
        // ------------------------------------------------------------ plan warps
        // kOrbPlanWarps warps compute the plan entries in the kernel (no plan
        // pre-pass): entry g of the CTA's sub-chunk sequence by warp g mod
        // kOrbPlanWarps, lane c / r: column run c / row r of the sub-chunk, each
        // window from two rank records
        const int pwi = warp - (kChainWarp + kChainWarps);
        uint64_t g = 0;
        for (CtaWork<kSplit> wk(p, sm.bandq, false, kProducerWarp, Cfg::kProds); wk.valid(); wk.next(p)) {
            const uint64_t j0 = wk.band() * kRows;
            const uint64_t lo_col = wk.lo();
            LaneRows lr;  // lane: row j0 + lane, its span [lo, hi) of this work item
            const uint64_t tend = tile_rows_split(p, j0, lane, lr, lo_col, wk.hi());
            const uint64_t iend = tend > lo_col ? tend : lo_col + 1;
            const uint64_t nch = (iend - lo_col + kCols - 1) / kCols;
            const uint64_t z = lr.z[0], rlo = lr.lo[0], rhi = lr.hi[0];
            uint64_t n = (pwi + kOrbPlanWarps - g % kOrbPlanWarps) % kOrbPlanWarps;  // first of mine
            for (; n < nch; n += kOrbPlanWarps) {
                const uint64_t ge = g + n;  // this entry's index in the CTA's sequence
                const uint64_t i0 = lo_col + n * kCols;
                const uint64_t cs = addmod(j0, mulmod_shoup(i0 + lane, p.m, p.m_sh, p.N), p.N);
                uint32_t cb, rb = 0;
                uint64_t cr, rr = 0;
                orb_window(p.orb, cs, cb, cr);
                if (cs + (kRows - 1) >= p.N) cr |= kOrbWrap;
                if (i0 < rhi && i0 + kCols > rlo) {  // the row's span meets the sub-chunk
                    uint32_t full;
                    orb_window(p.orb, z + i0, full, rr);
                    const uint32_t a0 = rlo > i0 ? static_cast<uint32_t>(rlo - i0) : 0u;
                    const uint32_t a1 = rhi - i0 < kCols ? static_cast<uint32_t>(rhi - i0) : uint32_t(kCols);
                    const uint32_t keep = (a1 >= 32 ? ~0u : ((1u << a1) - 1u)) & ~((1u << a0) - 1u);
                    rb = full & keep;
                    rr += __popc(full & ((1u << a0) - 1u));  // rank of the span's first position
                }
                const int ps = static_cast<int>(ge % kOrbPlanRing);
                mbar_wait(&sm.planempty[ps], static_cast<uint32_t>((ge / kOrbPlanRing) & 1) ^ 1);
                OrbPlan& e = sm.plan[ps];
                e.crank[lane] = cr;
                e.rrank[lane] = rr;
                e.cbits[lane] = cb;
                e.rbits[lane] = rb;
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.planfull[ps]);
            }
            g += nch;
        }
    } else if (kProbs && warp >= kChainWarp && warp < kChainWarp + kChainWarps) {
        // ------------------------------------------------------------ chains
        const int ct = tid - 32 * kChainWarp;  // one lane per (row, group)
        const int cr = ct % kRows, cg = ct / kRows;
        DigitWindow win;
        window_reset(win);
        uint64_t k = 0;
        for (CtaWork<kSplit> wk(p, sm.bandq, false, kProducerWarp, Cfg::kProds); wk.valid(); wk.next(p)) {
            const uint64_t j0 = wk.band() * kRows;
            const uint64_t lo_col = wk.lo();
            LaneRows lr;
            const uint64_t tend = tile_rows_split(p, j0, lane, lr, lo_col, wk.hi());
            const uint64_t iend = tend > lo_col ? tend : lo_col + 1;
            const int hsel = kRowsPerLane > 1 ? ((ct >> 5) % kRowsPerLane) : 0;  // row cr = lane + 32 hsel
            const uint64_t c_z = lr.z[hsel], c_len = lr.len[hsel];
            const uint64_t c_lo = lr.lo[hsel], c_hi = lr.hi[hsel];
            // head positions belong to the block shared with the predecessor row
            // (k_tile_fixup); c_lo > 0 is a block boundary, hence >= c_head
            const uint64_t c_head = (256 - (c_z & 255)) & 255;
            const uint64_t c_fast = c_lo > c_head ? c_lo : c_head;
            double c_s = 0.0;
            if constexpr (kOrb) {
                // Orbit variant: per slot, this row's members (compact, in z order)
                // sub-chunk by sub-chunk; positions off the orbit add +0.0 in the
                // reference, so skipping them leaves every fold unchanged. The head
                // positions (k_tile_fixup) are stored with zeros off the orbit.
                // (split plans: the row's span [c_lo, c_hi) of this work item; c_lo > 0
                // is a block boundary, hence past the head)
                const uint64_t nch = (iend - lo_col + kCols - 1) / kCols;
                for (uint64_t n = 0; n < nch; ++k) {
                    const int b = static_cast<int>(k % kNormBufs);
                    named_sync(kNormFull0 + b, kNormSync);
                    const OrbMeta& mt = sm.meta[b];
                    const int K = mt.nsub;
                    const double* nv = &sm.onrm[b][cg][0];
                    uint32_t e = mt.soff[cr];
                    // fold the next cnt members in order, 8 loads in flight at a time
                    // (padding adds +0.0, which leaves the non-negative sum unchanged)
                    auto fold = [&](uint32_t cnt) {
                        for (uint32_t t = 0; t < cnt; t += 8) {
                            double v[8];
#pragma unroll
                            for (int u = 0; u < 8; ++u) v[u] = t + u < cnt ? nv[e + t + u] : 0.0;
#pragma unroll
                            for (int u = 0; u < 8; ++u) c_s = __dadd_rn(c_s, v[u]);
                        }
                        e += cnt;
                    };
                    for (int j = 0; j < K; ++j) {
                        const uint64_t i0 = lo_col + (n + j) * kCols;
                        if (i0 >= c_hi) break;
                        if (i0 + kCols <= c_lo) continue;  // before this work item's span
                        uint32_t bits = mt.rbits[j][cr];
                        const int end = static_cast<int>(min(c_hi - i0, uint64_t(kCols)));
                        int start = c_lo > i0 ? static_cast<int>(c_lo - i0) : 0;
                        if (c_lo == 0 && i0 < c_head) {
                            const int qh = static_cast<int>(min(c_head - i0, uint64_t(end)));
                            double* head = p.head + ((j0 + cr) * 2 + cg) * 256 + i0;
                            for (int cc = 0; cc < qh; ++cc) head[cc] = ((bits >> cc) & 1u) ? nv[e++] : 0.0;
                            start = qh;
                            bits &= qh >= 32 ? 0u : ~((1u << qh) - 1u);
                        }
                        const int qb = static_cast<int>(255 - ((c_z + i0) & 255));
                        if (qb >= start && qb < end) {  // a block ends at column qb
                            const uint32_t lo = bits & (qb >= 31 ? ~0u : ((2u << qb) - 1u));
                            bits &= ~lo;
                            fold(__popc(lo));
                            p.S[cg * p.nb + ((c_z + i0 + qb) >> 8)] = c_s;
                            window_add(win, c_s, sm.digits[cg]);
                            c_s = 0.0;
                        }
                        fold(__popc(bits));
                    }
                    n += K;
                    __syncwarp();
                    named_arrive(kNormEmpty0 + b, kNormSync);
                }
            } else
            for (uint64_t i0 = lo_col; i0 < iend; i0 += kCols, ++k) {
                const int b = static_cast<int>(k % kNormBufs);
                named_sync(kNormFull0 + b, kNormSync);
                const double* row = &sm.nrm[b][cg][cr][0];
                if (i0 >= c_fast && i0 + kCols <= c_hi) {
                    // interior chunk (the common case): 64 in-order adds, branch-free.
                    // At most one block ends inside the chunk (kCols <= 256), at
                    // column qb: the block's fold continues in `a`, the next block
                    // starts in `nb`. Each chain adds the value or +0.0, which leaves
                    // a non-negative sum unchanged, so both folds are exactly the
                    // reference's (s = 0; s += x ...); the masking is off the chains.
                    const int qb = static_cast<int>(255 - ((c_z + i0) & 255));
                    double a = c_s, nb = 0.0;
#pragma unroll
                    for (int cc = 0; cc < kCols; cc += 2) {
                        const double2 x = *reinterpret_cast<const double2*>(row + cc);
                        const bool lo0 = cc <= qb, lo1 = cc + 1 <= qb;
                        a = __dadd_rn(a, lo0 ? x.x : 0.0);
                        nb = __dadd_rn(nb, lo0 ? 0.0 : x.x);
                        a = __dadd_rn(a, lo1 ? x.y : 0.0);
                        nb = __dadd_rn(nb, lo1 ? 0.0 : x.y);
                    }
                    if (qb < kCols) {
                        p.S[cg * p.nb + ((c_z + i0 + qb) >> 8)] = a;
                        window_add(win, a, sm.digits[cg]);
                        c_s = nb;
                    } else {
                        c_s = a;
                    }
                } else if (i0 < c_hi && i0 + kCols > c_lo) {
                    // span start / end: the row's head (stored for k_tile_fixup), then
                    // blocks folded in order
                    const int q1 = static_cast<int>(min(c_hi - i0, uint64_t(kCols)));
                    int qa = c_lo > i0 ? static_cast<int>(c_lo - i0) : 0;
                    if (i0 + qa < c_head) {
                        const int qh = static_cast<int>(min(c_head - i0, uint64_t(q1)));
                        double* head = p.head + ((j0 + cr) * 2 + cg) * 256 + i0;
                        for (int cc = qa; cc < qh; ++cc) head[cc] = row[cc];
                        qa = qh;
                    }
                    while (qa < q1) {
                        const int qb = qa + static_cast<int>(255 - ((c_z + i0 + qa) & 255));
                        if (qb < q1) {
                            for (int cc = qa; cc <= qb; ++cc) c_s = __dadd_rn(c_s, row[cc]);
                            p.S[cg * p.nb + ((c_z + i0 + qb) >> 8)] = c_s;
                            window_add(win, c_s, sm.digits[cg]);
                            c_s = 0.0;
                            qa = qb + 1;
                        } else {
                            for (int cc = qa; cc < q1; ++cc) c_s = __dadd_rn(c_s, row[cc]);
                            qa = q1;
                        }
                    }
                }
                __syncwarp();
                named_arrive(kNormEmpty0 + b, kNormSync);
            }
            if (c_len > 0 && c_hi == c_len && c_lo < c_hi) {  // this CTA ran the row's end
                const uint64_t end = c_z + c_len;
                if ((end & 255) != 0) {
                    if (end == p.N) {  // the final (partial) block of Z_N
                        p.S[cg * p.nb + ((p.N - 1) >> 8)] = c_s;
                        window_add(win, c_s, sm.digits[cg]);
                    } else {
                        p.tail[tile_row_succ(j0 + cr, p) * 2 + cg] = c_s;
                    }
                }
            }
        }
        window_flush(win, sm.digits[cg]);
    }
    if (kProbs) {
        __syncthreads();
        write_partials(sm.digits, p.partials + uint64_t(blockIdx.x) * 2 * kDigits, tid);
    }
#ifdef SHS_CTA_TRACE
    __syncthreads();
    if (tid == 0) {
        uint64_t t1;
        uint32_t smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        printf("CTA %d %d %d sm %u t0 %llu t1 %llu\n", int(kProbs), int(kSplit), blockIdx.x, smid,
               (unsigned long long)trace_t0, (unsigned long long)t1);
    }
#endif
}

// The block straddling the boundary between a row and its z-order predecessor:
// S_b = fold(predecessor's tail partial, this row's head norms), in z order.
// Each warp takes 32 (row, group) items at a time and walks their head runs
// (<= 255 norms each) in 32-column slabs: for every item the warp loads the
// slab's 32 norms coalesced (256 B), transposes them through a padded
// shared-memory tile, and lane i folds item i's 32 values in order — 32 serial
// chains per warp, every warp of the CTA folding.
constexpr int kFixWarps = 8;
constexpr int kFixStride = 33;  // doubles per transposed row (+1: conflict-free lanes)
constexpr size_t kFixSmem = sizeof(double) * kFixWarps * 32 * kFixStride;

static __global__ void __launch_bounds__(32 * kFixWarps, 2) k_tile_fixup(TileParams p, unsigned long long* slots) {
    extern __shared__ double fix_buf[];  // [kFixWarps][32][kFixStride]
    __shared__ unsigned long long digits[2][kDigits];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 2 * kDigits; i += blockDim.x) (&digits[0][0])[i] = 0ull;
    __syncthreads();
    double* buf = fix_buf + warp * 32 * kFixStride;
    DigitWindow win;
    window_reset(win);
    const int g = lane & 1;  // item base + lane has group (base + lane) & 1, base even
    const uint64_t items = 2 * p.H;
    for (uint64_t base = (uint64_t(blockIdx.x) * kFixWarps + warp) * 32; base < items;
         base += uint64_t(gridDim.x) * kFixWarps * 32) {
        const uint64_t idx = base + lane;
        uint32_t hl = 0;
        uint64_t z = 0;
        if (idx < items) {
            z = mulmod_shoup(idx >> 1, p.A, p.A_sh, p.N);
            hl = static_cast<uint32_t>((256 - (z & 255)) & 255);
        }
        double s = hl ? p.tail[idx] : 0.0;  // tail[j * 2 + g]
        const uint32_t maxhl = __reduce_max_sync(0xffffffffu, hl);
        // slab c0 of every item, lane = column: loaded one slab ahead of the fold
        double v[32];
        auto load_slab = [&](uint32_t c0) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const uint32_t hli = __shfl_sync(0xffffffffu, hl, i);
                v[i] = c0 + lane < hli ? p.head[(base + i) * 256 + c0 + lane] : 0.0;
            }
        };
        if (maxhl) load_slab(0);
        for (uint32_t c0 = 0; c0 < maxhl; c0 += 32) {
#pragma unroll
            for (int i = 0; i < 32; ++i) buf[i * kFixStride + lane] = v[i];
            __syncwarp();
            if (c0 + 32 < maxhl) load_slab(c0 + 32);
            const double* row = buf + lane * kFixStride;
#pragma unroll 8
            for (int cc = 0; cc < 32; ++cc) {
                const double x = row[cc];
                if (c0 + cc < hl) s = __dadd_rn(s, x);
            }
            __syncwarp();
        }
        if (hl) {
            p.S[g * p.nb + (z >> 8)] = s;
            window_add(win, s, digits[g]);
        }
    }
    window_flush(win, digits[g]);
    __syncthreads();
    write_partials(digits, slots + uint64_t(blockIdx.x) * 2 * kDigits, tid);
}

// k_tile_fixup for plans with few rows (2 H <= 32 x kFix1Ctas x SMs: config 3's
// 1536-row plans): one warp per CTA stages all of its 32 items' heads in shared
// memory with one round of 16 B cp.async copies, then each lane folds its item in
// order. The 8-warp kernel streams the heads slab by slab (32 columns, one slab
// in flight), a chain of up to 8 memory latencies per warp that set its time
// when there are too few warps to fill the GPU.
constexpr int kFix1Stride = 258;  // doubles per staged head (16 B aligned rows)
constexpr size_t kFix1Smem = sizeof(double) * 32 * kFix1Stride;
constexpr int kFix1Ctas = 3;      // per SM (66 KB of shared memory each)
static __global__ void __launch_bounds__(32) k_tile_fixup1(TileParams p, unsigned long long* slots) {
    extern __shared__ double fix1_buf[];  // [32][kFix1Stride]
    __shared__ unsigned long long digits[2][kDigits];
    const int lane = threadIdx.x;
    // launched as a programmatic dependent of k_tiled: wait for its heads,
    // tails and partials; the finalize may be scheduled right away
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    for (int i = lane; i < 2 * kDigits; i += 32) (&digits[0][0])[i] = 0ull;
    __syncwarp();
    DigitWindow win;
    window_reset(win);
    const int g = lane & 1;  // item base + lane has group (base + lane) & 1, base even
    const uint64_t items = 2 * p.H;
    for (uint64_t base = uint64_t(blockIdx.x) * 32; base < items; base += uint64_t(gridDim.x) * 32) {
        const uint64_t idx = base + lane;
        uint32_t hl = 0;
        uint64_t z = 0;
        if (idx < items) {
            z = mulmod_shoup(idx >> 1, p.A, p.A_sh, p.N);
            hl = static_cast<uint32_t>((256 - (z & 255)) & 255);
        }
        double s = hl ? p.tail[idx] : 0.0;  // tail[j * 2 + g]
        // item i's first hl values (pairs: the odd one past hl is never read)
        for (int i = 0; i < 32; ++i) {
            const uint32_t hli = __shfl_sync(0xffffffffu, hl, i);
            const double* src = p.head + (base + i) * 256;
            for (uint32_t c = 2 * lane; c < hli; c += 64) cp_async16(&fix1_buf[i * kFix1Stride + c], src + c);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        const double* row = fix1_buf + lane * kFix1Stride;
        for (uint32_t c = 0; c < hl; ++c) s = __dadd_rn(s, row[c]);
        if (hl) {
            p.S[g * p.nb + (z >> 8)] = s;
            window_add(win, s, digits[g]);
        }
        __syncwarp();  // the row reads end before the next items' copies
    }
    window_flush(win, digits[g]);
    __syncwarp();
    write_partials(digits, slots + uint64_t(blockIdx.x) * 2 * kDigits, lane);
}

}  // namespace shs
