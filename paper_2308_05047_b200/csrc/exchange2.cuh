// Sharded exchange, version 2: an all-to-all at the minimum link volume.
//
// Exchange v1 (exchange.cuh) has a third rank execute each tile: it pulls the
// tile's 32 source runs from their owners and pushes its 32 row runs to theirs,
// so an element crosses NVLink twice (2 x 16 B (N/G)(G-1)/G per GPU and
// direction). Here every element crosses once, sender -> receiver, and both HBM
// sides stay coalesced:
//
//   pack (sender q)   for every band b of the stage's tile plan and every
//                     32-column chunk, reads the source column runs it owns
//                     (sel[j + i m], 512 B runs of its own shard), and writes
//                     each element to the stream of the rank r owning its
//                     destination z = z_j + i, in the canonical order
//                     (band, column i, row k) — contiguous runs of the stream
//                     in r's receive buffer (peer stores over NVLink)
//   unpack (receiver) walks the same bands and chunks, takes each of its
//                     elements from the stream of the rank owning its source
//                     (local, contiguous per stream), transposes the chunk in
//                     shared memory and stores its row runs P[z] (coalesced)
//
// Both sides derive every stream position from the plan alone: for band b the
// pair (q -> r) owns count(b, q, r) consecutive stream slots starting at the
// exclusive prefix off(b, q, r) over bands (k_x2_count + a scan, computed once
// per engine and stage: the plan is data-independent), and inside a band the
// canonical order is column-major, ranked with warp ballots. Bands are split
// into K rounds so the receive buffer (two round slots) fits next to sel and P;
// pack of round g+1 (its own stream) overlaps unpack of round g.
#pragma once

#include "exchange.cuh"
#include "tiled.cuh"

namespace shs {

constexpr int kX2Warps = 4;  // one band per warp
constexpr int kX2Threads = 32 * kX2Warps;

struct X2Params {
    TileParams tp;          // plan (A, m, H, u, v, du, dv, ntiles); X / Y unused
    uint64_t S, S_inv;      // shard size, floor((2^64-1)/S)
    uint64_t N;
    int G, me;
    uint64_t b0, b1;        // bands of this round
    const double2* sel;     // pack: this shard's sel (local index)
    double2* P;             // unpack: this shard's P (local index)
    // pack: stream (me -> r) of this round in r's receive slot (round-relative:
    // band b's elements start at dst[r] + off(b, me, r) - off(b0, me, r))
    double2* dst[kMaxShards];
    // unpack: stream (q -> me) of this round in this shard's receive slot
    const double2* src[kMaxShards];
    // off[(peer) * (nbands + 1) + b]: pack = off(b, me, peer), unpack = off(b, peer, me)
    const unsigned long long* off;
    uint64_t mstep[33];     // c * m mod N, c <= 32 (host-computed)
};

__device__ __forceinline__ int x2_owner(uint64_t x, uint64_t S, uint64_t S_inv) {
    uint64_t q = __umul64hi(x, S_inv);
    if (x - q * S >= S) ++q;
    return static_cast<int>(q);
}

// The warp's band: lane k holds row j0 + k — its start z, length, the owner of
// its first element and the column where the owner changes (rows are shorter
// than a shard: at most one change; ~0 when none).
struct X2Row {
    uint64_t z, len, cut;
    int own;
};

__device__ __forceinline__ X2Row x2_row(const X2Params& p, uint64_t j) {
    X2Row r;
    r.len = tile_row_len(j, p.tp);
    r.z = r.len ? mulmod_shoup(j, p.tp.A, p.tp.A_sh, p.N) : 0;
    r.own = x2_owner(r.z, p.S, p.S_inv);
    const uint64_t end = (uint64_t(r.own) + 1) * p.S;  // first index of the next shard
    r.cut = r.z + r.len > end ? end - r.z : ~0ull;
    return r;
}

__device__ __forceinline__ uint64_t warp_max(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

// Pack side of band b, canonical order (column i ascending, then row k): the
// columns whose 32-element source run touches this shard, kX2Batch at a time
// (their loads issued together); lane k takes element (k, i). A row's
// destination rank only changes at its cut column, so the lanes' destination
// groups (match_any over the rows) are recomputed only when a cut is passed;
// per column the group is that mask & the column's ballot of live elements.
// `emit(n, live[], r[], grp[], v[])` sees each batch of n columns (r: this
// lane's row's rank).
constexpr int kX2Batch = 8;

template <typename Emit>
__device__ __forceinline__ void x2_pack_band(const X2Params& p, uint64_t b, bool load, Emit&& emit) {
    const int lane = threadIdx.x & 31;
    const uint64_t j0 = b * kRows;
    const X2Row row = x2_row(p, j0 + lane);
    const uint64_t maxlen = warp_max(row.len);
    const uint64_t lo = uint64_t(p.me) * p.S, hi = lo + p.S;
    const uint64_t m32 = p.mstep[32];  // source advance per 32 columns
    // lane c: the source run start of column i0 + c
    uint64_t cs = addmod(j0, p.mstep[lane], p.N);
    // destination groups valid for columns below next_cut
    uint64_t next_cut = 0;
    int r = 0;
    unsigned rowgrp = 0;
    unsigned pend = 0;      // touched columns of the current 32-column group not yet emitted
    uint64_t pend_i0 = 0;
    unsigned whole = 0;
    uint64_t pend_cs = cs;
    uint64_t i0 = 0;
    bool live[kX2Batch];
    double2 v[kX2Batch];
    unsigned grp[kX2Batch];
    int rr[kX2Batch];
    int n = 0;
    // gather kX2Batch touched columns (possibly from several 32-column groups),
    // then emit; every guard below is warp-uniform
    while (true) {
        while (!pend && i0 < maxlen) {  // next group with touched columns
            const uint64_t last = cs + (kRows - 1) >= p.N ? cs + (kRows - 1) - p.N : cs + (kRows - 1);
            const bool in0 = cs >= lo && cs < hi, in1 = last >= lo && last < hi;
            pend = __ballot_sync(0xffffffffu, i0 + lane < maxlen && (in0 || in1));
            whole = __ballot_sync(0xffffffffu, in0 && in1 && last > cs);  // no straddle
            pend_i0 = i0;
            pend_cs = cs;
            i0 += 32;
            cs = addmod(cs, m32, p.N);
        }
        if (!pend && n == 0) break;
        if (pend) {
            const int c = __ffs(pend) - 1;
            pend &= pend - 1;
            const uint64_t i = pend_i0 + c;
            const uint64_t c0 = __shfl_sync(0xffffffffu, pend_cs, c);
            uint64_t s = c0 + lane;
            if (s >= p.N) s -= p.N;
            const bool lv = i < row.len && (((whole >> c) & 1u) || (s >= lo && s < hi));
            if (i >= next_cut) {  // regroup the rows by destination
                r = row.own + (i >= row.cut ? 1 : 0);
                rowgrp = __match_any_sync(0xffffffffu, r);
                uint64_t nc = row.cut > i && row.cut < row.len ? row.cut : ~0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const uint64_t w = __shfl_xor_sync(0xffffffffu, nc, o);
                    nc = w < nc ? w : nc;
                }
                next_cut = nc;
            }
            const unsigned g = rowgrp & __ballot_sync(0xffffffffu, lv);
            const double2 val = load && lv ? __ldg(p.sel + (s - lo)) : make_double2(0.0, 0.0);
#pragma unroll
            for (int t = 0; t < kX2Batch; ++t)
                if (t == n) {
                    live[t] = lv;
                    grp[t] = g;
                    rr[t] = r;
                    v[t] = val;
                }
            ++n;
        }
        if (n == kX2Batch || (!pend && i0 >= maxlen)) {
            emit(n, live, rr, grp, v);
            n = 0;
        }
    }
}

// Unpack side of band b: this shard's rows of the band, compacted onto the
// lanes (lane L: row my[L % m], column offset L / m), so a warp step covers cpi
// columns (the largest power of two with cpi * m <= 32, so steps tile 32-column
// chunks) in canonical order (column, then row).
struct X2Lanes {
    unsigned rows;           // ballot of the band's rows with elements of this shard
    int m, cpi, ri, coff, k; // k: this lane's row (the ri-th set bit of rows)
    bool on;                 // lane < cpi * m
    uint64_t z, len, cut;    // row k
    int own;
};

// Walks the band in 32-column chunks. A chunk is "regular" when every one of its
// columns is inside every row of this shard (no band tail, no cut) and each
// column's source elements of those rows come from one sender q (no shard
// boundary or wrap inside the column's run): then the column holds m
// consecutive slots of q's stream and `fast(i0, q, L)` (lane c: column i0 + c)
// serves the chunk. Otherwise the chunk goes step by step through
// `take(n, mine[], q[], grp[], z[])`, kX2SlowBatch steps per call.
constexpr int kX2SlowBatch = 1;  // steps per take() call (irregular chunks only)

template <typename Fast, typename Take>
__device__ __forceinline__ void x2_unpack_band(const X2Params& p, uint64_t b, Fast&& fast,
                                               Take&& take) {
    const int lane = threadIdx.x & 31;
    const uint64_t j0 = b * kRows;
    const X2Row row = x2_row(p, j0 + lane);
    const bool has = row.len && (row.own == p.me || (row.cut != ~0ull && row.own + 1 == p.me));
    X2Lanes L;
    L.rows = __ballot_sync(0xffffffffu, has);
    if (!L.rows) return;
    L.m = __popc(L.rows);
    L.cpi = 1;
    while (L.cpi * 2 * L.m <= 32) L.cpi *= 2;
    L.ri = lane % L.m;
    L.coff = lane / L.m;
    L.on = lane < L.cpi * L.m;
    {
        unsigned rr = L.rows;
        for (int t = 0; t < L.ri; ++t) rr &= rr - 1;
        L.k = __ffs(rr) - 1;
    }
    L.z = __shfl_sync(0xffffffffu, row.z, L.k);
    L.len = __shfl_sync(0xffffffffu, row.len, L.k);
    L.cut = __shfl_sync(0xffffffffu, row.cut, L.k);
    L.own = __shfl_sync(0xffffffffu, row.own, L.k);
    const uint64_t maxlen = warp_max(has ? row.len : 0);
    // columns [rlo, rhi) are this shard's in every one of its rows
    uint64_t rlo = !has ? 0 : row.own == p.me ? 0 : row.cut;
    uint64_t rhi = !has ? ~0ull : row.own == p.me ? (row.cut < row.len ? row.cut : row.len) : row.len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t a = __shfl_xor_sync(0xffffffffu, rlo, o);
        const uint64_t c = __shfl_xor_sync(0xffffffffu, rhi, o);
        rlo = a > rlo ? a : rlo;
        rhi = c < rhi ? c : rhi;
    }
    const int kmin = __ffs(L.rows) - 1, kmax = 31 - __clz(L.rows);
    uint64_t cc = addmod(j0, p.mstep[lane], p.N);  // lane c: source run start of column i0 + c
    const uint64_t m32 = p.mstep[32];
    const int steps = kCols / L.cpi;
    bool mine[kX2SlowBatch];
    int qq[kX2SlowBatch];
    unsigned grp[kX2SlowBatch];
    uint64_t zz[kX2SlowBatch];
    for (uint64_t i0 = 0; i0 < maxlen; i0 += kCols) {
        const uint64_t i = i0 + lane;
        const int q = x2_owner(cc + kmin, p.S, p.S_inv);
        const bool reg = i >= rlo && i < rhi && cc + kmax < p.N &&
                         x2_owner(cc + kmax, p.S, p.S_inv) == q;
        if (__all_sync(0xffffffffu, reg)) {
            fast(i0, q, L);
        } else {
            for (int t0 = 0; t0 < steps; t0 += kX2SlowBatch) {
                int n = 0;
#pragma unroll
                for (int t = 0; t < kX2SlowBatch; ++t) {
                    const int c = (t0 + t) * L.cpi + L.coff;
                    const uint64_t ic = i0 + c;
                    uint64_t s = __shfl_sync(0xffffffffu, cc, c & 31) + L.k;
                    if (s >= p.N) s -= p.N;
                    const bool mn = t0 + t < steps && L.on && ic < L.len &&
                                    L.own + (ic >= L.cut ? 1 : 0) == p.me;
                    qq[t] = mn ? x2_owner(s, p.S, p.S_inv) : -1;
                    mine[t] = mn;
                    grp[t] = __match_any_sync(0xffffffffu, qq[t]);
                    zz[t] = L.z + ic;
                    if (t0 + t < steps && i0 + uint64_t(t0 + t) * L.cpi < maxlen) n = t + 1;
                }
                if (n) take(n, mine, qq, grp, zz);
            }
        }
        cc = addmod(cc, m32, p.N);
    }
}

// count(b, me, r) (kSend) or count(b, q, me) for every band, into
// counts[peer * (nbands + 1) + b]
template <bool kSend>
__global__ void __launch_bounds__(kX2Threads) k_x2_count(X2Params p,
                                                         unsigned long long* __restrict__ counts) {
    __shared__ unsigned int cnt[kX2Warps][kMaxShards];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t nb = p.tp.ntiles;
    for (uint64_t b = uint64_t(blockIdx.x) * kX2Warps + warp; b < nb;
         b += uint64_t(gridDim.x) * kX2Warps) {
        if (lane < kMaxShards) cnt[warp][lane] = 0;
        __syncwarp();
        auto add = [&](int n, const bool* mine, const int* peer, const unsigned* grp) {
#pragma unroll
            for (int t = 0; t < kX2Batch; ++t)
                if (t < n && mine[t] && (grp[t] & ((1u << lane) - 1)) == 0)
                    atomicAdd(&cnt[warp][peer[t]], __popc(grp[t]));
            __syncwarp();
        };
        if (kSend)
            x2_pack_band(p, b, false, [&](int n, const bool* live, const int* r,
                                          const unsigned* grp, const double2*) {
                add(n, live, r, grp);
            });
        else
            x2_unpack_band(
                p, b,
                [&](uint64_t, int q, const X2Lanes& L) {  // m elements per column from q
                    const unsigned g = __match_any_sync(0xffffffffu, q);
                    if ((g & ((1u << lane) - 1)) == 0) atomicAdd(&cnt[warp][q], L.m * __popc(g));
                    __syncwarp();
                },
                [&](int n, const bool* mine, const int* q, const unsigned* grp, const uint64_t*) {
                    add(n, mine, q, grp);
                });
        __syncwarp();
        if (lane < p.G) counts[uint64_t(lane) * (nb + 1) + b] = cnt[warp][lane];
        __syncwarp();
    }
}

// pack: this shard's source elements of the round's bands into the receivers'
// streams. Per band a row's destination rank only changes at its cut column,
// so for a "regular" column (its source run inside this shard, every live row
// still running, no cut passed) every lane's stream slot just advances by its
// destination group's size: the fast path is a load and a store per element
// (kX2Batch columns' loads in flight). Other columns (band tails, run
// straddles, cuts) take the general path; both write the canonical order.
__global__ void __launch_bounds__(kX2Threads) k_x2_pack(X2Params p) {
    __shared__ unsigned long long pos[kX2Warps][kMaxShards];  // next slot per receiver
    __shared__ double2* dstp[kMaxShards];  // (dynamically indexed: shared, not param space)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x < kMaxShards) dstp[threadIdx.x] = p.dst[threadIdx.x];
    __syncthreads();
    const uint64_t nb = p.tp.ntiles;
    const uint64_t lo = uint64_t(p.me) * p.S, hi = lo + p.S;
    const unsigned lt = (1u << lane) - 1;
    for (uint64_t b = p.b0 + uint64_t(blockIdx.x) * kX2Warps + warp; b < p.b1;
         b += uint64_t(gridDim.x) * kX2Warps) {
        if (lane < p.G) {
            const unsigned long long* o = p.off + uint64_t(lane) * (nb + 1);
            pos[warp][lane] = o[b] - o[p.b0];
        }
        __syncwarp();
        const uint64_t j0 = b * kRows;
        const X2Row row = x2_row(p, j0 + lane);
        const uint64_t maxlen = warp_max(row.len);
        uint64_t minlen = row.len ? row.len : ~0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t w = __shfl_xor_sync(0xffffffffu, minlen, o);
            minlen = w < minlen ? w : minlen;
        }
        const unsigned base = __ballot_sync(0xffffffffu, row.len > 0);
        // destination groups (valid below next_cut) and the fast-path pointer
        uint64_t next_cut = 0;
        int r = 0;
        unsigned rowgrp = 0, gsize = 0, rank = 0;
        double2* ptr = nullptr;
        uint64_t nreg = 0;  // regular columns written since pos was last updated
        auto flush = [&]() {  // fold the fast path's advance into pos
            if (nreg) {
                if (row.len && (rowgrp & base & lt) == 0) pos[warp][r] += nreg * gsize;
                nreg = 0;
            }
            __syncwarp();
        };
        auto regroup = [&](uint64_t i) {  // rows -> destination groups at column i
            r = row.own + (i >= row.cut ? 1 : 0);
            rowgrp = __match_any_sync(0xffffffffu, row.len ? r : -1);
            uint64_t nc = row.cut > i && row.cut < row.len ? row.cut : ~0ull;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const uint64_t w = __shfl_xor_sync(0xffffffffu, nc, o);
                nc = w < nc ? w : nc;
            }
            next_cut = nc;
            gsize = __popc(rowgrp & base);
            rank = __popc(rowgrp & base & lt);
        };
        auto repoint = [&]() {
            ptr = row.len ? dstp[r] + pos[warp][r] + rank : nullptr;
        };
        uint64_t cs = addmod(j0, p.mstep[lane], p.N);  // lane c: source run of column i0 + c
        for (uint64_t i0 = 0; i0 < maxlen; i0 += 32) {
            const uint64_t last = cs + (kRows - 1) >= p.N ? cs + (kRows - 1) - p.N : cs + (kRows - 1);
            const bool in0 = cs >= lo && cs < hi, in1 = last >= lo && last < hi;
            unsigned cols = __ballot_sync(0xffffffffu, i0 + lane < maxlen && (in0 || in1));
            const unsigned whole = __ballot_sync(0xffffffffu, in0 && in1 && last > cs);
            while (cols) {
                int ci[kX2Batch];
                int n = 0;
                bool regular = true;
#pragma unroll
                for (int t = 0; t < kX2Batch; ++t) {
                    ci[t] = cols ? __ffs(cols) - 1 : -1;
                    if (ci[t] >= 0) {
                        cols &= cols - 1;
                        n = t + 1;
                        const uint64_t i = i0 + ci[t];
                        regular = regular && ((whole >> ci[t]) & 1u) && i < minlen && i < next_cut;
                    }
                }
                if (regular) {  // all n columns: one load and one store per lane each
                    if (nreg == 0) repoint();
                    double2 v[kX2Batch];
#pragma unroll
                    for (int t = 0; t < kX2Batch; ++t)
                        if (t < n) {
                            const uint64_t c0 = __shfl_sync(0xffffffffu, cs, ci[t]);
                            uint64_t sx = c0 + lane;
                            if (sx >= p.N) sx -= p.N;
                            if (row.len) v[t] = __ldg(p.sel + (sx - lo));
                        }
#pragma unroll
                    for (int t = 0; t < kX2Batch; ++t)
                        if (t < n && row.len) {
                            *ptr = v[t];
                            ptr += gsize;
                        }
                    nreg += n;
                    continue;
                }
                flush();
#pragma unroll 1
                for (int t = 0; t < n; ++t) {  // the general path, column by column
                    const uint64_t i = i0 + ci[t];
                    if (i >= next_cut) regroup(i);
                    const uint64_t c0 = __shfl_sync(0xffffffffu, cs, ci[t]);
                    uint64_t sx = c0 + lane;
                    if (sx >= p.N) sx -= p.N;
                    const bool lv = i < row.len && sx >= lo && sx < hi;
                    const unsigned g = rowgrp & __ballot_sync(0xffffffffu, lv);
                    const unsigned below = g & lt;
                    if (lv) dstp[r][pos[warp][r] + __popc(below)] = __ldg(p.sel + (sx - lo));
                    __syncwarp();
                    if (lv && !below) pos[warp][r] += __popc(g);
                    __syncwarp();
                }
            }
            cs = addmod(cs, p.mstep[32], p.N);
        }
        flush();
    }
}

// unpack: this shard's destination elements of the round's bands from the
// senders' streams into P (a row's columns of one warp step are contiguous). In
// a regular chunk each column's m elements are consecutive in one stream: the
// column's stream pointer is ranked once per chunk, and a step is a shuffle, a
// load and a store per lane.
__global__ void __launch_bounds__(kX2Threads) k_x2_unpack(X2Params p) {
    __shared__ unsigned long long pos[kX2Warps][kMaxShards];  // next slot per sender
    __shared__ const double2* srcp[kMaxShards];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x < kMaxShards) srcp[threadIdx.x] = p.src[threadIdx.x];
    __syncthreads();
    const uint64_t nb = p.tp.ntiles;
    const uint64_t lo = uint64_t(p.me) * p.S;
    const unsigned lt = (1u << lane) - 1;
    for (uint64_t b = p.b0 + uint64_t(blockIdx.x) * kX2Warps + warp; b < p.b1;
         b += uint64_t(gridDim.x) * kX2Warps) {
        if (lane < p.G) {
            const unsigned long long* o = p.off + uint64_t(lane) * (nb + 1);
            pos[warp][lane] = o[b] - o[p.b0];
        }
        __syncwarp();
        x2_unpack_band(
            p, b,
            [&](uint64_t i0, int q, const X2Lanes& L) {
                const unsigned g = __match_any_sync(0xffffffffu, q);
                const unsigned below = g & lt;
                // lane c: the stream slot of column i0 + c's first element
                const unsigned long long col = reinterpret_cast<unsigned long long>(
                    srcp[q] + pos[warp][q] + uint64_t(L.m) * __popc(below));
                __syncwarp();
                if (!below) pos[warp][q] += uint64_t(L.m) * __popc(g);
                __syncwarp();
                double2* out = p.P + (L.z + i0 + L.coff - lo);
                const int steps = kCols / L.cpi;
                for (int t0 = 0; t0 < steps; t0 += kX2Batch) {
                    double2 v[kX2Batch];
#pragma unroll
                    for (int t = 0; t < kX2Batch; ++t) {
                        const unsigned long long c = __shfl_sync(
                            0xffffffffu, col, ((t0 + t) * L.cpi + L.coff) & 31);
                        if (L.on && t0 + t < steps)
                            v[t] = reinterpret_cast<const double2*>(c)[L.ri];
                    }
#pragma unroll
                    for (int t = 0; t < kX2Batch; ++t)
                        if (L.on && t0 + t < steps) out[(t0 + t) * L.cpi] = v[t];
                }
            },
            [&](int n, const bool* mine, const int* q, const unsigned* grp, const uint64_t* z) {
                unsigned long long at[kX2SlowBatch];
#pragma unroll
                for (int t = 0; t < kX2SlowBatch; ++t) {  // stream positions first (counters only) ...
                    if (t < n && mine[t]) {
                        const unsigned below = grp[t] & lt;
                        at[t] = pos[warp][q[t]] + __popc(below);
                        if (!below) pos[warp][q[t]] += __popc(grp[t]);
                    }
                    __syncwarp();
                }
                double2 v[kX2SlowBatch];
#pragma unroll
                for (int t = 0; t < kX2SlowBatch; ++t)  // ... then every load of the batch in flight
                    if (t < n && mine[t]) v[t] = srcp[q[t]][at[t]];
#pragma unroll
                for (int t = 0; t < kX2SlowBatch; ++t)
                    if (t < n && mine[t]) p.P[z[t] - lo] = v[t];
            });
        __syncwarp();
    }
}

}  // namespace shs
