// Host-side tile planning for the sorted-residue permutation tiles (tiled.cuh),
// shared by the single-GPU engine and the sharded engine.
#pragma once

#include <algorithm>
#include <cstdint>
#include <vector>

#include "../../include/shorsim_b200.h"
#include "host_model.hpp"
#include "tiled.cuh"

namespace shs {

inline constexpr double kDegenerateMass = 1e-300;  // statevector.cpp:19
inline constexpr uint64_t kKahanMaxBlocks = 1024;  // AUTO: sequential Kahan up to 2^18 amplitudes
inline constexpr uint64_t kTileAutoMinN = 1ull << 20;  // AUTO tiling from 16 MB of state
inline constexpr uint64_t kTileMinRow = 512;           // every 256-block touches <= 2 rows
#ifndef SHS_TILE_MAX_ROWS
#define SHS_TILE_MAX_ROWS (1ull << 18)
#endif
inline constexpr uint64_t kTileMaxRows = SHS_TILE_MAX_ROWS;  // head scratch <= 1 GB
inline constexpr uint64_t kTileMinRowsPlan = 256;      // >= 8 tiles of kRows rows
#ifndef SHS_TILE_AVG_ROW
#define SHS_TILE_AVG_ROW 640
#endif
#ifndef SHS_TILE_MIN_CHUNKS
#define SHS_TILE_MIN_CHUNKS 16
#endif
inline constexpr uint64_t kTileAvgRow = SHS_TILE_AVG_ROW;  // H <= N / kTileAvgRow
#ifndef SHS_TILE_TARGET_ROW
#define SHS_TILE_TARGET_ROW 8192
#endif
inline constexpr uint64_t kTileTargetRow = SHS_TILE_TARGET_ROW;  // preferred mean row length
// AUTO mode keeps the direct kernels when a plan has fewer chunks than this many
// per CTA (a CTA's range cut costs up to 256 / kCols partly masked chunks)
inline constexpr uint64_t kTileMinChunksPerCTA = SHS_TILE_MIN_CHUNKS;
// plans with at least this many bands per CTA run whole bands round-robin only
inline constexpr uint64_t kTileRoundRobinBands = 16;

// Host side of a stage's sorted-residue tiling (see tiled.cuh).
struct TilePlanHost {
    bool tiled = false;
    uint64_t H = 0, u = 0, v = 0, du = 0, dv = 0;
    uint64_t A = 0, A_sh = 0, m = 0, m_sh = 0, ntiles = 0;
    uint64_t chunks = 0;          // kRows x kCols chunks over all bands
    int grid = 0;                 // CTAs of k_tiled
    uint64_t bulk_rounds = 0;     // whole bands per CTA, round-robin
    bool split_tail = true;       // k_tiled<., true>: balanced remainder ranges
    std::vector<uint32_t> split;  // [grid + 1] x (band, chunk): each CTA's remainder range
};

// Longest row of band b (its chunk count is this / kCols, rounded up): rows
// j < H - u have length du, rows in [H - u, v) du + dv, the rest dv.
inline uint64_t tile_band_len(const TilePlanHost& pl, uint64_t b) {
    const uint64_t j0 = b * kRows, j1 = std::min<uint64_t>(j0 + kRows, pl.H);
    const uint64_t hu = pl.H - pl.u, vb = std::max(pl.v, hu);
    uint64_t mx = 0;
    if (j0 < hu) mx = std::max(mx, pl.du);
    if (j0 < pl.v && j1 > hu && hu < pl.v) mx = std::max(mx, pl.du + pl.dv);
    if (j1 > vb) mx = std::max(mx, pl.dv);
    return mx;
}

// Work split of the tiled kernels over `cap` CTAs (tiled.cuh, CtaWork): whole
// bands round-robin for floor(ntiles / cap) rounds, then the remaining bands'
// chunks, band-major, cut into cap contiguous ranges of equal size (within one
// chunk). Without full rounds the grid shrinks to the chunk count if smaller.
inline void make_tile_split(TilePlanHost& pl, int cap) {
    uint64_t G = static_cast<uint64_t>(cap);
    pl.split_tail = pl.ntiles < kTileRoundRobinBands * G;
    pl.bulk_rounds = pl.ntiles / G;
    const uint64_t b0 = std::min(pl.bulk_rounds * G, pl.ntiles);
    std::vector<uint64_t> pre(pl.ntiles - b0 + 1, 0);
    pl.chunks = 0;
    for (uint64_t b = 0; b < pl.ntiles; ++b) {
        const uint64_t nch = (tile_band_len(pl, b) + kCols - 1) / kCols;
        pl.chunks += nch;
        if (b >= b0) pre[b - b0 + 1] = pre[b - b0] + nch;
    }
    const uint64_t T = pre.back();
    if (pl.bulk_rounds == 0) G = std::min<uint64_t>(G, T);
    pl.grid = static_cast<int>(G);
    pl.split.assign(2 * (G + 1), 0);
    uint64_t b = 0;
    for (uint64_t g = 0; g <= G; ++g) {
        const uint64_t C = g * T / G;
        while (b < pl.ntiles - b0 && pre[b + 1] <= C) ++b;
        pl.split[2 * g] = static_cast<uint32_t>(b0 + b);
        pl.split[2 * g + 1] = static_cast<uint32_t>(C - pre[b]);
    }
}

// Pick a row count H (powers of two and 3 * 2^k up to N / kTileAvgRow) whose
// three gap lengths are all >= kTileMinRow and at most 3x the mean row, the
// largest such H <= N / kTileTargetRow or else the smallest above it: one
// O(H) scan of j*A mod N with running argmin / argmax gives u(H), v(H) for
// every candidate. Multipliers without such an H (tiny A, or A/N with a huge
// partial quotient) keep the direct gather, whose warps then read a few long
// runs anyway.
// Small multipliers (kTileMinRow <= A, N / A > the scan's row cap): the rows
// z_j = j A are the consecutive A-long runs of Z_N (u = 1, v = H - 1, the last
// row A + N mod A long), H = floor(N / A). The tile is then the same
// 32-row x 32-column transpose (gathered runs j..j+31 + i m); the price is one
// head run per row in the fixup scratch (H x 4 KB), so the single engine takes
// it only while that scratch stays within max_scratch bytes.
inline TilePlanHost make_small_a_plan(uint64_t A, uint64_t m, uint64_t N, uint64_t max_scratch) {
    TilePlanHost pl;
    if (A < kTileMinRow || A >= N / kTileMinRowsPlan) return pl;
    const uint64_t H = N / A;
    if (H <= kTileMaxRows || H * 2 * 257 * sizeof(double) > max_scratch) return pl;
    pl.tiled = true;
    pl.H = H;
    pl.u = 1;
    pl.v = H - 1;
    pl.du = A;
    pl.dv = A + N % A;
    pl.A = A;
    pl.A_sh = shoup(A, N);
    pl.m = m;
    pl.m_sh = shoup(m, N);
    pl.ntiles = (pl.H + kRows - 1) / kRows;
    return pl;
}

inline TilePlanHost make_tile_plan(uint64_t A, uint64_t m, uint64_t N, int tiling,
                                   uint64_t small_a_scratch = 0,
                                   uint64_t max_rows = kTileMaxRows) {
    TilePlanHost pl;
    if (tiling == SHS_TILING_OFF || A == 1) return pl;
    if (tiling == SHS_TILING_AUTO && N < kTileAutoMinN) return pl;
    if (small_a_scratch) {
        pl = make_small_a_plan(A, m, N, small_a_scratch);
        if (pl.tiled) return pl;
    }
    const uint64_t hmax = std::min<uint64_t>(N / kTileAvgRow, max_rows);
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
        // prefer rows of about kTileTargetRow (fewer rows: fewer heads to fix up):
        // the largest valid H <= N / kTileTargetRow, else the smallest valid H
        if (H >= kTileMinRowsPlan && du >= kTileMinRow && dv >= kTileMinRow &&
            du + dv <= 3 * (N / H + 1) && du + dv < (1ull << 31) &&  // 32-bit row spans
            (!pl.tiled || H * kTileTargetRow <= N)) {
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

}  // namespace shs
