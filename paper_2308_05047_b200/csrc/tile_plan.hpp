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
inline constexpr uint64_t kTileMaxRows = 1ull << 18;   // head scratch <= 1 GB
inline constexpr uint64_t kTileMinRowsPlan = 256;      // >= 8 tiles of kRows rows
#ifndef SHS_TILE_AVG_ROW
#define SHS_TILE_AVG_ROW 640
#endif
#ifndef SHS_TILE_MIN_TILES
#define SHS_TILE_MIN_TILES 1
#endif
inline constexpr uint64_t kTileAvgRow = SHS_TILE_AVG_ROW;  // H <= N / kTileAvgRow
// AUTO mode keeps the direct kernels when a plan has fewer tiles than this
// multiple of the SM count (too few tiles leave SMs idle: one CTA per tile row set)
inline constexpr uint64_t kTileMinTilesPerSM = SHS_TILE_MIN_TILES;

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
inline TilePlanHost make_tile_plan(uint64_t A, uint64_t m, uint64_t N, int tiling) {
    TilePlanHost pl;
    if (tiling == SHS_TILING_OFF || A == 1) return pl;
    if (tiling == SHS_TILING_AUTO && N < kTileAutoMinN) return pl;
    const uint64_t hmax = std::min<uint64_t>(N / kTileAvgRow, kTileMaxRows);
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

}  // namespace shs
