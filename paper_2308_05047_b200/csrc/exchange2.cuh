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

constexpr int kX2Warps = 8;
constexpr int kX2Threads = 32 * kX2Warps;
constexpr int kX2ColsPerWarp = kCols / kX2Warps;  // 4 columns of a 32-column chunk per warp

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
};

__device__ __forceinline__ int x2_owner(uint64_t x, uint64_t S, uint64_t S_inv) {
    uint64_t q = __umul64hi(x, S_inv);
    if (x - q * S >= S) ++q;
    return static_cast<int>(q);
}

// The rows of band b: z (start), len, the owner of its first element and the
// column where the owner changes (rows are shorter than a shard: at most one
// change; ~0 when none).
struct X2Rows {
    uint64_t z[kRows], len[kRows], cut[kRows];
    int own[kRows];
    uint64_t maxlen;
};

__device__ __forceinline__ void x2_load_rows(const X2Params& p, uint64_t b, X2Rows& R) {
    const int t = threadIdx.x;
    if (t < kRows) {
        const uint64_t j = b * kRows + t;
        const uint64_t len = tile_row_len(j, p.tp);
        const uint64_t z = len ? mulmod_shoup(j, p.tp.A, p.tp.A_sh, p.N) : 0;
        R.z[t] = z;
        R.len[t] = len;
        const int o = x2_owner(z, p.S, p.S_inv);
        R.own[t] = o;
        const uint64_t end = (uint64_t(o) + 1) * p.S;  // first index of the next shard
        R.cut[t] = z + len > end ? end - z : ~0ull;
    }
    __syncthreads();
    if (t == 0) {
        uint64_t mx = 0;
        for (int k = 0; k < kRows; ++k) mx = R.len[k] > mx ? R.len[k] : mx;
        R.maxlen = mx;
    }
    __syncthreads();
}

// (src owner, dst owner) of element (k, i): valid == false past the row's end
struct X2Elem {
    bool valid;
    int qs, rd;
    uint64_t src;
};

__device__ __forceinline__ X2Elem x2_elem(const X2Params& p, const X2Rows& R, uint64_t col_src,
                                          int k, uint64_t i) {
    X2Elem e;
    e.valid = i < R.len[k];
    uint64_t s = col_src + k;  // (j0 + i m + k) mod N, col_src < N
    if (s >= p.N) s -= p.N;
    e.src = s;
    e.qs = x2_owner(s, p.S, p.S_inv);
    e.rd = R.own[k] + (i >= R.cut[k] ? 1 : 0);
    return e;
}

// count(b, me, r) (kSend) or count(b, q, me) for every band of the plan, into
// counts[peer * (nbands + 1) + b]
template <bool kSend>
__global__ void __launch_bounds__(kX2Threads) k_x2_count(X2Params p,
                                                         unsigned long long* __restrict__ counts) {
    __shared__ X2Rows R;
    __shared__ unsigned int cnt[kMaxShards];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t nb = p.tp.ntiles;
    for (uint64_t b = blockIdx.x; b < nb; b += gridDim.x) {
        if (threadIdx.x < kMaxShards) cnt[threadIdx.x] = 0;
        x2_load_rows(p, b, R);
        const uint64_t j0 = b * kRows;
        for (uint64_t i = warp; i < R.maxlen; i += kX2Warps) {
            const uint64_t cs = addmod(j0, mulmod_shoup(i, p.tp.m, p.tp.m_sh, p.N), p.N);
            const X2Elem e = x2_elem(p, R, cs, lane, i);
            const bool mine = e.valid && (kSend ? e.qs == p.me : e.rd == p.me);
            const int peer = mine ? (kSend ? e.rd : e.qs) : -1;
            const unsigned grp = __match_any_sync(0xffffffffu, peer);
            if (mine && (grp & ((1u << lane) - 1)) == 0) atomicAdd(&cnt[peer], __popc(grp));
        }
        __syncthreads();
        if (threadIdx.x < p.G) counts[uint64_t(threadIdx.x) * (nb + 1) + b] = cnt[threadIdx.x];
        __syncthreads();
    }
}

// Chunk bookkeeping shared by pack and unpack: per-column element counts per
// peer, then their exclusive prefix in column order (one warp-wide scan per peer).
struct X2Chunk {
    unsigned int colcnt[kMaxShards][kCols];   // [peer][column]
    unsigned int colbase[kMaxShards][kCols];  // exclusive prefix over columns
    unsigned int total[kMaxShards];
};

__device__ __forceinline__ void x2_chunk_prefix(X2Chunk& C, int G) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int g = warp; g < G; g += kX2Warps) {
        const unsigned v = C.colcnt[g][lane];
        unsigned x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        C.colbase[g][lane] = x - v;
        if (lane == 31) C.total[g] = x;
    }
    __syncthreads();
}

// one column of a chunk: element (lane, i) classified against this shard's side
// (pack: its sources; unpack: its destinations), grouped by the other side's rank
struct X2Col {
    X2Elem e;
    int peer;      // -1: not this shard's element
    unsigned grp;  // lanes of this column with the same peer
};

template <bool kPack>
__device__ __forceinline__ X2Col x2_col(const X2Params& p, const X2Rows& R, uint64_t j0,
                                        uint64_t i, int lane) {
    X2Col c;
    const uint64_t cs = addmod(j0, mulmod_shoup(i, p.tp.m, p.tp.m_sh, p.N), p.N);
    c.e = x2_elem(p, R, cs, lane, i);
    const bool mine = c.e.valid && (kPack ? c.e.qs == p.me : c.e.rd == p.me);
    c.peer = mine ? (kPack ? c.e.rd : c.e.qs) : -1;
    c.grp = __match_any_sync(0xffffffffu, c.peer);
    return c;
}

__device__ __forceinline__ void x2_count_col(X2Chunk& C, const X2Col& c, int col, int lane) {
    if (c.peer >= 0 && (c.grp & ((1u << lane) - 1)) == 0) C.colcnt[c.peer][col] = __popc(c.grp);
}

// pack: this shard's source elements of the round's bands into the receivers' streams
__global__ void __launch_bounds__(kX2Threads) k_x2_pack(X2Params p) {
    __shared__ X2Rows R;
    __shared__ X2Chunk C;
    __shared__ unsigned long long pos[kMaxShards];  // band's next slot per receiver (round-relative)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t nb = p.tp.ntiles;
    const uint64_t lo = uint64_t(p.me) * p.S;
    for (uint64_t b = p.b0 + blockIdx.x; b < p.b1; b += gridDim.x) {
        x2_load_rows(p, b, R);
        if (threadIdx.x < p.G) {
            const unsigned long long* o = p.off + uint64_t(threadIdx.x) * (nb + 1);
            pos[threadIdx.x] = o[b] - o[p.b0];
        }
        const uint64_t j0 = b * kRows;
        for (uint64_t i0 = 0; i0 < R.maxlen; i0 += kCols) {
            for (int k = threadIdx.x; k < kMaxShards * kCols; k += kX2Threads)
                (&C.colcnt[0][0])[k] = 0;
            __syncthreads();
            X2Col col[kX2ColsPerWarp];
            double2 v[kX2ColsPerWarp];
#pragma unroll
            for (int h = 0; h < kX2ColsPerWarp; ++h) {
                const int c = warp + kX2Warps * h;
                col[h] = x2_col<true>(p, R, j0, i0 + c, lane);
                v[h] = col[h].peer >= 0 ? __ldg(p.sel + (col[h].e.src - lo)) : make_double2(0.0, 0.0);
                x2_count_col(C, col[h], c, lane);
            }
            __syncthreads();
            x2_chunk_prefix(C, p.G);
#pragma unroll
            for (int h = 0; h < kX2ColsPerWarp; ++h) {
                const int c = warp + kX2Warps * h;
                const int g = col[h].peer;
                if (g >= 0) {
                    const unsigned rank = __popc(col[h].grp & ((1u << lane) - 1));
                    p.dst[g][pos[g] + C.colbase[g][c] + rank] = v[h];
                }
            }
            __syncthreads();
            if (threadIdx.x < p.G) pos[threadIdx.x] += C.total[threadIdx.x];
        }
        __syncthreads();
    }
}

// unpack: this shard's destination elements of the round's bands from the
// senders' streams into P (rows through a shared-memory transpose)
__global__ void __launch_bounds__(kX2Threads) k_x2_unpack(X2Params p) {
    __shared__ X2Rows R;
    __shared__ X2Chunk C;
    __shared__ unsigned long long pos[kMaxShards];  // band's next slot per sender (round-relative)
    __shared__ double2 tile[kRows][kCols + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t nb = p.tp.ntiles;
    const uint64_t lo = uint64_t(p.me) * p.S;
    for (uint64_t b = p.b0 + blockIdx.x; b < p.b1; b += gridDim.x) {
        x2_load_rows(p, b, R);
        if (threadIdx.x < p.G) {
            const unsigned long long* o = p.off + uint64_t(threadIdx.x) * (nb + 1);
            pos[threadIdx.x] = o[b] - o[p.b0];
        }
        const uint64_t j0 = b * kRows;
        for (uint64_t i0 = 0; i0 < R.maxlen; i0 += kCols) {
            for (int k = threadIdx.x; k < kMaxShards * kCols; k += kX2Threads)
                (&C.colcnt[0][0])[k] = 0;
            __syncthreads();
            X2Col col[kX2ColsPerWarp];
#pragma unroll
            for (int h = 0; h < kX2ColsPerWarp; ++h) {
                const int c = warp + kX2Warps * h;
                col[h] = x2_col<false>(p, R, j0, i0 + c, lane);
                x2_count_col(C, col[h], c, lane);
            }
            __syncthreads();
            x2_chunk_prefix(C, p.G);
#pragma unroll
            for (int h = 0; h < kX2ColsPerWarp; ++h) {
                const int c = warp + kX2Warps * h;
                const int g = col[h].peer;
                if (g >= 0) {
                    const unsigned rank = __popc(col[h].grp & ((1u << lane) - 1));
                    tile[lane][c] = p.src[g][pos[g] + C.colbase[g][c] + rank];
                }
            }
            __syncthreads();
            for (int k = warp; k < kRows; k += kX2Warps) {  // row runs: lane = column
                const uint64_t i = i0 + lane;
                if (i < R.len[k] && R.own[k] + (i >= R.cut[k] ? 1 : 0) == p.me)
                    p.P[R.z[k] + i - lo] = tile[k][lane];
            }
            if (threadIdx.x < p.G) pos[threadIdx.x] += C.total[threadIdx.x];
            __syncthreads();
        }
        __syncthreads();
    }
}

}  // namespace shs
