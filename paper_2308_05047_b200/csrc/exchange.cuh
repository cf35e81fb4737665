// Sharded-state exchange for the multi-GPU engine (shard.cu).
//
// Shard q owns global amplitude indices [q*S, min(N, (q+1)*S)), S a multiple of
// kBlock, so the reference's fixed 256-blocks never straddle shards. A
// non-identity stage first gathers P[z] = sel[a_inv * z mod N] for every z into
// the owner's exchange buffer P; the probability and collapse passes then run
// shard-locally and elementwise on (sel, P) (stage_kernels.cuh, kSrcBuffer).
// Buffers are addressed through per-owner pointers: one device (virtual shards)
// or peer devices mapped over NVLink (CUDA IPC), where these loads and stores
// are NVLink transactions.
//
// With contiguous z-shards no rank owns both sides of a sorted-residue tile
// (consecutive rows j sit A apart in z), so each rank executes a round-robin
// share of the tiles as a pure exchange: it pulls each column's 256 B source run
// from that run's owner and pushes each row's 1 KB destination run into that
// run's owner's P. Per GPU and per direction this is 16 B * (N/G) * (G-1)/G of
// NVLink traffic, the all-to-all minimum, in whole-line granules.
#pragma once

#include "stage_kernels.cuh"
#include "tiled.cuh"

namespace shs {

constexpr int kMaxShards = 16;

struct ShardMap {
    uint64_t S;      // shard size
    uint64_t S_inv;  // floor((2^64 - 1) / S)
    int G;
    const double2* src[kMaxShards];  // owners' sel buffers
    double2* dst[kMaxShards];        // owners' exchange (P) buffers
};

// owner of global index x (x < N < 2^63): one mul.hi and one correction
__device__ __forceinline__ int shard_owner(uint64_t x, const ShardMap& sm) {
    uint64_t q = __umul64hi(x, sm.S_inv);
    if (x - q * sm.S >= sm.S) ++q;
    return static_cast<int>(q);
}

// Direct exchange for this rank's shard [z0, zend): P[z - z0] = sel[a_inv z mod N]
// pulled element-wise from the owner (stages without a tile plan).
static __global__ void __launch_bounds__(kThreads) k_exchange_direct(StageParams p, ShardMap sm,
                                                              double2* P) {
    const int tid = threadIdx.x;
    for (uint64_t c = blockIdx.x; c < p.nchunks; c += gridDim.x) {
        const uint64_t zg = p.z0 + c * kChunk + tid;
        uint64_t src = mulmod_shoup(zg, p.m, p.m_sh, p.N);
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const uint64_t z = zg + uint64_t(e) * kBlock;
            if (z < p.zend) {
                const int q = shard_owner(src, sm);
                P[z - p.z0] = sm.src[q][src - uint64_t(q) * sm.S];
            }
            src = addmod(src, p.m_step, p.N);
        }
    }
}

constexpr int kExStages = 8;
constexpr int kExchangeThreads = 32 * (kConsumerWarps + kProducerWarps);

struct ExchangeSmem {
    double2 src[kExStages][kCols][kRows + 1];  // ring of gathered columns (transposed)
    uint64_t row_z[kExStages][kRows];
    uint64_t row_l[kExStages][kRows];
    uint64_t i0[kExStages];
    uint64_t last[kExStages];
    uint64_t full[kExStages], empty[kExStages];
};

constexpr size_t exchange_smem_bytes() { return sizeof(ExchangeSmem); }

// Tiled exchange over this rank's tiles t = tile0 + tile_step * k: producers
// copy source runs from the owners' sel, consumers store destination runs to
// the owners' P. Same ring / mbarrier protocol as k_tiled, except that the
// producers use plain loads + shared stores + an mbarrier release instead of
// cp.async: sources are mostly peer memory (NVLink), whose per-SM bandwidth
// (~5 GB/s of 770 GB/s) 8 loads in flight per producer thread already cover.
static __global__ void __launch_bounds__(kExchangeThreads, 1)
    k_exchange(TileParams p, ShardMap shmap, uint64_t tile0, uint64_t tile_step) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    ExchangeSmem& sm = *reinterpret_cast<ExchangeSmem*>(smem_raw);
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < kExStages; ++s) {
            mbar_init(&sm.full[s], kProducers + 1);
            mbar_init(&sm.empty[s], kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t first = tile0 + uint64_t(blockIdx.x) * tile_step;  // (ring slots below)
    const uint64_t step = uint64_t(gridDim.x) * tile_step;

    if (warp >= kProducerWarp && warp < kProducerWarp + kProducerWarps) {
        const int pt = tid - 32 * kProducerWarp;
        const int r_src = pt & (kRows - 1);
        const int src_c0 = pt / kRows;
        int stage = 0;
        uint32_t phase = 0;
        for (uint64_t tile = first; tile < p.ntiles; tile += step) {
            const uint64_t j0 = tile * kRows;
            LaneRows lr;
            const uint64_t tlen = tile_rows(p, j0, lane, lr);
            const bool last_tile = tile + step >= p.ntiles;
            const uint64_t rl = lr.len[kRowsPerLane > 1 ? (r_src >> 5) : 0];
            uint64_t sidx[kCopiesPerProducer];
#pragma unroll
            for (int k = 0; k < kCopiesPerProducer; ++k) {
                const uint64_t c = src_c0 + (kProducers / kRows) * k;
                sidx[k] = addmod(j0 + r_src, mulmod_shoup(c, p.m, p.m_sh, p.N), p.N);
            }
            for (uint64_t i0 = 0; i0 < tlen; i0 += kCols) {
                mbar_wait(&sm.empty[stage], phase ^ 1);
                double2 v[kCopiesPerProducer];
#pragma unroll
                for (int k = 0; k < kCopiesPerProducer; ++k) {  // all loads in flight first
                    const int c = src_c0 + (kProducers / kRows) * k;
                    v[k] = make_double2(0.0, 0.0);
                    if (i0 + c < rl) {
                        const uint64_t x = sidx[k];
                        const int q = shard_owner(x, shmap);
                        v[k] = shmap.src[q][x - uint64_t(q) * shmap.S];
                    }
                    sidx[k] = addmod(sidx[k], p.m_chunk, p.N);
                }
#pragma unroll
                for (int k = 0; k < kCopiesPerProducer; ++k)
                    sm.src[stage][src_c0 + (kProducers / kRows) * k][r_src] = v[k];
                mbar_arrive(&sm.full[stage]);  // release of this thread's shared stores
                if (warp == kProducerWarp) {
                    store_rows(lr, lane, sm.row_z[stage], sm.row_l[stage]);
                    __syncwarp();
                    if (lane == 0) {
                        sm.i0[stage] = i0;
                        sm.last[stage] = (last_tile && i0 + kCols >= tlen) ? 1 : 0;
                        mbar_arrive(&sm.full[stage]);
                    }
                }
                if (++stage == kExStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp < kConsumerWarps) {
        int stage = 0;
        uint32_t phase = 0;
        const int c = tid & (kCols - 1);
        const int rg = tid / kCols;
        bool more = first < p.ntiles;
        while (more) {
            mbar_wait(&sm.full[stage], phase);
            const uint64_t pos = sm.i0[stage] + c;
            more = sm.last[stage] == 0;
#pragma unroll
            for (int q = 0; q < kRowsPerConsumer; ++q) {
                const int r = rg * kRowsPerConsumer + q;
                if (pos < sm.row_l[stage][r]) {
                    const uint64_t z = sm.row_z[stage][r] + pos;
                    const int d = shard_owner(z, shmap);
                    shmap.dst[d][z - uint64_t(d) * shmap.S] = sm.src[stage][c][r];
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[stage]);
            if (++stage == kExStages) {
                stage = 0;
                phase ^= 1;
            }
        }
    }
}

}  // namespace shs
