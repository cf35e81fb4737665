// HBM bandwidth of a gather of F-byte fragments at random 16 B-aligned offsets
// (the access pattern of the orbit-compressed stages: column runs of ~16 members
// = 256 B) against contiguous streaming, one B200.
// Each warp copies fragments: lane i moves 16 B at frag + 16 i (F / 16 lanes per
// fragment, 512 / F fragments per warp instruction) from a 64 GB source into a
// contiguous destination, so half the bytes are gathered reads and half
// contiguous writes, as in the compressed pass (reads src + dst, writes Y + Y1).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fragment_bw fragment_bw.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

template <int F>
__global__ void k_gather(const double2* __restrict__ src, uint64_t nsrc, double2* __restrict__ dst,
                         uint64_t nfrag_total, uint64_t seed) {
    constexpr int kLanes = F / 16;            // lanes per fragment (F <= 512)
    constexpr int kPer = 32 / kLanes;         // fragments per warp instruction
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t nwarps = (gridDim.x * uint64_t(blockDim.x)) >> 5;
    const uint64_t ninst = nfrag_total / kPer;
    for (uint64_t q = warp; q < ninst; q += nwarps) {
        const uint64_t f = q * kPer + lane / kLanes;
        const uint64_t off = mix(f ^ seed) % (nsrc - kLanes);
        const double2 v = __ldcg(src + off + (lane % kLanes));
        __stcg(dst + q * 32 + lane, v);
    }
}

// F > 512: a warp reads F / 512 consecutive 512 B pieces of one fragment
template <int F>
__global__ void k_gather_big(const double2* __restrict__ src, uint64_t nsrc, double2* __restrict__ dst,
                             uint64_t nfrag_total, uint64_t seed) {
    constexpr int kPieces = F / 512;
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t nwarps = (gridDim.x * uint64_t(blockDim.x)) >> 5;
    for (uint64_t f = warp; f < nfrag_total; f += nwarps) {
        const uint64_t off = mix(f ^ seed) % (nsrc - 32 * kPieces);
        double2 v[kPieces];
#pragma unroll
        for (int k = 0; k < kPieces; ++k) v[k] = __ldcg(src + off + 32 * k + lane);
#pragma unroll
        for (int k = 0; k < kPieces; ++k) __stcg(dst + (f * kPieces + k) * 32 + lane, v[k]);
    }
}

// both sides fragmented: F-byte reads and F-byte writes at independent random
// offsets (the compressed pass's stores are row runs of ~32 members = 512 B)
template <int F>
__global__ void k_gather_scatter(const double2* __restrict__ src, uint64_t nsrc, double2* __restrict__ dst,
                                 uint64_t nfrag_total, uint64_t seed) {
    constexpr int kLanes = F / 16;
    constexpr int kPer = 32 / kLanes;
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t nwarps = (gridDim.x * uint64_t(blockDim.x)) >> 5;
    const uint64_t ninst = nfrag_total / kPer;
    for (uint64_t q = warp; q < ninst; q += nwarps) {
        const uint64_t f = q * kPer + lane / kLanes;
        const uint64_t off = mix(f ^ seed) % (nsrc - kLanes);
        const uint64_t woff = mix(f ^ ~seed) % (nsrc - kLanes);
        __stcg(dst + woff + (lane % kLanes), __ldcg(src + off + (lane % kLanes)));
    }
}

// the compressed pass's pattern as streams: 4736 rows (148 CTAs x 32 warps), each with
// random 16 B-aligned bases in X (direct side), Y and Y1; per step a row reads G
// gathered fragments of F bytes at random offsets and D bytes at its X stream
// position, and writes D bytes at its Y and Y1 positions (F = 256, D = 512: the
// shipped 32-row bands at N / 2 density; F = 512, D = 1024: 64-row bands)
template <int F, int G, int D>
__global__ void __launch_bounds__(1024) k_streams(const double2* __restrict__ X, uint64_t nx,
                                                  double2* __restrict__ Y, double2* __restrict__ Y1,
                                                  uint64_t steps, uint64_t seed) {
    constexpr int kU = 4;  // steps in flight per row (the kernel keeps ~4 slots in flight)
    constexpr int kFL = F / 16, kDI = D / 512, kGI = G * kFL / 32;
    const int lane = threadIdx.x & 31;
    const uint64_t row = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;  // one row per warp
    const uint64_t span = steps * (D / 16);
    const uint64_t bx = mix(row * 3 + seed) % (nx - span), by = mix(row * 3 + 1 + seed) % (nx - span);
    for (uint64_t t0 = 0; t0 < steps; t0 += kU) {
        double2 g[kU][kGI], d[kU][kDI];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint64_t t = t0 + u;
#pragma unroll
            for (int k = 0; k < kGI; ++k) {
                const uint64_t f = (row * steps + t) * G + k * (32 / kFL) + lane / kFL;
                g[u][k] = __ldcg(X + mix(f ^ seed) % (nx - kFL) + lane % kFL);
            }
#pragma unroll
            for (int k = 0; k < kDI; ++k) d[u][k] = __ldcg(X + bx + t * (D / 16) + 32 * k + lane);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
#pragma unroll
            for (int k = 0; k < kDI; ++k) {
                double2 v = d[u][k];
#pragma unroll
                for (int q = 0; q < kGI; ++q) v.x += g[u][q].x;
                __stcg(Y + by + (t0 + u) * (D / 16) + 32 * k + lane, v);
                __stcg(Y1 + by + (t0 + u) * (D / 16) + 32 * k + lane, v);
            }
    }
}

template <int F, int G, int D>
static void run_streams(const double2* X, uint64_t nx, double2* Y, double2* Y1) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const uint64_t steps = 2048;
    k_streams<F, G, D><<<148, 1024>>>(X, nx, Y, Y1, steps, 1);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
        cudaEventRecord(a);
        k_streams<F, G, D><<<148, 1024>>>(X, nx, Y, Y1, steps, 7 + it);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    const double bytes = 148.0 * 32 * steps * (double(F) * G + 3.0 * D);
    printf("{\"kernel\": \"streams\", \"gathered\": \"%d x %d B\", \"stream_bytes\": %d, \"ms\": %.3f, \"GBps\": %.1f}\n",
           G, F, D, best, bytes / best / 1e6);
}

template <typename K>
static void run(const char* name, K kern, const double2* src, uint64_t nsrc, double2* dst, uint64_t nfrag,
                int F) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = 148 * 8, threads = 256;
    kern<<<blocks, threads>>>(src, nsrc, dst, nfrag, 1);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
        cudaEventRecord(a);
        kern<<<blocks, threads>>>(src, nsrc, dst, nfrag, 2 + it);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    const double bytes = 2.0 * double(nfrag) * F;  // gathered reads + contiguous writes
    printf("{\"fragment_bytes\": %d, \"kernel\": \"%s\", \"ms\": %.3f, \"GBps\": %.1f}\n", F, name, best,
           bytes / best / 1e6);
}

int main() {
    const uint64_t nsrc = (64ull << 30) / 16;  // 64 GB of 16 B elements
    const uint64_t bytes_moved = 8ull << 30;   // 8 GB gathered per launch
    double2 *src, *dst, *dst2;
    if (cudaMalloc(&src, nsrc * 16) != cudaSuccess || cudaMalloc(&dst, bytes_moved) != cudaSuccess ||
        cudaMalloc(&dst2, nsrc * 16) != cudaSuccess) {
        printf("alloc failed\n");
        return 1;
    }
    cudaMemset(src, 1, nsrc * 16);
    run("gather", k_gather<128>, src, nsrc, dst, bytes_moved / 128, 128);
    run("gather", k_gather<256>, src, nsrc, dst, bytes_moved / 256, 256);
    run("gather", k_gather<512>, src, nsrc, dst, bytes_moved / 512, 512);
    run("gather_big", k_gather_big<1024>, src, nsrc, dst, bytes_moved / 1024, 1024);
    run("gather_big", k_gather_big<2048>, src, nsrc, dst, bytes_moved / 2048, 2048);
    run("gather_big", k_gather_big<4096>, src, nsrc, dst, bytes_moved / 4096, 4096);
    run("gather_scatter", k_gather_scatter<256>, src, nsrc, dst2, bytes_moved / 256, 256);
    run("gather_scatter", k_gather_scatter<512>, src, nsrc, dst2, bytes_moved / 512, 512);
    run_streams<256, 2, 512>(src, nsrc / 2, dst2, dst2 + nsrc / 2);
    run_streams<512, 2, 1024>(src, nsrc / 2, dst2, dst2 + nsrc / 2);
    run_streams<512, 1, 512>(src, nsrc / 2, dst2, dst2 + nsrc / 2);
    return 0;
}
