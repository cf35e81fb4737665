// Sorted-residue tiles for the modular-multiplication permutation.
//
// For the stage multiplier A (m = A^-1 mod N) and a row count H, the residues
// z_j = j*A mod N (j < H) split Z_N into H rows [z_j, z_j + g_j) and
//                      src(z_j + i) = (j + i*m) mod N.
// So a tile of kRows consecutive rows j and kCols consecutive columns i reads
// the gathered side as kCols runs of kRows consecutive amplitudes (256 B) and
// the direct side / output as kRows runs of kCols consecutive amplitudes (1 KB):
// both HBM sides are coalesced; the transpose happens in shared memory. By the
// three-distance theorem a row's length and its successor in z order need no
// sort: with u = argmin_{0<j<H} (jA mod N), v = argmax_{0<j<H} (jA mod N),
//   j + u < H : length du = uA mod N,       successor j + u
//   j >= v    : length dv = N - (vA mod N),  successor j - v
//   otherwise : length du + dv,              successor j + u - v.
// Block partial sums (fixed 256-amplitude blocks in z order, bit-identical to
// proj/src/statevector.cpp:353-371) run as one sequential chain per (row,
// group); the block that straddles two rows is finished by k_tile_fixup from
// the predecessor's tail partial and the row's stored head norms.
#pragma once

#include "device_math.cuh"

namespace shs {

constexpr int kRows = 16;   // rows per tile
constexpr int kCols = 64;   // columns per chunk
constexpr int kTileThreads = 256;

struct TileParams {
    const double2* X;
    double2* Y;
    uint64_t N;
    uint64_t A, A_sh;   // z_j = j * A mod N
    uint64_t m, m_sh;   // src = j + i * m mod N
    uint64_t H, u, v, du, dv;
    uint64_t ntiles;
    StageScalars sc;
    double* S;          // block partials, S0 [0, nb), S1 [nb, 2nb)
    uint64_t nb;
    unsigned long long* partials;  // exact-accumulator slots, [slot][2][kDigits]
    double* head;       // [H][2][256] head norms of each row (before its first boundary)
    double* tail;       // [H][2]      predecessor's tail partial, indexed by successor row
    int sel;            // collapse: group kept
};

__device__ __forceinline__ uint64_t tile_row_len(uint64_t j, const TileParams& p) {
    if (j + p.u < p.H) return p.du;
    if (j >= p.v) return p.dv;
    return p.du + p.dv;
}

__device__ __forceinline__ uint64_t tile_row_succ(uint64_t j, const TileParams& p) {
    if (j + p.u < p.H) return j + p.u;
    if (j >= p.v) return j - p.v;
    return j + p.u - p.v;
}

__device__ __forceinline__ void write_partials(unsigned long long (*digits)[kDigits],
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

// kProbs: the probability pass (norms, block partials, exact accumulation).
// !kProbs: the collapse pass (writes Y[z] = h_sel).
template <bool kProbs>
__global__ void __launch_bounds__(kTileThreads) k_tiled(TileParams p) {
    __shared__ double2 src_s[kCols][kRows + 1];               // gathered side, transposed
    __shared__ double nrm[kProbs ? 2 : 1][kRows][kCols + 1];  // norms for the chains
    __shared__ uint64_t row_z[kRows], row_l[kRows];
    __shared__ unsigned long long digits[2][kDigits];
    const int tid = threadIdx.x;
    if (kProbs) {
        for (int i = tid; i < 2 * kDigits; i += kTileThreads) (&digits[0][0])[i] = 0ull;
    }
    DigitWindow win;
    window_reset(win);
    // chain lanes: warp 0, lane = g * kRows + r
    const int cr = tid & (kRows - 1), cg = (tid >> 4) & 1;
    const bool chain = kProbs && tid < 2 * kRows;

    for (uint64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
        const uint64_t j0 = tile * kRows;
        __syncthreads();  // previous tile fully consumed (row_z / row_l reuse)
        if (tid < kRows) {
            const uint64_t j = j0 + tid;
            if (j < p.H) {
                row_z[tid] = mulmod_shoup(j, p.A, p.A_sh, p.N);
                row_l[tid] = tile_row_len(j, p);
            } else {
                row_z[tid] = 0;
                row_l[tid] = 0;
            }
        }
        __syncthreads();
        uint64_t tile_len = 0;
#pragma unroll
        for (int r = 0; r < kRows; ++r) tile_len = row_l[r] > tile_len ? row_l[r] : tile_len;
        // chain state of this lane's (row, group)
        uint64_t c_z = 0, c_len = 0, c_head = 0;
        double c_s = 0.0;
        if (chain) {
            c_z = row_z[cr];
            c_len = row_l[cr];
            c_head = (256 - (c_z & 255)) & 255;
        }

        for (uint64_t i0 = 0; i0 < tile_len; i0 += kCols) {
            // gathered side: column c is a run of kRows amplitudes at (j0 + (i0+c) m) mod N
            {
                const int r = tid & (kRows - 1);
                const int cc = tid >> 4;
#pragma unroll
                for (int k = 0; k < kCols / 16; ++k) {
                    const int c = cc + 16 * k;
                    const uint64_t pos = i0 + c;
                    double2 v = make_double2(0.0, 0.0);
                    if (pos < row_l[r]) {
                        const uint64_t src = addmod(j0 + r, mulmod_shoup(pos, p.m, p.m_sh, p.N), p.N);
                        v = __ldg(p.X + src);
                    }
                    src_s[c][r] = v;
                }
            }
            // direct side: row r is a run of kCols amplitudes at z_j + i0
            const int c = tid & (kCols - 1);
            const int rg = tid >> 6;
            const uint64_t pos = i0 + c;
            double2 xz[kRows / 4];
#pragma unroll
            for (int k = 0; k < kRows / 4; ++k) {
                const int r = rg * (kRows / 4) + k;
                xz[k] = pos < row_l[r] ? __ldg(p.X + row_z[r] + pos) : make_double2(0.0, 0.0);
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < kRows / 4; ++k) {
                const int r = rg * (kRows / 4) + k;
                const bool live = pos < row_l[r];
                double h0r, h0i, h1r, h1i;
                stage_pair(p.sc, xz[k], src_s[c][r], h0r, h0i, h1r, h1i);
                if (kProbs) {
                    nrm[0][r][c] = live ? cnorm(h0r, h0i) : 0.0;
                    nrm[kProbs ? 1 : 0][r][c] = live ? cnorm(h1r, h1i) : 0.0;
                } else if (live) {
                    p.Y[row_z[r] + pos] = p.sel ? make_double2(h1r, h1i) : make_double2(h0r, h0i);
                }
            }
            __syncthreads();  // src_s / nrm complete; src_s free for the next chunk
            if (kProbs) {
                if (chain) {
                    const uint64_t jrow = j0 + cr;
                    double* head = p.head + (jrow * 2 + cg) * 256;
                    for (int cc = 0; cc < kCols; ++cc) {
                        const uint64_t q = i0 + cc;
                        if (q >= c_len) break;
                        const double n = nrm[cg][cr][cc];
                        if (q < c_head) {
                            head[q] = n;
                        } else {
                            c_s = __dadd_rn(c_s, n);
                            const uint64_t z = c_z + q;
                            if (((z + 1) & 255) == 0) {
                                p.S[cg * p.nb + (z >> 8)] = c_s;
                                window_add(win, c_s, digits[cg]);
                                c_s = 0.0;
                            }
                        }
                    }
                }
            }
        }
        if (chain && c_len > 0) {
            const uint64_t end = c_z + c_len;
            if ((end & 255) != 0) {
                if (end == p.N) {  // the final (partial) block of Z_N
                    p.S[cg * p.nb + ((p.N - 1) >> 8)] = c_s;
                    window_add(win, c_s, digits[cg]);
                } else {
                    p.tail[tile_row_succ(j0 + cr, p) * 2 + cg] = c_s;
                }
            }
        }
    }
    if (kProbs) {
        if (chain) window_flush(win, digits[cg]);
        __syncthreads();
        write_partials(digits, p.partials + uint64_t(blockIdx.x) * 2 * kDigits, tid);
    }
}

// The block straddling the boundary between a row and its z-order predecessor:
// S_b = fold(predecessor's tail partial, this row's head norms).
__global__ void __launch_bounds__(256) k_tile_fixup(TileParams p, unsigned long long* slots) {
    __shared__ unsigned long long digits[2][kDigits];
    const int tid = threadIdx.x;
    for (int i = tid; i < 2 * kDigits; i += blockDim.x) (&digits[0][0])[i] = 0ull;
    __syncthreads();
    DigitWindow w0, w1;
    window_reset(w0);
    window_reset(w1);
    for (uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + tid; idx < 2 * p.H;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t j = idx >> 1;
        const int g = static_cast<int>(idx & 1);
        const uint64_t z = mulmod_shoup(j, p.A, p.A_sh, p.N);
        const uint64_t hl = (256 - (z & 255)) & 255;
        if (hl == 0) continue;
        double s = p.tail[j * 2 + g];
        const double* head = p.head + (j * 2 + g) * 256;
        for (uint64_t q = 0; q < hl; ++q) s = __dadd_rn(s, head[q]);
        p.S[g * p.nb + (z >> 8)] = s;
        window_add(g ? w1 : w0, s, digits[g]);
    }
    window_flush(w0, digits[0]);
    window_flush(w1, digits[1]);
    __syncthreads();
    write_partials(digits, slots + uint64_t(blockIdx.x) * 2 * kDigits, tid);
}

}  // namespace shs
