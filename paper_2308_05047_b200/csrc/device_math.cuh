// Device-side arithmetic for the iterative-Shor stage kernels (sm_100a).
//
// Every floating-point operation is an explicitly rounded intrinsic
// (__dmul_rn / __dadd_rn / __dsub_rn), and the library is compiled with
// --fmad=false, so no multiply-add is ever contracted: each value rounds
// exactly where the reference's does under -ffp-contract=off
// (/root/reference/proj/CMakeLists.txt:17-20).
#pragma once

#include <cstdint>

namespace shs {

constexpr int kBlock = 256;              // reduction block, proj/src/statevector.cpp:16
constexpr int kThreads = 256;            // threads per CTA
constexpr int kPer = 8;                  // amplitudes per thread per chunk
constexpr int kChunk = kThreads * kPer;  // 2048 amplitudes = 8 reduction blocks
constexpr int kDigits = 40;              // exact accumulator: 40 x 32-bit digits
constexpr int kAnchor = 1088;            // value = F * 2^-kAnchor (covers 2^-1074 .. 2^191)
constexpr double kInvSqrt2 = 0.70710678118654752440;  // statevector.cpp:14

// r = z * m mod N by Shoup's method with m_sh = floor(m * 2^64 / N).
// Exact for N < 2^63, m < N, any z < 2^64 (A3: mulmod_u64, int128.hpp:28-30).
__device__ __forceinline__ uint64_t mulmod_shoup(uint64_t z, uint64_t m, uint64_t m_sh,
                                                 uint64_t n) {
    uint64_t q = __umul64hi(z, m_sh);
    uint64_t r = z * m - q * n;
    return r >= n ? r - n : r;
}

__device__ __forceinline__ uint64_t addmod(uint64_t x, uint64_t step, uint64_t n) {
    uint64_t r = x + step;
    return r >= n ? r - n : r;
}

// (a_r + i a_i)(b_r + i b_i) as GCC lowers std::complex<double> * with
// -ffp-contract=off: (a_r b_r - a_i b_i, a_r b_i + a_i b_r).
__device__ __forceinline__ void cmul(double ar, double ai, double br, double bi, double& r,
                                     double& i) {
    double rr = __dsub_rn(__dmul_rn(ar, br), __dmul_rn(ai, bi));
    double ii = __dadd_rn(__dmul_rn(ar, bi), __dmul_rn(ai, br));
    r = rr;
    i = ii;
}

// std::norm(z) = re*re + im*im (libstdc++ _Norm_helper, no contraction)
__device__ __forceinline__ double cnorm(double r, double i) {
    return __dadd_rn(__dmul_rn(r, r), __dmul_rn(i, i));
}

// Scalars of one stage, broadcast to every thread as kernel parameters.
struct StageScalars {
    double w0r, w0i, w1r, w1i;  // reinit pair (w0, w1), noise.cpp:89-95
    double phr, phi;            // std::polar(1, phi), statevector.cpp:338
    double inv;                 // 1/sqrt(p_src) of the previous collapse
    int phase_mul;              // gather || phi != 0 (statevector.cpp:345 / 349)
};

// A copy of shared-memory stage scalars that the compiler cannot hoist out of a loop.
__device__ __forceinline__ StageScalars load_scalars(const StageScalars& s) {
    const volatile StageScalars& v = s;
    StageScalars r;
    r.w0r = v.w0r;
    r.w0i = v.w0i;
    r.w1r = v.w1r;
    r.w1i = v.w1i;
    r.phr = v.phr;
    r.phi = v.phi;
    r.inv = v.inv;
    r.phase_mul = v.phase_mul;
    return r;
}

// Post-Hadamard pair of one amplitude index:
//   u  = w0 * (x * inv)                 g0[z] after reset   (statevector.cpp:396-397)
//   v  = (w1 * (xs * inv)) [* ph]       g1[src z] * ph      (statevector.cpp:345 / 360)
//   h0 = (u + v) * k, h1 = (u - v) * k                      (statevector.cpp:361-362)
template <class SC>
__device__ __forceinline__ void stage_pair(const SC& sc, double2 x, double2 xs,
                                           double& h0r, double& h0i, double& h1r,
                                           double& h1i) {
    double xr = __dmul_rn(x.x, sc.inv), xi = __dmul_rn(x.y, sc.inv);
    double sr = __dmul_rn(xs.x, sc.inv), si = __dmul_rn(xs.y, sc.inv);
    double ur, ui, vr, vi;
    cmul(sc.w0r, sc.w0i, xr, xi, ur, ui);
    cmul(sc.w1r, sc.w1i, sr, si, vr, vi);
    if (sc.phase_mul) cmul(vr, vi, sc.phr, sc.phi, vr, vi);
    h0r = __dmul_rn(__dadd_rn(ur, vr), kInvSqrt2);
    h0i = __dmul_rn(__dadd_rn(ui, vi), kInvSqrt2);
    h1r = __dmul_rn(__dsub_rn(ur, vr), kInvSqrt2);
    h1i = __dmul_rn(__dsub_rn(ui, vi), kInvSqrt2);
}

// ---------------------------------------------------------------------------
// Exact accumulation of non-negative doubles: value = F * 2^-kAnchor with F an
// integer held in 32-bit digits (uint64 lanes absorb 2^32 carries-free adds).
// A thread keeps a 4-digit window in registers and flushes it to shared
// memory with integer atomics only when the exponent moves out of the window,
// so the result is exact and independent of order, grid and GPU count.
struct DigitWindow {
    int base;
    unsigned long long d0, d1, d2, d3;
};

__device__ __forceinline__ void window_reset(DigitWindow& w) {
    w.base = -1;
    w.d0 = w.d1 = w.d2 = w.d3 = 0;
}

__device__ __forceinline__ void window_flush(DigitWindow& w, unsigned long long* digits) {
    if (w.base < 0) return;
    if (w.d0) atomicAdd(&digits[w.base], w.d0);
    if (w.d1) atomicAdd(&digits[w.base + 1], w.d1);
    if (w.d2) atomicAdd(&digits[w.base + 2], w.d2);
    if (w.d3) atomicAdd(&digits[w.base + 3], w.d3);
    window_reset(w);
}

__device__ __forceinline__ void window_add(DigitWindow& w, double v, unsigned long long* digits) {
    if (!(v > 0.0)) return;  // zero (and the impossible negatives / NaN) contribute nothing
    unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
    int ex = static_cast<int>((bits >> 52) & 0x7ff);
    unsigned long long mant = bits & ((1ull << 52) - 1);
    int shift;
    if (ex == 0) {
        shift = kAnchor - 1074;
    } else {
        mant |= 1ull << 52;
        shift = ex - 1075 + kAnchor;
    }
    int d = shift >> 5, off = shift & 31;
    unsigned long long lo = mant << off;
    unsigned long long hi = off ? (mant >> (64 - off)) : 0ull;
    unsigned long long p0 = lo & 0xffffffffull, p1 = lo >> 32, p2 = hi;
    if (w.base < 0 || d < w.base || d > w.base + 1) {
        window_flush(w, digits);
        w.base = d;
    }
    if (d == w.base) {
        w.d0 += p0;
        w.d1 += p1;
        w.d2 += p2;
    } else {
        w.d1 += p0;
        w.d2 += p1;
        w.d3 += p2;
    }
}

// Round an exact digit accumulator (normalised in place) to the nearest double,
// ties to even; subnormal results keep the 2^-1074 quantum. The mantissa, round
// and sticky bits are read word-wise (a bit-by-bit walk over shared memory cost
// ~2 us per call in the single-CTA finalize kernels).
__device__ __forceinline__ double digits_to_double(unsigned long long* acc) {
    unsigned long long carry = 0;
    for (int i = 0; i < kDigits; ++i) {
        unsigned long long v = acc[i] + carry;
        acc[i] = v & 0xffffffffull;
        carry = v >> 32;
    }
    int ti = kDigits - 1;
    while (ti >= 0 && !acc[ti]) --ti;
    if (ti < 0) return 0.0;
    const int top = ti * 32 + 63 - __clzll(acc[ti]);
    int lsb = top - 52;
    if (lsb < kAnchor - 1074) lsb = kAnchor - 1074;  // >= 14: round and sticky bits exist
    unsigned long long mant = 0;  // bits [lsb, top]
    if (top >= lsb) {
        const int k = lsb >> 5, sh = lsb & 31;
        const unsigned long long lo = acc[k] | (k + 1 < kDigits ? acc[k + 1] << 32 : 0ull);
        const unsigned long long d2 = k + 2 < kDigits ? acc[k + 2] : 0ull;
        const unsigned long long w = sh ? (lo >> sh) | (d2 << (64 - sh)) : lo;
        mant = w & ((2ull << (top - lsb)) - 1ull);
    }
    const int pr = lsb - 1;
    const bool round = (acc[pr >> 5] >> (pr & 31)) & 1ull;
    const int ps = lsb - 2;  // sticky: any bit in [0, ps]
    int j = ps >> 5;
    bool sticky = (acc[j] & ((2ull << (ps & 31)) - 1ull)) != 0;
    while (!sticky && --j >= 0) sticky = acc[j] != 0;
    if (round && (sticky || (mant & 1ull))) ++mant;
    return scalbn(static_cast<double>(mant), lsb - kAnchor);
}

}  // namespace shs
