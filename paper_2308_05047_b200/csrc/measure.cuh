// Device-side measurement of one stage: Philox4x32-10 + RngStream draws
// (proj/include/shorsim/rng.hpp:16-83) and sample_measurement with the error
// channels (proj/src/statevector.cpp:236-256, proj/src/noise.cpp:128-145),
// restated with explicitly rounded fp64 ops so the sampled bits are the host's
// (host_model.cpp) bit for bit. Used by the batched small-N engine (batch.cuh)
// and by the device-resident run of the large-state engine (k_finalize_measure):
// there the host never sits between a stage's |psi|^2 reduction and its
// collapse — it only supplies the two candidate phases of the NEXT stage
// (std::polar with glibc cos/sin, which the device cannot reproduce) one stage
// ahead.
#pragma once

#include "device_math.cuh"

namespace shs {

// ---- Philox4x32-10 (rng.hpp:16-31) and RngStream draws (rng.hpp:63-66)
__device__ __forceinline__ void philox_dev(uint64_t key, uint32_t c[4]) {
    uint32_t k0 = static_cast<uint32_t>(key), k1 = static_cast<uint32_t>(key >> 32);
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        const uint64_t p0 = uint64_t(0xD2511F53u) * c[0];
        const uint64_t p1 = uint64_t(0xCD9E8D57u) * c[2];
        const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c[1] ^ k0;
        const uint32_t n1 = static_cast<uint32_t>(p1);
        const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c[3] ^ k1;
        const uint32_t n3 = static_cast<uint32_t>(p0);
        c[0] = n0;
        c[1] = n1;
        c[2] = n2;
        c[3] = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

__device__ __forceinline__ double rng_double_dev(uint64_t seed, uint32_t a, uint32_t b,
                                                 uint32_t domain, uint32_t index) {
    uint32_t c[4] = {index, a, b, domain};
    philox_dev(seed, c);
    const uint64_t u = (uint64_t(c[0]) << 32) | c[1];
    return __dmul_rn(static_cast<double>(u >> 11), 0x1.0p-53);
}

// The run-constant inputs of sample_measurement.
struct MeasureCfg {
    uint64_t seed;
    uint32_t idx32;     // bitstring_index truncated to u32 (statevector.cpp:377)
    int kind;           // SHS_ERR_*
    double delta, px, py;
    int check_norms;
};

struct DevMeasure {
    int sbit, obit, flip, ebranch;
    int src_group;      // group kept by the collapse (statevector.cpp:385-386)
    double p_src;       // its mass: p1 or p0 (statevector.cpp:387)
    int status;         // 0, SHS_ERROR (norm drift), SHS_DEGENERATE_BRANCH
};

// sample_measurement + the collapse bookkeeping of stage s; `collapse` = s + 1 < t.
// Error precedence is the reference's: the norm check throws before sampling
// (statevector.cpp:374-375), the degenerate-branch check before the collapse
// (statevector.cpp:388-390).
__device__ __forceinline__ DevMeasure measure_dev(double p0, double p1, const MeasureCfg& m,
                                                  uint32_t s, bool collapse) {
    DevMeasure r{0, 0, 0, 0, 0, 0.0, 0};
    uint32_t draw = 0;
    if (m.kind == SHS_ERR_QUANTUM_MEASURE) {  // depolarizing_measure_branch, noise.cpp:133-145
        const double dxy = __dadd_rn(m.px, m.py);
        const double p1p = __dadd_rn(__dmul_rn(__dsub_rn(1.0, dxy), p1),
                                     __dmul_rn(dxy, __dsub_rn(1.0, p1)));
        r.sbit = rng_double_dev(m.seed, m.idx32, s, 0, draw++) < p1p ? 1 : 0;
        const double p_bit = r.sbit == 1 ? p1 : __dsub_rn(1.0, p1);
        const double p_other = __dsub_rn(1.0, p_bit);
        const double p_bit_prime = r.sbit == 1 ? p1p : __dsub_rn(1.0, p1p);
        const double p_err =
            p_bit_prime > 0.0 ? __ddiv_rn(__dmul_rn(dxy, p_other), p_bit_prime) : 0.0;
        r.ebranch = rng_double_dev(m.seed, m.idx32, s, 0, draw++) < p_err ? 1 : 0;
        r.obit = r.sbit;
    } else {
        r.sbit = rng_double_dev(m.seed, m.idx32, s, 0, draw++) < p1 ? 1 : 0;
        r.obit = r.sbit;
        if (m.kind == SHS_ERR_CLASSICAL_MEASURE) {  // classical_flip, noise.cpp:128-131
            r.flip = rng_double_dev(m.seed, m.idx32, s, 0, draw++) < m.delta ? 1 : 0;
            if (r.flip) r.obit = 1 - r.sbit;
        }
    }
    r.src_group = r.ebranch ? 1 - r.sbit : r.sbit;
    r.p_src = r.src_group == 1 ? p1 : p0;
    if (m.check_norms && fabs(__dsub_rn(__dadd_rn(p0, p1), 1.0)) > 1e-9) r.status = SHS_ERROR;
    else if (collapse && r.p_src < 1e-300) r.status = SHS_DEGENERATE_BRANCH;
    return r;
}

// The scalars a stage kernel reads from device memory in a device-resident
// run: slot s & 1 holds stage s's StageScalars (written by stage s-1's
// k_finalize_measure) and the group its collapse keeps (written by stage s's).
struct DevStage {
    StageScalars sc;
    int sel;
    int pad;
};

// Per-stage record of a device-resident run (host-mapped pinned memory).
struct StageRec {
    double p0, p1;
    int32_t sbit, obit, flip, ebranch;
    int32_t status, done;
};

// The next stage's phase for either value of this stage's observed bit: the
// host computes std::polar(1, stage_phase(s + 1, prefix | bit << s)) for both.
struct NextPhase {
    double phr[2], phi[2];
    int phase_mul[2];
};

}  // namespace shs
