// exhaustive_joint_distribution on the device (§8 f3): the exact distribution
// over observed bit strings by enumerating every measurement path, error
// branches marginalised (restates proj/src/statevector.cpp:420-579).
//
// The reference recurses depth-first; here every level of the path tree is one
// launch (one CTA per path node) and subtrees are processed chunk by chunk in
// depth-first order, so leaves come out in exactly the reference's DFS order
// and dist[j] += weight * w folds in the same sequence: the result is
// bit-identical, not just within the reference's 1e-10 tolerance. Per node:
//   stage_gates  h0/h1 from (sel, inv) with the node's phase (always applied,
//                as PathEnumerator::stage_gates does), statevector.cpp:441-457
//   flat_norm    sequential Kahan over the whole 2^L group, zeros included, :426-430
//   descend      the error model's children in call order, :486-527
//   project      child state = h_src, inv = 1/sqrt(p_src) (compressed form of :459-471)
// The per-(stage, prefix) phases come from a host table computed with glibc.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/shorsim_b200.h"
#include "device_math.cuh"
#include "host_model.hpp"

using namespace shs;

namespace {

#define EXH_CUDA(call)                                                                  \
    do {                                                                                \
        cudaError_t _e = (call);                                                        \
        if (_e != cudaSuccess) {                                                        \
            set_error(SHS_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(_e)); \
            throw SHS_CUDA_ERROR;                                                       \
        }                                                                               \
    } while (0)

constexpr int kExhThreads = 256;
constexpr uint32_t kExhChunk = 8192;  // nodes per launch (h buffers: chunk x 2 x N x 16 B)

struct ExhNode {        // one path-tree node of the current level
    uint32_t parent;    // index into the previous chunk's h buffers
    int32_t src_group;  // which of the parent's h0/h1 is this node's sel
    double inv;         // 1/sqrt(p_src)
    double weight;      // product of the branch weights on the path
    uint32_t observed;  // observed bits so far (t <= 14)
};

struct ExhSlot {        // up to 4 children per node, in descend() call order
    int32_t kind;       // 0 none, 1 child node, 2 leaf
    int32_t src_group;
    double inv;
    double weight;      // child weight (or leaf value weight * w)
    uint32_t observed;
};

struct ExhParams {
    uint64_t N, group;   // y_limit = N, group size 2^L
    uint32_t s, t;
    int root;            // level 0: sel = e_1, inv = 1
    int gather;          // a_pow != 1
    uint64_t m, m_sh;    // a_inv, Shoup companion
    double w0r, w0i, w1r, w1i;
    const double2* phase;  // (cos, sin) at (1 << s) - 1 + prefix
    int kind;
    double delta, px, py;
    const ExhNode* nodes;
    const double2* parent_h;  // previous chunk: [node][2][N]
    double2* h_out;           // this chunk: [node][2][N]
    ExhSlot* slots;           // [node][4]
};

__device__ __forceinline__ void kahan_flat(const double* x, uint64_t n, double& out) {
    double s = 0, c = 0;
    for (uint64_t i = 0; i < n; ++i) {  // kahan_add, statevector.cpp:21-26 (zeros too)
        const double y = __dsub_rn(x[i], c);
        const double t = __dadd_rn(s, y);
        c = __dsub_rn(__dsub_rn(t, s), y);
        s = t;
    }
    out = s;
}

__global__ void __launch_bounds__(kExhThreads) k_exh_stage(ExhParams p) {
    extern __shared__ double nrm[];  // [2][group]
    __shared__ double sh_p[2];
    const uint32_t node = blockIdx.x;
    const ExhNode nd = p.nodes[node];
    const double2* sel = p.root ? nullptr : p.parent_h + (uint64_t(nd.parent) * 2 + nd.src_group) * p.N;
    StageScalars sc;
    sc.w0r = p.w0r;
    sc.w0i = p.w0i;
    sc.w1r = p.w1r;
    sc.w1i = p.w1i;
    const double2 ph = p.phase[((uint64_t(1) << p.s) - 1) + nd.observed];
    sc.phr = ph.x;
    sc.phi = ph.y;
    sc.inv = p.root ? 1.0 : nd.inv;
    sc.phase_mul = 1;  // stage_gates multiplies by ph on every stage
    double2* h0 = p.h_out + uint64_t(node) * 2 * p.N;
    double2* h1 = h0 + p.N;
    for (uint64_t y = threadIdx.x; y < p.group; y += blockDim.x) {
        if (y < p.N) {
            const uint64_t src = p.gather ? mulmod_shoup(y, p.m, p.m_sh, p.N) : y;
            const double2 x = p.root ? make_double2(y == 1 ? 1.0 : 0.0, 0.0) : sel[y];
            const double2 xs = p.root ? make_double2(src == 1 ? 1.0 : 0.0, 0.0) : sel[src];
            double a, b, c, d;
            stage_pair(sc, x, xs, a, b, c, d);
            h0[y] = make_double2(a, b);
            h1[y] = make_double2(c, d);
            nrm[y] = cnorm(a, b);
            nrm[p.group + y] = cnorm(c, d);
        } else {  // y >= N: u = v = 0, so h = 0 (its norm still enters flat_norm)
            nrm[y] = 0.0;
            nrm[p.group + y] = 0.0;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) kahan_flat(nrm + p.group, p.group, sh_p[1]);  // p1 = flat_norm(g1)
    if (threadIdx.x == 32) kahan_flat(nrm, p.group, sh_p[0]);           // p0 = flat_norm(g0)
    __syncthreads();
    if (threadIdx.x != 0) return;
    const double p0 = sh_p[0], p1 = sh_p[1];
    const bool last = p.s + 1 == p.t;
    ExhSlot* out = p.slots + uint64_t(node) * 4;
    int k = 0;
    auto descend = [&](int observed_bit, int src_group, double w) {
        ExhSlot sl{};
        sl.kind = 0;
        if (w > 0.0) {
            sl.observed = nd.observed | (uint32_t(observed_bit) << p.s);
            const double p_src = src_group == 1 ? p1 : p0;
            if (last) {
                sl.kind = 2;
                sl.weight = __dmul_rn(nd.weight, w);
            } else if (p_src > 0.0) {
                sl.kind = 1;
                sl.src_group = src_group;
                sl.inv = __ddiv_rn(1.0, __dsqrt_rn(p_src));
                sl.weight = __dmul_rn(nd.weight, w);
            }
        }
        out[k++] = sl;
    };
    if (p.kind == SHS_ERR_QUANTUM_MEASURE) {
        const double dxy = __dadd_rn(p.px, p.py);
        for (int bit = 0; bit < 2; ++bit) {
            const double p_bit = bit == 1 ? p1 : p0;
            const double p_other = bit == 1 ? p0 : p1;
            descend(bit, bit, __dmul_rn(__dsub_rn(1.0, dxy), p_bit));
            descend(bit, 1 - bit, __dmul_rn(dxy, p_other));
        }
    } else if (p.kind == SHS_ERR_CLASSICAL_MEASURE) {
        for (int bit = 0; bit < 2; ++bit) {
            const double p_bit = bit == 1 ? p1 : p0;
            descend(bit, bit, __dmul_rn(p_bit, __dsub_rn(1.0, p.delta)));
            descend(1 - bit, bit, __dmul_rn(p_bit, p.delta));
        }
    } else {
        descend(0, 0, p0);
        descend(1, 1, p1);
    }
    for (; k < 4; ++k) out[k] = ExhSlot{};
}

struct Enumerator {
    ExhParams base{};
    std::vector<uint64_t> a_pows, a_invs;
    std::vector<double> dist;
    uint64_t budget = 0;
    size_t smem = 0;

    void count(uint64_t n) {
        if (n > budget) {
            set_error(SHS_BUDGET_EXCEEDED, "exhaustive_joint_distribution: node budget exhausted");
            throw SHS_BUDGET_EXCEEDED;
        }
        budget -= n;
    }

    // one level, nodes in DFS order; parent_h = the h buffers of their parents' chunk
    void level(uint32_t s, const std::vector<ExhNode>& nodes, const double2* parent_h) {
        for (size_t c0 = 0; c0 < nodes.size(); c0 += kExhChunk) {
            const uint32_t n = static_cast<uint32_t>(std::min<size_t>(kExhChunk, nodes.size() - c0));
            count(n);  // one recurse() call per node
            ExhNode* d_nodes = nullptr;
            double2* d_h = nullptr;
            ExhSlot* d_slots = nullptr;
            EXH_CUDA(cudaMalloc(&d_nodes, sizeof(ExhNode) * n));
            EXH_CUDA(cudaMalloc(&d_h, sizeof(double2) * 2 * base.N * n));
            EXH_CUDA(cudaMalloc(&d_slots, sizeof(ExhSlot) * 4 * n));
            EXH_CUDA(cudaMemcpy(d_nodes, nodes.data() + c0, sizeof(ExhNode) * n, cudaMemcpyHostToDevice));
            ExhParams p = base;
            p.s = s;
            p.root = s == 0;
            p.gather = a_pows[s] != 1;
            p.m = a_invs[s];
            p.m_sh = p.gather ? shoup(p.m, p.N) : 0;
            p.nodes = d_nodes;
            p.parent_h = parent_h;
            p.h_out = d_h;
            p.slots = d_slots;
            k_exh_stage<<<n, kExhThreads, smem>>>(p);
            EXH_CUDA(cudaGetLastError());
            std::vector<ExhSlot> slots(4 * size_t(n));
            EXH_CUDA(cudaMemcpy(slots.data(), d_slots, sizeof(ExhSlot) * 4 * n, cudaMemcpyDeviceToHost));
            cudaFree(d_nodes);
            cudaFree(d_slots);
            std::vector<ExhNode> children;
            for (uint32_t i = 0; i < n; ++i)
                for (int k = 0; k < 4; ++k) {
                    const ExhSlot& sl = slots[size_t(i) * 4 + k];
                    if (sl.kind == 2) {
                        count(1);  // the leaf's budget tick, statevector.cpp:491-493
                        dist[sl.observed] += sl.weight;  // in DFS order
                    } else if (sl.kind == 1) {
                        children.push_back(ExhNode{i, sl.src_group, sl.inv, sl.weight, sl.observed});
                    }
                }
            if (!children.empty()) level(s + 1, children, d_h);
            cudaFree(d_h);
        }
    }
};

}  // namespace

extern "C" int shs_exhaustive_distribution(const shs_problem* problem, const shs_error* error,
                                           uint64_t node_budget, int32_t device, double* out) {
    if (!problem || !error) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    // statevector.cpp:536-538: the reference's limits come first
    if (problem->t > 14 || problem->L + 1 > 12)
        return set_error(SHS_BUDGET_EXCEEDED,
                         "exhaustive_joint_distribution: t <= 14 and n <= 12 required");
    if (!out) return set_error(SHS_INVALID_ARGUMENT, "null argument");
    std::string why;
    if (validate_error(*error, &why)) return set_error(SHS_CONFIG_ERROR, why);
    if (problem->N < 2 || problem->t < 1 || problem->N > (uint64_t(1) << problem->L))
        return set_error(SHS_INVALID_ARGUMENT, "invalid problem");
    try {
        cudaError_t ce = cudaSetDevice(device);
        if (ce != cudaSuccess) {
            set_error(SHS_CUDA_ERROR, cudaGetErrorString(ce));
            return SHS_CUDA_ERROR;
        }
        Enumerator en;
        const uint32_t t = problem->t;
        const uint64_t N = problem->N, group = uint64_t(1) << problem->L;
        en.budget = node_budget;
        en.dist.assign(size_t(1) << t, 0.0);
        en.a_pows.assign(t, 0);
        en.a_invs.assign(t, 1);
        en.a_pows[t - 1] = problem->a % N;
        for (uint32_t s = t - 1; s > 0; --s) en.a_pows[s - 1] = mulmod(en.a_pows[s], en.a_pows[s], N);
        for (uint32_t s = 0; s < t; ++s) {
            if (en.a_pows[s] == 1) continue;
            u64 g = 0;
            if (mod_inverse(en.a_pows[s], N, &en.a_invs[s], &g) != SHS_OK)
                return set_error(SHS_NOT_INVERTIBLE, "not invertible: gcd(" +
                                                         std::to_string(en.a_pows[s]) + ", " +
                                                         std::to_string(N) + ") = " + std::to_string(g));
        }
        double w[4];
        reinit_state(*error, w);
        std::vector<double2> phase((size_t(1) << t) - 1);
        for (uint32_t s = 0; s < t; ++s)
            for (uint64_t pfx = 0; pfx < (uint64_t(1) << s); ++pfx) {
                const double phi = stage_phase(s, pfx);
                phase[((uint64_t(1) << s) - 1) + pfx] = make_double2(1.0 * std::cos(phi), 1.0 * std::sin(phi));
            }
        double2* d_phase = nullptr;
        EXH_CUDA(cudaMalloc(&d_phase, sizeof(double2) * phase.size()));
        EXH_CUDA(cudaMemcpy(d_phase, phase.data(), sizeof(double2) * phase.size(), cudaMemcpyHostToDevice));
        en.base.N = N;
        en.base.group = group;
        en.base.t = t;
        en.base.w0r = w[0];
        en.base.w0i = w[1];
        en.base.w1r = w[2];
        en.base.w1i = w[3];
        en.base.phase = d_phase;
        en.base.kind = error->kind;
        en.base.delta = error->delta;
        en.base.px = error->px;
        en.base.py = error->py;
        en.smem = sizeof(double) * 2 * group;
        EXH_CUDA(cudaFuncSetAttribute(k_exh_stage, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(en.smem)));
        std::vector<ExhNode> root{ExhNode{0, 0, 1.0, 1.0, 0}};
        try {
            en.level(0, root, nullptr);
        } catch (...) {
            cudaFree(d_phase);
            throw;
        }
        cudaFree(d_phase);
        if (error->kind == SHS_ERR_BITFLIP && error->delta > 0.0) {  // statevector.cpp:564-577
            auto& dist = en.dist;
            const double d = error->delta;
            for (unsigned bit = 0; bit < t; ++bit) {
                const size_t step = size_t(1) << bit;
                for (size_t j = 0; j < dist.size(); ++j) {
                    if (j & step) continue;
                    const double a = dist[j], b = dist[j | step];
                    dist[j] = (1.0 - d) * a + d * b;
                    dist[j | step] = (1.0 - d) * b + d * a;
                }
            }
        }
        std::memcpy(out, en.dist.data(), sizeof(double) * en.dist.size());
        return SHS_OK;
    } catch (int code) {
        return code;
    }
}
