/* TEST INFRASTRUCTURE ONLY — see shor_oracle.h. Compiled with
 * -ffp-contract=off, as the reference is (proj/CMakeLists.txt:17-20), so every
 * floating-point operation below rounds exactly where the reference's does. */
#include "shor_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

struct par_job_hdr { void (*fn)(void*, uint64_t, uint64_t); void* ctx; uint64_t lo, hi; };
static void* par_trampoline(void* p) {
    struct par_job_hdr* j = (struct par_job_hdr*)p;
    j->fn(j->ctx, j->lo, j->hi);
    return NULL;
}

typedef unsigned __int128 u128;
typedef __int128 i128;

enum {
    SO_OK = 0,
    SO_ERROR = 1,
    SO_CONFIG = 2,
    SO_CEILING = 3,
    SO_DEGENERATE = 4,
    SO_BUDGET = 5,
    SO_NOT_INVERTIBLE = 6,
    SO_INVALID = 7
};

enum { K_NONE = 0, K_AMP = 1, K_PHASE = 2, K_CLASSICAL = 3, K_QUANTUM = 4, K_BITFLIP = 5 };

static const double kInvSqrt2 = 0.70710678118654752440; /* statevector.cpp:14 */
static const double kPi = 3.14159265358979323846;       /* statevector.cpp:15 */
#define BLOCK 256u                                      /* statevector.cpp:16 */
static const double kNormTolerance = 1e-9;              /* statevector.cpp:18 */
static const double kDegenerateMass = 1e-300;           /* statevector.cpp:19 */

/* ---------------------------------------------------------------- rng */
/* philox::block, proj/include/shorsim/rng.hpp:16-31 */
void so_philox_block(uint64_t key, const uint32_t in[4], uint32_t out[4]) {
    uint32_t c0 = in[0], c1 = in[1], c2 = in[2], c3 = in[3];
    uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
    for (int round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* RngStream::at, rng.hpp:34-37 and 70 (counter = index, a, b, domain) */
uint64_t so_rng_u64(uint64_t seed, uint32_t a, uint32_t b, uint32_t domain, uint32_t index) {
    uint32_t ctr[4] = {index, a, b, domain}, out[4];
    so_philox_block(seed, ctr, out);
    return ((uint64_t)out[0] << 32) | out[1];
}

/* RngStream::next_double, rng.hpp:66 */
double so_rng_double(uint64_t seed, uint32_t a, uint32_t b, uint32_t domain, uint32_t index) {
    return (double)(so_rng_u64(seed, a, b, domain, index) >> 11) * 0x1.0p-53;
}

/* ---------------------------------------------------------- numtheory */
uint64_t so_mulmod(uint64_t a, uint64_t b, uint64_t m) { /* int128.hpp:28-30 */
    return (uint64_t)(((u128)a * b) % m);
}

/* ext_gcd + mod_inverse, numtheory.cpp:25-46 */
int so_mod_inverse(uint64_t a, uint64_t n, uint64_t* inv, uint64_t* gcd) {
    if (n < 2) return SO_INVALID;
    i128 old_r = (i128)(a % n), r = (i128)n, old_x = 1, x = 0;
    if (old_r == 0 && r == 0) return SO_INVALID;
    while (r != 0) {
        i128 q = old_r / r, tmp;
        tmp = old_r - q * r; old_r = r; r = tmp;
        tmp = old_x - q * x; old_x = x; x = tmp;
    }
    if (gcd) *gcd = (uint64_t)old_r;
    if (old_r != 1) return SO_NOT_INVERTIBLE;
    i128 v = old_x % (i128)n;
    if (v < 0) v += n;
    *inv = (uint64_t)v;
    return SO_OK;
}

unsigned so_bit_length(uint64_t n) { /* int128.hpp:20-24 */
    unsigned b = 0;
    while (n) { ++b; n >>= 1; }
    return b;
}

unsigned so_recommended_t(uint64_t n) { /* problems.cpp:17-23 */
    u128 n2 = (u128)n * n;
    unsigned t = 0;
    while (((u128)1 << t) < n2) ++t;
    return t;
}

int so_index_map(uint64_t a_pow, uint64_t n, uint64_t first, uint64_t count, uint64_t* out) {
    uint64_t inv, g;
    if (n < 2) return SO_INVALID;
    a_pow %= n;
    int rc = so_mod_inverse(a_pow, n, &inv, &g);
    if (rc) return rc;
    for (uint64_t i = 0; i < count; ++i) out[i] = so_mulmod(inv, first + i, n);
    return SO_OK;
}

/* -------------------------------------------------------------- noise */
int so_error_validate(const so_error* e) { /* noise.cpp:13-25 */
    if (e->delta < 0.0 || e->delta > 1.0) return SO_CONFIG;
    if (e->kind < K_NONE || e->kind > K_BITFLIP) return SO_CONFIG;
    if (e->kind == K_QUANTUM) {
        if (!e->has_pauli) return SO_CONFIG;
        if (e->px < 0 || e->py < 0 || e->pz < 0 || e->px + e->py + e->pz > 1.0) return SO_CONFIG;
        double d = e->px + e->py;
        if (fabs(d - e->delta) > 1e-12) return SO_CONFIG;
    } else if (e->has_pauli) {
        return SO_CONFIG;
    }
    return SO_OK;
}

/* reinit_state, noise.cpp:81-95 (std::polar(rho, th) = (rho cos th, rho sin th)) */
void so_reinit_state(const so_error* e, double out[4]) {
    if (e->kind == K_AMP) {
        out[0] = sqrt((1.0 + e->delta) / 2.0); out[1] = 0.0;
        out[2] = sqrt((1.0 - e->delta) / 2.0); out[3] = 0.0;
    } else if (e->kind == K_PHASE) {
        double th = kPi * e->delta;
        out[0] = kInvSqrt2; out[1] = 0.0;
        out[2] = kInvSqrt2 * cos(th); out[3] = kInvSqrt2 * sin(th);
    } else {
        out[0] = kInvSqrt2; out[1] = 0.0;
        out[2] = kInvSqrt2; out[3] = 0.0;
    }
}

/* stage_phase, statevector.cpp:201-206 */
double so_stage_phase(unsigned cbit, uint64_t lo, uint64_t hi) {
    if (cbit == 0) return 0.0;
    u128 prefix = ((u128)hi << 64) | lo;
    return kPi * (double)prefix * exp2(-(double)cbit);
}

/* sample_measurement, statevector.cpp:236-256, with classical_flip and
 * depolarizing_measure_branch from noise.cpp:128-145 */
void so_sample_measurement(double p1, uint64_t seed, uint32_t idx, uint32_t stage,
                           const so_error* e, int32_t out[4]) {
    uint32_t draw = 0;
#define NEXT() so_rng_double(seed, idx, stage, 0u, draw++)
    out[2] = 0;
    out[3] = 0;
    if (e->kind == K_QUANTUM) {
        double dxy = e->px + e->py;
        double p1p = (1.0 - dxy) * p1 + dxy * (1.0 - p1);
        int bit = NEXT() < p1p ? 1 : 0;
        double p_bit = bit == 1 ? p1 : 1.0 - p1;
        double p_other = 1.0 - p_bit;
        double p_bit_prime = bit == 1 ? p1p : 1.0 - p1p;
        double p_err = p_bit_prime > 0.0 ? dxy * p_other / p_bit_prime : 0.0;
        out[0] = bit;
        out[1] = bit;
        out[2] = NEXT() < p_err ? 1 : 0;
        return;
    }
    double r = NEXT();
    out[0] = r < p1 ? 1 : 0;
    out[1] = out[0];
    if (e->kind == K_CLASSICAL) {
        int flip = NEXT() < e->delta;
        out[1] = flip ? 1 - out[0] : out[0];
        out[3] = flip;
    }
#undef NEXT
}

/* bitflip_bitstring, noise.cpp:147-151, stream (seed, idx, 0, bitflip) */
void so_bitflip(uint64_t j[2], unsigned t, double delta, uint64_t seed, uint32_t idx) {
    u128 v = ((u128)j[1] << 64) | j[0];
    for (unsigned i = 0; i < t; ++i)
        if (so_rng_double(seed, idx, 0, 1u, i) < delta) v ^= (u128)1 << i;
    j[0] = (uint64_t)v;
    j[1] = (uint64_t)(v >> 64);
}

/* ------------------------------------------------------------ sums */
double so_combine_blocks(const double* blocks, uint64_t count) { /* statevector.cpp:21-40 */
    double sum = 0, comp = 0;
    for (uint64_t i = 0; i < count; ++i) {
        if (blocks[i] != 0.0) {
            double y = blocks[i] - comp;
            double t = sum + y;
            comp = (t - sum) - y;
            sum = t;
        }
    }
    return sum;
}

/* Exact fixed-point sum: value v = F * 2^-1088 with F held in 32-bit digits. */
#define XS_DIGITS 40
#define XS_ANCHOR 1088
static void xs_add(uint64_t* acc, double v) {
    if (v == 0.0) return;
    int e;
    double m = frexp(v, &e);                        /* v = m * 2^e, 0.5 <= m < 1 */
    uint64_t mant = (uint64_t)ldexp(m, 53);         /* exact: 53-bit integer */
    int shift = e - 53 + XS_ANCHOR;                 /* v = mant * 2^(shift - ANCHOR) */
    if (shift < 0) { mant >>= -shift; shift = 0; }  /* never for subnormal >= 2^-1074 */
    int d = shift / 32, off = shift % 32;
    u128 w = (u128)mant << off;                     /* < 2^85: spans 3 digits */
    acc[d] += (uint64_t)(w & 0xffffffffu);
    acc[d + 1] += (uint64_t)((w >> 32) & 0xffffffffu);
    acc[d + 2] += (uint64_t)(w >> 64);
}

static double xs_round(uint64_t* acc) {
    uint64_t carry = 0;
    for (int i = 0; i < XS_DIGITS; ++i) {
        uint64_t v = acc[i] + carry;
        acc[i] = v & 0xffffffffu;
        carry = v >> 32;
    }
    int top = -1;
    for (int i = XS_DIGITS - 1; i >= 0 && top < 0; --i)
        if (acc[i]) top = i * 32 + 63 - __builtin_clzll(acc[i]);
    if (top < 0) return 0.0;
#define BIT(p) ((p) >= 0 ? (int)((acc[(p) / 32] >> ((p) % 32)) & 1u) : 0)
    int lsb = top - 52;
    if (lsb < XS_ANCHOR - 1074) lsb = XS_ANCHOR - 1074; /* subnormal quantum */
    uint64_t mant = 0;
    for (int p = top; p >= lsb; --p) mant = (mant << 1) | (uint64_t)BIT(p);
    int round = BIT(lsb - 1);
    int sticky = 0;
    for (int p = lsb - 2; p >= 0 && !sticky; --p) sticky = BIT(p);
#undef BIT
    if (round && (sticky || (mant & 1))) ++mant;
    return ldexp((double)mant, lsb - XS_ANCHOR);
}

double so_exact_sum(const double* values, uint64_t count) {
    uint64_t acc[XS_DIGITS + 2];
    memset(acc, 0, sizeof(acc));
    for (uint64_t i = 0; i < count; ++i) xs_add(acc, values[i]);
    return xs_round(acc);
}

/* ------------------------------------------------------------- engine */
struct so_engine {
    uint64_t N, a;
    unsigned L, t;
    so_error err;
    int check_norms;
    double w[4];        /* reinit (w0, w1) */
    uint64_t* a_pows;   /* a^(2^(t-1-s)) mod N, statevector.cpp:302-306 */
    uint64_t* a_invs;   /* mod_inverse per stage (0 for identity stages) */
    double* sel;        /* N complex: selected post-Hadamard group, interleaved */
    double* nxt;        /* scratch for the next selection */
    double inv;         /* 1/sqrt(p_src) */
    uint64_t nblocks;
    double* bsum;       /* 2 * nblocks */
    /* pending stage */
    int pending;
    unsigned ps;
    double ph[2];
    int phase_mul;      /* gather || phi != 0 */
    double p0, p1;
};

static int engine_validate(uint64_t N, unsigned L, unsigned t, const so_error* e,
                           unsigned shard_count, unsigned qubit_ceiling) {
    int rc = so_error_validate(e); /* statevector.cpp:289 */
    if (rc) return rc;
    unsigned n = L + 1;
    if (n > qubit_ceiling) return SO_CEILING; /* statevector.cpp:291-294 */
    /* make_shard_layout validation, statevector.cpp:65-72 (the n <= 33 cap of
     * the u32 layout is lifted: indices are u64 here) */
    if (n < 2) return SO_INVALID;
    if (shard_count < 2 || (shard_count & (shard_count - 1)) != 0) return SO_INVALID;
    if ((unsigned)__builtin_ctz(shard_count) > n - 1) return SO_INVALID;
    if (N < 2 || t < 1 || L > 63 || N > ((uint64_t)1 << L)) return SO_INVALID;
    return SO_OK;
}

int so_engine_create(uint64_t N, uint64_t a, unsigned L, unsigned t, const so_error* e,
                     unsigned shard_count, unsigned qubit_ceiling, int check_norms,
                     so_engine** out) {
    int rc = engine_validate(N, L, t, e, shard_count, qubit_ceiling);
    if (rc) return rc;
    so_engine* g = (so_engine*)calloc(1, sizeof(so_engine));
    g->N = N; g->a = a; g->L = L; g->t = t; g->err = *e; g->check_norms = check_norms;
    so_reinit_state(e, g->w);
    g->a_pows = (uint64_t*)calloc(t, sizeof(uint64_t));
    g->a_invs = (uint64_t*)calloc(t, sizeof(uint64_t));
    g->a_pows[t - 1] = a % N;
    for (unsigned s = t - 1; s > 0; --s) g->a_pows[s - 1] = so_mulmod(g->a_pows[s], g->a_pows[s], N);
    for (unsigned s = 0; s < t; ++s) {
        if (g->a_pows[s] == 1) continue;
        uint64_t gcd;
        rc = so_mod_inverse(g->a_pows[s], N, &g->a_invs[s], &gcd);
        if (rc) { so_engine_destroy(g); return rc; }
    }
    g->sel = (double*)malloc(sizeof(double) * 2 * N);
    g->nxt = (double*)malloc(sizeof(double) * 2 * N);
    g->nblocks = (N + BLOCK - 1) / BLOCK;
    g->bsum = (double*)malloc(sizeof(double) * 2 * g->nblocks);
    if (!g->sel || !g->nxt || !g->bsum) { so_engine_destroy(g); return SO_INVALID; }
    so_state_init(g);
    *out = g;
    return SO_OK;
}

void so_engine_destroy(so_engine* g) {
    if (!g) return;
    free(g->a_pows); free(g->a_invs); free(g->sel); free(g->nxt); free(g->bsum);
    free(g);
}

int so_engine_multipliers(const so_engine* g, uint64_t* out) {
    memcpy(out, g->a_pows, sizeof(uint64_t) * g->t);
    return SO_OK;
}

uint64_t so_num_blocks(const so_engine* g) { return g->nblocks; }

/* run start, statevector.cpp:326-329, as sel = e_1 with inv = 1:
 * w_x * (e_1 * 1) == w_x numerically (only a zero's sign may differ). */
int so_state_init(so_engine* g) {
    memset(g->sel, 0, sizeof(double) * 2 * g->N);
    g->sel[2] = 1.0;
    g->inv = 1.0;
    g->pending = 0;
    return SO_OK;
}

/* complex multiply as GCC lowers it with -ffp-contract=off: (ac - bd, ad + bc) */
#define CMUL(ar, ai, br, bi, or_, oi) \
    do { double _r = (ar) * (br) - (ai) * (bi); double _i = (ar) * (bi) + (ai) * (br); \
         (or_) = _r; (oi) = _i; } while (0)

/* Post-Hadamard pair at z (Appendix A steps 1-3; statevector.cpp:344-364). */
static inline void stage_pair(const so_engine* g, uint64_t z, uint64_t src, double h[4]) {
    double inv = g->inv;
    double xr = g->sel[2 * z] * inv, xi = g->sel[2 * z + 1] * inv;
    double sr = g->sel[2 * src] * inv, si = g->sel[2 * src + 1] * inv;
    double ur, ui, vr, vi;
    CMUL(g->w[0], g->w[1], xr, xi, ur, ui);   /* g0[z] = w0 * v      (reset, :397) */
    CMUL(g->w[2], g->w[3], sr, si, vr, vi);   /* g1[src] = w1 * v    (reset, :398) */
    if (g->phase_mul) CMUL(vr, vi, g->ph[0], g->ph[1], vr, vi); /* * ph  (:345 / :360) */
    h[0] = (ur + vr) * kInvSqrt2;             /* h0 (:361) */
    h[1] = (ui + vi) * kInvSqrt2;
    h[2] = (ur - vr) * kInvSqrt2;             /* h1 (:362) */
    h[3] = (ui - vi) * kInvSqrt2;
}

/* Host-thread fan-out over independent index ranges (block partials are each a
 * sequential in-order sum, collapse is elementwise: results do not depend on
 * the thread count). SO_THREADS overrides the online core count. */
static void par_for(uint64_t n, void (*fn)(void*, uint64_t, uint64_t), void* ctx) {
    long nt = sysconf(_SC_NPROCESSORS_ONLN);
    const char* env = getenv("SO_THREADS");
    if (env) nt = atol(env);
    if (nt < 1) nt = 1;
    if (nt > 64) nt = 64;
    if (n < 65536 || nt == 1) { fn(ctx, 0, n); return; }
    pthread_t th[64];
    struct par_job { void (*fn)(void*, uint64_t, uint64_t); void* ctx; uint64_t lo, hi; } jobs[64];
    uint64_t per = (n + (uint64_t)nt - 1) / (uint64_t)nt;
    for (long i = 0; i < nt; ++i) {
        uint64_t lo = per * (uint64_t)i, hi = lo + per < n ? lo + per : n;
        jobs[i].fn = fn; jobs[i].ctx = ctx; jobs[i].lo = lo < n ? lo : n; jobs[i].hi = hi;
    }
    for (long i = 1; i < nt; ++i) pthread_create(&th[i], NULL, par_trampoline, &jobs[i]);
    fn(ctx, jobs[0].lo, jobs[0].hi);
    for (long i = 1; i < nt; ++i) pthread_join(th[i], NULL);
}

struct probs_ctx { const so_engine* g; int gather; uint64_t m; double* b0; double* b1; };
static void probs_range(void* vc, uint64_t lo, uint64_t hi) {
    struct probs_ctx* c = (struct probs_ctx*)vc;
    const uint64_t N = c->g->N;
    for (uint64_t b = lo; b < hi; ++b) { /* statevector.cpp:353-371 */
        uint64_t z = b * BLOCK, ze = z + BLOCK < N ? z + BLOCK : N;
        double s0 = 0, s1 = 0, h[4];
        for (; z < ze; ++z) {
            uint64_t src = c->gather ? so_mulmod(c->m, z, N) : z;
            stage_pair(c->g, z, src, h);
            s0 += h[0] * h[0] + h[1] * h[1]; /* std::norm */
            s1 += h[2] * h[2] + h[3] * h[3];
        }
        c->b0[b] = s0;
        c->b1[b] = s1;
    }
}

struct collapse_ctx { so_engine* g; int gather; uint64_t m; int src_group; };
static void collapse_range(void* vc, uint64_t lo, uint64_t hi) {
    struct collapse_ctx* c = (struct collapse_ctx*)vc;
    so_engine* g = c->g;
    for (uint64_t z = lo; z < hi; ++z) {
        double h[4];
        stage_pair(g, z, c->gather ? so_mulmod(c->m, z, g->N) : z, h);
        g->nxt[2 * z] = h[2 * c->src_group];
        g->nxt[2 * z + 1] = h[2 * c->src_group + 1];
    }
}

int so_stage_probs(so_engine* g, unsigned s, uint64_t lo, uint64_t hi, int combine_mode,
                   double* p0, double* p1) {
    if (s >= g->t) return SO_INVALID;
    double phi = so_stage_phase(s, lo, hi);
    g->ph[0] = 1.0 * cos(phi); /* std::polar(1.0, phi), statevector.cpp:338 */
    g->ph[1] = 1.0 * sin(phi);
    int gather = g->a_pows[s] != 1;
    g->phase_mul = gather || phi != 0.0;
    g->ps = s;
    uint64_t N = g->N, m = g->a_invs[s];
    double* b0 = g->bsum;
    double* b1 = g->bsum + g->nblocks;
    /* blocks are independent (each a sequential in-order sum): threads over blocks */
    struct probs_ctx c = {g, gather, m, b0, b1};
    par_for(g->nblocks, probs_range, &c);
    if (combine_mode == 0) {
        g->p0 = so_combine_blocks(b0, g->nblocks);
        g->p1 = so_combine_blocks(b1, g->nblocks);
    } else {
        g->p0 = so_exact_sum(b0, g->nblocks);
        g->p1 = so_exact_sum(b1, g->nblocks);
    }
    g->pending = 1;
    *p0 = g->p0;
    *p1 = g->p1;
    if (g->check_norms && fabs(g->p0 + g->p1 - 1.0) > kNormTolerance) return SO_ERROR; /* :374 */
    return SO_OK;
}

int so_stage_block_sums(so_engine* g, double* out) {
    if (!g->pending) return SO_INVALID;
    memcpy(out, g->bsum, sizeof(double) * 2 * g->nblocks);
    return SO_OK;
}

int so_stage_read(so_engine* g, int x, uint64_t first, uint64_t count, double* out) {
    if (!g->pending) return SO_INVALID;
    int gather = g->a_pows[g->ps] != 1;
    for (uint64_t i = 0; i < count; ++i) {
        uint64_t z = first + i;
        if (z >= g->N) { out[2 * i] = 0.0; out[2 * i + 1] = 0.0; continue; }
        double h[4];
        stage_pair(g, z, gather ? so_mulmod(g->a_invs[g->ps], z, g->N) : z, h);
        out[2 * i] = h[2 * x];
        out[2 * i + 1] = h[2 * x + 1];
    }
    return SO_OK;
}

/* collapse/reset, statevector.cpp:384-401: new sel = h_src, inv = 1/sqrt(p_src) */
int so_stage_collapse(so_engine* g, int src_group, double p_src) {
    if (!g->pending) return SO_INVALID;
    if (p_src < kDegenerateMass) return SO_DEGENERATE;
    int gather = g->a_pows[g->ps] != 1;
    uint64_t N = g->N, m = g->a_invs[g->ps];
    struct collapse_ctx c = {g, gather, m, src_group};
    par_for(N, collapse_range, &c);
    double* tmp = g->sel; g->sel = g->nxt; g->nxt = tmp;
    g->inv = 1.0 / sqrt(p_src);
    g->pending = 0;
    return SO_OK;
}

int so_state_read(so_engine* g, int x, uint64_t first, uint64_t count, double* out) {
    for (uint64_t i = 0; i < count; ++i) {
        uint64_t z = first + i;
        if (z >= g->N) { out[2 * i] = 0.0; out[2 * i + 1] = 0.0; continue; }
        double vr = g->sel[2 * z] * g->inv, vi = g->sel[2 * z + 1] * g->inv, r, im;
        CMUL(g->w[2 * x], g->w[2 * x + 1], vr, vi, r, im);
        out[2 * i] = r;
        out[2 * i + 1] = im;
    }
    return SO_OK;
}

/* IterativeShorEngine::run, statevector.cpp:323-412 */
int so_engine_run(so_engine* g, uint64_t seed, uint64_t idx, int combine_mode, uint64_t j[2],
                  uint64_t js[2], double* p1s, int32_t* ints) {
    so_state_init(g);
    u128 observed = 0, sampled = 0;
    for (unsigned s = 0; s < g->t; ++s) {
        double p0, p1;
        int rc = so_stage_probs(g, s, (uint64_t)observed, (uint64_t)(observed >> 64), combine_mode,
                                &p0, &p1);
        if (rc) return rc;
        int32_t mr[4];
        so_sample_measurement(p1, seed, (uint32_t)idx, s, &g->err, mr);
        if (p1s) p1s[s] = p1;
        if (ints) {
            ints[4 * s + 0] = mr[0];
            ints[4 * s + 1] = mr[1];
            ints[4 * s + 2] = mr[3];
            ints[4 * s + 3] = mr[2];
        }
        observed |= (u128)(unsigned)mr[1] << s;
        sampled |= (u128)(unsigned)mr[0] << s;
        if (s + 1 < g->t) {
            int src_group = mr[2] ? 1 - mr[0] : mr[0];
            double p_src = src_group == 1 ? p1 : p0;
            rc = so_stage_collapse(g, src_group, p_src);
            if (rc) return rc;
        }
    }
    js[0] = (uint64_t)sampled;
    js[1] = (uint64_t)(sampled >> 64);
    j[0] = (uint64_t)observed;
    j[1] = (uint64_t)(observed >> 64);
    if (g->err.kind == K_BITFLIP) so_bitflip(j, g->t, g->err.delta, seed, (uint32_t)idx);
    return SO_OK;
}

/* ------------------------------------------------- sparse-support engine
 * The same stage recipe (Appendix A; statevector.cpp:339-401) on the support
 * of the state only, for N too large for the dense restatement (config 4,
 * N ~ 2^32). From the run start e_1 (statevector.cpp:326-329), stage s can only
 * make amplitudes at z and A_s * z nonzero (the gather of :345 reads sel[a_inv
 * z]), so sel lives on a sorted set of indices. Every amplitude outside it is
 * exactly zero: its |h|^2 is +0.0 and adding +0.0 leaves the reference's
 * in-order 256-block sums (:354-370) unchanged, and all-zero blocks are
 * skipped by combine_blocks (:32-40). Hence p0/p1 and every support amplitude
 * equal the dense computation's; no assumption about the orbit is made (the
 * candidate set is a sorted union, so wraps and collisions are handled). */
struct so_sparse {
    uint64_t N;
    unsigned t;
    so_error err;
    int check_norms;
    double w[4];
    uint64_t* a_pows;
    uint64_t* a_invs;
    uint64_t n;       /* support size of sel */
    uint64_t* z;      /* sorted support */
    double* v;        /* sel values, interleaved */
    double inv;
    int pending;
    unsigned ps;
    double ph[2];
    int phase_mul;
    uint64_t nc;      /* pending stage: candidate indices (sorted) and h0, h1 */
    uint64_t* cz;
    double* ch;       /* 4 per candidate */
    double p0, p1;
};

void so_sparse_destroy(so_sparse* g) {
    if (!g) return;
    free(g->a_pows); free(g->a_invs); free(g->z); free(g->v); free(g->cz); free(g->ch);
    free(g);
}

int so_sparse_create(uint64_t N, uint64_t a, unsigned L, unsigned t, const so_error* e,
                     int check_norms, so_sparse** out) {
    int rc = engine_validate(N, L, t, e, 2, 127);
    if (rc) return rc;
    so_sparse* g = (so_sparse*)calloc(1, sizeof(so_sparse));
    g->N = N; g->t = t; g->err = *e; g->check_norms = check_norms;
    so_reinit_state(e, g->w);
    g->a_pows = (uint64_t*)calloc(t, sizeof(uint64_t));
    g->a_invs = (uint64_t*)calloc(t, sizeof(uint64_t));
    g->a_pows[t - 1] = a % N; /* statevector.cpp:302-306 */
    for (unsigned s = t - 1; s > 0; --s) g->a_pows[s - 1] = so_mulmod(g->a_pows[s], g->a_pows[s], N);
    for (unsigned s = 0; s < t; ++s) {
        if (g->a_pows[s] == 1) continue;
        uint64_t gcd;
        rc = so_mod_inverse(g->a_pows[s], N, &g->a_invs[s], &gcd);
        if (rc) { so_sparse_destroy(g); return rc; }
    }
    so_sparse_init(g);
    *out = g;
    return SO_OK;
}

int so_sparse_init(so_sparse* g) {
    free(g->z); free(g->v); free(g->cz); free(g->ch);
    g->cz = NULL; g->ch = NULL; g->nc = 0;
    g->n = 1;
    g->z = (uint64_t*)malloc(sizeof(uint64_t));
    g->v = (double*)malloc(2 * sizeof(double));
    g->z[0] = 1; g->v[0] = 1.0; g->v[1] = 0.0; /* e_1, inv = 1 (see so_state_init) */
    g->inv = 1.0;
    g->pending = 0;
    return SO_OK;
}

static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : x > y;
}

/* index of z in the sorted support, or -1 */
static int64_t sp_find(const so_sparse* g, uint64_t z) {
    uint64_t lo = 0, hi = g->n;
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (g->z[mid] < z) lo = mid + 1;
        else hi = mid;
    }
    return (lo < g->n && g->z[lo] == z) ? (int64_t)lo : -1;
}

int so_sparse_stage_probs(so_sparse* g, unsigned s, uint64_t lo, uint64_t hi, int combine_mode,
                          double* p0, double* p1) {
    if (s >= g->t) return SO_INVALID;
    double phi = so_stage_phase(s, lo, hi);
    g->ph[0] = 1.0 * cos(phi); /* std::polar(1.0, phi), statevector.cpp:338 */
    g->ph[1] = 1.0 * sin(phi);
    int gather = g->a_pows[s] != 1;
    g->phase_mul = gather || phi != 0.0;
    g->ps = s;
    uint64_t N = g->N, A = g->a_pows[s], m = g->a_invs[s];
    /* candidates: support ∪ A * support (z with sel[z] or sel[a_inv z] nonzero) */
    uint64_t nc = gather ? 2 * g->n : g->n;
    free(g->cz); free(g->ch);
    g->cz = (uint64_t*)malloc(sizeof(uint64_t) * nc);
    memcpy(g->cz, g->z, sizeof(uint64_t) * g->n);
    if (gather)
        for (uint64_t i = 0; i < g->n; ++i) g->cz[g->n + i] = so_mulmod(A, g->z[i], N);
    qsort(g->cz, nc, sizeof(uint64_t), cmp_u64);
    uint64_t k = 0;
    for (uint64_t i = 0; i < nc; ++i)
        if (k == 0 || g->cz[i] != g->cz[k - 1]) g->cz[k++] = g->cz[i];
    nc = k;
    g->nc = nc;
    g->ch = (double*)malloc(sizeof(double) * 4 * (nc ? nc : 1));
    /* block partials in z order over the candidate set (statevector.cpp:353-371) */
    double* b0 = (double*)malloc(sizeof(double) * (nc ? nc : 1));
    double* b1 = (double*)malloc(sizeof(double) * (nc ? nc : 1));
    uint64_t nb = 0, cur = UINT64_MAX;
    double s0 = 0, s1 = 0;
    const double inv = g->inv;
    for (uint64_t i = 0; i < nc; ++i) {
        uint64_t z = g->cz[i];
        if (z / BLOCK != cur) {
            if (cur != UINT64_MAX) { b0[nb] = s0; b1[nb] = s1; ++nb; }
            cur = z / BLOCK; s0 = 0; s1 = 0;
        }
        int64_t ix = sp_find(g, z);
        int64_t is = sp_find(g, gather ? so_mulmod(m, z, N) : z);
        double xr = ix >= 0 ? g->v[2 * ix] : 0.0, xi = ix >= 0 ? g->v[2 * ix + 1] : 0.0;
        double sr = is >= 0 ? g->v[2 * is] : 0.0, si = is >= 0 ? g->v[2 * is + 1] : 0.0;
        xr *= inv; xi *= inv; sr *= inv; si *= inv;
        double ur, ui, vr, vi, *h = g->ch + 4 * i;
        CMUL(g->w[0], g->w[1], xr, xi, ur, ui);   /* g0[z] = w0 * v      (reset, :397) */
        CMUL(g->w[2], g->w[3], sr, si, vr, vi);   /* g1[src] = w1 * v    (reset, :398) */
        if (g->phase_mul) CMUL(vr, vi, g->ph[0], g->ph[1], vr, vi); /* * ph  (:345 / :360) */
        h[0] = (ur + vr) * kInvSqrt2;             /* h0 (:361) */
        h[1] = (ui + vi) * kInvSqrt2;
        h[2] = (ur - vr) * kInvSqrt2;             /* h1 (:362) */
        h[3] = (ui - vi) * kInvSqrt2;
        s0 += h[0] * h[0] + h[1] * h[1];          /* std::norm */
        s1 += h[2] * h[2] + h[3] * h[3];
    }
    if (cur != UINT64_MAX) { b0[nb] = s0; b1[nb] = s1; ++nb; }
    if (combine_mode == 0) {
        g->p0 = so_combine_blocks(b0, nb);
        g->p1 = so_combine_blocks(b1, nb);
    } else {
        g->p0 = so_exact_sum(b0, nb);
        g->p1 = so_exact_sum(b1, nb);
    }
    free(b0); free(b1);
    g->pending = 1;
    *p0 = g->p0;
    *p1 = g->p1;
    if (g->check_norms && fabs(g->p0 + g->p1 - 1.0) > kNormTolerance) return SO_ERROR; /* :374 */
    return SO_OK;
}

/* collapse/reset, statevector.cpp:384-401: sel = h_src on the candidates */
int so_sparse_stage_collapse(so_sparse* g, int src_group, double p_src) {
    if (!g->pending) return SO_INVALID;
    if (p_src < kDegenerateMass) return SO_DEGENERATE;
    free(g->z); free(g->v);
    g->n = g->nc;
    g->z = g->cz;
    g->v = (double*)malloc(sizeof(double) * 2 * (g->n ? g->n : 1));
    for (uint64_t i = 0; i < g->n; ++i) {
        g->v[2 * i] = g->ch[4 * i + 2 * src_group];
        g->v[2 * i + 1] = g->ch[4 * i + 2 * src_group + 1];
    }
    free(g->ch);
    g->cz = NULL; g->ch = NULL; g->nc = 0;
    g->inv = 1.0 / sqrt(p_src);
    g->pending = 0;
    return SO_OK;
}

uint64_t so_sparse_size(const so_sparse* g) { return g->n; }

/* sorted support and the materialised g_x = w_x * (sel * inv) there */
int so_sparse_state(const so_sparse* g, int x, uint64_t* z_out, double* out) {
    for (uint64_t i = 0; i < g->n; ++i) {
        if (z_out) z_out[i] = g->z[i];
        if (out) {
            double vr = g->v[2 * i] * g->inv, vi = g->v[2 * i + 1] * g->inv, r, im;
            CMUL(g->w[2 * x], g->w[2 * x + 1], vr, vi, r, im);
            out[2 * i] = r;
            out[2 * i + 1] = im;
        }
    }
    return SO_OK;
}
