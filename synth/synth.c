/*
 * synth.c — seeded synthetic inputs for the sparse gated FFN (X, W_g, W_u, W_d).
 *
 * This module is INPUT GENERATION ONLY.  It holds none of the method's arithmetic
 * (no GEMM, no threshold, no TwELL packing); both the CPU oracle (oracle/) and the
 * CUDA path (paper_2603_23198_b200/) consume the arrays it writes, and neither of
 * them is imported here.
 *
 * Statistics mimicked (recipe in DESIGN.md §"Input recipe"):
 *   - ReLU gate, no MLP bias (Table 2): sparsity comes from a
 *     per-token "bias" carried on K_b reserved input channels times a per-neuron
 *     coefficient, plus zero-mean noise on the remaining channels.
 *   - heavy-tailed per-token nnz: "the maximum number of non-zeros often exceeds the
 *     layer's mean by more than an order of magnitude" -> lognormal per-token
 *     density, clipped at pmax_ratio x mean.
 *   - more non-zeros for the first tokens of a sequence -> (1+pos)^-alpha.
 *   - "non-zero activations tend to have high correlation within input sequences"
 *      -> a fraction of noise channels is shared by all tokens of a sequence.
 *   - dead neurons -> a fraction of hidden units whose gate weights
 *     are zero on the noise channels and negative on the bias channels.
 *   - lognormal per-neuron popularity (hot neurons fire for far more tokens than
 *     cold ones, Fig 8): neuron n's bias coefficient beta_n = clip(BETA0 - BETA_S z_n,
 *     BETA_MIN, 7), z_n ~ N(0,1), in steps of 1/64, spread over the K_b bias channels; its
 *     firing probability Phi_c(beta_n c_m / s_m) is then close to lognormal in z_n (log Phi_c is
 *     near-linear in beta at the operating point, slope ~ -1.4 per unit of beta); BETA_S = 0.7
 *     gives a standard deviation of log(popularity) of 1.0 over the live neurons at 7B / 99%
 *     (measured on a 2048-token window), i.e. LogNormal(., 1) popularity; the hottest neuron
 *     fires for ~20% of tokens.
 *
 * Exactness: every element is q * 2^-e with |q_x| <= 14, |q_w| <= 7,
 * so X*W products are integer multiples of 2^-11 and every partial sum of a length
 * K <= 8192 dot product is below 2^20 units: exact in fp32 under any summation order.
 *
 * The RNG is counter based (splitmix64 of (seed, stream, flat index)), so any row can
 * be generated alone and results are independent of the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

typedef struct {
    int64_t M, K, N;
    uint64_t seed;
    double sparsity;   /* target mean fraction of zeros of relu(X Wg^T), e.g. 0.99 */
    double dead_frac;  /* fraction of hidden units that never activate */
    double tok_sigma;  /* lognormal sigma of per-token density (0 = uniform) */
    double pmax_ratio; /* per-token density clip, multiple of the mean density */
    double pos_alpha;  /* position decay exponent of per-token density */
    int64_t seq_len;   /* tokens per sequence (2048) */
    int64_t Kb;        /* reserved bias channels (<= K/2) */
    int32_t share_q;   /* in quarters: share a noise channel with the sequence if (bits&3) < share_q */
    int32_t x_exp;     /* X = q * 2^-x_exp */
    int32_t w_exp;     /* W = q * 2^-w_exp */
} synth_cfg;

enum { S_XTOK = 1, S_XSEQ = 2, S_XI = 3, S_WG = 4, S_WU = 5, S_WD = 6, S_NEU = 7, S_PAT = 8, S_PATV = 9 };

/* per-neuron popularity: beta = clip(BETA0 - BETA_S * z, BETA_MIN, BETA_MAX), quantised to 1/64 */
#ifndef BETA0
#define BETA0 5.0
#endif
#ifndef BETA_S
#define BETA_S 0.7
#endif
#ifndef BETA_MIN
#define BETA_MIN 1.5
#endif
#define BETA_MAX 7.0
#define BETA_Q 64
#define QX_MAX 14
#define QW_NOISE_VAR 5.0

static inline uint64_t sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static inline uint64_t key_of(uint64_t seed, uint64_t stream) {
    return sm64(sm64(seed) ^ (stream * 0xD1B54A32D192ED03ULL));
}
static inline uint64_t rnd(uint64_t key, uint64_t idx) {
    return sm64(key ^ (idx * 0xD6E8FEB86659FD93ULL));
}
/* sum of four U{0..7} minus 14: range [-14,14], variance 21 */
static inline int qx(uint64_t r) {
    return (int)((r & 7) + ((r >> 8) & 7) + ((r >> 16) & 7) + ((r >> 24) & 7)) - 14;
}
/* sum of four U{0..3} minus 6: range [-6,6], variance 5 */
static inline int qw(uint64_t r) {
    return (int)((r & 3) + ((r >> 8) & 3) + ((r >> 16) & 3) + ((r >> 24) & 3)) - 6;
}

static inline uint16_t q_to_bf16(int q, int e) {
    float f = ldexpf((float)q, -e);
    uint32_t u;
    memcpy(&u, &f, 4);
    return (uint16_t)(u >> 16); /* exact: |q| < 2^4 needs no rounding */
}
static inline void put(void* out, int out_f32, int64_t i, int q, int e) {
    if (out_f32)
        ((float*)out)[i] = ldexpf((float)q, -e);
    else
        ((uint16_t*)out)[i] = q_to_bf16(q, e);
}

static inline int beta_q_of_z(double z) {
    double b = BETA0 - BETA_S * z;
    if (b < BETA_MIN) b = BETA_MIN;
    if (b > BETA_MAX) b = BETA_MAX;
    return (int)lround(b * BETA_Q);
}

/* neuron n: bias coefficient beta_n * 64 (integer) and the dead flag */
int synth_neuron(const synth_cfg* c, int64_t n, int32_t* bq_out, int32_t* dead_out) {
    uint64_t r = rnd(key_of(c->seed, S_NEU), (uint64_t)n);
    double u1 = ((double)(r & 0xFFFFFF) + 0.5) / 16777216.0;
    double u2 = ((double)((r >> 24) & 0xFFFFFF) + 0.5) / 16777216.0;
    double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    int dead = ((double)((r >> 48) & 0xFFFF) / 65536.0) < c->dead_frac;
    if (bq_out) *bq_out = dead ? (int32_t)(BETA_MAX * BETA_Q) : beta_q_of_z(z);
    if (dead_out) *dead_out = dead;
    return 0;
}

/* bias-channel weight magnitudes of a neuron with coefficient bq/64: Bresenham split over the Kb channels
 * (each channel floor or ceil of beta, prefix sums within 1 of beta * prefix length) */
static inline int bias_w(int32_t bq, int64_t k) {
    return (int)(((int64_t)bq * (k + 1)) / BETA_Q - ((int64_t)bq * k) / BETA_Q);
}

/* Per-token target densities p[0..M): mean (1-sparsity), heavy tail, position decay, clipped. */
int synth_token_targets(const synth_cfg* c, double* p) {
    const int64_t M = c->M;
    if (M <= 0) return 0;
    uint64_t key = key_of(c->seed, S_XI);
    double pbar = 1.0 - c->sparsity, pmax = c->pmax_ratio * pbar;
    if (pmax > 0.5) pmax = 0.5;
    for (int64_t m = 0; m < M; ++m) {
        uint64_t r = rnd(key, (uint64_t)m);
        double u1 = ((double)(r & 0xFFFFFFFFULL) + 0.5) / 4294967296.0;
        double u2 = ((double)(r >> 32) + 0.5) / 4294967296.0;
        double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
        double xi = exp(c->tok_sigma * z - 0.5 * c->tok_sigma * c->tok_sigma);
        double pos = (double)(m % c->seq_len);
        p[m] = xi * pow(1.0 + pos, -c->pos_alpha);
    }
    /* find scale s with mean(min(s*raw, pmax)) == pbar (monotone in s) */
    double lo = 0.0, hi = 1.0;
    for (;;) {
        double acc = 0;
        for (int64_t m = 0; m < M; ++m) acc += fmin(hi * p[m], pmax);
        if (acc / (double)M >= pbar || hi > 1e12) break;
        hi *= 2.0;
    }
    for (int it = 0; it < 80; ++it) {
        double mid = 0.5 * (lo + hi), acc = 0;
        for (int64_t m = 0; m < M; ++m) acc += fmin(mid * p[m], pmax);
        if (acc / (double)M < pbar) lo = mid; else hi = mid;
    }
    for (int64_t m = 0; m < M; ++m) p[m] = fmin(hi * p[m], pmax);
    return 0;
}

/* expected density of a token with bias c_units and noise std s (units of 2^-(x_exp+w_exp)): the mean over the
 * live neurons' beta distribution (midpoint rule on z in [-6, 6] weighted by the normal density) */
#define NZ 121
static double density_model(const synth_cfg* c, double cu, double s) {
    double acc = 0, wsum = 0;
    for (int i = 0; i < NZ; ++i) {
        const double z = -6.0 + 12.0 * (i + 0.5) / NZ;
        const double w = exp(-0.5 * z * z);
        const double beta = (double)beta_q_of_z(z) / BETA_Q;
        acc += w * 0.5 * erfc((beta * cu / s) / 1.4142135623730951);
        wsum += w;
    }
    return (1.0 - c->dead_frac) * acc / wsum;
}

/* X rows [row0, row0+nrows) -> out (row-major, K per row). p = synth_token_targets output (length M).
 * If c_out != NULL, the chosen integer bias units per row are written there. */
int synth_x(const synth_cfg* c, const double* p, int64_t row0, int64_t nrows, int out_f32, void* out,
            int32_t* c_out) {
    const int64_t K = c->K, Kb = c->Kb;
    const uint64_t ktok = key_of(c->seed, S_XTOK), kseq = key_of(c->seed, S_XSEQ);
    const int cmax = (int)(Kb * QX_MAX);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nrows; ++i) {
        const int64_t m = row0 + i, seq = m / c->seq_len;
        double ss = 0;
        for (int64_t k = Kb; k < K; ++k) {
            uint64_t r = rnd(ktok, (uint64_t)(m * K + k));
            int q = ((int)((r >> 40) & 3) < c->share_q) ? qx(rnd(kseq, (uint64_t)(seq * K + k))) : qx(r);
            put(out, out_f32, i * K + k, q, c->x_exp);
            ss += (double)q * q;
        }
        double s = sqrt(ss * QW_NOISE_VAR);
        if (s < 1.0) s = 1.0;
        /* smallest integer bias cu with model density <= target, then the nearer neighbour */
        int lo = 0, hi = cmax;
        double target = p[m];
        if (density_model(c, (double)hi, s) > target) lo = hi;
        while (lo < hi) {
            int mid = (lo + hi) / 2;
            if (density_model(c, (double)mid, s) <= target) hi = mid; else lo = mid + 1;
        }
        int cu = lo;
        if (cu > 0 && fabs(density_model(c, (double)(cu - 1), s) - target) < fabs(density_model(c, (double)cu, s) - target))
            cu -= 1;
        if (c_out) c_out[i] = cu;
        /* cu spread evenly over the Kb bias channels (each <= QX_MAX since cu <= Kb * QX_MAX), so the bias
         * term sum_k X[m,k] W_g[n,k] is ~ -cu * beta_n for every neuron */
        for (int64_t k = 0; k < Kb; ++k) {
            int q = (int)(cu / Kb) + (k < cu % Kb ? 1 : 0);
            put(out, out_f32, i * K + k, q, c->x_exp);
        }
    }
    return 0;
}

/* Weight rows [row0, row0+nrows) of which = 0 (W_g), 1 (W_u), 2 (W_d); all stored [N, K] row-major. */
int synth_w(const synth_cfg* c, int which, int64_t row0, int64_t nrows, int out_f32, void* out) {
    const int64_t K = c->K, Kb = c->Kb;
    const uint64_t key = key_of(c->seed, which == 0 ? S_WG : which == 1 ? S_WU : S_WD);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nrows; ++i) {
        const int64_t n = row0 + i;
        int32_t b = 0, dead = 0;
        if (which == 0) synth_neuron(c, n, &b, &dead);
        for (int64_t k = 0; k < K; ++k) {
            int q;
            if (which == 0 && k < Kb)
                q = -bias_w(b, k);
            else if (which == 0 && dead)
                q = 0;
            else
                q = qw(rnd(key, (uint64_t)(n * K + k)));
            put(out, out_f32, i * K + k, q, c->w_exp);
        }
    }
    return 0;
}

/* "Direct TwELL" mode: an activation pattern with values, WITHOUT a gate GEMM, for isolating the
 * fused up/down and for unpack tests.  Rows [row0, row0+nrows) of a dense bf16 [nrows, N] matrix H (zeros off the
 * pattern; the caller packs it with the oracle).  Unit n of token m is active with probability
 * min(1, p[m] * w_n), w_n = the neuron's lognormal popularity exp(sigma z_n - sigma^2/2) / (1 - dead_frac) (dead
 * neurons: 0), sigma = pop_sigma; active values are positive grid values q * 2^-4, q in 1..15. */
int synth_pattern(const synth_cfg* c, const double* p, int64_t row0, int64_t nrows, double pop_sigma,
                  uint16_t* out) {
    const int64_t N = c->N;
    const uint64_t kn = key_of(c->seed, S_NEU), kp = key_of(c->seed, S_PAT), kv = key_of(c->seed, S_PATV);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nrows; ++i) {
        const int64_t m = row0 + i;
        for (int64_t n = 0; n < N; ++n) {
            uint64_t r = rnd(kn, (uint64_t)n);
            double u1 = ((double)(r & 0xFFFFFF) + 0.5) / 16777216.0;
            double u2 = ((double)((r >> 24) & 0xFFFFFF) + 0.5) / 16777216.0;
            double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
            int dead = ((double)((r >> 48) & 0xFFFF) / 65536.0) < c->dead_frac;
            double w = dead ? 0.0 : exp(pop_sigma * z - 0.5 * pop_sigma * pop_sigma) / (1.0 - c->dead_frac);
            double q = p[m] * w;
            uint64_t ra = rnd(kp, (uint64_t)(m * N + n));
            double u = ((double)(ra >> 11) + 0.5) / 9007199254740992.0;
            int qv = 1 + (int)(rnd(kv, (uint64_t)(m * N + n)) % 15);
            out[i * N + n] = u < q ? q_to_bf16(qv, 4) : (uint16_t)0;
        }
    }
    return 0;
}
