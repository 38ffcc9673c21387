/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's NASG
 * guiding hot path (/root/reference/proj, C++20 + Eigen).  See nasg_oracle.h
 * for the pinning status.  Every function cites the reference file:line it
 * restates; arithmetic is done in the same precision (double for densities,
 * decode and KL gradient; float for the MLP and Adam) and in the same
 * operation order, so results are bit-identical to oracle/_ref wherever the
 * same libm calls are made.  Compiled with -ffp-contract=off.
 */
#define _GNU_SOURCE
#include "nasg_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define K_PI 3.14159265358979323846
#define K_TWO_PI (2.0 * K_PI)
#define LAMBDA_MIN 1e-3 /* sphdist.hpp:13 */
#define LAMBDA_MAX 3e3  /* sphdist.hpp:14 */
#define ECC_MAX 3e3     /* sphdist.hpp:15 */
#define SEL_MIN 0.01    /* guiding.hpp:22 */
#define SEL_MAX 0.99    /* guiding.hpp:23 */
#define DENSITY_FLOOR 1e-300 /* guiding.cpp:11 */
#define ONE_BLOB_BINS 19     /* encoding.hpp:11 */

static double clampd(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }
static double dot3(const double *a, const double *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

/* ---------------- L0: hashing and PCG32 (math.hpp:74-121) ---------------- */
uint64_t orc_hash_mix(uint64_t x) { /* math.hpp:74-79 splitmix64 finalizer */
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

uint64_t orc_hash_combine(uint64_t a, uint64_t b) { /* math.hpp:81-83 */
    return orc_hash_mix(a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2)));
}

typedef struct { uint64_t state, inc; } pcg_t;

static uint32_t pcg_next(pcg_t *g) { /* math.hpp:102-108 */
    uint64_t old = g->state;
    g->state = old * 6364136223846793005ull + g->inc;
    uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
    uint32_t rot = (uint32_t)(old >> 59u);
    return (xs >> rot) | (xs << ((~rot + 1u) & 31));
}

static void pcg_seed(pcg_t *g, uint64_t initstate, uint64_t initseq) { /* math.hpp:94-100 */
    g->state = 0u;
    g->inc = (initseq << 1u) | 1u;
    pcg_next(g);
    g->state += initstate;
    pcg_next(g);
}

static double pcg_double(pcg_t *g) { return pcg_next(g) * 0x1p-32; } /* math.hpp:111 */

static uint32_t pcg_below(pcg_t *g, uint32_t n) { /* math.hpp:114-116 */
    return (uint32_t)(((uint64_t)pcg_next(g) * n) >> 32);
}

void orc_pcg32(uint64_t initstate, uint64_t initseq, int n, uint32_t *out) {
    pcg_t g;
    pcg_seed(&g, initstate, initseq);
    for (int i = 0; i < n; ++i) out[i] = pcg_next(&g);
}

/* ---------------- network layout helpers ---------------- */
static void layer_dims(int out_dim, int dims[5]) {
    dims[0] = ORC_IN; dims[1] = dims[2] = dims[3] = ORC_HIDDEN; dims[4] = out_dim;
}
static size_t weight_count(int out_dim) {
    return (size_t)ORC_IN * ORC_HIDDEN + 2u * ORC_HIDDEN * ORC_HIDDEN + (size_t)ORC_HIDDEN * out_dim;
}
static size_t layer_offset(int out_dim, int l) {
    int d[5];
    layer_dims(out_dim, d);
    size_t off = 0;
    for (int i = 0; i < l; ++i) off += (size_t)d[i] * d[i + 1];
    return off;
}

/* init_network<float> net.hpp:43-57: Pcg32(hash_mix(seed), 0xda3e39cb94b95bdb),
 * row-major fill with (u*2-1)*sqrt(6/fan_in). */
void orc_init_network(uint64_t seed, int out_dim, float *w) { orc_init_network_hu(seed, ORC_HIDDEN, out_dim, w); }

/* The same fill with kHiddenUnits = hidden (the paper's Table 4 sweep; the
 * reference fixes 128): the canonical hidden-H layout, W1[64][H] .. W4[H][D]. */
void orc_init_network_hu(uint64_t seed, int hidden, int out_dim, float *w) {
    int d[5] = {ORC_IN, hidden, hidden, hidden, out_dim};
    pcg_t g;
    pcg_seed(&g, orc_hash_mix(seed), 0xda3e39cb94b95bdbull);
    for (int l = 0; l < 4; ++l) {
        double limit = sqrt(6.0 / d[l]);
        for (int r = 0; r < d[l]; ++r)
            for (int c = 0; c < d[l + 1]; ++c) *w++ = (float)((pcg_double(&g) * 2.0 - 1.0) * limit);
    }
}

/* ---------------- encoder (encoding.cpp:11-46) ---------------- */
void orc_one_blob(double x, int k, float *out) { /* encoding.cpp:11-19 */
    double sigma = 1.0 / k;
    double inv_two_sigma2 = 1.0 / (2.0 * sigma * sigma);
    for (int i = 0; i < k; ++i) {
        double center = (i + 0.5) / k;
        double dd = x - center;
        out[i] = (float)exp(-dd * dd * inv_two_sigma2);
    }
}

/* encode_inputs encoding.cpp:21-46; returns the number of clamped coordinates
 * (the reference's relaxed global counter, encoding.cpp:8,31-34). */
static int encode_one(const float *q9, const double *mn, const double *ext, float *enc) {
    int clamped = 0;
    for (int axis = 0; axis < 3; ++axis) {
        double t = ext[axis] > 0.0 ? ((double)q9[axis] - mn[axis]) / ext[axis] : 0.5;
        if (t < 0.0 || t > 1.0) {
            ++clamped;
            t = clampd(t, 0.0, 1.0);
        }
        orc_one_blob(t, ONE_BLOB_BINS, enc + axis * ONE_BLOB_BINS);
    }
    for (int k = 0; k < 6; ++k) enc[57 + k] = q9[3 + k];
    enc[63] = 1.0f;
    return clamped;
}

static void bounds_of(const float *bmin, const float *bmax, double mn[3], double ext[3]) {
    for (int a = 0; a < 3; ++a) {
        mn[a] = bmin[a];
        ext[a] = (double)bmax[a] - (double)bmin[a]; /* Aabb::extent math.hpp:70 */
    }
}

uint64_t orc_encode(int64_t n, const float *q9, const float *bmin, const float *bmax,
                    float *out64) {
    double mn[3], ext[3];
    bounds_of(bmin, bmax, mn, ext);
    uint64_t cnt = 0;
    for (int64_t i = 0; i < n; ++i) cnt += (uint64_t)encode_one(q9 + 9 * i, mn, ext, out64 + 64 * i);
    return cnt;
}

/* ---------------- tiny MLP (net.hpp:69-158) ---------------- */
/* Y[n x N] = X[n x K] * W[K x N] with float accumulation in ascending k, the
 * same order as the shim's (and Eigen's scalar) product. */
static void gemm_f(const float *x, const float *w, int64_t n, int K, int N, float *y, int relu) {
    for (int64_t i = 0; i < n; ++i) {
        float *yr = y + i * N;
        for (int j = 0; j < N; ++j) yr[j] = 0.0f;
        for (int k = 0; k < K; ++k) {
            float a = x[i * K + k];
            const float *wr = w + (size_t)k * N;
            for (int j = 0; j < N; ++j) yr[j] += a * wr[j];
        }
        if (relu)
            for (int j = 0; j < N; ++j) yr[j] = yr[j] < 0.0f ? 0.0f : yr[j]; /* cwiseMax net.hpp:74: std::max, NaN propagates */
    }
}

typedef struct {
    int64_t n;
    float *h[4]; /* h[0] = input batch, h[l] = relu output of hidden layer l */
    float *out;
} fcache_t;

static void fcache_free(fcache_t *c) {
    for (int l = 0; l < 4; ++l) free(c->h[l]);
    free(c->out);
    memset(c, 0, sizeof(*c));
}

/* forward net.hpp:69-76 */
static void forward_cached(const float *w, int out_dim, int64_t n, const float *in64, fcache_t *c) {
    int d[5];
    layer_dims(out_dim, d);
    c->n = n;
    c->h[0] = (float *)malloc(sizeof(float) * (size_t)n * d[0]);
    memcpy(c->h[0], in64, sizeof(float) * (size_t)n * d[0]);
    for (int l = 0; l < 3; ++l) {
        c->h[l + 1] = (float *)malloc(sizeof(float) * (size_t)n * d[l + 1]);
        gemm_f(c->h[l], w + layer_offset(out_dim, l), n, d[l], d[l + 1], c->h[l + 1], 1);
    }
    c->out = (float *)malloc(sizeof(float) * (size_t)n * out_dim);
    gemm_f(c->h[3], w + layer_offset(out_dim, 3), n, d[3], d[4], c->out, 0);
}

void orc_forward(const float *w, int out_dim, int64_t n, const float *in64, float *out) {
    fcache_t c = {0};
    forward_cached(w, out_dim, n, in64, &c);
    memcpy(out, c.out, sizeof(float) * (size_t)n * out_dim);
    fcache_free(&c);
}

/* Test knob: sum the dW reduction over batch rows in reverse order.  This is
 * "the reference under another valid summation order" and measures how far
 * the training trajectory moves from fp32 reassociation alone — the yardstick
 * for the GPU's tracking tolerance (tests/test_gpu_train.py). */
static int g_reverse_sum = 0;
void orc_set_reverse_sum(int on) { g_reverse_sum = on; }

/* backward net.hpp:95-110: dW_l = h_l^T delta; delta <- (delta W_l^T) .* [h_l > 0] */
static void backward_cached(const float *w, int out_dim, const fcache_t *c, const float *og,
                            float *dw) {
    int d[5];
    layer_dims(out_dim, d);
    int64_t n = c->n;
    float *delta = (float *)malloc(sizeof(float) * (size_t)n * out_dim);
    memcpy(delta, og, sizeof(float) * (size_t)n * out_dim);
    for (int l = 3; l >= 0; --l) {
        int K = d[l], N = d[l + 1];
        float *g = dw + layer_offset(out_dim, l);
        const float *h = c->h[l];
        for (int i = 0; i < K; ++i) {
            float *gr = g + (size_t)i * N;
            for (int j = 0; j < N; ++j) gr[j] = 0.0f;
            for (int64_t bb = 0; bb < n; ++bb) {
                const int64_t b = g_reverse_sum ? n - 1 - bb : bb;
                float a = h[b * K + i];
                const float *dr = delta + b * N;
                for (int j = 0; j < N; ++j) gr[j] += a * dr[j];
            }
        }
        if (l > 0) {
            const float *wl = w + layer_offset(out_dim, l);
            float *nd = (float *)malloc(sizeof(float) * (size_t)n * K);
            for (int64_t b = 0; b < n; ++b)
                for (int i = 0; i < K; ++i) {
                    float s = 0.0f;
                    for (int j = 0; j < N; ++j) s += delta[b * N + j] * wl[(size_t)i * N + j];
                    nd[b * K + i] = s * (h[b * K + i] > 0.0f ? 1.0f : 0.0f);
                }
            free(delta);
            delta = nd;
        }
    }
    free(delta);
}

void orc_backward(const float *w, int out_dim, int64_t n, const float *in64, const float *og,
                  float *dw) {
    fcache_t c = {0};
    forward_cached(w, out_dim, n, in64, &c);
    backward_cached(w, out_dim, &c, og, dw);
    fcache_free(&c);
}

/* adam_step<float> net.hpp:137-158; AdamState defaults net.hpp:119-122 */
static int adam_apply(size_t np, float *w, float *m, float *v, const float *g, int64_t *t, float lr) {
    const float b1 = 0.9f, b2 = 0.999f, eps = 1e-8f;
    for (size_t i = 0; i < np; ++i)
        if (!isfinite(g[i])) return 0; /* skip the whole update, net.hpp:140-144 */
    ++*t;
    float corr1 = 1.0f - powf(b1, (float)*t);
    float corr2 = 1.0f - powf(b2, (float)*t);
    for (size_t i = 0; i < np; ++i) {
        m[i] = b1 * m[i] + (1.0f - b1) * g[i];
        v[i] = b2 * v[i] + (1.0f - b2) * (g[i] * g[i]);
        float mh = m[i] / corr1, vh = v[i] / corr2;
        w[i] -= lr * mh / (sqrtf(vh) + eps);
    }
    return 1;
}

int orc_adam_step(int out_dim, float *w, float *m, float *v, const float *g, int64_t *t, float lr) {
    return adam_apply(weight_count(out_dim), w, m, v, g, t, lr);
}

/* ---------------- NASG density (sphdist.cpp) ---------------- */
typedef struct {
    double x[3], y[3], z[3];
    double lambda, a, eps;
} lobe_t;

static int renorm_pair(double *s, double *c) { /* sphdist.cpp:15-25 */
    double n = sqrt(*s * *s + *c * *c);
    if (n < 1e-6) {
        *s = 0.0;
        *c = 1.0;
        return 0;
    }
    *s /= n;
    *c /= n;
    return 1;
}

static int frame_from_euler(double ct, double sp, double cp, double st, double ctau, lobe_t *o) {
    /* sphdist.cpp:87-101 (Eq. 13) */
    int ok = 1;
    ok &= renorm_pair(&sp, &cp);
    ok &= renorm_pair(&st, &ctau);
    double c = clampd(ct, -1.0, 1.0);
    double s = sqrt(fmax(0.0, 1.0 - c * c));
    o->z[0] = cp * s; o->z[1] = sp * s; o->z[2] = c;
    o->x[0] = c * cp * ctau - sp * st;
    o->x[1] = c * sp * ctau + cp * st;
    o->x[2] = -s * ctau;
    /* y = cross(z, x) math.hpp:38-40 */
    o->y[0] = o->z[1] * o->x[2] - o->z[2] * o->x[1];
    o->y[1] = o->z[2] * o->x[0] - o->z[0] * o->x[2];
    o->y[2] = o->z[0] * o->x[1] - o->z[1] * o->x[0];
    return ok;
}

int orc_frame_from_euler(double ct, double sp, double cp, double st, double ctau, double *xyz9) {
    lobe_t l;
    int ok = frame_from_euler(ct, sp, cp, st, ctau, &l);
    memcpy(xyz9, l.x, 3 * sizeof(double));
    memcpy(xyz9 + 3, l.y, 3 * sizeof(double));
    memcpy(xyz9 + 6, l.z, 3 * sizeof(double));
    return ok;
}

typedef struct { double dz, dx, u, log_u, t2, denom, beta, m, u_pow_m; } leval_t;

static leval_t eval_lobe(const lobe_t *c, const double *v) { /* sphdist.cpp:71-83 */
    leval_t e;
    e.dz = dot3(v, c->z);
    e.dx = dot3(v, c->x);
    e.u = clampd((e.dz + 1.0) * 0.5, 1e-12, 1.0);
    e.log_u = log(e.u);
    e.denom = fmax(1.0 - e.dz * e.dz, 1e-12);
    e.t2 = clampd(e.dx * e.dx / e.denom, 0.0, 1.0);
    e.beta = c->a * e.t2;
    e.m = 1.0 + c->eps + e.beta;
    e.u_pow_m = pow(e.u, e.m);
    return e;
}

static double log_eval(const lobe_t *c, const double *v) { /* sphdist.cpp:133-140 */
    double dz = dot3(v, c->z);
    if (dz >= 1.0 - 1e-12) return 0.0;
    if (dz <= -1.0 + 1e-12) return -INFINITY;
    leval_t e = eval_lobe(c, v);
    return 2.0 * c->lambda * (e.u_pow_m - 1.0) + (c->eps + e.beta) * e.log_u;
}

static double norm_const(const lobe_t *c) { /* sphdist.cpp:142-146 (Eq. 12) */
    double one_eps = 1.0 + c->eps;
    return K_TWO_PI * (-expm1(-2.0 * c->lambda)) / (c->lambda * sqrt(one_eps * (one_eps + c->a)));
}

double orc_norm_const(double lambda, double a, double eps) {
    lobe_t l;
    memset(&l, 0, sizeof l);
    l.lambda = lambda; l.a = a; l.eps = eps;
    return norm_const(&l);
}

static double lobe_pdf(const lobe_t *c, const double *v) { /* sphdist.cpp:148-150 */
    return exp(log_eval(c, v)) / norm_const(c);
}

typedef struct {
    int n;
    lobe_t lobe[ORC_MAX_LOBES];
    double w[ORC_MAX_LOBES];
    double c, c_sig;
    double sig[5 * ORC_MAX_LOBES];
    double pair_norm[2 * ORC_MAX_LOBES];
    int lam_clamped[ORC_MAX_LOBES], a_clamped[ORC_MAX_LOBES];
} decoded_t;

static double mixture_pdf(const decoded_t *d, const double *v) { /* sphdist.cpp:152-157 */
    double pdf = 0.0;
    for (int i = 0; i < d->n; ++i) pdf += d->w[i] * lobe_pdf(&d->lobe[i], v);
    return pdf;
}

static void lobe_from_c12(const double *c12, lobe_t *l) {
    memcpy(l->x, c12, 3 * sizeof(double));
    memcpy(l->y, c12 + 3, 3 * sizeof(double));
    memcpy(l->z, c12 + 6, 3 * sizeof(double));
    l->lambda = c12[9]; l->a = c12[10]; l->eps = c12[11];
}

double orc_nasg_log_eval(const double *c12, const double *v) {
    lobe_t l;
    lobe_from_c12(c12, &l);
    return log_eval(&l, v);
}

/* nasg_sample sphdist.cpp:159-181 (Appendix C maps Phi_E / Phi_W) */
static void lobe_sample(const lobe_t *c, double xi0, double xi1, double xi2, double *v) {
    double emin = exp(-2.0 * c->lambda);
    double s = emin + xi0 * (1.0 - emin);
    double rho = (xi1 - 0.5) * K_PI;
    double one_eps = 1.0 + c->eps;
    double cos_rho = cos(rho);
    double expo = (one_eps + c->a - c->a * cos_rho * cos_rho) / (one_eps * (one_eps + c->a));
    double base = clampd(log(s) / (2.0 * c->lambda) + 1.0, 0.0, 1.0);
    double cos_t = clampd(2.0 * pow(base, expo) - 1.0, -1.0, 1.0);
    double sin_t = sqrt(1.0 - cos_t * cos_t);
    double stretch = sqrt((one_eps + c->a) / one_eps);
    double phi = atan2(stretch * sin(rho), cos_rho);
    if (xi2 <= 0.5) phi += K_PI; /* western chart */
    double cp = cos(phi), sp = sin(phi);
    for (int k = 0; k < 3; ++k) v[k] = c->x[k] * (sin_t * cp) + c->y[k] * (sin_t * sp) + c->z[k] * cos_t;
}

void orc_nasg_sample(const double *c12, double xi0, double xi1, double xi2, double *out) {
    lobe_t l;
    lobe_from_c12(c12, &l);
    lobe_sample(&l, xi0, xi1, xi2, out);
}

/* mixture_sample sphdist.cpp:183-198: first i with xi_sel < cumulative A_i */
static double mixture_sample(const decoded_t *d, const float *xi, double *dir) {
    int pick = d->n - 1;
    double acc = 0.0;
    for (int i = 0; i < d->n; ++i) {
        acc += d->w[i];
        if ((double)xi[0] < acc) {
            pick = i;
            break;
        }
    }
    lobe_sample(&d->lobe[pick], xi[1], xi[2], xi[3], dir);
    return mixture_pdf(d, dir);
}

/* ---------------- guider: decode (guiding.cpp:15-77) ---------------- */
static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); } /* guiding.cpp:9 */

static void decode_full(const float *raw, int n, decoded_t *d) {
    d->n = n;
    for (int i = 0; i < n; ++i) {
        double trig[5];
        for (int k = 0; k < 5; ++k) {
            double s = sigmoid(raw[5 * i + k]);
            d->sig[5 * i + k] = s;
            trig[k] = s * 2.0 - 1.0;
        }
        for (int p = 0; p < 2; ++p) { /* guiding.cpp:35-48 */
            double *s = &trig[1 + 2 * p], *c = &trig[2 + 2 * p];
            double norm = sqrt(*s * *s + *c * *c);
            if (norm < 1e-6) {
                *s = 0.0; *c = 1.0;
                d->pair_norm[2 * i + p] = 0.0;
            } else {
                *s /= norm; *c /= norm;
                d->pair_norm[2 * i + p] = norm;
            }
        }
        lobe_t *comp = &d->lobe[i];
        frame_from_euler(trig[0], trig[1], trig[2], trig[3], trig[4], comp);
        double lambda = exp((double)raw[5 * n + 2 * i]);
        double a = exp((double)raw[5 * n + 2 * i + 1]);
        comp->lambda = clampd(lambda, LAMBDA_MIN, LAMBDA_MAX);
        comp->a = fmin(a, ECC_MAX); /* std::min(a, 3e3); a is never NaN here unless raw is */
        if (a != a) comp->a = a;
        comp->eps = 0.0;
        d->lam_clamped[i] = comp->lambda != lambda;
        d->a_clamped[i] = comp->a != a;
    }
    double mx = -INFINITY; /* guiding.cpp:62-72 */
    for (int i = 0; i < n; ++i) mx = fmax(mx, (double)raw[7 * n + i]);
    double sum = 0.0;
    for (int i = 0; i < n; ++i) {
        double w = exp((double)raw[7 * n + i] - mx);
        d->w[i] = w;
        sum += w;
    }
    for (int i = 0; i < n; ++i) d->w[i] /= sum;
    d->c_sig = sigmoid(raw[8 * n]);
    d->c = clampd(d->c_sig, SEL_MIN, SEL_MAX);
}

void orc_decode(int64_t nq, int n_comp, const float *raw, double *out) {
    const int D = 8 * n_comp + 1;
    decoded_t d;
    for (int64_t q = 0; q < nq; ++q) {
        decode_full(raw + q * D, n_comp, &d);
        double *o = out + q * (13 * n_comp + 1);
        for (int i = 0; i < n_comp; ++i) {
            const lobe_t *l = &d.lobe[i];
            double *p = o + 13 * i;
            memcpy(p, l->z, 3 * sizeof(double));
            memcpy(p + 3, l->x, 3 * sizeof(double));
            memcpy(p + 6, l->y, 3 * sizeof(double));
            p[9] = l->lambda; p[10] = l->a; p[11] = d.w[i];
            p[12] = log(norm_const(l));
        }
        o[13 * n_comp] = d.c;
    }
}

void orc_decode_sample(int64_t nq, int n_comp, const float *raw, const float *xi, double *out4,
                       double *c_out, int nthreads) {
    const int D = 8 * n_comp + 1;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t q = 0; q < nq; ++q) {
        decoded_t d;
        decode_full(raw + q * D, n_comp, &d);
        double dir[3];
        double pdf = mixture_sample(&d, xi + 4 * q, dir);
        out4[4 * q] = dir[0]; out4[4 * q + 1] = dir[1]; out4[4 * q + 2] = dir[2];
        out4[4 * q + 3] = pdf;
        if (c_out) c_out[q] = d.c;
    }
}

/* guided_pdf guiding.cpp:81-85 */
static double guided_pdf(const decoded_t *d, double b, double bsdf, const double *v) {
    double c_eff = b * d->c;
    if (c_eff <= 0.0) return bsdf;
    return c_eff * mixture_pdf(d, v) + (1.0 - c_eff) * bsdf;
}

void orc_decode_pdf(int64_t nq, int n_comp, const float *raw, const float *dir3, double b,
                    const float *bsdf_pdf, double *mix_out, double *guided_out) {
    const int D = 8 * n_comp + 1;
    decoded_t d;
    for (int64_t q = 0; q < nq; ++q) {
        decode_full(raw + q * D, n_comp, &d);
        double v[3] = {dir3[3 * q], dir3[3 * q + 1], dir3[3 * q + 2]};
        if (mix_out) mix_out[q] = mixture_pdf(&d, v);
        if (guided_out) guided_out[q] = guided_pdf(&d, b, bsdf_pdf ? bsdf_pdf[q] : 0.0, v);
    }
}

/* infer_guide guiding.cpp:284-293 followed by mixture_sample */
void orc_query_sample(const float *w, int out_dim, int64_t nq, const float *q9, const float *xi,
                      const float *bmin, const float *bmax, float *out4, float *c_out, int nthreads) {
    double mn[3], ext[3];
    bounds_of(bmin, bmax, mn, ext);
    const int n_comp = (out_dim - 1) / 8;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t q = 0; q < nq; ++q) {
        float enc[64];
        float raw[8 * ORC_MAX_LOBES + 1];
        float h1[ORC_HIDDEN], h2[ORC_HIDDEN], h3[ORC_HIDDEN];
        encode_one(q9 + 9 * q, mn, ext, enc);
        gemm_f(enc, w + layer_offset(out_dim, 0), 1, ORC_IN, ORC_HIDDEN, h1, 1);
        gemm_f(h1, w + layer_offset(out_dim, 1), 1, ORC_HIDDEN, ORC_HIDDEN, h2, 1);
        gemm_f(h2, w + layer_offset(out_dim, 2), 1, ORC_HIDDEN, ORC_HIDDEN, h3, 1);
        gemm_f(h3, w + layer_offset(out_dim, 3), 1, ORC_HIDDEN, out_dim, raw, 0);
        decoded_t d;
        decode_full(raw, n_comp, &d);
        double dir[3];
        double pdf = mixture_sample(&d, xi + 4 * q, dir);
        out4[4 * q] = (float)dir[0]; out4[4 * q + 1] = (float)dir[1]; out4[4 * q + 2] = (float)dir[2];
        out4[4 * q + 3] = (float)pdf;
        if (c_out) c_out[q] = (float)d.c;
    }
}

/* ---------------- KL gradient (guiding.cpp:96-176, sphdist.cpp:200-274) ---------------- */
typedef struct { double ct, sp, cp, st, ctau; } euler_t;

static euler_t euler_from_frame(const lobe_t *f) { /* sphdist.cpp:33-57 */
    euler_t e;
    e.ct = clampd(f->z[2], -1.0, 1.0);
    double s = sqrt(fmax(0.0, 1.0 - e.ct * e.ct));
    if (s > 1e-9) {
        e.cp = f->z[0] / s;
        e.sp = f->z[1] / s;
        renorm_pair(&e.sp, &e.cp);
        e.ctau = -f->x[2] / s;
        e.st = f->x[1] * e.cp - f->x[0] * e.sp;
        renorm_pair(&e.st, &e.ctau);
    } else { /* gimbal pole: phi folded into tau */
        e.sp = 0.0;
        e.cp = 1.0;
        if (e.ct > 0.0) {
            e.ctau = f->x[0];
            e.st = f->x[1];
        } else {
            e.ctau = -f->x[0];
            e.st = f->x[1];
        }
        renorm_pair(&e.st, &e.ctau);
    }
    return e;
}

typedef struct { double d_ct, d_sp, d_cp, d_st, d_ctau, d_lambda, d_a; } pgrad_t;

/* nasg_grad_logpdf sphdist.cpp:200-274; q = mixture_pdf(m, v) is passed in
 * (the reference recomputes the identical value per component). */
static pgrad_t grad_logpdf(const decoded_t *m, int idx, const double *v, double q) {
    pgrad_t g;
    memset(&g, 0, sizeof g);
    const lobe_t *c = &m->lobe[idx];
    double dz = dot3(v, c->z);
    if (fabs(dz) > 1.0 - 1e-6) return g; /* pole guard sphdist.cpp:205 */
    if (!(q > 0.0) || !isfinite(q)) return g;
    leval_t e = eval_lobe(c, v);
    double log_g = 2.0 * c->lambda * (e.u_pow_m - 1.0) + (c->eps + e.beta) * e.log_u;
    double K = norm_const(c);
    double r = m->w[idx] * exp(log_g) / K / q;
    double expm2l = exp(-2.0 * c->lambda);
    double dlogK_dl = 2.0 * expm2l / (1.0 - expm2l) - 1.0 / c->lambda;
    double dlogK_da = -0.5 / (1.0 + c->eps + c->a);
    double dG_dbeta = (2.0 * c->lambda * e.u_pow_m + 1.0) * e.log_u;
    double dG_du = 2.0 * c->lambda * e.m * pow(e.u, e.m - 1.0) + (c->eps + e.beta) / e.u;
    double dt2_ddz = 2.0 * e.dz * e.t2 / e.denom;
    double dG_ddz = 0.5 * dG_du + dG_dbeta * c->a * dt2_ddz;
    double dG_ddx = dG_dbeta * c->a * 2.0 * e.dx / e.denom;
    g.d_lambda = r * (2.0 * (e.u_pow_m - 1.0) - dlogK_dl);
    g.d_a = r * (e.t2 * dG_dbeta - dlogK_da);

    euler_t t = euler_from_frame(c);
    double ct = t.ct;
    double st = sqrt(fmax(1e-18, 1.0 - ct * ct));
    double dst_dct = -ct / st;
    double dz_dct[3] = {t.cp * dst_dct, t.sp * dst_dct, 1.0};
    double dz_dsp[3] = {0.0, st, 0.0};
    double dz_dcp[3] = {st, 0.0, 0.0};
    double dx_dct[3] = {t.cp * t.ctau, t.sp * t.ctau, -dst_dct * t.ctau};
    double dx_dsp[3] = {-t.st, ct * t.ctau, 0.0};
    double dx_dcp[3] = {ct * t.ctau, t.st, 0.0};
    double dx_dst[3] = {-t.sp, t.cp, 0.0};
    double dx_dctau[3] = {ct * t.cp, ct * t.sp, -st};
    double g_ct = dG_ddz * dot3(v, dz_dct) + dG_ddx * dot3(v, dx_dct);
    double g_sp = dG_ddz * dot3(v, dz_dsp) + dG_ddx * dot3(v, dx_dsp);
    double g_cp = dG_ddz * dot3(v, dz_dcp) + dG_ddx * dot3(v, dx_dcp);
    double g_st = dG_ddx * dot3(v, dx_dst);
    double g_ctau = dG_ddx * dot3(v, dx_dctau);
    /* (I - p p^T) projection of pair gradients, sphdist.cpp:254-261 */
    double ps = t.cp * (t.cp * g_sp - t.sp * g_cp), pc = t.sp * (t.sp * g_cp - t.cp * g_sp);
    g_sp = ps; g_cp = pc;
    ps = t.ctau * (t.ctau * g_st - t.st * g_ctau); pc = t.st * (t.st * g_ctau - t.ctau * g_st);
    g_st = ps; g_ctau = pc;
    g.d_ct = r * g_ct; g.d_sp = r * g_sp; g.d_cp = r * g_cp;
    g.d_st = r * g_st; g.d_ctau = r * g_ctau;
    double all[7] = {g.d_ct, g.d_sp, g.d_cp, g.d_st, g.d_ctau, g.d_lambda, g.d_a};
    for (int k = 0; k < 7; ++k)
        if (!isfinite(all[k])) {
            memset(&g, 0, sizeof g);
            return g;
        }
    return g;
}

typedef struct { double pos[3], wo[3], nrm[3], wi[3], p, q, pbsdf; } tsample_t;

static tsample_t sample_from(const float *s) {
    tsample_t t;
    for (int k = 0; k < 3; ++k) {
        t.pos[k] = s[k]; t.wo[k] = s[4 + k]; t.nrm[k] = s[8 + k]; t.wi[k] = s[12 + k];
    }
    t.p = s[3]; t.q = s[7]; t.pbsdf = s[11];
    return t;
}

typedef struct { double q_mix, q_hat, c_eff; int usable; } blend_t;

static blend_t eval_blend(const tsample_t *s, const decoded_t *d, double b) { /* guiding.cpp:96-104 */
    blend_t e;
    e.q_mix = mixture_pdf(d, s->wi);
    e.c_eff = b * d->c;
    e.q_hat = e.c_eff * e.q_mix + (1.0 - e.c_eff) * s->pbsdf;
    e.usable = isfinite(e.q_mix) && e.q_mix > DENSITY_FLOOR && isfinite(e.q_hat) && e.q_hat > DENSITY_FLOOR;
    return e;
}

/* kl_loss_gradient guiding.cpp:108-165 */
static int kl_gradient(const tsample_t *s, const decoded_t *d, double b, double e, double *grad) {
    const int n = d->n, D = 8 * n + 1;
    for (int k = 0; k < D; ++k) grad[k] = 0.0;
    if (s->p == 0.0) return 1;
    blend_t bl = eval_blend(s, d, b);
    if (!bl.usable || !(s->q > 0.0)) return 0;
    const double w = s->p / s->q;
    const double mix_scale = e * (bl.c_eff * bl.q_mix / bl.q_hat) + (1.0 - e);
    for (int i = 0; i < n; ++i) {
        pgrad_t pg = grad_logpdf(d, i, s->wi, bl.q_mix);
        const double scale = -w * mix_scale;
        double dt[5] = {pg.d_ct, pg.d_sp, pg.d_cp, pg.d_st, pg.d_ctau};
        for (int p = 0; p < 2; ++p) {
            double norm = d->pair_norm[2 * i + p];
            double inv = norm > 0.0 ? 1.0 / norm : 0.0;
            dt[1 + 2 * p] *= inv;
            dt[2 + 2 * p] *= inv;
        }
        for (int k = 0; k < 5; ++k) {
            double sg = d->sig[5 * i + k];
            grad[5 * i + k] = scale * dt[k] * 2.0 * sg * (1.0 - sg);
        }
        grad[5 * n + 2 * i] = d->lam_clamped[i] ? 0.0 : scale * pg.d_lambda * d->lobe[i].lambda;
        grad[5 * n + 2 * i + 1] = d->a_clamped[i] ? 0.0 : scale * pg.d_a * d->lobe[i].a;
        double pdf_i = lobe_pdf(&d->lobe[i], s->wi);
        double r_i = d->w[i] * pdf_i / bl.q_mix;
        grad[7 * n + i] = scale * (r_i - d->w[i]);
    }
    double c_clamped = d->c != d->c_sig ? 0.0 : 1.0;
    double dsig_c = d->c_sig * (1.0 - d->c_sig) * c_clamped;
    grad[8 * n] = -w * e * b * (bl.q_mix - s->pbsdf) / bl.q_hat * dsig_c;
    for (int k = 0; k < D; ++k)
        if (!isfinite(grad[k])) {
            for (int j = 0; j < D; ++j) grad[j] = 0.0;
            return 0;
        }
    return 1;
}

static double loss_surrogate(const tsample_t *s, const decoded_t *d, double b, double e) {
    /* guiding.cpp:167-176 */
    if (s->p == 0.0) return 0.0;
    blend_t bl = eval_blend(s, d, b);
    if (!bl.usable || !(s->q > 0.0)) return NAN;
    double w = s->p / s->q;
    return -w * (e * log(bl.q_hat) + (1.0 - e) * log(bl.q_mix));
}

void orc_kl_grad(int64_t n, int n_comp, const float *raw, const float *samples, double b,
                 double loss_blend, double *grad_out, int *ok_out, double *loss_out) {
    const int D = 8 * n_comp + 1;
    decoded_t d;
    for (int64_t i = 0; i < n; ++i) {
        decode_full(raw + i * D, n_comp, &d);
        tsample_t s = sample_from(samples + 16 * i);
        ok_out[i] = kl_gradient(&s, &d, b, loss_blend, grad_out + i * D);
        loss_out[i] = loss_surrogate(&s, &d, b, loss_blend);
    }
}


/* ---------------- explicit mixtures and the vMF / SG baseline ----------------
 * sphdist.cpp:152-198 (NASG mixture pdf / sample), :200-274 (grad log pdf),
 * :276-340 (vMF).  Records as nasg.h: NASG 12 floats (x_axis, lambda,
 * y_axis, a, z_axis, epsilon), vMF 4 floats (mu, lambda); weights k floats. */
static void nasg_records(int k, const float *comp, const float *w, decoded_t *d) {
    d->n = k;
    for (int i = 0; i < k; ++i) {
        const float *r = comp + 12 * i;
        lobe_t *l = &d->lobe[i];
        for (int j = 0; j < 3; ++j) {
            l->x[j] = r[j];
            l->y[j] = r[4 + j];
            l->z[j] = r[8 + j];
        }
        l->lambda = r[3]; l->a = r[7]; l->eps = r[11];
        d->w[i] = w[i];
    }
}

typedef struct { double mu[3], lambda; } vmf_t;

static double vmf_log_eval(const vmf_t *c, const double *v) { return c->lambda * (dot3(c->mu, v) - 1.0); } /* :276-278 */
static double vmf_norm_const(const vmf_t *c) { return K_TWO_PI * (-expm1(-2.0 * c->lambda)) / c->lambda; } /* :280-282 */
static double vmf_pdf(const vmf_t *c, const double *v) { return exp(vmf_log_eval(c, v)) / vmf_norm_const(c); }
static double vmf_mixture_pdf(int k, const vmf_t *c, const double *w, const double *v) { /* :288-293 */
    double pdf = 0.0;
    for (int i = 0; i < k; ++i) pdf += w[i] * vmf_pdf(&c[i], v);
    return pdf;
}
static void normalize3(double *v) { /* math.hpp:43 */
    double l = sqrt(dot3(v, v));
    v[0] /= l; v[1] /= l; v[2] /= l;
}
static void cross3(const double *a, const double *b, double *o) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}
static void vmf_sample(const vmf_t *c, double xi0, double xi1, double *v) { /* :295-305 */
    double cos_t = clampd(1.0 + log1p(-xi0 * (-expm1(-2.0 * c->lambda))) / c->lambda, -1.0, 1.0);
    double sin_t = sqrt(1.0 - cos_t * cos_t);
    double phi = K_TWO_PI * xi1;
    double z[3] = {c->mu[0], c->mu[1], c->mu[2]}, x[3], y[3]; /* frame_around :103-110 */
    normalize3(z);
    double helper[3] = {1.0, 0.0, 0.0};
    if (!(fabs(z[0]) < 0.9)) { helper[0] = 0.0; helper[1] = 1.0; }
    cross3(helper, z, x);
    normalize3(x);
    cross3(z, x, y);
    for (int j = 0; j < 3; ++j) v[j] = x[j] * (sin_t * cos(phi)) + y[j] * (sin_t * sin(phi)) + z[j] * cos_t;
}
static void vmf_grad(const vmf_t *c, double wi, const double *v, double q, double *g4) { /* :324-340 */
    g4[0] = g4[1] = g4[2] = g4[3] = 0.0;
    if (!(q > 0.0) || !isfinite(q)) return;
    double r = wi * vmf_pdf(c, v) / q;
    double expm2l = exp(-2.0 * c->lambda);
    double dlogK = 2.0 * expm2l / (1.0 - expm2l) - 1.0 / c->lambda;
    g4[3] = r * ((dot3(c->mu, v) - 1.0) - dlogK);
    double gm[3] = {v[0] * c->lambda, v[1] * c->lambda, v[2] * c->lambda};
    double p = dot3(gm, c->mu);
    for (int j = 0; j < 3; ++j) g4[j] = (gm[j] - c->mu[j] * p) * r;
}
static void vmf_records(int k, const float *comp, const float *w, vmf_t *c, double *wd) {
    for (int i = 0; i < k; ++i) {
        for (int j = 0; j < 3; ++j) c[i].mu[j] = comp[4 * i + j];
        c[i].lambda = comp[4 * i + 3];
        wd[i] = w[i];
    }
}

void orc_dist_pdf(int kind, int64_t n, int k, const float *comp, const float *w, const float *dir4, double *out) {
    for (int64_t q = 0; q < n; ++q) {
        double v[3] = {dir4[4 * q], dir4[4 * q + 1], dir4[4 * q + 2]};
        if (kind == 0) {
            decoded_t d;
            nasg_records(k, comp + 12 * k * q, w + k * q, &d);
            out[q] = mixture_pdf(&d, v);
        } else {
            vmf_t c[ORC_MAX_LOBES];
            double wd[ORC_MAX_LOBES];
            vmf_records(k, comp + 4 * k * q, w + k * q, c, wd);
            out[q] = vmf_mixture_pdf(k, c, wd, v);
        }
    }
}

void orc_dist_sample(int kind, int64_t n, int k, const float *comp, const float *w, const float *xi4, double *out4) {
    for (int64_t q = 0; q < n; ++q) {
        const float *x = xi4 + 4 * q;
        double v[3];
        if (kind == 0) {
            decoded_t d;
            nasg_records(k, comp + 12 * k * q, w + k * q, &d);
            out4[4 * q + 3] = mixture_sample(&d, x, v);
        } else {
            vmf_t c[ORC_MAX_LOBES];
            double wd[ORC_MAX_LOBES];
            vmf_records(k, comp + 4 * k * q, w + k * q, c, wd);
            int pick = k - 1; /* vmf_mixture_sample :307-322 */
            double acc = 0.0;
            for (int i = 0; i < k; ++i) {
                acc += wd[i];
                if ((double)x[0] < acc) { pick = i; break; }
            }
            vmf_sample(&c[pick], x[1], x[2], v);
            out4[4 * q + 3] = vmf_mixture_pdf(k, c, wd, v);
        }
        for (int j = 0; j < 3; ++j) out4[4 * q + j] = v[j];
    }
}

void orc_dist_grad(int kind, int64_t n, int k, const float *comp, const float *w, const float *dir4, double *out) {
    for (int64_t q = 0; q < n; ++q) {
        double v[3] = {dir4[4 * q], dir4[4 * q + 1], dir4[4 * q + 2]};
        if (kind == 0) {
            decoded_t d;
            nasg_records(k, comp + 12 * k * q, w + k * q, &d);
            double qm = mixture_pdf(&d, v);
            for (int i = 0; i < k; ++i) {
                pgrad_t g = grad_logpdf(&d, i, v, qm);
                double *o = out + 8 * (k * q + i);
                o[0] = g.d_ct; o[1] = g.d_sp; o[2] = g.d_cp; o[3] = g.d_st; o[4] = g.d_ctau;
                o[5] = g.d_lambda; o[6] = g.d_a; o[7] = 0.0;
            }
        } else {
            vmf_t c[ORC_MAX_LOBES];
            double wd[ORC_MAX_LOBES];
            vmf_records(k, comp + 4 * k * q, w + k * q, c, wd);
            double qm = vmf_mixture_pdf(k, c, wd, v);
            for (int i = 0; i < k; ++i) vmf_grad(&c[i], wd[i], v, qm, out + 4 * (k * q + i));
        }
    }
}

/* The fit's vMF model (k_sphdist.cu header): raw = [k mean directions xyz,
 * k log-sharpness, k weight logits]; per-sample gradient of -w log q_mix with
 * w = p / q_s = 1 (samples drawn from the target, q_s = p), chained through
 * vmf_grad_logpdf.  p == 0 -> zero gradient, ok; unusable or non-finite ->
 * zero gradient, not ok (the kl_loss_gradient conventions, guiding.cpp:108-165). */
void orc_vmf_fit_grad(int k, const float *raw, int64_t n, const float *samples4, double *grad_out, int *ok_out) {
    vmf_t c[ORC_MAX_LOBES];
    double wd[ORC_MAX_LOBES], nr[ORC_MAX_LOBES], mx = -INFINITY, sum = 0.0;
    int clamped[ORC_MAX_LOBES];
    for (int i = 0; i < k; ++i) {
        double r[3] = {raw[3 * i], raw[3 * i + 1], raw[3 * i + 2]};
        nr[i] = sqrt(dot3(r, r));
        int deg = nr[i] < 1e-6;
        for (int j = 0; j < 3; ++j) c[i].mu[j] = deg ? (j == 2 ? 1.0 : 0.0) : r[j] / nr[i];
        if (deg) nr[i] = 0.0;
        double lam = exp((double)raw[3 * k + i]);
        c[i].lambda = clampd(lam, 1e-3, 3e3);
        clamped[i] = c[i].lambda != lam;
    }
    for (int i = 0; i < k; ++i) mx = fmax(mx, (double)raw[4 * k + i]);
    for (int i = 0; i < k; ++i) sum += (wd[i] = exp((double)raw[4 * k + i] - mx));
    for (int i = 0; i < k; ++i) wd[i] /= sum;
    const int D = 5 * k;
    for (int64_t s = 0; s < n; ++s) {
        double *g = grad_out + D * s;
        memset(g, 0, D * sizeof(double));
        ok_out[s] = 1;
        const float *sm = samples4 + 4 * s;
        if (sm[3] == 0.0f) continue;
        double v[3] = {sm[0], sm[1], sm[2]};
        double q = vmf_mixture_pdf(k, c, wd, v);
        if (!(isfinite(q) && q > DENSITY_FLOOR)) { ok_out[s] = 0; continue; }
        int fin = 1;
        for (int i = 0; i < k; ++i) {
            double g4[4];
            vmf_grad(&c[i], wd[i], v, q, g4);
            double inv = nr[i] > 0.0 ? 1.0 / nr[i] : 0.0;
            for (int j = 0; j < 3; ++j) g[3 * i + j] = -g4[j] * inv;
            g[3 * k + i] = clamped[i] ? 0.0 : -g4[3] * c[i].lambda;
            g[4 * k + i] = -(wd[i] * vmf_pdf(&c[i], v) / q - wd[i]);
        }
        for (int j = 0; j < D; ++j) fin &= isfinite(g[j]) != 0;
        if (!fin) { memset(g, 0, D * sizeof(double)); ok_out[s] = 0; }
    }
}

/* ---------------- schedules (guiding.hpp:78-92, guiding.cpp:178-182) ---------------- */
double orc_stride_update(double l, uint64_t s, uint64_t cap) {
    double next = l * sqrt((double)s / (double)cap);
    return next > 1.0 ? next : 1.0;
}

double orc_blend_coefficient(int64_t i, int m, int bsteps) {
    double b = (double)(i / m) / bsteps;
    return b < 1.0 ? b : 1.0;
}

/* ---------------- Trainer (guiding.cpp:184-282) ---------------- */
typedef struct {
    int n_comp, capacity, batch, step_factor;
    float lr;
    double loss_blend;
    uint64_t seed;
    float bmin[3], bmax[3];
    float *w, *m, *v;
    int64_t t;
    int64_t iterations;
} trainer_t;

void *orc_trainer_create(int n_comp, int capacity, int batch, int step_factor, float lr,
                         double loss_blend, uint64_t seed, const float *bmin, const float *bmax) {
    trainer_t *t = (trainer_t *)calloc(1, sizeof(trainer_t));
    t->n_comp = n_comp; t->capacity = capacity; t->batch = batch; t->step_factor = step_factor;
    t->lr = lr; t->loss_blend = loss_blend; t->seed = seed;
    memcpy(t->bmin, bmin, sizeof t->bmin);
    memcpy(t->bmax, bmax, sizeof t->bmax);
    int D = 8 * n_comp + 1;
    size_t np = weight_count(D);
    t->w = (float *)malloc(np * sizeof(float));
    t->m = (float *)calloc(np, sizeof(float));
    t->v = (float *)calloc(np, sizeof(float));
    orc_init_network(seed, D, t->w);
    return t;
}

void orc_trainer_destroy(void *p) {
    trainer_t *t = (trainer_t *)p;
    if (!t) return;
    free(t->w); free(t->m); free(t->v); free(t);
}

void orc_trainer_get_weights(void *p, float *w) {
    trainer_t *t = (trainer_t *)p;
    memcpy(w, t->w, weight_count(8 * t->n_comp + 1) * sizeof(float));
}

void orc_trainer_set_weights(void *p, const float *w) {
    trainer_t *t = (trainer_t *)p;
    memcpy(t->w, w, weight_count(8 * t->n_comp + 1) * sizeof(float));
}

void orc_trainer_train(void *p, int64_t n, const float *samples, double b, double *stats4) {
    trainer_t *t = (trainer_t *)p;
    stats4[0] = stats4[1] = stats4[2] = stats4[3] = 0.0;
    if (n == 0) { /* empty buffer: no-op + publish, guiding.cpp:198-202 */
        ++t->iterations;
        return;
    }
    const int D = 8 * t->n_comp + 1;
    const int tb = t->batch;
    const int steps = t->step_factor * ((t->capacity + tb - 1) / tb); /* config S, not n: :204-206 */
    double mn[3], ext[3];
    bounds_of(t->bmin, t->bmax, mn, ext);
    /* encode every sample once (guiding.cpp:209-214); remap the 16-float
     * sample layout to encode_one's (pos, omega_o, normal) triple. */
    float *enc = (float *)malloc(sizeof(float) * 64 * (size_t)n);
    for (int64_t s = 0; s < n; ++s) {
        float q9[9];
        const float *sm = samples + 16 * s;
        q9[0] = sm[0]; q9[1] = sm[1]; q9[2] = sm[2];
        q9[3] = sm[4]; q9[4] = sm[5]; q9[5] = sm[6];
        q9[6] = sm[8]; q9[7] = sm[9]; q9[8] = sm[10];
        encode_one(q9, mn, ext, enc + 64 * s);
    }
    pcg_t rng; /* guiding.cpp:216 */
    pcg_seed(&rng, orc_hash_combine(t->seed, 0x7261696e) + (uint64_t)t->iterations, 5);
    uint32_t *order = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) order[i] = (uint32_t)i;
#define RESHUFFLE()                                                   \
    for (int64_t i = n; i > 1; --i) {                                 \
        uint32_t j = pcg_below(&rng, (uint32_t)i);                    \
        uint32_t tmp = order[i - 1]; order[i - 1] = order[j]; order[j] = tmp; \
    }
    RESHUFFLE();
    int64_t cursor = 0;
    double loss_sum = 0.0;
    uint64_t loss_count = 0, dropped = 0, skipped = 0;
    size_t np = weight_count(D);
    float *dw = (float *)malloc(np * sizeof(float));
    for (int step = 0; step < steps; ++step) {
        if (cursor >= n) {
            RESHUFFLE();
            cursor = 0;
        }
        int64_t count = n - cursor < tb ? n - cursor : tb;
        float *batch = (float *)malloc(sizeof(float) * 64 * (size_t)count);
        for (int64_t r = 0; r < count; ++r) memcpy(batch + 64 * r, enc + 64 * (size_t)order[cursor + r], 64 * sizeof(float));
        fcache_t c = {0};
        forward_cached(t->w, D, count, batch, &c);
        float *og = (float *)calloc((size_t)count * D, sizeof(float));
        double grad[8 * ORC_MAX_LOBES + 1];
        decoded_t d;
        for (int64_t r = 0; r < count; ++r) {
            const float *raw = c.out + r * D;
            int finite = 1;
            for (int k = 0; k < D; ++k) finite &= isfinite(raw[k]) ? 1 : 0;
            if (!finite) { ++dropped; continue; }
            decode_full(raw, t->n_comp, &d);
            tsample_t s = sample_from(samples + 16 * (size_t)order[cursor + r]);
            if (!kl_gradient(&s, &d, b, t->loss_blend, grad)) { ++dropped; continue; }
            double inv = 1.0 / (double)count;
            for (int k = 0; k < D; ++k) og[r * D + k] = (float)(grad[k] * inv);
            double l = loss_surrogate(&s, &d, b, t->loss_blend);
            if (isfinite(l)) { loss_sum += l; ++loss_count; }
        }
        cursor += count;
        backward_cached(t->w, D, &c, og, dw);
        if (!adam_apply(np, t->w, t->m, t->v, dw, &t->t, t->lr)) ++skipped;
        fcache_free(&c);
        free(og);
        free(batch);
        stats4[0] += 1.0;
    }
#undef RESHUFFLE
    stats4[1] = loss_count > 0 ? loss_sum / (double)loss_count : 0.0;
    stats4[2] = (double)dropped;
    stats4[3] = (double)skipped;
    ++t->iterations;
    free(dw); free(order); free(enc);
}

/* ---------------- NASGNET1 checkpoint (net.cpp:31-82) ---------------- */
static void put_u32(FILE *f, uint32_t v) {
    unsigned char b[4] = {(unsigned char)v, (unsigned char)(v >> 8), (unsigned char)(v >> 16), (unsigned char)(v >> 24)};
    fwrite(b, 1, 4, f);
}
static uint32_t get_u32(FILE *f, int *ok) {
    unsigned char b[4];
    if (fread(b, 1, 4, f) != 4) *ok = 0;
    return (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
}

int orc_save_checkpoint(const char *path, const float *w, int out_dim, int n_comp) {
    FILE *f = fopen(path, "wb");
    if (!f) return -1;
    fwrite("NASGNET1", 1, 8, f);
    int d[5];
    layer_dims(out_dim, d);
    put_u32(f, (uint32_t)n_comp);
    put_u32(f, 5);
    for (int i = 0; i < 5; ++i) put_u32(f, (uint32_t)d[i]);
    size_t np = weight_count(out_dim);
    int ok = fwrite(w, sizeof(float), np, f) == np;
    ok &= fclose(f) == 0;
    return ok ? 0 : -1;
}

int orc_load_checkpoint(const char *path, float *w, int max_floats, int *n_comp) {
    FILE *f = fopen(path, "rb");
    if (!f) return -1;
    char magic[8];
    int ok = fread(magic, 1, 8, f) == 8 && memcmp(magic, "NASGNET1", 8) == 0;
    if (!ok) { fclose(f); return -1; }
    uint32_t n = get_u32(f, &ok), nd = get_u32(f, &ok);
    if (!ok || nd != 5) { fclose(f); return -1; }
    uint32_t d[5];
    for (int i = 0; i < 5; ++i) d[i] = get_u32(f, &ok);
    size_t total = 0;
    for (int l = 0; l < 4; ++l) total += (size_t)d[l] * d[l + 1];
    if ((int64_t)total > max_floats) { fclose(f); return -2; }
    ok &= fread(w, sizeof(float), total, f) == total;
    fclose(f);
    if (!ok) return -1;
    if (n_comp) *n_comp = (int)n;
    return (int)total;
}

/* ---------------- synthetic workloads ----------------
 * Byte-identical restatement of the product's nasg_synth_queries /
 * nasg_synth_samples, so the CPU arms of bench.py never load the CUDA library
 * (pinned by tests/test_abi.py::test_synth_generators_match). */
static float synth_f24(pcg_t *g) { return (float)(pcg_next(g) >> 8) * 0x1p-24f; }

static void synth_sphere(pcg_t *g, float *out) {
    const double z = 1.0 - 2.0 * synth_f24(g);
    const double phi = 2.0 * 3.14159265358979323846 * synth_f24(g);
    const double t = 1.0 - z * z;
    const double rr = sqrt(t > 0.0 ? t : 0.0);
    out[0] = (float)(rr * cos(phi));
    out[1] = (float)(rr * sin(phi));
    out[2] = (float)z;
    out[3] = 0.f;
}

void orc_synth_queries(uint64_t seed, int64_t first, int64_t n, const float *bmin, const float *bmax, float *x,
                       float *wo, float *nrm, float *xi) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        pcg_t g;
        pcg_seed(&g, orc_hash_combine(seed, (uint64_t)(first + i)), 0x51);
        for (int k = 0; k < 3; ++k) x[4 * i + k] = bmin[k] + (bmax[k] - bmin[k]) * synth_f24(&g);
        x[4 * i + 3] = 0.f;
        synth_sphere(&g, wo + 4 * i);
        synth_sphere(&g, nrm + 4 * i);
        for (int k = 0; k < 4; ++k) xi[4 * i + k] = synth_f24(&g);
    }
}

void orc_synth_samples(uint64_t seed, int64_t first, int64_t n, const float *bmin, const float *bmax, float *out16) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        pcg_t g;
        pcg_seed(&g, orc_hash_combine(seed, (uint64_t)(first + i)), 0x53);
        float *s = out16 + 16 * i;
        float wo[4], nn[4], wi[4];
        for (int k = 0; k < 3; ++k) s[k] = bmin[k] + (bmax[k] - bmin[k]) * synth_f24(&g);
        synth_sphere(&g, wo);
        synth_sphere(&g, nn);
        synth_sphere(&g, wi);
        for (int k = 0; k < 3; ++k) {
            s[4 + k] = wo[k];
            s[8 + k] = nn[k];
            s[12 + k] = wi[k];
        }
        const double dn = (double)wi[0] * nn[0] + (double)wi[1] * nn[1] + (double)wi[2] * nn[2];
        const double cosn = dn > 0.0 ? dn : 0.0;
        const double mu[3] = {sin(2.0 * s[0]) + 0.5, cos(3.0 * s[1]), 1.0 + 0.5 * sin((double)s[2])};
        const double inv = 1.0 / sqrt(mu[0] * mu[0] + mu[1] * mu[1] + mu[2] * mu[2]);
        const double d = (wi[0] * mu[0] + wi[1] * mu[1] + wi[2] * mu[2]) * inv;
        s[3] = (float)(exp(20.0 * (d - 1.0)) * cosn);
        s[7] = (float)(1.0 / (4.0 * 3.14159265358979323846));
        s[11] = (float)(cosn / 3.14159265358979323846);
        s[15] = 0.f;
    }
}
