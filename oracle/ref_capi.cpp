// TEST INFRASTRUCTURE ONLY — C-ABI harness around the UNMODIFIED reference.
//
// Linked (by oracle/Makefile) against /root/reference/proj/src/{sphdist,
// encoding,net,guiding}.cpp compiled with the Eigen-API shim, producing
// oracle/_ref/libnasg_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's reference/cpu_baseline legs may load it.  Every entry point
// calls the reference's own public functions (guiding.hpp, sphdist.hpp,
// encoding.hpp, net.hpp); this file adds only array marshalling and an
// optional OpenMP parallel-for over independent queries (the reference's
// query API is pure/reentrant, guiding.hpp:139-141).
//
// Array conventions (all little-endian, row-major):
//   query  : 9 floats  = position xyz, omega_o xyz, normal xyz
//   xi     : 4 floats  = xi_select, xi0, xi1, xi2
//   weights: W1(64x128) W2(128x128) W3(128x128) W4(128xD) concatenated
//   sample : 16 floats = pos xyz, p, omega_o xyz, q_sampling, normal xyz,
//            bsdf_pdf, omega_i xyz, pad
//   lobe   : 13 doubles = z xyz, x xyz, y xyz, lambda, a, weight, log K

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <cstring>
#include <span>
#include <vector>

#include "nasg/encoding.hpp"
#include "nasg/guiding.hpp"
#include "nasg/net.hpp"
#include "nasg/sphdist.hpp"

using namespace nasg;

namespace {

Vec3 v3(const float *p) { return {double(p[0]), double(p[1]), double(p[2])}; }

Aabb make_bounds(const float *bmin, const float *bmax) {
    Aabb b;
    b.min = v3(bmin);
    b.max = v3(bmax);
    return b;
}

NetworkParameters<float> params_from(const float *w, int out_dim) {
    NetworkParameters<float> p;
    int dims[5] = {kEncodedInputSize, kHiddenUnits, kHiddenUnits, kHiddenUnits, out_dim};
    for (int l = 0; l < kNumLayers; ++l) {
        p.w[l].resize(dims[l], dims[l + 1]);
        for (int r = 0; r < dims[l]; ++r)
            for (int c = 0; c < dims[l + 1]; ++c) p.w[l](r, c) = *w++;
    }
    return p;
}

void params_to(const NetworkParameters<float> &p, float *w) {
    for (int l = 0; l < kNumLayers; ++l)
        for (int r = 0; r < p.w[l].rows(); ++r)
            for (int c = 0; c < p.w[l].cols(); ++c) *w++ = p.w[l](r, c);
}

TrainingSample sample_from(const float *s) {
    TrainingSample t;
    t.position = v3(s + 0);
    t.p_value = s[3];
    t.omega_o = v3(s + 4);
    t.q_sampling = s[7];
    t.normal = v3(s + 8);
    t.bsdf_pdf_at_wi = s[11];
    t.omega_i = v3(s + 12);
    t.bsdf_is_delta = false;
    return t;
}

} // namespace

extern "C" {

int ref_version() { return 1; }

// ---- L0 / encoder -------------------------------------------------------
void ref_init_network(uint64_t seed, int out_dim, float *w_out) {
    params_to(init_network<float>(kEncodedInputSize, out_dim, seed), w_out);
}

void ref_pcg32(uint64_t initstate, uint64_t initseq, int n, uint32_t *out) {
    Pcg32 r(initstate, initseq);
    for (int i = 0; i < n; ++i) out[i] = r.next_u32();
}

uint64_t ref_hash_combine(uint64_t a, uint64_t b) { return hash_combine(a, b); }

void ref_one_blob(double x, int k, float *out) { one_blob(x, k, out); }

uint64_t ref_encode(int64_t n, const float *q9, const float *bmin, const float *bmax,
                    float *out64) {
    reset_encode_clamp_count();
    Aabb b = make_bounds(bmin, bmax);
    for (int64_t i = 0; i < n; ++i) {
        EncodedInput e = encode_inputs(v3(q9 + 9 * i), v3(q9 + 9 * i + 3), v3(q9 + 9 * i + 6), b);
        std::memcpy(out64 + 64 * i, e.data(), 64 * sizeof(float));
    }
    return encode_clamp_count();
}

// ---- tinynn --------------------------------------------------------------
void ref_forward(const float *w, int out_dim, int64_t n, const float *in64, float *out) {
    NetworkParameters<float> p = params_from(w, out_dim);
    Matrix<float> x(n, kEncodedInputSize);
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < kEncodedInputSize; ++k) x(i, k) = in64[64 * i + k];
    Matrix<float> y = forward(p, x);
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < out_dim; ++k) out[i * out_dim + k] = y(i, k);
}

void ref_backward(const float *w, int out_dim, int64_t n, const float *in64,
                  const float *out_grads, float *dw) {
    NetworkParameters<float> p = params_from(w, out_dim);
    Matrix<float> x(n, kEncodedInputSize);
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < kEncodedInputSize; ++k) x(i, k) = in64[64 * i + k];
    ForwardCache<float> cache;
    forward(p, x, &cache);
    Matrix<float> g(n, out_dim);
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < out_dim; ++k) g(i, k) = out_grads[i * out_dim + k];
    params_to(backward(p, cache, g), dw);
}

// One Adam step on flat arrays (w, m, v updated in place); returns 1 if applied.
int ref_adam_step(int out_dim, float *w, float *m, float *v, const float *g, int64_t *t,
                  float lr) {
    NetworkParameters<float> p = params_from(w, out_dim), gr = params_from(g, out_dim);
    AdamState<float> s = AdamState<float>::make(p, lr);
    s.m = params_from(m, out_dim).w;
    s.v = params_from(v, out_dim).w;
    s.t = *t;
    bool ok = adam_step(s, p, gr);
    params_to(p, w);
    NetworkParameters<float> tmp;
    tmp.w = s.m;
    params_to(tmp, m);
    tmp.w = s.v;
    params_to(tmp, v);
    *t = s.t;
    return ok ? 1 : 0;
}

// ---- sphdist -------------------------------------------------------------
double ref_norm_const(double lambda, double a, double eps) {
    NasgComponent c;
    c.lambda = lambda;
    c.a = a;
    c.epsilon = eps;
    return nasg_norm_const(c);
}

int ref_frame_from_euler(double ct, double sp, double cp, double st, double ctau,
                         double *xyz9) {
    Frame f;
    bool ok = frame_from_euler(ct, sp, cp, st, ctau, &f);
    const Vec3 *ax[3] = {&f.x_axis, &f.y_axis, &f.z_axis};
    for (int i = 0; i < 3; ++i) {
        xyz9[3 * i] = ax[i]->x;
        xyz9[3 * i + 1] = ax[i]->y;
        xyz9[3 * i + 2] = ax[i]->z;
    }
    return ok ? 1 : 0;
}

// Component given as frame (x,y,z axes, 9 doubles) + lambda, a, eps.
static NasgComponent comp_from(const double *c12) {
    NasgComponent c;
    c.frame.x_axis = {c12[0], c12[1], c12[2]};
    c.frame.y_axis = {c12[3], c12[4], c12[5]};
    c.frame.z_axis = {c12[6], c12[7], c12[8]};
    c.lambda = c12[9];
    c.a = c12[10];
    c.epsilon = c12[11];
    return c;
}

double ref_nasg_log_eval(const double *c12, const double *v) {
    return nasg_log_eval(comp_from(c12), {v[0], v[1], v[2]});
}

void ref_nasg_sample(const double *c12, double xi0, double xi1, double xi2, double *out) {
    Vec3 d = nasg_sample(comp_from(c12), xi0, xi1, xi2);
    out[0] = d.x;
    out[1] = d.y;
    out[2] = d.z;
}

// ---- guider: decode / sample / pdf on raw network outputs -----------------
static void write_lobes(const DecodedGuide &d, double *out) {
    for (int i = 0; i < d.n; ++i) {
        const NasgComponent &c = d.g.mixture.components[i];
        double *o = out + 13 * i;
        o[0] = c.frame.z_axis.x; o[1] = c.frame.z_axis.y; o[2] = c.frame.z_axis.z;
        o[3] = c.frame.x_axis.x; o[4] = c.frame.x_axis.y; o[5] = c.frame.x_axis.z;
        o[6] = c.frame.y_axis.x; o[7] = c.frame.y_axis.y; o[8] = c.frame.y_axis.z;
        o[9] = c.lambda; o[10] = c.a; o[11] = d.g.mixture.weights[i];
        o[12] = std::log(nasg_norm_const(c));
    }
    out[13 * d.n] = d.g.c;
}

// out: per query 13*N + 1 doubles
void ref_decode(int64_t nq, int n_comp, const float *raw, double *out) {
    const int D = 8 * n_comp + 1;
    for (int64_t i = 0; i < nq; ++i) {
        DecodedGuide d = decode_full(std::span<const float>(raw + i * D, D));
        write_lobes(d, out + i * (13 * n_comp + 1));
    }
}

// mixture_sample on decoded raw outputs: out4 = dir xyz, pdf; c_out = c.
void ref_decode_sample(int64_t nq, int n_comp, const float *raw, const float *xi,
                       double *out4, double *c_out, int nthreads) {
    const int D = 8 * n_comp + 1;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t i = 0; i < nq; ++i) {
        GuideDistribution g = decode(std::span<const float>(raw + i * D, D));
        const float *x = xi + 4 * i;
        DirectionSample s = mixture_sample(g.mixture, x[0], x[1], x[2], x[3]);
        out4[4 * i] = s.direction.x;
        out4[4 * i + 1] = s.direction.y;
        out4[4 * i + 2] = s.direction.z;
        out4[4 * i + 3] = s.pdf;
        if (c_out) c_out[i] = g.c;
    }
}

// mixture_pdf and guided_pdf at given directions.
void ref_decode_pdf(int64_t nq, int n_comp, const float *raw, const float *dir3, double b,
                    const float *bsdf_pdf, double *mix_out, double *guided_out) {
    const int D = 8 * n_comp + 1;
    for (int64_t i = 0; i < nq; ++i) {
        GuideDistribution g = decode(std::span<const float>(raw + i * D, D));
        Vec3 v = v3(dir3 + 3 * i);
        if (mix_out) mix_out[i] = mixture_pdf(g.mixture, v);
        if (guided_out) guided_out[i] = guided_pdf(g, b, bsdf_pdf ? bsdf_pdf[i] : 0.0, v);
    }
}

// The reference's own per-point query path, as a renderer calls it:
// infer_guide (encode + forward + decode) then mixture_sample.
void ref_query_sample(const float *w, int out_dim, int64_t nq, const float *q9,
                      const float *xi, const float *bmin, const float *bmax, float *out4,
                      float *c_out, int nthreads) {
    NetworkParameters<float> p = params_from(w, out_dim);
    Aabb b = make_bounds(bmin, bmax);
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t i = 0; i < nq; ++i) {
        const float *q = q9 + 9 * i;
        GuideDistribution g = infer_guide(p, v3(q), v3(q + 3), v3(q + 6), b);
        const float *x = xi + 4 * i;
        DirectionSample s = mixture_sample(g.mixture, x[0], x[1], x[2], x[3]);
        out4[4 * i] = float(s.direction.x);
        out4[4 * i + 1] = float(s.direction.y);
        out4[4 * i + 2] = float(s.direction.z);
        out4[4 * i + 3] = float(s.pdf);
        if (c_out) c_out[i] = float(g.c);
    }
}

// Per-sample KL gradient wrt raw outputs (65 doubles), ok flag and loss.
void ref_kl_grad(int64_t n, int n_comp, const float *raw, const float *samples, double b,
                 double loss_blend, double *grad_out, int *ok_out, double *loss_out) {
    const int D = 8 * n_comp + 1;
    Eigen::VectorXd g;
    for (int64_t i = 0; i < n; ++i) {
        DecodedGuide d = decode_full(std::span<const float>(raw + i * D, D));
        TrainingSample s = sample_from(samples + 16 * i);
        bool ok = kl_loss_gradient(s, d, b, loss_blend, &g);
        for (int k = 0; k < D; ++k) grad_out[i * D + k] = g[k];
        ok_out[i] = ok ? 1 : 0;
        loss_out[i] = loss_surrogate(s, d, b, loss_blend);
    }
}


// ---- explicit mixtures and the vMF / SG baseline (sphdist.hpp:33-121) --------
// Records as include/nasg/nasg.h: NASG 12 floats (x_axis, lambda, y_axis, a,
// z_axis, epsilon), vMF 4 floats (mu, lambda); weights k floats per query.
static NasgMixture nasg_mixture_of(int k, const float *comp, const float *w) {
    NasgMixture m;
    for (int i = 0; i < k; ++i) {
        const float *r = comp + 12 * i;
        NasgComponent c;
        c.frame.x_axis = v3(r);
        c.frame.y_axis = v3(r + 4);
        c.frame.z_axis = v3(r + 8);
        c.lambda = r[3];
        c.a = r[7];
        c.epsilon = r[11];
        m.components.push_back(c);
        m.weights.push_back(w[i]);
    }
    return m;
}
static VmfMixture vmf_mixture_of(int k, const float *comp, const float *w) {
    VmfMixture m;
    for (int i = 0; i < k; ++i) {
        VmfComponent c;
        c.mu = v3(comp + 4 * i);
        c.lambda = comp[4 * i + 3];
        m.components.push_back(c);
        m.weights.push_back(w[i]);
    }
    return m;
}

void ref_dist_pdf(int kind, int64_t n, int k, const float *comp, const float *w, const float *dir4, double *out) {
    for (int64_t q = 0; q < n; ++q) {
        Vec3 v = v3(dir4 + 4 * q);
        out[q] = kind == 0 ? mixture_pdf(nasg_mixture_of(k, comp + 12 * k * q, w + k * q), v)
                           : vmf_mixture_pdf(vmf_mixture_of(k, comp + 4 * k * q, w + k * q), v);
    }
}

void ref_dist_sample(int kind, int64_t n, int k, const float *comp, const float *w, const float *xi4, double *out4) {
    for (int64_t q = 0; q < n; ++q) {
        const float *x = xi4 + 4 * q;
        DirectionSample s = kind == 0 ? mixture_sample(nasg_mixture_of(k, comp + 12 * k * q, w + k * q), x[0], x[1], x[2], x[3])
                                      : vmf_mixture_sample(vmf_mixture_of(k, comp + 4 * k * q, w + k * q), x[0], x[1], x[2]);
        out4[4 * q] = s.direction.x;
        out4[4 * q + 1] = s.direction.y;
        out4[4 * q + 2] = s.direction.z;
        out4[4 * q + 3] = s.pdf;
    }
}

void ref_dist_grad(int kind, int64_t n, int k, const float *comp, const float *w, const float *dir4, double *out) {
    for (int64_t q = 0; q < n; ++q) {
        Vec3 v = v3(dir4 + 4 * q);
        if (kind == 0) {
            NasgMixture m = nasg_mixture_of(k, comp + 12 * k * q, w + k * q);
            for (int i = 0; i < k; ++i) {
                ParamGradient g = nasg_grad_logpdf(m, i, v);
                double *o = out + 8 * (k * q + i);
                o[0] = g.d_cos_theta; o[1] = g.d_sin_phi; o[2] = g.d_cos_phi; o[3] = g.d_sin_tau;
                o[4] = g.d_cos_tau; o[5] = g.d_lambda; o[6] = g.d_a; o[7] = 0.0;
            }
        } else {
            VmfMixture m = vmf_mixture_of(k, comp + 4 * k * q, w + k * q);
            for (int i = 0; i < k; ++i) {
                VmfParamGradient g = vmf_grad_logpdf(m, i, v);
                double *o = out + 4 * (k * q + i);
                o[0] = g.d_mu.x; o[1] = g.d_mu.y; o[2] = g.d_mu.z; o[3] = g.d_lambda;
            }
        }
    }
}

// The fit's vMF model (see nasg_oracle.c orc_vmf_fit_grad): the chain rule is
// this harness's, every density / gradient value is the reference's.
void ref_vmf_fit_grad(int k, const float *raw, int64_t n, const float *samples4, double *grad_out, int *ok_out) {
    VmfMixture m;
    std::vector<double> nr(k);
    std::vector<int> clamped(k);
    double mx = -std::numeric_limits<double>::infinity(), sum = 0.0;
    for (int i = 0; i < k; ++i) {
        Vec3 r{raw[3 * i], raw[3 * i + 1], raw[3 * i + 2]};
        nr[i] = length(r);
        VmfComponent c;
        if (nr[i] < 1e-6) {
            c.mu = Vec3{0.0, 0.0, 1.0};
            nr[i] = 0.0;
        } else {
            c.mu = r / nr[i];
        }
        double lam = std::exp((double)raw[3 * k + i]);
        c.lambda = std::clamp(lam, 1e-3, 3e3);
        clamped[i] = c.lambda != lam;
        m.components.push_back(c);
    }
    for (int i = 0; i < k; ++i) mx = std::max(mx, (double)raw[4 * k + i]);
    for (int i = 0; i < k; ++i) {
        m.weights.push_back(std::exp((double)raw[4 * k + i] - mx));
        sum += m.weights.back();
    }
    for (double &x : m.weights) x /= sum;
    const int D = 5 * k;
    for (int64_t s = 0; s < n; ++s) {
        double *g = grad_out + D * s;
        std::fill(g, g + D, 0.0);
        ok_out[s] = 1;
        const float *sm = samples4 + 4 * s;
        if (sm[3] == 0.0f) continue;
        Vec3 v = v3(sm);
        double q = vmf_mixture_pdf(m, v);
        if (!(std::isfinite(q) && q > 1e-300)) {
            ok_out[s] = 0;
            continue;
        }
        bool fin = true;
        for (int i = 0; i < k; ++i) {
            VmfParamGradient pg = vmf_grad_logpdf(m, i, v);
            double inv = nr[i] > 0.0 ? 1.0 / nr[i] : 0.0;
            g[3 * i] = -pg.d_mu.x * inv;
            g[3 * i + 1] = -pg.d_mu.y * inv;
            g[3 * i + 2] = -pg.d_mu.z * inv;
            g[3 * k + i] = clamped[i] ? 0.0 : -pg.d_lambda * m.components[i].lambda;
            g[4 * k + i] = -(m.weights[i] * vmf_pdf(m.components[i], v) / q - m.weights[i]);
        }
        for (int j = 0; j < D; ++j) fin = fin && std::isfinite(g[j]);
        if (!fin) {
            std::fill(g, g + D, 0.0);
            ok_out[s] = 0;
        }
    }
}

double ref_stride_update(double l, uint64_t s, uint64_t cap) { return stride_update(l, s, cap); }

double ref_blend_coefficient(int64_t i, int m, int bsteps) {
    BlendSchedule s;
    s.m = m;
    s.b_steps = bsteps;
    s.iteration = i;
    return s.coefficient();
}

// ---- Trainer ---------------------------------------------------------------
struct RefTrainer {
    Trainer t;
};

void *ref_trainer_create(int n_comp, int capacity, int batch, int step_factor, float lr,
                         double loss_blend, uint64_t seed, const float *bmin,
                         const float *bmax) {
    TrainerConfig c;
    c.n_components = n_comp;
    c.sample_capacity = capacity;
    c.batch_size = batch;
    c.step_factor = step_factor;
    c.learning_rate = lr;
    c.loss_blend = loss_blend;
    c.seed = seed;
    return new RefTrainer{Trainer(c, make_bounds(bmin, bmax))};
}

void ref_trainer_destroy(void *t) { delete static_cast<RefTrainer *>(t); }

// stats4: steps, mean_loss, dropped, skipped
void ref_trainer_train(void *t, int64_t n, const float *samples, double b, double *stats4) {
    std::vector<TrainingSample> buf(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) buf[i] = sample_from(samples + 16 * i);
    TrainStats s = static_cast<RefTrainer *>(t)->t.train_iteration(buf, b);
    stats4[0] = s.steps;
    stats4[1] = s.mean_loss;
    stats4[2] = double(s.dropped_samples);
    stats4[3] = double(s.skipped_updates);
}

void ref_trainer_get_weights(void *t, float *w) {
    params_to(static_cast<RefTrainer *>(t)->t.parameters(), w);
}

void ref_trainer_get_snapshot(void *t, float *w) {
    params_to(*static_cast<RefTrainer *>(t)->t.snapshot(), w);
}

void ref_trainer_set_weights(void *t, const float *w) {
    RefTrainer *r = static_cast<RefTrainer *>(t);
    r->t.mutable_parameters() = params_from(w, r->t.parameters().output_dim());
    r->t.publish();
}

// ---- checkpoint I/O ---------------------------------------------------------
int ref_save_checkpoint(const char *path, const float *w, int out_dim, int n_comp) {
    try {
        save_checkpoint(path, params_from(w, out_dim), n_comp);
        return 0;
    } catch (...) {
        return -1;
    }
}

int ref_load_checkpoint(const char *path, float *w, int max_floats, int *n_comp) {
    try {
        NetworkParameters<float> p = load_checkpoint(path, n_comp);
        int total = 0;
        for (int l = 0; l < kNumLayers; ++l) total += int(p.w[l].rows() * p.w[l].cols());
        if (total > max_floats) return -2;
        params_to(p, w);
        return total;
    } catch (...) {
        return -1;
    }
}

// ---- synthetic workloads ---------------------------------------------
// Byte-identical restatement of the product's nasg_synth_queries / nasg_synth_samples
// (paper_2303_08064_b200/csrc/nasg_api.cpp) on the reference's own Pcg32 and
// hash_combine (math.hpp:81-121), so the reference arm of bench.py builds its
// inputs without loading the CUDA library (tests/test_abi.py pins the equality).
static float synth_f24(Pcg32 &r) { return (float)(r.next_u32() >> 8) * 0x1p-24f; }

static void synth_sphere(Pcg32 &r, float *out) {
    const double z = 1.0 - 2.0 * synth_f24(r);
    const double phi = 2.0 * 3.14159265358979323846 * synth_f24(r);
    const double rr = std::sqrt(std::max(0.0, 1.0 - z * z));
    out[0] = (float)(rr * std::cos(phi));
    out[1] = (float)(rr * std::sin(phi));
    out[2] = (float)z;
    out[3] = 0.f;
}

void ref_synth_queries(uint64_t seed, int64_t first, int64_t n, const float *bmin, const float *bmax, float *x,
                       float *wo, float *nrm, float *xi) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        Pcg32 r(hash_combine(seed, (uint64_t)(first + i)), 0x51);
        for (int k = 0; k < 3; ++k) x[4 * i + k] = bmin[k] + (bmax[k] - bmin[k]) * synth_f24(r);
        x[4 * i + 3] = 0.f;
        synth_sphere(r, wo + 4 * i);
        synth_sphere(r, nrm + 4 * i);
        for (int k = 0; k < 4; ++k) xi[4 * i + k] = synth_f24(r);
    }
}

void ref_synth_samples(uint64_t seed, int64_t first, int64_t n, const float *bmin, const float *bmax, float *out16) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        Pcg32 r(hash_combine(seed, (uint64_t)(first + i)), 0x53);
        float *s = out16 + 16 * i;
        float wo[4], nn[4], wi[4];
        for (int k = 0; k < 3; ++k) s[k] = bmin[k] + (bmax[k] - bmin[k]) * synth_f24(r);
        synth_sphere(r, wo);
        synth_sphere(r, nn);
        synth_sphere(r, wi);
        for (int k = 0; k < 3; ++k) {
            s[4 + k] = wo[k];
            s[8 + k] = nn[k];
            s[12 + k] = wi[k];
        }
        const double cosn = std::max(0.0, (double)wi[0] * nn[0] + (double)wi[1] * nn[1] + (double)wi[2] * nn[2]);
        const double mu[3] = {std::sin(2.0 * s[0]) + 0.5, std::cos(3.0 * s[1]), 1.0 + 0.5 * std::sin((double)s[2])};
        const double inv = 1.0 / std::sqrt(mu[0] * mu[0] + mu[1] * mu[1] + mu[2] * mu[2]);
        const double d = (wi[0] * mu[0] + wi[1] * mu[1] + wi[2] * mu[2]) * inv;
        s[3] = (float)(std::exp(20.0 * (d - 1.0)) * cosn);
        s[7] = (float)(1.0 / (4.0 * 3.14159265358979323846));
        s[11] = (float)(cosn / 3.14159265358979323846);
        s[15] = 0.f;
    }
}

} // extern "C"
