// nasg_gpu.hpp — header-only C++ layer over the C ABI (nasg.h) that re-exposes
// the reference's guiding nouns (guiding.hpp: TrainerConfig, TrainStats,
// Trainer::train_iteration / publish / snapshot; infer_guide + mixture_sample,
// guided_pdf), batched over device buffers.  Errors throw nasg::gpu::Error
// (the C ABI itself never throws).
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "nasg/nasg.h"

namespace nasg::gpu {

struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string &what) : std::runtime_error(what), status(s) {}
};

inline void check(int s) {
    if (s != NASG_OK) throw Error(s, std::string(nasg_status_string(s)) + ": " + nasg_last_error());
}

// TrainerConfig (guiding.hpp:122-130), same defaults.
struct TrainerConfig {
    int n_components = 8;
    int sample_capacity = 1 << 16;
    int batch_size = 1 << 12;
    int step_factor = 1;
    float learning_rate = 0.002f;
    double loss_blend = 0.2;
    std::uint64_t seed = 0;
    int hidden_units = 128;  // 64: the paper's smaller network (nasg.h)
};

using TrainStats = nasg_train_stats;        // TrainStats (guiding.hpp:132-137)
using TrainingSample = nasg_train_sample;   // TrainingSample (guiding.hpp:54-63), 64 B

enum class Precision { FP32 = NASG_MLP_FP32, BF16 = NASG_MLP_BF16 };

// One GPU's Trainer + published NetworkSnapshot (guiding.hpp:142-166).
class Guide {
public:
    Guide(const TrainerConfig &c, int device, const float bmin[3], const float bmax[3]) {
        nasg_config cfg{c.n_components, c.sample_capacity, c.batch_size, c.step_factor,
                        c.learning_rate, c.loss_blend, c.seed, c.hidden_units};
        check(nasg_create(&cfg, device, bmin, bmax, &ctx_));
        n_ = c.n_components;
        hu_ = c.hidden_units ? c.hidden_units : 128;
    }
    ~Guide() { nasg_destroy(ctx_); }
    Guide(const Guide &) = delete;
    Guide &operator=(const Guide &) = delete;

    // Trainer::train_iteration over device-resident samples; publishes.
    TrainStats train_iteration(std::span<const TrainingSample> device_samples, double blend_b,
                               void *stream = nullptr) {
        TrainStats st{};
        check(nasg_train_iteration(ctx_, (std::int64_t)device_samples.size(), device_samples.data(),
                                   blend_b, &st, stream));
        return st;
    }
    void publish() { check(nasg_publish(ctx_)); }

    // infer_guide + mixture_sample for n queries (device float4 SoA).
    void sample(std::int64_t n, const float *x, const float *wo, const float *nrm, const float *xi,
                float *dir_pdf, float *c = nullptr, void *stream = nullptr) {
        check(nasg_query_sample(ctx_, n, x, wo, nrm, xi, dir_pdf, c, stream));
    }
    // mixture_pdf / guided_pdf (guiding.hpp:51) at given directions.
    void pdf(std::int64_t n, const float *x, const float *wo, const float *nrm, const float *dir,
             float b, const float *bsdf_pdf, float *mix_pdf, float *guided_pdf, void *stream = nullptr) {
        check(nasg_query_pdf(ctx_, n, x, wo, nrm, dir, b, bsdf_pdf, mix_pdf, guided_pdf, stream));
    }

    // guided scattering at wavefront vertices (nasg.h nasg_query_shade)
    void shade(std::int64_t n, const int *n_dev, const float *x, const float *wo, const float *nrm, const float *xi,
               const float *d_bsdf, const float *d_nee, float b, float *out, void *stream = nullptr) {
        check(nasg_query_shade(ctx_, n, n_dev, x, wo, nrm, xi, d_bsdf, d_nee, b, out, stream));
    }

    void set_precision(Precision p) { check(nasg_set_precision(ctx_, (int)p)); }
    void set_train_precision(Precision p) { check(nasg_set_train_precision(ctx_, (int)p)); }
    // p = 0 rows counted without the network pass (nasg_set_zero_row_skip; default on)
    void set_zero_row_skip(bool on) { check(nasg_set_zero_row_skip(ctx_, on ? 1 : 0)); }
    std::vector<float> parameters(bool published = false) const {
        std::vector<float> w((size_t)nasg_n_weights_hu(cfg_n(), hu_));
        check(nasg_get_weights(ctx_, w.data(), w.size(), published ? 1 : 0));
        return w;
    }
    void set_parameters(std::span<const float> w) { check(nasg_set_weights(ctx_, w.data(), w.size())); }
    void save_checkpoint(const std::string &p, bool optimizer = false) {
        check(optimizer ? nasg_save_checkpoint_ex(ctx_, p.c_str(), NASG_CKPT_OPTIMIZER) : nasg_save_checkpoint(ctx_, p.c_str()));
    }
    void load_checkpoint(const std::string &p) { check(nasg_load_checkpoint(ctx_, p.c_str())); }

    nasg_ctx *handle() { return ctx_; }

private:
    int cfg_n() const { return n_; }
    nasg_ctx *ctx_ = nullptr;
    int n_ = 8, hu_ = 128;
};

// ---- explicit mixtures (sphdist.hpp:33-121): NASG records and the vMF / SG baseline
struct NasgRecord {  // NasgComponent (sphdist.hpp:33-38) as 3 x float4
    float x_axis[3], lambda, y_axis[3], a, z_axis[3], epsilon;
};
struct VmfRecord {  // VmfComponent (sphdist.hpp:49-52)
    float mu[3], lambda;
};
enum class Family { NASG = NASG_DIST_NASG, VMF = NASG_DIST_VMF };

// mixture_pdf / vmf_mixture_pdf over n per-query mixtures of k components (device buffers)
inline void mixture_pdf(Family f, std::int64_t n, int k, const void *comp, const float *w, const float *dir, float *pdf,
                        void *stream = nullptr) {
    check(nasg_dist_mixture_pdf((int)f, n, k, static_cast<const float *>(comp), w, dir, pdf, stream));
}
// mixture_sample / vmf_mixture_sample -> float4 (direction, mixture pdf)
inline void mixture_sample(Family f, std::int64_t n, int k, const void *comp, const float *w, const float *xi,
                           float *dir_pdf, void *stream = nullptr) {
    check(nasg_dist_mixture_sample((int)f, n, k, static_cast<const float *>(comp), w, xi, dir_pdf, stream));
}
// nasg_grad_logpdf (8 floats per component) / vmf_grad_logpdf (4 floats per component)
inline void grad_logpdf(Family f, std::int64_t n, int k, const void *comp, const float *w, const float *dir,
                        float *grad, void *stream = nullptr) {
    check(nasg_dist_grad_logpdf((int)f, n, k, static_cast<const float *>(comp), w, dir, grad, stream));
}

// SPEC run_fit: n_fits guide distributions of one family fitted to a target mixture
struct FitResult {
    std::vector<float> raw;  // n_fits x checkpoints x raw_dim
    std::vector<double> kl;  // n_fits x checkpoints
    int raw_dim = 0;
};
inline FitResult fit(const nasg_fit_config &cfg, int n_fits, Family target, int target_k, const void *target_comp,
                     const float *target_w, int quad_nz = 256) {
    FitResult r;
    r.raw_dim = nasg_fit_raw_dim(cfg.model, cfg.n_components);
    if (r.raw_dim < 0) throw Error(NASG_ERR_UNSUPPORTED, "unsupported fit model");
    r.raw.resize((size_t)n_fits * cfg.checkpoints * r.raw_dim);
    r.kl.resize((size_t)n_fits * cfg.checkpoints);
    check(nasg_fit(&cfg, n_fits, (int)target, target_k, static_cast<const float *>(target_comp), target_w, nullptr,
                   r.raw.data(), r.kl.data(), quad_nz));
    return r;
}

// The SPEC tracer loop on one GPU's pixel rows (nasg_render_*).
class Render {
public:
    Render(Guide &g, const nasg_render_config &cfg) { check(nasg_render_create(g.handle(), &cfg, &r_)); }
    ~Render() { nasg_render_destroy(r_); }
    Render(const Render &) = delete;
    Render &operator=(const Render &) = delete;
    nasg_render_stats iteration() {
        nasg_render_stats st{};
        check(nasg_render_iteration(r_, &st));
        return st;
    }
    std::vector<float> image(std::int64_t pixels, bool last_frame = false) {
        std::vector<float> rgb((size_t)pixels * 3);
        check(nasg_render_image(r_, rgb.data(), last_frame ? 1 : 0));
        return rgb;
    }

private:
    nasg_render *r_ = nullptr;
};

}  // namespace nasg::gpu
