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
};

using TrainStats = nasg_train_stats;        // TrainStats (guiding.hpp:132-137)
using TrainingSample = nasg_train_sample;   // TrainingSample (guiding.hpp:54-63), 64 B

enum class Precision { FP32 = NASG_MLP_FP32, BF16 = NASG_MLP_BF16 };

// One GPU's Trainer + published NetworkSnapshot (guiding.hpp:142-166).
class Guide {
public:
    Guide(const TrainerConfig &c, int device, const float bmin[3], const float bmax[3]) {
        nasg_config cfg{c.n_components, c.sample_capacity, c.batch_size, c.step_factor,
                        c.learning_rate, c.loss_blend, c.seed};
        check(nasg_create(&cfg, device, bmin, bmax, &ctx_));
        n_ = c.n_components;
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

    void set_precision(Precision p) { check(nasg_set_precision(ctx_, (int)p)); }
    std::vector<float> parameters(bool published = false) const {
        std::vector<float> w((size_t)nasg_n_weights(cfg_n()));
        check(nasg_get_weights(ctx_, w.data(), w.size(), published ? 1 : 0));
        return w;
    }
    void set_parameters(std::span<const float> w) { check(nasg_set_weights(ctx_, w.data(), w.size())); }
    void save_checkpoint(const std::string &p) { check(nasg_save_checkpoint(ctx_, p.c_str())); }
    void load_checkpoint(const std::string &p) { check(nasg_load_checkpoint(ctx_, p.c_str())); }

    nasg_ctx *handle() { return ctx_; }

private:
    int cfg_n() const { return n_; }
    nasg_ctx *ctx_ = nullptr;
    int n_ = 8;
};

}  // namespace nasg::gpu
