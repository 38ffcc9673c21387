/* nasg.h — C ABI of the B200-native NASG path-guiding hot path.
 *
 * Drop-in for the reference's guiding API (/root/reference/proj/include/nasg),
 * batched and stream-ordered.  Every entry point cites the reference
 * interface it replaces.  Plain C types only: device buffers are passed as
 * raw pointers (cudaMalloc'd, 16-byte aligned), streams as `void *`
 * (a cudaStream_t, NULL = the context's stream).  No function throws; all
 * return an `int` nasg_status.  Host arrays are row-major, little-endian.
 *
 * Data layouts (device or host, per argument):
 *   query SoA    x, wo, nrm : n x float4 (xyz + ignored w)  — position,
 *                omega_o and shading normal of encode_inputs (encoding.hpp:26)
 *   xi           n x float4 = (xi_select, xi0, xi1, xi2) of mixture_sample
 *                (sphdist.hpp:97-98)
 *   dir_pdf      n x float4 = (direction xyz, mixture pdf)  — DirectionSample
 *                (sphdist.hpp:93-96)
 *   raw          n x (8N+1) float, reference raw-output order (guiding.hpp:25-30)
 *   train sample n x nasg_train_sample (64 B)  — TrainingSample (guiding.hpp:54-63)
 *   weights      W1(64x128) W2(128x128) W3(128x128) W4(128x(8N+1)) row-major,
 *                concatenated — NetworkParameters<float> (net.hpp:22-40)
 *
 * Threading (guiding.hpp:139-141): one context per GPU; the
 * training calls and nasg_publish are single-writer; query calls read the
 * published snapshot and may run concurrently on other streams.
 */
#ifndef NASG_H
#define NASG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    NASG_OK = 0,
    NASG_ERR_INVALID = 1,     /* bad argument / shape */
    NASG_ERR_CUDA = 2,        /* CUDA runtime error (or no sm_100a device) */
    NASG_ERR_NCCL = 3,        /* NCCL unavailable / failed */
    NASG_ERR_IO = 4,          /* checkpoint I/O (net.cpp:34-79 exceptions) */
    NASG_ERR_OOM = 5,
    NASG_ERR_UNSUPPORTED = 6  /* configuration not compiled in */
} nasg_status;

/* MLP arithmetic of the query path. */
typedef enum {
    NASG_MLP_FP32 = 0, /* fp32 FFMA, bit-for-tolerance with the fp32 reference */
    NASG_MLP_BF16 = 1  /* tcgen05/TMEM tensor cores, fp32 accumulate: queries and the
                          trainer's forward multiply f16 operands (same rate as bf16,
                          3 more mantissa bits; |activations| saturate at 65504), the
                          trainer's gradients flow in bf16 / row-scaled f16 (name kept
                          for ABI stability) */
} nasg_precision;

/* TrainerConfig (guiding.hpp:122-130); defaults via nasg_config_default. */
typedef struct {
    int n_components;     /* N = 8 */
    int sample_capacity;  /* S = 2^16 */
    int batch_size;       /* t = 2^12 */
    int step_factor;      /* nu = 1 */
    float learning_rate;  /* 0.002 */
    double loss_blend;    /* e = 0.2 */
    uint64_t seed;        /* 0 */
    int hidden_units;     /* 128 (kHiddenUnits, net.hpp); 64 is the paper's smaller
                             network (Table 4): it runs on the 128-wide kernels with
                             the extra units' weights held at exactly zero, which
                             computes the 64-unit network exactly (same cost as 128).
                             0 means 128. Weights, gradients and checkpoints are
                             exchanged in the 64-unit canonical layout. */
} nasg_config;

/* TrainStats (guiding.hpp:132-137). */
typedef struct {
    int steps;
    double mean_loss;
    uint64_t dropped_samples;
    uint64_t skipped_updates;
} nasg_train_stats;

/* TrainingSample (guiding.hpp:54-63) packed to 64 bytes. bsdf_is_delta
 * samples are never recorded (SPEC.md guider design decisions). */
typedef struct {
    float position[3];
    float p_value;        /* luminance target p */
    float omega_o[3];
    float q_sampling;     /* pdf the sample obeyed (> 0) */
    float normal[3];
    float bsdf_pdf_at_wi;
    float omega_i[3];
    float pad;
} nasg_train_sample;

typedef struct nasg_ctx nasg_ctx;

/* ---- lifetime (Trainer::Trainer guiding.cpp:184-190) ------------------- */
void nasg_config_default(nasg_config *cfg);
/* Initialises the live weights with init_network<float>(64, 8N+1, seed)
 * (net.hpp:43-57, bit-exact), zero Adam state, and publishes them. */
int nasg_create(const nasg_config *cfg, int device, const float bmin[3], const float bmax[3],
                nasg_ctx **out);
int nasg_destroy(nasg_ctx *ctx);
const char *nasg_status_string(int status);
const char *nasg_last_error(void);  /* thread-local detail of the last failure */
int nasg_n_weights(int n_components); /* 64*128 + 2*128*128 + 128*(8N+1) */
int nasg_n_weights_hu(int n_components, int hidden_units); /* 64*H + 2*H*H + H*(8N+1) */

/* ---- parameters / snapshots (Trainer::parameters/mutable_parameters/publish/
 * snapshot guiding.hpp:151-157; NetworkSnapshot net.hpp:161) -------------- */
int nasg_set_weights(nasg_ctx *ctx, const float *host_w, size_t n_floats); /* live, then publish */
int nasg_get_weights(nasg_ctx *ctx, float *host_w, size_t n_floats, int published);
int nasg_publish(nasg_ctx *ctx);  /* snapshot live -> published (stream-ordered) */
int nasg_set_precision(nasg_ctx *ctx, int precision); /* nasg_precision for queries */
int nasg_get_precision(nasg_ctx *ctx);
/* MLP arithmetic of training: NASG_MLP_FP32 (FFMA forward/backward, the
 * reference's float MLP; default) or NASG_MLP_BF16 (tcgen05 forward, backward
 * and dW GEMMs with bf16 operands, fp32 accumulation, fp32 master weights and
 * Adam).  The KL gradient is computed in double on both paths. */
int nasg_set_train_precision(nasg_ctx *ctx, int precision);
int nasg_get_train_precision(nasg_ctx *ctx);
/* Zero-gradient rows (p_value == 0: kl_loss_gradient returns a zero gradient,
 * guiding.cpp:112, and loss_surrogate 0, :170) skip the network pass of both
 * trainers: they are counted in TrainStats exactly as the reference counts
 * them, and the step's gradient is the same sum over the other rows.  Only
 * while every weight is below 1e7 in magnitude and the row's inputs are finite
 * (then its output is provably finite, so the reference would not drop it,
 * :247-250); otherwise the row takes the full path.  Applied to steps with
 * more tiles (128 rows tensor core, 64 fp32) than SMs (smaller steps are one
 * tile per SM either way).  Default on. */
int nasg_set_zero_row_skip(nasg_ctx *ctx, int on);
int nasg_get_zero_row_skip(nasg_ctx *ctx);
/* save_checkpoint / load_checkpoint (net.hpp:163-167, net.cpp:31-82): NASGNET1,
 * byte-identical with the reference's file.  nasg_save_checkpoint_ex with
 * NASG_CKPT_OPTIMIZER appends the Adam state (t, m, v) as a trailing chunk the
 * reference's loader skips; nasg_load_checkpoint restores it when present (the
 * reference persists weights only, so its resume restarts Adam). */
enum { NASG_CKPT_OPTIMIZER = 1 };
int nasg_save_checkpoint(nasg_ctx *ctx, const char *path);
int nasg_save_checkpoint_ex(nasg_ctx *ctx, const char *path, int flags);
int nasg_load_checkpoint(nasg_ctx *ctx, const char *path);

/* ---- queries (device buffers; read the published snapshot) -------------- */
/* infer_guide (guiding.hpp:169) + mixture_sample (sphdist.hpp:97): per query
 * encode -> MLP -> decode -> inverse-CDF lobe pick -> NASG sample -> mixture
 * pdf at the sample.  c (nullable) receives the clamped selection prob. */
int nasg_query_sample(nasg_ctx *ctx, int64_t n, const float *x, const float *wo,
                      const float *nrm, const float *xi, float *dir_pdf, float *c,
                      void *stream);
/* Same as nasg_query_sample with the packed row format: 13 floats per query
 * (position xyz, omega_o xyz, normal xyz, xi_select, xi0, xi1, xi2). */
int nasg_query_sample_packed(nasg_ctx *ctx, int64_t n, const float *q13, float *dir_pdf, float *c,
                             void *stream);
/* mixture_pdf (sphdist.hpp:84) and guided_pdf (guiding.hpp:51) at given
 * directions dir (n x float4).  Either output may be NULL. */
int nasg_query_pdf(nasg_ctx *ctx, int64_t n, const float *x, const float *wo, const float *nrm,
                   const float *dir, float b, const float *bsdf_pdf, float *mix_pdf,
                   float *guided_pdf, void *stream);
/* Guided scattering for a wavefront path tracer (SPEC.md tracer trace_path:
 * "scattering direction drawn from q-hat (mixture sample with probability c',
 * BSDF otherwise; pdf always the full blend)", guided_pdf guiding.cpp:81-85,
 * mixture_sample sphdist.cpp:183-198).  One network evaluation per vertex:
 *   in   x, wo, nrm, xi (n x float4 each, as nasg_query_sample)
 *        d_bsdf  n x float4: the caller's BSDF-sampled direction xyz, w = xi_t
 *        d_nee   n x float4: the NEE direction xyz, w > 0 when present
 *   out  out     2n x float4: [2i]   = (chosen direction xyz, q_mix there)
 *                             [2i+1] = (q_mix(d_nee) or 0, c' = b c,
 *                                       1 if the mixture was sampled else 0, c)
 * The blend pdf the renderer needs is c' q_mix + (1 - c') p_bsdf at each
 * direction (p_bsdf from its own material).  n_dev (nullable): a device int
 * read by the kernel as the row count (min with n), so a queue filled on the
 * device needs no host round trip; n is then the capacity. */
int nasg_query_shade(nasg_ctx *ctx, int64_t n, const int *n_dev, const float *x, const float *wo,
                     const float *nrm, const float *xi, const float *d_bsdf, const float *d_nee, float b,
                     float *out, void *stream);
/* encode_inputs + forward (infer_guide without decode): raw outputs in the
 * reference order, n x (8N+1).  Parity entry for the MLP. */
int nasg_query_raw(nasg_ctx *ctx, int64_t n, const float *x, const float *wo, const float *nrm,
                   float *raw, void *stream);
/* decode (guiding.hpp:47) + mixture_sample on given raw outputs — the
 * NASG epilogue alone (parity entry). */
int nasg_decode_sample_raw(nasg_ctx *ctx, int64_t n, const float *raw, const float *xi,
                           float *dir_pdf, float *c, void *stream);
int nasg_decode_pdf_raw(nasg_ctx *ctx, int64_t n, const float *raw, const float *dir, float b,
                        const float *bsdf_pdf, float *mix_pdf, float *guided_pdf, void *stream);
/* Host-buffer form of nasg_query_sample for callers without device memory:
 * pipelines H2D / kernel / D2H over chunks on the context's streams and
 * returns when dir_pdf (and c) are written.  Inputs are 4 floats/query. */
int nasg_query_sample_host(nasg_ctx *ctx, int64_t n, const float *x, const float *wo,
                           const float *nrm, const float *xi, float *dir_pdf, float *c);
/* Host-buffer form over packed 13-float rows: 52 B/query host->device instead
 * of 64 B, for PCIe-bound callers. */
int nasg_query_sample_host_packed(nasg_ctx *ctx, int64_t n, const float *q13, float *dir_pdf, float *c);

/* ---- training (Trainer::train_iteration guiding.hpp:149, guiding.cpp:196-282)
 * Runs T = nu*ceil(S/t) minibatch steps over the n samples (epochs reshuffled
 * with the reference's PCG32 Fisher-Yates), then publishes.  n == 0 is a
 * no-op + publish.  samples is a device array, complete when the call's first
 * kernel starts: stream order guarantees it, except after a producer kernel on
 * the same stream that releases its dependents early (programmatic dependent
 * launch, griddepcontrol.launch_dependents) — the step's first kernel reads the
 * rows before its own programmatic wait.  Blocks until stats are ready when
 * stats != NULL. */
int nasg_train_iteration(nasg_ctx *ctx, int64_t n, const nasg_train_sample *samples,
                         double blend_b, nasg_train_stats *stats, void *stream);
/* One data-parallel minibatch step on rows samples[order[0..count)] with the
 * 1/global_count scaling of guiding.cpp:262 (global_count = rows over all
 * ranks).  Accumulates loss/drop statistics into the context; gradient
 * exchange happens inside when a communicator is attached. */
int nasg_train_step(nasg_ctx *ctx, const nasg_train_sample *samples, const uint32_t *order,
                    int64_t count, int64_t global_count, double blend_b, void *stream);
/* Reads (and resets) the statistics accumulated by nasg_train_step. */
int nasg_train_stats_take(nasg_ctx *ctx, nasg_train_stats *stats);
/* Gradient of the last step (canonical weight layout, host copy). */
int nasg_get_last_grad(nasg_ctx *ctx, float *host_g, size_t n_floats);
int64_t nasg_adam_t(nasg_ctx *ctx);

/* ---- multi-GPU (NCCL over NVLink; one rank per GPU) ---------------------
 * Data-parallel train_iteration: rank r holds n_per_rank[r] samples.  The
 * global minibatch t is split over ranks in proportion to their buffers;
 * each rank walks its own PCG32-shuffled buffer with the reference's
 * cursor / epoch rule (guiding.cpp:236-243) for T = nu*ceil(S/t) steps.
 * Fills, per step, this rank's row count, the global row count (the 1/count
 * of guiding.cpp:262) and whether this rank reshuffles before the step.
 * With nranks == 1 the plan is exactly the reference's.  Host-only; returns
 * the number of steps, or -1 on bad arguments. */
int nasg_dp_plan(const nasg_config *cfg, const int64_t *n_per_rank, int nranks, int rank, int max_steps,
                 int64_t *local_count, int64_t *global_count, int32_t *reshuffle_before);
int nasg_comm_unique_id(void *out_128_bytes);
/* Create this rank's NCCL communicator (any nranks >= 1).  Once a context has a
 * communicator every Adam step runs the exchange (dW + statistics allreduce and
 * the finite re-check); with one rank it is an identity, bit for bit. */
int nasg_comm_init(nasg_ctx *ctx, const void *unique_id_128_bytes, int rank, int nranks);
/* Use a communicator the caller already has (an ncclComm_t, e.g. the one its
 * own data-parallel framework created over the same ranks) instead of creating
 * one; the context does not destroy it. */
int nasg_attach_nccl(nasg_ctx *ctx, void *nccl_comm, int rank, int nranks);

/* ---- counters (encode_clamp_count encoding.hpp:31-32) ------------------- */
typedef struct {
    uint64_t encode_clamps;    /* encode_clamp_count (encoding.hpp:31-32), this context */
    uint64_t kernel_launches;  /* device kernels launched by this context */
    int64_t adam_steps;        /* AdamState::t (net.hpp:115): applied, non-skipped updates */
    int64_t iterations;        /* Trainer::iterations_ (train_iteration calls) */
    int rank, nranks;          /* data-parallel position */
    uint64_t collectives;      /* NCCL launches issued: one grouped dW + statistics allreduce
                                  per Adam step, one buffer-size allgather per train_iteration */
} nasg_counters;
int nasg_get_counters(nasg_ctx *ctx, nasg_counters *out);  /* synchronises the device */
uint64_t nasg_encode_clamp_count(nasg_ctx *ctx);
void nasg_reset_encode_clamp_count(nasg_ctx *ctx);
/* Number of device kernel launches issued by this context since creation. */
uint64_t nasg_kernel_launches(nasg_ctx *ctx);

/* ---- host-side schedule helpers (guiding.hpp:77-120, guiding.cpp:178-182) */
double nasg_blend_coefficient(int64_t iteration, int m, int b_steps);
double nasg_stride_update(double l, uint64_t collected, uint64_t capacity);

/* ---- guided progressive render loop (SPEC.md tracer module :378-478; the
 * reference specifies it but ships no code) ---
 * A wavefront path tracer on the GPU: NEE + balance-heuristic MIS at every
 * non-delta vertex, scattering from the blend q-hat through nasg_query_shade,
 * Russian roulette from depth 5 (cap 0.95), max depth 16, per-vertex radiance
 * back-propagation into TrainingSamples for one pixel per l x l tile, then
 * train_iteration, stride_update and the progressive w_i ramp (SPEC accumulate).
 * Multi-GPU: each rank renders either the contiguous pixel rows [row_begin,
 * row_end) or (row_band > 0) every nshards-th band of row_band rows starting
 * with band `shard` — interleaved tile rows, so every rank sees the same mix
 * of scene content — and trains data-parallel through the context's NCCL
 * communicator (nasg_comm_init). */
typedef struct nasg_render nasg_render;
enum { NASG_SCENE_FURNACE = 0, NASG_SCENE_BOX = 1, NASG_SCENE_CRACK = 2, NASG_SCENE_DARK = 3, NASG_SCENE_ATTIC = 4,
       NASG_SCENE_INDIRECT = 5 /* SPEC acceptance 7: room lit only by the ceiling's bounce */ };
typedef struct {
    int scene;             /* NASG_SCENE_* */
    int width, height;     /* full image */
    int row_begin, row_end;/* this rank's rows; row_end <= 0 means height */
    uint64_t seed;
    int max_depth;         /* 16 */
    int rr_depth;          /* 5 */
    int guiding;           /* 1: blend schedule b = min(1, floor(i/M)/B); 0: b = 0 always */
    int collect;           /* 1: collect samples and train after every iteration */
    int ramp;              /* 1: accumulate with w_i = min(i+1, M B)/(M B); 0: plain mean */
    int schedule_m;        /* M = 4 */
    int schedule_b;        /* B = 64 */
    int nee;               /* 1: NEE + MIS (SPEC); 0: emitters reached by scattering only
                              (the brute-force reference of the SPEC's direct-light test) */
    int lazy_train_stats;  /* 0: stats.train is this iteration's TrainStats (the call waits for
                              training to finish); 1: stats.train is the previous iteration's
                              (no wait: the next iteration's tracing is queued behind training) */
    int pipelined;         /* 0: the SPEC loop (iteration i traces with the snapshot training i-1
                              published); 1: tracing of i+1 overlaps training i on a second stream,
                              so iteration i traces with the snapshot of training i-2 (one
                              iteration staler), and stats.train is training i-2's */
    int row_band;          /* > 0: interleaved sharding in bands of row_band rows (row_begin /
                              row_end ignored); this rank owns bands shard, shard + nshards, ...
                              and its image is those rows in order; collection tiles are laid
                              over that compacted image */
    int shard, nshards;    /* this rank's band phase and the band period (row_band > 0) */
} nasg_render_config;
typedef struct {
    int64_t iteration;     /* the iteration just rendered */
    double b;              /* blend coefficient used */
    double stride;         /* l used for collection (next one after stride_update) */
    int64_t paths, vertices, guided_vertices;
    int64_t collected;     /* samples produced by the selected pixels */
    int64_t kept;          /* min(collected, this rank's capacity) */
    int64_t nonfinite_paths;
    nasg_train_stats train;
} nasg_render_stats;
void nasg_render_config_default(nasg_render_config *cfg);
/* scene bounds for nasg_create (encoding's Aabb) */
int nasg_render_scene_bounds(int scene, float bmin[3], float bmax[3]);
int nasg_render_create(nasg_ctx *ctx, const nasg_render_config *cfg, nasg_render **out);
int nasg_render_destroy(nasg_render *r);
/* Render one sample per pixel, collect + train (cfg.collect), accumulate. */
int nasg_render_iteration(nasg_render *r, nasg_render_stats *stats);
/* Host copy of this rank's rows, (row_end-row_begin) x width x 3 floats:
 * which = 0 the accumulated image, 1 the last frame. */
int nasg_render_image(nasg_render *r, float *rgb, int which);
/* Device kernel launches issued by the render loop's own kernels. */
uint64_t nasg_render_kernel_launches(nasg_render *r);
/* MAPE (SPEC.md tracer mape, PAPER §7): per-pixel mean over channels of
 * |img - ref| / (ref + 0.01), the worst floor(0.1% of pixels) dropped. */
double nasg_mape(const float *img, const float *ref, int64_t npix);

/* ---- explicit-parameter mixtures: NASG and the vMF / SG baseline ----------
 * (sphdist.hpp:33-121).  Context-free, on the current CUDA
 * device, stream-ordered, device buffers.  Computed in double from fp32
 * records, as the reference computes in double.  Per query q, k components:
 *   NASG record  3 x float4 = (x_axis xyz, lambda), (y_axis xyz, a),
 *                (z_axis xyz, epsilon)    — NasgComponent sphdist.hpp:33-38
 *   vMF record   1 x float4 = (mu xyz, lambda) — VmfComponent sphdist.hpp:49-52
 *   comp         n x k records; weights n x k floats (sum to 1 per query)
 *   dir, xi      n x float4 (xi = xi_select, xi0, xi1, xi2; vMF ignores xi2)
 */
enum { NASG_DIST_NASG = 0, NASG_DIST_VMF = 1 };
/* mixture_pdf sphdist.hpp:84 / vmf_mixture_pdf :117 -> pdf (n floats) */
int nasg_dist_mixture_pdf(int kind, int64_t n, int k, const float *comp, const float *weights,
                          const float *dir, float *pdf, void *stream);
/* mixture_sample :97-98 / vmf_mixture_sample :119-120 -> dir_pdf (n x float4) */
int nasg_dist_mixture_sample(int kind, int64_t n, int k, const float *comp, const float *weights,
                             const float *xi, float *dir_pdf, void *stream);
/* nasg_grad_logpdf :68-71 (8 floats per component: d_cos_theta, d_sin_phi,
 * d_cos_phi, d_sin_tau, d_cos_tau, d_lambda, d_a, 0) / vmf_grad_logpdf :121
 * (4 floats: d_mu xyz, d_lambda) for every component of every query. */
int nasg_dist_grad_logpdf(int kind, int64_t n, int k, const float *comp, const float *weights,
                          const float *dir, float *grad, void *stream);

/* ---- NASG vs vMF expressiveness fit (SPEC.md run_fit :500-508, PAPER Fig. 5)
 * Fits n_fits independent position-free guide distributions (one CTA each)
 * to an analytic target mixture with the guider's KL gradient on directions
 * drawn from the target and the reference's Adam.  Model raw vectors:
 *   NASG  8N+1 floats in the network's raw-output order (guiding.hpp:25-30),
 *         decoded by decode_full (guiding.cpp:15-77); N in {1, 2, 4, 8, 16}
 *   vMF   5K floats: K unnormalised mean directions (xyz), K log-sharpness,
 *         K weight logits; K <= 32
 * Host buffers; blocks until done. */
typedef struct {
    int model;            /* NASG_DIST_NASG | NASG_DIST_VMF */
    int n_components;     /* the paper's comparison: 8 NASG (64 scalars) vs 14 vMF (70) */
    int batch;            /* target samples per Adam step */
    int steps;            /* Adam steps */
    int checkpoints;      /* raw snapshots, every steps/checkpoints steps (>= 1) */
    float learning_rate;
    uint64_t seed;
} nasg_fit_config;
int nasg_fit_raw_dim(int model, int n_components); /* -1 if unsupported */
/* target_comp / target_w: one explicit mixture of target_kind (records as
 * above, target_k <= 32).  raw_init (nullable): n_fits x raw_dim start
 * vectors, else a seeded init.  raw_out: n_fits x checkpoints x raw_dim.
 * kl_out (nullable): n_fits x checkpoints KL(target || model), integrated on
 * an equal-area grid of quad_nz x 2 quad_nz cells. */
int nasg_fit(const nasg_fit_config *cfg, int n_fits, int target_kind, int target_k,
             const float *target_comp, const float *target_w, const float *raw_init,
             float *raw_out, double *kl_out, int quad_nz);
/* The fit's mean gradient over given samples (n x float4: direction xyz,
 * target pdf p; q_sampling = p), raw_dim floats out — parity entry. */
int nasg_fit_gradient(int model, int n_components, const float *raw, int64_t n,
                      const float *samples, float *grad_out);
/* KL(target || model) for n_models raw vectors on the quad_nz grid. */
int nasg_fit_kl(int target_kind, int target_k, const float *target_comp, const float *target_w,
                int model, int n_components, int n_models, const float *raws, int quad_nz,
                double *kl_out);

/* ---- synthetic workloads (bench / tests) ----------------- */
/* Query i: Pcg32(hash_combine(seed, i), 0x51) -> x ~ U(bounds), omega_o and
 * normal ~ U(S^2), xi ~ U[0,1) as (u32 >> 8) * 2^-24.  Host arrays. */
void nasg_synth_queries(uint64_t seed, int64_t first, int64_t n, const float bmin[3],
                        const float bmax[3], float *x, float *wo, float *nrm, float *xi);
/* Sample i with the fixed analytic target of SURVEY §8d. */
void nasg_synth_samples(uint64_t seed, int64_t first, int64_t n, const float bmin[3],
                        const float bmax[3], nasg_train_sample *out);

#ifdef __cplusplus
}
#endif
#endif /* NASG_H */
