// Internal declarations shared by the host API (nasg_api.cpp) and the
// kernel translation units.  Not part of the C ABI.
#pragma once

#include <nvtx3/nvToolsExt.h>
#include <cstdint>
#include <utility>
#include <cuda_runtime.h>

#include "nasg/nasg.h"

namespace nasg {

constexpr int kIn = 64;        // encoding.hpp:12
constexpr int kHidden = 128;   // net.hpp:14
constexpr int kBins = 19;      // encoding.hpp:11
constexpr int kTileRows = 128; // query tile (one TMEM lane / thread per row)


// Packed raw-output layout of the last layer (see nasg_math.cuh): header of
// round_up(N + 1, 16) columns (weight logits, selection logit), then 8 columns per lobe.
__host__ __device__ constexpr int packed_header(int n) { return ((n + 1 + 15) / 16) * 16; }
__host__ __device__ constexpr int packed_width(int n) { return packed_header(n) + 8 * n; }

// fp32 packed weight image used by the SIMT kernels: W1[64][128], W2, W3, then
// the last layer in the packed raw order as f32_out_blocks(n) blocks of
// [128 k][128 packed cols] (zero-padded): one block for N <= 8, two for N = 16,
// three for N = 32.
__host__ __device__ constexpr int f32_out_blocks(int n) { return (packed_width(n) + 127) / 128; }
__host__ __device__ constexpr int packed_f32_floats(int n) {
    return kIn * kHidden + 2 * kHidden * kHidden + f32_out_blocks(n) * kHidden * 128;
}
// transposed copies for the backward delta GEMMs: W2^T, W3^T [128][128] and
// W4p^T [128 x blocks packed cols][128] (rows >= NP are zero).
__host__ __device__ constexpr int packed_t32_floats(int n) { return 2 * kHidden * kHidden + f32_out_blocks(n) * 128 * kHidden; }
// contraction length of the backward through W4p^T: NP rounded up to 16 (>= 128)
__host__ __device__ constexpr int f32_bwd_k(int n) { return packed_width(n) <= 128 ? 128 : (packed_width(n) + 15) / 16 * 16; }
// row stride of the fp32 trainer's delta4 (reference raw order, zero-padded;
// whole 128-column blocks past 80 so K_dw's block reads stay inside the row)
__host__ __device__ constexpr int d4_stride(int n) { return 8 * n + 1 <= 80 ? 80 : (8 * n + 1 + 127) / 128 * 128; }

__host__ __device__ inline int n_weights(int n) { return kIn * kHidden + 2 * kHidden * kHidden + kHidden * (8 * n + 1); }

// NVTX range for the scope of a host call (header-only NVTX 3: free unless a
// profiler is attached): train iterations / steps, query launches, render
// iterations and publishes show up as named ranges on the profiler timeline.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

// Makes `dev` current for the scope of one C-ABI call and restores the caller's
// device afterwards (one process may drive several contexts; a torch rank's
// current device must not move under it).
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev) {
        if (dev < 0) return;
        if (cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            prev = -1;
        }
        if (prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};
int ctx_device(const nasg_ctx *c);

// context accessors for the render loop (k_render.cu; nasg_ctx is opaque there)
int64_t ctx_sample_capacity(const nasg_ctx *c);  // TrainerConfig::sample_capacity S
int ctx_nranks(const nasg_ctx *c);
// start the next train_iteration's first-epoch shuffle for n rows on a host thread
int ctx_prefetch_shuffle(nasg_ctx *c, int64_t n);
// programmatic dependent launch of the training chain on (default) or off
void ctx_set_pdl(nasg_ctx *c, bool on);
// programmatic dependent launch of the query kernels (set by the serial render loop)
void ctx_set_query_pdl(nasg_ctx *c, bool on);
// enqueue on s: copy the training statistics accumulators (5 doubles) to a
// pinned host buffer and clear them; ctx_stats_from_acc converts after a sync
int ctx_train_stats_async(nasg_ctx *c, double *pinned_acc5, cudaStream_t s);
void ctx_stats_from_acc(const double *acc5, nasg_train_stats *st);               // data-parallel ranks (1 without NCCL)

struct Bounds {
    float bmin[3];
    double ext[3];      // bmax - bmin in double (Aabb::extent, math.hpp:70)
    float inv_ext[3];   // (float)(1 / ext), 0 for a degenerate axis (fp32 encoders)
};

// ---- kernels: packing -------------------------------------------------------
// wbig (nullable) is OR-ed with 1 when a weight is not finite or |w| >= kSafeWeight
void launch_pack_fp32(const float *w, int n_comp, float *wp, float *wtp, cudaStream_t s, int *wbig = nullptr);
// one-launch copy of up to three buffers (null src: skipped; sizes multiples of 16 B)
void launch_copy3(const void *const src[3], void *const dst[3], const size_t bytes[3], cudaStream_t s);

// Weight magnitude below which no forward pass can overflow for inputs with
// |feature| <= 2 (one-blob bins in [0,1], pad 1, direction components <= 2):
// |raw| <= 64 * 2 * 128^3 * B^4 = 2.7e36 < FLT_MAX at B = 1e7, bf16 rounding
// of the activations included.  Zero-gradient rows skip the network only
// while every weight is below it (train_classify_kernel).
constexpr float kSafeWeight = 1e7f;
// bf16 weight image for the tcgen05 kernel (smem image, UMMA core-matrix layout)
size_t tc_image_bytes(int n_comp);        // the query kernel's bf16 image
size_t tc_train_image_bytes(int n_comp);  // the bf16 trainer's f16 image + bf16 W4 copy
void launch_pack_tc(const float *w, int n_comp, void *img, cudaStream_t s, bool train = false);

// ---- kernels: queries -------------------------------------------------------
enum QueryMode { kModeSample = 0, kModePdf = 1, kModeRaw = 2, kModeShade = 3 };

struct QueryArgs {
    int64_t n;
    const float4 *x, *wo, *nrm;
    const float4 *xi;   // sample mode
    const float4 *dir;  // pdf mode
    const float *bsdf_pdf;
    float b;
    float4 *dir_pdf;
    float *c;
    float *mix_pdf, *guided_pdf;
    float *raw;  // raw mode (reference order)
    unsigned long long *clamp_count;
    Bounds bounds;
    // optional packed host format: 13 floats per query = position, omega_o,
    // normal (3 each) and xi (4); replaces x / wo / nrm / xi when non-null
    const float *packed;
    // optional device-side row count (a wavefront queue): rows = min(*n_dev, n)
    const int *n_dev;
    // shade mode (guided scattering at path vertices): BSDF sample + xi_t, NEE
    // direction + flag in; two float4 per row out (see guide_shade)
    const float4 *sh_bsdf, *sh_nee;
    float4 *sh_out;
};

#ifdef __CUDACC__
// Programmatic dependent launch: a kernel of the training chain lets the next
// one start its prologue (barrier init, TMEM allocation) while it still runs;
// griddepcontrol.wait then blocks until the previous grid has completed and its
// memory is visible, so it goes before the first read of the previous kernel's
// output.  The dependent grid launches only once every block of this one has
// started (and triggered), so waiting blocks can never starve it of SMs.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// pdl = false launches normally (no early start): when other streams run
// concurrent work (the pipelined render loop), early-started CTAs waiting in
// griddepcontrol.wait would hold SMs that work could use.
// cooperative = true additionally guarantees that every block of the grid is
// resident at once (a kernel with an in-kernel grid barrier).
template <class... KArgs, class... Args>
inline cudaError_t launch_ex(bool pdl, bool cooperative, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args &&...args) {
    if (!pdl && !cooperative) {
        k<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (pdl) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na++].val.programmaticStreamSerializationAllowed = 1;
    }
    if (cooperative) {
        at[na].id = cudaLaunchAttributeCooperative;
        at[na++].val.cooperative = 1;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(bool pdl, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args &&...args) {
    return launch_ex(pdl, false, k, grid, block, smem, s, std::forward<Args>(args)...);
}

__device__ __forceinline__ void load_query(const QueryArgs &a, int64_t q, float4 &x, float4 &wo, float4 &nrm) {
    if (a.packed) {
        const float *p = a.packed + q * 13;
        x = make_float4(p[0], p[1], p[2], 0.f);
        wo = make_float4(p[3], p[4], p[5], 0.f);
        nrm = make_float4(p[6], p[7], p[8], 0.f);
    } else {
        x = a.x[q];
        wo = a.wo[q];
        nrm = a.nrm[q];
    }
}
__device__ __forceinline__ float4 load_xi(const QueryArgs &a, int64_t q) {
    if (a.packed) {
        const float *p = a.packed + q * 13 + 9;
        return make_float4(p[0], p[1], p[2], p[3]);
    }
    return a.xi[q];
}
#endif

int query_fp32(int n_comp, QueryMode mode, const float *wp, const QueryArgs &a, int num_sms,
               cudaStream_t s);
int query_tc(int n_comp, QueryMode mode, const void *img, const QueryArgs &a, int num_sms,
             cudaStream_t s, bool pdl = false);
bool tc_supported(int n_comp);        // tensor-core query kernel compiled for this N
bool tc_train_supported(int n_comp);  // tensor-core trainer compiled for this N

int decode_raw(int n_comp, bool sample, bool fast, int64_t n, const float *raw, const float4 *xi,
               const float4 *dir, float b, const float *bsdf_pdf, float4 *dir_pdf, float *c,
               float *mix_pdf, float *guided_pdf, cudaStream_t s);

// ---- kernels: training ------------------------------------------------------
struct TrainScratch {
    // per-row activations (row-major [rows][features]) for the dW GEMMs
    float *h0, *h1, *h2, *h3;   // 64, 128, 128, 128 wide
    float *d1, *d2, *d3, *d4;   // 128, 128, 128, 80 (canonical raw order, padded)
    float *dw_partial;          // [splits][n_weights]
    double *tile_loss;          // per tile loss sum
    int *tile_loss_count, *tile_dropped;
    int64_t max_rows;
    int max_tiles;
    int splits;       // capacity of dw_partial
    int last_splits;  // splits used by the last train_dw
};

// bf16 tensor-core training scratch: per-128-row blocks of bf16 activations /
// deltas in the UMMA core-matrix layout, per-tile stats, dW partials.
struct TcTrainBufs {
    uint8_t *h0, *h1, *h2, *h3, *d1, *d2, *d3, *d4;
    double *tile_loss;
    int *tile_lc, *tile_dr;
    double *step_stats;
    float *partial;  // [4 layers][splits][128][128]
    int splits;
    int64_t max_blocks;
    // zero-gradient row skipping (train_classify_kernel): the step's rows that
    // need the network, in row order, and {live count, zero-row count}
    bool skip_zero = true;
    uint32_t *live = nullptr;  // two lists of live_cap rows: consecutive steps alternate
    int64_t *cls = nullptr;    // two {live, zero} pairs, same alternation
    int cls_par = 0;           // the list / pair the last train_classify wrote
    uint32_t *cur_live() const { return live + (size_t)cls_par * (size_t)live_cap; }
    int64_t *cur_cls() const { return cls + 2 * cls_par; }
    unsigned long long *scan_state = nullptr;  // decoupled look-back words, one per classify block
    int64_t scan_cap = 0;
    int64_t live_cap = 0;
    uint32_t scan_epoch = 0;
    const int *wbig = nullptr;  // set while some weight is >= kSafeWeight (or not finite)
};
size_t tc_train_block_bytes(int n_comp);
int train_tc_step(int n_comp, const void *img, const nasg_train_sample *samples, const uint32_t *order, int64_t count,
                  int64_t global_count, double b, double loss_blend, const Bounds &bounds, TcTrainBufs &tb,
                  int num_sms, unsigned long long *clamp_count, float *grad, int *nonfinite, cudaStream_t s,
                  bool pdl = true);
int train_step_stats_n(const double *tile_loss, const int *tile_lc, const int *tile_dr, int ntiles,
                       double *step_stats, cudaStream_t s);

// live_count (nullable): the classified step's row count on the device (order = its list)
int train_forward_backward(int n_comp, const float *wp, const float *wtp,
                           const nasg_train_sample *samples, const uint32_t *order,
                           int64_t count, const int64_t *live_count, int64_t global_count, double b,
                           double loss_blend, const Bounds &bounds, TrainScratch &sc, int num_sms,
                           unsigned long long *clamp_count, cudaStream_t s);
int train_dw(int n_comp, int64_t count, TrainScratch &sc, float *grad, cudaStream_t s,
             const int64_t *live_count = nullptr);
int train_reduce(int n_comp, const TrainScratch &sc, float *grad, int *nonfinite, cudaStream_t s);
int check_finite(const float *x, int n, int *nonfinite, cudaStream_t s);
int train_step_stats(const TrainScratch &sc, int64_t count, double *step_stats, cudaStream_t s,
                     const int64_t *cls = nullptr);
// zero-gradient row classification (k_train_tc.cu): the step's rows through the
// epoch order; p = 0 rows (finite inputs, weights below kSafeWeight) counted in
// tb.cls[1] (their encode clamps counted), the others listed in tb.live, tb.cls[0]
int train_classify(const nasg_train_sample *samples, const uint32_t *order, int64_t count, TcTrainBufs &tb,
                   const Bounds &bounds, unsigned long long *clamp_count, cudaStream_t s, bool pdl);
// skip decision, Adam t / bias corrections, accumulation of step stats into
// acc[0..4] = loss_sum, loss_count, dropped, skipped, steps
// Fused optimizer tail of one step (skip decision, t, bias corrections,
// adam_step, re-pack of the fp32 images and of the bf16 image when tc_img is
// set, statistics into acc, flag reset); nonfinite and ticket: 2 zeroed device
// words each.  recheck: the gradient was allreduced, so the skip flag is
// recomputed on it inside the launch (nonfinite[1], a grid barrier on
// ticket[1]; cooperative launch).
int train_adam(int n_comp, float *w, float *m, float *v, const float *grad, float lr, float *wp, float *wtp,
               void *tc_img, int *nonfinite, int64_t *adam_t, const double *step_stats, double *acc,
               unsigned int *ticket, cudaStream_t s, bool pdl, bool recheck, int *wbig);


// ---- explicit mixtures and the fit (k_sphdist.cu) --------------------------
// op 0 = pdf, 1 = sample, 2 = grad_logpdf
int dist_launch(int op, int kind, int64_t n, int k, const float *comp, const float *w, const float *in, float *out,
                cudaStream_t s);
struct FitLaunch {
    int model, k, tkind, tk;
    const float *tcomp, *tw;  // device
    int batch, steps, n_ckpt, n_fits;
    float lr;
    uint64_t seed;
    const float *raw_init;    // device, nullable
    const float *samples;     // device; non-null = gradient-only mode
    float *raw_out, *grad_out;
};
int fit_launch(const FitLaunch &L, cudaStream_t s);
int fit_max_components(int model);
int fit_max_target_components();
int fit_raw_dim_host(int model, int k);
int fit_target_grid(int tkind, int tk, const float *tcomp, const float *tw, int nz, double *p, cudaStream_t s);
int fit_kl(int model, int k, const float *raws, int n_models, int nz, const double *p, double *partial, int blocks,
           cudaStream_t s);

}  // namespace nasg
