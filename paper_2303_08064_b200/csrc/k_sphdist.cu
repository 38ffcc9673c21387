// Explicit-parameter spherical mixtures (NASG with epsilon, and the vMF / SG
// baseline) plus the NASG-vs-vMF fitting experiment.
//
// The reference's density layer (sphdist.hpp) works on explicit mixtures:
//   NASG  mixture_pdf :152-157, mixture_sample :183-198, nasg_grad_logpdf
//         :200-274 (with nasg_log_eval :133-140, nasg_norm_const :142-146,
//         nasg_sample :159-181, euler_from_frame :33-57; epsilon kept)
//   vMF   vmf_log_eval :276-278, vmf_norm_const :280-282, vmf_pdf :284-286,
//         vmf_mixture_pdf :288-293, vmf_sample :295-305 (frame_around :103-110),
//         vmf_mixture_sample :307-322, vmf_grad_logpdf :324-340
// The batched kernels below restate them in double (one thread per query,
// mixtures read from HBM as float4 records), exactly like the fp32 path's
// epilogue (nasg_refmath.cuh), so results agree with the reference to double
// rounding given the same fp32 inputs.
//
// The fit (SPEC.md run_fit :500-508, PAPER Fig. 5): one CTA owns one fit of a
// single position-free guide distribution to an analytic target mixture.
// Per Adam step it draws `batch` directions from the target (so w = p/q_s = 1),
// accumulates the guider's KL gradient over them in a fixed warp/lane order
// (deterministic), and applies the reference's Adam (net.hpp:137-158, float
// ops in the reference order).  The NASG model's raw vector is the network's
// raw output layout (guiding.hpp:25-30) and its per-sample gradient is
// kl_loss_gradient (guiding.cpp:108-165) at b = 0, e = 0, p_bsdf = 1/(4 pi) —
// i.e. -w d log q_mix / d raw — evaluated by the same device code as the
// fp32 trainer (ref::kl_grad_row).  The vMF model's raw vector is
//   [0, 3K)   unnormalised mean directions (mu = r / |r|)
//   [3K, 4K)  sharpness logits (lambda = clamp(exp(r), 1e-3, 3e3), as the NASG decode)
//   [4K, 5K)  weight logits (softmax)
// with the gradient chained through vmf_grad_logpdf (whose d_mu is already
// tangential, so d r = d_mu / |r|).  KL(target || model) is integrated on an
// equal-area (z, phi) grid, cell centres, in double.
#include <cstdint>
#include <cuda_runtime.h>

#include "nasg_internal.h"
#include "nasg_refmath.cuh"

namespace nasg {
namespace dist {

using ref::V3;
using ref::dot;
using ref::kPi;
using ref::kTwoPi;

constexpr double kUMin = 1e-12;       // sphdist.cpp:9
constexpr double kPoleGuard = 1e-6;   // sphdist.cpp:13
constexpr int kFitThreads = 256;
constexpr int kFitWarps = kFitThreads / 32;

__device__ __forceinline__ V3 v3(float4 f) { return {(double)f.x, (double)f.y, (double)f.z}; }
__device__ __forceinline__ V3 cross(const V3 &a, const V3 &b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ V3 normalize(const V3 &v) {  // math.hpp:43
    const double l = sqrt(dot(v, v));
    return {v.x / l, v.y / l, v.z / l};
}

// ---- NASG with epsilon (NasgComponent sphdist.hpp:33-38) --------------------
struct NasgC {
    V3 x, y, z;
    double lambda, a, eps;
};
// record: float4 (x_axis, lambda), (y_axis, a), (z_axis, epsilon)
__device__ __forceinline__ NasgC load_nasg(const float4 *p) {
    const float4 a = p[0], b = p[1], c = p[2];
    return {v3(a), v3(b), v3(c), (double)a.w, (double)b.w, (double)c.w};
}

struct LobeEval {  // sphdist.cpp:60-84
    double dz, dx, u, log_u, t2, denom, beta, m, u_pow_m;
};
__device__ __forceinline__ LobeEval eval_lobe(const NasgC &c, const V3 &v) {
    LobeEval e;
    e.dz = dot(v, c.z);
    e.dx = dot(v, c.x);
    e.u = fmin(fmax((e.dz + 1.0) * 0.5, kUMin), 1.0);
    e.log_u = log(e.u);
    e.denom = fmax(1.0 - e.dz * e.dz, 1e-12);
    e.t2 = fmin(fmax(e.dx * e.dx / e.denom, 0.0), 1.0);
    e.beta = c.a * e.t2;
    e.m = 1.0 + c.eps + e.beta;
    e.u_pow_m = pow(e.u, e.m);
    return e;
}
__device__ __forceinline__ double nasg_log_eval(const NasgC &c, const V3 &v) {  // :133-140
    const double dz = dot(v, c.z);
    if (dz >= 1.0 - 1e-12) return 0.0;
    if (dz <= -1.0 + 1e-12) return -INFINITY;
    const LobeEval e = eval_lobe(c, v);
    return 2.0 * c.lambda * (e.u_pow_m - 1.0) + (c.eps + e.beta) * e.log_u;
}
__device__ __forceinline__ double nasg_norm_const(const NasgC &c) {  // :142-146
    const double oe = 1.0 + c.eps;
    return kTwoPi * (-expm1(-2.0 * c.lambda)) / (c.lambda * sqrt(oe * (oe + c.a)));
}
__device__ __forceinline__ double nasg_pdf(const NasgC &c, const V3 &v) {  // :148-150
    return exp(nasg_log_eval(c, v)) / nasg_norm_const(c);
}
__device__ __forceinline__ V3 nasg_sample(const NasgC &c, double xi0, double xi1, double xi2) {  // :159-181
    const double emin = exp(-2.0 * c.lambda);
    const double s = emin + xi0 * (1.0 - emin);
    const double rho = (xi1 - 0.5) * kPi;
    const double oe = 1.0 + c.eps;
    const double cos_rho = cos(rho);
    const double expo = (oe + c.a - c.a * cos_rho * cos_rho) / (oe * (oe + c.a));
    const double base = fmin(fmax(log(s) / (2.0 * c.lambda) + 1.0, 0.0), 1.0);
    const double cos_t = fmin(fmax(2.0 * pow(base, expo) - 1.0, -1.0), 1.0);
    const double sin_t = sqrt(1.0 - cos_t * cos_t);
    const double stretch = sqrt((oe + c.a) / oe);
    double phi = atan2(stretch * sin(rho), cos_rho);
    if (xi2 <= 0.5) phi += kPi;
    const double cp = cos(phi), sp = sin(phi);
    return {c.x.x * (sin_t * cp) + c.y.x * (sin_t * sp) + c.z.x * cos_t,
            c.x.y * (sin_t * cp) + c.y.y * (sin_t * sp) + c.z.y * cos_t,
            c.x.z * (sin_t * cp) + c.y.z * (sin_t * sp) + c.z.z * cos_t};
}

struct Euler {
    double ct, sp, cp, st, ctau;
};
__device__ __forceinline__ Euler euler_from_frame(const NasgC &f) {  // :33-57
    Euler e;
    e.ct = fmin(fmax(f.z.z, -1.0), 1.0);
    const double s = sqrt(fmax(0.0, 1.0 - e.ct * e.ct));
    if (s > 1e-9) {
        e.cp = f.z.x / s;
        e.sp = f.z.y / s;
        ref::renorm_pair(e.sp, e.cp);
        e.ctau = -f.x.z / s;
        e.st = f.x.y * e.cp - f.x.x * e.sp;
        ref::renorm_pair(e.st, e.ctau);
    } else {
        e.sp = 0.0;
        e.cp = 1.0;
        e.ctau = e.ct > 0.0 ? f.x.x : -f.x.x;
        e.st = f.x.y;
        ref::renorm_pair(e.st, e.ctau);
    }
    return e;
}

// nasg_grad_logpdf (:200-274) for component c of weight wi, given q = mixture_pdf(m, v).
__device__ __forceinline__ void nasg_grad_logpdf(const NasgC &c, double wi, const V3 &v, double q, double g[7]) {
#pragma unroll
    for (int k = 0; k < 7; ++k) g[k] = 0.0;
    const double dz = dot(v, c.z);
    if (fabs(dz) > 1.0 - kPoleGuard) return;
    if (!(q > 0.0) || !isfinite(q)) return;
    const LobeEval e = eval_lobe(c, v);
    const double log_g = 2.0 * c.lambda * (e.u_pow_m - 1.0) + (c.eps + e.beta) * e.log_u;
    const double K = nasg_norm_const(c);
    const double r = wi * exp(log_g) / K / q;
    const double expm2l = exp(-2.0 * c.lambda);
    const double dlogK_dl = 2.0 * expm2l / (1.0 - expm2l) - 1.0 / c.lambda;
    const double dlogK_da = -0.5 / (1.0 + c.eps + c.a);
    const double dG_dbeta = (2.0 * c.lambda * e.u_pow_m + 1.0) * e.log_u;
    const double dG_du = 2.0 * c.lambda * e.m * pow(e.u, e.m - 1.0) + (c.eps + e.beta) / e.u;
    const double dt2_ddz = 2.0 * e.dz * e.t2 / e.denom;
    const double dG_ddz = 0.5 * dG_du + dG_dbeta * c.a * dt2_ddz;
    const double dG_ddx = dG_dbeta * c.a * 2.0 * e.dx / e.denom;
    g[5] = r * (2.0 * (e.u_pow_m - 1.0) - dlogK_dl);
    g[6] = r * (e.t2 * dG_dbeta - dlogK_da);
    const Euler t = euler_from_frame(c);
    const double ct = t.ct;
    const double st = sqrt(fmax(1e-18, 1.0 - ct * ct));
    const double dst = -ct / st;
    const V3 dz_dct = {t.cp * dst, t.sp * dst, 1.0}, dz_dsp = {0.0, st, 0.0}, dz_dcp = {st, 0.0, 0.0};
    const V3 dx_dct = {t.cp * t.ctau, t.sp * t.ctau, -dst * t.ctau};
    const V3 dx_dsp = {-t.st, ct * t.ctau, 0.0}, dx_dcp = {ct * t.ctau, t.st, 0.0};
    const V3 dx_dst = {-t.sp, t.cp, 0.0}, dx_dctau = {ct * t.cp, ct * t.sp, -st};
    double g_ct = dG_ddz * dot(v, dz_dct) + dG_ddx * dot(v, dx_dct);
    double g_sp = dG_ddz * dot(v, dz_dsp) + dG_ddx * dot(v, dx_dsp);
    double g_cp = dG_ddz * dot(v, dz_dcp) + dG_ddx * dot(v, dx_dcp);
    double g_st = dG_ddx * dot(v, dx_dst);
    double g_ctau = dG_ddx * dot(v, dx_dctau);
    double ps = t.cp * (t.cp * g_sp - t.sp * g_cp), pc = t.sp * (t.sp * g_cp - t.cp * g_sp);
    g_sp = ps;
    g_cp = pc;
    ps = t.ctau * (t.ctau * g_st - t.st * g_ctau);
    pc = t.st * (t.st * g_ctau - t.ctau * g_st);
    g_st = ps;
    g_ctau = pc;
    g[0] = r * g_ct;
    g[1] = r * g_sp;
    g[2] = r * g_cp;
    g[3] = r * g_st;
    g[4] = r * g_ctau;
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 7; ++k) ok &= isfinite(g[k]);
    if (!ok) {
#pragma unroll
        for (int k = 0; k < 7; ++k) g[k] = 0.0;
    }
}

// ---- vMF / normalised SG (VmfComponent sphdist.hpp:49-57) -------------------
struct VmfC {
    V3 mu;
    double lambda;
};
__device__ __forceinline__ VmfC load_vmf(const float4 *p) {
    const float4 a = p[0];
    return {v3(a), (double)a.w};
}
__device__ __forceinline__ double vmf_log_eval(const VmfC &c, const V3 &v) { return c.lambda * (dot(c.mu, v) - 1.0); }
__device__ __forceinline__ double vmf_norm_const(const VmfC &c) {
    return kTwoPi * (-expm1(-2.0 * c.lambda)) / c.lambda;
}
__device__ __forceinline__ double vmf_pdf(const VmfC &c, const V3 &v) { return exp(vmf_log_eval(c, v)) / vmf_norm_const(c); }
__device__ __forceinline__ V3 vmf_sample(const VmfC &c, double xi0, double xi1) {  // :295-305
    const double cos_t =
        fmin(fmax(1.0 + log1p(-xi0 * (-expm1(-2.0 * c.lambda))) / c.lambda, -1.0), 1.0);
    const double sin_t = sqrt(1.0 - cos_t * cos_t);
    const double phi = kTwoPi * xi1;
    // frame_around (:103-110)
    const V3 z = normalize(c.mu);
    const V3 helper = fabs(z.x) < 0.9 ? V3{1.0, 0.0, 0.0} : V3{0.0, 1.0, 0.0};
    const V3 x = normalize(cross(helper, z));
    const V3 y = cross(z, x);
    const double a1 = sin_t * cos(phi), a2 = sin_t * sin(phi);
    return {x.x * a1 + y.x * a2 + z.x * cos_t, x.y * a1 + y.y * a2 + z.y * cos_t, x.z * a1 + y.z * a2 + z.z * cos_t};
}
// vmf_grad_logpdf (:324-340) given q: out = (d_mu xyz, d_lambda)
__device__ __forceinline__ void vmf_grad_logpdf(const VmfC &c, double wi, const V3 &v, double q, double g[4]) {
    g[0] = g[1] = g[2] = g[3] = 0.0;
    if (!(q > 0.0) || !isfinite(q)) return;
    const double r = wi * vmf_pdf(c, v) / q;
    const double expm2l = exp(-2.0 * c.lambda);
    const double dlogK = 2.0 * expm2l / (1.0 - expm2l) - 1.0 / c.lambda;
    g[3] = r * ((dot(c.mu, v) - 1.0) - dlogK);
    const V3 gm = {v.x * c.lambda, v.y * c.lambda, v.z * c.lambda};
    const double p = dot(gm, c.mu);
    g[0] = (gm.x - c.mu.x * p) * r;
    g[1] = (gm.y - c.mu.y * p) * r;
    g[2] = (gm.z - c.mu.z * p) * r;
}

// Record stride (float4s per component) of each kind.
__host__ __device__ constexpr int rec4(int kind) { return kind == NASG_DIST_NASG ? 3 : 1; }

template <int KIND>
__device__ __forceinline__ double comp_pdf(const float4 *rec, const V3 &v) {
    if constexpr (KIND == NASG_DIST_NASG) return nasg_pdf(load_nasg(rec), v);
    else return vmf_pdf(load_vmf(rec), v);
}
template <int KIND>
__device__ __forceinline__ double mix_pdf(const float4 *comp, const float *w, int k, const V3 &v) {
    double pdf = 0.0;
    for (int i = 0; i < k; ++i) pdf += (double)w[i] * comp_pdf<KIND>(comp + rec4(KIND) * i, v);
    return pdf;
}

// ---- batched explicit-mixture kernels ---------------------------------------
template <int KIND>
__global__ void __launch_bounds__(128) dist_pdf_kernel(int64_t n, int k, const float4 *__restrict__ comp,
                                                       const float *__restrict__ w, const float4 *__restrict__ dir,
                                                       float *__restrict__ pdf) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    pdf[q] = (float)mix_pdf<KIND>(comp + q * k * rec4(KIND), w + q * k, k, v3(dir[q]));
}

template <int KIND>
__global__ void __launch_bounds__(128) dist_sample_kernel(int64_t n, int k, const float4 *__restrict__ comp,
                                                          const float *__restrict__ w, const float4 *__restrict__ xi,
                                                          float4 *__restrict__ dir_pdf) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const float4 *cq = comp + q * k * rec4(KIND);
    const float *wq = w + q * k;
    const float4 x = xi[q];
    int pick = k - 1;  // mixture_sample :185-193 / vmf_mixture_sample :309-317
    double acc = 0.0;
    for (int i = 0; i < k; ++i) {
        acc += (double)wq[i];
        if ((double)x.x < acc) {
            pick = i;
            break;
        }
    }
    V3 v;
    if constexpr (KIND == NASG_DIST_NASG)
        v = nasg_sample(load_nasg(cq + 3 * pick), (double)x.y, (double)x.z, (double)x.w);
    else
        v = vmf_sample(load_vmf(cq + pick), (double)x.y, (double)x.z);
    const double pdf = mix_pdf<KIND>(cq, wq, k, v);
    dir_pdf[q] = make_float4((float)v.x, (float)v.y, (float)v.z, (float)pdf);
}

// one thread per (query, component): NASG 8 floats (ParamGradient + pad), vMF 4 floats
template <int KIND>
__global__ void __launch_bounds__(128) dist_grad_kernel(int64_t n, int k, const float4 *__restrict__ comp,
                                                        const float *__restrict__ w, const float4 *__restrict__ dir,
                                                        float *__restrict__ grad) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * k) return;
    const int64_t q = t / k;
    const int i = (int)(t % k);
    const float4 *cq = comp + q * k * rec4(KIND);
    const float *wq = w + q * k;
    const V3 v = v3(dir[q]);
    const double qm = mix_pdf<KIND>(cq, wq, k, v);
    if constexpr (KIND == NASG_DIST_NASG) {
        double g[7];
        nasg_grad_logpdf(load_nasg(cq + 3 * i), (double)wq[i], v, qm, g);
        float4 *o = reinterpret_cast<float4 *>(grad) + 2 * t;
        o[0] = make_float4((float)g[0], (float)g[1], (float)g[2], (float)g[3]);
        o[1] = make_float4((float)g[4], (float)g[5], (float)g[6], 0.f);
    } else {
        double g[4];
        vmf_grad_logpdf(load_vmf(cq + i), (double)wq[i], v, qm, g);
        reinterpret_cast<float4 *>(grad)[t] = make_float4((float)g[0], (float)g[1], (float)g[2], (float)g[3]);
    }
}

// ---- fit -----------------------------------------------------------------------
constexpr int kMaxTargetK = 32;
constexpr int kMaxVmfK = 32;
constexpr int kMaxRaw = 5 * kMaxVmfK;  // >= packed_width(16) = 160 and 5K for vMF
static_assert(kMaxRaw >= packed_width(16), "fit scratch too small for N = 16");

struct FitShared {
    float raw[kMaxRaw];       // model parameters (NASG: packed layout; vMF: raw layout)
    float m[kMaxRaw], v[kMaxRaw];
    float part[kFitWarps][kMaxRaw];  // per-warp gradient sums (fixed order)
    float4 tcomp[3 * kMaxTargetK];
    float tw[kMaxTargetK];
    // decoded vMF model
    double vmu[kMaxVmfK][3], vlam[kMaxVmfK], vnorm[kMaxVmfK], vw[kMaxVmfK];
    int vclamp[kMaxVmfK];
    int skip;
    int t;  // AdamState::t: applied (non-skipped) steps
};

struct FitArgs {
    int model, k;           // model kind and lobes
    int tkind, tk;          // target kind and lobes
    const float4 *tcomp;    // target records
    const float *tw;        // target weights
    int batch, steps, ckpt_every, n_ckpt;
    float lr;
    uint64_t seed;
    const float *raw_init;  // [fits][P] reference layout, or null (seeded init)
    const float4 *samples;  // gradient-only mode: [batch] (dir xyz, p) with q_s = p
    float *raw_out;         // [fits][n_ckpt][P] reference layout
    float *grad_out;        // gradient-only mode: [P] reference layout
};

__host__ __device__ inline int fit_raw_dim(int model, int k) { return model == NASG_DIST_NASG ? 8 * k + 1 : 5 * k; }

// reference raw index j <-> model parameter slot
template <int N>
__device__ __forceinline__ int slot_of(int model, int j) {
    return model == NASG_DIST_NASG ? packed_col(j, N) : j;
}

__device__ __forceinline__ uint32_t pcg_hash(uint64_t &state) {  // PCG32 (math.hpp:87-121 generator family)
    const uint64_t old = state;
    state = old * 6364136223846793005ull + 1442695040888963407ull;
    const uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
    const uint32_t rot = (uint32_t)(old >> 59u);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
}
__device__ __forceinline__ double u01(uint64_t &s) { return (double)(pcg_hash(s) >> 8) * (1.0 / 16777216.0); }
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// draw one direction from the target (mixture_sample / vmf_mixture_sample)
__device__ __forceinline__ V3 target_sample(const FitShared &S, const FitArgs &a, uint64_t &rng, double &p) {
    const double xs = u01(rng), x0 = u01(rng), x1 = u01(rng), x2 = u01(rng);
    int pick = a.tk - 1;
    double acc = 0.0;
    for (int i = 0; i < a.tk; ++i) {
        acc += (double)S.tw[i];
        if (xs < acc) {
            pick = i;
            break;
        }
    }
    V3 v;
    if (a.tkind == NASG_DIST_NASG) {
        v = nasg_sample(load_nasg(S.tcomp + 3 * pick), x0, x1, x2);
        p = mix_pdf<NASG_DIST_NASG>(S.tcomp, S.tw, a.tk, v);
    } else {
        v = vmf_sample(load_vmf(S.tcomp + pick), x0, x1);
        p = mix_pdf<NASG_DIST_VMF>(S.tcomp, S.tw, a.tk, v);
    }
    return v;
}

// vMF decode of the raw vector into shared memory (threads < k)
__device__ __forceinline__ void vmf_decode(FitShared &S, int k) {
    const int i = threadIdx.x;
    if (i < k) {
        const double rx = S.raw[3 * i], ry = S.raw[3 * i + 1], rz = S.raw[3 * i + 2];
        const double nr = sqrt(rx * rx + ry * ry + rz * rz);
        const bool deg = nr < 1e-6;
        S.vmu[i][0] = deg ? 0.0 : rx / nr;
        S.vmu[i][1] = deg ? 0.0 : ry / nr;
        S.vmu[i][2] = deg ? 1.0 : rz / nr;
        S.vnorm[i] = deg ? 0.0 : nr;
        const double lam = exp((double)S.raw[3 * k + i]);
        S.vlam[i] = fmin(fmax(lam, 1e-3), 3e3);
        S.vclamp[i] = S.vlam[i] != lam;
    }
    if (threadIdx.x == 0) {  // softmax (guiding.cpp:62-70 form)
        double mx = -INFINITY, sum = 0.0;
        for (int j = 0; j < k; ++j) mx = fmax(mx, (double)S.raw[4 * k + j]);
        for (int j = 0; j < k; ++j) sum += (S.vw[j] = exp((double)S.raw[4 * k + j] - mx));
        for (int j = 0; j < k; ++j) S.vw[j] /= sum;
    }
}

// Per-sample gradient of -w log q_mix for the vMF model, reduced into part[warp].
// As kl_loss_gradient does for the NASG model, a sample whose gradient has any
// non-finite entry contributes nothing (guiding.cpp:159-163).
__device__ __forceinline__ void vmf_sample_grad(FitShared &S, int k, const V3 &v, double ws, double gscale,
                                                bool valid) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double q = 0.0;
    for (int i = 0; i < k; ++i) {
        const VmfC c = {{S.vmu[i][0], S.vmu[i][1], S.vmu[i][2]}, S.vlam[i]};
        q += S.vw[i] * vmf_pdf(c, v);
    }
    const bool usable = valid && isfinite(q) && q > 1e-300;
    const double scale = -ws;
    auto grads = [&](int i, float o[5]) {
        const VmfC c = {{S.vmu[i][0], S.vmu[i][1], S.vmu[i][2]}, S.vlam[i]};
        double g[4];
        vmf_grad_logpdf(c, S.vw[i], v, q, g);
        const double inv = S.vnorm[i] > 0.0 ? 1.0 / S.vnorm[i] : 0.0;
        const double r_i = S.vw[i] * vmf_pdf(c, v) / q;
        o[0] = (float)(scale * g[0] * inv * gscale);
        o[1] = (float)(scale * g[1] * inv * gscale);
        o[2] = (float)(scale * g[2] * inv * gscale);
        o[3] = S.vclamp[i] ? 0.f : (float)(scale * g[3] * S.vlam[i] * gscale);
        o[4] = (float)(scale * (r_i - S.vw[i]) * gscale);
    };
    bool fin = usable;
    for (int i = 0; i < k && fin; ++i) {
        float o[5];
        grads(i, o);
#pragma unroll
        for (int j = 0; j < 5; ++j) fin &= isfinite(o[j]);
    }
    for (int i = 0; i < k; ++i) {
        float o[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
        if (fin) grads(i, o);
        const int cols[5] = {3 * i, 3 * i + 1, 3 * i + 2, 3 * k + i, 4 * k + i};
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const float s = warp_sum(o[j]);
            if (lane == 0) S.part[warp][cols[j]] += s;
        }
    }
}

template <int N>
__device__ __forceinline__ void nasg_sample_grad(FitShared &S, const V3 &v, double p, double gscale, bool valid) {
    constexpr int PW = packed_width(N);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // kl_loss_gradient at b = 0, e = 0: q_hat = p_bsdf (uniform 1/(4 pi)), w = p / q_s
    TrainRow row;
    row.wi = make_float3((float)v.x, (float)v.y, (float)v.z);
    row.p = valid ? (float)p : 0.f;
    row.q_s = row.p;
    row.pbsdf = (float)(0.25 / kPi);
    double loss;
    float g[PW];  // compile-time columns: registers; the last put of a column wins
    auto raw = [&](int col) { return S.raw[col]; };
    auto put = [&](int col, float x) { g[col] = x; };
    ref::kl_grad_row<N>(raw, row, 0.0, 0.0, gscale, put, loss);
    static_for<0, PW>([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        const float s = warp_sum(g[j]);
        if (lane == 0) S.part[warp][j] += s;
    });
}

template <int N>
__device__ void fit_gradient(FitShared &S, const FitArgs &a, int P, int step, int fit, bool from_samples) {
    for (int j = threadIdx.x; j < kFitWarps * kMaxRaw; j += blockDim.x) (&S.part[0][0])[j] = 0.f;
    if (a.model == NASG_DIST_VMF) vmf_decode(S, a.k);
    __syncthreads();
    const double gscale = 1.0 / (double)a.batch;
    uint64_t rng = mix64(a.seed ^ mix64(((uint64_t)fit << 40) ^ ((uint64_t)step << 12) ^ threadIdx.x)) | 1ull;
    for (int base = 0; base < a.batch; base += blockDim.x) {
        const int idx = base + threadIdx.x;
        const bool valid = idx < a.batch;
        V3 v = {0.0, 0.0, 1.0};
        double p = 0.0;
        if (valid) {
            if (from_samples) {
                const float4 s = a.samples[idx];
                v = v3(s);
                p = (double)s.w;
            } else {
                v = target_sample(S, a, rng, p);
                // the sample record stores floats (TrainingSample's omega_i)
                v = {(double)(float)v.x, (double)(float)v.y, (double)(float)v.z};
            }
        }
        if (a.model == NASG_DIST_NASG) nasg_sample_grad<N>(S, v, p, gscale, valid);
        else vmf_sample_grad(S, a.k, v, 1.0, gscale, valid && p > 0.0);
        __syncwarp();
    }
    __syncthreads();
    // fixed-order sum over warps
    for (int j = threadIdx.x; j < P; j += blockDim.x) {
        float g = 0.f;
        for (int w = 0; w < kFitWarps; ++w) g += S.part[w][j];
        S.part[0][j] = g;
    }
    __syncthreads();
}

// One CTA per fit: init, steps x (gradient, Adam), checkpoints of the raw vector.
template <int N>
__global__ void __launch_bounds__(kFitThreads) fit_kernel(FitArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FitShared &S = *reinterpret_cast<FitShared *>(smem_raw);
    const int fit = blockIdx.x;
    const int D = fit_raw_dim(a.model, a.k);                                    // reference layout
    const int P = a.model == NASG_DIST_NASG ? packed_width(N) : D;              // slots
    for (int j = threadIdx.x; j < kMaxRaw; j += blockDim.x) S.raw[j] = S.m[j] = S.v[j] = 0.f;
    if (threadIdx.x == 0) S.t = 0;
    for (int j = threadIdx.x; j < rec4(a.tkind) * a.tk; j += blockDim.x) S.tcomp[j] = a.tcomp[j];
    for (int j = threadIdx.x; j < a.tk; j += blockDim.x) S.tw[j] = a.tw[j];
    __syncthreads();
    for (int j = threadIdx.x; j < D; j += blockDim.x) {
        float r;
        if (a.raw_init) {
            r = a.raw_init[(int64_t)fit * D + j];
        } else {  // seeded init: orientation / mean logits U(-1.5, 1.5), sharpness e^U(0, 2.3)
            uint64_t s = mix64(a.seed * 0x9e3779b97f4a7c15ull + (uint64_t)fit * 1000003ull + j) | 1ull;
            const double u = u01(s);
            const int k = a.k;
            if (a.model == NASG_DIST_NASG) {
                if (j < 5 * k) r = (float)(3.0 * u - 1.5);
                else if (j < 7 * k) r = ((j - 5 * k) % 2 == 0) ? (float)(2.3 * u) : (float)(2.3 * u - 2.3);
                else r = 0.f;  // weight logits and c
            } else {
                if (j < 3 * k) r = (float)(2.0 * u - 1.0);
                else if (j < 4 * k) r = (float)(2.3 * u);
                else r = 0.f;
            }
        }
        S.raw[slot_of<N>(a.model, j)] = r;
    }
    __syncthreads();
    const float b1 = 0.9f, b2 = 0.999f, eps = 1e-8f;
    int ck = 0;
    for (int step = 1; step <= a.steps; ++step) {
        fit_gradient<N>(S, a, P, step, fit, false);
        if (threadIdx.x == 0) {  // adam_step: non-finite gradient -> skip (net.hpp:139-143)
            int bad = 0;
            for (int j = 0; j < P; ++j) bad |= !isfinite(S.part[0][j]);
            S.skip = bad;
            if (!bad) ++S.t;
        }
        __syncthreads();
        if (!S.skip) {
            const float t = (float)S.t;
            const float c1 = 1.f - powf(b1, t), c2 = 1.f - powf(b2, t);
            for (int j = threadIdx.x; j < P; j += blockDim.x) {
                const float gi = S.part[0][j];
                const float mi = __fadd_rn(__fmul_rn(b1, S.m[j]), __fmul_rn(__fsub_rn(1.f, b1), gi));
                const float vi = __fadd_rn(__fmul_rn(b2, S.v[j]), __fmul_rn(__fsub_rn(1.f, b2), __fmul_rn(gi, gi)));
                const float mh = __fdiv_rn(mi, c1), vh = __fdiv_rn(vi, c2);
                S.raw[j] = __fsub_rn(S.raw[j], __fdiv_rn(__fmul_rn(a.lr, mh), __fadd_rn(__fsqrt_rn(vh), eps)));
                S.m[j] = mi;
                S.v[j] = vi;
            }
        }
        __syncthreads();
        if (step % a.ckpt_every == 0 && ck < a.n_ckpt) {
            float *o = a.raw_out + ((int64_t)fit * a.n_ckpt + ck) * D;
            for (int j = threadIdx.x; j < D; j += blockDim.x) o[j] = S.raw[slot_of<N>(a.model, j)];
            ++ck;
        }
        __syncthreads();
    }
}

// Gradient-only entry (parity): mean gradient over given samples, reference layout.
template <int N>
__global__ void __launch_bounds__(kFitThreads) fit_grad_kernel(FitArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FitShared &S = *reinterpret_cast<FitShared *>(smem_raw);
    const int D = fit_raw_dim(a.model, a.k);
    const int P = a.model == NASG_DIST_NASG ? packed_width(N) : D;
    for (int j = threadIdx.x; j < kMaxRaw; j += blockDim.x) S.raw[j] = 0.f;
    __syncthreads();
    for (int j = threadIdx.x; j < D; j += blockDim.x) S.raw[slot_of<N>(a.model, j)] = a.raw_init[j];
    __syncthreads();
    fit_gradient<N>(S, a, P, 0, 0, true);
    for (int j = threadIdx.x; j < D; j += blockDim.x) a.grad_out[j] = S.part[0][slot_of<N>(a.model, j)];
}

// ---- KL(target || model) quadrature ------------------------------------------
// equal-area grid: z_i = -1 + (i + 1/2) 2/nz, phi_j = (j + 1/2) 2 pi / (2 nz)
__device__ __forceinline__ V3 grid_dir(int64_t t, int nz) {
    const int nphi = 2 * nz;
    const int i = (int)(t / nphi), j = (int)(t % nphi);
    const double z = -1.0 + (i + 0.5) * (2.0 / nz);
    const double phi = (j + 0.5) * (kTwoPi / nphi);
    const double r = sqrt(fmax(0.0, 1.0 - z * z));
    return {r * cos(phi), r * sin(phi), z};
}

__global__ void target_grid_kernel(int tkind, int tk, const float4 *tcomp, const float *tw, int nz, double *p) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = (int64_t)nz * 2 * nz;
    if (t >= n) return;
    const V3 v = grid_dir(t, nz);
    p[t] = tkind == NASG_DIST_NASG ? mix_pdf<NASG_DIST_NASG>(tcomp, tw, tk, v) : mix_pdf<NASG_DIST_VMF>(tcomp, tw, tk, v);
}

// Decode one model raw vector (reference layout) into explicit records + weights.
// NASG: decode_full (guiding.cpp:15-77) through ref::decode_lobe; vMF: the fit's decode.
__device__ void decode_model(int model, int k, const float *raw, float4 *comp, float *w) {
    const int i = threadIdx.x;
    if (i < k) {
        if (model == NASG_DIST_NASG) {
            float r[7];
            for (int j = 0; j < 5; ++j) r[j] = raw[5 * i + j];
            r[5] = raw[5 * k + 2 * i];
            r[6] = raw[5 * k + 2 * i + 1];
            ref::Lobe L;
            ref::decode_lobe(r, L);
            comp[3 * i] = make_float4((float)L.x.x, (float)L.x.y, (float)L.x.z, (float)L.lambda);
            comp[3 * i + 1] = make_float4((float)L.y.x, (float)L.y.y, (float)L.y.z, (float)L.a);
            comp[3 * i + 2] = make_float4((float)L.z.x, (float)L.z.y, (float)L.z.z, 0.f);
        } else {
            const double rx = raw[3 * i], ry = raw[3 * i + 1], rz = raw[3 * i + 2];
            const double nr = sqrt(rx * rx + ry * ry + rz * rz);
            const bool deg = nr < 1e-6;
            const double lam = fmin(fmax(exp((double)raw[3 * k + i]), 1e-3), 3e3);
            comp[i] = make_float4(deg ? 0.f : (float)(rx / nr), deg ? 0.f : (float)(ry / nr), deg ? 1.f : (float)(rz / nr),
                                  (float)lam);
        }
    }
    if (threadIdx.x == 0) {
        const int off = model == NASG_DIST_NASG ? 7 * k : 4 * k;
        double mx = -INFINITY, sum = 0.0, e[kMaxVmfK];
        for (int j = 0; j < k; ++j) mx = fmax(mx, (double)raw[off + j]);
        for (int j = 0; j < k; ++j) sum += (e[j] = exp((double)raw[off + j] - mx));
        for (int j = 0; j < k; ++j) w[j] = (float)(e[j] / sum);
    }
}

// grid: (blocks over points, models); partial[model][block] = sum p log(p/q) dA
__global__ void __launch_bounds__(256) kl_kernel(int model, int k, const float *raws, int nz, const double *p,
                                                 double *partial) {
    __shared__ float4 comp[3 * kMaxVmfK];
    __shared__ float w[kMaxVmfK];
    __shared__ double red[256 / 32];
    const int D = fit_raw_dim(model, k);
    decode_model(model, k, raws + (int64_t)blockIdx.y * D, comp, w);
    __syncthreads();
    const int64_t n = (int64_t)nz * 2 * nz;
    const double dA = 4.0 * kPi / (double)n;
    double acc = 0.0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const double pt = p[t];
        if (!(pt > 0.0)) continue;
        const V3 v = grid_dir(t, nz);
        const double q = model == NASG_DIST_NASG ? mix_pdf<NASG_DIST_NASG>(comp, w, k, v) : mix_pdf<NASG_DIST_VMF>(comp, w, k, v);
        acc += pt * log(pt / fmax(q, 1e-300)) * dA;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int j = 0; j < (int)(blockDim.x >> 5); ++j) s += red[j];
        partial[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
    }
}

}  // namespace dist

// ---- launchers (nasg_internal.h) ----------------------------------------------
int dist_launch(int op, int kind, int64_t n, int k, const float *comp, const float *w, const float *in, float *out,
                cudaStream_t s) {
    if (n == 0) return 0;
    const int64_t rows = op == 2 ? n * k : n;
    const unsigned grid = (unsigned)((rows + 127) / 128);
    const float4 *c4 = reinterpret_cast<const float4 *>(comp);
    const float4 *i4 = reinterpret_cast<const float4 *>(in);
    if (kind == NASG_DIST_NASG) {
        if (op == 0) dist::dist_pdf_kernel<NASG_DIST_NASG><<<grid, 128, 0, s>>>(n, k, c4, w, i4, out);
        else if (op == 1) dist::dist_sample_kernel<NASG_DIST_NASG><<<grid, 128, 0, s>>>(n, k, c4, w, i4, reinterpret_cast<float4 *>(out));
        else dist::dist_grad_kernel<NASG_DIST_NASG><<<grid, 128, 0, s>>>(n, k, c4, w, i4, out);
    } else {
        if (op == 0) dist::dist_pdf_kernel<NASG_DIST_VMF><<<grid, 128, 0, s>>>(n, k, c4, w, i4, out);
        else if (op == 1) dist::dist_sample_kernel<NASG_DIST_VMF><<<grid, 128, 0, s>>>(n, k, c4, w, i4, reinterpret_cast<float4 *>(out));
        else dist::dist_grad_kernel<NASG_DIST_VMF><<<grid, 128, 0, s>>>(n, k, c4, w, i4, out);
    }
    return 1;
}

int fit_max_components(int model) { return model == NASG_DIST_NASG ? 16 : dist::kMaxVmfK; }
int fit_max_target_components() { return dist::kMaxTargetK; }
int fit_raw_dim_host(int model, int k) { return dist::fit_raw_dim(model, k); }

template <int N>
static int fit_launch_n(const FitLaunch &L, cudaStream_t s) {
    dist::FitArgs a{};
    a.model = L.model;
    a.k = L.k;
    a.tkind = L.tkind;
    a.tk = L.tk;
    a.tcomp = reinterpret_cast<const float4 *>(L.tcomp);
    a.tw = L.tw;
    a.batch = L.batch;
    a.steps = L.steps;
    a.n_ckpt = L.n_ckpt;
    a.ckpt_every = L.n_ckpt > 0 ? (L.steps / L.n_ckpt > 0 ? L.steps / L.n_ckpt : 1) : L.steps + 1;
    a.lr = L.lr;
    a.seed = L.seed;
    a.raw_init = L.raw_init;
    a.samples = reinterpret_cast<const float4 *>(L.samples);
    a.raw_out = L.raw_out;
    a.grad_out = L.grad_out;
    const size_t sm = sizeof(dist::FitShared);
    if (L.samples) {
        cudaFuncSetAttribute(dist::fit_grad_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        dist::fit_grad_kernel<N><<<1, dist::kFitThreads, sm, s>>>(a);
    } else {
        cudaFuncSetAttribute(dist::fit_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        dist::fit_kernel<N><<<L.n_fits, dist::kFitThreads, sm, s>>>(a);
    }
    return 1;
}

int fit_launch(const FitLaunch &L, cudaStream_t s) {
    if (L.model == NASG_DIST_VMF) return fit_launch_n<1>(L, s);  // N unused by the vMF model
    switch (L.k) {
        case 1: return fit_launch_n<1>(L, s);
        case 2: return fit_launch_n<2>(L, s);
        case 4: return fit_launch_n<4>(L, s);
        case 8: return fit_launch_n<8>(L, s);
        case 16: return fit_launch_n<16>(L, s);
        default: return -1;
    }
}

int fit_target_grid(int tkind, int tk, const float *tcomp, const float *tw, int nz, double *p, cudaStream_t s) {
    const int64_t n = (int64_t)nz * 2 * nz;
    dist::target_grid_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(tkind, tk, reinterpret_cast<const float4 *>(tcomp),
                                                                          tw, nz, p);
    return 1;
}

int fit_kl(int model, int k, const float *raws, int n_models, int nz, const double *p, double *partial, int blocks,
           cudaStream_t s) {
    dist::kl_kernel<<<dim3(blocks, n_models), 256, 0, s>>>(model, k, raws, nz, p, partial);
    return 1;
}

}  // namespace nasg
