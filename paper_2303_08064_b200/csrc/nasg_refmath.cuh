// Double-precision NASG epilogue of the fp32 path.
//
// The reference runs its MLP in float and everything after it — decode,
// densities, sampling and the KL gradient — in double (guiding.cpp:15-176,
// sphdist.cpp:15-274).  The fp32 path does the same on the GPU: these device
// functions restate those formulas in double, in the reference's operation
// order, so that given identical raw network outputs the fp32 path agrees
// with the reference to ~1e-12 (libm-vs-CUDA ulp differences only).  The
// bf16 tensor-core path uses the fp32 stable forms in nasg_math.cuh instead.
//
// Lobes are decoded on the fly from the packed raw outputs (one lobe's
// seven logits are contiguous, see nasg_math.cuh) to keep register pressure
// bounded; re-decoding is deterministic, so results equal a decode-once.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "nasg_math.cuh"

namespace nasg {
namespace ref {

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 2.0 * kPi;

// one_blob bin i of a normalised coordinate t (encoding.cpp:11-19): the
// Gaussian bump in double, rounded to float — identical to the reference's
// encoding up to CUDA-vs-glibc exp ulps.
__device__ __forceinline__ float one_blob_bin(double t, int i, int k = 19) {
    const double sigma = 1.0 / k;
    const double inv_two_sigma2 = 1.0 / (2.0 * sigma * sigma);
    const double center = (i + 0.5) / k;
    const double d = t - center;
    return (float)exp(-d * d * inv_two_sigma2);
}

struct V3 {
    double x, y, z;
};
__device__ __forceinline__ double dot(const V3 &a, const V3 &b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

struct Lobe {
    V3 x, y, z;
    double lambda, a;
    // decode intermediates for the KL chain (DecodedGuide guiding.hpp:34-42)
    double sig[5], pn[2];
    bool lam_clamped, a_clamped;
};

__device__ __forceinline__ double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }  // guiding.cpp:9

__device__ __forceinline__ bool renorm_pair(double &s, double &c) {  // sphdist.cpp:15-25
    double n = sqrt(s * s + c * c);
    if (n < 1e-6) {
        s = 0.0;
        c = 1.0;
        return false;
    }
    s /= n;
    c /= n;
    return true;
}

// decode_full for one lobe (guiding.cpp:26-60) + frame_from_euler (sphdist.cpp:87-101)
__device__ __forceinline__ void decode_lobe(const float r[7], Lobe &L) {
    double trig[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        L.sig[k] = sigmoid((double)r[k]);
        trig[k] = L.sig[k] * 2.0 - 1.0;
    }
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        double &s = trig[1 + 2 * p], &c = trig[2 + 2 * p];
        double norm = sqrt(s * s + c * c);
        if (norm < 1e-6) {
            s = 0.0;
            c = 1.0;
            L.pn[p] = 0.0;
        } else {
            s /= norm;
            c /= norm;
            L.pn[p] = norm;
        }
    }
    double sp = trig[1], cp = trig[2], st = trig[3], ctau = trig[4];
    renorm_pair(sp, cp);  // frame_from_euler renormalises again (sphdist.cpp:90-91)
    renorm_pair(st, ctau);
    const double c = fmin(fmax(trig[0], -1.0), 1.0);
    const double s = sqrt(fmax(0.0, 1.0 - c * c));
    L.z = {cp * s, sp * s, c};
    L.x = {c * cp * ctau - sp * st, c * sp * ctau + cp * st, -s * ctau};
    L.y = {L.z.y * L.x.z - L.z.z * L.x.y, L.z.z * L.x.x - L.z.x * L.x.z, L.z.x * L.x.y - L.z.y * L.x.x};
    const double lam = exp((double)r[5]), a = exp((double)r[6]);
    L.lambda = fmin(fmax(lam, 1e-3), 3e3);
    L.a = (3e3 < a) ? 3e3 : a;  // std::min(a, 3e3)
    L.lam_clamped = L.lambda != lam;
    L.a_clamped = L.a != a;
}

struct LEval {
    double dz, dx, u, log_u, t2, denom, beta, m, u_pow_m;
};

__device__ __forceinline__ LEval eval_lobe(const Lobe &c, const V3 &v) {  // sphdist.cpp:71-83
    LEval e;
    e.dz = dot(v, c.z);
    e.dx = dot(v, c.x);
    e.u = fmin(fmax((e.dz + 1.0) * 0.5, 1e-12), 1.0);
    e.log_u = log(e.u);
    e.denom = fmax(1.0 - e.dz * e.dz, 1e-12);
    e.t2 = fmin(fmax(e.dx * e.dx / e.denom, 0.0), 1.0);
    e.beta = c.a * e.t2;
    e.m = 1.0 + e.beta;
    e.u_pow_m = pow(e.u, e.m);
    return e;
}

__device__ __forceinline__ double log_eval(const Lobe &c, const V3 &v) {  // sphdist.cpp:133-140
    const double dz = dot(v, c.z);
    if (dz >= 1.0 - 1e-12) return 0.0;
    if (dz <= -1.0 + 1e-12) return -INFINITY;
    LEval e = eval_lobe(c, v);
    return 2.0 * c.lambda * (e.u_pow_m - 1.0) + e.beta * e.log_u;
}

__device__ __forceinline__ double norm_const(const Lobe &c) {  // sphdist.cpp:142-146 (eps = 0)
    return kTwoPi * (-expm1(-2.0 * c.lambda)) / (c.lambda * sqrt(1.0 * (1.0 + c.a)));
}

__device__ __forceinline__ double lobe_pdf(const Lobe &c, const V3 &v) {  // sphdist.cpp:148-150
    return exp(log_eval(c, v)) / norm_const(c);
}

// nasg_sample sphdist.cpp:159-181
__device__ __forceinline__ V3 lobe_sample(const Lobe &c, double xi0, double xi1, double xi2) {
    const double emin = exp(-2.0 * c.lambda);
    const double s = emin + xi0 * (1.0 - emin);
    const double rho = (xi1 - 0.5) * kPi;
    const double cos_rho = cos(rho);
    const double expo = (1.0 + c.a - c.a * cos_rho * cos_rho) / (1.0 * (1.0 + c.a));
    const double base = fmin(fmax(log(s) / (2.0 * c.lambda) + 1.0, 0.0), 1.0);
    const double cos_t = fmin(fmax(2.0 * pow(base, expo) - 1.0, -1.0), 1.0);
    const double sin_t = sqrt(1.0 - cos_t * cos_t);
    const double stretch = sqrt((1.0 + c.a) / 1.0);
    double phi = atan2(stretch * sin(rho), cos_rho);
    if (xi2 <= 0.5) phi += kPi;
    const double cp = cos(phi), sp = sin(phi);
    return {c.x.x * (sin_t * cp) + c.y.x * (sin_t * sp) + c.z.x * cos_t,
            c.x.y * (sin_t * cp) + c.y.y * (sin_t * sp) + c.z.y * cos_t,
            c.x.z * (sin_t * cp) + c.y.z * (sin_t * sp) + c.z.z * cos_t};
}

template <int N, class RawFn>
__device__ __forceinline__ void load_lobe(RawFn raw, int i, float (&r)[7]) {
    constexpr int H = packed_header(N);
#pragma unroll
    for (int k = 0; k < 7; ++k) r[k] = raw(H + 8 * i + k);
}

// softmax + clamped sigmoid of c (guiding.cpp:62-75)
template <int N, class RawFn>
__device__ __forceinline__ void decode_header(RawFn raw, double (&w)[N], double &c, double &c_sig) {
    double mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < N; ++i) mx = fmax(mx, (double)raw(i));
    double sum = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        w[i] = exp((double)raw(i) - mx);
        sum += w[i];
    }
#pragma unroll
    for (int i = 0; i < N; ++i) w[i] /= sum;
    c_sig = sigmoid((double)raw(N));
    c = fmin(fmax(c_sig, 0.01), 0.99);
}

template <int N, class RawFn>
__device__ __forceinline__ double mixture_pdf(RawFn raw, const double (&w)[N], const V3 &v) {  // :152-157
    double pdf = 0.0;
    static_for<0, N>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        float r[7];
        load_lobe<N>(raw, i, r);
        Lobe L;
        decode_lobe(r, L);
        pdf += w[i] * lobe_pdf(L, v);
    });
    return pdf;
}

// infer_guide's decode + mixture_sample (sphdist.cpp:183-198): (dir, pdf), c
template <int N, class RawFn>
__device__ __forceinline__ float4 guide_sample(RawFn raw, float4 xi, float &c_out) {
    double w[N], c, c_sig;
    decode_header<N>(raw, w, c, c_sig);
    c_out = (float)c;
    int pick = N - 1;
    double acc = 0.0;
    bool found = false;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        acc += w[i];
        const bool hit = !found && (double)xi.x < acc;
        pick = hit ? i : pick;
        found |= hit;
    }
    float rs[7];
    static_for<0, N>([&](auto ic) {  // register-resident raw: select without dynamic indexing
        constexpr int i = decltype(ic)::value;
        float r[7];
        load_lobe<N>(raw, i, r);
#pragma unroll
        for (int k = 0; k < 7; ++k) rs[k] = (i == pick) ? r[k] : (i == 0 ? r[k] : rs[k]);
    });
    Lobe Ls;
    decode_lobe(rs, Ls);
    const V3 v = lobe_sample(Ls, (double)xi.y, (double)xi.z, (double)xi.w);
    const double pdf = mixture_pdf<N>(raw, w, v);
    return make_float4((float)v.x, (float)v.y, (float)v.z, (float)pdf);
}

// mixture_pdf and guided_pdf at a direction (guiding.cpp:81-85)
template <int N, class RawFn>
__device__ __forceinline__ float2 guide_pdf(RawFn raw, float3 dir, float b, float bsdf_pdf) {
    double w[N], c, c_sig;
    decode_header<N>(raw, w, c, c_sig);
    const V3 v = {(double)dir.x, (double)dir.y, (double)dir.z};
    const double pdf = mixture_pdf<N>(raw, w, v);
    const double ce = (double)b * c;
    const double guided = ce <= 0.0 ? (double)bsdf_pdf : ce * pdf + (1.0 - ce) * (double)bsdf_pdf;
    return make_float2((float)pdf, (float)guided);
}

// guided scattering at a path vertex in double (same contract as nasg::guide_shade)
template <int N, class RawFn>
__device__ __forceinline__ void guide_shade(RawFn raw, float4 xi, float b, float4 dbsdf, float4 dnee, float4 &o0,
                                            float4 &o1) {
    double w[N], c, c_sig;
    ref::decode_header<N>(raw, w, c, c_sig);
    const double ce = (double)b * c;
    const bool tech = (double)dbsdf.w < ce;
    V3 v = {(double)dbsdf.x, (double)dbsdf.y, (double)dbsdf.z};
    double pv;
    if (tech) {
        float cc;
        const float4 s = ref::guide_sample<N>(raw, xi, cc);
        v = {(double)s.x, (double)s.y, (double)s.z};
        pv = (double)s.w;
    } else {
        pv = ref::mixture_pdf<N>(raw, w, v);
    }
    const V3 vn = {(double)dnee.x, (double)dnee.y, (double)dnee.z};
    const double pn = dnee.w > 0.f ? ref::mixture_pdf<N>(raw, w, vn) : 0.0;
    o0 = make_float4((float)v.x, (float)v.y, (float)v.z, (float)pv);
    o1 = make_float4((float)pn, (float)ce, tech ? 1.f : 0.f, (float)c);
}

// ---- lane-parallel forms for the fp32 query kernel: P consecutive lanes per
// query, each decoding N/P lobes for the mixture pdf (combined by shuffles, so
// the sum is pairwise instead of in lobe order: equal to double rounding).  The
// lobe pick and the sample are computed redundantly by every lane of the group
// (identical values).  All 32 lanes must call them (full-mask shuffles).
template <int N>
__device__ __forceinline__ double wsel(const double (&w)[N], int i) {  // w[i], runtime i, no local memory
    double x = w[0];
#pragma unroll
    for (int j = 1; j < N; ++j) x = i == j ? w[j] : x;
    return x;
}

template <int N, int P, class RawFn>
__device__ __forceinline__ double mixture_pdf_par(RawFn raw, const double (&w)[N], const V3 &v, int part) {
    constexpr int NL = N / P;
    double pdf = 0.0;
#pragma unroll
    for (int k = 0; k < NL; ++k) {
        const int i = part * NL + k;
        float r[7];
        load_lobe<N>(raw, i, r);
        Lobe L;
        decode_lobe(r, L);
        pdf += wsel<N>(w, i) * lobe_pdf(L, v);
    }
#pragma unroll
    for (int o = 1; o < P; o <<= 1) pdf += __shfl_xor_sync(0xffffffffu, pdf, o);
    return pdf;
}

template <int N, int P, class RawFn>
__device__ __forceinline__ float4 guide_sample_par(RawFn raw, float4 xi, int part, float &c_out) {
    double w[N], c, c_sig;
    decode_header<N>(raw, w, c, c_sig);
    c_out = (float)c;
    int pick = N - 1;
    double acc = 0.0;
    bool found = false;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        acc += w[i];
        const bool hit = !found && (double)xi.x < acc;
        pick = hit ? i : pick;
        found |= hit;
    }
    float rs[7];
    load_lobe<N>(raw, pick, rs);
    Lobe Ls;
    decode_lobe(rs, Ls);
    const V3 v = lobe_sample(Ls, (double)xi.y, (double)xi.z, (double)xi.w);
    const double pdf = mixture_pdf_par<N, P>(raw, w, v, part);
    return make_float4((float)v.x, (float)v.y, (float)v.z, (float)pdf);
}

template <int N, int P, class RawFn>
__device__ __forceinline__ float2 guide_pdf_par(RawFn raw, float3 dir, float b, float bsdf_pdf, int part) {
    double w[N], c, c_sig;
    decode_header<N>(raw, w, c, c_sig);
    const V3 v = {(double)dir.x, (double)dir.y, (double)dir.z};
    const double pdf = mixture_pdf_par<N, P>(raw, w, v, part);
    const double ce = (double)b * c;
    const double guided = ce <= 0.0 ? (double)bsdf_pdf : ce * pdf + (1.0 - ce) * (double)bsdf_pdf;
    return make_float2((float)pdf, (float)guided);
}

// ---- KL gradient (guiding.cpp:96-176, sphdist.cpp:200-274) -----------------------
struct Euler {
    double ct, sp, cp, st, ctau;
};

__device__ __forceinline__ Euler euler_from_frame(const Lobe &f) {  // sphdist.cpp:33-57
    Euler e;
    e.ct = fmin(fmax(f.z.z, -1.0), 1.0);
    const double s = sqrt(fmax(0.0, 1.0 - e.ct * e.ct));
    if (s > 1e-9) {
        e.cp = f.z.x / s;
        e.sp = f.z.y / s;
        renorm_pair(e.sp, e.cp);
        e.ctau = -f.x.z / s;
        e.st = f.x.y * e.cp - f.x.x * e.sp;
        renorm_pair(e.st, e.ctau);
    } else {
        e.sp = 0.0;
        e.cp = 1.0;
        e.ctau = e.ct > 0.0 ? f.x.x : -f.x.x;
        e.st = f.x.y;
        renorm_pair(e.st, e.ctau);
    }
    return e;
}

struct PGrad {
    double d[7];  // ct, sp, cp, st, ctau, lambda, a
};

// nasg_grad_logpdf with q = mixture_pdf(m, v) supplied (sphdist.cpp:200-274)
__device__ __forceinline__ PGrad grad_logpdf(const Lobe &c, double wi, const V3 &v, double q) {
    PGrad g;
#pragma unroll
    for (int k = 0; k < 7; ++k) g.d[k] = 0.0;
    const double dz = dot(v, c.z);
    if (fabs(dz) > 1.0 - 1e-6) return g;
    if (!(q > 0.0) || !isfinite(q)) return g;
    const LEval e = eval_lobe(c, v);
    const double log_g = 2.0 * c.lambda * (e.u_pow_m - 1.0) + e.beta * e.log_u;
    const double K = norm_const(c);
    const double r = wi * exp(log_g) / K / q;
    const double expm2l = exp(-2.0 * c.lambda);
    const double dlogK_dl = 2.0 * expm2l / (1.0 - expm2l) - 1.0 / c.lambda;
    const double dlogK_da = -0.5 / (1.0 + c.a);
    const double dG_dbeta = (2.0 * c.lambda * e.u_pow_m + 1.0) * e.log_u;
    const double dG_du = 2.0 * c.lambda * e.m * pow(e.u, e.m - 1.0) + e.beta / e.u;
    const double dt2_ddz = 2.0 * e.dz * e.t2 / e.denom;
    const double dG_ddz = 0.5 * dG_du + dG_dbeta * c.a * dt2_ddz;
    const double dG_ddx = dG_dbeta * c.a * 2.0 * e.dx / e.denom;
    g.d[5] = r * (2.0 * (e.u_pow_m - 1.0) - dlogK_dl);
    g.d[6] = r * (e.t2 * dG_dbeta - dlogK_da);
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
    g.d[0] = r * g_ct;
    g.d[1] = r * g_sp;
    g.d[2] = r * g_cp;
    g.d[3] = r * g_st;
    g.d[4] = r * g_ctau;
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 7; ++k) ok &= isfinite(g.d[k]);
    if (!ok) {
#pragma unroll
        for (int k = 0; k < 7; ++k) g.d[k] = 0.0;
    }
    return g;
}

// kl_loss_gradient (guiding.cpp:108-165) + loss_surrogate (:167-176), one pass
// over lobes for q_mix.  put(col, g) receives float(g * gscale) for every
// packed column (pads 0), as out_grads(r,k) = float(grad[k] * inv) (:262-264).
template <int N, class RawFn, class PutFn>
__device__ __forceinline__ bool kl_grad_row(RawFn raw, const TrainRow &s, double b, double e, double gscale,
                                            PutFn put, double &loss) {
    constexpr int H = packed_header(N);
    loss = 0.0;
    if (s.p == 0.f) {
        static_for<0, H + 8 * N>([&](auto jc) { put(decltype(jc)::value, 0.f); });
        return true;
    }
    double w[N], c, c_sig;
    decode_header<N>(raw, w, c, c_sig);
    const V3 v = {(double)s.wi.x, (double)s.wi.y, (double)s.wi.z};
    const double q_mix = mixture_pdf<N>(raw, w, v);  // eval_blend :96-104
    const double c_eff = b * c;
    const double q_hat = c_eff * q_mix + (1.0 - c_eff) * (double)s.pbsdf;
    const bool usable = isfinite(q_mix) && q_mix > 1e-300 && isfinite(q_hat) && q_hat > 1e-300;
    if (!usable || !(s.q_s > 0.f)) {
        static_for<0, H + 8 * N>([&](auto jc) { put(decltype(jc)::value, 0.f); });
        loss = NAN;
        return false;
    }
    const double ws = (double)s.p / (double)s.q_s;
    const double mix_scale = e * (c_eff * q_mix / q_hat) + (1.0 - e);
    const double scale = -ws * mix_scale;
    bool finite = true;
    const double c_clamped = c != c_sig ? 0.0 : 1.0;
    const double dsig_c = c_sig * (1.0 - c_sig) * c_clamped;
    const double gc = -ws * e * b * (q_mix - (double)s.pbsdf) / q_hat * dsig_c;
    finite &= isfinite(gc);
    put(N, (float)(gc * gscale));
    static_for<N + 1, H>([&](auto jc) { put(decltype(jc)::value, 0.f); });
    static_for<0, N>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        float r[7];
        load_lobe<N>(raw, i, r);
        Lobe L;
        decode_lobe(r, L);
        const PGrad pg = grad_logpdf(L, w[i], v, q_mix);
        double dt[5] = {pg.d[0], pg.d[1], pg.d[2], pg.d[3], pg.d[4]};
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const double inv = L.pn[p] > 0.0 ? 1.0 / L.pn[p] : 0.0;
            dt[1 + 2 * p] *= inv;
            dt[2 + 2 * p] *= inv;
        }
        double go[8];
#pragma unroll
        for (int k = 0; k < 5; ++k) go[k] = scale * dt[k] * 2.0 * L.sig[k] * (1.0 - L.sig[k]);
        go[5] = L.lam_clamped ? 0.0 : scale * pg.d[5] * L.lambda;
        go[6] = L.a_clamped ? 0.0 : scale * pg.d[6] * L.a;
        go[7] = 0.0;
        const double pdf_i = lobe_pdf(L, v);
        const double r_i = w[i] * pdf_i / q_mix;
        const double gl = scale * (r_i - w[i]);
        finite &= isfinite(gl);
        put(i, (float)(gl * gscale));
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            finite &= isfinite(go[k]);
            put(H + 8 * i + k, (float)(go[k] * gscale));
        }
    });
    if (!finite) {
        static_for<0, H + 8 * N>([&](auto jc) { put(decltype(jc)::value, 0.f); });
        return false;
    }
    loss = -ws * (e * log(q_hat) + (1.0 - e) * log(q_mix));
    return true;
}


// kl_grad_row with P consecutive lanes per row (the fp32 trainer: 4 lanes x 64
// rows keep all 8 warps busy in the double-precision epilogue instead of 2).
// Lane `part` owns lobes [part N/P, (part + 1) N/P): their decode, pdf, grad
// log pdf and output columns; q_mix and the finiteness of the row's gradient
// are combined over the P lanes with shuffles (q_mix summed pairwise rather
// than in lobe order: the reference's value to double rounding).  Part 0 also
// writes the selection-probability column, the header padding and the loss.
// Every lane of the warp must call it (the shuffles use the full mask); rows
// the caller does not use pass p = 0.  Returns the row status as kl_grad_row.
template <int N, int P, class RawFn, class PutFn>
__device__ __forceinline__ bool kl_grad_row_par(RawFn raw, const TrainRow &s, double b, double e, double gscale,
                                                int part, PutFn put, double &loss) {
    static_assert(N % P == 0 && (P & (P - 1)) == 0 && P <= 32, "lobes must split evenly over a power-of-2 group");
    constexpr int H = packed_header(N), NL = N / P;
    const int i0 = part * NL;
    double w[N], c, c_sig;
    decode_header<N>(raw, w, c, c_sig);
    const V3 v = {(double)s.wi.x, (double)s.wi.y, (double)s.wi.z};
    auto lobe_of = [&](int i, Lobe &L) {  // runtime lobe index: logits read from the caller's tile
        float r[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) r[k] = raw(H + 8 * i + k);
        decode_lobe(r, L);
    };
    auto wsel = [&](int i) { return ref::wsel<N>(w, i); };
    double q_part = 0.0;
#pragma unroll 1
    for (int k = 0; k < NL; ++k) {
        Lobe L;
        lobe_of(i0 + k, L);
        q_part += wsel(i0 + k) * lobe_pdf(L, v);
    }
    double q_mix = q_part;
#pragma unroll
    for (int o = 1; o < P; o <<= 1) q_mix += __shfl_xor_sync(0xffffffffu, q_mix, o);
    const double c_eff = b * c;
    const double q_hat = c_eff * q_mix + (1.0 - c_eff) * (double)s.pbsdf;
    const bool live = s.p != 0.f;
    const bool usable = isfinite(q_mix) && q_mix > 1e-300 && isfinite(q_hat) && q_hat > 1e-300 && s.q_s > 0.f;
    const double ws = (double)s.p / (double)s.q_s;
    const double mix_scale = e * (c_eff * q_mix / q_hat) + (1.0 - e);
    const double scale = -ws * mix_scale;
    bool finite = true;
    const double c_clamped = c != c_sig ? 0.0 : 1.0;
    const double dsig_c = c_sig * (1.0 - c_sig) * c_clamped;
    const double gc = -ws * e * b * (q_mix - (double)s.pbsdf) / q_hat * dsig_c;
    if (part == 0) finite &= isfinite(gc);
    float gl_own[NL], go_own[NL][8];
#pragma unroll
    for (int k = 0; k < NL; ++k) {
        const int i = i0 + k;
        Lobe L;
        lobe_of(i, L);
        const double wi = wsel(i);
        const PGrad pg = grad_logpdf(L, wi, v, q_mix);
        double dt[5] = {pg.d[0], pg.d[1], pg.d[2], pg.d[3], pg.d[4]};
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const double inv = L.pn[p] > 0.0 ? 1.0 / L.pn[p] : 0.0;
            dt[1 + 2 * p] *= inv;
            dt[2 + 2 * p] *= inv;
        }
        double go[8];
#pragma unroll
        for (int kk = 0; kk < 5; ++kk) go[kk] = scale * dt[kk] * 2.0 * L.sig[kk] * (1.0 - L.sig[kk]);
        go[5] = L.lam_clamped ? 0.0 : scale * pg.d[5] * L.lambda;
        go[6] = L.a_clamped ? 0.0 : scale * pg.d[6] * L.a;
        go[7] = 0.0;
        const double r_i = wi * lobe_pdf(L, v) / q_mix;
        const double gl = scale * (r_i - wi);
        finite &= isfinite(gl);
        gl_own[k] = (float)(gl * gscale);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            finite &= isfinite(go[kk]);
            go_own[k][kk] = (float)(go[kk] * gscale);
        }
    }
#pragma unroll
    for (int o = 1; o < P; o <<= 1) finite &= __shfl_xor_sync(0xffffffffu, (int)finite, o) != 0;
    __syncwarp();  // the group's reads of shared header columns precede every lane's writes
    const bool emit = live && usable && finite;
#pragma unroll
    for (int k = 0; k < NL; ++k) {
        const int i = i0 + k;
        put(i, emit ? gl_own[k] : 0.f);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) put(H + 8 * i + kk, emit ? go_own[k][kk] : 0.f);
    }
    if (part == 0) {
        put(N, emit ? (float)(gc * gscale) : 0.f);
        for (int j = N + 1; j < H; ++j) put(j, 0.f);
    }
    loss = 0.0;
    if (!live) return true;
    if (!usable) {
        loss = NAN;
        return false;
    }
    if (!finite) return false;
    loss = -ws * (e * log(q_hat) + (1.0 - e) * log(q_mix));
    return true;
}

}  // namespace ref
}  // namespace nasg
