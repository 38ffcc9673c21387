// Device-side NASG math shared by every kernel (query, pdf, train).
//
// Restates, in fp32 with cancellation-free forms, the reference's double
// precision density code:
//   decode_full           guiding.cpp:15-77
//   frame_from_euler      sphdist.cpp:87-101 (Eq. 13)
//   eval_lobe/log_eval    sphdist.cpp:71-83, 133-140 (Eq. 10)
//   nasg_norm_const       sphdist.cpp:142-146 (Eq. 12)
//   nasg_sample           sphdist.cpp:159-181 (Appendix C)
//   mixture_sample        sphdist.cpp:183-198
//   mixture_pdf           sphdist.cpp:152-157
//   guided_pdf            guiding.cpp:81-85
//
// Raw-output layout.  The MLP's last layer is stored with its columns
// permuted ("packed") so one lobe's seven logits are contiguous (one
// 8-column TMEM/smem load per lobe):
//   cols [0, N)           mixture-weight logits   (reference raw[7N + i])
//   col  N                selection logit c        (reference raw[8N])
//   cols [N+1, H)         zero padding, H = round_up(N + 1, 16)
//   cols H + 8i + {0..4}  orientation logits       (reference raw[5i + k])
//   col  H + 8i + 5       lambda logit             (reference raw[5N + 2i])
//   col  H + 8i + 6       eccentricity logit       (reference raw[5N + 2i + 1])
//   col  H + 8i + 7       zero padding
// Packed width NP = H + 8N (80 for N = 8).
//
// Precision.  `Precise = true` (the fp32 path) projects directions onto the
// lobe frame in double so that 1 - v.z keeps full relative accuracy for
// lambda up to 3e3 (fp32 frames are only unit-norm to ~6e-8, which a
// lambda = 3e3 lobe amplifies to ~4e-4 in log pdf).  `Precise = false`
// (the bf16 tensor-core path, whose raw outputs already differ by ~1e-2) is
// pure fp32.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace nasg {

constexpr float kPiF = 3.14159265358979323846f;
constexpr float kLog2Pi = 1.8378770664093453f;  // log(2*pi)
constexpr float kLambdaMinF = 1e-3f;            // sphdist.hpp:13
constexpr float kLambdaMaxF = 3e3f;             // sphdist.hpp:14
constexpr float kEccMaxF = 3e3f;                // sphdist.hpp:15
constexpr float kSelMin = 0.01f, kSelMax = 0.99f;  // guiding.hpp:22-23

__host__ __device__ constexpr int packed_header(int n) { return ((n + 1 + 15) / 16) * 16; }
__host__ __device__ constexpr int packed_width(int n) { return packed_header(n) + 8 * n; }

// Packed column of reference raw index j (guiding.hpp:25-30 layout).
__host__ __device__ inline int packed_col(int j, int n) {
    const int H = packed_header(n);
    if (j < 5 * n) return H + 8 * (j / 5) + (j % 5);
    if (j < 7 * n) return H + 8 * ((j - 5 * n) / 2) + 5 + ((j - 5 * n) % 2);
    if (j < 8 * n) return j - 7 * n;
    return n;  // j == 8n
}

struct Lobe {
    float3 x, y, z;   // frame axes (fp32)
    float lambda, a;  // clamped sharpness / eccentricity
    float log_k;      // log of nasg_norm_const
    float one_m_emin; // 1 - exp(-2 lambda) = -expm1(-2 lambda)
    // decode intermediates needed by the KL gradient (guiding.hpp:34-42)
    float sig[5], sigm[5];   // sigmoid(raw) and 1 - sigmoid(raw), accurate
    float ct, st;            // cos/sin theta used by the frame
    float sp, cp, stau, ctau;  // renormalised pairs
    float pn_phi, pn_tau;    // pre-normalisation pair norms (0 => degenerate)
    bool lam_clamped, a_clamped;
    // double-precision axes for the Precise projection
    double zd0, zd1, zd2, xd0, xd1, xd2;
};

__device__ __forceinline__ float dot3(float3 a, float3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

__device__ __forceinline__ float3 cross3(float3 a, float3 b) {
    return make_float3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}

// Accurate sigmoid pair: s = 1/(1+e^-r), sm = 1 - s computed without cancellation.
__device__ __forceinline__ void sigmoid_pair(float r, float &s, float &sm) {
    if (r >= 0.f) {
        float e = __expf(-r);
        s = __frcp_rn(1.f + e);
        sm = e * s;
    } else {
        float e = __expf(r);
        sm = __frcp_rn(1.f + e);
        s = e * sm;
    }
}

// Decode one lobe from its seven packed logits: orientation (5), lambda, a.
// guiding.cpp:26-60 + sphdist.cpp:87-101 + sphdist.cpp:142-146.
// Precise variant: the decode itself in double, as the reference does
// (guiding.cpp:26-60 computes sigmoid, trig, frame, lambda and a in double
// from the float raw outputs), so the lobe frame agrees with the oracle to
// ~1e-16 and only the per-direction evaluation runs in fp32.
__device__ __forceinline__ void decode_lobe_double(const float r[7], Lobe &L) {
    double trig[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const double s = 1.0 / (1.0 + exp(-(double)r[k]));  // sigmoid guiding.cpp:9
        L.sig[k] = (float)s;
        L.sigm[k] = (float)(1.0 - s);
        trig[k] = s * 2.0 - 1.0;
    }
    double n1 = sqrt(trig[1] * trig[1] + trig[2] * trig[2]);
    if (n1 < 1e-6) { trig[1] = 0.0; trig[2] = 1.0; L.pn_phi = 0.f; }
    else { trig[1] /= n1; trig[2] /= n1; L.pn_phi = (float)n1; }
    double n2 = sqrt(trig[3] * trig[3] + trig[4] * trig[4]);
    if (n2 < 1e-6) { trig[3] = 0.0; trig[4] = 1.0; L.pn_tau = 0.f; }
    else { trig[3] /= n2; trig[4] /= n2; L.pn_tau = (float)n2; }
    const double ct = fmin(fmax(trig[0], -1.0), 1.0);
    const double st = sqrt(fmax(0.0, 1.0 - ct * ct));
    const double sp = trig[1], cp = trig[2], stau = trig[3], ctau = trig[4];
    L.zd0 = cp * st; L.zd1 = sp * st; L.zd2 = ct;
    L.xd0 = ct * cp * ctau - sp * stau;
    L.xd1 = ct * sp * ctau + cp * stau;
    L.xd2 = -st * ctau;
    const double yd0 = L.zd1 * L.xd2 - L.zd2 * L.xd1, yd1 = L.zd2 * L.xd0 - L.zd0 * L.xd2,
                 yd2 = L.zd0 * L.xd1 - L.zd1 * L.xd0;
    L.z = make_float3((float)L.zd0, (float)L.zd1, (float)L.zd2);
    L.x = make_float3((float)L.xd0, (float)L.xd1, (float)L.xd2);
    L.y = make_float3((float)yd0, (float)yd1, (float)yd2);
    L.ct = (float)ct; L.st = (float)st; L.sp = (float)sp; L.cp = (float)cp;
    L.stau = (float)stau; L.ctau = (float)ctau;
    const double lam = exp((double)r[5]), a = exp((double)r[6]);
    const double lc = fmin(fmax(lam, 1e-3), 3e3), ac = fmin(a, 3e3);
    L.lam_clamped = lc != lam;
    L.a_clamped = ac != a;
    L.lambda = (float)lc;
    L.a = (float)ac;
    const double ome = -expm1(-2.0 * lc);
    L.one_m_emin = (float)ome;
    L.log_k = (float)(1.8378770664093453 + log(ome) - log(lc) - 0.5 * log1p(ac));
}

template <bool Precise>
__device__ __forceinline__ void decode_lobe(const float r[7], Lobe &L) {
    if (Precise) {
        decode_lobe_double(r, L);
        return;
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) sigmoid_pair(r[k], L.sig[k], L.sigm[k]);
    // trig = 2 sigmoid - 1 = s - (1 - s)
    float ct = L.sig[0] - L.sigm[0];
    float sp = L.sig[1] - L.sigm[1], cp = L.sig[2] - L.sigm[2];
    float st_ = L.sig[3] - L.sigm[3], ctau = L.sig[4] - L.sigm[4];
    // pair renormalisation, degenerate (norm < 1e-6) -> (0, 1)  guiding.cpp:35-48
    float n1 = sqrtf(sp * sp + cp * cp);
    if (n1 < 1e-6f) { sp = 0.f; cp = 1.f; L.pn_phi = 0.f; }
    else { float i = __frcp_rn(n1); sp *= i; cp *= i; L.pn_phi = n1; }
    float n2 = sqrtf(st_ * st_ + ctau * ctau);
    if (n2 < 1e-6f) { st_ = 0.f; ctau = 1.f; L.pn_tau = 0.f; }
    else { float i = __frcp_rn(n2); st_ *= i; ctau *= i; L.pn_tau = n2; }
    // sin(theta) = sqrt(1 - ct^2) = 2 sqrt(s (1 - s))
    float sth = 2.f * sqrtf(L.sig[0] * L.sigm[0]);
    L.ct = ct; L.st = sth; L.sp = sp; L.cp = cp; L.stau = st_; L.ctau = ctau;
    L.z = make_float3(cp * sth, sp * sth, ct);
    L.x = make_float3(ct * cp * ctau - sp * st_, ct * sp * ctau + cp * st_, -sth * ctau);
    L.y = cross3(L.z, L.x);
    // lambda = clamp(e^r, 1e-3, 3e3), a = min(e^r, 3e3)  guiding.cpp:53-59
    float lam = expf(r[5]), a = expf(r[6]);
    L.lambda = fminf(fmaxf(lam, kLambdaMinF), kLambdaMaxF);
    L.a = fminf(a, kEccMaxF);
    L.lam_clamped = L.lambda != lam;
    L.a_clamped = L.a != a;
    // K = 2 pi (1 - e^{-2 lambda}) / (lambda sqrt(1 + a))  (eps = 0)
    L.one_m_emin = -expm1f(-2.f * L.lambda);
    L.log_k = kLog2Pi + logf(L.one_m_emin) - logf(L.lambda) - 0.5f * log1pf(L.a);
}

// Local-frame quantities of a direction: w = 1 - dz, q = 1 + dz, t2 = dx^2/(1-dz^2).
struct LocalDir {
    float w, q, t2, dz, dx;
    bool pole;  // |dz| > 1 - 1e-6: zero parameter gradient (sphdist.cpp:205)
};

template <bool Precise>
__device__ __forceinline__ LocalDir project(const Lobe &L, float3 v) {
    LocalDir d;
    if (Precise) {
        double dz = (double)v.x * L.zd0 + (double)v.y * L.zd1 + (double)v.z * L.zd2;
        double dx = (double)v.x * L.xd0 + (double)v.y * L.xd1 + (double)v.z * L.xd2;
        d.w = (float)(1.0 - dz);
        d.q = (float)(1.0 + dz);
        d.dz = (float)dz;
        d.dx = (float)dx;
        d.pole = fabs(dz) > 1.0 - 1e-6;
    } else {
        float dz = dot3(v, L.z);
        // use v -/+ z (orthogonal to x) for dx, and the half squared chord for w
        float s = dz >= 0.f ? 1.f : -1.f;
        float3 e = make_float3(v.x - s * L.z.x, v.y - s * L.z.y, v.z - s * L.z.z);
        float h = 0.5f * dot3(e, e);
        d.w = dz >= 0.f ? h : 2.f - h;
        d.q = dz >= 0.f ? 2.f - h : h;
        d.dz = dz;
        d.dx = dot3(e, L.x);
        d.pole = fminf(d.w, d.q) < 1e-6f;
    }
    float denom = fmaxf(d.w * d.q, 1e-12f);  // 1 - dz^2, sphdist.cpp:77
    d.t2 = fminf(fmaxf(d.dx * d.dx / denom, 0.f), 1.f);
    return d;
}

// log G of the lobe at a direction given by its local quantities (eps = 0):
// 2 lambda (u^m - 1) + beta log u, u = (1 + dz)/2, m = 1 + beta, beta = a t2.
// sphdist.cpp:133-140 with u^m - 1 = expm1(m log u), log u = log1p(-w/2).
__device__ __forceinline__ float lobe_log_g(const Lobe &L, float w, float q, float t2) {
    if (q <= 1e-12f) return -INFINITY;  // v = -z sentinel branch
    float log_u = w < 1.f ? log1pf(-0.5f * w) : logf(0.5f * q);
    log_u = fmaxf(log_u, -27.631021f);   // u >= 1e-12 clamp (log 1e-12)
    float beta = L.a * t2;
    float m = 1.f + beta;
    return 2.f * L.lambda * expm1f(m * log_u) + beta * log_u;
}

// nasg_sample (sphdist.cpp:159-181) in cancellation-free form.  Returns the
// world direction and, for the pdf of the same lobe, its local w, q, t2.
__device__ __forceinline__ float3 sample_lobe(const Lobe &L, float xi0, float xi1, float xi2,
                                              float &w_out, float &q_out, float &t2_out) {
    // ln s with s = e^{-2l} + xi0 (1 - e^{-2l}) = 1 - (1 - xi0)(1 - e^{-2l})
    float ln_s = log1pf(-(1.f - xi0) * L.one_m_emin);
    float ratio = ln_s / (2.f * L.lambda);  // in [-1, 0]
    float srho, crho;
    sincospif(xi1 - 0.5f, &srho, &crho);    // rho = (xi1 - 1/2) pi
    float expo = (1.f + L.a * srho * srho) / (1.f + L.a);
    float one_m_c, one_p_c;                 // 1 - cos(theta), 1 + cos(theta)
    if (ratio <= -1.f) {
        one_m_c = 2.f; one_p_c = 0.f;       // base clamped to 0 -> theta = pi
    } else {
        float lb = log1pf(ratio);           // log(base)
        float bp = expf(expo * lb);         // base^expo
        one_m_c = -2.f * expm1f(expo * lb);
        one_p_c = 2.f * bp;
        one_m_c = fminf(fmaxf(one_m_c, 0.f), 2.f);
    }
    float cth = 1.f - one_m_c;
    float sth = sqrtf(fmaxf(one_m_c * one_p_c, 0.f));
    // phi = atan2(sqrt(1+a) sin rho, cos rho) (+pi on the western chart):
    // take (cos phi, sin phi) by normalising instead of atan2/cos/sin.
    float st = sqrtf(1.f + L.a) * srho;
    float inv = rsqrtf(crho * crho + st * st);
    float cph = crho * inv, sph = st * inv;
    if (xi2 <= 0.5f) { cph = -cph; sph = -sph; }
    float a1 = sth * cph, a2 = sth * sph;
    w_out = one_m_c;
    q_out = one_p_c;
    t2_out = cph * cph;  // dx^2 / (1 - dz^2) with dx = sin(theta) cos(phi)
    return make_float3(L.x.x * a1 + L.y.x * a2 + L.z.x * cth,
                       L.x.y * a1 + L.y.y * a2 + L.z.y * cth,
                       L.x.z * a1 + L.y.z * a2 + L.z.z * cth);
}

// Softmax over the N weight logits and the clamped selection probability.
// guiding.cpp:62-75.
template <int N, class RawFn>
__device__ __forceinline__ void decode_header(RawFn raw, float (&w)[N], float &c, float &c_sig) {
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < N; ++i) mx = fmaxf(mx, raw(i));
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < N; ++i) { w[i] = __expf(raw(i) - mx); sum += w[i]; }
    float inv = __frcp_rn(sum);
#pragma unroll
    for (int i = 0; i < N; ++i) w[i] *= inv;
    float s, sm;
    sigmoid_pair(raw(N), s, sm);
    c_sig = s;
    c = fminf(fmaxf(s, kSelMin), kSelMax);
}

// Full query epilogue on one row of packed raw outputs: decode, inverse-CDF
// lobe select, sample, and mixture pdf at the sampled direction.
// mixture_sample sphdist.cpp:183-198.
template <int N, bool Precise, class RawFn>
__device__ __forceinline__ float4 guide_sample(RawFn raw, float4 xi, float &c_out) {
    constexpr int H = packed_header(N);
    float w[N], c, c_sig;
    decode_header<N>(raw, w, c, c_sig);
    c_out = c;
    // first i with xi_sel < cumulative weight, else N-1
    int pick = N - 1;
    bool found = false;
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        acc += w[i];
        bool hit = !found && xi.x < acc;
        pick = hit ? i : pick;
        found |= hit;
    }
    float rs[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) rs[k] = raw(H + 8 * pick + k);
    Lobe Ls;
    decode_lobe<false>(rs, Ls);
    float ws, qs, t2s;
    float3 v = sample_lobe(Ls, xi.y, xi.z, xi.w, ws, qs, t2s);
    float pdf = 0.f;
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        float r[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) r[k] = raw(H + 8 * i + k);
        Lobe L;
        decode_lobe<Precise>(r, L);
        float lg;
        if (i == pick) {
            lg = lobe_log_g(L, ws, qs, t2s);
        } else {
            LocalDir d = project<Precise>(L, v);
            lg = lobe_log_g(L, d.w, d.q, d.t2);
        }
        pdf += w[i] * expf(lg - L.log_k);
    }
    return make_float4(v.x, v.y, v.z, pdf);
}

// Mixture pdf and guided pdf at a given direction (guiding.cpp:81-85).
template <int N, bool Precise, class RawFn>
__device__ __forceinline__ float2 guide_pdf(RawFn raw, float3 v, float b, float bsdf_pdf) {
    constexpr int H = packed_header(N);
    float w[N], c, c_sig;
    decode_header<N>(raw, w, c, c_sig);
    float pdf = 0.f;
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        float r[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) r[k] = raw(H + 8 * i + k);
        Lobe L;
        decode_lobe<Precise>(r, L);
        LocalDir d = project<Precise>(L, v);
        pdf += w[i] * expf(lobe_log_g(L, d.w, d.q, d.t2) - L.log_k);
    }
    float ce = b * c;
    float guided = ce <= 0.f ? bsdf_pdf : ce * pdf + (1.f - ce) * bsdf_pdf;
    return make_float2(pdf, guided);
}

// d log K / d lambda = 2 e^{-2l}/(1 - e^{-2l}) - 1/l = coth(l) - 1 - 1/l
// (sphdist.cpp:217), with a series below l = 0.05 to avoid cancellation.
__device__ __forceinline__ float dlogk_dlambda(float l, float one_m_emin) {
    if (l < 0.05f) {
        float l2 = l * l;
        return -1.f + l * (1.f / 3.f - l2 * (1.f / 45.f - l2 * (2.f / 945.f)));
    }
    return 2.f * (1.f - one_m_emin) / one_m_emin - 1.f / l;
}

struct TrainRow {
    float3 wi;
    float p, q_s, pbsdf;
};

// One-sample KL gradient with respect to the packed raw outputs
// (kl_loss_gradient guiding.cpp:108-165 with nasg_grad_logpdf
// sphdist.cpp:200-274, restated in a single O(N) pass: q_mix and the lobe
// pdfs are computed once instead of once per lobe).  `put(col, g)` receives
// every packed column's gradient (pads get 0).  Returns false when the sample
// must be dropped; `loss` receives loss_surrogate (guiding.cpp:167-176).
template <int N, bool Precise, class RawFn, class PutFn>
__device__ __forceinline__ bool kl_grad_row(RawFn raw, const TrainRow &s, float b, float e,
                                            float gscale, PutFn put, float &loss) {
    constexpr int H = packed_header(N);
    loss = 0.f;
    if (s.p == 0.f) {  // valid cheap path: zero gradient (guiding.cpp:112)
        for (int j = 0; j < H + 8 * N; ++j) put(j, 0.f);
        return true;
    }
    float w[N], c, c_sig;
    decode_header<N>(raw, w, c, c_sig);
    float pdf[N];
    float q_mix = 0.f;
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        float r[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) r[k] = raw(H + 8 * i + k);
        Lobe L;
        decode_lobe<Precise>(r, L);
        LocalDir d = project<Precise>(L, s.wi);
        pdf[i] = expf(lobe_log_g(L, d.w, d.q, d.t2) - L.log_k);
        q_mix += w[i] * pdf[i];
    }
    const float c_eff = b * c;
    const float q_hat = c_eff * q_mix + (1.f - c_eff) * s.pbsdf;
    const bool usable = isfinite(q_mix) && q_mix > 0.f && isfinite(q_hat) && q_hat > 0.f;
    if (!usable || !(s.q_s > 0.f)) {  // eval_blend floor (guiding.cpp:101-102)
        for (int j = 0; j < H + 8 * N; ++j) put(j, 0.f);
        loss = __int_as_float(0x7fc00000);
        return false;
    }
    const float ws = s.p / s.q_s;
    const float mix_scale = e * (c_eff * q_mix / q_hat) + (1.f - e);
    const float scale = -ws * mix_scale * gscale;
    const float inv_q = 1.f / q_mix;
    bool finite = true;
    // header: softmax logits (r_i - A_i), selection logit (guiding.cpp:150-158)
    {
        const bool c_clamped = c != c_sig;
        const float dsig = c_clamped ? 0.f : c_sig * (1.f - c_sig);
        float gc = -ws * e * b * (q_mix - s.pbsdf) / q_hat * dsig * gscale;
        finite &= isfinite(gc);
        put(N, gc);
        for (int j = N + 1; j < H; ++j) put(j, 0.f);
    }
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        float r[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) r[k] = raw(H + 8 * i + k);
        Lobe L;
        decode_lobe<Precise>(r, L);
        LocalDir d = project<Precise>(L, s.wi);
        const float ri = w[i] * pdf[i] * inv_q;  // posterior responsibility
        float gl = scale * (ri - w[i]);
        finite &= isfinite(gl);
        put(i, gl);
        float g7[7] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // d log q_mix / d (ct, sp, cp, st, ctau, l, a)
        if (!d.pole && pdf[i] > 0.f) {
            const float lam = L.lambda, a = L.a;
            float log_u = d.w < 1.f ? log1pf(-0.5f * d.w) : logf(0.5f * d.q);
            log_u = fmaxf(log_u, -27.631021f);
            const float u = fmaxf(0.5f * d.q, 1e-12f);
            const float beta = a * d.t2, m = 1.f + beta;
            const float um1 = expm1f(m * log_u);  // u^m - 1
            const float um = um1 + 1.f;
            const float denom = fmaxf(d.w * d.q, 1e-12f);
            const float dG_dbeta = (2.f * lam * um + 1.f) * log_u;
            const float dG_du = 2.f * lam * m * (um / u) + beta / u;
            const float dt2_ddz = 2.f * d.dz * d.t2 / denom;
            const float dG_ddz = 0.5f * dG_du + dG_dbeta * a * dt2_ddz;
            const float dG_ddx = dG_dbeta * a * 2.f * d.dx / denom;
            g7[5] = ri * (2.f * um1 - dlogk_dlambda(lam, L.one_m_emin));
            g7[6] = ri * (d.t2 * dG_dbeta + 0.5f / (1.f + a));
            // axis Jacobians contracted with v (sphdist.cpp:229-252)
            const float ct = L.ct, st = fmaxf(L.st, 1e-9f), dst = -ct / st;
            const float vx = s.wi.x, vy = s.wi.y, vz = s.wi.z;
            const float cpvx_spvy = L.cp * vx + L.sp * vy;
            float g_ct = dG_ddz * (dst * cpvx_spvy + vz) + dG_ddx * (L.ctau * cpvx_spvy - dst * L.ctau * vz);
            float g_sp = dG_ddz * (st * vy) + dG_ddx * (-L.stau * vx + ct * L.ctau * vy);
            float g_cp = dG_ddz * (st * vx) + dG_ddx * (ct * L.ctau * vx + L.stau * vy);
            float g_st = dG_ddx * (-L.sp * vx + L.cp * vy);
            float g_ctau = dG_ddx * (ct * L.cp * vx + ct * L.sp * vy - st * vz);
            // (I - p p^T) projection of the unit pairs (sphdist.cpp:254-261)
            float ps = L.cp * (L.cp * g_sp - L.sp * g_cp), pc = L.sp * (L.sp * g_cp - L.cp * g_sp);
            g_sp = ps; g_cp = pc;
            ps = L.ctau * (L.ctau * g_st - L.stau * g_ctau); pc = L.stau * (L.stau * g_ctau - L.ctau * g_st);
            g_st = ps; g_ctau = pc;
            g7[0] = ri * g_ct; g7[1] = ri * g_sp; g7[2] = ri * g_cp; g7[3] = ri * g_st; g7[4] = ri * g_ctau;
            bool ok = true;
#pragma unroll
            for (int k = 0; k < 7; ++k) ok &= isfinite(g7[k]);
            if (!ok) {
#pragma unroll
                for (int k = 0; k < 7; ++k) g7[k] = 0.f;
            }
        }
        // chain through pair renormalisation and sigmoid*2-1 (guiding.cpp:126-142)
        const float inv1 = L.pn_phi > 0.f ? 1.f / L.pn_phi : 0.f;
        const float inv2 = L.pn_tau > 0.f ? 1.f / L.pn_tau : 0.f;
        const float scl[5] = {1.f, inv1, inv1, inv2, inv2};
        float go[8];
#pragma unroll
        for (int k = 0; k < 5; ++k) go[k] = scale * g7[k] * scl[k] * 2.f * L.sig[k] * L.sigm[k];
        go[5] = L.lam_clamped ? 0.f : scale * g7[5] * L.lambda;
        go[6] = L.a_clamped ? 0.f : scale * g7[6] * L.a;
        go[7] = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            finite &= isfinite(go[k]);
            put(H + 8 * i + k, go[k]);
        }
    }
    if (!finite) {
        for (int j = 0; j < H + 8 * N; ++j) put(j, 0.f);
        return false;
    }
    loss = -ws * (e * logf(q_hat) + (1.f - e) * logf(q_mix));
    return true;
}

}  // namespace nasg
