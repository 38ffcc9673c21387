// fp32 NASG epilogue of the bf16 tensor-core path (K3/K4), plus the packed
// raw-output layout shared by every kernel.
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
// The fp32 (FFMA) path instead uses the double restatement in
// nasg_refmath.cuh, exactly as the reference computes after its float MLP.
//
// Stable forms: 1 - v.z = |v - z|^2 / 2 (and 1 + v.z = |v + z|^2 / 2),
// dx = (v -/+ z).x, log u = log1p(-w/2), u^m - 1 = expm1(m log u); the
// sampler builds (cos phi, sin phi) by normalising (cos rho, sqrt(1+a) sin rho)
// instead of atan2/cos/sin, and 1 -/+ cos(theta) from expm1/exp of the same
// logarithm.  The sampled lobe's pdf uses its exact local coordinates.
//
// Raw-output layout.  The MLP's last layer is stored with its columns
// permuted ("packed") so one lobe's seven logits are contiguous:
//   cols [0, N)           mixture-weight logits   (reference raw[7N + i])
//   col  N                selection logit c        (reference raw[8N])
//   cols [N+1, H)         zero padding, H = round_up(N + 1, 16)
//   cols H + 8i + {0..4}  orientation logits       (reference raw[5i + k])
//   col  H + 8i + 5       lambda logit             (reference raw[5N + 2i])
//   col  H + 8i + 6       eccentricity logit       (reference raw[5N + 2i + 1])
//   col  H + 8i + 7       zero padding
// Packed width NP = H + 8N (80 for N = 8).
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "nasg_internal.h"  // packed_header / packed_width

namespace nasg {

constexpr float kLog2Pi = 1.8378770664093453f;  // log(2*pi)
constexpr float kLambdaMinF = 1e-3f;            // sphdist.hpp:13
constexpr float kLambdaMaxF = 3e3f;             // sphdist.hpp:14
constexpr float kEccMaxF = 3e3f;                // sphdist.hpp:15
constexpr float kSelMin = 0.01f, kSelMax = 0.99f;  // guiding.hpp:22-23


// Packed column of reference raw index j (guiding.hpp:25-30 layout).
__host__ __device__ constexpr int packed_col(int j, int n) {
    const int H = packed_header(n);
    if (j < 5 * n) return H + 8 * (j / 5) + (j % 5);
    if (j < 7 * n) return H + 8 * ((j - 5 * n) / 2) + 5 + ((j - 5 * n) % 2);
    if (j < 8 * n) return j - 7 * n;
    return n;  // j == 8n
}

// Compile-time loop: lets lobe loops index register-resident raw outputs.
template <int I, int N, class F>
__device__ __forceinline__ void static_for(F &&f) {
    if constexpr (I < N) {
        f(std::integral_constant<int, I>{});
        static_for<I + 1, N>(f);
    }
}

// One recorded training sample as the KL epilogue needs it.
struct TrainRow {
    float3 wi;
    float p, q_s, pbsdf;
};

struct Lobe {
    float3 x, y, z;    // frame axes
    float lambda, a;   // clamped sharpness / eccentricity
    float log_k;       // log nasg_norm_const
    float one_m_emin;  // 1 - exp(-2 lambda)
};

__device__ __forceinline__ float dot3(float3 a, float3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

// ---- fast primitives (MUFU + short polynomials), accurate where the NASG
// formulas need relative accuracy ------------------------------------------------
__device__ __forceinline__ float rcp_fast(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float sqrt_fast(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// Branch-free select: both inputs are computed, so a lane-divergent choice
// between two short formulas does not split the warp into two passes.
__device__ __forceinline__ float sel(bool c, float a, float b) {
    float r;
    asm("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\tselp.f32 %0, %1, %2, p;\n\t}"
        : "=f"(r)
        : "f"(a), "f"(b), "r"((int)c));
    return r;
}

// log u for u = 1 - w/2 = q/2 (w = 1 - dz, q = 1 + dz from lobe_local): the
// log1p series below w = 1/2 (u near 1, where log(q/2) would cancel), MUFU.LG2
// of q/2 above it (u <= 3/4, relative error ~1e-7): one logarithm per call.
__device__ __forceinline__ float log_u_of(float w, float q) {
    const float x = -0.5f * fminf(w, 0.5f);
    const float sx = x * rcp_fast(2.f + x), s2 = sx * sx;
    const float ser = 2.f * sx * fmaf(s2, fmaf(s2, fmaf(s2, 1.f / 7.f, 1.f / 5.f), 1.f / 3.f), 1.f);
    return sel(w < 0.5f, ser, __logf(0.5f * q));
}

// log1p(x), x > -1: 2 atanh(x / (2 + x)) series for |x| < 1/4 (s^2 <= 0.0204,
// so the dropped s^8/9 term is < 2e-8 relative), log(1 + x) from MUFU.LG2
// otherwise (|log| > 0.22 there).
__device__ __forceinline__ float log1p_fast(float x) {
    const float sx = x * rcp_fast(2.f + x), s2 = sx * sx;
    const float ser = 2.f * sx * fmaf(s2, fmaf(s2, fmaf(s2, 1.f / 7.f, 1.f / 5.f), 1.f / 3.f), 1.f);
    return sel(fabsf(x) < 0.25f, ser, __logf(1.f + x));
}
// expm1(y): degree-6 Taylor polynomial for |y| < 1/4 (truncation < 5e-8
// relative), exp(y) - 1 from MUFU.EX2 otherwise (|result| > 0.22 there, so
// the EX2 error stays < 5e-7 relative).
__device__ __forceinline__ float expm1_fast(float y) {
    float p = fmaf(y, 1.f / 720.f, 1.f / 120.f);
    p = fmaf(p, y, 1.f / 24.f);
    p = fmaf(p, y, 1.f / 6.f);
    p = fmaf(p, y, 0.5f);
    p = fmaf(p, y, 1.f);
    return sel(fabsf(y) < 0.25f, p * y, __expf(y) - 1.f);
}

// s = 1/(1+e^-r) and 1 - s, both without cancellation.
__device__ __forceinline__ void sigmoid_pair(float r, float &s, float &sm) {
    const float e = __expf(-fabsf(r));
    const float big = rcp_fast(1.f + e), small = e * big;
    s = r >= 0.f ? big : small;
    sm = r >= 0.f ? small : big;
}

// 2 sigmoid(r) - 1 = tanh(r/2) = sign(r) (1 - e) / (1 + e) with e = exp(-|r|).
// A renormalised (sin, cos) pair only needs its direction, so both entries are
// scaled by (1 + e_a)(1 + e_b) and no reciprocal is taken; the degenerate-pair
// test (norm < 1e-6, sphdist.cpp:15-25) is applied to the unscaled norm.
__device__ __forceinline__ void tanh_half_pair(float ra, float rb, float &a, float &b, float &scale2) {
    const float ea = __expf(-fabsf(ra)), eb = __expf(-fabsf(rb));
    const float pa = 1.f + ea, pb = 1.f + eb;
    a = copysignf((1.f - ea) * pb, ra);
    b = copysignf((1.f - eb) * pa, rb);
    scale2 = (pa * pb) * (pa * pb);
}

// decode_full for one lobe (guiding.cpp:26-60) + frame_from_euler.
__device__ __forceinline__ void decode_lobe(const float r[7], Lobe &L) {
    const float e0 = __expf(-fabsf(r[0])), i0 = rcp_fast(1.f + e0);
    const float ct = copysignf((1.f - e0) * i0, r[0]);  // 2 sigmoid - 1
    const float sth = 2.f * sqrt_fast(e0) * i0;          // sqrt(1 - ct^2) = 2 sqrt(s (1 - s))
    float sp, cp, st, ctau, k1, k2;
    tanh_half_pair(r[1], r[2], sp, cp, k1);
    tanh_half_pair(r[3], r[4], st, ctau, k2);
    const float n1 = sp * sp + cp * cp, n2 = st * st + ctau * ctau;
    const bool d1 = n1 < 1e-12f * k1, d2 = n2 < 1e-12f * k2;  // degenerate pair -> (0, 1)
    const float i1 = rsqrtf(d1 ? 1.f : n1), i2 = rsqrtf(d2 ? 1.f : n2);
    sp = d1 ? 0.f : sp * i1;
    cp = d1 ? 1.f : cp * i1;
    st = d2 ? 0.f : st * i2;
    ctau = d2 ? 1.f : ctau * i2;
    L.z = make_float3(cp * sth, sp * sth, ct);
    L.x = make_float3(ct * cp * ctau - sp * st, ct * sp * ctau + cp * st, -sth * ctau);
    L.y = make_float3(L.z.y * L.x.z - L.z.z * L.x.y, L.z.z * L.x.x - L.z.x * L.x.z, L.z.x * L.x.y - L.z.y * L.x.x);
    L.lambda = fminf(fmaxf(__expf(r[5]), kLambdaMinF), kLambdaMaxF);
    L.a = fminf(__expf(r[6]), kEccMaxF);
    L.one_m_emin = -expm1_fast(-2.f * L.lambda);
    // log K = log 2pi + log((1 - e^{-2l}) / l) - log(1 + a) / 2  (absolute error ~1e-7)
    L.log_k = kLog2Pi + __logf(L.one_m_emin * rcp_fast(L.lambda)) - 0.5f * __logf(1.f + L.a);
}

// log G at v (sphdist.cpp:133-140), from local w = 1 - dz, q = 1 + dz, t2.
__device__ __forceinline__ float lobe_log_g(const Lobe &L, float w, float q, float t2) {
    float log_u = log_u_of(w, q);
    log_u = fmaxf(log_u, -27.631021f);  // u >= 1e-12
    const float beta = L.a * t2;
    const float lg = 2.f * L.lambda * expm1_fast((1.f + beta) * log_u) + beta * log_u;
    return q <= 1e-12f ? -INFINITY : lg;  // v = -z sentinel
}

// lobe-local coordinates of v: w = 1 - dz, q = 1 + dz (cancellation-free) and t2
__device__ __forceinline__ void lobe_local(const Lobe &L, float3 v, float &w, float &q, float &t2) {
    const float dz = dot3(v, L.z);
    const float sg = dz >= 0.f ? 1.f : -1.f;
    const float3 e = make_float3(v.x - sg * L.z.x, v.y - sg * L.z.y, v.z - sg * L.z.z);
    const float h = 0.5f * dot3(e, e);
    w = dz >= 0.f ? h : 2.f - h;
    q = dz >= 0.f ? 2.f - h : h;
    const float dx = dot3(e, L.x);
    t2 = fminf(fmaxf(dx * dx * rcp_fast(fmaxf(w * q, 1e-12f)), 0.f), 1.f);
}

__device__ __forceinline__ float lobe_log_g_at(const Lobe &L, float3 v) {
    float w, q, t2;
    lobe_local(L, v, w, q, t2);
    return lobe_log_g(L, w, q, t2);
}

// nasg_sample (sphdist.cpp:159-181); also returns the lobe-local w, q, t2.
__device__ __forceinline__ float3 sample_lobe(const Lobe &L, float xi0, float xi1, float xi2, float &w_out,
                                              float &q_out, float &t2_out) {
    const float ln_s = log1p_fast(-(1.f - xi0) * L.one_m_emin);  // s = 1 - (1-xi0)(1-e^-2l)
    const float ratio = fmaxf(ln_s * rcp_fast(2.f * L.lambda), -1.f);  // in [-1, 0]
    float srho, crho;
    __sincosf((xi1 - 0.5f) * 3.14159265358979f, &srho, &crho);  // rho = (xi1 - 1/2) pi
    const float expo = (1.f + L.a * srho * srho) * rcp_fast(1.f + L.a);
    float one_m_c = 2.f, one_p_c = 0.f;  // base clamped to 0 -> theta = pi
    if (ratio > -1.f) {
        const float el = expo * log1p_fast(ratio);
        one_m_c = fminf(fmaxf(-2.f * expm1_fast(el), 0.f), 2.f);
        one_p_c = 2.f * __expf(el);
    }
    const float cth = 1.f - one_m_c;
    const float sth = sqrt_fast(fmaxf(one_m_c * one_p_c, 0.f));
    const float st = sqrt_fast(1.f + L.a) * srho;  // phi = atan2(sqrt(1+a) sin rho, cos rho)
    const float inv = rsqrtf(crho * crho + st * st);
    float cph = crho * inv, sph = st * inv;
    if (xi2 <= 0.5f) { cph = -cph; sph = -sph; }  // western chart: phi + pi
    const float a1 = sth * cph, a2 = sth * sph;
    w_out = one_m_c;
    q_out = one_p_c;
    t2_out = cph * cph;
    return make_float3(L.x.x * a1 + L.y.x * a2 + L.z.x * cth, L.x.y * a1 + L.y.y * a2 + L.z.y * cth,
                       L.x.z * a1 + L.y.z * a2 + L.z.z * cth);
}

// Softmax over the N weight logits, clamped selection probability (guiding.cpp:62-75).
template <int N, class RawFn>
__device__ __forceinline__ void decode_header(RawFn raw, float (&w)[N], float &c) {
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < N; ++i) mx = fmaxf(mx, raw(i));
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        w[i] = __expf(raw(i) - mx);
        sum += w[i];
    }
    const float inv = __frcp_rn(sum);
#pragma unroll
    for (int i = 0; i < N; ++i) w[i] *= inv;
    float s, sm;
    sigmoid_pair(raw(N), s, sm);
    c = fminf(fmaxf(s, kSelMin), kSelMax);
}

template <int N, class RawFn>
__device__ __forceinline__ void lobe_logits(RawFn raw, int i, float (&r)[7]) {
    constexpr int H = packed_header(N);
#pragma unroll
    for (int k = 0; k < 7; ++k) r[k] = raw(H + 8 * i + k);
}

// decode + inverse-CDF lobe pick + sample + mixture pdf at the sample
// (infer_guide's decode, mixture_sample sphdist.cpp:183-198).
// The epilogues read the header through hraw(j) (j <= N) and each lobe's seven
// logits through lobe7(i, r) with a compile-time i: from a register array of the
// packed row (RawFn forms below), or streamed lobe by lobe from tensor memory by
// the 32-lobe tensor-core query, whose 304-column row does not fit in registers.
template <int N, class HdrFn, class Lobe7Fn>
__device__ __forceinline__ float4 guide_sample_src(HdrFn raw, Lobe7Fn lobe7, float4 xi, float &c_out) {
    float w[N];
    decode_header<N>(raw, w, c_out);
    int pick = N - 1;
    bool found = false;
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        acc += w[i];
        const bool hit = !found && xi.x < acc;
        pick = hit ? i : pick;
        found |= hit;
    }
    float rs[7];
    static_for<0, N>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        float r[7];
        lobe7(i, r);
#pragma unroll
        for (int k = 0; k < 7; ++k) rs[k] = (i == 0 || i == pick) ? r[k] : rs[k];
    });
    Lobe Ls;
    decode_lobe(rs, Ls);
    float ws, qs, t2s;
    const float3 v = sample_lobe(Ls, xi.y, xi.z, xi.w, ws, qs, t2s);
    float pdf = 0.f;
    static_for<0, N>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        float r[7];
        lobe7(i, r);
        Lobe L;
        decode_lobe(r, L);
        // the picked lobe uses the sampler's exact local coordinates; selecting
        // the inputs (not the evaluation) keeps one log G per lobe per lane
        float wl, ql, t2l;
        lobe_local(L, v, wl, ql, t2l);
        const bool me = i == pick;
        const float lg = lobe_log_g(L, sel(me, ws, wl), sel(me, qs, ql), sel(me, t2s, t2l));
        pdf += w[i] * __expf(lg - L.log_k);
    });
    return make_float4(v.x, v.y, v.z, pdf);
}
template <int N, class RawFn>
__device__ __forceinline__ float4 guide_sample(RawFn raw, float4 xi, float &c_out) {
    return guide_sample_src<N>(raw, [&](int i, float (&r)[7]) { lobe_logits<N>(raw, i, r); }, xi, c_out);
}

// mixture_pdf and guided_pdf at a given direction (guiding.cpp:81-85).
template <int N, class HdrFn, class Lobe7Fn>
__device__ __forceinline__ float2 guide_pdf_src(HdrFn raw, Lobe7Fn lobe7, float3 v, float b, float bsdf_pdf) {
    float w[N], c;
    decode_header<N>(raw, w, c);
    float pdf = 0.f;
    static_for<0, N>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        float r[7];
        lobe7(i, r);
        Lobe L;
        decode_lobe(r, L);
        pdf += w[i] * __expf(lobe_log_g_at(L, v) - L.log_k);
    });
    const float ce = b * c;
    return make_float2(pdf, ce <= 0.f ? bsdf_pdf : ce * pdf + (1.f - ce) * bsdf_pdf);
}
template <int N, class RawFn>
__device__ __forceinline__ float2 guide_pdf(RawFn raw, float3 v, float b, float bsdf_pdf) {
    return guide_pdf_src<N>(raw, [&](int i, float (&r)[7]) { lobe_logits<N>(raw, i, r); }, v, b, bsdf_pdf);
}

// Guided scattering at one path vertex (SPEC tracer trace_path; guided_pdf
// guiding.cpp:81-85): c' = b c; with probability c' (xi_t = dbsdf.w < c') the
// direction is the mixture sample (mixture_sample sphdist.cpp:183-198), else the
// caller's BSDF sample dbsdf.xyz.  One pass over the lobes evaluates the
// mixture pdf at the chosen direction and at the NEE direction dnee.xyz (the
// NEE pdf comes from the same network evaluation).
//   o0 = (dir, q_mix(dir)),  o1 = (q_mix(nee) or 0 if dnee.w <= 0, c', guided ? 1 : 0, c)
template <int N, class HdrFn, class Lobe7Fn>
__device__ __forceinline__ void guide_shade_src(HdrFn raw, Lobe7Fn lobe7, float4 xi, float b, float4 dbsdf,
                                                float4 dnee, float4 &o0, float4 &o1) {
    float w[N], c;
    decode_header<N>(raw, w, c);
    const float ce = b * c;
    const bool tech = dbsdf.w < ce;
    int pick = N - 1;
    bool found = false;
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        acc += w[i];
        const bool hit = !found && xi.x < acc;
        pick = hit ? i : pick;
        found |= hit;
    }
    float rs[7];
    static_for<0, N>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        float r[7];
        lobe7(i, r);
#pragma unroll
        for (int k = 0; k < 7; ++k) rs[k] = (i == 0 || i == pick) ? r[k] : rs[k];
    });
    Lobe Ls;
    decode_lobe(rs, Ls);
    float ws, qs, t2s;
    const float3 vm = sample_lobe(Ls, xi.y, xi.z, xi.w, ws, qs, t2s);
    const float3 v = make_float3(sel(tech, vm.x, dbsdf.x), sel(tech, vm.y, dbsdf.y), sel(tech, vm.z, dbsdf.z));
    const float3 vn = make_float3(dnee.x, dnee.y, dnee.z);
    float pv = 0.f, pn = 0.f;
    static_for<0, N>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        float r[7];
        lobe7(i, r);
        Lobe L;
        decode_lobe(r, L);
        float wl, ql, t2l;
        lobe_local(L, v, wl, ql, t2l);
        const bool me = tech && i == pick;
        pv += w[i] * __expf(lobe_log_g(L, sel(me, ws, wl), sel(me, qs, ql), sel(me, t2s, t2l)) - L.log_k);
        lobe_local(L, vn, wl, ql, t2l);
        pn += w[i] * __expf(lobe_log_g(L, wl, ql, t2l) - L.log_k);
    });
    o0 = make_float4(v.x, v.y, v.z, pv);
    o1 = make_float4(dnee.w > 0.f ? pn : 0.f, ce, tech ? 1.f : 0.f, c);
}
template <int N, class RawFn>
__device__ __forceinline__ void guide_shade(RawFn raw, float4 xi, float b, float4 dbsdf, float4 dnee, float4 &o0,
                                            float4 &o1) {
    guide_shade_src<N>(raw, [&](int i, float (&r)[7]) { lobe_logits<N>(raw, i, r); }, xi, b, dbsdf, dnee, o0, o1);
}

// Two-warpgroup forms (the split-lobe tensor-core query): warpgroup pt = 0 / 1
// owns lobes [pt N/2, pt N/2 + N/2) of the same row.  Both decode the header and
// the pick; the owner of the picked lobe passes its logits to the other
// (xc.picked), both sample from them, each sums its own lobes' pdf terms and
// part 1's sums reach part 0 (xc.to0).  Part 0's return value is the result (the
// pdf sums are (lobes of part 0) + (lobes of part 1)).  xc is the kernel's
// exchange between the two warpgroups (through tensor memory).
template <int N>
__device__ __forceinline__ bool own_lobe(int i, int pt) { return (i < N / 2) == (pt == 0); }

template <int N>
__device__ __forceinline__ int pick_lobe(const float (&w)[N], float xs) {
    int pick = N - 1;
    bool found = false;
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        acc += w[i];
        const bool hit = !found && xs < acc;
        pick = hit ? i : pick;
        found |= hit;
    }
    return pick;
}

template <int N, class Lobe7Fn, class Xchg>
__device__ __forceinline__ void share_picked(Lobe7Fn lobe7, int pick, int pt, Xchg &xc, float (&rs)[7]) {
#pragma unroll
    for (int k = 0; k < 7; ++k) rs[k] = 0.f;
    static_for<0, N>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        if (own_lobe<N>(i, pt)) {
            float r[7];
            lobe7(i, r);
#pragma unroll
            for (int k = 0; k < 7; ++k) rs[k] = i == pick ? r[k] : rs[k];
        }
    });
    xc.picked(rs, own_lobe<N>(pick, pt));
}

template <int N, class HdrFn, class Lobe7Fn, class Xchg>
__device__ __forceinline__ float4 guide_sample_pair(HdrFn raw, Lobe7Fn lobe7, float4 xi, float &c_out, int pt, Xchg &xc) {
    float w[N];
    decode_header<N>(raw, w, c_out);
    const int pick = pick_lobe<N>(w, xi.x);
    float rs[7];
    share_picked<N>(lobe7, pick, pt, xc, rs);
    Lobe Ls;
    decode_lobe(rs, Ls);
    float ws, qs, t2s;
    const float3 v = sample_lobe(Ls, xi.y, xi.z, xi.w, ws, qs, t2s);
    float pdf = 0.f;
    static_for<0, N>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        if (own_lobe<N>(i, pt)) {
            float r[7];
            lobe7(i, r);
            Lobe L;
            decode_lobe(r, L);
            float wl, ql, t2l;
            lobe_local(L, v, wl, ql, t2l);
            const bool me = i == pick;
            const float lg = lobe_log_g(L, sel(me, ws, wl), sel(me, qs, ql), sel(me, t2s, t2l));
            pdf += w[i] * __expf(lg - L.log_k);
        }
    });
    float dummy = 0.f;
    xc.to0(pdf, dummy);
    return make_float4(v.x, v.y, v.z, pdf);
}

template <int N, class HdrFn, class Lobe7Fn, class Xchg>
__device__ __forceinline__ float2 guide_pdf_pair(HdrFn raw, Lobe7Fn lobe7, float3 v, float b, float bsdf_pdf, int pt,
                                                 Xchg &xc) {
    float w[N], c;
    decode_header<N>(raw, w, c);
    float pdf = 0.f;
    static_for<0, N>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        if (own_lobe<N>(i, pt)) {
            float r[7];
            lobe7(i, r);
            Lobe L;
            decode_lobe(r, L);
            pdf += w[i] * __expf(lobe_log_g_at(L, v) - L.log_k);
        }
    });
    float dummy = 0.f;
    xc.to0(pdf, dummy);
    const float ce = b * c;
    return make_float2(pdf, ce <= 0.f ? bsdf_pdf : ce * pdf + (1.f - ce) * bsdf_pdf);
}

template <int N, class HdrFn, class Lobe7Fn, class Xchg>
__device__ __forceinline__ void guide_shade_pair(HdrFn raw, Lobe7Fn lobe7, float4 xi, float b, float4 dbsdf,
                                                 float4 dnee, float4 &o0, float4 &o1, int pt, Xchg &xc) {
    float w[N], c;
    decode_header<N>(raw, w, c);
    const float ce = b * c;
    const bool tech = dbsdf.w < ce;
    const int pick = pick_lobe<N>(w, xi.x);
    float rs[7];
    share_picked<N>(lobe7, pick, pt, xc, rs);
    Lobe Ls;
    decode_lobe(rs, Ls);
    float ws, qs, t2s;
    const float3 vm = sample_lobe(Ls, xi.y, xi.z, xi.w, ws, qs, t2s);
    const float3 v = make_float3(sel(tech, vm.x, dbsdf.x), sel(tech, vm.y, dbsdf.y), sel(tech, vm.z, dbsdf.z));
    const float3 vn = make_float3(dnee.x, dnee.y, dnee.z);
    float pv = 0.f, pn = 0.f;
    static_for<0, N>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        if (own_lobe<N>(i, pt)) {
            float r[7];
            lobe7(i, r);
            Lobe L;
            decode_lobe(r, L);
            float wl, ql, t2l;
            lobe_local(L, v, wl, ql, t2l);
            const bool me = tech && i == pick;
            pv += w[i] * __expf(lobe_log_g(L, sel(me, ws, wl), sel(me, qs, ql), sel(me, t2s, t2l)) - L.log_k);
            lobe_local(L, vn, wl, ql, t2l);
            pn += w[i] * __expf(lobe_log_g(L, wl, ql, t2l) - L.log_k);
        }
    });
    xc.to0(pv, pn);
    o0 = make_float4(v.x, v.y, v.z, pv);
    o1 = make_float4(dnee.w > 0.f ? pn : 0.f, ce, tech ? 1.f : 0.f, c);
}

// ---- KL gradient in fp32 (bf16 training path) --------------------------------
// Decode intermediates the chain rule needs (DecodedGuide guiding.hpp:34-42).
struct LobeG {
    Lobe L;
    float sig[5], sigm[5];      // sigmoid(raw) and 1 - sigmoid(raw)
    float ct, st, sp, cp, stau, ctau;
    float pn1, pn2;             // pre-normalisation pair norms (0 => degenerate)
    bool lam_cl, a_cl;
};

__device__ __forceinline__ void decode_lobe_g(const float r[7], LobeG &G) {
#pragma unroll
    for (int k = 0; k < 5; ++k) sigmoid_pair(r[k], G.sig[k], G.sigm[k]);
    const float ct = G.sig[0] - G.sigm[0];
    float sp = G.sig[1] - G.sigm[1], cp = G.sig[2] - G.sigm[2], st = G.sig[3] - G.sigm[3], ctau = G.sig[4] - G.sigm[4];
    const float n1 = sqrt_fast(sp * sp + cp * cp), n2 = sqrt_fast(st * st + ctau * ctau);
    const bool d1 = n1 < 1e-6f, d2 = n2 < 1e-6f;
    const float i1 = rcp_fast(d1 ? 1.f : n1), i2 = rcp_fast(d2 ? 1.f : n2);
    sp = d1 ? 0.f : sp * i1;
    cp = d1 ? 1.f : cp * i1;
    st = d2 ? 0.f : st * i2;
    ctau = d2 ? 1.f : ctau * i2;
    G.pn1 = d1 ? 0.f : n1;
    G.pn2 = d2 ? 0.f : n2;
    const float sth = 2.f * sqrt_fast(G.sig[0] * G.sigm[0]);
    G.ct = ct; G.st = sth; G.sp = sp; G.cp = cp; G.stau = st; G.ctau = ctau;
    Lobe &L = G.L;
    L.z = make_float3(cp * sth, sp * sth, ct);
    L.x = make_float3(ct * cp * ctau - sp * st, ct * sp * ctau + cp * st, -sth * ctau);
    L.y = make_float3(0.f, 0.f, 0.f);  // unused by the gradient
    const float lam = __expf(r[5]), a = __expf(r[6]);
    L.lambda = fminf(fmaxf(lam, kLambdaMinF), kLambdaMaxF);
    L.a = fminf(a, kEccMaxF);
    G.lam_cl = L.lambda != lam;
    G.a_cl = L.a != a;
    L.one_m_emin = -expm1_fast(-2.f * L.lambda);
    L.log_k = kLog2Pi + __logf(L.one_m_emin * rcp_fast(L.lambda)) - 0.5f * __logf(1.f + L.a);
}

// d log K / d lambda = coth(l) - 1 - 1/l, with a series below l = 0.05 (sphdist.cpp:217)
__device__ __forceinline__ float dlogk_dlambda(float l, float one_m_emin) {
    const float l2 = l * l;
    const float ser = -1.f + l * (1.f / 3.f - l2 * (1.f / 45.f - l2 * (2.f / 945.f)));
    return l < 0.05f ? ser : 2.f * (1.f - one_m_emin) * rcp_fast(one_m_emin) - rcp_fast(l);
}

// Outcome of one row's KL gradient (guiding.cpp:236-257 bookkeeping).
enum KlStatus : int {
    kKlZero = 0,  // p == 0: valid sample, zero gradient, zero loss (guiding.cpp:112)
    kKlOk = 1,    // gradient emitted; loss may still be non-finite (not accumulated)
    kKlDrop = 2,  // non-finite network row, unusable q, or non-finite gradient: dropped
};

// Pass 2 of the KL gradient for one lobe (guiding.cpp:118-152 with
// nasg_grad_logpdf sphdist.cpp:200-274, fp32 stable forms): the lobe's 8 raw
// logits r, its weighted pdf w_i pdf_i (wpi) and weight wi, 1 / q_mix and the
// sample's scale -> the weight-logit gradient gl and the lobe's 8 packed columns.
__device__ __forceinline__ void kl_lobe_grad(const float (&r)[8], const TrainRow &s, float wpi, float wi, float inv_q,
                                             float scale, float &gl, float (&g8)[8], bool &finite) {
    LobeG G;
    decode_lobe_g(r, G);
    const Lobe &L = G.L;
    const float ri = wpi * inv_q;  // posterior responsibility
    gl = scale * (ri - wi);
    finite &= isfinite(gl);
    // local frame of omega_i (stable fp32 forms, nasg_math.cuh header)
    const float3 v = s.wi;
    const float dz = dot3(v, L.z);
    const float sg = dz >= 0.f ? 1.f : -1.f;
    const float3 ev = make_float3(v.x - sg * L.z.x, v.y - sg * L.z.y, v.z - sg * L.z.z);
    const float hh = 0.5f * dot3(ev, ev);
    const float wl = dz >= 0.f ? hh : 2.f - hh, ql = dz >= 0.f ? 2.f - hh : hh;
    const float dx = dot3(ev, L.x);
    const float denom = fmaxf(wl * ql, 1e-12f);
    const float t2 = fminf(fmaxf(dx * dx * rcp_fast(denom), 0.f), 1.f);
    float g7[7] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // d log q / d (ct, sp, cp, st, ctau, lambda, a)
    if (fminf(wl, ql) >= 1e-6f && wpi > 0.f) {         // pole guard sphdist.cpp:205
        const float lam = L.lambda, a = L.a;
        float log_u = log_u_of(wl, ql);
        log_u = fmaxf(log_u, -27.631021f);
        const float u = fmaxf(0.5f * ql, 1e-12f);
        const float beta = a * t2, m = 1.f + beta;
        const float um1 = expm1_fast(m * log_u), um = um1 + 1.f;
        const float inv_u = rcp_fast(u), inv_den = rcp_fast(denom);
        const float dG_dbeta = (2.f * lam * um + 1.f) * log_u;
        const float dG_du = 2.f * lam * m * (um * inv_u) + beta * inv_u;
        const float dt2_ddz = 2.f * dz * t2 * inv_den;
        const float dG_ddz = 0.5f * dG_du + dG_dbeta * a * dt2_ddz;
        const float dG_ddx = dG_dbeta * a * 2.f * dx * inv_den;
        g7[5] = ri * (2.f * um1 - dlogk_dlambda(lam, L.one_m_emin));
        g7[6] = ri * (t2 * dG_dbeta + 0.5f * rcp_fast(1.f + a));
        const float ct = G.ct, st = fmaxf(G.st, 1e-9f), dst = -ct * rcp_fast(st);
        const float cs = G.cp * v.x + G.sp * v.y;
        float g_ct = dG_ddz * (dst * cs + v.z) + dG_ddx * (G.ctau * cs - dst * G.ctau * v.z);
        float g_sp = dG_ddz * (st * v.y) + dG_ddx * (-G.stau * v.x + ct * G.ctau * v.y);
        float g_cp = dG_ddz * (st * v.x) + dG_ddx * (ct * G.ctau * v.x + G.stau * v.y);
        float g_st = dG_ddx * (-G.sp * v.x + G.cp * v.y);
        float g_ctau = dG_ddx * (ct * G.cp * v.x + ct * G.sp * v.y - st * v.z);
        float ps = G.cp * (G.cp * g_sp - G.sp * g_cp), pc = G.sp * (G.sp * g_cp - G.cp * g_sp);
        g_sp = ps; g_cp = pc;
        ps = G.ctau * (G.ctau * g_st - G.stau * g_ctau);
        pc = G.stau * (G.stau * g_ctau - G.ctau * g_st);
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
    const float inv1 = G.pn1 > 0.f ? rcp_fast(G.pn1) : 0.f, inv2 = G.pn2 > 0.f ? rcp_fast(G.pn2) : 0.f;
    const float scl[5] = {1.f, inv1, inv1, inv2, inv2};
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        g8[k] = scale * g7[k] * scl[k] * 2.f * G.sig[k] * G.sigm[k];
        finite &= isfinite(g8[k]);
    }
    g8[5] = G.lam_cl ? 0.f : scale * g7[5] * L.lambda;
    g8[6] = G.a_cl ? 0.f : scale * g7[6] * L.a;
    g8[7] = 0.f;
    finite &= isfinite(g8[5]) && isfinite(g8[6]);
}

// One-sample KL gradient w.r.t. the packed raw outputs, fp32 restatement of
// kl_loss_gradient (guiding.cpp:108-165) + nasg_grad_logpdf (sphdist.cpp:200-274)
// in two O(N) passes over the lobes.  The raw row is never held whole:
//   hdr          packed header columns [0, H) (weight logits, c)
//   lobe(i, r)   loads lobe i's 8 packed columns (tensor-memory read in the kernel)
//   put_lobe(i, g) emits lobe i's 8 gradient columns (pass 2, in lobe order)
//   ghdr         receives the header's gradient columns
// Gradients carry the 1/count factor gscale.  On kKlOk every column has been
// emitted; on kKlZero / kKlDrop the caller writes zeros over the whole row
// (lobe columns may already hold values).  Non-finite raw outputs are checked
// before p == 0, as the trainer does (guiding.cpp:251-254 precede :112).
// lobe() is called for every i in both passes whatever the row's outcome (and
// for rows with valid = false), so a warp-collective load behind it stays
// convergent; only the arithmetic is predicated.
constexpr int kKlScStride = 128;  // rows per tile: per-row scratch interleaved across threads

template <int N, class LobeFn, class PutLobeFn>
__device__ __forceinline__ int kl_grad_row_fast(bool valid, const float (&hdr)[packed_header(N)], LobeFn lobe,
                                                const TrainRow &s, float b, float e, float gscale,
                                                float (&ghdr)[packed_header(N)], PutLobeFn put_lobe, float &loss,
                                                float *sc) {
    // The lobe loops are runtime loops (one copy of each body: the unrolled
    // 2 x N bodies overflowed the instruction cache); the per-lobe values that
    // cross from pass 1 to pass 2 live in this row's shared-memory scratch
    // sc[k * kKlScStride], k < 2N: [i] = w_i pdf_i (then the weight-logit
    // gradient), [N + i] = w_i.
    constexpr int H = packed_header(N);
    loss = 0.f;
    bool fin = true;
#pragma unroll
    for (int j = 0; j <= N; ++j) fin &= isfinite(hdr[j]);
    float w[N], c, c_sig;
    {
        float mx = -INFINITY;
#pragma unroll
        for (int i = 0; i < N; ++i) mx = fmaxf(mx, hdr[i]);
        float sum = 0.f;
#pragma unroll
        for (int i = 0; i < N; ++i) {
            w[i] = __expf(hdr[i] - mx);
            sum += w[i];
        }
        const float inv = rcp_fast(sum);
#pragma unroll
        for (int i = 0; i < N; ++i) sc[(N + i) * kKlScStride] = w[i] * inv;
        float sm;
        sigmoid_pair(hdr[N], c_sig, sm);
        c = fminf(fmaxf(c_sig, kSelMin), kSelMax);
    }
    const bool live = valid && s.p != 0.f;
    float q_mix = 0.f;
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        float r[8];
        lobe(i, r);
#pragma unroll
        for (int k = 0; k < 7; ++k) fin &= isfinite(r[k]);
        float wp = 0.f;
        if (live) {
            Lobe L;
            decode_lobe(r, L);
            wp = sc[(N + i) * kKlScStride] * __expf(lobe_log_g_at(L, s.wi) - L.log_k);
            q_mix += wp;
        }
        sc[i * kKlScStride] = wp;
    }
    const float c_eff = b * c;
    const float q_hat = c_eff * q_mix + (1.f - c_eff) * s.pbsdf;
    int status = kKlOk;
    if (!valid || (fin && !live)) {
        status = kKlZero;
    } else if (!fin) {
        status = kKlDrop;
    } else if (!(isfinite(q_mix) && q_mix > 0.f && isfinite(q_hat) && q_hat > 0.f) || !(s.q_s > 0.f)) {
        loss = __int_as_float(0x7fc00000);
        status = kKlDrop;
    }
    const bool go = status == kKlOk;
    const float ws = s.p / s.q_s;
    const float mix_scale = e * (c_eff * q_mix / q_hat) + (1.f - e);
    const float scale = -ws * mix_scale * gscale;
    const float inv_q = rcp_fast(q_mix);
    bool finite = true;
    {
        const float dsig = (c != c_sig) ? 0.f : c_sig * (1.f - c_sig);
        const float gc = -ws * e * b * (q_mix - s.pbsdf) / q_hat * dsig * gscale;
        finite &= isfinite(gc);
        ghdr[N] = gc;
#pragma unroll
        for (int j = N + 1; j < H; ++j) ghdr[j] = 0.f;
    }
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        float r[8];
        lobe(i, r);
        if (!go) continue;
        const float wpi = sc[i * kKlScStride], wi = sc[(N + i) * kKlScStride];
        float gl, g8[8];
        kl_lobe_grad(r, s, wpi, wi, inv_q, scale, gl, g8, finite);
        sc[i * kKlScStride] = gl;
        put_lobe(i, g8);
    }
    if (!go) return status;
#pragma unroll
    for (int i = 0; i < N; ++i) ghdr[i] = sc[i * kKlScStride];
    if (!finite) return kKlDrop;
    loss = -ws * (e * __logf(q_hat) + (1.f - e) * __logf(q_mix));
    return kKlOk;
}


template <int N>
__device__ __forceinline__ float wsel_f(const float (&w)[N], int i) {  // w[i] for a runtime i, in registers
    float x = w[0];
#pragma unroll
    for (int j = 1; j < N; ++j) x = i == j ? w[j] : x;
    return x;
}

// Cooperative kl_grad_row_fast for one tile shared by GW warpgroups (the bf16
// trainer's small-batch regime, one tile per CTA): warpgroup g decodes and
// differentiates lobes g, g + GW, ...  The row's per-lobe values cross through
// shared memory — sc: this row's column of a [3N][kKlScStride] scratch
// (w_i pdf_i, unused, weight-logit gradients), flg: [2 GW][kKlScStride]
// finiteness flags — and q_mix is summed in lobe order, so every value equals
// kl_grad_row_fast's.  sync(k), k = 0, 1, must be a barrier over all GW groups
// (with the proxy / tensor-memory fences the caller's put_lobe needs).  Group 0
// gets the header gradient, the status and the loss; the others return kKlZero.
template <int N, int GW, class LobeFn, class PutLobeFn, class SyncFn>
__device__ __forceinline__ int kl_grad_row_coop(int g, bool valid, const float (&hdr)[packed_header(N)], LobeFn lobe,
                                                const TrainRow &s, float b, float e, float gscale,
                                                float (&ghdr)[packed_header(N)], PutLobeFn put_lobe, float &loss,
                                                float *sc, int *flg, SyncFn sync) {
    constexpr int H = packed_header(N), S = kKlScStride;
    float *wp_s = sc, *gl_s = sc + 2 * N * S;
    loss = 0.f;
    bool fin = true;
#pragma unroll
    for (int j = 0; j <= N; ++j) fin &= isfinite(hdr[j]);
    float w[N], c, c_sig;
    {
        float mx = -INFINITY;
#pragma unroll
        for (int i = 0; i < N; ++i) mx = fmaxf(mx, hdr[i]);
        float sum = 0.f;
#pragma unroll
        for (int i = 0; i < N; ++i) {
            w[i] = __expf(hdr[i] - mx);
            sum += w[i];
        }
        const float inv = rcp_fast(sum);
#pragma unroll
        for (int i = 0; i < N; ++i) w[i] *= inv;
        float sm;
        sigmoid_pair(hdr[N], c_sig, sm);
        c = fminf(fmaxf(c_sig, kSelMin), kSelMax);
    }
    const bool live = valid && s.p != 0.f;
#pragma unroll 1
    for (int i = g; i < N; i += GW) {
        float r[8];
        lobe(i, r);
#pragma unroll
        for (int k = 0; k < 7; ++k) fin &= isfinite(r[k]);
        float wp = 0.f;
        if (live) {
            Lobe L;
            decode_lobe(r, L);
            wp = wsel_f<N>(w, i) * __expf(lobe_log_g_at(L, s.wi) - L.log_k);
        }
        wp_s[i * S] = wp;
    }
    flg[g * S] = fin;
    sync(0);
    float q_mix = 0.f;
#pragma unroll
    for (int i = 0; i < N; ++i) q_mix += wp_s[i * S];
#pragma unroll
    for (int k = 0; k < GW; ++k) fin = fin && flg[k * S] != 0;
    const float c_eff = b * c;
    const float q_hat = c_eff * q_mix + (1.f - c_eff) * s.pbsdf;
    int status = kKlOk;
    if (!valid || (fin && !live)) {
        status = kKlZero;
    } else if (!fin) {
        status = kKlDrop;
    } else if (!(isfinite(q_mix) && q_mix > 0.f && isfinite(q_hat) && q_hat > 0.f) || !(s.q_s > 0.f)) {
        loss = __int_as_float(0x7fc00000);
        status = kKlDrop;
    }
    const bool go = status == kKlOk;
    const float ws = s.p / s.q_s;
    const float mix_scale = e * (c_eff * q_mix / q_hat) + (1.f - e);
    const float scale = -ws * mix_scale * gscale;
    const float inv_q = rcp_fast(q_mix);
    bool finite = true;
    if (g == 0) {
        const float dsig = (c != c_sig) ? 0.f : c_sig * (1.f - c_sig);
        const float gc = -ws * e * b * (q_mix - s.pbsdf) / q_hat * dsig * gscale;
        finite &= isfinite(gc);
        ghdr[N] = gc;
#pragma unroll
        for (int j = N + 1; j < H; ++j) ghdr[j] = 0.f;
    }
#pragma unroll 1
    for (int i = g; i < N; i += GW) {
        float r[8];
        lobe(i, r);
        if (!go) continue;
        float gl, g8[8];
        kl_lobe_grad(r, s, wp_s[i * S], wsel_f<N>(w, i), inv_q, scale, gl, g8, finite);
        gl_s[i * S] = gl;
        put_lobe(i, g8);
    }
    flg[(GW + g) * S] = finite;
    sync(1);
    if (g != 0) return kKlZero;
#pragma unroll
    for (int k = 0; k < GW; ++k) finite = finite && flg[(GW + k) * S] != 0;
    if (!go) return status;
#pragma unroll
    for (int i = 0; i < N; ++i) ghdr[i] = gl_s[i * S];
    if (!finite) return kKlDrop;
    loss = -ws * (e * __logf(q_hat) + (1.f - e) * __logf(q_mix));
    return kKlOk;
}

}  // namespace nasg
