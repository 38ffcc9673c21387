// Analytic scenes, BSDFs, light sampling and counter-based random numbers for
// the guided wavefront path tracer (SPEC.md tracer module, lines 378-478: the
// reference specifies the tracer but ships no code for it).
//
// Scene: spheres and parallelogram quads (two-sided surfaces, one-sided
// emitters), materials lambertian / normalised Phong-glossy / mirror, a
// constant environment and a pinhole camera.  Everything lives in __constant__
// memory (a few hundred bytes), so intersection is a linear scan.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace nasg {
namespace rt {

constexpr int kMaxPrims = 24, kMaxMats = 8, kMaxLights = 4;
constexpr float kPiF = 3.14159265358979f, kInvPiF = 0.318309886183791f;
constexpr float kEps = 1e-4f;  // shadow-acne epsilon (SPEC.md: 1e-4 scene units)

enum PrimType : int { kSphere = 0, kQuad = 1 };
enum MatType : int { kLambert = 0, kPhong = 1, kMirror = 2, kEmitter = 3 };

struct Prim {
    int type, mat;
    float3 p;     // sphere centre / quad corner
    float3 u, v;  // quad edges (normal = normalize(u x v))
    float r;      // sphere radius
};
struct Mat {
    int type;
    float3 albedo;
    float exponent;  // Phong
    float3 emission; // emitters: radiance towards the quad normal
};
struct Camera {
    float3 pos, fwd, right, up;  // right/up scaled by tan(fov/2) (and aspect)
    int width, height;
};
struct Scene {
    int nprims, nlights;
    Prim prims[kMaxPrims];
    Mat mats[kMaxMats];
    int light_prim[kMaxLights];
    float light_cdf[kMaxLights];  // area CDF over the emitters
    float light_area_total;
    float3 env;
    Camera cam;
    float bmin[3], bmax[3];
};

struct Hit {
    float t;
    int prim;
    float3 x, n;  // geometric normal (quads: u x v side, spheres: outward)
};

__host__ __device__ inline float3 f3(float a, float b, float c) { return make_float3(a, b, c); }
__host__ __device__ inline float3 operator+(float3 a, float3 b) { return f3(a.x + b.x, a.y + b.y, a.z + b.z); }
__host__ __device__ inline float3 operator-(float3 a, float3 b) { return f3(a.x - b.x, a.y - b.y, a.z - b.z); }
__host__ __device__ inline float3 operator*(float3 a, float s) { return f3(a.x * s, a.y * s, a.z * s); }
__host__ __device__ inline float3 mul(float3 a, float3 b) { return f3(a.x * b.x, a.y * b.y, a.z * b.z); }
__host__ __device__ inline float dot(float3 a, float3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__host__ __device__ inline float3 cross(float3 a, float3 b) {
    return f3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__host__ __device__ inline float3 normalize(float3 a) { return a * (1.f / sqrtf(dot(a, a))); }
__host__ __device__ inline float lum(float3 c) { return 0.2126f * c.x + 0.7152f * c.y + 0.0722f * c.z; }

// ---- counter-based random numbers: (seed, pixel, iteration, bounce, dimension)
__host__ __device__ inline uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__host__ __device__ inline float rnd(uint64_t seed, uint64_t pixel, uint64_t iter, uint32_t bounce, uint32_t dim) {
    const uint64_t h = mix64(mix64(mix64(seed ^ 0x6e61736772656e64ull) + pixel) + (iter << 16) + (bounce << 8) + dim);
    return (float)(h >> 40) * (1.f / 16777216.f);  // [0, 1) on the float grid
}

// ---- intersection (nearest hit with t > kEps; linear scan) ---------------------
__device__ inline bool hit_prim(const Prim &p, float3 o, float3 d, float tmax, float &t, float3 &n) {
    if (p.type == kSphere) {
        const float3 oc = o - p.p;
        const float b = dot(oc, d), c = dot(oc, oc) - p.r * p.r;
        const float disc = b * b - c;
        if (disc < 0.f) return false;
        const float s = sqrtf(disc);
        float tt = -b - s;
        if (tt <= kEps) tt = -b + s;
        if (tt <= kEps || tt >= tmax) return false;
        t = tt;
        n = (o + d * tt - p.p) * (1.f / p.r);
        return true;
    }
    const float3 nn = cross(p.u, p.v);
    const float den = dot(nn, d);
    if (fabsf(den) < 1e-12f) return false;
    const float tt = dot(p.p - o, nn) / den;
    if (tt <= kEps || tt >= tmax) return false;
    const float3 h = o + d * tt - p.p;
    const float3 w = nn * (1.f / dot(nn, nn));
    const float a = dot(w, cross(h, p.v)), b = dot(w, cross(p.u, h));
    if (a < 0.f || a > 1.f || b < 0.f || b > 1.f) return false;
    t = tt;
    n = normalize(nn);
    return true;
}

__device__ inline bool intersect(const Scene &s, float3 o, float3 d, float tmax, Hit &h) {
    h.t = tmax;
    h.prim = -1;
    for (int i = 0; i < s.nprims; ++i) {
        float t;
        float3 n;
        if (hit_prim(s.prims[i], o, d, h.t, t, n)) {
            h.t = t;
            h.prim = i;
            h.n = n;
        }
    }
    if (h.prim < 0) return false;
    h.x = o + d * h.t;
    return true;
}

// Shadow ray towards a point on emitter `target`: that primitive is skipped, so
// the offset origin can never see the light itself as its own occluder (a point
// right under a light would otherwise lose its direct illumination).
__device__ inline bool occluded(const Scene &s, float3 o, float3 d, float dist, int target) {
    for (int i = 0; i < s.nprims; ++i) {
        float t;
        float3 n;
        if (i != target && hit_prim(s.prims[i], o, d, dist * (1.f - 1e-4f), t, n)) return true;
    }
    return false;
}

// ---- BSDFs (SPEC.md bsdf_sample_eval_pdf).  n faces wo.  No cosine in f. ------
__device__ inline float3 reflect(float3 wo, float3 n) { return n * (2.f * dot(n, wo)) - wo; }

__device__ inline void onb(float3 n, float3 &t, float3 &b) {  // branchless orthonormal basis
    const float sgn = copysignf(1.f, n.z);
    const float a = -1.f / (sgn + n.z), bb = n.x * n.y * a;
    t = f3(1.f + sgn * n.x * n.x * a, sgn * bb, -sgn * n.x);
    b = f3(bb, sgn + n.y * n.y * a, -n.y);
}

__device__ inline float3 bsdf_eval(const Mat &m, float3 n, float3 wo, float3 wi) {
    const float ci = dot(n, wi);
    if (ci <= 0.f || dot(n, wo) <= 0.f) return f3(0.f, 0.f, 0.f);
    if (m.type == kLambert) return m.albedo * kInvPiF;
    if (m.type == kPhong) {
        const float ca = fmaxf(dot(reflect(wo, n), wi), 0.f);
        return m.albedo * ((m.exponent + 2.f) * 0.5f * kInvPiF * powf(ca, m.exponent));
    }
    return f3(0.f, 0.f, 0.f);  // mirror / emitter: no non-delta lobe
}

__device__ inline float bsdf_pdf(const Mat &m, float3 n, float3 wo, float3 wi) {
    const float ci = dot(n, wi);
    if (ci <= 0.f) return 0.f;
    if (m.type == kLambert) return ci * kInvPiF;
    if (m.type == kPhong) {
        const float ca = fmaxf(dot(reflect(wo, n), wi), 0.f);
        return (m.exponent + 1.f) * 0.5f * kInvPiF * powf(ca, m.exponent);
    }
    return 0.f;
}

// Returns false for a zero-contribution sample: a glossy lobe direction below the
// surface.  One attempt, not SPEC's "resample up to 8 times": the retries would
// make the technique's density p_lobe (1 - P_below^8) / (1 - P_below) while the
// estimator and the MIS blend use p_lobe, biasing every grazing glossy vertex; a
// single attempt keeps the density exactly p_lobe (the failed mass contributes 0),
// which the SPEC's own unbiasedness invariant requires.
template <class Rng>
__device__ inline bool bsdf_sample(const Mat &m, float3 n, float3 wo, Rng rng, float3 &wi) {
    if (m.type == kLambert) {
        const float u1 = rng(0), u2 = rng(1);
        const float r = sqrtf(u1), phi = 2.f * kPiF * u2;
        float3 t, b;
        onb(n, t, b);
        wi = t * (r * cosf(phi)) + b * (r * sinf(phi)) + n * sqrtf(fmaxf(0.f, 1.f - u1));
        return true;
    }
    if (m.type == kPhong) {
        const float3 r = reflect(wo, n);
        float3 t, b;
        onb(r, t, b);
        const float u1 = rng(0), u2 = rng(1);
        const float ca = powf(u1, 1.f / (m.exponent + 1.f)), sa = sqrtf(fmaxf(0.f, 1.f - ca * ca));
        const float phi = 2.f * kPiF * u2;
        wi = t * (sa * cosf(phi)) + b * (sa * sinf(phi)) + r * ca;
        return dot(wi, n) > 0.f;
    }
    return false;
}

// ---- emitters: area sampling and the solid-angle pdf of a hit -------------------
__device__ inline float light_pdf_at(const Scene &s, float3 x, const Hit &h, float3 d) {
    const float cl = -dot(h.n, d);  // one-sided: emits towards its normal
    if (cl <= 0.f) return 0.f;
    return h.t * h.t / (cl * s.light_area_total);
}

struct LightSample {
    float3 dir, Le;
    float dist, pdf;  // pdf in solid angle at x; 0 if unusable
    int prim;         // the emitter primitive sampled
};

__device__ inline LightSample sample_light(const Scene &s, float3 x, float u0, float u1, float u2) {
    LightSample ls{f3(0.f, 0.f, 1.f), f3(0.f, 0.f, 0.f), 0.f, 0.f, -1};
    if (s.nlights == 0) return ls;
    int k = s.nlights - 1;
    for (int i = 0; i < s.nlights; ++i)
        if (u0 < s.light_cdf[i]) {
            k = i;
            break;
        }
    ls.prim = s.light_prim[k];
    const Prim &p = s.prims[ls.prim];
    const float3 y = p.p + p.u * u1 + p.v * u2;
    const float3 dv = y - x;
    const float d2 = dot(dv, dv);
    if (d2 <= 1e-12f) return ls;
    ls.dist = sqrtf(d2);
    ls.dir = dv * (1.f / ls.dist);
    const float3 nl = normalize(cross(p.u, p.v));
    const float cl = -dot(nl, ls.dir);
    if (cl <= 0.f) return ls;
    ls.pdf = d2 / (cl * s.light_area_total);
    ls.Le = s.mats[p.mat].emission;
    return ls;
}

}  // namespace rt
}  // namespace nasg
