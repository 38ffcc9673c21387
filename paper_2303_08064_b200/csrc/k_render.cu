// Guided progressive render loop (SPEC.md tracer module, :378-478; PAPER §6):
// a wavefront path tracer whose scattering at every non-delta vertex goes
// through the fused network query (nasg_query_shade), and whose selected
// pixels feed the online trainer (nasg_train_iteration) after every frame.
//
// One iteration (= 1 sample per pixel of this rank's rows):
//   K_begin     camera rays, path state, which pixel of each l x l tile collects
//   per bounce  K_isect  nearest hit; environment / emitter hits with the MIS
//                        weight of the previous scatter; mirror bounces; at
//                        non-delta vertices NEE (light sample + shadow ray), a
//                        BSDF pre-sample, and a slot in the guide queue
//               guide    nasg_query_shade over the queue (device row count):
//                        technique, direction, q_mix at it and at the NEE dir
//               K_update blend pdf, MIS-weighted NEE, throughput, training
//                        record of collected paths, Russian roulette
//   K_scan_* + K_records  per-vertex incident radiance by back-propagation
//                        (L_i = (L_end - L_before) / beta), TrainingSamples in
//                        deterministic tile order, an evenly spread S kept
//   K_accumulate film += w_i L (non-finite paths discarded and counted)
//   train_iteration + publish, stride_update (host)
// Path state is SoA in HBM (float4 per quantity); the guide queue is compacted
// with one atomic per guided vertex, so the query kernel runs over exactly the
// live vertices without a host round trip.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>
#ifdef NASG_RENDER_PROF  // development-only phase timing (scratch builds), compiled out of the library
#include <chrono>
namespace {
struct RProf {
    cudaEvent_t a = nullptr, b = nullptr, c = nullptr, pc = nullptr;  // trace start, trace end, train end
    double host[4] = {0, 0, 0, 0}, gpu[3] = {0, 0, 0};
    int n = 0, ng = 0;
    std::chrono::steady_clock::time_point t0;
    ~RProf() {
        if (n) fprintf(stderr, "[rprof] %d it: host enqueue-trace %.3f ms, wait-sync %.3f ms, train-call %.3f ms, rest %.3f ms | gpu trace %.3f, sync->train-end %.3f, idle-before-trace %.3f ms (%d)\n",
                       n, host[0] / n, host[1] / n, host[2] / n, host[3] / n, gpu[0] / ng, gpu[1] / ng, gpu[2] / ng, ng);
    }
};
RProf g_rprof;
double ms_since(std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}
}  // namespace
#endif

#include <cuda_runtime.h>

#include "nasg/nasg.h"
#include "nasg_internal.h"
#include "render_scene.cuh"

namespace nasg {
namespace rt {

__constant__ Scene c_scene;

constexpr int kMaxDepthCap = 16;
constexpr int kBlock = 256;

struct Paths {
    int64_t n;  // paths = pixels of this rank
    float4 *o, *d, *beta, *L;
    float *prev_pdf;        // q-hat of the last scatter; < 0: camera ray or delta bounce
    int *alive, *pending;   // pending: a non-delta vertex waiting for K_update
    int *act[2];            // compacted lists of the paths alive at the start of a bounce (by parity)
    int *nact;              // their lengths, one per bounce [kMaxDepthCap + 1] (zeroed per iteration)
    float4 *vx, *vn, *vwo, *vdb, *vdn, *vnee;
    int *slot, *rank, *bsdf_ok;
    // guide queue
    float4 *qx, *qwo, *qn, *qxi, *qdb, *qdn, *qout;
    int *qcount;            // guided queries queued at each bounce [kMaxDepthCap] (zeroed per iteration)
    // training records [depth][ncap]
    int64_t ncap;
    float4 *rx, *rwo, *rn, *rwi, *rfc, *rbeta, *rlb;
    int *rcnt, *rpix, *roff, *bsum, *boff;  // record counts, owning path, offsets (block-local + block)
    unsigned long long *ctr;  // 0 vertices, 1 guided, 2 nonfinite, 3 collected
    float4 *film, *frame;
    nasg_train_sample *samples;
    int64_t cap_samples;
};

struct Frame {
    uint64_t seed, iter;
    int width, height, row0;
    int band, shard, nshards;  // interleaved sharding (band > 0): see frame_row
    float l;          // collection stride
    int tile_row0;    // floor(row0 / l) (0 with interleaving: tiles over the compacted rows)
    int ntx;          // tiles per row
    int collect, max_depth, rr_depth;
    int nee;
};

// Image row of this rank's local row lr: contiguous rows from row0, or the
// lr-th row of the bands shard, shard + nshards, ... of `band` rows each.
__device__ __forceinline__ int frame_row(const Frame &F, int lr) {
    if (F.band <= 0) return F.row0 + lr;
    const int k = lr / F.band;
    return (k * F.nshards + F.shard) * F.band + (lr - k * F.band);
}

__device__ inline float4 f4(float3 v, float w) { return make_float4(v.x, v.y, v.z, w); }
__device__ inline float3 xyz(float4 v) { return make_float3(v.x, v.y, v.z); }

__global__ void k_begin(Paths P, Frame F) {
    pdl_trigger();
    pdl_wait();  // every input comes from the previous kernel on the stream
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.n) return;
    const Scene &S = c_scene;
    const int px = (int)(i % F.width), py = frame_row(F, (int)(i / F.width));
    const uint64_t pix = (uint64_t)py * F.width + px;
    const float jx = rnd(F.seed, pix, F.iter, 0, 0), jy = rnd(F.seed, pix, F.iter, 0, 1);
    const float sx = 2.f * (px + jx) / F.width - 1.f, sy = 1.f - 2.f * (py + jy) / F.height;
    const float3 d = normalize(S.cam.fwd + S.cam.right * sx + S.cam.up * sy);
    P.o[i] = f4(S.cam.pos, 0.f);
    P.d[i] = f4(d, 0.f);
    P.beta[i] = make_float4(1.f, 1.f, 1.f, 0.f);
    P.L[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    P.prev_pdf[i] = -1.f;
    P.alive[i] = 1;
    P.pending[i] = 0;
    P.act[0][i] = (int)i;
    if (i == 0) P.nact[0] = (int)P.n;
    int rank = -1;
    if (F.collect) {  // one pixel per l x l tile (PAPER §6), uniformly at random per tile and iteration
        // tiles over the image rows, or over the compacted local rows with interleaving
        const int ry = F.band > 0 ? (int)(i / F.width) : py;
        const uint64_t cseed = F.seed ^ 0x636f6c6cull ^ ((uint64_t)F.shard << 40);
        const int tx = (int)floorf(px / F.l), ty = (int)floorf(ry / F.l);
        const uint64_t tile = ((uint64_t)ty << 32) | (uint32_t)tx;
        const int cx = (int)floorf((tx + rnd(cseed, tile, F.iter, 0, 0)) * F.l);
        const int cy = (int)floorf((ty + rnd(cseed, tile, F.iter, 0, 1)) * F.l);
        if (cx == px && cy == ry) {
            const int64_t r = (int64_t)(ty - F.tile_row0) * F.ntx + tx;
            if (r >= 0 && r < P.ncap) {
                rank = (int)r;
                P.rpix[r] = (int)i;
            }
        }
    }
    P.rank[i] = rank;
    if (rank >= 0) P.rcnt[rank] = 0;
}

// per-bounce queue reset; the previous bounce's queue length feeds the counter;
// the list the coming bounce's survivors are appended to starts empty
__device__ __forceinline__ void isect_path(Paths &P, const Frame &F, int bounce, int guided, int64_t i) {
    if (!P.alive[i]) return;
    const Scene &S = c_scene;
    const int px = (int)(i % F.width), py = frame_row(F, (int)(i / F.width));
    const uint64_t pix = (uint64_t)py * F.width + px;
    auto R = [&](uint32_t dim) { return rnd(F.seed, pix, F.iter, (uint32_t)bounce + 1, dim); };
    const float3 o = xyz(P.o[i]), d = xyz(P.d[i]);
    float4 beta = P.beta[i], L = P.L[i];
    Hit h;
    if (!intersect(S, o, d, 1e30f, h)) {  // environment (not light-sampled: weight 1)
        L.x += beta.x * S.env.x;
        L.y += beta.y * S.env.y;
        L.z += beta.z * S.env.z;
        P.L[i] = L;
        P.alive[i] = 0;
        return;
    }
    const Prim &prim = S.prims[h.prim];
    const Mat &m = S.mats[prim.mat];
    if (m.type == kEmitter) {  // emitters absorb; MIS against NEE for scattered rays
        const float cl = -dot(h.n, d);
        if (cl > 0.f) {
            const float pp = P.prev_pdf[i];
            float w = 1.f;
            if (pp >= 0.f && F.nee) {
                const float pl = light_pdf_at(S, o, h, d);
                w = pp / (pp + pl);
            }
            L.x += beta.x * m.emission.x * w;
            L.y += beta.y * m.emission.y * w;
            L.z += beta.z * m.emission.z * w;
            P.L[i] = L;
        }
        P.alive[i] = 0;
        return;
    }
    atomicAdd(&P.ctr[0], 1ull);
    const float3 wo = d * -1.f;
    const float3 n = dot(h.n, wo) < 0.f ? h.n * -1.f : h.n;  // two-sided surfaces
    if (m.type == kMirror) {  // delta vertex: no guiding, no NEE, no training record
        const float3 r = reflect(wo, n);
        beta.x *= m.albedo.x;
        beta.y *= m.albedo.y;
        beta.z *= m.albedo.z;
        P.beta[i] = beta;
        P.o[i] = f4(h.x + n * kEps, 0.f);
        P.d[i] = f4(r, 0.f);
        P.prev_pdf[i] = -1.f;
        return;
    }
    // next-event estimation (SPEC nee_sample): one emitter by area, shadow ray
    LightSample ls = sample_light(S, h.x, R(0), R(1), R(2));
    if (!F.nee) ls.pdf = 0.f;
    float3 nee = f3(0.f, 0.f, 0.f);
    float pl = 0.f;
    if (ls.pdf > 0.f && dot(n, ls.dir) > 0.f && !occluded(S, h.x + n * kEps, ls.dir, ls.dist, ls.prim)) {
        const float3 f = bsdf_eval(m, n, wo, ls.dir);
        nee = mul(ls.Le, f) * (dot(n, ls.dir) / ls.pdf);
        pl = ls.pdf;
    }
    float3 db;
    const bool ok = bsdf_sample(m, n, wo, [&](int k) { return R(8 + k); }, db);
    if (!ok) db = n;
    P.vx[i] = f4(h.x, (float)prim.mat);
    P.vn[i] = f4(n, 0.f);
    P.vwo[i] = f4(wo, 0.f);
    P.vdb[i] = f4(db, R(3));                 // xi_t: technique selection
    P.vdn[i] = f4(ls.dir, pl > 0.f ? 1.f : 0.f);
    P.vnee[i] = f4(nee, pl);
    P.bsdf_ok[i] = ok ? 1 : 0;
    P.pending[i] = 1;
    int slot = -1;
    if (guided) {
        slot = atomicAdd(&P.qcount[bounce], 1);
        P.qx[slot] = f4(h.x, 0.f);
        P.qwo[slot] = f4(wo, 0.f);
        P.qn[slot] = f4(n, 0.f);
        P.qxi[slot] = make_float4(R(4), R(5), R(6), R(7));
        P.qdb[slot] = P.vdb[i];
        P.qdn[slot] = P.vdn[i];
    }
    P.slot[i] = slot;
}

__device__ __forceinline__ void update_path(Paths &P, const Frame &F, int bounce, int64_t i) {
    if (!P.pending[i]) return;
    P.pending[i] = 0;
    const Scene &S = c_scene;
    const int px = (int)(i % F.width), py = frame_row(F, (int)(i / F.width));
    const uint64_t pix = (uint64_t)py * F.width + px;
    const float4 vx = P.vx[i];
    const Mat &m = S.mats[(int)vx.w];
    const float3 x = xyz(vx), n = xyz(P.vn[i]), wo = xyz(P.vwo[i]);
    const float4 vdb = P.vdb[i], vdn = P.vdn[i], vnee = P.vnee[i];
    float3 v = xyz(vdb);
    float qv = 0.f, qn = 0.f, ce = 0.f;
    bool tech = false;
    const int slot = P.slot[i];
    if (slot >= 0) {
        const float4 o0 = P.qout[2 * slot], o1 = P.qout[2 * slot + 1];
        v = xyz(o0);
        qv = o0.w;
        qn = o1.x;
        ce = o1.y;
        tech = o1.z > 0.5f;
    }
    float4 beta = P.beta[i], L = P.L[i];
    // NEE with the balance heuristic against the full blend q-hat at its direction
    if (vdn.w > 0.f) {
        const float qhn = ce * qn + (1.f - ce) * bsdf_pdf(m, n, wo, xyz(vdn));
        const float w = vnee.w / (vnee.w + qhn);
        L.x += beta.x * vnee.x * w;
        L.y += beta.y * vnee.y * w;
        L.z += beta.z * vnee.z * w;
    }
    const float pb = bsdf_pdf(m, n, wo, v);
    const float qh = ce * qv + (1.f - ce) * pb;  // guided_pdf (guiding.cpp:81-85)
    const float cs = dot(n, v);
    const bool usable = (tech || P.bsdf_ok[i]) && qh > 0.f && isfinite(qh);
    const float3 fc = usable && cs > 0.f ? bsdf_eval(m, n, wo, v) * cs : f3(0.f, 0.f, 0.f);
    float4 nb = make_float4(beta.x * fc.x / qh, beta.y * fc.y / qh, beta.z * fc.z / qh, 0.f);
    bool live = usable && (nb.x > 0.f || nb.y > 0.f || nb.z > 0.f);
    if (live && bounce + 1 >= F.rr_depth) {  // Russian roulette from depth 5, capped at 0.95
        const float q = fminf(0.95f, lum(f3(nb.x, nb.y, nb.z)));
        if (rnd(F.seed, pix, F.iter, (uint32_t)bounce + 1, 31) >= q) {
            live = false;
        } else {
            nb.x /= q;
            nb.y /= q;
            nb.z /= q;
        }
    }
    const int r = P.rank[i];
    // training record (SPEC PathVertexRecord).  A direction whose radiance was never
    // traced (the path ended by Russian roulette or at the depth limit) has an
    // unknown, not a zero, target: such vertices are dropped; a zero f cos is a
    // genuine p = 0 sample and is kept.
    const bool zero_f = !(fc.x > 0.f || fc.y > 0.f || fc.z > 0.f);
    if (r >= 0 && usable && (zero_f || (live && bounce + 1 < F.max_depth))) {
        const int k = P.rcnt[r]++;
        const size_t at = (size_t)k * P.ncap + r;
        P.rx[at] = f4(x, 0.f);
        P.rwo[at] = f4(wo, qh);
        P.rn[at] = f4(n, pb);
        P.rwi[at] = f4(v, 0.f);
        P.rfc[at] = f4(fc, 0.f);
        P.rbeta[at] = zero_f ? make_float4(0.f, 0.f, 0.f, 0.f) : nb;
        P.rlb[at] = L;
    }
    P.L[i] = L;
    if (!live) {
        P.alive[i] = 0;
        return;
    }
    P.beta[i] = nb;
    P.o[i] = f4(x + n * kEps, 0.f);
    P.d[i] = f4(v, 0.f);
    P.prev_pdf[i] = qh;
}

// The bounce kernels walk the compacted list of paths alive at the bounce's
// start (warp-uniform strides, so whole warps vote together); late bounces,
// where Russian roulette has ended most paths, touch only the survivors.
__global__ void k_isect(Paths P, Frame F, int bounce, int guided) {
    pdl_trigger();
    pdl_wait();  // every input comes from the previous kernel on the stream
    const int *list = P.act[bounce & 1];
    const int cnt = P.nact[bounce];
    const int lane = threadIdx.x & 31;
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); w < cnt;
         w += (int64_t)gridDim.x * blockDim.x)
        if (w + lane < cnt) isect_path(P, F, bounce, guided, list[w + lane]);
}

// update, then append the paths still alive to the next bounce's list
// (one warp-aggregated atomic per warp; the list order never changes a path's
// arithmetic, so the film stays bitwise deterministic)
__global__ void k_update(Paths P, Frame F, int bounce) {
    pdl_trigger();
    pdl_wait();  // every input comes from the previous kernel on the stream
    const int *list = P.act[bounce & 1];
    int *next = P.act[(bounce + 1) & 1];
    int *ncount = &P.nact[bounce + 1];
    const int cnt = P.nact[bounce];
    const int lane = threadIdx.x & 31;
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); w < cnt;
         w += (int64_t)gridDim.x * blockDim.x) {
        const bool valid = w + lane < cnt;
        const int i = valid ? list[w + lane] : 0;
        if (valid) update_path(P, F, bounce, i);
        const bool keep = valid && P.alive[i] != 0;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        int base = 0;
        if (lane == 0 && bal) base = atomicAdd(ncount, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) next[base + __popc(bal & ((1u << lane) - 1u))] = i;
    }
}

// Exclusive prefix sum of the collected paths' record counts, in two passes:
// k_scan_local scans 1024-rank blocks (warp shuffles) and writes block totals,
// k_scan_blocks scans the block totals (ncap <= 1024^2); k_records adds both.
__device__ inline int warp_incl_scan(int v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) >= o) v += u;
    }
    return v;
}

__global__ void k_scan_local(Paths P) {
    pdl_trigger();
    pdl_wait();  // every input comes from the previous kernel on the stream
    __shared__ int wsum[32];
    const int64_t k = (int64_t)blockIdx.x * 1024 + threadIdx.x;
    const int c = (k < P.ncap && P.rpix[k] >= 0) ? P.rcnt[k] : 0;
    const int incl = warp_incl_scan(c);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
        const int t = warp_incl_scan(wsum[lane]);
        wsum[lane] = t;
    }
    __syncthreads();
    const int excl = incl - c + (w > 0 ? wsum[w - 1] : 0);
    if (k < P.ncap) P.roff[k] = excl;
    if (threadIdx.x == 1023) P.bsum[blockIdx.x] = excl + c;
}

__global__ void k_scan_blocks(Paths P, int nblocks) {
    pdl_trigger();
    pdl_wait();  // every input comes from the previous kernel on the stream
    __shared__ int wsum[32];
    const int i = threadIdx.x;
    const int c = i < nblocks ? P.bsum[i] : 0;
    const int incl = warp_incl_scan(c);
    const int w = i >> 5, lane = i & 31;
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
        const int t = warp_incl_scan(wsum[lane]);
        wsum[lane] = t;
    }
    __syncthreads();
    const int excl = incl - c + (w > 0 ? wsum[w - 1] : 0);
    if (i < nblocks) P.boff[i] = excl;
    if (i == 1023) {
        const unsigned long long total = (unsigned long long)(excl + c);
        P.ctr[3] += total;
        P.ctr[4] = total;
    }
}

// per-vertex incident radiance by back-propagation -> TrainingSamples
__global__ void k_records(Paths P) {
    pdl_trigger();
    pdl_wait();  // every input comes from the previous kernel on the stream
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= P.ncap) return;
    const int pi = P.rpix[r];
    if (pi < 0) return;
    const int cnt = P.rcnt[r];
    const float4 Le = P.L[pi];
    // more samples than the capacity S: keep an evenly spread S of them (sample o
    // goes to slot floor(o S / T) when that slot changes), not the first S rows
    const int64_t T = (int64_t)P.ctr[4], Sc = P.cap_samples;
    for (int k = 0; k < cnt; ++k) {
        int64_t o = (int64_t)P.roff[r] + P.boff[r >> 10] + k;
        if (T > Sc) {
            const int64_t a = o * Sc / T, b = (o + 1) * Sc / T;
            if (b == a) continue;
            o = a;
        }
        const size_t at = (size_t)k * P.ncap + r;
        const float4 b = P.rbeta[at], lb = P.rlb[at], fc = P.rfc[at];
        // incident radiance along omega_i: everything gathered after this vertex
        const float3 li = f3(b.x > 0.f ? (Le.x - lb.x) / b.x : 0.f, b.y > 0.f ? (Le.y - lb.y) / b.y : 0.f,
                             b.z > 0.f ? (Le.z - lb.z) / b.z : 0.f);
        float p = lum(mul(xyz(fc), li));  // luminance of f_s L_i |cos| (SPEC guider)
        if (!(p > 0.f) || !isfinite(p)) p = 0.f;
        const float4 x = P.rx[at], wo = P.rwo[at], n = P.rn[at], wi = P.rwi[at];
        nasg_train_sample s;
        s.position[0] = x.x; s.position[1] = x.y; s.position[2] = x.z;
        s.p_value = p;
        s.omega_o[0] = wo.x; s.omega_o[1] = wo.y; s.omega_o[2] = wo.z;
        s.q_sampling = wo.w;
        s.normal[0] = n.x; s.normal[1] = n.y; s.normal[2] = n.z;
        s.bsdf_pdf_at_wi = n.w;
        s.omega_i[0] = wi.x; s.omega_i[1] = wi.y; s.omega_i[2] = wi.z;
        s.pad = 0.f;
        P.samples[o] = s;
    }
}

__global__ void k_accumulate(Paths P, float w, int first, int depth) {
    pdl_trigger();
    pdl_wait();  // every input comes from the previous kernel on the stream
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {  // guided vertices of the iteration: the per-bounce query counts
        unsigned long long q = 0;
        for (int k = 0; k < depth; ++k) q += (unsigned long long)P.qcount[k];
        P.ctr[1] = q;
    }
    if (i >= P.n) return;
    float4 L = P.L[i];
    if (!(isfinite(L.x) && isfinite(L.y) && isfinite(L.z))) {  // discarded, counted, never on film
        atomicAdd(&P.ctr[2], 1ull);
        L = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    L.w = 1.f;
    P.frame[i] = L;
    float4 f = first ? make_float4(0.f, 0.f, 0.f, 0.f) : P.film[i];
    f.x += w * L.x;
    f.y += w * L.y;
    f.z += w * L.z;
    f.w += w;
    P.film[i] = f;
}

// ------------------------------------------------------------------ scenes --
static Prim quad(float3 p, float3 u, float3 v, int mat) {
    Prim q{};
    q.type = kQuad;
    q.mat = mat;
    q.p = p;
    q.u = u;
    q.v = v;
    return q;
}
static Prim sphere(float3 c, float r, int mat) {
    Prim s{};
    s.type = kSphere;
    s.mat = mat;
    s.p = c;
    s.r = r;
    return s;
}
static Mat mat(int type, float3 albedo, float e = 0.f, float3 em = f3(0.f, 0.f, 0.f)) {
    Mat m{};
    m.type = type;
    m.albedo = albedo;
    m.exponent = e;
    m.emission = em;
    return m;
}

static void look_at(Camera &c, float3 pos, float3 at, float3 up, float vfov_deg, int w, int h) {
    c.pos = pos;
    c.fwd = normalize(at - pos);
    const float3 r = normalize(cross(c.fwd, up));
    const float3 u = cross(r, c.fwd);
    const float th = tanf(vfov_deg * 0.5f * kPiF / 180.f);
    c.right = r * (th * (float)w / (float)h);
    c.up = u * th;
    c.width = w;
    c.height = h;
}

// Cornell-style box [0,1]^3 open at z = 0 (SPEC Scene: spheres, axis-aligned quads,
// lambertian / phong / mirror, area emitters); CRACK hides the light above a
// partition so the room is lit through a narrow slit (anisotropic indirect light,
// the case PAPER §7 targets).
static bool build_scene(int kind, int w, int h, Scene &s) {
    std::memset(&s, 0, sizeof(s));
    const float3 white = f3(0.73f, 0.73f, 0.73f), red = f3(0.65f, 0.05f, 0.05f), green = f3(0.12f, 0.45f, 0.15f);
    int np = 0, nm = 0;
    auto addm = [&](Mat m) { s.mats[nm] = m; return nm++; };
    auto addp = [&](Prim p) { s.prims[np++] = p; };
    if (kind == NASG_SCENE_FURNACE || kind == NASG_SCENE_DARK) {
        // SPEC trace_path examples: constant environment 1 over a lambertian plane
        // of albedo 0.5 (pixel expectation 0.5); DARK: no emitters, zero environment
        const int m0 = addm(mat(kLambert, f3(0.5f, 0.5f, 0.5f)));
        addp(quad(f3(-50.f, -50.f, 0.f), f3(100.f, 0.f, 0.f), f3(0.f, 100.f, 0.f), m0));
        s.env = kind == NASG_SCENE_FURNACE ? f3(1.f, 1.f, 1.f) : f3(0.f, 0.f, 0.f);
        look_at(s.cam, f3(0.f, -1.2f, 1.6f), f3(0.f, 0.f, 0.f), f3(0.f, 0.f, 1.f), 40.f, w, h);
        const float lo[3] = {-1.5f, -1.5f, -0.5f}, hi[3] = {1.5f, 1.5f, 2.5f};
        std::memcpy(s.bmin, lo, sizeof(lo));
        std::memcpy(s.bmax, hi, sizeof(hi));
    } else if (kind == NASG_SCENE_BOX || kind == NASG_SCENE_CRACK || kind == NASG_SCENE_ATTIC ||
               kind == NASG_SCENE_INDIRECT) {
        const bool indirect = kind == NASG_SCENE_INDIRECT;
        const bool crack = kind != NASG_SCENE_BOX && !indirect;
        const int mw = addm(mat(kLambert, white)), mr = addm(mat(kLambert, red)), mg = addm(mat(kLambert, green));
        const int mgl = addm(mat(kPhong, f3(0.8f, 0.8f, 0.8f), 60.f));
        const int mmi = addm(mat(kMirror, f3(0.95f, 0.95f, 0.95f)));
        const float3 le = kind == NASG_SCENE_BOX ? f3(17.f, 12.f, 4.f)
                          : (kind == NASG_SCENE_CRACK ? f3(60.f, 48.f, 30.f)
                             : (indirect ? f3(100.f, 80.f, 50.f) : f3(400.f, 320.f, 200.f)));
        const int mle = addm(mat(kEmitter, f3(0.f, 0.f, 0.f), 0.f, le));
        addp(quad(f3(0.f, 0.f, 0.f), f3(0.f, 0.f, 1.f), f3(1.f, 0.f, 0.f), crack ? mgl : mw));
        addp(quad(f3(0.f, 1.f, 0.f), f3(1.f, 0.f, 0.f), f3(0.f, 0.f, 1.f), mw));  // ceiling
        addp(quad(f3(0.f, 0.f, 1.f), f3(0.f, 1.f, 0.f), f3(1.f, 0.f, 0.f), mw));  // back
        addp(quad(f3(0.f, 0.f, 0.f), f3(0.f, 1.f, 0.f), f3(0.f, 0.f, 1.f), mr));  // left
        addp(quad(f3(1.f, 0.f, 0.f), f3(0.f, 0.f, 1.f), f3(0.f, 1.f, 0.f), mg));  // right
        if (indirect) {  // SPEC acceptance 7's "indirect-illumination box": a panel under the
                         // ceiling facing up, so everything below it is lit only by light that
                         // bounced off the ceiling and upper walls (NEE finds no unoccluded light)
            addp(quad(f3(0.35f, 0.8f, 0.35f), f3(0.f, 0.f, 0.3f), f3(0.3f, 0.f, 0.f), mle));
            addp(sphere(f3(0.3f, 0.2f, 0.6f), 0.2f, mw));
            addp(sphere(f3(0.72f, 0.18f, 0.35f), 0.18f, mmi));
        } else if (kind == NASG_SCENE_BOX) {
            addp(quad(f3(0.4f, 0.999f, 0.4f), f3(0.2f, 0.f, 0.f), f3(0.f, 0.f, 0.2f), mle));
            addp(sphere(f3(0.3f, 0.2f, 0.62f), 0.2f, mgl));
            addp(sphere(f3(0.72f, 0.18f, 0.35f), 0.18f, mmi));
        } else {
            // partition at y = 0.85 with a slit 0.47 < x < 0.53; the light lies above it
            addp(quad(f3(0.f, 0.85f, 0.f), f3(0.47f, 0.f, 0.f), f3(0.f, 0.f, 1.f), mw));
            addp(quad(f3(0.53f, 0.85f, 0.f), f3(0.47f, 0.f, 0.f), f3(0.f, 0.f, 1.f), mw));
            if (kind == NASG_SCENE_CRACK)  // light at the ceiling, partly visible through the slit
                addp(quad(f3(0.2f, 0.999f, 0.3f), f3(0.6f, 0.f, 0.f), f3(0.f, 0.f, 0.4f), mle));
            else  // ATTIC: light lying on the partition facing the ceiling; the room below
                  // only sees light that bounced off the ceiling and came through the slit
                addp(quad(f3(0.05f, 0.86f, 0.3f), f3(0.f, 0.f, 0.4f), f3(0.3f, 0.f, 0.f), mle));
            addp(sphere(f3(0.3f, 0.2f, 0.6f), 0.2f, mw));
            addp(sphere(f3(0.72f, 0.18f, 0.35f), 0.18f, mmi));
        }
        s.env = f3(0.f, 0.f, 0.f);
        look_at(s.cam, f3(0.5f, 0.5f, -1.25f), f3(0.5f, 0.45f, 0.5f), f3(0.f, 1.f, 0.f), 40.f, w, h);
        const float lo[3] = {-0.05f, -0.05f, -0.05f}, hi[3] = {1.05f, 1.05f, 1.05f};
        std::memcpy(s.bmin, lo, sizeof(lo));
        std::memcpy(s.bmax, hi, sizeof(hi));
    } else {
        return false;
    }
    s.nprims = np;
    float area = 0.f;
    for (int i = 0; i < np; ++i) {
        const Prim &p = s.prims[i];
        if (s.mats[p.mat].type != kEmitter) continue;
        if (p.type != kQuad || s.nlights == kMaxLights) return false;
        const float3 c = cross(p.u, p.v);
        area += sqrtf(dot(c, c));
        s.light_prim[s.nlights] = i;
        s.light_cdf[s.nlights++] = area;
    }
    for (int k = 0; k < s.nlights; ++k) s.light_cdf[k] /= area;
    s.light_area_total = area;
    return true;
}

}  // namespace rt
}  // namespace nasg

using namespace nasg;
using namespace nasg::rt;

struct nasg_render {
    nasg_ctx *ctx = nullptr;
    nasg_render_config cfg{};
    Scene scene{};
    Paths P{};
    cudaStream_t stream = nullptr;
    int rows = 0;
    int64_t iter = 0;
    double l = 1.0, l_min = 1.0;
    double wsum = 0.0;
    uint64_t launches = 0;
    std::vector<void *> bufs;
    int nranks = 1;
    int nsm = 148;
    bool pdl = true;  // programmatic dependent launch of the trace chain (serial loop only)
    double *h_acc = nullptr;   // pinned 2 x 5: training statistics (lazy_train_stats / pipelined)
    unsigned long long *h_ctr = nullptr;  // pinned: the iteration's counters
    bool acc_pending[2] = {false, false};
    // pipelined: trace i+1 overlaps training i (its own stream); two sample buffers
    nasg_train_sample *samples_buf[2] = {nullptr, nullptr};
    cudaStream_t tstream = nullptr;
    cudaEvent_t ev_train = nullptr, ev_acc[2] = {nullptr, nullptr};
    bool inflight = false;     // trace of iteration `iter` already launched
};

namespace {

thread_local char g_rerr[256];

int rfail(int code, const char *msg) {
    std::snprintf(g_rerr, sizeof(g_rerr), "%s", msg);
    return code;
}

#define RCUDA(x)                                                        \
    do {                                                                \
        cudaError_t e_ = (x);                                           \
        if (e_ != cudaSuccess) return rfail(NASG_ERR_CUDA, cudaGetErrorString(e_)); \
    } while (0)

template <class T>
int alloc(nasg_render *r, T **p, size_t count) {
    void *q = nullptr;
    RCUDA(cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T)));
    r->bufs.push_back(q);
    *p = static_cast<T *>(q);
    return NASG_OK;
}

unsigned grid_of(int64_t n) { return (unsigned)((n + kBlock - 1) / kBlock); }

}  // namespace

extern "C" {

void nasg_render_config_default(nasg_render_config *c) {
    if (!c) return;
    std::memset(c, 0, sizeof(*c));
    c->scene = NASG_SCENE_BOX;
    c->width = 256;
    c->height = 256;
    c->row_begin = 0;
    c->row_end = 0;
    c->seed = 1;
    c->max_depth = 16;
    c->rr_depth = 5;
    c->guiding = 1;
    c->collect = 1;
    c->ramp = 1;
    c->schedule_m = 4;
    c->schedule_b = 64;
    c->nee = 1;
}

int nasg_render_scene_bounds(int scene, float bmin[3], float bmax[3]) {
    Scene s;
    if (!bmin || !bmax || !build_scene(scene, 16, 16, s)) return NASG_ERR_INVALID;
    for (int k = 0; k < 3; ++k) {
        bmin[k] = s.bmin[k];
        bmax[k] = s.bmax[k];
    }
    return NASG_OK;
}

int nasg_render_destroy(nasg_render *r) {
    if (!r) return NASG_OK;
    DeviceScope ds_(ctx_device(r->ctx));
    if (r->stream) cudaStreamSynchronize(r->stream);
    if (r->tstream) cudaStreamSynchronize(r->tstream);
    if (r->cfg.pipelined && r->ctx) ctx_set_pdl(r->ctx, true);
    if (r->ctx) ctx_set_query_pdl(r->ctx, false);
    for (void *p : r->bufs) cudaFree(p);
    if (r->h_acc) cudaFreeHost(r->h_acc);
    if (r->h_ctr) cudaFreeHost(r->h_ctr);
    if (r->tstream) cudaStreamDestroy(r->tstream);
    for (cudaEvent_t e : {r->ev_train, r->ev_acc[0], r->ev_acc[1]})
        if (e) cudaEventDestroy(e);
    if (r->stream) cudaStreamDestroy(r->stream);
    delete r;
    return NASG_OK;
}

int nasg_render_create(nasg_ctx *ctx, const nasg_render_config *cfg, nasg_render **out) {
    if (!ctx || !cfg || !out) return NASG_ERR_INVALID;
    DeviceScope ds_(ctx_device(ctx));
    *out = nullptr;
    nasg_render_config c = *cfg;
    int band_rows = 0;  // rows owned with interleaving
    if (c.row_band > 0) {
        if (c.nshards < 1 || c.shard < 0 || c.shard >= c.nshards || c.height <= 0) return NASG_ERR_INVALID;
        const int nb = (c.height + c.row_band - 1) / c.row_band;
        for (int k = c.shard; k < nb; k += c.nshards) band_rows += std::min(c.height, (k + 1) * c.row_band) - k * c.row_band;
        if (band_rows == 0) return NASG_ERR_INVALID;  // more shards than bands
        c.row_begin = 0;
        c.row_end = band_rows;
    } else {
        c.row_band = 0;
        c.shard = 0;
        c.nshards = 1;
    }
    if (c.row_end <= 0) c.row_end = c.height;
    if (c.width <= 0 || c.height <= 0 || c.row_begin < 0 || c.row_end > c.height || c.row_begin >= c.row_end ||
        c.max_depth < 1 || c.max_depth > kMaxDepthCap || c.schedule_m < 1 || c.schedule_b < 1)
        return NASG_ERR_INVALID;
    auto *r = new nasg_render();
    r->ctx = ctx;
    r->cfg = c;
    if (!build_scene(c.scene, c.width, c.height, r->scene)) {
        delete r;
        return NASG_ERR_INVALID;
    }
    r->nranks = std::max(1, ctx_nranks(ctx));
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&r->nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    int rc = NASG_OK;
    auto fail_out = [&](int code) {
        nasg_render_destroy(r);
        return code;
    };
    if (cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking) != cudaSuccess) return fail_out(NASG_ERR_CUDA);
    if (cudaMallocHost(&r->h_acc, 10 * sizeof(double)) != cudaSuccess) return fail_out(NASG_ERR_OOM);
    if (cudaMallocHost(&r->h_ctr, 8 * sizeof(unsigned long long)) != cudaSuccess) return fail_out(NASG_ERR_OOM);
    ctx_set_query_pdl(ctx, !c.pipelined);
    if (c.pipelined) {
        // training shares the SMs with concurrent tracing: no early-started CTAs parked on them
        ctx_set_pdl(ctx, false);
        r->pdl = false;
        if (cudaStreamCreateWithFlags(&r->tstream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&r->ev_train, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&r->ev_acc[0], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&r->ev_acc[1], cudaEventDisableTiming) != cudaSuccess)
            return fail_out(NASG_ERR_CUDA);
    }
    r->rows = c.row_end - c.row_begin;
    Paths &P = r->P;
    P.n = (int64_t)r->rows * c.width;
    // this rank's share of the capacity S; record storage bounded to 4 S paths
    P.cap_samples = std::max<int64_t>(1, (ctx_sample_capacity(ctx) + r->nranks - 1) / r->nranks);
    // (and to the 1024 x 1024 ranks the two-pass scan covers)
    r->l_min = std::max(1.0, std::sqrt((double)P.n / (4.0 * (double)P.cap_samples)));
    for (;;) {
        const int64_t ntx_max = (int64_t)std::ceil(c.width / r->l_min) + 1;
        const int64_t nty_max = (int64_t)std::ceil(r->rows / r->l_min) + 2;
        P.ncap = ntx_max * nty_max;
        if (P.ncap <= 1024 * 1024) break;
        r->l_min *= 1.05;
    }
    r->l = r->l_min;
#define A(ptr, count) \
    if ((rc = alloc(r, &(ptr), (size_t)(count))) != NASG_OK) return fail_out(rc);
    A(P.o, P.n) A(P.d, P.n) A(P.beta, P.n) A(P.L, P.n) A(P.prev_pdf, P.n) A(P.alive, P.n) A(P.pending, P.n)
    A(P.vx, P.n) A(P.vn, P.n) A(P.vwo, P.n) A(P.vdb, P.n) A(P.vdn, P.n) A(P.vnee, P.n)
    A(P.slot, P.n) A(P.rank, P.n) A(P.bsdf_ok, P.n) A(P.act[0], P.n) A(P.act[1], P.n) A(P.nact, kMaxDepthCap + 1)
    A(P.qx, P.n) A(P.qwo, P.n) A(P.qn, P.n) A(P.qxi, P.n) A(P.qdb, P.n) A(P.qdn, P.n) A(P.qout, 2 * P.n)
    A(P.qcount, kMaxDepthCap)
    const size_t nrec = (size_t)P.ncap * kMaxDepthCap;
    A(P.rx, nrec) A(P.rwo, nrec) A(P.rn, nrec) A(P.rwi, nrec) A(P.rfc, nrec) A(P.rbeta, nrec) A(P.rlb, nrec)
    A(P.rcnt, P.ncap) A(P.rpix, P.ncap) A(P.roff, P.ncap) A(P.bsum, 1024) A(P.boff, 1024)
    A(P.ctr, 8) A(P.film, P.n) A(P.frame, P.n) A(r->samples_buf[0], P.cap_samples)
    if (c.pipelined) A(r->samples_buf[1], P.cap_samples)
    P.samples = r->samples_buf[0];
#undef A
    if (cudaMemsetAsync(P.film, 0, P.n * sizeof(float4), r->stream) != cudaSuccess) return fail_out(NASG_ERR_CUDA);
    *out = r;
    return NASG_OK;
}

uint64_t nasg_render_kernel_launches(nasg_render *r) { return r ? r->launches : 0; }

namespace {

// One iteration's tracing + collection on the render stream (everything but
// the accumulation): camera rays, up to max_depth bounces of intersection,
// guided scattering through the fused network query and the update, then the
// collected paths' training records into `samples`.
int launch_trace(nasg_render *r, int64_t iter, double b, nasg_train_sample *samples) {
    const nasg_render_config &c = r->cfg;
    Paths &P = r->P;
    cudaStream_t s = r->stream;
    P.samples = samples;
    RCUDA(cudaMemcpyToSymbolAsync(c_scene, &r->scene, sizeof(Scene), 0, cudaMemcpyHostToDevice, s));
    Frame F{};
    F.seed = c.seed;
    F.iter = (uint64_t)iter;
    F.width = c.width;
    F.height = c.height;
    F.row0 = c.row_begin;
    F.band = c.row_band;
    F.shard = c.shard;
    F.nshards = c.nshards;
    F.l = (float)r->l;
    F.tile_row0 = c.row_band > 0 ? 0 : (int)std::floor(c.row_begin / r->l);
    F.ntx = (int)std::ceil(c.width / r->l) + 1;
    F.collect = c.collect;
    F.max_depth = c.max_depth;
    F.rr_depth = c.rr_depth;
    F.nee = c.nee;
    RCUDA(cudaMemsetAsync(P.ctr, 0, 8 * sizeof(unsigned long long), s));
    RCUDA(cudaMemsetAsync(P.qcount, 0, kMaxDepthCap * sizeof(int), s));
    RCUDA(cudaMemsetAsync(P.nact, 0, (kMaxDepthCap + 1) * sizeof(int), s));
    if (c.collect) RCUDA(cudaMemsetAsync(P.rpix, 0xff, P.ncap * sizeof(int), s));
    // the buffer is usually full (kept = S): shuffle it on a host thread while the GPU traces
    if (c.collect) {
        const int rc = ctx_prefetch_shuffle(r->ctx, P.cap_samples);
        if (rc != NASG_OK) return rc;
    }
    const unsigned g = grid_of(P.n);
    launch_pdl(r->pdl, k_begin, dim3(g), dim3(kBlock), 0, s, P, F);
    r->launches++;
    const bool guided = b > 0.0;
    const unsigned gb = std::min<unsigned>(g, (unsigned)r->nsm * 8u);  // list-walking bounce kernels
    // per-bounce list lengths and query counts (zeroed above): no reset launches
    for (int bounce = 0; bounce < c.max_depth; ++bounce) {
        launch_pdl(r->pdl, k_isect, dim3(gb), dim3(kBlock), 0, s, P, F, bounce, guided ? 1 : 0);
        r->launches += 1;
        if (guided) {
            const int rc = nasg_query_shade(r->ctx, P.n, P.qcount + bounce, (const float *)P.qx, (const float *)P.qwo,
                                            (const float *)P.qn, (const float *)P.qxi, (const float *)P.qdb,
                                            (const float *)P.qdn, (float)b, (float *)P.qout, s);
            if (rc != NASG_OK) return rc;
        }
        launch_pdl(r->pdl, k_update, dim3(gb), dim3(kBlock), 0, s, P, F, bounce);
        r->launches++;
    }
    if (c.collect) {
        // pipelined: the training two iterations back read this sample buffer
        if (r->ev_train) RCUDA(cudaStreamWaitEvent(s, r->ev_train, 0));
        const int nb = (int)((P.ncap + 1023) / 1024);
        launch_pdl(r->pdl, k_scan_local, dim3(nb), dim3(1024), 0, s, P);
        launch_pdl(r->pdl, k_scan_blocks, dim3(1), dim3(1024), 0, s, P, nb);
        launch_pdl(r->pdl, k_records, dim3(grid_of(P.ncap)), dim3(kBlock), 0, s, P);
        r->launches += 3;
    }
    RCUDA(cudaGetLastError());
    return NASG_OK;
}

// SPEC accumulate: the progressive w_i ramp (or the plain mean)
int launch_accumulate(nasg_render *r, int64_t iter) {
    const nasg_render_config &c = r->cfg;
    const int64_t mb = (int64_t)c.schedule_m * c.schedule_b;
    const double w = c.ramp ? (double)std::min<int64_t>(iter + 1, mb) / (double)mb : 1.0;
    launch_pdl(r->pdl, k_accumulate, dim3(grid_of(r->P.n)), dim3(kBlock), 0, r->stream, r->P, (float)w, iter == 0 ? 1 : 0,
               r->cfg.max_depth);
    r->launches++;
    r->wsum += w;
    RCUDA(cudaGetLastError());
    return NASG_OK;
}

double blend_of(const nasg_render *r, int64_t iter) {
    return r->cfg.guiding ? nasg_blend_coefficient(iter, r->cfg.schedule_m, r->cfg.schedule_b) : 0.0;
}

}  // namespace

int nasg_render_iteration(nasg_render *r, nasg_render_stats *stats) {
    nasg::NvtxRange nv_("nasg_render_iteration");
    if (!r) return NASG_ERR_INVALID;
    DeviceScope ds_(ctx_device(r->ctx));
    const nasg_render_config &c = r->cfg;
    Paths &P = r->P;
    cudaStream_t s = r->stream;
    const int64_t i = r->iter;
    const double b = blend_of(r, i);
    int rc;
#ifdef NASG_RENDER_PROF
    RProf &pf = g_rprof;
    if (!pf.a) {
        cudaEventCreate(&pf.a); cudaEventCreate(&pf.b); cudaEventCreate(&pf.c); cudaEventCreate(&pf.pc);
    }
    auto T0 = std::chrono::steady_clock::now();
    const bool have_prev = pf.n > 0;
    cudaEventRecord(pf.a, s);
#endif
    if (!c.pipelined || !r->inflight) {
        if ((rc = launch_trace(r, i, b, r->samples_buf[c.pipelined ? (i & 1) : 0])) != NASG_OK) return rc;
    }
    if ((rc = launch_accumulate(r, i)) != NASG_OK) return rc;
    unsigned long long *ctr = r->h_ctr;  // pinned: the read-back never waits behind an upload
#ifdef NASG_RENDER_PROF
    cudaEventRecord(pf.b, s);
    pf.host[0] += ms_since(T0);
    auto T1 = std::chrono::steady_clock::now();
#endif
    RCUDA(cudaMemcpyAsync(ctr, P.ctr, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    RCUDA(cudaStreamSynchronize(s));
#ifdef NASG_RENDER_PROF
    pf.host[1] += ms_since(T1);
    {
        float x = 0.f;
        cudaEventElapsedTime(&x, pf.a, pf.b);
        pf.gpu[0] += x;
        if (have_prev) {
            cudaEventElapsedTime(&x, pf.pc, pf.a);  // previous train end -> this trace start
            pf.gpu[2] += x;
            ++pf.ng;
        }
    }
    auto T2 = std::chrono::steady_clock::now();
#endif
    r->inflight = false;
    nasg_render_stats st{};
    st.iteration = i;
    st.b = b;
    st.stride = r->l;
    st.paths = P.n;
    st.vertices = (int64_t)ctr[0];
    st.guided_vertices = (int64_t)ctr[1];
    st.nonfinite_paths = (int64_t)ctr[2];
    st.collected = (int64_t)ctr[4];
    st.kept = std::min<int64_t>(st.collected, P.cap_samples);
    if (c.collect) {
        // l = max(1, l sqrt(s / S)) (guiding.cpp:178-182) with the record-storage floor
        r->l = std::max(r->l_min, nasg_stride_update(r->l, (uint64_t)st.collected, (uint64_t)P.cap_samples));
    }
    if (c.pipelined) {
        // stats of the training two iterations back (finished: this iteration's
        // queries waited on the snapshot it published, or on its event below)
        const int slot = (int)(i & 1);
        if (r->acc_pending[slot]) {
            RCUDA(cudaEventSynchronize(r->ev_acc[slot]));
            ctx_stats_from_acc(r->h_acc + 5 * slot, &st.train);
            r->acc_pending[slot] = false;
        }
        // trace iteration i+1 now, against the snapshot of training i-1 ...
        if ((rc = launch_trace(r, i + 1, blend_of(r, i + 1), r->samples_buf[(i + 1) & 1])) != NASG_OK) return rc;
        r->inflight = true;
        // ... while training i runs on its own stream and publishes for i+2
        if (c.collect) {
            rc = nasg_train_iteration(r->ctx, st.kept, r->samples_buf[i & 1], b, nullptr, r->tstream);
            if (rc != NASG_OK) return rc;
            if (ctx_train_stats_async(r->ctx, r->h_acc + 5 * slot, r->tstream) != NASG_OK) return NASG_ERR_CUDA;
            RCUDA(cudaEventRecord(r->ev_acc[slot], r->tstream));
            RCUDA(cudaEventRecord(r->ev_train, r->tstream));
            r->acc_pending[slot] = true;
        }
    } else {
        if (c.lazy_train_stats && r->acc_pending[0]) {  // the previous training finished before the sync above
            ctx_stats_from_acc(r->h_acc, &st.train);
            r->acc_pending[0] = false;
        }
        if (c.collect) {
            // Trainer::train_iteration on this rank's buffer (data-parallel across ranks)
            rc = nasg_train_iteration(r->ctx, st.kept, r->samples_buf[0], b, c.lazy_train_stats ? nullptr : &st.train, s);
            if (rc != NASG_OK) return rc;
            if (c.lazy_train_stats) {
                if (ctx_train_stats_async(r->ctx, r->h_acc, s) != NASG_OK) return NASG_ERR_CUDA;
                r->acc_pending[0] = true;
            }
        }
    }
#ifdef NASG_RENDER_PROF
    pf.host[2] += ms_since(T2);
    cudaEventRecord(pf.pc, s);
    ++pf.n;
#endif
    ++r->iter;
    if (stats) *stats = st;
    return NASG_OK;
}

int nasg_render_image(nasg_render *r, float *rgb, int which) {
    if (!r || !rgb) return NASG_ERR_INVALID;
    DeviceScope ds_(ctx_device(r->ctx));
    const Paths &P = r->P;
    std::vector<float4> h((size_t)P.n);
    RCUDA(cudaMemcpyAsync(h.data(), which ? P.frame : P.film, P.n * sizeof(float4), cudaMemcpyDeviceToHost,
                          r->stream));
    RCUDA(cudaStreamSynchronize(r->stream));
    for (int64_t i = 0; i < P.n; ++i) {
        const float inv = which ? 1.f : (h[i].w > 0.f ? 1.f / h[i].w : 0.f);
        rgb[3 * i] = h[i].x * inv;
        rgb[3 * i + 1] = h[i].y * inv;
        rgb[3 * i + 2] = h[i].z * inv;
    }
    return NASG_OK;
}

double nasg_mape(const float *img, const float *ref, int64_t npix) {
    if (!img || !ref || npix <= 0) return -1.0;
    std::vector<double> e((size_t)npix);
    for (int64_t i = 0; i < npix; ++i) {
        double s = 0.0;
        for (int k = 0; k < 3; ++k) s += std::fabs((double)img[3 * i + k] - ref[3 * i + k]) / (ref[3 * i + k] + 0.01);
        e[i] = s / 3.0;
    }
    std::sort(e.begin(), e.end());
    const int64_t keep = npix - (int64_t)std::floor(npix * 0.001);
    double acc = 0.0;
    for (int64_t i = 0; i < keep; ++i) acc += e[i];
    return acc / (double)keep;
}

}  // extern "C"
