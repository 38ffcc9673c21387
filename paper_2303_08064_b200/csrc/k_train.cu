// fp32 training step (Trainer::train_iteration inner loop, guiding.cpp:236-276):
//
//   K_fb   per 64-row tile, on-chip: encode -> forward (h1..h3, raw) ->
//          KL gradient epilogue (delta4, loss, drops) -> delta3, delta2,
//          delta1 through W^T with the ReLU gates (backward net.hpp:95-110).
//          Activations and deltas are written row-major for K_dw.
//   K_dw   dW_l = h_l^T delta_{l+1}, split over rows into per-CTA partials
//          (fixed split boundaries -> deterministic).
//   K_red  grad = sum of partials in split order; non-finite flag.
//          [multi-GPU: ncclAllReduce of grad + step stats happens here]
//   K_fin  one thread: skip decision (net.hpp:140-144), t, bias corrections,
//          loss/drop accumulation in tile order.
//   K_adam adam_step<float> (net.hpp:146-156) with the reference's float
//          operation order (no FMA contraction), and re-packing of the
//          updated weights for the next step's K_fb.
#include <cstdio>

#include "nasg_internal.h"
#include "nasg_math.cuh"
#include "nasg_refmath.cuh"
#include "simt_gemm.cuh"
#include "tc_common.cuh"  // bf16 image layout (w_off) for the fused re-pack

namespace nasg {

constexpr int kTrainRows = 64;
constexpr int kTLda = kTrainRows + 4;  // 68

// smem carve-up of K_fb (floats).  da holds the packed raw outputs / delta4
// (160 rows for NP <= 160); db the next delta.  For N = 32 (NP = 304) the
// backward runs in place in da instead (tile_layer writes its outputs only
// after every thread has read its last input chunk), which keeps the tile
// inside one SM's shared memory.
constexpr int kOffH0 = 0;
constexpr int kOffH1 = kOffH0 + kIn * kTLda;
constexpr int kOffH2 = kOffH1 + kHidden * kTLda;
constexpr int kOffH3 = kOffH2 + kHidden * kTLda;
constexpr int kOffDA = kOffH3 + kHidden * kTLda;
constexpr bool bwd_in_place(int n) { return packed_width(n) > 160; }
constexpr int off_db(int n) { return bwd_in_place(n) ? kOffDA : kOffDA + 160 * kTLda; }
constexpr int off_w(int n) { return bwd_in_place(n) ? kOffDA + packed_width(n) * kTLda : off_db(n) + kHidden * kTLda; }
constexpr int off_row(int n) { return off_w(n) + 2 * kChunk * 128; }   // 64 x 8 per-row sample data
constexpr int off_loss(int n) { return off_row(n) + kTrainRows * 8; }  // 64 double losses + 64 int states
constexpr size_t fb_smem_f32(int n) { return (size_t)(off_loss(n) + kTrainRows * 3) * sizeof(float); }
static_assert(fb_smem_f32(32) <= 232448 && fb_smem_f32(16) <= 232448, "fp32 trainer tile fits one SM");

// feature-major smem [F][kTLda] -> row-major global [rows][F], rows < valid
template <int F>
__device__ __forceinline__ void store_rows(const float *sm, float *g, int64_t row0, int valid, int tid) {
    for (int idx = tid; idx < kTrainRows * (F / 4); idx += 256) {
        const int r = idx / (F / 4), f4 = (idx % (F / 4)) * 4;
        float4 v;
        if (r < valid) {
            v = make_float4(sm[f4 * kTLda + r], sm[(f4 + 1) * kTLda + r], sm[(f4 + 2) * kTLda + r],
                            sm[(f4 + 3) * kTLda + r]);
        } else {
            v = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        *reinterpret_cast<float4 *>(g + (row0 + r) * F + f4) = v;
    }
}

template <int N>
__global__ void __launch_bounds__(256, 1)
train_fb_kernel(const float *__restrict__ wp, const float *__restrict__ wtp,
                const nasg_train_sample *__restrict__ samples, const uint32_t *__restrict__ order,
                int64_t count, const int64_t *live_count, double gscale, double b, double e, Bounds bd,
                TrainScratch sc, unsigned long long *clamp_count) {
    constexpr int H = packed_header(N), NP = packed_width(N), D = 8 * N + 1;
    extern __shared__ __align__(16) float sm[];
    float *h0 = sm + kOffH0, *h1 = sm + kOffH1, *h2 = sm + kOffH2, *h3 = sm + kOffH3;
    float *da = sm + kOffDA, *db = sm + off_db(N), *wbuf = sm + off_w(N);
    float *rowd = sm + off_row(N);
    double *rloss = reinterpret_cast<double *>(sm + off_loss(N));
    int *rstate = reinterpret_cast<int *>(sm + off_loss(N) + 2 * kTrainRows);
    __shared__ int s_clamped;
    const int tid = threadIdx.x;
    const float *W1 = wp, *W2 = W1 + kIn * kHidden, *W3 = W2 + kHidden * kHidden, *W4 = W3 + kHidden * kHidden;
    const float *T2 = wtp, *T3 = T2 + kHidden * kHidden, *T4 = T3 + kHidden * kHidden;
    if (live_count) count = *live_count;  // the classified step: rows that need the network (order = their list)
    const int ntiles = (int)((count + kTrainRows - 1) / kTrainRows);
    if (tid == 0) s_clamped = 0;
    __syncthreads();
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t row0 = (int64_t)tile * kTrainRows;
        const int valid = (int)min((int64_t)kTrainRows, count - row0);
        // ---- K1: gather + encode (guiding.cpp:209-214, 242-244)
        if (tid < kTrainRows) {
            float *rd = rowd + tid * 8;
            if (tid < valid) {
                const int64_t src = order ? (int64_t)order[row0 + tid] : row0 + tid;
                const float4 *s4 = reinterpret_cast<const float4 *>(samples + src);
                float4 a = s4[0], o = s4[1], n = s4[2], w = s4[3];
                int cl = 0;
                const float xs[3] = {a.x, a.y, a.z};
#pragma unroll
                for (int axis = 0; axis < 3; ++axis) {
                    double t = bd.ext[axis] > 0.0 ? ((double)xs[axis] - (double)bd.bmin[axis]) / bd.ext[axis] : 0.5;
                    if (t < 0.0 || t > 1.0) { ++cl; t = fmin(fmax(t, 0.0), 1.0); }
#pragma unroll
                    for (int i = 0; i < kBins; ++i) {
                        h0[(axis * kBins + i) * kTLda + tid] = ref::one_blob_bin(t, i);
                    }
                }
                h0[57 * kTLda + tid] = o.x; h0[58 * kTLda + tid] = o.y; h0[59 * kTLda + tid] = o.z;
                h0[60 * kTLda + tid] = n.x; h0[61 * kTLda + tid] = n.y; h0[62 * kTLda + tid] = n.z;
                h0[63 * kTLda + tid] = 1.f;
                if (cl) atomicAdd(&s_clamped, cl);
                rd[0] = w.x; rd[1] = w.y; rd[2] = w.z;   // omega_i
                rd[3] = a.w; rd[4] = o.w; rd[5] = n.w;   // p, q_sampling, bsdf_pdf
            } else {
                for (int k = 0; k < kIn; ++k) h0[k * kTLda + tid] = 0.f;
            }
        }
        __syncthreads();
        // ---- K2: forward (net.hpp:69-76)
        tile_layer<kTrainRows, kIn, kEpiRelu, kTLda>(h0, h1, W1, wbuf, nullptr, tid);
        tile_layer<kTrainRows, kHidden, kEpiRelu, kTLda>(h1, h2, W2, wbuf, nullptr, tid);
        tile_layer<kTrainRows, kHidden, kEpiRelu, kTLda>(h2, h3, W3, wbuf, nullptr, tid);
        tile_layer<kTrainRows, kHidden, kEpiNone, kTLda>(h3, da, W4, wbuf, nullptr, tid);
        if constexpr (NP > 128)  // packed columns [128, NP): the further 128-column blocks of W4p
            tile_layer<kTrainRows, kHidden, kEpiNone, kTLda, (NP - 128 < 128 ? NP - 128 : 128)>(
                h3, da + 128 * kTLda, W4 + kHidden * 128, wbuf, nullptr, tid);
        if constexpr (NP > 256)
            tile_layer<kTrainRows, kHidden, kEpiNone, kTLda, NP - 256>(h3, da + 256 * kTLda, W4 + 2 * kHidden * 128,
                                                                        wbuf, nullptr, tid);
        store_rows<kIn>(h0, sc.h0, row0, valid, tid);
        store_rows<kHidden>(h1, sc.h1, row0, valid, tid);
        store_rows<kHidden>(h2, sc.h2, row0, valid, tid);
        store_rows<kHidden>(h3, sc.h3, row0, valid, tid);
        // ---- K5: KL gradient epilogue (guiding.cpp:250-270), 4 lanes per row: all
        // 8 warps run the double-precision math (kl_grad_row_par, 2 lobes per lane)
        {
            const int row = tid >> 2, part = tid & 3;
            float *col = da + row;
            bool rfin = true;  // non-finite network output row -> dropped (:251-254)
            for (int j = part; j < NP; j += 4) rfin &= isfinite(col[j * kTLda]);
#pragma unroll
            for (int o = 1; o < 4; o <<= 1) rfin &= __shfl_xor_sync(0xffffffffu, (int)rfin, o) != 0;
            const bool vrow = row < valid;
            const float *rd = rowd + row * 8;
            TrainRow s;
            s.wi = make_float3(rd[0], rd[1], rd[2]);
            s.p = (vrow && rfin) ? rd[3] : 0.f;  // p = 0: zero gradient (invalid and dropped rows too)
            s.q_s = rd[4];
            s.pbsdf = rd[5];
            double loss = 0.0;
            __syncwarp();  // the finiteness reads are done before any lane writes its columns
            auto raw = [&](int j) { return col[j * kTLda]; };
            auto put = [&](int j, float g) { col[j * kTLda] = g; };
            const bool ok = ref::kl_grad_row_par<N, 4>(raw, s, b, e, gscale, part, put, loss);
            for (int j = NP + part; j < kHidden; j += 4) col[j * kTLda] = 0.f;
            if (part == 0) {
                const int state = !vrow ? 0 : (!rfin ? 2 : (ok ? 1 : 2));  // 0 invalid row, 1 ok, 2 dropped
                rloss[row] = (state == 1 && isfinite(loss)) ? loss : 0.0;
                rstate[row] = state == 1 && isfinite(loss) ? 1 : (state == 2 ? 2 : 0);
            }
        }
        __syncthreads();
        // delta4 in reference raw order, padded to d4_stride(N) floats per row (K_dw operand)
        constexpr int DS = d4_stride(N);
        for (int idx = tid; idx < kTrainRows * DS; idx += 256) {
            const int r = idx / DS, j = idx % DS;
            sc.d4[(row0 + r) * DS + j] = (r < valid && j < D) ? da[packed_col(j, N) * kTLda + r] : 0.f;
        }
        if (tid == 0) {  // tile statistics in row order (deterministic)
            double ls = 0.0;
            int lc = 0, dr = 0;
            for (int r = 0; r < kTrainRows; ++r) {
                int st = rstate[r];
                ls += rloss[r];
                lc += st == 1;
                dr += st == 2;
            }
            sc.tile_loss[tile] = ls;
            sc.tile_loss_count[tile] = lc;
            sc.tile_dropped[tile] = dr;
        }
        // ---- K6: delta propagation with ReLU gates (net.hpp:101-107)
        tile_layer<kTrainRows, f32_bwd_k(N), kEpiMask, kTLda>(da, db, T4, wbuf, h3, tid);
        store_rows<kHidden>(db, sc.d3, row0, valid, tid);
        tile_layer<kTrainRows, kHidden, kEpiMask, kTLda>(db, da, T3, wbuf, h2, tid);
        store_rows<kHidden>(da, sc.d2, row0, valid, tid);
        tile_layer<kTrainRows, kHidden, kEpiMask, kTLda>(da, db, T2, wbuf, h1, tid);
        store_rows<kHidden>(db, sc.d1, row0, valid, tid);
        __syncthreads();
    }
    if (tid == 0 && s_clamped && clamp_count) atomicAdd(clamp_count, (unsigned long long)s_clamped);
}

int train_forward_backward(int n_comp, const float *wp, const float *wtp, const nasg_train_sample *samples,
                           const uint32_t *order, int64_t count, const int64_t *live_count, int64_t global_count,
                           double b, double loss_blend, const Bounds &bounds, TrainScratch &sc, int num_sms,
                           unsigned long long *clamp_count, cudaStream_t s) {
    const int ntiles = (int)((count + kTrainRows - 1) / kTrainRows);
    if (ntiles == 0) return 0;
    const int grid = ntiles < num_sms ? ntiles : num_sms;
    const double gscale = 1.0 / (double)global_count;  // guiding.cpp:262
    auto go = [&](auto kern, size_t smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, 256, smem, s>>>(wp, wtp, samples, order, count, live_count, gscale, b, loss_blend, bounds, sc,
                                     clamp_count);
        return 1;
    };
    switch (n_comp) {
        case 4: return go(train_fb_kernel<4>, fb_smem_f32(4));
        case 8: return go(train_fb_kernel<8>, fb_smem_f32(8));
        case 16: return go(train_fb_kernel<16>, fb_smem_f32(16));
        case 32: return go(train_fb_kernel<32>, fb_smem_f32(32));
        default: return -1;
    }
}

// ------------------------------------------------------------------ K_dw --
// partial[split][layer block] = sum over this split's rows of H^T Delta.
template <int M>
__global__ void __launch_bounds__(256)
dw_kernel(const float *__restrict__ Hm, const float *__restrict__ Dm, int ldd, int n_out, int ldo,
          int64_t rows, int rows_per_split, float *__restrict__ partial, size_t partial_stride,
          const int64_t *live_count) {
    __shared__ __align__(16) float As[2][kChunk][M];
    __shared__ __align__(16) float Bs[2][kChunk][128];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int split = blockIdx.x;
    if (live_count) {  // the classified step: its rows, spread over the launched splits
        rows = ((*live_count + kTrainRows - 1) / kTrainRows) * kTrainRows;
        rows_per_split = (int)((rows + gridDim.x - 1) / gridDim.x);
        rows_per_split = ((rows_per_split + kChunk - 1) / kChunk) * kChunk;
    }
    const int64_t r0 = (int64_t)split * rows_per_split;
    const int64_t r1 = min(rows, r0 + rows_per_split);
    constexpr int RM = M / 16;
    float acc[RM][8];
#pragma unroll
    for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    const int nchunks = r1 > r0 ? (int)((r1 - r0 + kChunk - 1) / kChunk) : 0;
    auto load = [&](int c, int buf) {
        const int64_t rb = r0 + (int64_t)c * kChunk;
        for (int e = tid; e < kChunk * M / 4; e += 256) {  // H rows (contiguous)
            const int rr = e / (M / 4), f4 = (e % (M / 4)) * 4;
            cp_async16(&As[buf][rr][f4], Hm + (rb + rr) * M + f4);
        }
        for (int e = tid; e < kChunk * 32; e += 256) {  // Delta rows, 128 cols (reads past ldd are discarded)
            const int rr = e / 32, f4 = (e % 32) * 4;
            cp_async16(&Bs[buf][rr][f4], Dm + (rb + rr) * ldd + f4);
        }
    };
    if (nchunks > 0) {
        load(0, 0);
        cp_async_commit();
    }
    for (int c = 0; c < nchunks; ++c) {
        if (c + 1 < nchunks) {
            load(c + 1, (c + 1) & 1);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const int buf = c & 1;
#pragma unroll
        for (int kk = 0; kk < kChunk; ++kk) {
            float a[RM];
#pragma unroll
            for (int h = 0; h < RM / 4; ++h) {
                float4 t = *reinterpret_cast<const float4 *>(&As[buf][kk][ty * 4 + 64 * h]);
                a[4 * h] = t.x; a[4 * h + 1] = t.y; a[4 * h + 2] = t.z; a[4 * h + 3] = t.w;
            }
            float4 b0 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][tx * 4]);
            float4 b1 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][64 + tx * 4]);
            float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < RM; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
        }
        __syncthreads();
    }
    float *out = partial + (size_t)split * partial_stride;
#pragma unroll
    for (int i = 0; i < RM; ++i) {
        const int m = ty * 4 + 64 * (i / 4) + (i % 4);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int n = (j < 4) ? tx * 4 + j : 64 + tx * 4 + (j - 4);
            if (n < n_out) out[(size_t)m * ldo + n] = acc[i][j];
        }
    }
}

__global__ void dw_reduce_kernel(const float *__restrict__ partial, int splits, size_t stride, int nw,
                                 float *__restrict__ grad, int *nonfinite) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nw) return;
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += partial[(size_t)k * stride + e];
    grad[e] = s;
    if (!isfinite(s)) atomicOr(nonfinite, 1);
}

// live_count (the classified step): the row count on the device, the splits
// re-spread over it by the kernel; splits without rows write zero partials.
int train_dw(int n_comp, int64_t count, TrainScratch &sc, float *grad, cudaStream_t s, const int64_t *live_count) {
    const int D = 8 * n_comp + 1;
    const int nw = n_weights(n_comp);
    const int64_t rows = ((count + kTrainRows - 1) / kTrainRows) * kTrainRows;  // zero-padded tail
    int splits = (int)((rows + 63) / 64);
    if (splits > sc.splits) splits = sc.splits;
    int rps = (int)((rows + splits - 1) / splits);
    rps = ((rps + kChunk - 1) / kChunk) * kChunk;
    splits = (int)((rows + rps - 1) / rps);
    const size_t stride = (size_t)nw;
    float *p = sc.dw_partial;
    const size_t o1 = kIn * kHidden, o2 = o1 + kHidden * kHidden, o3 = o2 + kHidden * kHidden;
    dw_kernel<64><<<splits, 256, 0, s>>>(sc.h0, sc.d1, 128, 128, 128, rows, rps, p, stride, live_count);
    dw_kernel<128><<<splits, 256, 0, s>>>(sc.h1, sc.d2, 128, 128, 128, rows, rps, p + o1, stride, live_count);
    dw_kernel<128><<<splits, 256, 0, s>>>(sc.h2, sc.d3, 128, 128, 128, rows, rps, p + o2, stride, live_count);
    // dW4 [128][D] in 128-column blocks of delta4 (two for N = 16, three for N = 32)
    const int ds = d4_stride(n_comp);
    for (int c0 = 0; c0 < D; c0 += 128)
        dw_kernel<128><<<splits, 256, 0, s>>>(sc.h3, sc.d4 + c0, ds, D - c0 < 128 ? D - c0 : 128, D, rows, rps,
                                               p + o3 + c0, stride, live_count);
    sc.last_splits = splits;
    return 3 + (D + 127) / 128;  // launches
}

int train_reduce(int n_comp, const TrainScratch &sc, float *grad, int *nonfinite, cudaStream_t s) {
    const int nw = n_weights(n_comp);
    dw_reduce_kernel<<<(nw + 255) / 256, 256, 0, s>>>(sc.dw_partial, sc.last_splits, (size_t)nw, nw, grad, nonfinite);
    return 1;
}

// step_stats[0..2] = loss_sum, loss_count, dropped of this step (tile order)
// One block: strided per-thread partial sums, then a fixed-shape tree
// (deterministic for a given tile count).
__global__ void step_stats_kernel(const double *tile_loss, const int *tile_lc, const int *tile_dr, int ntiles,
                                  double *step_stats, const int64_t *cls, int tile_rows) {
    __shared__ double sl[256], sc[256], sd[256];
    const int t = threadIdx.x;
    if (cls) ntiles = (int)((cls[0] + tile_rows - 1) / tile_rows);  // the classified step's tiles
    double ls = 0.0, lc = 0.0, dr = 0.0;
    for (int i = t; i < ntiles; i += 256) {
        ls += tile_loss[i];
        lc += tile_lc[i];
        dr += tile_dr[i];
    }
    sl[t] = ls; sc[t] = lc; sd[t] = dr;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (t < s) {
            sl[t] += sl[t + s];
            sc[t] += sc[t + s];
            sd[t] += sd[t + s];
        }
        __syncthreads();
    }
    if (t == 0) {
        step_stats[0] = sl[0];
        step_stats[1] = sc[0] + (cls ? (double)cls[1] : 0.0);  // zero-gradient rows: loss 0, counted
        step_stats[2] = sd[0];
    }
}

int train_step_stats_n(const double *tile_loss, const int *tile_lc, const int *tile_dr, int ntiles,
                       double *step_stats, cudaStream_t s) {
    step_stats_kernel<<<1, 256, 0, s>>>(tile_loss, tile_lc, tile_dr, ntiles, step_stats, nullptr, 1);
    return 1;
}

int train_step_stats(const TrainScratch &sc, int64_t count, double *step_stats, cudaStream_t s, const int64_t *cls) {
    const int ntiles = (int)((count + kTrainRows - 1) / kTrainRows);
    step_stats_kernel<<<1, 256, 0, s>>>(sc.tile_loss, sc.tile_loss_count, sc.tile_dropped, ntiles, step_stats, cls,
                                        kTrainRows);
    return 1;
}


// ---------------------------------------------------------------- K_adam --
// One launch per step for the whole optimizer tail: the step's skip decision
// and bias corrections (adam_step<float> net.hpp:137-147: a non-finite
// gradient skips the update and bumps `skipped`; t++; corr = 1 - beta^t as
// powf), the update (:148-155) with the reference's operation order and IEEE
// rounding of every float op (no FMA contraction), the re-pack of the fp32
// images and, when tc_img != null, of the bf16 tensor-core image, and the
// statistics accumulation.  Every block reads the step's flag and t before
// signalling completion; the last block to finish (atomic ticket) advances t,
// accumulates the step statistics and clears the flag for the next step.
__global__ void adam_kernel(int n_comp, float *__restrict__ w, float *__restrict__ m, float *__restrict__ v,
                            const float *__restrict__ g, float lr, float *__restrict__ wp, float *__restrict__ wtp,
                            __nv_bfloat16 *__restrict__ tc_img, int *nonfinite, int64_t *adam_t,
                            const double *step_stats, double *acc, unsigned int *ticket, int recheck, int *wbig) {
    __shared__ int s_skip;
    __shared__ float s_c1, s_c2;
    pdl_trigger();
    pdl_wait();  // the reduced gradient, its non-finite flag and the step statistics
    if (recheck) {
        // data-parallel step: the skip decision (net.hpp:140-144) is taken on the
        // allreduced gradient, identically on every rank.  Every block checks its
        // slice into nonfinite[1], then a grid barrier (the launch is cooperative,
        // so all blocks are co-resident) publishes the global verdict.
        const int e0 = blockIdx.x * blockDim.x + threadIdx.x;
        const int bad = e0 < n_weights(n_comp) && !isfinite(g[e0]);
        if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite + 1, 1);
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(ticket + 1, 1u);
            while (*(volatile unsigned int *)(ticket + 1) < gridDim.x) __nanosleep(32);
            __threadfence();
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        s_skip = *(volatile int *)(nonfinite + (recheck ? 1 : 0)) != 0;
        const int64_t t = *adam_t + 1;
        // corr = 1 - beta^t computed as powf would (float result), net.hpp:146-147
        s_c1 = 1.0f - (float)pow((double)0.9f, (double)(float)t);
        s_c2 = 1.0f - (float)pow((double)0.999f, (double)(float)t);
    }
    __syncthreads();
    const int nw = n_weights(n_comp);
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < nw && !s_skip) {
        const float b1 = 0.9f, b2 = 0.999f, eps = 1e-8f;
        const float c1 = s_c1, c2 = s_c2;
        const float gi = g[e];
        const float mi = __fadd_rn(__fmul_rn(b1, m[e]), __fmul_rn(__fsub_rn(1.f, b1), gi));
        const float vi = __fadd_rn(__fmul_rn(b2, v[e]), __fmul_rn(__fsub_rn(1.f, b2), __fmul_rn(gi, gi)));
        const float mh = __fdiv_rn(mi, c1), vh = __fdiv_rn(vi, c2);
        const float wi = __fsub_rn(w[e], __fdiv_rn(__fmul_rn(lr, mh), __fadd_rn(__fsqrt_rn(vh), eps)));
        m[e] = mi;
        v[e] = vi;
        w[e] = wi;
        if (!(fabsf(wi) < kSafeWeight)) atomicOr(wbig, 1);  // sticky until the next host re-pack
        // re-pack (same mappings as pack_fp32_kernel and pack_tc_kernel)
        const int o1 = kIn * kHidden, o2 = o1 + kHidden * kHidden, o3 = o2 + kHidden * kHidden;
        int l, n, k;  // layer, output column (packed for the last layer), input row
        if (e < o3) {
            wp[e] = wi;
            l = e < o1 ? 0 : (e < o2 ? 1 : 2);
            const int base = l == 0 ? 0 : (l == 1 ? o1 : o2);
            k = (e - base) / kHidden;
            n = (e - base) % kHidden;
            if (l > 0) wtp[(l - 1) * kHidden * kHidden + n * kHidden + k] = wi;
        } else {
            const int D = 8 * n_comp + 1;
            k = (e - o3) / D;
            n = packed_col((e - o3) % D, n_comp);
            l = 3;
            wp[o3 + (n / 128) * (kHidden * 128) + k * 128 + n % 128] = wi;
            wtp[2 * kHidden * kHidden + n * kHidden + k] = wi;
        }
        if (tc_img) {  // the bf16 trainer's image (train_img_bytes): f16 layers, bf16 copy of W4p^T
            const uint32_t byte = img_elem_off(l, n, k);
            uint16_t *im = reinterpret_cast<uint16_t *>(tc_img);
            im[byte / 2] = __half_as_ushort(__float2half_rn(sat_f16_range(wi)));
            if (l == 3) im[(img_bytes(n_comp) + byte - w_off(3)) / 2] = __bfloat16_as_ushort(__float2bfloat16_rn(wi));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(ticket, 1u) == gridDim.x - 1) {  // last block: every block has read flag and t
            const int sk = s_skip;
            if (!sk) *adam_t = *adam_t + 1;
            nonfinite[0] = 0;
            nonfinite[1] = 0;
            ticket[1] = 0;  // grid barrier of a recheck launch: every block is past it
            acc[0] += step_stats[0];
            acc[1] += step_stats[1];
            acc[2] += step_stats[2];
            acc[3] += sk;
            acc[4] += 1.0;
            *ticket = 0;
        }
    }
}

int train_adam(int n_comp, float *w, float *m, float *v, const float *grad, float lr, float *wp, float *wtp,
               void *tc_img, int *nonfinite, int64_t *adam_t, const double *step_stats, double *acc,
               unsigned int *ticket, cudaStream_t s, bool pdl, bool recheck, int *wbig) {
    const int nw = n_weights(n_comp);
    launch_ex(pdl, recheck, adam_kernel, dim3((nw + 255) / 256), dim3(256), 0, s, n_comp, w, m, v, grad, lr, wp,
               wtp, static_cast<__nv_bfloat16 *>(tc_img), nonfinite, adam_t, step_stats, acc, ticket, recheck ? 1 : 0, wbig);
    return 1;
}

}  // namespace nasg

namespace nasg {
__global__ void check_finite_kernel(const float *x, int n, int *nonfinite) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n && !isfinite(x[e])) atomicOr(nonfinite, 1);
}
int check_finite(const float *x, int n, int *nonfinite, cudaStream_t s) {
    check_finite_kernel<<<(n + 255) / 256, 256, 0, s>>>(x, n, nonfinite);
    return 1;
}
}  // namespace nasg
