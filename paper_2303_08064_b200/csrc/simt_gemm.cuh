// fp32 FFMA tile GEMM used by the fp32 query path and the fp32 training
// path: one CTA of 256 threads computes OUT[TM rows][128 cols] =
// IN[TM][K] * W[K][128] with the activations resident in shared memory in
// feature-major ("k-major") layout [K][LDA] and W streamed from global
// (L2-resident) in 16-row chunks with cp.async double buffering.
// Thread (tx, ty) = (tid % 16, tid / 16) owns rows {ty*4 + 64*j + i} and
// cols {tx*4 + 64*h + i}: 2 x LDS.128 of activations + 2 x LDS.128 of
// weights per 8 x 8 (TM = 128) or 4 x 8 (TM = 64) FFMAs.
#pragma once

#include <cuda_runtime.h>

namespace nasg {

constexpr int kLda = 132;   // 128 + 4 floats: keeps float4 alignment, spreads banks
constexpr int kChunk = 16;  // weight rows per cp.async stage

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Load weight rows [k0, k0 + 16) x 128 cols into wbuf (16 x 128 floats).
__device__ __forceinline__ void load_w_chunk(const float *__restrict__ W, int k0, float *wbuf,
                                             int tid) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        int e = (tid + 256 * i) * 4;  // float index within the chunk
        cp_async16(wbuf + e, W + (size_t)k0 * 128 + e);
    }
}

enum Epi { kEpiNone = 0, kEpiRelu = 1, kEpiMask = 2 };

// OUT[n][r] (feature-major) = epi( sum_k IN[k][r] * W[k][n] ).
// kEpiMask multiplies by [MASK[n][r] > 0] (ReLU gate of backward, net.hpp:106).
// Must be called by all 256 threads; ends with a __syncthreads().  Only output
// features n < NOUT are stored (the second 128-column block of a wide layer).
template <int TM, int K, int EPI, int LDA = kLda, int NOUT = 128>
__device__ __forceinline__ void tile_layer(const float *in, float *out,
                                           const float *__restrict__ W, float *wbuf,
                                           const float *mask, int tid) {
    constexpr int RM = TM / 16;  // rows per thread (8 or 4)
    constexpr int NC = K / kChunk;
    const int tx = tid & 15, ty = tid >> 4;
    float acc[RM][8];
#pragma unroll
    for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    load_w_chunk(W, 0, wbuf, tid);
    cp_async_commit();
#pragma unroll 1
    for (int kc = 0; kc < NC; ++kc) {
        if (kc + 1 < NC) {
            load_w_chunk(W, (kc + 1) * kChunk, wbuf + ((kc + 1) & 1) * kChunk * 128, tid);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const float *wb = wbuf + (kc & 1) * kChunk * 128;
#pragma unroll
        for (int kk = 0; kk < kChunk; ++kk) {
            const float *ar = in + (kc * kChunk + kk) * LDA + ty * 4;
            float a[RM];
#pragma unroll
            for (int h = 0; h < RM / 4; ++h) {
                float4 t = *reinterpret_cast<const float4 *>(ar + 64 * h);
                a[4 * h] = t.x; a[4 * h + 1] = t.y; a[4 * h + 2] = t.z; a[4 * h + 3] = t.w;
            }
            float4 b0 = *reinterpret_cast<const float4 *>(wb + kk * 128 + tx * 4);
            float4 b1 = *reinterpret_cast<const float4 *>(wb + kk * 128 + 64 + tx * 4);
            float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < RM; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int n = (j < 4) ? tx * 4 + j : 64 + tx * 4 + (j - 4);
        if (NOUT < 128 && n >= NOUT) continue;
#pragma unroll
        for (int h = 0; h < RM / 4; ++h) {
            float4 v = make_float4(acc[4 * h][j], acc[4 * h + 1][j], acc[4 * h + 2][j], acc[4 * h + 3][j]);
            if (EPI == kEpiRelu) {  // std::max(x, 0) as Eigen's cwiseMax: NaN propagates
                v.x = v.x < 0.f ? 0.f : v.x; v.y = v.y < 0.f ? 0.f : v.y;
                v.z = v.z < 0.f ? 0.f : v.z; v.w = v.w < 0.f ? 0.f : v.w;
            } else if (EPI == kEpiMask) {  // delta *= [h > 0] as a product (inf*0 = NaN, net.hpp:106)
                float4 m = *reinterpret_cast<const float4 *>(mask + n * LDA + ty * 4 + 64 * h);
                v.x *= m.x > 0.f ? 1.f : 0.f; v.y *= m.y > 0.f ? 1.f : 0.f;
                v.z *= m.z > 0.f ? 1.f : 0.f; v.w *= m.w > 0.f ? 1.f : 0.f;
            }
            *reinterpret_cast<float4 *>(out + n * LDA + ty * 4 + 64 * h) = v;
        }
    }
    __syncthreads();
}

}  // namespace nasg
