// Shared pieces of the tcgen05 kernels (query and training): the bf16 weight
// image layout, the one-blob encoder writing a bf16 A tile, and the
// warpgroup barrier.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "nasg_internal.h"
#include "nasg_math.cuh"
#include "tc_ptx.cuh"

namespace nasg {

// Weight image (f16 elements): per layer the UMMA B operand W_l^T as [N_out][K_in],
// K-major, no swizzle: 8-row x 16-byte core matrices, LBO = 128 B between the
// two K chunks of a K=16 slab, SBO = K_in * 16 B between 8-row groups.
__host__ __device__ constexpr uint32_t w_off(int l) {
    return l == 0 ? 0u : (l == 1 ? 16384u : (l == 2 ? 49152u : 81920u));
}
__host__ __device__ constexpr uint32_t img_bytes(int n) { return 81920u + (uint32_t)packed_width(n) * 256u; }
__host__ __device__ constexpr uint32_t align1k(uint32_t x) { return (x + 1023u) & ~1023u; }
// The bf16 trainer's live image: the same four layers in f16 (its forward and
// the backward through W3, W2 run f16 x f16), then W4p^T once more in bf16 at
// img_bytes(n) for the first backward layer, whose operand delta4 (the KL
// gradient, spanning decades) keeps bf16's exponent range.
__host__ __device__ constexpr uint32_t train_img_bytes(int n) { return img_bytes(n) + (uint32_t)packed_width(n) * 256u; }
// a weight clamped to f16's finite range for the trainer image; NaN stays NaN
// (a non-finite network must still poison its outputs and skip, net.hpp:140-144)
__device__ __forceinline__ float sat_f16_range(float v) { return v != v ? v : fminf(fmaxf(v, -65504.f), 65504.f); }
// byte offset of W_l^T[n][k] inside an image (core-matrix layout above)
__host__ __device__ constexpr uint32_t img_elem_off(int l, int n, int k) {
    return w_off(l) + (uint32_t)(n / 8) * (uint32_t)((l == 0 ? kIn : kHidden) * 16) + (uint32_t)(k / 8) * 128u +
           (uint32_t)(n % 8) * 16u + (uint32_t)(k % 8) * 2u;
}

// --------------------------------------------------------------- encoding --
// encode_inputs (encoding.cpp:21-46) in fp32 -> 64 bf16 features packed in 32
// registers (pairs in K order).  Returns the number of clamped coordinates.
__device__ __forceinline__ int encode_row_values(bool valid, float4 x, float4 wo, float4 nrm, const Bounds &bd,
                                                 const float (&inv_ext)[3], float (&e)[64]) {
    int clamped = 0;
    if (valid) {
        const float xs[3] = {x.x, x.y, x.z};
#pragma unroll
        for (int axis = 0; axis < 3; ++axis) {
            float t = inv_ext[axis] > 0.f ? (xs[axis] - bd.bmin[axis]) * inv_ext[axis] : 0.5f;
            if (t < 0.f || t > 1.f) {
                ++clamped;
                t = fminf(fmaxf(t, 0.f), 1.f);
            }
            // one_blob (encoding.cpp:11-19): e_i = exp(-180.5 (t - c_i)^2) = exp(-y_i^2 / 2)
            // with y_i = 19 t - i - 0.5 (sigma = 1/19).  Gaussian recurrence from the
            // centre bin (c_9 = 0.5 exactly): e_{i+1} = e_i q_i, q_i = exp(y_i - 1/2),
            // q_{i+1} = q_i / e (and downwards e_{i-1} = e_i p_i, p_i = exp(-y_i - 1/2)),
            // so 3 MUFU.EX2 per axis instead of 19.  Every factor derives from the one
            // rounded y_9, so the result is exp(-(y_i + eps)^2 / 2) for one consistent
            // eps ~ 1 ulp of y: p99 relative error 4e-6 (the direct 19-EX2 form's is 3e-6)
            constexpr float kL = 1.4426950408889634f;           // log2 e
            constexpr float kHalfL = 0.7213475204444817f;       // log2(e) / 2
            constexpr float kInvE = 0.36787944117144233f;       // e^-1
            const float y = fmaf(t, (float)kBins, -0.5f * kBins);
            const float e9 = tc::ex2_approx(-(y * y) * kHalfL);
            float q = tc::ex2_approx(fmaf(y, kL, -kHalfL));
            float p = tc::ex2_approx(fmaf(-y, kL, -kHalfL));
            float up = e9, dn = e9;
            e[axis * kBins + kBins / 2] = e9;
#pragma unroll
            for (int j = 1; j <= kBins / 2; ++j) {
                up *= q;
                dn *= p;
                e[axis * kBins + kBins / 2 + j] = up;
                e[axis * kBins + kBins / 2 - j] = dn;
                q *= kInvE;
                p *= kInvE;
            }
        }
        e[57] = wo.x; e[58] = wo.y; e[59] = wo.z;
        e[60] = nrm.x; e[61] = nrm.y; e[62] = nrm.z;
        e[63] = 1.f;
    } else {
#pragma unroll
        for (int k = 0; k < 64; ++k) e[k] = 0.f;
    }
    return clamped;
}

__device__ __forceinline__ int encode_row_pack_f16(bool valid, float4 x, float4 wo, float4 nrm, const Bounds &bd,
                                                   const float (&inv_ext)[3], uint32_t (&pk)[32]) {
    float e[64];
    const int clamped = encode_row_values(valid, x, wo, nrm, bd, inv_ext, e);
#pragma unroll
    for (int j = 0; j < 32; ++j) pk[j] = tc::pack_f16x2_sat(e[2 * j], e[2 * j + 1]);
    return clamped;
}

// row t's 8 16-byte chunks of the K=64 A tile (core-matrix layout); optionally
// also to `gdst` (a global row block with the same byte layout)
__device__ __forceinline__ void store_row_pack(const uint32_t (&pk)[32], uint32_t a_row, uint8_t *gdst = nullptr) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        tc::st_shared_v4(a_row + c * 128, pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
        if (gdst) *reinterpret_cast<uint4 *>(gdst + c * 128) = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
    }
}

// The trainer's encode: f16 features into the K=64 A tile (its forward runs
// in f16), bf16 into the global h0 block read by the dW GEMM.
__device__ __forceinline__ int encode_row_f16(bool valid, float4 x, float4 wo, float4 nrm, const Bounds &bd,
                                              const float (&inv_ext)[3], uint32_t a_row, uint8_t *gdst) {
    float e[64];
    const int clamped = encode_row_values(valid, x, wo, nrm, bd, inv_ext, e);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        uint32_t h[4], b[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            h[j] = tc::pack_f16x2_sat(e[8 * c + 2 * j], e[8 * c + 2 * j + 1]);
            b[j] = tc::pack_bf16x2(e[8 * c + 2 * j], e[8 * c + 2 * j + 1]);
        }
        tc::st_shared_v4(a_row + c * 128, h[0], h[1], h[2], h[3]);
        *reinterpret_cast<uint4 *>(gdst + c * 128) = make_uint4(b[0], b[1], b[2], b[3]);
    }
    return clamped;
}

// named barrier over the 128 threads of epilogue warpgroup g (id 0 is __syncthreads)
__device__ __forceinline__ void wg_sync(int g) { asm volatile("bar.sync %0, 128;" ::"r"(g + 1) : "memory"); }

// Wait until warpgroup g's accumulator is complete (its tcgen05.commit arrived):
// one warp of the group polls the mbarrier, the other three sleep on the group's
// named barrier instead of spending issue slots on try_wait.
__device__ __forceinline__ void wg_wait_acc(uint64_t *bar, uint32_t &phase, int g, int warp_in_group) {
    if (warp_in_group == 0) tc::mbar_wait(bar, phase);
    wg_sync(g);
    phase ^= 1u;
    tc::tc_fence_after();
}

}  // namespace nasg
