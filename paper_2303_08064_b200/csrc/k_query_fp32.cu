// fp32 query path: fused encode -> 4-layer MLP (FFMA) -> NASG epilogue,
// plus the weight-packing kernel and the raw-output parity kernels.
//
// Two persistent CTAs (256 threads) per SM walk 128-query tiles.  Per tile:
//   K1 encode     encode_inputs (encoding.cpp:21-46) into smem, feature-major
//   K2 MLP        forward<float> (net.hpp:69-76), 4 x tile_layer
//   K3 epilogue   decode + mixture_sample + mixture_pdf, or mixture/guided
//                 pdf at a given direction, one thread per query
// Only the 64 B/query of inputs and 16-20 B/query of outputs touch HBM.
#include <cstdio>

#include "nasg_internal.h"
#include "nasg_math.cuh"
#include "nasg_refmath.cuh"
#include "simt_gemm.cuh"

namespace nasg {

// ---------------------------------------------------------------- packing --
// wp : W1[64][128] W2[128][128] W3[128][128], W4p as f32_out_blocks blocks of
//      [128][128] (packed cols, block b = packed cols [128 b, 128 b + 128))
// wtp: W2^T[128][128] W3^T[128][128] W4p^T[128 x blocks][128] (rows = packed col)
__global__ void pack_fp32_kernel(const float *__restrict__ w, int n_comp, float *__restrict__ wp,
                                 float *__restrict__ wtp, int *wbig) {
    const int D = 8 * n_comp + 1;
    const int NP = packed_width(n_comp);
    const int o1 = kIn * kHidden, o2 = o1 + kHidden * kHidden, o3 = o2 + kHidden * kHidden;
    const int total = packed_f32_floats(n_comp);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        float v;
        int pc = 0, k = 0;
        if (e < o3) {
            v = w[e];
        } else {
            const int bk = (e - o3) / (kHidden * 128), rem = (e - o3) % (kHidden * 128);
            k = rem / 128;
            pc = bk * 128 + rem % 128;
            int j = -1;  // reference raw index of packed column pc
            if (pc < NP) {
                const int H = packed_header(n_comp);
                if (pc < n_comp) j = 7 * n_comp + pc;
                else if (pc == n_comp) j = 8 * n_comp;
                else if (pc >= H) {
                    const int i = (pc - H) / 8, kk = (pc - H) % 8;
                    j = kk < 5 ? 5 * i + kk : (kk == 5 ? 5 * n_comp + 2 * i : (kk == 6 ? 5 * n_comp + 2 * i + 1 : -1));
                }
            }
            v = j >= 0 ? w[o3 + k * D + j] : 0.f;
        }
        wp[e] = v;
        if (wbig && !(fabsf(v) < kSafeWeight)) atomicOr(wbig, 1);
        if (wtp && e >= o1) {  // transposed W2, W3, W4p
            if (e < o3) {
                const int l = e < o2 ? 0 : 1;
                const int base = l == 0 ? o1 : o2;
                const int kk = (e - base) / kHidden, col = (e - base) % kHidden;
                wtp[l * kHidden * kHidden + col * kHidden + kk] = v;
            } else {
                wtp[2 * kHidden * kHidden + pc * kHidden + k] = v;
            }
        }
    }
}

void launch_pack_fp32(const float *w, int n_comp, float *wp, float *wtp, cudaStream_t s, int *wbig) {
    pack_fp32_kernel<<<148, 256, 0, s>>>(w, n_comp, wp, wtp, wbig);
}

// Snapshot copy of up to three device buffers (16-byte multiples) in one launch.
struct Copy3 {
    const uint4 *src[3];
    uint4 *dst[3];
    int64_t n16[3];
};
__global__ void copy3_kernel(Copy3 c) {
#pragma unroll
    for (int k = 0; k < 3; ++k)
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.n16[k];
             i += (int64_t)gridDim.x * blockDim.x)
            c.dst[k][i] = c.src[k][i];
}

void launch_copy3(const void *const src[3], void *const dst[3], const size_t bytes[3], cudaStream_t s) {
    Copy3 c{};
    for (int k = 0; k < 3; ++k) {
        c.src[k] = static_cast<const uint4 *>(src[k]);
        c.dst[k] = static_cast<uint4 *>(dst[k]);
        c.n16[k] = src[k] ? (int64_t)(bytes[k] / 16) : 0;
    }
    copy3_kernel<<<148, 256, 0, s>>>(c);
}

// ------------------------------------------------------------- encoding --
// One-blob encoding of one query into column r of the feature-major tile.
// t = (p - min) / ext in double as in encoding.cpp:30; bins in fp32.
__device__ __forceinline__ int encode_row(const float4 x, const float4 wo, const float4 nrm,
                                          const Bounds &bd, float *act, int r) {
    int clamped = 0;
    const float xs[3] = {x.x, x.y, x.z};
#pragma unroll
    for (int axis = 0; axis < 3; ++axis) {
        double t = bd.ext[axis] > 0.0 ? ((double)xs[axis] - (double)bd.bmin[axis]) / bd.ext[axis] : 0.5;
        if (t < 0.0 || t > 1.0) {
            ++clamped;
            t = fmin(fmax(t, 0.0), 1.0);
        }
#pragma unroll
        for (int i = 0; i < kBins; ++i) {
            act[(axis * kBins + i) * kLda + r] = ref::one_blob_bin(t, i);
        }
    }
    act[57 * kLda + r] = wo.x; act[58 * kLda + r] = wo.y; act[59 * kLda + r] = wo.z;
    act[60 * kLda + r] = nrm.x; act[61 * kLda + r] = nrm.y; act[62 * kLda + r] = nrm.z;
    act[63 * kLda + r] = 1.f;
    return clamped;
}

// ---------------------------------------------------------- fused kernel --
// feature rows of the activation tile: the hidden width, or the packed raw width when wider
constexpr int act_rows(int n) { return packed_width(n) > kHidden ? packed_width(n) : kHidden; }
constexpr size_t query_smem(int n) { return (size_t)(act_rows(n) * kLda + 2 * kChunk * 128) * sizeof(float); }

template <int N, int MODE>
__global__ void __launch_bounds__(256, 2 * query_smem(N) <= 232448 ? 2 : 1)  // one CTA per SM at N = 32
query_fp32_kernel(const float *__restrict__ wp, QueryArgs a) {
    extern __shared__ __align__(16) float smem[];
    // one activation tile, updated in place: each layer keeps its outputs in
    // registers until every thread has read its last input chunk (tile_layer's
    // chunk barrier), so ~84 KB of smem -> two CTAs per SM, and one CTA's
    // half-occupied NASG epilogue overlaps the other's FFMA GEMMs
    float *actA = smem;                      // [max(128, NP)][kLda]
    float *wbuf = actA + act_rows(N) * kLda; // [2][16][128]
    __shared__ int s_clamped;
    const int tid = threadIdx.x;
    const int64_t nrows = a.n_dev ? min((int64_t)*a.n_dev, a.n) : a.n;  // a wavefront queue sets n_dev
    const int64_t ntiles = (nrows + kTileRows - 1) / kTileRows;
    const float *W1 = wp, *W2 = W1 + kIn * kHidden, *W3 = W2 + kHidden * kHidden,
                *W4 = W3 + kHidden * kHidden;
    if (tid == 0) s_clamped = 0;
    __syncthreads();
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t row0 = tile * kTileRows;
        if (tid < kTileRows) {
            const int64_t q = row0 + tid;
            if (q < nrows) {
                float4 qx, qwo, qn;
                load_query(a, q, qx, qwo, qn);
                int cl = encode_row(qx, qwo, qn, a.bounds, actA, tid);
                if (cl) atomicAdd(&s_clamped, cl);
            } else {
                for (int k = 0; k < kIn; ++k) actA[k * kLda + tid] = 0.f;
            }
        }
        __syncthreads();
        tile_layer<128, kIn, kEpiRelu>(actA, actA, W1, wbuf, nullptr, tid);
        tile_layer<128, kHidden, kEpiRelu>(actA, actA, W2, wbuf, nullptr, tid);
        tile_layer<128, kHidden, kEpiRelu>(actA, actA, W3, wbuf, nullptr, tid);
        constexpr int NP = packed_width(N);
        if constexpr (NP > 256)  // packed columns past 128 first, into rows the layer does not read
            tile_layer<128, kHidden, kEpiNone, kLda, NP - 256>(actA, actA + 256 * kLda, W4 + 2 * kHidden * 128, wbuf,
                                                               nullptr, tid);
        if constexpr (NP > 128)
            tile_layer<128, kHidden, kEpiNone, kLda, (NP - 128 < 128 ? NP - 128 : 128)>(
                actA, actA + 128 * kLda, W4 + kHidden * 128, wbuf, nullptr, tid);
        tile_layer<128, kHidden, kEpiNone>(actA, actA, W4, wbuf, nullptr, tid);
        if constexpr (MODE == kModeSample || MODE == kModePdf) {
            // double-precision epilogue on all 8 warps: 2 lanes per query, 4 lobes each
            const int row = tid >> 1, part = tid & 1;
            const int64_t q = row0 + row;
            const bool valid = q < nrows;
            const float *col = actA + row;
            auto raw = [&](int j) { return col[j * kLda]; };
            if constexpr (MODE == kModeSample) {
                float c;
                const float4 o = ref::guide_sample_par<N, 2>(raw, valid ? load_xi(a, q) : make_float4(0.f, 0.f, 0.f, 0.f),
                                                             part, c);
                if (valid && part == 0) {
                    a.dir_pdf[q] = o;
                    if (a.c) a.c[q] = c;
                }
            } else {
                const float4 d = valid ? a.dir[q] : make_float4(0.f, 0.f, 1.f, 0.f);
                const float2 p = ref::guide_pdf_par<N, 2>(raw, make_float3(d.x, d.y, d.z), a.b,
                                                          (valid && a.bsdf_pdf) ? a.bsdf_pdf[q] : 0.f, part);
                if (valid && part == 0) {
                    if (a.mix_pdf) a.mix_pdf[q] = p.x;
                    if (a.guided_pdf) a.guided_pdf[q] = p.y;
                }
            }
        } else if (tid < kTileRows) {
            const int64_t q = row0 + tid;
            if (q < nrows) {
                const float *col = actA + tid;
                auto raw = [&](int j) { return col[j * kLda]; };
                if (MODE == kModeShade) {
                    float4 o0, o1;
                    ref::guide_shade<N>(raw, load_xi(a, q), a.b, a.sh_bsdf[q], a.sh_nee[q], o0, o1);
                    a.sh_out[2 * q] = o0;
                    a.sh_out[2 * q + 1] = o1;
                } else {
                    constexpr int D = 8 * N + 1;
                    for (int j = 0; j < D; ++j) a.raw[q * D + j] = raw(packed_col(j, N));
                }
            }
        }
        __syncthreads();
    }
    if (tid == 0 && s_clamped && a.clamp_count) atomicAdd(a.clamp_count, (unsigned long long)s_clamped);
}


template <int N>
static int query_fp32_n(QueryMode mode, const float *wp, const QueryArgs &a, int num_sms, cudaStream_t s) {
    const int64_t ntiles = (a.n + kTileRows - 1) / kTileRows;
    constexpr int per_sm = 2 * query_smem(N) <= 232448 ? 2 : 1;  // two CTAs per SM (one at N = 32)
    const int grid = (int)(ntiles < per_sm * num_sms ? ntiles : per_sm * num_sms);
    if (grid == 0) return 0;
    switch (mode) {
#define NASG_LAUNCH(M)                                                                             \
    case M: {                                                                                      \
        auto k = query_fp32_kernel<N, M>;                                                          \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)query_smem(N));  \
        k<<<grid, 256, query_smem(N), s>>>(wp, a);                                                 \
        break;                                                                                     \
    }
        NASG_LAUNCH(kModeSample)
        NASG_LAUNCH(kModePdf)
        NASG_LAUNCH(kModeRaw)
        NASG_LAUNCH(kModeShade)
#undef NASG_LAUNCH
    }
    return 1;
}

int query_fp32(int n_comp, QueryMode mode, const float *wp, const QueryArgs &a, int num_sms, cudaStream_t s) {
    switch (n_comp) {  // N = 16: the last layer in two 128-column blocks (NP = 160)
        case 4: return query_fp32_n<4>(mode, wp, a, num_sms, s);
        case 8: return query_fp32_n<8>(mode, wp, a, num_sms, s);
        case 16: return query_fp32_n<16>(mode, wp, a, num_sms, s);
        case 32: return query_fp32_n<32>(mode, wp, a, num_sms, s);  // NP = 304: three blocks
        default: return -1;
    }
}

// ------------------------------------------------------ raw-output parity --
template <int N, bool SAMPLE, bool FAST>
__global__ void decode_raw_kernel(int64_t n, const float *__restrict__ raw, const float4 *xi,
                                  const float4 *dir, float b, const float *bsdf_pdf, float4 *dir_pdf,
                                  float *c, float *mix_pdf, float *guided_pdf) {
    constexpr int D = 8 * N + 1, H = packed_header(N);
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const float *row = raw + q * D;
    auto rawf = [&](int j) -> float {  // packed column -> reference raw index
        if (j < N) return row[7 * N + j];
        if (j == N) return row[8 * N];
        if (j < H) return 0.f;
        const int i = (j - H) >> 3, k = (j - H) & 7;
        return k < 5 ? row[5 * i + k] : (k == 5 ? row[5 * N + 2 * i] : (k == 6 ? row[5 * N + 2 * i + 1] : 0.f));
    };
    if (SAMPLE) {
        float cc;
        dir_pdf[q] = FAST ? guide_sample<N>(rawf, xi[q], cc) : ref::guide_sample<N>(rawf, xi[q], cc);
        if (c) c[q] = cc;
    } else {
        const float4 d = dir[q];
        const float3 v = make_float3(d.x, d.y, d.z);
        const float bp = bsdf_pdf ? bsdf_pdf[q] : 0.f;
        const float2 p = FAST ? guide_pdf<N>(rawf, v, b, bp) : ref::guide_pdf<N>(rawf, v, b, bp);
        if (mix_pdf) mix_pdf[q] = p.x;
        if (guided_pdf) guided_pdf[q] = p.y;
    }
}

template <int N, bool FAST>
static int decode_raw_n(bool sample, int64_t n, const float *raw, const float4 *xi, const float4 *dir, float b,
                        const float *bsdf_pdf, float4 *dir_pdf, float *c, float *mix_pdf, float *guided_pdf,
                        cudaStream_t s) {
    const int blocks = (int)((n + 127) / 128);
    if (blocks == 0) return 0;
    if (sample)
        decode_raw_kernel<N, true, FAST><<<blocks, 128, 0, s>>>(n, raw, xi, dir, b, bsdf_pdf, dir_pdf, c, mix_pdf,
                                                                guided_pdf);
    else
        decode_raw_kernel<N, false, FAST><<<blocks, 128, 0, s>>>(n, raw, xi, dir, b, bsdf_pdf, dir_pdf, c, mix_pdf,
                                                                 guided_pdf);
    return 1;
}

// fast = true: the fp32 epilogue of the bf16 tensor-core path (nasg_math.cuh);
// false: the double restatement used by the fp32 path (nasg_refmath.cuh).
int decode_raw(int n_comp, bool sample, bool fast, int64_t n, const float *raw, const float4 *xi, const float4 *dir,
               float b, const float *bsdf_pdf, float4 *dir_pdf, float *c, float *mix_pdf, float *guided_pdf,
               cudaStream_t s) {
#define NASG_DR(NN)                                                                                         \
    return fast ? decode_raw_n<NN, true>(sample, n, raw, xi, dir, b, bsdf_pdf, dir_pdf, c, mix_pdf, guided_pdf, s) \
                : decode_raw_n<NN, false>(sample, n, raw, xi, dir, b, bsdf_pdf, dir_pdf, c, mix_pdf, guided_pdf, s)
    switch (n_comp) {
        case 4: NASG_DR(4);
        case 8: NASG_DR(8);
        case 16: NASG_DR(16);
        case 32: NASG_DR(32);
        default: return -1;
    }
#undef NASG_DR
}

}  // namespace nasg
