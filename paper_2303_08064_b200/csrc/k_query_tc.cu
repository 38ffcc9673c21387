// bf16 tensor-core query path: fused encode -> 64-128-128-128-NP MLP on
// tcgen05 (UMMA M=128, accumulators in TMEM) -> fp32 NASG epilogue.
//
// Persistent CTA per SM, warp-specialised:
//   warps 0-11  three epilogue warpgroups; warpgroup g owns TMEM columns
//               [128g, 128g+128) and one 128-row activation tile in smem.
//               Thread t of the group owns query row t = TMEM lane t.
//               Per tile: encode (encoding.cpp:21-46) -> bf16 A tile; then for
//               layers 1-3: TMEM -> regs -> ReLU -> bf16 -> A tile (next
//               layer's operand); layer 4: TMEM -> 80 raw outputs in
//               registers -> decode / sample / pdf (nasg_math.cuh).
//               After writing an A tile the group syncs on its named barrier
//               and its thread 0 issues that layer's tcgen05.mma chain
//               (K/16 UMMAs) and tcgen05.commit -> acc_full[g].  The groups
//               run independently, drift out of phase, and the tensor core
//               interleaves one group's layers with the others' epilogues;
//               a tile's NASG epilogue overlaps the next tile's layer 1.
//   warp 12     TMEM allocator (512 columns) + one thread that TMA-bulk-copies
//               the 100 KB bf16 weight image into smem once per CTA.
// Only the 64 B/query of inputs and 16-20 B/query of outputs touch HBM.
#include <cuda_bf16.h>

#include "nasg_internal.h"
#include "nasg_math.cuh"
#include "tc_ptx.cuh"
#include "tc_common.cuh"

namespace nasg {

namespace {

constexpr int kWG = 3;                          // epilogue warpgroups
               // TMEM allocation + weight TMA warp
constexpr int kThreads = kWG * 128;  // 12 warps: 3 per SMSP -> up to 168 registers        // 416
constexpr uint32_t kABytes = 128 * 128 * 2;     // one bf16 activation tile, K = 128
constexpr uint32_t kTmemCols = 512;

template <int N>
constexpr size_t smem_bytes() {
    return align1k(img_bytes(N)) + kWG * kABytes + (kWG + 2) * sizeof(uint64_t);
}

}  // namespace

size_t tc_image_bytes(int n) { return img_bytes(n); }
bool tc_supported(int n) { return n == 4 || n == 8; }  // NP = 48 / 80: one UMMA N <= 256, N % 16 == 0

// ------------------------------------------------------------------ packing --
__global__ void pack_tc_kernel(const float *__restrict__ w, int n_comp, __nv_bfloat16 *__restrict__ img) {
    const int D = 8 * n_comp + 1, NP = packed_width(n_comp), H = packed_header(n_comp);
    const int o1 = kIn * kHidden, o2 = o1 + kHidden * kHidden, o3 = o2 + kHidden * kHidden;
    const int total = o3 + NP * kHidden;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        int l, n, k;
        float v;
        if (e < o1) {
            l = 0; n = e / kIn; k = e % kIn;
            v = w[k * kHidden + n];
        } else if (e < o3) {
            l = e < o2 ? 1 : 2;
            const int ee = e - (l == 1 ? o1 : o2);
            n = ee / kHidden; k = ee % kHidden;
            v = w[(l == 1 ? o1 : o2) + k * kHidden + n];
        } else {
            l = 3;
            const int ee = e - o3;
            n = ee / kHidden; k = ee % kHidden;
            int j = -1;  // reference raw index of packed column n
            if (n < n_comp) j = 7 * n_comp + n;
            else if (n == n_comp) j = 8 * n_comp;
            else if (n >= H) {
                const int i = (n - H) / 8, kk = (n - H) % 8;
                j = kk < 5 ? 5 * i + kk : (kk == 5 ? 5 * n_comp + 2 * i : (kk == 6 ? 5 * n_comp + 2 * i + 1 : -1));
            }
            v = j >= 0 ? w[o3 + k * D + j] : 0.f;
        }
        const int K = l == 0 ? kIn : kHidden;
        const uint32_t byte = w_off(l) + (n / 8) * (K * 16) + (k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2;
        img[byte / 2] = __float2bfloat16_rn(v);
    }
}

void launch_pack_tc(const float *w, int n_comp, void *img, cudaStream_t s) {
    pack_tc_kernel<<<148, 256, 0, s>>>(w, n_comp, static_cast<__nv_bfloat16 *>(img));
}

// ------------------------------------------------------------------ kernel --
template <int N, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
query_tc_kernel(const uint8_t *__restrict__ img, QueryArgs a) {
    constexpr int NP = packed_width(N);
    constexpr uint32_t IMG = img_bytes(N);
    constexpr uint32_t A_OFF = align1k(IMG);
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t *acc_full = reinterpret_cast<uint64_t *>(smem + A_OFF + kWG * kABytes);
    uint64_t *w_bar = acc_full + kWG;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(w_bar + 1);
    __shared__ int s_clamped;

    const int warp = threadIdx.x >> 5;
    const int64_t ntiles = (a.n + 127) / 128;

    if (threadIdx.x == 0) {
        for (int g = 0; g < kWG; ++g) tc::mbar_init(&acc_full[g], 1);
        tc::mbar_init(w_bar, 1);
        s_clamped = 0;
        tc::fence_mbar_init();
    }
    if (warp == 0) tc::tmem_alloc(tmem_slot, kTmemCols);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (threadIdx.x == 0) {  // weights: TMA bulk copies global -> smem, once per CTA
        tc::mbar_arrive_expect_tx(w_bar, IMG);
        for (uint32_t off = 0; off < IMG; off += 16384)
            tc::bulk_g2s(smem + off, img + off, (IMG - off) < 16384u ? (IMG - off) : 16384u, w_bar);
    }
    {
        const int g = warp >> 2, t = threadIdx.x & 127;
        const uint32_t my_tmem = tmem + g * 128 + ((uint32_t)((warp & 3) * 32) << 16);
        const uint32_t a_base = tc::smem_u32(smem + A_OFF + g * kABytes);
        const uint32_t a_row64 = a_base + (t >> 3) * 1024 + (t & 7) * 16;   // K = 64 layout
        const uint32_t a_row128 = a_base + (t >> 3) * 2048 + (t & 7) * 16;  // K = 128 layout
        const uint32_t sW = tc::smem_u32(smem);
        // The group's A tile is complete in smem (and its TMEM reads are done):
        // make it visible to the tensor core, then thread 0 of the group issues
        // the layer's UMMAs and commits them to acc_full[g].  Each group drives
        // its own chain, so the three groups drift out of phase and the
        // tensor core interleaves their layers with the others' epilogues.
        auto issue = [&](int l) {
            tc::fence_proxy_async_smem();
            tc::tc_fence_before();
            wg_sync(g);
            if (t == 0) {
                tc::mbar_wait(w_bar, 0);
                tc::tc_fence_after();
                const int K = l == 0 ? kIn : kHidden;
                const uint32_t sbo = (uint32_t)K * 16u;
                const uint32_t idesc = tc::idesc_bf16(128, l == 3 ? NP : kHidden);
                const uint32_t b0 = sW + w_off(l), d = tmem + g * 128;
                for (int k = 0; k < K / 16; ++k)
                    tc::mma_bf16(d, tc::smem_desc(a_base + k * 256, 128, sbo), tc::smem_desc(b0 + k * 256, 128, sbo),
                                 idesc, k > 0 ? 1u : 0u);
                tc::mma_commit(&acc_full[g]);
            }
        };
        float inv_ext[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) inv_ext[k] = a.bounds.ext[k] > 0.0 ? (float)(1.0 / a.bounds.ext[k]) : 0.f;
        uint32_t acc_ph = 0;
        int clamped = 0;
        int64_t tile = (int64_t)blockIdx.x * kWG + g;
        const int64_t stride = (int64_t)gridDim.x * kWG;
        if (tile < ntiles) {
            clamped += encode_tile_row(a, tile * 128 + t, inv_ext, a_row64);
            issue(0);
        }
        while (tile < ntiles) {
#pragma unroll 1
            for (int l = 1; l < 4; ++l) {  // hidden layers: TMEM -> ReLU -> bf16 -> next A operand
                wg_wait_acc(&acc_full[g], acc_ph, g, warp & 3);
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    float v[32];
                    tc::tmem_ld32(my_tmem + q4 * 32, v);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint32_t p[4];
#pragma unroll
                        for (int h = 0; h < 4; ++h) p[h] = tc::pack_bf16x2_relu(v[8 * c + 2 * h], v[8 * c + 2 * h + 1]);
                        tc::st_shared_v4(a_row128 + (q4 * 4 + c) * 128, p[0], p[1], p[2], p[3]);
                    }
                }
                issue(l);
            }
            // output layer ready: encode the next tile into the (now free) A tile,
            // drain the raw outputs, start the next tile, then run the NASG
            // epilogue of this tile while the tensor core works on the next
            wg_wait_acc(&acc_full[g], acc_ph, g, warp & 3);
            const int64_t next = tile + stride;
            if (next < ntiles) clamped += encode_tile_row(a, next * 128 + t, inv_ext, a_row64);
            float raw[NP];
            {
                float v[32];
#pragma unroll
                for (int q = 0; q < NP / 32; ++q) {
                    tc::tmem_ld32(my_tmem + q * 32, v);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; ++i) raw[q * 32 + i] = v[i];
                }
                if constexpr (NP % 32 != 0) {
                    float u[16];
                    tc::tmem_ld16(my_tmem + (NP / 32) * 32, u);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 16; ++i) raw[(NP / 32) * 32 + i] = u[i];
                }
            }
            if (next < ntiles) issue(0);
            const int64_t q = tile * 128 + t;
            if (q < a.n) {
                auto rawf = [&](int j) { return raw[j]; };
                if constexpr (MODE == kModeSample) {
                    float c;
                    a.dir_pdf[q] = guide_sample<N>(rawf, load_xi(a, q), c);
                    if (a.c) a.c[q] = c;
                } else if constexpr (MODE == kModePdf) {
                    const float4 d = a.dir[q];
                    const float2 p = guide_pdf<N>(rawf, make_float3(d.x, d.y, d.z), a.b, a.bsdf_pdf ? a.bsdf_pdf[q] : 0.f);
                    if (a.mix_pdf) a.mix_pdf[q] = p.x;
                    if (a.guided_pdf) a.guided_pdf[q] = p.y;
                } else {
                    constexpr int D = 8 * N + 1;
#pragma unroll
                    for (int j = 0; j < D; ++j) a.raw[q * D + j] = raw[packed_col(j, N)];
                }
            }
            tile = next;
        }
        if (clamped) atomicAdd(&s_clamped, clamped);
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem, kTmemCols);
    }
    if (threadIdx.x == 0 && s_clamped && a.clamp_count) atomicAdd(a.clamp_count, (unsigned long long)s_clamped);
}

template <int N>
static int query_tc_n(QueryMode mode, const void *img, const QueryArgs &a, int num_sms, cudaStream_t s) {
    const int64_t ntiles = (a.n + 127) / 128;
    const int64_t supers = (ntiles + kWG - 1) / kWG;
    const int grid = (int)(supers < num_sms ? supers : num_sms);
    if (grid == 0) return 0;
    constexpr size_t sm = smem_bytes<N>();
    const uint8_t *im = static_cast<const uint8_t *>(img);
    switch (mode) {
#define NASG_LAUNCH_TC(M)                                                                  \
    case M: {                                                                              \
        auto k = query_tc_kernel<N, M>;                                                    \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);     \
        k<<<grid, kThreads, sm, s>>>(im, a);                                               \
        break;                                                                             \
    }
        NASG_LAUNCH_TC(kModeSample)
        NASG_LAUNCH_TC(kModePdf)
        NASG_LAUNCH_TC(kModeRaw)
#undef NASG_LAUNCH_TC
    }
    return 1;
}

int query_tc(int n_comp, QueryMode mode, const void *img, const QueryArgs &a, int num_sms, cudaStream_t s) {
    switch (n_comp) {
        case 4: return query_tc_n<4>(mode, img, a, num_sms, s);
        case 8: return query_tc_n<8>(mode, img, a, num_sms, s);
        default: return -1;
    }
}

}  // namespace nasg
