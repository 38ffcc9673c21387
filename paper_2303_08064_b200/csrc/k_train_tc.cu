// Tensor-core training step (NASG_MLP_BF16; Trainer::train_iteration inner
// loop, guiding.cpp:236-276) — the fast training path; fp32 master weights + Adam.
//
//   classify (train_classify_kernel, steps with more tiles than SMs): the rows
//        with p = 0 are counted as zero-gradient rows; the others form the list
//        K_fb and K_dw work on.
//   K_fb (train_tc_fb_kernel)  persistent, 3 epilogue warpgroups x 128-row tiles
//        (1 at N = 16), like the query kernel: gather + encode -> 4 forward UMMA
//        layers on f16 operands (TMEM accumulators, ReLU fused into the f16
//        conversion, ReLU gate bits kept in registers) -> KL gradient of every
//        row in fp32 (kl_grad_row_fast, nasg_math.cuh; guiding.cpp:108-165) ->
//        delta4 (bf16) -> 3 backward UMMA layers delta_l = (delta_{l+1} W_l^T)
//        .* [h_l > 0] (net.hpp:101-107) that read the SAME smem weight image as
//        the forward as MN-major B operands (through a bf16 copy of W4 for
//        delta4, then row-scaled f16 deltas).  Every h_l / delta_l tile is
//        written once to HBM as bf16 in the tensor core's core-matrix layout.
//   K_dw (train_tc_dw_kernel)  dW_l = h_l^T delta_{l+1} (net.hpp:102) as a
//        split-K UMMA GEMM over 128-row blocks: both operands MN-major, TMA
//        bulk copies into a 2-stage smem ring, fp32 accumulation in TMEM,
//        per-split partials reduced in fixed order (deterministic) by
//        train_tc_reduce_kernel, whose extra block sums the step statistics.
//   then the one-launch optimizer tail shared with the fp32 path (k_train.cu
//   adam_kernel: skip decision, t, Adam, re-pack of every live image).  The
//   four launches of a step chain by programmatic dependent launch.
#include <cuda_bf16.h>

#include "nasg_internal.h"
#include "nasg_math.cuh"
#include "nasg_refmath.cuh"
#include "tc_common.cuh"
#include "tc_ptx.cuh"

// Development-only phase timestamps of K_fb (build with EXTRA=-DNASG_TRACE into
// a scratch directory; the shipped library compiles them out): clock64() of
// thread 0 of warpgroup 0 in CTA 0 at fixed points of its first 16 tiles.
#ifdef NASG_TRACE
__device__ unsigned long long g_fb_trace[16 * 16];
extern "C" int nasg_fb_trace_read(void *host) { return (int)cudaMemcpyFromSymbol(host, g_fb_trace, sizeof(g_fb_trace)); }
#define FB_TRACE(k, slot) \
    if (blockIdx.x == 0 && threadIdx.x == 0 && (k) < 16) g_fb_trace[(k) * 16 + (slot)] = clock64();
#else
#define FB_TRACE(k, slot)
#endif

namespace nasg {

namespace {

// Epilogue warpgroups (tile chains) per CTA: three for N <= 8 (12 warps, 3 per
// SMSP, up to 168 registers); one for N = 16, whose 160-column raw / delta4
// tile and 160 KB trainer image leave room for a single chain.
constexpr int kWGt = 3;
constexpr int wgt_for(int n) { return packed_width(n) > 128 ? 1 : kWGt; }
constexpr uint32_t kATile = 128 * 128 * 2;
constexpr uint32_t kTmemColsT = 512;

// The KL's per-row scratch (2N floats per row, kKlScStride-interleaved) sits in
// the tail of the warpgroup's own A tile: during the KL the tile holds only
// delta4 (K = NP columns, NP * 256 bytes); the cooperative small-batch KL uses
// warpgroup 1's tile, which has no tile of its own in that regime.
template <int N>
constexpr uint32_t kl_sc_off() { return (uint32_t)packed_width(N) * 256u; }
static_assert(packed_width(8) * 256 + 2 * 8 * kKlScStride * 4 <= kATile, "KL scratch fits the A tile tail");
static_assert((3 * 8 + 2 * kWGt) * kKlScStride * 4 <= kATile, "cooperative KL scratch fits an A tile");

// A tile of one chain: K = 128 activations / deltas, or delta4 (K = NP) with
// the KL scratch behind it when NP > 128
template <int N>
constexpr uint32_t a_tile_bytes() {
    return packed_width(N) <= 128 ? kATile
                                  : align1k((uint32_t)packed_width(N) * 256u + 2u * N * kKlScStride * 4u);
}

template <int N>
constexpr size_t fb_smem() {  // trainer image, A tiles, barriers, tile-stat partials
    return align1k(train_img_bytes(N)) + wgt_for(N) * a_tile_bytes<N>() + 64 + wgt_for(N) * 4 * 3 * sizeof(double);
}
static_assert(fb_smem<16>() <= 232448, "N = 16 trainer fits one SM's shared memory");

// Power-of-two scale exponent that maps a row maximum m to [2^13, 2^14)
// (0 for m = 0), bounded so the row's total scale 2^(E + k) stays a normal float.
__device__ __forceinline__ int row_scale_exp(float m, int E) {
    const int eb = (int)((__float_as_uint(m) >> 23) & 0xFFu);
    int k = eb == 0 ? 0 : 140 - eb;
    return min(max(k, -126 - E), 126 - E);
}
__device__ __forceinline__ float exp2i(int k) { return __uint_as_float((uint32_t)(k + 127) << 23); }  // |k| <= 126
__device__ __forceinline__ uint32_t mul_bf16x2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// byte offset of row t's 16-byte chunk c inside a 128-row block / A tile with F features
__device__ __forceinline__ uint32_t blk_off(int t, int F) { return (uint32_t)((t >> 3) * (F * 16) + (t & 7) * 16); }

__device__ __forceinline__ void st_g16(uint8_t *p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    *reinterpret_cast<uint4 *>(p) = make_uint4(a, b, c, d);
}

// the packed header columns of a row (16 for N <= 8, 32 for N = 16)
template <int HD>
__device__ __forceinline__ void tmem_ld_hdr(uint32_t taddr, float (&h)[HD]) {
    static_assert(HD == 16 || HD == 32, "packed header width");
    if constexpr (HD == 16) tc::tmem_ld16(taddr, h);
    else tc::tmem_ld32(taddr, h);
}

// ReLU gate flags of the 16 packed f16 pairs (32 columns) of a drain chunk in
// one register: pair j's halves set bits 15 - j and 31 - j.  After the ReLU
// satfinite conversion every half is a non-negative f16 <= 0x7BFF, so adding
// 0x7FFF to it sets its top bit exactly when it is non-zero, without a carry
// into the other half (3 instructions per pair: add, shift, and-or).
__device__ __forceinline__ uint32_t gate_flags(uint32_t acc, uint32_t p, int j) {
    const uint32_t q = p + 0x7FFF7FFFu;
    return acc | ((q >> j) & (0x80008000u >> j));
}
// 0xFFFF / 0x0000 per half of pair j from the chunk's flags: prmt replicates
// the sign bit of byte 1 (bit 15) over the low half and of byte 3 over the high
__device__ __forceinline__ uint32_t gate_mask(uint32_t flags, int j) {
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, 0xBB99;" : "=r"(r) : "r"(flags << j));
    return r;
}

// 128-row blocks of `rows` and how the dW GEMM spreads them over `splits`
// CTAs (the same plan on the host and, for a classified step, on the device)
__host__ __device__ __forceinline__ void split_plan(int64_t rows, int splits, int64_t &nb, int &bps) {
    nb = (rows + 127) / 128;
    bps = nb > 0 ? (int)((nb + splits - 1) / splits) : 0;
}

// ------------------------------------------------------------- classify --
// Rows with p = 0 take the zero-gradient path of kl_loss_gradient
// (guiding.cpp:112: zero gradient, valid) and loss_surrogate returns 0 for them
// (:170), counted (:267-270): the network output of such a row is only needed
// to decide "drop" when it is not finite (:247-250), which cannot happen while
// every weight is below kSafeWeight and the row's inputs are finite with
// |direction components| <= 2.  Those rows are counted and skipped; the rest
// (in row order, as source indices through the epoch permutation) form the
// step's list for K_fb and K_dw.  One pass, order-preserving, deterministic:
// 1024 rows per block, block offsets by decoupled look-back.  Consecutive
// steps alternate between two lists, so the classification of step s + 1 runs
// before the programmatic wait — overlapping step s's reduction and Adam — and
// only the weight flag (written by that Adam) is read after it: in the rare
// case it is set (some weight >= kSafeWeight), every row is kept instead.
constexpr int kClsThreads = 256, kClsRpt = 4, kClsRows = kClsThreads * kClsRpt;
constexpr int kClsEpochBits = 26, kClsValBits = 36;

__device__ __forceinline__ bool finite_dir(float4 v) {
    return fabsf(v.x) <= 2.f && fabsf(v.y) <= 2.f && fabsf(v.z) <= 2.f;  // false for NaN
}

__global__ void __launch_bounds__(kClsThreads)
train_classify_kernel(const nasg_train_sample *__restrict__ samples, const uint32_t *__restrict__ order, int64_t count,
                      const int *__restrict__ wbig, Bounds bd, uint32_t *__restrict__ live,
                      unsigned long long *state, uint32_t epoch, int64_t *cls, unsigned long long *clamp_count) {
    __shared__ int s_cnt[kClsRpt * 8], s_off[kClsRpt * 8];
    __shared__ long long s_prefix;
    __shared__ int s_clamped, s_total;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t base = (int64_t)blockIdx.x * kClsRows;
    if (tid == 0) s_clamped = 0;
    // the samples and the order were written before the previous step (host
    // uploads and copies are stream-ordered; a whole-buffer step has no order)
    uint32_t src[kClsRpt];
#pragma unroll
    for (int i = 0; i < kClsRpt; ++i) {
        const int64_t row = base + i * kClsThreads + tid;
        src[i] = row < count ? (order ? order[row] : (uint32_t)row) : 0u;
    }
    float4 a[kClsRpt], o[kClsRpt], n[kClsRpt];
#pragma unroll
    for (int i = 0; i < kClsRpt; ++i) {
        const int64_t row = base + i * kClsThreads + tid;
        if (row < count) {
            const float4 *sp = reinterpret_cast<const float4 *>(samples + src[i]);
            a[i] = sp[0]; o[i] = sp[1]; n[i] = sp[2];
        }
    }
    uint32_t bits = 0;
    int clamped = 0;
#pragma unroll
    for (int i = 0; i < kClsRpt; ++i) {
        const int64_t row = base + i * kClsThreads + tid;
        bool lv = false;
        if (row < count) {
            const bool zero = a[i].w == 0.f && isfinite(a[i].x) && isfinite(a[i].y) && isfinite(a[i].z) &&
                              finite_dir(o[i]) && finite_dir(n[i]);
            lv = !zero;
            if (zero) {  // its encode is skipped too: count its clamped coordinates here
                const float xs[3] = {a[i].x, a[i].y, a[i].z};
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) {
                    const float t = bd.inv_ext[ax] > 0.f ? (xs[ax] - bd.bmin[ax]) * bd.inv_ext[ax] : 0.5f;
                    clamped += (t < 0.f || t > 1.f) ? 1 : 0;
                }
            }
        }
        const uint32_t bl = __ballot_sync(0xffffffffu, lv);
        if (lane == 0) s_cnt[i * 8 + warp] = __popc(bl);
        bits |= (lv ? 1u : 0u) << i;
    }
    __syncthreads();
    if (warp == 0) {  // (i, warp) counts in row order -> exclusive offsets; block total; look-back
        const int v = s_cnt[lane];
        int inc = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += u;
        }
        s_off[lane] = inc - v;
        const int total = __shfl_sync(0xffffffffu, inc, 31);
        // decoupled look-back, a warp-wide window of 32 predecessors at a time:
        // lane i reads block (j - i); the window is summed up to the nearest
        // inclusive prefix (P), else wholly, and the walk moves 32 blocks back
        const unsigned long long tag = (unsigned long long)epoch << (kClsValBits + 2);
        const unsigned long long kA = 1ull << kClsValBits, kP = 2ull << kClsValBits;
        const unsigned long long vmask = (1ull << kClsValBits) - 1ull;
        long long prefix = 0;
        if (blockIdx.x == 0) {
            if (lane == 0) atomicExch(state, tag | kP | (unsigned long long)total);
        } else {
            if (lane == 0) atomicExch(state + blockIdx.x, tag | kA | (unsigned long long)total);
            for (int64_t j = (int64_t)blockIdx.x - 1;;) {
                const int64_t idx = j - lane;
                unsigned long long w = idx >= 0 ? *(volatile unsigned long long *)(state + idx) : (tag | kP);
                const bool ready = (w >> (kClsValBits + 2)) == epoch && (w & (kA | kP));
                if (!__all_sync(0xffffffffu, ready)) {  // a predecessor has not published yet
                    __nanosleep(32);
                    continue;
                }
                const uint32_t pm = __ballot_sync(0xffffffffu, (w & kP) != 0);
                const int stop = pm ? __ffs(pm) - 1 : 31;  // nearest inclusive prefix in the window
                long long v = lane <= stop ? (long long)(w & vmask) : 0;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
                prefix += v;
                if (pm) break;
                j -= 32;
            }
            if (lane == 0) atomicExch(state + blockIdx.x, tag | kP | (unsigned long long)(prefix + total));
        }
        if (lane == 0) {
            s_prefix = prefix;
            s_total = total;
        }
    }
    __syncthreads();
    pdl_wait();  // the previous step's Adam (its weight flag) and its readers of this list are done
    if (*(volatile const int *)wbig != 0) {  // rare: no row may skip the network; keep every row
#pragma unroll
        for (int i = 0; i < kClsRpt; ++i) {
            const int64_t row = base + i * kClsThreads + tid;
            if (row < count) live[row] = src[i];
        }
        if (blockIdx.x == 0 && tid == 0) {
            cls[0] = count;
            cls[1] = 0;
        }
        pdl_trigger();
        return;
    }
    if (clamped) atomicAdd(&s_clamped, clamped);  // the skipped rows' encode clamps (their encode is skipped)
    __syncthreads();
    if (tid == 0 && s_clamped && clamp_count) atomicAdd(clamp_count, (unsigned long long)s_clamped);
    if (tid == 0 && blockIdx.x == gridDim.x - 1) {  // {live, zero} after the weight flag is known
        cls[0] = s_prefix + s_total;
        cls[1] = count - (s_prefix + s_total);
    }
    const int64_t p0 = s_prefix;
#pragma unroll
    for (int i = 0; i < kClsRpt; ++i) {
        const bool lv = (bits >> i) & 1u;
        const uint32_t bl = __ballot_sync(0xffffffffu, lv);
        if (lv) {
            const int64_t at = p0 + s_off[i * 8 + warp] + __popc(bl & ((1u << lane) - 1u));
            NASG_CHECK(at < count, "classify: live list index");
            live[at] = src[i];
        }
    }
    pdl_trigger();
}

}  // namespace

size_t tc_train_block_bytes(int n_comp) {  // bf16 bytes per 128-row block over all 8 arrays
    return (size_t)(64 + 3 * 128 + 3 * 128 + packed_width(n_comp)) * 256;
}

// COOP (host-chosen when the step has no more tiles than SMs, kWGt > 1): one
// tile per CTA, and its three warpgroups split every phase of that tile's chain
// instead of warpgroup 0 running it alone: the forward and backward drains by
// 16-column units (unit u belongs to warpgroup u % 3; the ReLU gate bits stay
// with the warpgroup that drained those columns, the backward's row maximum is
// combined through shared memory) and the KL by lobes (kl_grad_row_coop).
// Warpgroup 0's warp 0 issues every MMA, after a barrier over all three.
template <int N, bool COOP>
__global__ void __launch_bounds__(wgt_for(N) * 128, 1)
train_tc_fb_kernel(const uint8_t *__restrict__ img, const nasg_train_sample *__restrict__ samples,
                   const uint32_t *__restrict__ order, int64_t count, const int64_t *live_count, double gscale,
                   double b, double e, Bounds bd, TcTrainBufs tb, unsigned long long *clamp_count) {
    constexpr int NP = packed_width(N);
    constexpr int kWGt = wgt_for(N);
    constexpr uint32_t kATile = a_tile_bytes<N>();
    constexpr uint32_t IMG = train_img_bytes(N);  // f16 layers + the bf16 copy of W4p^T at img_bytes(N)
    constexpr uint32_t A_OFF = align1k(IMG);
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t *acc_full = reinterpret_cast<uint64_t *>(smem + A_OFF + kWGt * kATile);
    uint64_t *w_bar = acc_full + kWGt;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(w_bar + 1);
    double *red = reinterpret_cast<double *>(smem + A_OFF + kWGt * kATile + 64);
    __shared__ int s_clamped;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int g = 0; g < kWGt; ++g) tc::mbar_init(&acc_full[g], 1);
        tc::mbar_init(w_bar, 1);
        s_clamped = 0;
        tc::fence_mbar_init();
    }
    if (warp == 0) tc::tmem_alloc(tmem_slot, kTmemColsT);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    NASG_CHECK(tc::dynamic_smem_bytes() >= fb_smem<N>(), "K_fb: dynamic shared memory");
    NASG_CHECK((kWGt - 1) * 128 + packed_width(N) <= (int)kTmemColsT, "K_fb: accumulators inside TMEM");
    pdl_trigger();
    pdl_wait();  // the weight image, the samples and the classified rows come from earlier work on the stream
    FB_TRACE(0, 15)
    if (live_count) count = *live_count;  // rows that need the network (order = their list)
    const int64_t ntiles = (count + 127) / 128;

    if (threadIdx.x == 0) {  // weights: TMA bulk copies global -> smem, once per CTA
        tc::mbar_arrive_expect_tx(w_bar, IMG);
        for (uint32_t off = 0; off < IMG; off += 16384)
            tc::bulk_g2s(smem + off, img + off, (IMG - off) < 16384u ? (IMG - off) : 16384u, w_bar);
    }
    {
        const int g = warp >> 2, t = threadIdx.x & 127;
        const int gt = COOP ? 0 : g;  // the warpgroup whose tile (accumulator, A tile) this thread works on
        const uint32_t my_tmem = tmem + gt * 128 + ((uint32_t)((warp & 3) * 32) << 16);
        const uint32_t a_base = tc::smem_u32(smem + A_OFF + gt * kATile);
        const uint32_t sW = tc::smem_u32(smem);
        // forward layer l (0..3): A = f16 activations (K = 64 | 128), B = the f16 W_l^T image (K-major)
        // backward through W_l (l = 3, 2, 1): A = delta (K = NP | 128), B = the image read MN-major:
        // l = 3 bf16 delta4 x the bf16 copy of W4p^T, l = 2, 1 row-scaled f16 deltas x the f16 image
        // warp 0 of the group issues with one elected lane; descriptors are rebuilt
        // from opaque base addresses (hoisted they would pin ~60 registers)
        auto issue = [&](int l, bool bwd) {
            tc::fence_proxy_async_smem();
            tc::tc_fence_before();
            if constexpr (COOP) asm volatile("bar.sync 8, %0;" ::"r"(kWGt * 128) : "memory");
            else wg_sync(g);
            if ((warp & 3) == 0 && (!COOP || g == 0)) {
                __syncwarp();
                tc::tc_fence_after();
                const uint32_t d = tmem + g * 128;
                const uint32_t abase = tc::opaque(a_base),
                               b0 = tc::opaque(sW) + ((bwd && l == 3) ? img_bytes(N) : w_off(l));
                if (!bwd) {
                    const int K = l == 0 ? kIn : kHidden;
                    const uint32_t sbo = (uint32_t)K * 16u;
                    const uint32_t idesc = tc::idesc_f16(128, l == 3 ? NP : kHidden);
                    const uint64_t ad = tc::smem_desc(abase, 128, sbo), bdsc = tc::smem_desc(b0, 128, sbo);
                    // +256 B per K=16 slab = +16 in the address field
                    if (l == 0) tc::mma_f16_chain_elect<kIn / 16>(d, ad, bdsc, idesc);
                    else tc::mma_f16_chain_elect<kHidden / 16>(d, ad, bdsc, idesc);
                } else {
                    constexpr uint32_t lbo_b = (uint32_t)kHidden * 16u;  // image rows (out index) in 8-groups
                    const uint32_t idesc = l == 3 ? tc::idesc_bf16(128, kHidden, false, true)
                                                  : tc::idesc_f16(128, kHidden, false, true);
                    const uint64_t bdsc = tc::smem_desc(b0, lbo_b, 128);
                    // contraction over W_l's output index; B advances 2 x 8 image rows per K=16 slab
                    if (l == 3)
                        tc::mma_f16_chain_elect<NP / 16, 16, 2 * lbo_b / 16>(
                            d, tc::smem_desc(abase, 128, (uint32_t)NP * 16u), bdsc, idesc);
                    else
                        tc::mma_f16_chain_elect<kHidden / 16, 16, 2 * lbo_b / 16>(
                            d, tc::smem_desc(abase, 128, (uint32_t)kHidden * 16u), bdsc, idesc);
                }
                tc::mma_commit_elect(&acc_full[g]);
            }
        };
        uint32_t acc_ph = 0;
        auto wait_acc = [&]() { wg_wait_acc(&acc_full[gt], acc_ph, g, warp & 3); };
        const float(&inv_ext)[3] = bd.inv_ext;
        int clamped = 0;
        const int64_t stride = (int64_t)gridDim.x * kWGt;
        float4 s0, s1, s2, s3;  // this row's sample; the next tile's is prefetched after the KL
        auto load_sample = [&](int64_t tl) {
            const int64_t row = tl * 128 + t;
            s0 = s1 = s2 = s3 = make_float4(0.f, 0.f, 0.f, 0.f);
            if (row < count) {  // gather through the epoch permutation (guiding.cpp:242-244)
                const int64_t src = order ? (int64_t)order[row] : row;
                const float4 *sp = reinterpret_cast<const float4 *>(samples + src);
                s0 = sp[0]; s1 = sp[1]; s2 = sp[2]; s3 = sp[3];
            }
        };
        // warpgroup-major tile order: a small batch (the render loop's t = 4096 is 32
        // tiles) spreads one tile per SM instead of three per SM on a third of them
        int64_t tile = COOP ? (int64_t)blockIdx.x : (int64_t)g * gridDim.x + blockIdx.x;
        // Small batch (no more tiles than CTAs): warpgroups 1 and 2 have no tile of
        // their own and take lobes of warpgroup 0's KL gradient instead (the step's
        // latency is one tile's chain; kl_grad_row_coop splits its longest link).
        // COOP: they also take their units of every drain.
        const bool coop = COOP || (kWGt > 1 && ntiles <= (int64_t)gridDim.x);
        float *rowmax = reinterpret_cast<float *>(smem + A_OFF + (kWGt - 1) * kATile);  // COOP: [3][128]
        float *coop_sc = reinterpret_cast<float *>(smem + A_OFF + kATile);           // [3N][128], group 1's tile
        int *coop_flg = reinterpret_cast<int *>(coop_sc + 3 * N * kKlScStride);     // [2 x 3][128]
        float *kl_scratch = reinterpret_cast<float *>(smem + A_OFF + g * kATile + kl_sc_off<N>());
        auto coop_sync = [&](int k) {  // the three warpgroups of the CTA; k = 0, 1 inside the KL, 2 at entry
            tc::fence_proxy_async_smem();  // delta4 chunks in the A tile -> visible to the tensor core
            tc::tc_fence_before();
            asm volatile("bar.sync %0, %1;" ::"r"(4 + k), "r"(kWGt * 128) : "memory");
            tc::tc_fence_after();
        };
        load_sample(tile);
        if ((warp & 3) == 0) tc::mbar_wait(w_bar, 0);  // weights resident before the first MMA issue
        FB_TRACE(0, 14)
        int ktr = 0;
        for (; tile < ntiles; tile += stride, ++ktr) {
            FB_TRACE(ktr, 0)
            NASG_CHECK(tile < tb.max_blocks, "K_fb: tile inside the h / delta block arrays");
            const int64_t row = tile * 128 + t;
            const bool valid = row < count;
            if (!COOP || g == 0)
                clamped += encode_row_f16(valid, s0, s1, s2, bd, inv_ext, a_base + blk_off(t, 64),
                                          tb.h0 + tile * (64 * 256) + blk_off(t, 64));
            FB_TRACE(ktr, 1)
            issue(0, false);
            uint32_t mask[3][4] = {};  // ReLU gate bits of h1..h3 (COOP: [layer][unit slot])
#pragma unroll 1
            for (int l = 1; l < 4; ++l) {  // hidden layers: ReLU, f16 A + gate bits, bf16 h_l block
                wait_acc();
                if constexpr (COOP) {  // this warpgroup's 16-column units u = g, g + 3, g + 6
                    uint8_t *gh = (l == 1 ? tb.h1 : (l == 2 ? tb.h2 : tb.h3)) + tile * (128 * 256) + blk_off(t, 128);
#pragma unroll
                    for (int sl = 0; sl < 3; ++sl) {
                        const int u = g + 3 * sl;
                        if (u < 8) {
                            float v[16];
                            tc::tmem_ld16(my_tmem + u * 16, v);
                            tc::tmem_ld_wait();
                            uint32_t bits = 0;
#pragma unroll
                            for (int c = 0; c < 2; ++c) {
                                uint32_t p[4], q[4];
#pragma unroll
                                for (int h = 0; h < 4; ++h) {
                                    p[h] = tc::pack_f16x2_relu_sat(v[8 * c + 2 * h], v[8 * c + 2 * h + 1]);
                                    q[h] = tc::pack_bf16x2_relu(v[8 * c + 2 * h], v[8 * c + 2 * h + 1]);
                                    bits = gate_flags(bits, p[h], 4 * c + h);
                                }
                                tc::st_shared_v4(a_base + blk_off(t, 128) + (2 * u + c) * 128, p[0], p[1], p[2], p[3]);
                                st_g16(gh + (2 * u + c) * 128, q[0], q[1], q[2], q[3]);
                            }
                            mask[0][sl] = l == 1 ? bits : mask[0][sl];
                            mask[1][sl] = l == 2 ? bits : mask[1][sl];
                            mask[2][sl] = l == 3 ? bits : mask[2][sl];
                        }
                    }
                    issue(l, false);
                    FB_TRACE(ktr, 1 + l)
                    continue;
                }
                uint8_t *gh = (l == 1 ? tb.h1 : (l == 2 ? tb.h2 : tb.h3)) + tile * (128 * 256) + blk_off(t, 128);
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    float v[32];
                    tc::tmem_ld32(my_tmem + q4 * 32, v);
                    tc::tmem_ld_wait();
                    uint32_t bits = 0;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint32_t p[4], q[4];
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            // a non-negative satfinite f16 is <= 0x7BFF: the same carry-free flag trick
                            p[h] = tc::pack_f16x2_relu_sat(v[8 * c + 2 * h], v[8 * c + 2 * h + 1]);
                            q[h] = tc::pack_bf16x2_relu(v[8 * c + 2 * h], v[8 * c + 2 * h + 1]);
                            bits = gate_flags(bits, p[h], 4 * c + h);
                        }
                        tc::st_shared_v4(a_base + blk_off(t, 128) + (q4 * 4 + c) * 128, p[0], p[1], p[2], p[3]);
                        st_g16(gh + (q4 * 4 + c) * 128, q[0], q[1], q[2], q[3]);
                    }
                    // register-resident gate bits: select instead of a dynamic index
                    mask[0][q4] = l == 1 ? bits : mask[0][q4];
                    mask[1][q4] = l == 2 ? bits : mask[1][q4];
                    mask[2][q4] = l == 3 ? bits : mask[2][q4];
                }
                issue(l, false);
                FB_TRACE(ktr, 1 + l)
            }
            wait_acc();
            FB_TRACE(ktr, 5)
            if (coop) coop_sync(2);  // the raw outputs are in tensor memory: helpers may read them
            // ---- KL gradient (fp32 stable forms) straight out of tensor memory:
            // header columns once, each lobe's 8 columns per pass; delta4 goes
            // to the A tile (K = NP) and the d4 block one 16-byte chunk at a time.
            constexpr int HD = packed_header(N);
            uint8_t *gd4 = tb.d4 + tile * (NP * 256) + blk_off(t, NP);
            const uint32_t a4 = a_base + blk_off(t, NP);
            auto put_chunk = [&](int c, const float *g8) {
                const uint32_t p0 = tc::pack_bf16x2(g8[0], g8[1]), p1 = tc::pack_bf16x2(g8[2], g8[3]),
                               p2 = tc::pack_bf16x2(g8[4], g8[5]), p3 = tc::pack_bf16x2(g8[6], g8[7]);
                tc::st_shared_v4(a4 + c * 128, p0, p1, p2, p3);
                st_g16(gd4 + c * 128, p0, p1, p2, p3);
            };
            float hdr[HD];
            tmem_ld_hdr(my_tmem, hdr);
            tc::tmem_ld_wait();
            TrainRow srow;
            srow.wi = make_float3(s3.x, s3.y, s3.z);
            srow.p = s0.w;
            srow.q_s = s1.w;
            srow.pbsdf = s2.w;
            float lossf = 0.f;
            int st;
            {  // every thread of the warp runs the tensor-memory loads (valid or not)
                float ghdr[HD];
                auto lobe = [&](int i, float (&r)[8]) {
                    __syncwarp();
                    tc::tmem_ld8_sync(my_tmem + HD + 8 * i, r);
                };
                auto put_lobe = [&](int i, const float (&g8)[8]) { put_chunk(HD / 8 + i, g8); };
                if (coop)
                    st = kl_grad_row_coop<N, kWGt>(COOP ? g : 0, valid, hdr, lobe, srow, (float)b, (float)e,
                                                   (float)gscale, ghdr, put_lobe, lossf, coop_sc + t, coop_flg + t,
                                                   coop_sync);
                else
                    st = kl_grad_row_fast<N>(valid, hdr, lobe, srow, (float)b, (float)e, (float)gscale, ghdr,
                                             put_lobe, lossf, kl_scratch + t);
                if (st == kKlOk) {
#pragma unroll
                    for (int c = 0; c < HD / 8; ++c) put_chunk(c, ghdr + 8 * c);
                }
            }
            if (st != kKlOk && (!COOP || g == 0)) {  // zero row: invalid, p = 0 or dropped
                const float z8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
                for (int c = 0; c < NP / 8; ++c) put_chunk(c, z8);
            }
            // 0 invalid row, 1 loss counted, 2 dropped, 3 ok but loss not finite
            const int state = !valid ? 0 : (st == kKlDrop ? 2 : ((st == kKlZero || isfinite(lossf)) ? 1 : 3));
            const double loss = lossf;
            FB_TRACE(ktr, 6)
            issue(3, true);
            load_sample(tile + stride);  // prefetch: in flight through the backward pass
            if (!COOP || g == 0) {  // tile statistics, deterministic order (warp tree, then warps 0..3)
                double ls = state == 1 ? loss : 0.0, lc = state == 1 ? 1.0 : 0.0, dr = state == 2 ? 1.0 : 0.0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    ls += __shfl_xor_sync(0xffffffffu, ls, o);
                    lc += __shfl_xor_sync(0xffffffffu, lc, o);
                    dr += __shfl_xor_sync(0xffffffffu, dr, o);
                }
                double *rg = red + g * 12;
                if (lane == 0) {
                    rg[(warp & 3) * 3] = ls;
                    rg[(warp & 3) * 3 + 1] = lc;
                    rg[(warp & 3) * 3 + 2] = dr;
                }
                wg_sync(g);
                if (t == 0) {
                    tb.tile_loss[tile] = ((rg[0] + rg[3]) + rg[6]) + rg[9];
                    tb.tile_lc[tile] = (int)(rg[1] + rg[4] + rg[7] + rg[10]);
                    tb.tile_dr[tile] = (int)(rg[2] + rg[5] + rg[8] + rg[11]);
                }
            }
            // ---- backward: delta_l = (delta_{l+1} W_l^T) .* [h_l > 0]
            // The accumulator of layer l holds delta_l * 2^E (E = 0 for delta3, which
            // comes from bf16 delta4 x bf16 W4).  Its f16 A operand for the next layer
            // is rescaled per row so the row maximum lands in [2^13, 2^14): deltas
            // keep f16's 11-bit precision whatever their magnitude (the 1/count
            // factor and w = p/q_s span decades), and the backward is row-linear, so
            // the next accumulator is exactly delta * 2^(E + k).  The bf16 copy for
            // the dW GEMM is unscaled (exact power-of-two multiply).
            int E = 0;
            static_for<0, 3>([&](auto jc) {
                constexpr int l = 3 - decltype(jc)::value;
                wait_acc();
                if constexpr (COOP) {  // this warpgroup's units; the row maximum combined over the three
                    uint8_t *gd = (l == 1 ? tb.d1 : (l == 2 ? tb.d2 : tb.d3)) + tile * (128 * 256) + blk_off(t, 128);
                    int k = 0;
                    if (l > 1) {
                        float m = 0.f;
#pragma unroll
                        for (int sl = 0; sl < 3; ++sl) {
                            const int u = g + 3 * sl;
                            if (u < 8) {
                                float v[16];
                                tc::tmem_ld16(my_tmem + u * 16, v);
                                tc::tmem_ld_wait();
#pragma unroll
                                for (int jj = 0; jj < 16; ++jj) m = fmaxf(m, fabsf(v[jj]));
                            }
                        }
                        rowmax[g * 128 + t] = m;
                        asm volatile("bar.sync 10, %0;" ::"r"(kWGt * 128) : "memory");
                        m = fmaxf(fmaxf(rowmax[t], rowmax[128 + t]), rowmax[256 + t]);
                        k = row_scale_exp(m, E);
                    }
                    const float ks = exp2i(k);
                    const uint32_t un = (uint32_t)(127 - E) << 7, unscale = un | (un << 16);  // 2^-E as bf16x2
#pragma unroll
                    for (int sl = 0; sl < 3; ++sl) {
                        const int u = g + 3 * sl;
                        if (u < 8) {
                            float v[16];
                            tc::tmem_ld16(my_tmem + u * 16, v);
                            tc::tmem_ld_wait();
                            const uint32_t bits = mask[l - 1][sl];
#pragma unroll
                            for (int c = 0; c < 2; ++c) {
                                uint32_t p[4], q[4];
#pragma unroll
                                for (int h = 0; h < 4; ++h) {
                                    const int i0 = 8 * c + 2 * h;
                                    const uint32_t gm = gate_mask(bits, 4 * c + h);
                                    q[h] = tc::pack_bf16x2(v[i0], v[i0 + 1]);
                                    if (l < 3) q[h] = mul_bf16x2(q[h], unscale);
                                    q[h] &= gm;
                                    if (l > 1) p[h] = tc::pack_f16x2_sat(v[i0] * ks, v[i0 + 1] * ks) & gm;
                                }
                                if (l > 1)
                                    tc::st_shared_v4(a_base + blk_off(t, 128) + (2 * u + c) * 128, p[0], p[1], p[2], p[3]);
                                st_g16(gd + (2 * u + c) * 128, q[0], q[1], q[2], q[3]);
                            }
                        }
                    }
                    E += k;
                    if (l > 1) issue(l - 1, true);
                    FB_TRACE(ktr, 10 - l)
                    return;
                }
                uint8_t *gd = (l == 1 ? tb.d1 : (l == 2 ? tb.d2 : tb.d3)) + tile * (128 * 256) + blk_off(t, 128);
                int k = 0;
                if (l > 1) {  // pass 1: the row's maximum |value|
                    float m = 0.f;
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        float v[32];
                        tc::tmem_ld32(my_tmem + q4 * 32, v);
                        tc::tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 32; ++j) m = fmaxf(m, fabsf(v[j]));
                    }
                    k = row_scale_exp(m, E);
                }
                const float ks = exp2i(k);
                const uint32_t un = (uint32_t)(127 - E) << 7, unscale = un | (un << 16);  // 2^-E as bf16x2
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    float v[32];
                    tc::tmem_ld32(my_tmem + q4 * 32, v);
                    tc::tmem_ld_wait();
                    const uint32_t bits = mask[l - 1][q4];
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint32_t p[4], q[4];
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            const int i0 = 8 * c + 2 * h;
                            const uint32_t gm = gate_mask(bits, 4 * c + h);
                            q[h] = tc::pack_bf16x2(v[i0], v[i0 + 1]);
                            if (l < 3) q[h] = mul_bf16x2(q[h], unscale);
                            q[h] &= gm;
                            if (l > 1) p[h] = tc::pack_f16x2_sat(v[i0] * ks, v[i0 + 1] * ks) & gm;
                        }
                        if (l > 1) tc::st_shared_v4(a_base + blk_off(t, 128) + (q4 * 4 + c) * 128, p[0], p[1], p[2], p[3]);
                        st_g16(gd + (q4 * 4 + c) * 128, q[0], q[1], q[2], q[3]);
                    }
                }
                E += k;
                if (l > 1) issue(l - 1, true);
                FB_TRACE(ktr, 10 - l)
            });
            tc::tc_fence_before();
        }
        if (!COOP && coop && g > 0 && (int64_t)blockIdx.x < ntiles) {  // helper in warpgroup 0's KL
            constexpr int HD = packed_header(N);
            const int64_t tl = blockIdx.x;
            load_sample(tl);
            const bool valid = tl * 128 + t < count;
            const uint32_t tm0 = tmem + ((uint32_t)((warp & 3) * 32) << 16);  // group 0's columns, this lane quarter
            uint8_t *gd4 = tb.d4 + tl * (NP * 256) + blk_off(t, NP);
            const uint32_t a4 = tc::smem_u32(smem + A_OFF) + blk_off(t, NP);  // group 0's A tile
            auto put_lobe = [&](int i, const float (&g8)[8]) {
                const uint32_t p0 = tc::pack_bf16x2(g8[0], g8[1]), p1 = tc::pack_bf16x2(g8[2], g8[3]),
                               p2 = tc::pack_bf16x2(g8[4], g8[5]), p3 = tc::pack_bf16x2(g8[6], g8[7]);
                const int c = HD / 8 + i;
                tc::st_shared_v4(a4 + c * 128, p0, p1, p2, p3);
                st_g16(gd4 + c * 128, p0, p1, p2, p3);
            };
            auto lobe = [&](int i, float (&r)[8]) {
                __syncwarp();
                tc::tmem_ld8_sync(tm0 + HD + 8 * i, r);
            };
            coop_sync(2);
            float hdr[HD], ghdr[HD];
            tmem_ld_hdr(tm0, hdr);
            tc::tmem_ld_wait();
            TrainRow srow;
            srow.wi = make_float3(s3.x, s3.y, s3.z);
            srow.p = s0.w;
            srow.q_s = s1.w;
            srow.pbsdf = s2.w;
            float lossf = 0.f;
            kl_grad_row_coop<N, kWGt>(g, valid, hdr, lobe, srow, (float)b, (float)e, (float)gscale, ghdr, put_lobe,
                                      lossf, coop_sc + t, coop_flg + t, coop_sync);
        }
        if (clamped) atomicAdd(&s_clamped, clamped);
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem, kTmemColsT);
    }
    if (threadIdx.x == 0 && s_clamped && clamp_count) atomicAdd(clamp_count, (unsigned long long)s_clamped);
}

// ------------------------------------------------------------------- K_dw --
// row stride (floats) of one split's [128][.] dW partial: 128, or NP when wider
__host__ __device__ constexpr int partial_stride(int np) { return np > 128 ? np : 128; }

// grid (splits, 4 layers).  Layer L computes D[128][FB] = A^T-contraction over
// rows of A block [rows][128] and B block [rows][FB], both MN-major:
//   L0: A = delta1, B = h0 -> dW1^T   L1: A = h1, B = delta2 -> dW2
//   L2: A = h2, B = delta3 -> dW3     L3: A = h3, B = delta4 -> dW4 (packed cols)
__global__ void __launch_bounds__(128, 1)
train_tc_dw_kernel(TcTrainBufs tb, int64_t nblocks, int bps, int np, const int64_t *live_count) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int L = blockIdx.y;
    const uint8_t *A = L == 0 ? tb.d1 : (L == 1 ? tb.h1 : (L == 2 ? tb.h2 : tb.h3));
    const uint8_t *B = L == 0 ? tb.h0 : (L == 1 ? tb.d2 : (L == 2 ? tb.d3 : tb.d4));
    const int FB = L == 0 ? 64 : (L == 3 ? np : 128);
    const uint32_t abytes = 128u * 256u, bbytes = (uint32_t)FB * 256u;
    constexpr uint32_t kStage = 73728;  // A block 32 KB + B block up to 160 x 256 B
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + 2 * kStage);
    uint64_t *empty = full + 2;
    uint64_t *done = full + 4;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(full + 5);
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(done, 1);
        tc::fence_mbar_init();
    }
    if (warp == 0) tc::tmem_alloc(tmem_slot, 256);  // FB <= 160 fp32 columns
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_trigger();
    pdl_wait();  // the h / delta blocks of K_fb
    if (live_count) split_plan(*live_count, gridDim.x, nblocks, bps);
    const int64_t b0 = (int64_t)blockIdx.x * bps, b1 = min(nblocks, b0 + bps);
    NASG_CHECK(tc::dynamic_smem_bytes() >= 2 * kStage + 64 && (int)blockIdx.x < tb.splits && nblocks <= tb.max_blocks &&
                   FB <= 256,
               "K_dw: shared memory, split index, block range, accumulator columns");
    if (threadIdx.x == 0 && b1 > b0) {
        const uint32_t idesc = tc::idesc_bf16(128, FB, true, true);
        auto load = [&](int64_t blk, int s) {
            tc::mbar_arrive_expect_tx(&full[s], abytes + bbytes);
            for (uint32_t off = 0; off < abytes; off += 16384)
                tc::bulk_g2s(smem + s * kStage + off, A + blk * abytes + off, 16384, &full[s]);
            for (uint32_t off = 0; off < bbytes; off += 16384)
                tc::bulk_g2s(smem + s * kStage + abytes + off, B + blk * bbytes + off,
                             (bbytes - off) < 16384u ? (bbytes - off) : 16384u, &full[s]);
        };
        uint32_t fph[2] = {0, 0}, eph[2] = {0, 0};
        load(b0, 0);
        if (b0 + 1 < b1) load(b0 + 1, 1);
        for (int64_t i = b0; i < b1; ++i) {
            const int s = (int)((i - b0) & 1);
            tc::mbar_wait(&full[s], fph[s]);
            fph[s] ^= 1u;
            tc::tc_fence_after();
            const uint32_t sa = tc::smem_u32(smem + s * kStage), sb = sa + abytes;
            for (int k = 0; k < 8; ++k)  // 128 rows = 8 x K16
                tc::mma_bf16(tmem, tc::smem_desc(sa + k * 2 * 2048, 2048, 128),
                             tc::smem_desc(sb + k * 2 * (FB * 16), FB * 16, 128), idesc, (i > b0 || k > 0) ? 1u : 0u);
            tc::mma_commit(&empty[s]);
            if (i + 2 < b1) {
                tc::mbar_wait(&empty[s], eph[s]);
                eph[s] ^= 1u;
                load(i + 2, s);
            }
        }
        tc::mma_commit(done);
    }
    __syncthreads();
    if (b1 > b0) {
        tc::mbar_wait(done, 0);
        tc::tc_fence_after();
        const int ps = partial_stride(np);
        float *out = tb.partial + ((size_t)L * tb.splits + blockIdx.x) * (128 * ps) + threadIdx.x * ps;
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
        for (int q = 0; q < FB / 16; ++q) {
            float v[16];
            tc::tmem_ld16(ta + q * 16, v);
            tc::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; i += 4)
                *reinterpret_cast<float4 *>(out + q * 16 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem, 256);
    }
}

// canonical grad[e] = sum over splits (fixed order) of the layer partials; the
// grid's extra last block reduces the per-tile loss / count / drop statistics
// of the step (same fixed order as step_stats_kernel), saving a launch.
__global__ void train_tc_reduce_kernel(TcTrainBufs tb, int splits, int n_comp, float *grad, int *nonfinite,
                                       int ntiles, const int64_t *cls) {
    pdl_trigger();
    pdl_wait();  // K_dw's partials
    double zero_rows = 0.0;
    if (cls) {  // the classified step: live tiles, the splits that got blocks, rows skipped as zero-gradient
        int64_t nb;
        int bps;
        split_plan(cls[0], splits, nb, bps);
        ntiles = (int)nb;
        splits = bps > 0 ? (int)((nb + bps - 1) / bps) : 0;
        zero_rows = (double)cls[1];
    }
    if (blockIdx.x == gridDim.x - 1) {
        __shared__ double sl[128], sc[128], sd[128];
        const int t = threadIdx.x;
        double ls = 0.0, lc = 0.0, dr = 0.0;
        for (int i = t; i < ntiles; i += 128) {
            ls += tb.tile_loss[i];
            lc += tb.tile_lc[i];
            dr += tb.tile_dr[i];
        }
        sl[t] = ls; sc[t] = lc; sd[t] = dr;
        __syncthreads();
        for (int h = 64; h > 0; h >>= 1) {
            if (t < h) {
                sl[t] += sl[t + h];
                sc[t] += sc[t + h];
                sd[t] += sd[t + h];
            }
            __syncthreads();
        }
        if (t == 0) {  // zero-gradient rows: loss 0, counted (guiding.cpp:170, :267-270)
            tb.step_stats[0] = sl[0];
            tb.step_stats[1] = sc[0] + zero_rows;
            tb.step_stats[2] = sd[0];
        }
        return;
    }
    // 4 warps per block share 32 consecutive weights: warp q sums the splits
    // k = q, q + 4, ...; the four partial sums are added in fixed order
    // ((s0 + s1) + (s2 + s3)): deterministic, a quarter of the dependent chain
    __shared__ float quarter[4][32];
    const int nw = n_weights(n_comp), D = 8 * n_comp + 1;
    const int o1 = kIn * kHidden, o2 = o1 + kHidden * kHidden, o3 = o2 + kHidden * kHidden;
    const int q = threadIdx.x >> 5;
    int e = blockIdx.x * 32 + (threadIdx.x & 31);
    const bool has = e < nw;
    if (!has) e = nw - 1;
    int L, m, n;
    // dW1^T[n_out][k_in] partials: consecutive threads take consecutive k_in so
    // the split loads coalesce; the canonical W1 index (k_in * 128 + n_out) is
    // then a strided store, once per weight
    if (e < o1) { L = 0; m = e / kIn; n = e % kIn; e = n * kHidden + m; }
    else if (e < o2) { L = 1; m = (e - o1) / kHidden; n = (e - o1) % kHidden; }
    else if (e < o3) { L = 2; m = (e - o2) / kHidden; n = (e - o2) % kHidden; }
    else { L = 3; m = (e - o3) / D; n = packed_col((e - o3) % D, n_comp); }
    const int ps = partial_stride(packed_width(n_comp));
    const float *p = tb.partial + (size_t)L * tb.splits * (128 * ps) + m * ps + n;
    float s = 0.f;
    for (int k = q; k < splits; k += 4) s += p[(size_t)k * (128 * ps)];
    quarter[q][threadIdx.x & 31] = s;
    __syncthreads();
    if (q == 0 && has) {
        const int l = threadIdx.x & 31;
        s = (quarter[0][l] + quarter[1][l]) + (quarter[2][l] + quarter[3][l]);
        grad[e] = s;
        if (!isfinite(s)) atomicOr(nonfinite, 1);
    }
}

int train_classify(const nasg_train_sample *samples, const uint32_t *order, int64_t count, TcTrainBufs &tb,
                   const Bounds &bounds, unsigned long long *clamp_count, cudaStream_t s, bool pdl) {
    const int nblk = (int)((count + kClsRows - 1) / kClsRows);
    if (++tb.scan_epoch >= (1u << kClsEpochBits)) {  // look-back tags wrapped: start clean
        cudaMemsetAsync(tb.scan_state, 0, tb.scan_cap * sizeof(unsigned long long), s);
        tb.scan_epoch = 1;
    }
    tb.cls_par ^= 1;  // the other list: the previous step's readers may still be running
    launch_pdl(pdl, train_classify_kernel, dim3(nblk), dim3(kClsThreads), 0, s, samples, order, count, tb.wbig, bounds,
               tb.cur_live(), tb.scan_state, tb.scan_epoch, tb.cur_cls(), clamp_count);
    return 1;
}

int train_tc_step(int n_comp, const void *img, const nasg_train_sample *samples, const uint32_t *order, int64_t count,
                  int64_t global_count, double b, double loss_blend, const Bounds &bounds, TcTrainBufs &tb,
                  int num_sms, unsigned long long *clamp_count, float *grad, int *nonfinite, cudaStream_t s,
                  bool pdl) {
    if (n_comp != 8 && n_comp != 4 && n_comp != 16) return -1;
    const int64_t ntiles = (count + 127) / 128;
    const double gscale = 1.0 / (double)global_count;
    int launches = 0;
    if (ntiles > 0) {
        // zero-gradient rows out of the network pass (train_classify_kernel): K_fb
        // walks the list of the others, K_dw and the reduction size themselves
        // from its length on the device.  Only when there are more tiles than
        // SMs: below that every tile already has its own CTA (the step is one
        // tile's latency chain) and the extra launch would only add to it.
        const int64_t *live_count = nullptr;
        const uint32_t *rows = order;
        if (tb.skip_zero && ntiles > num_sms) {
            launches += train_classify(samples, order, count, tb, bounds, clamp_count, s, pdl);
            live_count = tb.cur_cls();
            rows = tb.cur_live();
        }
        const int grid = (int)(ntiles < num_sms ? ntiles : num_sms);
        const uint8_t *im = static_cast<const uint8_t *>(img);
        // one tile per CTA and no classification: the three warpgroups split the tile's chain
        const bool coop_split = !live_count && ntiles <= num_sms && getenv("NASG_NO_COOP_SPLIT") == nullptr;
        auto launch_fb = [&](auto nc) {
            constexpr int NC = decltype(nc)::value;
            constexpr size_t sm = fb_smem<NC>();
            auto go = [&](auto kern) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                launch_pdl(pdl, kern, dim3(grid), dim3(wgt_for(NC) * 128), sm, s, im, samples, rows, count,
                           live_count, gscale, b, loss_blend, bounds, tb, clamp_count);
            };
            if constexpr (wgt_for(NC) > 1) {
                if (coop_split) {
                    go(train_tc_fb_kernel<NC, true>);
                    return;
                }
            }
            go(train_tc_fb_kernel<NC, false>);
        };
        if (n_comp == 8) launch_fb(std::integral_constant<int, 8>{});
        else if (n_comp == 4) launch_fb(std::integral_constant<int, 4>{});
        else launch_fb(std::integral_constant<int, 16>{});
        int64_t nb;
        int bps;
        int splits = (int)(ntiles < tb.splits ? ntiles : tb.splits);
        split_plan(count, splits, nb, bps);
        if (!live_count) splits = (int)((ntiles + bps - 1) / bps);  // every launched split gets blocks
        const size_t sm = 2 * 73728 + 64;
        cudaFuncSetAttribute(train_tc_dw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        launch_pdl(pdl, train_tc_dw_kernel, dim3(splits, 4), dim3(128), sm, s, tb, ntiles, bps, packed_width(n_comp),
                   live_count);
        const int nw = n_weights(n_comp);
        launch_pdl(pdl, train_tc_reduce_kernel, dim3((nw + 31) / 32 + 1), dim3(128), 0, s, tb, splits, n_comp, grad,
                   nonfinite, (int)ntiles, live_count);
        launches += 3;
    }
    return launches;
}

}  // namespace nasg
