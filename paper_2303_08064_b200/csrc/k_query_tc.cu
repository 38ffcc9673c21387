// Tensor-core query path (NASG_MLP_BF16): fused encode -> 64-128-128-128-NP
// MLP on tcgen05 kind::f16 with f16 operands (UMMA M=128, fp32 accumulators
// in TMEM) -> fp32 NASG epilogue.  f16 rather than bf16 operands: the same
// tensor-core rate and bytes, 3 more mantissa bits (raw outputs ~8x closer to
// the fp32 reference); the MLP's weights and activations sit far inside f16's
// range (conversions saturate at +-65504, NaN propagates).
//
// Persistent CTA per SM (16 warps), warp-specialised into two pipelines
// ("pairs").  Pair m = one MLP warpgroup + one NASG warpgroup; thread t of a
// group owns row t of the pair's current 128-row tile (= TMEM lane t).
//   MLP warpgroup m (warps 4m..4m+3, 104 registers): only the latency-critical
//     chain.  Layer 0 reads the encoded tile E_m straight from smem; for
//     layers 1-3 the group drains its TMEM accumulator [128m, 128m+128) ->
//     ReLU -> f16 -> A tile; warp 0 issues each layer's UMMAs with one
//     elected lane and commits them to acc_full[m].  The output layer writes
//     the pair's raw buffer (TMEM [256+128m, 256+128m+NP)) once the NASG group
//     has emptied it and commits to raw_full[m].
//   NASG warpgroup m (warps 8+4m..11+4m, 152 registers): everything with
//     slack.  It stages tile inputs by TMA bulk copies two tiles ahead, encodes
//     the NEXT tile (one-blob, encoding.cpp:21-46) into E_m as soon as the
//     MLP's layer 0 has consumed it (e_empty[m]), then waits raw_full[m],
//     copies its rows' raw outputs to registers, releases the buffer and runs
//     decode / sample / pdf (nasg_math.cuh) while the MLP computes the next tile.
// The MLP chain (4 MMA round trips) is bound by latency, the NASG side by
// instruction issue; this split keeps the chain free of every instruction
// that can run elsewhere.  setmaxnreg moves registers from MLP to NASG groups.
// N = 16 (NP = 160): one MLP warpgroup and two NASG warpgroups ("slots") that
// take its tiles alternately, each with its own E buffer, input stage and raw
// buffer (TMEM [128 + 160 j, ...)) — the 16-lobe epilogue is about twice the
// MLP's work per tile.  N = 32 (NP = 304): one MLP warpgroup and one NASG lane
// served by two warpgroups that split each row's lobes (16 each; the picked
// lobe's logits and the partial pdf sums cross through TMEM columns behind the
// raw buffer), raw buffer TMEM [128, 432) written by two
// output MMAs (N = 256 + 48); they stream the row's lobes out of tensor memory
// (the 304 columns do not fit in registers).
// Only the 52 B/query of inputs and 16-20 B/query of outputs touch HBM.
#include <cuda_bf16.h>

#include "nasg_internal.h"
#include "nasg_math.cuh"
#include "tc_ptx.cuh"
#include "tc_common.cuh"


// Development-only phase timestamps (build with EXTRA=-DNASG_TRACE into a
// scratch directory; the shipped library compiles them out): clock64() of
// thread 0 of pair 0 in CTA 0 at fixed points of the first 32 tiles.
#ifdef NASG_TRACE
__device__ unsigned long long g_trace[2 * 32 * 16];
extern "C" int nasg_trace_read(void *host) { return (int)cudaMemcpyFromSymbol(host, g_trace, sizeof(g_trace)); }
#define NASG_TRACE_AT(role, k, slot)                                                   \
    if (blockIdx.x == 0 && t == 0 && m == 0 && j == 0 && (k) < 32)                     \
        g_trace[((role) * 32 + (k)) * 16 + (slot)] = clock64();
#else
#define NASG_TRACE_AT(role, k, slot)
#endif

namespace nasg {

namespace {

// MLP warpgroups ("pairs") per CTA and NASG warpgroups ("slots") per MLP
// warpgroup.  N <= 8 (NP <= 80): two pairs of one MLP + one NASG warpgroup, raw
// buffers TMEM [256 + 128 m, ...).  N = 16 (NP = 160): one MLP warpgroup feeding
// two NASG warpgroups that take its tiles alternately (the 16-lobe epilogue is
// twice the MLP's work per tile), raw buffers TMEM [128, 288) and [288, 448).
constexpr int pairs_for(int n) { return packed_width(n) > 128 ? 1 : 2; }
constexpr int slots_for(int n) { return packed_width(n) > 256 ? 1 : (packed_width(n) > 128 ? 2 : 1); }
// N = 32: the row's lobes streamed from TMEM by two warpgroups per NASG lane (the
// 304 columns do not fit in registers).  The same split at N = 8 (four NASG
// warpgroups at 96 registers, MLP at 48) ran at 5.77e9 vs 8.02e9 q/s: reverted.
constexpr bool streamed(int n) { return packed_width(n) > 256; }
constexpr int nasg_wgs(int n) { return streamed(n) ? 2 : 1; }      // warpgroups per NASG lane
constexpr int threads_for(int n) { return pairs_for(n) * (1 + slots_for(n) * nasg_wgs(n)) * 128; }
constexpr uint32_t raw_col(int n, int lane) {  // first TMEM column of NASG lane (pair m, slot j) = m * S + j
    return pairs_for(n) == 2 ? 256u + 128u * (uint32_t)lane : 128u + 160u * (uint32_t)lane;
}
// setmaxnreg split between the MLP and the NASG warpgroups.  The NASG groups
// can only grow into what the MLP groups release from the launch allocation
// (the kernel's register count: 128 at 512 threads, 168 at 384), or they wait
// forever: P x 4 x (launch - MLP) >= P x S x 4 x (NASG - launch).
//   N <= 8 (launch 128): N = 8 runs NASG-bound (96 / 160 measured +0.9 % over
//   104 / 152), N = 4's lighter epilogue leaves the MLP side the longer chain
//   (104 / 152: 9.50e9 vs 8.46e9 q/s);  N = 16 (launch 168): 96 / 200 / 200.
constexpr int regs_mlp(int n) { return n == 4 ? 104 : 96; }
constexpr int launch_regs(int n) { return pairs_for(n) == 2 ? 128 : 168; }
constexpr int regs_nasg(int n) { return pairs_for(n) == 2 ? 256 - regs_mlp(n) : 200; }
static_assert(4 * (launch_regs(16) - regs_mlp(16)) >= 2 * 4 * (regs_nasg(16) - launch_regs(16)),
              "N = 16: the NASG groups' setmaxnreg.inc fits what the MLP group releases");
static_assert(4 * (launch_regs(8) - regs_mlp(8)) >= 4 * (regs_nasg(8) - launch_regs(8)), "N = 8 register split");
static_assert(4 * (launch_regs(32) - regs_mlp(32)) >= 2 * 4 * (regs_nasg(32) - launch_regs(32)), "N = 32 register split");
constexpr uint32_t kABytes = 128 * 128 * 2;     // one f16 activation tile, K = 128
constexpr uint32_t kTmemCols = 512;             // [acc0 | acc1 | raw0 | raw1], 128 columns each

constexpr uint32_t kEBytes = 128 * 64 * 2;      // one encoded tile (layer 0's A operand, K = 64)
constexpr uint32_t kInBytes = 128 * 52;         // one tile of inputs: 13-float rows or 3 x 2 KB SoA

template <int N>
constexpr size_t smem_bytes() {
    constexpr int P = pairs_for(N), Q = pairs_for(N) * slots_for(N);
    return align1k(img_bytes(N)) + P * kABytes + Q * kEBytes + 2 * Q * kInBytes + (P + 6 * Q + 2) * sizeof(uint64_t);
}
static_assert(smem_bytes<32>() <= 232448, "N = 32 query kernel fits one SM's shared memory");

}  // namespace

size_t tc_image_bytes(int n) { return img_bytes(n); }
size_t tc_train_image_bytes(int n) { return train_img_bytes(n); }
// queries: NP = 48 / 80 / 160 / 304 (N % 16 == 0; two output MMAs past 256)
bool tc_supported(int n) { return n == 4 || n == 8 || n == 16 || n == 32; }
// training: the trainer's f16 image + bf16 W4 copy + delta4 tile fit one SM up to N = 16
bool tc_train_supported(int n) { return n == 4 || n == 8 || n == 16; }

// ------------------------------------------------------------------ packing --
// f16 image of the four layers (both tensor-core kernels); train = 1 appends
// the trainer's bf16 copy of W4p^T (train_img_bytes)
__global__ void pack_tc_kernel(const float *__restrict__ w, int n_comp, uint16_t *__restrict__ img, int train) {
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
        const uint32_t byte = img_elem_off(l, n, k);
        img[byte / 2] = __half_as_ushort(__float2half_rn(sat_f16_range(v)));
        if (train && l == 3) img[(img_bytes(n_comp) + byte - w_off(3)) / 2] = __bfloat16_as_ushort(__float2bfloat16_rn(v));
    }
}

void launch_pack_tc(const float *w, int n_comp, void *img, cudaStream_t s, bool train) {
    pack_tc_kernel<<<148, 256, 0, s>>>(w, n_comp, static_cast<uint16_t *>(img), train ? 1 : 0);
}

// ------------------------------------------------------------------ kernel --
template <int N, int MODE>
__global__ void __launch_bounds__(threads_for(N), 1)
query_tc_kernel(const uint8_t *__restrict__ img, QueryArgs a) {
    constexpr int NP = packed_width(N);
    constexpr int kPairs = pairs_for(N), S = slots_for(N), Q = kPairs * S;
    constexpr uint32_t IMG = img_bytes(N);
    constexpr uint32_t A_OFF = align1k(IMG);
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr uint32_t E_OFF = A_OFF + kPairs * kABytes;    // encoded tiles E_l, one per NASG lane
    constexpr uint32_t IN_OFF = E_OFF + Q * kEBytes;        // input staging: [NASG lane][2 buffers]
    uint64_t *acc_full = reinterpret_cast<uint64_t *>(smem + IN_OFF + 2 * Q * kInBytes);  // [pair]
    uint64_t *raw_full = acc_full + kPairs;  // [NASG lane] from here on
    uint64_t *raw_empty = raw_full + Q;
    uint64_t *in_full = raw_empty + Q;  // [lane][buffer]
    uint64_t *e_full = in_full + 2 * Q;
    uint64_t *e_empty = e_full + Q;
    uint64_t *w_bar = e_empty + Q;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(w_bar + 1);
    __shared__ int s_clamped;

    pdl_trigger();
    pdl_wait();  // the queue (n_dev) and its rows come from the previous kernel on the stream
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = warp >> 2;        // warpgroup: named barrier g + 1
    // warpgroups [0, P): MLP of pair g; then the NASG warpgroups, lane (pair m, slot j)
    // warpgroups [P, P + Q): NASG lanes 0..Q-1 (part 0); streamed: [P + Q, P + 2Q) their part 1
    const int lnq = g < kPairs ? 0 : (g - kPairs) % Q;
    const int pt = g < kPairs ? 0 : (g - kPairs) / Q;  // which half of the lobes (streamed)
    const int m = g < kPairs ? g : lnq / S;
    const int j = g < kPairs ? 0 : lnq % S;
    const int wq = warp & 3;        // TMEM lane quarter of this warp
    const int t = threadIdx.x & 127;
    const int64_t nrows = a.n_dev ? min((int64_t)*a.n_dev, a.n) : a.n;  // a wavefront queue sets n_dev
    const int64_t ntiles = (nrows + 127) / 128;
    const int64_t stride = (int64_t)gridDim.x * kPairs;
    // a short device-sized queue (n_dev, the render loop's late bounces) leaves most
    // CTAs without a tile: they leave before allocating TMEM and loading weights
    if ((int64_t)blockIdx.x * kPairs >= ntiles) return;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kPairs; ++i) tc::mbar_init(&acc_full[i], 1);
        for (int i = 0; i < Q; ++i) {
            tc::mbar_init(&raw_full[i], 1);
            tc::mbar_init(&raw_empty[i], 4 * nasg_wgs(N));  // one arrival per NASG warp
            tc::mbar_init(&in_full[2 * i], 1);
            tc::mbar_init(&in_full[2 * i + 1], 1);
            tc::mbar_init(&e_full[i], 1);
            tc::mbar_init(&e_empty[i], 1);
        }
        tc::mbar_init(w_bar, 1);
        s_clamped = 0;
        tc::fence_mbar_init();
    }
    if (warp == 0) tc::tmem_alloc(tmem_slot, kTmemCols);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    NASG_CHECK(tc::dynamic_smem_bytes() >= smem_bytes<N>(), "query kernel: dynamic shared memory");
    NASG_CHECK((tmem & 0xFFFFu) == 0u, "query kernel: TMEM allocation starts at column 0");
    if (threadIdx.x == 0) {  // weights: TMA bulk copies global -> smem, once per CTA
        tc::mbar_arrive_expect_tx(w_bar, IMG);
        for (uint32_t off = 0; off < IMG; off += 16384)
            tc::bulk_g2s(smem + off, img + off, (IMG - off) < 16384u ? (IMG - off) : 16384u, w_bar);
    }

    if (g < kPairs) {
        // ============================ MLP warpgroup ============================
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(regs_mlp(N)));
        const uint32_t my_acc = tmem + m * 128 + ((uint32_t)(wq * 32) << 16);
        const uint32_t a_base = tc::smem_u32(smem + A_OFF + m * kABytes);
        const uint32_t e_base0 = tc::smem_u32(smem + E_OFF + m * S * kEBytes);  // + slot * kEBytes
        const uint32_t a_row128 = a_base + (t >> 3) * 2048 + (t & 7) * 16;  // K = 128 layout
        const uint32_t sW = tc::smem_u32(smem);
        uint32_t acc_ph = 0;
        // The A operand is complete in smem (and our TMEM reads are done): warp 0
        // issues layer L with one elected lane.  Layer 0 reads E of the NASG lane
        // that owns tile k (once it has filled it), layers 1-2 accumulate into the
        // group's TMEM columns, the output layer into that lane's raw buffer once
        // it is empty.  Tile k of the pair goes to slot k % S.
        auto issue = [&](int L, int64_t k) {
            const int lk = m * S + (int)(k % S);
            const int64_t ks = k / S;  // use count of that lane's buffers
            if (L > 0) {
                tc::fence_proxy_async_smem();
                tc::tc_fence_before();
                wg_sync(g);
            }
            if (wq == 0) {
                __syncwarp();
                if (L == 0) tc::mbar_wait(&e_full[lk], (uint32_t)(ks & 1));
                if (L == 3 && ks > 0) tc::mbar_wait(&raw_empty[lk], (uint32_t)((ks - 1) & 1));
                tc::tc_fence_after();
                auto chain = [&](auto lc) {
                    constexpr int LL = decltype(lc)::value;
                    constexpr int K = LL == 0 ? kIn : kHidden;
                    constexpr int NO = LL == 3 ? NP : kHidden;  // output columns
                    constexpr int N0 = NO > 256 ? 256 : NO;     // first MMA's columns (UMMA N <= 256)
                    constexpr uint32_t idesc = tc::idesc_f16(128, N0);
                    // descriptors rebuilt at issue time from opaque copies of the base
                    // addresses: hoisted out of the tile loop they would occupy ~60
                    // registers and spill
                    const uint32_t abase = tc::opaque(LL == 0 ? e_base0 + (uint32_t)(k % S) * kEBytes : a_base);
                    const uint32_t bbase = tc::opaque(sW) + w_off(LL);
                    const uint64_t ad = tc::smem_desc(abase, 128, K * 16);
                    const uint64_t bd = tc::smem_desc(bbase, 128, K * 16);
                    const uint32_t d = tmem + (LL == 3 ? raw_col(N, lk) : (uint32_t)m * 128u);
                    // +256 B per K=16 slab = +16 in the address field
                    tc::mma_f16_chain_elect<K / 16, 16, 16, (N != 4)>(d, ad, bd, idesc);
                    if constexpr (NO > 256) {  // packed columns [256, NP): image rows 256.. (32 row groups on)
                        constexpr uint32_t idesc1 = tc::idesc_f16(128, NO - 256);
                        const uint64_t bd1 = tc::smem_desc(bbase + 32u * (uint32_t)(K * 16), 128, K * 16);
                        tc::mma_f16_chain_elect<K / 16>(d + 256u, ad, bd1, idesc1);
                    }
                    tc::mma_commit_elect(LL == 3 ? &raw_full[lk] : &acc_full[m]);
                };
                switch (L) {
                    case 0: chain(std::integral_constant<int, 0>{}); break;
                    case 1: chain(std::integral_constant<int, 1>{}); break;
                    case 2: chain(std::integral_constant<int, 2>{}); break;
                    default: chain(std::integral_constant<int, 3>{}); break;
                }
            }
        };
        if (wq == 0) tc::mbar_wait(w_bar, 0);  // weights resident before the first MMA issue
        int64_t k = 0;
        for (int64_t tile = (int64_t)blockIdx.x * kPairs + m; tile < ntiles; tile += stride, ++k) {
            NASG_TRACE_AT(0, k, 0)
            issue(0, k);
            NASG_TRACE_AT(0, k, 1)
#pragma unroll 1
            for (int l = 1; l < 4; ++l) {  // hidden layers: TMEM -> ReLU -> f16 -> next A operand
                // (layer 1's wait also covers the previous tile's output layer,
                //  which still read the A tile: commits track all earlier MMAs)
                wg_wait_acc(&acc_full[m], acc_ph, g, wq);
                NASG_TRACE_AT(0, k, 2 * l)
                if (l == 1 && t == 0) tc::mbar_arrive(&e_empty[m * S + (int)(k % S)]);  // layer 0 has consumed E
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    float v[32];
                    tc::tmem_ld32(my_acc + q4 * 32, v);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint32_t p[4];
#pragma unroll
                        for (int h = 0; h < 4; ++h)
                            p[h] = tc::pack_f16x2_relu_sat(v[8 * c + 2 * h], v[8 * c + 2 * h + 1]);
                        tc::st_shared_v4(a_row128 + (q4 * 4 + c) * 128, p[0], p[1], p[2], p[3]);
                    }
                }
                issue(l, k);
                NASG_TRACE_AT(0, k, 2 * l + 1)
            }
        }
    } else {
        // ============================ NASG warpgroup ===========================
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(regs_nasg(N)));
        const int ln = m * S + j;  // this warpgroup's NASG lane: its E, input stage and raw buffer
        NASG_CHECK(ln < Q && raw_col(N, ln) + (uint32_t)NP + (streamed(N) ? 18u : 0u) <= kTmemCols &&
                       (kPairs == 1 || raw_col(N, ln) >= (uint32_t)kPairs * 128u),
                   "query kernel: NASG lane's raw / exchange columns inside TMEM, clear of the accumulators");
        const uint32_t my_raw = tmem + raw_col(N, ln) + ((uint32_t)(wq * 32) << 16);
        const uint32_t e_row64 = tc::smem_u32(smem + E_OFF + ln * kEBytes) + (t >> 3) * 1024 + (t & 7) * 16;
        const int64_t lstride = stride * S;  // this lane's tiles: every S-th tile of the pair
        const float(&inv_ext)[3] = a.bounds.inv_ext;
        int clamped = 0;
        // Inputs arrive two tiles ahead by TMA bulk copies into a double-buffered
        // smem stage; kt = index of the tile within this pair's sequence.
        const bool tma_in = a.packed ? ((reinterpret_cast<uintptr_t>(a.packed) & 15) == 0) : true;
        auto load_tile = [&](int64_t tl, int buf) {  // thread 0 only
            if (tl >= ntiles) return;
            const int64_t q0 = tl * 128, rows = min((int64_t)128, nrows - q0);
            uint64_t *bar = &in_full[2 * ln + buf];
            uint8_t *dst = smem + IN_OFF + (2 * ln + buf) * kInBytes;
            if (!tma_in) {
                tc::mbar_arrive_expect_tx(bar, 0);
            } else if (a.packed) {
                const uint32_t bytes = (uint32_t)(rows * 52) & ~15u;
                tc::mbar_arrive_expect_tx(bar, bytes);
                if (bytes) tc::bulk_g2s(dst, a.packed + q0 * 13, bytes, bar);
            } else {
                const uint32_t bytes = (uint32_t)rows * 16u;
                tc::mbar_arrive_expect_tx(bar, 3 * bytes);
                tc::bulk_g2s(dst, a.x + q0, bytes, bar);
                tc::bulk_g2s(dst + 2048, a.wo + q0, bytes, bar);
                tc::bulk_g2s(dst + 4096, a.nrm + q0, bytes, bar);
            }
        };
        // encode tile tl (this lane's kt-th) into its E and hand it to the MLP group
        auto encode = [&](int64_t tl, int64_t kt) {
            const int buf = (int)(kt & 1);
            tc::mbar_wait(&in_full[2 * ln + buf], (uint32_t)((kt >> 1) & 1));
            const int64_t q = tl * 128 + t;
            const bool valid = q < nrows;
            float4 x = make_float4(0.f, 0.f, 0.f, 0.f), wo = x, nrm = x;
            const uint8_t *src = smem + IN_OFF + (2 * ln + buf) * kInBytes;
            if (valid) {
                if (!tma_in) {
                    load_query(a, q, x, wo, nrm);
                } else if (a.packed) {
                    const int64_t rows = min((int64_t)128, nrows - tl * 128);
                    if ((uint32_t)(t * 52 + 52) <= ((uint32_t)(rows * 52) & ~15u)) {
                        const float *p = reinterpret_cast<const float *>(src + t * 52);
                        x = make_float4(p[0], p[1], p[2], 0.f);
                        wo = make_float4(p[3], p[4], p[5], 0.f);
                        nrm = make_float4(p[6], p[7], p[8], 0.f);
                    } else {
                        load_query(a, q, x, wo, nrm);  // tail rows past the 16-byte-rounded copy
                    }
                } else {
                    x = *reinterpret_cast<const float4 *>(src + t * 16);
                    wo = *reinterpret_cast<const float4 *>(src + 2048 + t * 16);
                    nrm = *reinterpret_cast<const float4 *>(src + 4096 + t * 16);
                }
            }
            uint32_t pk[32];
            clamped += encode_row_pack_f16(valid, x, wo, nrm, a.bounds, inv_ext, pk);
            store_row_pack(pk, e_row64);
            tc::fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core
            wg_sync(g);
            if (t == 0) {
                tc::mbar_arrive(&e_full[ln]);
                load_tile(tl + 2 * lstride, buf);  // every row of this buffer has been read
            }
        };
        int64_t tile = (int64_t)blockIdx.x * kPairs + m + (int64_t)j * stride;
        if (t == 0 && pt == 0) {
            load_tile(tile, 0);
            load_tile(tile + lstride, 1);
        }
        if (tile < ntiles && pt == 0) encode(tile, 0);
        uint32_t e_ph = 0;
        for (int64_t k = 0; tile < ntiles; tile += lstride, ++k) {
            // the next tile's encoding first: the MLP needs it right after this
            // tile's output layer, the raw outputs arrive only then
            NASG_TRACE_AT(1, k, 0)
            if (tile + lstride < ntiles && pt == 0) {
                wg_wait_acc(&e_empty[ln], e_ph, g, wq);
                NASG_TRACE_AT(1, k, 1)
                encode(tile + lstride, k + 1);
            }
            NASG_TRACE_AT(1, k, 2)
            const int64_t q = tile * 128 + t;
            const bool valid = q < nrows;
            float4 xi = make_float4(0.f, 0.f, 0.f, 0.f), dir = xi, dnee = xi;
            float bsdf = 0.f;
            if (valid) {  // issued before the wait: the loads land while the MLP finishes
                if constexpr (MODE == kModeSample || MODE == kModeShade) xi = load_xi(a, q);
                if constexpr (MODE == kModeShade) {
                    dir = a.sh_bsdf[q];
                    dnee = a.sh_nee[q];
                }
                if constexpr (MODE == kModePdf) {
                    dir = a.dir[q];
                    bsdf = a.bsdf_pdf ? a.bsdf_pdf[q] : 0.f;
                }
            }
            uint32_t ph = (uint32_t)(k & 1);
            wg_wait_acc(&raw_full[ln], ph, g, wq);
            NASG_TRACE_AT(1, k, 3)
            if constexpr (streamed(N)) {
                // every lane runs the tensor-memory loads (warp-collective), valid row or not
                constexpr int HD = packed_header(N);
                float hdr[HD];
                {
                    float v[16];
#pragma unroll
                    for (int c0 = 0; c0 < HD; c0 += 16) {
                        tc::tmem_ld16(my_raw + c0, v);
                        tc::tmem_ld_wait();
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) hdr[c0 + jj] = v[jj];
                    }
                }
                auto hraw = [&](int jj) { return hdr[jj]; };
                auto lobe7 = [&](int i, float (&r)[7]) {
                    float r8[8];
                    __syncwarp();
                    tc::tmem_ld8_sync(my_raw + HD + 8 * i, r8);
#pragma unroll
                    for (int kk = 0; kk < 7; ++kk) r[kk] = r8[kk];
                };
                // the lane's two warpgroups exchange through tensor memory behind the
                // raw columns: [0, 8) part 0's picked logits, [8, 16) part 1's, [16, 18) sums
                struct Xchg {
                    uint32_t base;
                    int pt, bar;
                    __device__ __forceinline__ void sync() const {
                        tc::tmem_st_wait();
                        tc::tc_fence_before();
                        asm volatile("bar.sync %0, 256;" ::"r"(bar) : "memory");
                        tc::tc_fence_after();
                    }
                    __device__ __forceinline__ void picked(float (&rs)[7], bool own) const {
                        const float v8[8] = {rs[0], rs[1], rs[2], rs[3], rs[4], rs[5], rs[6], 0.f};
                        tc::tmem_st8(base + 8u * (uint32_t)pt, v8);
                        sync();
                        float o[8];
                        tc::tmem_ld8_sync(base + 8u * (uint32_t)(1 - pt), o);
#pragma unroll
                        for (int k = 0; k < 7; ++k) rs[k] = own ? rs[k] : o[k];
                    }
                    __device__ __forceinline__ void to0(float &a, float &b) const {
                        if (pt == 1) tc::tmem_st2(base + 16u, a, b);
                        sync();
                        if (pt == 0) {
                            float x, y;
                            tc::tmem_ld2_sync(base + 16u, x, y);
                            a += x;
                            b += y;
                        }
                    }
                };
                Xchg xc{my_raw + (uint32_t)NP, pt, 9 + ln};
                const bool out = valid && pt == 0;
                if constexpr (MODE == kModeSample) {
                    float c;
                    const float4 o = guide_sample_pair<N>(hraw, lobe7, xi, c, pt, xc);
                    if (out) {
                        a.dir_pdf[q] = o;
                        if (a.c) a.c[q] = c;
                    }
                } else if constexpr (MODE == kModePdf) {
                    const float2 p = guide_pdf_pair<N>(hraw, lobe7, make_float3(dir.x, dir.y, dir.z), a.b, bsdf, pt, xc);
                    if (out) {
                        if (a.mix_pdf) a.mix_pdf[q] = p.x;
                        if (a.guided_pdf) a.guided_pdf[q] = p.y;
                    }
                } else if constexpr (MODE == kModeShade) {
                    float4 o0, o1;
                    guide_shade_pair<N>(hraw, lobe7, xi, a.b, dir, dnee, o0, o1, pt, xc);
                    if (out) {
                        a.sh_out[2 * q] = o0;
                        a.sh_out[2 * q + 1] = o1;
                    }
                } else {  // raw outputs in the reference order (packed_col), lobes split by halves
                    constexpr int D = 8 * N + 1;
                    float *dst = a.raw + q * D;
                    if (out) {
#pragma unroll
                        for (int i = 0; i <= N; ++i) dst[i < N ? 7 * N + i : 8 * N] = hdr[i];
                    }
#pragma unroll 1
                    for (int i = pt * (N / 2); i < pt * (N / 2) + N / 2; ++i) {
                        float r[7];
                        lobe7(i, r);
                        if (valid) {
#pragma unroll
                            for (int kk = 0; kk < 5; ++kk) dst[5 * i + kk] = r[kk];
                            dst[5 * N + 2 * i] = r[5];
                            dst[5 * N + 2 * i + 1] = r[6];
                        }
                    }
                }
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&raw_empty[ln]);  // buffer free for the next output layer
                NASG_TRACE_AT(1, k, 4)
                continue;
            }
            float raw[NP];
            {
                float v[32];
#pragma unroll
                for (int i = 0; i < NP / 32; ++i) {
                    tc::tmem_ld32(my_raw + i * 32, v);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) raw[i * 32 + j] = v[j];
                }
                if constexpr (NP % 32 != 0) {
                    float u[16];
                    tc::tmem_ld16(my_raw + (NP / 32) * 32, u);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 16; ++j) raw[(NP / 32) * 32 + j] = u[j];
                }
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&raw_empty[ln]);  // buffer free for the next output layer
            if (valid) {
                auto rawf = [&](int j) { return raw[j]; };
                if constexpr (MODE == kModeSample) {
                    float c;
                    a.dir_pdf[q] = guide_sample<N>(rawf, xi, c);
                    if (a.c) a.c[q] = c;
                } else if constexpr (MODE == kModePdf) {
                    const float2 p = guide_pdf<N>(rawf, make_float3(dir.x, dir.y, dir.z), a.b, bsdf);
                    if (a.mix_pdf) a.mix_pdf[q] = p.x;
                    if (a.guided_pdf) a.guided_pdf[q] = p.y;
                } else if constexpr (MODE == kModeShade) {
                    float4 o0, o1;
                    guide_shade<N>(rawf, xi, a.b, dir, dnee, o0, o1);
                    a.sh_out[2 * q] = o0;
                    a.sh_out[2 * q + 1] = o1;
                } else {
                    constexpr int D = 8 * N + 1;
#pragma unroll
                    for (int j = 0; j < D; ++j) a.raw[q * D + j] = raw[packed_col(j, N)];
                }
            }
            NASG_TRACE_AT(1, k, 4)
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
static int query_tc_n(QueryMode mode, const void *img, const QueryArgs &a, int num_sms, cudaStream_t s, bool pdl) {
    constexpr int kPairs = pairs_for(N);
    const int64_t ntiles = (a.n + 127) / 128;
    const int64_t supers = (ntiles + kPairs - 1) / kPairs;
    const int grid = (int)(supers < num_sms ? supers : num_sms);
    if (grid == 0) return 0;
    constexpr size_t sm = smem_bytes<N>();
    const uint8_t *im = static_cast<const uint8_t *>(img);
    switch (mode) {
#define NASG_LAUNCH_TC(M)                                                                  \
    case M: {                                                                              \
        auto k = query_tc_kernel<N, M>;                                                    \
        static const bool regs_ok = [&] {  /* the setmaxnreg split assumes this allocation */ \
            cudaFuncAttributes fa;                                                         \
            return cudaFuncGetAttributes(&fa, k) == cudaSuccess &&                         \
                   (streamed(N) || fa.numRegs == launch_regs(N));                          \
        }();                                                                               \
        if (!regs_ok) return -2;                                                           \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);     \
        launch_pdl(pdl, k, dim3(grid), dim3(threads_for(N)), sm, s, im, a);                 \
        break;                                                                             \
    }
        NASG_LAUNCH_TC(kModeSample)
        NASG_LAUNCH_TC(kModePdf)
        NASG_LAUNCH_TC(kModeRaw)
        NASG_LAUNCH_TC(kModeShade)
#undef NASG_LAUNCH_TC
    }
    return 1;
}

int query_tc(int n_comp, QueryMode mode, const void *img, const QueryArgs &a, int num_sms, cudaStream_t s, bool pdl) {
    switch (n_comp) {
        case 4: return query_tc_n<4>(mode, img, a, num_sms, s, pdl);
        case 8: return query_tc_n<8>(mode, img, a, num_sms, s, pdl);
        case 16: return query_tc_n<16>(mode, img, a, num_sms, s, pdl);
        case 32: return query_tc_n<32>(mode, img, a, num_sms, s, pdl);
        default: return -1;
    }
}

}  // namespace nasg
