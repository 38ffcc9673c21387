// Thin inline-PTX wrappers for the sm_100a primitives the tensor-core query
// kernel uses: mbarriers, TMA bulk copy, tcgen05 (alloc / mma / commit / ld /
// fences) and UMMA shared-memory + instruction descriptors.
#pragma once

#include <cstdint>
#ifdef NASG_CHECKED
#include <cstdio>
#endif
#include <cuda_runtime.h>

namespace nasg {
namespace tc {

// a value the compiler cannot see through (keeps derived values from being hoisted)
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
    asm volatile("mov.b32 %0, %0;" : "+r"(x));
    return x;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier ----------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// Blocking wait on a phase.  The suspend-time hint lets the hardware park the
// warp until the phase completes instead of re-polling, so waiting warps do
// not steal issue slots from the epilogue warps that share the SM.
#ifdef NASG_CHECKED
// Checked builds (EXTRA=-DNASG_CHECKED, profiles/r2_checked_build.txt): the
// kernels' protocol invariants — shared-memory and tensor-memory ranges, tile and
// list indices, and every mbarrier wait bounded to ~4 s — trap with a message
// instead of corrupting memory or hanging.  Compiled out of the library.
#define NASG_CHECK(cond, what)                                                                              \
    do {                                                                                                     \
        if (!(cond)) {                                                                                       \
            printf("NASG_CHECK failed: %s [%s:%d] block %d thread %d\n", what, __FILE__, __LINE__, blockIdx.x, \
                   threadIdx.x);                                                                             \
            __trap();                                                                                        \
        }                                                                                                    \
    } while (0)
#else
#define NASG_CHECK(cond, what) \
    do {                       \
    } while (0)
#endif

__device__ __forceinline__ uint32_t dynamic_smem_bytes() {
    uint32_t r;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
#ifdef NASG_CHECKED
    for (int it = 0;; ++it) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity), "r"(1000000)
            : "memory");
        if (ok) break;
        if (it > 4000) {
            printf("NASG_CHECK failed: mbarrier wait (smem 0x%x parity %u) block %d thread %d\n", a, parity,
                   blockIdx.x, threadIdx.x);
            __trap();
        }
    }
#else
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(a),
        "r"(parity), "r"(0x989680)
        : "memory");
#endif
}

// ---- TMA bulk copy global -> shared (1D), completes on an mbarrier ------------
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// generic-proxy smem writes -> visible to the async proxy (tensor core)
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- tcgen05 -----------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem], kind::f16 (bf16 in, fp32 accumulate), M = 128.
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// arrive on an mbarrier when all previously issued tcgen05.mma of this thread complete
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// Warp-collective forms: the whole (converged) warp calls them and one elected
// lane issues, so descriptors stay warp-uniform (no per-lane issue loop).
__device__ __forceinline__ void mma_bf16_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// NK MMAs of one K-chain in one elected issue block instead of an elect and
// register moves per MMA.  Slab kk uses adesc + kk*AINC and bdesc + kk*BINC
// (descriptor address units of 16 B); the first MMA accumulates into D when
// acc != 0, the others always.  BRANCH: the elected lane branches into an
// unpredicated block, so ptxas keeps the chain in uniform registers
// (back-to-back UTCHMMA: the query kernel 4.9 k -> 3.8 k static instructions);
// otherwise every MMA is predicated on the elect (4.4 k), which measured faster
// for the N = 4 query only (profiles/r2_query_knobs.txt).
#define NASG_MMA_STEP_B "add.s64 a, a, %5;\n\tadd.s64 b, b, %6;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, pt;\n\t"
#define NASG_MMA_STEP_P "add.s64 a, a, %5;\n\tadd.s64 b, b, %6;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, pt;\n\t"
#define NASG_MMA_HEAD_B                                             \
    "{\n\t.reg .pred e, pf, pt;\n\t.reg .b64 a, b;\n\t"               \
    "elect.sync _|e, 0xffffffff;\n\t@!e bra MMA_SKIP_%=;\n\t"          \
    "setp.ne.b32 pf, %4, 0;\n\tsetp.eq.u32 pt, 0, 0;\n\t"              \
    "mov.b64 a, %1;\n\tmov.b64 b, %2;\n\t"                             \
    "tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, pf;\n\t"
#define NASG_MMA_HEAD_P                                             \
    "{\n\t.reg .pred e, pf, pt;\n\t.reg .b64 a, b;\n\t"               \
    "elect.sync _|e, 0xffffffff;\n\t"                                  \
    "setp.ne.b32 pf, %4, 0;\n\tsetp.eq.u32 pt, 0, 0;\n\t"              \
    "mov.b64 a, %1;\n\tmov.b64 b, %2;\n\t"                             \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, pf;\n\t"
#define NASG_MMA_TAIL_B "MMA_SKIP_%=:\n\t}"
#define NASG_MMA_TAIL_P "}"
#define NASG_MMA_ARGS ::"r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc), "n"(AINC), "n"(BINC)
#define NASG_MMA_CHAIN(H, S, T)                                                                              \
    if constexpr (NK == 3) asm volatile(H S S T NASG_MMA_ARGS);                                             \
    else if constexpr (NK == 4) asm volatile(H S S S T NASG_MMA_ARGS);                                      \
    else if constexpr (NK == 5) asm volatile(H S S S S T NASG_MMA_ARGS);                                    \
    else if constexpr (NK == 8) asm volatile(H S S S S S S S T NASG_MMA_ARGS);                              \
    else if constexpr (NK == 10) asm volatile(H S S S S S S S S S T NASG_MMA_ARGS);                         \
    else asm volatile(H S S S S S S S S S S S S S S S S S S T NASG_MMA_ARGS);
template <int NK, int AINC = 16, int BINC = 16, bool BRANCH = true>
__device__ __forceinline__ void mma_f16_chain_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                    uint32_t acc = 0) {
    static_assert(NK == 3 || NK == 4 || NK == 5 || NK == 8 || NK == 10 || NK == 19, "K / 16 slabs");
    if constexpr (BRANCH) {
        NASG_MMA_CHAIN(NASG_MMA_HEAD_B, NASG_MMA_STEP_B, NASG_MMA_TAIL_B)
    } else {
        NASG_MMA_CHAIN(NASG_MMA_HEAD_P, NASG_MMA_STEP_P, NASG_MMA_TAIL_P)
    }
}
#undef NASG_MMA_CHAIN
#undef NASG_MMA_ARGS
#undef NASG_MMA_TAIL_P
#undef NASG_MMA_TAIL_B
#undef NASG_MMA_HEAD_P
#undef NASG_MMA_HEAD_B
#undef NASG_MMA_STEP_P
#undef NASG_MMA_STEP_B
__device__ __forceinline__ void mma_commit_elect(uint64_t *bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 8 consecutive 32-bit columns, completed by the wait inside (the
// registers are tied to the wait so no use can be scheduled before it)
__device__ __forceinline__ void tmem_ld8_sync(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7])
                 :
                 : "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// stores: 32 lanes x 8 (or 2) consecutive 32-bit columns from this thread's
// registers into its lane; tmem_st_wait() completes them before a fence + barrier
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
                 "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                 "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                 "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
                 : "memory");
}
__device__ __forceinline__ void tmem_st2(uint32_t taddr, float a, float b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(taddr), "r"(__float_as_uint(a)),
                 "r"(__float_as_uint(b))
                 : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld2_sync(uint32_t taddr, float &a, float &b) {
    uint32_t r0, r1;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r0), "+r"(r1) : : "memory");
    a = __uint_as_float(r0);
    b = __uint_as_float(r1);
}

// 32 lanes x 16 consecutive 32-bit columns: thread i gets lane (base + i), cols [c, c+16)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// ---- UMMA descriptors (K-major, no swizzle: 8-row x 16-byte core matrices) ----
// start address, LBO = byte distance between the two 16-byte K chunks of a
// K=16 slab, SBO = byte distance between 8-row groups; version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
    // base_offset = 0, lbo_mode = 0, layout_type (bits 61-63) = 0: SWIZZLE_NONE
    return d;
}

// Instruction descriptor for kind::f16: A = B = bf16, D = f32.  a_mn / b_mn
// select MN-major operands (bits 15 / 16); default K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn = false, bool b_mn = false) {
    return (1u << 4)                      // D format f32
           | (1u << 7)                    // A format bf16
           | (1u << 10)                   // B format bf16
           | ((a_mn ? 1u : 0u) << 15)     // A major
           | ((b_mn ? 1u : 0u) << 16)     // B major
           | ((uint32_t)(N >> 3) << 17)   // N / 8
           | ((uint32_t)(M >> 4) << 24);  // M / 16
}

// kind::f16 with A = B = f16 (format code 0), D = f32: the bf16 trainer's
// forward and its backward through W3, W2 (k_train_tc.cu)
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, bool a_mn = false, bool b_mn = false) {
    return (1u << 4) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

// f16x2 conversions saturating to +-65504 (never inf); the relu form fuses max(x, 0)
__device__ __forceinline__ uint32_t pack_f16x2_sat(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ uint32_t pack_f16x2_relu_sat(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.relu.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// 2^x on the MUFU (flush-to-zero: no denormal range fix-up around it)
__device__ __forceinline__ float ex2_approx(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// max(x, 0) of both values fused into the bf16 conversion (one F2FP.RELU).
__device__ __forceinline__ uint32_t pack_bf16x2_relu(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

}  // namespace tc
}  // namespace nasg
