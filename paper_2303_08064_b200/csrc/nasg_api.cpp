// Host side of the B200-native NASG guiding path: context, snapshots,
// training loop, checkpoint I/O, NCCL, synthetic workloads — all behind the
// C ABI in include/nasg/nasg.h.  Mirrors the reference's C++ guiding API
// (guiding.hpp, net.hpp, sphdist.hpp) with batched, stream-ordered calls.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "nasg/nasg.h"
#include "nasg_internal.h"

using namespace nasg;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CUDA_TRY(x)                                                                        \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) return fail(NASG_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define CHECK_LAUNCH()                                                                     \
    do {                                                                                   \
        cudaError_t e_ = cudaGetLastError();                                               \
        if (e_ != cudaSuccess) return fail(NASG_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
    } while (0)

// splitmix64 / hash_combine / PCG32 (math.hpp:74-121) — the specified RNG of
// the reference's weight init, epoch shuffle and our synthetic inputs.
uint64_t hash_mix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
uint64_t hash_combine(uint64_t a, uint64_t b) { return hash_mix(a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2))); }

struct Pcg32 {
    uint64_t state = 0, inc = 0;
    Pcg32(uint64_t initstate, uint64_t initseq) {
        inc = (initseq << 1u) | 1u;
        next();
        state += initstate;
        next();
    }
    uint32_t next() {
        uint64_t old = state;
        state = old * 6364136223846793005ull + inc;
        uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
        uint32_t rot = (uint32_t)(old >> 59u);
        return (xs >> rot) | (xs << ((~rot + 1u) & 31));
    }
    double next_double() { return next() * 0x1p-32; }
    uint32_t next_below(uint32_t n) { return (uint32_t)(((uint64_t)next() * n) >> 32); }
    float next_f24() { return (float)(next() >> 8) * 0x1p-24f; }
};

// init_network<float> (net.hpp:43-57), bit-exact; `hidden` is kHiddenUnits
// (128 in the reference; 64 fills the same PCG32 stream over the smaller
// matrices, the paper's Table 4 network).
void init_network(uint64_t seed, int n_comp, int hidden, float *w) {
    const int dims[5] = {kIn, hidden, hidden, hidden, 8 * n_comp + 1};
    Pcg32 rng(hash_mix(seed), 0xda3e39cb94b95bdbull);
    for (int l = 0; l < 4; ++l) {
        const double limit = std::sqrt(6.0 / dims[l]);
        for (int r = 0; r < dims[l]; ++r)
            for (int c = 0; c < dims[l + 1]; ++c) *w++ = (float)((rng.next_double() * 2.0 - 1.0) * limit);
    }
}

// ---- NCCL, loaded lazily (the query path never needs it) ----------------------
struct Nccl {
    void *h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    ncclResult_t (*commCount)(const ncclComm_t, int *) = nullptr;
    ncclResult_t (*commCuDevice)(const ncclComm_t, int *) = nullptr;
    const char *(*errStr)(ncclResult_t) = nullptr;
    bool load() {
        if (h) return true;
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return false;
        getUniqueId = (decltype(getUniqueId))dlsym(h, "ncclGetUniqueId");
        commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
        allReduce = (decltype(allReduce))dlsym(h, "ncclAllReduce");
        commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
        allGather = (decltype(allGather))dlsym(h, "ncclAllGather");
        errStr = (decltype(errStr))dlsym(h, "ncclGetErrorString");
        groupStart = (decltype(groupStart))dlsym(h, "ncclGroupStart");
        groupEnd = (decltype(groupEnd))dlsym(h, "ncclGroupEnd");
        commCount = (decltype(commCount))dlsym(h, "ncclCommCount");
        commCuDevice = (decltype(commCuDevice))dlsym(h, "ncclCommCuDevice");
        return getUniqueId && commInitRank && allReduce && allGather && commDestroy && groupStart && groupEnd &&
               commCount && commCuDevice;
    }
};
Nccl g_nccl;
std::mutex g_nccl_mu;

// Canonical weight count of a network with `hidden` units per hidden layer.
size_t n_weights_hu(int n_comp, int hidden) {
    return (size_t)kIn * hidden + 2u * hidden * hidden + (size_t)hidden * (8 * n_comp + 1);
}

// A hidden-64 network lives in the 128-wide device layout with the extra
// units' rows and columns zero.  Their gradients are exactly zero (their
// activations are ReLU(0) = 0 and their outgoing weights are 0), so Adam keeps
// them at zero and every kernel computes the 64-unit network unchanged.
// embed: canonical hidden-H layout -> 128-wide layout; extract: the inverse.
void hu_embed(int n_comp, int hidden, const float *e, float *w) {
    const int D = 8 * n_comp + 1;
    const int rows[4] = {kIn, hidden, hidden, hidden}, cols[4] = {hidden, hidden, hidden, D};
    const int wrows[4] = {kIn, kHidden, kHidden, kHidden}, wcols[4] = {kHidden, kHidden, kHidden, D};
    std::fill(w, w + n_weights(n_comp), 0.f);
    for (int l = 0; l < 4; ++l) {
        for (int r = 0; r < rows[l]; ++r)
            std::copy(e + (size_t)r * cols[l], e + (size_t)r * cols[l] + cols[l], w + (size_t)r * wcols[l]);
        e += (size_t)rows[l] * cols[l];
        w += (size_t)wrows[l] * wcols[l];
    }
}
void hu_extract(int n_comp, int hidden, const float *w, float *e) {
    const int D = 8 * n_comp + 1;
    const int rows[4] = {kIn, hidden, hidden, hidden}, cols[4] = {hidden, hidden, hidden, D};
    const int wrows[4] = {kIn, kHidden, kHidden, kHidden}, wcols[4] = {kHidden, kHidden, kHidden, D};
    for (int l = 0; l < 4; ++l) {
        for (int r = 0; r < rows[l]; ++r)
            std::copy(w + (size_t)r * wcols[l], w + (size_t)r * wcols[l] + cols[l], e + (size_t)r * cols[l]);
        e += (size_t)rows[l] * cols[l];
        w += (size_t)wrows[l] * wcols[l];
    }
}

}  // namespace

struct nasg_ctx {
    nasg_config cfg{};
    int device = 0, N = 8, D = 65, nw = 0, num_sms = 148;
    int hu = kHidden, nw_ext = 0;  // hidden units; canonical (caller-facing) weight count
    Bounds bounds{};
    float bmax[3]{};
    cudaStream_t stream = nullptr;
    cudaStream_t lanes[3] = {nullptr, nullptr, nullptr};
    // live parameters + Adam (Trainer::params_, adam_ guiding.hpp:162-163)
    float *w = nullptr, *m = nullptr, *v = nullptr, *grad = nullptr;
    float *wp = nullptr, *wtp = nullptr;  // packed live (training forward/backward)
    // published snapshot (NetworkSnapshot net.hpp:161)
    // two snapshot slots (shared_ptr<const> snapshots, net.hpp:161): a publish
    // fills the slot no reader can still be using, then makes it current
    struct PubSlot {
        float *w = nullptr, *wp = nullptr;
        void *tc = nullptr;
        cudaEvent_t ev = nullptr;  // recorded on `stream` when the slot's snapshot is complete
        std::vector<std::pair<cudaStream_t, cudaEvent_t>> readers;  // last query per foreign stream
    } pub[2];
    int cur = 0;
    // the current slot's images (aliases of pub[cur])
    float *w_pub = nullptr, *wp_pub = nullptr;
    void *tc_pub = nullptr;
    int precision = NASG_MLP_FP32;        // query path MLP arithmetic
    int train_precision = NASG_MLP_FP32;  // training path MLP arithmetic
    void *tc_live = nullptr;              // trainer image of the live weights (bf16 training: f16 layers + bf16 W4)
    TcTrainBufs tcb{};
    unsigned long long *d_clamp = nullptr;
    // Adam / step state on device
    int64_t *d_adam_t = nullptr;
    int *d_nonfinite = nullptr;
    int *d_wbig = nullptr;  // some live weight >= kSafeWeight or not finite (disables zero-row skipping)
    unsigned int *d_ticket = nullptr;  // last-block ticket of the fused Adam kernel
    cudaEvent_t xev = nullptr;  // reusable: orders the context stream after a caller stream
    double *h_acc = nullptr;    // pinned: TrainStats read-back (a D2H copy engine, never behind an upload)
    double *d_step_stats = nullptr, *d_acc = nullptr;
    TrainScratch sc{};
    uint32_t *d_order = nullptr, *h_order[2] = {nullptr, nullptr};
    cudaEvent_t order_ev[2] = {nullptr, nullptr};  // recorded after each h_order[i] upload
    int order_slot = 0;
    // first-epoch shuffle computed ahead on a host thread (ctx_prefetch_shuffle)
    struct Prefetch {
        std::thread th;
        bool active = false;
        int64_t n = 0;
        uint64_t iteration = 0;
        int slot = 0;
        uint64_t rng_state = 0, rng_inc = 0;  // the shuffle stream after the first epoch
    } pf;
    size_t order_cap = 0;
    int64_t iterations = 0;
    // host pipeline buffers (nasg_query_sample_host)
    float *lane_in[3] = {nullptr, nullptr, nullptr}, *lane_out[3] = {nullptr, nullptr, nullptr};
    int64_t lane_cap = 0;
    // NCCL
    ncclComm_t comm = nullptr;
    bool comm_owned = true;
    // per-iteration buffer-size exchange (allocated with the communicator)
    int64_t *d_nall = nullptr, *h_nall = nullptr;
    cudaEvent_t nall_ev = nullptr;
    bool pdl = true;  // programmatic dependent launch of the training chain
    bool query_pdl = false;  // ... and of the query kernels (serial render loop)  // false: attached by the caller (nasg_attach_nccl), not destroyed here
    int rank = 0, nranks = 1;
    uint64_t launches = 0;
    uint64_t collectives = 0;  // NCCL launches (grouped exchange per step, allgather per iteration)
    cudaEvent_t pub_ev = nullptr;  // = pub[cur].ev
};

namespace nasg {
int64_t ctx_sample_capacity(const nasg_ctx *c) { return c ? (int64_t)c->cfg.sample_capacity : 0; }
int ctx_nranks(const nasg_ctx *c) { return c ? c->nranks : 1; }
int ctx_device(const nasg_ctx *c) { return c ? c->device : 0; }
}  // namespace nasg

namespace {

int ensure_scratch(nasg_ctx *c, int64_t count) {
    const int64_t rows = ((count + 63) / 64) * 64;
    if (rows <= c->sc.max_rows) return NASG_OK;
    TrainScratch &s = c->sc;
    float **bufs[8] = {&s.h0, &s.h1, &s.h2, &s.h3, &s.d1, &s.d2, &s.d3, &s.d4};
    const int widths[8] = {64, 128, 128, 128, 128, 128, 128, d4_stride(c->N)};
    for (int i = 0; i < 8; ++i) {
        if (*bufs[i]) cudaFree(*bufs[i]);
        *bufs[i] = nullptr;
        CUDA_TRY(cudaMalloc(bufs[i], (size_t)(rows * widths[i] + 128) * sizeof(float)));
    }
    const int tiles = (int)(rows / 64);
    if (s.tile_loss) cudaFree(s.tile_loss);
    if (s.tile_loss_count) cudaFree(s.tile_loss_count);
    if (s.tile_dropped) cudaFree(s.tile_dropped);
    CUDA_TRY(cudaMalloc(&s.tile_loss, tiles * sizeof(double)));
    CUDA_TRY(cudaMalloc(&s.tile_loss_count, tiles * sizeof(int)));
    CUDA_TRY(cudaMalloc(&s.tile_dropped, tiles * sizeof(int)));
    if (!s.dw_partial) {
        s.splits = 128;
        CUDA_TRY(cudaMalloc(&s.dw_partial, (size_t)s.splits * c->nw * sizeof(float)));
    }
    s.max_rows = rows;
    s.max_tiles = tiles;
    return NASG_OK;
}

void join_prefetch(nasg_ctx *c);

int ensure_order(nasg_ctx *c, size_t n) {
    if (n <= c->order_cap) return NASG_OK;
    join_prefetch(c);  // a prefetch writes into the old buffers
    c->pf.active = false;
    CUDA_TRY(cudaDeviceSynchronize());  // uploads from the old buffers are done
    if (c->d_order) cudaFree(c->d_order);
    CUDA_TRY(cudaMalloc(&c->d_order, n * sizeof(uint32_t)));
    for (int i = 0; i < 2; ++i) {
        if (c->h_order[i]) cudaFreeHost(c->h_order[i]);
        c->h_order[i] = nullptr;
        CUDA_TRY(cudaMallocHost(&c->h_order[i], n * sizeof(uint32_t)));
        if (!c->order_ev[i]) CUDA_TRY(cudaEventCreateWithFlags(&c->order_ev[i], cudaEventDisableTiming));
    }
    c->order_cap = n;
    return NASG_OK;
}

void join_prefetch(nasg_ctx *c) {
    if (c->pf.th.joinable()) c->pf.th.join();
}

// The shuffle stream of train_iteration (guiding.cpp:216-225): rank r uses
// stream 5 + 2r of Pcg32(hash_combine(seed, 0x7261696e) + iteration).
Pcg32 shuffle_rng(const nasg_ctx *c, uint64_t iteration) {
    return Pcg32(hash_combine(c->cfg.seed, 0x7261696e) + iteration, 5 + 2 * (uint64_t)c->rank);
}

// Fisher-Yates of the identity (the first epoch of an iteration, :219-225).
void first_epoch_shuffle(uint32_t *ord, int64_t n, Pcg32 &rng) {
    for (int64_t i = 0; i < n; ++i) ord[i] = (uint32_t)i;
    for (int64_t i = n; i > 1; --i) {
        uint32_t j = rng.next_below((uint32_t)i);
        std::swap(ord[i - 1], ord[j]);
    }
}

int do_publish(nasg_ctx *c) {
    auto &P = c->pub[c->cur ^ 1];
    // queries still reading that older snapshot on other streams finish first; the
    // list then starts over (a destroyed event stays valid for waits already queued)
    for (auto &rd : P.readers) CUDA_TRY(cudaStreamWaitEvent(c->stream, rd.second, 0));
    for (auto &rd : P.readers) cudaEventDestroy(rd.second);
    P.readers.clear();
    if (!P.tc || c->tc_live) {
        // the live packed images are current with c->w (every Adam step and every
        // host weight change re-packs them), and the query image is the first
        // img_bytes of the trainer's: the snapshot is three copies in one launch
        const void *src[3] = {c->w, c->wp, P.tc ? c->tc_live : nullptr};
        void *dst[3] = {P.w, P.wp, P.tc};
        const size_t bytes[3] = {c->nw * sizeof(float), packed_f32_floats(c->N) * sizeof(float),
                                 P.tc ? tc_image_bytes(c->N) : 0};
        launch_copy3(src, dst, bytes, c->stream);
        c->launches++;
    } else {  // N = 32: a query image without a trainer image
        CUDA_TRY(cudaMemcpyAsync(P.w, c->w, c->nw * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
        launch_pack_fp32(P.w, c->N, P.wp, nullptr, c->stream);
        launch_pack_tc(P.w, c->N, P.tc, c->stream);
        c->launches += 2;
    }
    CHECK_LAUNCH();
    CUDA_TRY(cudaEventRecord(P.ev, c->stream));
    c->cur ^= 1;
    c->w_pub = P.w;
    c->wp_pub = P.wp;
    c->tc_pub = P.tc;
    c->pub_ev = P.ev;
    return NASG_OK;
}

// A query on stream s read the current snapshot: remember it so the publish
// that next overwrites this slot waits for it.
int note_reader(nasg_ctx *c, cudaStream_t s) {
    if (s == c->stream) return NASG_OK;  // stream order already covers it
    auto &rd = c->pub[c->cur].readers;
    cudaEvent_t ev = nullptr;
    for (auto &x : rd)
        if (x.first == s) ev = x.second;
    if (!ev) {
        CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        rd.emplace_back(s, ev);
    }
    CUDA_TRY(cudaEventRecord(ev, s));
    return NASG_OK;
}

int repack_live(nasg_ctx *c) {
    CUDA_TRY(cudaMemsetAsync(c->d_wbig, 0, sizeof(int), c->stream));
    launch_pack_fp32(c->w, c->N, c->wp, c->wtp, c->stream, c->d_wbig);
    c->launches++;
    if (c->tc_live) {
        launch_pack_tc(c->w, c->N, c->tc_live, c->stream, true);
        c->launches++;
    }
    CHECK_LAUNCH();
    return NASG_OK;
}

int ensure_tc_scratch(nasg_ctx *c, int64_t count) {
    const int64_t blocks = (count + 127) / 128;
    TcTrainBufs &t = c->tcb;
    if (blocks <= t.max_blocks) return NASG_OK;
    uint8_t **bufs[8] = {&t.h0, &t.h1, &t.h2, &t.h3, &t.d1, &t.d2, &t.d3, &t.d4};
    const int feats[8] = {64, 128, 128, 128, 128, 128, 128, packed_width(c->N)};
    for (int i = 0; i < 8; ++i) {
        if (*bufs[i]) cudaFree(*bufs[i]);
        *bufs[i] = nullptr;
        CUDA_TRY(cudaMalloc(bufs[i], (size_t)blocks * feats[i] * 256));
    }
    if (t.tile_loss) cudaFree(t.tile_loss);
    if (t.tile_lc) cudaFree(t.tile_lc);
    if (t.tile_dr) cudaFree(t.tile_dr);
    CUDA_TRY(cudaMalloc(&t.tile_loss, blocks * sizeof(double)));
    CUDA_TRY(cudaMalloc(&t.tile_lc, blocks * sizeof(int)));
    CUDA_TRY(cudaMalloc(&t.tile_dr, blocks * sizeof(int)));
    if (!t.partial) {
        // 4 layers x 37 splits = one wave of 148 CTAs (one per SM: 131 KB of
        // smem each); 74 splits (two waves) measured 5 us slower per 2^18 step
        // (profiles/r2_dw_splits.txt)
        t.splits = 37;
        const int ps = packed_width(c->N) > 128 ? packed_width(c->N) : 128;  // partial_stride (k_train_tc.cu)
        CUDA_TRY(cudaMalloc(&t.partial, (size_t)4 * 2 * 37 * 128 * ps * sizeof(float)));
    }
    t.step_stats = c->d_step_stats;
    t.max_blocks = blocks;
    return NASG_OK;
}

// The zero-row classification's buffers (train_classify, both trainers): the
// step's row list (u32 per row), one look-back word per 1024 rows, {live, zero}.
int ensure_classify(nasg_ctx *c, int64_t count) {
    TcTrainBufs &t = c->tcb;
    const int64_t rows = ((count + 1023) / 1024) * 1024;
    if (!t.cls) CUDA_TRY(cudaMalloc(&t.cls, 4 * sizeof(int64_t)));
    t.wbig = c->d_wbig;
    if (rows <= t.live_cap) return NASG_OK;
    if (t.live) cudaFree(t.live);
    if (t.scan_state) cudaFree(t.scan_state);
    t.live = nullptr;
    t.scan_state = nullptr;
    t.scan_cap = rows / 1024;
    CUDA_TRY(cudaMalloc(&t.live, 2 * (size_t)rows * sizeof(uint32_t)));
    CUDA_TRY(cudaMalloc(&t.scan_state, (size_t)t.scan_cap * sizeof(unsigned long long)));
    CUDA_TRY(cudaMemset(t.scan_state, 0, (size_t)t.scan_cap * sizeof(unsigned long long)));
    t.scan_epoch = 0;
    t.live_cap = rows;
    return NASG_OK;
}

cudaStream_t pick(nasg_ctx *c, void *s) { return s ? (cudaStream_t)s : c->stream; }

QueryArgs base_args(nasg_ctx *c, int64_t n) {
    QueryArgs a{};
    a.n = n;
    a.bounds = c->bounds;
    a.clamp_count = c->d_clamp;
    return a;
}

int run_query(nasg_ctx *c, QueryMode mode, const QueryArgs &a, cudaStream_t s) {
    static const char *const kNames[] = {"nasg_query_sample", "nasg_query_pdf", "nasg_query_raw", "nasg_query_shade"};
    NvtxRange nv_(kNames[(int)mode & 3]);
    if (a.n == 0) return NASG_OK;
    if (s != c->stream) CUDA_TRY(cudaStreamWaitEvent(s, c->pub_ev, 0));  // read a complete snapshot
    int r;
    if (c->precision == NASG_MLP_BF16) {
        if (!c->tc_pub) return fail(NASG_ERR_UNSUPPORTED, "bf16 tensor-core path not available for this N");
        r = query_tc(c->N, mode, c->tc_pub, a, c->num_sms, s, c->query_pdl);
    } else {
        r = query_fp32(c->N, mode, c->wp_pub, a, c->num_sms, s);
    }
    if (r == -2) return fail(NASG_ERR_CUDA, "query kernel register allocation differs from its setmaxnreg split");
    if (r < 0) return fail(NASG_ERR_UNSUPPORTED, "n_components not compiled for this path");
    c->launches += r;
    CHECK_LAUNCH();
    return note_reader(c, s);
}

// One minibatch step (guiding.cpp:236-276) on rows samples[order[0..count)].
// count_clamps: the reference encodes every buffer row once per train_iteration
// (guiding.cpp:209-214), so encode clamps are counted on a row's first-epoch visit only.
int train_step_impl(nasg_ctx *c, const nasg_train_sample *samples, const uint32_t *order, int64_t count,
                    int64_t global_count, double b, cudaStream_t s, bool count_clamps = true) {
    NvtxRange nv_("nasg_train_step");
    unsigned long long *clamp = count_clamps ? c->d_clamp : nullptr;
    if (count <= 0 && c->nranks == 1) return NASG_OK;
    const bool tc = c->train_precision == NASG_MLP_BF16;
    int r = tc ? ensure_tc_scratch(c, std::max<int64_t>(count, 1)) : ensure_scratch(c, std::max<int64_t>(count, 1));
    if (!r) r = ensure_classify(c, std::max<int64_t>(count, 1));
    if (r) return r;
    if (count > 0 && tc) {
        const int k = train_tc_step(c->N, c->tc_live, samples, order, count, global_count, b, c->cfg.loss_blend,
                                    c->bounds, c->tcb, c->num_sms, clamp, c->grad, c->d_nonfinite, s, c->pdl);
        if (k < 0) return fail(NASG_ERR_UNSUPPORTED, "n_components not compiled for bf16 training");
        c->launches += k;
    } else if (count > 0) {
        // zero-gradient rows out of the network pass, as on the tensor-core path,
        // when the step has more 64-row tiles than SMs
        const int64_t *live_count = nullptr;
        const uint32_t *rows = order;
        if (c->tcb.skip_zero && (count + 63) / 64 > c->num_sms) {
            c->launches += train_classify(samples, order, count, c->tcb, c->bounds, clamp, s, false);
            live_count = c->tcb.cur_cls();
            rows = c->tcb.cur_live();
        }
        if (train_forward_backward(c->N, c->wp, c->wtp, samples, rows, count, live_count, global_count, b,
                                   c->cfg.loss_blend, c->bounds, c->sc, c->num_sms, clamp, s) < 0)
            return fail(NASG_ERR_UNSUPPORTED, "n_components not compiled for training");
        const int ndw = train_dw(c->N, count, c->sc, c->grad, s, live_count);
        train_reduce(c->N, c->sc, c->grad, c->d_nonfinite, s);
        train_step_stats(c->sc, count, c->d_step_stats, s, live_count);
        c->launches += 3 + ndw;  // forward/backward, dW GEMMs, reduction, statistics
    } else {
        CUDA_TRY(cudaMemsetAsync(c->grad, 0, c->nw * sizeof(float), s));
        CUDA_TRY(cudaMemsetAsync(c->d_step_stats, 0, 3 * sizeof(double), s));
    }
    CHECK_LAUNCH();
    if (c->comm) {
        // data-parallel exchange (any attached communicator, 1 rank included): the
        // sum of the ranks' unnormalised-by-rank gradients and step statistics, as
        // ONE grouped NCCL launch per Adam step
        ncclResult_t e0 = g_nccl.groupStart();
        ncclResult_t e1 = g_nccl.allReduce(c->grad, c->grad, c->nw, ncclFloat32, ncclSum, c->comm, s);
        ncclResult_t e2 = g_nccl.allReduce(c->d_step_stats, c->d_step_stats, 3, ncclFloat64, ncclSum, c->comm, s);
        ncclResult_t e3 = g_nccl.groupEnd();
        if (e0 != ncclSuccess || e1 != ncclSuccess || e2 != ncclSuccess || e3 != ncclSuccess)
            return fail(NASG_ERR_NCCL, "grouped ncclAllReduce failed");
        c->collectives++;
    }
    // skip decision (re-taken on the reduced gradient when one was exchanged), t,
    // Adam, re-pack of every live image (the bf16 operands of the next step
    // included) and the statistics, in one launch
    train_adam(c->N, c->w, c->m, c->v, c->grad, c->cfg.learning_rate, c->wp, c->wtp, c->tc_live, c->d_nonfinite,
               c->d_adam_t, c->d_step_stats, c->d_acc, c->d_ticket, s, c->pdl, c->comm != nullptr, c->d_wbig);
    c->launches += 1;
    CHECK_LAUNCH();
    return NASG_OK;
}

bool is_pinned(const void *p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}


// ---- explicit mixtures and the NASG-vs-vMF fit (k_sphdist.cu) ---------------
int check_current_device() {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    cudaDeviceProp prop{};
    CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10 || prop.minor != 0)
        return fail(NASG_ERR_CUDA, "this build targets sm_100a (B200); device is sm_" +
                                       std::to_string(prop.major * 10 + prop.minor));
    return NASG_OK;
}

int dist_call(int op, int kind, int64_t n, int k, const float *comp, const float *w, const float *in, float *out,
              void *stream) {
    if (kind != NASG_DIST_NASG && kind != NASG_DIST_VMF) return fail(NASG_ERR_INVALID, "unknown distribution kind");
    if (n < 0 || k <= 0) return fail(NASG_ERR_INVALID, "n must be >= 0 and k > 0");
    if (n > 0 && (!comp || !w || !in || !out)) return fail(NASG_ERR_INVALID, "null buffer");
    if (n == 0) return NASG_OK;
    int r = check_current_device();
    if (r) return r;
    dist_launch(op, kind, n, k, comp, w, in, out, (cudaStream_t)stream);
    CHECK_LAUNCH();
    return NASG_OK;
}

// RAII device buffer for the blocking fit calls
struct DevBuf {
    void *p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    int alloc(size_t bytes) {
        if (cudaMalloc(&p, bytes ? bytes : 16) != cudaSuccess) {
            cudaGetLastError();
            return fail(NASG_ERR_OOM, "cudaMalloc failed");
        }
        return NASG_OK;
    }
    template <class T>
    T *as() const { return static_cast<T *>(p); }
};

int fit_check_model(int model, int k) {
    if (model != NASG_DIST_NASG && model != NASG_DIST_VMF) return fail(NASG_ERR_INVALID, "unknown model kind");
    if (model == NASG_DIST_NASG && k != 1 && k != 2 && k != 4 && k != 8 && k != 16)
        return fail(NASG_ERR_UNSUPPORTED, "NASG fit: n_components must be 1, 2, 4, 8 or 16");
    if (model == NASG_DIST_VMF && (k < 1 || k > fit_max_components(NASG_DIST_VMF)))
        return fail(NASG_ERR_UNSUPPORTED, "vMF fit: n_components must be in [1, 32]");
    return NASG_OK;
}

int fit_upload_target(int tkind, int tk, const float *tcomp, const float *tw, DevBuf &dc, DevBuf &dw) {
    if (tkind != NASG_DIST_NASG && tkind != NASG_DIST_VMF) return fail(NASG_ERR_INVALID, "unknown target kind");
    if (tk < 1 || tk > fit_max_target_components()) return fail(NASG_ERR_INVALID, "target_k must be in [1, 32]");
    if (!tcomp || !tw) return fail(NASG_ERR_INVALID, "null target");
    const size_t cb = (size_t)tk * (tkind == NASG_DIST_NASG ? 12 : 4) * sizeof(float);
    int r = dc.alloc(cb);
    if (!r) r = dw.alloc(tk * sizeof(float));
    if (r) return r;
    CUDA_TRY(cudaMemcpy(dc.p, tcomp, cb, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(dw.p, tw, tk * sizeof(float), cudaMemcpyHostToDevice));
    return NASG_OK;
}

// KL of n_models device raw vectors against the target grid p (device, nz x 2nz)
int fit_kl_device(int model, int k, const float *d_raws, int n_models, int nz, const double *d_p, double *kl_out) {
    const int blocks = 148;
    DevBuf part;
    int r = part.alloc((size_t)blocks * n_models * sizeof(double));
    if (r) return r;
    fit_kl(model, k, d_raws, n_models, nz, d_p, part.as<double>(), blocks, 0);
    CHECK_LAUNCH();
    std::vector<double> h((size_t)blocks * n_models);
    CUDA_TRY(cudaMemcpy(h.data(), part.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost));
    for (int m = 0; m < n_models; ++m) {
        double s = 0.0;
        for (int b = 0; b < blocks; ++b) s += h[(size_t)m * blocks + b];
        kl_out[m] = s;
    }
    return NASG_OK;
}
}  // namespace

namespace nasg {
// Starts the next train_iteration's first-epoch shuffle for a buffer of n rows
// on a host thread (used by the render loop while the GPU traces); the
// iteration consumes it when its buffer has exactly n rows and computes the
// permutation itself otherwise.  Results are identical either way.
int ctx_prefetch_shuffle(nasg_ctx *c, int64_t n) {
    if (!c || n <= 1 || n > 0xffffffffll) return NASG_OK;
    join_prefetch(c);
    c->pf.active = false;
    int r = ensure_order(c, (size_t)n);
    if (r) return r;
    c->pf.n = n;
    c->pf.iteration = (uint64_t)c->iterations;
    c->pf.slot = c->order_slot ^ 1;
    c->pf.active = true;
    c->pf.th = std::thread([c, n]() {
        cudaSetDevice(c->device);
        cudaEventSynchronize(c->order_ev[c->pf.slot]);  // the slot's last upload has left
        Pcg32 rng = shuffle_rng(c, c->pf.iteration);
        first_epoch_shuffle(c->h_order[c->pf.slot], n, rng);
        c->pf.rng_state = rng.state;
        c->pf.rng_inc = rng.inc;
    });
    return NASG_OK;
}

void ctx_set_pdl(nasg_ctx *c, bool on) {
    if (c) c->pdl = on;
}

void ctx_set_query_pdl(nasg_ctx *c, bool on) {
    if (c) c->query_pdl = on;
}

int ctx_train_stats_async(nasg_ctx *c, double *acc, cudaStream_t s) {
    CUDA_TRY(cudaMemcpyAsync(acc, c->d_acc, 5 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemsetAsync(c->d_acc, 0, 5 * sizeof(double), s));
    return NASG_OK;
}

void ctx_stats_from_acc(const double *acc, nasg_train_stats *st) {  // TrainStats (guiding.cpp:278-281)
    st->steps = (int)acc[4];
    st->mean_loss = acc[1] > 0 ? acc[0] / acc[1] : 0.0;
    st->dropped_samples = (uint64_t)acc[2];
    st->skipped_updates = (uint64_t)acc[3];
}
}  // namespace nasg

extern "C" {

const char *nasg_status_string(int s) {
    switch (s) {
        case NASG_OK: return "ok";
        case NASG_ERR_INVALID: return "invalid argument";
        case NASG_ERR_CUDA: return "cuda error";
        case NASG_ERR_NCCL: return "nccl error";
        case NASG_ERR_IO: return "i/o error";
        case NASG_ERR_OOM: return "out of memory";
        case NASG_ERR_UNSUPPORTED: return "unsupported";
        default: return "unknown";
    }
}

const char *nasg_last_error(void) { return g_err.c_str(); }

int nasg_n_weights(int n_components) { return n_weights(n_components); }
int nasg_n_weights_hu(int n_components, int hidden_units) {
    return (int)n_weights_hu(n_components, hidden_units ? hidden_units : kHidden);
}

void nasg_config_default(nasg_config *c) {
    c->n_components = 8;
    c->sample_capacity = 1 << 16;
    c->batch_size = 1 << 12;
    c->step_factor = 1;
    c->learning_rate = 0.002f;
    c->loss_blend = 0.2;
    c->seed = 0;
    c->hidden_units = kHidden;
}

int nasg_create(const nasg_config *cfg, int device, const float bmin[3], const float bmax[3], nasg_ctx **out) {
    if (!cfg || !out || !bmin || !bmax) return fail(NASG_ERR_INVALID, "null argument");
    if (cfg->n_components != 4 && cfg->n_components != 8 && cfg->n_components != 16 && cfg->n_components != 32)
        return fail(NASG_ERR_UNSUPPORTED, "n_components must be 4, 8, 16 or 32 in this build");
    if (cfg->batch_size <= 0 || cfg->sample_capacity <= 0 || cfg->step_factor <= 0)
        return fail(NASG_ERR_INVALID, "batch_size, sample_capacity, step_factor must be > 0");
    if (cfg->hidden_units != 0 && cfg->hidden_units != 64 && cfg->hidden_units != kHidden)
        return fail(NASG_ERR_UNSUPPORTED, "hidden_units must be 64 or 128 in this build");
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(NASG_ERR_INVALID, "bad device ordinal");
    DeviceScope ds_(device);  // the caller's current device is restored on return
    cudaDeviceProp prop{};
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
        return fail(NASG_ERR_CUDA, "this build targets sm_100a (B200); device is sm_" +
                                       std::to_string(prop.major * 10 + prop.minor));
    nasg_ctx *c = new nasg_ctx();
    c->cfg = *cfg;
    c->device = device;
    c->N = cfg->n_components;
    c->D = 8 * c->N + 1;
    c->nw = n_weights(c->N);
    c->hu = cfg->hidden_units ? cfg->hidden_units : kHidden;
    c->cfg.hidden_units = c->hu;
    c->nw_ext = (int)n_weights_hu(c->N, c->hu);
    c->num_sms = prop.multiProcessorCount;
    for (int k = 0; k < 3; ++k) {
        c->bounds.bmin[k] = bmin[k];
        c->bmax[k] = bmax[k];
        c->bounds.ext[k] = (double)bmax[k] - (double)bmin[k];
        c->bounds.inv_ext[k] = c->bounds.ext[k] > 0.0 ? (float)(1.0 / c->bounds.ext[k]) : 0.f;
    }
    auto cleanup_fail = [&](int code) {
        nasg_destroy(c);
        return code;
    };
#define ALLOC(p, bytes)                                                             \
    do {                                                                            \
        if (cudaMalloc(&(p), (bytes)) != cudaSuccess) {                            \
            cudaGetLastError();                                                     \
            fail(NASG_ERR_OOM, "cudaMalloc failed");                                \
            return cleanup_fail(NASG_ERR_OOM);                                      \
        }                                                                           \
    } while (0)
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
        return cleanup_fail(fail(NASG_ERR_CUDA, "stream create failed"));
    if (cudaEventCreateWithFlags(&c->xev, cudaEventDisableTiming) != cudaSuccess)
        return cleanup_fail(fail(NASG_ERR_CUDA, "event create failed"));
    if (cudaMallocHost(&c->h_acc, 5 * sizeof(double)) != cudaSuccess)
        return cleanup_fail(fail(NASG_ERR_OOM, "cudaMallocHost failed"));
    for (auto &l : c->lanes)
        if (cudaStreamCreateWithFlags(&l, cudaStreamNonBlocking) != cudaSuccess)
            return cleanup_fail(fail(NASG_ERR_CUDA, "stream create failed"));
    const size_t wb = c->nw * sizeof(float);
    ALLOC(c->w, wb); ALLOC(c->m, wb); ALLOC(c->v, wb); ALLOC(c->grad, wb);
    for (auto &P : c->pub) {
        ALLOC(P.w, wb);
        ALLOC(P.wp, packed_f32_floats(c->N) * sizeof(float));
        if (tc_supported(c->N)) ALLOC(P.tc, tc_image_bytes(c->N));
        if (cudaEventCreateWithFlags(&P.ev, cudaEventDisableTiming) != cudaSuccess)
            return cleanup_fail(fail(NASG_ERR_CUDA, "event create failed"));
    }
    ALLOC(c->wp, packed_f32_floats(c->N) * sizeof(float));
    ALLOC(c->wtp, packed_t32_floats(c->N) * sizeof(float));
    if (tc_train_supported(c->N)) ALLOC(c->tc_live, tc_train_image_bytes(c->N));
    ALLOC(c->d_clamp, sizeof(unsigned long long));
    ALLOC(c->d_adam_t, sizeof(int64_t));
    ALLOC(c->d_nonfinite, 2 * sizeof(int));
    ALLOC(c->d_wbig, sizeof(int));
    ALLOC(c->d_ticket, 2 * sizeof(unsigned int));
    ALLOC(c->d_step_stats, 3 * sizeof(double));
    ALLOC(c->d_acc, 5 * sizeof(double));
#undef ALLOC
    cudaMemsetAsync(c->m, 0, wb, c->stream);
    cudaMemsetAsync(c->v, 0, wb, c->stream);
    cudaMemsetAsync(c->d_clamp, 0, sizeof(unsigned long long), c->stream);
    cudaMemsetAsync(c->d_adam_t, 0, sizeof(int64_t), c->stream);
    cudaMemsetAsync(c->d_nonfinite, 0, 2 * sizeof(int), c->stream);
    cudaMemsetAsync(c->d_wbig, 0, sizeof(int), c->stream);
    cudaMemsetAsync(c->d_ticket, 0, 2 * sizeof(unsigned int), c->stream);
    cudaMemsetAsync(c->d_acc, 0, 5 * sizeof(double), c->stream);
    std::vector<float> w(c->nw);
    if (c->hu == kHidden) {
        init_network(cfg->seed, c->N, kHidden, w.data());
    } else {
        std::vector<float> e(c->nw_ext);
        init_network(cfg->seed, c->N, c->hu, e.data());
        hu_embed(c->N, c->hu, e.data(), w.data());
    }
    if (cudaMemcpyAsync(c->w, w.data(), wb, cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
        return cleanup_fail(fail(NASG_ERR_CUDA, "weight upload failed"));
    int r = repack_live(c);
    if (!r) r = do_publish(c);
    if (!r && cudaStreamSynchronize(c->stream) != cudaSuccess) r = fail(NASG_ERR_CUDA, "init sync failed");
    if (r) return cleanup_fail(r);
    *out = c;
    return NASG_OK;
}

int nasg_destroy(nasg_ctx *c) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c) return NASG_OK;
    join_prefetch(c);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->comm && c->comm_owned && g_nccl.commDestroy) g_nccl.commDestroy(c->comm);
    if (c->h_nall) cudaFreeHost(c->h_nall);
    if (c->nall_ev) cudaEventDestroy(c->nall_ev);
    void *bufs[] = {c->d_nall, c->tc_live, c->tcb.h0, c->tcb.h1, c->tcb.h2, c->tcb.h3, c->tcb.d1, c->tcb.d2, c->tcb.d3,
                    c->tcb.d4, c->tcb.tile_loss, c->tcb.tile_lc, c->tcb.tile_dr, c->tcb.partial,
                    c->tcb.live, c->tcb.cls, c->tcb.scan_state, c->d_wbig,
                    c->w, c->m, c->v, c->grad, c->wp, c->wtp, c->pub[0].w, c->pub[0].wp, c->pub[0].tc,
                    c->pub[1].w, c->pub[1].wp, c->pub[1].tc, c->d_clamp,
                    c->d_adam_t, c->d_ticket, c->d_nonfinite, c->d_step_stats, c->d_acc, c->d_order,
                    c->sc.h0, c->sc.h1, c->sc.h2, c->sc.h3, c->sc.d1, c->sc.d2, c->sc.d3, c->sc.d4,
                    c->sc.dw_partial, c->sc.tile_loss, c->sc.tile_loss_count, c->sc.tile_dropped,
                    c->lane_in[0], c->lane_in[1], c->lane_in[2], c->lane_out[0], c->lane_out[1], c->lane_out[2]};
    for (void *p : bufs)
        if (p) cudaFree(p);
    for (int i = 0; i < 2; ++i) {
        if (c->h_order[i]) cudaFreeHost(c->h_order[i]);
        if (c->order_ev[i]) cudaEventDestroy(c->order_ev[i]);
    }
    for (auto l : c->lanes)
        if (l) cudaStreamDestroy(l);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->xev) cudaEventDestroy(c->xev);
    if (c->h_acc) cudaFreeHost(c->h_acc);
    for (auto &P : c->pub) {
        if (P.ev) cudaEventDestroy(P.ev);
        for (auto &rd : P.readers) cudaEventDestroy(rd.second);
    }
    delete c;
    return NASG_OK;
}

// Device 128-wide parameter vector -> caller's canonical layout (host-synchronous).
static int copy_out_wide(nasg_ctx *c, const float *dev, float *host) {
    CUDA_TRY(cudaDeviceSynchronize());  // host-synchronous getter: order after all caller streams
    if (c->hu == kHidden) {
        CUDA_TRY(cudaMemcpyAsync(host, dev, c->nw * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        return NASG_OK;
    }
    std::vector<float> wide(c->nw);
    CUDA_TRY(cudaMemcpyAsync(wide.data(), dev, c->nw * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    hu_extract(c->N, c->hu, wide.data(), host);
    return NASG_OK;
}

// Caller's canonical layout -> device 128-wide parameter vector (synchronous).
static int copy_in_wide(nasg_ctx *c, const float *host, float *dev) {
    std::vector<float> wide;
    if (c->hu != kHidden) {
        wide.resize(c->nw);
        hu_embed(c->N, c->hu, host, wide.data());
        host = wide.data();
    }
    CUDA_TRY(cudaMemcpy(dev, host, c->nw * sizeof(float), cudaMemcpyHostToDevice));
    return NASG_OK;
}

int nasg_set_weights(nasg_ctx *c, const float *host_w, size_t n) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c || !host_w) return fail(NASG_ERR_INVALID, "null argument");
    if (n != (size_t)c->nw_ext) return fail(NASG_ERR_INVALID, "weight count mismatch");
    std::vector<float> wide;
    if (c->hu != kHidden) {
        wide.resize(c->nw);
        hu_embed(c->N, c->hu, host_w, wide.data());
        host_w = wide.data();
        n = wide.size();
    }
    CUDA_TRY(cudaDeviceSynchronize());  // training may be in flight on a caller stream
    CUDA_TRY(cudaMemcpyAsync(c->w, host_w, n * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    int r = repack_live(c);
    if (!r) r = do_publish(c);
    if (!r) CUDA_TRY(cudaStreamSynchronize(c->stream));
    return r;
}

int nasg_get_weights(nasg_ctx *c, float *host_w, size_t n, int published) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c || !host_w) return fail(NASG_ERR_INVALID, "null argument");
    if (n != (size_t)c->nw_ext) return fail(NASG_ERR_INVALID, "weight count mismatch");
    return copy_out_wide(c, published ? c->w_pub : c->w, host_w);
}

int nasg_publish(nasg_ctx *c) {
    DeviceScope ds_(c ? c->device : -1);
    NvtxRange nv_("nasg_publish");
    if (!c) return fail(NASG_ERR_INVALID, "null context");
    return do_publish(c);
}

int nasg_set_precision(nasg_ctx *c, int p) {
    if (!c) return fail(NASG_ERR_INVALID, "null context");
    if (p != NASG_MLP_FP32 && p != NASG_MLP_BF16) return fail(NASG_ERR_INVALID, "bad precision");
    if (p == NASG_MLP_BF16 && !c->tc_pub) return fail(NASG_ERR_UNSUPPORTED, "bf16 path unavailable");
    c->precision = p;
    return NASG_OK;
}

int nasg_get_precision(nasg_ctx *c) { return c ? c->precision : -1; }

int nasg_set_train_precision(nasg_ctx *c, int p) {
    if (!c) return fail(NASG_ERR_INVALID, "null context");
    if (p != NASG_MLP_FP32 && p != NASG_MLP_BF16) return fail(NASG_ERR_INVALID, "bad precision");
    if (p == NASG_MLP_BF16 && !c->tc_live) return fail(NASG_ERR_UNSUPPORTED, "bf16 training unavailable");
    c->train_precision = p;
    return NASG_OK;
}

int nasg_get_train_precision(nasg_ctx *c) { return c ? c->train_precision : -1; }

int nasg_set_zero_row_skip(nasg_ctx *c, int on) {
    if (!c) return fail(NASG_ERR_INVALID, "null context");
    c->tcb.skip_zero = on != 0;
    return NASG_OK;
}

int nasg_get_zero_row_skip(nasg_ctx *c) { return c ? (c->tcb.skip_zero ? 1 : 0) : -1; }

// NASGNET1 (net.cpp:31-82): magic, u32 N, u32 5, u32 dims[5], row-major f32 W1..W4.
// With NASG_CKPT_OPTIMIZER the Adam state follows as a trailing chunk
// ("NASGADM1", u64 t, u32 n, f32 m[n], f32 v[n]); the reference's loader reads
// the weights and ignores what follows them (net.cpp:54-82), so such a file
// still loads there.
int nasg_save_checkpoint(nasg_ctx *c, const char *path) { return nasg_save_checkpoint_ex(c, path, 0); }

int nasg_save_checkpoint_ex(nasg_ctx *c, const char *path, int flags) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c || !path) return fail(NASG_ERR_INVALID, "null argument");
    if (flags & ~NASG_CKPT_OPTIMIZER) return fail(NASG_ERR_INVALID, "unknown checkpoint flags");
    std::vector<float> w(c->nw_ext), m, v;
    int r = nasg_get_weights(c, w.data(), w.size(), 0);
    if (r) return r;
    int64_t t = 0;
    if (flags & NASG_CKPT_OPTIMIZER) {
        m.resize(c->nw_ext);
        v.resize(c->nw_ext);
        if ((r = copy_out_wide(c, c->m, m.data())) || (r = copy_out_wide(c, c->v, v.data()))) return r;
        CUDA_TRY(cudaMemcpy(&t, c->d_adam_t, sizeof(t), cudaMemcpyDeviceToHost));
    }
    FILE *f = std::fopen(path, "wb");
    if (!f) return fail(NASG_ERR_IO, std::string("cannot open checkpoint for writing: ") + path);
    auto u32 = [&](uint32_t v) {
        unsigned char b[4] = {(unsigned char)v, (unsigned char)(v >> 8), (unsigned char)(v >> 16), (unsigned char)(v >> 24)};
        std::fwrite(b, 1, 4, f);
    };
    std::fwrite("NASGNET1", 1, 8, f);
    u32((uint32_t)c->N);
    u32(5);
    const uint32_t dims[5] = {(uint32_t)kIn, (uint32_t)c->hu, (uint32_t)c->hu, (uint32_t)c->hu, (uint32_t)c->D};
    for (uint32_t d : dims) u32(d);
    bool ok = std::fwrite(w.data(), sizeof(float), w.size(), f) == w.size();
    if (flags & NASG_CKPT_OPTIMIZER) {
        ok &= std::fwrite("NASGADM1", 1, 8, f) == 8;
        for (int k = 0; k < 8; ++k) {
            const unsigned char b = (unsigned char)((uint64_t)t >> (8 * k));
            ok &= std::fwrite(&b, 1, 1, f) == 1;
        }
        u32((uint32_t)c->nw_ext);
        ok &= std::fwrite(m.data(), sizeof(float), m.size(), f) == m.size();
        ok &= std::fwrite(v.data(), sizeof(float), v.size(), f) == v.size();
    }
    ok &= std::fclose(f) == 0;
    return ok ? NASG_OK : fail(NASG_ERR_IO, std::string("short write on checkpoint: ") + path);
}

int nasg_load_checkpoint(nasg_ctx *c, const char *path) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c || !path) return fail(NASG_ERR_INVALID, "null argument");
    FILE *f = std::fopen(path, "rb");
    if (!f) return fail(NASG_ERR_IO, std::string("cannot open checkpoint: ") + path);
    char magic[8];
    bool ok = std::fread(magic, 1, 8, f) == 8 && std::memcmp(magic, "NASGNET1", 8) == 0;
    auto u32 = [&]() -> uint32_t {
        unsigned char b[4] = {0, 0, 0, 0};
        if (std::fread(b, 1, 4, f) != 4) ok = false;
        return (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
    };
    if (!ok) {
        std::fclose(f);
        return fail(NASG_ERR_IO, std::string("not a network checkpoint: ") + path);
    }
    const uint32_t n = u32(), nd = u32();
    if (!ok || nd != 5) {
        std::fclose(f);
        return fail(NASG_ERR_IO, std::string("unexpected layer count in checkpoint: ") + path);
    }
    uint32_t dims[5];
    for (auto &d : dims) d = u32();
    if ((int)n != c->N || dims[0] != (uint32_t)kIn || dims[1] != (uint32_t)c->hu || dims[2] != (uint32_t)c->hu ||
        dims[3] != (uint32_t)c->hu || dims[4] != (uint32_t)c->D) {
        std::fclose(f);
        return fail(NASG_ERR_INVALID, "checkpoint shape does not match this context");
    }
    std::vector<float> w(c->nw_ext);
    ok &= std::fread(w.data(), sizeof(float), w.size(), f) == w.size();
    if (!ok) {
        std::fclose(f);
        return fail(NASG_ERR_IO, std::string("truncated checkpoint: ") + path);
    }
    // optional Adam chunk (nasg_save_checkpoint_ex); anything else after the
    // weights is ignored, as the reference's loader does
    bool adam = false;
    uint64_t t = 0;
    std::vector<float> m, v;
    char tag[8];
    if (std::fread(tag, 1, 8, f) == 8 && std::memcmp(tag, "NASGADM1", 8) == 0) {
        unsigned char b[8];
        bool ok2 = std::fread(b, 1, 8, f) == 8;
        for (int k = 0; k < 8; ++k) t |= (uint64_t)b[k] << (8 * k);
        const uint32_t nw = u32();
        ok2 &= ok && nw == (uint32_t)c->nw_ext;
        if (ok2) {
            m.resize(nw);
            v.resize(nw);
            ok2 &= std::fread(m.data(), sizeof(float), nw, f) == nw && std::fread(v.data(), sizeof(float), nw, f) == nw;
        }
        if (!ok2) {
            std::fclose(f);
            return fail(NASG_ERR_IO, std::string("truncated or mismatched optimizer chunk in checkpoint: ") + path);
        }
        adam = true;
    }
    std::fclose(f);
    int r = nasg_set_weights(c, w.data(), w.size());
    if (r || !adam) return r;
    const int64_t ts = (int64_t)t;
    if ((r = copy_in_wide(c, m.data(), c->m)) || (r = copy_in_wide(c, v.data(), c->v))) return r;
    CUDA_TRY(cudaMemcpy(c->d_adam_t, &ts, sizeof(ts), cudaMemcpyHostToDevice));
    return NASG_OK;
}

// ---- queries --------------------------------------------------------------------
int nasg_query_sample(nasg_ctx *c, int64_t n, const float *x, const float *wo, const float *nrm, const float *xi,
                      float *dir_pdf, float *cc, void *stream) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c || n < 0 || (n > 0 && (!x || !wo || !nrm || !xi || !dir_pdf))) return fail(NASG_ERR_INVALID, "bad argument");
    QueryArgs a = base_args(c, n);
    a.x = (const float4 *)x; a.wo = (const float4 *)wo; a.nrm = (const float4 *)nrm; a.xi = (const float4 *)xi;
    a.dir_pdf = (float4 *)dir_pdf; a.c = cc;
    return run_query(c, kModeSample, a, pick(c, stream));
}

int nasg_query_sample_packed(nasg_ctx *c, int64_t n, const float *q13, float *dir_pdf, float *cc, void *stream) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c || n < 0 || (n > 0 && (!q13 || !dir_pdf))) return fail(NASG_ERR_INVALID, "bad argument");
    QueryArgs a = base_args(c, n);
    a.packed = q13;
    a.dir_pdf = (float4 *)dir_pdf;
    a.c = cc;
    return run_query(c, kModeSample, a, pick(c, stream));
}

// Packed host rows (52 B/query in, 16 + 4 B out): the PCIe-lean form of
// nasg_query_sample_host, same 3-lane H2D / kernel / D2H pipeline.
int nasg_query_sample_host_packed(nasg_ctx *c, int64_t n, const float *q13, float *dir_pdf, float *cc) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c || n < 0 || (n > 0 && (!q13 || !dir_pdf))) return fail(NASG_ERR_INVALID, "bad argument");
    if (n == 0) return NASG_OK;
    // 2^19-row chunks (27 MB in): 1.013e9 q/s from pinned rows on one B200,
    // vs 1.000e9 at 2^20 (longer pipeline drain) and 0.96e9 at 2^17 or 2^21
    const int64_t chunk = std::min<int64_t>(n, 1 << 19);
    if (chunk > c->lane_cap) {
        for (int k = 0; k < 3; ++k) {
            if (c->lane_in[k]) cudaFree(c->lane_in[k]);
            if (c->lane_out[k]) cudaFree(c->lane_out[k]);
            c->lane_in[k] = c->lane_out[k] = nullptr;
            CUDA_TRY(cudaMalloc(&c->lane_in[k], chunk * 16 * sizeof(float)));
            CUDA_TRY(cudaMalloc(&c->lane_out[k], chunk * 5 * sizeof(float)));
        }
        c->lane_cap = chunk;
    }
    cudaEvent_t ready;
    CUDA_TRY(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(ready, c->stream));
    for (auto l : c->lanes) CUDA_TRY(cudaStreamWaitEvent(l, ready, 0));
    cudaEventDestroy(ready);
    int64_t i = 0;
    for (int64_t off = 0; off < n; off += chunk, ++i) {
        const int64_t m = std::min(chunk, n - off);
        const int k = (int)(i % 3);
        cudaStream_t s = c->lanes[k];
        float *in = c->lane_in[k], *out = c->lane_out[k];
        CUDA_TRY(cudaMemcpyAsync(in, q13 + off * 13, (size_t)m * 13 * sizeof(float), cudaMemcpyHostToDevice, s));
        int r = nasg_query_sample_packed(c, m, in, out, cc ? out + chunk * 4 : nullptr, s);
        if (r) return r;
        CUDA_TRY(cudaMemcpyAsync(dir_pdf + off * 4, out, (size_t)m * 4 * sizeof(float), cudaMemcpyDeviceToHost, s));
        if (cc) CUDA_TRY(cudaMemcpyAsync(cc + off, out + chunk * 4, m * sizeof(float), cudaMemcpyDeviceToHost, s));
    }
    for (auto l : c->lanes) CUDA_TRY(cudaStreamSynchronize(l));
    return NASG_OK;
}

int nasg_query_pdf(nasg_ctx *c, int64_t n, const float *x, const float *wo, const float *nrm, const float *dir,
                   float b, const float *bsdf_pdf, float *mix_pdf, float *guided_pdf, void *stream) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c || n < 0 || (n > 0 && (!x || !wo || !nrm || !dir))) return fail(NASG_ERR_INVALID, "bad argument");
    QueryArgs a = base_args(c, n);
    a.x = (const float4 *)x; a.wo = (const float4 *)wo; a.nrm = (const float4 *)nrm; a.dir = (const float4 *)dir;
    a.b = b; a.bsdf_pdf = bsdf_pdf; a.mix_pdf = mix_pdf; a.guided_pdf = guided_pdf;
    return run_query(c, kModePdf, a, pick(c, stream));
}

int nasg_query_shade(nasg_ctx *c, int64_t n, const int *n_dev, const float *x, const float *wo, const float *nrm,
                     const float *xi, const float *d_bsdf, const float *d_nee, float b, float *out, void *stream) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c || n < 0 || (n > 0 && (!x || !wo || !nrm || !xi || !d_bsdf || !d_nee || !out)))
        return fail(NASG_ERR_INVALID, "bad argument");
    QueryArgs a = base_args(c, n);
    a.x = (const float4 *)x; a.wo = (const float4 *)wo; a.nrm = (const float4 *)nrm; a.xi = (const float4 *)xi;
    a.n_dev = n_dev; a.b = b;
    a.sh_bsdf = (const float4 *)d_bsdf; a.sh_nee = (const float4 *)d_nee; a.sh_out = (float4 *)out;
    return run_query(c, kModeShade, a, pick(c, stream));
}

int nasg_query_raw(nasg_ctx *c, int64_t n, const float *x, const float *wo, const float *nrm, float *raw,
                   void *stream) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c || n < 0 || (n > 0 && (!x || !wo || !nrm || !raw))) return fail(NASG_ERR_INVALID, "bad argument");
    QueryArgs a = base_args(c, n);
    a.x = (const float4 *)x; a.wo = (const float4 *)wo; a.nrm = (const float4 *)nrm; a.raw = raw;
    return run_query(c, kModeRaw, a, pick(c, stream));
}

int nasg_decode_sample_raw(nasg_ctx *c, int64_t n, const float *raw, const float *xi, float *dir_pdf, float *cc,
                           void *stream) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c || n < 0 || (n > 0 && (!raw || !xi || !dir_pdf))) return fail(NASG_ERR_INVALID, "bad argument");
    if (n == 0) return NASG_OK;
    if (decode_raw(c->N, true, c->precision == NASG_MLP_BF16, n, raw, (const float4 *)xi, nullptr, 0.f, nullptr, (float4 *)dir_pdf, cc, nullptr,
                   nullptr, pick(c, stream)) < 0)
        return fail(NASG_ERR_UNSUPPORTED, "n_components");
    c->launches++;
    CHECK_LAUNCH();
    return NASG_OK;
}

int nasg_decode_pdf_raw(nasg_ctx *c, int64_t n, const float *raw, const float *dir, float b, const float *bsdf_pdf,
                        float *mix_pdf, float *guided_pdf, void *stream) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c || n < 0 || (n > 0 && (!raw || !dir))) return fail(NASG_ERR_INVALID, "bad argument");
    if (n == 0) return NASG_OK;
    if (decode_raw(c->N, false, c->precision == NASG_MLP_BF16, n, raw, nullptr, (const float4 *)dir, b, bsdf_pdf, nullptr, nullptr, mix_pdf,
                   guided_pdf, pick(c, stream)) < 0)
        return fail(NASG_ERR_UNSUPPORTED, "n_components");
    c->launches++;
    CHECK_LAUNCH();
    return NASG_OK;
}

// Host-buffer query: 3 lanes (streams) x chunk; lane k: H2D(i) -> kernel(i) ->
// D2H(i), so copies in both directions overlap the kernels of other chunks.
int nasg_query_sample_host(nasg_ctx *c, int64_t n, const float *x, const float *wo, const float *nrm,
                           const float *xi, float *dir_pdf, float *cc) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c || n < 0 || (n > 0 && (!x || !wo || !nrm || !xi || !dir_pdf))) return fail(NASG_ERR_INVALID, "bad argument");
    if (n == 0) return NASG_OK;
    const int64_t chunk = std::min<int64_t>(n, 1 << 19);
    if (chunk > c->lane_cap) {
        for (int k = 0; k < 3; ++k) {
            if (c->lane_in[k]) cudaFree(c->lane_in[k]);
            if (c->lane_out[k]) cudaFree(c->lane_out[k]);
            c->lane_in[k] = c->lane_out[k] = nullptr;
            CUDA_TRY(cudaMalloc(&c->lane_in[k], chunk * 16 * sizeof(float)));
            CUDA_TRY(cudaMalloc(&c->lane_out[k], chunk * 5 * sizeof(float)));
        }
        c->lane_cap = chunk;
    }
    // the snapshot must be complete before any lane reads it
    cudaEvent_t ready;
    CUDA_TRY(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(ready, c->stream));
    for (auto l : c->lanes) CUDA_TRY(cudaStreamWaitEvent(l, ready, 0));
    cudaEventDestroy(ready);
    int64_t i = 0;
    for (int64_t off = 0; off < n; off += chunk, ++i) {
        const int64_t m = std::min(chunk, n - off);
        const int k = (int)(i % 3);
        cudaStream_t s = c->lanes[k];
        float *in = c->lane_in[k], *out = c->lane_out[k];
        const size_t vb = (size_t)m * 4 * sizeof(float);
        CUDA_TRY(cudaMemcpyAsync(in, x + off * 4, vb, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(in + chunk * 4, wo + off * 4, vb, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(in + chunk * 8, nrm + off * 4, vb, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(in + chunk * 12, xi + off * 4, vb, cudaMemcpyHostToDevice, s));
        int r = nasg_query_sample(c, m, in, in + chunk * 4, in + chunk * 8, in + chunk * 12, out,
                                  cc ? out + chunk * 4 : nullptr, s);
        if (r) return r;
        CUDA_TRY(cudaMemcpyAsync(dir_pdf + off * 4, out, vb, cudaMemcpyDeviceToHost, s));
        if (cc) CUDA_TRY(cudaMemcpyAsync(cc + off, out + chunk * 4, m * sizeof(float), cudaMemcpyDeviceToHost, s));
    }
    for (auto l : c->lanes) CUDA_TRY(cudaStreamSynchronize(l));
    return NASG_OK;
}

// ---- training -----------------------------------------------------------------------
int nasg_train_step(nasg_ctx *c, const nasg_train_sample *samples, const uint32_t *order, int64_t count,
                    int64_t global_count, double b, void *stream) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c || count < 0 || global_count <= 0 || (count > 0 && !samples)) return fail(NASG_ERR_INVALID, "bad argument");
    cudaStream_t s = pick(c, stream);
    int r = train_step_impl(c, samples, order, count, global_count, b, s);
    if (r) return r;
    if (s != c->stream) {  // nasg_train_stats_take reads the accumulators on the context stream
        CUDA_TRY(cudaEventRecord(c->xev, s));
        CUDA_TRY(cudaStreamWaitEvent(c->stream, c->xev, 0));
    }
    return NASG_OK;
}

int nasg_train_stats_take(nasg_ctx *c, nasg_train_stats *st) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c || !st) return fail(NASG_ERR_INVALID, "null argument");
    // the training steps that fed the accumulators are ordered before c->stream
    CUDA_TRY(cudaMemcpyAsync(c->h_acc, c->d_acc, 5 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaMemsetAsync(c->d_acc, 0, 5 * sizeof(double), c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    const double *acc = c->h_acc;
    ctx_stats_from_acc(acc, st);
    return NASG_OK;
}

// Data-parallel minibatch plan (see nasg.h).  Global batch t is split over the
// ranks in proportion to their buffer sizes; each rank walks its own shuffled
// buffer with the reference's cursor/epoch rule (guiding.cpp:236-243).
int nasg_dp_plan(const nasg_config *cfg, const int64_t *n_per_rank, int nranks, int rank, int max_steps,
                 int64_t *local_count, int64_t *global_count, int32_t *reshuffle_before) {
    if (!cfg || !n_per_rank || nranks < 1 || rank < 0 || rank >= nranks || cfg->batch_size <= 0 ||
        cfg->sample_capacity <= 0 || cfg->step_factor <= 0)
        return -1;
    const int64_t t = cfg->batch_size;
    const int steps = cfg->step_factor * (int)((cfg->sample_capacity + t - 1) / t);  // guiding.cpp:204-206
    if (steps > max_steps) return -1;
    int64_t total = 0;
    for (int k = 0; k < nranks; ++k) {
        if (n_per_rank[k] < 0) return -1;
        total += n_per_rank[k];
    }
    if (total == 0) return 0;  // empty global buffer: no-op (guiding.cpp:198-202)
    std::vector<int64_t> tr(nranks), cur(nranks, 0);
    int64_t assigned = 0;
    for (int k = 0; k < nranks; ++k) {
        tr[k] = (int64_t)(((unsigned __int128)t * (uint64_t)n_per_rank[k]) / (uint64_t)total);
        assigned += tr[k];
    }
    for (int k = 0; assigned < t && k < nranks; ++k)  // remainder to the first non-empty ranks
        if (n_per_rank[k] > 0) {
            ++tr[k];
            ++assigned;
        }
    for (int k = 0; k < nranks; ++k)
        if (n_per_rank[k] > 0 && tr[k] == 0) tr[k] = 1;
    for (int step = 0; step < steps; ++step) {
        int64_t g = 0;
        for (int k = 0; k < nranks; ++k) {
            int64_t cnt = 0;
            bool resh = step == 0;
            if (n_per_rank[k] > 0) {
                if (cur[k] >= n_per_rank[k]) {
                    cur[k] = 0;
                    resh = true;
                }
                cnt = std::min(tr[k], n_per_rank[k] - cur[k]);
                cur[k] += cnt;
            }
            g += cnt;
            if (k == rank) {
                local_count[step] = cnt;
                if (reshuffle_before) reshuffle_before[step] = (resh && n_per_rank[k] > 0) ? 1 : 0;
            }
        }
        global_count[step] = g;
    }
    return steps;
}

// Trainer::train_iteration (guiding.cpp:196-282).
int nasg_train_iteration(nasg_ctx *c, int64_t n, const nasg_train_sample *samples, double b,
                         nasg_train_stats *stats, void *stream) {
    DeviceScope ds_(c ? c->device : -1);
    NvtxRange nv_("nasg_train_iteration");
    if (!c || n < 0 || (n > 0 && !samples)) return fail(NASG_ERR_INVALID, "bad argument");
    cudaStream_t s = pick(c, stream);
    if (s != c->stream) {  // the context's own stream carries publish; order it after s
        CUDA_TRY(cudaEventRecord(c->xev, s));
        CUDA_TRY(cudaStreamWaitEvent(c->stream, c->xev, 0));
    }
    if (n == 0 && c->nranks == 1) {  // empty buffer: no-op + publish (:198-202)
        ++c->iterations;
        int r = do_publish(c);
        if (stats) *stats = nasg_train_stats{0, 0.0, 0, 0};
        return r;
    }
    if (n > 0xffffffffll) return fail(NASG_ERR_INVALID, "buffer too large");
    // Data-parallel plan: every rank learns every rank's buffer size, then walks
    // the same deterministic schedule (single rank: exactly guiding.cpp:204-276).
    std::vector<int64_t> n_all((size_t)c->nranks, 0);
    n_all[(size_t)c->rank] = n;
    if (c->comm) {  // buffers allocated with the communicator; one event wait, no device-wide sync
        c->h_nall[c->rank] = n;
        CUDA_TRY(cudaMemcpyAsync(c->d_nall + c->rank, c->h_nall + c->rank, sizeof(int64_t), cudaMemcpyHostToDevice, s));
        if (g_nccl.allGather(c->d_nall + c->rank, c->d_nall, 1, ncclInt64, c->comm, s) != ncclSuccess)
            return fail(NASG_ERR_NCCL, "ncclAllGather of buffer sizes failed");
        c->collectives++;
        CUDA_TRY(cudaMemcpyAsync(c->h_nall, c->d_nall, sizeof(int64_t) * c->nranks, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaEventRecord(c->nall_ev, s));
        CUDA_TRY(cudaEventSynchronize(c->nall_ev));
        std::copy(c->h_nall, c->h_nall + c->nranks, n_all.begin());
    }
    const int max_steps = c->cfg.step_factor * ((c->cfg.sample_capacity + c->cfg.batch_size - 1) / c->cfg.batch_size);
    std::vector<int64_t> local(max_steps), global(max_steps);
    std::vector<int32_t> resh(max_steps);
    const int steps = nasg_dp_plan(&c->cfg, n_all.data(), c->nranks, c->rank, max_steps, local.data(),
                                   global.data(), resh.data());
    if (steps < 0) return fail(NASG_ERR_INVALID, "bad data-parallel plan");
    int r = ensure_order(c, (size_t)std::max<int64_t>(n, 1));
    if (r) return r;
    // epoch shuffle (guiding.cpp:216-225); rank 0 uses the reference's stream 5
    Pcg32 rng = shuffle_rng(c, (uint64_t)c->iterations);
    // When every minibatch is this rank's whole buffer (config 3: S = t), each
    // step sums over the same set of rows whatever the permutation, so the
    // shuffle cannot change which samples a step sees: rows are read in place
    // (order = nullptr). Otherwise the host Fisher-Yates runs into one of two
    // pinned order buffers while the GPU still works on the previous upload.
    bool whole = true;
    for (int step = 0; step < steps; ++step) whole = whole && local[step] == n;
    uint32_t *ord = nullptr;
    auto reshuffle = [&]() -> int {  // Fisher-Yates :219-224, continuing one rng stream per iteration
        uint32_t *prev = ord;
        if (!prev && c->pf.active) {  // first epoch computed ahead by ctx_prefetch_shuffle
            join_prefetch(c);
            c->pf.active = false;
            if (c->pf.n == n && c->pf.iteration == (uint64_t)c->iterations) {
                c->order_slot = c->pf.slot;
                ord = c->h_order[c->order_slot];
                rng.state = c->pf.rng_state;
                rng.inc = c->pf.rng_inc;
                return NASG_OK;
            }
        }
        c->order_slot ^= 1;
        CUDA_TRY(cudaEventSynchronize(c->order_ev[c->order_slot]));  // its last upload has left
        ord = c->h_order[c->order_slot];
        if (!prev) {
            first_epoch_shuffle(ord, n, rng);
            return NASG_OK;
        }
        std::memcpy(ord, prev, n * sizeof(uint32_t));
        for (int64_t i = n; i > 1; --i) {
            uint32_t j = rng.next_below((uint32_t)i);
            std::swap(ord[i - 1], ord[j]);
        }
        return NASG_OK;
    };
    if (stats) CUDA_TRY(cudaMemsetAsync(c->d_acc, 0, 5 * sizeof(double), s));
    int64_t cursor = 0;
    int epoch = 0;
    for (int step = 0; step < steps; ++step) {
        if (resh[step] && step > 0) ++epoch;
        if (resh[step] && !whole) {
            r = reshuffle();
            if (r) return r;
            CUDA_TRY(cudaMemcpyAsync(c->d_order, ord, n * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
            CUDA_TRY(cudaEventRecord(c->order_ev[c->order_slot], s));
            cursor = 0;
        }
        r = train_step_impl(c, samples, whole ? nullptr : c->d_order + cursor, local[step], global[step], b, s,
                            epoch == 0);
        if (r) return r;
        cursor += local[step];
    }
    if (c->pf.active) {  // prefetched for a different buffer size / unused (whole-buffer steps)
        join_prefetch(c);
        c->pf.active = false;
    }
    ++c->iterations;
    if (s != c->stream) {
        CUDA_TRY(cudaEventRecord(c->xev, s));
        CUDA_TRY(cudaStreamWaitEvent(c->stream, c->xev, 0));
    }
    r = do_publish(c);
    if (r) return r;
    if (stats) return nasg_train_stats_take(c, stats);
    return NASG_OK;
}

int nasg_get_last_grad(nasg_ctx *c, float *host_g, size_t n) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c || !host_g || n != (size_t)c->nw_ext) return fail(NASG_ERR_INVALID, "bad argument");
    return copy_out_wide(c, c->grad, host_g);
}

int64_t nasg_adam_t(nasg_ctx *c) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c) return -1;
    int64_t t = 0;
    if (cudaDeviceSynchronize() != cudaSuccess) return -1;
    if (cudaMemcpy(&t, c->d_adam_t, sizeof(t), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    return t;
}

// ---- multi-GPU ------------------------------------------------------------------------
int nasg_comm_unique_id(void *out) {
    if (!out) return fail(NASG_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (!g_nccl.load()) return fail(NASG_ERR_NCCL, "libnccl.so.2 not loadable");
    ncclUniqueId id;
    if (g_nccl.getUniqueId(&id) != ncclSuccess) return fail(NASG_ERR_NCCL, "ncclGetUniqueId failed");
    std::memcpy(out, &id, sizeof(id));
    return NASG_OK;
}

namespace {
// Binds `comm` (already created) as the context's communicator: the size
// exchange buffers are (re)allocated first, so a failure leaves the previous
// communicator and its rank/nranks in place.
int bind_comm(nasg_ctx *c, ncclComm_t comm, bool owned, int rank, int nranks) {
    int64_t *d = nullptr, *h = nullptr;
    if (cudaMalloc(&d, sizeof(int64_t) * nranks) != cudaSuccess ||
        cudaMallocHost(&h, sizeof(int64_t) * nranks) != cudaSuccess) {
        cudaGetLastError();
        if (d) cudaFree(d);
        return fail(NASG_ERR_OOM, "communicator buffers");
    }
    if (!c->nall_ev && cudaEventCreateWithFlags(&c->nall_ev, cudaEventDisableTiming) != cudaSuccess) {
        cudaFree(d);
        cudaFreeHost(h);
        return fail(NASG_ERR_CUDA, "event create failed");
    }
    cudaDeviceSynchronize();  // nothing may still use the old communicator
    if (c->comm && c->comm_owned && g_nccl.commDestroy) g_nccl.commDestroy(c->comm);
    if (c->d_nall) cudaFree(c->d_nall);
    if (c->h_nall) cudaFreeHost(c->h_nall);
    c->d_nall = d;
    c->h_nall = h;
    c->comm = comm;
    c->comm_owned = owned;
    c->rank = rank;
    c->nranks = nranks;
    return NASG_OK;
}
}  // namespace

int nasg_comm_init(nasg_ctx *c, const void *uid, int rank, int nranks) {
    if (!c || !uid || nranks < 1 || rank < 0 || rank >= nranks) return fail(NASG_ERR_INVALID, "bad argument");
    DeviceScope ds(c->device);
    {
        std::lock_guard<std::mutex> lk(g_nccl_mu);
        if (!g_nccl.load()) return fail(NASG_ERR_NCCL, "libnccl.so.2 not loadable");
    }
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    ncclComm_t comm = nullptr;  // the old communicator stays bound until the new one exists
    ncclResult_t e = g_nccl.commInitRank(&comm, nranks, id, rank);
    if (e != ncclSuccess)
        return fail(NASG_ERR_NCCL, std::string("ncclCommInitRank: ") + (g_nccl.errStr ? g_nccl.errStr(e) : ""));
    int r = bind_comm(c, comm, true, rank, nranks);
    if (r) g_nccl.commDestroy(comm);
    return r;
}

int nasg_attach_nccl(nasg_ctx *c, void *comm, int rank, int nranks) {
    if (!c || nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !comm))
        return fail(NASG_ERR_INVALID, "bad argument");
    if (nranks == 1 && !comm) return NASG_OK;
    DeviceScope ds(c->device);
    {
        std::lock_guard<std::mutex> lk(g_nccl_mu);
        if (!g_nccl.load()) return fail(NASG_ERR_NCCL, "libnccl.so.2 not loadable");
    }
    int count = 0, dev = -1;
    ncclComm_t cm = static_cast<ncclComm_t>(comm);
    if (g_nccl.commCount(cm, &count) != ncclSuccess || g_nccl.commCuDevice(cm, &dev) != ncclSuccess)
        return fail(NASG_ERR_NCCL, "cannot query the communicator");
    if (count != nranks) return fail(NASG_ERR_INVALID, "communicator size != nranks");
    if (dev != c->device) return fail(NASG_ERR_INVALID, "communicator is bound to another device");
    return bind_comm(c, cm, false, rank, nranks);
}

// ---- counters / schedules ------------------------------------------------------------
int nasg_get_counters(nasg_ctx *c, nasg_counters *out) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c || !out) return fail(NASG_ERR_INVALID, "null argument");
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaDeviceSynchronize());
    unsigned long long clamps = 0;
    int64_t t = 0;
    CUDA_TRY(cudaMemcpy(&clamps, c->d_clamp, sizeof(clamps), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(&t, c->d_adam_t, sizeof(t), cudaMemcpyDeviceToHost));
    out->encode_clamps = clamps;
    out->kernel_launches = c->launches;
    out->adam_steps = t;
    out->iterations = c->iterations;
    out->rank = c->rank;
    out->nranks = c->nranks;
    out->collectives = c->collectives;
    return NASG_OK;
}

uint64_t nasg_encode_clamp_count(nasg_ctx *c) {
    DeviceScope ds_(c ? c->device : -1);
    if (!c) return 0;
    unsigned long long v = 0;
    cudaStreamSynchronize(c->stream);
    cudaDeviceSynchronize();
    cudaMemcpy(&v, c->d_clamp, sizeof(v), cudaMemcpyDeviceToHost);
    return v;
}

void nasg_reset_encode_clamp_count(nasg_ctx *c) {
    DeviceScope ds_(c ? c->device : -1);
    if (c) cudaMemset(c->d_clamp, 0, sizeof(unsigned long long));
}

uint64_t nasg_kernel_launches(nasg_ctx *c) { return c ? c->launches : 0; }

double nasg_blend_coefficient(int64_t i, int m, int b_steps) {  // BlendSchedule guiding.hpp:78-88
    double b = (double)(i / m) / b_steps;
    return b < 1.0 ? b : 1.0;
}

double nasg_stride_update(double l, uint64_t s, uint64_t cap) {  // guiding.cpp:178-182
    double next = l * std::sqrt((double)s / (double)cap);
    return std::max(1.0, next);
}

}  // extern "C"

// ---- synthetic workloads ---------------------------------------------------------------
static void sphere(Pcg32 &r, float *out) {
    const double z = 1.0 - 2.0 * r.next_f24();
    const double phi = 2.0 * 3.14159265358979323846 * r.next_f24();
    const double rr = std::sqrt(std::max(0.0, 1.0 - z * z));
    out[0] = (float)(rr * std::cos(phi));
    out[1] = (float)(rr * std::sin(phi));
    out[2] = (float)z;
    out[3] = 0.f;
}

template <class F>
static void parallel_for(int64_t n, F f) {
    const int64_t per = 1 << 16;
    int nt = (int)std::min<int64_t>((n + per - 1) / per, std::max(1u, std::thread::hardware_concurrency()));
    if (nt <= 1) {
        f(0, n);
        return;
    }
    std::vector<std::thread> th;
    const int64_t step = (n + nt - 1) / nt;
    for (int k = 0; k < nt; ++k) {
        const int64_t a = k * step, b = std::min(n, a + step);
        if (a < b) th.emplace_back(f, a, b);
    }
    for (auto &t : th) t.join();
}

extern "C" {

void nasg_synth_queries(uint64_t seed, int64_t first, int64_t n, const float bmin[3], const float bmax[3], float *x,
                        float *wo, float *nrm, float *xi) {
    parallel_for(n, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) {
            Pcg32 r(hash_combine(seed, (uint64_t)(first + i)), 0x51);
            for (int k = 0; k < 3; ++k) x[4 * i + k] = bmin[k] + (bmax[k] - bmin[k]) * r.next_f24();
            x[4 * i + 3] = 0.f;
            sphere(r, wo + 4 * i);
            sphere(r, nrm + 4 * i);
            for (int k = 0; k < 4; ++k) xi[4 * i + k] = r.next_f24();
        }
    });
}

void nasg_synth_samples(uint64_t seed, int64_t first, int64_t n, const float bmin[3], const float bmax[3],
                        nasg_train_sample *out) {
    parallel_for(n, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) {
            Pcg32 r(hash_combine(seed, (uint64_t)(first + i)), 0x53);
            nasg_train_sample &s = out[i];
            float wo[4], nn[4], wi[4];
            for (int k = 0; k < 3; ++k) s.position[k] = bmin[k] + (bmax[k] - bmin[k]) * r.next_f24();
            sphere(r, wo);
            sphere(r, nn);
            sphere(r, wi);
            for (int k = 0; k < 3; ++k) {
                s.omega_o[k] = wo[k];
                s.normal[k] = nn[k];
                s.omega_i[k] = wi[k];
            }
            const double cosn = std::max(0.0, (double)wi[0] * nn[0] + (double)wi[1] * nn[1] + (double)wi[2] * nn[2]);
            // fixed analytic target field mu(x)
            double mu[3] = {std::sin(2.0 * s.position[0]) + 0.5, std::cos(3.0 * s.position[1]),
                            1.0 + 0.5 * std::sin((double)s.position[2])};
            const double inv = 1.0 / std::sqrt(mu[0] * mu[0] + mu[1] * mu[1] + mu[2] * mu[2]);
            const double d = (wi[0] * mu[0] + wi[1] * mu[1] + wi[2] * mu[2]) * inv;
            s.p_value = (float)(std::exp(20.0 * (d - 1.0)) * cosn);
            s.q_sampling = (float)(1.0 / (4.0 * 3.14159265358979323846));
            s.bsdf_pdf_at_wi = (float)(cosn / 3.14159265358979323846);
            s.pad = 0.f;
        }
    });
}


int nasg_dist_mixture_pdf(int kind, int64_t n, int k, const float *comp, const float *weights, const float *dir,
                          float *pdf, void *stream) {
    return dist_call(0, kind, n, k, comp, weights, dir, pdf, stream);
}
int nasg_dist_mixture_sample(int kind, int64_t n, int k, const float *comp, const float *weights, const float *xi,
                             float *dir_pdf, void *stream) {
    return dist_call(1, kind, n, k, comp, weights, xi, dir_pdf, stream);
}
int nasg_dist_grad_logpdf(int kind, int64_t n, int k, const float *comp, const float *weights, const float *dir,
                          float *grad, void *stream) {
    return dist_call(2, kind, n, k, comp, weights, dir, grad, stream);
}

int nasg_fit_raw_dim(int model, int k) {
    if (model == NASG_DIST_NASG)
        return (k == 1 || k == 2 || k == 4 || k == 8 || k == 16) ? fit_raw_dim_host(model, k) : -1;
    if (model == NASG_DIST_VMF) return (k >= 1 && k <= fit_max_components(model)) ? fit_raw_dim_host(model, k) : -1;
    return -1;
}

int nasg_fit(const nasg_fit_config *cfg, int n_fits, int target_kind, int target_k, const float *target_comp,
             const float *target_w, const float *raw_init, float *raw_out, double *kl_out, int quad_nz) {
    if (!cfg || n_fits <= 0 || !raw_out) return fail(NASG_ERR_INVALID, "bad argument");
    int r = fit_check_model(cfg->model, cfg->n_components);
    if (r) return r;
    if (cfg->batch <= 0 || cfg->steps <= 0 || cfg->checkpoints <= 0 || cfg->checkpoints > cfg->steps)
        return fail(NASG_ERR_INVALID, "batch, steps > 0 and 1 <= checkpoints <= steps");
    if (kl_out && quad_nz <= 0) return fail(NASG_ERR_INVALID, "quad_nz must be > 0");
    if ((r = check_current_device())) return r;
    DevBuf dc, dw, dinit, dout, dp;
    if ((r = fit_upload_target(target_kind, target_k, target_comp, target_w, dc, dw))) return r;
    const int D = fit_raw_dim_host(cfg->model, cfg->n_components);
    const size_t outn = (size_t)n_fits * cfg->checkpoints * D;
    if ((r = dout.alloc(outn * sizeof(float)))) return r;
    if (raw_init) {
        if ((r = dinit.alloc((size_t)n_fits * D * sizeof(float)))) return r;
        CUDA_TRY(cudaMemcpy(dinit.p, raw_init, (size_t)n_fits * D * sizeof(float), cudaMemcpyHostToDevice));
    }
    FitLaunch L{};
    L.model = cfg->model;
    L.k = cfg->n_components;
    L.tkind = target_kind;
    L.tk = target_k;
    L.tcomp = dc.as<float>();
    L.tw = dw.as<float>();
    L.batch = cfg->batch;
    L.steps = cfg->steps;
    L.n_ckpt = cfg->checkpoints;
    L.n_fits = n_fits;
    L.lr = cfg->learning_rate;
    L.seed = cfg->seed;
    L.raw_init = raw_init ? dinit.as<float>() : nullptr;
    L.raw_out = dout.as<float>();
    if (fit_launch(L, 0) < 0) return fail(NASG_ERR_UNSUPPORTED, "fit configuration not compiled");
    CHECK_LAUNCH();
    CUDA_TRY(cudaMemcpy(raw_out, dout.p, outn * sizeof(float), cudaMemcpyDeviceToHost));
    if (kl_out) {
        const int64_t npt = (int64_t)quad_nz * 2 * quad_nz;
        if ((r = dp.alloc(npt * sizeof(double)))) return r;
        fit_target_grid(target_kind, target_k, dc.as<float>(), dw.as<float>(), quad_nz, dp.as<double>(), 0);
        CHECK_LAUNCH();
        if ((r = fit_kl_device(cfg->model, cfg->n_components, dout.as<float>(), n_fits * cfg->checkpoints, quad_nz,
                               dp.as<double>(), kl_out)))
            return r;
    }
    return NASG_OK;
}

int nasg_fit_gradient(int model, int k, const float *raw, int64_t n, const float *samples, float *grad_out) {
    int r = fit_check_model(model, k);
    if (r) return r;
    if (!raw || !grad_out || n <= 0 || !samples || n > (1 << 24)) return fail(NASG_ERR_INVALID, "bad argument");
    if ((r = check_current_device())) return r;
    const int D = fit_raw_dim_host(model, k);
    DevBuf draw, ds, dg;
    if ((r = draw.alloc(D * sizeof(float))) || (r = ds.alloc((size_t)n * 4 * sizeof(float))) ||
        (r = dg.alloc(D * sizeof(float))))
        return r;
    CUDA_TRY(cudaMemcpy(draw.p, raw, D * sizeof(float), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(ds.p, samples, (size_t)n * 4 * sizeof(float), cudaMemcpyHostToDevice));
    FitLaunch L{};
    L.model = model;
    L.k = k;
    L.batch = (int)n;
    L.n_fits = 1;
    L.raw_init = draw.as<float>();
    L.samples = ds.as<float>();
    L.grad_out = dg.as<float>();
    if (fit_launch(L, 0) < 0) return fail(NASG_ERR_UNSUPPORTED, "fit configuration not compiled");
    CHECK_LAUNCH();
    CUDA_TRY(cudaMemcpy(grad_out, dg.p, D * sizeof(float), cudaMemcpyDeviceToHost));
    return NASG_OK;
}

int nasg_fit_kl(int target_kind, int target_k, const float *target_comp, const float *target_w, int model, int k,
                int n_models, const float *raws, int quad_nz, double *kl_out) {
    int r = fit_check_model(model, k);
    if (r) return r;
    if (n_models <= 0 || !raws || !kl_out || quad_nz <= 0) return fail(NASG_ERR_INVALID, "bad argument");
    if ((r = check_current_device())) return r;
    DevBuf dc, dw, draws, dp;
    if ((r = fit_upload_target(target_kind, target_k, target_comp, target_w, dc, dw))) return r;
    const int D = fit_raw_dim_host(model, k);
    if ((r = draws.alloc((size_t)n_models * D * sizeof(float)))) return r;
    CUDA_TRY(cudaMemcpy(draws.p, raws, (size_t)n_models * D * sizeof(float), cudaMemcpyHostToDevice));
    const int64_t npt = (int64_t)quad_nz * 2 * quad_nz;
    if ((r = dp.alloc(npt * sizeof(double)))) return r;
    fit_target_grid(target_kind, target_k, dc.as<float>(), dw.as<float>(), quad_nz, dp.as<double>(), 0);
    CHECK_LAUNCH();
    return fit_kl_device(model, k, draws.as<float>(), n_models, quad_nz, dp.as<double>(), kl_out);
}

}  // extern "C"
