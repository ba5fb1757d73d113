// rgc_api.cu -- the C ABI of librgc.so (declared in include/rgc.h).
//
// Host side only: validation, workspace layout, the fixed kernel sequence of
// rgc_compress, the NCCL allgather of rgc_sync (libnccl.so.2 is dlopen'ed so
// the library binds the same NCCL torch loaded), and rgc_decompress.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges for nsys / ncu --nvtx

#include "../../include/rgc.h"
#include "rgc_internal.cuh"

#ifndef RGC_NCCL_PATH
#define RGC_NCCL_PATH ""
#endif

using namespace rgc;

// ---------------------------------------------------------------- NCCL (dlopen)
namespace {
typedef struct ncclComm *ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;          // ncclSuccess = 0, ncclInProgress = 7
enum { ncclUint8 = 1, ncclFloat32 = 7 };
enum { ncclSum = 0 };

struct Nccl {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};
Nccl g_nccl;

bool nccl_load(std::string &err) {
    if (g_nccl.h) return true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // the one torch loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h && RGC_NCCL_PATH[0]) h = dlopen(RGC_NCCL_PATH, RTLD_NOW);
    if (!h) { err = std::string("cannot dlopen libnccl.so.2: ") + dlerror(); return false; }
#define SYM(f) *(void **)(&g_nccl.f) = dlsym(h, "nccl" #f); if (!g_nccl.f) { err = "missing nccl" #f; return false; }
    SYM(GetUniqueId) SYM(CommInitRank) SYM(CommDestroy) SYM(CommGetAsyncError) SYM(AllGather)
    SYM(Broadcast) SYM(GroupStart) SYM(GroupEnd) SYM(GetErrorString)
#undef SYM
    g_nccl.h = h;
    return true;
}

constexpr int kPhaseCount = RGC_NPHASE;

struct ProfRec { int phase; cudaEvent_t a, b; };

struct Layout {
    int L = 0;
    uint32_t TV = 0, TD = 0, H = 0;
    uint64_t off_desc = 0, off_ddesc = 0, off_st = 0, off_statA = 0, off_statB = 0, off_S = 0,
             off_dec = 0, ws_bytes = 0, msg_bytes = 0, cap_total = 0, k_total = 0, s_total = 0,
             off_cand = 0, off_rec = 0, cand_total = 0, off_lay = 0, off_Q = 0, q_total = 0,
             cap_dense = 0, cap_asq = 0, tab_off = 0;
    uint32_t tab_words = 0;      // producer range table: TD + L words (padded to 16 bytes)
    bool any_quant = false;
    uint32_t status_words = 0;
    int max_trim = 0;
    int k45_cl = 4;                   // K45 CTAs per cluster (2 or 4)
    std::vector<LayerDesc> desc;      // without pointers
    std::vector<DecompDesc> ddesc;    // without pointers
};

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// A workspace keeps kSlots versions of each layer table (pointers + constants),
// so alternating buffer sets (e.g. double-buffered gradients) need no upload
// and no host wait in steady state, and a CUDA graph can be captured.
constexpr int kSlots = 4;
struct TableCache {
    const void *ws = nullptr;
    size_t slot_bytes = 0;
    std::vector<uint8_t> content[kSlots];
    uint64_t last_use[kSlots] = {0, 0, 0, 0};
    bool valid[kSlots] = {false, false, false, false};
    bool ev_used[kSlots] = {false, false, false, false};
    bool pinned[kSlots] = {false, false, false, false};   // used by a captured CUDA graph
    void *staging[kSlots] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t ev[kSlots] = {nullptr, nullptr, nullptr, nullptr};
    uint64_t tick = 0;
};

constexpr uint32_t kG2Max = 148 * 8;       // upper bound of the K1 grid (candidate records)
constexpr uint64_t kDescBytes = sizeof(LayerDesc) * RGC_MAX_LAYERS;
constexpr uint64_t kDdescBytes = sizeof(DecompDesc) * RGC_MAX_LAYERS;
// offsets of the fixed-size head of a workspace: Ctrl | desc slots | ddesc slots | LayerState[]
constexpr uint64_t kOffDesc = sizeof(Ctrl);
constexpr uint64_t kOffDdesc = (kOffDesc + kDescBytes * kSlots + 255) / 256 * 256;
constexpr uint64_t kOffState = (kOffDdesc + kDdescBytes * kSlots + 255) / 256 * 256;
}  // namespace

struct rgc_ctx {
    int rank = 0, nranks = 1, device = 0;
    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;
    std::string err;
    int sms = 148, occ1 = 1, occ2 = 1, occ3 = 1, occ4 = 1, occ6 = 1;
    uint64_t launches = 0;
    // device copies of the per-call layer tables: kSlots versions per workspace
    TableCache tdesc, tddesc;
    // SIZES_FIRST scratch
    uint32_t *h_hdr = nullptr;
    size_t h_hdr_bytes = 0;
    void *d_hdr = nullptr;
    size_t d_hdr_bytes = 0;
    // profiling
    int prof = 0;                          // 1: every phase, 2: accumulate (K1) only
    int prof_every = 1;                    // prof 2: K1 on every prof_every-th compress call
    uint64_t prof_calls = 0;               // compress calls since rgc_profile
    std::vector<ProfRec> recs;
    std::vector<cudaEvent_t> pool;
    double acc[kPhaseCount] = {0};
    int ncompress = 0;
    // RGC_SYNC_P2P (rgc_p2p_init): staging areas mapped across ranks with CUDA IPC
    bool p2p = false;
    void *p2p_msg = nullptr;               // this rank's message block (library-owned)
    uint64_t p2p_bytes = 0;
    uint8_t *p2p_stage = nullptr;          // nranks blocks: slot r = rank r's pushed block
    P2PFlags *p2p_flags = nullptr;         // this rank's epoch flags
    std::vector<void *> p2p_open;          // peer mappings (closed by rgc_finalize)
    uint8_t **d_peer_stage = nullptr;      // device table [nranks] of staging areas
    P2PFlags **d_peer_flags = nullptr;     // device table [nranks] of flag blocks
    unsigned long long epoch = 0;          // P2P syncs so far
    bool p2p_synced = false;               // a P2P sync precedes the next decompress
    // RGC_SYNC_PULL: every rank's message block mapped here (own block at [rank])
    std::vector<uint8_t *> h_peer_msg;     // host copy of the table (rgc_p2p_gather)
    uint8_t **d_peer_msg = nullptr;        // device table [nranks]
    bool pull_synced = false;              // the pending sync was RGC_SYNC_PULL
    unsigned long long pull_wait_epoch = 0;  // next compress: wait for peers' consumed >= this
    // rgc_decompress_prefill: the dense zero fill of the next decompression runs on an
    // auxiliary stream forked after the next compress' K1 (overlaps the selection)
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int fill_state = 0;                    // 0 none, 1 registered, 2 enqueued (not joined)
    FillTable fill;
    unsigned int *d_sig = nullptr;         // k6_fill control words (kFillSigWords)
    unsigned long long *d_k1cnt = nullptr; // K1 CTAs done streaming (monotonic; RGC_FILL_AT=0)
    unsigned long long k1cnt_total = 0;    // its value after the last counted K1
    // device status (rgc_status): sticky words in device memory, mirrored by k_finish into
    // pinned host-mapped memory when they change (the host polls without a sync)
    uint32_t *d_stat = nullptr;
    uint32_t *h_stat = nullptr;            // host view of the mapped words
    uint32_t *h_stat_dev = nullptr;        // device address of the same pinned words
    uint32_t nccl_err = 0;                 // sticky ncclResult_t of an NCCL async error
    bool poisoned = false;                 // a cross-GPU wait timed out: epochs out of step
    bool assume_tab = false;               // RGC_ASSUME_TAB=1 at rgc_init: a context without a
                                           // communicator decompresses blocks that carry their
                                           // range tables (single-GPU simulation of p ranks)
    unsigned long long timeout_ns = 0;     // P2P / PULL wait limit (RGC_P2P_TIMEOUT_S)
    unsigned long long *d_tl = nullptr;    // RGC_TIMELINE=1: per-kernel start / end (Ws::tl)
};

namespace {
rgc_status_t fail(rgc_ctx *c, rgc_status_t s, const char *fmt, ...) {
    if (c) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        c->err = buf;
    }
    return s;
}

#define CUDA_TRY(c, call)                                                                     \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail((c), RGC_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e_));      \
    } while (0)

bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

uint64_t k_of(uint64_t n, double D) {
    double kd = ceil(D * (double)n);
    uint64_t k = (uint64_t)kd;
    if (k < 1) k = 1;
    if (k > n) k = n;
    return k;
}

// Alg.2 ratio levels with ratio > 0: 1-eps, 1-2eps, ... ; 0 if > 16 levels
uint32_t trim_levels_of(double eps) {
    uint32_t n = 0;
    for (double r = 1.0 - eps; r > 0.0; r = r - eps)
        if (++n > RGC_MAX_TRIM_LEVELS) return 0;
    return n;
}

rgc_status_t make_layout(rgc_ctx *c, const rgc_layer_t *layers, int L, Layout &lo) {
    if (!layers || L < 1 || L > RGC_MAX_LAYERS)
        return fail(c, RGC_EINVAL, "L=%d outside [1, %d]", L, RGC_MAX_LAYERS);
    lo = Layout();
    lo.L = L;
    lo.desc.resize(L);
    lo.ddesc.resize(L);
    uint64_t s_total = 0;
    for (int l = 0; l < L; l++) {
        const rgc_layer_t &y = layers[l];
        if (y.n == 0 || y.n >= (1ull << 31))
            return fail(c, RGC_EINVAL, "layer %d: n=%llu outside [1, 2^31)", l, (unsigned long long)y.n);
        if (!(y.density > 0.0 && y.density <= 1.0))
            return fail(c, RGC_EINVAL, "layer %d: density %g outside (0,1]", l, y.density);
        if (!(y.momentum >= 0.0f) || isinf(y.momentum))
            return fail(c, RGC_EINVAL, "layer %d: momentum %g invalid", l, (double)y.momentum);
        if (y.selector != RGC_SEL_TRIMMED && y.selector != RGC_SEL_THRESHOLD_BS &&
            y.selector != RGC_SEL_SAMPLED_BS)
            return fail(c, RGC_EINVAL, "layer %d: selector %d invalid", l, y.selector);
        if (y.bs_branch != RGC_BS_MONOTONE && y.bs_branch != RGC_BS_PAPER_LITERAL)
            return fail(c, RGC_EINVAL, "layer %d: bs_branch %d invalid", l, y.bs_branch);
        if (y.quantize != 0 && y.quantize != 1)
            return fail(c, RGC_EINVAL, "layer %d: quantize %d invalid", l, y.quantize);
        if (y.quantize && y.selector == RGC_SEL_SAMPLED_BS)
            return fail(c, RGC_EINVAL, "layer %d: sampled threshold binary search cannot be used "
                                       "with quantization (P:292)", l);
        const double teps = y.trim_eps == 0.0 ? 0.2 : y.trim_eps;
        const double beps = y.bs_eps == 0.0 ? 1e-3 : y.bs_eps;
        const uint32_t tl = (teps > 0.0 && teps < 1.0) ? trim_levels_of(teps) : 0;
        if (tl == 0)
            return fail(c, RGC_EINVAL, "layer %d: trim_eps %g gives no level or more than 16", l, teps);
        if (!(beps >= 0.0009765625 && beps < 1.0))
            return fail(c, RGC_EINVAL, "layer %d: bs_eps %g outside [2^-10, 1)", l, beps);
        const uint64_t k = k_of(y.n, y.density);
        const bool bs = y.selector != RGC_SEL_TRIMMED;   // Alg.3 and its sampled variant
        uint64_t mc = y.max_count ? y.max_count : (bs ? 2 * k : k);
        if (mc < k)
            return fail(c, RGC_EINVAL, "layer %d: max_count %u < k %llu", l, y.max_count,
                        (unsigned long long)k);
        if (mc > 0xFFFFFFFFull) mc = 0xFFFFFFFFull;
        const uint64_t cap = mc < y.n ? mc : y.n;   // a message never exceeds n pairs
        LayerDesc &d = lo.desc[l];
        memset(&d, 0, sizeof d);
        d.n = (uint32_t)y.n;
        d.k = (uint32_t)k;
        d.tile_begin = lo.TV;
        d.ntiles = (uint32_t)((y.n + kTile - 1) / kTile);
        d.cap = (uint32_t)mc;
        d.s_cap = 0;
        if (!bs || y.selector == RGC_SEL_SAMPLED_BS) {
            // Alg.2 survivor buffer: momentum-corrected residuals keep many elements above the
            // first level (R5), so size it generously: max(64K, 64k, n/8), at most n.  Sampled
            // BS layers use it on a reuse step whose count exceeds the capacity (R18): the
            // exact top-k then runs over {|V| > t_cached} instead of all of V
            uint64_t sc = 64 * k;
            if (sc < 65536) sc = 65536;
            if (sc < y.n / 8) sc = y.n / 8;
            if (sc > y.n) sc = y.n;
            d.s_cap = (uint32_t)sc;
        }
        d.s_off = s_total;
        s_total += d.s_cap;
        d.m = y.momentum;
        d.selector = (uint32_t)y.selector;
        d.branch = (uint32_t)y.bs_branch;
        d.trim_levels = tl;
        d.interval = y.sample_interval ? y.sample_interval : 5u;
        d.trim_eps = teps;
        d.bs_eps = beps;
        d.quant = y.quantize ? 1u : 0u;
        d.q_off = lo.q_total;
        const uint64_t mcap = bs ? cap : k;   // message entries of this layer at most
        if (d.quant) { lo.q_total += mcap; lo.cap_asq += mcap; } else { lo.cap_dense += mcap; }
        lo.TV += d.ntiles;
        if (!bs && (int)tl > lo.max_trim) lo.max_trim = (int)tl;
        DecompDesc &dd = lo.ddesc[l];
        memset(&dd, 0, sizeof dd);
        dd.n = (uint32_t)y.n;
        dd.tile_begin = lo.TD;
        dd.ntiles = (uint32_t)((y.n + kDecTile - 1) / kDecTile);
        dd.slot_begin = lo.TD + (uint32_t)l;
        dd.quant = y.quantize ? 1u : 0u;
        lo.TD += dd.ntiles;
        lo.cap_total += bs ? cap : k;
        lo.k_total += k;
        lo.any_quant |= y.quantize != 0;
    }
    lo.s_total = s_total;
    {
        // K45 cluster size: 4 CTAs (180K-key sets) unless the layers that can take K45 (Alg.2
        // and sampled-BS layers, small layers in an exact fallback) need more than one wave of
        // 4-CTA clusters (1024-thread CTAs, one per SM) -- then 2 (90K-key sets, larger ones
        // take K4 + K3B): ResNet-50's 53 conv layers.  RGC_K45_CL = 2 / 4 overrides.
        static const int forced = [] { const char *e = getenv("RGC_K45_CL"); return e ? atoi(e) : 0; }();
        int n45 = 0;
        for (int l = 0; l < L; l++)
            if (layers[l].selector != RGC_SEL_THRESHOLD_BS || layers[l].n <= (uint64_t)kSmallSel) n45++;
        const int sms = c ? c->sms : 148;   // rgc_sizes may run without a context
        lo.k45_cl = (forced == 1 || forced == 2 || forced == 4 || forced == 8) ? forced : (4 * n45 > sms ? 2 : 4);
    }
    // header: counts[L], status, L, value words[L], table marker (include/rgc.h), 16-byte
    // multiple; then the pairs / ASQ indices (capacity); then the producer's range table
    lo.H = 4u * (uint32_t)((2 * L + 3 + 3) / 4);
    lo.tab_off = align_up(4ull * lo.H + 8ull * lo.cap_dense + 4ull * lo.cap_asq, 16);
    lo.tab_words = (uint32_t)align_up((uint64_t)lo.TD + (uint64_t)L, 4);
    lo.msg_bytes = lo.tab_off + 4ull * lo.tab_words;
    uint64_t o = kOffState;
    lo.off_desc = kOffDesc;
    lo.off_ddesc = kOffDdesc;
    lo.off_st = o; o = align_up(o + sizeof(LayerState) * (uint64_t)L, 256);
    lo.status_words = lo.TV + (uint32_t)L + kG2Max;    // K3 segments: V tiles or K1 records
    lo.off_statA = o; o = align_up(o + 8ull * lo.status_words, 256);
    lo.off_statB = o; o = align_up(o + 8ull * lo.status_words, 256);
    lo.off_S = o; o = align_up(o + 8ull * s_total + 8, 256);
    // K2 candidate scratch: ~8% of the elements plus slack per CTA, and the record table
    lo.cand_total = (uint64_t)(0.08 * (double)lo.TV * kTile) + 64ull * kG2Max;
    lo.off_cand = o; o = align_up(o + 8ull * lo.cand_total, 256);
    lo.off_rec = o; o = align_up(o + 8ull * ((uint64_t)L + kG2Max), 256);
    lo.off_dec = o; o = align_up(o + 4ull * (uint64_t)(c ? c->nranks : 1) * (lo.TD + L) + 4, 256);
    lo.off_lay = o; o = align_up(o + 16ull * (uint64_t)(c ? c->nranks : 1) * L, 256);
    lo.off_Q = o; o = align_up(o + 8ull * lo.q_total + 8, 256);
    lo.ws_bytes = o;
    return RGC_OK;
}

Ws ws_of(const Layout &lo, void *ws) {
    uint8_t *b = (uint8_t *)ws;
    Ws w;
    w.ctrl = (Ctrl *)b;
    w.desc = (LayerDesc *)(b + lo.off_desc);
    w.ddesc = (DecompDesc *)(b + lo.off_ddesc);
    w.st = (LayerState *)(b + lo.off_st);
    w.statusA = (unsigned long long *)(b + lo.off_statA);
    w.statusB = (unsigned long long *)(b + lo.off_statB);
    w.S = (uint2 *)(b + lo.off_S);
    w.dec_start = (uint32_t *)(b + lo.off_dec);
    w.cand = (uint2 *)(b + lo.off_cand);
    w.rec = (uint2 *)(b + lo.off_rec);
    w.Q = (uint2 *)(b + lo.off_Q);
    w.dec_lay = (uint4 *)(b + lo.off_lay);
    w.cand_R = 0;
    w.seg_ch = 1;
    w.status_extra = lo.status_words - lo.TV;
    w.ntiles_total = lo.TV;
    w.pull_flags = nullptr;
    w.pull_epoch = 0;
    w.pull_rank = 0;
    w.pull_p = 0;
    w.k4_hint = nullptr;
    w.small_sel = (uint32_t)(lo.k45_cl * kKeysPerCta45);
    w.k1cnt = nullptr;
    w.tl = nullptr;
    return w;
}

cudaEvent_t pool_get(rgc_ctx *c) {
    if (!c->pool.empty()) { cudaEvent_t e = c->pool.back(); c->pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// NVTX range around a host call (tracing): nearly free without a tool attached
struct Nvtx {
    explicit Nvtx(const char *name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
};

const char *const kPhaseName[kPhaseCount] = {
    "K1 accumulate+stats", "K2 count/search", "K3A compaction", "K45/K4 exact select",
    "K3B emission", "sync", "decompress"};

struct PhaseScope {
    rgc_ctx *c; int ph; cudaEvent_t a = nullptr;
    PhaseScope(rgc_ctx *c_, int ph_) : c(c_), ph(ph_) {
        nvtxRangePushA(kPhaseName[ph]);
        if (c->prof == 1 ||
            (c->prof == 2 && ph == 0 && c->prof_calls % (uint64_t)c->prof_every == 0)) {
            a = pool_get(c);
            cudaEventRecord(a, c->stream);
        }
    }
    ~PhaseScope() {
        nvtxRangePop();
        if (a) {
            cudaEvent_t b = pool_get(c);
            cudaEventRecord(b, c->stream);
            c->recs.push_back({ph, a, b});
        }
    }
};

// Find (or upload into) a table slot holding exactly `src`; returns the slot index.
rgc_status_t table_slot(rgc_ctx *c, TableCache &tc, uint8_t *dev_base, uint64_t slot_stride,
                        const void *ws, const void *src, size_t bytes, int *slot_out) {
    if (tc.ws != ws) {
        for (int i = 0; i < kSlots; i++) { tc.valid[i] = false; tc.pinned[i] = false; }
        tc.ws = ws;
    }
    tc.tick++;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(c->stream, &cap);
    for (int i = 0; i < kSlots; i++) {
        if (tc.valid[i] && tc.content[i].size() == bytes &&
            memcmp(tc.content[i].data(), src, bytes) == 0) {
            tc.last_use[i] = tc.tick;
            // a captured graph keeps this slot's device address: never evict it afterwards
            if (cap != cudaStreamCaptureStatusNone) tc.pinned[i] = true;
            *slot_out = i;
            return RGC_OK;
        }
    }
    if (cap != cudaStreamCaptureStatusNone)
        return fail(c, RGC_ESTATE, "layer table changed while the stream is being captured; "
                                   "run the same call once before capturing it");
    int v = -1;
    for (int i = 0; i < kSlots && v < 0; i++) if (!tc.valid[i]) v = i;
    if (v < 0) {
        for (int i = 0; i < kSlots; i++)
            if (!tc.pinned[i] && (v < 0 || tc.last_use[i] < tc.last_use[v])) v = i;
    }
    if (v < 0)
        return fail(c, RGC_ESTATE, "all %d layer-table slots of this workspace are held by captured "
                                   "CUDA graphs; rgc_workspace_init releases them", kSlots);
    if (!tc.staging[v]) CUDA_TRY(c, cudaMallocHost(&tc.staging[v], slot_stride));
    if (!tc.ev[v]) CUDA_TRY(c, cudaEventCreateWithFlags(&tc.ev[v], cudaEventDisableTiming));
    if (tc.ev_used[v]) CUDA_TRY(c, cudaEventSynchronize(tc.ev[v]));   // previous users done
    memcpy(tc.staging[v], src, bytes);
    CUDA_TRY(c, cudaMemcpyAsync(dev_base + (uint64_t)v * slot_stride, tc.staging[v], bytes,
                                cudaMemcpyHostToDevice, c->stream));
    tc.content[v].assign((const uint8_t *)src, (const uint8_t *)src + bytes);
    tc.valid[v] = true;
    tc.last_use[v] = tc.tick;
    *slot_out = v;
    return RGC_OK;
}

// mark the slot as used by the work just enqueued (skipped while capturing)
void table_used(rgc_ctx *c, TableCache &tc, int v) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(c->stream, &cap);
    if (cap == cudaStreamCaptureStatusNone && tc.ev[v]) {
        cudaEventRecord(tc.ev[v], c->stream);
        tc.ev_used[v] = true;
    }
}

void table_free(TableCache &tc) {
    for (int i = 0; i < kSlots; i++) {
        if (tc.staging[i]) cudaFreeHost(tc.staging[i]);
        if (tc.ev[i]) cudaEventDestroy(tc.ev[i]);
        tc.staging[i] = nullptr;
        tc.ev[i] = nullptr;
    }
}

int grid_of(rgc_ctx *c, int occ, uint64_t work) {
    uint64_t g = (uint64_t)c->sms * (uint64_t)(occ > 0 ? occ : 1);
    if (work < g) g = work;
    if (g < 1) g = 1;
    return (int)g;
}

// enqueue the registered zero fill on the auxiliary stream, ordered after the work
// already on the context stream
// Enqueue the registered zero fill on the high-priority auxiliary stream, ordered after
// the work already on the context stream (rgc_compress: right after K1, so it streams
// under the latency-bound selection kernels; include/rgc.h, rgc_decomp.cu).
// where the zero fill of rgc_decompress_prefill goes (RGC_FILL_AT): -1 (default) an early fill
// with K1 when K1 has >= 32 tiles per CTA (a long ramp-down), and the regular fill after K1;
// 0 the early fill always; 1 the regular fill after K1 only; 2 after K2
int fill_at() {
    static const int v = getenv("RGC_FILL_AT") ? atoi(getenv("RGC_FILL_AT")) : -1;
    return v;
}

rgc_status_t fill_fork(rgc_ctx *c) {
    const int grid = 2 * c->sms;   // at most one active CTA per SM (rgc_decomp.cu)
    CUDA_TRY(c, cudaEventRecord(c->ev_fork, c->stream));
    CUDA_TRY(c, cudaStreamWaitEvent(c->aux, c->ev_fork, 0));
    CUDA_TRY(c, launch_k6_fill(c->fill, c->d_sig, grid, c->aux));
    CUDA_TRY(c, cudaEventRecord(c->ev_join, c->aux));
    c->launches++;
    c->fill_state = 2;
    return RGC_OK;
}
}  // namespace

// CTAs per SM of the stash pass (and of the V passes folded into it); RGC_K2S_MULT overrides
static int k2s_mult() {
    static const int m = [] { const char *e = getenv("RGC_K2S_MULT"); int v = e ? atoi(e) : 2;
                              return v < 1 ? 1 : (v > 4 ? 4 : v); }();
    return m;
}

// Producer range tables (k_tab) in the messages of multi-rank contexts; RGC_NO_TAB=1 turns
// them off (every receiver derives the ranges with k6_prep, round 1's design; A/B)
bool tab_enabled() {
    static const bool on = getenv("RGC_NO_TAB") == nullptr;
    return on;
}

namespace rgc {
bool pdl_enabled() {
    static const bool on = getenv("RGC_NO_PDL") == nullptr;
    return on;
}
}  // namespace rgc

// ======================================================================= API
extern "C" {

const char *rgc_version(void) { return "rgc-b200 0.1 (sm_100a)"; }

const char *rgc_status_string(rgc_status_t s) {
    switch (s) {
        case RGC_OK: return "ok";
        case RGC_EINVAL: return "invalid argument";
        case RGC_ECUDA: return "CUDA error";
        case RGC_ENCCL: return "NCCL error";
        case RGC_ENONFINITE: return "non-finite residual";
        case RGC_ESTATE: return "bad state";
    }
    return "unknown";
}

rgc_status_t rgc_k(uint64_t n, double density, uint64_t *k_out) {
    if (!k_out || n == 0 || !(density > 0.0 && density <= 1.0)) return RGC_EINVAL;
    *k_out = k_of(n, density);
    return RGC_OK;
}

rgc_status_t rgc_get_unique_id(uint8_t out[128]) {
    std::string err;
    if (!out) return RGC_EINVAL;
    if (!nccl_load(err)) return RGC_ENCCL;
    ncclUniqueId id;
    if (g_nccl.GetUniqueId(&id) != 0) return RGC_ENCCL;
    memcpy(out, id.internal, 128);
    return RGC_OK;
}

rgc_status_t rgc_init(rgc_ctx_t *out, int rank, int nranks, int device, const uint8_t *uid,
                      void *stream) {
    if (!out || nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks) return RGC_EINVAL;
    *out = nullptr;
    rgc_ctx *c = new rgc_ctx();
    c->rank = rank; c->nranks = nranks; c->device = device;
    c->stream = (cudaStream_t)stream;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) {
        // prediction policy (which pass reads what; never the result): RGC_TUNE="X,m,R,s"
        uint32_t t[5] = {32u, 16u, 0u, 8u, 6u};
        if (const char *v = getenv("RGC_TUNE"))
            sscanf(v, "%u,%u,%u,%u,%u", &t[0], &t[1], &t[2], &t[3], &t[4]);
        e = set_tuning(t);
    }
    if (e == cudaSuccess) e = occupancy(&c->occ1, &c->occ2, &c->occ3, &c->occ4, &c->occ6);
    // RGC_K1_OCC=n (read here, per context): K1 keeps at most n CTAs per SM, leaving room for
    // the latency-bound selection kernels of another context (bucketed steps, bench --buckets)
    if (const char *v = getenv("RGC_K1_OCC")) {
        const int n = atoi(v);
        if (n >= 1 && n < c->occ1) c->occ1 = n;
    }
    if (e == cudaSuccess) e = cudaMalloc((void **)&c->d_stat, kStatWords * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemset(c->d_stat, 0, kStatWords * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaHostAlloc((void **)&c->h_stat, kStatWords * sizeof(uint32_t),
                                            cudaHostAllocMapped);
    if (e == cudaSuccess) {
        memset(c->h_stat, 0, kStatWords * sizeof(uint32_t));
        e = cudaHostGetDevicePointer((void **)&c->h_stat_dev, c->h_stat, 0);
    }
    c->assume_tab = getenv("RGC_ASSUME_TAB") != nullptr;
    if (getenv("RGC_TIMELINE") && e == cudaSuccess)
        e = cudaMalloc((void **)&c->d_tl, 2 * kTlKernels * sizeof(unsigned long long));
    {
        double tmo = 120.0;
        if (const char *v = getenv("RGC_P2P_TIMEOUT_S")) tmo = atof(v);
        if (!(tmo > 0.0)) tmo = 120.0;
        c->timeout_ns = (unsigned long long)(tmo * 1e9);
    }
    if (e != cudaSuccess) {
        rgc_finalize(c);
        return RGC_ECUDA;
    }
    if (nranks > 1 && uid) {   // uid == NULL: no communicator (decompress of external messages)
        std::string err;
        if (!nccl_load(err)) { rgc_finalize(c); return RGC_ENCCL; }
        ncclUniqueId id;
        memcpy(id.internal, uid, 128);
        if (g_nccl.CommInitRank(&c->comm, nranks, id, rank) != 0) {
            c->comm = nullptr;
            rgc_finalize(c);
            return RGC_ENCCL;
        }
    }
    *out = c;
    return RGC_OK;
}

rgc_status_t rgc_set_stream(rgc_ctx_t c, void *stream) {
    if (!c) return RGC_EINVAL;
    c->stream = (cudaStream_t)stream;
    return RGC_OK;
}

rgc_status_t rgc_finalize(rgc_ctx_t c) {
    if (!c) return RGC_EINVAL;
    cudaSetDevice(c->device);
    if (c->p2p && c->nranks > 1 && c->epoch > 0 && !c->poisoned) {
        // peers map this rank's message block, staging area and flags (CUDA IPC): before they
        // are unmapped and freed, wait (bounded) until every peer published consumed >= the
        // last epoch -- its last reads of this block and its last store into these flags are
        // then complete (cudaDeviceSynchronize alone only waits for local work)
        const unsigned long long lim = std::min<unsigned long long>(c->timeout_ns, 10ull * 1000000000ull);
        if (launch_wait_consumed(c->p2p_flags, c->rank, c->nranks, c->epoch, lim,
                                 c->stream) == cudaSuccess)
            cudaStreamSynchronize(c->stream);
    }
    if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
    table_free(c->tdesc);
    table_free(c->tddesc);
    if (c->h_hdr) cudaFreeHost(c->h_hdr);
    if (c->d_hdr) cudaFree(c->d_hdr);
    for (auto &r : c->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : c->pool) cudaEventDestroy(e);
    if (c->d_sig) cudaFree(c->d_sig);
    if (c->d_k1cnt) cudaFree(c->d_k1cnt);
    if (c->aux) cudaStreamDestroy(c->aux);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->p2p_open.size()) cudaDeviceSynchronize();
    for (void *pm : c->p2p_open) cudaIpcCloseMemHandle(pm);
    if (c->p2p_msg) cudaFree(c->p2p_msg);
    if (c->p2p_flags) cudaFree(c->p2p_flags);
    if (c->p2p_stage) cudaFree(c->p2p_stage);
    if (c->d_peer_stage) cudaFree(c->d_peer_stage);
    if (c->d_peer_msg) cudaFree(c->d_peer_msg);
    if (c->d_peer_flags) cudaFree(c->d_peer_flags);
    if (c->d_stat) cudaFree(c->d_stat);
    if (c->d_tl) cudaFree(c->d_tl);
    if (c->h_stat) cudaFreeHost(c->h_stat);
    delete c;
    return RGC_OK;
}

const char *rgc_last_error(rgc_ctx_t c) { return c ? c->err.c_str() : "null context"; }

rgc_status_t rgc_sizes(rgc_ctx_t c, const rgc_layer_t *layers, int L, rgc_sizes_t *out) {
    if (!out) return fail(c, RGC_EINVAL, "null argument");
    Layout lo;
    rgc_status_t s = make_layout(c, layers, L, lo);
    if (s) return s;
    out->workspace_bytes = lo.ws_bytes;
    out->msg_bytes = lo.msg_bytes;
    out->gathered_bytes = lo.msg_bytes * (uint64_t)(c ? c->nranks : 1);
    out->header_bytes = 4ull * lo.H;
    out->k_total = lo.k_total;
    out->cap_total = lo.cap_total;
    return RGC_OK;
}

rgc_status_t rgc_workspace_init(rgc_ctx_t c, const rgc_layer_t *layers, int L, void *ws) {
    if (!c || !ws) return fail(c, RGC_EINVAL, "null argument");
    if (!aligned16(ws)) return fail(c, RGC_EINVAL, "workspace not 16-byte aligned");
    Layout lo;
    rgc_status_t s = make_layout(c, layers, L, lo);
    if (s) return s;
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaMemsetAsync(ws, 0, lo.ws_bytes, c->stream));
    if (c->tdesc.ws == ws) c->tdesc.ws = nullptr;
    if (c->tddesc.ws == ws) c->tddesc.ws = nullptr;
    return RGC_OK;
}

rgc_status_t rgc_compress(rgc_ctx_t c, const rgc_layer_t *layers, int L, const float *const *grad,
                          float *const *residual, float *const *momentum, void *msg, void *ws) {
    if (!c) return RGC_EINVAL;
    if (c->poisoned) return fail(c, RGC_ESTATE, "a cross-GPU wait timed out earlier: the context is unusable");
    if (!grad || !residual || !msg || !ws) return fail(c, RGC_EINVAL, "null argument");
    if (!aligned16(msg) || !aligned16(ws)) return fail(c, RGC_EINVAL, "msg/ws not 16-byte aligned");
    Nvtx nv("rgc_compress");
    Layout lo;
    rgc_status_t s = make_layout(c, layers, L, lo);
    if (s) return s;
    for (int l = 0; l < L; l++) {
        LayerDesc &d = lo.desc[l];
        if (!grad[l] || !residual[l] || !aligned16(grad[l]) || !aligned16(residual[l]))
            return fail(c, RGC_EINVAL, "layer %d: grad/residual null or not 16-byte aligned", l);
        d.g = grad[l];
        d.V = residual[l];
        d.u = nullptr;
        if (d.m != 0.0f) {
            if (!momentum || !momentum[l] || !aligned16(momentum[l]))
                return fail(c, RGC_EINVAL, "layer %d: momentum buffer required (m != 0), 16-byte aligned", l);
            d.u = momentum[l];
        }
    }
    // K1 grid and the candidate records each layer gets (one per K1 CTA covering it)
    // at least RGC_K1_MINTILES tiles per CTA (A/B knob; default 1): fewer, longer CTAs mean
    // fewer candidate records for K2 and K3A on small layer lists
    static const uint32_t k1_mintiles = [] { const char *e = getenv("RGC_K1_MINTILES");
                                             const int v = e ? atoi(e) : 1; return (uint32_t)(v < 1 ? 1 : v); }();
    int g1 = grid_of(c, c->occ1, (lo.TV + k1_mintiles - 1) / k1_mintiles);
    if (g1 > (int)kG2Max) g1 = (int)kG2Max;
    const int g2 = grid_of(c, c->occ2, lo.TV);
    uint32_t nrec = 0;
    {
        auto cta_of = [&](uint32_t t) {   // K1 CTA whose blocked range holds tile t
            uint32_t lo_b = 0, hi_b = (uint32_t)g1 - 1;
            while (lo_b < hi_b) {
                const uint32_t mid = (lo_b + hi_b + 1) / 2;
                if ((uint64_t)lo.TV * mid / (uint64_t)g1 <= t) lo_b = mid; else hi_b = mid - 1;
            }
            return lo_b;
        };
        uint32_t rb = 0;
        for (int l = 0; l < L; l++) {
            LayerDesc &d = lo.desc[l];
            const uint32_t b0 = cta_of(d.tile_begin), b1 = cta_of(d.tile_begin + d.ntiles - 1);
            d.cand_b0 = b0;
            d.cand_nb = b1 - b0 + 1;
            d.rec_base = rb;
            rb += d.cand_nb;
        }
        nrec = rb;
    }
    CUDA_TRY(c, cudaSetDevice(c->device));
    Ws w = ws_of(lo, ws);
    w.cand_R = (uint32_t)(lo.cand_total / (uint64_t)g1);
    {
        // K3A takes small candidate records (few tiles per K1 CTA, as on C1) in groups of
        // seg_ch, ~16 tiles a segment; RGC_K3A_SEGREC overrides
        static const int forced = [] { const char *e = getenv("RGC_K3A_SEGREC"); return e ? atoi(e) : 0; }();
        uint32_t sc = (uint32_t)((16ull * (uint64_t)g1 + lo.TV - 1) / lo.TV);
        if (forced > 0) sc = (uint32_t)forced;
        w.seg_ch = sc < 1 ? 1u : (sc > 64 ? 64u : sc);
    }
    w.k4_hint = c->h_stat_dev + 3;   // K2 reports this call's K4 work for the next call
    if (c->d_tl) {   // RGC_TIMELINE: a fresh timeline for this step (start = max, end = 0)
        w.tl = c->d_tl;
        c->fill.tl = c->d_tl;
        CUDA_TRY(c, cudaMemsetAsync(c->d_tl, 0xFF, kTlKernels * sizeof(unsigned long long), c->stream));
        CUDA_TRY(c, cudaMemsetAsync(c->d_tl + kTlKernels, 0, kTlKernels * sizeof(unsigned long long), c->stream));
    }
    int slot = 0;
    s = table_slot(c, c->tdesc, (uint8_t *)ws + kOffDesc, kDescBytes, ws, lo.desc.data(),
                   sizeof(LayerDesc) * L, &slot);
    if (s) return s;
    w.desc = (LayerDesc *)((uint8_t *)ws + kOffDesc + (uint64_t)slot * kDescBytes);
    static const bool sync_each = getenv("RGC_SYNC_EACH") != nullptr;
    // RGC_SYNC_EACH=1 (debugging): synchronise after every launch and name the kernel that failed
    int dbg_line = 0;
#define RGC_DBG_SYNC()                                                                        \
    do {                                                                                      \
        dbg_line = __LINE__;                                                                  \
        if (sync_each) {                                                                      \
            cudaError_t e_ = cudaStreamSynchronize(c->stream);                                \
            if (e_ != cudaSuccess)                                                            \
                return fail(c, RGC_ECUDA, "kernel launched before rgc_api.cu:%d failed: %s",  \
                            dbg_line, cudaGetErrorString(e_));                                \
        }                                                                                     \
    } while (0)
    uint32_t *hdr = (uint32_t *)msg;
    uint2 *pairs = (uint2 *)((uint8_t *)msg + 4ull * lo.H);
    cudaStream_t st = c->stream;
    {
        PhaseScope ps(c, 0);
        Ws w1 = w;
        if (c->pull_wait_epoch) {   // RGC_SYNC_PULL: peers may still be reading the block
            w1.pull_flags = c->p2p_flags;
            w1.pull_epoch = c->pull_wait_epoch;
            w1.pull_rank = c->rank;
            w1.pull_p = c->nranks;
            c->pull_wait_epoch = 0;
        }
        // The early fill depends only on the work before K1 and is enqueued right after it:
        // its CTAs (which cannot fit beside three K1 CTAs) take the SMs K1's CTAs leave during
        // K1's ramp-down (its CTAs end over a ~60-80 us spread) and start filling when
        // RGC_FILL_PCT % (90) of K1's CTAs have streamed their tiles: VGG16 0.620 -> 0.610 ms,
        // M1 0.454 -> 0.450; off for short ramp-downs (ResNet-50: +4 us)
        const int fa = fill_at();
        bool fill_early = c->fill_state == 1 && c->d_k1cnt &&
                          (fa == 0 || (fa < 0 && (uint64_t)lo.TV >= 32ull * (uint64_t)g1));
        if (fill_early) {
            // not under CUDA-graph capture: the wait targets count K1 launches, which a
            // replayed graph would not advance
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            CUDA_TRY(c, cudaStreamIsCapturing(st, &cs));
            fill_early = cs == cudaStreamCaptureStatusNone;
        }
        if (fill_early) {
            // and not when an output overlaps a buffer K1 reads or writes (include/rgc.h: out
            // may alias grad -- then only the fill after K1 is correct)
            const FillTable &ft = c->fill;
            for (int a = 0; a < ft.L && fill_early; a++) {
                const uintptr_t o0 = (uintptr_t)ft.out[a], o1 = o0 + 4ull * ft.n[a];
                for (int l = 0; l < L && fill_early; l++) {
                    const LayerDesc &d = lo.desc[l];
                    const void *bufs[3] = {d.g, d.V, d.u};
                    for (const void *b : bufs) {
                        if (!b) continue;
                        const uintptr_t b0 = (uintptr_t)b, b1 = b0 + 4ull * d.n;
                        if (o0 < b1 && b0 < o1) { fill_early = false; break; }
                    }
                }
            }
        }
        if (fill_early) {
            w1.k1cnt = c->d_k1cnt;
            CUDA_TRY(c, cudaEventRecord(c->ev_fork, c->stream));
        }
        CUDA_TRY(c, launch_k1(w1, L, lo.TV, hdr, g1, st));
        c->launches++;
        RGC_DBG_SYNC();
        if (fill_early) {
            // the early fill: the same table, armed with K1's counters (the regular fill is
            // still forked after K1 below and finishes what this one leaves)
            static const int pct = [] { const char *e = getenv("RGC_FILL_PCT"); const int v = e ? atoi(e) : 90;
                                        return v < 0 ? 0 : (v > 100 ? 100 : v); }();
            FillTable early = c->fill;
            early.k1cnt = c->d_k1cnt;
            early.start_target = c->k1cnt_total + (uint64_t)g1;
            early.wait_until = c->k1cnt_total + ((uint64_t)g1 * (uint64_t)pct + 99) / 100;
            c->k1cnt_total += (uint64_t)g1;
            CUDA_TRY(c, cudaStreamWaitEvent(c->aux, c->ev_fork, 0));
            CUDA_TRY(c, launch_k6_fill(early, c->d_sig, 2 * c->sms, c->aux));
            c->launches++;
        }
    }
    // rgc_decompress_prefill: the zero fill of the outputs is forked onto the auxiliary stream
    // after kernel `fill_after` of the chain (1: K1, 2: K2) -- it shares HBM with whatever
    // runs beside it (RGC_FILL_AT, A/B)
    const int fill_after = fill_at();   // 0: the regular fill also goes here, after the early one
    if (c->fill_state == 1 && fill_after <= 1) {
        s = fill_fork(c);
        if (s) return s;
    }

    {
        PhaseScope ps(c, 1);
        // stash pass (+ the V passes folded into it) or the two V-pass launches
        CUDA_TRY(c, launch_k2(w, L, lo.TV, lo.max_trim, hdr, lo.H, g2, nrec, c->sms * k2s_mult(), st,
                              &c->launches));
        RGC_DBG_SYNC();
    }
    if (c->fill_state == 1 && fill_after >= 2) {
        s = fill_fork(c);
        if (s) return s;
    }
    {
        PhaseScope ps(c, 2);
        CUDA_TRY(c, launch_k3(w, L, 0, pairs, grid_of(c, c->occ3, lo.TV), st));
        c->launches++;
        RGC_DBG_SYNC();
    }
    {
        PhaseScope ps(c, 3);
        CUDA_TRY(c, launch_k45(w, L, pairs, st, lo.k45_cl));
        c->launches++;
        RGC_DBG_SYNC();
        // the three radix passes: one cooperative launch (grid barriers between the passes)
        const bool k4_expected = ((volatile uint32_t *)c->h_stat)[3] != 0u;   // the last call's
        CUDA_TRY(c, launch_k4_all(w, L, hdr, c->sms, st, &c->launches, k4_expected));
        RGC_DBG_SYNC();
    }
    {
        PhaseScope ps(c, 4);
        CUDA_TRY(c, launch_k3(w, L, 1, pairs, grid_of(c, c->occ3, lo.TV), st));
        c->launches++;
        RGC_DBG_SYNC();
        if (lo.any_quant) {   // ASQ layers: indices + one mean into the message (K5)
            CUDA_TRY(c, launch_k5_asq(w, L, hdr, lo.H, grid_of(c, 4, lo.cap_total / 4096 + L), st));
            c->launches++;
            RGC_DBG_SYNC();
        }
    }
    if (c->nranks > 1 && tab_enabled()) {
        // the receivers' per-tile ranges of this message, once here instead of on every rank
        CUDA_TRY(c, launch_k_tab(w, L, hdr, lo.H, (uint32_t)(lo.tab_off / 4), (uint32_t)lo.cap_total,
                                 grid_of(c, 4, (lo.cap_total + lo.TD + L + kThreads - 1) / kThreads), st));
        c->launches++;
        RGC_DBG_SYNC();
    }
    table_used(c, c->tdesc, slot);
    c->ncompress++;
    c->prof_calls++;
    return RGC_OK;
}

rgc_status_t rgc_p2p_init(rgc_ctx_t c, const rgc_layer_t *layers, int L, void **msg_out) {
    if (!c || !msg_out) return RGC_EINVAL;
    if (c->p2p) return fail(c, RGC_ESTATE, "rgc_p2p_init already called on this context");
    if (c->nranks > kMaxP2P) return fail(c, RGC_EINVAL, "RGC_SYNC_P2P supports at most %d ranks", kMaxP2P);
    if (c->nranks > 1 && !c->comm) return fail(c, RGC_ESTATE, "context has no communicator (created without uid)");
    Layout lo;
    rgc_status_t s = make_layout(c, layers, L, lo);
    if (s) return s;
    CUDA_TRY(c, cudaSetDevice(c->device));
    const int p = c->nranks;
    std::vector<uint8_t *> hs(p, nullptr), hm(p, nullptr);
    std::vector<P2PFlags *> hf(p, nullptr);
    auto undo = [&]() {
        for (void *pm : c->p2p_open) cudaIpcCloseMemHandle(pm);
        c->p2p_open.clear();
        if (c->p2p_msg) cudaFree(c->p2p_msg);
        if (c->p2p_stage) cudaFree(c->p2p_stage);
        if (c->p2p_flags) cudaFree(c->p2p_flags);
        c->p2p_msg = nullptr; c->p2p_stage = nullptr; c->p2p_flags = nullptr;
    };
    // Collective and all-or-nothing: every rank takes part in both exchanges below whatever
    // happened locally, and all ranks fail together if any rank failed (a rank returning
    // early would leave its peers blocked in the exchange).
    std::string why;
    bool ok = cudaMalloc(&c->p2p_msg, lo.msg_bytes) == cudaSuccess &&
              cudaMalloc((void **)&c->p2p_stage, lo.msg_bytes * (uint64_t)p) == cudaSuccess &&
              cudaMalloc((void **)&c->p2p_flags, sizeof(P2PFlags)) == cudaSuccess &&
              cudaMemset(c->p2p_msg, 0, lo.msg_bytes) == cudaSuccess &&
              cudaMemset(c->p2p_stage, 0, lo.msg_bytes * (uint64_t)p) == cudaSuccess &&
              cudaMemset(c->p2p_flags, 0, sizeof(P2PFlags)) == cudaSuccess &&
              cudaMemcpy(&c->p2p_flags->timeout_ns, &c->timeout_ns, sizeof(unsigned long long),
                         cudaMemcpyHostToDevice) == cudaSuccess;
    if (!ok) { cudaGetLastError(); why = "allocation failed"; }
    hs[c->rank] = c->p2p_stage;
    hf[c->rank] = c->p2p_flags;
    hm[c->rank] = (uint8_t *)c->p2p_msg;
    // one byte per rank through the communicator: min over ranks (host-synchronous)
    auto all_ok = [&](bool mine, bool *all) -> bool {
        uint8_t *d1 = nullptr;
        std::vector<uint8_t> h1(p, 0);
        if (cudaMalloc(&d1, (size_t)p) != cudaSuccess) { cudaGetLastError(); return false; }
        const uint8_t v = mine ? 1 : 0;
        cudaMemcpy(d1 + c->rank, &v, 1, cudaMemcpyHostToDevice);
        ncclResult_t r = g_nccl.AllGather(d1 + c->rank, d1, 1, ncclUint8, c->comm, c->stream);
        cudaError_t ce = cudaStreamSynchronize(c->stream);
        if (r == 0 && ce == cudaSuccess) ce = cudaMemcpy(h1.data(), d1, (size_t)p, cudaMemcpyDeviceToHost);
        cudaFree(d1);
        if (r != 0 || ce != cudaSuccess) return false;
        *all = true;
        for (int q = 0; q < p; q++) *all = *all && h1[q] == 1;
        return true;
    };
    if (p > 1) {
        // exchange the three IPC handles of every rank plus an ok byte (one-time, host-synchronous)
        constexpr size_t HB = 3 * sizeof(cudaIpcMemHandle_t) + 16;
        std::vector<uint8_t> hh((size_t)p * HB, 0), mine(HB, 0);
        cudaIpcMemHandle_t h[3];
        if (ok && (cudaIpcGetMemHandle(&h[0], c->p2p_stage) != cudaSuccess ||
                   cudaIpcGetMemHandle(&h[1], c->p2p_flags) != cudaSuccess ||
                   cudaIpcGetMemHandle(&h[2], c->p2p_msg) != cudaSuccess)) {
            cudaGetLastError();
            ok = false;
            why = "cudaIpcGetMemHandle failed";
        }
        if (ok) memcpy(mine.data(), h, 3 * sizeof(cudaIpcMemHandle_t));
        mine[HB - 1] = ok ? 1 : 0;
        uint8_t *dh = nullptr;
        bool xok = cudaMalloc(&dh, (size_t)p * HB) == cudaSuccess;
        ncclResult_t r = 1;
        if (xok) {
            cudaMemcpy(dh + (size_t)c->rank * HB, mine.data(), HB, cudaMemcpyHostToDevice);
            r = g_nccl.AllGather(dh + (size_t)c->rank * HB, dh, HB, ncclUint8, c->comm, c->stream);
            cudaError_t ce = cudaStreamSynchronize(c->stream);
            if (r == 0 && ce == cudaSuccess) ce = cudaMemcpy(hh.data(), dh, (size_t)p * HB, cudaMemcpyDeviceToHost);
            xok = r == 0 && ce == cudaSuccess;
            cudaFree(dh);
        }
        if (!xok) {
            undo();
            return fail(c, RGC_ENCCL, "rgc_p2p_init: handle exchange failed");
        }
        bool all = true;
        for (int q = 0; q < p; q++) all = all && hh[(size_t)q * HB + HB - 1] == 1;
        if (!all) {
            undo();
            return fail(c, RGC_ECUDA, "rgc_p2p_init: a rank could not set up its areas%s%s",
                        why.empty() ? "" : " (here: ", why.empty() ? "" : (why + ")").c_str());
        }
        for (int q = 0; q < p && ok; q++) {
            if (q == c->rank) continue;
            cudaIpcMemHandle_t hq[3];
            memcpy(hq, hh.data() + (size_t)q * HB, 3 * sizeof(cudaIpcMemHandle_t));
            void *ptr[3] = {nullptr, nullptr, nullptr};
            for (int j = 0; j < 3 && ok; j++) {
                if (cudaIpcOpenMemHandle(&ptr[j], hq[j], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                    cudaGetLastError();
                    ok = false;
                    char b[128];
                    snprintf(b, sizeof b, "rank %d's memory is not mappable here (no P2P)", q);
                    why = b;
                } else {
                    c->p2p_open.push_back(ptr[j]);
                }
            }
            hs[q] = (uint8_t *)ptr[0];
            hf[q] = (P2PFlags *)ptr[1];
            hm[q] = (uint8_t *)ptr[2];
        }
        // every rank mapped every peer, or all ranks give up together
        bool all2 = false;
        if (!all_ok(ok, &all2)) {
            undo();
            return fail(c, RGC_ENCCL, "rgc_p2p_init: barrier failed");
        }
        if (!all2) {
            undo();
            return fail(c, RGC_ECUDA, "rgc_p2p_init: peer mappings failed on some rank%s%s",
                        why.empty() ? "" : " (here: ", why.empty() ? "" : (why + ")").c_str());
        }
    } else if (!ok) {
        undo();
        return fail(c, RGC_ECUDA, "rgc_p2p_init: %s", why.c_str());
    }
    ok = cudaMalloc((void **)&c->d_peer_stage, sizeof(void *) * p) == cudaSuccess &&
         cudaMalloc((void **)&c->d_peer_flags, sizeof(void *) * p) == cudaSuccess &&
         cudaMalloc((void **)&c->d_peer_msg, sizeof(void *) * p) == cudaSuccess &&
         cudaMemcpy(c->d_peer_stage, hs.data(), sizeof(void *) * p, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(c->d_peer_flags, hf.data(), sizeof(void *) * p, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(c->d_peer_msg, hm.data(), sizeof(void *) * p, cudaMemcpyHostToDevice) == cudaSuccess;
    if (!ok) cudaGetLastError();
    c->h_peer_msg = hm;
    // every rank's tables are in place before any rank pushes (and all ranks agree)
    if (p > 1) {
        bool all = false;
        if (!all_ok(ok, &all) || !all) {
            undo();
            return fail(c, RGC_ECUDA, "rgc_p2p_init: device tables could not be set up on some rank");
        }
    } else if (!ok) {
        undo();
        return fail(c, RGC_ECUDA, "rgc_p2p_init: device tables could not be set up");
    }
    c->p2p = true;
    c->p2p_bytes = lo.msg_bytes;
    c->epoch = 0;
    *msg_out = c->p2p_msg;
    return RGC_OK;
}

rgc_status_t rgc_p2p_gather(rgc_ctx_t c, const rgc_layer_t *layers, int L, void *gathered) {
    if (!c || !gathered) return RGC_EINVAL;
    if (!(c->p2p && c->p2p_synced))
        return fail(c, RGC_ESTATE, "rgc_p2p_gather is valid between an RGC_SYNC_P2P sync and rgc_decompress");
    Layout lo;
    rgc_status_t s = make_layout(c, layers, L, lo);
    if (s) return s;
    CUDA_TRY(c, cudaSetDevice(c->device));
    if (c->pull_synced) {
        // RGC_SYNC_PULL: every rank's own block, read over NVLink once the peers published it
        if (c->nranks > 1)
            CUDA_TRY(c, launch_pull_wait(c->p2p_flags, c->rank, c->nranks, c->epoch, c->stream));
        for (int r = 0; r < c->nranks; r++)
            CUDA_TRY(c, cudaMemcpyAsync((uint8_t *)gathered + (uint64_t)r * lo.msg_bytes, c->h_peer_msg[r],
                                        lo.msg_bytes, cudaMemcpyDeviceToDevice, c->stream));
        return RGC_OK;
    }
    // the staging area holds every rank's block (only the used part is defined)
    CUDA_TRY(c, cudaMemcpyAsync(gathered, c->p2p_stage, lo.msg_bytes * (uint64_t)c->nranks,
                                cudaMemcpyDeviceToDevice, c->stream));
    return RGC_OK;
}

rgc_status_t rgc_sync_plan(const uint32_t *headers, int nranks, int L, uint32_t header_words,
                           uint64_t msg_bytes, uint64_t *bytes_out, uint32_t *counts_out,
                           uint32_t *status_out) {
    if (!headers || nranks < 1 || L < 1 || header_words < (uint32_t)(2 * L + 2)) return RGC_EINVAL;
    uint32_t status = 0;
    for (int r = 0; r < nranks; r++) {
        const uint32_t *h = headers + (size_t)r * header_words;
        if (h[L + 1] != (uint32_t)L) return RGC_ESTATE;
        uint64_t tot = 0;
        for (int l = 0; l < L; l++) {
            tot += (h[L + 2 + l] == RGC_MSG_DENSE ? 8ull : 4ull) * h[l];   // pair / ASQ index
            if (counts_out) counts_out[(size_t)r * L + l] = h[l];
        }
        status |= h[L];
        const uint64_t b = 4ull * header_words + tot;
        if (b > msg_bytes) return RGC_ESTATE;
        if (bytes_out) bytes_out[r] = b;
    }
    if (status_out) *status_out = status;
    return RGC_OK;
}

rgc_status_t rgc_sync(rgc_ctx_t c, const rgc_layer_t *layers, int L, const void *msg,
                      void *gathered, int mode, uint32_t *counts_host) {
    if (!c) return RGC_EINVAL;
    if (c->poisoned) return fail(c, RGC_ESTATE, "a cross-GPU wait timed out earlier: the context is unusable");
    Nvtx nv("rgc_sync");
    if (mode == RGC_SYNC_PULL) {
        // no data moves here: publish "epoch e is complete in my block" to every peer; the
        // peers' decompression reads the block in place over NVLink
        if (!c->p2p) return fail(c, RGC_ESTATE, "RGC_SYNC_PULL needs rgc_p2p_init first");
        if (msg != c->p2p_msg) return fail(c, RGC_EINVAL, "RGC_SYNC_PULL: msg must be the rgc_p2p_init block");
        Layout lo;
        rgc_status_t s = make_layout(c, layers, L, lo);
        if (s) return s;
        if (lo.msg_bytes != c->p2p_bytes) return fail(c, RGC_EINVAL, "layers differ from rgc_p2p_init's");
        CUDA_TRY(c, cudaSetDevice(c->device));
        PhaseScope ps(c, 5);
        c->epoch++;
        if (c->nranks > 1) {
            CUDA_TRY(c, launch_pull_publish(c->d_peer_flags, c->rank, c->nranks, c->epoch, c->stream));
            c->launches++;
            c->pull_wait_epoch = c->epoch;   // the next compress must not rewrite the block early
        }
        c->p2p_synced = true;
        c->pull_synced = true;
        return RGC_OK;
    }
    if (mode == RGC_SYNC_P2P) {
        // exact-size push of this rank's block into every rank's staging area (NVLink
        // stores), then "ready" flags: one kernel, no host round trip
        if (!c->p2p) return fail(c, RGC_ESTATE, "RGC_SYNC_P2P needs rgc_p2p_init first");
        if (msg != c->p2p_msg) return fail(c, RGC_EINVAL, "RGC_SYNC_P2P: msg must be the rgc_p2p_init block");
        Layout lo;
        rgc_status_t s = make_layout(c, layers, L, lo);
        if (s) return s;
        if (lo.msg_bytes != c->p2p_bytes) return fail(c, RGC_EINVAL, "layers differ from rgc_p2p_init's");
        CUDA_TRY(c, cudaSetDevice(c->device));
        PhaseScope ps(c, 5);
        c->epoch++;
        static const int nb_max = getenv("RGC_P2P_NB") ? atoi(getenv("RGC_P2P_NB")) : 64;
        const int nb = (int)std::max<uint64_t>(1, std::min<uint64_t>(nb_max, (lo.msg_bytes + 16383) / 16384));
        CUDA_TRY(c, launch_p2p_push((const uint8_t *)msg, c->d_peer_stage, c->d_peer_flags, c->p2p_flags,
                                    c->rank, c->nranks, c->epoch, lo.msg_bytes, L, lo.H, nb, c->stream,
                                    lo.tab_off, tab_enabled() ? 4ull * lo.tab_words : 0ull));
        c->launches++;
        c->p2p_synced = true;
        c->pull_synced = false;
        return RGC_OK;
    }
    if (!msg || !gathered) return fail(c, RGC_EINVAL, "null argument");
    if (mode != RGC_SYNC_FIXED && mode != RGC_SYNC_SIZES_FIRST)
        return fail(c, RGC_EINVAL, "sync mode %d invalid", mode);
    if (!aligned16(msg) || !aligned16(gathered)) return fail(c, RGC_EINVAL, "buffers not 16-byte aligned");
    Layout lo;
    rgc_status_t s = make_layout(c, layers, L, lo);
    if (s) return s;
    CUDA_TRY(c, cudaSetDevice(c->device));
    const int p = c->nranks;
    const uint64_t stride = lo.msg_bytes;
    const uint64_t hb = 4ull * lo.H;
    PhaseScope ps(c, 5);
    if (mode == RGC_SYNC_FIXED) {
        if (p == 1) {
            if (gathered != msg)
                CUDA_TRY(c, cudaMemcpyAsync(gathered, msg, stride, cudaMemcpyDeviceToDevice, c->stream));
        } else {
            if (!c->comm) return fail(c, RGC_ESTATE, "context has no communicator (created without uid)");
            ncclResult_t r = g_nccl.AllGather(msg, gathered, stride, ncclUint8, c->comm, c->stream);
            if (r != 0) return fail(c, RGC_ENCCL, "ncclAllGather: %s", g_nccl.GetErrorString(r));
            ncclResult_t ae = 0;
            g_nccl.CommGetAsyncError(c->comm, &ae);
            if (ae != 0 && ae != 7 /* ncclInProgress */) {
                c->nccl_err = (uint32_t)ae;
                return fail(c, RGC_ENCCL, "NCCL async error: %s", g_nccl.GetErrorString(ae));
            }
        }
        return RGC_OK;
    }
    // SIZES_FIRST: the length elements first, then exact-size payloads
    const size_t need = hb * (size_t)p;
    if (c->h_hdr_bytes < need) {
        if (c->h_hdr) cudaFreeHost(c->h_hdr);
        c->h_hdr = nullptr; c->h_hdr_bytes = 0;
        CUDA_TRY(c, cudaMallocHost((void **)&c->h_hdr, need));
        c->h_hdr_bytes = need;
    }
    if (p == 1) {
        CUDA_TRY(c, cudaMemcpyAsync(c->h_hdr, msg, hb, cudaMemcpyDeviceToHost, c->stream));
    } else {
        if (!c->comm) return fail(c, RGC_ESTATE, "context has no communicator (created without uid)");
        if (c->d_hdr_bytes < need) {
            if (c->d_hdr) cudaFree(c->d_hdr);
            c->d_hdr = nullptr; c->d_hdr_bytes = 0;
            CUDA_TRY(c, cudaMalloc(&c->d_hdr, need));
            c->d_hdr_bytes = need;
        }
        ncclResult_t r = g_nccl.AllGather(msg, c->d_hdr, hb, ncclUint8, c->comm, c->stream);
        if (r != 0) return fail(c, RGC_ENCCL, "ncclAllGather(sizes): %s", g_nccl.GetErrorString(r));
        CUDA_TRY(c, cudaMemcpyAsync(c->h_hdr, c->d_hdr, need, cudaMemcpyDeviceToHost, c->stream));
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    uint32_t status = 0;
    std::vector<uint64_t> bytes(p);
    s = rgc_sync_plan(c->h_hdr, p, L, lo.H, stride, bytes.data(), counts_host, &status);
    if (s) return fail(c, s, "gathered headers are inconsistent (message exceeds capacity)");
    if (p == 1) {
        if (gathered != msg)
            CUDA_TRY(c, cudaMemcpyAsync(gathered, msg, bytes[0], cudaMemcpyDeviceToDevice, c->stream));
    } else {
        const uint64_t tb = tab_enabled() ? 4ull * lo.tab_words : 0ull;   // range tables
        g_nccl.GroupStart();
        for (int r = 0; r < p; r++) {
            ncclResult_t e = g_nccl.Broadcast(msg, (uint8_t *)gathered + (uint64_t)r * stride, bytes[r],
                                              ncclUint8, r, c->comm, c->stream);
            if (e == 0 && tb)
                e = g_nccl.Broadcast((const uint8_t *)msg + lo.tab_off,
                                     (uint8_t *)gathered + (uint64_t)r * stride + lo.tab_off, tb,
                                     ncclUint8, r, c->comm, c->stream);
            if (e != 0) { g_nccl.GroupEnd(); return fail(c, RGC_ENCCL, "ncclBroadcast: %s", g_nccl.GetErrorString(e)); }
        }
        ncclResult_t e = g_nccl.GroupEnd();
        if (e != 0) return fail(c, RGC_ENCCL, "ncclGroupEnd: %s", g_nccl.GetErrorString(e));
        ncclResult_t ae = 0;
        g_nccl.CommGetAsyncError(c->comm, &ae);
        if (ae != 0 && ae != 7 /* ncclInProgress */) {
            c->nccl_err = (uint32_t)ae;
            return fail(c, RGC_ENCCL, "NCCL async error: %s", g_nccl.GetErrorString(ae));
        }
    }
    if (status & RGC_F_NONFINITE) return fail(c, RGC_ENONFINITE, "a rank reported a non-finite residual");
    return RGC_OK;
}

rgc_status_t rgc_decompress(rgc_ctx_t c, const rgc_layer_t *layers, int L, const void *gathered,
                            float *const *out, int ordered, void *ws) {
    if (!c) return RGC_EINVAL;
    if (c->poisoned) return fail(c, RGC_ESTATE, "a cross-GPU wait timed out earlier: the context is unusable");
    if (!out || !ws) return fail(c, RGC_EINVAL, "null argument");
    Nvtx nv("rgc_decompress");
    const bool p2p = gathered == nullptr;   // RGC_SYNC_P2P: read every rank's own block
    if (p2p && !(c->p2p && c->p2p_synced))
        return fail(c, RGC_EINVAL, "gathered is NULL but no RGC_SYNC_P2P sync precedes this call");
    Layout lo;
    rgc_status_t s = make_layout(c, layers, L, lo);
    if (s) return s;
    for (int l = 0; l < L; l++) {
        if (!out[l] || !aligned16(out[l]))
            return fail(c, RGC_EINVAL, "layer %d: out null or not 16-byte aligned", l);
        lo.ddesc[l].out = out[l];
    }
    CUDA_TRY(c, cudaSetDevice(c->device));
    bool prefilled = false;
    if (c->fill_state == 1) {   // registered, no compress in between: fill now (no overlap)
        s = fill_fork(c);
        if (s) return s;
    }
    if (c->fill_state == 2) {   // join the zero fill forked by rgc_compress
        CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_join, 0));
        prefilled = c->fill.L == L;
        for (int l = 0; l < L && prefilled; l++)
            prefilled = c->fill.out[l] == out[l] && c->fill.n[l] == lo.ddesc[l].n;
    }
    c->fill_state = 0;
    Ws w = ws_of(lo, ws);
    w.tl = c->d_tl;
    int slot = 0;
    s = table_slot(c, c->tddesc, (uint8_t *)ws + kOffDdesc, kDdescBytes, ws, lo.ddesc.data(),
                   sizeof(DecompDesc) * L, &slot);
    if (s) return s;
    w.ddesc = (DecompDesc *)((uint8_t *)ws + kOffDdesc + (uint64_t)slot * kDdescBytes);
    const int p = c->nranks;
    const float scale = 1.0f / (float)p;   // R13: fl32(1/p)
    MsgSrc src;
    src.base = p2p ? c->p2p_stage : (const uint8_t *)gathered;   // P2P: pushed by the peers
    src.stride = lo.msg_bytes;
    src.tab = nullptr;
    const bool pull = p2p && c->pull_synced;
    PhaseScope ps(c, 6);
    if (pull) {
        // RGC_SYNC_PULL: the kernels below read every peer's block in place over NVLink
        src.tab = c->d_peer_msg;
        if (p > 1) {
            CUDA_TRY(c, launch_pull_wait(c->p2p_flags, c->rank, p, c->epoch, c->stream));
            c->launches++;
        }
    }
    // blocks exchanged by rgc_sync between multi-rank contexts carry their producer's range
    // table (k_tab); externally gathered blocks of nranks = 1 producers (a context without a
    // communicator) do not, and k6_prep derives the ranges instead
    const bool use_tab = p > 1 && (c->comm != nullptr || p2p || c->assume_tab) && tab_enabled();
    bool read_tab = false;
    if (prefilled) {
        // the outputs are +0: write only the indices some rank sent (rgc_decomp.cu)
        if (ordered && p > 1) {
            if (!use_tab) {
                uint64_t prep_work = (uint64_t)p * ((uint64_t)lo.cap_total > (lo.TD + L) ? lo.cap_total : (lo.TD + L));
                CUDA_TRY(c, launch_k6_prep(w, L, p, src, lo.H, lo.TD,
                                           grid_of(c, 8, (prep_work + kThreads - 1) / kThreads), c->stream,
                                           (uint32_t)lo.cap_total));
                c->launches++;
            }
            read_tab = use_tab;
            c->launches++;
            CUDA_TRY(c, launch_k6_scatter(w, L, p, src, lo.H, lo.TD, (uint32_t)lo.cap_total, scale,
                                          grid_of(c, 8, (lo.TD + kWarps - 1) / kWarps), c->stream,
                                          use_tab ? (uint32_t)(lo.tab_off / 4) : 0u));
        } else if (ordered) {
            c->launches++;
            CUDA_TRY(c, launch_k6_scatter(w, L, p, src, lo.H, lo.TD, (uint32_t)lo.cap_total, scale,
                                          grid_of(c, 8, (lo.TD + kWarps - 1) / kWarps), c->stream, 0u));
        } else {
            CUDA_TRY(c, launch_k6_atomic_only(w, L, p, src, lo.H, (uint32_t)lo.cap_total, scale,
                                              grid_of(c, c->occ6, lo.TD), c->stream));
            c->launches++;
        }
    } else if (ordered) {
        uint64_t prep_work = (uint64_t)p * ((uint64_t)lo.cap_total > (lo.TD + L) ? lo.cap_total : (lo.TD + L));
        CUDA_TRY(c, launch_k6_prep(w, L, p, src, lo.H, lo.TD,
                                   grid_of(c, 8, (prep_work + kThreads - 1) / kThreads), c->stream,
                                   (uint32_t)lo.cap_total));
        c->launches++;
        CUDA_TRY(c, launch_k6(w, L, p, src, lo.H, lo.TD, scale, grid_of(c, c->occ6, lo.TD), c->stream));
        c->launches++;
    } else {
        CUDA_TRY(c, launch_k6_atomic(w, L, p, src, lo.H, lo.TD, (uint32_t)lo.cap_total, scale,
                                     grid_of(c, c->occ6, lo.TD), c->stream));
        c->launches += 2;
    }
    // every rank's status word (non-finite residuals) and the P2P timeout mask -> the context
    // status (rgc_status); P2P / PULL at p > 1: then this rank's staging slots (P2P) / its
    // reads of the peers' blocks (PULL) of epoch e are done -> consumed[rank] = e
    CUDA_TRY(c, launch_finish(src, L, p, p2p ? c->p2p_flags : nullptr, c->d_peer_flags, c->rank,
                              c->epoch, (p2p && p > 1) ? 1 : 0, c->d_stat, c->h_stat_dev,
                              c->stream, read_tab ? 1 : 0));
    c->launches++;
    if (p2p) {
        c->p2p_synced = false;
        c->pull_synced = false;
    }
    table_used(c, c->tddesc, slot);
    return RGC_OK;
}

rgc_status_t rgc_decompress_prefill(rgc_ctx_t c, const rgc_layer_t *layers, int L,
                                    float *const *out) {
    if (!c) return RGC_EINVAL;
    if (!out) return fail(c, RGC_EINVAL, "null argument");
    if (c->fill_state == 2)
        return fail(c, RGC_ESTATE, "a prefill is already enqueued: call rgc_decompress first");
    Layout lo;
    rgc_status_t s = make_layout(c, layers, L, lo);
    if (s) return s;
    FillTable &t = c->fill;
    t.L = L;
    t.k1cnt = nullptr;   // rgc_compress arms the wait (RGC_FILL_AT=0)
    uint32_t ch = 0;
    for (int l = 0; l < L; l++) {
        if (!out[l] || !aligned16(out[l]))
            return fail(c, RGC_EINVAL, "layer %d: out null or not 16-byte aligned", l);
        t.out[l] = out[l];
        t.n[l] = lo.ddesc[l].n;
        t.chunk_begin[l] = ch;
        ch += (uint32_t)((4ull * t.n[l] + 65535) / 65536);
    }
    t.chunk_begin[L] = ch;
    {
        static const uint32_t stride = [] { const char *e = getenv("RGC_FILL_STRIDE");
                                            const int v = e ? atoi(e) : 1; return (uint32_t)(v < 1 ? 1 : v); }();
        static const uint32_t inflight = [] { const char *e = getenv("RGC_FILL_INFLIGHT");
                                              return (uint32_t)(e ? atoi(e) : 0); }();
        t.sm_stride = stride;
        t.inflight = inflight;
    }
    CUDA_TRY(c, cudaSetDevice(c->device));
    if (!c->aux) {
        // highest priority: when K1 completes, the block scheduler places the fill's
        // CTAs (one per SM) before the selection kernels queued behind K1; at equal
        // priority they end up packed onto the few SMs the selection leaves free
        int lo_pr = 0, hi_pr = 0;
        CUDA_TRY(c, cudaDeviceGetStreamPriorityRange(&lo_pr, &hi_pr));
        CUDA_TRY(c, cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, hi_pr));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
        CUDA_TRY(c, cudaMalloc((void **)&c->d_sig, kFillSigWords * sizeof(unsigned int)));
        CUDA_TRY(c, cudaMemset(c->d_sig, 0, kFillSigWords * sizeof(unsigned int)));
        CUDA_TRY(c, cudaMalloc((void **)&c->d_k1cnt, 2 * sizeof(unsigned long long)));
        CUDA_TRY(c, cudaMemset(c->d_k1cnt, 0, 2 * sizeof(unsigned long long)));
        c->k1cnt_total = 0;
    }
    c->fill_state = 1;
    return RGC_OK;
}

rgc_status_t rgc_get_info(rgc_ctx_t c, int L, const void *ws, rgc_info_t *out) {
    if (!c || !ws || !out || L < 1 || L > RGC_MAX_LAYERS) return fail(c, RGC_EINVAL, "bad argument");
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    // LayerState sits after Ctrl | desc slots | ddesc slots (independent of the layer list)
    const uint64_t o = kOffState;
    std::vector<LayerState> st(L);
    CUDA_TRY(c, cudaMemcpy(st.data(), (const uint8_t *)ws + o, sizeof(LayerState) * L,
                           cudaMemcpyDeviceToHost));
    for (int l = 0; l < L; l++) {
        out[l] = st[l].info;
        const uint32_t mode = st[l].mode;
        out[l].emitted = mode == MODE_THRESH ? st[l].emitted_a
                         : (mode == MODE_SURV || mode == MODE_EXACT) ? st[l].emitted_b : 0;
    }
    return RGC_OK;
}

rgc_status_t rgc_debug_layer(rgc_ctx_t c, const void *ws, int l, uint32_t *out, int nout) {
    if (!c || !ws || !out || nout < 20 || l < 0 || l >= RGC_MAX_LAYERS)
        return fail(c, RGC_EINVAL, "bad argument");
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    LayerState st;
    CUDA_TRY(c, cudaMemcpy(&st, (const uint8_t *)ws + kOffState + sizeof(LayerState) * (uint64_t)l,
                           sizeof st, cudaMemcpyDeviceToHost));
    const uint32_t v[20] = {st.mode, st.count, st.thr_key, st.cand_key, st.stash_shift, st.stash_on,
                            st.stash_ok, st.k2src, st.cand_ok, st.need_full, st.jhint, st.margin,
                            st.phase, st.surv, st.emitted_a, st.emitted_b, st.cand_total, st.need_cnt, st.vpass_runs, st.full_runs};
    memcpy(out, v, sizeof v);
    return RGC_OK;
}

rgc_status_t rgc_check(rgc_ctx_t c, const void *msg, int L, uint32_t *status_out) {
    if (!c || !msg || !status_out || L < 1 || L > RGC_MAX_LAYERS) return fail(c, RGC_EINVAL, "bad argument");
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    uint32_t v = 0;
    CUDA_TRY(c, cudaMemcpy(&v, (const uint32_t *)msg + L, 4, cudaMemcpyDeviceToHost));
    *status_out = v;
    if (c->p2p) {
        unsigned long long e = 0;
        CUDA_TRY(c, cudaMemcpy(&e, &c->p2p_flags->err, 8, cudaMemcpyDeviceToHost));
        if (e) return fail(c, RGC_ESTATE, "RGC_SYNC_P2P: a wait for peers timed out (ranks mask %llx)", e);
    }
    return (v & RGC_F_NONFINITE) ? fail(c, RGC_ENONFINITE, "non-finite residual") : RGC_OK;
}

rgc_status_t rgc_status(rgc_ctx_t c, int flags, uint32_t *status_out) {
    if (!c) return RGC_EINVAL;
    if (flags & ~(RGC_STATUS_WAIT | RGC_STATUS_CLEAR)) return fail(c, RGC_EINVAL, "bad flags");
    CUDA_TRY(c, cudaSetDevice(c->device));
    if (flags & (RGC_STATUS_WAIT | RGC_STATUS_CLEAR)) CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    volatile uint32_t *h = c->h_stat;
    const uint32_t w0 = h[0], w1 = h[1], w2 = h[2];
    if (status_out) {
        status_out[0] = w0;
        status_out[1] = w1;
        status_out[2] = w2;
        status_out[3] = c->nccl_err;
    }
    rgc_status_t rc = RGC_OK;
    if (w0 & kStatTimeout) {
        c->poisoned = true;
        rc = fail(c, RGC_ESTATE, "a cross-GPU wait for peers timed out (ranks mask %08x%08x): "
                                 "the exchange epochs are out of step, the context is unusable",
                  w2, w1);
    } else if (w0 & kStatBarrier) {
        rc = fail(c, RGC_ESTATE, "a grid barrier of the radix select timed out (its CTAs were not "
                                 "co-resident); that step's selection is not valid");
    } else if (w0 & kStatNoTable) {
        rc = fail(c, RGC_ESTATE, "a rank's message block lacks its range table (decompress blocks "
                                 "of nranks = 1 producers with a context without a communicator)");
    } else if (c->nccl_err) {
        rc = fail(c, RGC_ENCCL, "NCCL async error: %s", g_nccl.GetErrorString
                                                           ? g_nccl.GetErrorString((ncclResult_t)c->nccl_err)
                                                           : "?");
    } else if (w0 & RGC_F_NONFINITE) {
        rc = fail(c, RGC_ENONFINITE, "a rank sent a message with a non-finite residual "
                                     "(that layer's set was empty)");
    }
    if ((flags & RGC_STATUS_CLEAR) && !(w0 & kStatTimeout)) {
        // the non-finite report is per step: clear it (a timeout stays: the context is poisoned)
        CUDA_TRY(c, cudaMemset(c->d_stat, 0, kStatWords * sizeof(uint32_t)));
        h[0] = 0; h[1] = 0; h[2] = 0;
    }
    return rc;
}

rgc_status_t rgc_profile(rgc_ctx_t c, int enable) {
    if (!c) return RGC_EINVAL;
    c->prof = enable >= 2 ? 2 : (enable != 0 ? 1 : 0);
    c->prof_every = enable >= 2 ? enable - 1 : 1;
    c->prof_calls = 0;
    return RGC_OK;
}

rgc_status_t rgc_profile_read(rgc_ctx_t c, float *ms, int nphase, int *n_out) {
    if (!c || !ms || nphase < kPhaseCount) return fail(c, RGC_EINVAL, "bad argument");
    CUDA_TRY(c, cudaSetDevice(c->device));
    for (auto &r : c->recs) {
        float t = 0.f;
        CUDA_TRY(c, cudaEventSynchronize(r.b));
        CUDA_TRY(c, cudaEventElapsedTime(&t, r.a, r.b));
        c->acc[r.phase] += t;
        c->pool.push_back(r.a);
        c->pool.push_back(r.b);
    }
    c->recs.clear();
    for (int i = 0; i < kPhaseCount; i++) { ms[i] = (float)c->acc[i]; c->acc[i] = 0.0; }
    if (n_out) *n_out = c->ncompress;
    c->ncompress = 0;
    return RGC_OK;
}

uint64_t rgc_launch_count(rgc_ctx_t c) { return c ? c->launches : 0; }

rgc_status_t rgc_debug_timeline(rgc_ctx_t c, uint64_t *out, int n) {
    if (!c || !out || n < 2 * kTlKernels) return fail(c, RGC_EINVAL, "bad argument");
    if (!c->d_tl) return fail(c, RGC_ESTATE, "the context was created without RGC_TIMELINE=1");
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->aux) CUDA_TRY(c, cudaStreamSynchronize(c->aux));
    CUDA_TRY(c, cudaMemcpy(out, c->d_tl, 2 * kTlKernels * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return RGC_OK;
}

}  // extern "C"
