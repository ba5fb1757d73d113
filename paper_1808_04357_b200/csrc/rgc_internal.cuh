// rgc_internal.cuh -- device-side data layout shared by the kernels and the
// host API of librgc.so (never exported, never seen by the oracle).
//
// Workspace (caller-owned device memory, rgc_sizes().workspace_bytes):
//   Ctrl | LayerDesc[RGC_MAX_LAYERS] | DecompDesc[RGC_MAX_LAYERS] |
//   LayerState[L] | statusA[TV] | statusB[TV] | S pairs[sum s_cap] |
//   dec_start[nranks][TD + L]
// TV = total 4096-element tiles over the layers; TD = total 8192-element
// decompress tiles.  Every accumulator is reset by the kernel that consumes it,
// so the workspace stays valid from call to call after rgc_workspace_init.
#pragma once
#include <stdint.h>
#include "../../include/rgc.h"

namespace rgc {

constexpr int kTile = RGC_TILE;            // 4096 elements (= mean_fx tile, R2)
constexpr int kThreads = 256;              // threads per CTA for the streaming kernels
constexpr int kPerThread = kTile / kThreads;  // 16
constexpr int kWarps = kThreads / 32;      // 8
constexpr int kMeanBins = 277;             // tile exponents -149..127
constexpr int kBsLevels = 1024;            // eps >= 2^-10 -> every ratio is j/1024 (R8)
constexpr int kBsTable = kBsLevels + 2;    // keys t_0..t_1024 + sentinel
constexpr int kRadixBins = 2048;
constexpr int kDecTile = 8192;             // decompress tile (elements)
constexpr int kMaxTrim = RGC_MAX_TRIM_LEVELS;
constexpr int kSegTiles = 16;                  // K3 work unit: 16 tiles
constexpr uint32_t kSeg = kSegTiles * kTile;   // = 65536 elements
constexpr uint32_t kSegB = 8192;              // K3 pass B segment (exact emission: more CTAs)
#ifndef RGC_K3A_SEG
#define RGC_K3A_SEG 65536
#endif
constexpr uint32_t kSegA = RGC_K3A_SEG;        // K3 pass A segment over V
constexpr int kStash = 4096;                   // K3 shared-memory stash (pairs, 32 KB)
constexpr int kK1Stash = 256;                  // K1 warp-private candidate staging (pairs)
constexpr int kK1Batch = 8;                    // K1 tiles per staging drain
#ifndef RGC_SMALLSEL
#define RGC_SMALLSEL 180224
#endif
constexpr int kSmallSel = RGC_SMALLSEL;
constexpr int kKeysPerCta45 = kSmallSel / 4;   // K45 keys per CTA (176 KB of shared memory)
// K45: candidate sets up to kSmallSel take one cluster per layer (RGC_K45_CL CTAs)

enum Mode : uint32_t { MODE_NONE = 0, MODE_THRESH = 1, MODE_SURV = 2, MODE_EXACT = 3 };

// per-layer constants (device table written by the host when it changes)
struct LayerDesc {
    const float *g;
    float *u;            // nullptr when m == 0
    float *V;
    uint32_t n, k, tile_begin, ntiles;
    uint32_t cap;        // message capacity (pairs) -> capacity fallback (R18)
    uint32_t s_cap;      // Alg.2 survivor capacity (pairs), 0 for BS layers
    uint64_t s_off;      // survivor buffer offset (pairs)
    float m;
    uint32_t selector;
    uint32_t branch;
    uint32_t trim_levels;
    uint32_t interval;     // sampled BS search interval
    uint32_t cand_b0;      // first K1 CTA whose tile range covers this layer
    uint32_t cand_nb;      // number of K1 CTAs covering it (= candidate records)
    uint32_t rec_base;     // first candidate record of this layer
    uint32_t quant;        // ASQ layer: selection on the signed view, mean message
    uint32_t pad_q;
    uint64_t q_off;        // ASQ: the layer's emission scratch in Ws::Q (pairs)
    double trim_eps;
    double bs_eps;
};

struct DecompDesc {
    float *out;
    uint32_t n;
    uint32_t tile_begin;   // first 8192-element tile
    uint32_t ntiles;
    uint32_t slot_begin;   // tile_begin + layer index (room for the per-layer sentinel)
    uint32_t quant;        // ASQ layer: the message holds indices + one value (hdr[L+2+l])
};

// Per-layer state, in two parts.  LayerHot: what the per-layer finalisations (K1, K2) read and
// decide -- they copy it into shared memory in one parallel load, decide from there and write
// it back in one parallel store (a thread walking it in global memory paid one dependent L2
// round trip per field: 6-23 us per finalisation).  Nothing else writes a layer's LayerHot
// while its finalisation runs.  LayerState adds the accumulators other CTAs add into.
struct alignas(16) LayerHot {
    // ---- per-call results ----
    double mean;
    unsigned int maxkey, flags, mode, thr_key;
    unsigned int count, surv, msg_off, pad0;
    unsigned int rs_prefix, rs_krem, rs_above, rs_src;   // radix select state
    unsigned int k3a_begin, k3a_tiles, k3b_begin, k3b_tiles;
    unsigned int k4_begin, k4_tiles, emitted_a, emitted_b;  // pairs written by K3 A / B
    // sampled threshold BS state (persists across calls; reset by rgc_workspace_init)
    unsigned int step, cache_valid, cache_key, reuse_cnt, small, need_cnt, pad1, pad2;
    // Alg.3 bounded histogram: hint (previous chosen threshold index), margin, fallback flag
    unsigned int jhint, margin, need_full, full_runs;   // full_runs: pass-1 re-counts (diagnostics)
    // Alg.3 bounded histogram of this call: levels j >= jlo_cur are counted exactly (K1)
    unsigned int jlo_cur, rs_two, rs_base, pad9;   // rs_*: K4 two-digit select over survivors
    // K1 candidate stash {|V| > tau}, tau = cand_key predicted by the previous call;
    // serves K2 (k2src) and K3's first pass (cand_ok) in place of reading V again
    unsigned int cand_key, cand_ok, stash_on, pad3;
    unsigned int stash_ok, k2src, stash_shift, cand_total;   // cand_total: stash records (diagnostics)
    unsigned int tkeys[kBsTable];         // threshold keys (Alg.3 table / Alg.2 levels)
    // ASQ (R21): phase of this call (0 positive, 1 negative; flipped by K5 at the end of
    // the call) and the selection key of the call: skey(b) = ((b ^ skx) & ska) ? 0 : |b|
    unsigned int phase, skx, ska, pad4;
    // the other phase's prediction state (Alg.3 hint/margin, stash key/shift/on): the two
    // signs have different histories, so K5 swaps these with the live ones at each flip
    unsigned int alt_jhint, alt_margin, alt_cand_key, alt_shift, alt_stash_on, vpass_runs, pad8[2];
    rgc_info_t info;
};
static_assert(sizeof(LayerHot) % 16 == 0, "LayerHot moves as uint4");

struct alignas(16) LayerState : LayerHot {
    // ---- accumulators (reset by their consumer) ----
    unsigned long long bins[kMeanBins + 3];
    unsigned int maxkey_acc;
    unsigned int k1_done, k2_done, k4_done;
    unsigned int trim_cnt[kMaxTrim];
    unsigned int hist[kRadixBins];        // K2 Alg.3 histogram (1026 bins) / K4 radix digits
    unsigned int k1_cnt, cand_acc, cand_bad, qdone;
    unsigned long long qbins[256];        // R22: significand sums per biased exponent
};

struct alignas(16) Ctrl {
    unsigned int layers_done;
    unsigned int k3a_total, k3b_total, k4_total;
    unsigned int ticketA, ticketB;
    unsigned int status;
    unsigned int any_full;
    unsigned int any_vpass;     // some layer needs K2's V pass this call
    unsigned int dense_pairs;   // pairs of the plain layers this call (ASQ indices follow them)
    unsigned int bar_count, bar_gen;   // grid barrier of the one-launch K4 (three digit passes)
    unsigned int pad[52];
};
static_assert(sizeof(Ctrl) == 256, "Ctrl must be 256 bytes");

struct P2PFlags;
struct Ws {
    Ctrl *ctrl;
    LayerDesc *desc;
    DecompDesc *ddesc;
    LayerState *st;
    unsigned long long *statusA, *statusB;
    uint2 *S;
    uint32_t *dec_start;
    uint2 *cand;          // K1 candidate stash: cand_R pairs per K1 CTA
    uint2 *rec;           // candidate records: {offset in the CTA region, count}
    uint2 *Q;             // ASQ layers' emission scratch (pairs; K5 packs the message)
    uint4 *dec_lay;       // [nranks][L] where each rank's set of each layer sits (k6_prep)
    uint32_t cand_R;
    uint32_t seg_ch;      // K3A over the stash: candidate records per segment (small records
                          // are grouped; 1 = one record per segment)
    uint32_t status_extra;   // look-back status words beyond the tile count (zeroed by K1)
    uint32_t ntiles_total;
    // RGC_SYNC_PULL write-after-read guard: before this compress may rewrite the message
    // block the peers read in place last epoch, K1 (block 0, at its end) waits until every
    // peer published consumed[peer] >= pull_epoch in this rank's flags (NULL: no wait)
    P2PFlags *pull_flags;
    unsigned long long pull_epoch;
    int pull_rank, pull_p;
    // pinned host-mapped word: K2's message layout writes the call's K4 work there, so the
    // host can pick the next call's K4 launch form (one cooperative launch when idle)
    volatile uint32_t *k4_hint;
    // K1 CTAs count themselves here when their tiles are streamed (NULL: no count)
    unsigned long long *k1cnt;
    // K45 cluster capacity (keys) = CTAs per cluster x kKeysPerCta45: candidate sets up to it
    // take the one-cluster select + emission
    uint32_t small_sel;
    // diagnostics (RGC_TIMELINE=1 at rgc_init, else NULL): per kernel id the earliest CTA
    // start after griddepcontrol.wait ([id]) and the latest CTA exit ([kTlKernels + id]),
    // globaltimer ns -- the warm step's timeline with the zero fill beside it (ncu serialises)
    unsigned long long *tl;
};
constexpr int kTlKernels = 32;
enum TlId { TL_K1 = 0, TL_K2S, TL_K2V0, TL_K2V1, TL_K3A, TL_K3B, TL_K45, TL_K4, TL_K5, TL_FILL,
            TL_SCATTER, TL_PREP, TL_TAB, TL_K6,
            // sub-phases: K1's tile streaming (end = the last CTA's last tile), the per-layer
            // finalisations of K1 and K2, K2's global finalisation (the message layout)
            TL_K1S, TL_K1F, TL_K2F, TL_K2G,
            TL_P0 };   // TL_P0 + i: development probes (tl_probe)

// rank r's message block: base + r*stride (the gathered buffer of the NCCL modes, or the
// local staging area the peers pushed into in RGC_SYNC_P2P mode), or tab[r] in
// RGC_SYNC_PULL mode: every rank's own block, peers' mapped over NVLink (CUDA IPC)
struct MsgSrc {
    const uint8_t *base;
    uint64_t stride;
    const uint8_t *const *tab;
    __device__ __forceinline__ const uint8_t *of(int r) const {
        return tab ? tab[r] : base + (uint64_t)r * stride;
    }
};

// RGC_SYNC_P2P epoch flags, one block per rank (library-owned, IPC-exported).  Rank r
// stores into peer q's block: ready[r] = e once its epoch-e message sits in q's staging
// area, consumed[r] = e once it has decompressed epoch e (its staging slots are free).
constexpr int kMaxP2P = 64;
struct alignas(128) P2PFlags {
    unsigned long long ready[kMaxP2P];
    unsigned long long consumed[kMaxP2P];
    unsigned long long pushed;     // CTAs of this rank's push kernels that finished (monotone)
    unsigned long long err;        // nonzero: a wait timed out (bit q: waiting for rank q)
    unsigned long long timeout_ns; // wait limit (rgc_p2p_init: RGC_P2P_TIMEOUT_S, default 120 s)
};

// Device status of a context (library-owned, rgc_status): word 0 = sticky OR of the status
// words of every message block a decompression consumed (RGC_F_NONFINITE from any rank) and
// kStatTimeout when a cross-GPU wait gave up; words 1 / 2 = OR of the P2P timeout masks
// (bit q of ranks 0-31 / 32-63: a wait for rank q gave up).  k_finish keeps the sticky copy in device memory and mirrors it into
// pinned, host-mapped memory only when it changes, so the host can poll it without a sync.
constexpr uint32_t kStatTimeout = 1u << 30;
constexpr int kStatWords = 4;

constexpr int kFillSigWords = 4 + 1024 + 4;   // k6_fill control words (rgc_decomp.cu)

// Producer range table (multi-rank contexts): k_tab writes, into the table region at the end
// of the message block, tab[slot_begin_l + t] = the entry index (in this rank's entry
// sequence) of layer l's first entry with element index >= 8192 t, t = 0..ntiles_l, and sets
// the header word hdr[2L+2] to kTabMarker.  Receivers read it instead of re-deriving every
// rank's ranges (k6_prep) -- the work moves from p receivers to 1 producer.
constexpr uint32_t kTabMarker = RGC_MSG_TABLE;
constexpr uint32_t kStatNoTable = 1u << 29;   // a rank's block lacked the table (rgc_status)
constexpr uint32_t kStatBarrier = 1u << 28;   // a grid barrier gave up (co-residency failed)

// dense outputs of one decompression, passed by value to k6_fill (rgc_decomp.cu)
struct FillTable {
    unsigned long long *tl;   // timeline (Ws::tl) or NULL
    float *out[RGC_MAX_LAYERS];
    uint32_t n[RGC_MAX_LAYERS];
    uint32_t chunk_begin[RGC_MAX_LAYERS + 1];   // prefix of 64 KB fill chunks per layer
    int L;
    uint32_t sm_stride;       // SMs that fill: smid % sm_stride == 0 (RGC_FILL_STRIDE, default 1)
    uint32_t inflight;        // bulk groups in flight per filling SM, 0 = unbounded (RGC_FILL_INFLIGHT)
    // the early fill (RGC_FILL_AT=0, enqueued with K1): k1cnt[0] counts K1's CTAs started,
    // k1cnt[1] those done streaming (both monotonic); a CTA works only if k1cnt[0] reached
    // start_target (every K1 CTA resident), from when k1cnt[1] reaches wait_until; NULL: the
    // regular fill
    const unsigned long long *k1cnt;
    unsigned long long start_target, wait_until;
};

// host-side launchers (rgc_kernels.cu)
struct Launch {
    int grid_stream;   // persistent grid for the streaming kernels
    int grid_k3;
    int grid_k4;
    int grid_k6;
    int grid_small;
};

cudaError_t launch_k1(const Ws &w, int L, uint32_t total_tiles, uint32_t *msg_hdr, int grid,
                      cudaStream_t s);
cudaError_t launch_k2(const Ws &w, int L, uint32_t total_tiles, int max_trim_levels,
                      uint32_t *msg_hdr, uint32_t hdr_words, int grid, uint32_t nrec,
                      int grid_stash, cudaStream_t s, uint64_t *launches);
cudaError_t launch_k3(const Ws &w, int L, int pass, uint2 *msg_pairs, int grid, cudaStream_t s);
cudaError_t launch_k4(const Ws &w, int L, int pass, int grid, cudaStream_t s);
// the three radix passes in ONE cooperative launch with grid barriers between them (falls
// back to three launches if the cooperative launch is refused); *launches += kernels used
cudaError_t launch_k4_all(const Ws &w, int L, uint32_t *msg_hdr, int sms, cudaStream_t s,
                          uint64_t *launches, bool expect_work);
cudaError_t launch_k6_prep(const Ws &w, int L, int p, const MsgSrc &src, uint32_t hdr_words,
                           uint32_t total_dec_tiles, int grid, cudaStream_t s, uint32_t max_pairs);
cudaError_t launch_k6(const Ws &w, int L, int p, const MsgSrc &src, uint32_t hdr_words,
                      uint32_t total_dec_tiles, float scale, int grid, cudaStream_t s);
cudaError_t launch_k6_atomic(const Ws &w, int L, int p, const MsgSrc &src, uint32_t hdr_words,
                             uint32_t total_dec_tiles, uint32_t max_pairs, float scale, int grid,
                             cudaStream_t s);
cudaError_t occupancy(int *k1, int *k2, int *k3, int *k4, int *k6);
cudaError_t set_tuning(const uint32_t *t);   // stash / bounded-histogram policy (rgc_kernels.cu)
cudaError_t occupancy_k3(int *k3);
// decompression split (rgc_decomp.cu)
cudaError_t launch_k6_fill(const FillTable &t, unsigned int *sig, int grid, cudaStream_t s);
cudaError_t launch_k6_scatter(const Ws &w, int L, int p, const MsgSrc &src, uint32_t hdr_words,
                              uint32_t total_dec_tiles, uint32_t max_pairs, float scale, int grid,
                              cudaStream_t s, uint32_t tab_woff);
// producer range table of this rank's message (rgc_decomp.cu)
cudaError_t launch_k_tab(const Ws &w, int L, uint32_t *msg, uint32_t hdr_words, uint32_t tab_woff,
                         uint32_t max_pairs, int grid, cudaStream_t s);
cudaError_t launch_k6_atomic_only(const Ws &w, int L, int p, const MsgSrc &src, uint32_t hdr_words,
                                  uint32_t max_pairs, float scale, int grid, cudaStream_t s);
// ASQ message packing (rgc_asq.cu)
cudaError_t launch_k5_asq(const Ws &w, int L, uint32_t *msg_hdr, uint32_t hdr_words, int grid,
                          cudaStream_t s);
cudaError_t launch_k45(const Ws &w, int L, uint2 *msg_pairs, cudaStream_t s, int cl);
// RGC_SYNC_P2P (rgc_p2p.cu)
cudaError_t launch_p2p_push(const uint8_t *msg, uint8_t *const *stage, P2PFlags *const *peer_flags,
                            P2PFlags *mine, int rank, int p, unsigned long long epoch,
                            uint64_t msg_bytes, int L, uint32_t hdr_words, int nb, cudaStream_t s,
                            uint64_t tab_off, uint64_t tab_bytes);
// RGC_SYNC_PULL (rgc_p2p.cu): publish ready[rank] = e in every peer / wait for every peer's
cudaError_t launch_pull_publish(P2PFlags *const *peer_flags, int rank, int p,
                                unsigned long long epoch, cudaStream_t s);
cudaError_t launch_pull_wait(P2PFlags *mine, int rank, int p, unsigned long long epoch,
                             cudaStream_t s);
// End of every decompression (rgc_p2p.cu): OR the status word of every rank's block into the
// context status (and the P2P timeout mask), then -- P2P / PULL at p > 1 -- publish
// consumed[rank] = epoch in every peer
cudaError_t launch_finish(const MsgSrc &src, int L, int p, P2PFlags *mine,
                          P2PFlags *const *peer_flags, int rank, unsigned long long epoch,
                          int publish, uint32_t *d_stat, volatile uint32_t *h_stat, cudaStream_t s,
                          int need_tab);
// rgc_finalize (rgc_p2p.cu): wait (bounded) until every peer published consumed >= epoch, i.e.
// no peer still reads this rank's message block or stores into its flags
cudaError_t launch_wait_consumed(P2PFlags *mine, int rank, int p, unsigned long long epoch,
                                 unsigned long long limit_ns, cudaStream_t s);

}  // namespace rgc
