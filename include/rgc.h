/*
 * rgc.h -- C ABI of the B200 (sm_100a) RedSync Residual Gradient Compression
 * synchronisation hot path (Fang et al., arXiv 1808.04357).
 *
 * Citations "P:<n>" are lines of /root/reference/PAPER.md; "R<n>" are the
 * readings of silent / ambiguous passages listed in DESIGN.md.
 *
 * The calls follow the paper's statement of the per-layer problem
 * (Algorithm 1, and its prose P:137-151): every node keeps a
 * residual V per layer, adds its gradient, selects a
 * communication-set of density D by magnitude (Alg. 2 P:202-222 /
 * Alg. 3), packs <indices, values> into one message whose initial
 * element gives the length, zeroes the sent residual entries
 * (P:130), all-gathers the messages and decompresses all N sets
 * into the dense averaged gradient.
 *
 *   rgc_compress   : Alg.1 lines V += G, select, compress, V *= (1-Masks)
 *   rgc_sync       : Sparse-Allreduce implemented as Allgather
 *   rgc_decompress : decompress(G)
 *
 * Conventions
 *  - Every call returns an rgc_status_t; nothing crosses the ABI as an
 *    exception.  On error, rgc_last_error(ctx) gives a message.
 *  - All device buffers are owned by the caller (e.g. torch allocations);
 *    the library owns only the opaque context (and, when created from a
 *    unique id, its NCCL communicator).  Device pointers must be 16-byte
 *    aligned.
 *  - rgc_compress and rgc_decompress only enqueue kernels on the context's
 *    stream (asynchronous).  rgc_sync enqueues NCCL calls on the same stream;
 *    in RGC_SYNC_SIZES_FIRST mode it waits for the counts (the single
 *    device->host crossing of the path).  In RGC_SYNC_P2P mode it enqueues one
 *    kernel that stores the message into every peer over NVLink; in
 *    RGC_SYNC_PULL mode only an epoch flag (the decompression reads the peers).
 *  - Data-dependent decisions (threshold level, search path, fallbacks) are
 *    taken on the device; the host launches a fixed sequence of kernels, so
 *    compress + RGC_SYNC_FIXED + decompress can be captured in a CUDA graph.
 *  - A context is not thread-safe.
 */
#ifndef RGC_H
#define RGC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rgc_ctx *rgc_ctx_t;

typedef enum {
    RGC_OK = 0,
    RGC_EINVAL = 1,      /* bad argument: n==0 or n>=2^31, D not in (0,1], m<0, eps out of range,
                            unaligned pointer, L out of [1, RGC_MAX_LAYERS], nranks mismatch */
    RGC_ECUDA = 2,       /* a CUDA runtime call failed */
    RGC_ENCCL = 3,       /* NCCL missing or an NCCL call failed (incl. async errors) */
    RGC_ENONFINITE = 4,  /* a residual held Inf/NaN after accumulation (that layer sent 0 pairs) */
    RGC_ESTATE = 5       /* call out of order / workspace not initialised */
} rgc_status_t;

#define RGC_MAX_LAYERS 128
#define RGC_TILE 4096            /* elements per tile; also the mean_fx tile of R2 */
#define RGC_MAX_TRIM_LEVELS 16

/* selector (A11) */
enum { RGC_SEL_TRIMMED = 0,        /* Algorithm 2: exact top-k after trimming */
       RGC_SEL_THRESHOLD_BS = 1,   /* Algorithm 3: threshold binary search */
       RGC_SEL_SAMPLED_BS = 2 };   /* sampled threshold BS: reuse the searched threshold for
                                      sample_interval-1 calls (R20) */
/* branch rule of Alg.3 line 9 (R7) */
enum { RGC_BS_MONOTONE = 0,        /* nnz <= k -> r = ratio, else l = ratio (default) */
       RGC_BS_PAPER_LITERAL = 1 }; /* nnz < k/2 -> r = ratio, else l = ratio   */
/* allgather variants of rgc_sync */
enum { RGC_SYNC_FIXED = 0,         /* one allgather of the whole fixed-capacity message */
       RGC_SYNC_SIZES_FIRST = 1,   /* allgather of the length elements, then exact-size payloads */
       RGC_SYNC_P2P = 2,           /* exact-size push of every block over NVLink in one kernel
                                      (CUDA IPC mappings from rgc_p2p_init; epoch flags) */
       RGC_SYNC_PULL = 3 };        /* no copy: publish an epoch flag; the decompression reads
                                      every peer's block in place over NVLink (rgc_p2p_init) */

/* result flags (rgc_info_t.flags); numeric values listed in DESIGN.md "Flags" */
#define RGC_F_DEGENERATE (1u << 0)  /* max|V|==0 or mean==max -> exact top-k (R10) */
#define RGC_F_TRIM_ALL   (1u << 1)  /* Alg.2: no ratio>0 level reached k -> exact top-k on V */
#define RGC_F_BS_BREAK   (1u << 2)  /* Alg.3: k < nnz < 2k reached */
#define RGC_F_EPS_HIGH   (1u << 3)  /* Alg.3: eps-terminated, kept, nnz >= 2k */
#define RGC_F_EPS_BEST   (1u << 4)  /* Alg.3: eps-terminated with nnz<k; best nnz>=k used */
#define RGC_F_EPS_EXACT  (1u << 5)  /* Alg.3: eps-terminated, no nnz>=k seen -> exact top-k */
#define RGC_F_CAP_EXACT  (1u << 6)  /* chosen count > max_count -> exact top-k (R18) */
#define RGC_F_NONFINITE  (1u << 7)  /* residual not finite (error) */
#define RGC_F_EPS_KEEP   (1u << 8)  /* Alg.3: eps-terminated, last nnz >= k kept */
#define RGC_F_SAMPLED_REUSE (1u << 9) /* sampled BS: the cached threshold was reused */
#define RGC_F_SURV_CAP   (1u << 16) /* implementation note: Alg.2 survivors exceeded the
                                       workspace; exact top-k over V instead (same result) */

/* One compressed layer.  k = min(n, max(1, ceil(density*n))) (R1). */
typedef struct {
    uint64_t n;          /* elements, 1 <= n < 2^31 */
    double   density;    /* D in (0,1] */
    float    momentum;   /* DGC momentum correction m >= 0 (R15); 0 -> V += g */
    int32_t  selector;   /* RGC_SEL_* */
    int32_t  bs_branch;  /* RGC_BS_* */
    double   trim_eps;   /* Alg.2 step epsilon; 0 -> 0.2; at most 16 levels */
    double   bs_eps;     /* Alg.3 termination epsilon (R8); 0 -> 1e-3; in [2^-10, 1) */
    uint32_t max_count;  /* message capacity in pairs; 0 -> k (trimmed) or 2k (BS) (R18) */
    uint32_t sample_interval; /* RGC_SEL_SAMPLED_BS: full search every this many calls; 0 -> 5
                                 ("the interval of search is empirically set to 5") */
    int32_t  quantize;   /* 1: ASQ, Alternating Signs Quantization (R21, R22): the
                            call selects among the positive residuals (largest k) or, on the next
                            call, the negative ones (smallest k), alternating per layer from
                            positive, and the message carries the indices plus ONE value, the
                            mean of the selected values.  Not with RGC_SEL_SAMPLED_BS (P:292,
                            RGC_EINVAL).  The paper leaves the output layer unquantized:
                            the caller's choice.  0: plain <index, value> messages. */
} rgc_layer_t;

/* Per-layer diagnostics written by the device (read with rgc_get_info). */
typedef struct {
    uint32_t flags;          /* RGC_F_* */
    uint32_t iters;          /* count_nonzero evaluations (Alg.2 levels / Alg.3 steps) */
    uint32_t trim_level;     /* Alg.2: level used (== trim_levels if TRIM_ALL) */
    uint32_t trim_levels;    /* Alg.2: number of ratio > 0 levels */
    uint64_t count;          /* message length c */
    float    threshold;      /* threshold defining the set by strict '>' (0 for exact paths) */
    uint32_t maxkey;         /* bits of max|V| */
    double   mean;           /* mean_fx |V| (R2) */
    uint64_t level_count[RGC_MAX_TRIM_LEVELS];
    float    level_thresh[RGC_MAX_TRIM_LEVELS];
    uint64_t survivors;      /* Alg.2: survivors after trimming */
    uint32_t kth_key;        /* exact paths: bits of the k-th largest |V| */
    uint32_t tie_quota;      /* exact paths: how many elements equal to kth_key were taken */
    uint64_t emitted;        /* pairs the compaction kernel actually wrote (== count) */
    uint32_t lb_mask;        /* Alg.3: bit i set -> level_count[i] is a lower bound (the step
                                was decided by a bound from the bounded histogram) */
    uint32_t stashed;        /* 1: the compaction read the counting pass's candidate stash
                                instead of re-reading the residual (implementation detail) */
} rgc_info_t;

/* Buffer sizes for a layer list (bytes). */
typedef struct {
    uint64_t workspace_bytes;  /* device workspace (rgc_workspace_init before first use) */
    uint64_t msg_bytes;        /* one message block: header + pair capacity */
    uint64_t gathered_bytes;   /* nranks * msg_bytes */
    uint64_t header_bytes;     /* 4 * header words: counts[L], status, L, padding to 16 B */
    uint64_t k_total;          /* sum of k over layers */
    uint64_t cap_total;        /* sum of message capacities (pairs) */
} rgc_sizes_t;

/*
 * Message block layout (device, written by rgc_compress; the paper's "initial
 * element which indicates the length", one per layer):
 *   uint32 hdr[H]   H = 4*ceil((2L+3)/4): hdr[l] = c_l (entries of layer l),
 *                   hdr[L] = status (OR of RGC_F_NONFINITE over layers),
 *                   hdr[L+1] = L,
 *                   hdr[L+2+l] = RGC_MSG_DENSE for a plain layer, or the bits of the
 *                   layer's single fp32 value for an ASQ layer (0 if c_l == 0),
 *                   hdr[2L+2] = RGC_MSG_TABLE if the range table below is written, else 0
 *   uint2 pairs[]   at byte offset 4*H: the plain layers' pairs, layer order, compact;
 *                   pair = {uint32 index, uint32 bits of the fp32 value}
 *   uint32 idx[]    right after them: the ASQ layers' indices, layer order, compact
 *   (ascending index within a layer, R11).  Used bytes = 4*H + 8*sum_plain c_l +
 *   4*sum_ASQ c_l.
 *   uint32 tab[]    at the END of the block (byte offset msg_bytes - 4*T, T = a multiple of 4
 *                   >= sum_l (ceil(n_l/8192) + 1)): the range table (an implementation aid of
 *                   the decompression, not a paper element), written by rgc_compress of a
 *                   context with nranks > 1: for layer l with slot base b_l = sum_{l'<l}
 *                   (ceil(n_l'/8192) + 1), tab[b_l + t] = the index, in this block's entry
 *                   sequence, of layer l's first entry with element index >= 8192*t,
 *                   t = 0..ceil(n_l/8192).  rgc_sync moves it with the used bytes (P2P push,
 *                   SIZES_FIRST broadcast; FIXED moves the whole block), so the receivers
 *                   read every rank's per-tile ranges instead of deriving them.
 *   msg_bytes is the capacity.
 * gathered = nranks blocks at stride msg_bytes, rank-major.
 */
#define RGC_MSG_DENSE 0xFFFFFFFFu
#define RGC_MSG_TABLE 0x7AB1E001u   /* hdr[2L+2]: the block carries its range table */

const char  *rgc_version(void);
const char  *rgc_status_string(rgc_status_t s);

/* k for (n, D): min(n, max(1, ceil(D*n))) in IEEE double (R1). */
rgc_status_t rgc_k(uint64_t n, double density, uint64_t *k_out);

/* NCCL unique id for a library-owned communicator (128 bytes).  Requires
 * libnccl.so.2 (dlopen'ed; the one torch loaded if present). */
rgc_status_t rgc_get_unique_id(uint8_t out[128]);

/* Create a context on CUDA device `device`.  nranks == 1: no NCCL needed, uid
 * may be NULL.  nranks > 1: uid is the unique id from rank 0 (collective call
 * over all ranks, like ncclCommInitRank); uid == NULL creates a context without
 * a communicator (rgc_sync returns RGC_ESTATE) that can still decompress
 * nranks externally gathered message blocks.  stream: cudaStream_t (NULL =
 * legacy default stream) on which all work is enqueued. */
rgc_status_t rgc_init(rgc_ctx_t *ctx, int rank, int nranks, int device,
                      const uint8_t *uid, void *stream);
rgc_status_t rgc_set_stream(rgc_ctx_t ctx, void *stream);
rgc_status_t rgc_finalize(rgc_ctx_t ctx);
const char  *rgc_last_error(rgc_ctx_t ctx);

/* Buffer sizes for `layers` (validates every layer; EINVAL names the first bad one).
 * ctx may be NULL (host-only call, nranks = 1). */
rgc_status_t rgc_sizes(rgc_ctx_t ctx, const rgc_layer_t *layers, int L, rgc_sizes_t *out);

/* Zero-fill and initialise a workspace of rgc_sizes().workspace_bytes for `layers`.
 * Must be called once before the first rgc_compress with this workspace and layer
 * list (the kernels keep the workspace reset between calls). Asynchronous. */
rgc_status_t rgc_workspace_init(rgc_ctx_t ctx, const rgc_layer_t *layers, int L, void *ws);

/* Alg.1 lines 5-8 for L layers on this node:
 *   u = m*u + g; V = V + u   (or V = V + g when m == 0)
 *   select the communication-set of layer l by its selector
 *   write <indices, values> (values = V before zeroing) into msg
 *   V[i] = 0 (and u[i] = 0) for every sent i
 * grad[l], residual[l], momentum[l]: device fp32 arrays of n_l elements;
 * momentum[l] may be NULL iff layers[l].momentum == 0.  residual and momentum
 * are updated in place.  msg: device block of rgc_sizes().msg_bytes.
 * ws: the initialised workspace.  Asynchronous on the context stream. */
rgc_status_t rgc_compress(rgc_ctx_t ctx, const rgc_layer_t *layers, int L,
                          const float *const *grad, float *const *residual,
                          float *const *momentum, void *msg, void *ws);

/* Sparse-Allreduce as Allgather: every rank receives every rank's
 * message block into gathered[r * msg_bytes].  mode RGC_SYNC_FIXED: one
 * ncclAllGather of msg_bytes (no host sync).  RGC_SYNC_SIZES_FIRST: allgather
 * of the headers (the length elements), a device->host read of the counts,
 * then one ncclBroadcast per rank of exactly header + 8*sum_l c_{r,l} bytes
 * (grouped; plus each rank's range table, see the block layout).  counts_host (optional, nranks*L uint32, rank-major) receives the
 * counts in SIZES_FIRST mode.  nranks == 1: gathered may equal msg (no copy).
 * Returns RGC_ENONFINITE (after completing the exchange) if any rank flagged a
 * non-finite residual in SIZES_FIRST mode (the one mode that reads the headers on the
 * host); RGC_ENCCL if NCCL reports an asynchronous error (FIXED and SIZES_FIRST check
 * ncclCommGetAsyncError after enqueuing).  In every mode the decompression also folds
 * every rank's status word into the context status, reported by rgc_status.
 * mode RGC_SYNC_P2P (after rgc_p2p_init; msg = its block, gathered ignored): one
 * kernel pushes the used part of the block into every rank's staging area over
 * NVLink and exchanges epoch flags.  mode RGC_SYNC_PULL (same setup): one tiny
 * kernel publishes "epoch e ready" to every peer; nothing is copied, the next
 * rgc_decompress(gathered = NULL) reads the peers' blocks in place.  Both: no
 * host synchronisation; RGC_ESTATE without rgc_p2p_init, RGC_EINVAL if msg is
 * not the rgc_p2p_init block or the layers differ from rgc_p2p_init's. */
rgc_status_t rgc_sync(rgc_ctx_t ctx, const rgc_layer_t *layers, int L, const void *msg,
                      void *gathered, int mode, uint32_t *counts_host);

/* RGC_SYNC_P2P setup (collective: every rank of the context calls it once).
 * Allocates, in library-owned device memory, this rank's message block
 * (rgc_sizes().msg_bytes for these layers), a staging area of nranks blocks and
 * epoch flags; exchanges the IPC handles of the staging area and the flags over
 * the context's communicator and maps every peer's (NVLink/NVSwitch peer access).
 * *msg_out receives the message block: pass it as msg to rgc_compress and
 * rgc_sync(..., RGC_SYNC_P2P) (gathered ignored, may be NULL), then call
 * rgc_decompress with gathered = NULL.  The sync is then ONE kernel: it stores
 * the used part of this rank's block (header + the pairs its length elements
 * count) into slot `rank` of every rank's staging area over NVLink,
 * publishes "epoch e ready" in every peer and waits for every peer's; the
 * decompression reads its local staging area and then publishes "epoch e
 * consumed", which a peer waits for before pushing epoch e+1 into it.  No host
 * synchronisation; a wait longer than RGC_P2P_TIMEOUT_S seconds (environment,
 * read by rgc_init; default 120) gives up, and the next decompression turns it
 * into the context status: rgc_status then returns RGC_ESTATE and the context is
 * unusable (every later compress / sync / decompress returns RGC_ESTATE) -- a
 * timed-out exchange means the ranks' epochs are out of step.
 * Collective and all-or-nothing: if any rank cannot allocate or map its peers'
 * areas, every rank returns the error (so all can fall back to RGC_SYNC_FIXED).  The same setup serves RGC_SYNC_PULL: it also maps
 * every peer's message block; rgc_sync(..., RGC_SYNC_PULL) then only publishes
 * "epoch e ready" (one tiny kernel, nothing copied) and rgc_decompress(gathered =
 * NULL) reads the peers' blocks in place (see rgc_decompress).  Freed by
 * rgc_finalize.
 * Errors: RGC_ESTATE (no communicator, or already initialised), RGC_ECUDA
 * (a peer area cannot be mapped: no P2P between the GPUs), RGC_EINVAL
 * (nranks > 64). */
rgc_status_t rgc_p2p_init(rgc_ctx_t ctx, const rgc_layer_t *layers, int L, void **msg_out);

/* Inspection copy for RGC_SYNC_P2P / RGC_SYNC_PULL (tests, diagnostics): enqueue a
 * copy of every rank's block (P2P: the local staging area the peers pushed into;
 * PULL: each rank's own block, read over NVLink after waiting for its epoch flag;
 * bytes past a block's used part are undefined) into gathered[r * msg_bytes].
 * Valid only between rgc_sync(..., RGC_SYNC_P2P or RGC_SYNC_PULL) and the following
 * rgc_decompress (the peers overwrite the blocks only after it); RGC_ESTATE
 * otherwise. */
rgc_status_t rgc_p2p_gather(rgc_ctx_t ctx, const rgc_layer_t *layers, int L, void *gathered);

/* Host-side planning step of RGC_SYNC_SIZES_FIRST (no GPU needed): from the
 * nranks gathered headers (rank-major, header_words u32 each) compute the
 * exact bytes each rank broadcasts (4*header_words + 8*sum_plain c_{r,l} +
 * 4*sum_ASQ c_{r,l}, a layer's kind read from hdr[L+2+l]), the counts
 * (nranks*L, optional) and the OR of the status words (optional).
 * RGC_EINVAL if header_words < 2L+2; RGC_ESTATE if a header does not describe
 * L layers or exceeds msg_bytes. */
rgc_status_t rgc_sync_plan(const uint32_t *headers, int nranks, int L, uint32_t header_words,
                           uint64_t msg_bytes, uint64_t *bytes_out, uint32_t *counts_out,
                           uint32_t *status_out);

/* decompress into the dense averaged gradient (R13, R14):
 *   ordered = 1: out[l][i] = fl32( sum over ranks r = 0..p-1, in rank order from +0,
 *                of the value rank r sent for index i ) * fl32(1/p)   -- bit-exact;
 *   ordered = 0: unordered atomic variant (tolerance 1e-6 relative, R14).
 * out[l]: device fp32 arrays of n_l elements (fully overwritten).
 * gathered: nranks blocks at stride msg_bytes (RGC_SYNC_FIXED / SIZES_FIRST),
 * or NULL after an RGC_SYNC_P2P sync: the staging area the peers pushed into
 * (RGC_EINVAL if no such sync precedes the call); also NULL after an
 * RGC_SYNC_PULL sync: the decompression first waits (one small kernel) for every
 * peer's epoch flag, then its kernels load the peers' pairs in place over NVLink
 * (CUDA IPC mappings of the peers' message blocks) -- the gather and the
 * scatter-add are one pass -- and finally publishes "consumed"; a peer's next
 * rgc_compress waits for that (inside its accumulate kernel) before rewriting
 * its block.  The last kernel of every decompression folds every rank's status word
 * into the context status (rgc_status). */
rgc_status_t rgc_decompress(rgc_ctx_t ctx, const rgc_layer_t *layers, int L,
                            const void *gathered, float *const *out, int ordered, void *ws);

/* Overlap of the decompression's dense part with the selection (implementation of
 * P:310-312 / R13; not a paper step).  The dense averaged gradient is +0 except at the
 * indices some rank sent, and zeroing it is the whole HBM cost of the decompression
 * (4 bytes per element) while it depends on no message.  This call registers the
 * outputs (out[l]: device fp32 arrays of layers[l].n elements, 16-byte aligned) of the
 * NEXT rgc_decompress: the next rgc_compress then enqueues, right after its
 * accumulate pass (K1), a zero fill of every out[l] (TMA bulk stores, one CTA per SM)
 * on a library-owned auxiliary stream forked from the context stream, so it streams
 * while the latency-bound selection kernels and the sync run; the next rgc_decompress
 * with the same out pointers waits for it and writes only the indices some rank sent
 * (bit-identical to the full decompression in both modes).  When K1 has many tiles per
 * CTA an early part of the fill is enqueued with K1 and fills the SMs K1's finished CTAs
 * leave; it is skipped when an out[l] overlaps a grad / residual / momentum buffer, so
 * out[l] may still alias grad[l] (the fill after K1 then does everything).  If no rgc_compress intervenes, rgc_decompress
 * enqueues the fill itself (same result, no overlap).  If rgc_decompress gets other
 * outputs, the full decompression runs (the registered buffers have been zeroed
 * nevertheless).  Stream capture: capture the compress and the decompress that
 * joins the fill in the same graph.  RGC_ESTATE if a registered fill is still
 * enqueued (call rgc_decompress first); RGC_EINVAL on bad layers / pointers. */
rgc_status_t rgc_decompress_prefill(rgc_ctx_t ctx, const rgc_layer_t *layers, int L,
                                    float *const *out);

/* Synchronous diagnostics: copy the per-layer info of the last compress. */
rgc_status_t rgc_get_info(rgc_ctx_t ctx, int L, const void *ws, rgc_info_t *out);

/* Synchronous diagnostics of the implementation's per-layer state (not a paper step):
 * out[0..15] = mode, count, threshold key, stash key, stash shift, stash on, stash ok,
 * K2 source = stash, K3 source = stash, full-histogram pass needed, Alg.3 hint, Alg.3
 * margin, ASQ phase, survivors, emitted (first pass), emitted (exact pass), stash
 * records of the last accumulate pass, count at the lowest key the call needed, calls
 * so far whose counts re-read the residual (stash miss), calls so far that needed
 * Alg.3's full-histogram pass.  RGC_EINVAL if nout < 20 or l is out of range. */
rgc_status_t rgc_debug_layer(rgc_ctx_t ctx, const void *ws, int l, uint32_t *out, int nout);

/* Synchronous check of the last compress' status word (RGC_F_NONFINITE etc.). */
rgc_status_t rgc_check(rgc_ctx_t ctx, const void *msg, int L, uint32_t *status_out);

/* Context status, every sync mode (the exchange surfaces device status flags).
 * Every rgc_decompress ends with one small kernel that ORs the status word (hdr[L]) of every
 * rank's message block it consumed -- RGC_F_NONFINITE: some rank's residual held Inf/NaN,
 * its set for that layer was empty -- and the P2P / PULL wait-timeout mask into a sticky
 * device word, mirrored into pinned host-mapped memory when it changes.  rgc_status reads
 * that copy WITHOUT synchronising (flags = 0: it reflects the decompressions that have
 * completed so far, so an error of step i surfaces at a later poll), or after
 * cudaStreamSynchronize of the context stream (RGC_STATUS_WAIT).  RGC_STATUS_CLEAR (implies
 * WAIT) resets the non-finite report.  status_out (optional, 4 words): [0] status bits
 * (RGC_F_NONFINITE; bit 30 = a cross-GPU wait timed out; bit 29 = a block read for its range
 * table did not carry one; bit 28 = a grid barrier of the one-launch radix select gave up),
 * [1]/[2] the ranks a wait gave up on (bits of ranks 0-31 / 32-63), [3] the NCCL async error
 * code seen by rgc_sync (0 none).  Returns, in this order of precedence: RGC_ESTATE (a wait
 * timed out: the context is unusable from now on; or bit 28 / 29: that step's result is not
 * valid), RGC_ENCCL, RGC_ENONFINITE, else RGC_OK. */
#define RGC_STATUS_WAIT 1
#define RGC_STATUS_CLEAR 2
rgc_status_t rgc_status(rgc_ctx_t ctx, int flags, uint32_t *status_out);

/* Phase timing with CUDA events recorded on the context stream.
 * rgc_profile(ctx, 1) enables recording of every phase, rgc_profile(ctx, 2) of phase
 * [0] only (two events per compress: the dominant kernel timed live with the least
 * perturbation), rgc_profile(ctx, k) with k > 2 of phase [0] on every (k-1)-th compress
 * call only, counting from this call (events break the programmatic-dependent-launch
 * overlap at K1's edges, ~7 us per recorded call), 0 disables it; rgc_profile_read waits for the
 * recorded events and returns accumulated milliseconds per phase since the
 * previous read:  [0] accumulate+stats  [1] threshold count/search
 * [2] compaction (survivors / BS pairs)  [3] exact select  [4] final emission
 * [5] sync  [6] decompress.  n_out receives the number of compress calls
 * accumulated.  Returns RGC_EINVAL if nphase < 7. */
#define RGC_NPHASE 7
rgc_status_t rgc_profile(rgc_ctx_t ctx, int enable);
rgc_status_t rgc_profile_read(rgc_ctx_t ctx, float *ms, int nphase, int *n_out);

/* Diagnostics: the per-kernel timeline of the last step, for a context created with the
 * environment variable RGC_TIMELINE=1 (else RGC_ESTATE).  Every kernel records its earliest
 * CTA start after its programmatic-dependent-launch wait and its latest CTA exit (globaltimer
 * ns); out[id] = start, out[32 + id] = end, id = K1 0, K2 stash 1, K2 V passes 2 / 3, K3A 4,
 * K3B 5, K45 6, K4 7, K5 8, zero fill 9, scatter 10, k6_prep 11, k_tab 12 (start = UINT64_MAX:
 * did not run).  Waits for the context and auxiliary streams.  n >= 64. */
rgc_status_t rgc_debug_timeline(rgc_ctx_t ctx, uint64_t *out, int n);

/* Number of kernels this context has launched (host counter). */
uint64_t rgc_launch_count(rgc_ctx_t ctx);

#ifdef __cplusplus
}
#endif
#endif /* RGC_H */
