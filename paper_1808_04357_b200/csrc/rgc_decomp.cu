// rgc_decomp.cu -- the decompression (R13, R14) split in two so that its
// dense part leaves the critical path.
//
// The dense averaged gradient is +0 everywhere except at the indices some rank sent
// (D = 0.1 %: ~0.1 % x p of the elements).  Writing those 4 bytes/element is the whole
// HBM cost of the decompression, and it does not depend on the messages:
//
//   k6_fill     zero-fills the outputs with TMA bulk stores (cp.async.bulk
//               shared::cta -> global from one zeroed 8 KB smem buffer; one issuing
//               thread per CTA, one active CTA per SM).  rgc_api.cu enqueues it on a
//               high-priority auxiliary stream forked right after K1, so it streams
//               while the latency-bound selection kernels (K2..K3B) and the sync run.
//   k6_scatter1 p == 1: every pair g writes out[i] = fl32(+0 + v) * fl32(1/p)
//               (one thread per pair; no tiling needed).
//   k6_scatter  p > 1: one warp per 8192-element tile (ranges from k6_prep).  The
//               leader of an index -- the entry of the lowest rank that sent it --
//               adds every rank's value in rank order from +0 (binary searches in
//               the other ranks' sorted ranges of the tile) and stores the scaled
//               sum once: out[i] = fl32(sum_r v_r[i]) * fl32(1/p), bit-identical to
//               k6_decompress's full-tile accumulation (R14).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "rgc_device.cuh"

namespace rgc {

constexpr int kFillSmem = 8192;             // zero source of the bulk stores (bytes)
constexpr uint32_t kFillChunk = 65536;      // bytes of output per work item

// Control words sig[]: [1] fill CTAs exited, [2] chunk ticket, [4 + smid] "an active
// fill CTA runs on this SM", [1028] debug slot counter.
//
// Placement decides this kernel's speed: the block scheduler puts a CTA on the first SM
// with room, and when the fill becomes ready together with the selection kernels (right
// after K1) plain 32-thread CTAs were packed ~25 to an SM on 6 SMs (0.36 TB/s, measured
// with RGC_FILL_DEBUG).  So (1) a CTA that finds another fill CTA on its SM exits at once
// (the grid is 2 per SM, 512 threads each), (2) the active CTAs take 64 KB chunks from a
// ticket, so the work follows whichever SMs hold an active CTA, and (3) the stream has
// the highest priority.  Measured: one active CTA on each of the 148 SMs, 85 us for
// VGG16's 553 MB alone (6.5 TB/s).  The last CTA to exit resets the control words.
constexpr int kFillThreads = 512;
constexpr int kFillMaxSM = 1024;

__global__ void __launch_bounds__(kFillThreads, 1)
k6_fill(FillTable t, unsigned int *sig, unsigned long long *dbg) {
    TlMark tlm(t.tl, TL_FILL);
    __shared__ alignas(128) uint4 z[kFillSmem / 16];
    __shared__ int s_work;
    __shared__ unsigned int s_sm;
    const int tid = threadIdx.x;
    unsigned long long dt0 = 0;
    if (tid == 0) {
        unsigned int smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        s_sm = smid % kFillMaxSM;
        s_work = (smid % t.sm_stride) == 0u && atomicExch(sig + 4 + s_sm, 1u) == 0u;
    }
    __syncthreads();
    if (t.k1cnt) {
        // the early fill, enqueued with K1 (the regular fill after K1 does whatever it leaves):
        // a CTA placed before all of K1's CTAs are resident must not hold a slot K1 needs --
        // it leaves at once; else it waits until enough of K1 has streamed (the fill has no
        // data dependency on K1: this only keeps it off K1's bandwidth), at most 2 ms
        if (tid == 0 && s_work) {
            if (*(volatile const unsigned long long *)&t.k1cnt[0] < t.start_target) {
                s_work = 0;
            } else {
                const unsigned long long t0 = globaltimer_ns();
                while (*(volatile const unsigned long long *)&t.k1cnt[1] < t.wait_until &&
                       globaltimer_ns() - t0 < 2000000ull)
                    __nanosleep(256);
            }
            if (!s_work) atomicExch(sig + 4 + s_sm, 0u);
        }
        __syncthreads();
    }
    if (s_work) {
        for (int i = tid; i < kFillSmem / 16; i += kFillThreads) z[i] = make_uint4(0u, 0u, 0u, 0u);
        // generic-proxy writes of the smem source -> visible to the async (TMA) proxy
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            if (dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(dt0));
            const uint32_t zs = (uint32_t)__cvta_generic_to_shared(z);
            const uint32_t nchunks = t.chunk_begin[t.L];
            const uint64_t pol = l2_policy_evict_first();   // keep the K1 stash in L2
            for (uint32_t c = atomicAdd(sig + 2, 1u); c < nchunks; c = atomicAdd(sig + 2, 1u)) {
                int lo = 0, hi = t.L - 1;              // layer of chunk c
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (t.chunk_begin[mid] <= c) lo = mid; else hi = mid - 1;
                }
                const uint64_t nbytes = 4ull * t.n[lo];
                const uint64_t b0 = (uint64_t)(c - t.chunk_begin[lo]) * kFillChunk;
                const uint64_t b1 = b0 + kFillChunk < nbytes ? b0 + kFillChunk : nbytes;
                const uint64_t bulk_end = b0 + ((b1 - b0) & ~15ull);   // 16-byte granules
                uint8_t *base = reinterpret_cast<uint8_t *>(t.out[lo]);
                for (uint64_t b = b0; b < bulk_end; b += kFillSmem) {
                    const uint32_t sz = (uint32_t)(bulk_end - b < (uint64_t)kFillSmem ? bulk_end - b
                                                                                        : kFillSmem);
#ifdef RGC_NO_L2HINT
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                                 ::"l"(base + b), "r"(zs), "r"(sz) : "memory");
#else
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                                 ::"l"(base + b), "r"(zs), "r"(sz), "l"(pol) : "memory");
#endif
                    if (t.inflight) {
                        // paced: at most inflight 8 KB stores pending per filling SM, so the
                        // HBM write queues do not back up into the selection chain's loads
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                        switch (t.inflight) {
                            case 1: asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); break;
                            case 2: asm volatile("cp.async.bulk.wait_group 2;" ::: "memory"); break;
                            case 3: asm volatile("cp.async.bulk.wait_group 3;" ::: "memory"); break;
                            case 4: asm volatile("cp.async.bulk.wait_group 4;" ::: "memory"); break;
                            case 6: asm volatile("cp.async.bulk.wait_group 6;" ::: "memory"); break;
                            case 8: asm volatile("cp.async.bulk.wait_group 8;" ::: "memory"); break;
                            case 12: asm volatile("cp.async.bulk.wait_group 12;" ::: "memory"); break;
                            default: asm volatile("cp.async.bulk.wait_group 16;" ::: "memory"); break;
                        }
                    }
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                // the last < 16 bytes of a layer whose n is not a multiple of 4
                for (uint64_t b = bulk_end; b < b1; b += 4) *reinterpret_cast<float *>(base + b) = 0.f;
            }
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            if (dbg) {
                unsigned long long dt1;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(dt1));
                const unsigned int slot = atomicAdd(sig + 1028, 1u);
                dbg[3 * slot] = s_sm;
                dbg[3 * slot + 1] = dt0;
                dbg[3 * slot + 2] = dt1;
            }
            atomicExch(sig + 4 + s_sm, 0u);
        }
    }
    if (tid == 0 && !t.k1cnt) {   // (the early fill leaves the counters to the regular one)
        __threadfence();
        if (atomicAdd(sig + 1, 1u) == gridDim.x - 1) {   // everyone is past the wait
            if (dbg) dbg[3 * 1023] = sig[1028];
            atomicExch(sig + 1028, 0u);
            atomicExch(sig + 1, 0u);
            atomicExch(sig + 2, 0u);
        }
    }
}

// Producer range table (rgc_compress of a multi-rank context, after the message is
// final): k6_prep's derivation of the per-tile entry ranges, done once by the producer of the
// message instead of by every receiver.  slot_begin / decompress tiles per layer come from
// the layer sizes (the decompression's table is not uploaded at compress time).
__global__ void __launch_bounds__(kThreads)
k_tab(Ws w, int L, uint32_t *msg, uint32_t hdr_words, uint32_t tab_woff, uint32_t max_pairs) {
    pdl_wait();
    TlMark tlm(w.tl, TL_TAB);
    __shared__ uint32_t s_off[RGC_MAX_LAYERS + 1], s_ao[RGC_MAX_LAYERS + 1];
    __shared__ uint32_t s_sb[RGC_MAX_LAYERS + 1], s_nt[RGC_MAX_LAYERS];
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid < 32) {   // slot_begin_l = sum over l' < l of (ntiles_l' + 1)
        uint32_t carry = 0;
        for (int l0 = 0; l0 < L; l0 += 32) {
            const int l = l0 + lane;
            const uint32_t nt = l < L ? (w.desc[l].n + kDecTile - 1) / kDecTile : 0u;
            const uint32_t v = l < L ? nt + 1u : 0u;
            uint32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULLMASK, x, o);
                if (lane >= o) x += y;
            }
            if (l < L) { s_sb[l] = carry + x - v; s_nt[l] = nt; }
            carry += __shfl_sync(FULLMASK, x, 31);
        }
        if (lane == 0) s_sb[L] = carry;
    }
    MsgSrc src;
    src.base = reinterpret_cast<const uint8_t *>(msg);
    src.stride = 0;
    src.tab = nullptr;
    load_layout(src, L, 1, s_off, s_ao);   // (synchronises the block)
    uint32_t *tab = msg + tab_woff;
    const uint32_t gtid = blockIdx.x * kThreads + tid, stride = gridDim.x * kThreads;
    for (uint32_t sl = gtid; sl < s_sb[L]; sl += stride) {   // empty sets: the layer offset
        const int l = find_layer(s_sb, L, sl);
        RGC_DCHECK(sl < s_sb[L]);
        if (s_off[l + 1] == s_off[l]) tab[sl] = s_off[l];
    }
    const uint32_t *pw = msg + hdr_words;
    const uint32_t tot = min(s_off[L], max_pairs);
    for (uint32_t g = gtid; g < tot; g += stride) {           // tile boundaries
        const int l = find_layer(s_off, L, g);
        const uint4 v = layer_view(msg, s_off, s_ao, L, l);
        uint32_t *out = tab + s_sb[l];
        const int t = (int)(view_entry(pw, v, g).x / kDecTile);
        const int tprev = (g > s_off[l]) ? (int)(view_entry(pw, v, g - 1).x / kDecTile) : -1;
        RGC_DCHECK(t >= 0 && (uint32_t)t <= s_nt[l]);
        for (int tt = tprev + 1; tt <= t; tt++) out[tt] = g;
        if (g + 1 == s_off[l + 1])
            for (uint32_t tt = t + 1; tt <= s_nt[l]; tt++) out[tt] = g + 1;
    }
    if (blockIdx.x == 0 && tid == 0) msg[2 * L + 2] = kTabMarker;
}

cudaError_t launch_k_tab(const Ws &w, int L, uint32_t *msg, uint32_t hdr_words, uint32_t tab_woff,
                         uint32_t max_pairs, int grid, cudaStream_t s) {
    return launch_pdl(k_tab, grid, kThreads, 0, s, w, L, msg, hdr_words, tab_woff, max_pairs);
}

// A value alone in its 32-byte output sector is stored as the whole sector (the value and
// seven +0, which the zero fill wrote there anyway): a full-sector write needs no DRAM
// read-modify-write when L2 evicts it, where a 4-byte store into a sector the fill left
// in DRAM costs a 32-byte read (~20 MB of reads per p = 4 VGG16 decompression, ncu).
// Needs a 32-byte aligned output (else the plain 4-byte store).
#ifdef RGC_NO_SECTOR_STORE
constexpr bool kSectorStore = false;   // A/B: plain 4-byte stores
#else
constexpr bool kSectorStore = true;
#endif
__device__ __forceinline__ void store_alone_in_sector(float *out, uint32_t i, float v) {
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
    const uint32_t s = i & 7u;
    if (s < 4) (&a.x)[s] = v; else (&b.x)[s - 4] = v;
    float4 *q = reinterpret_cast<float4 *>(out + (i & ~7u));
    q[0] = a;
    q[1] = b;
}

// p == 1: out[i] = fl32(+0 + v) * scale for every pair (R13: +0 + (-0) = +0)
__global__ void __launch_bounds__(kThreads)
k6_scatter1(Ws w, int L, MsgSrc src, uint32_t hdr_words, uint32_t max_pairs, float scale) {
    pdl_wait();
    TlMark tlm(w.tl, TL_SCATTER);
    __shared__ uint32_t s_off[RGC_MAX_LAYERS + 1], s_ao[RGC_MAX_LAYERS + 1];
    __shared__ uint4 s_v[RGC_MAX_LAYERS];
    load_layout(src, L, 1, s_off, s_ao);
    const uint32_t *hdr = reinterpret_cast<const uint32_t *>(src.of(0));
    for (int l = threadIdx.x; l < L; l += kThreads) s_v[l] = layer_view(hdr, s_off, s_ao, L, l);
    __syncthreads();
    const uint32_t total = s_off[L];
    const uint32_t *pw = hdr + hdr_words;
    for (uint32_t g = blockIdx.x * kThreads + threadIdx.x; g < total && g < max_pairs;
         g += gridDim.x * kThreads) {
        const int l = find_layer(s_off, L, g);
        const uint2 pr = view_entry(pw, s_v[l], g);
        // plain 4-byte stores: at p = 1 the neighbour loads a whole-sector store needs cost
        // more than the read-modify-writes they save (decompress 18.8 -> 21.5 us on VGG16)
        RGC_DCHECK(pr.x < w.ddesc[l].n);
        w.ddesc[l].out[pr.x] = __fmul_rn(__fadd_rn(0.f, __uint_as_float(pr.y)), scale);
    }
}

// index x among the ascending entries [a, b) of a set? -> its value bits
__device__ __forceinline__ bool find_pair(const uint32_t *pw, const uint4 &v, uint32_t a, uint32_t b,
                                          uint32_t x, uint32_t *bits) {
    while (a < b) {
        const uint32_t mid = (a + b) >> 1;
        const uint2 pr = view_entry(pw, v, mid);
        if (pr.x == x) { *bits = pr.y; return true; }
        if (pr.x < x) a = mid + 1; else b = mid;
    }
    return false;
}

constexpr int kMaxRanks = 64;

// p > 1: one warp per decompress tile; dec_start from k6_prep.  The tile's entries of
// all ranks (S of them, rank-major, ascending index within a rank) are staged in the
// warp's shared memory with independent loads; two 8192-bit maps mark the indices seen
// once and more than once.  An index one rank sent (the common case: P:300 reports ~1.5%
// overlap) is written directly; for a shared one the entry of the lowest rank sums the
// ranks' values in rank order from +0 (R14).  Tiles with more than kWarpEnt entries
// search the message blocks instead.
constexpr int kWarpEnt = 256;

// tab_woff != 0: every rank's block carries its range table (k_tab) at word tab_woff and
// the layer views come from the headers (no k6_prep); 0: dec_start / dec_lay from k6_prep
__global__ void __launch_bounds__(kThreads)
k6_scatter(Ws w, int L, int p, MsgSrc src, uint32_t hdr_words, uint32_t total_dec_tiles,
           float scale, uint32_t tab_woff) {
    pdl_wait();
    TlMark tlm(w.tl, TL_SCATTER);
    extern __shared__ uint32_t s_lay[];   // tab_woff: [p][L+1] offsets, [p][L+1] ASQ offsets
    __shared__ uint32_t s_tb[RGC_MAX_LAYERS + 1];
    __shared__ uint32_t s_rng[kWarps][2 * kMaxRanks];
    __shared__ uint32_t s_pre[kWarps][kMaxRanks + 1];
    __shared__ uint4 s_v[kWarps][kMaxRanks];
    __shared__ uint2 s_ent[kWarps][kWarpEnt];
    __shared__ uint32_t s_seen[kWarps][kDecTile / 32], s_dup[kWarps][kDecTile / 32];
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    for (int l = tid; l < L; l += kThreads) s_tb[l] = w.ddesc[l].tile_begin;
    if (tid == 0) s_tb[L] = total_dec_tiles;
    for (int i = tid; i < kWarps * (kDecTile / 32); i += kThreads) {
        (&s_seen[0][0])[i] = 0u;
        (&s_dup[0][0])[i] = 0u;
    }
    if (tab_woff) load_layout(src, L, p, s_lay, s_lay + p * (L + 1));   // (synchronises)
    __syncthreads();
    const uint32_t nslots = total_dec_tiles + L;
    uint32_t *rng = s_rng[wp], *pre = s_pre[wp];
    uint4 *sv = s_v[wp];
    uint2 *ent = s_ent[wp];
    uint32_t *seen = s_seen[wp], *dup = s_dup[wp];
    auto rank_of = [&](uint32_t e) {             // last r with pre[r] <= e
        int r = 0, hi = p - 1;
        while (r < hi) {
            const int mid = (r + hi + 1) >> 1;
            if (pre[mid] <= e) r = mid; else hi = mid - 1;
        }
        return r;
    };
    for (uint32_t tile = blockIdx.x * kWarps + wp; tile < total_dec_tiles;
         tile += gridDim.x * kWarps) {
        const int l = find_layer(s_tb, L, tile);
        const DecompDesc &dd = w.ddesc[l];
        const uint32_t lt = tile - s_tb[l];
        for (int r = lane; r < p; r += 32) {
            if (tab_woff) {
                const uint32_t *hr = reinterpret_cast<const uint32_t *>(src.of(r));
                const uint32_t *ds = hr + tab_woff + dd.slot_begin + lt;
                rng[2 * r] = ds[0];
                rng[2 * r + 1] = ds[1];
                const uint32_t *o = s_lay + r * (L + 1), *ao = s_lay + (p + r) * (L + 1);
                // layer_view without the header load for a plain layer (no ASQ entries before
                // the next layer's: its value word is RGC_MSG_DENSE)
                const bool asq = ao[l + 1] != ao[l];
                sv[r] = asq ? make_uint4(2u * (o[L] - ao[L]) + ao[l], 1u, hr[L + 2 + l], o[l])
                            : make_uint4(2u * (o[l] - ao[l]), 2u, RGC_MSG_DENSE, o[l]);
            } else {
                const uint32_t *ds = w.dec_start + (uint64_t)r * nslots + dd.slot_begin + lt;
                rng[2 * r] = ds[0];
                rng[2 * r + 1] = ds[1];
                sv[r] = w.dec_lay[r * L + l];
            }
        }
        __syncwarp();
        // pre[r] = entries of ranks < r (warp scan over ranks, 32 at a time)
        uint32_t carry = 0;
        for (int r0 = 0; r0 < p; r0 += 32) {
            const int r = r0 + lane;
            const uint32_t c = r < p ? rng[2 * r + 1] - rng[2 * r] : 0u;
            uint32_t x = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULLMASK, x, o);
                if (lane >= o) x += y;
            }
            if (r < p) pre[r] = carry + x - c;
            carry += __shfl_sync(FULLMASK, x, 31);
        }
        if (lane == 0) pre[p] = carry;
        __syncwarp();
        const uint32_t S = carry;
        float *out = dd.out;
        if (S <= (uint32_t)kWarpEnt) {
            // stage the tile's entries, 4 independent loads in flight per lane
            for (uint32_t e0 = lane; e0 < S; e0 += 128) {
                uint2 v[4];
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const uint32_t e = e0 + 32 * j;
                    if (e < S) {
                        const int r = rank_of(e);
                        const uint32_t *pw = reinterpret_cast<const uint32_t *>(src.of(r)) + hdr_words;
                        v[j] = view_entry(pw, sv[r], rng[2 * r] + (e - pre[r]));
                    }
                }
#pragma unroll
                for (int j = 0; j < 4; j++)
                    if (e0 + 32 * j < S) ent[e0 + 32 * j] = v[j];
            }
            __syncwarp();
            // tile bitmaps: indices seen once / more than once (only the touched words
            // are cleared again below, so the maps stay zero between tiles)
            const uint32_t t0 = lt * (uint32_t)kDecTile;
            for (uint32_t e = lane; e < S; e += 32) {
                const uint32_t li = ent[e].x - t0, bit = 1u << (li & 31);
                if (atomicOr(&seen[li >> 5], bit) & bit) atomicOr(&dup[li >> 5], bit);
            }
            __syncwarp();
            const bool al32 = kSectorStore && ((uintptr_t)out & 31u) == 0;
            for (uint32_t e = lane; e < S; e += 32) {
                const uint2 pr = ent[e];
                const uint32_t li = pr.x - t0;
                RGC_DCHECK(pr.x < dd.n && li < (uint32_t)kDecTile);
                // this index alone in its 32-byte sector (the tile starts sector-aligned)
                const bool alone = al32 && __popc((seen[li >> 5] >> (li & 24u)) & 0xFFu) == 1;
                if (!((dup[li >> 5] >> (li & 31)) & 1u)) {   // one rank sent it: +0 + v (R14)
                    const float v = __fmul_rn(__fadd_rn(0.f, __uint_as_float(pr.y)), scale);
                    if (alone) store_alone_in_sector(out, pr.x, v); else out[pr.x] = v;
                    continue;
                }
                // several ranks sent it (rare): the lowest rank's entry sums in rank order
                const int r = rank_of(e);
                bool lead = true;
                for (uint32_t f = 0; f < pre[r] && lead; f++) lead = ent[f].x != pr.x;
                if (!lead) continue;
                float acc = __fadd_rn(0.f, __uint_as_float(pr.y));
                for (uint32_t f = pre[r + 1]; f < S; f++)   // rank-major = rank order
                    if (ent[f].x == pr.x) acc = __fadd_rn(acc, __uint_as_float(ent[f].y));
                if (alone) store_alone_in_sector(out, pr.x, __fmul_rn(acc, scale));
                else out[pr.x] = __fmul_rn(acc, scale);
            }
            __syncwarp();
            for (uint32_t e = lane; e < S; e += 32) {
                const uint32_t li = ent[e].x - t0;
                seen[li >> 5] = 0u;
                dup[li >> 5] = 0u;
            }
        } else {
            for (uint32_t e = lane; e < S; e += 32) {
                const int r = rank_of(e);
                const uint32_t *pw_r = reinterpret_cast<const uint32_t *>(src.of(r)) + hdr_words;
                const uint2 pr = view_entry(pw_r, sv[r], rng[2 * r] + (e - pre[r]));
                uint32_t bits;
                bool lead = true;
                for (int q = 0; q < r && lead; q++) {
                    const uint32_t *pq = reinterpret_cast<const uint32_t *>(src.of(q)) + hdr_words;
                    lead = !find_pair(pq, sv[q], rng[2 * q], rng[2 * q + 1], pr.x, &bits);
                }
                if (!lead) continue;
                float acc = __fadd_rn(0.f, __uint_as_float(pr.y));
                for (int q = r + 1; q < p; q++) {
                    const uint32_t *pq = reinterpret_cast<const uint32_t *>(src.of(q)) + hdr_words;
                    if (find_pair(pq, sv[q], rng[2 * q], rng[2 * q + 1], pr.x, &bits))
                        acc = __fadd_rn(acc, __uint_as_float(bits));
                }
                out[pr.x] = __fmul_rn(acc, scale);
            }
        }
        __syncwarp();
    }
}

cudaError_t launch_k6_fill(const FillTable &t, unsigned int *sig, int grid, cudaStream_t s) {
    static unsigned long long *dbg = nullptr;
    static const bool want = getenv("RGC_FILL_DEBUG") != nullptr;   // placement diagnostics
    static int calls = 0;
    if (want && !dbg) cudaMalloc(&dbg, 3 * 8 * 1024);
    if (want && calls++ % 10 == 9) {   // report the previous call
        static unsigned long long h[3 * 1024];
        cudaDeviceSynchronize();
        cudaMemcpy(h, dbg, sizeof(h), cudaMemcpyDeviceToHost);
        const int nw = (int)h[3 * 1023];
        unsigned long long t0 = ~0ull, t1 = 0, s1 = 0;
        for (int i = 0; i < nw && i < 1000; i++) {
            t0 = h[3 * i + 1] < t0 ? h[3 * i + 1] : t0;
            s1 = h[3 * i + 1] > s1 ? h[3 * i + 1] : s1;
            t1 = h[3 * i + 2] > t1 ? h[3 * i + 2] : t1;
        }
        fprintf(stderr, "fill debug: %d CTAs, %d active (one per SM), start spread %.1f us, "
                        "span %.1f us\n", grid, nw, (s1 - t0) * 1e-3, (t1 - t0) * 1e-3);
    }
    k6_fill<<<grid, kFillThreads, 0, s>>>(t, sig, want ? dbg : nullptr);
    return cudaGetLastError();
}

cudaError_t launch_k6_scatter(const Ws &w, int L, int p, const MsgSrc &src, uint32_t hdr_words,
                              uint32_t total_dec_tiles, uint32_t max_pairs, float scale, int grid,
                              cudaStream_t s, uint32_t tab_woff) {
    if (p == 1) {
        const uint64_t g = ((uint64_t)max_pairs + kThreads - 1) / kThreads;
        const int gr = (int)(g < (uint64_t)grid ? (g ? g : 1) : (uint64_t)grid);
        return launch_pdl(k6_scatter1, gr, kThreads, 0, s, w, L, src, hdr_words, max_pairs, scale);
    } else {
        const size_t smem = tab_woff ? (size_t)2 * p * (L + 1) * sizeof(uint32_t) : 0;
        static cudaError_t attr = cudaFuncSetAttribute(
            (const void *)k6_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
            (int)((size_t)2 * kMaxRanks * (RGC_MAX_LAYERS + 1) * sizeof(uint32_t)));
        if (attr != cudaSuccess) return attr;
        return launch_pdl(k6_scatter, grid, kThreads, smem, s, w, L, p, src, hdr_words, total_dec_tiles,
                          scale, tab_woff);
    }
    return cudaGetLastError();
}

}  // namespace rgc
