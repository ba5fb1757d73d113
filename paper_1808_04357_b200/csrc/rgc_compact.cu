// rgc_compact.cu -- K3: ordered stream compaction nonzero_indices(|X| > t)
// with the gather of values and the
// residual / momentum masking V <- V (.) (1 - Masks).
//
// Work unit: a segment of consecutive elements of one layer's source -- the
// residual V (pass A: 65536 elements), one K1 stash record (pass A), or the
// ascending Alg.2 survivor list S / V in the exact emission (pass B: 8192
// elements, so a large set spreads over many CTAs).  Each of the 8 warps of a
// CTA owns a contiguous 1/8 chunk of the segment and
// streams it with no block barrier: 128-bit loads, one ballot per (128-element
// round, slot), popc ranks, and an in-order copy of the chunk's candidates into
// a warp-private shared-memory stash.  One decoupled look-back per segment
// (warp-wide window over 32 predecessors) gives the segment's global offsets;
// the stashes are then written out in index order.  A warp whose candidates
// overflow its stash re-reads its chunk and writes directly (pass 2).
// Exact-top-k emission (PASS 1) also takes the first q elements equal to the
// k-th key (lower index wins, R6) using a second ballot.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "rgc_device.cuh"

namespace rgc {

constexpr int kWarpStash = kStash / kWarps;     // 512 pairs per warp



// one 512-element round of a warp over V: lane holds 4 x float4 at
// pos + j*128 + lane*4 (j = 0..3); index order = (j, lane, slot)
__device__ __forceinline__ void load_round_v(const float *V, uint32_t pos, uint32_t nsrc,
                                             float4 *x) {
    const int lane = threadIdx.x & 31;
    if (pos + 512 <= nsrc) {
#pragma unroll
        for (int j = 0; j < 4; j++)
            x[j] = __ldcs(reinterpret_cast<const float4 *>(V + pos + j * 128 + lane * 4));
    } else {
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t p = pos + j * 128 + lane * 4;
            x[j].x = p + 0 < nsrc ? V[p + 0] : 0.f;
            x[j].y = p + 1 < nsrc ? V[p + 1] : 0.f;
            x[j].z = p + 2 < nsrc ? V[p + 2] : 0.f;
            x[j].w = p + 3 < nsrc ? V[p + 3] : 0.f;
        }
    }
}

__device__ __forceinline__ uint32_t f4get(const float4 &v, int s) {
    return __float_as_uint(s == 0 ? v.x : (s == 1 ? v.y : (s == 2 ? v.z : v.w)));
}

// Ballots of one round: gt = |x| > T, eq = |x| == T (TIE only).  Elements past
// nsrc are excluded.
template <bool FROM_S, bool TIE>
__device__ __forceinline__ void ballots(const uint32_t *vb, uint32_t pos, uint32_t nsrc,
                                        uint32_t T, uint32_t skx, uint32_t ska, uint32_t *gtb,
                                        uint32_t *eqb) {
    const int lane = threadIdx.x & 31;
    constexpr int NI = 16;
#pragma unroll
    for (int i = 0; i < NI; i++) {
        const uint32_t p = FROM_S ? pos + i * 32 + lane : pos + (i >> 2) * 128 + lane * 4 + (i & 3);
        const bool valid = p < nsrc;
        const uint32_t kk = skey(vb[i], skx, ska);
        gtb[i] = __ballot_sync(FULLMASK, valid && kk > T);
        eqb[i] = TIE ? __ballot_sync(FULLMASK, valid && kk == T) : 0u;
    }
}

// A segment of several K1 candidate records: their pieces of consecutive K1 CTAs' stash
// regions concatenated, flat index p -> record j = the last with pref[j] <= p, entry
// roff[j] + p - pref[j] of region j (cand_R pairs each)
struct StashMap {
    const uint32_t *pref;   // shared: exclusive prefix of the record counts, npref + 1 entries
    const uint32_t *roff;   // shared: the records' offsets in their regions
    int npref;
    const uint2 *base;      // region of the segment's first record
    uint32_t cand_R;
};

// Load one round (V: 512 elements as 4x4 per lane; S: 16 x 32 pairs, one per lane, from the
// survivor list / one stash record, or through sm when sm.pref is set)
template <bool FROM_S>
__device__ __forceinline__ void load_round(const float *V, const uint2 *src, uint32_t pos,
                                           uint32_t nsrc, uint32_t *vb, uint32_t *ix,
                                           const StashMap &sm) {
    const int lane = threadIdx.x & 31;
    if (FROM_S && sm.pref) {
        // the lane's 16 indices ascend: walk the record forward from the first one's
        int j = find_layer(sm.pref, sm.npref, min(pos + lane, nsrc > 0 ? nsrc - 1 : 0u));
#pragma unroll
        for (int i = 0; i < 16; i++) {
            const uint32_t p = pos + i * 32 + lane;
            uint2 pr = make_uint2(0u, 0u);
            if (p < nsrc) {
                while (j + 1 < sm.npref && sm.pref[j + 1] <= p) j++;
                pr = __ldcg(&sm.base[(uint64_t)j * sm.cand_R + sm.roff[j] + (p - sm.pref[j])]);
            }
            vb[i] = pr.y;
            ix[i] = pr.x;
        }
        return;
    }
    if (!FROM_S) {
        float4 x[4];
        load_round_v(V, pos, nsrc, x);
#pragma unroll
        for (int i = 0; i < 16; i++) {
            vb[i] = f4get(x[i >> 2], i & 3);
            ix[i] = pos + (i >> 2) * 128 + lane * 4 + (i & 3);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 16; i++) {
            const uint32_t p = pos + i * 32 + lane;
            const uint2 pr = p < nsrc ? src[p] : make_uint2(0u, 0u);
            vb[i] = pr.y;
            ix[i] = pr.x;
        }
    }
}

// Number of elements of the round before this lane's element i, among mask bits
// of all 16 (round-major) ballots, in index order.
//   V order: (j, lane, slot) with i = 4j + slot;  S order: (i, lane).
template <bool FROM_S>
__device__ __forceinline__ uint32_t rank_before(const uint32_t *m, int i) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t r = 0;
    if (FROM_S) {
#pragma unroll
        for (int t = 0; t < 16; t++)
            if (t < i) r += __popc(m[t]);
        r += __popc(m[i] & lt);
    } else {
        const int j = i >> 2, s = i & 3;
#pragma unroll
        for (int t = 0; t < 16; t++) {
            const int tj = t >> 2, ts = t & 3;
            if (tj < j) r += __popc(m[t]);
            else if (tj == j) r += __popc(m[t] & lt) + ((ts < s) ? ((m[t] >> lane) & 1u) : 0u);
        }
    }
    return r;
}

// CTAs per SM the register allocation must allow: pass A (the common path, ~460 stash
// records on VGG16) and pass B (exact emission; its tie-quota code needs more registers)
#ifndef RGC_K3A_MINB
#define RGC_K3A_MINB 1
#endif
#ifndef RGC_K3_MINB
#define RGC_K3_MINB 1
#endif
template <int PASS>
__global__ void __launch_bounds__(kThreads, PASS == 0 ? RGC_K3A_MINB : RGC_K3_MINB)
k3_compact(Ws w, int L, uint2 *msg_pairs) {
    pdl_wait();
    TlMark tlm(w.tl, PASS == 0 ? TL_K3A : TL_K3B);
    constexpr bool TIE = (PASS == 1);
    __shared__ uint2 s_stash[kStash];
    __shared__ uint32_t s_tb[RGC_MAX_LAYERS + 1];
    __shared__ uint32_t s_seg;
    __shared__ uint32_t s_pref[65], s_roff[64];
    __shared__ uint32_t s_wg[kWarps], s_we[kWarps], s_wo[kWarps];
    __shared__ unsigned long long s_ex;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t total = PASS == 0 ? w.ctrl->k3a_total : w.ctrl->k3b_total;
    if (total == 0) return;
    for (int l = tid; l < L; l += kThreads) s_tb[l] = PASS == 0 ? w.st[l].k3a_begin : w.st[l].k3b_begin;
    if (tid == 0) s_tb[L] = total;
    unsigned int *ticket = PASS == 0 ? &w.ctrl->ticketA : &w.ctrl->ticketB;
    unsigned long long *status = PASS == 0 ? w.statusA : w.statusB;
    uint2 *wst = s_stash + warp * kWarpStash;

    for (;;) {
        if (tid == 0) s_seg = atomicAdd(ticket, 1u);
        __syncthreads();
        const uint32_t seg = s_seg;
        if (seg >= total) break;
        const int l = find_layer(s_tb, L, seg);
        const uint32_t ls = seg - s_tb[l];
        const LayerDesc &d = w.desc[l];
        LayerState &S = w.st[l];
        const uint32_t mode = S.mode;
        const uint32_t skx = S.skx, ska = S.ska;
        bool fromS = (PASS == 1 && mode == MODE_SURV);
        uint32_t T, q;
        uint2 *dst;
        bool zero;
        if (PASS == 0) {
            // Alg.3 set {|V| > t} straight into the message, or Alg.2 survivors into S
            T = S.thr_key; q = 0;
            zero = (mode == MODE_THRESH);
            dst = zero ? (d.quant ? w.Q : msg_pairs) + S.msg_off : w.S + d.s_off;
        } else {
            // exact top-k: {|x| > T*} plus the first q elements with |x| == T*
            T = S.rs_prefix; q = S.rs_krem;
            zero = true;
            dst = (d.quant ? w.Q : msg_pairs) + S.msg_off;
        }
        uint32_t nsrc = fromS ? S.surv : d.n;
#ifdef RGC_CHECK
        const uint32_t dlim = (PASS == 0 && !zero) ? d.s_cap : max(d.cap, d.k);
#endif
        // pass A over V: 65536-element segments (8192 measured slower on stash-miss layers);
        // pass B (exact emission over the survivors or V): 8192-element segments, so a large
        // set spreads over many CTAs; pass A from the K1 stash takes one record per segment
        constexpr uint32_t SEG = PASS == 0 ? kSegA : kSegB, WCH = SEG / kWarps;
        uint32_t c0 = ls * SEG + warp * WCH;                            // this warp's chunk
        uint32_t c1 = min(c0 + WCH, nsrc);
        const uint2 *src = w.S + d.s_off;
        StashMap sm = {nullptr, nullptr, 0, nullptr, 0u};
#ifndef RGC_NO_RECSRC
        if (PASS == 0 && S.cand_ok && w.seg_ch > 1) {
            // K1 stashed the candidates in small records: segment ls = the layer's records
            // ls * seg_ch ... (pieces of consecutive K1 CTAs' regions, in index order), one
            // flat index through the prefix of their counts
            const uint32_t q0 = ls * w.seg_ch;
            const uint32_t nck = min(w.seg_ch, d.cand_nb - q0);
            const uint2 rec_t = tid < (int)nck ? __ldcg(&w.rec[d.rec_base + q0 + tid]) : make_uint2(0u, 0u);
            uint32_t inc = rec_t.y;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULLMASK, inc, o);
                if (lane >= o) inc += y;
            }
            if (tid < 64) { s_pref[tid + 1] = inc; s_roff[tid] = rec_t.x; }
            if (tid == 0) s_pref[0] = 0u;
            __syncthreads();
            if (tid >= 32 && tid < 64) s_pref[tid + 1] += s_pref[32];
            __syncthreads();
            sm.pref = s_pref;
            sm.roff = s_roff;
            sm.npref = (int)nck;
            sm.base = w.cand + (uint64_t)(d.cand_b0 + q0) * w.cand_R;
            sm.cand_R = w.cand_R;
            nsrc = s_pref[nck];
            const uint32_t per = ((nsrc + kWarps - 1) / kWarps + 511u) / 512u * 512u;
            c0 = min(nsrc, warp * per);
            c1 = min(nsrc, c0 + per);
            fromS = true;
        } else if (PASS == 0 && S.cand_ok) {
            // K1 stashed the candidates: segment ls = the record of K1 CTA cand_b0 + ls
            const uint2 rec = w.rec[d.rec_base + ls];
            src = w.cand + (uint64_t)(d.cand_b0 + ls) * w.cand_R + rec.x;
            nsrc = rec.y;
            const uint32_t per = ((nsrc + kWarps - 1) / kWarps + 511u) / 512u * 512u;
            c0 = min(nsrc, warp * per);
            c1 = min(nsrc, c0 + per);
            fromS = true;
        }
#endif
        float *V = d.V;
        float *u = d.u;

        // ---- pass 1 (per warp, no block barrier): count + stash candidates in order
        uint32_t cg = 0, ce = 0;
        bool over = false;
        for (uint32_t pos = c0; pos < c1; pos += 512) {
            uint32_t vb[16], ix[16], gtb[16], eqb[16];
            if (!fromS) {
                load_round<false>(V, src, pos, nsrc, vb, ix, sm);
                ballots<false, TIE>(vb, pos, nsrc, T, skx, ska, gtb, eqb);
            } else {
                load_round<true>(V, src, pos, nsrc, vb, ix, sm);
                ballots<true, TIE>(vb, pos, nsrc, T, skx, ska, gtb, eqb);
            }
            uint32_t cm[16];
            uint32_t rc = 0, rg = 0, re = 0;
#pragma unroll
            for (int i = 0; i < 16; i++) {
                cm[i] = gtb[i] | eqb[i];
                rc += __popc(cm[i]); rg += __popc(gtb[i]); re += __popc(eqb[i]);
            }
            if (rc) {
                const uint32_t at = cg + ce;
                if (!over && at + rc <= (uint32_t)kWarpStash) {
#pragma unroll
                    for (int i = 0; i < 16; i++) {
                        if ((cm[i] >> lane) & 1u) {
                            const uint32_t r = fromS ? rank_before<true>(cm, i) : rank_before<false>(cm, i);
                            wst[at + r] = make_uint2(ix[i], vb[i]);
                        }
                    }
                } else {
                    over = true;
                }
            }
            cg += rg; ce += re;
        }
        if (lane == 0) { s_wg[warp] = cg; s_we[warp] = ce; s_wo[warp] = over; }
        __syncthreads();
        uint32_t pg = 0, pe = 0, lg = 0, le = 0, anyover = 0;
#pragma unroll
        for (int i = 0; i < kWarps; i++) {
            if (i < warp) { pg += s_wg[i]; pe += s_we[i]; }
            lg += s_wg[i]; le += s_we[i]; anyover |= s_wo[i];
        }

        // ---- one decoupled look-back per segment (packed gt:31 | eq:31)
        if (warp == 0) {
            const unsigned long long agg = ((unsigned long long)lg << 31) | le;
            unsigned long long ex = 0;
            if (ls == 0) {
                if (lane == 0) st_volatile_u64(&status[seg], kFlagInc | agg);
            } else {
                if (lane == 0) st_volatile_u64(&status[seg], kFlagAgg | agg);
                int j = (int)seg - 1 - lane;        // window of 32 predecessors
                const int first = (int)(seg - ls); // this layer's first segment
                for (;;) {
                    // warp-uniform wait until every in-layer predecessor of the window published
                    unsigned long long v = 0;
                    bool ready = j < first;
                    while (!__all_sync(FULLMASK, ready)) {
                        if (!ready) {
                            v = ld_volatile_u64(&status[j]);
                            ready = (v >> 62) != 0;
                        }
                    }
                    const bool inc = (j < first) || ((v >> 62) == 2);
                    const uint32_t incm = __ballot_sync(FULLMASK, inc);
                    const int stop = incm ? __ffs(incm) - 1 : 32;   // nearest inclusive lane
                    unsigned long long add = (lane <= stop && j >= first) ? (v & kCntMask) : 0ull;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(FULLMASK, add, o);
                    ex += add;
                    if (incm) break;
                    j -= 32;
                }
                if (lane == 0) st_volatile_u64(&status[seg], kFlagInc | (ex + agg));
            }
            if (lane == 0) {
                s_ex = ex;
                const uint32_t nseg = PASS == 0 ? S.k3a_tiles : S.k3b_tiles;
                if (ls + 1 == nseg) {   // last segment of the layer: pairs actually written
                    const uint32_t tg = (uint32_t)((ex + agg) >> 31);
                    const uint32_t te = (uint32_t)((ex + agg) & 0x7FFFFFFFull);
                    const uint32_t emitted = tg + min(te, q);
                    if (PASS == 0) S.emitted_a = emitted; else S.emitted_b = emitted;
                }
            }
        }
        __syncthreads();
        const unsigned long long ex = s_ex;
        // running (gt, eq) ranks at the start of this warp's chunk
        uint32_t gb0 = (uint32_t)(ex >> 31) + pg;
        uint32_t eb0 = (uint32_t)(ex & 0x7FFFFFFFull) + pe;

        if (!anyover && !TIE) {
            // ---- write the warp's stash: <index, value> + masking
            for (uint32_t j = lane; j < cg; j += 32) {
                const uint2 e = wst[j];
                RGC_DCHECK(gb0 + j < dlim && e.x < d.n, "pass %d seg %u l %d gb0 %u j %u dlim %u ex %llx e.x %u n %u\n",
                         PASS, seg, l, gb0, j, dlim, (unsigned long long)ex, e.x, d.n);
                dst[gb0 + j] = e;
                if (zero) { V[e.x] = 0.0f; if (u) u[e.x] = 0.0f; }
            }
        } else if (!anyover) {
            // tie quota: walk the stash 32 entries at a time in index order
            const uint32_t nc = cg + ce;
            for (uint32_t b = 0; b < nc; b += 32) {
                const uint32_t j = b + lane;
                const bool ok = j < nc;
                const uint2 e = ok ? wst[j] : make_uint2(0u, 0u);
                const uint32_t kk = skey(e.y, skx, ska);
                const bool isg = ok && kk > T, ise = ok && kk == T;
                const uint32_t G = __ballot_sync(FULLMASK, isg), E = __ballot_sync(FULLMASK, ise);
                const uint32_t lt = (1u << lane) - 1u;
                const uint32_t gb = gb0 + __popc(G & lt), eb = eb0 + __popc(E & lt);
                if (isg || (ise && eb < q)) {
                    const uint32_t outpos = isg ? gb + min(eb, q) : gb + eb;
                    RGC_DCHECK(outpos < dlim && e.x < d.n, "tie seg %u\n", seg);
                    dst[outpos] = e;
                    V[e.x] = 0.0f;
                    if (u) u[e.x] = 0.0f;
                }
                gb0 += __popc(G); eb0 += __popc(E);
            }
        } else {
            // ---- pass 2 (a stash overflowed): every warp re-reads its chunk, writes directly
            for (uint32_t pos = c0; pos < c1; pos += 512) {
                uint32_t vb[16], ix[16], gtb[16], eqb[16];
                if (!fromS) {
                    load_round<false>(V, src, pos, nsrc, vb, ix, sm);
                    ballots<false, TIE>(vb, pos, nsrc, T, skx, ska, gtb, eqb);
                } else {
                    load_round<true>(V, src, pos, nsrc, vb, ix, sm);
                    ballots<true, TIE>(vb, pos, nsrc, T, skx, ska, gtb, eqb);
                }
                uint32_t rg = 0, re = 0;
#pragma unroll
                for (int i = 0; i < 16; i++) { rg += __popc(gtb[i]); re += __popc(eqb[i]); }
                if (rg | re) {
#pragma unroll
                    for (int i = 0; i < 16; i++) {
                        const bool isg = (gtb[i] >> lane) & 1u, ise = (eqb[i] >> lane) & 1u;
                        if (isg || ise) {
                            const uint32_t gr = gb0 + (fromS ? rank_before<true>(gtb, i) : rank_before<false>(gtb, i));
                            const uint32_t er = eb0 + (fromS ? rank_before<true>(eqb, i) : rank_before<false>(eqb, i));
                            if (isg || er < q) {
                                const uint32_t outpos = isg ? gr + min(er, q) : gr + er;
                                RGC_DCHECK(outpos < dlim && ix[i] < d.n, "p2 seg %u\n", seg);
                                dst[outpos] = make_uint2(ix[i], vb[i]);
                                if (zero) { V[ix[i]] = 0.0f; if (u) u[ix[i]] = 0.0f; }
                            }
                        }
                    }
                }
                gb0 += rg; eb0 += re;
            }
        }
        __syncthreads();
    }
}

cudaError_t launch_k3(const Ws &w, int L, int pass, uint2 *msg_pairs, int grid, cudaStream_t s) {
    if (pass == 0) return launch_pdl(k3_compact<0>, grid, kThreads, 0, s, w, L, msg_pairs);
    return launch_pdl(k3_compact<1>, grid, kThreads, 0, s, w, L, msg_pairs);
}

cudaError_t occupancy_k3(int *k3) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(k3, k3_compact<0>, kThreads, 0);
}

}  // namespace rgc
