// rgc_kernels.cu -- sm_100a kernels of the RGC synchronisation hot path.
//
//   K1 k1_accumulate : u = m*u + g ; V += u + max|V| and mean_fx
//                      (R2) in the same HBM pass; last CTA per layer finalises the
//                      statistics and the threshold table
//   K2 k2_count      : count_nonzero(|V| > t) for every Alg.2 level (register
//                      counters) or a one-pass 1026-bin histogram over the 1025
//                      Alg.3 thresholds; last CTA per layer runs Alg.2's level choice
//                       or Alg.3's binary search on the counts
//   K3 k3_compact    : ordered stream compaction nonzero_indices(|V| > t) (P:183,
//                      P:219) with warp ballot/popc ranks, decoupled look-back
//                      between tiles, gather of values and the
//                      residual/momentum masking in the same pass
//   K4 k4_radix      : radixSelect of the k-th largest |V| over
//                      the Alg.2 survivors or over V (fallback), 11/11/9-bit digits
//   K6 k6_decompress : rank-ordered scatter-add of all gathered sets into the dense
//                      averaged gradient (R13, R14) per 8192-element tile
//                      in shared memory, 128-bit stores
// No tensor cores: nothing on this path is a dense contraction.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "rgc_device.cuh"

namespace rgc {

// lowest Alg.3 threshold index whose count this call bins exactly
// Stash / bounded-histogram prediction policy (only decides which pass reads what; the
// results never depend on it).  c_tune = {halve the Alg.3 margin when c(t_jlo) > X*k,
// smallest margin, tighten the stash key when it stashed > R x what the call needed
// (0: never), largest shift, F: an Alg.3 layer's next stash key sits at the highest
// level whose count reached F*k (0: at this call's t_jlo)}.  Measured on VGG16 (tools/gpu_tune.sh): tighter settings
// shrink the stash ~2x but the selection kernels are latency-bound, not record-bound,
// and the step time did not move beyond run-to-run noise; the defaults stay wide.  Defaults set by set_tuning() (rgc_init; RGC_TUNE env).
__constant__ uint32_t c_tune[5];
cudaError_t set_tuning(const uint32_t *t) { return cudaMemcpyToSymbol(c_tune, t, sizeof(c_tune)); }

// lowest Alg.3 level a residual pass bins: the previous call's chosen level minus a margin
__device__ __forceinline__ uint32_t bs_jlo_hint(const LayerHot &S) {
    const uint32_t margin = S.margin ? S.margin : 64u;
    return S.jhint > margin ? S.jhint - margin : 0u;
}
// this call's lowest exactly-counted level (K1 decides: from the stash key when the stash
// serves K2, else bs_jlo_hint); pass 1 is the full histogram
__device__ __forceinline__ uint32_t bs_jlo(const LayerHot &S, int pass) {
    return pass == 1 ? 0u : S.jlo_cur;
}

// stash key scale 1 - 2^-shift (shift 0 in a fresh workspace = the default 4)
__device__ __forceinline__ uint32_t stash_shift(const LayerHot &S) {
    return S.stash_shift ? S.stash_shift : 4u;
}

// A finalisation's working copies (all threads of the CTA; L2, not L1: other CTAs wrote the
// state since this SM may have cached it).  hot_load + desc_load are one round trip.
__device__ __forceinline__ void hot_load(LayerHot &dst, const LayerHot &src) {
    const uint4 *s = reinterpret_cast<const uint4 *>(&src);
    uint4 *d = reinterpret_cast<uint4 *>(&dst);
    for (int i = threadIdx.x; i < (int)(sizeof(LayerHot) / 16); i += blockDim.x) d[i] = __ldcg(s + i);
}
__device__ __forceinline__ void hot_store(LayerHot &dst, const LayerHot &src) {
    const uint4 *s = reinterpret_cast<const uint4 *>(&src);
    uint4 *d = reinterpret_cast<uint4 *>(&dst);
    for (int i = threadIdx.x; i < (int)(sizeof(LayerHot) / 16); i += blockDim.x) __stcg(d + i, s[i]);
}
__device__ __forceinline__ void desc_load(LayerDesc &dst, const LayerDesc &src) {
    static_assert(sizeof(LayerDesc) % 8 == 0, "LayerDesc moves as uint2");
    const uint2 *s = reinterpret_cast<const uint2 *>(&src);
    uint2 *d = reinterpret_cast<uint2 *>(&dst);
    for (int i = threadIdx.x; i < (int)(sizeof(LayerDesc) / 8); i += blockDim.x) d[i] = s[i];
}

// ============================================================================
// K1: residual accumulation + momentum correction + statistics + candidate stash
// ============================================================================
__device__ void k1_finalize(const Ws &w, int l, unsigned long long *s_bins, uint32_t *s_misc) {
    TlMark tlm(w.tl, TL_K1F);
    __threadfence();
    LayerState &G = w.st[l];
    __shared__ LayerHot s_hot;
    __shared__ LayerDesc s_desc;
    __shared__ uint32_t s_jlo;   // lowest Alg.3 level with t_j >= the stash key
    __shared__ uint32_t s_acc[3];
    LayerHot &S = s_hot;
    const LayerDesc &d = s_desc;
    hot_load(s_hot, G);
    desc_load(s_desc, w.desc[l]);
    for (int b = threadIdx.x; b < kMeanBins; b += kThreads)
        s_bins[b] = atomicExch(&G.bins[b], 0ull);
    if (threadIdx.x == 0) {
        s_misc[0] = atomicExch(&G.maxkey_acc, 0u);
        s_acc[0] = atomicExch(&G.k1_cnt, 0u);    // sampled-BS reuse count (0 on other calls)
        s_acc[1] = atomicExch(&G.cand_bad, 0u);
        s_acc[2] = atomicExch(&G.cand_acc, 0u);
        G.k1_done = 0;
        s_jlo = 0xFFFFFFFFu;
    }
    __syncthreads();
    tl_probe(w.tl, TL_P0 + 0);
    __shared__ double s_mean;
    __shared__ uint32_t s_flags;
    __shared__ uint32_t s_nz[(kMeanBins + 31) / 32];
    if (threadIdx.x < 32) {
        // which exponent bins are non-zero (adding a zero term leaves the sum's bits unchanged)
        for (int b0 = 0; b0 < kMeanBins; b0 += 32) {
            const int b = b0 + threadIdx.x;
            const uint32_t m = __ballot_sync(FULLMASK, b < kMeanBins && s_bins[b] != 0ull);
            if (threadIdx.x == 0) s_nz[b0 / 32] = m;
        }
    }
    __syncwarp();
    if (threadIdx.x == 0) {
        // mean_fx (R2): sum_E ascending of B[E] * 2^(E-30), then / n, in double
        double acc = 0.0;
        for (int q = 0; q < (kMeanBins + 31) / 32; q++) {
            uint32_t m = s_nz[q];
            while (m) {
                const int b = q * 32 + __ffs(m) - 1;
                m &= m - 1u;
                acc = __dadd_rn(acc, __dmul_rn(__ull2double_rn(s_bins[b]), pow2d((b - 149) - 30)));
            }
        }
        double mean = __ddiv_rn(acc, (double)d.n);
        uint32_t maxkey = s_misc[0];
        uint32_t flags = 0;
        uint32_t mode = MODE_NONE;
        const bool reuse = d.selector == RGC_SEL_SAMPLED_BS && S.cache_valid &&
                           (S.step % d.interval) != 0u;
        if (maxkey >= 0x7F800000u) {
            flags |= RGC_F_NONFINITE;
        } else if (reuse) {
            // sampled BS reuse step: {|V| > t_cached}, counted in this pass
            const uint32_t c = s_acc[0];
            flags |= RGC_F_SAMPLED_REUSE;
            S.reuse_cnt = c;
            if (c > d.cap) {                  // R18
                flags |= RGC_F_CAP_EXACT;
                S.count = d.k;
                if (c <= d.s_cap) {
                    // the exact top-k lies inside {|V| > t_cached} (c >= k of them): select it
                    // from those c survivors (K3A, then K45 / K4 + K3B), not from all of V
                    mode = MODE_SURV;
                    S.thr_key = S.cache_key;
                    S.surv = c;
                } else {
                    mode = MODE_EXACT;
                }
            } else {
                mode = MODE_THRESH;
                S.thr_key = S.cache_key;
                S.count = c;
            }
        } else if (maxkey == 0u || mean == (double)__uint_as_float(maxkey)) {
            flags |= RGC_F_DEGENERATE;       // R10
            mode = MODE_EXACT;
        }
        S.mean = mean;
        S.maxkey = maxkey;
        S.flags = flags;
        S.mode = mode;
        S.cand_ok = 0u;
        // ASQ (R21): this call's phase picks the sign the selection keys keep
        S.ska = d.quant ? 0x80000000u : 0u;
        S.skx = (d.quant && (S.phase & 1u)) ? 0x80000000u : 0u;
        s_mean = mean;
        s_flags = flags;
    }
    __syncthreads();
    tl_probe(w.tl, TL_P0 + 1);
    for (int b = threadIdx.x; b < kMeanBins; b += kThreads) s_bins[b] = 0ull;
    const uint32_t flags = s_flags;
    if (!(flags & (RGC_F_NONFINITE | RGC_F_DEGENERATE | RGC_F_SAMPLED_REUSE))) {
        const double mean = s_mean;
        const double maxd = (double)__uint_as_float(S.maxkey);
        if (d.selector == RGC_SEL_TRIMMED) {
            if (threadIdx.x == 0) {
                // Alg.2 lines 2/5/7: ratio = 1-eps, then ratio -= eps
                double ratio = __dsub_rn(1.0, d.trim_eps);
                for (int j = 0; j < kMaxTrim; j++) {
                    S.tkeys[j] = (j < (int)d.trim_levels)
                                     ? fkey(thresh_at(mean, maxd, ratio)) : 0x7FFFFFFFu;
                    ratio = __dsub_rn(ratio, d.trim_eps);
                }
            }
        } else {
            // Alg.3: every ratio the search can visit is j/1024 (R8).  The lowest level whose
            // key reaches the stash key (the stash verdict below) is found while the table is
            // written: the keys ascend with j, so it is the smallest such j (sentinel 1025)
            const uint32_t ck = S.cand_key;
            for (int j = threadIdx.x; j <= kBsLevels; j += kThreads) {
                const uint32_t kk = fkey(thresh_at(mean, maxd, __dmul_rn((double)j, 0.0009765625)));
                S.tkeys[j] = kk;
                if (kk >= ck) atomicMin(&s_jlo, (uint32_t)j);
            }
            if (threadIdx.x == 0) S.tkeys[kBsLevels + 1] = 0xFFFFFFFFu;
        }
    }
    __syncthreads();
    tl_probe(w.tl, TL_P0 + 2);
    if (threadIdx.x == 0) {
        // The stash holds every |V| > tau (tau = S.cand_key, predicted by the previous
        // call) of this layer iff no CTA overflowed; it serves this call iff tau does not
        // exceed the lowest key the call needs: t_0 (Alg.2 levels), t_jlo (Alg.3's
        // bounded histogram) or the cached threshold (sampled BS reuse step).
        const uint32_t bad = s_acc[1];
        S.cand_total = s_acc[2];
        bool ok = S.stash_on && !(flags & (RGC_F_NONFINITE | RGC_F_DEGENERATE));
        uint32_t sh = stash_shift(S);
        if (ok && bad) { ok = false; sh = min(sh + 1u, c_tune[3]); }  // too many: tighten
        uint32_t jlo = bs_jlo_hint(S);
        if (ok && d.selector != RGC_SEL_TRIMMED && !(flags & RGC_F_SAMPLED_REUSE)) {
            // Alg.3 from the stash: every level with t_j >= tau is counted exactly, so the
            // bounded histogram starts at the lowest such level (a value-space window: it
            // follows this call's thresholds when max|V| jumps, as with heavy tails).  When
            // the counts it gives do not decide the search, K2 re-counts over V (pass 1).
            const uint32_t lo = min(s_jlo, (uint32_t)kBsLevels + 1u);
            if (lo <= kBsLevels) jlo = lo;
            else { ok = false; sh = max(sh, 2u) - 1u; }                     // too few: widen
        } else if (ok) {
            const uint32_t need = (flags & RGC_F_SAMPLED_REUSE) ? S.cache_key
                                  : (d.selector == RGC_SEL_TRIMMED ? S.tkeys[0] : S.tkeys[jlo]);
            if (S.cand_key > need) { ok = false; sh = max(sh, 2u) - 1u; }  // too few: widen
        }
        S.jlo_cur = jlo;
        S.stash_shift = sh;
        S.stash_ok = ok ? 1u : 0u;
        const bool k2src = ok && !(flags & RGC_F_SAMPLED_REUSE);
        S.k2src = k2src ? 1u : 0u;
        if (!k2src) atomicOr(&w.ctrl->any_vpass, 1u);
        if (!k2src && !(flags & (RGC_F_NONFINITE | RGC_F_DEGENERATE | RGC_F_SAMPLED_REUSE))) S.vpass_runs++;
    }
    __syncthreads();
    tl_probe(w.tl, TL_P0 + 3);
    hot_store(G, s_hot);
    __syncthreads();
}

__device__ void k1_flush(const Ws &w, int l, uint32_t ntl, uint32_t cta_max,
                         unsigned long long *s_bins, uint32_t *s_misc, uint32_t rcnt) {
    LayerState &S = w.st[l];
    rcnt = __reduce_add_sync(0xffffffffu, rcnt);
    if ((threadIdx.x & 31) == 0 && rcnt) atomicAdd(&S.k1_cnt, rcnt);
    __syncthreads();
    for (int b = threadIdx.x; b < kMeanBins; b += kThreads) {
        unsigned long long v = s_bins[b];
        if (v) { atomicAdd(&S.bins[b], v); s_bins[b] = 0ull; }
    }
    if (threadIdx.x == 0 && cta_max) atomicMax(&S.maxkey_acc, cta_max);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int old = atomicAdd(&S.k1_done, ntl);
        s_misc[1] = (old + ntl == w.desc[l].ntiles);
    }
    __syncthreads();
    if (s_misc[1]) k1_finalize(w, l, s_bins, s_misc);
}

#ifndef RGC_K1_MINB
#define RGC_K1_MINB 3   // 3 CTAs per SM (<= 85 registers, no spills): K1 489 -> 468 us on VGG16
#endif
__global__ void __launch_bounds__(kThreads, RGC_K1_MINB)
k1_accumulate(Ws w, int L, uint32_t total) {
    pdl_wait();
    if (w.k1cnt && threadIdx.x == 0) atomicAdd(&w.k1cnt[0], 1ull);   // resident (early fill)
    TlMark tlm(w.tl, TL_K1);
    const unsigned long long tlm_start = w.tl ? tl_now() : 0ull;
    __shared__ uint32_t s_tb[RGC_MAX_LAYERS + 1];
    __shared__ unsigned long long s_bins[kMeanBins];
    // per-warp tile maxima, double-buffered by tile parity: with one block barrier per tile a
    // warp may write the next tile's entry while a slower one still reads this tile's
    __shared__ uint32_t s_wmax[2][kWarps];
#ifdef RGC_K1_TWOBAR
    __shared__ unsigned long long s_wsum[kWarps];
#endif
    __shared__ uint32_t s_misc[4];
    __shared__ uint2 s_cst[kWarps][kK1Stash];        // warp-private candidate staging
    __shared__ uint32_t s_tcnt[kK1Batch][kWarps];    // candidates per (tile of the batch, warp)
    __shared__ uint32_t s_toff[kK1Batch][kWarps];    // their offsets in the CTA region
    __shared__ uint32_t s_btot;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int l = tid; l < L; l += kThreads) s_tb[l] = w.desc[l].tile_begin;
    if (tid == 0) s_tb[L] = total;
    for (int b = tid; b < kMeanBins; b += kThreads) s_bins[b] = 0ull;
    if (blockIdx.x == 0) {
        if (tid == 0) { w.ctrl->ticketA = 0; w.ctrl->ticketB = 0; }
        for (uint32_t i = tid; i < w.status_extra; i += kThreads) {   // segments beyond the tiles
            w.statusA[w.ntiles_total + i] = 0ull;
            w.statusB[w.ntiles_total + i] = 0ull;
        }
    }
    __syncthreads();

    int cur = -1;
    uint32_t ntl = 0, cta_max = 0, rcnt = 0, tc = 0, tpar = 0;
    bool reuse = false;
    const float *g = nullptr;
    float *u = nullptr, *V = nullptr;
    uint32_t n = 0, tb = 0;
    float m = 0.f;
    // candidate stash: |V| > tau in index order, this CTA's region, one record per layer
    uint2 *region = w.cand + (uint64_t)blockIdx.x * w.cand_R;
    uint32_t cta_cnt = 0, layer_start = 0, nbt = 0, wfill = 0, tau = 0, st_skx = 0, st_ska = 0;
    bool st_on = false, over = false;

    // move the batch's staged candidates into the CTA region in index order
    // (tile-major, warp-minor); block-uniform call
    const uint64_t pol_keep = l2_policy_evict_last();   // the stash stays in L2 for K2/K3
    auto drain = [&]() {
        over = __syncthreads_or(over) != 0;
        if (warp == 0) {
            constexpr int E = kK1Batch * kWarps;
            const int ne = (int)nbt * kWarps;
            uint32_t carry = 0;
#pragma unroll
            for (int e0 = 0; e0 < E; e0 += 32) {
                const int e = e0 + lane;
                const uint32_t v = e < ne ? s_tcnt[e / kWarps][e % kWarps] : 0u;
                uint32_t a = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) { uint32_t y = __shfl_up_sync(FULLMASK, a, o); if (lane >= o) a += y; }
                if (e < ne) s_toff[e / kWarps][e % kWarps] = carry + a - v;
                carry += __shfl_sync(FULLMASK, a, 31);
            }
            if (lane == 0) s_btot = carry;
        }
        __syncthreads();
        const uint32_t btot = s_btot;
        if (!over && cta_cnt + btot <= w.cand_R) {
            uint32_t src = 0;
            for (uint32_t t = 0; t < nbt; t++) {
                const uint32_t cnt = s_tcnt[t][warp];
                uint2 *dst = region + cta_cnt + s_toff[t][warp];
                RGC_DCHECK(cta_cnt + s_toff[t][warp] + cnt <= w.cand_R);
                for (uint32_t i = lane; i < cnt; i += 32) st_u2_hint(dst + i, s_cst[warp][src + i], pol_keep);
                src += cnt;
            }
            cta_cnt += btot;
        } else {
            over = true;
        }
        nbt = 0;
        wfill = 0;
        __syncthreads();
    };

    auto flush = [&](int l) {
        if (st_on) {
            if (nbt) drain();
            if (tid == 0) {
                const LayerDesc &d = w.desc[l];
                w.rec[d.rec_base + (blockIdx.x - d.cand_b0)] = make_uint2(layer_start, cta_cnt - layer_start);
                atomicAdd(&w.st[l].cand_acc, cta_cnt - layer_start);
                if (over) atomicOr(&w.st[l].cand_bad, 1u);
            }
        }
        k1_flush(w, l, ntl, cta_max, s_bins, s_misc, rcnt);
    };

    // blocked tile ranges: each CTA streams a contiguous range (touches few layers)
    const uint32_t t_beg = (uint32_t)(((uint64_t)total * blockIdx.x) / gridDim.x);
    const uint32_t t_end = (uint32_t)(((uint64_t)total * (blockIdx.x + 1)) / gridDim.x);
    // warp w owns tile elements [512w, 512w + 512): float4 j of a lane sits at
    // 512w + 128j + 4*lane, so the warp's candidates come out in index order (j, lane, slot)
    const uint32_t wo = warp * 512 + lane * 4;
    for (uint32_t tile = t_beg; tile < t_end; tile++) {
        int l = find_layer(s_tb, L, tile);
        if (l != cur) {
            if (cur >= 0) flush(cur);
            cur = l; ntl = 0; cta_max = 0; rcnt = 0;
            const LayerDesc &d = w.desc[l];
            g = d.g; u = d.u; V = d.V; n = d.n; tb = d.tile_begin; m = d.m;
            const LayerState &S = w.st[l];
            reuse = d.selector == RGC_SEL_SAMPLED_BS && S.cache_valid && (S.step % d.interval) != 0u;
            tc = S.cache_key;
#ifdef RGC_NO_STASH
            st_on = false;
#else
            st_on = S.stash_on != 0u;
#endif
            tau = S.cand_key;
            // ASQ (R21): only the sign this call selects is a candidate
            st_ska = d.quant ? 0x80000000u : 0u;
            st_skx = (d.quant && (S.phase & 1u)) ? 0x80000000u : 0u;
            over = false;
            layer_start = cta_cnt;
            nbt = 0; wfill = 0;
        }
        const uint32_t t0 = (tile - tb) * kTile;
        const uint32_t cnt = min((uint32_t)kTile, n - t0);
        float gv[kPerThread], uv[kPerThread], vv[kPerThread];
        const bool full = (cnt == kTile);
        const bool mom = (m != 0.f);
        if (full) {
            float4 G[4], U[4], X[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                G[j] = __ldcs(reinterpret_cast<const float4 *>(g + t0 + wo + j * 128));
                X[j] = ld_stream(V + t0 + wo + j * 128);
            }
            if (mom) {
#pragma unroll
                for (int j = 0; j < 4; j++) U[j] = ld_stream(u + t0 + wo + j * 128);
            }
#pragma unroll
            for (int j = 0; j < 4; j++) {
                gv[4 * j] = G[j].x; gv[4 * j + 1] = G[j].y; gv[4 * j + 2] = G[j].z; gv[4 * j + 3] = G[j].w;
                vv[4 * j] = X[j].x; vv[4 * j + 1] = X[j].y; vv[4 * j + 2] = X[j].z; vv[4 * j + 3] = X[j].w;
                if (mom) { uv[4 * j] = U[j].x; uv[4 * j + 1] = U[j].y; uv[4 * j + 2] = U[j].z; uv[4 * j + 3] = U[j].w; }
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4; j++)
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    uint32_t p = wo + j * 128 + c;
                    bool ok = p < cnt;
                    gv[4 * j + c] = ok ? g[t0 + p] : 0.f;
                    vv[4 * j + c] = ok ? V[t0 + p] : 0.f;
                    uv[4 * j + c] = (ok && mom) ? u[t0 + p] : 0.f;
                }
        }
        // u <- m*u + g (one rounding, DGC momentum correction); V <- V + u
#pragma unroll
        for (int e = 0; e < kPerThread; e++) {
            if (mom) {
                uv[e] = __fmaf_rn(m, uv[e], gv[e]);
                vv[e] = __fadd_rn(vv[e], uv[e]);
            } else {
                vv[e] = __fadd_rn(vv[e], gv[e]);
            }
        }
        if (full) {
#pragma unroll
            for (int j = 0; j < 4; j++)
                st_stream(V + t0 + wo + j * 128, make_float4(vv[4 * j], vv[4 * j + 1], vv[4 * j + 2], vv[4 * j + 3]));
            if (mom) {
#pragma unroll
                for (int j = 0; j < 4; j++)
                    st_stream(u + t0 + wo + j * 128, make_float4(uv[4 * j], uv[4 * j + 1], uv[4 * j + 2], uv[4 * j + 3]));
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4; j++)
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    uint32_t p = wo + j * 128 + c;
                    if (p < cnt) {
                        V[t0 + p] = vv[4 * j + c];
                        if (mom) u[t0 + p] = uv[4 * j + c];
                    }
                }
        }
        // candidates |V| > tau staged in index order (padding past cnt is 0, never staged)
        if (st_on) {
            const uint32_t lt = (1u << lane) - 1u;
            uint32_t wc = 0;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                uint32_t mk = 0;
#pragma unroll
                for (int c = 0; c < 4; c++)
                    mk |= (uint32_t)(skey(__float_as_uint(vv[4 * j + c]), st_skx, st_ska) > tau) << c;
                if (__ballot_sync(FULLMASK, mk != 0u)) {
                    const uint32_t q0 = __ballot_sync(FULLMASK, mk & 1u);
                    const uint32_t q1 = __ballot_sync(FULLMASK, mk & 2u);
                    const uint32_t q2 = __ballot_sync(FULLMASK, mk & 4u);
                    const uint32_t q3 = __ballot_sync(FULLMASK, mk & 8u);
                    const uint32_t rtot = __popc(q0) + __popc(q1) + __popc(q2) + __popc(q3);
                    if (wfill + wc + rtot <= (uint32_t)kK1Stash) {
                        uint32_t pos = wfill + wc + __popc(q0 & lt) + __popc(q1 & lt) +
                                       __popc(q2 & lt) + __popc(q3 & lt);
                        const uint32_t ib = t0 + wo + j * 128;
#pragma unroll
                        for (int c = 0; c < 4; c++)
                            if ((mk >> c) & 1u) s_cst[warp][pos++] = make_uint2(ib + c, __float_as_uint(vv[4 * j + c]));
                        wc += rtot;
                    } else {
                        over = true;
                    }
                }
            }
            if (lane == 0) s_tcnt[nbt][warp] = wc;
            wfill += wc;
            nbt++;
        }
        // tile max of |V| on 31-bit keys (P:211 max(abs(X)))
        uint32_t km = 0;
#pragma unroll
        for (int e = 0; e < kPerThread; e++) km = max(km, fkey(vv[e]));
        if (reuse) {   // sampled BS reuse step: count_nonzero(|V| > t_cached) in this pass
#pragma unroll
            for (int e = 0; e < kPerThread; e++) rcnt += fkey(vv[e]) > tc ? 1u : 0u;
        }
        km = __reduce_max_sync(FULLMASK, km);
        uint32_t *wmax = s_wmax[tpar & 1u];
        tpar++;
        if (lane == 0) wmax[warp] = km;
        __syncthreads();
        uint32_t tmax = wmax[0];
#pragma unroll
        for (int i = 1; i < kWarps; i++) tmax = max(tmax, wmax[i]);
        cta_max = max(cta_max, tmax);
        // mean_fx terms: floor(|x| * 2^(30-E_t)) exactly from the significand (R2)
        unsigned long long sum = 0;
        int Et = 0;
        if (tmax != 0u && tmax < 0x7F800000u) {
            const int eb = (int)(tmax >> 23);
            Et = eb > 0 ? eb - 127 : (31 - __clz(tmax & 0x7FFFFFu)) - 149;
#pragma unroll
            for (int e = 0; e < kPerThread; e++) {
                const uint32_t k = fkey(vv[e]);
                const int ebx = (int)(k >> 23);
                const uint32_t s = (k & 0x7FFFFFu) | (ebx ? 0x800000u : 0u);
                const int sh = (max(ebx, 1) - 150) + 30 - Et;
                uint32_t term = sh >= 0 ? (s << sh) : ((-sh) < 32 ? (s >> (-sh)) : 0u);
                sum += term;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(FULLMASK, sum, o);
        }
#ifdef RGC_K1_TWOBAR
        if (lane == 0) s_wsum[warp] = sum;
        __syncthreads();
        if (tid == 0) {
            if (tmax != 0u && tmax < 0x7F800000u) {
                unsigned long long S = 0;
#pragma unroll
                for (int i = 0; i < kWarps; i++) S += s_wsum[i];
                s_bins[Et + 149] += S;
            }
        }
#else
        // the tile's term sum goes straight into its exponent bin (integer adds commute: the
        // same bits as the ordered combine); no second block barrier per tile (k1_flush
        // synchronises before it reads the bins)
        if (lane == 0 && sum) atomicAdd(&s_bins[Et + 149], sum);
#endif
        if (tid == 0) {
            // fresh look-back status words for this call's K3 launches
            w.statusA[tile] = 0ull;
            w.statusB[tile] = 0ull;
        }
        if (st_on && nbt == (uint32_t)kK1Batch) drain();
        ntl++;
    }
    if (w.tl && tid == 0) atomicMin(&w.tl[TL_K1S], tlm_start);
    tl_end(w.tl, TL_K1S);
    tl_probe(w.tl, TL_P0 + 12);   // min / max over the CTAs: the spread of K1's ramp-down
    if (w.k1cnt && tid == 0) atomicAdd(&w.k1cnt[1], 1ull);   // the early fill waits on it
    if (cur >= 0) flush(cur);
    // RGC_SYNC_PULL: the peers read last epoch's message block in place; K2 (which waits
    // for this grid) rewrites it only after every peer has published "consumed"
    if (w.pull_flags && blockIdx.x == 0 && tid < w.pull_p && tid != w.pull_rank)
        wait_flag(w.pull_flags, &w.pull_flags->consumed[tid], tid, w.pull_epoch);
}

// ============================================================================
// K2: threshold counts (Alg.2 levels) / Alg.3 histogram + device-side decision
// ============================================================================
// Grid barrier for a cooperative launch (all CTAs co-resident): arrive on a counter, the last
// CTA bumps the generation.  A wait longer than 2 s gives up (flag in the message status
// word -> rgc_status) instead of hanging the device.
#ifndef RGC_BAR_SLEEP_MAX
#define RGC_BAR_SLEEP_MAX 1024u
#endif
__device__ void grid_barrier(Ctrl *c, uint32_t *msg_hdr, int L) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int gen = *(volatile unsigned int *)&c->bar_gen;
        __threadfence();
        if (atomicAdd(&c->bar_count, 1u) == gridDim.x - 1) {
            c->bar_count = 0u;
            __threadfence();
            atomicAdd(&c->bar_gen, 1u);
        } else {
            // exponential back-off (64 ns .. RGC_BAR_SLEEP_MAX): a waiting CTA's polls hit one
            // L2 line, and the CTAs still working (the per-layer finalisations) are chains of
            // dependent L2 round trips that tight polling from ~300 CTAs slows down
            const unsigned long long t0 = globaltimer_ns();
            unsigned int ns = 64u;
            while (*(volatile unsigned int *)&c->bar_gen == gen) {
                if (globaltimer_ns() - t0 > 2000000000ull) { atomicOr(&msg_hdr[L], kStatBarrier); break; }
                __nanosleep(ns);
                ns = ns < RGC_BAR_SLEEP_MAX ? 2u * ns : ns;
            }
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULLMASK, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

// every layer is decided: message offsets (compact) and the K3/K4 work spaces.
// One warp; lane i takes layers i, i+32, ... with running carries between rounds.
__device__ void k2_global_finalize(const Ws &w, int L, uint32_t *msg_hdr, uint32_t hdr_words) {
    const int lane = threadIdx.x & 31;
    uint32_t off = 0, a = 0, b = 0, c4 = 0, status = 0;
    for (int l0 = 0; l0 < L; l0 += 32) {
        const int l = l0 + lane;
        uint32_t cnt = 0, ta = 0, tb = 0, t4 = 0, small = 0;
        if (l < L) {
            LayerState &S = w.st[l];
            const LayerDesc &d = w.desc[l];
            const uint32_t mode = __ldcg(&S.mode);
            // ASQ layers emit into their scratch; K5 appends their indices after the pairs
            cnt = d.quant ? 0u : __ldcg(&S.count);
            const uint32_t surv = __ldcg(&S.surv);
            status |= __ldcg(&S.flags) & RGC_F_NONFINITE;
            const uint32_t stiles = (surv + kTile - 1) / kTile;           // K4 work units
            const uint32_t vsegs = (d.n + kSegA - 1) / kSegA;             // K3A work units
            const uint32_t ssegs = (surv + kSegB - 1) / kSegB;            // K3B units
            const uint32_t vsegsB = (d.n + kSegB - 1) / kSegB;
            // exact top-k over a small candidate set: one cluster does select + emission (K45)
            small = (mode == MODE_SURV && surv <= w.small_sel) ||
                    (mode == MODE_EXACT && d.n <= w.small_sel);
            const bool cand = __ldcg(&S.cand_ok) != 0u;
            // K3A over the stash (segments of seg_ch records) or over V
            const uint32_t asegs = cand ? (d.cand_nb + w.seg_ch - 1) / w.seg_ch : vsegs;
            if (mode == MODE_THRESH) ta = asegs;
            else if (mode == MODE_SURV) { ta = asegs; if (!small) { tb = ssegs; t4 = stiles; } }
            else if (mode == MODE_EXACT && !small) { tb = vsegsB; t4 = d.ntiles; }
        }
        const uint32_t ioff = warp_incl_scan(cnt), ia = warp_incl_scan(ta);
        const uint32_t ib = warp_incl_scan(tb), i4 = warp_incl_scan(t4);
        if (l < L) {
            LayerState &S = w.st[l];
            const LayerDesc &d = w.desc[l];
            S.small = small;
            S.msg_off = d.quant ? (uint32_t)d.q_off : off + ioff - cnt;
            msg_hdr[L + 2 + l] = d.quant ? 0u : RGC_MSG_DENSE;
            S.k3a_begin = a + ia - ta; S.k3a_tiles = ta;
            S.k3b_begin = b + ib - tb; S.k3b_tiles = tb;
            S.k4_begin = c4 + i4 - t4; S.k4_tiles = t4;
        }
        off += __shfl_sync(FULLMASK, ioff, 31);
        a += __shfl_sync(FULLMASK, ia, 31);
        b += __shfl_sync(FULLMASK, ib, 31);
        c4 += __shfl_sync(FULLMASK, i4, 31);
    }
    tl_probe(w.tl, TL_P0 + 10);
    status = __reduce_or_sync(FULLMASK, status);
    if (lane == 0) {
        w.ctrl->k3a_total = a;
        w.ctrl->k3b_total = b;
        w.ctrl->k4_total = c4;
        w.ctrl->status = status;
        w.ctrl->dense_pairs = off;
        if (w.k4_hint) *w.k4_hint = c4;
        msg_hdr[L] = status;
        msg_hdr[L + 1] = (uint32_t)L;
    }
    tl_probe(w.tl, TL_P0 + 11);
    for (uint32_t i = 2 * L + 2 + lane; i < hdr_words; i += 32) msg_hdr[i] = 0u;
}

// Alg.3 on the counts cnt[j] = #{|V| > t_j}, t_j = tk[j].
// cnt[j] is exact for j >= jlo; for j < jlo only c(j) >= cnt[jlo] is known (the
// histogram binned only |V| > t_jlo).  Whenever that lower bound does not
// determine the algorithm's path and result exactly, return false: the caller
// then re-runs the full histogram (jlo = 0) for this layer.
// tp[j].x = t_j's key: the (t_j, t_{j+1}) table the counting kernel staged in shared memory
// (the search's dependent steps then cost shared-memory, not L2, latency)
__device__ bool bs_search(const LayerDesc &d, LayerHot &S, const uint32_t *cnt,
                          const uint2 *tp, uint32_t jlo) {
    const uint64_t k = d.k;
    const uint32_t clo = cnt[jlo];
    const bool lb_forced = (uint64_t)clo >= 2 * k;   // every j < jlo has c >= 2k
    double l = 0.0, r = 1.0;
    uint32_t it = 0, flags = S.flags, lbmask = 0;
    uint32_t jsel = 0, c = 0;
    bool have_best = false, broke = false, any_lb = false, last_lb = false;
    uint32_t best_j = 0, best_c = 0;
    while (__dsub_rn(r, l) > d.bs_eps) {
        // (r - l) / 2 as a multiplication by 0.5: the same bits (r - l >= 2^-10 is dyadic and
        // far from the subnormals, so halving it is exact either way), no division sequence
        const double ratio = __dadd_rn(l, __dmul_rn(__dsub_rn(r, l), 0.5));
        const uint32_t j = (uint32_t)__dmul_rn(ratio, 1024.0);   // exact: ratio = j/1024
        const bool lb = j < jlo;
        if (lb && !lb_forced) return false;
        c = lb ? clo : cnt[j];
        last_lb = lb;
        any_lb |= lb;
        jsel = j;
        if (it < (uint32_t)kMaxTrim) {
            S.info.level_count[it] = c;             // a lower bound when lb (info.lb_mask)
            S.info.level_thresh[it] = __uint_as_float(tp[j].x);
            if (lb) lbmask |= 1u << it;
        }
        it++;
        if (lb) {                                  // c >= 2k: no break, the left border moves
            have_best = true;
            l = ratio;
            continue;
        }
        if ((uint64_t)c >= k && (!have_best || c < best_c)) { have_best = true; best_j = j; best_c = c; }
        if ((uint64_t)c > k && 2 * k > (uint64_t)c) { broke = true; break; }
        if (d.branch == RGC_BS_PAPER_LITERAL) {
            if (2 * (uint64_t)c < k) r = ratio; else l = ratio;
        } else {
            if ((uint64_t)c <= k) r = ratio; else l = ratio;
        }
    }
    bool exact = false;
    if (broke) {
        flags |= RGC_F_BS_BREAK;
    } else if (it > 0 && (uint64_t)c >= k) {
        if (last_lb) return false;                 // the kept set's size must be exact
        flags |= RGC_F_EPS_KEEP;
        if ((uint64_t)c >= 2 * k) flags |= RGC_F_EPS_HIGH;
    } else if (have_best) {
        if (any_lb) return false;                  // best may be a bounded step
        flags |= RGC_F_EPS_BEST;
        jsel = best_j; c = best_c;
    } else {
        flags |= RGC_F_EPS_EXACT;
        exact = true;
    }
    if (!exact && c > d.cap) { flags |= RGC_F_CAP_EXACT; exact = true; }
    S.info.iters = it;
    S.info.lb_mask = lbmask;
    S.flags = flags;
    if (exact) {
        S.mode = MODE_EXACT;
        S.count = d.k;
        S.info.threshold = 0.f;
    } else {
        S.mode = MODE_THRESH;
        S.thr_key = tp[jsel].x;
        S.count = c;
        S.info.threshold = __uint_as_float(tp[jsel].x);
    }
    // next call's hint: bin only above the chosen threshold minus the margin
    S.jhint = exact ? 0u : jsel;
    return true;
}


// s_last (shared) tells the CTA whether its decision was the call's last one
template <int NL, int NT>
__device__ void k2_finalize(const Ws &w, int l, int L, uint32_t *s_hist, uint32_t *s_w,
                            const uint2 *s_tp, uint32_t *msg_hdr, uint32_t hdr_words, int pass) {
    TlMark tlm(w.tl, TL_K2F);
    __shared__ int s_last, s_decided;
    __shared__ LayerHot s_hot;
    __shared__ LayerDesc s_desc;
    __threadfence();
    LayerState &G = w.st[l];
    LayerHot &S = s_hot;
    const LayerDesc &d = s_desc;
    hot_load(s_hot, G);
    desc_load(s_desc, w.desc[l]);
    // the histogram, taken in the same round trip as the state (whatever the layer: it is
    // all zeros unless this is an Alg.3 layer K2 counted -- K4 leaves its digits zeroed)
    constexpr int PER = (kBsTable + NT - 1) / NT;
    uint32_t loc[PER];
    uint32_t tsum = 0;
#pragma unroll
    for (int i = 0; i < PER; i++) {
        const int b = threadIdx.x * PER + i;
        loc[i] = (b < kBsTable) ? atomicExch(&G.hist[b], 0u) : 0u;
        tsum += loc[i];
    }
    __syncthreads();
    tl_probe(w.tl, TL_P0 + 4);
    const uint32_t flags0 = S.flags;
    const bool skip = flags0 & (RGC_F_NONFINITE | RGC_F_DEGENERATE | RGC_F_SAMPLED_REUSE);
    const bool bs = d.selector != RGC_SEL_TRIMMED;
    if (!skip && bs) {
        // cnt[j] = sum_{b > j} hist[b]  (suffix sums of the one-pass histogram)
        uint32_t incl = block_incl_scan(tsum, s_w);
        __shared__ uint32_t s_total;
        if (threadIdx.x == NT - 1) s_total = incl;
        __syncthreads();
        uint32_t run = incl - tsum;
#pragma unroll
        for (int i = 0; i < PER; i++) {
            int b = threadIdx.x * PER + i;
            run += loc[i];
            if (b < kBsTable) s_hist[b] = s_total - run;   // count of elements in bins > b
        }
        __syncthreads();
    }
    tl_probe(w.tl, TL_P0 + 5);
    if (threadIdx.x == 0) {
        const uint32_t k = d.k;
        const uint32_t surv_k1 = S.surv;   // a sampled reuse step's survivors (set by K1)
        S.rs_prefix = 0; S.rs_krem = k; S.rs_above = 0;
        S.surv = 0;
        S.emitted_a = 0; S.emitted_b = 0;
        // fresh diagnostics for this call
        S.info.iters = 0; S.info.trim_level = 0; S.info.trim_levels = 0;
        S.info.threshold = 0.f; S.info.survivors = 0; S.info.kth_key = 0; S.info.tie_quota = 0;
        S.info.emitted = 0; S.info.lb_mask = 0; S.info.stashed = 0;
        for (int j = 0; j < kMaxTrim; j++) { S.info.level_count[j] = 0; S.info.level_thresh[j] = 0.f; }
        if (!bs && !(flags0 & (RGC_F_NONFINITE | RGC_F_DEGENERATE))) S.info.trim_levels = d.trim_levels;
        bool decided = true;
        // decision of this call, kept in registers and stored once below
        uint32_t mode = S.mode, flags = flags0, thr = S.thr_key, count = S.count, surv = 0;
        int tlevel = -1;
        if (flags0 & RGC_F_NONFINITE) {
            mode = MODE_NONE; count = 0;
        } else if (flags0 & RGC_F_SAMPLED_REUSE) {
            // decided in K1 (mode, count, thr_key, surv): one count_nonzero at the cached threshold
            if (mode == MODE_SURV) surv = surv_k1;
            S.info.iters = 1;
            S.info.level_count[0] = S.reuse_cnt;
            S.info.level_thresh[0] = __uint_as_float(S.cache_key);
            S.info.threshold = mode == MODE_THRESH ? __uint_as_float(S.cache_key) : 0.f;
        } else if (flags0 & RGC_F_DEGENERATE) {
            mode = MODE_EXACT; count = k;
        } else if (!bs) {
            // Alg.2 lines 3-8: the first level whose count reaches k (R4, R5)
            uint32_t cnts[kMaxTrim];
#pragma unroll
            for (int j = 0; j < NL; j++) cnts[j] = atomicExch(&G.trim_cnt[j], 0u);
            // counted from the K1 stash {|V| > tau}: a level below tau has only a lower
            // bound; reaching one re-counts the layer over V (pass 1)
            const bool from_stash = pass == 0 && S.k2src;
            int jsel = -1;
            for (int j = 0; j < (int)d.trim_levels && j < NL; j++) {
                if (from_stash && S.tkeys[j] < S.cand_key) { decided = false; break; }
                S.info.level_count[j] = cnts[j];
                S.info.level_thresh[j] = __uint_as_float(S.tkeys[j]);
                if (cnts[j] >= k) { jsel = j; break; }
            }
            if (!decided) {
                S.need_full = 1u;
                atomicOr(&w.ctrl->any_full, 1u);
            } else {
                count = k;
                if (jsel < 0) {
                    flags |= RGC_F_TRIM_ALL;
                    S.info.iters = d.trim_levels;
                    S.info.trim_level = d.trim_levels;
                    S.info.survivors = d.n;
                    mode = MODE_EXACT;
                } else {
                    S.info.iters = jsel + 1;
                    S.info.trim_level = jsel;
                    S.info.survivors = cnts[jsel];
                    S.need_cnt = cnts[jsel];
                    tlevel = jsel;
                    if (cnts[jsel] <= d.s_cap) {
                        mode = MODE_SURV;
                        thr = S.tkeys[jsel];
                        surv = cnts[jsel];
                    } else {
                        flags |= RGC_F_SURV_CAP;
                        mode = MODE_EXACT;
                    }
                }
                S.info.threshold = 0.f;
            }
        } else {
            const uint32_t jlo = bs_jlo(S, pass);
            const uint32_t margin = S.margin ? S.margin : 64u;
            const bool bs_ok = bs_search(d, S, s_hist, s_tp, jlo);
            tl_probe(w.tl, TL_P0 + 6);
            if (bs_ok) {
                mode = S.mode; flags = S.flags; thr = S.thr_key; count = S.count;
                if (pass == 1) {                    // the hint was too tight: widen it
                    S.need_full = 0u;
                    S.full_runs++;
                    if (S.k2src) S.stash_shift = max(stash_shift(S), 2u) - 1u;   // and the stash key
                    S.margin = min(1024u, 2u * margin);
                } else if ((uint64_t)s_hist[jlo] > (uint64_t)c_tune[0] * k && margin > c_tune[1]) {
                    S.margin = margin / 2u;         // binned too much: tighten
                }
                S.need_cnt = s_hist[jlo];
            } else {
                // the bound did not determine Alg.3's path: full histogram in pass 1
                S.need_full = 1u;
                atomicOr(&w.ctrl->any_full, 1u);
                decided = false;
            }
        }
        if (decided) {
            if (pass == 1) S.need_full = 0u;
            S.mode = mode; S.flags = flags; S.thr_key = thr; S.count = count; S.surv = surv;
            // K4 over the Alg.2 survivors: two offset digits when they span < 2^22 keys
            S.rs_two = (mode == MODE_SURV && S.maxkey - thr < (1u << 22)) ? 1u : 0u;
            S.rs_base = thr + 1u;
            // K3's first pass reads the K1 stash when it holds the whole selected set /
            // the Alg.2 survivors (every |V| > tau, tau <= the compaction threshold)
            const uint32_t tau = S.cand_key;
            const uint32_t ok = (S.stash_ok && (mode == MODE_THRESH || mode == MODE_SURV) &&
                                 thr >= tau) ? 1u : 0u;
#ifdef RGC_NO_STASH
            S.cand_ok = 0u;
            S.info.stashed = 0u;
#else
            S.cand_ok = ok;
            S.info.stashed = ok;
#endif
            if (flags0 & RGC_F_DEGENERATE) S.info.threshold = 0.f;
            if (d.selector == RGC_SEL_SAMPLED_BS) {
                // a full search caches its threshold (or clears the cache after an exact fallback)
                if (!(flags & RGC_F_SAMPLED_REUSE)) {
                    S.cache_valid = (mode == MODE_THRESH) ? 1u : 0u;
                    S.cache_key = thr;
                }
                if (flags & RGC_F_NONFINITE) S.cache_valid = 0u;
                S.step = S.step + 1u;
            }
            // next call's stash key: the lowest key this call needed, scaled by 1 - 2^-shift
            // (the next call's mean/max move the thresholds; K1 checks the prediction)
            if (!(flags & (RGC_F_NONFINITE | RGC_F_DEGENERATE))) {
                uint32_t need;
                if (d.selector == RGC_SEL_TRIMMED) {
                    // the level Alg.2 stopped at (all levels above it are needed too)
                    const int lv = tlevel >= 0 ? tlevel : (int)min(d.trim_levels, (uint32_t)NL) - 1;
                    need = S.tkeys[max(lv, 0)];
                } else {
                    // the highest level whose count reached F*k (exact for j >= jlo of
                    // this pass), else this pass's t_jlo
                    const uint32_t jl = bs_jlo(S, pass);
                    uint32_t jn = jl;
                    const uint64_t want = (uint64_t)c_tune[4] * d.k;
                    if (c_tune[4] && mode == MODE_THRESH && (uint64_t)s_hist[jl] >= want) {
                        // the highest j in [jl, max(jhint, jl)] with count >= want: the suffix
                        // counts do not increase with j, so a bisection (it was a walk down
                        // from jhint, up to ~1000 dependent steps)
                        uint32_t lo = jl, hi = max(S.jhint, jl);   // s_hist[lo] >= want
                        while (lo < hi) {
                            const uint32_t mid = (lo + hi + 1u) >> 1;
                            if ((uint64_t)s_hist[mid] >= want) lo = mid; else hi = mid - 1u;
                        }
                        jn = lo;
                    }
                    need = s_tp[jn].x;
                    if (d.selector == RGC_SEL_SAMPLED_BS && S.cache_valid) need = min(need, S.cache_key);
                }
                // stashed far more than the call needed: move the key closer (next call)
                if (c_tune[2] && S.k2src && S.cand_total > c_tune[2] * max(S.need_cnt, 1u) &&
                    stash_shift(S) < c_tune[3])
                    S.stash_shift = stash_shift(S) + 1u;
                const float scale = 1.0f - __uint_as_float((127u - stash_shift(S)) << 23);
                S.cand_key = fkey(__fmul_rn(__uint_as_float(need), scale));
                S.stash_on = 1u;
            } else {
                S.stash_on = 0u;
            }
            S.info.flags = flags;
            S.info.count = count;
            S.info.maxkey = S.maxkey;
            S.info.mean = S.mean;
            msg_hdr[l] = count;
        }
        G.k2_done = 0;
        s_decided = decided;
    }
    __syncthreads();
    tl_probe(w.tl, TL_P0 + 7);
    hot_store(G, s_hot);
    if (L > 1) __threadfence();   // before the layers_done count another CTA's layout reads
    __syncthreads();
    tl_probe(w.tl, TL_P0 + 8);
    if (threadIdx.x == 0) {
        s_last = 0;
        if (s_decided) {
            // the last layer decided this call lays out the message and the K3/K4 spaces
            // (a single layer is its own last: no counter round trip)
            const unsigned int old = L == 1 ? 0u : atomicAdd(&w.ctrl->layers_done, 1u);
            s_last = (old + 1u == (unsigned int)L);
        }
    }
    __syncthreads();
    if (s_last && threadIdx.x < 32) {
        // acquire the other layers' decisions (a single layer's are this CTA's own stores,
        // visible across the block barrier)
        if (L > 1) __threadfence();
        { TlMark tlg(w.tl, TL_K2G); k2_global_finalize(w, L, msg_hdr, hdr_words); }
        tl_probe(w.tl, TL_P0 + 9);
        if (threadIdx.x == 0) {
            w.ctrl->layers_done = 0u;
            w.ctrl->any_full = 0u;
            w.ctrl->any_vpass = 0u;
        }
    }
    if (!skip && bs) {
        for (int j = threadIdx.x; j < kBsTable; j += NT) s_hist[j] = 0u;
    }
    __syncthreads();
}


// V tile loader shared by K2: full tiles with 128-bit loads, ragged tails guarded
__device__ __forceinline__ void k2_load(const Ws &w, const uint32_t *s_tb, int L, uint32_t tile,
                                        float4 *X) {
    const int tid = threadIdx.x;
    const int l = find_layer(s_tb, L, tile);
    const LayerDesc &d = w.desc[l];
    const uint32_t t0 = (tile - d.tile_begin) * kTile;
    const uint32_t cnt = min((uint32_t)kTile, d.n - t0);
    const float *V = d.V + t0;
    if (cnt == kTile) {
#pragma unroll
        for (int j = 0; j < 4; j++) X[j] = reinterpret_cast<const float4 *>(V)[j * kThreads + tid];
    } else {
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t p = (j * kThreads + tid) * 4;
            X[j].x = p + 0 < cnt ? V[p + 0] : 0.f;
            X[j].y = p + 1 < cnt ? V[p + 1] : 0.f;
            X[j].z = p + 2 < cnt ? V[p + 2] : 0.f;
            X[j].w = p + 3 < cnt ? V[p + 3] : 0.f;
        }
    }
}

#ifndef RGC_K2_MINB
#define RGC_K2_MINB 4
#endif
// V pass (fallback to the K1 stash): K2 over the residual itself.
// pass 0: layers without a usable stash (Alg.2 level counts; Alg.3 histogram of
//         |V| > t_jlo only), and the skipped ones (non-finite, degenerate, reuse steps)
// pass 1: only Alg.3 layers whose bounded histogram did not determine the search
// One V pass by the whole grid (a device function: the k2_count kernel below, or the tail of
// k2_stash); shared buffers from the caller
template <int NL>
__device__ __forceinline__ void k2_vpass(const Ws &w, int L, uint32_t total, uint32_t *msg_hdr,
                                         uint32_t hdr_words, int pass, uint32_t *s_tb,
                                         uint2 *s_tp, uint32_t *s_hist, uint32_t *s_cnt,
                                         uint32_t *s_w, int *s_flag) {
    const int tid = threadIdx.x, lane = tid & 31;
    for (int l = tid; l < L; l += kThreads) s_tb[l] = w.desc[l].tile_begin;
    if (tid == 0) s_tb[L] = total;
    for (int b = tid; b < kBsTable; b += kThreads) s_hist[b] = 0u;
    if (tid < kMaxTrim) s_cnt[tid] = 0u;
    __syncthreads();

    int cur = -1;
    uint32_t ntl = 0;
    bool skip = true, bs = false, active = false;
    uint32_t tk[NL];
    uint32_t c[NL];
#pragma unroll
    for (int j = 0; j < NL; j++) { c[j] = 0; tk[j] = 0x7FFFFFFFu; }
    uint32_t tlo = 0, skx = 0, ska = 0;
    float mean_f = 0.f, inv_d = 0.f;

    auto layer_active = [&](int l) -> bool {
        return pass == 0 ? w.st[l].k2src == 0u : w.st[l].need_full != 0u;
    };

    auto flush = [&](int l) {
        if (!active) return;
        LayerState &S = w.st[l];
        if (!skip && !bs) {
#pragma unroll
            for (int j = 0; j < NL; j++) {
                uint32_t v = __reduce_add_sync(FULLMASK, c[j]);
                if (lane == 0 && v) atomicAdd(&s_cnt[j], v);
                c[j] = 0;
            }
        }
        __syncthreads();
        if (!skip && !bs && tid < NL) {
            if (s_cnt[tid]) atomicAdd(&S.trim_cnt[tid], s_cnt[tid]);
            s_cnt[tid] = 0;
        }
        if (!skip && bs) {
            for (int b = tid; b < kBsTable; b += kThreads) {
                uint32_t v = s_hist[b];
                if (v) { atomicAdd(&S.hist[b], v); s_hist[b] = 0u; }
            }
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            unsigned int old = atomicAdd(&S.k2_done, ntl);
            s_flag[1] = (old + ntl == w.desc[l].ntiles);
        }
        __syncthreads();
        if (s_flag[1]) k2_finalize<NL, kThreads>(w, l, L, s_hist, s_w, s_tp, msg_hdr, hdr_words, pass);
    };

    // a layer whose tiles this pass reads: active and not decided without counts (non-finite,
    // degenerate, sampled-BS reuse step -- K2 only runs their finalisation; a reuse step
    // used to re-read the whole residual here for nothing)
    auto layer_loads = [&](int l) -> bool {
        return layer_active(l) &&
               !(w.st[l].flags & (RGC_F_NONFINITE | RGC_F_DEGENERATE | RGC_F_SAMPLED_REUSE));
    };

    float4 X[4];
    // blocked tile ranges: each CTA streams a contiguous range (touches few layers)
    const uint32_t t_beg = (uint32_t)(((uint64_t)total * blockIdx.x) / gridDim.x);
    const uint32_t t_end = (uint32_t)(((uint64_t)total * (blockIdx.x + 1)) / gridDim.x);
    uint32_t tile = t_beg;
    bool have = false;
    if (tile < t_end && layer_loads(find_layer(s_tb, L, tile))) { k2_load(w, s_tb, L, tile, X); have = true; }
    while (tile < t_end) {
        const int l = find_layer(s_tb, L, tile);
        if (l != cur) {
            if (cur >= 0) flush(cur);
            cur = l; ntl = 0;
            active = layer_active(l);
            const LayerDesc &d = w.desc[l];
            const LayerState &S = w.st[l];
            skip = !active || (S.flags & (RGC_F_NONFINITE | RGC_F_DEGENERATE | RGC_F_SAMPLED_REUSE));
            bs = d.selector != RGC_SEL_TRIMMED;
            skx = S.skx; ska = S.ska;
            if (!skip && bs) {
                for (int j = tid; j <= kBsLevels; j += kThreads)
                    s_tp[j] = make_uint2(S.tkeys[j], S.tkeys[j + 1]);
                const float mx = __uint_as_float(S.maxkey);
                mean_f = (float)S.mean;
                inv_d = 1024.0f / (mx - mean_f);
                tlo = S.tkeys[bs_jlo(S, pass)];
            } else if (!skip) {
#pragma unroll
                for (int j = 0; j < NL; j++) tk[j] = S.tkeys[j];
            }
            __syncthreads();
        }
        if (skip) {
            // nothing to count in this layer: account for this CTA's tiles of it at once
            const uint32_t lend = min(t_end, s_tb[l + 1]);
            if (active) ntl += lend - tile;
            tile = lend;
            have = false;
            if (tile < t_end && layer_loads(find_layer(s_tb, L, tile))) { k2_load(w, s_tb, L, tile, X); have = true; }
            continue;
        }
        // prefetch the next tile of this CTA while the current one is counted
        const uint32_t nt = tile + 1;
        float4 Y[4];
        bool nhave = false;
        if (nt < t_end && layer_loads(find_layer(s_tb, L, nt))) { k2_load(w, s_tb, L, nt, Y); nhave = true; }
        if (!skip && have) {
            uint32_t key[kPerThread];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                key[4 * j] = skey(__float_as_uint(X[j].x), skx, ska);
                key[4 * j + 1] = skey(__float_as_uint(X[j].y), skx, ska);
                key[4 * j + 2] = skey(__float_as_uint(X[j].z), skx, ska);
                key[4 * j + 3] = skey(__float_as_uint(X[j].w), skx, ska);
            }
            if (!bs) {
                // count_nonzero(abs(X) > threshold) for every Alg.2 level at once
#pragma unroll
                for (int e = 0; e < kPerThread; e++)
#pragma unroll
                    for (int j = 0; j < NL; j++) c[j] += (key[e] > tk[j]) ? 1u : 0u;
            } else {
                // bin b = #{j : t_j < |x|} (count(t_j) = #{x : b(x) > j}) for |x| > t_jlo only:
                // estimate from the linear threshold spacing, verified against the exact
                // key pair (t_{b-1}, t_b); the rare misses take a binary search
                uint32_t act = 0;
#pragma unroll
                for (int e = 0; e < kPerThread; e++) act |= (uint32_t)(key[e] > tlo) << e;
                while (act) {
                    const int e = __ffs(act) - 1;
                    act &= act - 1;
                    uint32_t kk = 0;
#pragma unroll
                    for (int i = 0; i < kPerThread; i++) kk = (i == e) ? key[i] : kk;
                    const float jf = (__uint_as_float(kk) - mean_f) * inv_d;
                    int b = __float2int_rz(fminf(fmaxf(jf, 0.f), 1024.f));
                    const uint2 pr = s_tp[b];
                    if ((pr.x < kk) & (kk <= pr.y)) {
                        b += 1;
                    } else {
                        int lo = 1, hi = kBsLevels + 1;   // smallest b with kk <= t_b
                        while (lo < hi) {
                            const int mid = (lo + hi) >> 1;
                            if (kk <= s_tp[mid].x) hi = mid; else lo = mid + 1;
                        }
                        b = lo;
                    }
                    atomicAdd(&s_hist[b], 1u);
                }
            }
        }
        if (active) ntl++;
#pragma unroll
        for (int j = 0; j < 4; j++) X[j] = Y[j];
        have = nhave;
        tile = nt;
    }
    if (cur >= 0) flush(cur);
    __syncthreads();   // the caller may reuse the shared buffers
}

// the V pass as a call from the stash kernel: its register allocation stays apart from the
// stash body's (inlined, the stash loop spilled and the stash pass ran ~10 us longer)
template <int NL>
__device__ __noinline__ void k2_vpass_call(const Ws &w, int L, uint32_t total, uint32_t *msg_hdr,
                                           uint32_t hdr_words, int pass, uint32_t *s_tb,
                                           uint2 *s_tp, uint32_t *s_hist, uint32_t *s_cnt,
                                           uint32_t *s_w, int *s_flag) {
    k2_vpass<NL>(w, L, total, msg_hdr, hdr_words, pass, s_tb, s_tp, s_hist, s_cnt, s_w, s_flag);
}

template <int NL>
__global__ void __launch_bounds__(kThreads, RGC_K2_MINB)
k2_count(Ws w, int L, uint32_t total, uint32_t *msg_hdr, uint32_t hdr_words, int pass) {
    pdl_wait();
    TlMark tlm(w.tl, pass == 0 ? TL_K2V0 : TL_K2V1);
    __shared__ uint32_t s_tb[RGC_MAX_LAYERS + 1];
    __shared__ uint2 s_tp[kBsLevels + 1];   // (t_j, t_{j+1}) keys, j = 0..1024 (t_1025 = inf)
    __shared__ uint32_t s_hist[kBsTable];
    __shared__ uint32_t s_cnt[kMaxTrim];
    __shared__ uint32_t s_w[kWarps];
    __shared__ int s_flag[2];
    if (pass == 1 && w.ctrl->any_full == 0u) return;
    if (pass == 0 && w.ctrl->any_vpass == 0u) return;
    k2_vpass<NL>(w, L, total, msg_hdr, hdr_words, pass, s_tb, s_tp, s_hist, s_cnt, s_w, s_flag);
}

// Stash pass: Alg.2 level counts / Alg.3 bounded histogram from the K1 candidate
// records of the layers whose stash covers this call (S.k2src).  The records of all
// layers form one list (layer l owns [rec_base, rec_base + cand_nb)); each CTA takes a
// blocked range of it and the last CTA to finish a layer's records runs k2_finalize.
#ifndef RGC_K2S_MINB
#define RGC_K2S_MINB 3   // 2 CTAs/SM launched: room beside them for a zero-fill CTA
#endif
template <int NL>
__global__ void __launch_bounds__(kThreads, RGC_K2S_MINB)
k2_stash(Ws w, int L, uint32_t nrec, uint32_t *msg_hdr, uint32_t hdr_words, uint32_t total_tiles,
         int fold) {
    pdl_wait();
    TlMark tlm(w.tl, TL_K2S);
    __shared__ uint32_t s_rb[RGC_MAX_LAYERS + 1];
    __shared__ uint2 s_tp[kBsLevels + 1];
    __shared__ uint32_t s_hist[kBsTable];
    __shared__ uint32_t s_cnt[kMaxTrim];
    __shared__ uint32_t s_w[kWarps];
    __shared__ int s_flag[2];
    const int tid = threadIdx.x, lane = tid & 31;
    // fold: the V passes run at the end of this kernel (no separate launches, each of which
    // cost ~3.5 us of chain); K1 decided any_vpass, and it stays set until every layer is
    // decided -- which cannot happen before the V pass 0 that needs it
    const bool vpass0 = fold && *(volatile unsigned int *)&w.ctrl->any_vpass != 0u;
    for (int l = tid; l < L; l += kThreads) s_rb[l] = w.desc[l].rec_base;
    if (tid == 0) s_rb[L] = nrec;
    for (int b = tid; b < kBsTable; b += kThreads) s_hist[b] = 0u;
    if (tid < kMaxTrim) s_cnt[tid] = 0u;
    __syncthreads();
    const uint32_t r_beg = (uint32_t)(((uint64_t)nrec * blockIdx.x) / gridDim.x);
    const uint32_t r_end = (uint32_t)(((uint64_t)nrec * (blockIdx.x + 1)) / gridDim.x);
    int cur = -1;
    bool on = false, bs = false;
    uint32_t nr = 0, tlo = 0, skx = 0, ska = 0;
    uint32_t tk[NL], c[NL];
#pragma unroll
    for (int j = 0; j < NL; j++) { c[j] = 0; tk[j] = 0x7FFFFFFFu; }
    float mean_f = 0.f, inv_d = 0.f;

    auto flush = [&](int l) {
        if (!on) return;
        LayerState &S = w.st[l];
        if (!bs) {
#pragma unroll
            for (int j = 0; j < NL; j++) {
                uint32_t v = __reduce_add_sync(FULLMASK, c[j]);
                if (lane == 0 && v) atomicAdd(&s_cnt[j], v);
                c[j] = 0;
            }
        }
        __syncthreads();
        if (!bs && tid < NL) {
            if (s_cnt[tid]) atomicAdd(&S.trim_cnt[tid], s_cnt[tid]);
            s_cnt[tid] = 0;
        }
        if (bs) {
            for (int b = tid; b < kBsTable; b += kThreads) {
                uint32_t v = s_hist[b];
                if (v) { atomicAdd(&S.hist[b], v); s_hist[b] = 0u; }
            }
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            unsigned int old = atomicAdd(&S.k2_done, nr);
            s_flag[1] = (old + nr == w.desc[l].cand_nb);
        }
        __syncthreads();
        if (s_flag[1]) k2_finalize<NL, kThreads>(w, l, L, s_hist, s_w, s_tp, msg_hdr, hdr_words, 0);
    };

    constexpr int U = 8;    // independent loads in flight per thread
    for (uint32_t r = r_beg; r < r_end; r++) {
        const int l = find_layer(s_rb, L, r);
        const uint2 rec = w.rec[r];     // issued with the layer's state below (one round trip)
        const LayerDesc &d = w.desc[l];
        const uint2 *src = w.cand + (uint64_t)(d.cand_b0 + (r - s_rb[l])) * w.cand_R + rec.x;
        // a batch of raw value bits (0 past the record: key 0 counts nowhere)
        uint32_t kq[U];
        auto load_batch = [&](uint32_t i0) {
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t i = i0 + u * kThreads + tid;
                kq[u] = i < rec.y ? __ldcg(&src[i].y) : 0u;
            }
        };
        if (l != cur) {
            if (cur >= 0) flush(cur);
            cur = l; nr = 0;
            const LayerState &S = w.st[l];
            // every field the layer needs, loaded together (no load behind a branch on another;
            // the threshold table is read whatever the selector: one round trip, not two)
            const uint32_t k2src = S.k2src, sel = d.selector, sx = S.skx, sa = S.ska;
            const uint32_t mk = S.maxkey, jl = bs_jlo(S, 0);
            const double mean = S.mean;
            constexpr int TPQ = (kBsLevels + kThreads) / kThreads;   // table entries per thread
            uint32_t tq0[TPQ], tq1[TPQ], tl0[NL];
#pragma unroll
            for (int q = 0; q < TPQ; q++) {
                const int j = tid + q * kThreads;
                tq0[q] = j <= kBsLevels ? S.tkeys[j] : 0u;
                tq1[q] = j <= kBsLevels ? S.tkeys[j + 1] : 0u;
            }
#pragma unroll
            for (int j = 0; j < NL; j++) tl0[j] = S.tkeys[j];
            on = k2src != 0u;
            bs = sel != RGC_SEL_TRIMMED;
            skx = sx; ska = sa;
            if (on && bs) {
#pragma unroll
                for (int q = 0; q < TPQ; q++) {
                    const int j = tid + q * kThreads;
                    if (j <= kBsLevels) s_tp[j] = make_uint2(tq0[q], tq1[q]);
                }
                const float mx = __uint_as_float(mk);
                mean_f = (float)mean;
                inv_d = 1024.0f / (mx - mean_f);
            } else if (on) {
#pragma unroll
                for (int j = 0; j < NL; j++) tk[j] = tl0[j];
            }
            if (on) load_batch(0);      // in flight across the barrier
            __syncthreads();
            if (on && bs) tlo = s_tp[jl].x;   // t_jlo, from the staged table
        } else if (on) {
            load_batch(0);
        }
        if (!on) continue;
        for (uint32_t i0 = 0; i0 < rec.y; i0 += U * kThreads) {
          if (i0) load_batch(i0);
#pragma unroll
          for (int u = 0; u < U; u++) kq[u] = skey(kq[u], skx, ska);
#pragma unroll
          for (int u = 0; u < U; u++) {
            const uint32_t kk = kq[u];
            if (!bs) {
#pragma unroll
                for (int j = 0; j < NL; j++) c[j] += (kk > tk[j]) ? 1u : 0u;
            } else if (kk > tlo) {
                // bin b = #{j : t_j < |x|}: linear estimate verified on (t_{b-1}, t_b)
                const float jf = (__uint_as_float(kk) - mean_f) * inv_d;
                int b = __float2int_rz(fminf(fmaxf(jf, 0.f), 1024.f));
                const uint2 pr = s_tp[b];
                if ((pr.x < kk) & (kk <= pr.y)) {
                    b += 1;
                } else {
                    int lo = 1, hi = kBsLevels + 1;   // smallest b with kk <= t_b
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (kk <= s_tp[mid].x) hi = mid; else lo = mid + 1;
                    }
                    b = lo;
                }
                atomicAdd(&s_hist[b], 1u);
            }
          }
        }
        nr++;
    }
    if (cur >= 0) flush(cur);
    if (!fold) return;
    __syncthreads();
    // V pass 0 over the layers the stash did not cover (independent of the stash pass's
    // layers: no barrier before it)
    if (vpass0)
        k2_vpass_call<NL>(w, L, total_tiles, msg_hdr, hdr_words, 0, s_rb, s_tp, s_hist, s_cnt, s_w, s_flag);
    // V pass 1 needs every decision of the stash pass and pass 0 (need_full / any_full): one
    // grid barrier (the grid is small enough to be co-resident beside a zero-fill CTA)
    grid_barrier(w.ctrl, msg_hdr, L);
    if (*(volatile unsigned int *)&w.ctrl->any_full != 0u)
        k2_vpass_call<NL>(w, L, total_tiles, msg_hdr, hdr_words, 1, s_rb, s_tp, s_hist, s_cnt, s_w, s_flag);
}

// ============================================================================
// K4: radix select of the k-th largest key (11/11/9-bit digits)
// ============================================================================
__device__ void k4_finalize(const Ws &w, int l, int pass, uint32_t *s_hist, uint32_t *s_w) {
    __threadfence();
    LayerState &S = w.st[l];
    const bool two = S.rs_two != 0u;
    if (two && pass == 2) {                 // decided after two digits (K4 pass 1)
        __syncthreads();
        if (threadIdx.x == 0) S.k4_done = 0;
        __syncthreads();
        return;
    }
    const int shift = two ? (pass == 0 ? 11 : 0) : (pass == 0 ? 20 : (pass == 1 ? 9 : 0));
    const int nb = (!two && pass == 2) ? 512 : 2048;
    uint32_t loc[8];
    uint32_t tsum = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        int b = threadIdx.x * 8 + i;
        loc[i] = b < nb ? atomicExch(&S.hist[b], 0u) : 0u;
        tsum += loc[i];
    }
    uint32_t incl = block_incl_scan(tsum, s_w);
    __shared__ uint32_t s_total, s_digit, s_above;
    if (threadIdx.x == kThreads - 1) s_total = incl;
    __syncthreads();
    const uint32_t krem = S.rs_krem;
    uint32_t run = incl - tsum;   // elements in bins < this thread's first bin
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const uint32_t above = s_total - run - loc[i];   // elements in bins > b
        if (loc[i] && above < krem && krem <= above + loc[i]) {
            s_digit = threadIdx.x * 8 + i;
            s_above = above;
        }
        run += loc[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        S.rs_prefix |= s_digit << shift;
        S.rs_above += s_above;
        S.rs_krem = krem - s_above;
        // ASQ: fewer than k keys of the phase's sign -> only those (no tie at key 0)
        if (pass == 2 && S.ska && S.rs_prefix == 0u) S.rs_krem = 0u;
        if (two && pass == 1) {             // offset digits -> the k-th key itself
            S.rs_prefix += S.rs_base;
            S.info.kth_key = S.rs_prefix;
            S.info.tie_quota = S.rs_krem;
        }
        if (pass == 2) {
            S.info.kth_key = S.rs_prefix;
            S.info.tie_quota = S.rs_krem;
        }
        S.k4_done = 0;
    }
    __syncthreads();
}

// K4: radix passes pass_begin .. pass_end-1 (one per launch, or all three in one cooperative
// launch with grid barriers between them; the next pass reads the digits the previous
// pass's per-layer finalisations chose)
__global__ void __launch_bounds__(kThreads)
k4_radix(Ws w, int L, int pass_begin, int pass_end, uint32_t *msg_hdr) {
    pdl_wait();
    TlMark tlm(w.tl, TL_K4);
    __shared__ uint32_t s_tb[RGC_MAX_LAYERS + 1];
    __shared__ uint32_t s_hist[kRadixBins];
    __shared__ uint32_t s_w[kWarps];
    __shared__ int s_last;
    const int tid = threadIdx.x;
    const uint32_t total = w.ctrl->k4_total;
    if (total == 0) return;
  for (int pass = pass_begin; pass < pass_end; pass++) {
    if (pass > pass_begin) grid_barrier(w.ctrl, msg_hdr, L);
    for (int l = tid; l < L; l += kThreads) s_tb[l] = w.st[l].k4_begin;
    if (tid == 0) s_tb[L] = total;
    for (int b = tid; b < kRadixBins; b += kThreads) s_hist[b] = 0u;
    __syncthreads();
    // digit geometry per layer: three digits of the raw key (11/11/9 bits), or two 11-bit
    // digits of the offset key - rs_base for Alg.2 survivors within 2^22 keys above the
    // level threshold (S.rs_two; pass 2 then only closes the layer)
    int shift = 0, hishift = 31;
    uint32_t dmask = 2047u, base = 0;
    bool skip = false;
    int cur = -1;
    uint32_t ntl = 0, prefix = 0, nsrc = 0, skx = 0, ska = 0;
    bool fromS = false;
    const float *V = nullptr;
    const uint2 *src = nullptr;

    auto flush = [&](int l) {
        __syncthreads();
        LayerState &S = w.st[l];
        for (int b = tid; b <= (int)dmask; b += kThreads) {
            uint32_t v = s_hist[b];
            if (v) { atomicAdd(&S.hist[b], v); s_hist[b] = 0u; }
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            unsigned int old = atomicAdd(&S.k4_done, ntl);
            s_last = (old + ntl == S.k4_tiles);
        }
        __syncthreads();
        if (s_last) k4_finalize(w, l, pass, s_hist, s_w);
    };

    for (uint32_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
        const int l = find_layer(s_tb, L, tile);
        if (l != cur) {
            if (cur >= 0) flush(cur);
            cur = l; ntl = 0;
            const LayerState &S = w.st[l];
            const LayerDesc &d = w.desc[l];
            prefix = S.rs_prefix;
            skx = S.skx; ska = S.ska;
            fromS = S.mode == MODE_SURV;
            nsrc = fromS ? S.surv : d.n;
            V = d.V;
            src = w.S + d.s_off;
            const bool two = S.rs_two != 0u;
            base = two ? S.rs_base : 0u;
            skip = two && pass == 2;
            shift = two ? (pass == 0 ? 11 : 0) : (pass == 0 ? 20 : (pass == 1 ? 9 : 0));
            dmask = (!two && pass == 2) ? 511u : 2047u;
            hishift = pass == 0 ? 31 : (two ? 11 : (pass == 1 ? 20 : 9));
        }
        const uint32_t t0 = (tile - s_tb[l]) * kTile;
        if (!skip) {
#pragma unroll 4
            for (int e = 0; e < kPerThread; e++) {
                const uint32_t p = t0 + e * kThreads + tid;
                if (p < nsrc) {
                    const uint32_t kk = skey(fromS ? src[p].y : __float_as_uint(V[p]), skx, ska) - base;
                    if (hishift == 31 || (kk >> hishift) == (prefix >> hishift))
                        atomicAdd(&s_hist[(kk >> shift) & dmask], 1u);
                }
            }
        }
        ntl++;
    }
    if (cur >= 0) flush(cur);
  }
}

// ============================================================================
// K6: decompress -- rank-ordered scatter-add into the dense averaged gradient
// ============================================================================
// load_layout(), layer_view(), view_entry(): rgc_device.cuh

// dec_start[r][slot]: index (in rank r's compact pair array) of the first pair
// whose element index >= 8192*t, for slot = ddesc[l].slot_begin + t, t = 0..ntiles_l.
__global__ void __launch_bounds__(kThreads)
k6_prep(Ws w, int L, int p, MsgSrc src, uint32_t hdr_words, uint32_t total_dec_tiles,
        uint32_t max_pairs) {
    pdl_wait();
    TlMark tlm(w.tl, TL_PREP);
    extern __shared__ uint32_t s_dyn[];
    uint32_t *s_off = s_dyn;                      // [p][L+1] rank-local layer offsets (entries)
    uint32_t *s_ao = s_dyn + p * (L + 1);         // [p][L+1] ASQ entries before each layer
    uint32_t *s_sb = s_dyn + 2 * p * (L + 1);     // [L] slot_begin
    const int tid = threadIdx.x;
    for (int l = tid; l < L; l += kThreads) s_sb[l] = w.ddesc[l].slot_begin;
    load_layout(src, L, p, s_off, s_ao);
    if (blockIdx.x == 0 && blockIdx.y == 0)   // where every (rank, layer) set sits, for K6
        for (int i = tid; i < p * L; i += kThreads) {
            const int r = i / L, l = i % L;
            w.dec_lay[i] = layer_view(reinterpret_cast<const uint32_t *>(src.of(r)),
                                      s_off + r * (L + 1), s_ao + r * (L + 1), L, l);
        }
    const uint32_t nslots = total_dec_tiles + L;
    // grid (x, p): blockIdx.y = the rank whose block this CTA indexes (no divisions)
    const int r = blockIdx.y;
    const uint32_t *o = s_off + r * (L + 1);
    uint32_t *dst = w.dec_start + (uint64_t)r * nslots;
    const uint32_t gtid = blockIdx.x * kThreads + tid, stride = gridDim.x * kThreads;
    // empty (rank, layer) sets: every slot of the layer = the layer offset
    for (uint32_t sl = gtid; sl < nslots; sl += stride) {
        const int l = find_layer(s_sb, L, sl);
        if (o[l + 1] == o[l]) dst[sl] = o[l];
    }
    // non-empty sets: tile boundaries between consecutive (ascending) indices
    const uint32_t *hdr = reinterpret_cast<const uint32_t *>(src.of(r));
    const uint32_t *pw = hdr + hdr_words;
    const uint32_t tot = min(o[L], max_pairs);
    for (uint32_t g = gtid; g < tot; g += stride) {
        const int l = find_layer(o, L, g);
        const uint4 v = layer_view(hdr, o, s_ao + r * (L + 1), L, l);
        uint32_t *out = dst + s_sb[l];
        const int t = (int)(view_entry(pw, v, g).x / kDecTile);
        const int tprev = (g > o[l]) ? (int)(view_entry(pw, v, g - 1).x / kDecTile) : -1;
        for (int tt = tprev + 1; tt <= t; tt++) out[tt] = g;
        if (g + 1 == o[l + 1]) {
            const uint32_t nt = w.ddesc[l].ntiles;
            for (uint32_t tt = t + 1; tt <= nt; tt++) out[tt] = g + 1;
        }
    }
}

__global__ void __launch_bounds__(kThreads)
k6_decompress(Ws w, int L, int p, MsgSrc src, uint32_t hdr_words, uint32_t total_dec_tiles,
              float scale) {
    pdl_wait();
    __shared__ float4 acc4[kDecTile / 4];
    __shared__ uint32_t s_tb[RGC_MAX_LAYERS + 1];
    __shared__ uint32_t s_rng[2 * 64];
    __shared__ int s_any;
    float *acc = reinterpret_cast<float *>(acc4);
    const int tid = threadIdx.x;
    for (int l = tid; l < L; l += kThreads) s_tb[l] = w.ddesc[l].tile_begin;
    if (tid == 0) s_tb[L] = total_dec_tiles;
    __syncthreads();
    const uint32_t nslots = total_dec_tiles + L;
    for (uint32_t tile = blockIdx.x; tile < total_dec_tiles; tile += gridDim.x) {
        const int l = find_layer(s_tb, L, tile);
        const DecompDesc &dd = w.ddesc[l];
        const uint32_t lt = tile - s_tb[l];
        const uint32_t t0 = lt * kDecTile;
        const uint32_t cnt = min((uint32_t)kDecTile, dd.n - t0);
        if (tid == 0) s_any = 0;
        __syncthreads();
        for (int r = tid; r < p; r += kThreads) {
            const uint32_t *ds = w.dec_start + (uint64_t)r * nslots + dd.slot_begin + lt;
            const uint32_t a = ds[0], b = ds[1];
            s_rng[2 * r] = a; s_rng[2 * r + 1] = b;
            if (b > a) s_any = 1;
        }
        __syncthreads();
        float *out = dd.out + t0;
        if (!s_any) {
            // no rank sent an index of this tile: +0 * (1/p) = +0
            if (cnt == kDecTile) {
                float4 *o4 = reinterpret_cast<float4 *>(out);
#pragma unroll
                for (int j = 0; j < kDecTile / 4 / kThreads; j++)
                    o4[j * kThreads + tid] = make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
                for (uint32_t i = tid; i < cnt; i += kThreads) out[i] = 0.f;
            }
            __syncthreads();
            continue;
        }
#pragma unroll
        for (int j = 0; j < kDecTile / 4 / kThreads; j++)
            acc4[j * kThreads + tid] = make_float4(0.f, 0.f, 0.f, 0.f);
        __syncthreads();
        for (int r = 0; r < p; r++) {
            const uint32_t *pw = reinterpret_cast<const uint32_t *>(src.of(r)) + hdr_words;
            const uint32_t a = s_rng[2 * r], b = s_rng[2 * r + 1];
            const uint4 v = w.dec_lay[r * L + l];
            for (uint32_t j = a + tid; j < b; j += kThreads) {
                const uint2 pr = view_entry(pw, v, j);
                float *dstp = acc + (pr.x - t0);
                *dstp = __fadd_rn(*dstp, __uint_as_float(pr.y));   // rank order (R14)
            }
            __syncthreads();
        }
        if (cnt == kDecTile) {
            float4 *o4 = reinterpret_cast<float4 *>(out);
#pragma unroll
            for (int j = 0; j < kDecTile / 4 / kThreads; j++) {
                float4 v = acc4[j * kThreads + tid];
                o4[j * kThreads + tid] = make_float4(__fmul_rn(v.x, scale), __fmul_rn(v.y, scale),
                                                     __fmul_rn(v.z, scale), __fmul_rn(v.w, scale));
            }
        } else {
            for (uint32_t i = tid; i < cnt; i += kThreads) out[i] = __fmul_rn(acc[i], scale);
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kThreads)
k6_zero(Ws w, int L, uint32_t total_dec_tiles) {
    pdl_wait();
    __shared__ uint32_t s_tb[RGC_MAX_LAYERS + 1];
    const int tid = threadIdx.x;
    for (int l = tid; l < L; l += kThreads) s_tb[l] = w.ddesc[l].tile_begin;
    if (tid == 0) s_tb[L] = total_dec_tiles;
    __syncthreads();
    for (uint32_t tile = blockIdx.x; tile < total_dec_tiles; tile += gridDim.x) {
        const int l = find_layer(s_tb, L, tile);
        const DecompDesc &dd = w.ddesc[l];
        const uint32_t t0 = (tile - s_tb[l]) * kDecTile;
        const uint32_t cnt = min((uint32_t)kDecTile, dd.n - t0);
        float *out = dd.out + t0;
        if (cnt == kDecTile) {
            float4 *o4 = reinterpret_cast<float4 *>(out);
#pragma unroll
            for (int j = 0; j < kDecTile / 4 / kThreads; j++)
                o4[j * kThreads + tid] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
            for (uint32_t i = tid; i < cnt; i += kThreads) out[i] = 0.f;
        }
    }
}

// unordered variant: out[i] += v * (1/p) with atomics (tolerance-checked, R14)
__global__ void __launch_bounds__(kThreads)
k6_atomic(Ws w, int L, int p, MsgSrc src, uint32_t hdr_words, uint32_t max_pairs, float scale) {
    pdl_wait();
    extern __shared__ uint32_t s_dyn[];
    uint32_t *s_off = s_dyn, *s_ao = s_dyn + p * (L + 1);
    const int tid = threadIdx.x;
    load_layout(src, L, p, s_off, s_ao);
    for (uint64_t it = blockIdx.x * (uint64_t)kThreads + tid; it < (uint64_t)p * max_pairs;
         it += (uint64_t)gridDim.x * kThreads) {
        const int r = (int)(it / max_pairs);
        const uint32_t g = (uint32_t)(it % max_pairs);
        const uint32_t *o = s_off + r * (L + 1);
        if (g >= o[L]) continue;
        const int lo = find_layer(o, L, g);
        const uint32_t *hdr = reinterpret_cast<const uint32_t *>(src.of(r));
        const uint2 pr = view_entry(hdr + hdr_words, layer_view(hdr, o, s_ao + r * (L + 1), L, lo), g);
        atomicAdd(w.ddesc[lo].out + pr.x, __fmul_rn(__uint_as_float(pr.y), scale));
    }
}

// ============================================================================
// launchers
// ============================================================================
cudaError_t launch_k1(const Ws &w, int L, uint32_t total_tiles, uint32_t *, int grid,
                      cudaStream_t s) {
    cudaError_t e = launch_pdl(k1_accumulate, grid, kThreads, 0, s, w, L, total_tiles);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_k2(const Ws &w, int L, uint32_t total_tiles, int max_trim_levels,
                      uint32_t *msg_hdr, uint32_t hdr_words, int grid, uint32_t nrec,
                      int grid_stash, cudaStream_t s, uint64_t *launches) {
    // fold the V passes into the stash launch for small layer lists only (<= 1024 tiles = 4M
    // elements; RGC_FOLD_K2_TILES overrides, RGC_NO_FOLD_K2 disables): C1 (1M) 76 -> 69 us, but
    // on VGG16 / ResNet-50 / M1 a V pass that works runs slower on the stash grid (2 CTAs/SM)
    // than as its own launch (4/SM) and the steps lose 1-4 us (profiles/r02/k2_fold_ab.txt)
    static const uint32_t fold_max = [] {
        if (getenv("RGC_NO_FOLD_K2")) return 0u;
        const char *e = getenv("RGC_FOLD_K2_TILES");
        return e ? (uint32_t)strtoul(e, nullptr, 10) : 1024u;
    }();
    const int fold = (nrec && total_tiles <= fold_max) ? 1 : 0;
    if (nrec) {
        const int gs = (int)(nrec < (uint32_t)grid_stash ? nrec : (uint32_t)grid_stash);
        cudaError_t e;
        if (max_trim_levels <= 5) e = launch_pdl(k2_stash<5>, gs, kThreads, 0, s, w, L, nrec, msg_hdr, hdr_words, total_tiles, fold);
        else if (max_trim_levels <= 8) e = launch_pdl(k2_stash<8>, gs, kThreads, 0, s, w, L, nrec, msg_hdr, hdr_words, total_tiles, fold);
        else e = launch_pdl(k2_stash<16>, gs, kThreads, 0, s, w, L, nrec, msg_hdr, hdr_words, total_tiles, fold);
        if (e != cudaSuccess) return e;
        if (launches) *launches += 1;
    }
    if (fold) return cudaSuccess;   // the V passes ran inside k2_stash
    for (int pass = 0; pass < 2; pass++) {
        cudaError_t e;
        if (max_trim_levels <= 5)
            e = launch_pdl(k2_count<5>, grid, kThreads, 0, s, w, L, total_tiles, msg_hdr, hdr_words, pass);
        else if (max_trim_levels <= 8)
            e = launch_pdl(k2_count<8>, grid, kThreads, 0, s, w, L, total_tiles, msg_hdr, hdr_words, pass);
        else
            e = launch_pdl(k2_count<16>, grid, kThreads, 0, s, w, L, total_tiles, msg_hdr, hdr_words, pass);
        if (e != cudaSuccess) return e;
        if (launches) *launches += 1;
    }
    return cudaSuccess;
}

cudaError_t launch_k4(const Ws &w, int L, int pass, int grid, cudaStream_t s) {
    return launch_pdl(k4_radix, grid, kThreads, 0, s, w, L, pass, pass + 1, (uint32_t *)nullptr);
}

cudaError_t launch_k4_all(const Ws &w, int L, uint32_t *msg_hdr, int sms, cudaStream_t s,
                          uint64_t *launches, bool expect_work) {
    static int occ = -1;
    if (occ < 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k4_radix, kThreads, 0) != cudaSuccess)
            occ = 0;
    }
    // The one-launch form saves two launches when K4 has no work (the common case: Alg.2's
    // survivors fit K45's clusters) but its grid barriers cost more than the launch
    // boundaries when it does (VGG16 all-trimmed +5 us, M1 trimmed +10 us): the host uses it
    // when the previous call had no K4 work (expect_work false).  Both forms are exact.
    static const bool coop_ok = getenv("RGC_NO_COOP_K4") == nullptr;
    if (coop_ok && occ > 0 && !expect_work) {
        cudaLaunchConfig_t cfg = {};
        // at most 4 CTAs per SM: they stay co-resident beside a zero-fill CTA still running
        // on the auxiliary stream (512 threads, 16K registers)
        cfg.gridDim = dim3(sms * (occ < 4 ? occ : 4));
        cfg.blockDim = dim3(kThreads);
        cfg.stream = s;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl_enabled() ? 2 : 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k4_radix, w, L, 0, 3, msg_hdr);
        if (e == cudaSuccess) { *launches += 1; return e; }
        cudaGetLastError();   // refused (e.g. co-residency): three plain launches instead
    }
    for (int pass = 0; pass < 3; pass++) {
        cudaError_t e = launch_k4(w, L, pass, sms * (occ > 0 ? occ : 1), s);
        if (e != cudaSuccess) return e;
        *launches += 1;
    }
    return cudaSuccess;
}

// dynamic shared memory above the 48 KB default (p up to 64 ranks, L up to 128 layers)
static cudaError_t allow_smem(const void *f) {
    return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)((2 * 64 * (RGC_MAX_LAYERS + 1) + RGC_MAX_LAYERS) * 4));
}

cudaError_t launch_k6_prep(const Ws &w, int L, int p, const MsgSrc &src, uint32_t hdr_words,
                           uint32_t total_dec_tiles, int grid, cudaStream_t s, uint32_t max_pairs) {
    static cudaError_t attr = allow_smem((const void *)k6_prep);
    if (attr != cudaSuccess) return attr;
    size_t smem = ((size_t)2 * p * (L + 1) + L) * sizeof(uint32_t);
    // one grid row per rank: (grid / p) x p CTAs (at least one per rank)
    const int gx = grid / p > 0 ? grid / p : 1;
    return launch_pdl(k6_prep, dim3(gx, p), dim3(kThreads), smem, s, w, L, p, src, hdr_words,
                      total_dec_tiles, max_pairs);
}

cudaError_t launch_k6(const Ws &w, int L, int p, const MsgSrc &src, uint32_t hdr_words,
                      uint32_t total_dec_tiles, float scale, int grid, cudaStream_t s) {
    return launch_pdl(k6_decompress, grid, kThreads, 0, s, w, L, p, src, hdr_words, total_dec_tiles, scale);
}

cudaError_t launch_k6_atomic(const Ws &w, int L, int p, const MsgSrc &src, uint32_t hdr_words,
                             uint32_t total_dec_tiles, uint32_t max_pairs, float scale, int grid,
                             cudaStream_t s) {
    k6_zero<<<grid, kThreads, 0, s>>>(w, L, total_dec_tiles);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    static cudaError_t attr = allow_smem((const void *)k6_atomic);
    if (attr != cudaSuccess) return attr;
    size_t smem = (size_t)2 * p * (L + 1) * sizeof(uint32_t);
    k6_atomic<<<grid, kThreads, smem, s>>>(w, L, p, src, hdr_words, max_pairs, scale);
    return cudaGetLastError();
}

cudaError_t launch_k6_atomic_only(const Ws &w, int L, int p, const MsgSrc &src, uint32_t hdr_words,
                                  uint32_t max_pairs, float scale, int grid, cudaStream_t s) {
    static cudaError_t attr = allow_smem((const void *)k6_atomic);
    if (attr != cudaSuccess) return attr;
    size_t smem = (size_t)2 * p * (L + 1) * sizeof(uint32_t);
    k6_atomic<<<grid, kThreads, smem, s>>>(w, L, p, src, hdr_words, max_pairs, scale);
    return cudaGetLastError();
}

cudaError_t occupancy(int *k1, int *k2, int *k3, int *k4, int *k6) {
    cudaError_t e0 = occupancy_k3(k3);
    if (e0 != cudaSuccess) return e0;
    cudaError_t e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(k1, k1_accumulate, kThreads, 0))) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(k2, k2_count<5>, kThreads, 0))) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(k4, k4_radix, kThreads, 0))) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(k6, k6_decompress, kThreads, 0))) return e;
    return cudaSuccess;
}

}  // namespace rgc
