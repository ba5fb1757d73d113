// rgc_select.cu -- K45: exact top-k (radixSelect) and the
// ordered emission of the selected <index, value> pairs with the residual /
// momentum masking, fused in ONE thread-block cluster per layer
// for candidate sets of up to kSmallSel elements: the Alg.2 survivors (P:181
// "radixSelect on the remaining elements") or a small layer in an exact
// fallback.  Larger sets take the multi-CTA K4 passes + K3 pass B.
//
// Cluster of 4 (or 2, chosen by the host from the layer list) CTAs of 1024 threads;
// CTA r stages the 31-bit keys of its contiguous slice of the candidates in its shared
// memory once (up to 45056 keys, 176 KB).
// Select: three MSB-first digit passes (11/11/9 bits) -- or two 11-bit digits of
// key - (t_j + 1) when the Alg.2 survivors span < 2^22 keys; each CTA histograms
// its slice in shared memory, cluster rank 0 sums the histograms through
// distributed shared memory (DSMEM) and picks the digit holding the k-th
// largest key.  Result: T* and the number q of elements equal to T* to take
// (lower index first, R6).
// Emit: per-CTA (gt, eq) counts, a cluster prefix over DSMEM, then per-warp
// chunks with ballot ranks -- ascending index order overall.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "rgc_device.cuh"

namespace cg = cooperative_groups;

namespace rgc {

#ifndef RGC_T45
#define RGC_T45 1024
#endif
constexpr int kT45 = RGC_T45;                    // threads per CTA
constexpr int kW45 = kT45 / 32;
constexpr int kBpt = kRadixBins / kT45;          // histogram bins per thread in the scan
constexpr int kKeysPerCta = kKeysPerCta45;   // keys per CTA (dynamic smem, 176 KB)

// CL CTAs per layer: 4 (180K-key sets), or 2 (90K-key sets) when the layers that can take K45
// need more than one wave of 4-CTA clusters (ResNet-50: 53 conv layers; the host picks, from
// the layer list, rgc_api.cu)
template <int CL>
__global__ void __launch_bounds__(kT45, 1024 / kT45)
k45_cluster(Ws w, int L, uint2 *msg_pairs) {
    constexpr int kCluster = CL;
    pdl_wait();
    TlMark tlm(w.tl, TL_K45);
    extern __shared__ uint32_t s_key[];          // [kKeysPerCta] keys of this CTA's slice
    __shared__ uint32_t s_hist[kRadixBins];
    __shared__ uint32_t s_part[kW45];
    __shared__ uint32_t s_wg[kW45], s_we[kW45];
    __shared__ uint32_t s_ctl[4];                // [0] digit [1] above (rank 0); [2] gt [3] eq
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int l = blockIdx.x / kCluster;
    if (l >= L) return;                          // uniform over the cluster
    LayerState &S = w.st[l];
    if (!S.small) return;                        // uniform over the cluster
    const LayerDesc &d = w.desc[l];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool fromS = S.mode == MODE_SURV;
    const uint32_t n = fromS ? S.surv : d.n;
    const uint2 *src = w.S + d.s_off;
    float *V = d.V;
    float *u = d.u;
    const uint32_t chunk = (n + kCluster - 1) / kCluster;
    const uint32_t c0 = min(n, (uint32_t)rank * chunk);
    const uint32_t m = min(n, c0 + chunk) - c0;   // <= kKeysPerCta

    // ---- stage this slice's keys (8 loads in flight per thread)
    for (uint32_t i0 = 0; i0 < m; i0 += 8 * kT45) {
        uint32_t kv[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint32_t i = i0 + j * kT45 + tid;
            kv[j] = i < m ? skey(fromS ? src[c0 + i].y : __float_as_uint(V[c0 + i]), S.skx, S.ska)
                          : 0u;
        }
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint32_t i = i0 + j * kT45 + tid;
            if (i < m) s_key[i] = kv[j];
        }
    }

    // ---- radix select of the k-th largest key over the whole cluster.  Alg.2 survivors
    // all lie in (t_j, max|V|]; when that range spans < 2^22 keys (t_0 >= 0.8 max: the usual
    // case) the select runs on the offset key - (t_j + 1) in two 11-bit digits instead of
    // three digits of the raw 31-bit key (one histogram pass and two cluster barriers fewer)
    const bool two = fromS && S.maxkey - S.thr_key < (1u << 22);
    const uint32_t base = two ? S.thr_key + 1u : 0u;
    const int npass = two ? 2 : 3;
    uint32_t prefix = 0, krem = d.k;
#pragma unroll 1
    for (int pass = 0; pass < npass; pass++) {
        const int shift = two ? (pass == 0 ? 11 : 0) : (pass == 0 ? 20 : (pass == 1 ? 9 : 0));
        const uint32_t dmask = (!two && pass == 2) ? 511u : 2047u;
        const int hishift = pass == 0 ? 31 : (two ? 11 : (pass == 1 ? 20 : 9));
        for (int b = tid; b < kRadixBins; b += kT45) s_hist[b] = 0u;
        __syncthreads();
        for (uint32_t i = tid; i < m; i += kT45) {
            const uint32_t kk = s_key[i] - base;
            if (hishift == 31 || (kk >> hishift) == (prefix >> hishift))
                atomicAdd(&s_hist[(kk >> shift) & dmask], 1u);
        }
        cluster.sync();
        if (rank == 0) {
            // sum the cluster's histograms (kBpt bins per thread) and scan from the top
            uint32_t h[kBpt], hs = 0;
#pragma unroll
            for (int i = 0; i < kBpt; i++) h[i] = 0u;
#pragma unroll
            for (int r = 0; r < kCluster; r++) {
                const uint32_t *rh = cluster.map_shared_rank(s_hist, r);
#pragma unroll
                for (int i = 0; i < kBpt; i++) h[i] += rh[kBpt * tid + i];
            }
#pragma unroll
            for (int i = 0; i < kBpt; i++) hs += h[i];
            uint32_t x = hs;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_down_sync(FULLMASK, x, o);
                if (lane + o < 32) x += y;
            }
            if (lane == 0) s_part[warp] = x;
            __syncthreads();
            uint32_t addw = 0;
            for (int i = warp + 1; i < kW45; i++) addw += s_part[i];
            uint32_t above = x + addw - hs;               // keys in bins > kBpt*tid + kBpt-1
#pragma unroll
            for (int i = kBpt - 1; i >= 0; i--) {         // above = keys in bins > kBpt*tid + i
                if (h[i] && above < krem && krem <= above + h[i]) { s_ctl[0] = kBpt * tid + i; s_ctl[1] = above; }
                above += h[i];
            }
        }
        cluster.sync();
        const uint32_t *ctl0 = cluster.map_shared_rank(s_ctl, 0);
        const uint32_t digit = ctl0[0], above = ctl0[1];
        prefix |= digit << shift;
        krem -= above;
    }
    const uint32_t T = prefix + base;
    // ASQ: fewer than k keys of the phase's sign -> only those (no tie at key 0)
    const uint32_t q = (S.ska && T == 0u) ? 0u : krem;

    // ---- ordered emission: CTA totals, cluster prefix over DSMEM, warp ballot ranks
    const uint32_t per = (m + kW45 - 1) / kW45;
    const uint32_t w0 = min(m, warp * per), w1 = min(m, w0 + per);
    uint32_t wg = 0, we = 0;
    for (uint32_t b = w0; b < w1; b += 32) {
        const uint32_t i = b + lane;
        const uint32_t kk = i < w1 ? s_key[i] : 0u;
        wg += __popc(__ballot_sync(FULLMASK, i < w1 && kk > T));
        we += __popc(__ballot_sync(FULLMASK, i < w1 && kk == T));
    }
    if (lane == 0) { s_wg[warp] = wg; s_we[warp] = we; }
    __syncthreads();
    if (tid == 0) {
        uint32_t tg = 0, te = 0;
        for (int i = 0; i < kW45; i++) { tg += s_wg[i]; te += s_we[i]; }
        s_ctl[2] = tg; s_ctl[3] = te;
    }
    cluster.sync();
    uint32_t gb = 0, eb = 0;
    for (int r = 0; r < rank; r++) {
        const uint32_t *cr = cluster.map_shared_rank(s_ctl, r);
        gb += cr[2]; eb += cr[3];
    }
    for (int i = 0; i < warp; i++) { gb += s_wg[i]; eb += s_we[i]; }
    uint2 *dst = (d.quant ? w.Q : msg_pairs) + S.msg_off;
    const uint32_t lt = (1u << lane) - 1u;
    for (uint32_t b = w0; b < w1; b += 32) {
        const uint32_t i = b + lane;
        const uint32_t kk = i < w1 ? s_key[i] : 0u;
        const bool isg = i < w1 && kk > T, ise = i < w1 && kk == T;
        const uint32_t G = __ballot_sync(FULLMASK, isg), E = __ballot_sync(FULLMASK, ise);
        const uint32_t g = gb + __popc(G & lt), eq = eb + __popc(E & lt);
        if (isg || (ise && eq < q)) {
            const uint32_t outpos = isg ? g + min(eq, q) : g + eq;
            const uint32_t gi = c0 + i;
            const uint2 e = fromS ? src[gi] : make_uint2(gi, __float_as_uint(V[gi]));
            RGC_DCHECK(outpos < max(d.cap, d.k) && e.x < d.n);
            dst[outpos] = e;                      // <index, value>
            V[e.x] = 0.0f;                        // V <- V (.) (1 - Masks)
            if (u) u[e.x] = 0.0f;                 // momentum masking
        }
        gb += __popc(G); eb += __popc(E);
    }
    if (rank == 0 && tid == 0) {
        S.rs_prefix = T;
        S.rs_krem = q;
        S.info.kth_key = T;
        S.info.tie_quota = q;
        S.emitted_b = d.k - krem + q;
    }
    cluster.sync();                               // peers' shared memory stays live until here
}

template <int CL>
cudaError_t launch_k45_cl(const Ws &w, int L, uint2 *msg_pairs, cudaStream_t s) {
    static bool attr = false;
    const size_t smem = sizeof(uint32_t) * kKeysPerCta;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k45_cluster<CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(L * CL);
    cfg.blockDim = dim3(kT45);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, k45_cluster<CL>, w, L, msg_pairs);
}

cudaError_t launch_k45(const Ws &w, int L, uint2 *msg_pairs, cudaStream_t s, int cl) {
    return cl == 1 ? launch_k45_cl<1>(w, L, msg_pairs, s)
         : cl == 2 ? launch_k45_cl<2>(w, L, msg_pairs, s)
         : cl == 8 ? launch_k45_cl<8>(w, L, msg_pairs, s) : launch_k45_cl<4>(w, L, msg_pairs, s);
}

}  // namespace rgc
