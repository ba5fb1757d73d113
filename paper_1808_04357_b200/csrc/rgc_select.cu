// rgc_select.cu -- K45: exact top-k (radixSelect) and the
// ordered emission of the selected <index, value> pairs with the residual /
// momentum masking, fused in ONE CTA per layer, for small
// candidate sets: the Alg.2 survivors ("radixSelect on the remaining
// elements") or a small layer in an exact fallback.  Large sets take the
// multi-CTA K4 passes + K3 pass B instead.
//
// Select: three MSB-first digit passes (11/11/9 bits of the 31-bit magnitude
// key) with shared-memory histograms; the k-th largest key T* and the number q
// of elements equal to T* to take (lower index first, R6).
// Emit: each warp owns a contiguous chunk of the (ascending) candidate list;
// one block-level prefix of the per-warp (gt, eq) counts, then ballot ranks.
#include <cuda_runtime.h>
#include <stdint.h>

#include "rgc_device.cuh"

namespace rgc {

constexpr int kT45 = 1024;          // threads per CTA
constexpr int kW45 = kT45 / 32;

__global__ void __launch_bounds__(kT45)
k45_small(Ws w, int L, uint2 *msg_pairs) {
    extern __shared__ uint32_t s_key[];    // [kSmallSel] candidate keys, staged once
    __shared__ uint32_t s_hist[kRadixBins];
    __shared__ uint32_t s_part[kW45];
    __shared__ uint32_t s_wg[kW45], s_we[kW45];
    __shared__ uint32_t s_digit, s_above;
    const int l = blockIdx.x;
    if (l >= L) return;
    LayerState &S = w.st[l];
    if (!S.small) return;
    const LayerDesc &d = w.desc[l];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool fromS = S.mode == MODE_SURV;
    const uint32_t n = fromS ? S.surv : d.n;
    const uint2 *src = w.S + d.s_off;
    float *V = d.V;
    float *u = d.u;
    // stage the candidates' 31-bit keys in shared memory (8 loads in flight per thread)
    for (uint32_t i0 = 0; i0 < n; i0 += 8 * kT45) {
        uint32_t kv[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint32_t i = i0 + j * kT45 + tid;
            kv[j] = i < n ? (fromS ? ukey(src[i].y) : fkey(V[i])) : 0u;
        }
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint32_t i = i0 + j * kT45 + tid;
            if (i < n) s_key[i] = kv[j];
        }
    }
    __syncthreads();
    auto key_at = [&](uint32_t i) -> uint32_t { return s_key[i]; };

    // ---- radix select of the k-th largest key
    uint32_t prefix = 0, krem = d.k;
#pragma unroll 1
    for (int pass = 0; pass < 3; pass++) {
        const int shift = pass == 0 ? 20 : (pass == 1 ? 9 : 0);
        const uint32_t dmask = pass == 2 ? 511u : 2047u;
        const int hishift = pass == 0 ? 31 : (pass == 1 ? 20 : 9);
        for (int b = tid; b < kRadixBins; b += kT45) s_hist[b] = 0u;
        __syncthreads();
        for (uint32_t i = tid; i < n; i += kT45) {
            const uint32_t kk = key_at(i);
            if (hishift == 31 || (kk >> hishift) == (prefix >> hishift))
                atomicAdd(&s_hist[(kk >> shift) & dmask], 1u);
        }
        __syncthreads();
        // digit whose cumulative count from the top reaches krem (2 bins per thread)
        const uint32_t h0 = s_hist[2 * tid], h1 = s_hist[2 * tid + 1];
        uint32_t v = h0 + h1;
        // inclusive scan from the top: reverse thread order
        const int rt = kT45 - 1 - tid;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_down_sync(FULLMASK, x, o);
            if (lane + o < 32) x += y;
        }
        // x = sum over lanes >= lane within the warp (bins above, warp-local)
        if (lane == 0) s_part[warp] = x;
        __syncthreads();
        uint32_t addw = 0;
        for (int i = warp + 1; i < kW45; i++) addw += s_part[i];
        const uint32_t incl = x + addw;                 // bins >= 2*tid
        const uint32_t above1 = incl - h0 - h1;         // bins > 2*tid+1
        (void)rt;
        if (h1 && above1 < krem && krem <= above1 + h1) { s_digit = 2 * tid + 1; s_above = above1; }
        const uint32_t above0 = above1 + h1;
        if (h0 && above0 < krem && krem <= above0 + h0) { s_digit = 2 * tid; s_above = above0; }
        __syncthreads();
        prefix |= s_digit << shift;
        krem -= s_above;
        __syncthreads();
    }
    const uint32_t T = prefix, q = krem;

    // ---- ordered emission: chunk per warp, counts, block prefix, ballot ranks
    const uint32_t per = (n + kW45 - 1) / kW45;
    const uint32_t c0 = min(n, warp * per), c1 = min(n, c0 + per);
    uint32_t wg = 0, we = 0;
    for (uint32_t b = c0; b < c1; b += 32) {
        const uint32_t i = b + lane;
        const uint32_t kk = i < c1 ? key_at(i) : 0u;
        wg += __popc(__ballot_sync(FULLMASK, i < c1 && kk > T));
        we += __popc(__ballot_sync(FULLMASK, i < c1 && kk == T));
    }
    if (lane == 0) { s_wg[warp] = wg; s_we[warp] = we; }
    __syncthreads();
    uint32_t gb = 0, eb = 0;
    for (int i = 0; i < warp; i++) { gb += s_wg[i]; eb += s_we[i]; }
    uint2 *dst = msg_pairs + S.msg_off;
    const uint32_t lt = (1u << lane) - 1u;
    for (uint32_t b = c0; b < c1; b += 32) {
        const uint32_t i = b + lane;
        const uint32_t kk = i < c1 ? s_key[i] : 0u;
        const bool isg = i < c1 && kk > T, ise = i < c1 && kk == T;
        const uint32_t G = __ballot_sync(FULLMASK, isg), E = __ballot_sync(FULLMASK, ise);
        const uint32_t g = gb + __popc(G & lt), eq = eb + __popc(E & lt);
        if (isg || (ise && eq < q)) {
            const uint32_t outpos = isg ? g + min(eq, q) : g + eq;
            const uint2 e = fromS ? src[i] : make_uint2(i, __float_as_uint(V[i]));
            dst[outpos] = e;                      // <index, value>
            V[e.x] = 0.0f;                        // V <- V (.) (1 - Masks)
            if (u) u[e.x] = 0.0f;                 // momentum masking
        }
        gb += __popc(G); eb += __popc(E);
    }
    if (tid == 0) {
        S.rs_prefix = T;
        S.rs_krem = q;
        S.info.kth_key = T;
        S.info.tie_quota = q;
        S.emitted_b = d.k;
    }
}

cudaError_t launch_k45(const Ws &w, int L, uint2 *msg_pairs, cudaStream_t s) {
    static bool attr = false;
    const size_t smem = sizeof(uint32_t) * kSmallSel;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k45_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    k45_small<<<L, kT45, smem, s>>>(w, L, msg_pairs);
    return cudaGetLastError();
}

}  // namespace rgc
