// rgc_asq.cu -- K5: the message of the ASQ layers (Alternating Signs Quantization,
// P:274-294; readings R21, R22 in DESIGN.md).
//
// K3/K45 emit an ASQ layer's selected <index, value> pairs (one sign only, R21) into
// its scratch Ws::Q in ascending index order and zero the residual there, exactly as
// for a plain layer (Alg.1 zeroes the selected entries).  K5 then
//   * appends the layer's indices to the message after the plain layers' pairs
//     ("transmitting only one average element instead of k elements"),
//   * quantizes the values to their mean (R22: exact per-exponent integer sums of the
//     24-bit significands, combined in double in ascending exponent order, / c,
//     rounded once to fp32 -- the same bits for any thread mapping), stored in the
//     header word hdr[L+2+l],
//   * writes the layer's length element hdr[l] and flips its phase for the next call
//     ("if we select the largest k elements ... at current iteration, we will choose
//     smallest k elements ... for the next iteration").
// Work unit: 4096 pairs of one ASQ layer (at least one unit per ASQ layer, so an empty
// message still gets its header and its phase flip); the last unit of a layer to
// finish takes the mean.
#include <cuda_runtime.h>
#include <stdint.h>

#include "rgc_device.cuh"

namespace rgc {

constexpr uint32_t kQUnit = 4096;

__global__ void __launch_bounds__(kThreads)
k5_asq(Ws w, int L, uint32_t *msg_hdr, uint32_t hdr_words) {
    pdl_wait();
    TlMark tlm(w.tl, TL_K5);
    __shared__ uint32_t s_ub[RGC_MAX_LAYERS + 1];   // first work unit of each layer
    __shared__ uint32_t s_e[RGC_MAX_LAYERS];        // entries of each ASQ layer
    __shared__ uint32_t s_ao[RGC_MAX_LAYERS];       // its first index word after the pairs
    __shared__ uint32_t s_w[kWarps];
    __shared__ unsigned long long s_bins[256];
    __shared__ unsigned long long s_wbins[kWarps][256];   // warp-private (no atomics)
    __shared__ uint32_t s_nz[8];                    // nonzero bins (finalize)
    __shared__ int s_last;
    const int tid = threadIdx.x, lane = tid & 31;
    // per-layer entries and units (one thread per layer, L <= 128 < kThreads)
    uint32_t e = 0, units = 0;
    if (tid < L) {
        const LayerDesc &d = w.desc[tid];
        const LayerState &S = w.st[tid];
        if (d.quant) {
            const uint32_t mode = S.mode;
            e = mode == MODE_THRESH ? S.emitted_a
                : (mode == MODE_SURV || mode == MODE_EXACT) ? S.emitted_b : 0u;
            units = e ? (e + kQUnit - 1) / kQUnit : 1u;
        }
    }
    const uint32_t ie = block_incl_scan(e, s_w);
    const uint32_t iu = block_incl_scan(units, s_w);
    if (tid < L) { s_e[tid] = e; s_ao[tid] = ie - e; s_ub[tid] = iu - units; }
    if (tid == L - 1) s_ub[L] = iu;
    __syncthreads();
    const uint32_t total = s_ub[L];
    uint32_t *idx_base = msg_hdr + hdr_words + 2ull * w.ctrl->dense_pairs;
    for (uint32_t unit = blockIdx.x; unit < total; unit += gridDim.x) {
        const int l = find_layer(s_ub, L, unit);
        const LayerDesc &d = w.desc[l];
        LayerState &S = w.st[l];
        const uint32_t c = s_e[l];
        const uint32_t j0 = (unit - s_ub[l]) * kQUnit;
        const uint32_t j1 = min(c, j0 + kQUnit);
        const uint2 *src = w.Q + d.q_off;
        uint32_t *dst = idx_base + s_ao[l];
        unsigned long long *wb = s_wbins[tid >> 5];
        for (int b = lane; b < 256; b += 32) wb[b] = 0ull;
        __syncwarp();
        // all of the thread's pairs are loaded at once (independent loads), then the
        // significands go to the bins in warp-uniform rounds of 32 pairs
        constexpr int R = kQUnit / kThreads;    // 16
        uint32_t ex[R], sg[R];
#pragma unroll
        for (int i = 0; i < R; i++) {
            const uint32_t j = j0 + (uint32_t)(i * kThreads + tid);
            ex[i] = 0xFFFFFFFFu; sg[i] = 0u;
            if (j < j1) {
                const uint2 pr = src[j];
                dst[j] = pr.x;
                const uint32_t m = pr.y & 0x7FFFFFFFu;
                ex[i] = m >> 23;
                sg[i] = (m & 0x7FFFFFu) | (ex[i] ? 0x800000u : 0u);
            }
        }
#pragma unroll
        for (int i = 0; i < R; i++) {
            // one integer sum per distinct exponent of the round (< 2^29: exact in u32)
            bool done = ex[i] == 0xFFFFFFFFu;
            uint32_t todo = __ballot_sync(FULLMASK, !done);
            while (todo) {
                const int lead = __ffs(todo) - 1;
                const uint32_t le = __shfl_sync(FULLMASK, ex[i], lead);
                const bool in = !done && ex[i] == le;
                const uint32_t sum = __reduce_add_sync(FULLMASK, in ? sg[i] : 0u);
                if (lane == lead) wb[le] += sum;          // one writer per warp and round
                done |= in;
                todo = __ballot_sync(FULLMASK, !done);
            }
        }
        __syncthreads();
        for (int b = tid; b < 255; b += kThreads) {
            unsigned long long v = 0;
#pragma unroll
            for (int wq = 0; wq < kWarps; wq++) v += s_wbins[wq][b];
            if (v) atomicAdd(&S.qbins[b], v);
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            const uint32_t nunits = s_ub[l + 1] - s_ub[l];
            s_last = atomicAdd(&S.qdone, 1u) + 1u == nunits;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            if (tid < 8) s_nz[tid] = 0u;
            __syncthreads();
            for (int b = tid; b < 255; b += kThreads) {
                s_bins[b] = atomicExch(&S.qbins[b], 0ull);
                if (s_bins[b]) atomicOr(&s_nz[b >> 5], 1u << (b & 31));
            }
            __syncthreads();
            if (tid == 0) {
                float mean = 0.f;
                if (c) {
                    // ascending exponent order; empty bins add +0.0 (an identity for acc >= 0)
                    double acc = 0.0;
                    for (int wd = 0; wd < 8; wd++) {
                        for (uint32_t m = s_nz[wd]; m; m &= m - 1u) {
                            const int x = wd * 32 + __ffs(m) - 1;
                            acc = __dadd_rn(acc, __dmul_rn(__ull2double_rn(s_bins[x]),
                                                           pow2d((x > 1 ? x : 1) - 150)));
                        }
                    }
                    mean = __double2float_rn(__ddiv_rn(acc, (double)c));
                    if (S.phase & 1u) mean = -mean;     // the negative phase's values
                }
                msg_hdr[l] = c;
                msg_hdr[L + 2 + l] = __float_as_uint(mean);
                S.info.count = c;
                S.count = c;
                S.qdone = 0u;
                S.phase ^= 1u;
                // the next call selects the other sign: restore that sign's predictions
                unsigned int t;
                t = S.jhint; S.jhint = S.alt_jhint; S.alt_jhint = t;
                t = S.margin; S.margin = S.alt_margin; S.alt_margin = t;
                t = S.cand_key; S.cand_key = S.alt_cand_key; S.alt_cand_key = t;
                t = S.stash_shift; S.stash_shift = S.alt_shift; S.alt_shift = t;
                t = S.stash_on; S.stash_on = S.alt_stash_on; S.alt_stash_on = t;
            }
        }
        __syncthreads();
    }
}

cudaError_t launch_k5_asq(const Ws &w, int L, uint32_t *msg_hdr, uint32_t hdr_words, int grid,
                          cudaStream_t s) {
    return launch_pdl(k5_asq, grid, kThreads, 0, s, w, L, msg_hdr, hdr_words);
}

}  // namespace rgc
