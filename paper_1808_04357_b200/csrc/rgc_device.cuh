// rgc_device.cuh -- small device helpers shared by the kernels of librgc.so.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rgc_internal.cuh"

namespace rgc {

#define FULLMASK 0xffffffffu

__device__ __forceinline__ uint32_t fkey(float x) { return __float_as_uint(x) & 0x7FFFFFFFu; }
__device__ __forceinline__ uint32_t ukey(uint32_t b) { return b & 0x7FFFFFFFu; }

// largest l with tb[l] <= t (tb ascending, tb[L] = total)
__device__ __forceinline__ int find_layer(const uint32_t *tb, int L, uint32_t t) {
    int lo = 0, hi = L - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (tb[mid] <= t) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// threshold <- mean + ratio * (max - mean), double, one rounding to f32 (R3)
__device__ __forceinline__ float thresh_at(double mean, double maxd, double ratio) {
    double d = __dsub_rn(maxd, mean);
    double p = __dmul_rn(ratio, d);
    double t = __dadd_rn(mean, p);
    return __double2float_rn(t);
}

__device__ __forceinline__ double pow2d(int e) {  // exact 2^e, -1022 <= e <= 1023
    return __longlong_as_double((long long)(e + 1023) << 52);
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long *p) {
    return *(const volatile unsigned long long *)p;
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long *p, unsigned long long v) {
    *(volatile unsigned long long *)p = v;
}

// inclusive block scan of one u32 per thread (kThreads threads)
__device__ __forceinline__ uint32_t block_incl_scan(uint32_t v, uint32_t *s_w /*[kWarps]*/) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(FULLMASK, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) s_w[warp] = v;
    __syncthreads();
    uint32_t add = 0;
    for (int i = 0; i < warp; i++) add += s_w[i];
    __syncthreads();
    return v + add;
}

constexpr unsigned long long kFlagAgg = 1ull << 62;   // look-back: aggregate published
constexpr unsigned long long kFlagInc = 2ull << 62;   // look-back: inclusive prefix published
constexpr unsigned long long kCntMask = (1ull << 62) - 1;

// s_off[r][l] = first pair of layer l in rank r's block (l = 0..L), from the headers'
// length elements: all p*L words loaded at once, then scanned in smem
__device__ inline void load_offsets(const MsgSrc &src, int L, int p, uint32_t *s_off) {
    for (int i = threadIdx.x; i < p * L; i += kThreads) {
        const int r = i / L, l = i % L;
        s_off[r * (L + 1) + l] = reinterpret_cast<const uint32_t *>(src.of(r))[l];
    }
    __syncthreads();
    for (int r = threadIdx.x; r < p; r += kThreads) {
        uint32_t o = 0;
        for (int l = 0; l < L; l++) { const uint32_t c = s_off[r * (L + 1) + l]; s_off[r * (L + 1) + l] = o; o += c; }
        s_off[r * (L + 1) + L] = o;
    }
    __syncthreads();
}

}  // namespace rgc
