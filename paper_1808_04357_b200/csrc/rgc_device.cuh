// rgc_device.cuh -- small device helpers shared by the kernels of librgc.so.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <utility>

#include "rgc_internal.cuh"

namespace rgc {

#define FULLMASK 0xffffffffu

// RGC_CHECK builds (the "checked" library variant: tools/mkvar.sh checked -DRGC_CHECK): every
// store of a message entry, a residual / momentum / output index and a table slot is checked
// against its bound first; the first violation is printed and the kernel traps.  A device-
// side stand-in for a memory checker (compute-sanitizer is not used on this pool).
#ifdef RGC_CHECK
#define RGC_DCHECK(cond, ...)                                                                 \
    do { if (!(cond)) { printf("RGC_CHECK failed %s:%d: " #cond "\n", __FILE__, __LINE__);    \
                        asm volatile("trap;"); } } while (0)
#else
#define RGC_DCHECK(cond, ...) do { } while (0)
#endif

// Programmatic dependent launch: a kernel launched with launch_pdl() may start while its
// predecessor in the stream drains; it must call pdl_wait() before touching anything the
// predecessor writes (griddepcontrol.wait returns once the predecessor grid completed and
// its memory is visible; a no-op for a normal launch).
__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef RGC_PDL_EARLY
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

bool pdl_enabled();   // rgc_api.cu (RGC_NO_PDL=1 disables it)

__device__ __forceinline__ unsigned long long tl_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Timeline marks (Ws::tl): constructed right after pdl_wait(), destroyed when thread 0 leaves
struct TlMark {
    unsigned long long *tl;
    int k;
    __device__ __forceinline__ TlMark(unsigned long long *tl_, int k_) : tl(tl_), k(k_) {
        if (tl && threadIdx.x == 0) atomicMin(&tl[k], tl_now());
    }
    __device__ __forceinline__ ~TlMark() {
        if (tl && threadIdx.x == 0) atomicMax(&tl[kTlKernels + k], tl_now());
    }
};

// a point in time (start = end = now; min / max over the CTAs that pass it)
__device__ __forceinline__ void tl_probe(unsigned long long *tl, int k) {
    if (tl && threadIdx.x == 0) {
        const unsigned long long now = tl_now();
#ifdef RGC_CYCLES   // development: SM cycles instead of time (one CTA's probes compare)
        const unsigned long long cyc = (unsigned long long)clock64();
        tl[k] = cyc;
        tl[kTlKernels + k] = cyc;
        return;
#endif
        atomicMin(&tl[k], now);
        atomicMax(&tl[kTlKernels + k], now);
    }
}
__device__ __forceinline__ void tl_end(unsigned long long *tl, int k) {
    if (tl && threadIdx.x == 0) atomicMax(&tl[kTlKernels + k], tl_now());
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---- cross-GPU epoch flags (RGC_SYNC_P2P / RGC_SYNC_PULL; P2PFlags in rgc_internal.cuh)
constexpr unsigned long long kP2PTimeoutNs = 120ull * 1000 * 1000 * 1000;   // default 120 s

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// spin until *flag >= epoch (one thread); false on timeout (recorded in mine->err and
// reported as an error by the next decompression's k_finish -> rgc_status)
__device__ inline bool wait_flag(P2PFlags *mine, const unsigned long long *flag, int q,
                                 unsigned long long epoch) {
    const unsigned long long t0 = globaltimer_ns();
    const unsigned long long lim = mine->timeout_ns ? mine->timeout_ns : kP2PTimeoutNs;
    while (ld_acquire_sys(flag) < epoch) {
        if (globaltimer_ns() - t0 > lim) {
            atomicOr(&mine->err, 1ull << (q & 63));
            return false;
        }
        __nanosleep(64);
    }
    return true;
}

// ---- L2 eviction priorities.  K1 streams 20 B/element through L2 while it writes the
// candidate stash (~1-2 % of the elements) that K2/K3 read right after it, under the
// decompression's zero fill: the streams are marked evict-first and the stash evict-last,
// so the stash is still in L2 when the latency-bound selection kernels read it.
// RGC_NO_L2HINT turns the hints off (A/B experiments).
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_u2_hint(uint2 *p, uint2 v, uint64_t pol) {
#ifdef RGC_NO_L2HINT
    *p = v;
#else
    asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;"
                 ::"l"(p), "r"(v.x), "r"(v.y), "l"(pol) : "memory");
#endif
}
// K1's residual / momentum loads and stores: plain (default L2 policy).  Marking them
// evict-first (ld/st .cs) was measured 7 us slower on VGG16's K1 (tools/gpu_ab.sh,
// variant RGC_STREAM_HINT); only the stash (evict-last) and the zero fill (evict-first)
// carry hints.
__device__ __forceinline__ float4 ld_stream(const float *p) {
#ifdef RGC_STREAM_HINT
    return __ldcs(reinterpret_cast<const float4 *>(p));
#else
    return *reinterpret_cast<const float4 *>(p);
#endif
}
__device__ __forceinline__ void st_stream(float *p, float4 v) {
#ifdef RGC_STREAM_HINT
    __stcs(reinterpret_cast<float4 *>(p), v);
#else
    *reinterpret_cast<float4 *>(p) = v;
#endif
}

__device__ __forceinline__ uint32_t fkey(float x) { return __float_as_uint(x) & 0x7FFFFFFFu; }
__device__ __forceinline__ uint32_t ukey(uint32_t b) { return b & 0x7FFFFFFFu; }
// selection key of a layer: |x| on 31 bits, or for an ASQ layer (R21) the magnitude of the
// phase's sign only (ska = 0x80000000; skx = 0 positive phase, 0x80000000 negative phase)
__device__ __forceinline__ uint32_t skey(uint32_t b, uint32_t skx, uint32_t ska) {
    return ((b ^ skx) & ska) ? 0u : (b & 0x7FFFFFFFu);
}

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

// Message layout per rank (include/rgc.h): s_off[r][l] = first entry of layer l in
// rank r's entry sequence (l = 0..L, from the length elements) and
// s_ao[r][l] = ASQ entries before layer l (a layer is ASQ iff its header value word
// hdr[L+2+l] is not RGC_MSG_DENSE).  Plain layers' pairs come first, the ASQ layers'
// indices after them.  All p*L words are loaded at once, then scanned in smem.
__device__ inline void load_layout(const MsgSrc &src, int L, int p, uint32_t *s_off,
                                   uint32_t *s_ao) {
    for (int i = threadIdx.x; i < p * L; i += blockDim.x) {
        const int r = i / L, l = i % L;
        const uint32_t *h = reinterpret_cast<const uint32_t *>(src.of(r));
        s_off[r * (L + 1) + l] = h[l];
        s_ao[r * (L + 1) + l] = h[L + 2 + l] != RGC_MSG_DENSE ? 1u : 0u;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < p; r += blockDim.x) {
        uint32_t o = 0, a = 0;
        for (int l = 0; l < L; l++) {
            const uint32_t c = s_off[r * (L + 1) + l], q = s_ao[r * (L + 1) + l];
            s_off[r * (L + 1) + l] = o;
            s_ao[r * (L + 1) + l] = a;
            o += c;
            a += q ? c : 0u;
        }
        s_off[r * (L + 1) + L] = o;
        s_ao[r * (L + 1) + L] = a;
    }
    __syncthreads();
}

// Where layer l's entries sit in a rank's block: {x: word offset of its first entry
// from the pairs base (4*H bytes into the block), y: words per entry (2 pair / 1 ASQ
// index), z: the ASQ value bits (or RGC_MSG_DENSE), w: global entry index of its first
// entry}.  o, ao: that rank's s_off / s_ao rows.
__device__ __forceinline__ uint4 layer_view(const uint32_t *hdr, const uint32_t *o,
                                            const uint32_t *ao, int L, int l) {
    const uint32_t vb = hdr[L + 2 + l];
    if (vb == RGC_MSG_DENSE) return make_uint4(2u * (o[l] - ao[l]), 2u, vb, o[l]);
    const uint32_t plain = o[L] - ao[L];
    return make_uint4(2u * plain + ao[l], 1u, vb, o[l]);
}

// entry g (global entry index, inside the layer of view v) -> {index, value bits}
__device__ __forceinline__ uint2 view_entry(const uint32_t *pw, const uint4 &v, uint32_t g) {
    const uint32_t at = v.x + v.y * (g - v.w);
    return v.y == 2u ? make_uint2(pw[at], pw[at + 1]) : make_uint2(pw[at], v.z);
}

}  // namespace rgc
