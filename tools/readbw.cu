// readbw.cu -- microbenchmark: read-only streaming count (|x| > t) with
// (a) register double-buffered 128-bit loads, (b) per-warp cp.async.bulk (TMA
// bulk copy) pipelines into shared memory completed on mbarriers.
// Development tool for choosing the K2/K3 streaming design (not part of librgc).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t fkey(float x) { return __float_as_uint(x) & 0x7FFFFFFFu; }

template <bool IL>
__global__ void __launch_bounds__(256) count_reg(const float *V, size_t n, uint32_t T, unsigned long long *out) {
    const size_t tiles = n / 4096;
    const size_t tb = tiles * blockIdx.x / gridDim.x, te = tiles * (blockIdx.x + 1) / gridDim.x;
    if (IL) {
        uint32_t c = 0;
        const float4 *v4 = reinterpret_cast<const float4 *>(V);
        for (size_t t = blockIdx.x; t < tiles; t += gridDim.x) {
            float4 X[4];
            for (int j = 0; j < 4; j++) X[j] = v4[t * 1024 + j * 256 + threadIdx.x];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                c += fkey(X[j].x) > T; c += fkey(X[j].y) > T; c += fkey(X[j].z) > T; c += fkey(X[j].w) > T;
            }
        }
        atomicAdd(out, (unsigned long long)c);
        return;
    }
    uint32_t c = 0;
    float4 X[4], Y[4];
    const float4 *v4 = reinterpret_cast<const float4 *>(V);
    if (tb < te) for (int j = 0; j < 4; j++) X[j] = v4[tb * 1024 + j * 256 + threadIdx.x];
    for (size_t t = tb; t < te; t++) {
        if (t + 1 < te) for (int j = 0; j < 4; j++) Y[j] = v4[(t + 1) * 1024 + j * 256 + threadIdx.x];
#pragma unroll
        for (int j = 0; j < 4; j++) {
            c += fkey(X[j].x) > T; c += fkey(X[j].y) > T; c += fkey(X[j].z) > T; c += fkey(X[j].w) > T;
        }
        for (int j = 0; j < 4; j++) X[j] = Y[j];
    }
    atomicAdd(out, (unsigned long long)c);
}

template <int STAGES, int CHUNK, bool IL, int NW = 8>   // CHUNK floats per warp stage
__global__ void __launch_bounds__(NW * 32) count_tma(const float *V, size_t n, uint32_t T, unsigned long long *out) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float *buf = reinterpret_cast<float *>(smem) + (size_t)warp * STAGES * CHUNK;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + sizeof(float) * NW * STAGES * CHUNK) + warp * STAGES;
    const size_t chunks = n / CHUNK;
    const size_t gw = (size_t)gridDim.x * NW, wid = (size_t)blockIdx.x * NW + warp;
    size_t cb = chunks * wid / gw, ce = chunks * (wid + 1) / gw;
    // IL: the CTA owns a blocked range; its warps take consecutive chunks of it
    const size_t c0 = chunks * blockIdx.x / gridDim.x, c1 = chunks * (blockIdx.x + 1) / gridDim.x;
    if (IL) { cb = 0; ce = (c1 - c0 > (size_t)warp) ? (c1 - c0 - warp + NW - 1) / NW : 0; }
    auto cidx = [&](size_t k) -> size_t { return IL ? c0 + warp + k * NW : k; };
    if (lane == 0)
        for (int s = 0; s < STAGES; s++) {
            uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
        }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    auto issue = [&](size_t ch, int s) {
        uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
        uint32_t d = (uint32_t)__cvta_generic_to_shared(buf + s * CHUNK);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(CHUNK * 4) : "memory");
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(d), "l"(V + cidx(ch) * CHUNK), "r"(CHUNK * 4), "r"(a) : "memory");
    };
    if (lane == 0)
        for (int s = 0; s < STAGES && cb + s < ce; s++) issue(cb + s, s);
    uint32_t c = 0;
    for (size_t ch = cb; ch < ce; ch++) {
        const int s = (int)((ch - cb) % STAGES);
        const uint32_t ph = (uint32_t)(((ch - cb) / STAGES) & 1);
        uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
        asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(a), "r"(ph) : "memory");
        const float4 *b4 = reinterpret_cast<const float4 *>(buf + s * CHUNK);
#pragma unroll
        for (int j = 0; j < CHUNK / 128; j++) {
            float4 x = b4[j * 32 + lane];
            c += fkey(x.x) > T; c += fkey(x.y) > T; c += fkey(x.z) > T; c += fkey(x.w) > T;
        }
        __syncwarp();
        if (lane == 0 && ch + STAGES < ce) issue(ch + STAGES, s);
    }
    atomicAdd(out, (unsigned long long)c);
}


// CTA-wide ring: thread 0 issues one 16 KB bulk copy per tile; NW consumer warps
// take a slice each and release the stage on an "empty" barrier
template <int ST, int NW>
__global__ void __launch_bounds__(NW * 32, 1) count_ring(const float *V, size_t n, uint32_t T, unsigned long long *out) {
    extern __shared__ __align__(128) unsigned char smem[];
    float *ring = reinterpret_cast<float *>(smem);
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + ST * 4096), *empty = full + ST;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const size_t tiles = n / 4096;
    const size_t tb = tiles * blockIdx.x / gridDim.x, te = tiles * (blockIdx.x + 1) / gridDim.x;
    auto sa = [](const void *p) { return (uint32_t)__cvta_generic_to_shared(p); };
    if (tid == 0) for (int s = 0; s < ST; s++) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[s])), "r"(NW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    auto wait = [&](uint64_t *b, uint32_t ph) {
        asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(sa(b)), "r"(ph) : "memory");
    };
    size_t issued = 0;
    auto top = [&](size_t limit) {
        if (tid) return;
        while (issued < limit && tb + issued < te) {
            const int s = issued % ST;
            if (issued >= ST) wait(&empty[s], ((issued / ST) - 1) & 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(16384) : "memory");
            asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(sa(ring + s * 4096)), "l"(V + (tb + issued) * 4096), "r"(16384), "r"(sa(&full[s])) : "memory");
            issued++;
        }
    };
    top(ST);
    uint32_t c = 0;
    for (size_t q = 0; tb + q < te; q++) {
        top(q + ST - 1);
        const int s = q % ST;
        wait(&full[s], (q / ST) & 1);
        const float4 *b4 = reinterpret_cast<const float4 *>(ring + s * 4096 + warp * (4096 / NW));
#pragma unroll
        for (int j = 0; j < 4096 / NW / 128; j++) {
            float4 x = b4[j * 32 + lane];
            c += fkey(x.x) > T; c += fkey(x.y) > T; c += fkey(x.z) > T; c += fkey(x.w) > T;
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
    }
    atomicAdd(out, (unsigned long long)c);
}

__global__ void __launch_bounds__(256) copy_il(const float4 *a, float4 *b, size_t n4) {
    for (size_t i = blockIdx.x * 256 + threadIdx.x; i < n4; i += (size_t)gridDim.x * 256) b[i] = a[i];
}
__global__ void fillk(float *V, size_t n) {
    for (size_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256)
        V[i] = (float)((i * 2654435761u) & 0xFFFF) * 1e-5f - 0.3f;
}
int main() {
    const size_t n = (size_t)1 << 27;   // 128M floats = 512 MB
    float *V; unsigned long long *out;
    cudaMalloc(&V, n * 4); cudaMalloc(&out, 8);
    fillk<<<1184, 256>>>(V, n);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto time = [&](const char *name, auto launch) {
        for (int i = 0; i < 3; i++) launch();
        cudaEventRecord(a);
        for (int i = 0; i < 20; i++) launch();
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("%-28s %8.1f us  %7.0f GB/s  (%s)\n", name, ms / 20 * 1e3, n * 4.0 / (ms / 20 * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    };
#define TMAI(S, C, OCC, IL, NW)                                                                              \
    {                                                                                              \
        size_t sm = (size_t)NW * S * C * 4 + NW * S * 8;                                             \
        cudaFuncSetAttribute(count_tma<S, C, IL, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
        char nm[64]; snprintf(nm, 64, "tma%s S=%d C=%d occ=%d nw=%d", IL ? "-cta" : "", S, C, OCC, NW);                         \
        time(nm, [&] { count_tma<S, C, IL, NW><<<sms * OCC, NW * 32, sm>>>(V, n, 1u, out); });               \
    }
#define RING(ST, NW) { size_t sm = (size_t)ST * 16384 + 16 * ST; \
        cudaFuncSetAttribute(count_ring<ST, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
        char nm[64]; snprintf(nm, 64, "ring ST=%d NW=%d", ST, NW); \
        time(nm, [&] { count_ring<ST, NW><<<sms, NW * 32, sm>>>(V, n, 1u, out); }); }
    RING(10, 8) RING(12, 8) RING(10, 16) RING(10, 4) RING(6, 8) RING(4, 8)
    TMAI(6, 2048, 1, true, 4) TMAI(6, 1024, 1, false, 8)
    return 0;
}
