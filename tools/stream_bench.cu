// stream_bench.cu -- ceiling of K1's traffic pattern on this B200 (development tool, not
// part of librgc).  K1 reads g, u, V and writes u, V (3 reads + 2 writes of 4 B per
// element, 20 B/element; u = fma(m,u,g), V = V + u).  This measures the same pattern with
// the K1 arithmetic but no statistics, in several implementations, next to a 1R:1W copy
// (the pattern MEASURED_PEAKS.json's hbm_gbs is taken with), so K1's fraction of the
// measured copy peak can be read against the best a plain 3R:2W stream reaches.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_bench tools/stream_bench.cu
//   tools/stream_bench [n_elements]      (default 138,342,400 = VGG16's compressed elements)
//
// Variants (GB/s = algorithmic bytes / best-of-10 CUDA-event time):
//   copy      : 1R:1W float4 grid-stride copy (calibration against hbm_gbs)
//   gs<U>     : 3R:2W grid-stride, U float4 per array per thread in flight
//   blk<W>    : 3R:2W, each CTA a contiguous blocked range of 4096-element tiles (K1's
//               layout), 256 threads, W CTAs per SM
//   tma<S>    : 3R:2W through shared memory: one thread per CTA issues cp.async.bulk loads
//               of g, u, V tiles (S-stage mbarrier ring), the CTA computes in shared memory,
//               one thread issues cp.async.bulk stores of u, V (bulk groups)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <functional>
#include <string>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void k_copy(const float4 *a, float4 *b, size_t n4) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

template <int U>
__global__ void __launch_bounds__(256) k_gs(const float4 *g, float4 *u, float4 *V, float m, size_t n4) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n4; i += U * stride) {
        float4 G[U], X[U], Y[U];
#pragma unroll
        for (int k = 0; k < U; k++) { G[k] = g[i + k * stride]; X[k] = u[i + k * stride]; Y[k] = V[i + k * stride]; }
#pragma unroll
        for (int k = 0; k < U; k++) {
            X[k].x = fmaf(m, X[k].x, G[k].x); X[k].y = fmaf(m, X[k].y, G[k].y);
            X[k].z = fmaf(m, X[k].z, G[k].z); X[k].w = fmaf(m, X[k].w, G[k].w);
            Y[k].x += X[k].x; Y[k].y += X[k].y; Y[k].z += X[k].z; Y[k].w += X[k].w;
            u[i + k * stride] = X[k]; V[i + k * stride] = Y[k];
        }
    }
    for (; i < n4; i += stride) {
        float4 G = g[i], X = u[i], Y = V[i];
        X.x = fmaf(m, X.x, G.x); X.y = fmaf(m, X.y, G.y); X.z = fmaf(m, X.z, G.z); X.w = fmaf(m, X.w, G.w);
        Y.x += X.x; Y.y += X.y; Y.z += X.z; Y.w += X.w;
        u[i] = X; V[i] = Y;
    }
}

// K1's layout: blocked tile ranges, each warp a 512-element slice per step (4 float4 per lane)
__global__ void __launch_bounds__(256) k_blk(const float4 *g, float4 *u, float4 *V, float m, size_t tiles) {
    const size_t t0 = tiles * blockIdx.x / gridDim.x, t1 = tiles * (blockIdx.x + 1) / gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (size_t t = t0; t < t1; t++) {
        const size_t base = t * 1024 + warp * 128 + lane;   // float4 index: 4096 floats / tile
        float4 G[4], X[4], Y[4];
#pragma unroll
        for (int k = 0; k < 4; k++) { G[k] = g[base + k * 32]; X[k] = u[base + k * 32]; Y[k] = V[base + k * 32]; }
#pragma unroll
        for (int k = 0; k < 4; k++) {
            X[k].x = fmaf(m, X[k].x, G[k].x); X[k].y = fmaf(m, X[k].y, G[k].y);
            X[k].z = fmaf(m, X[k].z, G[k].z); X[k].w = fmaf(m, X[k].w, G[k].w);
            Y[k].x += X[k].x; Y[k].y += X[k].y; Y[k].z += X[k].z; Y[k].w += X[k].w;
            u[base + k * 32] = X[k]; V[base + k * 32] = Y[k];
        }
    }
}

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// TMA bulk ring: tiles of TE elements; stage s holds g, u, V (3 * TE * 4 bytes)
template <int S, int TE>
__global__ void __launch_bounds__(256, 1) k_tma(const float *g, float *u, float *V, float m, size_t tiles) {
    extern __shared__ __align__(128) unsigned char smem[];
    float *buf = reinterpret_cast<float *>(smem);                       // [S][3][TE]
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + sizeof(float) * S * 3 * TE);
    const size_t t0 = tiles * blockIdx.x / gridDim.x, t1 = tiles * (blockIdx.x + 1) / gridDim.x;
    const size_t nt = t1 - t0;
    constexpr uint32_t TB = TE * 4;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](size_t k) {   // tile t0 + k into stage k % S
        const int s = (int)(k % S);
        const size_t e0 = (t0 + k) * TE;
        float *b = buf + (size_t)s * 3 * TE;
        const uint32_t bar = sa(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(3 * TB) : "memory");
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(b)), "l"(g + e0), "r"(TB), "r"(bar) : "memory");
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(b + TE)), "l"(u + e0), "r"(TB), "r"(bar) : "memory");
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(b + 2 * TE)), "l"(V + e0), "r"(TB), "r"(bar) : "memory");
    };
    if (threadIdx.x == 0)
        for (int k = 0; k < S - 1 && k < (int)nt; k++) issue(k);
    for (size_t k = 0; k < nt; k++) {
        const int s = (int)(k % S);
        if (threadIdx.x == 0 && k + S - 1 < nt) {
            // stage (k+S-1) % S was stored from at iteration k-1: its bulk store must have
            // finished reading shared memory before the refill (at most 1 group pending)
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            issue(k + S - 1);
        }
        const uint32_t ph = (uint32_t)((k / S) & 1);
        asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n"
                     ::"r"(sa(&full[s])), "r"(ph) : "memory");
        float4 *b = reinterpret_cast<float4 *>(buf + (size_t)s * 3 * TE);
        for (int i = threadIdx.x; i < TE / 4; i += 256) {
            const float4 G = b[i];
            float4 X = b[TE / 4 + i], Y = b[2 * (TE / 4) + i];
            X.x = fmaf(m, X.x, G.x); X.y = fmaf(m, X.y, G.y); X.z = fmaf(m, X.z, G.z); X.w = fmaf(m, X.w, G.w);
            Y.x += X.x; Y.y += X.y; Y.z += X.z; Y.w += X.w;
            b[TE / 4 + i] = X; b[2 * (TE / 4) + i] = Y;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            const size_t e0 = (t0 + k) * TE;
            float *bb = buf + (size_t)s * 3 * TE;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         ::"l"(u + e0), "r"(sa(bb + TE)), "r"(TB) : "memory");
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         ::"l"(V + e0), "r"(sa(bb + 2 * TE)), "r"(TB) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// blk + one block barrier per tile with a CTA-wide max (K1's tile max of |V|)
__global__ void __launch_bounds__(256) k_blkbar(const float4 *g, float4 *u, float4 *V, float m, size_t tiles,
                                                unsigned *sink) {
    __shared__ unsigned s_w[8];
    const size_t t0 = tiles * blockIdx.x / gridDim.x, t1 = tiles * (blockIdx.x + 1) / gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned acc = 0;
    for (size_t t = t0; t < t1; t++) {
        const size_t base = t * 1024 + warp * 128 + lane;
        float4 G[4], X[4], Y[4];
#pragma unroll
        for (int k = 0; k < 4; k++) { G[k] = g[base + k * 32]; X[k] = u[base + k * 32]; Y[k] = V[base + k * 32]; }
        unsigned km = 0;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            X[k].x = fmaf(m, X[k].x, G[k].x); X[k].y = fmaf(m, X[k].y, G[k].y);
            X[k].z = fmaf(m, X[k].z, G[k].z); X[k].w = fmaf(m, X[k].w, G[k].w);
            Y[k].x += X[k].x; Y[k].y += X[k].y; Y[k].z += X[k].z; Y[k].w += X[k].w;
            u[base + k * 32] = X[k]; V[base + k * 32] = Y[k];
            km = max(km, max(max(__float_as_uint(Y[k].x) & 0x7fffffffu, __float_as_uint(Y[k].y) & 0x7fffffffu),
                             max(__float_as_uint(Y[k].z) & 0x7fffffffu, __float_as_uint(Y[k].w) & 0x7fffffffu)));
        }
        km = __reduce_max_sync(0xffffffffu, km);
        if (lane == 0) s_w[warp] = km;
        __syncthreads();
        unsigned tm = s_w[0];
        for (int i = 1; i < 8; i++) tm = max(tm, s_w[i]);
        acc += tm;
        __syncthreads();
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

// TMA bulk loads (S-stage ring), compute from shared memory, plain 128-bit stores from
// registers (no bulk stores: a stage is free once the CTA passed its barrier)
template <int S, int TE>
__global__ void __launch_bounds__(256) k_tmald(const float *g, float *u, float *V, float m, size_t tiles) {
    extern __shared__ __align__(128) unsigned char smem[];
    float *buf = reinterpret_cast<float *>(smem);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + sizeof(float) * S * 3 * TE);
    const size_t t0 = tiles * blockIdx.x / gridDim.x, t1 = tiles * (blockIdx.x + 1) / gridDim.x;
    const size_t nt = t1 - t0;
    constexpr uint32_t TB = TE * 4;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](size_t k) {
        const int s = (int)(k % S);
        const size_t e0 = (t0 + k) * TE;
        float *b = buf + (size_t)s * 3 * TE;
        const uint32_t bar = sa(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(3 * TB) : "memory");
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(b)), "l"(g + e0), "r"(TB), "r"(bar) : "memory");
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(b + TE)), "l"(u + e0), "r"(TB), "r"(bar) : "memory");
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(b + 2 * TE)), "l"(V + e0), "r"(TB), "r"(bar) : "memory");
    };
    if (threadIdx.x == 0)
        for (int k = 0; k < S && k < (int)nt; k++) issue(k);
    for (size_t k = 0; k < nt; k++) {
        const int s = (int)(k % S);
        const uint32_t ph = (uint32_t)((k / S) & 1);
        asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n"
                     ::"r"(sa(&full[s])), "r"(ph) : "memory");
        const float4 *b = reinterpret_cast<const float4 *>(buf + (size_t)s * 3 * TE);
        const size_t e4 = (t0 + k) * (TE / 4);
        for (int i = threadIdx.x; i < TE / 4; i += 256) {
            const float4 G = b[i];
            float4 X = b[TE / 4 + i], Y = b[2 * (TE / 4) + i];
            X.x = fmaf(m, X.x, G.x); X.y = fmaf(m, X.y, G.y); X.z = fmaf(m, X.z, G.z); X.w = fmaf(m, X.w, G.w);
            Y.x += X.x; Y.y += X.y; Y.z += X.z; Y.w += X.w;
            reinterpret_cast<float4 *>(u)[e4 + i] = X;
            reinterpret_cast<float4 *>(V)[e4 + i] = Y;
        }
        __syncthreads();   // stage s fully consumed -> refill it with tile k + S
        if (threadIdx.x == 0 && k + S < nt) issue(k + S);
    }
}

// K1's layout with tiles dealt round-robin in chunks of C tiles: CTA b takes chunks b, b+G, ...
// (C = 1: the whole grid sweeps one contiguous window, like the grid-stride variant)
template <int C>
__global__ void __launch_bounds__(256) k_rr(const float4 *g, float4 *u, float4 *V, float m, size_t tiles) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t chunks = (tiles + C - 1) / C;
    for (size_t c = blockIdx.x; c < chunks; c += gridDim.x)
        for (size_t t = c * C; t < (c + 1) * C && t < tiles; t++) {
            const size_t base = t * 1024 + warp * 128 + lane;
            float4 G[4], X[4], Y[4];
#pragma unroll
            for (int k = 0; k < 4; k++) { G[k] = g[base + k * 32]; X[k] = u[base + k * 32]; Y[k] = V[base + k * 32]; }
#pragma unroll
            for (int k = 0; k < 4; k++) {
                X[k].x = fmaf(m, X[k].x, G[k].x); X[k].y = fmaf(m, X[k].y, G[k].y);
                X[k].z = fmaf(m, X[k].z, G[k].z); X[k].w = fmaf(m, X[k].w, G[k].w);
                Y[k].x += X[k].x; Y[k].y += X[k].y; Y[k].z += X[k].z; Y[k].w += X[k].w;
                u[base + k * 32] = X[k]; V[base + k * 32] = Y[k];
            }
        }
}

// like k_blk / k_rr<1>, but each step of a warp moves ONE float4 per array per lane (the
// tile's 4 steps issue their loads one step at a time, like the grid-stride gs1 variant)
template <bool RR>
__global__ void __launch_bounds__(256) k_u1(const float4 *__restrict__ g, float4 *__restrict__ u,
                                            float4 *__restrict__ V, float m, size_t tiles) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t t0 = RR ? blockIdx.x : tiles * blockIdx.x / gridDim.x;
    const size_t t1 = RR ? tiles : tiles * (blockIdx.x + 1) / gridDim.x;
    const size_t ts = RR ? gridDim.x : 1;
    for (size_t t = t0; t < t1; t += ts) {
#pragma unroll 1
        for (int k = 0; k < 4; k++) {
            const size_t i = t * 1024 + k * 256 + threadIdx.x;   // 1024 contiguous floats per step
            float4 G = g[i], X = u[i], Y = V[i];
            X.x = fmaf(m, X.x, G.x); X.y = fmaf(m, X.y, G.y); X.z = fmaf(m, X.z, G.z); X.w = fmaf(m, X.w, G.w);
            Y.x += X.x; Y.y += X.y; Y.z += X.z; Y.w += X.w;
            u[i] = X; V[i] = Y;
        }
    }
    (void)warp; (void)lane;
}

struct Timer {
    cudaEvent_t a, b;
    Timer() { cudaEventCreate(&a); cudaEventCreate(&b); }
    template <class F> float best(F f, int reps = 10) {
        f(); CK(cudaDeviceSynchronize());
        float bt = 1e30f;
        for (int r = 0; r < reps; r++) {
            cudaEventRecord(a); f(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b); if (ms < bt) bt = ms;
        }
        CK(cudaGetLastError());
        return bt;
    }
};

int main(int argc, char **argv) {
    size_t n = argc > 1 ? strtoull(argv[1], nullptr, 10) : 138342400ull;
    const int rounds = argc > 2 ? atoi(argv[2]) : 3;
    n = n / 16384 * 16384;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    float *g, *u, *V, *a, *b;
    unsigned *sink;
    CK(cudaMalloc(&g, n * 4)); CK(cudaMalloc(&u, n * 4)); CK(cudaMalloc(&V, n * 4));
    CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&b, n * 8)); CK(cudaMalloc(&sink, 64));
    CK(cudaMemset(g, 0, n * 4)); CK(cudaMemset(u, 0, n * 4)); CK(cudaMemset(V, 0, n * 4));
    CK(cudaMemset(a, 0, n * 8));
    Timer T;
    const double alg = 20.0 * n;
    const size_t n4 = n / 4, tiles = n / 4096;
    struct Var { std::string name; double bytes; std::function<void()> run; };
    std::vector<Var> vars;
    for (int occ : {4, 8})
        vars.push_back({"copy_occ" + std::to_string(occ), 16.0 * n,
                        [=] { k_copy<<<sms * occ, 256>>>((const float4 *)a, (float4 *)b, 2 * n / 4); }});
    for (int occ : {3, 8}) {
        vars.push_back({"gs1_occ" + std::to_string(occ), alg,
                        [=] { k_gs<1><<<sms * occ, 256>>>((const float4 *)g, (float4 *)u, (float4 *)V, 0.9f, n4); }});
        vars.push_back({"gs4_occ" + std::to_string(occ), alg,
                        [=] { k_gs<4><<<sms * occ, 256>>>((const float4 *)g, (float4 *)u, (float4 *)V, 0.9f, n4); }});
    }
    for (int occ : {2, 3, 4, 8})
        vars.push_back({"blk_occ" + std::to_string(occ), alg,
                        [=] { k_blk<<<sms * occ, 256>>>((const float4 *)g, (float4 *)u, (float4 *)V, 0.9f, tiles); }});
    for (int occ : {3, 4}) {
        vars.push_back({"rr1_occ" + std::to_string(occ), alg,
                        [=] { k_rr<1><<<sms * occ, 256>>>((const float4 *)g, (float4 *)u, (float4 *)V, 0.9f, tiles); }});
        vars.push_back({"rr2_occ" + std::to_string(occ), alg,
                        [=] { k_rr<2><<<sms * occ, 256>>>((const float4 *)g, (float4 *)u, (float4 *)V, 0.9f, tiles); }});
        vars.push_back({"rr8_occ" + std::to_string(occ), alg,
                        [=] { k_rr<8><<<sms * occ, 256>>>((const float4 *)g, (float4 *)u, (float4 *)V, 0.9f, tiles); }});
        vars.push_back({"rr64_occ" + std::to_string(occ), alg,
                        [=] { k_rr<64><<<sms * occ, 256>>>((const float4 *)g, (float4 *)u, (float4 *)V, 0.9f, tiles); }});
    }
    for (int occ : {3, 4, 8}) {
        vars.push_back({"blku1_occ" + std::to_string(occ), alg,
                        [=] { k_u1<false><<<sms * occ, 256>>>((const float4 *)g, (float4 *)u, (float4 *)V, 0.9f, tiles); }});
        vars.push_back({"rru1_occ" + std::to_string(occ), alg,
                        [=] { k_u1<true><<<sms * occ, 256>>>((const float4 *)g, (float4 *)u, (float4 *)V, 0.9f, tiles); }});
    }
    for (int occ : {3, 8})
        vars.push_back({"blkbar_occ" + std::to_string(occ), alg,
                        [=] { k_blkbar<<<sms * occ, 256>>>((const float4 *)g, (float4 *)u, (float4 *)V, 0.9f, tiles, sink); }});
    auto add_tma = [&](auto kern, int S, int TE, const char *name) {
        const size_t smem = sizeof(float) * S * 3 * TE + 8 * S;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem));
        const size_t t = n / TE;
        vars.push_back({std::string(name) + "_occ" + std::to_string(occ), alg,
                        [=] { kern<<<sms * occ, 256, smem>>>(g, u, V, 0.9f, t); }});
    };
    add_tma(k_tma<4, 2048>, 4, 2048, "tma_s4_t2048");
    add_tma(k_tma<6, 1024>, 6, 1024, "tma_s6_t1024");
    add_tma(k_tmald<3, 4096>, 3, 4096, "tmald_s3_t4096");
    add_tma(k_tmald<4, 2048>, 4, 2048, "tmald_s4_t2048");
    add_tma(k_tmald<6, 1024>, 6, 1024, "tmald_s6_t1024");
    add_tma(k_tmald<8, 1024>, 8, 1024, "tmald_s8_t1024");
    add_tma(k_tmald<3, 2048>, 3, 2048, "tmald_s3_t2048");
    std::vector<std::vector<float>> ms(vars.size());
    for (int r = 0; r < rounds; r++)
        for (size_t i = 0; i < vars.size(); i++) ms[i].push_back(T.best(vars[i].run, 5));
    printf("{\"n\": %zu, \"sms\": %d, \"rounds\": %d, \"results\": [\n", n, sms, rounds);
    for (size_t i = 0; i < vars.size(); i++) {
        std::vector<float> v = ms[i];
        std::sort(v.begin(), v.end());
        const float med = v[v.size() / 2], best = v[0];
        printf("  {\"variant\": \"%s\", \"ms_median\": %.4f, \"GBps_median\": %.1f, \"GBps_best\": %.1f}%s\n",
               vars[i].name.c_str(), med, vars[i].bytes / med / 1e6, vars[i].bytes / best / 1e6,
               i + 1 < vars.size() ? "," : "");
    }
    printf("]}\n");
    return 0;
}
