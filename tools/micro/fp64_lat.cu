// FP64 dependent-chain latency on this GPU (development microbenchmark): cycles per op
#include <cstdio>
__global__ void k(double *out, long long *cyc, double a, double b, unsigned long long u) {
    double x = a;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; i++) x = __dadd_rn(x, b);
    long long t1 = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; i++) x = __dmul_rn(x, b);
    long long t2 = clock64();
#pragma unroll 1
    for (int i = 0; i < 64; i++) x = __ddiv_rn(x, b);
    long long t3 = clock64();
#pragma unroll 1
    for (int i = 0; i < 64; i++) { u = u * 3 + 1; x = __dadd_rn(x, __ull2double_rn(u)); }
    long long t4 = clock64();
    float f = (float)x;
#pragma unroll 1
    for (int i = 0; i < 256; i++) f = __fadd_rn(f, (float)b);
    long long t5 = clock64();
    out[0] = x + f;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
}
int main() {
    double *o; long long *c; cudaMalloc(&o, 8); cudaMalloc(&c, 64);
    for (int r = 0; r < 3; r++) k<<<1, 1>>>(o, c, 1.0, 1.0000001, 12345);
    long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
    printf("{\"dadd_cyc\": %.1f, \"dmul_cyc\": %.1f, \"ddiv_cyc\": %.1f, \"u2d_dadd_cyc\": %.1f, \"fadd_cyc\": %.1f}\n",
           h[0] / 256.0, h[1] / 256.0, h[2] / 64.0, h[3] / 64.0, h[4] / 256.0);
    return 0;
}
