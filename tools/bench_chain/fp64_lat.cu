// Micro-benchmark (dev tool): dependent-chain latency of FP64 and integer ops
// on one warp (cycles per op).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double a, double b, long long* out, double* sink)
{
    double x = a + threadIdx.x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 4096; ++i) { x = __dadd_rn(x, b); x = __dadd_rn(x, -b); }
    long long t1 = clock64();
    double y = a + threadIdx.x;
#pragma unroll 1
    for (int i = 0; i < 4096; ++i) { y = __dmul_rn(y, b); y = __dmul_rn(y, 1.0 / b); }
    long long t2 = clock64();
    double z = a + threadIdx.x;
#pragma unroll 1
    for (int i = 0; i < 4096; ++i) { z = rint(z + 0.25); z = trunc(z * 0.5 + 0.75); }
    long long t3 = clock64();
    long long w = threadIdx.x;
#pragma unroll 1
    for (int i = 0; i < 4096; ++i) { w = w * 3 + 1; w = w ^ (w >> 7); }
    long long t4 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; }
    sink[threadIdx.x] = x + y + z + (double)w;
}

int main()
{
    long long* d; double* s; cudaMalloc(&d, 64); cudaMalloc(&s, 1024);
    long long h[4];
    for (int r = 0; r < 2; ++r) {
        k<<<1, 32>>>(1.5, 1.0000001, d, s);
        cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
        printf("DADD %.1f  DMUL %.1f  (rint+DADD,trunc+DMUL+DADD)/2 %.1f  (IMAD,SHF+LOP)/2 %.1f cycles per op\n",
               h[0] / 8192.0, h[1] / 8192.0, h[2] / 8192.0, h[3] / 8192.0);
    }
}
