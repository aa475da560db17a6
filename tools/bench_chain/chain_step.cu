// Micro-benchmark (dev tool): cycles per step of the serial reference chain
// (codec.cpp:224-247) in three formulations, one chain per thread.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

__device__ __noinline__ double slow_div(double a, double b) { return __ddiv_rn(a, b); }

template <int V>
__global__ void k(const double* x, int n, double delta, double td, double inv, double lim, long long* cyc, double* out)
{
    const double* xr = x + (size_t)threadIdx.x * n;
    double P = 0.0;
    long long t0 = clock64();
    uint32_t acc = 0;
    for (int i = 0; i < n; ++i) {
        const double xx = xr[i];
        const double diff = __dsub_rn(xx, P);
        double Pn = xx;
        if (fabs(diff) < lim) {
            double qd;
            if (V == 0) qd = __ddiv_rn(diff, td);
            else {
                qd = __dmul_rn(diff, inv);
                const double fr = fabs(__dsub_rn(qd, trunc(qd)));
                if (fabs(__dsub_rn(fr, 0.5)) <= fabs(qd) * 9.094947017729282e-13) qd = slow_div(diff, td);
            }
            double t;
            if (V == 2) t = round(qd);  // half away from zero == llround
            else {
                t = trunc(qd);
                if (fabs(__dsub_rn(qd, t)) >= 0.5) t = __dadd_rn(t, copysign(1.0, qd));
            }
            if (t > -32768.0 && t < 32768.0) {
                const double recon = __dadd_rn(P, __dmul_rn(td, t));
                if (fabs(__dsub_rn(xx, recon)) <= delta) { Pn = recon; acc += (uint32_t)(int)t; }
            }
        }
        P = Pn;
    }
    long long t1 = clock64();
    cyc[threadIdx.x] = t1 - t0;
    out[threadIdx.x] = P + acc;
}

int main()
{
    const int n = 16384, T = 32;
    double* hx = new double[(size_t)n * T];
    for (int t = 0; t < T; ++t)
        for (int i = 0; i < n; ++i) hx[(size_t)t * n + i] = cos(6.283185307179586 * 0.00731 * i * (t + 1)) / 1024.0;
    double *dx, *dout; long long* dc;
    cudaMalloc(&dx, sizeof(double) * n * T); cudaMalloc(&dout, 8 * T); cudaMalloc(&dc, 8 * T);
    cudaMemcpy(dx, hx, sizeof(double) * n * T, cudaMemcpyHostToDevice);
    const double delta = 1e-6, td = 2e-6, inv = 1.0 / td, lim = td * 32768;
    long long hc[T];
    for (int rep = 0; rep < 2; ++rep) {
        k<0><<<1, T>>>(dx, n, delta, td, inv, lim, dc, dout); cudaMemcpy(hc, dc, 8 * T, cudaMemcpyDeviceToHost);
        printf("div:        %.1f cyc/step\n", (double)hc[0] / n);
        k<1><<<1, T>>>(dx, n, delta, td, inv, lim, dc, dout); cudaMemcpy(hc, dc, 8 * T, cudaMemcpyDeviceToHost);
        printf("mul+check:  %.1f cyc/step\n", (double)hc[0] / n);
        k<2><<<1, T>>>(dx, n, delta, td, inv, lim, dc, dout); cudaMemcpy(hc, dc, 8 * T, cudaMemcpyDeviceToHost);
        printf("mul+round:  %.1f cyc/step\n", (double)hc[0] / n);
    }
    return 0;
}
