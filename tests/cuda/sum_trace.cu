// Debug harness: trace sumsq_iteration on a stride pair loaded from a file.
#include <cstdio>
#include <vector>
#define SUMSQ_TRACE 1
#include "../../paper_1811_05140_b200/csrc/qcs_codec.cuh"
using namespace qcs;
__global__ void k(const double* re, const double* im, int n, double* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* xs = reinterpret_cast<double*>(smem);
  int16_t* code = reinterpret_cast<int16_t*>(xs + 2 * PLANE_LANES * XS_STRIDE);
  EncShared& S = *reinterpret_cast<EncShared*>(smem + ENC_S_OFF);
  int pl = threadIdx.x >> 7, lane = threadIdx.x & 127;
  for (int i = lane; i < ITER; i += 128) xs_at(xs, pl, i) = i < n ? (pl ? im[i] : re[i]) : 0.0;
  if (threadIdx.x == 0) S.s = 0.0;
  __syncthreads();
  sumsq_iteration(xs, n, S, nullptr);
  __syncthreads();
  if (threadIdx.x == 0) *out = S.s;
}
int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb"); int n = atoi(argv[2]);
  std::vector<double> h(2 * n); fread(h.data(), 8, 2 * n, f); fclose(f);
  double *d, *o; cudaMalloc(&d, 16 * n); cudaMalloc(&o, 8);
  cudaMemcpy(d, h.data(), 16 * n, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ENC_SMEM);
  k<<<1, 256, ENC_SMEM>>>(d, d + n, n, o);
  double r; cudaMemcpy(&r, o, 8, cudaMemcpyDeviceToHost);
  double s = 0; for (int i = 0; i < n; ++i) s = s + (h[i] * h[i] + h[n + i] * h[n + i]);
  printf("device %.17g serial %.17g\n", r, s);
}
