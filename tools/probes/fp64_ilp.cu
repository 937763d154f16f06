// Single-warp issue rate of independent fp64 instructions (ILP): K independent DADD chains
// interleaved in one warp; cycles per DADD.  Also: one dependent DADD chain with J independent
// integer instructions between consecutive adds (do they fit in the 8-cycle shadow?).
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void ilp(double* out, long long* cyc, double b, int n) {
  double s[K];
#pragma unroll
  for (int k = 0; k < K; ++k) s[k] = b + threadIdx.x + k;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int k = 0; k < K; ++k) s[k] = __dadd_rn(s[k], b);
  }
  long long t1 = clock64();
  double r = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) r += s[k];
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int J>
__global__ void shadow(double* out, long long* cyc, double b, int n, unsigned m) {
  double s = b + threadIdx.x;
  unsigned x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 7 + j;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s = __dadd_rn(s, b);
#pragma unroll
      for (int j = 0; j < J; ++j) x[j & 7] = (x[j & 7] >> 3) ^ (x[(j + 1) & 7] & m);
    }
  }
  long long t1 = clock64();
  unsigned r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r += x[j];
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + r;
}

int main() {
  double* out; long long* cyc; long long h;
  cudaMalloc(&out, 8 << 20); cudaMalloc(&cyc, 8);
  const int n = 4096;
  for (int threads : {32, 64, 256}) {
    printf("%d threads:\n", threads);
#define RUN(K) ilp<K><<<1, threads>>>(out, cyc, 1.0000001, n); ilp<K><<<1, threads>>>(out, cyc, 1.0000001, n); \
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("  %d independent DADD chains: %.2f cycles per DADD\n", K, (double)h / (n * 8.0 * K));
    RUN(1) RUN(2) RUN(4) RUN(8)
#define RUNS(J) shadow<J><<<1, threads>>>(out, cyc, 1.0000001, n, 0x8fffffffu); shadow<J><<<1, threads>>>(out, cyc, 1.0000001, n, 0x8fffffffu); \
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("  dependent DADD + %d integer ops between: %.2f cycles per step\n", J, (double)h / (n * 8.0));
    RUNS(0) RUNS(2) RUNS(4) RUNS(6) RUNS(8) RUNS(12)
  }
  return 0;
}
