// Dependent-chain latency of fp64 add / mul / fma and of the fp32->fp64 conversion on this GPU
// (one warp; cycles per dependent instruction), and the same with 2..8 warps on one SM
// sub-partition set (throughput sharing).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_lat fp64_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, long long* cyc, double a, double b, int n) {
  double s = a + threadIdx.x;
  float f = (float)a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (OP == 0) s = __dadd_rn(s, b);
      if (OP == 1) s = __dmul_rn(s, b);
      if (OP == 2) s = __fma_rn(s, b, a);
      if (OP == 3) { s = __dadd_rn((double)f, b); f = (float)s; }  // F2F both ways + DADD
      if (OP == 4) { double d = __dadd_rn(b, -s); s = __dadd_rn(s, __dmul_rn(d, d)); }  // sub,mul,add all dependent
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + f;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8 * 1024 * 1024); cudaMalloc(&cyc, 8);
  const char* names[] = {"DADD", "DMUL", "DFMA", "F2F.F64.F32 + DADD + F2F.F32.F64", "DADD -> DMUL -> DADD"};
  const int n = 4096;
  for (int threads : {32, 128, 256, 512, 1024}) {
    printf("%d threads on one SM:\n", threads);
    for (int op = 0; op < 5; ++op) {
      long long h;
      auto go = [&](int o) {
        if (o == 0) chain<0><<<1, threads>>>(out, cyc, 1.5, 1.0000001, n);
        if (o == 1) chain<1><<<1, threads>>>(out, cyc, 1.5, 1.0000001, n);
        if (o == 2) chain<2><<<1, threads>>>(out, cyc, 1.5, 1.0000001, n);
        if (o == 3) chain<3><<<1, threads>>>(out, cyc, 1.5, 1.0000001, n);
        if (o == 4) chain<4><<<1, threads>>>(out, cyc, 1.5, 1.0000001, n);
      };
      go(op); go(op);
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("  %-36s %6.1f cycles per step\n", names[op], (double)h / (n * 16.0));
    }
  }
  return 0;
}
