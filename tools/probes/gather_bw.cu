// Random-gather bandwidth probe: how many GB/s does B200 HBM deliver for random accesses of
// G bytes (32 / 64 / 128 / 256), versus a streaming copy?  Each warp issues U independent
// random G-byte gathers per round (lanes split each gather into 16-byte pieces).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bw gather_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}

template <int G, int U>
__global__ void gather(const uint4* __restrict__ buf, uint64_t nchunks, int rounds, uint4* out) {
  constexpr int LPG = G / 16;        // lanes per gather
  constexpr int GPW = 32 / LPG;      // gathers per warp instruction
  const int lane = threadIdx.x & 31;
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int r = 0; r < rounds; ++r) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t g = mix(w * 1000003ull + r * 7919ull + u * 104729ull + lane / LPG) % nchunks;
      v[u] = __ldcg(buf + g * LPG + (lane % LPG));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) { acc.x ^= v[u].x; acc.y += v[u].y; acc.z |= v[u].z; acc.w ^= v[u].w; }
  }
  if (acc.x == 0x12345678u) out[0] = acc;
}

template <int G>
void run(const uint4* buf, uint64_t bytes, uint4* out, int sms) {
  const uint64_t nchunks = bytes / G;
  const int blocks = sms * 8, threads = 256, rounds = 64;
  constexpr int U = 8;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  gather<G, U><<<blocks, threads>>>(buf, nchunks, 4, out);
  cudaEventRecord(a);
  gather<G, U><<<blocks, threads>>>(buf, nchunks, rounds, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double gathers = (double)blocks * threads / 32 * (32 / (G / 16)) * U * rounds;
  printf("random %4d-byte gathers: %8.1f GB/s useful (%.2f G gathers/s)\n", G, gathers * G / ms / 1e6,
         gathers / ms / 1e6);
}

__global__ void stream_copy(const uint4* __restrict__ s, uint4* __restrict__ d, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t bytes = 2ull << 30;
  uint4 *buf, *out, *dst;
  cudaMalloc(&buf, bytes); cudaMalloc(&out, 64); cudaMalloc(&dst, bytes);
  cudaMemset(buf, 1, bytes);
  run<16>(buf, bytes, out, sms);
  run<32>(buf, bytes, out, sms);
  run<64>(buf, bytes, out, sms);
  run<128>(buf, bytes, out, sms);
  run<256>(buf, bytes, out, sms);
  run<512>(buf, bytes, out, sms);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  stream_copy<<<sms * 8, 256>>>(buf, dst, bytes / 16);
  cudaEventRecord(a);
  stream_copy<<<sms * 8, 256>>>(buf, dst, bytes / 16);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("stream copy: %.1f GB/s (read + write)\n", 2.0 * bytes / ms / 1e6);
  return 0;
}
