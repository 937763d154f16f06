// Row-walk bandwidth probe: the real-valued routing kernel reads C random 3,840-byte rows per
// expansion with 8 warps per SM.  How fast can the memory system deliver them
//   (A) one row per lane, 16-byte loads, S slots of 64 bytes in flight per lane (the kernel's
//       register pipeline): every L1 miss is a single-sector request;
//   (B) 8 lanes per 128-byte line, 4 rows per warp instruction, U line-columns in flight:
//       every request is a whole line?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rowwalk_bw rowwalk_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}
constexpr int kRowB = 3840, kRow16 = kRowB / 16;

template <int S>
__global__ void lane_rows(const uint4* __restrict__ buf, uint64_t nrows, int rounds, int C, uint4* out) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int r = 0; r < rounds; ++r) {
    if (lane < C) {
      const uint4* row = buf + (mix(w * 1000003ull + r * 7919ull + lane) % nrows) * kRow16;
      uint4 v[S][4];
#pragma unroll
      for (int s = 0; s < S; ++s)
#pragma unroll
        for (int u = 0; u < 4; ++u) v[s][u] = __ldg(row + s * 4 + u);
      for (int c = 0; c < kRow16 / 4; c += S) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
#pragma unroll
          for (int u = 0; u < 4; ++u) { acc.x ^= v[s][u].x; acc.y += v[s][u].y; acc.z |= v[s][u].z; acc.w ^= v[s][u].w; }
          if (c + s + S < kRow16 / 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) v[s][u] = __ldg(row + (c + s + S) * 4 + u);
          }
        }
      }
    }
    __syncwarp();
  }
  if (acc.x == 0x12345678u) out[0] = acc;
}

template <int U>
__global__ void line_rows(const uint4* __restrict__ buf, uint64_t nrows, int rounds, int C, uint4* out) {
  const int lane = threadIdx.x & 31;
  const int sub = lane & 7, grp = lane >> 3;  // 8 lanes per line, 4 rows per instruction
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int r = 0; r < rounds; ++r) {
    for (int r0 = 0; r0 < C; r0 += 4) {
      const bool on = r0 + grp < C;
      const uint4* row = buf + (mix(w * 1000003ull + r * 7919ull + r0 + grp) % nrows) * kRow16;
      for (int c = 0; c < kRow16 / 8; c += U) {  // 30 lines per row
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (on && c + u < kRow16 / 8) v[u] = __ldg(row + (c + u) * 8 + sub);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (on && c + u < kRow16 / 8) { acc.x ^= v[u].x; acc.y += v[u].y; acc.z |= v[u].z; acc.w ^= v[u].w; }
      }
    }
  }
  if (acc.x == 0x12345678u) out[0] = acc;
}

template <class K>
void timeit(const char* name, K launch, double bytes) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  launch(2);
  cudaEventRecord(a);
  launch(40);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%-58s %8.1f GB/s\n", name, bytes * 40 / ms / 1e6);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t bytes = 4ull << 30, nrows = bytes / kRowB;
  uint4 *buf, *out;
  cudaMalloc(&buf, bytes); cudaMalloc(&out, 64);
  cudaMemset(buf, 1, bytes);
  for (int wps : {8, 16}) {
    const int threads = 256, blocks = sms * wps / 8;
    for (int C : {8, 32}) {
      const double per_round = (double)blocks * 8 * C * kRowB;
      char nm[128];
      snprintf(nm, sizeof nm, "%d warps/SM, %2d rows: lane per row, 4 x 64 B in flight", wps, C);
      timeit(nm, [&](int rounds) { lane_rows<4><<<blocks, threads>>>(buf, nrows, rounds, C, out); }, per_round);
      snprintf(nm, sizeof nm, "%d warps/SM, %2d rows: lane per row, 8 x 64 B in flight", wps, C);
      timeit(nm, [&](int rounds) { lane_rows<8><<<blocks, threads>>>(buf, nrows, rounds, C, out); }, per_round);
      snprintf(nm, sizeof nm, "%d warps/SM, %2d rows: 8 lanes per line, 4 columns in flight", wps, C);
      timeit(nm, [&](int rounds) { line_rows<4><<<blocks, threads>>>(buf, nrows, rounds, C, out); }, per_round);
      snprintf(nm, sizeof nm, "%d warps/SM, %2d rows: 8 lanes per line, 8 columns in flight", wps, C);
      timeit(nm, [&](int rounds) { line_rows<8><<<blocks, threads>>>(buf, nrows, rounds, C, out); }, per_round);
      snprintf(nm, sizeof nm, "%d warps/SM, %2d rows: 8 lanes per line, 16 columns in flight", wps, C);
      timeit(nm, [&](int rounds) { line_rows<16><<<blocks, threads>>>(buf, nrows, rounds, C, out); }, per_round);
    }
  }
  return 0;
}
