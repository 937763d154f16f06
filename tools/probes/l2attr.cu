#include <cstdio>
#include <cuda_runtime.h>
int main() {
  int v[4];
  cudaDeviceGetAttribute(&v[0], cudaDevAttrL2CacheSize, 0);
  cudaDeviceGetAttribute(&v[1], cudaDevAttrMaxPersistingL2CacheSize, 0);
  cudaDeviceGetAttribute(&v[2], cudaDevAttrMaxAccessPolicyWindowSize, 0);
  printf("L2 %d B, max persisting %d B, max access-policy window %d B\n", v[0], v[1], v[2]);
}
