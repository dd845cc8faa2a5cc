// p2p_probe.cu -- peer-store bandwidth probe between GPU 0 and GPU 1 (one process):
// 8-byte stores from a kernel into peer memory vs into local memory.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void store(double* dst, const double* src, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) dst[i] = src[i];
}
int main() {
  int n = 0; cudaGetDeviceCount(&n);
  if (n < 2) { printf("need 2 GPUs\n"); return 0; }
  int can = 0; cudaDeviceCanAccessPeer(&can, 0, 1);
  printf("canAccessPeer(0,1)=%d\n", can);
  cudaSetDevice(1); double* remote; cudaMalloc(&remote, 64 << 20);
  cudaSetDevice(0); double *local, *src; cudaMalloc(&local, 64 << 20); cudaMalloc(&src, 64 << 20);
  cudaMemset(src, 0, 64 << 20);
  printf("enablePeer: %s\n", cudaGetErrorString(cudaDeviceEnablePeerAccess(1, 0)));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (long bytes : {1L << 20, 8L << 20, 64L << 20}) {
    for (int which = 0; which < 2; ++which) {
      double* dst = which ? remote : local;
      long cnt = bytes / 8;
      int grid = (int)((cnt + 255) / 256); if (grid > 592) grid = 592;
      store<<<grid, 256>>>(dst, src, cnt);
      cudaEventRecord(a);
      for (int r = 0; r < 10; ++r) store<<<grid, 256>>>(dst, src, cnt);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("%s %8ld B: %.3f us/launch, %.1f GB/s\n", which ? "peer " : "local", bytes, ms * 100, bytes / (ms / 10 * 1e-3) / 1e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
