// p2p_probe_ipc.cu -- peer-store bandwidth through a CUDA IPC mapping (two processes,
// GPU 1 exports a cudaMalloc buffer, GPU 0 maps it with cudaIpcMemLazyEnablePeerAccess).
#include <cstdio>
#include <unistd.h>
#include <sys/wait.h>
#include <cuda_runtime.h>
__global__ void store(double* dst, const double* src, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) dst[i] = src[i];
}
int main() {
  int p2c[2], c2p[2]; pipe(p2c); pipe(c2p);
  pid_t pid = fork();
  if (pid == 0) {  // exporter on GPU 1
    cudaSetDevice(1); double* buf; cudaMalloc(&buf, 64 << 20);
    cudaIpcMemHandle_t h; cudaIpcGetMemHandle(&h, buf);
    write(c2p[1], &h, sizeof h);
    char done; read(p2c[0], &done, 1);
    return 0;
  }
  cudaIpcMemHandle_t h; read(c2p[0], &h, sizeof h);
  cudaSetDevice(0);
  double *remote = nullptr, *local, *src;
  printf("open: %s\n", cudaGetErrorString(cudaIpcOpenMemHandle((void**)&remote, h, cudaIpcMemLazyEnablePeerAccess)));
  cudaMalloc(&local, 64 << 20); cudaMalloc(&src, 64 << 20); cudaMemset(src, 0, 64 << 20);
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
      printf("%s %8ld B: %.3f us/launch, %.1f GB/s\n", which ? "ipc-peer" : "local   ", bytes, ms * 100, bytes / (ms / 10 * 1e-3) / 1e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  char d = 1; write(p2c[1], &d, 1); wait(nullptr);
  return 0;
}
