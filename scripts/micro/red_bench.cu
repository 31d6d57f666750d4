// Dev microbenchmark: global RED.ADD.64 throughput on B200 for the access
// patterns of the moment flush (not part of the product).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;

// pattern 0: 32 consecutive int64 per warp instruction (coalesced)
// pattern 1: slot-flush shape: lane (c = lane&7, g = lane>>3) -> acc[g*NN + node + off(c)]
// pattern 2: random address per lane
__global__ void red_kernel(u64* acc, int NN, int pattern, int iters, int NY, int NZ) {
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int c = lane & 7, g = lane >> 3;
  const int off = (c & 1) * NY * NZ + ((c >> 1) & 1) * NZ + ((c >> 2) & 1);
  unsigned h = (unsigned)gw * 2654435761u;
  for (int it = 0; it < iters; ++it) {
    h = h * 1664525u + 1013904223u;
    long long a;
    if (pattern == 0) a = ((long long)(h % (unsigned)(10 * NN / 32))) * 32 + lane;
    else if (pattern == 1) a = (long long)g * NN + (h % (unsigned)(NN - NY * NZ - NZ - 2)) + off;
    else { unsigned r = (h ^ (lane * 0x9E3779B9u)) * 2246822519u; a = r % (unsigned)(10 * NN); }
    atomicAdd(acc + a, 1ull);
  }
}

int main() {
  const int NX = 129, NY = 65, NZ = 65, NN = NX * NY * NZ;
  u64* acc; cudaMalloc(&acc, sizeof(u64) * 10 * NN);
  cudaMemset(acc, 0, sizeof(u64) * 10 * NN);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * 8, threads = 256, iters = 512;
  for (int p = 0; p < 3; ++p) {
    red_kernel<<<blocks, threads>>>(acc, NN, p, 16, NY, NZ);
    cudaEventRecord(e0);
    red_kernel<<<blocks, threads>>>(acc, NN, p, iters, NY, NZ);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)blocks * threads * iters;
    printf("pattern %d: %.0f M RED.64 in %.3f ms = %.1f G/s\n", p, n / 1e6, ms, n / ms / 1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
