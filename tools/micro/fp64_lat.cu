// FP64 latency / throughput probe for B200 (sm_100a): dependent DADD/DMUL/DFMA
// chains per warp, and issue throughput with many independent chains.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP, int CHAINS>
__global__ void chain(double* out, double x0, int iters, long long* cycles) {
  double v[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) v[c] = x0 + threadIdx.x + c;
  const double m = 1.0000001, a = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (OP == 0) v[c] = v[c] + a;
      if (OP == 1) v[c] = v[c] * m;
      if (OP == 2) v[c] = fma(v[c], m, a);
      if (OP == 3) v[c] = __drcp_rn(v[c]);
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
}

template <int OP, int CHAINS>
void run(const char* name, int blocks, int threads) {
  double* out; long long* cyc;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaMalloc(&cyc, sizeof(long long));
  const int iters = 4096;
  chain<OP, CHAINS><<<blocks, threads>>>(out, 1.0, iters, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  chain<OP, CHAINS><<<blocks, threads>>>(out, 1.0, iters, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double ops = (double)blocks * threads * iters * CHAINS;
  printf("%-6s chains=%2d blocks=%5d thr=%4d: %7.2f cyc/op/lane (block0)  %8.1f Gop/s\n", name,
         CHAINS, blocks, threads, (double)c / (iters * CHAINS), ops / ms / 1e6);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  run<0, 1>("DADD", 1, 32);
  run<1, 1>("DMUL", 1, 32);
  run<2, 1>("DFMA", 1, 32);
  run<3, 1>("DRCP", 1, 32);
  run<0, 8>("DADD", 1, 32);
  run<0, 8>("DADD", 148 * 8, 256);
  run<1, 8>("DMUL", 148 * 8, 256);
  run<2, 8>("DFMA", 148 * 8, 256);
  run<3, 8>("DRCP", 148 * 8, 256);
  return 0;
}
