// Dependent-chain latencies of FP64 ops on the GPU (cycles per op), single warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double* out, long long* cyc, double a, double b) {
  double x = a, y = b;
  long long t0, t1;
  const int R = 256;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < R; ++i) x = fma(x, y, 1e-300);
  t1 = clock64(); cyc[0] = (t1 - t0) / R;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < R; ++i) x = x + y;
  t1 = clock64(); cyc[1] = (t1 - t0) / R;
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < R; ++i) x = sqrt(x + 1.0);
  t1 = clock64(); cyc[2] = (t1 - t0) / R;
  // division chain
  t0 = clock64();
  for (int i = 0; i < R; ++i) x = y / (x + 1.0);
  t1 = clock64(); cyc[3] = (t1 - t0) / R;
  // rsqrt chain
  t0 = clock64();
  for (int i = 0; i < R; ++i) x = rsqrt(x + 1.0);
  t1 = clock64(); cyc[4] = (t1 - t0) / R;
  // drcp chain
  t0 = clock64();
  for (int i = 0; i < R; ++i) x = __drcp_rn(x + 1.0);
  t1 = clock64(); cyc[5] = (t1 - t0) / R;
  // shuffle (double) chain
  t0 = clock64();
  for (int i = 0; i < R; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
  t1 = clock64(); cyc[6] = (t1 - t0) / R;
  // shared load chain
  __shared__ double sm[64];
  sm[threadIdx.x] = x; __syncwarp();
  int idx = threadIdx.x & 7;
  t0 = clock64();
  for (int i = 0; i < R; ++i) { x = sm[idx] + x; idx = ((int)x & 7) | (threadIdx.x & 0); }
  t1 = clock64(); cyc[7] = (t1 - t0) / R;
  // syncthreads with 1 warp
  t0 = clock64();
  for (int i = 0; i < R; ++i) __syncthreads();
  t1 = clock64(); cyc[8] = (t1 - t0) / R;
  out[threadIdx.x] = x + y;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 64 * 8); cudaMallocManaged(&cyc, 16 * 8);
  probe<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999);
  cudaDeviceSynchronize();
  const char* n[] = {"dfma", "dadd", "sqrt", "div", "rsqrt", "drcp", "shfl+dadd", "lds+dadd+cvt", "bar(1 warp)"};
  for (int i = 0; i < 9; ++i) printf("%-14s %lld cycles\n", n[i], cyc[i]);
  return 0;
}
