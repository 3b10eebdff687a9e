// Throughput probe: legacy warp-level IMMA (mma.sync m16n8k32 s8 -> s32) and DMMA on this GPU.
// usage: ./imma_probe   (prints TOPS for several CTA counts per SM)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void imma_loop(int* out, int iters) {
  int a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  int c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x, b = a * 0.5;
  double c[8][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* o;
  cudaMalloc(&o, 1 << 26);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int per : {1, 2, 4, 8}) {
    for (int warps : {4, 8}) {
      const int iters = 4096, grid = sms * per, thr = 32 * warps;
      imma_loop<<<grid, thr>>>(o, 16);
      cudaEventRecord(e0);
      imma_loop<<<grid, thr>>>(o, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 2.0 * 16 * 8 * 32 * 8 * (double)iters * grid * warps;
      printf("IMMA m16n8k32 s8: ctas/SM %d warps %d: %.1f TOPS\n", per, warps, ops / ms / 1e9);
      dmma_loop<<<grid, thr>>>((double*)o, 16);
      cudaEventRecord(e0);
      dmma_loop<<<grid, thr>>>((double*)o, iters / 4);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double fl = 2.0 * 8 * 8 * 4 * 8 * (double)(iters / 4) * grid * warps;
      printf("DMMA m8n8k4 f64: ctas/SM %d warps %d: %.2f TFLOPS\n", per, warps, fl / ms / 1e9);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
