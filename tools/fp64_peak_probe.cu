// FP64 peak probe for the roofline denominator (DMMA tensor pipe and DFMA pipe).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak_probe fp64_peak_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(double* out, int iters){
  double a=threadIdx.x*1e-3, b=1.0000001;
  double c0[2]={0,0}, c1[2]={0,0}, c2[2]={0,0}, c3[2]={0,0};
  for(int i=0;i<iters;i++){
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0[0]),"+d"(c0[1]) : "d"(a),"d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c1[0]),"+d"(c1[1]) : "d"(a),"d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c2[0]),"+d"(c2[1]) : "d"(a),"d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c3[0]),"+d"(c3[1]) : "d"(a),"d"(b));
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=c0[0]+c0[1]+c1[0]+c1[1]+c2[0]+c2[1]+c3[0]+c3[1];
}
__global__ void dfma_loop(double* out, int iters){
  double a=threadIdx.x*1e-3, b=1.0000001;
  double c[8]={0,1,2,3,4,5,6,7};
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int j=0;j<8;j++) c[j]=fma(a,c[j],b);
  }
  double s=0; for(int j=0;j<8;j++) s+=c[j];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  double* d; cudaMalloc(&d, 148*64*1024*sizeof(double));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters=20000;
  for(int bpsm=1;bpsm<=8;bpsm*=2){
    int blocks=148*bpsm, threads=256;
    dmma_loop<<<blocks,threads>>>(d,100);
    cudaEventRecord(e0); dmma_loop<<<blocks,threads>>>(d,iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double flops=(double)blocks*(threads/32)*iters*4*(2.0*8*8*4);
    printf("DMMA m8n8k4 blocks/SM=%d: %.2f TFLOP/s\n",bpsm,flops/ms/1e9);
    dfma_loop<<<blocks,threads>>>(d,100);
    cudaEventRecord(e0); dfma_loop<<<blocks,threads>>>(d,iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms,e0,e1);
    flops=(double)blocks*threads*iters*8*2.0;
    printf("DFMA blocks/SM=%d: %.2f TFLOP/s\n",bpsm,flops/ms/1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
