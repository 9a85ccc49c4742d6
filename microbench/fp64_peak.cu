// FP64 ceiling microbenchmark for sm_100a: DFMA pipe, DMMA (mma.sync m8n8k4 f64) pipe.
// Also verifies the m8n8k4 f64 fragment layout assumed by the contraction kernel.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);} }while(0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i=0;i<iters;i++){
    x0=fma(x0,a,b); x1=fma(x1,a,b); x2=fma(x2,a,b); x3=fma(x3,a,b);
    x4=fma(x4,a,b); x5=fma(x5,a,b); x6=fma(x6,a,b); x7=fma(x7,a,b);
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}

__device__ __forceinline__ void dmma(double& d0,double& d1,double a,double b){
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};\n"
    : "+d"(d0),"+d"(d1) : "d"(a),"d"(b));
}
template<int NACC>
__global__ void dmma_kernel(double* out, int iters) {
  double acc0[NACC], acc1[NACC];
  double a = 1.0 + threadIdx.x*1e-3, b = 1.0 - threadIdx.x*1e-3;
  #pragma unroll
  for (int j=0;j<NACC;j++){acc0[j]=j; acc1[j]=-j;}
  for (int i=0;i<iters;i++){
    #pragma unroll
    for (int j=0;j<NACC;j++) dmma(acc0[j],acc1[j],a,b);
  }
  double s=0;
  #pragma unroll
  for (int j=0;j<NACC;j++) s+=acc0[j]+acc1[j];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
// layout check: A 8x4 row-major, B 4x8 (stored as B[k][n]), C 8x8
__global__ void dmma_layout(const double* A, const double* B, double* C){
  int l=threadIdx.x;
  double a=A[(l>>2)*4+(l&3)];
  double b=B[(l&3)*8+(l>>2)];
  double d0=0,d1=0;
  dmma(d0,d1,a,b);
  C[(l>>2)*8+(l&3)*2]=d0; C[(l>>2)*8+(l&3)*2+1]=d1;
}

int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  int clk=0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s SMs %d clock(max) %d kHz\n", p.name, p.multiProcessorCount, clk);
  // layout check
  double hA[32],hB[32],hC[64],ref[64];
  for(int i=0;i<32;i++){hA[i]=i*0.5+1; hB[i]=i*0.25-3;}
  for(int m=0;m<8;m++)for(int n=0;n<8;n++){double s=0;for(int k=0;k<4;k++)s+=hA[m*4+k]*hB[k*8+n];ref[m*8+n]=s;}
  double *dA,*dB,*dC; CK(cudaMalloc(&dA,256));CK(cudaMalloc(&dB,256));CK(cudaMalloc(&dC,512));
  CK(cudaMemcpy(dA,hA,256,cudaMemcpyHostToDevice));CK(cudaMemcpy(dB,hB,256,cudaMemcpyHostToDevice));
  dmma_layout<<<1,32>>>(dA,dB,dC); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(hC,dC,512,cudaMemcpyDeviceToHost));
  double err=0; for(int i=0;i<64;i++) err=fmax(err,fabs(hC[i]-ref[i]));
  printf("dmma m8n8k4 layout max err %g\n", err);

  int sms=p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, sizeof(double)*sms*64*1024));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int tpb : {256, 512, 1024}) for (int bps : {1,2,4}) {
    int iters=20000; int blocks=sms*bps;
    dfma_kernel<<<blocks,tpb>>>(out,100,1.0000001,1e-9);
    cudaEventRecord(e0); dfma_kernel<<<blocks,tpb>>>(out,iters,1.0000001,1e-9); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1);
    double fl=2.0*8*iters*(double)blocks*tpb;
    printf("DFMA tpb %4d blocks/SM %d: %.2f TFLOP/s (%.3f ms)\n",tpb,bps,fl/ms/1e9,ms);
  }
  for (int tpb : {128, 256, 512}) for (int bps : {1,2,4}) {
    int iters=20000; int blocks=sms*bps;
    dmma_kernel<8><<<blocks,tpb>>>(out,100);
    cudaEventRecord(e0); dmma_kernel<8><<<blocks,tpb>>>(out,iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1);
    double fl=512.0*8*iters*(double)blocks*(tpb/32);
    printf("DMMA8 tpb %4d blocks/SM %d: %.2f TFLOP/s (%.3f ms)\n",tpb,bps,fl/ms/1e9,ms);
  }
  for (int tpb : {128, 256}) {
    int iters=20000; int blocks=sms*2;
    dmma_kernel<4><<<blocks,tpb>>>(out,100);
    cudaEventRecord(e0); dmma_kernel<4><<<blocks,tpb>>>(out,iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1);
    double fl=512.0*4*iters*(double)blocks*(tpb/32);
    printf("DMMA4 tpb %4d blocks/SM 2: %.2f TFLOP/s (%.3f ms)\n",tpb,fl/ms/1e9,ms);
  }
  return 0;
}
