// Throughput probe: 32-weight INT4 dot products per SM per cycle,
// (a) subnormal-fp16 FHFMA path, (b) dp4a (IDP.4A) fixed-point path.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
__device__ __forceinline__ float fl(uint32_t a, uint32_t b, float c){float d;asm("{.reg .f16 a0,a1,b0,b1;\n mov.b32 {a0,a1},%1;\n mov.b32 {b0,b1},%2;\n fma.rn.f32.f16 %0,a0,b0,%3;}":"=f"(d):"r"(a),"r"(b),"f"(c));return d;}
__device__ __forceinline__ float fh(uint32_t a, uint32_t b, float c){float d;asm("{.reg .f16 a0,a1,b0,b1;\n mov.b32 {a0,a1},%1;\n mov.b32 {b0,b1},%2;\n fma.rn.f32.f16 %0,a1,b1,%3;}":"=f"(d):"r"(a),"r"(b),"f"(c));return d;}
__global__ void kf(const uint4* __restrict__ src, float* out, int iters){
  uint32_t P[16]; for(int i=0;i<16;i++) P[i]=0x3c003c00u+threadIdx.x*i;
  uint4 c = src[threadIdx.x & 63];
  float acc[4]={0,0,0,0};
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int r=0;r<4;r++){
      float tl=0.f, th=0.f;
      uint32_t w[4]={c.x^r, c.y^r, c.z^r, c.w^r};
      #pragma unroll
      for(int m=0;m<4;m++){ uint32_t x=w[m], x8=x>>8;
        tl=fl(x&0x000F000Fu,P[4*m],tl); th=fl(x&0x00F000F0u,P[4*m+1],th);
        tl=fh(x&0x000F000Fu,P[4*m],tl); th=fh(x&0x00F000F0u,P[4*m+1],th);
        tl=fl(x8&0x000F000Fu,P[4*m+2],tl); th=fl(x8&0x00F000F0u,P[4*m+3],th);
        tl=fh(x8&0x000F000Fu,P[4*m+2],tl); th=fh(x8&0x00F000F0u,P[4*m+3],th);}
      acc[r]+=fmaf(0.0625f,th,tl);
    }
    c.x+=1;
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=acc[0]+acc[1]+acc[2]+acc[3];
}
__global__ void ki(const uint4* __restrict__ src, float* out, int iters){
  uint32_t X[16]; for(int i=0;i<16;i++) X[i]=0x01020304u*(threadIdx.x+i);
  uint4 c = src[threadIdx.x & 63];
  float acc[4]={0,0,0,0};
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int r=0;r<4;r++){
      int hi=0; unsigned lo=0;
      uint32_t w[4]={c.x^r, c.y^r, c.z^r, c.w^r};
      #pragma unroll
      for(int m=0;m<4;m++){ uint32_t e=w[m]&0x0F0F0F0Fu, o=(w[m]>>4)&0x0F0F0F0Fu; int t; unsigned t2;
        asm("dp4a.u32.s32 %0,%1,%2,%3;":"=r"(t):"r"(e),"r"(X[4*m]),"r"(hi)); hi=t;
        asm("dp4a.u32.s32 %0,%1,%2,%3;":"=r"(t):"r"(o),"r"(X[4*m+1]),"r"(hi)); hi=t;
        asm("dp4a.u32.u32 %0,%1,%2,%3;":"=r"(t2):"r"(e),"r"(X[4*m+2]),"r"(lo)); lo=t2;
        asm("dp4a.u32.u32 %0,%1,%2,%3;":"=r"(t2):"r"(o),"r"(X[4*m+3]),"r"(lo)); lo=t2;}
      acc[r]+=(float)(hi*256+(int)lo);
    }
    c.x+=1;
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=acc[0]+acc[1]+acc[2]+acc[3];
}
int main(){
  uint4* s; float* o; cudaMalloc(&s, 64*16); cudaMemset(s,0x5a,64*16); cudaMalloc(&o, 148*8*512*4);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters=4096;
  for(int v=0; v<2; v++){
    for(int rep=0;rep<3;rep++){
      cudaEventRecord(a);
      if(v==0) kf<<<148*4,256>>>(s,o,iters); else ki<<<148*4,256>>>(s,o,iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms,a,b);
      double weights = 148.0*4*256*iters*4*32;
      if(rep==2) printf("%s: %.3f ms  %.1f Tweights/s  (%.2f weights/clk/SM at 1.965GHz)\n", v?"dp4a":"fhfma", ms, weights/ms/1e9, weights/(ms*1e-3)/148/1.965e9);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
