// probe: does fma.rn.f32.f16 keep fp16 subnormal inputs?  does cvt e4m3x2->f16x2 give q*2^-9?
#include <cstdio>
#include <cuda_fp16.h>
__global__ void k(float* out) {
  unsigned a2 = 0x00050003u;            // halves: 3*2^-24, 5*2^-24 (subnormal)
  unsigned b2 = 0x3c003c00u;            // 1.0, 1.0
  float d0, d1;
  asm volatile("{.reg .f16 a0,a1,b0,b1;\n mov.b32 {a0,a1}, %2;\n mov.b32 {b0,b1}, %3;\n fma.rn.f32.f16 %0, a0, b0, 0f00000000;\n fma.rn.f32.f16 %1, a1, b1, 0f00000000;\n}" : "=f"(d0), "=f"(d1) : "r"(a2), "r"(b2));
  out[0] = d0 * 16777216.f; out[1] = d1 * 16777216.f;
  unsigned short e = 0x0f05;  // bytes 0x05, 0x0f -> e4m3 q=5, q=15
  unsigned h2;
  asm volatile("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(e));
  __half2 hh = *reinterpret_cast<__half2*>(&h2);
  out[2] = __low2float(hh) * 512.f; out[3] = __high2float(hh) * 512.f;
  // hfma2 with subnormal
  __half2 s = *reinterpret_cast<__half2*>(&a2);
  __half2 r = __hmul2(s, __floats2half2_rn(1024.f, 1024.f));
  out[4] = __low2float(r); out[5] = __high2float(r);
}
int main() {
  float* d; cudaMalloc(&d, 64); k<<<1,1>>>(d); float h[6]; cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  printf("fhfma subnormal: %g %g (expect 3 5)\ncvt e4m3: %g %g (expect 5 15)\nhmul2 subnormal*1024: %g %g (expect 3/16384 5/16384 = %g %g)\n", h[0], h[1], h[2], h[3], h[4], h[5], 3.0/16384, 5.0/16384);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
