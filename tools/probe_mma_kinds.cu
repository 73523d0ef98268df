// Probe: mma.sync throughput on sm_100a for the operand kinds a bs=1 INT4 GEMV could use:
// f16 m16n8k16 (256 MAC/row-col... 2048 MAC), e4m3 m16n8k32, u8.s8 m16n8k32, u4.s4 m16n8k64.
// Reports MMA instructions per clock per SM and A-elements (weights) per clock per SM.
#include <cstdio>
#include <cstdint>
#define MMA_F16(D, a, b) asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};" \
  : "+f"(D[0]), "+f"(D[1]), "+f"(D[2]), "+f"(D[3]) : "r"(a), "r"(a ^ 1), "r"(a + 2), "r"(a + 3), "r"(b), "r"(b))
#define MMA_E4M3(D, a, b) asm volatile("mma.sync.aligned.m16n8k32.row.col.f32.e4m3.e4m3.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};" \
  : "+f"(D[0]), "+f"(D[1]), "+f"(D[2]), "+f"(D[3]) : "r"(a), "r"(a ^ 1), "r"(a + 2), "r"(a + 3), "r"(b), "r"(b))
#define MMA_S8(D, a, b) asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};" \
  : "+r"(D[0]), "+r"(D[1]), "+r"(D[2]), "+r"(D[3]) : "r"(a), "r"(a ^ 1), "r"(a + 2), "r"(a + 3), "r"(b), "r"(b))
#define MMA_S4(D, a, b) asm volatile("mma.sync.aligned.m16n8k64.row.col.s32.u4.s4.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};" \
  : "+r"(D[0]), "+r"(D[1]), "+r"(D[2]), "+r"(D[3]) : "r"(a), "r"(a ^ 1), "r"(a + 2), "r"(a + 3), "r"(b), "r"(b))

template <int KIND>
__global__ void k(float* out, int iters) {
  uint32_t a = 0x01020304u + threadIdx.x, b = 0x3c003c00u ^ threadIdx.x;
  if (KIND == 0 || KIND == 1) {
    float D[8][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 8; j++) {
        if (KIND == 0) MMA_F16(D[j], a, b); else MMA_E4M3(D[j], a, b);
      }
      a += 0x10;
    }
    float s = 0; for (int j = 0; j < 8; j++) s += D[j][0] + D[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  } else {
    int D[8][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 8; j++) {
        if (KIND == 2) MMA_S8(D[j], a, b); else MMA_S4(D[j], a, b);
      }
      a += 0x10;
    }
    int s = 0; for (int j = 0; j < 8; j++) s += D[j][0] + D[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  }
}

// exactness of u4 x s4 (A row-major 16x64 nibbles, B col-major 64x8 nibbles)
__global__ void kex(const uint8_t* A, const int8_t* B, int* out) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  // A fragment m16n8k64 (.u4): a0: row g, k 8t..8t+7; a1: row g+8, same; a2: row g, k 32+8t..; a3: row g+8, k 32+8t..
  auto pa = [&](int r, int k0) { uint32_t v = 0; for (int i = 0; i < 8; i++) v |= (uint32_t)(A[r * 64 + k0 + i] & 15) << (4 * i); return v; };
  auto pb = [&](int n, int k0) { uint32_t v = 0; for (int i = 0; i < 8; i++) v |= (uint32_t)(B[n * 64 + k0 + i] & 15) << (4 * i); return v; };
  uint32_t a0 = pa(g, 8 * t), a1 = pa(g + 8, 8 * t), a2 = pa(g, 32 + 8 * t), a3 = pa(g + 8, 32 + 8 * t);
  uint32_t b0 = pb(g, 8 * t), b1 = pb(g, 32 + 8 * t);
  int D[4] = {0, 0, 0, 0};
  asm volatile("mma.sync.aligned.m16n8k64.row.col.s32.u4.s4.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+r"(D[0]), "+r"(D[1]), "+r"(D[2]), "+r"(D[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  out[g * 8 + 2 * t] = D[0]; out[g * 8 + 2 * t + 1] = D[1]; out[(g + 8) * 8 + 2 * t] = D[2]; out[(g + 8) * 8 + 2 * t + 1] = D[3];
}

int main() {
  float* dout; cudaMalloc(&dout, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[4] = {"f16 m16n8k16", "e4m3 m16n8k32", "u8.s8 m16n8k32", "u4.s4 m16n8k64"};
  const int kdim[4] = {16, 32, 32, 64};
  int iters = 2048;
  for (int kind = 0; kind < 4; kind++) for (int warps = 4; warps <= 16; warps *= 2) {
    float ms = 0;
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(e0);
      if (kind == 0) k<0><<<148, warps * 32>>>(dout, iters);
      if (kind == 1) k<1><<<148, warps * 32>>>(dout, iters);
      if (kind == 2) k<2><<<148, warps * 32>>>(dout, iters);
      if (kind == 3) k<3><<<148, warps * 32>>>(dout, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    double mmas = 148.0 * warps * iters * 8;
    double per_clk = mmas / (ms * 1e-3) / 148 / 1.965e9;
    printf("%-16s warps=%2d: %.3f ms  %.3f mma/clk/SM  (%.1f clk/mma/SMSP)  %.0f A-elem/clk/SM\n", names[kind], warps, ms, per_clk,
           4.0 / per_clk, per_clk * 16 * kdim[kind]);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  // exactness u4.s4
  uint8_t hA[16 * 64]; int8_t hB[8 * 64];
  srand(3);
  for (int i = 0; i < 16 * 64; i++) hA[i] = rand() & 15;
  for (int i = 0; i < 8 * 64; i++) hB[i] = (int8_t)((rand() & 15) - 8);
  uint8_t* dA; int8_t* dB; int* dD; cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, 512);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  kex<<<1, 32>>>(dA, dB, dD);
  int hD[128]; cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < 16; r++) for (int n = 0; n < 8; n++) {
    int ref = 0; for (int kk = 0; kk < 64; kk++) ref += hA[r * 64 + kk] * hB[n * 64 + kk];
    if (ref != hD[r * 8 + n]) bad++;
  }
  printf("u4.s4 exactness: %d / 128 wrong; err %s\n", bad, cudaGetErrorString(cudaGetLastError()));
}
