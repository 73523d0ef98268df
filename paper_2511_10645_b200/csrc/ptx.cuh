// ptx.cuh -- thin inline-PTX helpers for sm_100a (mbarrier, bulk async copy,
// cluster / DSMEM, programmatic dependent launch).  No ParoQuant arithmetic.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

#define PARO_DEV __device__ __forceinline__
#ifndef PARO_MBAR_SUSPEND_NS
#define PARO_MBAR_SUSPEND_NS 1000000u
#endif

namespace paro {

PARO_DEV uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// ---------------------------------------------------------------- mbarrier
PARO_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
PARO_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
PARO_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
PARO_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
PARO_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
PARO_DEV bool mbar_try_wait_spin(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
PARO_DEV bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  // suspend-time hint: the waiting warp is parked by the hardware until the phase completes
  // (or the hint expires) instead of spinning on issue slots and the shared-memory pipe
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(PARO_MBAR_SUSPEND_NS)
      : "memory");
  return ok != 0;
}
PARO_DEV uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Wait for the phase with the given parity.  Watchdog: a phase that never completes (a protocol
// bug) traps after 4 s instead of hanging the GPU; the clock is read every 256 retries only.
PARO_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
#if PARO_MBAR_SPIN
  if (mbar_try_wait_spin(bar, parity)) return;
#else
  if (mbar_try_wait(bar, parity)) return;
#endif
  const uint64_t t0 = globaltimer_ns();
  uint32_t n = 0;
#if PARO_MBAR_SPIN
  while (!mbar_try_wait_spin(bar, parity)) {
#else
  while (!mbar_try_wait(bar, parity)) {
#endif
    if ((++n & 255u) == 0u && globaltimer_ns() - t0 > 4000000000ull) __trap();
  }
}

// spin variant (no suspend hint) for short waits on the critical path (e.g. tcgen05.commit)
PARO_DEV void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait_spin(bar, parity)) return;
  const uint64_t t0 = globaltimer_ns();
  uint32_t n = 0;
  while (!mbar_try_wait_spin(bar, parity)) {
    if ((++n & 1023u) == 0u && globaltimer_ns() - t0 > 4000000000ull) __trap();
  }
}

// ---------------------------------------------------------------- bulk async copy (TMA engine, 1-D)
// global -> shared::cta, completion counted on an mbarrier (complete_tx), L2 evict-first hint.
PARO_DEV uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
PARO_DEV void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

PARO_DEV void bulk_g2s_nohint(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// ---------------------------------------------------------------- cluster / DSMEM
PARO_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
PARO_DEV uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
PARO_DEV void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
PARO_DEV void cluster_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory"); }
PARO_DEV void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
PARO_DEV uint32_t mapa(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
// asynchronous DSMEM store; completion counted (bytes) on the receiver's mbarrier
PARO_DEV void st_async_v2(uint32_t remote_addr, uint32_t v0, uint32_t v1, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];" ::"r"(remote_addr),
               "r"(v0), "r"(v1), "r"(remote_bar)
               : "memory");
}
PARO_DEV void st_async_b32(uint32_t remote_addr, uint32_t v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(remote_addr), "r"(v),
               "r"(remote_bar)
               : "memory");
}
PARO_DEV void prefetch_l2_bulk(const void* gmem, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gmem), "r"(bytes) : "memory");
}
PARO_DEV void st_cluster_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// ---------------------------------------------------------------- named barrier
PARO_DEV void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// non-.aligned form: the threads of a warp may reach it from different branches
PARO_DEV void named_bar_sync_na(uint32_t id, uint32_t nthreads) {
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
PARO_DEV void named_bar_arrive(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}


// ---------------------------------------------------------------- grid-wide barrier (persistent chains)
// Flat flags: every CTA publishes its arrival at barrier k of the launch with epoch e as
// flag[cta] = 64 e + k + 1 (st.release), and a waiter polls all flags until each is >= that
// value -- one store and one poll round trip, no read-modify-write on the critical path.  The
// epoch word is read once per launch (after the previous kernel on the stream completed) and
// bumped by CTA 0 when it exits, so flags left by earlier launches never satisfy a wait.
// All CTAs of the grid are co-resident (one wave, grid <= occupancy); < 64 barriers per launch.
struct GridBar {
  uint32_t* epoch;  // workspace word
  uint32_t* flags;  // [gridDim.x]
};
PARO_DEV uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
PARO_DEV void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
PARO_DEV void st_relaxed_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
PARO_DEV void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// one thread per CTA, after a CTA barrier that orders the CTA's writes before it
PARO_DEV void grid_arrive(const GridBar& gb, uint32_t target) { st_release_gpu(gb.flags + blockIdx.x, target); }
// one full warp; returns when every CTA's flag reached `target` (then CTA-barrier the rest)
PARO_DEV void grid_wait_warp(const GridBar& gb, uint32_t target, int lane) {
  const int n = static_cast<int>(gridDim.x);
  const uint64_t t0 = globaltimer_ns();
  for (;;) {
    bool ok = true;
    for (int j = lane; j < n; j += 32) ok &= static_cast<int>(ld_relaxed_gpu(gb.flags + j) - target) >= 0;
    if (__all_sync(0xffffffffu, ok)) break;
    if (globaltimer_ns() - t0 > 2000000000ull) __trap();  // a CTA never arrived: error, not a hang
  }
  fence_acq_rel_gpu();
}

// ---------------------------------------------------------------- programmatic dependent launch
PARO_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
PARO_DEV void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------- shared loads
PARO_DEV uint4 lds128(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}

// shared loads by 32-bit shared-window address (volatile: never hoisted above the
// mbarrier wait that guards the data)
PARO_DEV uint4 lds128_a(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
PARO_DEV unsigned short lds_u16_a(uint32_t addr) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}
PARO_DEV uint32_t lds_u8_a(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

PARO_DEV uint32_t lds_u32_a(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
PARO_DEV uint2 lds_u64_a(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
PARO_DEV uint32_t lds_u16z_a(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
PARO_DEV float2 lds_f2_a(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}

// ---------------------------------------------------------------- warp-level tensor-core MMA
// D(16x8, fp32) += A(16x16, fp16, row) * B(16x8, fp16, col)  (SASS HMMA.16816.F32).
// Fragments (g = lane / 4, t = lane % 4): a0 = A[g][2t..2t+1], a1 = A[g+8][2t..], a2 = A[g][2t+8..],
// a3 = A[g+8][2t+8..]; b0 = B[2t..2t+1][g], b1 = B[2t+8..2t+9][g]; d = D[g][2t], D[g][2t+1],
// D[g+8][2t], D[g+8][2t+1].  fp16 subnormal A inputs are exact (tools/probe_hmma.cu).
PARO_DEV void mma_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
PARO_DEV void mma_16816_z(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%10,%10,%10};"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(0.f));
}

}  // namespace paro

// D(16x8, s32) += A(16x32, u8, row) * B(32x8, s8, col)  (SASS IMMA.16832.U8.S8, native on sm_100a:
// 512 A elements per instruction, 2x the HMMA.16816 rate per A element; tools/probe_mma_kinds.cu).
// Fragments: a0 = A[g][4t..4t+3], a1 = A[g+8][4t..], a2 = A[g][16+4t..], a3 = A[g+8][16+4t..];
// b0 = B[4t..4t+3][g], b1 = B[16+4t..16+4t+3][g]; d as for mma_16816.  Exact integer arithmetic.
PARO_DEV void imma_16832(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
PARO_DEV void imma_16832_z(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%10,%10,%10};"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "r"(0));
}
PARO_DEV void st_async_v4(uint32_t remote_addr, uint4 v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   remote_addr),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(remote_bar)
               : "memory");
}
