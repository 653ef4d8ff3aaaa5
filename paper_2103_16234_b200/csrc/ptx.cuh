// Inline-PTX helpers shared by the kernels: mbarriers (producer/consumer
// pipelines), elect.sync, cp.async completion tracking and TMA tensor loads.
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace b2c {

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// mbarrier wait.  limit_ns == 0 (default): unbounded — a correct kernel may be
// preempted or time-sliced for any length of time.  limit_ns > 0 (watchdog,
// B2C_WATCHDOG_MS, set by the test suite): a protocol bug traps (kernel error)
// instead of hanging the GPU; wall time (globaltimer), checked every 256 polls.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity, unsigned long long limit_ns,
                                          unsigned int *dbg = nullptr, unsigned code = 0) {
  unsigned long long t0 = 0;
  unsigned n = 0;
  while (!mbar_try_wait(bar, parity)) {
    if (limit_ns && (++n & 255u) == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t0 == 0) {
        t0 = t;
      } else if (t - t0 > limit_ns) {
        if (dbg) atomicExch(dbg, code);
        __threadfence_system();
        __trap();
      }
    }
  }
}

// One lane of a converged warp (elect.sync): the warp runs the role's loop
// together so descriptors and loop state stay warp-uniform (uniform
// datapath), and the elected lane issues the single-thread tcgen05 / bulk ops.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// The mbarrier tracks every cp.async this thread issued before the call: its
// arrive fires when they have landed (noinc: the arrive counts against the
// barrier's expected count, so every issuing thread is one expected arrival).
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
// Named CTA barriers (ids 1..15; 0 is __syncthreads): the consumers of a
// stage arrive without waiting, the producer that refills it waits.  Used for
// stage release (write-after-read), where compute-sanitizer's racecheck
// models the ordering (it does not model an mbarrier ordering later cp.async
// writes after earlier shared-memory reads).
__device__ __forceinline__ void named_bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
// 1-D bulk copy global -> shared (TMA engine; 16-byte aligned, size a multiple
// of 16), completion as transaction bytes on `bar`.
__device__ __forceinline__ void bulk_copy_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
// Raise the transaction count of the current phase without arriving.
__device__ __forceinline__ void mbar_expect_tx_only(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// 2-D TMA tile load (tensor map in param/global space), completion as
// transaction bytes on `bar`; out-of-range elements are zero-filled.
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int x0, int x1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x0), "r"(x1), "r"(bar)
      : "memory");
}

}  // namespace b2c
