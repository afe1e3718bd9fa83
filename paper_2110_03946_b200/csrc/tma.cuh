// Tensor Memory Accelerator helpers (sm_100a): a 3-D tensor map over a planar
// [C][H][W] image, one bulk tile copy per CTA into shared memory, completion
// through an mbarrier transaction count.  Out-of-image elements of a box
// (negative or past-the-end coordinates) arrive as zeros, which is exactly
// the zero ghost ring the stencils need.
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace sib {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)),
               "r"(bytes));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity));
}

// Box at (x, y, c) of the map into dst (128-byte aligned shared memory).
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int c,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(c), "r"(smem_addr(bar))
      : "memory");
}

// Box at (x, y) of a 2-D map into dst.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_addr(bar))
      : "memory");
}

}  // namespace sib

// ---- Tensor memory (TMEM) as a register-file extension ---------------------
// The sweep keeps one CG vector (x: 16 doubles per thread) in TMEM instead of
// registers: 32 columns per CTA, warp w addresses TMEM lanes 32w..32w+31
// (its sub-partition), thread t of the warp lane 32w+t, so a thread's 16
// doubles are columns 0..31 of its own lane.  One warp allocates (and later
// frees) the columns; tcgen05.ld/st move 32 columns per instruction.
namespace sib {

// Warp 0 allocates COLS columns (a power of two >= 32); every thread returns
// the base address after the fence / barrier / fence handshake.  `slot` is a
// shared word.
template <uint32_t COLS>
__device__ __forceinline__ uint32_t tmem_alloc_cta(uint32_t* slot) {
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_addr(slot)),
                 "n"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  return *reinterpret_cast<volatile uint32_t*>(slot);
}

// Every thread is done with the columns (caller synchronised the CTA).
template <uint32_t COLS>
__device__ __forceinline__ void tmem_free_cta(uint32_t base) {
  if ((threadIdx.x >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base),
                 "n"(COLS));
}

// This warp's lane quarter of the allocation.
__device__ __forceinline__ uint32_t tmem_warp_addr(uint32_t base) {
  return base + ((static_cast<uint32_t>(threadIdx.x >> 5) * 32u) << 16);
}

// 16 doubles <-> 32 columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_store16(uint32_t taddr, const double (&v)[16]) {
  uint32_t w[32];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    w[2 * i] = static_cast<uint32_t>(__double2loint(v[i]));
    w[2 * i + 1] = static_cast<uint32_t>(__double2hiint(v[i]));
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
      "%29, %30, %31, %32};\n" ::"r"(taddr),
      "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
      "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]),
      "r"(w[15]), "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19]), "r"(w[20]), "r"(w[21]),
      "r"(w[22]), "r"(w[23]), "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]), "r"(w[28]),
      "r"(w[29]), "r"(w[30]), "r"(w[31])
      : "memory");
}

__device__ __forceinline__ void tmem_load16(uint32_t taddr, double (&v)[16]) {
  uint32_t w[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
      "%29, %30, %31}, [%32];\n"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
        "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]),
        "=r"(w[14]), "=r"(w[15]), "=r"(w[16]), "=r"(w[17]), "=r"(w[18]), "=r"(w[19]),
        "=r"(w[20]), "=r"(w[21]), "=r"(w[22]), "=r"(w[23]), "=r"(w[24]), "=r"(w[25]),
        "=r"(w[26]), "=r"(w[27]), "=r"(w[28]), "=r"(w[29]), "=r"(w[30]), "=r"(w[31])
      : "r"(taddr)
      : "memory");
  // the wait "rewrites" the registers so no use is scheduled above it
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]),
                 "+r"(w[6]), "+r"(w[7]), "+r"(w[8]), "+r"(w[9]), "+r"(w[10]), "+r"(w[11]),
                 "+r"(w[12]), "+r"(w[13]), "+r"(w[14]), "+r"(w[15]), "+r"(w[16]), "+r"(w[17]),
                 "+r"(w[18]), "+r"(w[19]), "+r"(w[20]), "+r"(w[21]), "+r"(w[22]), "+r"(w[23]),
                 "+r"(w[24]), "+r"(w[25]), "+r"(w[26]), "+r"(w[27]), "+r"(w[28]), "+r"(w[29]),
                 "+r"(w[30]), "+r"(w[31])
               :
               : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i)
    v[i] = __hiloint2double(static_cast<int>(w[2 * i + 1]), static_cast<int>(w[2 * i]));
}

// 4 doubles <-> 8 columns.
__device__ __forceinline__ void tmem_store4(uint32_t taddr, const double (&v)[4]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(
          taddr),
      "r"(__double2loint(v[0])), "r"(__double2hiint(v[0])), "r"(__double2loint(v[1])),
      "r"(__double2hiint(v[1])), "r"(__double2loint(v[2])), "r"(__double2hiint(v[2])),
      "r"(__double2loint(v[3])), "r"(__double2hiint(v[3]))
      : "memory");
}

// Stores issued by this thread have landed (before re-reading the columns).
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}

}  // namespace sib
