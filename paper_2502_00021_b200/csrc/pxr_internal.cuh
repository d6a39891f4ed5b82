// Shared helpers of the libpxr translation units: status/error plumbing for
// the C ABI and the sm_100a bulk-copy (TMA 1-D) primitives.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/pxr.h"

// PXR_DCHECK: bounds / invariant checks of the kernels, compiled in only for
// the checked build (libpxr_checked.so, -DPXR_CHECKED; make checked). A
// failed check prints the condition and traps, so the launch fails loudly;
// tests/test_gpu_checked.py runs the fuzz and overflow cases through it.
#ifdef PXR_CHECKED
#include <cstdio>
#define PXR_DCHECK(cond)                                                            \
  do {                                                                              \
    if (!(cond)) {                                                                  \
      printf("PXR_DCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x, #cond);                             \
      __trap();                                                                     \
    }                                                                               \
  } while (0)
#else
#define PXR_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

namespace pxr {

void set_last_error(const char *msg);

inline pxr_status set_invalid(const char *msg) {
  set_last_error(msg);
  return PXR_ERR_INVALID;
}
inline pxr_status set_unsupported(const char *msg) {
  set_last_error(msg);
  return PXR_ERR_UNSUPPORTED;
}
pxr_status set_cuda(cudaError_t e, const char *where);

// Debug / test knobs (forced raster budgets, row bands, physics variant,
// workload counters). Read from the PXR_DEBUG_* environment once, at the
// first query; pxr_set_debug() changes them at run time (the tests). Never
// consulted per element: the launch paths read them once per call.
enum DebugKnob {
  kDbgFragLimit,     // PXR_DEBUG_FRAG_LIMIT: fragment list limit
  kDbgRowCap,        // PXR_DEBUG_ROW_CAP: bbox rows per raster round
  kDbgCap,           // PXR_DEBUG_CAP: live-triangle records per round
  kDbgStatsPtr,      // PXR_DEBUG_STATS_PTR: device int32 workload counters
  kDbgBandH,         // PXR_DEBUG_BAND_H: rows per band
  kDbgNoPackedScan,  // PXR_DEBUG_NO_PACKED_SCAN: two-scan block scan
  kDbgPhys,          // PXR_DEBUG_PHYS: warp|half|quarter|thread physics kernel
  kDbgGrid,          // PXR_DEBUG_GRID: at most this many CTAs (several envs per CTA)
  kDbgProf,          // PXR_DEBUG_PROF: device int64 (grid, 12) per-CTA phase cycles
  kDbgNoUpscale,     // PXR_DEBUG_NO_UPSCALE: gather video texels even with an upscaled pack
  kDbgNoPdl,         // PXR_DEBUG_NO_PDL: launch the render kernel without programmatic dependent launch
  kDbgNoSplit,       // PXR_DEBUG_NO_SPLIT: small batches keep one CTA per env
  kDbgCount
};
// value of a knob, or nullptr when unset
const char *debug_knob(int id);
inline int64_t debug_int(int id, int64_t dflt) {
  const char *s = debug_knob(id);
  return s != nullptr ? (int64_t)strtoll(s, nullptr, 0) : dflt;
}

// Per-device launch facts, queried once per device: SM count and the opt-in
// shared memory per block.
struct DeviceFacts {
  int device, num_sms, max_smem_optin;
};
const DeviceFacts &device_facts();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) + occupancy query for
// (kernel, device, smem), cached: the first launch of a configuration pays
// for the driver calls, later launches only look the answer up.
pxr_status kernel_occupancy(const void *kernel, int threads, int smem, int *per_sm);

inline pxr_status check_launch(const char *where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda(e, where);
  return PXR_OK;
}

// Programmatic dependent launch trigger: a kernel that may precede the
// render launch lets it be scheduled early (its CTAs then wait in
// griddepcontrol.wait for this grid to complete and flush, so the trigger's
// position does not matter for correctness). No-op without a PDL dependent.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- TMA bulk (non-tensor) copies, shared::cta -> global -----------------

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// One thread's shared-memory atomic add, returning the old value. atomicAdd
// would be wrapped in the compiler's warp aggregation (vote, leader, shuffle:
// ~12 instructions and a lane-id read on the critical path) even where a
// single lane issues it.
__device__ __forceinline__ int smem_atomic_add(int *p, int v) {
  int old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
  return old;
}

// Make generic-proxy smem writes visible to the async (TMA) proxy.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void bulk_store_s2g(void *gdst, const void *ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :
               : "l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// Wait until all committed bulk stores have finished READING shared memory.
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// Wait until all committed bulk stores are complete.
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---- mbarrier + TMA bulk load, global -> shared::cta ----------------------

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// 1-D bulk copy global -> this CTA's shared memory, completing on `bar`.
__device__ __forceinline__ void bulk_load_g2s(void *sdst, const void *gsrc, uint32_t bytes,
                                              uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

}  // namespace pxr
