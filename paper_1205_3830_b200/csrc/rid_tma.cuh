// rid_tma.cuh — mbarrier and TMA (cp.async.bulk.tensor) building blocks shared by the kernels
// that stream operands with the Tensor Memory Accelerator (k_qrcp.cu: the QR column pass;
// k_zgemm3m_tma.cu: the sketch). PTX only; host side: the driver's cuTensorMapEncodeTiled.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

namespace rid {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
// make the mbarrier inits visible to the async proxy (TMA complete_tx) and the other threads
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
// Order this thread's generic-proxy accesses to shared memory (the LDS of a consumed stage)
// before later async-proxy (TMA) writes to the same bytes: every consumer thread executes it
// before its warp releases a ring slot (WAR across proxies; without it a refill was measured to
// land under a lagging warp's reads, rarely: 1 in ~6 runs of one generation shape).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// L2 prefetch of `bytes` (a multiple of 16) contiguous bytes by the bulk-copy engine: no shared
// memory, no load-store-unit slots
__device__ __forceinline__ void bulk_prefetch_l2(const void* gmem, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// one 2D box (x = inner coordinate in elements, y = outer) into shared memory; completion is
// counted in bytes on the mbarrier b (out-of-bounds elements are zero-filled and counted)
__device__ __forceinline__ void tma_box_g2s(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(b))
      : "memory");
}
// the same with an L2 eviction-priority policy (createpolicy) for the box's lines
__device__ __forceinline__ void tma_box_g2s_hint(void* dst, const CUtensorMap* map, int x, int y,
                                                 uint64_t* b, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(b)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}

// host: the driver's tensor-map encoder (resolved once through the runtime)
inline cudaError_t tensor_map_encoder(PFN_cuTensorMapEncodeTiled* out) {
  static PFN_cuTensorMapEncodeTiled encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult qr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode,
                                            cudaEnableDefault, &qr);
    if (e != cudaSuccess) return e;
    if (qr != cudaDriverEntryPointSuccess || !encode) return cudaErrorSymbolNotFound;
  }
  *out = encode;
  return cudaSuccess;
}

}  // namespace rid
