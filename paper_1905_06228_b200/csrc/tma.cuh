// TMA (cp.async.bulk.tensor) staging of 2D image regions into shared memory:
// host-side tensor-map encoding through the driver entry point (no -lcuda),
// device-side mbarrier + bulk-tensor load helpers. Out-of-image box elements
// are zero-filled by the copy engine, which is exactly the staging semantics
// of the refinement kernels (zero outside the image).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>

namespace dicb200 {

// Two tensor maps (reference, target) passed as one __grid_constant__ kernel parameter.
struct alignas(64) TmaPair {
  CUtensorMap ref;
  CUtensorMap tgt;
  CUtensorMap aux;  // pre-converted refinement staging: the reference's 2 grad image
};

// 2D tiled map over a dense fp32 (elem 4) or 8-byte (float2, elem 8) image
// with box box_w x box_h; zero fill outside. false: layout rules not met.
inline bool tma_encode_2d_f(CUtensorMap* map, const void* base, int elem_bytes, int width, int height, int pitch,
                            int box_w, int box_h) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) return false;
  const uint64_t stride = (uint64_t)pitch * elem_bytes;
  if (((uintptr_t)base & 15) || (stride & 15) || ((box_w * elem_bytes) & 15) || box_w > 256 || box_h > 256)
    return false;
  const cuuint64_t dims[2] = {(cuuint64_t)width, (cuuint64_t)height};
  const cuuint64_t strides[1] = {stride};
  const cuuint32_t box[2] = {(cuuint32_t)box_w, (cuuint32_t)box_h};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT64, 2,
                const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2D tiled map over a u8/u16 image (width x height, pitch in elements) with box
// box_w x box_h. false: the image does not meet TMA's layout rules (16-byte
// aligned base and row pitch, box_w * elem a multiple of 16 bytes) or the
// driver entry point is unavailable -> callers stage without TMA.
inline bool tma_encode_2d(CUtensorMap* map, const void* base, int elem_bytes, int width, int height, int pitch,
                          int box_w, int box_h) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) return false;
  const uint64_t stride = (uint64_t)pitch * elem_bytes;
  if (((uintptr_t)base & 15) || (stride & 15) || ((box_w * elem_bytes) & 15) || box_w > 256 || box_h > 256)
    return false;
  const cuuint64_t dims[2] = {(cuuint64_t)width, (cuuint64_t)height};
  const cuuint64_t strides[1] = {stride};
  const cuuint32_t box[2] = {(cuuint32_t)box_w, (cuuint32_t)box_h};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, elem_bytes == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 2,
                const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

#if defined(__CUDACC__)
__device__ __forceinline__ uint32_t tma_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tma_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(tma_smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void tma_mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(tma_smem_u32(bar)), "r"(bytes)
               : "memory");
}

// Box of `map` with its top-left element at (x, y) (may lie outside the image:
// zero fill) -> shared memory dst (16-byte aligned), completing on `bar`.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          tma_smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(tma_smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(tma_smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
#endif

}  // namespace dicb200
