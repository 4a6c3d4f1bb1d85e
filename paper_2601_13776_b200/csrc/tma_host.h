// Host-side TMA tensor-map construction (cuTensorMapEncodeTiled obtained
// through the runtime's driver entry point, so no libcuda link is needed).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

namespace orth {

inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 3-D map over the BF16 GEMM-layout conv kernel (C_o, k*k, C_i/g): box = 64
// channels x 1 tap x `rows` output channels, SWIZZLE_128B, OOB -> 0.  The box
// lands in shared memory exactly as a K-major SW128 UMMA operand tile.
inline bool make_weight_tmap(CUtensorMap* out, const void* w, int co_f, int taps, int ci_g, int rows) {
  using Key = std::tuple<const void*, int, int, int, int>;
  static std::map<Key, CUtensorMap> cache;
  static std::mutex mu;
  const Key key{w, co_f, taps, ci_g, rows};
  {
    std::lock_guard<std::mutex> lk(mu);
    auto itc = cache.find(key);
    if (itc != cache.end()) {
      *out = itc->second;
      return true;
    }
  }
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)ci_g, (cuuint64_t)taps, (cuuint64_t)co_f};
  const cuuint64_t strides[2] = {(cuuint64_t)ci_g * 2, (cuuint64_t)taps * ci_g * 2};
  const cuuint32_t box[3] = {64, 1, (cuuint32_t)rows};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(w), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = m;
  *out = m;
  return true;
}

}  // namespace orth
