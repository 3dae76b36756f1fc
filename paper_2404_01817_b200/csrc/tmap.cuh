// Host-side TMA descriptor encoding (cuTensorMapEncodeTiled resolved through
// the runtime's driver entry point: no link against libcuda, no cached state).
#pragma once

#include <cuda.h>          // CUtensorMap (types only)
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled
#include <cuda_runtime.h>

namespace tneat {

inline PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q) !=
          cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return encode;
}

}  // namespace tneat
