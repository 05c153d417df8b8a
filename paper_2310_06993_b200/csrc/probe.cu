// NVLink / HBM bandwidth probes (measurement only, not on the hot path):
// a grid-stride float4 copy run with a peer pointer as source (SM pull over
// NVLink), as destination (SM push), or both local (HBM copy).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/optr.h"

namespace {
__global__ void probe_copy_kernel(float4* __restrict__ dst, const float4* __restrict__ src, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
}  // namespace

extern "C" {

int optr_probe_enable_peer(int device, int peer) {
  if (cudaSetDevice(device) != cudaSuccess) return OPTR_ECUDA;
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return OPTR_ECUDA;
  cudaGetLastError();
  return OPTR_OK;
}

int optr_probe_copy(void* dst, const void* src, int64_t bytes, int blocks, int device, void* stream) {
  if (!dst || !src || bytes <= 0 || (bytes & 15) || blocks <= 0) return OPTR_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return OPTR_ECUDA;
  probe_copy_kernel<<<blocks, 512, 0, (cudaStream_t)stream>>>((float4*)dst, (const float4*)src, bytes / 16);
  return cudaGetLastError() == cudaSuccess ? OPTR_OK : OPTR_ECUDA;
}

}  // extern "C"
