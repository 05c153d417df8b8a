// Ring all-reduce steps of the sans-IO baseline (collectives.py:248-292):
// the partial sums travel as float32 but accumulate in a float64 buffer,
// exactly as the reference's numpy code does (buf = entries.astype(float64);
// chunk += received; chunk[m] = received[m]; (buf / n).astype(float32)).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/optr.h"
#include "internal.h"

namespace {

constexpr int kThreads = 256;

unsigned grid_for(int64_t n) {
  int64_t b = (n + kThreads - 1) / kThreads;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)(b > 0 ? b : 1);
}

__global__ void cast_kernel(const double* __restrict__ c, int64_t n, float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __double2float_rn(c[i]);
}

// gather == 0: chunk += data (missing entries arrive as 0.0)
// gather == 1: chunk[m] = data[m] (keep the partial value where dropped)
__global__ void step_kernel(double* __restrict__ chunk, const float* __restrict__ data,
                            const uint8_t* __restrict__ mask, int64_t n, int gather) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (gather) {
      if (mask == nullptr || mask[i]) chunk[i] = (double)data[i];
    } else {
      chunk[i] += (double)data[i];
    }
  }
}

__global__ void finish_kernel(const double* __restrict__ buf, double n, int64_t len, float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __double2float_rn(buf[i] / n);
}

int done() { return cudaGetLastError() == cudaSuccess ? OPTR_OK : OPTR_ECUDA; }

}  // namespace

extern "C" {

int optr_ring_cast(const double* chunk, int64_t n, float* out, void* stream) {
  if (n < 0 || (n > 0 && (!chunk || !out))) return OPTR_EINVAL;
  if (n == 0) return OPTR_OK;
  optr_bind_stream_device(stream);
  cast_kernel<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(chunk, n, out);
  optr_note_launches(1);
  return done();
}

int optr_ring_step(double* chunk, const float* data, const uint8_t* mask, int64_t n, int gather, void* stream) {
  if (n < 0 || (n > 0 && (!chunk || !data))) return OPTR_EINVAL;
  if (n == 0) return OPTR_OK;
  optr_bind_stream_device(stream);
  step_kernel<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(chunk, data, mask, n, gather ? 1 : 0);
  optr_note_launches(1);
  return done();
}

int optr_ring_finish(const double* buf, int nodes, int64_t len, float* out, void* stream) {
  if (nodes < 1 || len < 0 || (len > 0 && (!buf || !out))) return OPTR_EINVAL;
  if (len == 0) return OPTR_OK;
  optr_bind_stream_device(stream);
  finish_kernel<<<grid_for(len), kThreads, 0, (cudaStream_t)stream>>>(buf, (double)nodes, len, out);
  optr_note_launches(1);
  return done();
}

}  // extern "C"
