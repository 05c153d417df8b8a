// Float64 RHT codec (hadamard.py:76-123 in the reference's own arithmetic).
//
// The reference transforms numpy float64 arrays with the radix-2 butterfly
// of fwht_in_place, stage h = 1, 2, 4, ... in turn, [a, b] -> [a + b, a - b].
// These kernels apply the same stages in the same order -- K consecutive
// stages per pass, the 2^K values of one butterfly group in registers -- so
// every output is the same sequence of float64 additions and the results are
// bit-identical to the reference's.  Encode multiplies the zero-padded input
// by the +-1 signs first and divides by sqrt(dim) last; decode zero-fills the
// misses, scales by dim / received, transforms, applies the signs and divides
// by sqrt(dim) (hadamard.py:93-123), also in the reference's order.
//
// This is the facade's path for float64 data (numpy arrays, like the
// reference); the TAR hot path runs the float32 tile kernels of tma.cuh.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/optr.h"
#include "internal.h"

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double sign_of(const uint32_t* s, int64_t g) {
  return ((s[g >> 5] >> (g & 31)) & 1u) ? 1.0 : -1.0;
}

// Stages b .. b+K-1 (bits of the index), in increasing order.
template <int K>
__global__ void __launch_bounds__(kThreads) fwht64_pass(double* __restrict__ v, int64_t dim, int b) {
  const int64_t groups = dim >> K;
  for (int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < groups;
       gi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = gi & ((1LL << b) - 1);
    const int64_t base = ((gi >> b) << (b + K)) | lo;
    double r[1 << K];
#pragma unroll
    for (int j = 0; j < (1 << K); ++j) r[j] = v[base + ((int64_t)j << b)];
#pragma unroll
    for (int s = 0; s < K; ++s) {
#pragma unroll
      for (int j = 0; j < (1 << K); ++j) {
        if (!((j >> s) & 1)) {
          const double a = r[j], c = r[j | (1 << s)];
          r[j] = a + c;
          r[j | (1 << s)] = a - c;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < (1 << K); ++j) v[base + ((int64_t)j << b)] = r[j];
  }
}

// padded = zeros(dim); padded[:L] = x; padded * signs   (hadamard.py:98-100)
__global__ void enc_prologue64(const double* __restrict__ x, int64_t L, const uint32_t* __restrict__ signs,
                               double* __restrict__ v, int64_t dim) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < dim; g += (int64_t)gridDim.x * blockDim.x)
    v[g] = (g < L ? x[g] : 0.0) * sign_of(signs, g);
}

// y /= sqrt(dim)   (hadamard.py:101)
__global__ void div64(double* __restrict__ v, int64_t dim, double root) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < dim; g += (int64_t)gridDim.x * blockDim.x)
    v[g] = v[g] / root;
}

// y = where(received, y_recv, 0.0) * scale   (hadamard.py:119-120)
__global__ void dec_prologue64(const double* __restrict__ y, const uint8_t* __restrict__ mask, double scale,
                               double* __restrict__ v, int64_t dim) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < dim; g += (int64_t)gridDim.x * blockDim.x)
    v[g] = ((mask == nullptr || mask[g]) ? y[g] : 0.0) * scale;
}

// x = signs * fwht(y); x /= sqrt(dim); x[:L]   (hadamard.py:121-123)
__global__ void dec_epilogue64(const double* __restrict__ v, const uint32_t* __restrict__ signs, double root,
                               double* __restrict__ out, int64_t L) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < L; g += (int64_t)gridDim.x * blockDim.x)
    out[g] = (sign_of(signs, g) * v[g]) / root;
}

__global__ void count64(const uint8_t* __restrict__ mask, int64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x)
    c += mask[g] ? 1 : 0;
  for (int o = 16; o; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

unsigned grid_for(int64_t items) {
  int64_t b = (items + kThreads - 1) / kThreads;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)(b > 0 ? b : 1);
}

bool pow2(int64_t d) { return d > 0 && (d & (d - 1)) == 0; }

int log2i(int64_t d) {
  int k = 0;
  while ((1LL << k) < d) ++k;
  return k;
}

int fwht64(double* v, int64_t dim, cudaStream_t st) {
  const int k = log2i(dim);
  for (int b = 0; b < k; b += 5) {
    const int K = k - b < 5 ? k - b : 5;
    const unsigned g = grid_for(dim >> K);
    switch (K) {
      case 1: fwht64_pass<1><<<g, kThreads, 0, st>>>(v, dim, b); break;
      case 2: fwht64_pass<2><<<g, kThreads, 0, st>>>(v, dim, b); break;
      case 3: fwht64_pass<3><<<g, kThreads, 0, st>>>(v, dim, b); break;
      case 4: fwht64_pass<4><<<g, kThreads, 0, st>>>(v, dim, b); break;
      default: fwht64_pass<5><<<g, kThreads, 0, st>>>(v, dim, b); break;
    }
    optr_note_launches(1);
  }
  return cudaGetLastError() == cudaSuccess ? OPTR_OK : OPTR_ECUDA;
}

}  // namespace

extern "C" {

int optr_fwht_f64(double* v, int64_t dim, void* stream) {
  if (!pow2(dim) || !v) return OPTR_EINVAL;  // hadamard.py:78-81
  optr_bind_stream_device(stream);
  return fwht64(v, dim, (cudaStream_t)stream);
}

int optr_rht_encode_f64(const double* x, int64_t L, double* y, int64_t dim, uint64_t seed, void* stream) {
  if (!pow2(dim) || L > dim || L < 0 || !y || (L > 0 && !x)) return OPTR_EINVAL;  // hadamard.py:45-48,96-97
  optr_bind_stream_device(stream);
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* signs = nullptr;
  if (cudaMallocAsync((void**)&signs, (size_t)((dim + 31) / 32) * 4 + 16, st) != cudaSuccess) return OPTR_ENOMEM;
  int rc = optr_rht_signs(signs, dim, seed, stream);
  if (!rc) {
    enc_prologue64<<<grid_for(dim), kThreads, 0, st>>>(x, L, signs, y, dim);
    optr_note_launches(1);
    rc = fwht64(y, dim, st);
  }
  if (!rc) {
    div64<<<grid_for(dim), kThreads, 0, st>>>(y, dim, sqrt((double)dim));
    optr_note_launches(1);
    rc = cudaGetLastError() == cudaSuccess ? OPTR_OK : OPTR_ECUDA;
  }
  cudaFreeAsync(signs, st);
  return rc;
}

int optr_rht_decode_f64(const double* y, const uint8_t* mask, int64_t dim, int64_t L, uint64_t seed, double* out,
                        void* stream) {
  if (!pow2(dim) || L > dim || L < 0 || !y || (L > 0 && !out)) return OPTR_EINVAL;
  optr_bind_stream_device(stream);
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long count = (unsigned long long)dim;
  if (mask) {  // DropMask.received_count (hadamard.py:116-118)
    unsigned long long* dc = nullptr;
    if (cudaMallocAsync((void**)&dc, sizeof(*dc), st) != cudaSuccess) return OPTR_ENOMEM;
    cudaMemsetAsync(dc, 0, sizeof(*dc), st);
    count64<<<grid_for(dim), kThreads, 0, st>>>(mask, dim, dc);
    optr_note_launches(1);
    cudaMemcpyAsync(&count, dc, sizeof(count), cudaMemcpyDeviceToHost, st);
    const cudaError_t e = cudaStreamSynchronize(st);
    cudaFreeAsync(dc, st);
    if (e != cudaSuccess) return OPTR_ECUDA;
  }
  if (count == 0) return OPTR_EEMPTY;
  uint32_t* signs = nullptr;
  double* tmp = nullptr;
  if (cudaMallocAsync((void**)&signs, (size_t)((dim + 31) / 32) * 4 + 16, st) != cudaSuccess) return OPTR_ENOMEM;
  if (cudaMallocAsync((void**)&tmp, (size_t)dim * 8, st) != cudaSuccess) {
    cudaFreeAsync(signs, st);
    return OPTR_ENOMEM;
  }
  int rc = optr_rht_signs(signs, dim, seed, stream);
  if (!rc) {
    const double scale = (double)dim / (double)count;  // ctx.dim / received
    dec_prologue64<<<grid_for(dim), kThreads, 0, st>>>(y, mask, scale, tmp, dim);
    optr_note_launches(1);
    rc = fwht64(tmp, dim, st);
  }
  if (!rc && L > 0) {
    dec_epilogue64<<<grid_for(L), kThreads, 0, st>>>(tmp, signs, sqrt((double)dim), out, L);
    optr_note_launches(1);
    rc = cudaGetLastError() == cudaSuccess ? OPTR_OK : OPTR_ECUDA;
  }
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(signs, st);
  return rc;
}

}  // extern "C"
