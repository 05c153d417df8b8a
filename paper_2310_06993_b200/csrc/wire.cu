// GPU packetizer for a lossy datagram path (wire.py:36-85,176-208): frames a
// shard's float32 bytes into packets of [9-byte big-endian header | payload]
// and reassembles received packets into a zero-filled shard plus per-entry
// received flags.  One CTA per packet; header fields:
//   bucket_id u16 | byte_offset u32 | timeout_share u8 | flags u8 | reserved u8
// flags bit 0 = last-percentile tag (the final max(1, total/100) packets),
// bits 1-7 = incast advert.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/optr.h"
#include "internal.h"

namespace {

constexpr int kHeader = 9;

__global__ void packetize_kernel(const uint8_t* __restrict__ src, int64_t nbytes, int64_t total, int bucket_id,
                                 uint32_t base, int max_payload, int timeout_share, int incast,
                                 uint8_t* __restrict__ out, int64_t stride) {
  const int64_t k = blockIdx.x;
  if (k >= total) return;
  uint8_t* const p = out + k * stride;
  const int64_t lo = k * max_payload;
  const int64_t len = nbytes - lo < max_payload ? nbytes - lo : max_payload;
  if (threadIdx.x == 0) {
    const uint32_t off = base + (uint32_t)lo;
    const int64_t tagged_from = total - (total / 100 > 1 ? total / 100 : 1);
    p[0] = (uint8_t)(bucket_id >> 8);
    p[1] = (uint8_t)bucket_id;
    p[2] = (uint8_t)(off >> 24);
    p[3] = (uint8_t)(off >> 16);
    p[4] = (uint8_t)(off >> 8);
    p[5] = (uint8_t)off;
    p[6] = (uint8_t)timeout_share;
    p[7] = (uint8_t)((k >= tagged_from ? 1 : 0) | (incast << 1));
    p[8] = 0;
  }
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) p[kHeader + i] = src[lo + i];
}

// errors[0]: packets with a bad header (reserved byte, bucket, offset range)
__global__ void depacketize_kernel(const uint8_t* __restrict__ in, int64_t npk, int64_t stride,
                                   const uint8_t* __restrict__ delivered, int bucket_id, uint32_t base,
                                   int max_payload, uint8_t* __restrict__ dst, uint8_t* __restrict__ mask,
                                   int64_t nbytes, unsigned int* errors) {
  const int64_t k = blockIdx.x;
  if (k >= npk || (delivered && !delivered[k])) return;
  const uint8_t* const p = in + k * stride;
  const int bid = (p[0] << 8) | p[1];
  const uint32_t off = ((uint32_t)p[2] << 24) | ((uint32_t)p[3] << 16) | ((uint32_t)p[4] << 8) | p[5];
  const int64_t rel = (int64_t)off - (int64_t)base;
  if (p[8] != 0 || bid != bucket_id || rel < 0 || rel >= nbytes || (rel % 4) != 0) {
    if (threadIdx.x == 0) atomicAdd(errors, 1u);
    return;
  }
  const int64_t len = nbytes - rel < max_payload ? nbytes - rel : max_payload;
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) dst[rel + i] = p[kHeader + i];
  for (int64_t e = threadIdx.x; e < len / 4; e += blockDim.x) mask[rel / 4 + e] = 1;
}

}  // namespace

extern "C" {

int optr_packetize(const float* shard, int64_t n_entries, int bucket_id, uint32_t base_byte_offset,
                   int max_payload, int timeout_share, int incast, uint8_t* packets, int64_t stride,
                   void* stream) {
  if (n_entries < 0 || max_payload <= 0 || (max_payload & 3) || stride < kHeader + max_payload) return OPTR_EINVAL;
  if (bucket_id < 0 || bucket_id > 0xFFFF || timeout_share < 0 || timeout_share > 0xFF || incast < 0 || incast > 127)
    return OPTR_EINVAL;  // wire.py:44-53 HeaderError
  const int64_t nbytes = n_entries * 4;
  if ((uint64_t)base_byte_offset + (uint64_t)nbytes > 0x100000000ULL) return OPTR_EINVAL;
  if (n_entries == 0) return OPTR_OK;
  if (!shard || !packets) return OPTR_EINVAL;
  optr_bind_stream_device(stream);
  const int64_t total = (nbytes + max_payload - 1) / max_payload;  // wire.py:176-180
  packetize_kernel<<<(unsigned)total, 128, 0, (cudaStream_t)stream>>>((const uint8_t*)shard, nbytes, total, bucket_id,
                                                                      base_byte_offset, max_payload, timeout_share,
                                                                      incast, packets, stride);
  optr_note_launches(1);
  return cudaGetLastError() == cudaSuccess ? OPTR_OK : OPTR_ECUDA;
}

int optr_depacketize(const uint8_t* packets, int64_t n_packets, int64_t stride, const uint8_t* delivered,
                     int bucket_id, uint32_t base_byte_offset, int max_payload, float* shard_out,
                     uint8_t* mask_out, int64_t n_entries, unsigned int* errors, void* stream) {
  if (n_packets < 0 || n_entries < 0 || max_payload <= 0 || (max_payload & 3) || stride < kHeader + max_payload ||
      !errors)
    return OPTR_EINVAL;
  if (n_entries > 0 && (!shard_out || !mask_out)) return OPTR_EINVAL;
  optr_bind_stream_device(stream);
  cudaStream_t st = (cudaStream_t)stream;
  if (n_entries > 0) {
    if (cudaMemsetAsync(shard_out, 0, (size_t)n_entries * 4, st) != cudaSuccess ||
        cudaMemsetAsync(mask_out, 0, (size_t)n_entries, st) != cudaSuccess)
      return OPTR_ECUDA;
  }
  if (n_packets == 0) return OPTR_OK;
  if (!packets) return OPTR_EINVAL;
  depacketize_kernel<<<(unsigned)n_packets, 128, 0, st>>>(packets, n_packets, stride, delivered, bucket_id,
                                                          base_byte_offset, max_payload, (uint8_t*)shard_out,
                                                          mask_out, n_entries * 4, errors);
  optr_note_launches(1);
  return cudaGetLastError() == cudaSuccess ? OPTR_OK : OPTR_ECUDA;
}

}  // extern "C"
