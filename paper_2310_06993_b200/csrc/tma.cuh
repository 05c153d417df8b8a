// TMA-pipelined strided FWHT pass (sm_100a).
//
// The strided pass transforms index bits [LO, LO+KS) of a vector; its tile is
// 2^KS rows x 8 columns (32-byte row segments, rows 2^LO entries apart).
// Through the LSU each warp load of such a tile touches 16 cache lines, so the
// pass is L1-bound even on L2-resident data.  Here the tile moves with TMA
// tensor copies instead (8 x 256 boxes, cp.async.bulk.tensor), double
// buffered through shared memory with mbarrier completion, and is written
// back with TMA tensor stores:
//
//   thread 0 : load tile k+1 (after the store of tile k-1 has read its
//              buffer), then store tile k after the CTA has transformed it;
//   all      : wait full[k&1] -> registers (round A) -> padded work buffer
//              rounds B, C -> dense buffer -> fence.proxy.async -> store.
//
// The gather variant reads each box from the owning worker's aggregate shard
// (TAR stage-2 receive, collectives.py:140-150) and applies the stage-2 mask
// after the load.
#pragma once
#include <cuda.h>

#include "kernels.cuh"

namespace optr {

struct TmaMaps {
  CUtensorMap m[kMaxW];
};

struct TmaStridedArgs {
  int64_t ntiles;
  int lo;        // first transformed bit (row stride 2^lo entries)
  int outer_sh;  // log2(rows * 2^lo): outer block stride
  int box_rows;  // rows per TMA box (<= 256)
  float scale;   // applied to the result (1/sqrt(D) on the last encode pass)
  // gather variant
  int q, n, r;
  int shard_shift;  // log2(entries per shard) (equal power-of-two shards)
  MaskView m;
  uint8_t* got;
  int64_t dim;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
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
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(dst)), "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   (uint64_t)map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int T>
constexpr size_t tma_smem_bytes() {
  return (size_t)2 * (sizeof(float) << T) + sizeof(float) * ((size_t)pad(1 << T) + 8) + 64 + 1024;
}

// Issue the TMA loads of tile t into `buf`.
template <int T, bool GATHER>
__device__ __forceinline__ void tma_issue_load(const TmaMaps& src, const TmaStridedArgs& a, int64_t t, float* buf,
                                               uint64_t* bar) {
  constexpr int KS = T - 3;
  const int cgb = a.lo - 3;
  const int c0 = (int)((t & ((1LL << cgb) - 1)) << 3);
  const int outer = (int)(t >> cgb);
  const int nbox = (1 << KS) / a.box_rows;
  mbar_expect_tx(bar, (uint32_t)(sizeof(float) << T));
  for (int b = 0; b < nbox; ++b) {
    const int row = b * a.box_rows;
    float* dst = buf + (size_t)row * 8;
    if (GATHER) {
      // rows are global (outer == 0): shard j holds rows [j*2^(shift-lo), ...)
      const int rsh = a.shard_shift - a.lo;
      const int j = row >> rsh;
      const int owner = shard_owner(j, a.r, a.n);
      tma_load_3d(dst, &src.m[owner], bar, c0, row - (j << rsh), 0);
    } else {
      tma_load_3d(dst, &src.m[0], bar, c0, row, outer);
    }
  }
}

template <int T, bool GATHER>
__global__ void __launch_bounds__(1 << (T - 5)) tma_strided_kernel(const __grid_constant__ TmaMaps src,
                                                                 const __grid_constant__ CUtensorMap dst,
                                                                 const __grid_constant__ TmaStridedArgs a) {
  constexpr int CB = 3;
  constexpr RPlan P = make_rplan(T, CB);
  constexpr int NR = P.nr;
  static_assert(NR == 3, "strided TMA kernel expects three register rounds");
  static_assert(P.pos[0][0] == 0 && P.pos[0][1] == 1, "round A holds float4 columns");
  extern __shared__ unsigned char smraw[];
  // 1024-byte aligned base for the TMA buffers
  unsigned char* base = (unsigned char*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  float* const stage0 = (float*)base;
  float* work = (float*)base + 2 * (1 << T);
  uint64_t* full = (uint64_t*)(work + pad(1 << T) + 8);

  const int tid = threadIdx.x;
  const int b0 = thread_base<T>(P, 0, tid);
  const int b1 = thread_base<T>(P, 1, tid);
  const int b2 = thread_base<T>(P, 2, tid);
  float* const w0 = work + pad(b0);
  float* const w1 = work + pad(b1);
  float* const w2 = work + pad(b2);

  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t stride = gridDim.x;
  int64_t t = blockIdx.x;
  if (tid == 0) {
    if (t < a.ntiles) tma_issue_load<T, GATHER>(src, a, t, stage0, &full[0]);
    if (t + stride < a.ntiles) tma_issue_load<T, GATHER>(src, a, t + stride, stage0 + (1 << T), &full[1]);
  }
  const int cgb = a.lo - 3;
  for (int k = 0; t < a.ntiles; ++k, t += stride) {
    const int buf = k & 1;
    if (tid == 0 && k >= 1 && t + stride < a.ntiles) {
      bulk_wait_read0();  // the store of tile k-1 has read stage[buf^1]
      tma_issue_load<T, GATHER>(src, a, t + stride, stage0 + ((buf ^ 1) << T), &full[buf ^ 1]);
    }
    mbar_wait(&full[buf], (uint32_t)((k >> 1) & 1));
    float* sb = stage0 + (buf << T);
    float v[32];
    // round A: dense tile, float4 per (row, 4 columns)
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const int i = b0 + roff(P, 0, 4 * m);
      float4 q4 = *reinterpret_cast<const float4*>(sb + i);
      if (GATHER) {
        const int64_t c0 = (t & ((1LL << cgb) - 1)) << 3;
        const int64_t g = ((int64_t)(i >> 3) << a.lo) + c0 + (i & 7);
        const int j = (int)(g >> a.shard_shift);
        const uint32_t e = (uint32_t)(g - ((int64_t)j << a.shard_shift));
        const int owner = shard_owner(j, a.r, a.n);
        if (owner != a.q) {
          const uint32_t* row = a.m.row(1, a.q, owner);
          const Pkt4 pk = pkt4(e, (uint32_t)a.m.epp);
          const bool k0 = row_bit(row, pk.p[0]), k1 = row_bit(row, pk.p[1]);
          const bool k2 = row_bit(row, pk.p[2]), k3 = row_bit(row, pk.p[3]);
          q4.x = k0 ? q4.x : 0.f;
          q4.y = k1 ? q4.y : 0.f;
          q4.z = k2 ? q4.z : 0.f;
          q4.w = k3 ? q4.w : 0.f;
          if (a.got) *reinterpret_cast<uchar4*>(a.got + g) = make_uchar4(k0, k1, k2, k3);
        } else if (a.got) {
          *reinterpret_cast<uchar4*>(a.got + g) = make_uchar4(1, 1, 1, 1);
        }
      }
      v[4 * m] = q4.x;
      v[4 * m + 1] = q4.y;
      v[4 * m + 2] = q4.z;
      v[4 * m + 3] = q4.w;
    }
    bfly32<P.xm[0]>(v);
#pragma unroll
    for (int j = 0; j < 32; ++j) w0[pad(roff(P, 0, j))] = v[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = w1[pad(roff(P, 1, j))];
    bfly32<P.xm[1]>(v);
#pragma unroll
    for (int j = 0; j < 32; ++j) w1[pad(roff(P, 1, j))] = v[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = w2[pad(roff(P, 2, j))];
    bfly32<P.xm[2]>(v);
    // back to the dense buffer (every thread finished reading it before the
    // first __syncthreads above)
    const float s = a.scale;
    if constexpr (P.pos[2][0] == 0 && P.pos[2][1] == 1) {
#pragma unroll
      for (int m = 0; m < 8; ++m)
        *reinterpret_cast<float4*>(sb + b2 + roff(P, 2, 4 * m)) =
            make_float4(v[4 * m] * s, v[4 * m + 1] * s, v[4 * m + 2] * s, v[4 * m + 3] * s);
    } else if constexpr (P.pos[2][0] == 0) {
#pragma unroll
      for (int m = 0; m < 16; ++m)
        *reinterpret_cast<float2*>(sb + b2 + roff(P, 2, 2 * m)) = make_float2(v[2 * m] * s, v[2 * m + 1] * s);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) sb[b2 + roff(P, 2, j)] = v[j] * s;
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      constexpr int KS = T - 3;
      const int c0 = (int)((t & ((1LL << cgb) - 1)) << 3);
      const int outer = GATHER ? 0 : (int)(t >> cgb);
      const int nbox = (1 << KS) / a.box_rows;
      for (int b = 0; b < nbox; ++b) tma_store_3d(&dst, sb + (size_t)b * a.box_rows * 8, c0, b * a.box_rows, outer);
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait0();
}

}  // namespace optr

namespace optr {

// ------------------------------------------------ TMA contiguous pass
// Tiles are 2^T contiguous entries.  Loads are 1D bulk copies
// (cp.async.bulk) into a two-stage shared-memory ring; the source transform
// (encode: pad + signs + bf16 upcast; gather: owner shard + stage-2 mask) is
// applied when the tile is read out of shared memory; results are stored
// with vector STG (each warp writes 512 contiguous bytes).
enum ContigSrc { CS_BUF = 0, CS_ENC = 1, CS_GATHER = 2 };

struct TmaContigArgs {
  int64_t ntiles;
  // CS_BUF / CS_ENC: source vector (fp32, or x of dtype_in for CS_ENC)
  const void* x;
  int dtype;
  int64_t L;              // CS_ENC: entries of x (the rest of the tile is padding)
  const uint32_t* signs;  // CS_ENC
  // CS_GATHER (collectives.py:140-150)
  const float* A[kMaxW];
  int q, n, r;
  int shard_shift;  // equal power-of-two shards of 2^shard_shift >= 2^T entries
  MaskView m;
  uint8_t* got;  // optional, already offset to worker q
};

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int T, int SK>
__device__ __forceinline__ void contig_issue(const TmaContigArgs& a, int64_t t, unsigned char* stage, uint32_t* sgn,
                                             uint64_t* bar) {
  const int64_t g0 = t << T;
  if (SK == CS_GATHER) {
    const int j = (int)(g0 >> a.shard_shift);
    const int owner = shard_owner(j, a.r, a.n);
    const int64_t e0 = g0 - ((int64_t)j << a.shard_shift);
    mbar_expect_tx(bar, (uint32_t)(sizeof(float) << T));
    bulk_load(stage, a.A[owner] + e0, (uint32_t)(sizeof(float) << T), bar);
    return;
  }
  if (SK == CS_BUF) {
    mbar_expect_tx(bar, (uint32_t)(sizeof(float) << T));
    bulk_load(stage, (const float*)a.x + g0, (uint32_t)(sizeof(float) << T), bar);
    return;
  }
  // CS_ENC: the valid part of x (16-byte multiple) and the tile's sign words
  const int esz = a.dtype == OPTR_BF16 ? 2 : 4;
  int64_t valid = a.L - g0;
  if (valid > (1 << T)) valid = 1 << T;
  if (valid < 0) valid = 0;
  uint32_t bytes = (uint32_t)((valid * esz) & ~15LL);
  const uint32_t sbytes = (uint32_t)(sizeof(uint32_t) << (T - 5));
  mbar_expect_tx(bar, bytes + sbytes);
  if (bytes) bulk_load(stage, (const unsigned char*)a.x + g0 * esz, bytes, bar);
  bulk_load(sgn, a.signs + (g0 >> 5), sbytes, bar);
}

template <int T>
constexpr size_t tma_contig_smem_bytes() {
  return (size_t)2 * (sizeof(float) << T) + (size_t)2 * (sizeof(uint32_t) << (T - 5)) +
         sizeof(float) * ((size_t)pad(1 << T) + 8) + 64 + 1024;
}

template <int T, int SK, class Snk>
__global__ void __launch_bounds__(1 << (T - 5)) tma_contig_kernel(const __grid_constant__ TmaContigArgs a,
                                                                const __grid_constant__ Snk snk, int worker) {
  constexpr RPlan P = make_rplan(T, 0);
  constexpr int NR = P.nr;
  static_assert(NR == 3, "contiguous TMA kernel expects three register rounds");
  extern __shared__ unsigned char smraw[];
  unsigned char* base = (unsigned char*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  unsigned char* const stage0 = base;
  uint32_t* const sgw0 = (uint32_t*)(base + 2 * (sizeof(float) << T));
  float* work = (float*)(base + 2 * (sizeof(float) << T) + 2 * (sizeof(uint32_t) << (T - 5)));
  uint64_t* full = (uint64_t*)(work + pad(1 << T) + 8);

  const int tid = threadIdx.x;
  const int b0 = thread_base<T>(P, 0, tid);
  const int b1 = thread_base<T>(P, 1, tid);
  const int b2 = thread_base<T>(P, 2, tid);
  float* const w0 = work + pad(b0);
  float* const w1 = work + pad(b1);
  float* const w2 = work + pad(b2);
  const auto d = snk.bind(worker);

  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t stride = gridDim.x;
  int64_t t = blockIdx.x;
  if (tid == 0) {
    if (t < a.ntiles) contig_issue<T, SK>(a, t, stage0, sgw0, &full[0]);
    if (t + stride < a.ntiles)
      contig_issue<T, SK>(a, t + stride, stage0 + (sizeof(float) << T), sgw0 + (1 << (T - 5)), &full[1]);
  }
  for (int k = 0; t < a.ntiles; ++k, t += stride) {
    const int buf = k & 1;
    mbar_wait(&full[buf], (uint32_t)((k >> 1) & 1));
    const int64_t g0 = t << T;
    unsigned char* const sb = stage0 + ((size_t)buf * (sizeof(float) << T));
    const uint32_t* const sw0 = sgw0 + (buf << (T - 5));
    int64_t bulk_end = 0;
    if (SK == CS_ENC) {
      const int lsh = a.dtype == OPTR_BF16 ? 1 : 2;
      bulk_end = g0 + ((((a.L - g0) << lsh) & ~15LL) >> lsh);
    }
    float v[32];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const int i = b0 + roff(P, 0, 4 * m);
      float4 q4;
      if (SK == CS_ENC) {
        const int64_t g = g0 + i;
        if (a.dtype == OPTR_BF16) {
          const uint2 u = *reinterpret_cast<const uint2*>(sb + (size_t)i * 2);
          const float2 fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
          const float2 fb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
          q4 = make_float4(fa.x, fa.y, fb.x, fb.y);
        } else {
          q4 = *reinterpret_cast<const float4*>(sb + (size_t)i * 4);
        }
        if (g + 4 > bulk_end) {  // past the bulk copy: unaligned tail of x, then padding
          float e[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (g + c < a.L) e[c] = load_elem(a.x, a.dtype, g + c);
          q4 = make_float4(e[0], e[1], e[2], e[3]);
        }
        const uint32_t sw = sw0[i >> 5];
        const int bb = i & 31;
        q4.x = sgn(sw, bb, q4.x);
        q4.y = sgn(sw, bb + 1, q4.y);
        q4.z = sgn(sw, bb + 2, q4.z);
        q4.w = sgn(sw, bb + 3, q4.w);
      } else {
        q4 = *reinterpret_cast<const float4*>(sb + (size_t)i * 4);
        if (SK == CS_GATHER) {
          const int64_t g = g0 + i;
          const int j = (int)(g >> a.shard_shift);
          const int owner = shard_owner(j, a.r, a.n);
          const uint32_t e = (uint32_t)(g - ((int64_t)j << a.shard_shift));
          if (owner != a.q) {
            const uint32_t* row = a.m.row(1, a.q, owner);
            const Pkt4 pk = pkt4(e, (uint32_t)a.m.epp);
            const bool k0 = row_bit(row, pk.p[0]), k1 = row_bit(row, pk.p[1]);
            const bool k2 = row_bit(row, pk.p[2]), k3 = row_bit(row, pk.p[3]);
            q4.x = k0 ? q4.x : 0.f;
            q4.y = k1 ? q4.y : 0.f;
            q4.z = k2 ? q4.z : 0.f;
            q4.w = k3 ? q4.w : 0.f;
            if (a.got) *reinterpret_cast<uchar4*>(a.got + g) = make_uchar4(k0, k1, k2, k3);
          } else if (a.got) {
            *reinterpret_cast<uchar4*>(a.got + g) = make_uchar4(1, 1, 1, 1);
          }
        }
      }
      v[4 * m] = q4.x;
      v[4 * m + 1] = q4.y;
      v[4 * m + 2] = q4.z;
      v[4 * m + 3] = q4.w;
    }
    bfly32<P.xm[0]>(v);
#pragma unroll
    for (int j = 0; j < 32; ++j) w0[pad(roff(P, 0, j))] = v[j];
    __syncthreads();  // everyone has read stage[buf]; work holds round A
    if (tid == 0 && t + 2 * stride < a.ntiles)
      contig_issue<T, SK>(a, t + 2 * stride, sb, sgw0 + (buf << (T - 5)), &full[buf]);
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = w1[pad(roff(P, 1, j))];
    bfly32<P.xm[1]>(v);
#pragma unroll
    for (int j = 0; j < 32; ++j) w1[pad(roff(P, 1, j))] = v[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = w2[pad(roff(P, 2, j))];
    bfly32<P.xm[2]>(v);
    if constexpr (P.pos[2][0] == 0 && P.pos[2][1] == 1) {
#pragma unroll
      for (int m = 0; m < 8; ++m)
        d.store4(g0 + b2 + roff(P, 2, 4 * m), make_float4(v[4 * m], v[4 * m + 1], v[4 * m + 2], v[4 * m + 3]));
    } else if constexpr (P.pos[2][0] == 0) {
#pragma unroll
      for (int m = 0; m < 16; ++m) d.store2(g0 + b2 + roff(P, 2, 2 * m), v[2 * m], v[2 * m + 1]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) d.store1(g0 + b2 + roff(P, 2, j), v[j]);
    }
    __syncthreads();  // work is free for the next tile
  }
}

}  // namespace optr
