// TMA-pipelined FWHT passes (sm_100a).
//
// A pass transforms index bits [lo, lo+ks) of a vector in tiles of 2^T
// entries (see kernels.cuh PassGeom).  Tiles stream through a 3-stage
// shared-memory ring per CTA, filled by one elected thread with TMA:
//
//   contiguous pass (lo = 0): one 1D bulk copy (cp.async.bulk) per tile;
//   strided pass (cb = 3): 8 x box_rows tensor boxes (cp.async.bulk.tensor),
//     because through the LSU each warp load of 32-byte row segments touches
//     16 cache lines and the pass is L1-bound even on L2-resident data.
//
// Each tile is transformed in place in its stage buffer: round A reads the
// dense tile (float4), rounds B and C go through an XOR-swizzled copy of the
// same buffer (conflict-free for every layout here), and the result leaves
// either through vector STG (contiguous pass: each warp stores 512 bytes)
// or through TMA tensor stores from the dense buffer (strided pass).  The
// fused source transforms (encode pad/signs/bf16 upcast, TAR stage-2 gather
// with masks) are applied when round A reads the tile.
#pragma once
#include <cuda.h>

#include <type_traits>

#include "kernels.cuh"

namespace optr {


struct TmaMaps {
  CUtensorMap m[kMaxW];
};

enum TileSrc { TS_BUF = 0, TS_ENC = 1, TS_GATHER = 2 };

struct TmaArgs {
  int64_t ntiles;
  int lo;        // strided: first transformed bit (row stride 2^lo entries)
  int box_rows;  // strided: rows per TMA box (<= 256)
  float scale;   // strided sink: result scale
  // TS_BUF / TS_ENC (contiguous): source vector of each worker; TS_ENC: x of
  // `dtype`, L entries
  const void* xw[kMaxW];
  int dtype;
  int64_t L;
  const uint32_t* signs;
  // TS_GATHER (collectives.py:140-150): owner shards, stage-2 masks
  const float* A[kMaxW];
  int n, r;
  int shard_shift;  // equal power-of-two shards of 2^shard_shift entries
  MaskView m;
  uint8_t* got;  // optional [worker][dim]
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
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// XOR-linear swizzle: swzc(b | c) = swzc(b) ^ swzc(c) for disjoint b, c
__host__ __device__ constexpr int swzc(int i) { return i ^ ((i >> 5) & 31); }

// tile + its sign words, rounded to 1 KB so every stage (a TMA destination)
// stays 128-byte aligned
template <int T>
__host__ __device__ constexpr size_t tma_stage_bytes() {
  return ((sizeof(float) << T) + (sizeof(uint32_t) << (T - 5)) + 1023) / 1024 * 1024;
}
template <int T, int S>
__host__ __device__ constexpr size_t tma_smem_bytes() {
  return S * tma_stage_bytes<T>() + 64 + 1024;
}

// Issue the loads of tile t into stage buffer `st` (sign words after the tile).
template <int T, bool STRIDED, int SK, int CBW>
__device__ __forceinline__ void tile_issue(const TmaMaps& maps, const TmaArgs& a, int w, int64_t t,
                                           unsigned char* st, uint64_t* bar) {
  if constexpr (STRIDED) {
    constexpr int KS = T - CBW;
    const int cgb = a.lo - CBW;
    const int c0 = (int)((t & ((1LL << cgb) - 1)) << CBW);
    const int outer = (int)(t >> cgb);
    const int nbox = (1 << KS) / a.box_rows;
    mbar_expect_tx(bar, (uint32_t)(sizeof(float) << T));
    for (int b = 0; b < nbox; ++b) {
      const int row = b * a.box_rows;
      float* dst = (float*)st + ((size_t)row << CBW);
      if (SK == TS_GATHER) {
        const int rsh = a.shard_shift - a.lo;  // rows per shard = 2^rsh (outer == 0)
        const int j = row >> rsh;
        tma_load_3d(dst, &maps.m[shard_owner(j, a.r, a.n)], bar, c0, row - (j << rsh), 0);
      } else {
        tma_load_3d(dst, &maps.m[w], bar, c0, row, outer);
      }
    }
  } else {
    const int64_t g0 = t << T;
    if (SK == TS_GATHER) {
      const int j = (int)(g0 >> a.shard_shift);
      const int64_t e0 = g0 - ((int64_t)j << a.shard_shift);
      mbar_expect_tx(bar, (uint32_t)(sizeof(float) << T));
      bulk_load(st, a.A[shard_owner(j, a.r, a.n)] + e0, (uint32_t)(sizeof(float) << T), bar);
    } else if (SK == TS_BUF) {
      mbar_expect_tx(bar, (uint32_t)(sizeof(float) << T));
      bulk_load(st, (const float*)a.xw[w] + g0, (uint32_t)(sizeof(float) << T), bar);
    } else {
      const int lsh = a.dtype == OPTR_BF16 ? 1 : 2;
      int64_t valid = a.L - g0;
      if (valid > (1 << T)) valid = 1 << T;
      if (valid < 0) valid = 0;
      const uint32_t bytes = (uint32_t)((valid << lsh) & ~15LL);
      const uint32_t sbytes = (uint32_t)(sizeof(uint32_t) << (T - 5));
      mbar_expect_tx(bar, bytes + sbytes);
      if (bytes) bulk_load(st, (const unsigned char*)a.xw[w] + (g0 << lsh), bytes, bar);
      bulk_load(st + (sizeof(float) << T), a.signs + (g0 >> 5), sbytes, bar);
    }
  }
}

// Masked float4 of worker q's stage-2 receive at global index g (4 entries
// inside one shard).
__device__ __forceinline__ float4 gather_mask4(const TmaArgs& a, int q, uint8_t* got, int64_t g, float4 v) {
  const int j = (int)(g >> a.shard_shift);
  const int owner = shard_owner(j, a.r, a.n);
  if (owner == q) {
    if (got) *reinterpret_cast<uchar4*>(got + g) = make_uchar4(1, 1, 1, 1);
    return v;
  }
  const uint32_t e = (uint32_t)(g - ((int64_t)j << a.shard_shift));
  const uint32_t kk = keep4(a.m.row(1, q, owner), e, a.m);
  if (kk == 0xFu) {
    if (got) *reinterpret_cast<uchar4*>(got + g) = make_uchar4(1, 1, 1, 1);
    return v;
  }
  const bool k0 = kk & 1u, k1 = kk & 2u, k2 = kk & 4u, k3 = kk & 8u;
  if (got) *reinterpret_cast<uchar4*>(got + g) = make_uchar4(k0, k1, k2, k3);
  return make_float4(k0 ? v.x : 0.f, k1 ? v.y : 0.f, k2 ? v.z : 0.f, k3 ? v.w : 0.f);
}

// One tile of a TMA pass, from its filled stage buffer `sb` to its issued
// result.  `refill()` is called by thread 0 once the stage may be reused for
// the next load: for a contiguous tile right after the tile has been read
// (the results then leave by STG), for a strided tile after its TMA store
// group is committed (the refill policy decides which stage to wait for).
template <int T, bool STRIDED, int SK, class Snk, int CBW, class Refill>
__device__ __forceinline__ void tma_tile(const TmaMaps& maps, const CUtensorMap& dst, const TmaArgs& a,
                                         const typename Snk::B& d, int worker, uint8_t* gotw, int64_t t,
                                         unsigned char* sb, Refill&& refill) {
  constexpr int CB = STRIDED ? CBW : 0;  // untransformed column bits (8 or 32 columns)
  constexpr int CM = (1 << CB) - 1;
  constexpr RPlan P = make_rplan(T, CB);
  static_assert(P.nr == 2 || P.nr == 3, "TMA pass expects two or three register rounds");
  constexpr int LR = P.nr - 1;  // last round
  static_assert(P.pos[0][0] == 0 && P.pos[0][1] == 1, "round A holds float4 groups");
  static_assert(!STRIDED || !std::is_same<Snk, SnkDecode>::value || (P.pos[LR][0] == 0 && P.pos[LR][1] == 1),
                "decode epilogue stores float4 groups");
  static_assert(sizeof(float) * pad(1 << T) <= tma_stage_bytes<T>(), "padded tile fits the stage");
  const int tid = threadIdx.x;
  const int b0 = thread_base<T>(P, 0, tid);
  const int b1 = thread_base<T>(P, 1, tid);
  const int b2 = thread_base<T>(P, LR, tid);  // last-round base
  const int p0 = pad(b0), p1 = pad(b1), p2 = pad(b2);
  float* const tile = (float*)sb;
  const int cgb = STRIDED ? a.lo - CB : 0;
  // global index of tile element 0
  const int64_t g0 = STRIDED ? (((t >> cgb) << (a.lo + T - CB)) + ((t & ((1LL << cgb) - 1)) << CB)) : (t << T);
  float v[32];
  // ---- round A: dense tile, float4 groups, fused source transform
  int64_t bulk_end = 0;
  bool enc_fast = true;
  if constexpr (SK == TS_ENC) {
    const int lsh = a.dtype == OPTR_BF16 ? 1 : 2;
    bulk_end = g0 + ((((a.L - g0) << lsh) & ~15LL) >> lsh);
    enc_fast = g0 + (1 << T) <= bulk_end;
  }
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const int i = b0 + roff(P, 0, 4 * m);
    const int64_t g = STRIDED ? (g0 + ((int64_t)(i >> CB) << a.lo) + (i & CM)) : (g0 + i);
    float4 q4;
    if constexpr (SK == TS_ENC) {
      if (a.dtype == OPTR_BF16) {
        const uint2 u = *reinterpret_cast<const uint2*>(sb + (size_t)i * 2);
        const float2 fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
        const float2 fb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
        q4 = make_float4(fa.x, fa.y, fb.x, fb.y);
      } else {
        q4 = *reinterpret_cast<const float4*>(tile + i);
      }
      if (!enc_fast && g + 4 > bulk_end) {  // past the bulk copy: unaligned tail of x, then padding
        float e[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (g + c < a.L) e[c] = load_elem(a.xw[worker], a.dtype, g + c);
        q4 = make_float4(e[0], e[1], e[2], e[3]);
      }
      const uint32_t sw = reinterpret_cast<const uint32_t*>(sb + (sizeof(float) << T))[i >> 5] >> (i & 31);
      q4 = make_float4(__int_as_float(__float_as_int(q4.x) ^ ((~sw & 1u) << 31)),
                       __int_as_float(__float_as_int(q4.y) ^ ((~sw & 2u) << 30)),
                       __int_as_float(__float_as_int(q4.z) ^ ((~sw & 4u) << 29)),
                       __int_as_float(__float_as_int(q4.w) ^ ((~sw & 8u) << 28)));
    } else {
      q4 = *reinterpret_cast<const float4*>(tile + i);
      if constexpr (SK == TS_GATHER) q4 = gather_mask4(a, worker, gotw, g, q4);
    }
    v[4 * m] = q4.x;
    v[4 * m + 1] = q4.y;
    v[4 * m + 2] = q4.z;
    v[4 * m + 3] = q4.w;
  }
  bfly32<P.xm[0]>(v);
  __syncthreads();  // the dense tile has been read
  // rounds B, C in the padded layout (it ends exactly where the stage's
  // sign words end; those were consumed in round A)
#pragma unroll
  for (int j = 0; j < 32; ++j) tile[p0 + pad(roff(P, 0, j))] = v[j];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = tile[p1 + pad(roff(P, 1, j))];
  bfly32<P.xm[1]>(v);
  if constexpr (P.nr == 3) {
#pragma unroll
    for (int j = 0; j < 32; ++j) tile[p1 + pad(roff(P, 1, j))] = v[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = tile[p2 + pad(roff(P, 2, j))];
    bfly32<P.xm[2]>(v);
  }
  __syncthreads();  // the padded tile has been read: the stage is free
  if constexpr (!STRIDED) {
    if (tid == 0) refill();
    if constexpr (P.pos[LR][0] == 0 && P.pos[LR][1] == 1) {
#pragma unroll
      for (int m = 0; m < 8; ++m)
        d.store4(g0 + b2 + roff(P, LR, 4 * m), make_float4(v[4 * m], v[4 * m + 1], v[4 * m + 2], v[4 * m + 3]));
    } else if constexpr (P.pos[LR][0] == 0) {
#pragma unroll
      for (int m = 0; m < 16; ++m) d.store2(g0 + b2 + roff(P, LR, 2 * m), v[2 * m], v[2 * m + 1]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) d.store1(g0 + b2 + roff(P, LR, j), v[j]);
    }
  } else if constexpr (std::is_same<Snk, SnkDecode>::value) {
    // decode epilogue (hadamard.py:119-123, runner.py:253-256): scale,
    // signs, cast, then TMA store into `out` for the rows inside [0, L)
    // (the map stops at the last full row; the partial row goes by STG)
    const int64_t rows_full = d.L >> a.lo;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const int i = b2 + roff(P, LR, 4 * m);
      const int64_t g = g0 + ((int64_t)(i >> CB) << a.lo) + (i & CM);
      const uint32_t w = __ldg(d.signs + (g >> 5)) >> (g & 31);
      float4 o4 = make_float4(v[4 * m] * d.scale, v[4 * m + 1] * d.scale, v[4 * m + 2] * d.scale,
                              v[4 * m + 3] * d.scale);
      o4 = make_float4(__int_as_float(__float_as_int(o4.x) ^ ((~w & 1u) << 31)),
                       __int_as_float(__float_as_int(o4.y) ^ ((~w & 2u) << 30)),
                       __int_as_float(__float_as_int(o4.z) ^ ((~w & 4u) << 29)),
                       __int_as_float(__float_as_int(o4.w) ^ ((~w & 8u) << 28)));
      if ((i >> CB) >= rows_full) {  // partial last row / padding rows
        const float r4[4] = {o4.x, o4.y, o4.z, o4.w};
        for (int c = 0; c < 4; ++c)
          if (g + c < d.L) store_elem(d.out, d.dtype, g + c, r4[c]);
      }
      if (d.dtype == OPTR_BF16) {
        const __nv_bfloat162 lo2 = __floats2bfloat162_rn(o4.x, o4.y), hi2 = __floats2bfloat162_rn(o4.z, o4.w);
        uint2 u;
        u.x = *reinterpret_cast<const uint32_t*>(&lo2);
        u.y = *reinterpret_cast<const uint32_t*>(&hi2);
        *reinterpret_cast<uint2*>(sb + (size_t)i * 2) = u;
      } else {
        *reinterpret_cast<float4*>(tile + i) = o4;
      }
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      const int c0 = (int)((t & ((1LL << cgb) - 1)) << CB);
      const int nbox = (1 << (T - CB)) / a.box_rows;
      const int esz = d.dtype == OPTR_BF16 ? 2 : 4;
      for (int b = 0; b < nbox; ++b)
        if ((int64_t)b * a.box_rows < rows_full)
          tma_store_3d(&dst, sb + ((size_t)b * a.box_rows << CB) * esz, c0, b * a.box_rows, 0);
      bulk_commit();
      refill();
    }
  } else {
    // dense result -> TMA tensor store
    const float sc = a.scale;
    if constexpr (P.pos[LR][0] == 0 && P.pos[LR][1] == 1) {
#pragma unroll
      for (int m = 0; m < 8; ++m)
        *reinterpret_cast<float4*>(tile + b2 + roff(P, LR, 4 * m)) =
            make_float4(v[4 * m] * sc, v[4 * m + 1] * sc, v[4 * m + 2] * sc, v[4 * m + 3] * sc);
    } else if constexpr (P.pos[LR][0] == 0) {
#pragma unroll
      for (int m = 0; m < 16; ++m)
        *reinterpret_cast<float2*>(tile + b2 + roff(P, LR, 2 * m)) = make_float2(v[2 * m] * sc, v[2 * m + 1] * sc);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) tile[b2 + roff(P, LR, j)] = v[j] * sc;
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      const int c0 = (int)((t & ((1LL << cgb) - 1)) << CB);
      const int outer = SK == TS_GATHER ? 0 : (int)(t >> cgb);
      const int nbox = (1 << (T - CB)) / a.box_rows;
      for (int b = 0; b < nbox; ++b)
        tma_store_3d(&dst, tile + ((size_t)b * a.box_rows << CB), c0, b * a.box_rows, outer);
      bulk_commit();
      refill();
    }
  }
}

template <int T, int kStages, bool STRIDED, int SK, class Snk, int CBW>
__global__ void __launch_bounds__(1 << (T - 5)) tma_pass_kernel(const __grid_constant__ TmaMaps maps,
                                                              const __grid_constant__ TmaMaps dmaps,
                                                              const __grid_constant__ TmaArgs a,
                                                              const __grid_constant__ Snk snk, int worker_base) {
  const int worker = worker_base + blockIdx.y;
  const CUtensorMap& dst = dmaps.m[worker];
  uint8_t* const gotw = (SK == TS_GATHER && a.got) ? a.got + (int64_t)worker * a.dim : nullptr;
  constexpr size_t SB = tma_stage_bytes<T>();
  extern __shared__ __align__(16) unsigned char smraw[];
  // 1024-byte aligned ring; indexing smraw keeps the shared address space
  unsigned char* const base = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  uint64_t* const full = reinterpret_cast<uint64_t*>(base + kStages * SB);
  const int tid = threadIdx.x;
  const auto d = snk.bind(worker);

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // programmatic dependent launch: let the next kernel in the stream get
  // scheduled now, and wait here until the previous one's memory is visible
  // (both are no-ops for a normal launch)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t stride = gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      const int64_t ts = blockIdx.x + s * stride;
      if (ts < a.ntiles) tile_issue<T, STRIDED, SK, CBW>(maps, a, worker, ts, base + s * SB, &full[s]);
    }
  }
  int k = 0;
  for (int64_t t = blockIdx.x; t < a.ntiles; t += stride, ++k) {
    const int s = k % kStages;
    unsigned char* const sb = base + s * SB;
    mbar_wait(&full[s], (uint32_t)((k / kStages) & 1));
    tma_tile<T, STRIDED, SK, Snk, CBW>(maps, dst, a, d, worker, gotw, t, sb, [&]() {
      if constexpr (!STRIDED) {
        // contiguous: the stage was read; refill it while the results leave by STG
        if (t + kStages * stride < a.ntiles)
          tile_issue<T, STRIDED, SK, CBW>(maps, a, worker, t + kStages * stride, sb, &full[s]);
      } else if constexpr (kStages == 1) {
        bulk_wait_read0();  // single stage: refill once this tile's store has left it
        if (t + stride < a.ntiles) tile_issue<T, STRIDED, SK, CBW>(maps, a, worker, t + stride, base, &full[0]);
      } else if (k >= 1) {
        bulk_wait_read1();  // the store of tile k-1 has left its stage
        const int64_t tn = t + (kStages - 1) * stride;
        const int sp = (k - 1) % kStages;
        if (tn < a.ntiles) tile_issue<T, STRIDED, SK, CBW>(maps, a, worker, tn, base + sp * SB, &full[sp]);
      }
    });
  }
  if constexpr (STRIDED) {
    if (tid == 0) bulk_wait0();
  }
}

// ------------------------------------------------ persistent two-pass chain
// Both passes of a two-pass transform (contiguous bits [0,T), then strided
// bits [T,n) on 2^(T-CB) x 2^CB tiles: the same tile size) for several
// workers in ONE persistent launch.  Tiles are handed out by a global ticket
// counter in job order w0.p0, w1.p0, w0.p1, w2.p0, w1.p1, ..., so each
// worker's intermediate is still L2-resident when its second pass reads it,
// and no pass pays a launch ramp or a tail.  A pass-1 tile of worker w
// depends on every pass-0 tile of w (per-worker completion counter).
//
// Thread 0 claims tickets in processing order (slot k % S holds position k;
// a strided slot is refilled one tile late, once its store has read it).  A
// pass-1 tile whose dependency is not met at claim time is deferred: its load
// is issued when the CTA reaches it, after all of the CTA's earlier tiles
// are finished and signalled, so waiting never blocks a tile it depends on.
template <int T, int S>
__host__ __device__ constexpr size_t tma_chain_smem_bytes() {
  return S * tma_stage_bytes<T>() + 128 + 1024;  // ring, barriers + slot records, alignment
}

struct ChainSched {
  unsigned int* ctr;  // [0] ticket, [1] CTAs done, [2 + w] pass-0 tiles done; zero on entry, reset by the last CTA
  int nw;
  int64_t nt0, nt1;  // tiles per worker of pass 0 / pass 1
  int njobs;
  int8_t jpass[2 * kMaxW];
  int8_t jw[2 * kMaxW];
  int64_t jstart[2 * kMaxW + 1];  // first ticket of each job; jstart[njobs] = total
};

__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

template <int T, int kStages, int SK0, class Snk1, int CBW>
__global__ void __launch_bounds__(1 << (T - 5)) tma_chain_kernel(const __grid_constant__ TmaMaps maps1,
                                                               const __grid_constant__ TmaMaps dmaps1,
                                                               const __grid_constant__ TmaArgs a0,
                                                               const __grid_constant__ TmaArgs a1,
                                                               const __grid_constant__ SnkBuf snk0,
                                                               const __grid_constant__ Snk1 snk1,
                                                               const __grid_constant__ ChainSched cs) {
  constexpr size_t SB = tma_stage_bytes<T>();
  extern __shared__ __align__(16) unsigned char smraw[];
  unsigned char* const base = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  uint64_t* const full = reinterpret_cast<uint64_t*>(base + kStages * SB);
  int* const slot_job = reinterpret_cast<int*>(full + kStages);          // job of each slot, -1 = end
  int64_t* const slot_tile = reinterpret_cast<int64_t*>(slot_job + 4);   // tile within the job
  const int tid = threadIdx.x;
  unsigned int* const ticket = cs.ctr;
  unsigned int* const done = cs.ctr + 2;
  const int64_t total = cs.jstart[cs.njobs];

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  // thread-0 state
  bool ended = false;
  int lag = -1;                  // strided slot whose refill is pending
  unsigned deferred = 0;         // slots claimed but not yet issued (bit s)
  auto do_issue = [&](int s) {
    const int j = slot_job[s];
    const int w = cs.jw[j];
    const int64_t t = slot_tile[s];
    if (cs.jpass[j] == 0) {
      tile_issue<T, false, SK0, CBW>(maps1, a0, w, t, base + s * SB, &full[s]);
    } else {
      fence_proxy_async_global();  // pass-0 results (generic stores) before these TMA reads
      tile_issue<T, true, TS_BUF, CBW>(maps1, a1, w, t, base + s * SB, &full[s]);
    }
  };
  auto claim_issue = [&](int s) {
    int j = -1;
    int64_t t = 0;
    if (!ended) {
      const int64_t tk = atomicAdd(ticket, 1u);
      if (tk >= total) {
        ended = true;
      } else {
        j = 0;
        while (tk >= cs.jstart[j + 1]) ++j;
        t = tk - cs.jstart[j];
      }
    }
    slot_job[s] = j;
    slot_tile[s] = t;
    if (j < 0) {
      mbar_arrive(&full[s]);  // end marker: completes the phase with no data
    } else if (cs.jpass[j] == 1 && ld_acquire_gpu(done + cs.jw[j]) < (unsigned)cs.nt0) {
      deferred |= 1u << s;
    } else {
      do_issue(s);
    }
  };
  if (tid == 0)
    for (int s = 0; s < kStages; ++s) claim_issue(s);

  for (int k = 0;; ++k) {
    const int s = k % kStages;
    unsigned char* const sb = base + s * SB;
    if (tid == 0 && (deferred >> s & 1u)) {
      const unsigned int* dw = done + cs.jw[slot_job[s]];
      while (ld_acquire_gpu(dw) < (unsigned)cs.nt0) __nanosleep(64);
      do_issue(s);
      deferred &= ~(1u << s);
    }
    mbar_wait(&full[s], (uint32_t)((k / kStages) & 1));
    const int j = slot_job[s];
    if (j < 0) break;
    const int w = cs.jw[j];
    const int64_t t = slot_tile[s];  // read before tma_tile's first barrier; refills come after it
    if (cs.jpass[j] == 0) {
      uint8_t* const gotw = (SK0 == TS_GATHER && a0.got) ? a0.got + (int64_t)w * a0.dim : nullptr;
      tma_tile<T, false, SK0, SnkBuf, CBW>(maps1, dmaps1.m[w], a0, snk0.bind(w), w, gotw, t, sb, [&]() {
        if (lag >= 0) {
          bulk_wait_read0();
          claim_issue(lag);
          lag = -1;
        }
        claim_issue(s);
      });
      __syncthreads();  // all results of the tile are stored
      if (tid == 0) {
        __threadfence();
        fence_proxy_async_global();
        atomicAdd(done + w, 1u);
      }
    } else {
      tma_tile<T, true, TS_BUF, Snk1, CBW>(maps1, dmaps1.m[w], a1, snk1.bind(w), w, nullptr, t, sb, [&]() {
        if (lag >= 0) {
          bulk_wait_read1();  // the previous strided store has left its slot
          claim_issue(lag);
        }
        lag = s;
      });
    }
  }
  if (tid == 0) {
    bulk_wait0();
    __threadfence();
    const unsigned int prev = atomicAdd(cs.ctr + 1, 1u);
    if (prev == gridDim.x - 1) {  // last CTA out: reset the counters for the next launch
      cs.ctr[0] = 0;
      cs.ctr[1] = 0;
      for (int w = 0; w < cs.nw; ++w) done[w] = 0;
      __threadfence();
    }
  }
}

}  // namespace optr

namespace optr {

// ------------------------------------------------ TMA stage-1 aggregate
// TAR stage 1 at owner o (collectives.py:113-125, _mean_received :77-94):
// the owner's shard of every worker's wire vector streams into shared
// memory in CH-entry chunks by 1D bulk copies (peer-mapped buffers in the
// multi-GPU path, so the NVLink requests are whole chunks), two chunks in
// flight per CTA; each thread then takes the fp64 mean of 4 entries in
// ascending node order under the stage-1 masks.
struct TmaAggArgs {
  const float* Y[kMaxW];  // wire vector of each worker
  float* A[kMaxW];        // aggregate shard of each owner
  float* G[kMaxW];        // push mode: every rank's stage-2 receive vector (peer-mapped)
  int push;               // 1: write the mean into G[q] + off for every rank q (TAR stage 2 fused)
  Shards sh;
  int n, r, owner_base;
  MaskView m;
};

template <int CH>
__host__ __device__ constexpr size_t tma_agg_smem_bytes(int n) {
  return (size_t)2 * n * CH * sizeof(float) + 64 + 1024;
}

template <int CH, int NW>
__global__ void __launch_bounds__(CH / 4) tma_agg_kernel(const __grid_constant__ TmaAggArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  unsigned char* const base = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  float* const buf = reinterpret_cast<float*>(base);  // [2][n][CH]
  uint64_t* const full = reinterpret_cast<uint64_t*>(base + (size_t)2 * a.n * CH * sizeof(float));
  const int tid = threadIdx.x;
  const int n = NW > 0 ? NW : a.n;  // compile-time worker count for the common n
  const int o = a.owner_base + blockIdx.y;
  const int j = owned_shard(o, a.r, n);
  const int64_t off = a.sh.off(j), len = a.sh.len(j);
  const int64_t nchunks = (len + CH - 1) / CH;
  float* const A = a.A[o];
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // programmatic dependent launch: let the next kernel in the stream get
  // scheduled now, and wait here until the previous one's memory is visible
  // (both are no-ops for a normal launch)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  auto issue = [&](int64_t c, int s) {
    const int64_t e0 = c * CH;
    int64_t cnt = len - e0;
    if (cnt > CH) cnt = CH;
    const uint32_t bytes = (uint32_t)(cnt * sizeof(float));
    mbar_expect_tx(&full[s], bytes * (uint32_t)n);
    for (int i = 0; i < n; ++i) bulk_load(buf + ((size_t)s * n + i) * CH, a.Y[i] + off + e0, bytes, &full[s]);
  };
  const int64_t stride = gridDim.x;
  int64_t c = blockIdx.x;
  if (tid == 0) {
    if (c < nchunks) issue(c, 0);
    if (c + stride < nchunks) issue(c + stride, 1);
  }
  for (int k = 0; c < nchunks; ++k, c += stride) {
    const int s = k & 1;
    mbar_wait(&full[s], (uint32_t)((k >> 1) & 1));
    const int64_t e = c * CH + tid * 4;
    float4 res = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e < len) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      uint32_t c4[4] = {0u, 0u, 0u, 0u};
      const float* src = buf + (size_t)s * n * CH + tid * 4;
#pragma unroll
      for (int i = 0; i < (NW > 0 ? NW : kMaxW); ++i) {
        if (NW == 0 && i >= n) break;
        const float4 v = *reinterpret_cast<const float4*>(src + (size_t)i * CH);
        const uint32_t kk = i == o ? 0xFu : keep4(a.m.row(0, o, i), (uint32_t)e, a.m);
        // misses add +0.0 (the reference adds its zero-filled buffer)
        acc[0] += (kk & 1u) ? (double)v.x : 0.0;
        acc[1] += (kk & 2u) ? (double)v.y : 0.0;
        acc[2] += (kk & 4u) ? (double)v.z : 0.0;
        acc[3] += (kk & 8u) ? (double)v.w : 0.0;
        c4[0] += kk & 1u;
        c4[1] += (kk >> 1) & 1u;
        c4[2] += (kk >> 2) & 1u;
        c4[3] += (kk >> 3) & 1u;
      }
      res = make_float4(mean_of(acc[0], (double)c4[0]), mean_of(acc[1], (double)c4[1]),
                        mean_of(acc[2], (double)c4[2]), mean_of(acc[3], (double)c4[3]));
    }
    __syncthreads();  // stage s has been read
    if (tid == 0 && c + 2 * stride < nchunks) issue(c + 2 * stride, s);
    if (e + 4 <= len) {
      if (a.push) {
        // stage 2 (collectives.py:133-137): the owner's mean goes to every rank
#pragma unroll
        for (int q = 0; q < (NW > 0 ? NW : kMaxW); ++q) {
          if (NW == 0 && q >= n) break;
          st4(a.G[q] + off + e, res);
        }
      } else {
        st4(A + e, res);
      }
    }
  }
}

}  // namespace optr
