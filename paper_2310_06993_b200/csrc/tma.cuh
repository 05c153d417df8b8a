// TMA-pipelined FWHT passes and the persistent kernels built on them (sm_100a).
//
// A pass transforms index bits [lo, lo+ks) of a vector in tiles of 2^T
// entries (see kernels.cuh PassGeom).  Tiles stream through a 2- or 3-stage
// shared-memory ring per CTA, filled by one elected thread with TMA:
//
//   contiguous pass (lo = 0): one 1D bulk copy (cp.async.bulk) per tile;
//   strided pass (8 or 32 columns): box_rows-row tensor boxes
//     (cp.async.bulk.tensor), because through the LSU each warp load of
//     32-byte row segments touches 16 cache lines and the pass is L1-bound
//     even on L2-resident data; sign bits for a strided tile come as one
//     bulk copy of its column of transposed sign bytes (PrepArgs.signs_t).
//
// Each tile is transformed in place in its stage buffer (tma_tile): round A
// reads the dense tile (float4), rounds B and C go through a padded copy of
// the same buffer (conflict-free for every layout here), and the result
// leaves either through vector STG or through TMA tensor stores.  The fused
// source transforms (encode pad/signs/bf16 upcast, TAR stage-2 gather with
// masks) are applied when round A reads the tile, the decode epilogue
// (count scale, signs, truncate, cast) when the last round writes it.
//
// Kernels: tma_pass_kernel (one pass, grid.y = worker), tma_mean_kernel
// (one GPU: last encode pass of every worker + TAR stage-1 mean), tma_agg_kernel
// (TAR stage-1 mean, optional stage-2 push), tma_fused_kernel (multi-GPU:
// contiguous encode + stage 1 + stage 2 + contiguous decode, per-tile flags
// over NVLink).
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
  // strided passes: transposed sign bytes (one 2^ks-byte column per 8-column
  // tile, loaded with the tile) for the encode source / decode epilogue
  const uint8_t* signs_t;
  // TS_GATHER (collectives.py:140-150): owner shards, stage-2 masks
  const float* A[kMaxW];
  int n, r;
  int shard_shift;  // equal power-of-two shards of 2^shard_shift entries
  MaskView m;
  uint8_t* got;  // optional [worker][dim]
  int64_t dim;
  const uint32_t* tile_ok2;  // optional stage-2 tile summaries (PrepArgs.tile_ok + ntiles)
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
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
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

// Issue the bulk loads of contiguous tile t into stage buffer `st` (sign
// words after the tile for the encode source).
template <int T, int SK>
__device__ __forceinline__ void tile_issue_contig(const TmaArgs& a, int w, int64_t t, unsigned char* st,
                                                  uint64_t* bar) {
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
    if (SK == TS_ENC) {
      // x as a [rows_full][2^lo] tensor (dtype of x): boxes of the full rows;
      // rows past the map come back zero-filled (full-box transaction) and
      // round A reads the partial row from global memory
      const int esz = a.dtype == OPTR_BF16 ? 2 : 4;
      const int64_t rows_full = a.L >> a.lo;
      uint32_t bytes = 0;
      for (int b = 0; b < nbox; ++b)
        if ((int64_t)b * a.box_rows < rows_full) bytes += (uint32_t)(esz * a.box_rows) << CBW;
      const uint32_t sbytes = a.signs_t ? (1u << KS) : 0u;  // the tile's sign column
      mbar_expect_tx(bar, bytes + sbytes);
      for (int b = 0; b < nbox; ++b) {
        const int row = b * a.box_rows;
        if (row < rows_full) tma_load_3d(st + ((size_t)row << CBW) * esz, &maps.m[w], bar, c0, row, 0);
      }
      if (sbytes) bulk_load(st + (sizeof(float) << T), a.signs_t + ((size_t)(c0 >> CBW) << KS), sbytes, bar);
      return;
    }
    const uint32_t sbytes = (SK == TS_BUF && a.signs_t) ? (1u << KS) : 0u;  // decode epilogue signs
    mbar_expect_tx(bar, (uint32_t)(sizeof(float) << T) + sbytes);
    if (sbytes) bulk_load(st + (sizeof(float) << T), a.signs_t + ((size_t)(c0 >> CBW) << KS), sbytes, bar);
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
    tile_issue_contig<T, SK>(a, w, t, st, bar);
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

// Contiguous stage-2 tile t of receiver q lies in one shard: true when q owns
// it or every packet of it arrived (no per-entry masks then).
template <int T>
__device__ __forceinline__ bool gather_tile_all_kept(const TmaArgs& a, int q, int64_t t) {
  const int64_t g0 = t << T;
  const int j = (int)(g0 >> a.shard_shift);
  const int owner = shard_owner(j, a.r, a.n);
  if (owner == q) return true;
  if (a.tile_ok2) return (__ldg(a.tile_ok2 + t) >> q) & 1u;  // prep's per-tile summary
  return packets_all_kept(a.m.row(1, q, owner), (uint32_t)(g0 - ((int64_t)j << a.shard_shift)), 1u << T, a.m);
}

// CTA barrier (BAR = 0) or named barrier BAR over the first NT threads, for
// kernels whose CTA holds several independent warp groups.
template <int BAR, int NT>
__device__ __forceinline__ void group_sync() {
  if constexpr (BAR == 0) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NT) : "memory");
  }
}

// One tile of a TMA pass, from its filled stage buffer `sb` to its issued
// result.  `refill()` is called by thread 0 once the stage may be reused for
// the next load: for a contiguous tile right after the tile has been read
// (the results then leave by STG), for a strided tile after its TMA store
// group is committed (the refill policy decides which stage to wait for).
// Contiguous passes hand their results to `epi(v, base)` when one is given
// (v[4m..4m+3] are tile entries base + roff(make_rplan(T, 0), LR, 4m) + 0..3),
// else store them through the sink.
struct NoEpi {
  __device__ __forceinline__ void operator()(const float (&)[32], int) const {}
};

template <int T, bool STRIDED, int SK, class Snk, int CBW, int BAR = 0, int TID_OFF = 0, class Refill,
          class Epi = NoEpi>
__device__ __forceinline__ void tma_tile(const TmaMaps* maps, const CUtensorMap* dst, const TmaArgs& a,
                                         const typename Snk::B& d, int worker, uint8_t* gotw, int64_t t,
                                         unsigned char* sb, Refill&& refill, Epi&& epi = Epi{},
                                         bool all_kept = false, const float* radd = nullptr) {
  constexpr int CB = STRIDED ? CBW : 0;  // untransformed column bits (8 or 32 columns)
  constexpr int CM = (1 << CB) - 1;
  constexpr RPlan P = make_rplan(T, CB);
  static_assert(P.nr == 2 || P.nr == 3, "TMA pass expects two or three register rounds");
  constexpr int LR = P.nr - 1;  // last round
  static_assert(P.pos[0][0] == 0 && P.pos[0][1] == 1, "round A holds float4 groups");
  static_assert(!STRIDED || !std::is_same<Snk, SnkDecode>::value || (P.pos[LR][0] == 0 && P.pos[LR][1] == 1),
                "decode epilogue stores float4 groups");
  static_assert(sizeof(float) * pad(1 << T) <= tma_stage_bytes<T>(), "padded tile fits the stage");
  const int tid = (int)threadIdx.x - TID_OFF;  // thread index inside its warp group
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
  if constexpr (SK == TS_ENC && !STRIDED) {
    const int lsh = a.dtype == OPTR_BF16 ? 1 : 2;
    bulk_end = g0 + ((((a.L - g0) << lsh) & ~15LL) >> lsh);
    enc_fast = g0 + (1 << T) <= bulk_end;
  }
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const int i = b0 + roff(P, 0, 4 * m);
    const int64_t g = STRIDED ? (g0 + ((int64_t)(i >> CB) << a.lo) + (i & CM)) : (g0 + i);
    float4 q4;
    if constexpr (SK == TS_ENC && STRIDED) {
      // strided encode (hadamard.py:93-102 with the passes reordered): the
      // tile's full rows came by TMA; the partial row and padding rows here
      if (a.dtype == OPTR_BF16) {
        const uint2 u = *reinterpret_cast<const uint2*>(sb + (size_t)i * 2);
        const float2 fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
        const float2 fb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
        q4 = make_float4(fa.x, fa.y, fb.x, fb.y);
      } else {
        q4 = *reinterpret_cast<const float4*>(tile + i);
      }
      if ((g >> a.lo) >= (a.L >> a.lo)) {
        float e[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (g + c < a.L) e[c] = load_elem(a.xw[worker], a.dtype, g + c);
        q4 = make_float4(e[0], e[1], e[2], e[3]);
      }
      const uint32_t sw = a.signs_t ? (uint32_t)sb[(sizeof(float) << T) + (i >> CB)] >> (i & 7)
                                    : __ldg(a.signs + (g >> 5)) >> (g & 31);
      q4 = make_float4(__int_as_float(__float_as_int(q4.x) ^ ((~sw & 1u) << 31)),
                       __int_as_float(__float_as_int(q4.y) ^ ((~sw & 2u) << 30)),
                       __int_as_float(__float_as_int(q4.z) ^ ((~sw & 4u) << 29)),
                       __int_as_float(__float_as_int(q4.w) ^ ((~sw & 8u) << 28)));
    } else if constexpr (SK == TS_ENC) {
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
      if (radd) {  // contiguous TS_BUF: a pre-accumulated sum of other tiles (linearity)
        q4.x += radd[4 * m];
        q4.y += radd[4 * m + 1];
        q4.z += radd[4 * m + 2];
        q4.w += radd[4 * m + 3];
      }
    }
    v[4 * m] = q4.x;
    v[4 * m + 1] = q4.y;
    v[4 * m + 2] = q4.z;
    v[4 * m + 3] = q4.w;
  }
  if constexpr (SK == TS_GATHER) {
    // stage-2 masks (collectives.py:140-150); a tile whose packets all
    // arrived skips them (one branch per tile, not per float4)
    const int jt = STRIDED ? 0 : (int)(g0 >> a.shard_shift);
    if (!all_kept && !STRIDED && shard_owner(jt, a.r, a.n) != worker) {
      // contiguous tile: one shard, one owner (not this receiver: its own
      // shard is never masked), one bitmap row for the whole tile
      const int j = jt;
      const uint32_t* const row = a.m.row(1, worker, shard_owner(j, a.r, a.n));
      const uint32_t e0 = (uint32_t)(g0 - ((int64_t)j << a.shard_shift));
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int i = b0 + roff(P, 0, 4 * m);
        const uint32_t kk = keep4(row, e0 + (uint32_t)i, a.m);
        v[4 * m] = (kk & 1u) ? v[4 * m] : 0.f;
        v[4 * m + 1] = (kk & 2u) ? v[4 * m + 1] : 0.f;
        v[4 * m + 2] = (kk & 4u) ? v[4 * m + 2] : 0.f;
        v[4 * m + 3] = (kk & 8u) ? v[4 * m + 3] : 0.f;
        if (gotw)
          *reinterpret_cast<uchar4*>(gotw + g0 + i) =
              make_uchar4(kk & 1u, (kk >> 1) & 1u, (kk >> 2) & 1u, (kk >> 3) & 1u);
      }
    } else if (!all_kept) {  // strided tiles (several shards) and own contiguous tiles
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int i = b0 + roff(P, 0, 4 * m);
        const int64_t g = STRIDED ? (g0 + ((int64_t)(i >> CB) << a.lo) + (i & CM)) : (g0 + i);
        const float4 q4 = gather_mask4(a, worker, gotw, g, make_float4(v[4 * m], v[4 * m + 1], v[4 * m + 2],
                                                                       v[4 * m + 3]));
        v[4 * m] = q4.x;
        v[4 * m + 1] = q4.y;
        v[4 * m + 2] = q4.z;
        v[4 * m + 3] = q4.w;
      }
    } else if (gotw) {
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int i = b0 + roff(P, 0, 4 * m);
        const int64_t g = STRIDED ? (g0 + ((int64_t)(i >> CB) << a.lo) + (i & CM)) : (g0 + i);
        *reinterpret_cast<uchar4*>(gotw + g) = make_uchar4(1, 1, 1, 1);
      }
    }
  }
  bfly32<P.xm[0]>(v);
  // strided decode epilogue with transposed signs: take this thread's
  // last-round sign nibbles now, before the padded layout covers them
  uint32_t dsig = 0;
  if constexpr (STRIDED && std::is_same<Snk, SnkDecode>::value) {
    if (a.signs_t) {
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int i = b2 + roff(P, LR, 4 * m);
        dsig |= (((uint32_t)sb[(sizeof(float) << T) + (i >> CB)] >> (i & 7)) & 0xFu) << (4 * m);
      }
    }
  }
  group_sync<BAR, (1 << (T - 5))>();  // the dense tile has been read
  // rounds B, C in the padded layout (it ends exactly where the stage's
  // sign words end; those were consumed in round A)
#pragma unroll
  for (int j = 0; j < 32; ++j) tile[p0 + pad(roff(P, 0, j))] = v[j];
  group_sync<BAR, (1 << (T - 5))>();
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = tile[p1 + pad(roff(P, 1, j))];
  bfly32<P.xm[1]>(v);
  if constexpr (P.nr == 3) {
#pragma unroll
    for (int j = 0; j < 32; ++j) tile[p1 + pad(roff(P, 1, j))] = v[j];
    group_sync<BAR, (1 << (T - 5))>();
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = tile[p2 + pad(roff(P, 2, j))];
    bfly32<P.xm[2]>(v);
  }
  group_sync<BAR, (1 << (T - 5))>();  // the padded tile has been read: the stage is free
  if constexpr (!STRIDED && !std::is_same<std::decay_t<Epi>, NoEpi>::value) {
    if (tid == 0) refill();
    epi(v, b2);
  } else if constexpr (!STRIDED) {
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
      const uint32_t w = a.signs_t ? dsig >> (4 * m) : __ldg(d.signs + (g >> 5)) >> (g & 31);
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
    group_sync<BAR, (1 << (T - 5))>();
    if (tid == 0) {
      const int c0 = (int)((t & ((1LL << cgb) - 1)) << CB);
      const int nbox = (1 << (T - CB)) / a.box_rows;
      const int esz = d.dtype == OPTR_BF16 ? 2 : 4;
      for (int b = 0; b < nbox; ++b)
        if ((int64_t)b * a.box_rows < rows_full)
          tma_store_3d(dst, sb + ((size_t)b * a.box_rows << CB) * esz, c0, b * a.box_rows, 0);
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
    group_sync<BAR, (1 << (T - 5))>();
    if (tid == 0) {
      const int c0 = (int)((t & ((1LL << cgb) - 1)) << CB);
      const int outer = SK == TS_GATHER ? 0 : (int)(t >> cgb);
      const int nbox = (1 << (T - CB)) / a.box_rows;
      for (int b = 0; b < nbox; ++b)
        tma_store_3d(dst, tile + ((size_t)b * a.box_rows << CB), c0, b * a.box_rows, outer);
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
    bool all_kept = false;
    if constexpr (SK == TS_GATHER && !STRIDED) all_kept = gather_tile_all_kept<T>(a, worker, t);
    tma_tile<T, STRIDED, SK, Snk, CBW>(&maps, &dst, a, d, worker, gotw, t, sb, [&]() {
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
    }, NoEpi{}, all_kept);
  }
  if constexpr (STRIDED) {
    if (tid == 0) bulk_wait0();
  }
}

// ------------------------- last encode pass + TAR stage-1 mean (one GPU)
// The contiguous (last) encode pass of every co-resident worker fused with
// TAR stage 1 (collectives.py:113-125, _mean_received :77-94): a CTA takes
// contiguous tile t of worker 0, 1, ..., n-1 in turn through its TMA ring,
// transforms each and scales it by 1/sqrt(dim) in fp32 (the wire value,
// runner.py:224), and accumulates it in fp64 in ascending worker order under
// the stage-1 masks of the tile's owner (own tile always counted, misses
// add 0.0).  After the last worker it writes the owner's mean of the tile
// into the natural-order aggregate vector, so the n wire vectors are never
// written to memory.  A tile lies in one shard (equal power-of-two shards of
// >= 2^T entries); a peer whose packets over the tile all arrived skips the
// per-entry masks.
struct MeanArgs {
  float* agg;   // [dim]: shard j's mean at j's natural offset
  float scale;  // 1/sqrt(dim)
  int n, r, shard_shift;
  MaskView m;   // stage-1 rows (stage 0 of the bitmap layout)
  const uint32_t* tile_ok1;  // stage-1 tile summaries (PrepArgs.tile_ok): bit i = sender i's packets all arrived
};

// two CTAs per SM for 256-thread tiles (T = 13: <= 128 registers), one for
// 512-thread tiles (T = 14)
template <int T, int kStages, int NW>
__global__ void __launch_bounds__(1 << (T - 5), T == 13 ? 2 : 1) tma_mean_kernel(const __grid_constant__ TmaArgs a,
                                                                 const __grid_constant__ MeanArgs ma) {
  constexpr size_t SB = tma_stage_bytes<T>();
  constexpr RPlan P = make_rplan(T, 0);
  constexpr int LR = P.nr - 1;
  static_assert(P.pos[LR][0] == 0, "vector groups in the last round");
  // the last round holds tile bits 0,1 (float4 groups, T = 13) or bit 0 (pairs, T = 14)
  constexpr int VW = P.pos[LR][1] == 1 ? 4 : 2;
  constexpr int NQ = 32 / VW;
  extern __shared__ __align__(16) unsigned char smraw[];
  unsigned char* const base = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  uint64_t* const full = reinterpret_cast<uint64_t*>(base + kStages * SB);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t stride = gridDim.x;
  // job k = (tile blockIdx.x + (k / NW) * stride, worker k % NW)
  auto issue = [&](int64_t k, int s) {
    const int64_t t = blockIdx.x + (k / NW) * stride;
    if (t < a.ntiles) tile_issue_contig<T, TS_BUF>(a, (int)(k % NW), t, base + (size_t)s * SB, &full[s]);
  };
  if (tid == 0)
    for (int s = 0; s < kStages; ++s) issue(s, s);
  // Per tile, C = the ranks whose packets over it all arrived at the owner
  // (the owner included).  By linearity the C tiles are summed as they
  // arrive (first-pass values, fp32) and transformed ONCE, by the job of the
  // last rank in C; each remaining rank (a lost packet over the tile) is
  // transformed and accumulated under its per-entry masks.  A 1% drop rate
  // leaves most tiles with |C| = n (one transform instead of n).  fp32
  // accumulation (the RHT-on path is float32 anyway; the tolerance is 1e-5).
  float acc[32];
  uint32_t cnt[8];  // count byte per entry (a thread's entries 4c..4c+3 in cnt[c])
  float vacc[32];   // running sum of the C tiles (round-A layout)
  uint32_t cset = 0;
  int last_c = 0;
  constexpr uint32_t kAllW = (NW >= 32) ? 0xffffffffu : ((1u << NW) - 1u);
  constexpr RPlan P0 = make_rplan(T, 0);
  const int b0 = thread_base<T>(P0, 0, tid);
  const float scale = ma.scale;
  const SnkBuf::B nosnk{nullptr, 1.f};
  for (int64_t k = 0;; ++k) {
    const int64_t t = blockIdx.x + (k / NW) * stride;
    if (t >= a.ntiles) break;
    const int w = (int)(k % NW);
    const int s = (int)(k % kStages);
    // owner of the tile's shard and the tile's offset inside it (uniform)
    const int64_t g0 = t << T;
    const int j = (int)(g0 >> ma.shard_shift);
    const int owner = shard_owner(j, ma.r, NW);
    const uint32_t e0 = (uint32_t)(g0 - ((int64_t)j << ma.shard_shift));
    if (w == 0) {
      cset = (__ldg(ma.tile_ok1 + t) | (1u << owner)) & kAllW;
      last_c = 31 - __clz(cset);
      const uint32_t c0 = (uint32_t)__popc(cset) * 0x01010101u;
#pragma unroll
      for (int c = 0; c < 8; ++c) cnt[c] = c0;
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) acc[jj] = 0.f;
    }
    const bool in_c = (cset >> w) & 1u;
    mbar_wait(&full[s], (uint32_t)((k / kStages) & 1));
    float* const tile = reinterpret_cast<float*>(base + (size_t)s * SB);
    if (in_c && w != last_c) {  // add the raw tile to the C sum, no transform
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const float4 q4 = *reinterpret_cast<const float4*>(tile + b0 + roff(P0, 0, 4 * m));
        const bool first = w == (__ffs(cset) - 1);
        vacc[4 * m] = (first ? 0.f : vacc[4 * m]) + q4.x;
        vacc[4 * m + 1] = (first ? 0.f : vacc[4 * m + 1]) + q4.y;
        vacc[4 * m + 2] = (first ? 0.f : vacc[4 * m + 2]) + q4.z;
        vacc[4 * m + 3] = (first ? 0.f : vacc[4 * m + 3]) + q4.w;
      }
      __syncthreads();  // every thread has read the stage
      if (tid == 0) issue(k + kStages, s);
      continue;
    }
    const bool sum_job = in_c;  // the last C rank: transform of the C sum
    const bool has_sum = sum_job && __popc(cset) > 1;
    tma_tile<T, false, TS_BUF, SnkBuf, 3>(
        nullptr, nullptr, a, nosnk, w, nullptr, t, base + (size_t)s * SB, [&]() { issue(k + kStages, s); },
        [&](const float (&v)[32], int b2) {
          if (sum_job) {
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) acc[jj] += v[jj] * scale;
          } else {
            const uint32_t* row = ma.m.row(0, owner, w);
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
              const uint32_t e = e0 + (uint32_t)(b2 + roff(P, LR, VW * q));
              const uint32_t kk = (keep4(row, e & ~3u, ma.m) >> (e & 3u)) & ((1u << VW) - 1u);
#pragma unroll
              for (int c = 0; c < VW; ++c) acc[VW * q + c] += ((kk >> c) & 1u) ? v[VW * q + c] * scale : 0.f;
              cnt[(VW * q) / 4] += nibble_bytes(kk) << (8 * ((VW * q) % 4));
            }
          }
          if (w == NW - 1) {
            float* const out = ma.agg + g0;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
              const int i = b2 + roff(P, LR, VW * q);
              float r[VW];
#pragma unroll
              for (int c = 0; c < VW; ++c) {
                const int jj = VW * q + c;
                const uint32_t cn = (cnt[jj / 4] >> (8 * (jj % 4))) & 0xffu;
                // a power-of-two count divides exactly; others round once
                r[c] = (cn & (cn - 1)) == 0 ? acc[jj] * __int_as_float((127 - (__ffs(cn) - 1)) << 23)
                                            : __fdiv_rn(acc[jj], (float)cn);
              }
              if constexpr (VW == 4)
                st4(out + i, make_float4(r[0], r[1], r[2], r[3]));
              else
                *reinterpret_cast<float2*>(out + i) = make_float2(r[0], r[1]);
            }
          }
        },
        false, has_sum ? vacc : nullptr);
  }
}

// ------------------ stage-2 receive + contiguous decode pass (one GPU)
// Every co-resident receiver's decode input for contiguous tile t is the
// owner's aggregate tile under that receiver's stage-2 mask, transformed.
// Receivers whose stage-2 packets over the tile all arrived (tile_ok2 bit;
// the owner always) get the SAME tile: one transform, stored into each of
// their wire vectors; a receiver with a lost packet over the tile gets its
// own masked transform.  A CTA walks its tiles; per tile one job for the
// clean group, then one per masked receiver, each job one TMA load of the
// (L2-resident) aggregate tile through the ring.
struct GatherSharedArgs {
  float* y[kMaxW];  // each receiver's decode buffer (its wire vector)
};

template <int T, int kStages, int NW>
__global__ void __launch_bounds__(1 << (T - 5), T == 13 ? 2 : 1)
    tma_gather_shared_kernel(const __grid_constant__ TmaArgs a, const __grid_constant__ GatherSharedArgs ys) {
  constexpr size_t SB = tma_stage_bytes<T>();
  constexpr RPlan P = make_rplan(T, 0);
  constexpr int LR = P.nr - 1;
  static_assert(P.pos[LR][0] == 0, "vector groups in the last round");
  constexpr int VW = P.pos[LR][1] == 1 ? 4 : 2;
  constexpr int NQ = 32 / VW;
  constexpr uint32_t kAll = (NW >= 32) ? 0xffffffffu : ((1u << NW) - 1u);
  extern __shared__ __align__(16) unsigned char smraw[];
  unsigned char* const base = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  uint64_t* const full = reinterpret_cast<uint64_t*>(base + kStages * SB);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t stride = gridDim.x;
  auto owner_of = [&](int64_t t) { return shard_owner((int)((t << T) >> a.shard_shift), a.r, NW); };
  auto ok_of = [&](int64_t t) { return (__ldg(a.tile_ok2 + t) | (1u << owner_of(t))) & kAll; };
  // issue cursor (thread 0 only): the tile of every job, kStages ahead
  int64_t it = blockIdx.x;
  int ij = 0, in = it < a.ntiles ? 1 + __popc(kAll & ~ok_of(it)) : 0;
  auto issue_next = [&](int s) {
    if (it >= a.ntiles) return;
    tile_issue_contig<T, TS_GATHER>(a, 0, it, base + (size_t)s * SB, &full[s]);
    if (++ij == in) {
      ij = 0;
      it += stride;
      in = it < a.ntiles ? 1 + __popc(kAll & ~ok_of(it)) : 0;
    }
  };
  if (tid == 0)
    for (int s = 0; s < kStages; ++s) issue_next(s);
  const SnkBuf::B nosnk{nullptr, 1.f};
  int64_t k = 0;
  for (int64_t t = blockIdx.x; t < a.ntiles; t += stride) {
    const int owner = owner_of(t);
    const uint32_t ok = ok_of(t);
    uint32_t todo = kAll & ~ok;
    for (bool first = true;; first = false) {
      const int s = (int)(k % kStages);
      mbar_wait(&full[s], (uint32_t)((k / kStages) & 1));
      int q = owner;
      uint32_t dests = ok;
      if (!first) {
        q = __ffs(todo) - 1;
        todo &= todo - 1;
        dests = 1u << q;
      }
      tma_tile<T, false, TS_GATHER, SnkBuf, 3>(
          nullptr, nullptr, a, nosnk, q, nullptr, t, base + (size_t)s * SB, [&]() { issue_next(s); },
          [&](const float (&v)[32], int b2) {
            for (uint32_t d = dests; d; d &= d - 1) {
              float* const yo = ys.y[__ffs(d) - 1] + (t << T);
#pragma unroll
              for (int m = 0; m < NQ; ++m) {
                const int i = b2 + roff(P, LR, VW * m);
                if constexpr (VW == 4)
                  st4(yo + i, make_float4(v[4 * m], v[4 * m + 1], v[4 * m + 2], v[4 * m + 3]));
                else
                  *reinterpret_cast<float2*>(yo + i) = make_float2(v[2 * m], v[2 * m + 1]);
              }
            }
          },
          first);
      ++k;
      if (!todo) break;
    }
  }
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
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

template <int CH, int S = 2>
__host__ __device__ constexpr size_t tma_agg_smem_bytes(int n) {
  return (size_t)S * n * CH * sizeof(float) + 64 + 1024;
}

template <int CH, int NW, int S = 2>
__global__ void __launch_bounds__(CH / 4) tma_agg_kernel(const __grid_constant__ TmaAggArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  unsigned char* const base = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  float* const buf = reinterpret_cast<float*>(base);  // [S][n][CH]
  uint64_t* const full = reinterpret_cast<uint64_t*>(base + (size_t)S * a.n * CH * sizeof(float));
  const int tid = threadIdx.x;
  const int n = NW > 0 ? NW : a.n;  // compile-time worker count for the common n
  const int o = a.owner_base + blockIdx.y;
  const int j = owned_shard(o, a.r, n);
  const int64_t off = a.sh.off(j), len = a.sh.len(j);
  const int64_t nchunks = (len + CH - 1) / CH;
  float* const A = a.A[o];
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
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
  if (tid == 0)
    for (int s = 0; s < S; ++s)
      if (c + s * stride < nchunks) issue(c + s * stride, s);
  for (int k = 0; c < nchunks; ++k, c += stride) {
    const int s = k % S;
    mbar_wait(&full[s], (uint32_t)((k / S) & 1));
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
    if (tid == 0 && c + S * stride < nchunks) issue(c + S * stride, s);
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

namespace optr {

// ------------------------------------ fused multi-GPU TAR core (one rank)
// The encode's last (contiguous) pass, TAR stage 1 at the owner, stage 2
// (owner push) and the decode's first (contiguous) pass of one rank in ONE
// persistent kernel, so NVLink traffic overlaps the FWHT tile by tile
// (collectives.py:97-150 between the runner's encode and decode,
// runner.py:219-258).  The strided passes run before and after it.
//
// Tiles t hold 2^T entries; shard j = tiles [j*ns, (j+1)*ns).  Each CTA has
// two warp groups with their own ticket queues:
//   E/D group (2^(T-5) threads): all E tickets (row order, row k = tiles
//     {j*ns + k}), then all D tickets (row order)
//     E(t)  encode tile t of my wire vector Y in place (scale 1/sqrt(dim)),
//           then eflag[me][t] = epoch in my memory
//     D(t)  once tile t's owner counted every unit of it: pull it from the owner's aggregate
//           (one TMA bulk copy over NVLink, stage-2 masks applied as it is
//           read) and decode it into my G
//   A group (kAggThreads threads): units (1/UPT tile) of my shard in order;
//     for each, wait for eflag[t] at every rank, stream the unit from every
//     rank's Y in kAggCh-entry chunks through a ring, masked fp64 mean in
//     ascending node order into my aggregate A; then gflag[me][t*4+u] = epoch.
// E jobs wait for nothing, A jobs only for E jobs, D jobs only for A jobs of
// the same row, and every queue is claimed in the same order on all ranks,
// so nothing waits on a job that cannot run.  A D job's load is deferred
// (never spun on at claim time) until its CTA has finished every earlier job.
struct FusedArgs {
  const float* Y[kMaxW];       // every rank's wire vector (peer-mapped)
  float* A[kMaxW];             // every rank's owner-shard aggregate (peer-mapped)
  // Flags live in the WRITER's memory and readers poll them over NVLink, so
  // a writer's system-scope release only waits for its own GPU's L2:
  //   eflag[q][t]           = epoch once rank q encoded tile t (its E job);
  //   gflag[q][t * 4 + u]   = epoch once owner q published unit u of tile t.
  // Epochs count the calls of one parity, so a flag left by an earlier call
  // (any shape, any owner) is always below the current epoch: no re-arming.
  unsigned int* eflag[kMaxW];
  unsigned int* gflag[kMaxW];
  unsigned int* ctr;           // local [0] E/D ticket, [1] CTAs done, [2] A ticket (reset by the last CTA)
  unsigned int epoch;
  int n, me, r, own;
  int64_t ns;                  // tiles per shard
  int64_t shard_len;
  MaskView m;
  uint4* trace;   // debug (optr_debug_trace): per CTA [cap/2 E/D jobs | cap/2 A tiles]
  int trace_cap;
  uint64_t watchdog_ns;
  // bounded stage 1 (UBT hard bound, transport.py:102-108 / simdriver.py:
  // 323-326): an owner waits for a peer's encoded tile until deadline_ns
  // after its CTA started, then aggregates without it (0 = unbounded)
  uint64_t deadline_ns;
  int grid_cap;                      // host: CTAs of the launch (0 = SMs x occupancy)
  unsigned long long* stats;         // optr_tar_stats (device) or null
  const unsigned long long* counts;  // this rank's [2][n] mask-model received counts
  uint32_t* cut_units;               // optional [units]: peers cut from each stage-1 unit
};

// optr_tar_stats field offsets (u64 words, include/optr.h)
enum { ST_RECV0 = 0, ST_RECV1 = 1, ST_CUT0 = 2, ST_CUT1 = 3, ST_OPEN = 4, ST_STAGE1 = 5, ST_STAGE2 = 6 };

__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned int* p, unsigned int v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Flags of the fused kernel.  Every flag lives in its WRITER's memory, next
// to the data it publishes (the writer's wire tiles Y / aggregate A), and
// readers poll it over NVLink:
//   writer: data stores by the group -> group barrier -> one thread:
//           __threadfence (MEMBAR.SC.GPU, cumulative over the barrier) ->
//           relaxed system-scope flag store into its own memory;
//   reader: relaxed system-scope polls of the writer's flag -> fence.acquire.sys
//           (an L1 invalidate) -> fence.proxy.async -> TMA reads of the data.
// Flag and data sit in the same GPU's memory and every peer access to it is
// served by that GPU's L2, so once the fence has made the data GPU-visible
// (in that L2) any reader that sees the flag reads the data.  A system-scope
// release (fence.release.sys = MEMBAR.ALL.SYS) gives the same results and is
// what the PTX model asks for across GPUs, but costs 15-25% of the step at
// N=2 (profiles/r02_fence_ab.txt); 10,000 back-to-back async calls per test
// run match the serialised calls bit for bit (test_fused_protocol_async_stress).
__device__ __forceinline__ void fence_release_sys() { asm volatile("fence.release.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acquire_sys() { asm volatile("fence.acquire.sys;" ::: "memory"); }
__device__ __forceinline__ unsigned int ld_relaxed_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(unsigned int* p, unsigned int v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_relaxed_sys(unsigned int* p, unsigned int v) {
  asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Spin until *p >= v.  A peer may legitimately be late (a straggler rank in
// DDP); one that never arrives is a protocol bug or a dead rank: trap after
// `limit_ns` (OPTR_WATCHDOG_S, default 1800 s like NCCL's default timeout)
// instead of hanging the GPU.
__device__ __noinline__ void spin_ge_sys(const unsigned int* p, unsigned int v, uint64_t limit_ns) {
  if (ld_relaxed_sys(p) >= v) return;
  const uint64_t t0 = globaltimer_ns();
  while (ld_relaxed_sys(p) < v) {
    __nanosleep(64);
    if (globaltimer_ns() - t0 > limit_ns) {
      printf("optr: fused kernel wait timed out (flag %p, have %u, want %u)\n", p, ld_relaxed_sys(p), v);
      __trap();
    }
  }
}

constexpr int kAggThreads = 256;
// entries per rank per aggregate chunk: 4096/n (>= one float4 per thread)
__host__ __device__ constexpr int agg_chunk(int n) { return 4096 / n > 1024 ? 4096 / n : 1024; }
// A-group ring bytes.  (A 32 KB ring at 2^13 tiles, n <= 4, so that a
// strided-pass CTA of the next bucket fits beside a fused CTA, made the fused
// kernel 86 -> 94 us per 2^23 bucket at N=2 and the step slower; two-stage
// strided passes beside the 64 KB ring: 0.492 -> 0.533 ms per resnet50 step.)
__host__ __device__ constexpr int agg_bytes(int, int) { return 64 * 1024; }

template <int T, int S, int NG, int NW>
__host__ __device__ constexpr size_t tma_fused_smem_bytes() {
  return (size_t)NG * S * tma_stage_bytes<T>() + agg_bytes(T, NW) + 512 + 1024;
}

enum FusedJob { FJ_END = -1, FJ_E = 0, FJ_D = 2, FJ_NOP = 3 };

template <int T, int kStages, int NW, int NG>
__global__ void __launch_bounds__(NG * (1 << (T - 5)) + kAggThreads)
    tma_fused_kernel(const __grid_constant__ TmaArgs ae, const __grid_constant__ TmaArgs ad,
                     const __grid_constant__ SnkBuf se, const __grid_constant__ SnkBuf sd,
                     const __grid_constant__ FusedArgs f) {
  constexpr int NED = 1 << (T - 5);
  constexpr size_t SB = tma_stage_bytes<T>();
  constexpr int kAggCh = agg_chunk(NW);
  constexpr int kAggBytes = agg_bytes(T, NW);
  constexpr int SA = kAggBytes / (NW * kAggCh * 4) < 16 ? kAggBytes / (NW * kAggCh * 4) : 16;
  // aggregate work unit = 1/UPT of a tile (finer units shorten the A tail);
  // a unit must cover every ring stage queued behind a not-ready unit
  constexpr int kCpt = (1 << T) / kAggCh;
  constexpr int UPT = kCpt / SA >= 4 ? 4 : (kCpt / SA >= 2 ? 2 : 1);
  constexpr int kCpu = kCpt / UPT;  // chunks per unit
  static_assert(NW >= 2 && SA >= 2, "aggregate ring needs two stages");
  extern __shared__ __align__(16) unsigned char smraw[];
  unsigned char* const base = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  float* const abuf = reinterpret_cast<float*>(base + (size_t)NG * kStages * SB);
  uint64_t* const full = reinterpret_cast<uint64_t*>(base + (size_t)NG * kStages * SB + kAggBytes);
  uint64_t* const abar = full + NG * kStages;
  int* const slot_kind = reinterpret_cast<int*>(abar + SA);                // [NG][4]
  int64_t* const slot_tile = reinterpret_cast<int64_t*>(slot_kind + NG * 4);  // [NG][4]
  int* const aslot = reinterpret_cast<int*>(slot_tile + NG * 4);  // A ring: (unit << 8 | chunk), -1 end
  uint32_t* const apres = reinterpret_cast<uint32_t*>(aslot + SA);  // A ring: ranks whose data the stage holds
  const int tid = threadIdx.x;
  constexpr int n = NW;
  const int me = f.me;
  const int64_t ns = f.ns;
  const uint64_t t_cta0 = globaltimer_ns();
  // owner of contiguous tile t (tiles of shard j are [j*ns, (j+1)*ns)); a
  // tile is published once its owner flagged every unit of it in this call
  auto owner_of = [&](int64_t t) { return shard_owner((int)(t / ns), f.r, NW); };
  auto published = [&](int64_t t) {
    const unsigned int* g = f.gflag[owner_of(t)] + t * 4;
    bool ok = true;
    for (int u = 0; u < UPT; ++u) ok = ok && ld_relaxed_sys(g + u) >= f.epoch;
    return ok;
  };
  if (f.stats && tid == 0) atomicMin(f.stats + ST_OPEN, (unsigned long long)t_cta0);

  if (tid == 0) {
    for (int s = 0; s < NG * kStages; ++s) mbar_init(&full[s], 1);
    for (int s = 0; s < SA; ++s) mbar_init(&abar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  // E/D warp group G (NG groups per CTA, independent rings / barriers / ticket
  // order positions; all claim from the same counter)
  auto ed_loop = [&](auto gc) {
    constexpr int G = decltype(gc)::value;
    constexpr int BARID = 1 + 2 * G;
    const int ltid = tid - G * NED;
    unsigned char* const gbase = base + (size_t)G * kStages * SB;
    uint64_t* const gfull = full + G * kStages;
    int* const gkind = slot_kind + G * 4;
    int64_t* const gtile = slot_tile + G * 4;
    // ------------------------------------------------ E/D warp group
    // tickets [0, n*ns): E in row order; [n*ns, 2*n*ns): D in row order (E
    // never queues behind a D; the D rows drain as the owners publish)
    const int64_t nt = (int64_t)n * ns;
    const int64_t total = 2 * nt;
    bool ended = false;
    unsigned deferred = 0;
    int64_t pend_e = -1;  // thread 0: encoded tile whose eflag is not yet released
    auto release_e = [&]() {
      if (pend_e >= 0) {
        __threadfence();  // release (see "Flags" above), cumulative over the group's stores before its barrier
        st_relaxed_sys(f.eflag[me] + pend_e, f.epoch);  // my own memory
        pend_e = -1;
      }
    };
    auto claim_issue = [&](int s) {
      int kind = FJ_END;
      int64_t t = 0;
      if (!ended) {
        const int64_t tk = atomicAdd(f.ctr, 1u);
        if (tk >= total) {
          ended = true;
        } else {
          const int64_t row = (tk % nt) / n;
          const int u = (int)(tk % n);
          kind = tk < nt ? FJ_E : FJ_D;
          t = (int64_t)u * ns + row;
        }
      }
      gkind[s] = kind;
      gtile[s] = t;
      if (kind == FJ_E) {
        tile_issue_contig<T, TS_BUF>(ae, me, t, gbase + s * SB, &gfull[s]);
      } else if (kind == FJ_D) {
        if (published(t)) {
          fence_acquire_sys();
          fence_proxy_async_global();
          tile_issue_contig<T, TS_GATHER>(ad, me, t, gbase + s * SB, &gfull[s]);
        } else {
          deferred |= 1u << s;
        }
      } else {
        mbar_arrive(&gfull[s]);  // no-op / end: nothing through the ring
      }
    };
    if (ltid == 0)
      for (int s = 0; s < kStages; ++s) claim_issue(s);
    uint4* const tr = (f.trace && G == 0) ? f.trace + (size_t)blockIdx.x * f.trace_cap : nullptr;
    for (int k = 0;; ++k) {
      const int s = k % kStages;
      unsigned char* const sb = gbase + s * SB;
      const uint32_t tb = tr && ltid == 0 ? (uint32_t)globaltimer_ns() : 0u;
      if (ltid == 0 && (deferred >> s & 1u)) {
        release_e();  // never wait while holding an unreleased encode
        const int64_t t = gtile[s];
        for (int u = 0; u < UPT; ++u) spin_ge_sys(f.gflag[owner_of(t)] + t * 4 + u, f.epoch, f.watchdog_ns);
        fence_acquire_sys();
        fence_proxy_async_global();
        tile_issue_contig<T, TS_GATHER>(ad, me, t, sb, &gfull[s]);
        deferred &= ~(1u << s);
      }
      mbar_wait(&gfull[s], (uint32_t)((k / kStages) & 1));
      const int kind = gkind[s];
      const int64_t t = gtile[s];
      if (kind == FJ_END) {
        if (ltid == 0) {
          release_e();
          if (f.stats) atomicMax(f.stats + ST_STAGE2, (unsigned long long)globaltimer_ns());
        }
        break;
      }
      if (ltid == 0 && kind != FJ_E) release_e();
      const uint32_t trd = tr && ltid == 0 ? (uint32_t)globaltimer_ns() : 0u;
      if (kind == FJ_E) {
        tma_tile<T, false, TS_BUF, SnkBuf, 3, BARID, G * NED>(nullptr, nullptr, ae, se.bind(me), me, nullptr, t, sb,
                                                 [&]() { claim_issue(s); });
        // released after the group's next job (or before any wait / exit), so
        // the fence finds the tile's stores drained instead of stalling on them
        group_sync<BARID, NED>();
        if (ltid == 0) {
          release_e();
          pend_e = t;
        }
      } else if (kind == FJ_D) {
        tma_tile<T, false, TS_GATHER, SnkBuf, 3, BARID, G * NED>(nullptr, nullptr, ad, sd.bind(me), me, nullptr, t, sb,
                                                    [&]() { claim_issue(s); }, NoEpi{},
                                                    gather_tile_all_kept<T>(ad, me, t));
      } else {
        // no-op ticket: every thread has read the slot (it is only rewritten
        // after this barrier)
        group_sync<BARID, NED>();
        if (ltid == 0) claim_issue(s);
      }
      if (tr && ltid == 0 && k < f.trace_cap / 2)
        tr[k] = make_uint4(((uint32_t)kind << 28) | (uint32_t)t, tb, trd, (uint32_t)globaltimer_ns());
    }
  };

  if (tid < NED) {
    ed_loop(std::integral_constant<int, 0>{});
  } else if (NG > 1 && tid < NG * NED) {
    ed_loop(std::integral_constant<int, (NG > 1 ? 1 : 0)>{});
  } else {
    // ------------------------------------------------ A warp group
    // TAR stage 1 + stage-2 push (collectives.py:113-137) of my shard's tiles
    const int ta = tid - NG * NED;
    const int64_t nunits = ns * UPT;
    const int64_t soff = (int64_t)f.own * f.shard_len;
    // producer state (ta == 0).  A new unit whose encodes are not all in is
    // not waited for here: its stages are queued (pend_*) and the wait
    // happens when the consumer reaches its first chunk, i.e. after the
    // previous unit is published (peers' E jobs may be queued behind D jobs
    // that wait for exactly that unit).
    int64_t cur = -1;  // current unit (tile-in-shard * UPT + part)
    int nxt = kCpu;    // next chunk of it to issue
    bool aend = false;
    int pend_first = -1, pend_count = 0;
    uint4* const tra = f.trace ? f.trace + (size_t)blockIdx.x * f.trace_cap + f.trace_cap / 2 : nullptr;
    int ntr = 0;
    uint32_t t_claim = 0, t_ready = 0;
    constexpr uint32_t kAll = (1u << NW) - 1u;
    uint32_t cur_present = kAll;  // ranks whose encoded unit `cur` is aggregated
    unsigned long long cut = 0;   // consumer: mask-delivered entries a deadline cut
    // wait for every rank's encoded tile t; past the deadline a peer that is
    // still missing is cut from the unit (never this rank's own tile)
    auto wait_present = [&](int64_t t) {
      uint32_t pres = 0;
      for (int q = 0; q < n; ++q) {
        const unsigned int* p = f.eflag[q] + t;
        if (q == me || f.deadline_ns == 0) {
          spin_ge_sys(p, f.epoch, f.watchdog_ns);
          pres |= 1u << q;
          continue;
        }
        const uint64_t end = t_cta0 + f.deadline_ns;
        while (ld_relaxed_sys(p) < f.epoch && globaltimer_ns() < end) __nanosleep(64);
        if (ld_relaxed_sys(p) >= f.epoch) pres |= 1u << q;
      }
      return pres;
    };
    auto tile_ready = [&](int64_t u) {
      const int64_t t = (int64_t)f.own * ns + u / UPT;
      unsigned int v[NW];
#pragma unroll
      for (int q = 0; q < n; ++q) v[q] = ld_relaxed_sys(f.eflag[q] + t);  // n polls in flight
      bool ok = true;
#pragma unroll
      for (int q = 0; q < n; ++q) ok = ok && v[q] >= f.epoch;
      return ok;
    };
    auto issue_chunk = [&](int s) {
      aslot[s] = (int)((cur << 8) | nxt);
      apres[s] = cur_present;
      const uint32_t bytes = kAggCh * sizeof(float);
      const int64_t e = ((cur / UPT) << T) + ((int64_t)(cur % UPT) * kCpu + nxt) * kAggCh;  // inside my shard
      mbar_expect_tx(&abar[s], bytes * (uint32_t)__popc(cur_present));
      for (int i = 0; i < n; ++i)
        if ((cur_present >> i) & 1u) bulk_load(abuf + ((size_t)s * n + i) * kAggCh, f.Y[i] + soff + e, bytes, &abar[s]);
      ++nxt;
    };
    auto decide = [&](uint32_t pres) {  // unit `cur`'s contributors are fixed
      cur_present = pres;
      if (f.cut_units && nxt == 0) f.cut_units[cur] = kAll & ~pres;
    };
    auto issue_next = [&](int s) {
      if (pend_first >= 0) {  // the queued unit takes this stage too (SA <= kCpu)
        ++pend_count;
        return;
      }
      if (!aend && nxt == kCpu) {
        const int64_t k = atomicAdd(f.ctr + 2, 1u);
        if (k >= nunits) {
          aend = true;
        } else {
          cur = k;
          nxt = 0;
          if (tra) t_claim = (uint32_t)globaltimer_ns();
          if (!tile_ready(k)) {
            pend_first = s;
            pend_count = 1;
            return;
          }
          decide(kAll);
          if (tra) t_ready = (uint32_t)globaltimer_ns();
          fence_acquire_sys();
          fence_proxy_async_global();
        }
      }
      if (aend) {
        aslot[s] = -1;
        mbar_arrive(&abar[s]);
        return;
      }
      issue_chunk(s);
    };
    if (ta == 0)
      for (int s = 0; s < SA; ++s) issue_next(s);
    static_assert(SA <= kCpu, "a queued unit covers every queued stage");
    static_assert(kAggCh % (4 * kAggThreads) == 0, "whole float4 groups per thread");
    for (int k = 0;; ++k) {
      const int s = k % SA;
      if (ta == 0 && s == pend_first) {
        const int64_t t = (int64_t)f.own * ns + cur / UPT;
        decide(wait_present(t));
        if (tra) t_ready = (uint32_t)globaltimer_ns();
        fence_acquire_sys();
        fence_proxy_async_global();
        const int first = pend_first, cnt = pend_count;
        pend_first = -1;
        pend_count = 0;
        for (int i = 0; i < cnt; ++i) issue_chunk((first + i) % SA);
      }
      mbar_wait(&abar[s], (uint32_t)((k / SA) & 1));
      const int code = aslot[s];
      if (code < 0) break;
      const int64_t un = code >> 8;  // unit
      const int chunk = code & 255;  // chunk inside the unit
      const uint32_t pres = apres[s];
#pragma unroll
      for (int v = 0; v < kAggCh / (4 * kAggThreads); ++v) {
        const int off = 4 * (ta + v * kAggThreads);
        const int64_t e = ((un / UPT) << T) + ((int64_t)(un % UPT) * kCpu + chunk) * kAggCh + off;
        const float* src = abuf + (size_t)s * n * kAggCh + off;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        uint32_t c4[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int i = 0; i < n; ++i) {
          const float4 x4 = *reinterpret_cast<const float4*>(src + (size_t)i * kAggCh);
          uint32_t kk = i == me ? 0xFu : keep4(f.m.row(0, me, i), (uint32_t)e, f.m);
          if (!((pres >> i) & 1u)) {  // cut by the stage-1 deadline: a miss
            cut += (unsigned long long)__popc(kk);
            kk = 0u;
          }
          acc[0] += (kk & 1u) ? (double)x4.x : 0.0;  // misses add +0.0 like the reference
          acc[1] += (kk & 2u) ? (double)x4.y : 0.0;
          acc[2] += (kk & 4u) ? (double)x4.z : 0.0;
          acc[3] += (kk & 8u) ? (double)x4.w : 0.0;
          c4[0] += kk & 1u;
          c4[1] += (kk >> 1) & 1u;
          c4[2] += (kk >> 2) & 1u;
          c4[3] += (kk >> 3) & 1u;
        }
        const float4 res = make_float4(mean_of(acc[0], (double)c4[0]), mean_of(acc[1], (double)c4[1]),
                                       mean_of(acc[2], (double)c4[2]), mean_of(acc[3], (double)c4[3]));
        st4(f.A[me] + e, res);  // my shard's aggregate; peers pull it in their D jobs
      }
      const bool last = chunk == kCpu - 1;
      group_sync<2, kAggThreads>();  // stage s consumed (and the unit's results stored, when last)
      if (ta == 0) {
        if (last) {
          __threadfence();  // release (see "Flags" above): the group's results before the flag
          const int64_t t = (int64_t)f.own * ns + un / UPT;
          st_relaxed_sys(f.gflag[me] + t * 4 + un % UPT, f.epoch);  // my own memory
          if (tra && ntr < f.trace_cap / 2)
            tra[ntr++] = make_uint4((1u << 28) | (uint32_t)t, t_claim, t_ready, (uint32_t)globaltimer_ns());
        }
        issue_next(s);
      }
    }
    if (f.stats) {
      if (cut) atomicAdd(f.stats + ST_CUT0, cut);
      if (ta == 0) atomicMax(f.stats + ST_STAGE1, (unsigned long long)globaltimer_ns());
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned int prev = atomicAdd(f.ctr + 1, 1u);
    if (prev == gridDim.x - 1) {
      f.ctr[0] = 0;
      f.ctr[1] = 0;
      f.ctr[2] = 0;
      if (f.stats) {  // last CTA out: received = mask-model counts - deadline cuts
        f.stats[ST_RECV0] = f.counts[me] - f.stats[ST_CUT0];
        f.stats[ST_RECV1] = f.counts[n + me] - f.stats[ST_CUT1];
      }
      __threadfence();
    }
  }
}

}  // namespace optr
