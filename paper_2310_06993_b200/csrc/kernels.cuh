// Device kernels of the TAR+RHT hot path (sm_100a).
//
//   prep_kernel       Rademacher sign bits (hadamard.py:49-51), drop-mask packet
//                     bitmaps (datagram.py:70-72,117-124 coin or caller bitmaps),
//                     per-(stage,dst) received counts (simdriver.py:328-341).
//   rtile_kernel      one pass of the Sylvester FWHT (hadamard.py:76-90) over a
//                     2^T-entry tile held in registers (32 per thread) with two
//                     shared-memory transposes; H_D is the product of passes over
//                     disjoint index-bit ranges.  The encode sign/pad/cast is fused
//                     into the first pass, the decode gather/mask/scale/sign/
//                     truncate/cast into the first and last passes.
//   smem_tile_kernel  the same for small tiles (D < 2^10), shared-memory rounds.
//   aggregate_kernel  TAR stage-1 owner mean (collectives.py:77-94,125): fp64
//                     accumulate in ascending node order under stage-1 masks.
//   assemble_kernel   TAR stage-2 assembly without RHT (collectives.py:140-150).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "../../include/optr.h"
#include "pcg.h"

namespace optr {

constexpr int kMaxW = OPTR_MAX_WORKERS;

// ------------------------------------------------------------------ geometry
// Shard split of a `len`-entry vector over n owners (wire.py:121-133): the
// first `extra` shards hold base+1 entries.
struct Shards {
  int64_t base;
  int64_t extra;
  int n;
  __host__ __device__ __forceinline__ int64_t len(int j) const { return base + (j < extra ? 1 : 0); }
  __host__ __device__ __forceinline__ int64_t off(int j) const {
    return (int64_t)j * base + (j < extra ? j : extra);
  }
  // shard containing entry g (g < total): estimate in double, then correct
  __host__ __device__ __forceinline__ int of(int64_t g) const {
    int j = (int)((double)g / (double)(base + 1));
    if (j > n - 1) j = n - 1;
    while (j > 0 && off(j) > g) --j;
    while (j < n - 1 && off(j + 1) <= g) ++j;
    return j;
  }
};

__host__ __device__ __forceinline__ Shards make_shards(int64_t len, int n) {
  Shards s;
  s.base = len / n;
  s.extra = len % n;
  s.n = n;
  return s;
}

__host__ __device__ __forceinline__ int owned_shard(int node, int r, int n) {  // schedule.py:47-49
  return ((node - r) % n + n) % n;
}
__host__ __device__ __forceinline__ int shard_owner(int j, int r, int n) {  // schedule.py:42-44
  return (j + r) % n;
}
__host__ __device__ __forceinline__ int64_t n_packets(int64_t len, int epp) {
  return len > 0 ? (len + epp - 1) / epp : 0;
}

// Exact e / d for 32-bit e via a 64-bit multiply-high: q = umulhi64(e, M),
// M = ceil(2^64 / d); the error e(Md - 2^64)/(d 2^64) < e/2^64 < 1/d.
struct Divider {
  uint64_t m;  // 0 when d == 1
  __device__ __forceinline__ uint32_t div(uint32_t e) const {
    return m ? (uint32_t)__umul64hi((unsigned long long)e, (unsigned long long)m) : e;
  }
};
inline Divider make_divider(uint32_t d) {
  Divider v;
  if (d <= 1) {
    v.m = 0;
  } else {
    unsigned __int128 one = (unsigned __int128)1 << 64;
    v.m = (uint64_t)((one + d - 1) / d);
  }
  return v;
}

// Packet-bitmap addressing (optr.h): stage 0/1, receiver dst, sender src.
struct MaskView {
  const uint32_t* bits;
  int64_t pw;  // u32 words per pair
  int n;
  int epp;
  Divider dv;  // division by epp
  __device__ __forceinline__ const uint32_t* row(int stage, int dst, int src) const {
    return bits + ((int64_t)(stage * n + dst) * n + src) * pw;
  }
};

__device__ __forceinline__ bool row_bit(const uint32_t* row, uint32_t pkt) {
  return (__ldg(row + (pkt >> 5)) >> (pkt & 31)) & 1u;
}

// Keep-flags (bit c = entry e+c delivered) of 4 consecutive shard entries
// e..e+3 from a packet bitmap row: one word load, one packet boundary at most
// when epp >= 4.
__device__ __forceinline__ uint32_t keep4(const uint32_t* row, uint32_t e, const MaskView& m) {
  const uint32_t epp = (uint32_t)m.epp;
  if (epp >= 4) {
    const uint32_t p0 = m.dv.div(e), rem = e - p0 * epp;
    const uint32_t w = __ldg(row + (p0 >> 5)) >> (p0 & 31);
    const uint32_t b0 = w & 1u;
    if (rem + 3 < epp) return b0 ? 0xFu : 0u;
    const uint32_t b1 = (p0 & 31) == 31 ? (__ldg(row + (p0 >> 5) + 1) & 1u) : ((w >> 1) & 1u);
    const uint32_t split = epp - rem;  // entries 0..split-1 in p0, the rest in p0+1
    const uint32_t lo = (1u << split) - 1u;
    return (b0 ? lo : 0u) | (b1 ? (0xFu & ~lo) : 0u);
  }
  uint32_t k = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) k |= (row_bit(row, (e + c) / epp) ? 1u : 0u) << c;
  return k;
}

// True when every packet covering shard entries [e0, e0 + len) is delivered
// (uniform per tile: the per-entry mask work is skipped).
__device__ __forceinline__ bool packets_all_kept(const uint32_t* row, uint32_t e0, uint32_t len, const MaskView& m) {
  const uint32_t p0 = m.dv.div(e0), p1 = m.dv.div(e0 + len - 1);
  for (uint32_t w = p0 >> 5; w <= (p1 >> 5); ++w) {
    uint32_t need = 0xffffffffu;
    if (w == (p0 >> 5)) need &= 0xffffffffu << (p0 & 31);
    if (w == (p1 >> 5)) need &= 0xffffffffu >> (31 - (p1 & 31));
    if ((__ldg(row + w) & need) != need) return false;
  }
  return true;
}

// keep-flag nibble -> one count byte per entry (entries 0..3 of a float4)
__device__ __forceinline__ uint32_t nibble_bytes(uint32_t kk) {
  return (kk & 1u) | ((kk & 2u) << 7) | ((kk & 4u) << 14) | ((kk & 8u) << 21);
}

// packet index of entries e..e+3 of a shard (epp = entries per packet)
struct Pkt4 {
  uint32_t p[4];
};
__device__ __forceinline__ Pkt4 pkt4(uint32_t e, uint32_t epp) {
  Pkt4 r;
  uint32_t p0 = e / epp;
  uint32_t rem = e - p0 * epp;
  if (epp >= 4) {
#pragma unroll
    for (int m = 0; m < 4; ++m) r.p[m] = p0 + (rem + m >= epp ? 1u : 0u);
  } else {
#pragma unroll
    for (int m = 0; m < 4; ++m) r.p[m] = p0 + (rem + m) / epp;
  }
  return r;
}

// -------------------------------------------------------------------- prep
// LCG jump table: advancing 2^i steps maps s -> A_i s + inc * G_i.
struct JumpTable {
  u128 a[64];
  u128 g[64];
};
__constant__ JumpTable c_jump;

inline JumpTable make_jump_table() {
  JumpTable t;
  u128 a = pcg_mult(), g = 1;
  for (int i = 0; i < 64; ++i) {
    t.a[i] = a;
    t.g[i] = g;
    g = g * (a + 1);
    a = a * a;
  }
  return t;
}

// state after k steps from s (table-driven; uniform loop over the bit index
// so the constant-bank reads broadcast across the warp)
__device__ __forceinline__ u128 jump(u128 s, u128 inc, uint64_t k) {
  int top = 64 - __clzll((long long)(k | 1));
  for (int i = 0; i < top; ++i) {
    if ((k >> i) & 1) s = c_jump.a[i] * s + inc * c_jump.g[i];
  }
  return s;
}

struct PrepArgs {
  // signs: each thread writes 4 words = 128 signs = 64 PCG outputs
  uint32_t* signs;
  int64_t dim;
  u128 sign_state, sign_inc;
  int64_t sign_threads;
  // optional second layout for strided passes (tma.cuh): sign byte of
  // entries row*2^t_lo + 8*cg .. +7 at signs_t[cg * 2^t_ks + row]
  uint8_t* signs_t;
  int t_lo, t_ks;
  // masks
  int kind;
  int n, r, epp;
  Shards sh;
  int64_t pw;
  uint32_t* bitmap_out;       // COIN / NONE: written here
  const uint32_t* bitmap_in;  // BITMAP: read from here
  u128 coin_state[kMaxW];
  u128 coin_inc[kMaxW];
  double drop_prob;
  int dst_lo, dst_hi;
  int64_t mask_threads;
  unsigned long long* counts;  // [2][n] received entries per (stage,dst)
  // optional per-tile summaries of the masks (tiles of 2^tile_shift vector
  // entries, preset to all ones): tile_ok[stage * ntiles + t] bit i is
  // cleared when a packet over tile t is lost -- stage 1: from sender i to
  // the tile's owner; stage 2: from the tile's owner to receiver i
  uint32_t* tile_ok;
  int tile_shift;
  int64_t ntiles;
};

constexpr int kSignsPerThread = 128;

// Running packet index of sender `src`'s first packet to `dst` in `stage`
// (datagram.py:117-124 draws one coin per packet in send order: stage 1 to
// dst = src+1..src+n-1 (schedule.py:67-78) then stage 2 the same order).
__device__ __forceinline__ uint64_t coin_base(const PrepArgs& a, int stage, int src, int dst) {
  int n = a.n;
  int o = ((dst - src) % n + n) % n;
  uint64_t base = 0;
  if (stage == 0) {
    for (int k = 1; k < o; ++k) base += n_packets(a.sh.len(owned_shard((src + k) % n, a.r, n)), a.epp);
  } else {
    for (int k = 1; k < n; ++k) base += n_packets(a.sh.len(owned_shard((src + k) % n, a.r, n)), a.epp);
    base += (uint64_t)(o - 1) * n_packets(a.sh.len(owned_shard(src, a.r, n)), a.epp);
  }
  return base;
}

__device__ __forceinline__ void prep_item(const PrepArgs& a, int64_t t);

// One work item per thread; a capped grid strides over the items (the
// multi-GPU path runs prep as a thin background kernel on a side stream).
// (translation units that only need the device helpers -- small.cu --
// define OPTR_NO_GLOBAL_KERNELS: the non-template kernels live in api.cu)
#ifndef OPTR_NO_GLOBAL_KERNELS
__global__ void __launch_bounds__(256) prep_kernel(const __grid_constant__ PrepArgs a) {
  const int64_t total = a.sign_threads + a.mask_threads;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x)
    prep_item(a, t);
}
#endif

__device__ __forceinline__ void prep_item(const PrepArgs& a, int64_t t) {
  if (t < a.sign_threads) {
    // signs 128c .. 128c+127 = outputs 64c .. 64c+63; Lemire bit of u32 halves.
    // Natural layout: chunk c = t.  With the transposed layout too, a warp
    // takes 32 consecutive rows of one 128-column chunk (coalesced bytes).
    int64_t c = t, row = 0, cg16 = 0;
    if (a.signs_t) {
      const int64_t rows = 1LL << a.t_ks;
      const int64_t w = t >> 5;
      row = ((w % (rows >> 5)) << 5) | (t & 31);
      cg16 = w / (rows >> 5);
      c = ((row << a.t_lo) >> 7) + cg16;
    }
    u128 s = jump(a.sign_state, a.sign_inc, (uint64_t)c * 64 + 1);
    const int64_t nwords = (a.dim + 31) >> 5;
    const int64_t w0 = c * 4;
#pragma unroll
    for (int wd = 0; wd < 4; ++wd) {
      uint32_t word = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        uint64_t out = pcg_xsl_rr(s);
        word |= (uint32_t)((out >> 31) & 1u) << (2 * i);
        word |= (uint32_t)(out >> 63) << (2 * i + 1);
        s = pcg_step(s, a.sign_inc);
      }
      int64_t wi = w0 + wd;
      if (wi < nwords) {
        int64_t valid = a.dim - wi * 32;  // zero the bits past dim
        if (valid < 32) word &= (1u << valid) - 1u;
        a.signs[wi] = word;
        if (a.signs_t) {
          const int64_t rows = 1LL << a.t_ks;
#pragma unroll
          for (int b = 0; b < 4; ++b)
            a.signs_t[(cg16 * 16 + wd * 4 + b) * rows + row] = (uint8_t)(word >> (8 * b));
        }
      }
    }
    return;
  }
  t -= a.sign_threads;
  if (t >= a.mask_threads) return;
  // one thread per bitmap word of one (stage, dst, src) pair
  int per_dst = 2 * (a.n - 1);
  int64_t pair = t / a.pw;
  int64_t word = t - pair * a.pw;
  int dsti = (int)(pair / per_dst);
  int rem = (int)(pair - (int64_t)dsti * per_dst);
  int stage = rem / (a.n - 1);
  int srci = rem - stage * (a.n - 1);
  int dst = a.dst_lo + dsti;
  int src = srci < dst ? srci : srci + 1;
  int j = stage == 0 ? owned_shard(dst, a.r, a.n) : owned_shard(src, a.r, a.n);
  int64_t len = a.sh.len(j);
  int64_t np = n_packets(len, a.epp);
  int64_t p0 = word * 32;
  int64_t idx = ((int64_t)(stage * a.n + dst) * a.n + src) * a.pw + word;
  uint32_t bits = 0;
  int64_t rem_p = np - p0;
  int cnt = rem_p <= 0 ? 0 : (rem_p >= 32 ? 32 : (int)rem_p);
  if (a.kind == OPTR_MASK_COIN) {
    if (cnt > 0) {
      uint64_t k = coin_base(a, stage, src, dst) + (uint64_t)p0;
      u128 s = jump(a.coin_state[src], a.coin_inc[src], k + 1);
      for (int i = 0; i < cnt; ++i) {
        if (!coin_drops(pcg_xsl_rr(s), a.drop_prob)) bits |= 1u << i;
        s = pcg_step(s, a.coin_inc[src]);
      }
    }
    a.bitmap_out[idx] = bits;
  } else if (a.kind == OPTR_MASK_BITMAP) {
    bits = cnt > 0 ? a.bitmap_in[idx] : 0u;
    if (cnt < 32) bits &= (cnt > 0 ? ((1u << cnt) - 1u) : 0u);
  } else {
    bits = cnt >= 32 ? 0xffffffffu : (cnt > 0 ? ((1u << cnt) - 1u) : 0u);
    a.bitmap_out[idx] = bits;
  }
  if (a.tile_ok && cnt > 0) {
    uint32_t lost = ~bits & (cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u));
    const int64_t off = a.sh.off(j);
    const uint32_t bit = 1u << (stage == 0 ? src : dst);
    while (lost) {  // rare: one atomic per lost packet per tile it touches
      const int b = __ffs(lost) - 1;
      lost &= lost - 1;
      const int64_t e_lo = off + (p0 + b) * a.epp;
      const int64_t e_hi = off + ((p0 + b + 1) * a.epp < len ? (p0 + b + 1) * a.epp : len) - 1;
      for (int64_t tt = e_lo >> a.tile_shift; tt <= (e_hi >> a.tile_shift); ++tt)
        atomicAnd(a.tile_ok + stage * a.ntiles + tt, ~bit);
    }
  }
  if (bits) {
    unsigned long long e = (unsigned long long)__popc(bits) * (unsigned long long)a.epp;
    // the last packet of a transfer is short (simdriver.py:188-189)
    if (p0 + cnt == np && ((bits >> (cnt - 1)) & 1u)) e -= (unsigned long long)(np * a.epp - len);
    atomicAdd(a.counts + stage * a.n + dst, e);
  }
}

// ------------------------------------------------------ element helpers
__device__ __forceinline__ float load_elem(const void* p, int dtype, int64_t g) {
  if (dtype == OPTR_BF16) return __bfloat162float(((const __nv_bfloat16*)p)[g]);
  return ((const float*)p)[g];
}
__device__ __forceinline__ void store_elem(void* p, int dtype, int64_t g, float v) {
  if (dtype == OPTR_BF16)
    ((__nv_bfloat16*)p)[g] = __float2bfloat16_rn(v);
  else
    ((float*)p)[g] = v;
}
__device__ __forceinline__ float sgn(uint32_t word, int bit, float v) {
  return ((word >> bit) & 1u) ? v : -v;
}
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

// --------------------------------------------------- sources and sinks
// Each parameter struct binds to one worker (`bind(w)`) to give a small
// register-resident view with load4 / store{1,2,4} on global indices.

// pad(x) * signs   (hadamard.py:98-100)
struct SrcEncode {
  const void* x[kMaxW];
  int dtype;
  int64_t L;
  const uint32_t* signs;
  const uint8_t* signs_t;  // optional transposed sign bytes (strided TMA pass, PrepArgs)
  struct B {
    const void* x;
    int dtype;
    int64_t L;
    const uint32_t* signs;
    __device__ __forceinline__ void begin_tile(int64_t, int64_t) {}
    __device__ __forceinline__ float load1(int64_t g) const {
      if (g >= L) return 0.f;
      return sgn(__ldg(signs + (g >> 5)), (int)(g & 31), load_elem(x, dtype, g));
    }
    // vector loads need x 16-byte (fp32) / 8-byte (bf16) aligned
    __device__ __forceinline__ bool vec_ok() const {
      return (((uintptr_t)x) & (dtype == OPTR_F32 ? 15 : 7)) == 0;
    }
    __device__ __forceinline__ float4 load4(int64_t g) const {
      if (g + 4 <= L && vec_ok()) {
        float4 v;
        if (dtype == OPTR_F32) {
          v = ldg4((const float*)x + g);
        } else {
          uint2 u = __ldg(reinterpret_cast<const uint2*>((const __nv_bfloat16*)x + g));
          __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&u.x);
          __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&u.y);
          float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
          v = make_float4(fa.x, fa.y, fb.x, fb.y);
        }
        uint32_t w = __ldg(signs + (g >> 5));
        int b0 = (int)(g & 31);
        v.x = sgn(w, b0, v.x);
        v.y = sgn(w, b0 + 1, v.y);
        v.z = sgn(w, b0 + 2, v.z);
        v.w = sgn(w, b0 + 3, v.w);
        return v;
      }
      return make_float4(load1(g), load1(g + 1), load1(g + 2), load1(g + 3));
    }
  };
  __device__ __forceinline__ B bind(int w) const { return B{x[w], dtype, L, signs}; }
};

struct SrcBuf {
  float* y[kMaxW];
  struct B {
    const float* y;
    __device__ __forceinline__ void begin_tile(int64_t, int64_t) {}
    __device__ __forceinline__ float load1(int64_t g) const { return y[g]; }
    __device__ __forceinline__ float4 load4(int64_t g) const { return ld4(y + g); }
  };
  __device__ __forceinline__ B bind(int w) const { return B{y[w]}; }
};

// where(mask, y, 0) with a byte mask (hadamard.py:120)
struct SrcMasked {
  const float* y;
  const uint8_t* mask;
  struct B {
    const float* y;
    const uint8_t* mask;
    __device__ __forceinline__ void begin_tile(int64_t, int64_t) {}
    __device__ __forceinline__ float load1(int64_t g) const {
      return (mask == nullptr || mask[g]) ? y[g] : 0.f;
    }
    __device__ __forceinline__ float4 load4(int64_t g) const {
      return make_float4(load1(g), load1(g + 1), load1(g + 2), load1(g + 3));
    }
  };
  __device__ __forceinline__ B bind(int) const { return B{y, mask}; }
};

// received flags of 4 consecutive entries (the row base q*dim may be odd)
__device__ __forceinline__ void put_got(uint8_t* p, bool a, bool b, bool c, bool d) {
  if ((((uintptr_t)p) & 3) == 0) {
    *reinterpret_cast<uchar4*>(p) = make_uchar4(a, b, c, d);
  } else {
    p[0] = a;
    p[1] = b;
    p[2] = c;
    p[3] = d;
  }
}

// TAR stage-2 receive of worker q (collectives.py:140-150): own shard from
// its own aggregate, peer shards from the owner's aggregate (peer-mapped in
// the multi-GPU path) under the stage-2 mask, zero-filled misses.
struct SrcGather {
  const float* A[kMaxW];
  Shards sh;
  int n, r;
  MaskView m;
  uint8_t* got;  // optional [n][dim]
  int64_t dim;
  int pow2_shift;  // log2(shard length) when all shards are one power of two, else -1
  const uint32_t* tile_ok2;  // optional stage-2 tile summaries (TMA contiguous passes)
  struct B {
    const SrcGather* p;  // param space
    int q;
    // tile-uniform shard (fast path)
    int uj;
    const float* ua;
    const uint32_t* urow;
    int64_t uoff;
    __device__ __forceinline__ void begin_tile(int64_t g0, int64_t g1) {
      int j0 = p->sh.of(g0), j1 = p->sh.of(g1);
      uj = j0 == j1 ? j0 : -1;
      if (uj >= 0 && (((uintptr_t)p->A[shard_owner(uj, p->r, p->n)]) & 15)) uj = -1;  // float4 needs 16B
      if (uj >= 0) {
        int owner = shard_owner(uj, p->r, p->n);
        uoff = p->sh.off(uj);
        ua = p->A[owner] - uoff;
        urow = owner == q ? nullptr : p->m.row(1, q, owner);
      }
    }
    __device__ __forceinline__ float load1(int64_t g) const {
      int j = p->sh.of(g);
      int64_t e = g - p->sh.off(j);
      int owner = shard_owner(j, p->r, p->n);
      bool ok = owner == q ? true : row_bit(p->m.row(1, q, owner), (uint32_t)e / (uint32_t)p->m.epp);
      if (p->got) p->got[(int64_t)q * p->dim + g] = ok ? 1 : 0;
      return ok ? p->A[owner][e] : 0.f;
    }
    // 4 consecutive entries inside one shard, e = offset of the first
    __device__ __forceinline__ float4 load4_in(const float* a, const uint32_t* row, uint32_t e, int64_t g) const {
      float4 v = ldg4(a + e);
      if (row) {
        const uint32_t kk = keep4(row, e, p->m);
        const bool k0 = kk & 1u, k1 = kk & 2u, k2 = kk & 4u, k3 = kk & 8u;
        v.x = k0 ? v.x : 0.f;
        v.y = k1 ? v.y : 0.f;
        v.z = k2 ? v.z : 0.f;
        v.w = k3 ? v.w : 0.f;
        if (p->got) put_got(p->got + (int64_t)q * p->dim + g, k0, k1, k2, k3);
      } else if (p->got) {
        put_got(p->got + (int64_t)q * p->dim + g, true, true, true, true);
      }
      return v;
    }
    __device__ __forceinline__ float4 load4(int64_t g) const {
      if (uj >= 0 && ((g - uoff) & 3) == 0) return load4_in(ua + uoff, urow, (uint32_t)(g - uoff), g);
      if (p->pow2_shift >= 0) {  // equal power-of-two shards (pow2 dim, pow2 n)
        const int j = (int)(g >> p->pow2_shift);
        const uint32_t e = (uint32_t)(g & ((1LL << p->pow2_shift) - 1));
        if ((e & 3) == 0 && (int64_t)e + 4 <= (1LL << p->pow2_shift)) {
          const int owner = shard_owner(j, p->r, p->n);
          return load4_in(p->A[owner], owner == q ? nullptr : p->m.row(1, q, owner), e, g);
        }
      } else {  // general ceil split: one shard lookup per group
        const int j = p->sh.of(g);
        const int64_t e = g - p->sh.off(j);
        const int owner = shard_owner(j, p->r, p->n);
        if ((e & 3) == 0 && e + 4 <= p->sh.len(j) && (((uintptr_t)p->A[owner]) & 15) == 0)
          return load4_in(p->A[owner], owner == q ? nullptr : p->m.row(1, q, owner), (uint32_t)e, g);
      }
      return make_float4(load1(g), load1(g + 1), load1(g + 2), load1(g + 3));
    }
  };
  __device__ __forceinline__ B bind(int q) const {
    B b;
    b.p = this;
    b.q = q;
    b.uj = -1;
    b.ua = nullptr;
    b.urow = nullptr;
    b.uoff = 0;
    return b;
  }
};

struct SnkBuf {
  float* y[kMaxW];
  float scale;
  struct B {
    float* y;
    float scale;
    __device__ __forceinline__ void store1(int64_t g, float v) const { y[g] = v * scale; }
    __device__ __forceinline__ void store2(int64_t g, float a, float b) const {
      *reinterpret_cast<float2*>(y + g) = make_float2(a * scale, b * scale);
    }
    __device__ __forceinline__ void store4(int64_t g, float4 v) const {
      st4(y + g, make_float4(v.x * scale, v.y * scale, v.z * scale, v.w * scale));
    }
  };
  __device__ __forceinline__ B bind(int w) const { return B{y[w], scale}; }
};

// signs * v * (dim/count)/sqrt(dim), truncated to L, cast (hadamard.py:116-123,
// runner.py:253-256: count 0 -> zeros).
struct SnkDecode {
  void* out[kMaxW];
  int dtype;
  int64_t L;
  const uint32_t* signs;
  const uint8_t* signs_t;  // optional transposed sign bytes (strided TMA pass, PrepArgs)
  const unsigned long long* count_extra;  // device: + received entries (may be null)
  int64_t count_base[kMaxW];              // host-known part of count
  int count_stride;
  double dim;
  struct B {
    void* out;
    int dtype;
    int64_t L;
    const uint32_t* signs;
    float scale;
    __device__ __forceinline__ void store1(int64_t g, float v) const {
      if (g >= L) return;
      store_elem(out, dtype, g, sgn(__ldg(signs + (g >> 5)), (int)(g & 31), v * scale));
    }
    // vector stores need out 16-byte (fp32 x4) / 8-byte aligned
    __device__ __forceinline__ bool vec_ok(int bytes) const { return (((uintptr_t)out) & (bytes - 1)) == 0; }
    __device__ __forceinline__ void store2(int64_t g, float a, float b) const {
      if (g + 2 <= L && vec_ok(dtype == OPTR_F32 ? 8 : 4)) {
        uint32_t w = __ldg(signs + (g >> 5));
        int b0 = (int)(g & 31);
        a = sgn(w, b0, a * scale);
        b = sgn(w, b0 + 1, b * scale);
        if (dtype == OPTR_F32)
          *reinterpret_cast<float2*>((float*)out + g) = make_float2(a, b);
        else
          *reinterpret_cast<__nv_bfloat162*>((__nv_bfloat16*)out + g) = __floats2bfloat162_rn(a, b);
        return;
      }
      store1(g, a);
      store1(g + 1, b);
    }
    __device__ __forceinline__ void store4(int64_t g, float4 v) const {
      if (g + 4 <= L && vec_ok(dtype == OPTR_F32 ? 16 : 8)) {
        uint32_t w = __ldg(signs + (g >> 5));
        int b0 = (int)(g & 31);
        v.x = sgn(w, b0, v.x * scale);
        v.y = sgn(w, b0 + 1, v.y * scale);
        v.z = sgn(w, b0 + 2, v.z * scale);
        v.w = sgn(w, b0 + 3, v.w * scale);
        if (dtype == OPTR_F32) {
          st4((float*)out + g, v);
        } else {
          __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
          uint2 u;
          u.x = *reinterpret_cast<uint32_t*>(&a);
          u.y = *reinterpret_cast<uint32_t*>(&b);
          *reinterpret_cast<uint2*>((__nv_bfloat16*)out + g) = u;
        }
        return;
      }
      store1(g, v.x);
      store1(g + 1, v.y);
      store1(g + 2, v.z);
      store1(g + 3, v.w);
    }
  };
  __device__ __forceinline__ B bind(int w) const {
    unsigned long long c = (unsigned long long)count_base[w];
    if (count_extra) c += count_extra[w * count_stride];
    float s = c == 0 ? 0.f : (float)((dim / (double)c) / sqrt(dim));
    return B{out[w], dtype, L, signs, s};
  }
};

// ------------------------------------------------------------ tile geometry
// A pass transforms index bits [lo, lo+ks) of the vector.  A tile holds
// 2^(cb+ks) entries: tile bits [0,cb) are untransformed columns (vector bits
// [0,cb), contiguous), tile bits [cb, cb+ks) are the transformed bits.  Tile
// t covers column group t mod 2^(lo-cb) of outer block t >> (lo-cb).
struct PassGeom {
  int lo, ks, cb;
  int64_t ntiles;
};

__device__ __forceinline__ int64_t tile_origin(const PassGeom& pg, int64_t t) {
  const int cgb = pg.lo - pg.cb;
  const int64_t cgroup = t & ((1LL << cgb) - 1);
  const int64_t outer = t >> cgb;
  return (outer << (pg.lo + pg.ks)) + (cgroup << pg.cb);
}
__device__ __forceinline__ int64_t tile_remap(const PassGeom& pg, int i) {
  return ((int64_t)(i >> pg.cb) << pg.lo) | (int64_t)(i & ((1 << pg.cb) - 1));
}

// Shared-memory bank swizzle of the small-tile kernel: XOR index bits 0-4
// with bits 5-9 (conflict-free when warp lanes sit on five tile bits < 10
// that are distinct mod 5).
__device__ __forceinline__ int swz(int i) { return i ^ ((i >> 5) & 31); }

// ---------------------------------------------- register-layout tile FWHT
// Plan: round 0 holds tile bits {0,1,T-3,T-2,T-1} in registers (float4
// global loads); each later round holds up to 5 more transform bits, moved
// through shared memory; the last round also holds bits 0(,1) when it can,
// for vector stores.  (Prototyped and checked in numpy.)
struct RPlan {
  int nr;
  int pos[4][5];
  unsigned xm[4];
};

__host__ __device__ constexpr RPlan make_rplan(int T, int CB) {
  RPlan p{};
  bool done[32] = {};
  const int A[5] = {0, 1, T - 3, T - 2, T - 1};
  unsigned x0 = 0;
  for (int k = 0; k < 5; ++k) {
    p.pos[0][k] = A[k];
    if (A[k] >= CB) {
      x0 |= 1u << k;
      done[A[k]] = true;
    }
  }
  p.xm[0] = x0;
  p.nr = 1;
  int rem[32] = {};
  int nrem = 0;
  for (int b = CB; b < T; ++b)
    if (!done[b]) rem[nrem++] = b;
  int ri = 0;
  while (ri < nrem && p.nr < 4) {
    int cur[5] = {};
    int nc = 0;
    while (nc < 5 && ri < nrem) cur[nc++] = rem[ri++];
    const bool last = ri >= nrem;
    int pos[5] = {};
    int np = 0;
    if (last) {
      if (nc <= 3) {
        pos[np++] = 0;
        pos[np++] = 1;
      } else if (nc == 4) {
        pos[np++] = 0;
      }
    }
    for (int c = 0; c < nc; ++c) pos[np++] = cur[c];
    for (int b = 0; b < T && np < 5; ++b) {
      bool in = false;
      for (int q = 0; q < np; ++q) in = in || pos[q] == b;
      if (!in) pos[np++] = b;
    }
    unsigned x = 0;
    for (int k = 0; k < 5; ++k) {
      p.pos[p.nr][k] = pos[k];
      for (int c = 0; c < nc; ++c)
        if (pos[k] == cur[c]) x |= 1u << k;
    }
    p.xm[p.nr] = x;
    p.nr++;
  }
  return p;
}

// tile offset of register j in round r
__host__ __device__ constexpr int roff(const RPlan& p, int r, int j) {
  int o = 0;
  for (int k = 0; k < 5; ++k)
    if ((j >> k) & 1) o |= 1 << p.pos[r][k];
  return o;
}

// tile offset contributed by the thread id in round r (thread bits ascend
// over the positions not held in registers)
template <int T>
__device__ __forceinline__ int thread_base(const RPlan& p, int r, int tid) {
  int o = 0, m = 0;
#pragma unroll
  for (int b = 0; b < T; ++b) {
    bool in = false;
#pragma unroll
    for (int k = 0; k < 5; ++k) in = in || p.pos[r][k] == b;
    if (!in) {
      o |= ((tid >> m) & 1) << b;
      ++m;
    }
  }
  return o;
}

// Packed fp32x2 add/sub (sm_100a FADD2): two butterflies per instruction.
__device__ __forceinline__ void add_sub2(float& a0, float& a1, float& b0, float& b1) {
  float s0, s1, d0, d1;
  asm("{.reg .b64 ra, rb, rs, rd;\n"
      " mov.b64 ra, {%4, %5};\n mov.b64 rb, {%6, %7};\n"
      " add.rn.f32x2 rs, ra, rb;\n sub.rn.f32x2 rd, ra, rb;\n"
      " mov.b64 {%0, %1}, rs;\n mov.b64 {%2, %3}, rd;}"
      : "=f"(s0), "=f"(s1), "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
  a0 = s0;
  a1 = s1;
  b0 = d0;
  b1 = d1;
}

// Butterfly stages over the register-index bits set in XM.  Registers pair
// up as (2m, 2m+1); stages over bits 1..4 run as packed FADD2 on pairs, the
// stage over bit 0 (inside a pair) as scalar FADDs.
template <unsigned XM>
__device__ __forceinline__ void bfly32(float (&v)[32]) {
  if constexpr ((XM & 1u) != 0) {
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      const float a = v[j], b = v[j + 1];
      v[j] = a + b;
      v[j + 1] = a - b;
    }
  }
#pragma unroll
  for (int k = 1; k < 5; ++k) {
    if ((XM >> k) & 1u) {
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        if (((j >> k) & 1) == 0) add_sub2(v[j], v[j + 1], v[j | (1 << k)], v[(j | (1 << k)) + 1]);
      }
    }
  }
}

// Padded shared-memory index: one spare word per 32.  It is additive over
// disjoint bit sets (pad(b|c) = pad(b) + pad(c)), so every access is a
// per-thread base plus a compile-time immediate, and it is conflict-free for
// every layout here (warp lanes sit on five tile bits < 10, distinct mod 5).
__host__ __device__ constexpr int pad(int i) { return i + (i >> 5); }

// global offset of tile element i (tile bits >= CB move up to LO)
template <int CB, int LO>
__host__ __device__ constexpr int64_t remap_c(int i) {
  return ((int64_t)(i >> CB) << LO) | (int64_t)(i & ((1 << CB) - 1));
}

// Sources with a two-step load (raw4: every memory access, fix4: the math
// on the loaded words) declare `static constexpr bool kSplit = true`.
template <class S, class = void>
struct split_load : std::false_type {};
template <class S>
struct split_load<S, std::enable_if_t<S::kSplit>> : std::true_type {};

// Sinks with a two-step store (pre: the word a group of stores needs, e.g.
// its sign word; store4w / store2w: the stores) declare kSplitStore.
template <class S, class = void>
struct split_store : std::false_type {};
template <class S>
struct split_store<S, std::enable_if_t<S::kSplitStore>> : std::true_type {};

// One 2^T-entry tile t of a pass over vector bits [LO, LO + T - CB) with
// 2^CB contiguous columns, by a CTA of 2^(T-5) threads (32 values each in
// registers, rounds exchanged through `sm`, pad(2^T) floats).  Callable in a
// loop: the leading barrier protects the previous tile's shared-memory reads.
template <int T, int CB, int LO, class SB, class DB>
__device__ __forceinline__ void rtile_do(SB& s, const DB& d, int64_t t, float* sm) {
  constexpr RPlan P = make_rplan(T, CB);
  constexpr int NR = P.nr;
  constexpr int KS = T - CB;
  const int tid = threadIdx.x;
  const int b0 = thread_base<T>(P, 0, tid);
  const int b1 = NR > 1 ? thread_base<T>(P, 1, tid) : 0;
  const int b2 = NR > 2 ? thread_base<T>(P, 2, tid) : 0;
  const int b3 = NR > 3 ? thread_base<T>(P, 3, tid) : 0;
  constexpr int LR = NR - 1;
  const int bl = LR == 0 ? b0 : (LR == 1 ? b1 : (LR == 2 ? b2 : b3));
  const int64_t r0 = remap_c<CB, LO>(b0), rl = remap_c<CB, LO>(bl);
  float* const s0 = sm + pad(b0);
  float* const s1 = sm + pad(b1);
  float* const s2 = sm + pad(b2);
  float* const s3 = sm + pad(b3);
  {
    constexpr int CGB = LO - CB;
    const int64_t g0 = ((t >> CGB) << (LO + KS)) + ((t & ((1LL << CGB) - 1)) << CB);
    s.begin_tile(g0, g0 + remap_c<CB, LO>((1 << T) - 1));
    float v[32];
#pragma unroll
    if constexpr (split_load<SB>::value) {
      // latency-bound callers (the small-bucket kernel: one tile per CTA):
      // all eight raw loads in flight before any result is used
      typename SB::Raw raw[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) raw[m] = s.raw4(g0 + r0 + remap_c<CB, LO>(roff(P, 0, 4 * m)));
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const float4 q = s.fix4(g0 + r0 + remap_c<CB, LO>(roff(P, 0, 4 * m)), raw[m]);
        v[4 * m] = q.x;
        v[4 * m + 1] = q.y;
        v[4 * m + 2] = q.z;
        v[4 * m + 3] = q.w;
      }
    } else {
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const float4 q = s.load4(g0 + r0 + remap_c<CB, LO>(roff(P, 0, 4 * m)));
        v[4 * m] = q.x;
        v[4 * m + 1] = q.y;
        v[4 * m + 2] = q.z;
        v[4 * m + 3] = q.w;
      }
    }
    bfly32<P.xm[0]>(v);
    if constexpr (NR > 1) {
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 32; ++j) s0[pad(roff(P, 0, j))] = v[j];
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = s1[pad(roff(P, 1, j))];
      bfly32<P.xm[1]>(v);
    }
    if constexpr (NR > 2) {
#pragma unroll
      for (int j = 0; j < 32; ++j) s1[pad(roff(P, 1, j))] = v[j];
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = s2[pad(roff(P, 2, j))];
      bfly32<P.xm[2]>(v);
    }
    if constexpr (NR > 3) {
#pragma unroll
      for (int j = 0; j < 32; ++j) s2[pad(roff(P, 2, j))] = v[j];
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = s3[pad(roff(P, 3, j))];
      bfly32<P.xm[3]>(v);
    }
    if constexpr (P.pos[LR][0] == 0 && P.pos[LR][1] == 1 && split_store<DB>::value) {
      uint32_t wd[8];  // every sink-side load in flight before the stores
#pragma unroll
      for (int m = 0; m < 8; ++m) wd[m] = d.pre(g0 + rl + remap_c<CB, LO>(roff(P, LR, 4 * m)));
#pragma unroll
      for (int m = 0; m < 8; ++m)
        d.store4w(g0 + rl + remap_c<CB, LO>(roff(P, LR, 4 * m)),
                  make_float4(v[4 * m], v[4 * m + 1], v[4 * m + 2], v[4 * m + 3]), wd[m]);
    } else if constexpr (P.pos[LR][0] == 0 && P.pos[LR][1] == 1) {
#pragma unroll
      for (int m = 0; m < 8; ++m)
        d.store4(g0 + rl + remap_c<CB, LO>(roff(P, LR, 4 * m)),
                 make_float4(v[4 * m], v[4 * m + 1], v[4 * m + 2], v[4 * m + 3]));
    } else if constexpr (P.pos[LR][0] == 0 && split_store<DB>::value) {
      uint32_t wd[16];
#pragma unroll
      for (int m = 0; m < 16; ++m) wd[m] = d.pre(g0 + rl + remap_c<CB, LO>(roff(P, LR, 2 * m)));
#pragma unroll
      for (int m = 0; m < 16; ++m)
        d.store2w(g0 + rl + remap_c<CB, LO>(roff(P, LR, 2 * m)), v[2 * m], v[2 * m + 1], wd[m]);
    } else if constexpr (P.pos[LR][0] == 0) {
#pragma unroll
      for (int m = 0; m < 16; ++m)
        d.store2(g0 + rl + remap_c<CB, LO>(roff(P, LR, 2 * m)), v[2 * m], v[2 * m + 1]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) d.store1(g0 + rl + remap_c<CB, LO>(roff(P, LR, j)), v[j]);
    }
  }
}

template <int T, int CB, int LO, class Src, class Snk>
__global__ void __launch_bounds__(1 << (T - 5)) rtile_kernel(PassGeom pg, int worker_base,
                                                          const __grid_constant__ Src src,
                                                          const __grid_constant__ Snk snk) {
  extern __shared__ float sm[];
  const int w = worker_base + blockIdx.y;
  auto s = src.bind(w);
  const auto d = snk.bind(w);
  for (int64_t t = blockIdx.x; t < pg.ntiles; t += gridDim.x) rtile_do<T, CB, LO>(s, d, t, sm);
}

// ------------------------------------------------ small tiles (shared mem)
template <int E>
__device__ __forceinline__ void butterfly(float (&v)[1 << E]) {
#pragma unroll
  for (int h = 1; h < (1 << E); h <<= 1) {
#pragma unroll
    for (int j = 0; j < (1 << E); ++j) {
      if ((j & h) == 0) {
        float a = v[j], b = v[j + h];
        v[j] = a + b;
        v[j + h] = a - b;
      }
    }
  }
}

template <int E>
__device__ __forceinline__ void smem_round(float* s, int b, int nelem, int tid, int nthr) {
  int ngroups = nelem >> E;
  int lomask = (1 << b) - 1;
  for (int g = tid; g < ngroups; g += nthr) {
    int base = (g & lomask) | ((g & ~lomask) << E);
    float v[1 << E];
#pragma unroll
    for (int j = 0; j < (1 << E); ++j) v[j] = s[swz(base + (j << b))];
    butterfly<E>(v);
#pragma unroll
    for (int j = 0; j < (1 << E); ++j) s[swz(base + (j << b))] = v[j];
  }
}

__device__ __forceinline__ void tile_fwht(float* s, int b, int nbits, int nelem) {
  int end = b + nbits;
  while (b < end) {
    int e = min(5, end - b);
    switch (e) {
      case 5: smem_round<5>(s, b, nelem, threadIdx.x, blockDim.x); break;
      case 4: smem_round<4>(s, b, nelem, threadIdx.x, blockDim.x); break;
      case 3: smem_round<3>(s, b, nelem, threadIdx.x, blockDim.x); break;
      case 2: smem_round<2>(s, b, nelem, threadIdx.x, blockDim.x); break;
      default: smem_round<1>(s, b, nelem, threadIdx.x, blockDim.x); break;
    }
    __syncthreads();
    b += e;
  }
}

template <class Src, class Snk>
__global__ void __launch_bounds__(256) smem_tile_kernel(PassGeom pg, int worker_base, const __grid_constant__ Src src,
                                                            const __grid_constant__ Snk snk) {
  extern __shared__ float smem[];
  const int nelem = 1 << (pg.cb + pg.ks);
  const int w = worker_base + blockIdx.y;
  auto s = src.bind(w);
  const auto d = snk.bind(w);
  for (int64_t t = blockIdx.x; t < pg.ntiles; t += gridDim.x) {
    const int64_t g0 = tile_origin(pg, t);
    s.begin_tile(g0, g0 + tile_remap(pg, nelem - 1));
    __syncthreads();
    for (int i = threadIdx.x; i < nelem; i += blockDim.x) smem[swz(i)] = s.load1(g0 + tile_remap(pg, i));
    __syncthreads();
    tile_fwht(smem, pg.cb, pg.ks, nelem);
    for (int i = threadIdx.x; i < nelem; i += blockDim.x) d.store1(g0 + tile_remap(pg, i), smem[swz(i)]);
  }
}

// ------------------------------------------------------------- aggregate
struct AggArgs {
  const float* Y[kMaxW];  // wire vectors of every worker (peer-mapped in multi-GPU)
  float* A[kMaxW];        // aggregate shard of each owner
  float* G[kMaxW];        // push mode (TMA aggregate only): every rank's receive vector
  int push;
  Shards sh;
  int n, r;
  MaskView m;
  int owner_base;
};

// acc / cnt with cnt in 1..n: a power-of-two count divides exactly by
// multiplying with its reciprocal; otherwise IEEE division (np.divide).
__device__ __forceinline__ float mean_of(double acc, double cnt) {
  const unsigned c = (unsigned)cnt;
  if ((c & (c - 1)) == 0) {  // exact: multiply by 2^-log2(c), built from its exponent bits
    const long long e = 1023 - (long long)(__ffs(c) - 1);
    return (float)(acc * __longlong_as_double(e << 52));
  }
  return (float)(acc / cnt);
}

// collectives.py:77-94 with the own shard at its rank position and
// zero-filled misses (acc += 0.0 keeps the reference's -0.0 + 0.0 behaviour).
template <bool VEC>
__global__ void __launch_bounds__(256) aggregate_kernel(const __grid_constant__ AggArgs a) {
  const int o = a.owner_base + blockIdx.y;
  const int j = owned_shard(o, a.r, a.n);
  const int64_t len = a.sh.len(j), off = a.sh.off(j);
  const int n = a.n;
  const uint32_t epp = (uint32_t)a.m.epp;
  float* out = a.A[o];
  if (VEC) {
    const int64_t n4 = len >> 2;
    for (int64_t e4 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e4 < n4;
         e4 += (int64_t)gridDim.x * blockDim.x) {
      const int64_t e = e4 * 4;
      double acc[4] = {0.0, 0.0, 0.0, 0.0}, cnt[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int i = 0; i < kMaxW; ++i) {
        if (i < n) {
          const float4 v = ldg4(a.Y[i] + off + e);
          if (i == o) {
            acc[0] += (double)v.x;
            acc[1] += (double)v.y;
            acc[2] += (double)v.z;
            acc[3] += (double)v.w;
            cnt[0] += 1.0;
            cnt[1] += 1.0;
            cnt[2] += 1.0;
            cnt[3] += 1.0;
          } else {
            const uint32_t kk = keep4(a.m.row(0, o, i), (uint32_t)e, a.m);
            const bool k0 = kk & 1u, k1 = kk & 2u, k2 = kk & 4u, k3 = kk & 8u;
            acc[0] += k0 ? (double)v.x : 0.0;
            acc[1] += k1 ? (double)v.y : 0.0;
            acc[2] += k2 ? (double)v.z : 0.0;
            acc[3] += k3 ? (double)v.w : 0.0;
            cnt[0] += k0 ? 1.0 : 0.0;
            cnt[1] += k1 ? 1.0 : 0.0;
            cnt[2] += k2 ? 1.0 : 0.0;
            cnt[3] += k3 ? 1.0 : 0.0;
          }
        }
      }
      st4(out + e, make_float4(mean_of(acc[0], cnt[0]), mean_of(acc[1], cnt[1]), mean_of(acc[2], cnt[2]),
                               mean_of(acc[3], cnt[3])));
    }
  }
  const int64_t start = VEC ? (len & ~3LL) : 0;
  for (int64_t e = start + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < len;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t pkt = (uint32_t)e / epp;
    double acc = 0.0, cnt = 0.0;
    for (int i = 0; i < n; ++i) {
      if (i == o) {
        acc += (double)a.Y[i][off + e];
        cnt += 1.0;
      } else {
        const bool ok = row_bit(a.m.row(0, o, i), pkt);
        acc += ok ? (double)a.Y[i][off + e] : 0.0;
        cnt += ok ? 1.0 : 0.0;
      }
    }
    out[e] = mean_of(acc, cnt);
  }
}

// collectives.py:77-94 over explicit per-peer buffers (the sans-IO protocol's
// StageResult: zero-filled data + per-entry masks), for the generator-level
// collectives (tar / tar2d / ring / ps) of the facade.
struct MeanRecvArgs {
  const float* own;
  const float* peers[kMaxW];   // nullptr: peer not in result.data
  const uint8_t* masks[kMaxW]; // nullptr: all received
  int n, rank;
  int64_t len;
  float* out;
};

#ifndef OPTR_NO_GLOBAL_KERNELS
__global__ void __launch_bounds__(256) mean_received_kernel(const __grid_constant__ MeanRecvArgs a) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < a.len; e += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0, cnt = 0.0;
    for (int i = 0; i < a.n; ++i) {
      if (i == a.rank) {
        acc += (double)a.own[e];
        cnt += 1.0;
      } else if (a.peers[i]) {
        acc += (double)a.peers[i][e];
        cnt += (a.masks[i] == nullptr || a.masks[i][e]) ? 1.0 : 0.0;
      }
    }
    a.out[e] = cnt > 0.0 ? mean_of(acc, cnt) : 0.f;
  }
}
#endif

// ------------------------------------------------------------- assemble
struct AsmArgs {
  SrcGather gather;
  void* out[kMaxW];
  int dtype;
  int64_t L;
  int worker_base;
};

#ifndef OPTR_NO_GLOBAL_KERNELS
__global__ void __launch_bounds__(256) assemble_kernel(const __grid_constant__ AsmArgs a) {
  const int q = a.worker_base + blockIdx.y;
  auto s = a.gather.bind(q);
  void* const out = a.out[q];
  // float4 groups (fast path inside equal power-of-two shards), scalar tail
  const int64_t n4 = a.L >> 2;
  for (int64_t g4 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g4 < n4; g4 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = g4 * 4;
    const float4 v = s.load4(g);
    if (a.dtype == OPTR_F32 && (((uintptr_t)out) & 15) == 0) {
      st4((float*)out + g, v);
    } else {
      store_elem(out, a.dtype, g, v.x);
      store_elem(out, a.dtype, g + 1, v.y);
      store_elem(out, a.dtype, g + 2, v.z);
      store_elem(out, a.dtype, g + 3, v.w);
    }
  }
  for (int64_t g = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < a.L;
       g += (int64_t)gridDim.x * blockDim.x)
    store_elem(out, a.dtype, g, s.load1(g));
}
#endif

// fp32/bf16 -> fp32 copy (RHT off: the wire carries float32, runner.py:228)
#ifndef OPTR_NO_GLOBAL_KERNELS
__global__ void cast_copy_kernel(const void* x, int dtype, float* y, int64_t n) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x)
    y[g] = load_elem(x, dtype, g);
}

__global__ void count_mask_kernel(const uint8_t* mask, int64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x)
    c += mask[g] ? 1 : 0;
  for (int o = 16; o; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}
#endif

}  // namespace optr
