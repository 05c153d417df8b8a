// Device kernels of the TAR+RHT hot path (sm_100a).
//
//   prep_kernel       Rademacher sign bits (hadamard.py:49-51), drop-mask packet
//                     bitmaps (datagram.py:70-72,117-124 coin or caller bitmaps),
//                     per-(stage,dst) received counts (simdriver.py:328-341).
//   fwht_pass_kernel  one tile pass of the Sylvester FWHT (hadamard.py:76-90),
//                     H_D = prod of passes over disjoint index-bit ranges, with
//                     the encode sign/pad/cast fused into the first pass and the
//                     decode gather/mask/scale/sign/truncate fused into the ends.
//   aggregate_kernel  TAR stage-1 owner mean (collectives.py:77-94,125): fp64
//                     accumulate in ascending node order under stage-1 masks.
//   assemble_kernel   TAR stage-2 assembly without RHT (collectives.py:140-150).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

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
  __host__ __device__ __forceinline__ int of(int64_t g) const {
    int64_t big = extra * (base + 1);
    if (g < big) return (int)(g / (base + 1));
    return (int)(extra + (g - big) / base);
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

// Packet-bitmap addressing (optr.h): stage 0/1, receiver dst, sender src.
struct MaskView {
  const uint32_t* bits;
  int64_t pw;  // u32 words per pair
  int n;
  int epp;
  __device__ __forceinline__ bool get(int stage, int dst, int src, int64_t pkt) const {
    const uint32_t* p = bits + ((int64_t)(stage * n + dst) * n + src) * pw;
    return (__ldg(p + (pkt >> 5)) >> (pkt & 31)) & 1u;
  }
};

// -------------------------------------------------------------------- prep
struct PrepArgs {
  // signs
  uint32_t* signs;
  int64_t dim;
  u128 sign_state, sign_inc;
  int64_t sign_threads;  // dim/64 rounded up (0 = no signs)
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
};

// Running packet index of sender `src`'s first packet to `dst` in `stage`
// (datagram.py:117-124 draws one coin per packet in send order: stage 1 to
// dst = src+1..src+n-1 (schedule.py:67-78) then stage 2 the same order).
__device__ __forceinline__ uint64_t coin_base(const PrepArgs& a, int stage, int src, int dst) {
  int n = a.n;
  int o = ((dst - src) % n + n) % n;
  uint64_t base = 0;
  if (stage == 0) {
    for (int k = 1; k < o; ++k)
      base += n_packets(a.sh.len(owned_shard((src + k) % n, a.r, n)), a.epp);
  } else {
    for (int k = 1; k < n; ++k)
      base += n_packets(a.sh.len(owned_shard((src + k) % n, a.r, n)), a.epp);
    base += (uint64_t)(o - 1) * n_packets(a.sh.len(owned_shard(src, a.r, n)), a.epp);
  }
  return base;
}

__global__ void prep_kernel(PrepArgs a) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < a.sign_threads) {
    // 64 signs = 32 consecutive PCG64 outputs starting at output 32t
    int64_t k0 = t * 64;
    u128 s = pcg_advance(a.sign_state, a.sign_inc, (uint64_t)(t * 32) + 1);
    uint32_t w0 = 0, w1 = 0;
#pragma unroll 4
    for (int i = 0; i < 32; ++i) {
      uint64_t out = pcg_xsl_rr(s);
      uint32_t b0 = (uint32_t)((out >> 31) & 1u), b1 = (uint32_t)(out >> 63);
      int bit = 2 * i;
      if (bit < 32) {
        w0 |= (b0 << bit) | (b1 << (bit + 1));
      } else {
        w1 |= (b0 << (bit - 32)) | (b1 << (bit - 31));
      }
      s = pcg_step(s, a.sign_inc);
    }
    int64_t wi = k0 >> 5;
    int64_t nwords = (a.dim + 31) >> 5;
    if (wi < nwords) a.signs[wi] = w0;
    if (wi + 1 < nwords) a.signs[wi + 1] = w1;
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
      u128 s = pcg_advance(a.coin_state[src], a.coin_inc[src], k + 1);
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
  if (bits) {
    unsigned long long e = (unsigned long long)__popc(bits) * (unsigned long long)a.epp;
    // the last packet of a transfer is short (simdriver.py:188-189)
    if (p0 + cnt == np && ((bits >> (cnt - 1)) & 1u)) e -= (unsigned long long)(np * a.epp - len);
    atomicAdd(a.counts + stage * a.n + dst, e);
  }
}

// ------------------------------------------------------------ FWHT tiles
// Shared-memory bank swizzle: XOR index bits 0-4 with bits 5-9.  Every
// register round below maps warp lanes onto the lowest index bits outside
// its butterfly range, which this swizzle makes conflict-free.
__device__ __forceinline__ int swz(int i) { return i ^ ((i >> 5) & 31); }

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

// Butterflies over tile-index bits [b, b+E) for all 2^(nbits-E) groups.
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

// Geometry of one pass: tile = 2^(cb+ks) elements; tile bits [0,cb) are
// columns (index bits [0,cb) of the vector, not transformed here... but see
// below), tile bits [cb,cb+ks) are the transformed index bits [lo, lo+ks).
// Global index of tile element i in tile t:
//   g = outer*2^(lo+ks) + row*2^lo + cgroup*2^cb + col,
//   cgroup = t mod 2^(lo-cb), outer = t >> (lo-cb).
struct PassGeom {
  int lo, ks, cb;
};

__device__ __forceinline__ int64_t tile_global(const PassGeom& pg, int64_t t, int i) {
  int64_t ncg_bits = pg.lo - pg.cb;
  int64_t cgroup = t & ((1LL << ncg_bits) - 1);
  int64_t outer = t >> ncg_bits;
  int col = i & ((1 << pg.cb) - 1);
  int64_t row = i >> pg.cb;
  return (outer << (pg.lo + pg.ks)) + (row << pg.lo) + (cgroup << pg.cb) + col;
}

// ---- sources (first pass input) and sinks (last pass output)
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
__device__ __forceinline__ bool sign_pos(const uint32_t* signs, int64_t g) {
  return (__ldg(signs + (g >> 5)) >> (g & 31)) & 1u;
}

// pad(x) * signs   (hadamard.py:98-100)
struct SrcEncode {
  const void* x[kMaxW];
  int dtype;
  int64_t L;
  const uint32_t* signs;
  __device__ __forceinline__ float load(int w, int64_t g) const {
    if (g >= L) return 0.f;
    float v = load_elem(x[w], dtype, g);
    return sign_pos(signs, g) ? v : -v;
  }
};

struct SrcBuf {
  float* y[kMaxW];
  __device__ __forceinline__ float load(int w, int64_t g) const { return y[w][g]; }
};

// where(mask, y, 0) with a byte mask (hadamard.py:120)
struct SrcMasked {
  const float* y;
  const uint8_t* mask;
  __device__ __forceinline__ float load(int, int64_t g) const {
    return (mask == nullptr || mask[g]) ? y[g] : 0.f;
  }
};

// TAR stage-2 receive of worker q (collectives.py:140-150): own shard from
// its own aggregate, peer shards from the owner's aggregate under the
// stage-2 mask, zero-filled misses.  Optionally records `received`.
struct SrcGather {
  const float* A[kMaxW];
  Shards sh;
  int n, r;
  MaskView m;
  uint8_t* got;  // optional [n][dim]
  int64_t dim;
  __device__ __forceinline__ float load(int q, int64_t g) const {
    int j = sh.of(g);
    int64_t e = g - sh.off(j);
    int owner = shard_owner(j, r, n);
    bool ok = owner == q ? true : m.get(1, q, owner, (int64_t)((uint32_t)e / (uint32_t)m.epp));
    if (got) got[(int64_t)q * dim + g] = ok ? 1 : 0;
    return ok ? A[owner][e] : 0.f;
  }
};

struct SnkBuf {
  float* y[kMaxW];
  float scale;
  __device__ __forceinline__ void store(int w, int64_t g, float v) const { y[w][g] = v * scale; }
};

// signs * v * (dim/count)/sqrt(dim), truncated to L, cast (hadamard.py:116-123,
// runner.py:253-256: count 0 -> zeros).
struct SnkDecode {
  void* out[kMaxW];
  int dtype;
  int64_t L;
  const uint32_t* signs;
  const unsigned long long* count_extra;  // device: + received entries (may be null)
  int64_t count_base[kMaxW];              // host-known part of count
  int count_stride;                       // index of worker's count_extra entry
  double dim;
  __device__ __forceinline__ float scale_for(int w) const {
    unsigned long long c = (unsigned long long)count_base[w];
    if (count_extra) c += count_extra[w * count_stride];
    if (c == 0) return 0.f;
    return (float)((dim / (double)c) / sqrt(dim));
  }
  __device__ __forceinline__ void store(int w, int64_t g, float v, float scale) const {
    if (g >= L) return;
    float r = v * scale;
    store_elem(out[w], dtype, g, sign_pos(signs, g) ? r : -r);
  }
};

template <class S>
struct HasScale {
  static constexpr bool value = false;
};
template <>
struct HasScale<SnkDecode> {
  static constexpr bool value = true;
};

template <class Src, class Snk>
__global__ void __launch_bounds__(1024) fwht_pass_kernel(PassGeom pg, int worker_base, Src src, Snk snk) {
  extern __shared__ float smem[];
  const int nelem = 1 << (pg.cb + pg.ks);
  const int64_t t = blockIdx.x;
  const int w = worker_base + blockIdx.y;
  for (int i = threadIdx.x; i < nelem; i += blockDim.x) smem[swz(i)] = src.load(w, tile_global(pg, t, i));
  __syncthreads();
  tile_fwht(smem, pg.cb, pg.ks, nelem);
  float scale = 1.f;
  if constexpr (HasScale<Snk>::value) scale = snk.scale_for(w);
  for (int i = threadIdx.x; i < nelem; i += blockDim.x) {
    if constexpr (HasScale<Snk>::value)
      snk.store(w, tile_global(pg, t, i), smem[swz(i)], scale);
    else
      snk.store(w, tile_global(pg, t, i), smem[swz(i)]);
  }
}

// ------------------------------------------------------------- aggregate
struct AggArgs {
  const float* Y[kMaxW];  // wire vectors of every worker (peer-mapped in multi-GPU)
  float* A[kMaxW];        // aggregate shard of each owner
  Shards sh;
  int n, r;
  MaskView m;
  int owner_base;
};

// collectives.py:77-94 with own shard at its rank position, zero-filled misses
// (acc += 0.0 keeps -0.0 + 0.0 semantics bit-identical to the reference).
__global__ void __launch_bounds__(256) aggregate_kernel(AggArgs a) {
  const int o = a.owner_base + blockIdx.y;
  const int j = owned_shard(o, a.r, a.n);
  const int64_t len = a.sh.len(j), off = a.sh.off(j);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < len;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t pkt = (int64_t)((uint64_t)e / (uint64_t)a.m.epp);
    double acc = 0.0, cnt = 0.0;
    for (int i = 0; i < a.n; ++i) {
      if (i == o) {
        acc += (double)a.Y[i][off + e];
        cnt += 1.0;
      } else {
        bool ok = a.m.get(0, o, i, pkt);
        float v = ok ? a.Y[i][off + e] : 0.f;
        acc += (double)v;
        cnt += ok ? 1.0 : 0.0;
      }
    }
    a.A[o][e] = (float)(acc / cnt);
  }
}

// ------------------------------------------------------------- assemble
struct AsmArgs {
  SrcGather gather;
  void* out[kMaxW];
  int dtype;
  int64_t L;
  int worker_base;
};

__global__ void __launch_bounds__(256) assemble_kernel(AsmArgs a) {
  const int q = a.worker_base + blockIdx.y;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < a.L;
       g += (int64_t)gridDim.x * blockDim.x)
    store_elem(a.out[q], a.dtype, g, a.gather.load(q, g));
}

// fp32/bf16 -> fp32 copy (RHT off: the wire carries float32, runner.py:228)
__global__ void cast_copy_kernel(const void* x, int dtype, float* y, int64_t n) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x)
    y[g] = load_elem(x, dtype, g);
}

__global__ void count_mask_kernel(const uint8_t* mask, int64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x)
    c += mask[g] ? 1 : 0;
  for (int o = 16; o; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

}  // namespace optr
