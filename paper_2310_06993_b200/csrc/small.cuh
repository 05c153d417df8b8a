// Small-bucket TAR+RHT, one worker per GPU, ONE launch per call.
//
// Buckets of 2^13..2^20 entries (32 KB..4 MB fp32: DDP's first bucket, the
// small end of the BASELINE sweep) are latency-bound: the multi-launch path
// pays ~65 us in launches, stream hops and barrier kernels for a few us of
// data movement.  Here one cooperative kernel (every CTA co-resident) runs
// the whole call -- signs, masks, both encode passes, stage 1, stage 2 and
// both decode passes -- separated by grid barriers on the GPU and by two
// flag handshakes over NVLink:
//
//   phase 1  each tile CTA: its tile's signs (one PCG jump per 32), then
//            encode pass 1 (contiguous 2^13 tiles of x -> Y[me]: pad, signs,
//            bf16 upcast); the other CTAs: packet masks and received counts
//   phase 2  encode pass 2: strided bits [13, K) in place, x 1/sqrt(D)
//            -> ready1: push my epoch into every peer's flag block
//   phase 3  wait ready1 of every peer; stage 1: masked fp64 mean of my
//            shard over every rank's Y (peer loads), and stage 2 as a push:
//            the mean goes into every rank's Y at my shard's offset under
//            that receiver's stage-2 mask (peer stores; system-scope fence)
//            -> ready2
//   phase 4  wait ready2 of every peer (my Y now holds the stage-2
//            receive); decode pass 1: contiguous tiles in place
//   phase 5  decode pass 2: strided bits, D/count scale, signs, truncate,
//            cast -> out
//
// References: hadamard.py:93-123 (encode / decode), collectives.py:97-150
// (tar_allreduce), collectives.py:77-94 (_mean_received), datagram.py:70-72
// (coin masks, via prep_item).
//
// Buffer reuse needs no extra synchronisation: in phase 3 owner j reads
// every rank's Y at shard j's offset and writes its mean back to exactly
// those entries (same thread, read before write); other owners touch other
// shards.  Owner j pushes call c+1's means into my Y only after my ready1 of
// c+1, i.e. after my whole call c (stream order).  Flags carry the call
// epoch and only grow.
#pragma once

#include "kernels.cuh"

namespace optr {

constexpr int kSmallT = 13;        // tile bits of both passes (256 threads, 32 values each)
constexpr int kSmallMinLog = 13;   // 32 KB fp32
constexpr int kSmallMaxLog = 20;   // 4 MB fp32
constexpr int kSmallBarriers = 4;  // grid barriers per call
constexpr int kSmallMaxRanks = 8;

__device__ __forceinline__ uint64_t small_clock_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct SmallArgs {
  PrepArgs pa;  // masks + counts of dst = me (pa.sign_threads = 0)
  uint32_t* signs;
  u128 sign_state, sign_inc;
  const void* x;
  void* out;
  int dtype_in, dtype_out;
  int64_t L, dim;
  float* Y[kMaxW];                   // every rank's wire / stage-2 receive vector (peer-mapped)
  unsigned long long* flags[kMaxW];  // every rank's flag block [2][kMaxW]
  unsigned long long* bar;           // grid-barrier arrivals (monotonic)
  unsigned long long bar_base;
  unsigned long long epoch;
  unsigned long long* counts;        // [2][n] received entries at me (this call's parity)
  unsigned long long* counts_next;   // the next call's [2][n], zeroed here
  unsigned long long* received_out;  // optional [2]
  MaskView m;
  int n, me, r, shard_shift;
  uint64_t watchdog_ns;
  unsigned long long* trace;  // optional debug stamps: [call % 64][16] globaltimer ns (CTA 0)
};

__device__ __forceinline__ void small_stamp(const SmallArgs& a, int i) {
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[(a.epoch % 64) * 16 + i] = small_clock_ns();
}

__device__ __forceinline__ void small_grid_sync(unsigned long long* bar, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
    unsigned long long v;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// ready flag `slot` of this call: every peer's epoch landed in my block
__device__ __forceinline__ void small_wait_peers(const SmallArgs& a, int slot) {
  if (threadIdx.x == 0) {
    const unsigned long long* f = a.flags[a.me] + slot * kMaxW;
    uint64_t t0 = 0;
    for (int p = 0; p < a.n; ++p) {
      if (p == a.me) continue;
      for (;;) {
        unsigned long long v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f + p) : "memory");
        if (v >= a.epoch) break;
        if (!t0) t0 = small_clock_ns();
        else if (small_clock_ns() - t0 > a.watchdog_ns) {
          printf("optr: small-bucket kernel wait timed out (rank %d, peer %d, slot %d)\n", a.me, p, slot);
          __trap();
        }
      }
    }
  }
  __syncthreads();
}

// After a grid barrier: publish this rank's progress into every peer's flag
// block.  The data a peer reads next (my Y / A) lives in MY memory and peer
// loads of it are served by my L2, so the GPU-scope fence (the grid
// barrier's release/acquire, then MEMBAR.GPU here) makes it readable before
// the flag leaves; a system-scope release (MEMBAR.SYS) is what the PTX model
// asks for across GPUs and cost ~3.6 us per handshake, measured (the fused
// kernel's protocol, tma.cuh, argues and measures the same; the multi-GPU
// stress test interleaves this kernel's calls).
__device__ __forceinline__ void small_signal(const SmallArgs& a, int slot) {
  if (blockIdx.x == 0 && threadIdx.x < a.n && threadIdx.x != a.me) {
    __threadfence();
    unsigned long long* dst = a.flags[threadIdx.x] + slot * kMaxW + a.me;
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(dst), "l"(a.epoch) : "memory");
  }
}

// PCG jump from a shared-memory copy of the jump table (the constant-bank
// table misses line by line on a cold SM: one load round here instead)
struct JumpSmem {
  u128 a[64], g[64];
};
__device__ __forceinline__ u128 jump_s(u128 s, u128 inc, uint64_t k, const JumpSmem& t) {
  const int top = 64 - __clzll((long long)(k | 1));
  for (int i = 0; i < top; ++i)
    if ((k >> i) & 1) s = t.a[i] * s + inc * t.g[i];
  return s;
}

__device__ __forceinline__ float4 ld_cg4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }

// pad(x) * signs with a scalar path for unaligned x (hadamard.py:98-100).
// Two-step loads (kSplit): raw4 issues the x and sign-word loads, fix4
// converts and applies the signs once all of a thread's loads are in flight.
struct SmallEncodeSrc {
  static constexpr bool kSplit = true;
  SrcEncode::B e;
  bool vec;
  struct Raw {
    float4 v;
    uint32_t w;
  };
  __device__ __forceinline__ void begin_tile(int64_t, int64_t) {}
  __device__ __forceinline__ bool fast(int64_t g) const { return vec && g + 4 <= e.L; }
  __device__ __forceinline__ Raw raw4(int64_t g) const {
    Raw r;
    if (fast(g)) {
      if (e.dtype == OPTR_F32) {
        r.v = ldg4((const float*)e.x + g);
      } else {
        const uint2 u = __ldg(reinterpret_cast<const uint2*>((const __nv_bfloat16*)e.x + g));
        r.v = make_float4(__uint_as_float(u.x), __uint_as_float(u.y), 0.f, 0.f);
      }
      r.w = __ldcg(e.signs + (g >> 5));  // written by this CTA in this phase
    } else {
      float f[4];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        f[c] = g + c < e.L ? sgn(__ldcg(e.signs + ((g + c) >> 5)), (int)((g + c) & 31), load_elem(e.x, e.dtype, g + c))
                           : 0.f;
      r.v = make_float4(f[0], f[1], f[2], f[3]);
      r.w = 0;
    }
    return r;
  }
  __device__ __forceinline__ float4 fix4(int64_t g, const Raw& r) const {
    if (!fast(g)) return r.v;
    float4 v = r.v;
    if (e.dtype != OPTR_F32) {
      const uint32_t ux = __float_as_uint(r.v.x), uy = __float_as_uint(r.v.y);
      const float2 fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ux));
      const float2 fb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&uy));
      v = make_float4(fa.x, fa.y, fb.x, fb.y);
    }
    const int b0 = (int)(g & 31);
    return make_float4(sgn(r.w, b0, v.x), sgn(r.w, b0 + 1, v.y), sgn(r.w, b0 + 2, v.z), sgn(r.w, b0 + 3, v.w));
  }
};

struct SmallBufSrc {
  const float* y;
  __device__ __forceinline__ void begin_tile(int64_t, int64_t) {}
  __device__ __forceinline__ float4 load4(int64_t g) const { return ld4(y + g); }
};

// keep flags of entries e..e+3 of a shard from the two bitmap words that can
// cover them (keep4 with the loads hoisted out)
__device__ __forceinline__ uint32_t keep4_words(uint32_t e, uint32_t w0, uint32_t w1, const MaskView& m) {
  const uint32_t epp = (uint32_t)m.epp;
  if (epp >= 4) {
    const uint32_t p0 = m.dv.div(e), rem = e - p0 * epp;
    const uint32_t w = w0 >> (p0 & 31);
    const uint32_t b0 = w & 1u;
    if (rem + 3 < epp) return b0 ? 0xFu : 0u;
    const uint32_t b1 = (p0 & 31) == 31 ? (w1 & 1u) : ((w >> 1) & 1u);
    const uint32_t lo = (1u << (epp - rem)) - 1u;
    return (b0 ? lo : 0u) | (b1 ? (0xFu & ~lo) : 0u);
  }
  uint32_t k = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint32_t p = (e + c) / epp, d = p - (m.dv.div(e) & ~31u);  // 0..63 words from w0
    k |= (((d < 32 ? (w0 >> d) : (w1 >> (d - 32))) & 1u)) << c;
  }
  return k;
}

// signs * v * (D/count)/sqrt(D), truncated, cast; scalar stores for unaligned out
struct SmallDecodeSnk {
  static constexpr bool kSplitStore = true;
  SnkDecode::B d;
  bool vec;
  __device__ __forceinline__ bool fast(int64_t g, int k) const { return vec && g + k <= d.L; }
  __device__ __forceinline__ uint32_t pre(int64_t g) const { return g < d.L ? __ldg(d.signs + (g >> 5)) : 0u; }
  __device__ __forceinline__ void store4w(int64_t g, float4 v, uint32_t w) const {
    if (!fast(g, 4)) {
      store4(g, v);
      return;
    }
    const int b0 = (int)(g & 31);
    v = make_float4(sgn(w, b0, v.x * d.scale), sgn(w, b0 + 1, v.y * d.scale), sgn(w, b0 + 2, v.z * d.scale),
                    sgn(w, b0 + 3, v.w * d.scale));
    if (d.dtype == OPTR_F32) {
      st4((float*)d.out + g, v);
    } else {
      __nv_bfloat162 p = __floats2bfloat162_rn(v.x, v.y), q = __floats2bfloat162_rn(v.z, v.w);
      *reinterpret_cast<uint2*>((__nv_bfloat16*)d.out + g) =
          make_uint2(*reinterpret_cast<uint32_t*>(&p), *reinterpret_cast<uint32_t*>(&q));
    }
  }
  __device__ __forceinline__ void store2w(int64_t g, float p, float q, uint32_t w) const {
    if (!fast(g, 2)) {
      store2(g, p, q);
      return;
    }
    const int b0 = (int)(g & 31);
    p = sgn(w, b0, p * d.scale);
    q = sgn(w, b0 + 1, q * d.scale);
    if (d.dtype == OPTR_F32)
      *reinterpret_cast<float2*>((float*)d.out + g) = make_float2(p, q);
    else
      *reinterpret_cast<__nv_bfloat162*>((__nv_bfloat16*)d.out + g) = __floats2bfloat162_rn(p, q);
  }
  __device__ __forceinline__ void store1(int64_t g, float v) const { d.store1(g, v); }
  __device__ __forceinline__ void store2(int64_t g, float p, float q) const {
    if (vec) {
      d.store2(g, p, q);
    } else {
      d.store1(g, p);
      d.store1(g + 1, q);
    }
  }
  __device__ __forceinline__ void store4(int64_t g, float4 v) const {
    if (vec) {
      d.store4(g, v);
    } else {
      d.store1(g, v.x);
      d.store1(g + 1, v.y);
      d.store1(g + 2, v.z);
      d.store1(g + 3, v.w);
    }
  }
};

// Packet masks, one packet per thread, a warp per bitmap word (prep_item's
// per-word loop, spread out: the coin of packet k is output k of the
// sender's stream, datagram.py:70-72,122): my receive rows (stage, dst = me,
// src) with the received entries per stage (simdriver.py:188-189: the last
// packet of a transfer is short), then my stage-2 send rows (dst = q, src =
// me) for the push.  Every row has np packets (equal shards).
__device__ __forceinline__ void small_masks(const SmallArgs& a, int64_t gtid, int64_t gthreads,
                                            const JumpSmem& jt) {
  const PrepArgs& pa = a.pa;
  const int n = a.n, me = a.me;
  const int64_t len = 1LL << a.shard_shift;
  const int64_t np = n_packets(len, pa.epp);
  const int64_t per_row = pa.pw * 32;
  const int64_t total = (int64_t)3 * (n - 1) * per_row;  // a multiple of 32: whole warps per word
  for (int64_t t = gtid; t < total; t += gthreads) {
    const int row = (int)(t / per_row);
    const int64_t p = t - (int64_t)row * per_row;
    const bool recv = row < 2 * (n - 1);
    const int stage = recv ? row / (n - 1) : 1, oi = row - (recv ? stage : 2) * (n - 1);
    const int other = oi < me ? oi : oi + 1;
    const int src = recv ? other : me, dst = recv ? me : other;
    const int64_t widx = ((int64_t)(stage * n + dst) * n + src) * pa.pw + (p >> 5);
    bool keep = p < np;
    if (pa.kind == OPTR_MASK_COIN && keep) {
      const u128 s = jump_s(pa.coin_state[src], pa.coin_inc[src], coin_base(pa, stage, src, dst) + (uint64_t)p + 1, jt);
      keep = !coin_drops(pcg_xsl_rr(s), pa.drop_prob);
    } else if (pa.kind == OPTR_MASK_BITMAP && keep) {
      keep = (__ldg(pa.bitmap_in + widx) >> (p & 31)) & 1u;
    }
    const uint32_t bits = __ballot_sync(0xffffffffu, keep);
    if ((threadIdx.x & 31) == 0) {
      if (pa.kind != OPTR_MASK_BITMAP) pa.bitmap_out[widx] = bits;
      if (bits && recv) {
        unsigned long long e = (unsigned long long)__popc(bits) * (unsigned long long)pa.epp;
        const int64_t last = np - 1 - (p & ~31LL);  // bit of the short last packet, if in this word
        if (last >= 0 && last < 32 && ((bits >> last) & 1u)) e -= (unsigned long long)(np * pa.epp - len);
        atomicAdd(a.counts + stage * n + me, e);
      }
    }
  }
}

// Stage 1 at the owner (collectives.py:77-94; aggregate_kernel): masked
// mean of my shard over every rank's Y, fp64 in ascending rank order; then
// stage 2 (collectives.py:133-150) as a push: the mean into every rank's Y
// at the same entries, zero where my packet to that receiver was lost.
// Each thread keeps 8 / NR float4 groups' loads (NR ranks each, mostly over
// NVLink) in flight before it computes.
template <int NR>
__device__ __forceinline__ void small_mean(const SmallArgs& a, int64_t gtid, int64_t gthreads) {
  constexpr int U = 8 / NR;
  const int j = owned_shard(a.me, a.r, NR);
  const int64_t n4 = (1LL << a.shard_shift) >> 2, off = (int64_t)j << a.shard_shift;
  for (int64_t b4 = gtid; b4 < n4; b4 += gthreads * U) {
    float4 v[U][NR];
    uint32_t w0[U][NR], w1[U][NR], s0[U][NR], s1[U][NR];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e4 = b4 + u * gthreads;
      if (e4 < n4) {
        const uint32_t e = (uint32_t)(e4 * 4), wi = a.m.dv.div(e) >> 5;
#pragma unroll
        for (int i = 0; i < NR; ++i) {
          v[u][i] = ld_cg4(a.Y[i] + off + e);
          const uint32_t* row = a.m.row(0, a.me, i);
          w0[u][i] = i == a.me ? 0xffffffffu : __ldg(row + wi);
          w1[u][i] = (i == a.me || wi + 1 >= (uint32_t)a.m.pw) ? 0xffffffffu : __ldg(row + wi + 1);
          const uint32_t* srow = a.m.row(1, i, a.me);  // my stage-2 packets to receiver i
          s0[u][i] = i == a.me ? 0xffffffffu : __ldg(srow + wi);
          s1[u][i] = (i == a.me || wi + 1 >= (uint32_t)a.m.pw) ? 0xffffffffu : __ldg(srow + wi + 1);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e4 = b4 + u * gthreads;
      if (e4 < n4) {
        const uint32_t e = (uint32_t)(e4 * 4);
        double acc[4] = {0.0, 0.0, 0.0, 0.0}, cnt[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int i = 0; i < NR; ++i) {
          const uint32_t kk = i == a.me ? 0xFu : keep4_words(e, w0[u][i], w1[u][i], a.m);
          acc[0] += (kk & 1u) ? (double)v[u][i].x : 0.0;
          acc[1] += (kk & 2u) ? (double)v[u][i].y : 0.0;
          acc[2] += (kk & 4u) ? (double)v[u][i].z : 0.0;
          acc[3] += (kk & 8u) ? (double)v[u][i].w : 0.0;
          cnt[0] += (kk & 1u) ? 1.0 : 0.0;
          cnt[1] += (kk & 2u) ? 1.0 : 0.0;
          cnt[2] += (kk & 4u) ? 1.0 : 0.0;
          cnt[3] += (kk & 8u) ? 1.0 : 0.0;
        }
        const float4 mv = make_float4(mean_of(acc[0], cnt[0]), mean_of(acc[1], cnt[1]), mean_of(acc[2], cnt[2]),
                                      mean_of(acc[3], cnt[3]));
#pragma unroll
        for (int i = 0; i < NR; ++i) {
          const uint32_t kk = i == a.me ? 0xFu : keep4_words(e, s0[u][i], s1[u][i], a.m);
          st4(a.Y[i] + off + e, make_float4((kk & 1u) ? mv.x : 0.f, (kk & 2u) ? mv.y : 0.f, (kk & 4u) ? mv.z : 0.f,
                                            (kk & 8u) ? mv.w : 0.f));
        }
      }
    }
  }
}

template <int K>
__global__ void __launch_bounds__(1 << (kSmallT - 5)) tar_small_kernel(const __grid_constant__ SmallArgs a) {
  extern __shared__ float sm[];
  constexpr int T = kSmallT;
  constexpr int CB = 2 * T - K;  // strided pass: 2^(K-T) rows x 2^CB columns per tile
  const int64_t ntiles = a.dim >> T;
  const int G = gridDim.x;
  const int tid = threadIdx.x;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + tid;
  const int64_t gthreads = (int64_t)G * blockDim.x;
  float* const ym = a.Y[a.me];
  small_stamp(a, 0);
  __shared__ JumpSmem jt;
  if (tid < 64) {
    jt.a[tid] = c_jump.a[tid];
    jt.g[tid] = c_jump.g[tid];
  }
  __syncthreads();
  if (blockIdx.x == 0 && tid < 2 * a.n) a.counts_next[tid] = 0ULL;
  // packet masks and received counts, from the last CTA down (the tile CTAs
  // are the first ones)
  small_masks(a, (int64_t)(G - 1 - blockIdx.x) * blockDim.x + tid, gthreads, jt);
  small_stamp(a, 1);

  // phase 1: per tile, its 2^13 signs = PCG64 outputs 16w..16w+15 of words
  // w = 256t + tid (hadamard.py:49-51), then encode pass 1 (contiguous)
  {
    SrcEncode::B eb{a.x, a.dtype_in, a.L, a.signs};
    SmallEncodeSrc src{eb, (((uintptr_t)a.x) & (a.dtype_in == OPTR_F32 ? 15 : 7)) == 0};
    const SnkBuf::B dst{ym, K == T ? (float)(1.0 / sqrt((double)a.dim)) : 1.f};
    for (int64_t t = blockIdx.x; t < ntiles; t += G) {
      const int64_t w = (t << (T - 5)) + tid;  // 2^(T-5) threads: one sign word each
      u128 st = jump_s(a.sign_state, a.sign_inc, (uint64_t)w * 16 + 1, jt);
      uint32_t word = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint64_t o = pcg_xsl_rr(st);
        word |= (uint32_t)((o >> 31) & 1u) << (2 * i);
        word |= (uint32_t)(o >> 63) << (2 * i + 1);
        st = pcg_step(st, a.sign_inc);
      }
      a.signs[w] = word;
      __syncthreads();  // the tile's sign words are written (read back through L2)
      rtile_do<T, 0, 0>(src, dst, t, sm);
    }
  }
  small_stamp(a, 4);
  small_grid_sync(a.bar, a.bar_base + 1ULL * G);
  small_stamp(a, 5);

  // phase 2: encode pass 2 (strided, in place) -> ready1
  if constexpr (K > T) {
    SmallBufSrc src{ym};
    const SnkBuf::B dst{ym, (float)(1.0 / sqrt((double)a.dim))};
    for (int64_t t = blockIdx.x; t < ntiles; t += G) rtile_do<T, CB, T>(src, dst, t, sm);
  }
  small_stamp(a, 6);
  small_grid_sync(a.bar, a.bar_base + 2ULL * G);
  small_stamp(a, 7);
  small_signal(a, 0);
  small_stamp(a, 8);

  // phase 3: stage 1 at the owner + the stage-2 push -> ready2
  small_wait_peers(a, 0);
  small_stamp(a, 9);
  switch (a.n) {
    case 2: small_mean<2>(a, gtid, gthreads); break;
    case 4: small_mean<4>(a, gtid, gthreads); break;
    default: small_mean<8>(a, gtid, gthreads); break;
  }
  // my peer stores have landed before this CTA arrives at the barrier, so
  // before the flag that follows it (the data lives in the READER's memory)
  __threadfence_system();
  small_stamp(a, 10);
  small_grid_sync(a.bar, a.bar_base + 3ULL * G);
  small_signal(a, 1);
  small_stamp(a, 11);

  // phase 4: every owner's push landed in my Y; decode pass 1 (contiguous, in place)
  small_wait_peers(a, 1);
  small_stamp(a, 12);
  SnkDecode::B db;
  {
    const unsigned long long c = (1ULL << a.shard_shift) + __ldcg(a.counts + a.n + a.me);
    const double D = (double)a.dim;
    db = SnkDecode::B{a.out, a.dtype_out, a.L, a.signs, c == 0 ? 0.f : (float)((D / (double)c) / sqrt(D))};
  }
  const bool ovec = (((uintptr_t)a.out) & (a.dtype_out == OPTR_F32 ? 15 : 7)) == 0;
  {
    SmallBufSrc src{ym};
    if constexpr (K == T) {
      const SmallDecodeSnk dst{db, ovec};
      for (int64_t t = blockIdx.x; t < ntiles; t += G) rtile_do<T, 0, 0>(src, dst, t, sm);
    } else {
      const SnkBuf::B dst{ym, 1.f};
      for (int64_t t = blockIdx.x; t < ntiles; t += G) rtile_do<T, 0, 0>(src, dst, t, sm);
    }
  }
  small_stamp(a, 13);
  small_grid_sync(a.bar, a.bar_base + 4ULL * G);
  small_stamp(a, 14);

  // phase 5: decode pass 2 (strided) -> out
  if constexpr (K > T) {
    SmallBufSrc src{ym};
    const SmallDecodeSnk dst{db, ovec};
    for (int64_t t = blockIdx.x; t < ntiles; t += G) rtile_do<T, CB, T>(src, dst, t, sm);
  }
  if (a.received_out && blockIdx.x == 0 && tid < 2) a.received_out[tid] = __ldcg(a.counts + tid * a.n + a.me);
  small_stamp(a, 15);
}

}  // namespace optr

namespace optr {

// ---------------------------------------------------------------------------
// The same one-launch plan for n co-resident workers on ONE GPU
// (optr_tar_local, the reference simulator's shape: BASELINE configs[0]),
// without flags: (0) signs + every (stage, dst, src) mask row + counts;
// (1), (2) both encode passes of every worker; (3) every owner's stage-1
// mean pushed into every receiver's Y under its stage-2 mask (received
// flags optional); (4), (5) both decode passes of every worker.  Five grid
// barriers on a counter the caller zeroes with the counts.
struct SmallLocalArgs {
  PrepArgs pa;  // every (stage, dst) row; counts zeroed before the launch
  uint32_t* signs;
  u128 sign_state, sign_inc;
  const void* x[kMaxW];
  void* out[kMaxW];
  int dtype_in, dtype_out;
  int64_t L, dim;
  float* Y[kMaxW];                 // per-worker wire / stage-2 receive vectors
  unsigned long long* bar;         // grid-barrier arrivals (zeroed before the launch)
  unsigned long long* counts;      // [2][n]
  uint8_t* got;                    // optional [n][dim] received flags
  unsigned long long* received_out;  // optional [2][n] copy of the counts
  MaskView m;
  int n, r, shard_shift;
  unsigned long long* trace;  // optional debug stamps [8] (CTA 0, globaltimer ns)
};

__device__ __forceinline__ void small_local_stamp(const SmallLocalArgs& a, int i) {
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[i] = small_clock_ns();
}

// every row (stage, dst, src != dst), one packet per thread (small_masks)
__device__ __forceinline__ void small_local_masks(const SmallLocalArgs& a, int64_t gtid, int64_t gthreads,
                                                  const JumpSmem& jt) {
  const PrepArgs& pa = a.pa;
  const int n = a.n;
  const int64_t len = 1LL << a.shard_shift;
  const int64_t np = n_packets(len, pa.epp);
  const int64_t per_row = pa.pw * 32;
  const int64_t total = (int64_t)2 * n * (n - 1) * per_row;
  for (int64_t t = gtid; t < total; t += gthreads) {
    const int row = (int)(t / per_row);
    const int64_t p = t - (int64_t)row * per_row;
    const int stage = row / (n * (n - 1));
    const int rem = row - stage * n * (n - 1);
    const int dst = rem / (n - 1), srci = rem - dst * (n - 1);
    const int src = srci < dst ? srci : srci + 1;
    const int64_t widx = ((int64_t)(stage * n + dst) * n + src) * pa.pw + (p >> 5);
    bool keep = p < np;
    if (pa.kind == OPTR_MASK_COIN && keep) {
      const u128 s = jump_s(pa.coin_state[src], pa.coin_inc[src], coin_base(pa, stage, src, dst) + (uint64_t)p + 1, jt);
      keep = !coin_drops(pcg_xsl_rr(s), pa.drop_prob);
    } else if (pa.kind == OPTR_MASK_BITMAP && keep) {
      keep = (__ldg(pa.bitmap_in + widx) >> (p & 31)) & 1u;
    }
    const uint32_t bits = __ballot_sync(0xffffffffu, keep);
    if ((threadIdx.x & 31) == 0) {
      if (pa.kind != OPTR_MASK_BITMAP) pa.bitmap_out[widx] = bits;
      if (bits) {
        unsigned long long e = (unsigned long long)__popc(bits) * (unsigned long long)pa.epp;
        const int64_t last = np - 1 - (p & ~31LL);
        if (last >= 0 && last < 32 && ((bits >> last) & 1u)) e -= (unsigned long long)(np * pa.epp - len);
        atomicAdd(a.counts + stage * n + dst, e);
      }
    }
  }
}

// every owner's masked mean (fp64, ascending worker order) pushed into every
// receiver's Y under its stage-2 mask (collectives.py:77-94, 133-150)
template <int NR>
__device__ __forceinline__ void small_local_mean(const SmallLocalArgs& a, int64_t gtid, int64_t gthreads) {
  const int64_t n4 = a.dim >> 2;
  const int64_t smask = (1LL << a.shard_shift) - 1;
#pragma unroll 2
  for (int64_t g4 = gtid; g4 < n4; g4 += gthreads) {
    const int64_t g = g4 * 4;
    const int j = (int)(g >> a.shard_shift);
    const int o = shard_owner(j, a.r, NR);
    const uint32_t e = (uint32_t)(g & smask), wi = a.m.dv.div(e) >> 5;
    float4 v[NR];
    uint32_t w0[NR], w1[NR], s0[NR], s1[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      v[i] = ld_cg4(a.Y[i] + g);
      const uint32_t* row = a.m.row(0, o, i);  // stage 1: sender i -> owner o
      const uint32_t* srow = a.m.row(1, i, o);  // stage 2: owner o -> receiver i
      const bool own = i == o;
      w0[i] = own ? 0xffffffffu : __ldg(row + wi);
      w1[i] = (own || wi + 1 >= (uint32_t)a.m.pw) ? 0xffffffffu : __ldg(row + wi + 1);
      s0[i] = own ? 0xffffffffu : __ldg(srow + wi);
      s1[i] = (own || wi + 1 >= (uint32_t)a.m.pw) ? 0xffffffffu : __ldg(srow + wi + 1);
    }
    double acc[4] = {0.0, 0.0, 0.0, 0.0}, cnt[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const uint32_t kk = i == o ? 0xFu : keep4_words(e, w0[i], w1[i], a.m);
      acc[0] += (kk & 1u) ? (double)v[i].x : 0.0;
      acc[1] += (kk & 2u) ? (double)v[i].y : 0.0;
      acc[2] += (kk & 4u) ? (double)v[i].z : 0.0;
      acc[3] += (kk & 8u) ? (double)v[i].w : 0.0;
      cnt[0] += (kk & 1u) ? 1.0 : 0.0;
      cnt[1] += (kk & 2u) ? 1.0 : 0.0;
      cnt[2] += (kk & 4u) ? 1.0 : 0.0;
      cnt[3] += (kk & 8u) ? 1.0 : 0.0;
    }
    const float4 mv = make_float4(mean_of(acc[0], cnt[0]), mean_of(acc[1], cnt[1]), mean_of(acc[2], cnt[2]),
                                  mean_of(acc[3], cnt[3]));
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      const uint32_t kk = q == o ? 0xFu : keep4_words(e, s0[q], s1[q], a.m);
      st4(a.Y[q] + g, make_float4((kk & 1u) ? mv.x : 0.f, (kk & 2u) ? mv.y : 0.f, (kk & 4u) ? mv.z : 0.f,
                                  (kk & 8u) ? mv.w : 0.f));
      if (a.got)
        *reinterpret_cast<uchar4*>(a.got + (int64_t)q * a.dim + g) =
            make_uchar4(kk & 1u, (kk >> 1) & 1u, (kk >> 2) & 1u, (kk >> 3) & 1u);
    }
  }
}

template <int K>
__global__ void __launch_bounds__(1 << (kSmallT - 5)) tar_small_local_kernel(const __grid_constant__ SmallLocalArgs a) {
  extern __shared__ float sm[];
  constexpr int T = kSmallT;
  constexpr int CB = 2 * T - K;
  const int64_t ntiles = a.dim >> T;
  const int64_t njobs = ntiles * a.n;  // job = worker * ntiles + tile
  const int G = gridDim.x;
  const int tid = threadIdx.x;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + tid;
  const int64_t gthreads = (int64_t)G * blockDim.x;
  small_local_stamp(a, 0);
  __shared__ JumpSmem jt;
  if (tid < 64) {
    jt.a[tid] = c_jump.a[tid];
    jt.g[tid] = c_jump.g[tid];
  }
  __syncthreads();

  // phase 0: signs (32 per item, hadamard.py:49-51), masks, counts
  for (int64_t w = gtid; w < (a.dim >> 5); w += gthreads) {
    u128 s = jump_s(a.sign_state, a.sign_inc, (uint64_t)w * 16 + 1, jt);
    uint32_t word = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint64_t o = pcg_xsl_rr(s);
      word |= (uint32_t)((o >> 31) & 1u) << (2 * i);
      word |= (uint32_t)(o >> 63) << (2 * i + 1);
      s = pcg_step(s, a.sign_inc);
    }
    a.signs[w] = word;
  }
  small_local_masks(a, (int64_t)(G - 1 - blockIdx.x) * blockDim.x + tid, gthreads, jt);
  small_grid_sync(a.bar, 1ULL * G);
  small_local_stamp(a, 1);

  // phase 1: encode pass 1 (contiguous) of every worker
  for (int64_t k = blockIdx.x; k < njobs; k += G) {
    const int w = (int)(k / ntiles);
    SrcEncode::B eb{a.x[w], a.dtype_in, a.L, a.signs};
    SmallEncodeSrc src{eb, (((uintptr_t)a.x[w]) & (a.dtype_in == OPTR_F32 ? 15 : 7)) == 0};
    const SnkBuf::B dst{a.Y[w], K == T ? (float)(1.0 / sqrt((double)a.dim)) : 1.f};
    rtile_do<T, 0, 0>(src, dst, k - (int64_t)w * ntiles, sm);
  }
  small_grid_sync(a.bar, 2ULL * G);
  small_local_stamp(a, 2);

  // phase 2: encode pass 2 (strided, in place)
  if constexpr (K > T) {
    for (int64_t k = blockIdx.x; k < njobs; k += G) {
      const int w = (int)(k / ntiles);
      SmallBufSrc src{a.Y[w]};
      const SnkBuf::B dst{a.Y[w], (float)(1.0 / sqrt((double)a.dim))};
      rtile_do<T, CB, T>(src, dst, k - (int64_t)w * ntiles, sm);
    }
  }
  small_grid_sync(a.bar, 3ULL * G);
  small_local_stamp(a, 3);

  // phase 3: stage 1 at every owner, stage 2 pushed into every receiver
  switch (a.n) {
    case 2: small_local_mean<2>(a, gtid, gthreads); break;
    case 4: small_local_mean<4>(a, gtid, gthreads); break;
    default: small_local_mean<8>(a, gtid, gthreads); break;
  }
  small_grid_sync(a.bar, 4ULL * G);
  small_local_stamp(a, 4);
  if (a.received_out && blockIdx.x == 0 && tid < 2 * a.n) a.received_out[tid] = __ldcg(a.counts + tid);

  // phases 4, 5: the decode passes of every worker (count scale, signs, cast)
  const double D = (double)a.dim;
  auto dec_sink = [&](int w) {
    const unsigned long long c = (1ULL << a.shard_shift) + __ldcg(a.counts + a.n + w);
    const SnkDecode::B db{a.out[w], a.dtype_out, a.L, a.signs, c == 0 ? 0.f : (float)((D / (double)c) / sqrt(D))};
    return SmallDecodeSnk{db, (((uintptr_t)a.out[w]) & (a.dtype_out == OPTR_F32 ? 15 : 7)) == 0};
  };
  for (int64_t k = blockIdx.x; k < njobs; k += G) {
    const int w = (int)(k / ntiles);
    SmallBufSrc src{a.Y[w]};
    if constexpr (K == T) {
      rtile_do<T, 0, 0>(src, dec_sink(w), k - (int64_t)w * ntiles, sm);
    } else {
      const SnkBuf::B dst{a.Y[w], 1.f};
      rtile_do<T, 0, 0>(src, dst, k - (int64_t)w * ntiles, sm);
    }
  }
  if constexpr (K > T) {
    small_grid_sync(a.bar, 5ULL * G);
    small_local_stamp(a, 5);
    for (int64_t k = blockIdx.x; k < njobs; k += G) {
      const int w = (int)(k / ntiles);
      SmallBufSrc src{a.Y[w]};
      rtile_do<T, CB, T>(src, dec_sink(w), k - (int64_t)w * ntiles, sm);
    }
  }
  small_local_stamp(a, 6);
}

}  // namespace optr
