// C-ABI entry points (include/optr.h): host-side planning + kernel launches.
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <type_traits>
#include <mutex>
#include <vector>

#include "../../include/optr.h"
#include "kernels.cuh"
#include "tma.cuh"
#include "small.cuh"
#include "internal.h"

#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>

using namespace optr;

namespace {

// NVTX range around a public entry point (visible in nsys / ncu --nvtx)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

#define CK(call)                                                          \
  do {                                                                    \
    cudaError_t _e = (call);                                              \
    if (_e != cudaSuccess) {                                              \
      fprintf(stderr, "optr: %s failed: %s\n", #call, cudaGetErrorString(_e)); \
      return OPTR_ECUDA;                                                  \
    }                                                                     \
  } while (0)

int log2_exact(int64_t d) {
  int k = 0;
  while ((1LL << k) < d) ++k;
  return k;
}

bool is_pow2(int64_t d) { return d > 0 && (d & (d - 1)) == 0; }

int64_t next_pow2_i(int64_t n) {
  if (n <= 1) return 1;
  int64_t d = 1;
  while (d < n) d <<= 1;
  return d;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// ------------------------------------------------------ launch accounting
std::atomic<int64_t> g_launches{0};
std::mutex g_tmu;
bool g_timing = false;
struct TRec {
  int cls;
  int units;
  cudaEvent_t a, b;
};
std::vector<TRec> g_trecs;

// Brackets the kernel launches of one class with CUDA events on `st` when
// timing is enabled; always counts launches.
struct KScope {
  cudaStream_t st;
  int cls;
  int units;
  cudaEvent_t a = nullptr, b = nullptr;
  KScope(int c, cudaStream_t s, int u = 1) : st(s), cls(c), units(u) {
    g_launches += 1;
    if (g_timing) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, st);
    }
  }
  ~KScope() {
    if (a) {
      cudaEventRecord(b, st);
      std::lock_guard<std::mutex> lk(g_tmu);
      g_trecs.push_back(TRec{cls, units, a, b});
    }
  }
};

// Make this library's runtime use the device of the caller's stream (the
// library links its own static cudart; the caller's current device lives in
// the caller's runtime).
int bind_device(void* stream) {
  if (stream) {
    int dev = -1;
    if (cudaStreamGetDevice((cudaStream_t)stream, &dev) == cudaSuccess && dev >= 0) {
      int cur = -1;
      cudaGetDevice(&cur);
      if (cur != dev) CK(cudaSetDevice(dev));
    }
  }
  return OPTR_OK;
}

// Passes realising H_D = product over disjoint index-bit ranges.
// contiguous: bits [0, 13) on 8192-entry tiles; strided: bits [13, n) on
// 2^ks-row x 8-column tiles (split in two when n > 25).
constexpr int kContigBits = 13;
constexpr int kColBits = 3;

int plan_passes(int n, PassGeom* out, bool encode_order) {
  // A contiguous pass on 2^c-entry tiles plus strided passes of <= 11 row
  // bits on 2^ks x 8 tiles (T = ks + 3 <= 14: one CTA's registers).  Encode
  // runs the contiguous pass first (x streams from HBM) and decode runs it
  // last (out streams to HBM), so the strided passes, whose 32-byte row
  // segments are poor DRAM bursts, work on an L2-resident vector.
  PassGeom p[3];
  int np = 0;
  if (n <= kContigBits) {
    p[np++] = PassGeom{0, n, 0, 1};
  } else if (n <= kContigBits + 11) {
    p[np++] = PassGeom{0, kContigBits, 0, 0};
    p[np++] = PassGeom{kContigBits, n - kContigBits, kColBits, 0};
  } else if (n == kContigBits + 12) {
    p[np++] = PassGeom{0, kContigBits + 1, 0, 0};
    p[np++] = PassGeom{kContigBits + 1, n - kContigBits - 1, kColBits, 0};
  } else {
    // three passes (D >= 2^26): the strided passes take 32 columns (128-byte
    // rows, full L2 lines) while T = ks + 5 <= 14; with 8 columns their tiles
    // were 2^9..2^10 entries of 32-byte rows at multi-MB strides (~1.2-1.5
    // TB/s).
    // The high pass takes 6 bits (T = 11): the multi-GPU decode ends with it
    // and the TMA decode epilogue needs float4 groups in its last register
    // round (32-column T = 11 / 14 tiles; T = 12 / 13 end on other bits).
    int rest = n - kContigBits;
    int k1 = rest - 6 <= 9 ? rest - 6 : rest / 2;
    const int cb = k1 + 5 <= 14 ? 5 : kColBits;
    p[np++] = PassGeom{0, kContigBits, 0, 0};
    p[np++] = PassGeom{kContigBits, k1, cb, 0};
    p[np++] = PassGeom{kContigBits + k1, rest - k1, cb, 0};
  }
  for (int i = 0; i < np; ++i) p[i].ntiles = (1LL << n) >> (p[i].cb + p[i].ks);
  for (int i = 0; i < np; ++i) out[i] = encode_order ? p[i] : p[np - 1 - i];
  return np;
}

std::mutex g_attr_mu;

// one-time per-device setup: PCG jump table in constant memory
int ensure_device_init() {
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_attr_mu);
  if (!done[dev & 63]) {
    JumpTable t = make_jump_table();
    CK(cudaMemcpyToSymbol(c_jump, &t, sizeof(t)));
    done[dev & 63] = true;
  }
  return OPTR_OK;
}

// After a launch: on failure report the kernel's resource limits.
template <class K>
int launch_check(K kernel, const char* name, int T, int CB, int gx, int gy, int threads, size_t smem) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return OPTR_OK;
  cudaFuncAttributes fa;
  memset(&fa, 0, sizeof(fa));
  cudaFuncGetAttributes(&fa, kernel);
  fprintf(stderr,
          "optr: %s<T=%d,CB=%d> launch grid=(%d,%d) block=%d smem=%zu failed: %s "
          "(regs=%d maxThreads=%d maxDynSmem=%d)\n",
          name, T, CB, gx, gy, threads, smem, cudaGetErrorString(e), fa.numRegs, fa.maxThreadsPerBlock,
          fa.maxDynamicSharedSizeBytes);
  return OPTR_ECUDA;
}

template <class K>
int set_smem_attr(K kernel, size_t smem) {
  if (smem <= 48 * 1024) return OPTR_OK;
  CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return OPTR_OK;
}

constexpr int64_t kMaxGrid = 148 * 16;

template <int T, int CB, int LO, class Src, class Snk>
int launch_rtile(int cls, const PassGeom& pg, int worker_base, int nworkers, const Src& src, const Snk& snk,
                 cudaStream_t st) {
  const size_t smem = sizeof(float) * (size_t)pad(1 << T);
  int rc = set_smem_attr(rtile_kernel<T, CB, LO, Src, Snk>, smem);
  if (rc) return rc;
  const int64_t gx = pg.ntiles < kMaxGrid ? pg.ntiles : kMaxGrid;
  KScope ks(cls, st, nworkers);
  rtile_kernel<T, CB, LO, Src, Snk><<<dim3((unsigned)gx, (unsigned)nworkers), 1 << (T - 5), smem, st>>>(
      pg, worker_base, src, snk);
  return launch_check(rtile_kernel<T, CB, LO, Src, Snk>, "rtile", T, CB, (int)gx, nworkers, 1 << (T - 5), smem);
}

template <class Src, class Snk>
int launch_smem(int cls, const PassGeom& pg, int worker_base, int nworkers, const Src& src, const Snk& snk,
                cudaStream_t st) {
  const int nelem = 1 << (pg.cb + pg.ks);
  const size_t smem = (size_t)nelem * sizeof(float);
  int rc = set_smem_attr(smem_tile_kernel<Src, Snk>, smem);
  if (rc) return rc;
  const int64_t gx = pg.ntiles < kMaxGrid ? pg.ntiles : kMaxGrid;
  int threads = nelem / 32;
  if (threads < 32) threads = 32;
  if (threads > 256) threads = 256;
  KScope ks(cls, st, nworkers);
  smem_tile_kernel<Src, Snk><<<dim3((unsigned)gx, (unsigned)nworkers), threads, smem, st>>>(pg, worker_base, src,
                                                                                            snk);
  return launch_check(smem_tile_kernel<Src, Snk>, "smem_tile", pg.cb + pg.ks, pg.cb, (int)gx, nworkers, threads,
                      smem);
}



// Launch with programmatic stream serialization (PDL) so the kernel is
// scheduled while its predecessor drains; the kernels call
// griddepcontrol.wait before touching dependent memory.  Off while timing
// (the per-launch events would serialise anyway).
template <class K, class... Args>
cudaError_t launch_ex(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_timing ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// ------------------------------------------------------------ TMA strided
PFN_cuTensorMapEncodeTiled_v12000 g_encode_tiled = nullptr;
int g_tma_mode = -1;  // -1 unknown, 0 off, 1 on

// TMA tensor maps need the driver's cuTensorMapEncodeTiled
bool tma_enabled() {
  if (g_tma_mode < 0) {
    g_tma_mode = 1;
    {
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&g_encode_tiled, cudaEnableDefault, &q) !=
              cudaSuccess ||
          q != cudaDriverEntryPointSuccess || !g_encode_tiled)
        g_tma_mode = 0;
    }
  }
  return g_tma_mode == 1;
}

// tensor [d2][d1][d0] (d0 contiguous) of fp32 / bf16, boxes of box0 x box1 x 1.
// Encoded maps are cached per host thread (the key determines the map): the
// same buckets / workspaces recur every step.
struct MapKey {
  const void* base;
  uint64_t d0, d1, d2;
  uint32_t box0, box1;
  int dtype;
  bool operator==(const MapKey& o) const {
    return base == o.base && d0 == o.d0 && d1 == o.d1 && d2 == o.d2 && box0 == o.box0 && box1 == o.box1 &&
           dtype == o.dtype;
  }
};
bool make_map3_uncached(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t box1,
                        int dtype, uint32_t box0);
bool make_map3(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t box1,
               int dtype = OPTR_F32, uint32_t box0 = 8) {
  constexpr int kSlots = 256;
  struct Slot {
    MapKey k;
    CUtensorMap m;
    bool valid;
  };
  thread_local Slot cache[kSlots];
  const MapKey k{base, d0, d1, d2, box0, box1, dtype};
  uint64_t h = (uint64_t)(uintptr_t)base * 0x9E3779B97F4A7C15ULL ^ (d0 * 31 + d1 * 17 + d2 * 7 + box0 * 3 + box1 + dtype);
  h ^= h >> 29;
  Slot& sl = cache[h % kSlots];
  if (sl.valid && sl.k == k) {
    *m = sl.m;
    return true;
  }
  if (!make_map3_uncached(m, base, d0, d1, d2, box1, dtype, box0)) return false;
  sl.k = k;
  sl.m = *m;
  sl.valid = true;
  return true;
}
bool make_map3_uncached(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t box1,
                        int dtype, uint32_t box0) {
  if (((uintptr_t)base) & 15) return false;  // TMA needs a 16-byte aligned global address: LSU path
  const uint64_t esz = dtype == OPTR_BF16 ? 2 : 4;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0 * esz, d0 * d1 * esz};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode_tiled(m, dtype == OPTR_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                              3, const_cast<void*>(base), dims, strides, box,
                              es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fprintf(stderr, "optr: cuTensorMapEncodeTiled failed (%d)\n", (int)r);
  return r == CUDA_SUCCESS;
}

template <int T, int S, bool STRIDED, int SK, class Snk, int CBW>
int launch_tma_pass_s(int cls, const TmaMaps& maps, const TmaMaps& dmaps, const TmaArgs& a, const Snk& snk,
                      int worker, int nworkers, cudaStream_t st) {
  const size_t smem = tma_smem_bytes<T, S>();
  auto kern = tma_pass_kernel<T, S, STRIDED, SK, Snk, CBW>;
  int rc = set_smem_attr(kern, smem);
  if (rc) return rc;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  // CTAs per SM by shared memory, capped by what is resident (registers can
  // bind first: a grid past residency runs as a partial second wave)
  int per_sm = (int)((227 * 1024) / (smem + 1024));
  int resident = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, kern, 1 << (T - 5), smem) == cudaSuccess &&
      resident >= 1 && resident < per_sm)
    per_sm = resident;
  if (per_sm < 1) per_sm = 1;
  int64_t gx = ((int64_t)nsm * per_sm + nworkers - 1) / nworkers;
  if (gx > a.ntiles) gx = a.ntiles;
  KScope ks(cls, st, nworkers);
  launch_ex(kern, dim3((unsigned)gx, (unsigned)nworkers), dim3(1 << (T - 5)), smem, st, maps, dmaps, a, snk, worker);
  return launch_check(kern, STRIDED ? "tma_strided" : "tma_contig", T, STRIDED ? 3 : 0, (int)gx, nworkers,
                      1 << (T - 5), smem);
}

// ring depth of the TMA pass kernels: 2, strided T >= 13 tiles 3 (D = 2^25:
// the strided pass waits on its 32-byte-row TMA boxes with one CTA per SM;
// a third stage takes it from 90 to 60 us; at D = 2^23 with the workers
// batched, 2 CTAs x 3 stages beat 3 x 2 by ~2%; contiguous is flat from 2 up;
// profiles/r01_stage_sweep.jsonl).
template <int T, bool STRIDED, int SK, class Snk, int CBW = 3>
int launch_tma_pass(int cls, const TmaMaps& maps, const TmaMaps& dmaps, const TmaArgs& a, const Snk& snk,
                    int worker, int nworkers, cudaStream_t st) {
  // (T = 14 strided with one stage at two CTAs per SM: 242 -> 262 us at N=1)
  if constexpr (STRIDED && T >= 13)
    return launch_tma_pass_s<T, 3, STRIDED, SK, Snk, CBW>(cls, maps, dmaps, a, snk, worker, nworkers, st);
  else
    return launch_tma_pass_s<T, 2, STRIDED, SK, Snk, CBW>(cls, maps, dmaps, a, snk, worker, nworkers, st);
}

// A pass through the TMA ring kernel when the shapes allow it; -1 when the
// caller should use the LSU kernels instead.  Workers [worker, worker+nworkers)
// go in one launch (grid.y = worker).
template <class Src, class Snk>
int try_tma(int cls, const PassGeom& pg, int nlog, int worker, int nworkers, const Src& src, const Snk& snk,
            cudaStream_t st) {
  constexpr bool kBuf = std::is_same<Src, SrcBuf>::value;
  constexpr bool kEnc = std::is_same<Src, SrcEncode>::value;
  constexpr bool kGather = std::is_same<Src, SrcGather>::value;
  constexpr bool kSnkBuf = std::is_same<Snk, SnkBuf>::value;
  constexpr int SK = kBuf ? TS_BUF : (kEnc ? TS_ENC : TS_GATHER);
  if constexpr (!(kBuf || kEnc || kGather)) {
    return -1;
  } else {
    const int T = pg.cb + pg.ks;
    if (!tma_enabled()) return -1;
    TmaArgs a;
    memset(&a, 0, sizeof(a));
    a.ntiles = pg.ntiles;
    a.lo = pg.lo;
    TmaMaps maps, dmaps;
    memset(&maps, 0, sizeof(maps));
    memset(&dmaps, 0, sizeof(dmaps));
    if constexpr (kGather) {
      for (int o = 0; o < src.n; ++o) a.A[o] = src.A[o];
      a.n = src.n;
      a.r = src.r;
      a.shard_shift = src.pow2_shift;
      a.m = src.m;
      a.got = src.got;
      a.dim = src.dim;
      a.tile_ok2 = (pg.cb == 0 && pg.lo == 0) ? src.tile_ok2 : nullptr;  // tiles of the fast plan's contiguous pass
    }
    if (pg.cb == 3 || pg.cb == 5) {  // strided: tensor boxes in, tensor boxes out
      if constexpr (kEnc) {
        // strided-first encode (the fused multi-GPU path): x as [rows_full][2^lo]
        if (pg.cb != 3 || (T != 13 && T != 14)) return -1;
        const uint64_t d0 = 1ULL << pg.lo, d1 = 1ULL << pg.ks;
        if (nlog != pg.lo + pg.ks) return -1;  // two-pass plans only (no outer blocks)
        const int64_t rows_full = src.L >> pg.lo;
        if (rows_full < 1) return -1;
        const int box = (int)(d1 < 256 ? d1 : 256);
        for (int w = worker; w < worker + nworkers; ++w) {
          if (((uintptr_t)src.x[w] & 15) || !make_map3(&maps.m[w], src.x[w], d0, (uint64_t)rows_full, 1,
                                                         (uint32_t)box, src.dtype))
            return -1;
          a.xw[w] = src.x[w];
          if (!make_map3(&dmaps.m[w], snk.y[w], d0, d1, 1, (uint32_t)box)) return -1;
        }
        a.dtype = src.dtype;
        a.L = src.L;
        a.signs = src.signs;
        a.signs_t = src.signs_t;
        a.scale = snk.scale;
        a.box_rows = box;
        if (T == 13) return launch_tma_pass<13, true, SK>(cls, maps, dmaps, a, snk, worker, nworkers, st);
        return launch_tma_pass<14, true, SK>(cls, maps, dmaps, a, snk, worker, nworkers, st);
      } else {
        if (T < 9 || T > 14 || (pg.cb == 5 && T < 11)) return -1;
        const uint32_t bw = 1u << pg.cb;
        const uint64_t d0 = 1ULL << pg.lo, d1 = 1ULL << pg.ks, d2 = 1ULL << (nlog - pg.lo - pg.ks);
        int box = (int)(d1 < 256 ? d1 : 256);
        if constexpr (kGather) {
          if (src.pow2_shift < pg.lo || d2 != 1) return -1;
          const int64_t srows = 1LL << (src.pow2_shift - pg.lo);
          if (srows < box) box = (int)srows;
          for (int o = 0; o < src.n; ++o)
            if (!make_map3(&maps.m[o], src.A[o], d0, (uint64_t)srows, 1, (uint32_t)box, OPTR_F32, bw)) return -1;
        }
        for (int w = worker; w < worker + nworkers; ++w) {
          if constexpr (kBuf) {
            if (!make_map3(&maps.m[w], src.y[w], d0, d1, d2, (uint32_t)box, OPTR_F32, bw)) return -1;
          }
          if constexpr (kSnkBuf) {
            if (!make_map3(&dmaps.m[w], snk.y[w], d0, d1, d2, (uint32_t)box, OPTR_F32, bw)) return -1;
          } else {  // decode epilogue: map over the full rows of `out`
            if (d2 != 1) return -1;
            const int64_t rows_full = snk.L >> pg.lo;
            if (rows_full > 0 &&
                !make_map3(&dmaps.m[w], snk.out[w], d0, (uint64_t)rows_full, 1, (uint32_t)box, snk.dtype, bw))
              return -1;
            if (((uintptr_t)snk.out[w] & 15) || ((uintptr_t)snk.signs & 15)) return -1;
          }
        }
        if constexpr (kSnkBuf) a.scale = snk.scale;
        if constexpr (!kSnkBuf) {
          if (pg.cb == 3) a.signs_t = snk.signs_t;
        }
        a.box_rows = box;
        if (pg.cb == 5) {
          if constexpr (kSnkBuf) {  // three-pass plans (32-column tiles)
            switch (T) {
              case 11: return launch_tma_pass<11, true, SK, Snk, 5>(cls, maps, dmaps, a, snk, worker, nworkers, st);
              case 12: return launch_tma_pass<12, true, SK, Snk, 5>(cls, maps, dmaps, a, snk, worker, nworkers, st);
              case 13: return launch_tma_pass<13, true, SK, Snk, 5>(cls, maps, dmaps, a, snk, worker, nworkers, st);
              default: break;
            }
          }
          if (T == 11) return launch_tma_pass<11, true, SK, Snk, 5>(cls, maps, dmaps, a, snk, worker, nworkers, st);
          if (T != 14) return -1;
          return launch_tma_pass<14, true, SK, Snk, 5>(cls, maps, dmaps, a, snk, worker, nworkers, st);
        }
        if constexpr (kSnkBuf) {  // small strided tiles (3-pass plans of D >= 2^26)
          switch (T) {
            case 9: return launch_tma_pass<9, true, SK>(cls, maps, dmaps, a, snk, worker, nworkers, st);
            case 10: return launch_tma_pass<10, true, SK>(cls, maps, dmaps, a, snk, worker, nworkers, st);
            case 11: return launch_tma_pass<11, true, SK>(cls, maps, dmaps, a, snk, worker, nworkers, st);
            default: break;
          }
        } else {
          if (T < 12) return -1;  // the decode epilogue needs float4 groups in the last round
        }
        switch (T) {
          case 12: return launch_tma_pass<12, true, SK>(cls, maps, dmaps, a, snk, worker, nworkers, st);
          case 13: return launch_tma_pass<13, true, SK>(cls, maps, dmaps, a, snk, worker, nworkers, st);
          default: return launch_tma_pass<14, true, SK>(cls, maps, dmaps, a, snk, worker, nworkers, st);
        }
      }
    }
    if (pg.cb != 0 || pg.lo != 0 || (T != 13 && T != 14)) return -1;
    for (int w = worker; w < worker + nworkers; ++w) {
      if constexpr (kBuf) {
        a.xw[w] = src.y[w];
      } else if constexpr (kEnc) {
        a.xw[w] = src.x[w];
        if (((uintptr_t)a.xw[w] & 15) || ((uintptr_t)src.signs & 15)) return -1;
      }
    }
    if constexpr (kEnc) {
      a.dtype = src.dtype;
      a.L = src.L;
      a.signs = src.signs;
    }
    if constexpr (kGather) {
      if (src.pow2_shift < T) return -1;
    }
    if (T == 13) return launch_tma_pass<13, false, SK>(cls, maps, dmaps, a, snk, worker, nworkers, st);
    return launch_tma_pass<14, false, SK>(cls, maps, dmaps, a, snk, worker, nworkers, st);
  }
}

constexpr int kAggChunk = 1024;

int launch_tma_aggregate(const AggArgs& ag, int nowners, int64_t smax, cudaStream_t st) {
  TmaAggArgs a;
  memset(&a, 0, sizeof(a));
  for (int i = 0; i < ag.n; ++i) {
    a.Y[i] = ag.Y[i];
    a.A[i] = ag.A[i];
    a.G[i] = ag.G[i];
  }
  a.push = ag.push;
  a.sh = ag.sh;
  a.n = ag.n;
  a.r = ag.r;
  a.owner_base = ag.owner_base;
  a.m = ag.m;
  // chunk ring depth 2 (4 measured slower on one GPU, 1.013 vs 0.988 ms/step:
  // more CTAs per SM beat a deeper ring here)
  const size_t smem = tma_agg_smem_bytes<kAggChunk, 2>(ag.n);
  auto kern = ag.n == 2 ? tma_agg_kernel<kAggChunk, 2, 2>
              : ag.n == 4 ? tma_agg_kernel<kAggChunk, 4, 2>
              : ag.n == 8 ? tma_agg_kernel<kAggChunk, 8, 2>
                          : tma_agg_kernel<kAggChunk, 0, 2>;
  int rc = set_smem_attr(kern, smem);
  if (rc) return rc;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  int per_sm = (int)((227 * 1024) / (smem + 1024));
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 8) per_sm = 8;
  const int64_t nchunks = (smax + kAggChunk - 1) / kAggChunk;
  int64_t gx = (int64_t)nsm * per_sm / nowners;
  if (gx < 1) gx = 1;
  if (gx > nchunks) gx = nchunks;
  KScope ks(OPTR_K_AGG, st, nowners);
  launch_ex(kern, dim3((unsigned)gx, (unsigned)nowners), dim3(kAggChunk / 4), smem, st, a);
  return launch_check(kern, "tma_aggregate", 0, 0, (int)gx, nowners, kAggChunk / 4, smem);
}

template <class S>
constexpr bool kStridedSrc = !std::is_same<S, SrcEncode>::value;
template <class S>
constexpr bool kStridedSnk = !std::is_same<S, SnkDecode>::value;

template <class Src, class Snk>
int launch_pass(int cls, const PassGeom& pg, int nlog, int worker_base, int nworkers, const Src& src,
                const Snk& snk, cudaStream_t st) {
  const int T = pg.cb + pg.ks;
  {
    int rc = try_tma(cls, pg, nlog, worker_base, nworkers, src, snk, st);
    if (rc >= 0) return rc;
  }
  if (pg.cb == 0 && pg.lo == 0 && T == 13) return launch_rtile<13, 0, 0>(cls, pg, worker_base, nworkers, src, snk, st);
  if (pg.cb == 0 && pg.lo == 0 && T == 14) return launch_rtile<14, 0, 0>(cls, pg, worker_base, nworkers, src, snk, st);
  if constexpr (kStridedSrc<Src> && kStridedSnk<Snk>) {
    if (pg.cb == 3 && pg.lo == 13) {
      switch (T) {
        case 11: return launch_rtile<11, 3, 13>(cls, pg, worker_base, nworkers, src, snk, st);
        case 12: return launch_rtile<12, 3, 13>(cls, pg, worker_base, nworkers, src, snk, st);
        case 13: return launch_rtile<13, 3, 13>(cls, pg, worker_base, nworkers, src, snk, st);
        case 14: return launch_rtile<14, 3, 13>(cls, pg, worker_base, nworkers, src, snk, st);
        default: break;
      }
    }
    if (pg.cb == 3 && pg.lo == 14) {
      switch (T) {
        case 13: return launch_rtile<13, 3, 14>(cls, pg, worker_base, nworkers, src, snk, st);
        case 14: return launch_rtile<14, 3, 14>(cls, pg, worker_base, nworkers, src, snk, st);
        default: break;
      }
    }
  }
  return launch_smem(cls, pg, worker_base, nworkers, src, snk, st);
}

// Run the pass list with a fused first-pass source and last-pass sink; the
// intermediate passes work in place on `buf`.
template <class Src, class Snk>
int run_transform(int nlog, bool encode_order, int worker_base, int nworkers, const Src& src,
                  const SrcBuf& buf, const Snk& snk, cudaStream_t st, int cls0 = OPTR_K_OTHER) {
  const int c_first = cls0, c_mid = cls0 == OPTR_K_OTHER ? cls0 : cls0 + 1,
            c_last = cls0 == OPTR_K_OTHER ? cls0 : cls0 + 2;
  PassGeom ps[3];
  int np = plan_passes(nlog, ps, encode_order);
  SnkBuf mid;
  for (int i = 0; i < kMaxW; ++i) mid.y[i] = buf.y[i];
  mid.scale = 1.f;
  int rc;
  if (np == 1) return launch_pass(c_first, ps[0], nlog, worker_base, nworkers, src, snk, st);
  if ((rc = launch_pass(c_first, ps[0], nlog, worker_base, nworkers, src, mid, st))) return rc;
  for (int i = 1; i < np - 1; ++i)
    if ((rc = launch_pass(c_mid, ps[i], nlog, worker_base, nworkers, buf, mid, st))) return rc;
  return launch_pass(c_last, ps[np - 1], nlog, worker_base, nworkers, buf, snk, st);
}


// float4 path of the aggregate needs every shard offset and buffer 16B-aligned
bool agg_vec_ok(const AggArgs& a) {
  if (a.sh.extra != 0 || (a.sh.base & 3) != 0) return false;
  for (int i = 0; i < a.n; ++i)
    if (((uintptr_t)a.Y[i] & 15) || ((uintptr_t)a.A[i] & 15)) return false;
  return true;
}

int launch_tma_aggregate(const AggArgs& ag, int nowners, int64_t smax, cudaStream_t st);

int launch_aggregate(const AggArgs& ag, int nowners, int64_t smax, cudaStream_t st) {
  if (smax <= 0) return OPTR_OK;
  if (agg_vec_ok(ag) && tma_enabled()) return launch_tma_aggregate(ag, nowners, smax, st);
  int64_t blocks = (smax / 4 + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > kMaxGrid) blocks = kMaxGrid;
  KScope ks(OPTR_K_AGG, st, nowners);
  if (agg_vec_ok(ag))
    aggregate_kernel<true><<<dim3((unsigned)blocks, nowners), 256, 0, st>>>(ag);
  else
    aggregate_kernel<false><<<dim3((unsigned)blocks, nowners), 256, 0, st>>>(ag);
  CK(cudaGetLastError());
  return OPTR_OK;
}

Pcg sign_pcg(uint64_t seed) { return pcg_from_u64s(&seed, 1); }

// Decode pass order: contiguous first (the stage-2 receive then works on
// whole packets per tile, and over NVLink pulls whole owner chunks with bulk
// copies) whenever the strided pass can finish into `out` with the TMA decode
// epilogue and transposed signs (two passes, 8-column strided tiles of
// T >= 12); strided first otherwise.
// Multi-GPU (unfused) always decodes contiguous-first.
bool decode_contig_first(int nlog, bool multi_gpu) {
  PassGeom ps[3];
  return multi_gpu || (plan_passes(nlog, ps, true) == 2 && ps[1].cb == 3 && ps[1].ks + 3 >= 12);
}

void fill_sign_args(PrepArgs& a, uint32_t* signs, int64_t dim, uint64_t seed) {
  Pcg p = sign_pcg(seed);
  a.signs = signs;
  a.dim = dim;
  a.sign_state = p.state;
  a.sign_inc = p.inc;
  a.sign_threads = (dim + kSignsPerThread - 1) / kSignsPerThread;
}

// cap_per_sm > 0: at most that many CTAs per SM (grid-stride), for a prep
// that runs in the background beside another call's kernels.
int launch_prep(const PrepArgs& a, cudaStream_t st, int cap_per_sm = 0) {
  int64_t total = a.sign_threads + a.mask_threads;
  if (total == 0) return OPTR_OK;
  int rc = ensure_device_init();
  if (rc) return rc;
  // (128-thread background CTAs measured slower at N=4: 0.639 vs 0.612 ms)
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (cap_per_sm > 0) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (blocks > (int64_t)nsm * cap_per_sm) blocks = (int64_t)nsm * cap_per_sm;
  }
  KScope ks(OPTR_K_PREP, st);
  prep_kernel<<<(unsigned)blocks, threads, 0, st>>>(a);
  CK(cudaGetLastError());
  return OPTR_OK;
}

int64_t mask_words(int64_t dim, int n, int epp) {
  Shards sh = make_shards(dim, n);
  int64_t maxlen = sh.base + (sh.extra ? 1 : 0);
  int64_t np = n_packets(maxlen, epp);
  int64_t w = (np + 31) / 32;
  return w > 0 ? w : 1;
}

// Mask/count setup shared by local and multi-GPU paths.
int setup_masks(PrepArgs& a, const optr_mask_spec* ms, int64_t dim, int n, int r, int epp,
                uint32_t* bitmap_ws, unsigned long long* counts, int dst_lo, int dst_hi,
                const uint32_t** bitmap_for_consumers) {
  a.kind = ms ? ms->kind : OPTR_MASK_NONE;
  a.n = n;
  a.r = r;
  a.epp = epp;
  a.sh = make_shards(dim, n);
  a.pw = mask_words(dim, n, epp);
  a.bitmap_out = bitmap_ws;
  a.bitmap_in = (ms && ms->kind == OPTR_MASK_BITMAP) ? ms->bitmap : nullptr;
  if (a.kind == OPTR_MASK_BITMAP && !a.bitmap_in) return OPTR_EINVAL;
  if (a.kind != OPTR_MASK_NONE && a.kind != OPTR_MASK_COIN && a.kind != OPTR_MASK_BITMAP)
    return OPTR_EINVAL;
  a.drop_prob = ms ? ms->drop_prob : 0.0;
  if (a.kind == OPTR_MASK_COIN) {
    for (int s = 0; s < n; ++s) {
      uint64_t ent[2] = {ms->seed, (uint64_t)s};
      Pcg p = pcg_from_u64s(ent, 2);
      // a continued stream starts after the sender's earlier draws
      a.coin_state[s] = ms->stream_offsets ? pcg_advance(p.state, p.inc, ms->stream_offsets[s]) : p.state;
      a.coin_inc[s] = p.inc;
    }
  }
  a.dst_lo = dst_lo;
  a.dst_hi = dst_hi;
  a.mask_threads = (int64_t)(dst_hi - dst_lo) * 2 * (n - 1) * a.pw;
  a.counts = counts;
  *bitmap_for_consumers = a.kind == OPTR_MASK_BITMAP ? a.bitmap_in : bitmap_ws;
  return OPTR_OK;
}

int check_common(int n, int64_t L, int dtype_in, int dtype_out, const optr_mask_spec* ms) {
  if (n < 2 || n > OPTR_MAX_WORKERS) return OPTR_EINVAL;  // schedule.py:21-22
  if (L < 0) return OPTR_EINVAL;
  if ((dtype_in != OPTR_F32 && dtype_in != OPTR_BF16) || (dtype_out != OPTR_F32 && dtype_out != OPTR_BF16))
    return OPTR_EINVAL;
  int epp = ms ? ms->epp : 350;
  if (epp <= 0) return OPTR_EINVAL;
  if (ms && ms->kind == OPTR_MASK_COIN && !(ms->drop_prob >= 0.0 && ms->drop_prob <= 1.0)) return OPTR_EINVAL;
  return OPTR_OK;
}

}  // namespace

void optr_note_launches(int k) { g_launches += k; }
void optr_bind_stream_device(void* stream) { bind_device(stream); }

extern "C" {

// ------------------------------------------------------------ host helpers
uint64_t optr_derive_seed(uint64_t job_seed, uint64_t bucket_id, uint64_t generation) {
  return derive_seed(job_seed, bucket_id, generation);
}

uint64_t optr_pcg64_output(const uint64_t* entropy, int n_entropy, uint64_t k) {
  Pcg p = pcg_from_u64s(entropy, n_entropy);
  return pcg_output_at(p, k);
}

int64_t optr_next_pow2(int64_t n) { return next_pow2_i(n); }

int64_t optr_mask_words(int64_t dim, int n, int epp) {
  if (n < 1 || epp <= 0 || dim < 0) return -1;
  return mask_words(dim, n, epp);
}

int optr_coin_packets(uint64_t seed, int src, uint64_t start, int64_t count, double p, uint8_t* keep) {
  if (src < 0 || count < 0 || (count > 0 && !keep) || !(p >= 0.0 && p <= 1.0)) return OPTR_EINVAL;
  uint64_t ent[2] = {seed, (uint64_t)src};
  Pcg g = pcg_from_u64s(ent, 2);
  u128 s = pcg_advance(g.state, g.inc, start);
  for (int64_t k = 0; k < count; ++k) {
    s = pcg_step(s, g.inc);
    keep[k] = coin_drops(pcg_xsl_rr(s), p) ? 0 : 1;
  }
  return OPTR_OK;
}

int optr_masks_host(uint32_t* bm, int64_t dim, int n, int rotation, uint64_t seed, double p, int epp) {
  if (n < 2 || n > OPTR_MAX_WORKERS || epp <= 0 || dim < 0 || !bm) return OPTR_EINVAL;
  int r = ((rotation % n) + n) % n;
  Shards sh = make_shards(dim, n);
  int64_t pw = mask_words(dim, n, epp);
  memset(bm, 0, sizeof(uint32_t) * (size_t)(2 * n * n * pw));
  for (int src = 0; src < n; ++src) {
    uint64_t ent[2] = {seed, (uint64_t)src};
    Pcg g = pcg_from_u64s(ent, 2);
    u128 s = g.state;
    for (int stage = 0; stage < 2; ++stage) {
      for (int o = 1; o < n; ++o) {
        int dst = (src + o) % n;
        int j = stage == 0 ? owned_shard(dst, r, n) : owned_shard(src, r, n);
        int64_t np = n_packets(sh.len(j), epp);
        uint32_t* row = bm + ((int64_t)(stage * n + dst) * n + src) * pw;
        for (int64_t k = 0; k < np; ++k) {
          bool keep = true;
          if (p > 0) {  // datagram.py:122 draws only when drop_prob > 0
            s = pcg_step(s, g.inc);
            keep = !coin_drops(pcg_xsl_rr(s), p);
          }
          if (keep) row[k >> 5] |= 1u << (k & 31);
        }
      }
    }
  }
  return OPTR_OK;
}

int optr_mean_received(const float* own, const float* const* peers, const uint8_t* const* masks, int n, int rank,
                       int64_t len, float* out, void* stream) {
  if (n < 1 || n > OPTR_MAX_WORKERS || rank < 0 || rank >= n || len < 0 || !peers) return OPTR_EINVAL;
  if (len > 0 && (!own || !out)) return OPTR_EINVAL;
  if (len == 0) return OPTR_OK;
  bind_device(stream);
  MeanRecvArgs a;
  memset(&a, 0, sizeof(a));
  a.own = own;
  for (int i = 0; i < n; ++i) {
    a.peers[i] = peers[i];
    a.masks[i] = masks ? masks[i] : nullptr;
  }
  a.n = n;
  a.rank = rank;
  a.len = len;
  a.out = out;
  int64_t blocks = (len + 255) / 256;
  if (blocks > kMaxGrid) blocks = kMaxGrid;
  KScope ks(OPTR_K_AGG, (cudaStream_t)stream);
  mean_received_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(a);
  CK(cudaGetLastError());
  return OPTR_OK;
}

const char* optr_version(void) { return "optr 0.1 sm_100a"; }

// ---------------------------------------------------------------- codec
int optr_rht_signs(uint32_t* sign_bits, int64_t dim, uint64_t seed, void* stream) {
  if (!is_pow2(dim) || !sign_bits) return OPTR_EINVAL;
  bind_device(stream);
  PrepArgs a;
  memset(&a, 0, sizeof(a));
  fill_sign_args(a, sign_bits, dim, seed);
  return launch_prep(a, (cudaStream_t)stream);
}

int optr_fwht(float* v, int64_t dim, void* stream) {
  if (!is_pow2(dim) || !v) return OPTR_EINVAL;  // hadamard.py:78-81
  bind_device(stream);
  SrcBuf b;
  memset(&b, 0, sizeof(b));
  b.y[0] = v;
  SnkBuf s;
  memset(&s, 0, sizeof(s));
  s.y[0] = v;
  s.scale = 1.f;
  return run_transform(log2_exact(dim), true, 0, 1, b, b, s, (cudaStream_t)stream);
}

int optr_rht_encode(const void* x, int dtype_in, int64_t L, float* y, int64_t dim, uint64_t seed,
                    void* stream) {
  if (!is_pow2(dim) || L > dim || L < 0 || !y || (L > 0 && !x)) return OPTR_EINVAL;  // hadamard.py:45-48,96-97
  if (dtype_in != OPTR_F32 && dtype_in != OPTR_BF16) return OPTR_EINVAL;
  bind_device(stream);
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* signs = nullptr;
  size_t sbytes = (size_t)((dim + 31) / 32) * 4;
  CK(cudaMallocAsync((void**)&signs, sbytes + 16, st));
  PrepArgs a;
  memset(&a, 0, sizeof(a));
  fill_sign_args(a, signs, dim, seed);
  int rc = launch_prep(a, st);
  if (!rc) {
    SrcEncode src;
    memset(&src, 0, sizeof(src));
    src.x[0] = x;
    src.dtype = dtype_in;
    src.L = L;
    src.signs = signs;
    SrcBuf buf;
    memset(&buf, 0, sizeof(buf));
    buf.y[0] = y;
    SnkBuf snk;
    memset(&snk, 0, sizeof(snk));
    snk.y[0] = y;
    snk.scale = (float)(1.0 / sqrt((double)dim));
    rc = run_transform(log2_exact(dim), true, 0, 1, src, buf, snk, st, OPTR_K_ENC_FIRST);
  }
  cudaFreeAsync(signs, st);
  return rc;
}

int optr_rht_decode(const float* y, const uint8_t* mask, int64_t dim, int64_t L, uint64_t seed, void* out,
                    int dtype_out, void* stream) {
  if (!is_pow2(dim) || L > dim || L < 0 || !y || (L > 0 && !out)) return OPTR_EINVAL;
  if (dtype_out != OPTR_F32 && dtype_out != OPTR_BF16) return OPTR_EINVAL;
  bind_device(stream);
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long count = (unsigned long long)dim;
  unsigned long long* dcount = nullptr;
  if (mask) {
    CK(cudaMallocAsync((void**)&dcount, sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(dcount, 0, sizeof(unsigned long long), st));
    int64_t blocks = (dim + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    {
      KScope ks(OPTR_K_OTHER, st);
      count_mask_kernel<<<(unsigned)blocks, 256, 0, st>>>(mask, dim, dcount);
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&count, dcount, sizeof(count), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    cudaFreeAsync(dcount, st);
  }
  if (count == 0) return OPTR_EEMPTY;  // hadamard.py:117-118
  uint32_t* signs = nullptr;
  float* tmp = nullptr;
  CK(cudaMallocAsync((void**)&signs, (size_t)((dim + 31) / 32) * 4, st));
  CK(cudaMallocAsync((void**)&tmp, (size_t)dim * 4, st));
  PrepArgs a;
  memset(&a, 0, sizeof(a));
  fill_sign_args(a, signs, dim, seed);
  int rc = launch_prep(a, st);
  if (!rc) {
    SrcMasked src{y, mask};
    SrcBuf buf;
    memset(&buf, 0, sizeof(buf));
    buf.y[0] = tmp;
    SnkDecode snk;
    memset(&snk, 0, sizeof(snk));
    snk.out[0] = out;
    snk.dtype = dtype_out;
    snk.L = L;
    snk.signs = signs;
    snk.count_extra = nullptr;
    snk.count_base[0] = (int64_t)count;
    snk.dim = (double)dim;
    rc = run_transform(log2_exact(dim), false, 0, 1, src, buf, snk, st, OPTR_K_DEC_FIRST);
  }
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(signs, st);
  return rc;
}


}  // extern "C"

namespace {
// Async co-resident calls: two slots, each with its own work stream, so
// consecutive buckets overlap (one bucket's aggregate
// and decode with the next one's encode).
struct LocalAsync {
  bool init = false;
  cudaStream_t ws[2];
  cudaEvent_t fork[2], done[2];
  bool recorded[2] = {false, false};
  std::mutex mu;
};
LocalAsync g_lasync[64];

LocalAsync* local_async() {
  int dev = 0;
  cudaGetDevice(&dev);
  LocalAsync* a = &g_lasync[dev & 63];
  std::lock_guard<std::mutex> lk(g_attr_mu);
  if (!a->init) {
    for (int i = 0; i < 2; ++i) {
      if (cudaStreamCreateWithFlags(&a->ws[i], cudaStreamNonBlocking) != cudaSuccess) return nullptr;
      if (cudaEventCreateWithFlags(&a->fork[i], cudaEventDisableTiming) != cudaSuccess) return nullptr;
      if (cudaEventCreateWithFlags(&a->done[i], cudaEventDisableTiming) != cudaSuccess) return nullptr;
    }
    a->init = true;
  }
  return a;
}

int tar_local_impl(const void* const* x, void* const* out, int n, int64_t L, int dtype_in, int dtype_out,
                   uint64_t job_seed, uint64_t bucket_id, uint64_t generation, int rotation, int ht,
                   const optr_mask_spec* masks, void* workspace, size_t workspace_bytes,
                   uint64_t* received_out, uint8_t* got_out, cudaStream_t st, int set);
}  // namespace

extern "C" {

// -------------------------------------------------- TAR, n workers, one GPU
struct LocalLayout {
  size_t y, a, signs, signs_t, bitmap, counts, bar, tileok, total;
  int64_t dim, smax, astride, pw;
};

static LocalLayout local_layout(int n, int64_t L, int ht, int epp) {
  LocalLayout l;
  l.dim = ht ? next_pow2_i(L) : L;
  Shards sh = make_shards(l.dim, n);
  l.smax = sh.base + (sh.extra ? 1 : 0);
  l.astride = (l.smax + 63) / 64 * 64;  // owner aggregates 256-byte aligned (float4 / TMA)
  l.pw = mask_words(l.dim, n, epp);
  size_t off = 0;
  l.y = off;
  off = align_up(off + (size_t)n * l.dim * 4, 256);
  l.a = off;
  off = align_up(off + (size_t)n * (l.astride > 0 ? l.astride : 1) * 4, 256);
  l.signs = off;
  off = align_up(off + (size_t)((l.dim + 31) / 32 + 2) * 4, 256);
  l.signs_t = off;  // transposed sign bytes for the strided decode pass
  off = align_up(off + (size_t)(ht ? l.dim / 8 + 16 : 16), 256);
  l.bitmap = off;
  off = align_up(off + (size_t)2 * n * n * l.pw * 4, 256);
  l.counts = off;
  off = align_up(off + (size_t)2 * n * 8, 8);
  l.bar = off;  // small-bucket kernel's grid-barrier counter (zeroed with the counts)
  off = align_up(off + 8, 256);
  l.tileok = off;  // per-tile mask summaries of the fast plan: 2 x (dim / 2^13) words
  off = align_up(off + (size_t)2 * ((l.dim >> 13) + 1) * 4, 256);
  l.total = off;
  return l;
}

size_t optr_tar_local_workspace(int n, int64_t L, int ht, int epp) {
  if (n < 2 || n > OPTR_MAX_WORKERS || L < 0 || epp <= 0) return 0;
  return local_layout(n, L, ht, epp).total;
}

int optr_tar_local(const void* const* x, void* const* out, int n, int64_t L, int dtype_in, int dtype_out,
                   uint64_t job_seed, uint64_t bucket_id, uint64_t generation, int rotation, int ht,
                   const optr_mask_spec* masks, void* workspace, size_t workspace_bytes,
                   uint64_t* received_out, uint8_t* got_out, void* stream) {
  NvtxRange nr("optr_tar_local");
  bind_device(stream);
  return tar_local_impl(x, out, n, L, dtype_in, dtype_out, job_seed, bucket_id, generation, rotation, ht, masks,
                        workspace, workspace_bytes, received_out, got_out, (cudaStream_t)stream, 0);
}

int optr_tar_local_async(const void* const* x, void* const* out, int n, int64_t L, int dtype_in, int dtype_out,
                         uint64_t job_seed, uint64_t bucket_id, uint64_t generation, int rotation, int ht,
                         const optr_mask_spec* masks, void* workspace, size_t workspace_bytes,
                         uint64_t* received_out, uint8_t* got_out, int slot, void* stream) {
  NvtxRange nr("optr_tar_local_async");
  if (slot < 0 || slot > 1) return OPTR_EINVAL;
  bind_device(stream);
  LocalAsync* la = local_async();
  if (!la) return OPTR_ECUDA;
  std::lock_guard<std::mutex> lk(la->mu);
  const cudaStream_t ws = la->ws[slot];
  CK(cudaEventRecord(la->fork[slot], (cudaStream_t)stream));
  CK(cudaStreamWaitEvent(ws, la->fork[slot], 0));
  int rc = tar_local_impl(x, out, n, L, dtype_in, dtype_out, job_seed, bucket_id, generation, rotation, ht, masks,
                          workspace, workspace_bytes, received_out, got_out, ws, 1 + slot);
  CK(cudaEventRecord(la->done[slot], ws));
  la->recorded[slot] = true;
  return rc;
}

int optr_local_join(void* stream) {
  bind_device(stream);
  LocalAsync* la = local_async();
  if (!la) return OPTR_ECUDA;
  std::lock_guard<std::mutex> lk(la->mu);
  for (int i = 0; i < 2; ++i)
    if (la->recorded[i]) CK(cudaStreamWaitEvent((cudaStream_t)stream, la->done[i], 0));
  return OPTR_OK;
}

}  // extern "C"

namespace {
// Fast one-GPU plan (RHT on, D = 2^23..2^25, equal power-of-two shards of
// whole contiguous tiles): strided encode pass from x (signs, pad, cast) ->
// contiguous encode pass of every worker fused with the stage-1 mean
// (tma_mean_kernel: the wire vectors never reach memory) -> contiguous decode
// pass with the stage-2 receive from the aggregate -> strided decode pass
// into `out`.  Four launches per bucket; -1 when the shapes do not fit.
struct FastPlan {
  PassGeom contig, strided;
  int nlog;
};

bool local_fast_plan(int64_t L, int64_t dim, int n, int ht, const void* const* x, void* const* out,
                     FastPlan* fp) {
  if (!ht || !tma_enabled() || !is_pow2(dim)) return false;
  PassGeom ps[3];
  const int nlog = log2_exact(dim);
  if (plan_passes(nlog, ps, true) != 2) return false;
  const int Tc = ps[0].ks, Ts = ps[1].ks + ps[1].cb;
  if (ps[0].cb != 0 || (Tc != 13 && Tc != 14) || ps[1].cb != 3 || (Ts != 13 && Ts != 14)) return false;
  const Shards sh = make_shards(dim, n);
  if (sh.extra != 0 || !is_pow2(sh.base) || sh.base < (1LL << Tc)) return false;
  if ((L >> ps[1].lo) < 1) return false;
  for (int w = 0; w < n; ++w)
    if (((uintptr_t)x[w] & 15) || ((uintptr_t)out[w] & 15)) return false;
  fp->contig = ps[0];
  fp->strided = ps[1];
  fp->nlog = nlog;
  return true;
}

template <int T, int NW>
int launch_mean_t(const TmaArgs& a, const MeanArgs& m, cudaStream_t st) {
  // two CTAs per SM (<= 128 registers: the fp64 accumulators take 64) with a
  // two-stage ring: 61.5 us per 2^23 bucket of 4 workers against 71.6 us for
  // one CTA with three stages (140 registers; profiles/r02_quick_mean_ab.txt);
  // three stages at two CTAs per SM measured the same (0.795 vs 0.798 ms)
  constexpr int S = 2;
  const size_t smem = tma_smem_bytes<T, S>();
  auto kern = tma_mean_kernel<T, S, NW>;
  int rc = set_smem_attr(kern, smem);
  if (rc) return rc;
  int dev = 0, nsm = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 1 << (T - 5), smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  // equal tile counts per CTA (no tail of CTAs with one tile more)
  const int64_t cap = (int64_t)nsm * per_sm;
  const int64_t per_cta = (a.ntiles + cap - 1) / cap;
  const int64_t gx = (a.ntiles + per_cta - 1) / per_cta;
  KScope ks(OPTR_K_ENC_MEAN, st, m.n);
  launch_ex(kern, dim3((unsigned)gx), dim3(1 << (T - 5)), smem, st, a, m);
  return launch_check(kern, "tma_mean", T, 0, (int)gx, 1, 1 << (T - 5), smem);
}

// stage-2 receive + contiguous decode of every co-resident worker, shared
// across the receivers with clean tiles (tma_gather_shared_kernel)
template <int T, int NW>
int launch_gather_shared_t(const TmaArgs& a, const GatherSharedArgs& ys, cudaStream_t st) {
  constexpr int S = 2;  // (three stages: the same, 47.8 vs 47.4 us)
  const size_t smem = tma_smem_bytes<T, S>();
  auto kern = tma_gather_shared_kernel<T, S, NW>;
  int rc = set_smem_attr(kern, smem);
  if (rc) return rc;
  int dev = 0, nsm = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 1 << (T - 5), smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const int64_t cap = (int64_t)nsm * per_sm;
  const int64_t per_cta = (a.ntiles + cap - 1) / cap;
  const int64_t gx = (a.ntiles + per_cta - 1) / per_cta;
  KScope ks(OPTR_K_DEC_FIRST, st, a.n);
  launch_ex(kern, dim3((unsigned)gx), dim3(1 << (T - 5)), smem, st, a, ys);
  return launch_check(kern, "tma_gather_shared", T, 0, (int)gx, 1, 1 << (T - 5), smem);
}

template <int T>
int launch_gather_shared(const TmaArgs& a, const GatherSharedArgs& ys, cudaStream_t st) {
  switch (a.n) {
    case 2: return launch_gather_shared_t<T, 2>(a, ys, st);
    case 4: return launch_gather_shared_t<T, 4>(a, ys, st);
    case 8: return launch_gather_shared_t<T, 8>(a, ys, st);
    case 16: return launch_gather_shared_t<T, 16>(a, ys, st);
    default: return OPTR_EINVAL;
  }
}

template <int T>
int launch_mean_n(const TmaArgs& a, const MeanArgs& m, cudaStream_t st) {
  switch (m.n) {
    case 2: return launch_mean_t<T, 2>(a, m, st);
    case 4: return launch_mean_t<T, 4>(a, m, st);
    case 8: return launch_mean_t<T, 8>(a, m, st);
    case 16: return launch_mean_t<T, 16>(a, m, st);
    default: return OPTR_EINVAL;
  }
}

void* g_small_trace = nullptr;  // optr_debug_trace with per_cta < 0: small-kernel phase stamps

bool small_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("OPTR_SMALL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// n co-resident workers, D = 2^13..2^20 (RHT on, n a power of two <= 8):
// the whole call in one cooperative launch (small.cuh)
int tar_local_small(const void* const* x, void* const* out, int n, int64_t L, int dtype_in, int dtype_out,
                    uint64_t seed, int r, const optr_mask_spec* masks, char* ws, const LocalLayout& lay,
                    int epp, uint64_t* received_out, uint8_t* got_out, cudaStream_t st) {
  const int64_t dim = lay.dim;
  unsigned long long* counts = (unsigned long long*)(ws + lay.counts);
  CK(cudaMemsetAsync(counts, 0, lay.bar + 8 - lay.counts, st));  // counts + barrier counter
  SmallLocalArgs a;
  memset(&a, 0, sizeof(a));
  const uint32_t* cb = nullptr;
  int rc = setup_masks(a.pa, masks, dim, n, r, epp, (uint32_t*)(ws + lay.bitmap), counts, 0, n, &cb);
  if (rc) return rc;
  if ((rc = ensure_device_init())) return rc;
  const Pcg sp = sign_pcg(seed);
  a.signs = (uint32_t*)(ws + lay.signs);
  a.sign_state = sp.state;
  a.sign_inc = sp.inc;
  for (int w = 0; w < n; ++w) {
    a.x[w] = x[w];
    a.out[w] = out[w];
    a.Y[w] = (float*)(ws + lay.y) + (size_t)w * dim;
  }
  a.dtype_in = dtype_in;
  a.dtype_out = dtype_out;
  a.L = L;
  a.dim = dim;
  a.bar = (unsigned long long*)(ws + lay.bar);
  a.counts = counts;
  a.got = got_out;
  a.received_out = (unsigned long long*)received_out;
  a.m = MaskView{cb, a.pa.pw, n, epp, make_divider((uint32_t)epp)};
  a.n = n;
  a.r = r;
  a.shard_shift = log2_exact(dim / n);
  a.trace = (unsigned long long*)g_small_trace;
  {
    KScope ks(OPTR_K_SMALL, st, n);
    rc = optr_small_local_launch(log2_exact(dim), a, st);
  }
  return rc;
}

int tar_local_impl(const void* const* x, void* const* out, int n, int64_t L, int dtype_in, int dtype_out,
                   uint64_t job_seed, uint64_t bucket_id, uint64_t generation, int rotation, int ht,
                   const optr_mask_spec* masks, void* workspace, size_t workspace_bytes,
                   uint64_t* received_out, uint8_t* got_out, cudaStream_t st, int set) {
  (void)set;
  int rc = check_common(n, L, dtype_in, dtype_out, masks);
  if (rc) return rc;
  if (!x || !out || !workspace) return OPTR_EINVAL;
  int epp = masks ? masks->epp : 350;
  LocalLayout lay = local_layout(n, L, ht, epp);
  if (workspace_bytes < lay.total) return OPTR_EINVAL;
  if (L == 0) return OPTR_OK;
  char* ws = (char*)workspace;
  const int64_t dim = lay.dim;
  const int r = ((rotation % n) + n) % n;
  float* Y = (float*)(ws + lay.y);
  float* A = (float*)(ws + lay.a);
  uint32_t* signs = (uint32_t*)(ws + lay.signs);
  uint32_t* bitmap = (uint32_t*)(ws + lay.bitmap);
  unsigned long long* counts = (unsigned long long*)(ws + lay.counts);
  const Shards sh = make_shards(dim, n);
  const int nlog = ht ? log2_exact(dim) : 0;
  if (ht && small_enabled() && nlog >= kSmallMinLog && nlog <= kSmallMaxLog && n <= kSmallMaxRanks &&
      (n & (n - 1)) == 0)
    return tar_local_small(x, out, n, L, dtype_in, dtype_out, derive_seed(job_seed, bucket_id, generation), r,
                           masks, ws, lay, epp, received_out, got_out, st);
  FastPlan fp;
  const bool fast = local_fast_plan(L, dim, n, ht, x, out, &fp);

  // 1. signs (+ transposed sign bytes for the strided passes) + masks + counts
  CK(cudaMemsetAsync(counts, 0, (size_t)2 * n * 8, st));
  PrepArgs pa;
  memset(&pa, 0, sizeof(pa));
  if (ht) fill_sign_args(pa, signs, dim, derive_seed(job_seed, bucket_id, generation));
  // general plan: two-pass plans decode contiguous-first and finish with the
  // strided pass, whose signs come from the transposed sign bytes
  PassGeom dps[3];
  const int dnp = ht ? plan_passes(nlog, dps, true) : 0;
  const bool dec_cf = ht && decode_contig_first(nlog, false);
  uint8_t* const signs_t =
      (ht && (fast || (dec_cf && dnp == 2 && dps[1].cb == 3))) ? (uint8_t*)(ws + lay.signs_t) : nullptr;
  if (signs_t) {
    pa.signs_t = signs_t;
    pa.t_lo = dps[1].lo;
    pa.t_ks = dps[1].ks;
  }
  const uint32_t* cbits = nullptr;
  if ((rc = setup_masks(pa, masks, dim, n, r, epp, bitmap, counts, 0, n, &cbits))) return rc;
  uint32_t* const tile_ok = fast ? (uint32_t*)(ws + lay.tileok) : nullptr;
  if (tile_ok) {  // per-tile summaries of the masks, cleared by prep where a packet is lost
    pa.tile_ok = tile_ok;
    pa.tile_shift = fp.contig.ks;
    pa.ntiles = dim >> fp.contig.ks;
    CK(cudaMemsetAsync(tile_ok, 0xFF, (size_t)2 * pa.ntiles * 4, st));
  }
  if ((rc = launch_prep(pa, st))) return rc;
  MaskView mv{cbits, pa.pw, n, epp, make_divider((uint32_t)epp)};

  // stage-2 receive source (collectives.py:140-150)
  SrcGather ga;
  memset(&ga, 0, sizeof(ga));
  ga.sh = sh;
  ga.n = n;
  ga.r = r;
  ga.m = mv;
  ga.got = got_out;
  ga.dim = dim;
  ga.pow2_shift = (sh.extra == 0 && is_pow2(sh.base)) ? log2_exact(sh.base) : -1;
  SnkDecode dec;
  memset(&dec, 0, sizeof(dec));
  for (int w = 0; w < n; ++w) {
    dec.out[w] = out[w];
    dec.count_base[w] = sh.len(owned_shard(w, r, n));
  }
  dec.dtype = dtype_out;
  dec.L = L;
  dec.signs = signs;
  dec.signs_t = signs_t;
  dec.count_extra = counts + n;  // stage-2 row
  dec.count_stride = 1;
  dec.dim = (double)dim;

  if (fast) {
    // 2. strided encode pass x -> Y (signs, pad, bf16 upcast fused)
    SrcEncode src;
    memset(&src, 0, sizeof(src));
    src.dtype = dtype_in;
    src.L = L;
    src.signs = signs;
    src.signs_t = signs_t;
    SnkBuf mid;
    memset(&mid, 0, sizeof(mid));
    mid.scale = 1.f;
    for (int w = 0; w < n; ++w) {
      src.x[w] = x[w];
      mid.y[w] = Y + (size_t)w * dim;
    }
    if ((rc = launch_pass(OPTR_K_ENC_FIRST, fp.strided, nlog, 0, n, src, mid, st))) return rc;
    // 3. contiguous encode pass of every worker + stage-1 mean -> A (natural order)
    TmaArgs ta;
    memset(&ta, 0, sizeof(ta));
    ta.ntiles = fp.contig.ntiles;
    for (int w = 0; w < n; ++w) ta.xw[w] = Y + (size_t)w * dim;
    MeanArgs ma;
    memset(&ma, 0, sizeof(ma));
    ma.agg = A;
    ma.scale = (float)(1.0 / sqrt((double)dim));
    ma.n = n;
    ma.r = r;
    ma.shard_shift = log2_exact(sh.base);
    ma.m = mv;
    ma.tile_ok1 = tile_ok;
    rc = fp.contig.ks == 13 ? launch_mean_n<13>(ta, ma, st) : launch_mean_n<14>(ta, ma, st);
    if (rc) return rc;
    // 4. contiguous decode pass with the stage-2 receive, A -> Y
    for (int o = 0; o < n; ++o) ga.A[o] = A + sh.off(owned_shard(o, r, n));
    ga.tile_ok2 = tile_ok + (dim >> fp.contig.ks);
    SrcBuf buf;
    memset(&buf, 0, sizeof(buf));
    for (int w = 0; w < n; ++w) buf.y[w] = mid.y[w];
    // one transform per tile for the receivers it reached intact (without
    // received flags to write): 52.8 -> 47.5 us per 4 x 2^23 launch, resnet50
    // 0.823 -> 0.802 ms per step, headline 0.960 -> 0.923 ms
    if (!got_out) {
      TmaArgs ta2;
      memset(&ta2, 0, sizeof(ta2));
      ta2.ntiles = fp.contig.ntiles;
      for (int o = 0; o < n; ++o) ta2.A[o] = ga.A[o];
      ta2.n = n;
      ta2.r = r;
      ta2.shard_shift = log2_exact(sh.base);
      ta2.m = mv;
      ta2.dim = dim;
      ta2.tile_ok2 = ga.tile_ok2;
      GatherSharedArgs ys;
      memset(&ys, 0, sizeof(ys));
      for (int w = 0; w < n; ++w) ys.y[w] = mid.y[w];
      rc = fp.contig.ks == 13 ? launch_gather_shared<13>(ta2, ys, st) : launch_gather_shared<14>(ta2, ys, st);
      if (rc) return rc;
    } else if ((rc = launch_pass(OPTR_K_DEC_FIRST, fp.contig, nlog, 0, n, ga, mid, st))) {
      return rc;
    }
    // 5. strided decode pass Y -> out (count scale, signs, truncate, cast)
    if ((rc = launch_pass(OPTR_K_DEC_LAST, fp.strided, nlog, 0, n, buf, dec, st))) return rc;
    if (received_out) CK(cudaMemcpyAsync(received_out, counts, (size_t)2 * n * 8, cudaMemcpyDeviceToDevice, st));
    return OPTR_OK;
  }

  // ---- general plan (RHT off, other sizes and shard splits)
  // 2. wire vectors
  const float* Yw[kMaxW];
  if (ht) {
    SrcEncode src;
    memset(&src, 0, sizeof(src));
    src.dtype = dtype_in;
    src.L = L;
    src.signs = signs;
    SrcBuf buf;
    memset(&buf, 0, sizeof(buf));
    SnkBuf snk;
    memset(&snk, 0, sizeof(snk));
    for (int w = 0; w < n; ++w) {
      src.x[w] = x[w];
      buf.y[w] = snk.y[w] = Y + (size_t)w * dim;
      Yw[w] = Y + (size_t)w * dim;
    }
    snk.scale = (float)(1.0 / sqrt((double)dim));
    if ((rc = run_transform(nlog, true, 0, n, src, buf, snk, st, OPTR_K_ENC_FIRST))) return rc;
  } else {
    for (int w = 0; w < n; ++w) {
      if (dtype_in == OPTR_F32) {
        Yw[w] = (const float*)x[w];
      } else {
        float* yw = Y + (size_t)w * dim;
        KScope ks(OPTR_K_OTHER, st);
        cast_copy_kernel<<<1184, 256, 0, st>>>(x[w], dtype_in, yw, dim);
        CK(cudaGetLastError());
        Yw[w] = yw;
      }
    }
  }

  // 3. stage 1: owner means
  AggArgs ag;
  memset(&ag, 0, sizeof(ag));
  for (int w = 0; w < n; ++w) {
    ag.Y[w] = Yw[w];
    ag.A[w] = A + (size_t)w * lay.astride;
  }
  ag.sh = sh;
  ag.n = n;
  ag.r = r;
  ag.m = mv;
  ag.owner_base = 0;
  if ((rc = launch_aggregate(ag, n, lay.smax, st))) return rc;

  // 4. stage 2 receive (+ decode)
  for (int w = 0; w < n; ++w) ga.A[w] = ag.A[w];
  if (ht) {
    SrcBuf buf;
    memset(&buf, 0, sizeof(buf));
    for (int w = 0; w < n; ++w) buf.y[w] = Y + (size_t)w * dim;  // encoded vectors are dead after stage 1
    if ((rc = run_transform(nlog, dec_cf, 0, n, ga, buf, dec, st, OPTR_K_DEC_FIRST))) return rc;
  } else {
    AsmArgs as;
    memset(&as, 0, sizeof(as));
    as.gather = ga;
    for (int w = 0; w < n; ++w) as.out[w] = out[w];
    as.dtype = dtype_out;
    as.L = L;
    int64_t blocks = (L + 255) / 256;
    if (blocks > 4736) blocks = 4736;
    KScope ks(OPTR_K_ASSEMBLE, st, n);
    assemble_kernel<<<dim3((unsigned)blocks, n), 256, 0, st>>>(as);
    CK(cudaGetLastError());
  }
  if (received_out) CK(cudaMemcpyAsync(received_out, counts, (size_t)2 * n * 8, cudaMemcpyDeviceToDevice, st));
  return OPTR_OK;
}
}  // namespace

extern "C" {

// ------------------------------------------------ TAR, one worker per GPU
struct optr_comm_s {
  int rank, n, epp, device;
  int64_t max_dim;
  // two parities of [Y | A] so consecutive calls can overlap; three flag
  // sets (one per parity, one for the public barrier)
  size_t off_flags[3], off_y[2], off_a[2], off_g[2], off_ef[2], off_gf[2], sym_bytes;
  char* sym;
  char* peer[OPTR_MAX_WORKERS];
  bool opened[OPTR_MAX_WORKERS];
  char* local;  // two parities of signs | bitmap | counts
  size_t off_signs, off_signs_t, off_bitmap, off_counts, off_ctr, local_bytes;  // within one parity
  unsigned int* fused_ctr[2];  // chain / fused kernel counters of each parity (self-resetting)
  unsigned int fepoch[2];      // fused-kernel tile-flag epochs of each parity
  cudaEvent_t fused_done[2];   // fused kernels of consecutive calls never overlap
  bool fused_recorded[2];
  cudaEvent_t enc_done[2];     // fused path: the next call's prep starts after this strided encode
  bool enc_recorded[2];
  unsigned long long epoch[3];
  cudaStream_t ws[2];       // per-parity work streams
  cudaEvent_t fork[2];
  // prep (signs + masks + counts) runs on its own stream into the buffers of
  // call parity p as soon as call c-2 (the last user of p) is done, so it
  // overlaps the previous call's kernels
  cudaStream_t pstream;
  cudaEvent_t prep_ready[2], done[2];
  bool done_recorded[2];
  uint64_t calls;
  int fused_grid;  // CTAs of the persistent fused kernel (0 = SMs x occupancy)
  // small-bucket path (tar_small_kernel): wire / receive vector Y | flags
  // [2][kMaxW] in the symmetric block, signs | bitmap | counts | barrier
  // counter in `slocal`; 0 bytes when max_len is below the small range
  int64_t small_dim;  // largest small-path dim (0 = off)
  size_t off_sy, off_sf;
  char* slocal;
  size_t s_signs, s_bitmap, s_counts, s_bar;
  unsigned long long s_epoch, s_bar_base;
};

size_t optr_comm_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

int optr_comm_create(optr_comm* out, int device, int rank, int n, int64_t max_len, int epp) {
  if (!out || n < 2 || n > OPTR_MAX_WORKERS || rank < 0 || rank >= n || max_len < 1 || epp <= 0 ||
      device < 0)
    return OPTR_EINVAL;
  CK(cudaSetDevice(device));
  optr_comm c = (optr_comm)calloc(1, sizeof(optr_comm_s));
  if (!c) return OPTR_ENOMEM;
  c->rank = rank;
  c->n = n;
  c->epp = epp;
  c->device = device;
  c->max_dim = next_pow2_i(max_len);
  Shards sh = make_shards(c->max_dim, n);
  int64_t smax = sh.base + (sh.extra ? 1 : 0);
  size_t off = 0;
  for (int f = 0; f < 3; ++f) {
    c->off_flags[f] = off;
    off = align_up(off + OPTR_MAX_WORKERS * 8, 256);
  }
  for (int p = 0; p < 2; ++p) {
    c->off_y[p] = off;
    off = align_up(off + (size_t)c->max_dim * 4, 1024);
    c->off_a[p] = off;
    off = align_up(off + (size_t)smax * 4, 1024);
    c->off_g[p] = off;  // stage-2 receive vector, written by every owner's push
    off = align_up(off + (size_t)c->max_dim * 4, 1024);
    c->off_ef[p] = off;  // fused kernel: my encode flags [tiles], my published-unit flags [tiles][4]
    off = align_up(off + (size_t)(c->max_dim >> 13 > 0 ? c->max_dim >> 13 : 1) * 4, 256);
    c->off_gf[p] = off;
    off = align_up(off + (size_t)4 * (c->max_dim >> 13 > 0 ? c->max_dim >> 13 : 1) * 4, 1024);
  }
  c->small_dim = c->max_dim < (1LL << kSmallMinLog) ? 0
                 : (c->max_dim < (1LL << kSmallMaxLog) ? c->max_dim : (1LL << kSmallMaxLog));
  if (c->small_dim) {
    c->off_sy = off;
    off = align_up(off + (size_t)c->small_dim * 4, 1024);
    c->off_sf = off;
    off = align_up(off + (size_t)2 * kMaxW * 8, 1024);
  }
  c->sym_bytes = off;
  int64_t pw = mask_words(c->max_dim, n, 1);  // epp >= 1 bound
  off = 0;
  c->off_signs = off;
  off = align_up(off + (size_t)((c->max_dim + 31) / 32 + 2) * 4, 256);
  c->off_signs_t = off;  // transposed sign bytes for the fused path's strided passes
  off = align_up(off + (size_t)(c->max_dim / 8 + 16), 256);
  c->off_bitmap = off;
  off = align_up(off + (size_t)2 * n * n * pw * 4, 256);
  c->off_counts = off;
  off = align_up(off + (size_t)2 * n * 8, 256);
  c->off_ctr = off;
  off = align_up(off + 4 * sizeof(unsigned int), 256);
  c->local_bytes = off;
  size_t soff = 0;
  if (c->small_dim) {
    const int64_t spw = mask_words(c->small_dim, n, 1);
    c->s_signs = soff;
    soff = align_up(soff + (size_t)(c->small_dim / 32) * 4, 256);
    c->s_bitmap = soff;
    soff = align_up(soff + (size_t)2 * n * n * spw * 4, 256);
    c->s_counts = soff;  // two call parities of [2][n]
    soff = align_up(soff + (size_t)2 * 2 * n * 8, 256);
    c->s_bar = soff;
    soff = align_up(soff + 8, 256);
  }
  if (cudaMalloc((void**)&c->sym, c->sym_bytes) != cudaSuccess ||
      cudaMalloc((void**)&c->local, 2 * c->local_bytes) != cudaSuccess ||
      (soff && cudaMalloc((void**)&c->slocal, soff) != cudaSuccess)) {
    cudaFree(c->sym);
    cudaFree(c->local);
    free(c);
    return OPTR_ENOMEM;
  }
  CK(cudaMemset(c->sym, 0, c->sym_bytes));
  CK(cudaMemset(c->local, 0, 2 * c->local_bytes));
  if (soff) CK(cudaMemset(c->slocal, 0, soff));
  for (int p = 0; p < 2; ++p) c->fused_ctr[p] = (unsigned int*)(c->local + p * c->local_bytes + c->off_ctr);
  // prep (ALU-heavy, off the critical path) at the lowest priority, the call
  // streams at the highest: the block scheduler gives prep leftover SMs
  int prio_lo = 0, prio_hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  CK(cudaStreamCreateWithPriority(&c->pstream, cudaStreamNonBlocking, prio_lo));
  for (int p = 0; p < 2; ++p) {
    CK(cudaEventCreateWithFlags(&c->prep_ready[p], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->done[p], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->fork[p], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->fused_done[p], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->enc_done[p], cudaEventDisableTiming));
    CK(cudaStreamCreateWithPriority(&c->ws[p], cudaStreamNonBlocking, prio_hi));
  }
  CK(cudaDeviceSynchronize());
  c->peer[rank] = c->sym;
  *out = c;
  return OPTR_OK;
}

int optr_comm_get_handle(optr_comm c, void* handle_out) {
  if (!c || !handle_out) return OPTR_EINVAL;
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, c->sym));
  memcpy(handle_out, &h, sizeof(h));
  return OPTR_OK;
}

int optr_comm_open(optr_comm c, const void* all_handles) {
  if (!c || !all_handles) return OPTR_EINVAL;
  CK(cudaSetDevice(c->device));
  const char* hb = (const char*)all_handles;
  for (int i = 0; i < c->n; ++i) {
    if (i == c->rank || c->opened[i]) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, hb + (size_t)i * sizeof(h), sizeof(h));
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->peer[i] = (char*)p;
    c->opened[i] = true;
  }
  return OPTR_OK;
}

int optr_comm_destroy(optr_comm c) {
  if (!c) return OPTR_EINVAL;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int i = 0; i < c->n; ++i)
    if (c->opened[i]) cudaIpcCloseMemHandle(c->peer[i]);
  cudaFree(c->sym);
  cudaFree(c->local);
  if (c->slocal) cudaFree(c->slocal);
  cudaStreamDestroy(c->pstream);
  for (int p = 0; p < 2; ++p) {
    cudaEventDestroy(c->prep_ready[p]);
    cudaEventDestroy(c->done[p]);
    cudaEventDestroy(c->fork[p]);
    cudaEventDestroy(c->fused_done[p]);
    cudaEventDestroy(c->enc_done[p]);
    cudaStreamDestroy(c->ws[p]);
  }
  free(c);
  return OPTR_OK;
}

struct FlagPtrs {
  unsigned long long* f[OPTR_MAX_WORKERS];
};

__global__ void barrier_kernel2(FlagPtrs peers, unsigned long long* mine, int rank, int n,
                                unsigned long long epoch) {
  int i = threadIdx.x;
  if (i >= n || i == rank) return;
  __threadfence_system();
  unsigned long long* dst = peers.f[i] + rank;
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst), "l"(epoch) : "memory");
  unsigned long long v;
  do {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine + i) : "memory");
  } while (v < epoch);
}

static int comm_barrier(optr_comm c, int set, cudaStream_t st) {
  FlagPtrs fp;
  memset(&fp, 0, sizeof(fp));
  for (int i = 0; i < c->n; ++i) {
    if (!c->peer[i]) return OPTR_EINVAL;
    fp.f[i] = (unsigned long long*)(c->peer[i] + c->off_flags[set]);
  }
  c->epoch[set] += 1;
  KScope ks(OPTR_K_BARRIER, st);
  barrier_kernel2<<<1, 32, 0, st>>>(fp, (unsigned long long*)(c->sym + c->off_flags[set]), c->rank, c->n,
                                     c->epoch[set]);
  CK(cudaGetLastError());
  return OPTR_OK;
}

int optr_comm_set_fused_grid(optr_comm c, int ctas) {
  if (!c || ctas < 0) return OPTR_EINVAL;
  c->fused_grid = ctas;
  return OPTR_OK;
}

int optr_comm_barrier(optr_comm c, void* stream) {
  if (!c) return OPTR_EINVAL;
  CK(cudaSetDevice(c->device));
  return comm_barrier(c, 2, (cudaStream_t)stream);
}

int optr_comm_join(optr_comm c, void* stream) {
  if (!c) return OPTR_EINVAL;
  CK(cudaSetDevice(c->device));
  for (int p = 0; p < 2; ++p)
    if (c->done_recorded[p]) CK(cudaStreamWaitEvent((cudaStream_t)stream, c->done[p], 0));
  return OPTR_OK;
}

static int tar_enqueue(optr_comm c, const void* x, void* out, int64_t L, int dtype_in, int dtype_out,
                       uint64_t job_seed, uint64_t bucket_id, uint64_t generation, int rotation, int ht,
                       const optr_mask_spec* masks, uint64_t* received_out, void* stream, bool async,
                       uint64_t deadline_ns = 0, optr_tar_stats* stats = nullptr, uint32_t* cut_units = nullptr);

int optr_tar(optr_comm c, const void* x, void* out, int64_t L, int dtype_in, int dtype_out, uint64_t job_seed,
             uint64_t bucket_id, uint64_t generation, int rotation, int ht, const optr_mask_spec* masks,
             uint64_t* received_out, void* stream) {
  return tar_enqueue(c, x, out, L, dtype_in, dtype_out, job_seed, bucket_id, generation, rotation, ht, masks,
                     received_out, stream, false);
}

int optr_tar_async(optr_comm c, const void* x, void* out, int64_t L, int dtype_in, int dtype_out,
                   uint64_t job_seed, uint64_t bucket_id, uint64_t generation, int rotation, int ht,
                   const optr_mask_spec* masks, uint64_t* received_out, void* stream) {
  return tar_enqueue(c, x, out, L, dtype_in, dtype_out, job_seed, bucket_id, generation, rotation, ht, masks,
                     received_out, stream, true);
}

int optr_tar_bounded(optr_comm c, const void* x, void* out, int64_t L, int dtype_in, int dtype_out,
                     uint64_t job_seed, uint64_t bucket_id, uint64_t generation, int rotation, int ht,
                     const optr_mask_spec* masks, uint64_t stage1_deadline_ns, optr_tar_stats* stats,
                     uint32_t* cut_units, int async, void* stream) {
  return tar_enqueue(c, x, out, L, dtype_in, dtype_out, job_seed, bucket_id, generation, rotation, ht, masks,
                     nullptr, stream, async != 0, stage1_deadline_ns, stats, cut_units);
}

}  // extern "C"

namespace {
void* g_fused_trace = nullptr;  // optr_debug_trace
int g_fused_trace_cap = 0;
// OPTR_FUSED=0 keeps the barrier-separated encode / aggregate / decode path.
// Fused-kernel watchdog: a peer that never arrives traps the kernel after
// OPTR_WATCHDOG_S seconds (default 1800 s, NCCL's default timeout).
uint64_t watchdog_ns() {
  static const uint64_t wd = [] {
    const char* w = getenv("OPTR_WATCHDOG_S");
    const double sec = (w && atof(w) > 0) ? atof(w) : 1800.0;
    return (uint64_t)(sec * 1e9);
  }();
  return wd;
}

bool fused_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("OPTR_FUSED");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// optr_tar_stats bookkeeping (stats words: ST_* in tma.cuh)
__global__ void stats_init_kernel(unsigned long long* s) {
  for (int i = 0; i < 7; ++i) s[i] = i == ST_OPEN ? ~0ULL : 0ULL;
}
__global__ void stats_stamp_kernel(unsigned long long* s, int field) {
  const unsigned long long t = (unsigned long long)globaltimer_ns();
  if (field == ST_OPEN) atomicMin(s + field, t);
  else atomicMax(s + field, t);
}
__global__ void stats_finish_kernel(unsigned long long* s, const unsigned long long* counts, int me, int n) {
  s[ST_RECV0] = counts[me] - s[ST_CUT0];
  s[ST_RECV1] = counts[n + me] - s[ST_CUT1];
}
int stats_open(optr_tar_stats* s, cudaStream_t st) {
  stats_init_kernel<<<1, 1, 0, st>>>((unsigned long long*)s);
  CK(cudaGetLastError());
  return OPTR_OK;
}
int stats_stamp(optr_tar_stats* s, int field, cudaStream_t st) {
  stats_stamp_kernel<<<1, 1, 0, st>>>((unsigned long long*)s, field);
  CK(cudaGetLastError());
  return OPTR_OK;
}

template <int T, int NW, int S, int NG>
int launch_fused_t(const TmaArgs& ae, const TmaArgs& ad, const SnkBuf& se, const SnkBuf& sd, const FusedArgs& f,
                   cudaStream_t st) {
  const size_t smem = tma_fused_smem_bytes<T, S, NG, NW>();
  auto kern = tma_fused_kernel<T, S, NW, NG>;
  int rc = set_smem_attr(kern, smem);
  if (rc) return rc;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  int per_sm = 0;
  const int threads = NG * (1 << (T - 5)) + kAggThreads;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  int grid = nsm * per_sm;
  // a communicator's cap (optr_comm_set_fused_grid: leave SMs to the
  // backward pass in DDP), else OPTR_FUSED_GRID
  if (f.grid_cap > 0 && f.grid_cap < grid) {
    grid = f.grid_cap;
  } else {
    const char* e = getenv("OPTR_FUSED_GRID");
    if (e && atoi(e) > 0 && atoi(e) < grid) grid = atoi(e);
  }
  KScope ks(OPTR_K_FUSED, st);
  launch_ex(kern, dim3((unsigned)grid), dim3(threads), smem, st, ae, ad, se, sd, f);
  return launch_check(kern, "tma_fused", T, 0, grid, 1, threads, smem);
}

int launch_small(int K, const SmallArgs& a, int grid, cudaStream_t st) {
  KScope ks(OPTR_K_SMALL, st);
  return optr_small_launch(K, a, grid, st);
}

// CTAs of the small kernel: one per SM (stage 1's NVLink loads, the signs
// and the masks spread over the whole grid; the tile passes use D/2^13)
int small_grid(int K) {
  static int cap = 0;
  if (!cap) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cap = nsm > 0 ? nsm : 148;
    const char* e = getenv("OPTR_SMALL_GRID");
    if (e && atoi(e) > 0 && atoi(e) < cap) cap = atoi(e);
  }
  (void)K;
  return cap;
}

int launch_fused(int T, const TmaArgs& ae, const TmaArgs& ad, const SnkBuf& se, const SnkBuf& sd,
                 const FusedArgs& f, cudaStream_t st) {
  // (a 3-stage E/D ring for T = 13 measured slower: 0.504 vs 0.490 ms/step)
  // (two E/D warp groups per CTA for T = 13 made the kernel 2% faster but the
  // step slower, 0.507 vs 0.494 ms: the larger CTA crowds out the neighbour
  // buckets' strided passes; the kernel keeps the NG parameter)
  switch (T * 100 + f.n) {
    case 1302: return launch_fused_t<13, 2, 2, 1>(ae, ad, se, sd, f, st);
    case 1304: return launch_fused_t<13, 4, 2, 1>(ae, ad, se, sd, f, st);
    case 1308: return launch_fused_t<13, 8, 2, 1>(ae, ad, se, sd, f, st);
    case 1402: return launch_fused_t<14, 2, 2, 1>(ae, ad, se, sd, f, st);
    case 1404: return launch_fused_t<14, 4, 2, 1>(ae, ad, se, sd, f, st);
    case 1408: return launch_fused_t<14, 8, 2, 1>(ae, ad, se, sd, f, st);
    default: return -1;
  }
}
}  // namespace

extern "C" {

static int tar_enqueue(optr_comm c, const void* x, void* out, int64_t L, int dtype_in, int dtype_out,
                       uint64_t job_seed, uint64_t bucket_id, uint64_t generation, int rotation, int ht,
                       const optr_mask_spec* masks, uint64_t* received_out, void* stream, bool async,
                       uint64_t deadline_ns, optr_tar_stats* stats, uint32_t* cut_units) {
  NvtxRange nr("optr_tar");
  if (!c) return OPTR_EINVAL;
  int n = c->n;
  int rc = check_common(n, L, dtype_in, dtype_out, masks);
  if (rc) return rc;
  int epp = masks ? masks->epp : 350;
  int64_t dim = ht ? next_pow2_i(L) : L;
  if (dim > c->max_dim) return OPTR_EINVAL;
  if (L == 0) {  // nothing to exchange: zero received entries
    if (received_out) {
      CK(cudaSetDevice(c->device));
      CK(cudaMemsetAsync(received_out, 0, 2 * sizeof(uint64_t), (cudaStream_t)stream));
    }
    return OPTR_OK;
  }
  if (L > 0 && (!x || !out)) return OPTR_EINVAL;
  for (int i = 0; i < n; ++i)
    if (!c->peer[i]) return OPTR_EINVAL;  // optr_comm_open not called
  CK(cudaSetDevice(c->device));
  const cudaStream_t caller = (cudaStream_t)stream;
  const int me = c->rank;
  const int r = ((rotation % n) + n) % n;
  const int par = (int)(c->calls++ & 1);
  // ---- small buckets (2^13..2^20 entries, power-of-two n <= 8): the whole
  // call is one cooperative kernel (small.cuh).  Serialised after the
  // previous call, on the caller's stream (no stream hop); the next call's
  // fused kernel waits for it.
  const Shards sh = make_shards(dim, n);
  const int klog = ht ? log2_exact(dim) : 0;
  if (ht && small_enabled() && c->small_dim && dim <= c->small_dim && klog >= kSmallMinLog &&
      klog <= kSmallMaxLog && n <= kSmallMaxRanks && (n & (n - 1)) == 0 && deadline_ns == 0 && !stats &&
      !cut_units) {
    const cudaStream_t st = caller;
    if (c->done_recorded[par ^ 1]) CK(cudaStreamWaitEvent(st, c->done[par ^ 1], 0));
    char* const sl = c->slocal;
    SmallArgs a;
    memset(&a, 0, sizeof(a));
    unsigned long long* const scounts = (unsigned long long*)(sl + c->s_counts);
    uint32_t* const sbitmap = (uint32_t*)(sl + c->s_bitmap);
    const uint32_t* cb = nullptr;
    if ((rc = setup_masks(a.pa, masks, dim, n, r, epp, sbitmap, scounts, me, me + 1, &cb))) return rc;
    if ((rc = ensure_device_init())) return rc;
    const Pcg sp = sign_pcg(derive_seed(job_seed, bucket_id, generation));
    a.signs = (uint32_t*)(sl + c->s_signs);
    a.sign_state = sp.state;
    a.sign_inc = sp.inc;
    a.x = x;
    a.out = out;
    a.dtype_in = dtype_in;
    a.dtype_out = dtype_out;
    a.L = L;
    a.dim = dim;
    for (int i = 0; i < n; ++i) {
      a.Y[i] = (float*)(c->peer[i] + c->off_sy);
      a.flags[i] = (unsigned long long*)(c->peer[i] + c->off_sf);
    }
    const int grid = small_grid(klog);
    a.bar = (unsigned long long*)(sl + c->s_bar);
    a.bar_base = c->s_bar_base;
    a.epoch = ++c->s_epoch;
    a.counts = scounts + (c->s_epoch & 1) * 2 * n;  // zeroed by the previous call (or at create)
    a.counts_next = scounts + ((c->s_epoch + 1) & 1) * 2 * n;
    a.received_out = (unsigned long long*)received_out;
    a.m = MaskView{cb, a.pa.pw, n, epp, make_divider((uint32_t)epp)};
    a.n = n;
    a.me = me;
    a.r = r;
    a.shard_shift = log2_exact(sh.base);
    a.watchdog_ns = watchdog_ns();
    a.trace = (unsigned long long*)g_small_trace;
    if ((rc = launch_small(klog, a, grid, st))) return rc;
    c->s_bar_base += (unsigned long long)kSmallBarriers * grid;
    CK(cudaEventRecord(c->done[par], st));
    c->done_recorded[par] = true;
    CK(cudaEventRecord(c->fused_done[par], st));  // the next fused kernel starts after it
    c->fused_recorded[par] = true;
    return OPTR_OK;
  }

  // this call's kernels run on the parity's work stream, after the caller's
  // prior work (inputs ready)
  const cudaStream_t st = c->ws[par];
  CK(cudaEventRecord(c->fork[par], caller));
  CK(cudaStreamWaitEvent(st, c->fork[par], 0));
  char* const loc = c->local + (size_t)par * c->local_bytes;
  uint32_t* signs = (uint32_t*)(loc + c->off_signs);
  uint32_t* bitmap = (uint32_t*)(loc + c->off_bitmap);
  unsigned long long* counts = (unsigned long long*)(loc + c->off_counts);
  float* Yp[kMaxW];
  float* Ap[kMaxW];
  float* Gp[kMaxW];
  for (int i = 0; i < n; ++i) {
    Yp[i] = (float*)(c->peer[i] + c->off_y[par]);
    Ap[i] = (float*)(c->peer[i] + c->off_a[par]);
    Gp[i] = (float*)(c->peer[i] + c->off_g[par]);
  }
  // ---- fused path: strided encode pass, then ONE persistent kernel for the
  // contiguous encode pass + stage 1 + stage 2 + contiguous decode pass with
  // per-tile flags over NVLink (no barriers), then the strided decode pass.
  // Decided before prep, which also lays out the signs for it.
  PassGeom fps[3];
  const int nlog = ht ? log2_exact(dim) : 0;
  const int np = ht ? plan_passes(nlog, fps, true) : 0;
  const int Tc = np == 2 ? fps[0].ks : 0;
  const bool fused = ht && fused_enabled() && tma_enabled() && np == 2 && fps[0].cb == 0 &&
                     (Tc == 13 || Tc == 14) && fps[1].cb == 3 && (fps[1].ks + 3 == 13 || fps[1].ks + 3 == 14) &&
                     (n == 2 || n == 4 || n == 8) && sh.extra == 0 && (sh.base >> Tc) >= 1 &&
                     ((sh.base >> Tc) << Tc) == sh.base && (L >> fps[1].lo) >= 1;
  // (every input of this decision is the same on all ranks: a rank taking the
  // other path would leave its peers waiting; the strided passes fall back
  // per rank on their own, e.g. for unaligned x / out)
  const cudaStream_t ps = c->pstream;
  if (c->done_recorded[par]) CK(cudaStreamWaitEvent(ps, c->done[par], 0));
  // the host runs ahead: without this, this call's prep (ALU-heavy) would run
  // beside the previous call's HBM-bound strided encode instead of beside its
  // NVLink-bound fused kernel
  if (fused && c->enc_recorded[par ^ 1]) CK(cudaStreamWaitEvent(ps, c->enc_done[par ^ 1], 0));

  CK(cudaMemsetAsync(counts, 0, (size_t)2 * n * 8, ps));
  PrepArgs pa;
  memset(&pa, 0, sizeof(pa));
  if (ht) fill_sign_args(pa, signs, dim, derive_seed(job_seed, bucket_id, generation));
  uint8_t* const signs_t = fused ? (uint8_t*)(loc + c->off_signs_t) : nullptr;
  if (fused) {
    pa.signs_t = signs_t;
    pa.t_lo = fps[1].lo;
    pa.t_ks = fps[1].ks;
  }
  const uint32_t* cbits = nullptr;
  if ((rc = setup_masks(pa, masks, dim, n, r, epp, bitmap, counts, me, me + 1, &cbits))) return rc;
  // background prep: a few small CTAs per SM, beside the previous call's
  // fused kernel (a full-width prep delayed the strided passes; on the call
  // stream at full width it costs more than its overlap with the strided
  // decode pass does; two PCG chains per thread or rank-sharded signs stored
  // into every rank's copy were slower too, profiles/r02_prep_ab.txt)
  if ((rc = launch_prep(pa, ps, 2))) return rc;
  CK(cudaEventRecord(c->prep_ready[par], ps));
  CK(cudaStreamWaitEvent(st, c->prep_ready[par], 0));
  MaskView mv{cbits, pa.pw, n, epp, make_divider((uint32_t)epp)};

  if (fused) {
    // Fused kernels of consecutive calls never overlap.  Letting the next one
    // fill the previous one's tail deadlocked (watchdog, 2 GPUs): a rank's
    // next fused kernel spins on SMs while a peer's next call still needs SM
    // space for its prep / strided encode, held by that peer's previous
    // fused kernel waiting on this rank -- a resource cycle outside the
    // ticket order.  Serialised, every rank's fused(c) finishes before its
    // fused(c+1) holds an SM.
    if (c->fused_recorded[par ^ 1]) CK(cudaStreamWaitEvent(st, c->fused_done[par ^ 1], 0));
    {  // strided encode pass: x -> Y (signs, pad, upcast fused)
      SrcEncode src;
      memset(&src, 0, sizeof(src));
      src.x[me] = x;
      src.dtype = dtype_in;
      src.L = L;
      src.signs = signs;
      src.signs_t = signs_t;
      SnkBuf snk;
      memset(&snk, 0, sizeof(snk));
      snk.y[me] = Yp[me];
      snk.scale = 1.f;
      if ((rc = launch_pass(OPTR_K_ENC_FIRST, fps[1], nlog, me, 1, src, snk, st))) return rc;
      CK(cudaEventRecord(c->enc_done[par], st));
      c->enc_recorded[par] = true;
    }
    TmaArgs ae, ad;
    memset(&ae, 0, sizeof(ae));
    memset(&ad, 0, sizeof(ad));
    ae.ntiles = fps[0].ntiles;
    ae.xw[me] = Yp[me];
    ad.ntiles = fps[0].ntiles;
    for (int o = 0; o < n; ++o) ad.A[o] = Ap[o];  // stage 2: pull from the owners
    ad.n = n;
    ad.r = r;
    ad.shard_shift = log2_exact(sh.base);
    ad.m = mv;
    ad.dim = dim;
    SnkBuf se, sd;
    memset(&se, 0, sizeof(se));
    memset(&sd, 0, sizeof(sd));
    se.y[me] = Yp[me];
    se.scale = (float)(1.0 / sqrt((double)dim));
    sd.y[me] = Gp[me];
    sd.scale = 1.f;
    FusedArgs f;
    memset(&f, 0, sizeof(f));
    for (int i = 0; i < n; ++i) {
      f.Y[i] = Yp[i];
      f.A[i] = Ap[i];
      f.eflag[i] = (unsigned int*)(c->peer[i] + c->off_ef[par]);
      f.gflag[i] = (unsigned int*)(c->peer[i] + c->off_gf[par]);
    }
    f.ctr = c->fused_ctr[par];
    f.epoch = ++c->fepoch[par];
    f.n = n;
    f.me = me;
    f.r = r;
    f.own = owned_shard(me, r, n);
    f.ns = sh.base >> Tc;
    f.shard_len = sh.base;
    f.m = mv;
    f.trace = (uint4*)g_fused_trace;
    f.trace_cap = g_fused_trace_cap;
    f.watchdog_ns = watchdog_ns();
    f.grid_cap = c->fused_grid;
    f.deadline_ns = deadline_ns;
    f.stats = (unsigned long long*)stats;
    f.counts = counts;
    f.cut_units = cut_units;
    if (stats && (rc = stats_open(stats, st))) return rc;
    if ((rc = launch_fused(Tc, ae, ad, se, sd, f, st))) return rc < 0 ? OPTR_ECUDA : rc;
    CK(cudaEventRecord(c->fused_done[par], st));
    c->fused_recorded[par] = true;
    {  // strided decode pass: G -> out (scale, signs, truncate, cast)
      SrcBuf gb;
      memset(&gb, 0, sizeof(gb));
      gb.y[me] = Gp[me];
      SnkDecode snk;
      memset(&snk, 0, sizeof(snk));
      snk.out[me] = out;
      snk.count_base[me] = sh.len(owned_shard(me, r, n));
      snk.dtype = dtype_out;
      snk.L = L;
      snk.signs = signs;
      snk.signs_t = signs_t;
      snk.count_extra = counts + n;
      snk.count_stride = 1;
      snk.dim = (double)dim;
      if ((rc = launch_pass(OPTR_K_DEC_LAST, fps[1], nlog, me, 1, gb, snk, st))) return rc;
    }
    if (received_out) {
      CK(cudaMemcpyAsync(received_out, counts + me, 8, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(received_out + 1, counts + n + me, 8, cudaMemcpyDeviceToDevice, st));
    }
    CK(cudaEventRecord(c->done[par], st));
    c->done_recorded[par] = true;
    if (!async) CK(cudaStreamWaitEvent(caller, c->done[par], 0));
    return OPTR_OK;
  }

  // encode into my symmetric wire buffer
  if (ht) {
    SrcEncode src;
    memset(&src, 0, sizeof(src));
    src.x[me] = x;
    src.dtype = dtype_in;
    src.L = L;
    src.signs = signs;
    SrcBuf buf;
    memset(&buf, 0, sizeof(buf));
    buf.y[me] = Yp[me];
    SnkBuf snk;
    memset(&snk, 0, sizeof(snk));
    snk.y[me] = Yp[me];
    snk.scale = (float)(1.0 / sqrt((double)dim));
    rc = run_transform(log2_exact(dim), true, me, 1, src, buf, snk, st, OPTR_K_ENC_FIRST);
    if (rc) return rc;
  } else {
    KScope ks(OPTR_K_OTHER, st);
    cast_copy_kernel<<<1184, 256, 0, st>>>(x, dtype_in, Yp[me], dim);
    CK(cudaGetLastError());
  }
  if ((rc = comm_barrier(c, par, st))) return rc;
  if (stats && ((rc = stats_open(stats, st)) || (rc = stats_stamp(stats, ST_OPEN, st)))) return rc;

  // stage 1: pull my shard from every peer over NVLink, masked mean
  AggArgs ag;
  memset(&ag, 0, sizeof(ag));
  for (int i = 0; i < n; ++i) {
    ag.Y[i] = Yp[i];
    ag.A[i] = Ap[i];
  }
  ag.sh = sh;
  ag.n = n;
  ag.r = r;
  ag.m = mv;
  ag.owner_base = me;
  // Stage 2 fused into stage 1 (push): the owner writes its mean chunk into
  // every rank's receive vector G while it pulls the next chunk, so the
  // decode reads stage-2 data locally.  Needs the TMA aggregate.
  const bool push = agg_vec_ok(ag) && tma_enabled();
  if (push) {
    for (int i = 0; i < n; ++i) ag.G[i] = Gp[i];
    ag.push = 1;
  }
  int64_t smax = sh.base + (sh.extra ? 1 : 0);
  if ((rc = launch_aggregate(ag, 1, smax, st))) return rc;
  if ((rc = comm_barrier(c, par, st))) return rc;
  if (stats && (rc = stats_stamp(stats, ST_STAGE1, st))) return rc;

  // stage 2 receive fused into the first decode pass: from the local G
  // (push) or pulled from every owner's aggregate over NVLink
  SrcGather ga;
  memset(&ga, 0, sizeof(ga));
  for (int i = 0; i < n; ++i) ga.A[i] = push ? Gp[me] + sh.off(owned_shard(i, r, n)) : Ap[i];
  ga.sh = sh;
  ga.n = n;
  ga.r = r;
  ga.m = mv;
  ga.got = nullptr;
  ga.dim = dim;
  ga.pow2_shift = (sh.extra == 0 && is_pow2(sh.base)) ? log2_exact(sh.base) : -1;
  if (ht) {
    SrcBuf buf;
    memset(&buf, 0, sizeof(buf));
    buf.y[me] = Yp[me];  // peers finished reading my wire vector (barrier 2)
    SnkDecode snk;
    memset(&snk, 0, sizeof(snk));
    snk.out[me] = out;
    snk.count_base[me] = sh.len(owned_shard(me, r, n));
    snk.dtype = dtype_out;
    snk.L = L;
    snk.signs = signs;
    snk.count_extra = counts + n;
    snk.count_stride = 1;
    snk.dim = (double)dim;
    rc = run_transform(log2_exact(dim), true, me, 1, ga, buf, snk, st, OPTR_K_DEC_FIRST);
    if (rc) return rc;
  } else {
    AsmArgs as;
    memset(&as, 0, sizeof(as));
    as.gather = ga;
    as.out[me] = out;
    as.dtype = dtype_out;
    as.L = L;
    as.worker_base = me;
    int64_t blocks = (L + 255) / 256;
    if (blocks > 4736) blocks = 4736;
    KScope ks(OPTR_K_ASSEMBLE, st);
    assemble_kernel<<<dim3((unsigned)blocks, 1), 256, 0, st>>>(as);
    CK(cudaGetLastError());
  }
  if (received_out) {
    CK(cudaMemcpyAsync(received_out, counts + me, 8, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(received_out + 1, counts + n + me, 8, cudaMemcpyDeviceToDevice, st));
  }
  if (stats) {  // no deadline on this path: received = the mask-model counts
    if ((rc = stats_stamp(stats, ST_STAGE2, st))) return rc;
    stats_finish_kernel<<<1, 1, 0, st>>>((unsigned long long*)stats, counts, me, n);
    CK(cudaGetLastError());
  }
  CK(cudaEventRecord(c->done[par], st));
  c->done_recorded[par] = true;
  if (!async) CK(cudaStreamWaitEvent(caller, c->done[par], 0));
  return OPTR_OK;
}

// Entries per stage-1 unit of the fused kernel (the granularity of deadline
// cut-offs, optr_tar_bounded's cut_units); 0 when (dim, n) takes the barrier
// path.  Mirrors tma_fused_kernel's constants.
int64_t optr_fused_unit_entries(int64_t dim, int n) {
  if (!is_pow2(dim) || (n != 2 && n != 4 && n != 8)) return 0;
  PassGeom ps[3];
  const int nlog = log2_exact(dim);
  if (plan_passes(nlog, ps, true) != 2 || ps[0].cb != 0) return 0;
  const int T = ps[0].ks;
  if ((T != 13 && T != 14) || ps[1].cb != 3 || (ps[1].ks + 3 != 13 && ps[1].ks + 3 != 14)) return 0;
  if ((dim / n) < (1LL << T)) return 0;
  const int ch = agg_chunk(n);
  int sa = agg_bytes(T, n) / (n * ch * 4);
  if (sa > 16) sa = 16;
  const int cpt = (1 << T) / ch;
  const int upt = cpt / sa >= 4 ? 4 : (cpt / sa >= 2 ? 2 : 1);
  return (1LL << T) / upt;
}

// ------------------------------------------------------ instrumentation
int optr_debug_trace(void* dev_buf, int64_t per_cta) {
  if (per_cta < 0) {  // small-bucket kernel: [64][16] u64 phase stamps
    g_small_trace = dev_buf;
    return OPTR_OK;
  }
  g_fused_trace = dev_buf;
  g_fused_trace_cap = (int)per_cta;
  return OPTR_OK;
}

int optr_timing_enable(int on) {
  std::lock_guard<std::mutex> lk(g_tmu);
  g_timing = on != 0;
  return OPTR_OK;
}

int optr_timing_collect(double* ms_out, int64_t* launches_out, int64_t* units_out) {
  std::vector<TRec> recs;
  {
    std::lock_guard<std::mutex> lk(g_tmu);
    recs.swap(g_trecs);
  }
  if (ms_out)
    for (int i = 0; i < OPTR_K_CLASSES; ++i) ms_out[i] = 0.0;
  if (launches_out)
    for (int i = 0; i < OPTR_K_CLASSES; ++i) launches_out[i] = 0;
  if (units_out)
    for (int i = 0; i < OPTR_K_CLASSES; ++i) units_out[i] = 0;
  int rc = OPTR_OK;
  for (auto& r : recs) {
    float ms = 0.f;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess)
      rc = OPTR_ECUDA;
    if (r.cls >= 0 && r.cls < OPTR_K_CLASSES) {
      if (ms_out) ms_out[r.cls] += ms;
      if (launches_out) launches_out[r.cls] += 1;
      if (units_out) units_out[r.cls] += r.units;
    }
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  return rc;
}

int64_t optr_launch_count(void) { return g_launches.load(); }

}  // extern "C"
