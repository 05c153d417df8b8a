// Launchers of the small-bucket kernels (small.cuh), in their own
// translation unit: the 16 kernel instantiations compile beside api.cu.
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <mutex>

#include "../../include/optr.h"
#define OPTR_NO_GLOBAL_KERNELS
#include "kernels.cuh"
#include "small.cuh"
#include "internal.h"

using namespace optr;

namespace {

// this translation unit's copy of the PCG jump table (constant memory is
// per translation unit without relocatable device code)
int ensure_jump_table() {
  static std::mutex mu;
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!done[dev & 63]) {
    const JumpTable t = make_jump_table();
    if (cudaMemcpyToSymbol(c_jump, &t, sizeof(t)) != cudaSuccess) return OPTR_ECUDA;
    done[dev & 63] = true;
  }
  return OPTR_OK;
}

template <class K, class A>
int launch_coop(K kern, const A& a, int grid, cudaStream_t st, const char* name, int k) {
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(1u << (kSmallT - 5));
  cfg.dynamicSmemBytes = sizeof(float) * (size_t)pad(1 << kSmallT);  // < 48 KB: no attribute
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // grid barriers: every CTA co-resident
  attr[0].val.cooperative = 1;                   // (a plain launch measured the same)
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  if (e != cudaSuccess) {
    fprintf(stderr, "optr: %s<%d> grid=%d launch failed: %s\n", name, k, grid, cudaGetErrorString(e));
    return OPTR_ECUDA;
  }
  return OPTR_OK;
}

template <int K>
int local_t(const SmallLocalArgs& a, cudaStream_t st) {
  auto kern = tar_small_local_kernel<K>;
  const size_t smem = sizeof(float) * (size_t)pad(1 << kSmallT);
  int dev = 0, nsm = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (nsm <= 0) nsm = 148;
  // every co-resident CTA (cooperative): more tile jobs per pass in flight
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 1 << (kSmallT - 5), smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  if (per_sm > 2) per_sm = 2;
  if ((a.dim >> kSmallT) * a.n <= nsm) per_sm = 1;  // few tile jobs: cheaper barriers
  return launch_coop(kern, a, nsm * per_sm, st, "tar_small_local_kernel", K);
}

}  // namespace

int optr_small_launch(int K, const SmallArgs& a, int grid, cudaStream_t st) {
  int rc = ensure_jump_table();
  if (rc) return rc;
  switch (K) {
    case 13: return launch_coop(tar_small_kernel<13>, a, grid, st, "tar_small_kernel", K);
    case 14: return launch_coop(tar_small_kernel<14>, a, grid, st, "tar_small_kernel", K);
    case 15: return launch_coop(tar_small_kernel<15>, a, grid, st, "tar_small_kernel", K);
    case 16: return launch_coop(tar_small_kernel<16>, a, grid, st, "tar_small_kernel", K);
    case 17: return launch_coop(tar_small_kernel<17>, a, grid, st, "tar_small_kernel", K);
    case 18: return launch_coop(tar_small_kernel<18>, a, grid, st, "tar_small_kernel", K);
    case 19: return launch_coop(tar_small_kernel<19>, a, grid, st, "tar_small_kernel", K);
    case 20: return launch_coop(tar_small_kernel<20>, a, grid, st, "tar_small_kernel", K);
    default: return OPTR_EINVAL;
  }
}

int optr_small_local_launch(int K, const SmallLocalArgs& a, cudaStream_t st) {
  int rc = ensure_jump_table();
  if (rc) return rc;
  switch (K) {
    case 13: return local_t<13>(a, st);
    case 14: return local_t<14>(a, st);
    case 15: return local_t<15>(a, st);
    case 16: return local_t<16>(a, st);
    case 17: return local_t<17>(a, st);
    case 18: return local_t<18>(a, st);
    case 19: return local_t<19>(a, st);
    case 20: return local_t<20>(a, st);
    default: return OPTR_EINVAL;
  }
}
