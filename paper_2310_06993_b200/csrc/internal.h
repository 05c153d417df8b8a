// Library-internal helpers shared by the translation units of liboptr.so
// (not part of the C ABI in include/optr.h).
#pragma once
#include <stdint.h>

// count `k` kernel launches in optr_launch_count()
void optr_note_launches(int k);
// make this library's runtime use the device of the caller's stream
void optr_bind_stream_device(void* stream);

// small-bucket kernels (small.cu: their own translation unit, compiled in
// parallel with api.cu); cooperative launches, OPTR_* status
#include <cuda_runtime.h>
namespace optr {
struct SmallArgs;
struct SmallLocalArgs;
}  // namespace optr
int optr_small_launch(int K, const optr::SmallArgs& a, int grid, cudaStream_t st);
int optr_small_local_launch(int K, const optr::SmallLocalArgs& a, cudaStream_t st);
