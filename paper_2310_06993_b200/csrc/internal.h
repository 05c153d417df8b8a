// Library-internal helpers shared by the translation units of liboptr.so
// (not part of the C ABI in include/optr.h).
#pragma once
#include <stdint.h>

// count `k` kernel launches in optr_launch_count()
void optr_note_launches(int k);
// make this library's runtime use the device of the caller's stream
void optr_bind_stream_device(void* stream);
