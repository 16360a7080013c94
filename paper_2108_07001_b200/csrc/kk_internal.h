// Host-side internals shared by the translation units of libkkb200.so:
// status codes (mirrored in include/kkb200.h), the thread-local last-error
// string, and the lazily built per-device twiddle table.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/kkb200.h"

namespace kk {

void clear_error();
int set_error(int code, const char* msg);
int set_cuda_error(const char* where);
int check_launch(const char* name);

// W_32768 two-level table on the current device: [hi(512) | lo(64)] float2.
// Built once per device (std::call_once), immutable afterwards.
const float2* twiddle_table_device();

// SM count of the current device (cached per device)
int num_sms();

// cudaFuncAttributeMaxDynamicSharedMemorySize for `fn` on the current device,
// set once per (device, kernel) for the whole process (thread-safe)
int ensure_smem_attr(const void* fn, size_t smem, const char* what);

// float64 power-of-two FFT (kk_fft.cu): twiddle tables for 2^log_n points
// (table_bytes of device memory, built stream-ordered), and the batched
// forward transform of `batch` rows ping-ponging between a and b (*result is
// whichever holds the output).
namespace fft64 {
size_t table_bytes(int log_n);
int build_tables(void* mem, int log_n, cudaStream_t st);
int forward_pow2(double2* a, double2* b, int log_n, int64_t batch, const void* tables, cudaStream_t st,
                 double2** result);
}  // namespace fft64

}  // namespace kk
