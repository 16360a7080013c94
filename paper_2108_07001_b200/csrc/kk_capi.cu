// C-ABI plumbing for libkkb200.so: thread-local last error, status codes,
// lazily built immutable twiddle tables (one per device, std::call_once).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <set>
#include <utility>
#include <vector>

#include "kk_common.cuh"
#include "kk_internal.h"

namespace kk {

static thread_local char g_err[512] = {0};
static unsigned long long g_launches = 0;   // kernels launched through this library

void clear_error() { g_err[0] = 0; }

int set_error(int code, const char* msg) {
    std::snprintf(g_err, sizeof(g_err), "%s", msg ? msg : "error");
    return code;
}

int set_cuda_error(const char* where) {
    const cudaError_t e = cudaGetLastError();
    std::snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return KK_ERR_CUDA;
}

int check_launch(const char* name) {
    __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        std::snprintf(g_err, sizeof(g_err), "launch %s: %s", name, cudaGetErrorString(e));
        return KK_ERR_CUDA;
    }
    return KK_OK;
}

namespace {
constexpr int kMaxDev = 64;
std::once_flag g_tw_once[kMaxDev];
float2* g_tw[kMaxDev] = {nullptr};
}  // namespace

int ensure_smem_attr(const void* fn, size_t smem, const char* what) {
    static std::mutex mu;
    static std::set<std::pair<int, const void*>> done;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return set_cuda_error("cudaGetDevice");
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({dev, fn})) return KK_OK;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
        return set_cuda_error(what);
    done.insert({dev, fn});
    return KK_OK;
}

int num_sms() {
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (!cached[dev]) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        cached[dev] = n;
    }
    return cached[dev];
}

const float2* twiddle_table_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) {
        set_cuda_error("cudaGetDevice");
        return nullptr;
    }
    std::call_once(g_tw_once[dev], [dev]() {
        std::vector<float2> h(kTwEntries + kTwPassEntries);
        const double two_pi = 6.283185307179586476925286766559;
        for (int M = 256; M <= 32768; M *= 2) {
            const int o = tw_offset(M);
            for (int i = 0; i < 32; ++i) {          // L_M[i] = W_M^i
                const double a = -two_pi * i / M;
                h[o + i] = make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
            }
            for (int i = 0; i < M / 32; ++i) {      // H_M[i] = W_M^(32 i)
                const double a = -two_pi * (32.0 * i) / M;
                h[o + 32 + i] = make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
            }
        }
        // K1's per-pass tables (kk_common.cuh DirectTwiddle), after the two-level ones
        for (int r = 1; r < 16; ++r)
            for (int m = 0; m < 16; ++m) {
                const double a = -two_pi * ((r * m) % 256) / 256.0;
                h[kTwEntries + kTwPass16 + (r - 1) * 16 + m] =
                    make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
            }
        for (int r = 1; r < 4; ++r)
            for (int m = 0; m < 256; ++m) {
                const double a = -two_pi * ((r * m) % 1024) / 1024.0;
                h[kTwEntries + kTwPass4 + (r - 1) * 256 + m] =
                    make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
            }
        float2* d = nullptr;
        const size_t nt = kTwEntries + kTwPassEntries;
        if (cudaMalloc(&d, nt * sizeof(float2)) == cudaSuccess &&
            cudaMemcpy(d, h.data(), nt * sizeof(float2), cudaMemcpyHostToDevice) == cudaSuccess)
            g_tw[dev] = d;
    });
    if (!g_tw[dev]) set_error(KK_ERR_CUDA, "twiddle table allocation failed");
    return g_tw[dev];
}

}  // namespace kk

extern "C" const char* kk_last_error(void) { return kk::g_err; }

extern "C" int kk_version(void) { return KK_ABI_VERSION; }

extern "C" unsigned long long kk_launch_count(void) { return __atomic_load_n(&kk::g_launches, __ATOMIC_RELAXED); }

extern "C" int kk_device_sync(void) {
    kk::clear_error();
    if (cudaDeviceSynchronize() != cudaSuccess) return kk::set_cuda_error("cudaDeviceSynchronize");
    return KK_OK;
}

// ---------------------------------------------------------------------------
// Small host->device uploads through kernel parameters.  A DMA copy (pinned
// or pageable above 64 KB) issued while bulk input copies are queued waits
// for them on the host->device copy engine; kernel parameters travel in the
// launch itself, so per-stream set-up data (equaliser tables, reference
// symbols) lands in order on its own stream.  16 KB per launch.
// ---------------------------------------------------------------------------
namespace kk {
constexpr int kUpBlob = 16384;
struct alignas(16) UpBlob {
    unsigned char b[kUpBlob];
};
// __grid_constant__: indexed straight from the parameter bank (a plain by-
// value struct indexed dynamically is first copied to local memory per thread)
__global__ void upload_blob_kernel(unsigned char* __restrict__ dst, const __grid_constant__ UpBlob blob,
                                   int nbytes) {
    const int i = threadIdx.x * 16;
    if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0 && i + 16 <= nbytes) {
        *reinterpret_cast<uint4*>(dst + i) = *reinterpret_cast<const uint4*>(blob.b + i);
    } else {
        for (int k = i; k < min(i + 16, nbytes); ++k) dst[k] = blob.b[k];
    }
}
}  // namespace kk

extern "C" int kk_upload(void* dst, const void* src, int64_t bytes, void* stream) {
    kk::clear_error();
    if (bytes < 0 || (bytes > 0 && (!dst || !src))) return kk::set_error(KK_ERR_PARAM, "kk_upload: bad arguments");
    static kk::UpBlob blob;   // staging for the launch arguments (copied at launch)
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    const auto* s = static_cast<const unsigned char*>(src);
    auto* d = static_cast<unsigned char*>(dst);
    for (int64_t off = 0; off < bytes; off += kk::kUpBlob) {
        const int n = static_cast<int>(std::min<int64_t>(kk::kUpBlob, bytes - off));
        std::memcpy(blob.b, s + off, n);
        kk::upload_blob_kernel<<<1, kk::kUpBlob / 16, 0, static_cast<cudaStream_t>(stream)>>>(d + off, blob, n);
        if (int rc = kk::check_launch("upload_blob_kernel")) return rc;
    }
    return KK_OK;
}

// ---------------------------------------------------------------------------
// FP32 FMA throughput microbenchmark (the roofline denominator for the
// FP32-bound FFT kernels; MEASURED_PEAKS.json has no FP32 entry).  Each
// thread runs 8 independent FFMA chains; returns FLOP/s (2 per FFMA).
// ---------------------------------------------------------------------------
namespace kk {
__global__ void fma_peak_kernel(float* out, int iters, float a, float b) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
          x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
            x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
        }
    }
    const float s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 1234.5f) out[threadIdx.x] = s;   // keep the chains alive
}
}  // namespace kk

extern "C" int kk_fma_peak(double* flops_per_s, void* stream) {
    kk::clear_error();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    float* out = nullptr;
    if (cudaMalloc(&out, 1024 * sizeof(float)) != cudaSuccess) return kk::set_cuda_error("fma peak alloc");
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kk::fma_peak_kernel<<<blocks, threads, 0, s>>>(out, 64, 0.999f, 1e-3f);   // warm-up
    cudaEventRecord(e0, s);
    kk::fma_peak_kernel<<<blocks, threads, 0, s>>>(out, iters, 0.999f, 1e-3f);
    cudaEventRecord(e1, s);
    int rc = kk::check_launch("fma_peak_kernel");
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (rc) return rc;
    const double flops = 2.0 * 8 * 16 * double(iters) * blocks * threads;
    *flops_per_s = flops / (ms * 1e-3);
    return KK_OK;
}
