// Throughput of scalar vs packed (f32x2) FP32 instructions on sm_100a:
// FFMA / FFMA2, FADD / FADD2, FMUL / FMUL2 with register operands (the form
// FFT butterflies use).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// tools/f32x2_bench.cu -o /tmp/f32x2 && /tmp/f32x2
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) {
    u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r;
}
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
    u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;
}
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) {
    u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r;
}
__device__ __forceinline__ u64 fmul2(u64 a, u64 b) {
    u64 r; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r;
}
__device__ __forceinline__ float ffma1(float a, float b, float c) {
    float r; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r;
}
__device__ __forceinline__ float fadd1(float a, float b) {
    float r; asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r;
}

template <int OP>
__global__ void bench(float* out, int iters, const float* in) {
    const int t = threadIdx.x;
    float y[8], z[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { y[i] = in[(t + i) & 255]; z[i] = in[(t + 3 * i + 1) & 255]; }
    if (OP < 2) {   // scalar: 16 chains
        float x[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = in[(t + 7 * i) & 255];
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < 16; ++i) x[i] = OP == 0 ? ffma1(x[i], y[i & 7], z[i & 7]) : fadd1(x[i], y[i & 7]);
        }
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) s += x[i];
        if (s == 1234.5f) out[t] = s;
    } else {        // packed: 8 chains of 2 lanes = 16 FP32 ops per iteration as well
        u64 x[8], yy[4], zz[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = pk(in[(t + 7 * i) & 255], in[(t + 7 * i + 3) & 255]);
#pragma unroll
        for (int i = 0; i < 4; ++i) { yy[i] = pk(y[2 * i], y[2 * i + 1]); zz[i] = pk(z[2 * i], z[2 * i + 1]); }
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                x[i] = OP == 2 ? ffma2(x[i], yy[i & 3], zz[i & 3]) : (OP == 3 ? fadd2(x[i], yy[i & 3]) : fmul2(x[i], yy[i & 3]));
        }
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) { float2 v = *reinterpret_cast<float2*>(&x[i]); s += v.x + v.y; }
        if (s == 1234.5f) out[t] = s;
    }
}

template <int OP>
double run(float* out, const float* in, int sms) {
    const int blocks = sms * 8, threads = 256, iters = 8192;
    bench<OP><<<blocks, threads>>>(out, 16, in);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench<OP><<<blocks, threads>>>(out, iters, in);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 16.0 * iters * blocks * threads;   // FP32 lane-ops (an FMA counts once)
    return ops / (ms * 1e-3) / 1e12;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out, *in; cudaMalloc(&out, 1024 * 4); cudaMalloc(&in, 256 * 4);
    float h[256]; for (int i = 0; i < 256; ++i) h[i] = 1.0f + 1e-6f * i;
    cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 2; ++rep) {
        printf("FFMA  reg: %7.2f T lane-op/s\n", run<0>(out, in, sms));
        printf("FADD  reg: %7.2f T lane-op/s\n", run<1>(out, in, sms));
        printf("FFMA2 reg: %7.2f T lane-op/s\n", run<2>(out, in, sms));
        printf("FADD2 reg: %7.2f T lane-op/s\n", run<3>(out, in, sms));
        printf("FMUL2 reg: %7.2f T lane-op/s\n", run<4>(out, in, sms));
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
