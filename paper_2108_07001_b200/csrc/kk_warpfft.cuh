// Warp-level FFT building blocks (four-step factorisations whose inner
// transforms run inside one warp, so only __syncwarp separates their passes).
//
//   warp_fft1024: 1024 = 32 x 32.  Lane a holds y[a + 32 b] (b = 0..31),
//     DFT32 over b, twiddle W1024^{a c}, transpose through the warp's own
//     row (rotation swizzle, conflict-free), DFT32 over a -> Y[c + 32 d] in
//     lane c, written back in natural order.
//   warp_fft512: 512 = 32 x 16.  Lane a holds y[a + 32 b] (b = 0..15),
//     DFT16 over b, twiddle W512^{a c}, transpose, then each 32-point column
//     DFT is split over a lane pair (c, h): one radix-2 DIF stage in
//     registers (h = 0 even, h = 1 odd outputs) and a DFT16 each.
//
// The block-level step (a DFT16 over a stride of N/16 and the W_N twiddle)
// is the caller's: it is fused with the kernels' global loads.
#pragma once

#include "kk_common.cuh"

namespace kk {

// cos/sin(2*pi*t/32), t in [0, 16)
__host__ __device__ constexpr float c32(int t) {
    return t == 0 ? 1.0f : t == 1 ? 0.98078528040323044913f : t == 2 ? 0.92387953251128675613f
         : t == 3 ? 0.83146961230254523708f : t == 4 ? 0.70710678118654752440f
         : t == 5 ? 0.55557023301960222474f : t == 6 ? 0.38268343236508977173f
         : t == 7 ? 0.19509032201612826785f : t == 8 ? 0.0f : t == 9 ? -0.19509032201612826785f
         : t == 10 ? -0.38268343236508977173f : t == 11 ? -0.55557023301960222474f
         : t == 12 ? -0.70710678118654752440f : t == 13 ? -0.83146961230254523708f
         : t == 14 ? -0.92387953251128675613f : -0.98078528040323044913f;
}
__host__ __device__ constexpr float s32(int t) { return c32(t < 8 ? 8 - t : t - 8); }

// multiply by W32^t (forward exp(-2 pi i t/32); inverse: conjugate); t must
// fold to a constant (template or unrolled loop index)
template <bool INV>
__device__ __forceinline__ float2 tw32(float2 a, int t) {
    if (t == 0) return a;
    if (t == 8) return INV ? mul_pj(a) : mul_mj(a);
    const float c = c32(t), s = INV ? s32(t) : -s32(t);
    return cmul_const(a, c, s);
}

template <bool INV, int K = 0>
__device__ __forceinline__ void dif32_stage(float2 (&v)[32], float2 (&s)[16], float2 (&t)[16]) {
    if constexpr (K < 16) {
        s[K] = cadd(v[K], v[K + 16]);
        t[K] = tw32<INV>(csub(v[K], v[K + 16]), K);
        dif32_stage<INV, K + 1>(v, s, t);
    }
}

// In-register 32-point DFT, natural order in and out.
template <bool INV>
__device__ __forceinline__ void dft32(float2 (&v)[32]) {
    float2 s[16], t[16];
    dif32_stage<INV>(v, s, t);
    dft_reg<16, INV>(s);
    dft_reg<16, INV>(t);
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        v[2 * m] = s[m];
        v[2 * m + 1] = t[m];
    }
}

// w^r for r = 1..R-1 applied in place to v[r] (running product from w1)
template <int R, bool INV>
__device__ __forceinline__ void apply_twiddle_chain(float2 (&v)[R], float2 w1) {
    if constexpr (INV) w1 = cconj(w1);
    float2 wr = w1;
#pragma unroll
    for (int r = 1; r < R; ++r) {
        v[r] = cmul(v[r], wr);
        if (r + 1 < R) wr = cmul(wr, w1);
    }
}

// conflict-free in-row transpose slot of element (c, a) of a [C][32] tile
__device__ __forceinline__ int xpose_slot(int c, int a) { return c * 32 + ((a + c) & 31); }

// 1024-point FFT by one warp with fused I/O: input element i comes from
// load(i) (i = lane + 32 b), output k = lane + 32 d goes to store(d, k, v)
// (d compile-time after unrolling); row[0..1024) is the transpose scratch.
template <bool INV, class Load, class Store>
__device__ __forceinline__ void warp_fft1024_io(float2* row, int lane, const Twiddle& tw, const Load& load,
                                                const Store& store) {
    float2 v[32];
#pragma unroll
    for (int b = 0; b < 32; ++b) v[b] = load(lane + 32 * b);
    dft32<INV>(v);
    apply_twiddle_chain<32, INV>(v, tw.template w<1024>(lane));
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 32; ++c) row[xpose_slot(c, lane)] = v[c];
    __syncwarp();
#pragma unroll
    for (int a = 0; a < 32; ++a) v[a] = row[xpose_slot(lane, a)];
    dft32<INV>(v);
    __syncwarp();
#pragma unroll
    for (int d = 0; d < 32; ++d) store(d, lane + 32 * d, v[d]);
    __syncwarp();
}

// 1024-point FFT of row[0..1024) (natural order in and out) by one warp.
template <bool INV>
__device__ __forceinline__ void warp_fft1024(float2* row, int lane, const Twiddle& tw) {
    warp_fft1024_io<INV>(row, lane, tw, [&](int i) { return row[i]; },
                         [&](int, int k, float2 v) { row[k] = v; });
}

// 512-point FFT of row[0..512) by one warp; output k = c + 16 (2 d + h) of
// lane (c = lane & 15, h = lane >> 4), register d, goes to store(k, value).
template <bool INV, class Store>
__device__ __forceinline__ void warp_fft512(float2* row, int lane, const Twiddle& tw, const Store& store) {
    float2 v[16];
#pragma unroll
    for (int b = 0; b < 16; ++b) v[b] = row[lane + 32 * b];
    dft_reg<16, INV>(v);
    apply_twiddle_chain<16, INV>(v, tw.template w<512>(lane));
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 16; ++c) row[xpose_slot(c, lane)] = v[c];
    __syncwarp();
    const int c = lane & 15, h = lane >> 4;
    const float sg = h ? -1.f : 1.f;
#pragma unroll
    for (int a = 0; a < 16; ++a) {
        const float2 z0 = row[xpose_slot(c, a)], z1 = row[xpose_slot(c, a + 16)];
        const float2 d = make_float2(fmaf(sg, z1.x, z0.x), fmaf(sg, z1.y, z0.y));
        // h = 1: (z0 - z1) W32^a  (radix-2 DIF stage of the column DFT32)
        const float2 dt = tw32<INV>(d, a);
        v[a] = h ? dt : d;
    }
    dft_reg<16, INV>(v);
    __syncwarp();
#pragma unroll
    for (int d = 0; d < 16; ++d) store(c + 16 * (2 * d + h), v[d]);
}

}  // namespace kk
