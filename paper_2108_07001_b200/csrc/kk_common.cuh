// Shared device building blocks for the B200 KK receiver kernels.
//
// * complex helpers on float2,
// * in-register radix-{2,4,8,16} DFTs (DIF, compile-time twiddles),
// * an in-place shared-memory Stockham pass engine: every pass reads all of
//   its inputs into registers, barriers, butterflies, writes the outputs to
//   the autosorted positions and barriers again, so one padded buffer
//   (float2, one pad slot per 16) serves all passes.
//   The first pass can read through a functor (global memory, fused
//   pre-processing) and the last pass can write through a functor (fused
//   epilogue), so only the middle passes touch shared memory.
// * per-size two-level twiddle tables W_M^k = H_M[k>>5] L_M[k&31] for
//   M = 256..32768 (conflict-free for the lanes of a pass).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace kk {


// KK_PACKED_ADD / KK_PACKED_MUL: complex adds and multiplies on sm_100's
// packed FP32 instructions (FADD2 / FMUL2 / FFMA2: one instruction per re/im
// pair).  Same roundings as the scalar form (every lane is one add.rn /
// mul.rn / fma.rn of the same operands), so results are bit-identical; what
// changes is the issue count of the instruction-bound FFT kernels
// (tools/f32x2_bench.cu: packed and scalar ops have the same lane
// throughput, the packed ones take half the issue slots).  Per translation
// unit (set before this header is included), A/B'd per kernel: K1 (kk_kk.cu)
// packs all three, 7.13 -> 6.63 ms per 2^30 samples; K2 (kk_static.cu) the
// adds and constant-twiddle multiplies, 11.80 -> 11.51 ms.  KK_PACKED_CONST
// (constant multiplies) follows KK_PACKED_MUL unless set.
#ifndef KK_PACKED_ADD
#define KK_PACKED_ADD 0
#endif
#ifndef KK_PACKED_MUL
#define KK_PACKED_MUL 0
#endif
#if KK_PACKED_ADD
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
#else
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
#endif
#ifndef KK_PACKED_CONST
#define KK_PACKED_CONST KK_PACKED_MUL
#endif
// KK_PACKED_NP: the forms below let ptxas fold the one-lane negation into the
// FFMA2 addend (the ".NP" operand modifier) and the re/im swap into an operand
// selector, so a complex multiply is FMUL2 + FFMA2 with no pair-forming moves
#ifndef KK_PACKED_NP
#define KK_PACKED_NP 1
#endif
#if KK_PACKED_CONST
// a * (c + i s) with c, s compile-time constants: (a.x c - a.y s, a.x s + a.y c)
__device__ __forceinline__ float2 cmul_const(float2 a, float c, float s) {
#if KK_PACKED_NP
    const float2 t = __fmul2_rn(make_float2(a.y, a.y), make_float2(s, c));
    return __ffma2_rn(make_float2(a.x, a.x), make_float2(c, s), make_float2(-t.x, t.y));
#else
    const float2 t = __fmul2_rn(make_float2(a.y, a.y), make_float2(-s, c));
    return __ffma2_rn(make_float2(a.x, a.x), make_float2(c, s), t);
#endif
}
#else
__device__ __forceinline__ float2 cmul_const(float2 a, float c, float s) {
    return make_float2(fmaf(a.x, c, -a.y * s), fmaf(a.x, s, a.y * c));
}
#endif
#if KK_PACKED_MUL && KK_PACKED_NP
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    const float2 t = __fmul2_rn(make_float2(a.y, a.y), make_float2(b.y, b.x));
    return __ffma2_rn(make_float2(a.x, a.x), b, make_float2(-t.x, t.y));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
    const float2 t = __fmul2_rn(make_float2(a.y, a.x), make_float2(b.y, b.y));
    return __ffma2_rn(a, make_float2(b.x, b.x), make_float2(t.x, -t.y));
}
#elif KK_PACKED_MUL
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    const float2 t = __fmul2_rn(make_float2(a.y, a.y), make_float2(-b.y, b.x));
    return __ffma2_rn(make_float2(a.x, a.x), b, t);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
    const float2 t = __fmul2_rn(make_float2(a.y, a.x), make_float2(b.y, -b.y));
    return __ffma2_rn(a, make_float2(b.x, b.x), t);
}
#else
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
    return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
#endif
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 mul_mj(float2 a) { return make_float2(a.y, -a.x); }   // * (-j)
__device__ __forceinline__ float2 mul_pj(float2 a) { return make_float2(-a.y, a.x); }   // * (+j)

// x mod d for 0 <= x < 2^25 via a float reciprocal (+-1 quotient fix-up)
__device__ __forceinline__ unsigned fmod_u(unsigned x, unsigned d, float inv_d, unsigned* quot = nullptr) {
    unsigned q = __float2uint_rz(__uint2float_rn(x) * inv_d);
    int r = static_cast<int>(x) - static_cast<int>(q * d);
    if (r < 0) { r += d; --q; }
    if (r >= static_cast<int>(d)) { r -= d; ++q; }
    if (quot) *quot = q;
    return static_cast<unsigned>(r);
}

// Downshift rotation of a general tone (rot_q == 0, rot_step != 0 in the C
// ABI): exp(-2 pi i ph / 2^64), ph = g * rot_step (mod 2^64) the phase of
// global sample g as a 64-bit fixed-point fraction of a cycle (exact at any
// stream index; sigcore.py frequency_shift :286-299 computes the same phase
// in float64).  Fast: the top 32 bits through the SFU (~1e-6 absolute);
// precise: float64 sincospi of the whole phase.
__device__ __forceinline__ float2 rot_phase_fast(unsigned long long ph) {
    const float x = static_cast<float>(static_cast<int>(static_cast<unsigned>(ph >> 32))) * 2.3283064365386963e-10f;
    float s, c;
    __sincosf(-6.283185307179586f * x, &s, &c);     // x in [-0.5, 0.5): no range reduction needed
    return make_float2(c, s);
}
__device__ __forceinline__ float2 rot_phase_precise(unsigned long long ph) {
    double s, c;
    sincospi(-2.0 * static_cast<double>(static_cast<long long>(ph)) * 5.421010862427522170e-20, &s, &c);
    return make_float2(static_cast<float>(c), static_cast<float>(s));
}

// cos/sin(2*pi*t/16) for t in [0,8)
__host__ __device__ constexpr float c16(int t) {
    return t == 0 ? 1.0f : t == 1 ? 0.92387953251128674f : t == 2 ? 0.70710678118654752f
         : t == 3 ? 0.38268343236508977f : t == 4 ? 0.0f : t == 5 ? -0.38268343236508977f
         : t == 6 ? -0.70710678118654752f : -0.92387953251128674f;
}
__host__ __device__ constexpr float s16(int t) {
    return t == 0 ? 0.0f : t == 1 ? 0.38268343236508977f : t == 2 ? 0.70710678118654752f
         : t == 3 ? 0.92387953251128674f : t == 4 ? 1.0f : t == 5 ? 0.92387953251128674f
         : t == 6 ? 0.70710678118654752f : 0.38268343236508977f;
}

// multiply by W16^t (forward: exp(-2*pi*i*t/16); inverse: conjugate), t compile-time
template <int T, bool INV>
__device__ __forceinline__ float2 tw16(float2 a) {
    if constexpr (T == 0) {
        return a;
    } else if constexpr (T == 4) {
        return INV ? mul_pj(a) : mul_mj(a);
    } else {
        constexpr float c = c16(T);
        constexpr float s = INV ? s16(T) : -s16(T);
        return cmul_const(a, c, s);
    }
}

template <int LOG>
__host__ __device__ constexpr int bitrev(int i) {
    int r = 0;
    for (int b = 0; b < LOG; ++b) r |= ((i >> b) & 1) << (LOG - 1 - b);
    return r;
}
template <int R> struct Log2;
template <> struct Log2<2> { static constexpr int v = 1; };
template <> struct Log2<4> { static constexpr int v = 2; };
template <> struct Log2<8> { static constexpr int v = 3; };
template <> struct Log2<16> { static constexpr int v = 4; };

// radix-2 DIF stage with span S inside an R-point register DFT
template <int R, int S, bool INV>
__device__ __forceinline__ void dif_stage(float2 (&v)[R]) {
#pragma unroll
    for (int j = 0; j < R; j += 2 * S) {
#pragma unroll
        for (int k = 0; k < S; ++k) {
            float2 a = v[j + k], b = v[j + k + S];
            v[j + k] = cadd(a, b);
            float2 d = csub(a, b);
            // W_{2S}^k = W16^{k * 16/(2S)}
            switch (k * (16 / (2 * S))) {
                case 0: v[j + k + S] = tw16<0, INV>(d); break;
                case 1: v[j + k + S] = tw16<1, INV>(d); break;
                case 2: v[j + k + S] = tw16<2, INV>(d); break;
                case 3: v[j + k + S] = tw16<3, INV>(d); break;
                case 4: v[j + k + S] = tw16<4, INV>(d); break;
                case 5: v[j + k + S] = tw16<5, INV>(d); break;
                case 6: v[j + k + S] = tw16<6, INV>(d); break;
                default: v[j + k + S] = tw16<7, INV>(d); break;
            }
        }
    }
}

// In-register R-point DFT, natural order in and out.
template <int R, bool INV>
__device__ __forceinline__ void dft_reg(float2 (&v)[R]) {
    if constexpr (R >= 16) dif_stage<R, 8, INV>(v);
    if constexpr (R >= 8) dif_stage<R, 4, INV>(v);
    if constexpr (R >= 4) dif_stage<R, 2, INV>(v);
    dif_stage<R, 1, INV>(v);
    float2 t[R];
#pragma unroll
    for (int i = 0; i < R; ++i) t[i] = v[bitrev<Log2<R>::v>(i)];
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = t[i];
}

// ---------------------------------------------------------------------------
// twiddles: for every power of two M in [256, 32768] a two-level table
//   W_M^k = H_M[k >> 5] * L_M[k & 31],  L_M[i] = W_M^i, H_M[i] = W_M^(32 i)
// so that 32 consecutive k (the lanes of a Stockham pass) read 32
// consecutive L entries (conflict-free) and one or two broadcast H entries.
// Packed [L_256 H_256 | L_512 H_512 | ... | L_32768 H_32768], built once per
// device on the host in float64 (kk_capi.cu) and staged into smem.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int ilog2c(int m) { return m <= 1 ? 0 : 1 + ilog2c(m >> 1); }
__host__ __device__ constexpr int tw_offset(int M) { return 32 * (ilog2c(M) - 8) + M / 32 - 8; }
constexpr int kTwEntries = tw_offset(65536);   // 2296 float2 = 18.4 KB

struct Twiddle {
    const float2* t;
    // W_M^k (forward sign), 0 <= k < M
    template <int M>
    __device__ __forceinline__ float2 w(int k) const {
        static_assert(M >= 256 && M <= 32768, "twiddle size");
        constexpr int o = tw_offset(M);
        return cmul(t[o + 32 + (k >> 5)], t[o + (k & 31)]);
    }
};

// Per-pass twiddle tables of K1's 1024-point transforms, appended to the
// global table after kTwEntries: W_256^{r m} (r = 1..15, m = 0..15) for the
// radix-16 pass with NS = 16 and W_1024^{r m} (r = 1..3, m = 0..255) for the
// radix-4 pass with NS = 256 -- one load per twiddle instead of a running
// product (fewer instructions, correctly rounded twiddles).  Read through the
// read-only path (L1 resident; K1's shared memory is its occupancy limit).
constexpr int kTwPass16 = 0;
constexpr int kTwPass4 = 15 * 16;
constexpr int kTwPassEntries = kTwPass4 + 3 * 256;

struct DirectTwiddle : Twiddle {
    const float2* p;     // pass tables (global)
    static constexpr bool kDirect = true;
    template <int NS, int R>
    __device__ __forceinline__ float2 d(int r, int m) const {
        if constexpr (NS == 16 && R == 16) return __ldg(p + kTwPass16 + (r - 1) * 16 + m);
        else return __ldg(p + kTwPass4 + (r - 1) * 256 + m);
    }
};
template <class T, class = void>
struct has_direct { static constexpr bool value = false; };
template <class T>
struct has_direct<T, decltype(void(T::kDirect))> { static constexpr bool value = T::kDirect; };

__device__ __forceinline__ void load_twiddles(float2* sm, const float2* __restrict__ g, int tid, int nt) {
    for (int i = tid; i < kTwEntries; i += nt) sm[i] = g[i];
}

// w[r] = w1^r for r in [0, R), by a power tree of depth <= 4 (accuracy ~1e-7)
template <int R>
__device__ __forceinline__ void twiddle_powers(float2 w1, float2 (&w)[R]) {
    w[0] = make_float2(1.f, 0.f);
    if constexpr (R > 1) w[1] = w1;
    if constexpr (R > 2) w[2] = cmul(w1, w1);
    if constexpr (R > 3) w[3] = cmul(w[2], w1);
    if constexpr (R > 4) {
        w[4] = cmul(w[2], w[2]);
        w[5] = cmul(w[4], w1);
        w[6] = cmul(w[4], w[2]);
        w[7] = cmul(w[4], w[3]);
    }
    if constexpr (R > 8) {
        w[8] = cmul(w[4], w[4]);
#pragma unroll
        for (int r = 1; r < 8; ++r) w[8 + r] = cmul(w[8], w[r]);
    }
}

// ---------------------------------------------------------------------------
// padded planar shared-memory buffer
// ---------------------------------------------------------------------------
// float2 elements with one pad slot per 16: every Stockham access pattern
// used here (consecutive, stride-R with R = 16, the NS = 16 scatter) maps the
// 16 lanes of each LDS.64/STS.64 wavefront to 16 distinct bank pairs.
__host__ __device__ constexpr int padi(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int padded(int n) { return n + (n >> 4); }

struct SmemPlanes {
    float2* d;
    __device__ __forceinline__ float2 ld(int i) const { return d[padi(i)]; }
    __device__ __forceinline__ void st(int i, float2 v) const { d[padi(i)] = v; }
};

struct LoadPlanes {
    static constexpr bool kPlanes = true;
    SmemPlanes s;
    __device__ __forceinline__ float2 operator()(int i) const { return s.ld(i); }
};
struct StorePlanes {
    static constexpr bool kPlanes = true;
    SmemPlanes s;
    __device__ __forceinline__ void operator()(int i, float2 v) const { s.st(i, v); }
};

// does the functor address the padded smem buffer directly?  Then the pass
// engine hoists the padding math: padi(x + y) == padi(x) + y + y/16 for y a
// multiple of 16, and == padi(x) + y when x is a multiple of 16 and y < 16.
template <class F, class = void>
struct is_planes { static constexpr bool value = false; };
template <class F>
struct is_planes<F, decltype(void(F::kPlanes))> { static constexpr bool value = F::kPlanes; };

// One in-place Stockham (autosort, DIT-twiddle) pass of an N-point FFT with
// radix R, run by NT threads; NS = product of the radices of earlier passes.
// Butterfly j reads x[j + r*N/R], applies W_{NS*R}^{r*(j%NS)}, does an
// R-point DFT and writes x[(j/NS)*NS*R + j%NS + r*NS].
template <int N, int R, int NT>
struct PassShape {
    static constexpr int NB = N / R;
    static_assert(NB % NT == 0 || NT % NB == 0, "butterflies must split evenly over threads");
    static constexpr int BPT = NB >= NT ? NB / NT : 1;
    static constexpr bool PARTIAL = NB < NT;   // threads tid >= NB idle in this pass
};

template <int N, int R, int NT, class Load>
__device__ __forceinline__ void stockham_load(int tid, const Load& load, float2 (&v)[PassShape<N, R, NT>::BPT][R]) {
    constexpr int NB = PassShape<N, R, NT>::NB;
    if (PassShape<N, R, NT>::PARTIAL && tid >= NB) return;
#pragma unroll
    for (int q = 0; q < PassShape<N, R, NT>::BPT; ++q) {
        const int j = tid + q * NT;
        if constexpr (is_planes<Load>::value && NB % 16 == 0) {
            const float2* p = load.s.d + padi(j);
#pragma unroll
            for (int r = 0; r < R; ++r) v[q][r] = p[r * (NB + NB / 16)];
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) v[q][r] = load(j + r * NB);
        }
    }
}

template <int N, int R, int NS, int NT, bool INV, int NBF = PassShape<N, R, NT>::BPT, class Store, class TW>
__device__ __forceinline__ void stockham_compute_store(int tid, const TW& tw, float2 (&v)[NBF][R],
                                                       const Store& store) {
    if (PassShape<N, R, NT>::PARTIAL && tid >= PassShape<N, R, NT>::NB) return;
    constexpr bool kDirect = has_direct<TW>::value && NS > 1 && ((NS == 16 && R == 16) || (NS == 256 && R == 4));
    // when NT is a multiple of NS every butterfly of this thread has the same
    // twiddle index (j % NS == tid % NS): build the chain once, apply to all
    constexpr bool kShared = !kDirect && (NS > 1) && (NT % NS == 0) && (NBF > 1);
    if constexpr (kShared) {
        const float2 w1 = tw.template w<NS * R>(tid % NS);
        float2 wr = w1;
#pragma unroll
        for (int r = 1; r < R; ++r) {
#pragma unroll
            for (int q = 0; q < NBF; ++q) v[q][r] = INV ? cmulc(v[q][r], wr) : cmul(v[q][r], wr);
            if (r + 1 < R) wr = cmul(wr, w1);
        }
    }
#pragma unroll
    for (int q = 0; q < NBF; ++q) {
        const int j = tid + q * NT;
        if constexpr (kDirect) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
                const float2 w = tw.template d<NS, R>(r, j % NS);
                v[q][r] = INV ? cmulc(v[q][r], w) : cmul(v[q][r], w);
            }
        } else if constexpr (NS > 1 && !kShared) {
            // w_r = w1^r by a running product (2 live registers; error <= R ulp)
            const float2 w1 = tw.template w<NS * R>(j % NS);
            float2 wr = w1;
#pragma unroll
            for (int r = 1; r < R; ++r) {
                v[q][r] = INV ? cmulc(v[q][r], wr) : cmul(v[q][r], wr);
                if (r + 1 < R) wr = cmul(wr, w1);
            }
        }
        dft_reg<R, INV>(v[q]);
        const int d0 = (j / NS) * NS * R + (j % NS);
        if constexpr (is_planes<Store>::value && NS % 16 == 0) {
            float2* p = store.s.d + padi(d0);
#pragma unroll
            for (int r = 0; r < R; ++r) p[r * (NS + NS / 16)] = v[q][r];
        } else if constexpr (is_planes<Store>::value && NS == 1 && R <= 16 && 16 % R == 0) {
            float2* p = store.s.d + padi(d0);        // d0 = j*R, R | 16: no pad crossing
#pragma unroll
            for (int r = 0; r < R; ++r) p[r] = v[q][r];
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) store(d0 + r * NS, v[q][r]);
        }
    }
}

// SYNC_IN: barrier between the read and write phases (needed whenever the
// loader reads the same buffer the storer writes).
// SYNC_IN == false means the pass is out of place (loader and storer touch
// different memory): butterflies then stream one at a time (R live values).
struct BlockBarrier {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
// named barrier over the NT threads of one sub-group (id 1..15) of the CTA
struct GroupBarrier {
    int id, nt;
    __device__ __forceinline__ void operator()() const {
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nt) : "memory");
    }
};

template <int N, int R, int NS, int NT, bool INV, bool SYNC_IN, class Load, class Store, class Bar = BlockBarrier,
          class TW = Twiddle>
__device__ __forceinline__ void stockham_pass(int tid, const TW& tw, const Load& load, const Store& store,
                                              const Bar& bar = Bar{}) {
    if constexpr (SYNC_IN) {
        float2 v[PassShape<N, R, NT>::BPT][R];
        stockham_load<N, R, NT>(tid, load, v);
        bar();
        stockham_compute_store<N, R, NS, NT, INV>(tid, tw, v, store);
    } else {
        constexpr int NB = PassShape<N, R, NT>::NB;
        if (PassShape<N, R, NT>::PARTIAL && tid >= NB) return;
#pragma unroll 1
        for (int q = 0; q < PassShape<N, R, NT>::BPT; ++q) {
            float2 v[1][R];
            const int j = tid + q * NT;
            if constexpr (is_planes<Load>::value && NB % 16 == 0) {
                const float2* p = load.s.d + padi(j);
#pragma unroll
                for (int r = 0; r < R; ++r) v[0][r] = p[r * (NB + NB / 16)];
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) v[0][r] = load(j + r * NB);
            }
            stockham_compute_store<N, R, NS, NT, INV, 1>(tid + q * NT, tw, v, store);
        }
    }
}

}  // namespace kk
