// K1 kk_fused: blockwise Kramers-Kronig field reconstruction fused with the
// downshift / mirror and the per-hop carrier sums.
//
// Reference semantics (rxdsp.py `kk_reconstruct` :184-244, `_hilbert_multiplier`
// :170-181, `_run_downshift` :690-696 -> sigcore `frequency_shift` :286-299,
// and the segment sums of `_run_carrier` :685-687):
//   per hop (512) mean m; dead if m <= 0; safe = max(x, 1e-12|m|) (1 if dead)
//   amp = sqrt(safe), u = 0.5 ln(safe)
//   block j = [u(hop j-1), u(hop j)] (1024): phi = irfft(rfft(block) * M)[512:]
//   M[k] = (-j)^(k+1) (the -j sgn multiplier delayed by 256), M[0] = M[512] = 0
//   field[g] = amp[g-256] exp(j phi[g]), 0 where the delayed hop is dead
//   z[g] = conj(field[g] * exp(-2 pi i (p g mod q)/q))          (mirror on)
//
// B200 mapping: one 64-thread group per PAIR of blocks (global even hop 2p
// and 2p+1) packed as the real and imaginary parts of one complex 1024-point
// FFT (the multiplier is Hermitian, so the two real results separate
// exactly).  A 256-thread CTA runs 4 pairs = 8 output hops and stages the 9
// hops of u/amp it needs once in shared memory.  FFT = Stockham radix
// 16x16x4 in padded float2 smem; the inverse FFT's last pass writes the field
// straight to HBM (coalesced) with the rotation/mirror and the hop sums fused.
#include <algorithm>
#include <type_traits>

// packed FP32 complex arithmetic (kk_common.cuh; measured 7.13 -> 6.63 ms)
#ifndef KK_K1_PACKED_ADD
#define KK_K1_PACKED_ADD 1
#endif
#ifndef KK_K1_PACKED_MUL
#define KK_K1_PACKED_MUL 1
#endif
#define KK_PACKED_ADD KK_K1_PACKED_ADD
#define KK_PACKED_MUL KK_K1_PACKED_MUL
#ifdef KK_K1_PACKED_CONST
#define KK_PACKED_CONST KK_K1_PACKED_CONST
#endif
#include "kk_common.cuh"
#include "kk_internal.h"

namespace kk {

constexpr int kHop = 512;
constexpr int kN1 = 1024;
constexpr int kPairsPerCta = 4;
constexpr int kGroupThreads = 64;
constexpr int kK1Threads = kPairsPerCta * kGroupThreads;      // 256
constexpr int kStageHops = 2 * kPairsPerCta + 1;              // 9
constexpr int kPlane1 = padded(kN1);                          // 1088 float2

// K1 only indexes the W_256 / W_1024 twiddle tables: stage that prefix
constexpr int kK1TwEntries = tw_offset(2048);

struct K1Smem {
    float u[kStageHops * kHop];          // 0.5 ln(safe); amp = exp(u) is recomputed
    float ahist[kHop / 2];               // amp of the state hop (initial state: zeros)
    float2 buf[kPairsPerCta][kPlane1];
    float2 tw[kK1TwEntries];
    float2 red[kK1Threads / 32][2];
    double h0part[kK1Threads / 32];
    int dead[kStageHops];
    uint8_t dead_hist[kHop / 2];   // per-sample dead flags of hop -1 (state)
    unsigned int clamped;
};

// x reduced to [-pi, pi] (exact multiple-of-2pi removal for |x| << 2^20)
__device__ __forceinline__ float reduce_2pi(float x) {
    const float k = rintf(x * 0.15915494309189535f);
    return fmaf(-k, 6.28318548202514648f, fmaf(-k, -1.7484555314695172e-7f, x));
}

// Packed 12-bit wire format (KK_DTYPE_P12): two 12-bit two's-complement ADC
// codes c (12-bit converter, frontend.py:82-118; odd half-LSB code h = 2c+1)
// per 3 bytes, little-endian: byte0 = c0[7:0], byte1 = c0[11:8] | c1[3:0] << 4,
// byte2 = c1[11:4].  1.5 B/sample on the wire instead of int16's 2.
struct P12 {};
template <typename TIn> struct InElem { using T = TIn; };
template <> struct InElem<P12> { using T = uint8_t; };

// raw input value at sample i: the code h (int16, P12) or the sample (f32/f64)
template <typename TIn>
__device__ __forceinline__ auto raw_at(const typename InElem<TIn>::T* p, int64_t i) {
    if constexpr (std::is_same<TIn, P12>::value) {
        const int64_t b = 3 * (i >> 1);                       // first byte of the pair
        const uint32_t* w = reinterpret_cast<const uint32_t*>(p + (b & ~int64_t(3)));
        // the second word only when the 3 bytes straddle it ((b & 3) >= 2): every
        // word read then overlaps the data, so nothing past its end is touched
        const uint32_t hi = (b & 2) ? __ldg(w + 1) : 0u;
        const uint32_t v = __funnelshift_r(__ldg(w), hi, static_cast<unsigned>(b & 3) * 8u);
        const int c = (i & 1) ? (static_cast<int>(v << 8) >> 20) : (static_cast<int>(v << 20) >> 20);
        return static_cast<int16_t>(2 * c + 1);
    } else {
        return p[i];
    }
}
template <typename TIn>
__device__ __forceinline__ float load_in(const typename InElem<TIn>::T* p, int64_t i, float scale) {
    if constexpr (std::is_same<TIn, double>::value)
        return static_cast<float>(p[i] * static_cast<double>(scale));
    else
        return static_cast<float>(raw_at<TIn>(p, i)) * scale;
}

// Hilbert multiplier on the full 1024-bin spectrum (Hermitian extension of
// the rfft multiplier): k in [1,511]: (-j)^(k+1); k in [513,1023]:
// conj((-j)^(1025-k)); 0 at DC and Nyquist.
// Branch-free (the lanes of a pass hold different k: a switch diverged).
// (-j)^e z for e = 0..3: (x, y), (y, -x), (-x, -y), (-y, x); the conjugated
// multiplier (+j)^e is (-j)^{-e}.
__device__ __forceinline__ float2 apply_mult(int k, float2 z) {
    const int e = k < 512 ? ((k + 1) & 3) : ((k - 1025) & 3);     // (1025-k) conj -> -(1025-k)
    const bool swap = e & 1;
    const float a = swap ? z.y : z.x, b = swap ? z.x : z.y;
    const float zero = (k & 511) == 0 ? 0.f : 1.f;                  // DC and Nyquist
    const float sr = (e & 2) ? -zero : zero;
    const float si = ((e + 1) & 2) ? -zero : zero;
    return make_float2(a * sr, b * si);
}

// PRECISE: correctly-rounded logf/expf/sincosf instead of the SFU
// approximations (the functional kk_reconstruct API, whose reference tests
// demand e.g. a constant current reconstructed to 1e-8 absolute,
// test_rxdsp.py:83-89); the streaming pipeline uses the fast variant.
// The fast forms are __logf / __expf without their subnormal fix-ups (the
// .ftz MUFU forms; 3 instructions less each, same results for normal
// operands and results): log's argument is >= the clamp threshold or 1, and
// an amplitude below 2^-126 flushes to 0 (an absolute difference < 1.2e-38).
__device__ __forceinline__ float log_ftz(float x) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r * 0.693147180559945309f;
}
__device__ __forceinline__ float exp_ftz(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x * 1.442695040888963407f));
    return r;
}
#ifndef KK_K1_FTZ
#define KK_K1_FTZ 1
#endif
#ifndef KK_K1_EPI_PACKED      // epilogue phase scaling / amplitude products as packed pairs
#define KK_K1_EPI_PACKED 1
#endif
template <bool PRECISE>
__device__ __forceinline__ float k1_log(float x) { return PRECISE ? logf(x) : (KK_K1_FTZ ? log_ftz(x) : __logf(x)); }
template <bool PRECISE>
__device__ __forceinline__ float k1_exp(float x) { return PRECISE ? expf(x) : (KK_K1_FTZ ? exp_ftz(x) : __expf(x)); }
// sin/cos of a phase; the fast form first reduces to [-pi, pi]
template <bool PRECISE>
__device__ __forceinline__ void k1_sincos(float x, float* s, float* c) {
    if (PRECISE) sincosf(x, s, c);
    else __sincosf(reduce_2pi(x), s, c);
}

#ifndef KK_K1_MINB
#define KK_K1_MINB 4
#endif
template <typename TIn, bool PRECISE>
__device__ __forceinline__ void
k1_body(const int bx, const typename InElem<TIn>::T* __restrict__ in, float in_scale, float clamp_rel, int64_t n_hops,
        const float* __restrict__ st_u, const float* __restrict__ st_a,
        const uint8_t* __restrict__ st_dead,
        float* __restrict__ new_u, float* __restrict__ new_a, uint8_t* __restrict__ new_dead,
        float2* __restrict__ out, float2* __restrict__ hop_sum, uint8_t* __restrict__ hop_dead,
        unsigned long long* __restrict__ clamped_total,
        int64_t n0_global, int rot_p, int rot_q, const float2* __restrict__ rot_tab,
        unsigned long long rot_step, int mirror, const float2* __restrict__ tw_g)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K1Smem& S = *reinterpret_cast<K1Smem*>(smem_raw);
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int64_t hop0 = int64_t(bx) * (2 * kPairsPerCta) - 1;   // chunk hop of stage hop 0

    for (int i = tid; i < kK1TwEntries; i += kK1Threads) S.tw[i] = tw_g[i];
    if (tid == 0) S.clamped = 0;
    __syncthreads();

    // ---- stage 9 hops: means, dead flags, clamp, u = 0.5 ln(safe) ----
    // Warp w stages hop w + 1 whole; hop 0 (the previous CTA's last hop,
    // needed for the first block's history half) is shared by all 8 warps,
    // 64 samples each, so no warp stages two hops.  Sums of int16 codes are
    // exact integers.
    using Acc = typename std::conditional<std::is_same<TIn, int16_t>::value || std::is_same<TIn, P12>::value, int,
                                          double>::type;
    auto hop_params = [&](int64_t h, double sum, int& dead, float& thr) {
        // mean = sum * scale / 512 (exact for int16 codes: integer sum)
        const double mean = sum * static_cast<double>(in_scale) / kHop;
        dead = !(mean > 0.0) ? 1 : 0;
        thr = dead ? 1.0f : static_cast<float>(static_cast<double>(clamp_rel) * fabs(mean));
    };
    auto stage_val = [&](float xin, int dead, float thr, unsigned& ncl) {
        const float x = xin * in_scale;
        float sv;
        if (dead) {
            sv = 1.0f;
        } else {
            ncl += (x < thr) ? 1u : 0u;
            sv = fmaxf(x, thr);
        }
        return 0.5f * k1_log<PRECISE>(sv);
    };
    const int64_t h0 = hop0;                       // stage hop 0
    const bool h0_real = h0 >= 0 && h0 < n_hops;
    float x0v[2];
    {
        // (a) own hop L = warp + 1, (b) this warp's 64 samples of hop 0
        const int L = warp + 1;
        const int64_t h = hop0 + L;
        float* u = S.u + L * kHop;
        if (h >= n_hops) {  // dummy partner beyond the last real hop
            for (int i = lane; i < kHop; i += 32) u[i] = 0.f;
            if (lane == 0) S.dead[L] = 1;
        } else {
            float xv[kHop / 32];
            Acc sum = 0;
#pragma unroll
            for (int i = 0; i < kHop / 32; ++i) {
                const auto r = raw_at<TIn>(in, h * kHop + lane + 32 * i);
                xv[i] = static_cast<float>(r);
                sum += static_cast<Acc>(r);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            int dead;
            float thr;
            hop_params(h, static_cast<double>(sum), dead, thr);
            unsigned int ncl = 0;
#pragma unroll
            for (int i = 0; i < kHop / 32; ++i) u[lane + 32 * i] = stage_val(xv[i], dead, thr, ncl);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ncl += __shfl_xor_sync(0xffffffffu, ncl, o);
            if (lane == 0) {
                S.dead[L] = dead;
                if (ncl) atomicAdd(&S.clamped, ncl);
                hop_dead[h] = static_cast<uint8_t>(dead);
            }
        }
        Acc p0 = 0;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int i = warp * 64 + lane + 32 * e;
            x0v[e] = 0.f;
            if (h0_real) {
                const auto r = raw_at<TIn>(in, h0 * kHop + i);
                x0v[e] = static_cast<float>(r);
                p0 += static_cast<Acc>(r);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) p0 += __shfl_xor_sync(0xffffffffu, p0, o);
        if (lane == 0) S.h0part[warp] = static_cast<double>(p0);
    }
    __syncthreads();
    {
        float* u = S.u;
        if (h0 < 0) {   // previous-chunk state (rxdsp.py:208-213 initial zeros)
            for (int i = tid; i < kHop; i += kK1Threads) u[i] = st_u[i];
            for (int i = tid; i < kHop / 2; i += kK1Threads) {
                S.ahist[i] = st_a[i];
                S.dead_hist[i] = st_dead[i];
            }
            if (tid == 0) S.dead[0] = 0;
        } else if (!h0_real) {
            for (int i = tid; i < kHop; i += kK1Threads) u[i] = 0.f;
            if (tid == 0) S.dead[0] = 1;
        } else {
            double sum = 0.0;
            for (int w = 0; w < kK1Threads / 32; ++w) sum += S.h0part[w];   // fixed order
            int dead;
            float thr;
            hop_params(h0, sum, dead, thr);
            unsigned int ncl = 0;   // stage hop 0 is counted by the previous CTA
#pragma unroll
            for (int e = 0; e < 2; ++e) u[warp * 64 + lane + 32 * e] = stage_val(x0v[e], dead, thr, ncl);
            if (tid == 0) S.dead[0] = dead;
        }
    }
    __syncthreads();

    // ---- per pair: forward FFT1024 of u_a + j u_b, multiplier, inverse ----
    const int g = tid / kGroupThreads;
    const int gt = tid % kGroupThreads;
    const int64_t pair = int64_t(bx) * kPairsPerCta + g;
    const int64_t hop_a = 2 * pair;          // output hop of the real-part block
    const bool active = hop_a < n_hops;
#ifndef KK_K1_DIRECT_TW
#define KK_K1_DIRECT_TW 0   // per-pass tables: 4 % fewer instructions but 120 B of spills at the 64-register cap (measured slower)
#endif
#if KK_K1_DIRECT_TW
    DirectTwiddle tw;
    tw.t = S.tw;
    tw.p = tw_g + kTwEntries;
#else
    const Twiddle tw{S.tw};
#endif
    SmemPlanes P{S.buf[g]};
    const float* ua = S.u + (2 * g) * kHop;          // block a: stage hops 2g, 2g+1
    const float* ub = S.u + (2 * g + 1) * kHop;      // block b: stage hops 2g+1, 2g+2

    // The Hilbert multiplier is 0 at DC (M[0] = 0), so a constant shift of a
    // block's u leaves phi unchanged: subtract u at the first sample of stage
    // hop 2g+1 (common to both blocks of the pair).  This keeps the transform
    // at the block's AC level (a constant current gives phi == 0 exactly).
    const float u_ref = S.u[(2 * g + 1) * kHop];
    auto ld_u = [&](int i) { return make_float2(ua[i] - u_ref, ub[i] - u_ref); };
    // the four pairs of the CTA are independent: each 64-thread group syncs
    // on its own named barrier between passes
    const GroupBarrier gb{g + 1, kGroupThreads};
    stockham_pass<kN1, 16, 1, kGroupThreads, false, false>(gt, tw, ld_u, StorePlanes{P});
    gb();
    stockham_pass<kN1, 16, 16, kGroupThreads, false, true>(gt, tw, LoadPlanes{P}, StorePlanes{P}, gb);
    gb();
    stockham_pass<kN1, 4, 256, kGroupThreads, false, true>(gt, tw, LoadPlanes{P}, StorePlanes{P}, gb);
    gb();
    auto ld_m = [&](int k) { return apply_mult(k, P.ld(k)); };
    stockham_pass<kN1, 16, 1, kGroupThreads, true, true>(gt, tw, ld_m, StorePlanes{P}, gb);
    gb();
    stockham_pass<kN1, 16, 16, kGroupThreads, true, true>(gt, tw, LoadPlanes{P}, StorePlanes{P}, gb);
    gb();

    // last inverse pass: outputs n = j + 256 r; n >= 512 are the new hop
    float2 acc_a = make_float2(0.f, 0.f), acc_b = make_float2(0.f, 0.f);
    const float* ua_d = S.u + (2 * g) * kHop + kHop / 2;      // u at (new hop pos - 256), block a
    const float* ub_d = S.u + (2 * g + 1) * kHop + kHop / 2;  // block b
    const int dead_a0 = S.dead[2 * g], dead_a1 = S.dead[2 * g + 1], dead_b1 = S.dead[2 * g + 2];
    const bool hist = (hop0 + 2 * g) < 0;   // stage hop 2g is the state hop
    // rotation index (rot_p * g mod rot_q) of the pair's first output sample
    unsigned rot_base = 0;
    const float inv_q = rot_q > 0 ? 1.0f / static_cast<float>(rot_q) : 0.f;
    const float two_pi_over_q = rot_q > 0 ? 6.283185307179586f / static_cast<float>(rot_q) : 0.f;
    // (32-bit arithmetic: n0_global arrives reduced mod q, hop_a < 2^31)
    // (one integer modulo for the unbounded hop index; the small arguments,
    // all < 2^25, reduce through the float reciprocal)
    if (rot_q > 0 && active) {
        const unsigned Q = static_cast<unsigned>(rot_q);
        const unsigned h = static_cast<unsigned>(hop_a) % Q;
        rot_base = fmod_u(static_cast<unsigned>(n0_global) + h * fmod_u(512u, Q, inv_q), Q, inv_q);
    }
    float2 rot_cache = make_float2(1.f, 0.f), r256 = rot_cache, r512 = rot_cache;
    const bool rotate = rot_q > 0 || rot_step != 0ull;
    if (rot_q > 0) {
        const unsigned Q = static_cast<unsigned>(rot_q), Pp = static_cast<unsigned>(rot_p);
        r256 = __ldg(rot_tab + fmod_u(256u * Pp, Q, inv_q));     // exp(-2 pi i (256 p mod q) / q)
        r512 = __ldg(rot_tab + fmod_u(512u * Pp, Q, inv_q));
    } else if (rot_step) {
        r256 = PRECISE ? rot_phase_precise(256ull * rot_step) : rot_phase_fast(256ull * rot_step);
        r512 = PRECISE ? rot_phase_precise(512ull * rot_step) : rot_phase_fast(512ull * rot_step);
    }
    const bool has_b = (hop_a + 1) < n_hops;
    auto st_out = [&](int n, float2 v) {
        if (n < kHop) return;
        const int i = n - kHop;
        // delayed dead flags: position i-256 of the new hop lies in the
        // previous hop when i < 256
        bool da = (i < kHop / 2) ? (hist ? (S.dead_hist[i] != 0) : (dead_a0 != 0)) : (dead_a1 != 0);
        bool db = (i < kHop / 2) ? (dead_a1 != 0) : (dead_b1 != 0);
        // phases (the fast sin/cos reduces to [-pi, pi]: abs err ~1e-6)
        const float amp_a = (hist && i < kHop / 2) ? S.ahist[i] : k1_exp<PRECISE>(ua_d[i]);
        const float amp_b = k1_exp<PRECISE>(ub_d[i]);
        float sa, ca, sb, cb;
#if KK_K1_EPI_PACKED
        const float2 ph = __fmul2_rn(v, make_float2(1.0f / 1024.0f, 1.0f / 1024.0f));
        k1_sincos<PRECISE>(ph.x, &sa, &ca);
        k1_sincos<PRECISE>(ph.y, &sb, &cb);
        float2 fa = da ? make_float2(0.f, 0.f) : __fmul2_rn(make_float2(amp_a, amp_a), make_float2(ca, sa));
        float2 fb = db ? make_float2(0.f, 0.f) : __fmul2_rn(make_float2(amp_b, amp_b), make_float2(cb, sb));
#else
        k1_sincos<PRECISE>(v.x * (1.0f / 1024.0f), &sa, &ca);
        k1_sincos<PRECISE>(v.y * (1.0f / 1024.0f), &sb, &cb);
        float2 fa = da ? make_float2(0.f, 0.f) : make_float2(amp_a * ca, amp_a * sa);
        float2 fb = db ? make_float2(0.f, 0.f) : make_float2(amp_b * cb, amp_b * sb);
#endif
        if (!active) return;
        acc_a = cadd(acc_a, fa);
        const int64_t pa = hop_a * kHop + i;           // chunk positions
        const int64_t pb = pa + kHop;
        float2 za = fa, zb = fb;
        if (rotate) {
            // field * exp(-2 pi i a/q) (or the general tone's phase).  A
            // butterfly's outputs i = j and j + 256 of hops a and b are 256 /
            // 512 samples apart: one sincos for the first, exact constant
            // rotations (table entries) for the others
            if (i < kHop / 2) {
                if (rot_q > 0) {
                    const unsigned Q = static_cast<unsigned>(rot_q), P = static_cast<unsigned>(rot_p);
                    const int ia = static_cast<int>(fmod_u((rot_base + i) * P, Q, inv_q));
                    float sr, cr;
                    k1_sincos<PRECISE>(-two_pi_over_q * static_cast<float>(ia), &sr, &cr);
                    rot_cache = make_float2(cr, sr);
                } else {
                    const unsigned long long ph = static_cast<unsigned long long>(n0_global + pa) * rot_step;
                    rot_cache = PRECISE ? rot_phase_precise(ph) : rot_phase_fast(ph);
                }
            } else {
                rot_cache = cmul(rot_cache, r256);
            }
            za = cmul(fa, rot_cache);
            zb = cmul(fb, cmul(rot_cache, r512));
        }
        if (mirror) { za = cconj(za); zb = cconj(zb); }
        out[pa] = za;
        if (has_b) {
            acc_b = cadd(acc_b, fb);
            out[pb] = zb;
        }
    };
    stockham_pass<kN1, 4, 256, kGroupThreads, true, true>(gt, tw, LoadPlanes{P}, st_out, gb);

    // ---- deterministic per-hop field sums (fixed shuffle tree) ----
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc_a.x += __shfl_xor_sync(0xffffffffu, acc_a.x, o);
        acc_a.y += __shfl_xor_sync(0xffffffffu, acc_a.y, o);
        acc_b.x += __shfl_xor_sync(0xffffffffu, acc_b.x, o);
        acc_b.y += __shfl_xor_sync(0xffffffffu, acc_b.y, o);
    }
    if (lane == 0) { S.red[warp][0] = acc_a; S.red[warp][1] = acc_b; }
    __syncthreads();
    if (gt == 0 && active) {
        const int w0 = warp;   // first warp of the group (gt == 0)
        hop_sum[hop_a] = cadd(S.red[w0][0], S.red[w0 + 1][0]);
        if (hop_a + 1 < n_hops) hop_sum[hop_a + 1] = cadd(S.red[w0][1], S.red[w0 + 1][1]);
    }
    if (tid == 0 && S.clamped) atomicAdd(clamped_total, static_cast<unsigned long long>(S.clamped));

    // ---- state for the next chunk: u, amp, dead of the last real hop ----
    const int64_t last = n_hops - 1;
    const int64_t Ll = last - hop0;
    if (Ll >= 1 && Ll < kStageHops) {
        for (int i = tid; i < kHop; i += kK1Threads) new_u[i] = S.u[Ll * kHop + i];
        for (int i = tid; i < kHop / 2; i += kK1Threads) {
            new_a[i] = (hop0 + Ll < 0) ? S.ahist[i] : k1_exp<PRECISE>(S.u[Ll * kHop + kHop / 2 + i]);
            new_dead[i] = static_cast<uint8_t>(S.dead[Ll]);
        }
    }
}

template <typename TIn, bool PRECISE>
__global__ void __launch_bounds__(kK1Threads, KK_K1_MINB)
kk_pairs_kernel(const typename InElem<TIn>::T* __restrict__ in, float in_scale, float clamp_rel, int64_t n_hops,
                const float* __restrict__ st_u, const float* __restrict__ st_a,
                const uint8_t* __restrict__ st_dead,
                float* __restrict__ new_u, float* __restrict__ new_a, uint8_t* __restrict__ new_dead,
                float2* __restrict__ out, float2* __restrict__ hop_sum, uint8_t* __restrict__ hop_dead,
                unsigned long long* __restrict__ clamped_total,
                int64_t n0_global, int rot_p, int rot_q, const float2* __restrict__ rot_tab,
                unsigned long long rot_step, int mirror, const float2* __restrict__ tw_g) {
    k1_body<TIn, PRECISE>(blockIdx.x, in, in_scale, clamp_rel, n_hops, st_u, st_a, st_dead, new_u, new_a, new_dead, out,
                          hop_sum, hop_dead, clamped_total, n0_global, rot_p, rot_q, rot_tab, rot_step, mirror, tw_g);
}

// Batched K1 (independent streams -- sweep points -- in one launch, SURVEY
// §8(f)3): blockIdx.y selects the stream's job, CTAs beyond its own grid
// return at once.
constexpr int kK1BatchMax = 32;
struct K1Batch {
    kk_k1_job job[kK1BatchMax];
};

template <typename TIn, bool PRECISE>
__global__ void __launch_bounds__(kK1Threads, KK_K1_MINB)
kk_pairs_batch_kernel(const __grid_constant__ K1Batch b, const float2* __restrict__ tw_g) {
    const kk_k1_job& j = b.job[blockIdx.y];
    const int64_t ctas = ((j.n_hops + 1) / 2 + kPairsPerCta - 1) / kPairsPerCta;
    if (blockIdx.x >= ctas) return;
    const int q = j.rot_q;
    // rational tones need the stream index modulo q only; general tones the index itself
    const int64_t n0m = q > 0 ? ((j.n0_global % q) + q) % q : j.n0_global;
    k1_body<TIn, PRECISE>(blockIdx.x, static_cast<const typename InElem<TIn>::T*>(j.in), j.in_scale, j.clamp_rel,
                          j.n_hops, j.st_u, j.st_a, j.st_dead, j.new_u, j.new_a, j.new_dead,
                          static_cast<float2*>(j.out), static_cast<float2*>(j.hop_sum), j.hop_dead, j.clamped, n0m,
                          j.rot_p, q, static_cast<const float2*>(j.rot_tab), j.rot_step, j.mirror, tw_g);
}

template <typename TIn, bool PRECISE>
static int launch_k1_batch(const kk_k1_job* jobs, int n, cudaStream_t s) {
    const float2* tw = twiddle_table_device();
    if (!tw) return KK_ERR_CUDA;
    const size_t smem = sizeof(K1Smem);
    if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(kk_pairs_batch_kernel<TIn, PRECISE>), smem,
                                  "K1 batch smem attr"))
        return rc;
    for (int a = 0; a < n; a += kK1BatchMax) {
        K1Batch b;
        const int m = std::min(kK1BatchMax, n - a);
        int64_t gx = 0;
        for (int i = 0; i < m; ++i) {
            b.job[i] = jobs[a + i];
            if (b.job[i].n_hops >= (int64_t(1) << 31)) return set_error(KK_ERR_PARAM, "n_hops must be < 2^31 per job");
            gx = std::max<int64_t>(gx, ((b.job[i].n_hops + 1) / 2 + kPairsPerCta - 1) / kPairsPerCta);
        }
        if (gx == 0) continue;
        kk_pairs_batch_kernel<TIn, PRECISE><<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(m)), kK1Threads,
                                                smem, s>>>(b, tw);
        if (int rc = check_launch("kk_pairs_batch_kernel")) return rc;
    }
    return KK_OK;
}

template <typename TIn, bool PRECISE>
static int launch_k1(const void* in, float in_scale, float clamp_rel, int64_t n_hops, const float* st_u, const float* st_a,
                     const uint8_t* st_dead, float* new_u, float* new_a, uint8_t* new_dead, float2* out,
                     float2* hop_sum, uint8_t* hop_dead, unsigned long long* clamped, int64_t n0,
                     int rot_p, int rot_q, const float2* rot_tab, unsigned long long rot_step, int mirror,
                     cudaStream_t s) {
    const float2* tw = twiddle_table_device();
    if (!tw) return KK_ERR_CUDA;
    const size_t smem = sizeof(K1Smem);
    if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(kk_pairs_kernel<TIn, PRECISE>), smem, "K1 smem attr"))
        return rc;
    if (n_hops >= (int64_t(1) << 31)) return set_error(KK_ERR_PARAM, "n_hops must be < 2^31 per call");
    const int64_t pairs = (n_hops + 1) / 2;
    const int64_t grid = (pairs + kPairsPerCta - 1) / kPairsPerCta;
    // a rational tone needs the stream index modulo its period only
    const int64_t n0m = rot_q > 0 ? ((n0 % rot_q) + rot_q) % rot_q : n0;
    kk_pairs_kernel<TIn, PRECISE><<<static_cast<unsigned>(grid), kK1Threads, smem, s>>>(
        static_cast<const typename InElem<TIn>::T*>(in), in_scale, clamp_rel, n_hops, st_u, st_a, st_dead, new_u, new_a,
        new_dead, out,
        hop_sum, hop_dead, clamped, n0m, rot_p, rot_q, rot_tab, rot_step, mirror, tw);
    return check_launch("kk_pairs_kernel");
}

}  // namespace kk

extern "C" int kk_reconstruct_pairs(int in_dtype, const void* in, float in_scale, float clamp_rel, int64_t n_hops,
                                    const float* st_u, const float* st_a, const uint8_t* st_dead,
                                    float* new_u, float* new_a, uint8_t* new_dead, void* out,
                                    void* hop_sum, uint8_t* hop_dead, unsigned long long* clamped,
                                    int64_t n0_global, int rot_p, int rot_q, const void* rot_tab,
                                    unsigned long long rot_step, int mirror, void* stream) {
    using namespace kk;
    clear_error();
    if (n_hops <= 0) return set_error(KK_ERR_PARAM, "n_hops must be positive");
    if (rot_q > 0 && !rot_tab) return set_error(KK_ERR_PARAM, "rotation table missing");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    float2* o = static_cast<float2*>(out);
    float2* hs = static_cast<float2*>(hop_sum);
    const float2* rt = static_cast<const float2*>(rot_tab);
    const bool precise = (in_dtype & KK_DTYPE_PRECISE) != 0;
#define KK_LAUNCH_K1(T, PR)                                                                                    \
    return launch_k1<T, PR>(in, in_scale, clamp_rel, n_hops, st_u, st_a, st_dead, new_u, new_a, new_dead, o, hs, \
                            hop_dead, clamped, n0_global, rot_p, rot_q, rt, rot_step, mirror, s)
    switch (in_dtype & ~KK_DTYPE_PRECISE) {
        case KK_DTYPE_I16:
            if (precise) KK_LAUNCH_K1(int16_t, true);
            KK_LAUNCH_K1(int16_t, false);
        case KK_DTYPE_F32:
            if (precise) KK_LAUNCH_K1(float, true);
            KK_LAUNCH_K1(float, false);
        case KK_DTYPE_F64:
            if (precise) KK_LAUNCH_K1(double, true);
            KK_LAUNCH_K1(double, false);
        case KK_DTYPE_P12:
            if (reinterpret_cast<uintptr_t>(in) & 3) return set_error(KK_ERR_PARAM, "packed 12-bit input must be 4-byte aligned");
            if (precise) KK_LAUNCH_K1(P12, true);
            KK_LAUNCH_K1(P12, false);
        default:
            return set_error(KK_ERR_PARAM, "unsupported input dtype");
    }
#undef KK_LAUNCH_K1
}

// ---------------------------------------------------------------------------
// packed 12-bit -> int16 odd half-LSB codes (the flush remainder of a packed
// stream, which needs exact zero padding, and general conversion)
// ---------------------------------------------------------------------------
namespace kk {
__global__ void unpack12_kernel(const uint8_t* __restrict__ in, int64_t n, int16_t* __restrict__ out) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = 3 * (i >> 1);
        const int lo = in[b + (i & 1)], hi = in[b + 1 + (i & 1)];
        const int c = (i & 1) ? (((hi << 4) | (lo >> 4)) & 0xFFF) : (((hi & 0xF) << 8) | lo);
        out[i] = static_cast<int16_t>(2 * ((c ^ 0x800) - 0x800) + 1);
    }
}
}  // namespace kk

// ---------------------------------------------------------------------------
// Standalone downshift (the functional downshift_dc, rx:247-257 ->
// sigcore.py frequency_shift :286-299), complex128: y[i] = x[i] *
// exp(j theta), theta = ((2 pi df) * n) * (1 / fs) with n = start + i in
// float64 -- numpy evaluates the reference's `2j*pi*df*n / fs` as a complex
// quotient, i.e. times the reciprocal of fs -- and the complex product without
// FMA contraction, as numpy forms it.  (The pipeline's downshift is fused in
// K1.)
// ---------------------------------------------------------------------------
namespace kk {
__global__ void frequency_shift_kernel(const double2* __restrict__ x, double2* __restrict__ y, int64_t n,
                                       double two_pi_df, double inv_fs, int64_t start) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const double th = __dmul_rn(__dmul_rn(two_pi_df, static_cast<double>(start + i)), inv_fs);
        double s, c;
        sincos(th, &s, &c);
        const double2 v = x[i];
        y[i] = make_double2(__dsub_rn(__dmul_rn(v.x, c), __dmul_rn(v.y, s)),
                            __dadd_rn(__dmul_rn(v.x, s), __dmul_rn(v.y, c)));
    }
}
}  // namespace kk

extern "C" int kk_frequency_shift(const void* x, void* y, int64_t n, double two_pi_df, double fs, int64_t start_index,
                                  void* stream) {
    using namespace kk;
    clear_error();
    if (n < 0 || !(fs > 0) || (n > 0 && (!x || !y))) return set_error(KK_ERR_PARAM, "kk_frequency_shift: bad arguments");
    if (n == 0) return KK_OK;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
    frequency_shift_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const double2*>(x), static_cast<double2*>(y), n, two_pi_df, 1.0 / fs, start_index);
    return check_launch("frequency_shift_kernel");
}

extern "C" int kk_unpack12(const uint8_t* in, int64_t n, int16_t* out, void* stream) {
    using namespace kk;
    clear_error();
    if (n <= 0) return KK_OK;
    if (n & 1) return set_error(KK_ERR_PARAM, "packed 12-bit streams hold an even number of samples");
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 32);
    unpack12_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(in, n, out);
    return check_launch("unpack12_kernel");
}

extern "C" int kk_reconstruct_pairs_batch(int in_dtype, const kk_k1_job* jobs, int n_jobs, void* stream) {
    using namespace kk;
    clear_error();
    if (n_jobs <= 0) return KK_OK;
    if (!jobs) return set_error(KK_ERR_PARAM, "jobs missing");
    for (int i = 0; i < n_jobs; ++i) {
        if (jobs[i].n_hops < 0) return set_error(KK_ERR_PARAM, "n_hops must be >= 0");
        if (jobs[i].rot_q > 0 && !jobs[i].rot_tab) return set_error(KK_ERR_PARAM, "rotation table missing");
        if ((in_dtype & ~KK_DTYPE_PRECISE) == KK_DTYPE_P12 && (reinterpret_cast<uintptr_t>(jobs[i].in) & 3))
            return set_error(KK_ERR_PARAM, "packed 12-bit input must be 4-byte aligned");
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool precise = (in_dtype & KK_DTYPE_PRECISE) != 0;
    switch (in_dtype & ~KK_DTYPE_PRECISE) {
        case KK_DTYPE_I16: return precise ? launch_k1_batch<int16_t, true>(jobs, n_jobs, s)
                                          : launch_k1_batch<int16_t, false>(jobs, n_jobs, s);
        case KK_DTYPE_F32: return precise ? launch_k1_batch<float, true>(jobs, n_jobs, s)
                                          : launch_k1_batch<float, false>(jobs, n_jobs, s);
        case KK_DTYPE_F64: return precise ? launch_k1_batch<double, true>(jobs, n_jobs, s)
                                          : launch_k1_batch<double, false>(jobs, n_jobs, s);
        case KK_DTYPE_P12: return precise ? launch_k1_batch<P12, true>(jobs, n_jobs, s)
                                          : launch_k1_batch<P12, false>(jobs, n_jobs, s);
        default: return set_error(KK_ERR_PARAM, "unsupported input dtype");
    }
}
