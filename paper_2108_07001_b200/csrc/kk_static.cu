// K2 static_fused: carrier-mean subtraction + fused static equaliser / CD
// compensation + 2:1 decimation, one 32768-point overlap-save block per CTA.
//
// Reference semantics (rxdsp.py `_run_carrier` :671-688, `_run_static`
// :698-720 == `static_equalize_and_resample` :414-453, `_static_response`
// :401-411):
//   s[g] = z[g] - conj(mean_seg(g) * rot[g])      (carrier removed, mirrored)
//   block b = s[16384(b-1) .. 16384(b+1))          (zeros before the stream)
//   Y = ifft16384( fft32768(block)[kept] * H ) * 0.5 ;  out = Y[8192:]
//   kept = [0, 8192) U [24576, 32768)
//
// B200 mapping (the 256 KB block does not fit one CTA's 227 KB of shared
// memory, so it is never materialised):
//   radix-2 DIF split  a = x0 + x1 -> E = FFT16384(a) = even bins
//                      b = (x0 - x1) W32768^n -> O = FFT16384(b) = odd bins
//   kept bins of E/O are their low and high quarters -> 8192 each
//   A = IFFT8192(E_kept * H_even), B = IFFT8192(O_kept * H_odd)
//   out[r] = (A[r] - W16384^{-r} B[r]) * 0.5/16384
// One 512-thread CTA (16 warps) per block, four-step factorisations whose
// inner transforms are warp-local (kk_warpfft.cuh):
//   FFT16384 = DFT16 over stride 1024 (fused with the HBM loads, carrier
//              subtraction, DIF pre-twiddle; then W16384^{n2 k1}) into 16
//              rows, then one warp_fft1024 per row (warp k1)
//   IFFT8192 = DFT16 over stride 512 of the kept bins x H (then
//              W8192^{-m2 p1}) into 16 rows, then one warp_fft512 per row
// so each transform needs two block barriers instead of one per radix pass.
// Chain 0's A is parked in smem (natural order, padded); chain 1 combines
// out = (A - W16384^{-r} B) * 0.5/16384 in place and the block is written
// to HBM coalesced.
#include <algorithm>

// packed FP32 complex arithmetic (kk_common.cuh), A/B'd per operation:
// adds 11.82 -> 11.79 ms, constant-twiddle multiplies -> 11.51 ms; the
// general multiplies (running twiddle products) measured slower packed
// (both packed: 12.03 ms), so they stay scalar
#ifndef KK_K2_PACKED_ADD
#define KK_K2_PACKED_ADD 1
#endif
#ifndef KK_K2_PACKED_MUL
#define KK_K2_PACKED_MUL 0
#endif
#ifndef KK_K2_PACKED_CONST
#define KK_K2_PACKED_CONST 1
#endif
#define KK_PACKED_ADD KK_K2_PACKED_ADD
#define KK_PACKED_MUL KK_K2_PACKED_MUL
#define KK_PACKED_CONST KK_K2_PACKED_CONST
#ifndef KK_K2_PACKED_NP     // the .NP multiply forms: K1 6.37 -> 6.15 ms, K2 11.51 -> 11.62 (not used here)
#define KK_K2_PACKED_NP 0
#endif
#define KK_PACKED_NP KK_K2_PACKED_NP
#include "kk_common.cuh"
#include "kk_internal.h"
#include "kk_warpfft.cuh"

namespace kk {

constexpr int kNS = 32768;        // static block
constexpr int kHopS = 16384;      // hop / half FFT
constexpr int kNOut = 8192;       // outputs per block
constexpr int kK2Threads = 512;
constexpr int kRowE = 1025;              // FFT16384 rows (16 x 1024, +1 pad)
constexpr int kRowI = 513;               // IFFT8192 rows (16 x 512, +1 pad)
constexpr int kRotMax = 1024;            // rotation-table entries held in smem

struct K2Smem {
    float2 buf[16 * kRowE];              // 131,200 B
    float2 A[padded(kNOut)];             // 69,632 B: chain 0 result / output staging
    float2 tw[kTwEntries];               // 18,368 B
    float2 rot[kRotMax];                 // 8,192 B
};
static_assert(sizeof(K2Smem) <= 232448, "K2 shared memory");

struct K2Params {
    const float2* z;        // KK output stream (conj(field * rot)), z[0] = global index z_index0
    int64_t z_index0;
    int64_t hb0;            // global static hop of the first block of this launch
    int64_t valid_end;      // global index: samples at/after are zero padding
    const float2* seg_mean; // carrier mean per segment, seg_mean[0] = segment seg_index0
    int64_t seg_index0;
    int seg_len;
    int carrier;            // subtract the carrier mean
    int rot_p, rot_q;       // rotation exp(-2 pi i (p g mod q)/q); q == 0 -> rot_step
    const float2* rot_tab;
    unsigned long long rot_step;   // general tone: exp(-2 pi i (g rot_step mod 2^64)/2^64); 0 -> none
    int mirror;
    const float2* h_even;   // H at kept index 2m'  (8192)
    const float2* h_odd;    // H at kept index 2m'+1 (8192)
    float2* out;            // 8192 per block
    int prefetch_ahead;     // CTAs resident at once (SM count)
};

// per-CTA constants for the carrier-removed input of one 32768-sample block
struct BlockIn {
    int64_t base;      // global index of block sample 0 (may be negative: stream start)
    unsigned c0;       // (p * base) mod q
    unsigned rb;       // base mod seg_len (floor)
    int64_t sb;        // floor(base / seg_len) - seg_index0
    float inv_q, inv_seg;
};

__device__ __forceinline__ BlockIn make_block_in(const K2Params& p, int64_t base) {
    BlockIn b;
    b.base = base;
    b.inv_q = p.rot_q > 0 ? 1.0f / static_cast<float>(p.rot_q) : 0.f;
    b.inv_seg = p.seg_len > 0 ? 1.0f / static_cast<float>(p.seg_len) : 0.f;
    if (p.rot_q > 0) {
        int64_t m = base % p.rot_q;
        if (m < 0) m += p.rot_q;
        b.c0 = static_cast<unsigned>((m * p.rot_p) % p.rot_q);
    } else {
        b.c0 = 0;
    }
    if (p.seg_len > 0) {
        int64_t sq = base / p.seg_len;
        int64_t r = base - sq * p.seg_len;
        if (r < 0) { r += p.seg_len; --sq; }
        b.rb = static_cast<unsigned>(r);
        b.sb = sq - p.seg_index0;
    } else {
        b.rb = 0;
        b.sb = 0;
    }
    return b;
}

// carrier-removed static-stage input at block position n (global base + n)
__device__ __forceinline__ float2 static_input(const K2Params& p, const BlockIn& b, const float2* rot_s, int n) {
    const int64_t g = b.base + n;
    if (g < 0 || g >= p.valid_end) return make_float2(0.f, 0.f);
    float2 v = __ldg(p.z + (g - p.z_index0));
    if (p.carrier) {
        unsigned ds;
        fmod_u(b.rb + static_cast<unsigned>(n), static_cast<unsigned>(p.seg_len), b.inv_seg, &ds);
        float2 mr = __ldg(p.seg_mean + (b.sb + ds));
        if (p.rot_q > 0) {
            const unsigned a = fmod_u(b.c0 + static_cast<unsigned>(p.rot_p) * static_cast<unsigned>(n),
                                      static_cast<unsigned>(p.rot_q), b.inv_q);
            const float2 r = (p.rot_q <= kRotMax) ? rot_s[a] : __ldg(p.rot_tab + a);
            mr = cmul(mr, r);
        } else if (p.rot_step) {
            mr = cmul(mr, rot_phase_fast(static_cast<unsigned long long>(g) * p.rot_step));
        }
        if (p.mirror) mr = cconj(mr);
        v = csub(v, mr);
    }
    return v;
}

// ---------------------------------------------------------------------------
// TMEM as a per-thread scratch: chain 0's first pass also forms the odd
// chain's column input b and parks it in tensor memory (256 KB/SM, unused by
// this kernel otherwise); chain 1 reads it back instead of re-reading HBM/L2
// and recomputing the carrier.  Warp w owns TMEM lanes 32 (w % 4) .. +32 and
// columns 64 (w / 4) .. +64: 16 complex per column j, 2 columns per thread.
// ---------------------------------------------------------------------------
constexpr int kTmemCols = 256;

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float2 (&v)[8]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};\n" ::"r"(taddr),
        "f"(v[0].x), "f"(v[0].y), "f"(v[1].x), "f"(v[1].y), "f"(v[2].x), "f"(v[2].y), "f"(v[3].x), "f"(v[3].y),
        "f"(v[4].x), "f"(v[4].y), "f"(v[5].x), "f"(v[5].y), "f"(v[6].x), "f"(v[6].y), "f"(v[7].x), "f"(v[7].y)
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float2 (&v)[8]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];\n"
        : "=f"(v[0].x), "=f"(v[0].y), "=f"(v[1].x), "=f"(v[1].y), "=f"(v[2].x), "=f"(v[2].y), "=f"(v[3].x),
          "=f"(v[3].y), "=f"(v[4].x), "=f"(v[4].y), "=f"(v[5].x), "=f"(v[5].y), "=f"(v[6].x), "=f"(v[6].y),
          "=f"(v[7].x), "=f"(v[7].y)
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// Bulk (TMA-engine) copies global -> shared with mbarrier completion: the
// second column's inputs of chain 0 (x0 and x1 halves, 16 runs of 512
// samples each = 128 KB) are copied by one thread while the first column is
// transformed, instead of 16 per-thread cp.async + 16 __ldg per thread.
#ifndef KK_K2_BULK
#define KK_K2_BULK 1
#endif
#ifndef KK_K2_BULK_X1
#define KK_K2_BULK_X1 0
#endif
__device__ __forceinline__ void mbar_init(uint32_t bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, unsigned parity) {
    asm volatile(
        "{\n.reg .pred p;\nKK_MBAR_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra KK_MBAR_WAIT_%=;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, unsigned bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// Chain 0 column j: v[r] = a(n), and the odd chain's b(n) W32^r parked in
// TMEM at taddr (+16 columns for r >= 8).
template <bool FAST>
__device__ __forceinline__ void k2_load_column_ab(const K2Params& p, const BlockIn& b, const float2* rot_s, int j,
                                                  float2 mA, float2 mB, int bnd, unsigned s1024, unsigned s16384,
                                                  float2 (&v)[16], uint32_t taddr, const float2* x0_s = nullptr,
                                                  const float2* x1_s = nullptr) {
    float2 w[8];
    if constexpr (FAST) {
        const float2* z0 = p.z + (b.base - p.z_index0) + j;
        float2 ca = make_float2(0.f, 0.f), cb = ca, st = make_float2(1.f, 0.f);
        if (p.carrier) {
            const float2 m1 = bnd <= kHopS ? mB : mA;
            float2 c0 = mA, c1 = m1;
            const unsigned Q = static_cast<unsigned>(p.rot_q);
            if (Q) {
                const unsigned a0 = fmod_u(b.c0 + static_cast<unsigned>(p.rot_p) * static_cast<unsigned>(j), Q, b.inv_q);
                unsigned a1 = a0 + s16384;
                a1 -= (a1 >= Q) ? Q : 0u;
                c0 = cmul(c0, rot_s[a0]);
                c1 = cmul(c1, rot_s[a1]);
                st = rot_s[s1024];
            } else if (p.rot_step) {
                const unsigned long long ph0 = static_cast<unsigned long long>(b.base + j) * p.rot_step;
                c0 = cmul(c0, rot_phase_fast(ph0));
                c1 = cmul(c1, rot_phase_fast(ph0 + 16384ull * p.rot_step));
                st = rot_phase_fast(1024ull * p.rot_step);
            }
            ca = cadd(c0, c1);
            cb = csub(c0, c1);
            if (p.mirror) {
                ca = cconj(ca);
                cb = cconj(cb);
                st = cconj(st);
            }
        }
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            // x0 of the second column arrives early in smem (cp.async at chain start)
            const float2 x0 = x0_s ? x0_s[r * kK2Threads] : __ldg(z0 + 1024 * r);
            // x1 staged by the bulk copies: run r at row r of the FFT buffer,
            // right half, +1 slot on odd rows (16 B alignment)
            const float2 x1 = x1_s ? x1_s[r * kRowE + (r & 1)] : __ldg(z0 + kHopS + 1024 * r);
            float2 ua = cadd(x0, x1), ub = csub(x0, x1);
            if (p.carrier) {
                ua = csub(ua, ca);
                ub = csub(ub, cb);
                ca = cmul(ca, st);
                cb = cmul(cb, st);
            }
            v[r] = ua;
            w[r & 7] = tw32<false>(ub, r);
            if ((r & 7) == 7) {
                tmem_st16(taddr + (r >> 3) * 16, w);
                tmem_wait_st();
            }
        }
    } else {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int n = j + 1024 * r;
            const float2 x0 = static_input(p, b, rot_s, n), x1 = static_input(p, b, rot_s, kHopS + n);
            v[r] = cadd(x0, x1);
            w[r & 7] = tw32<false>(csub(x0, x1), r);
            if ((r & 7) == 7) {
                tmem_st16(taddr + (r >> 3) * 16, w);
                tmem_wait_st();
            }
        }
    }
}

template <bool FAST>
__device__ __forceinline__ void k2_body(const int bx, const int64_t grid_x, const K2Params& p,
                                        const float2* __restrict__ tw_g) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K2Smem& S = *reinterpret_cast<K2Smem*>(smem_raw);
    const int tid = threadIdx.x;
    // twiddle + rotation tables (26 KB from L2): every load issued before
    // any store, so the CTA pays one latency instead of one per loop trip
    {
        constexpr int kTw4 = kTwEntries / 2;                      // float4 = 2 entries
        static_assert(kTwEntries % 2 == 0, "twiddle table");
        constexpr int kPer = (kTw4 + kK2Threads - 1) / kK2Threads;
        const float4* g4 = reinterpret_cast<const float4*>(tw_g);
        float4* s4 = reinterpret_cast<float4*>(S.tw);
        float4 tv[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int i = tid + k * kK2Threads;
            tv[k] = i < kTw4 ? __ldg(g4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float2 rv[(kRotMax + kK2Threads - 1) / kK2Threads];
        const bool rot = p.carrier && p.rot_q > 0 && p.rot_q <= kRotMax;
#pragma unroll
        for (int k = 0; k < (kRotMax + kK2Threads - 1) / kK2Threads; ++k) {
            const int i = tid + k * kK2Threads;
            rv[k] = (rot && i < p.rot_q) ? __ldg(p.rot_tab + i) : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int i = tid + k * kK2Threads;
            if (i < kTw4) s4[i] = tv[k];
        }
#pragma unroll
        for (int k = 0; k < (kRotMax + kK2Threads - 1) / kK2Threads; ++k) {
            const int i = tid + k * kK2Threads;
            if (rot && i < p.rot_q) S.rot[i] = rv[k];
        }
    }
    __syncthreads();

    const Twiddle tw{S.tw};
    const SmemPlanes P{S.buf};
    const int64_t hb = p.hb0 + bx;
    // L2 prefetch of the input of the block this SM most likely runs next
    // (one CTA per SM, CTAs dispatched in index order -> this block + #SMs):
    // pass 1 of both chains then reads L2 instead of stalling on HBM latency
    // with only 16 warps per SM (measured: 20.8 -> 18.3 ms per 2^30 samples;
    // a persistent-CTA variant with the exact next block was slower)
    if (FAST && tid < 16) {
        const int64_t nb = static_cast<int64_t>(bx) + p.prefetch_ahead;
        if (nb < grid_x) {
            const int64_t g0 = (p.hb0 + nb - 1) * kHopS - p.z_index0;   // first sample of that block
            const char* a0 = reinterpret_cast<const char*>(p.z + g0) + tid * (kNS * 8 / 16);
            const uintptr_t al = reinterpret_cast<uintptr_t>(a0) & ~uintptr_t(15);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(al), "r"(kNS * 8 / 16) : "memory");
        }
    }
    const int64_t base = (hb - 1) * kHopS;   // global index of block sample 0
    const BlockIn bi = make_block_in(p, base);
    float2 mA = make_float2(0.f, 0.f), mB = mA;
    int bnd = kNS;
    unsigned s1024 = 0, s16384 = 0;
    if (FAST && p.carrier) {
        mA = __ldg(p.seg_mean + bi.sb);
        bnd = p.seg_len - static_cast<int>(bi.rb);
        if (bnd < kNS) mB = __ldg(p.seg_mean + bi.sb + 1);
        if (p.rot_q > 0) {
            s1024 = static_cast<unsigned>((1024ll * p.rot_p) % p.rot_q);
            s16384 = static_cast<unsigned>((16384ll * p.rot_p) % p.rot_q);
        }
    }

    const int warp = tid >> 5, lane = tid & 31;
    float2* E = S.buf;
    __shared__ __align__(8) unsigned long long bulk_bar;
    const uint32_t bar_a = static_cast<uint32_t>(__cvta_generic_to_shared(&bulk_bar));
    const float2* zq = p.z + (bi.base - p.z_index0);
    const bool bulk = KK_K2_BULK && FAST && ((reinterpret_cast<uintptr_t>(zq) & 15) == 0);
    if (bulk && tid == 0) {
        mbar_init(bar_a, 1);
        mbar_expect_tx(bar_a, (KK_K2_BULK_X1 ? 32u : 16u) * kK2Threads * sizeof(float2));
#pragma unroll 1
        for (int r = 0; r < 16; ++r) {
            bulk_g2s(static_cast<uint32_t>(__cvta_generic_to_shared(S.A + r * kK2Threads)), zq + kK2Threads + 1024 * r,
                     kK2Threads * sizeof(float2), bar_a);
            if (KK_K2_BULK_X1)
                bulk_g2s(static_cast<uint32_t>(__cvta_generic_to_shared(E + r * kRowE + kK2Threads + (r & 1))),
                         zq + kHopS + kK2Threads + 1024 * r, kK2Threads * sizeof(float2), bar_a);
        }
    }
    // TMEM scratch (one CTA per SM: the allocation always succeeds)
    __shared__ uint32_t tmem_base_sh;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_base_sh))),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem_thread = tmem_base_sh + (static_cast<uint32_t>(32 * (warp & 3)) << 16) +
                                 static_cast<uint32_t>(64 * (warp >> 2));
    for (int chain = 0; chain < 2; ++chain) {
        // ---- FFT16384 step 1: column n2 = j, DFT16 over n1 (stride 1024),
        //      W16384^{j k1}, -> row k1, position j ----
#pragma unroll 1
        for (int q = 0; q < 1024 / kK2Threads; ++q) {
            float2 v[16];
            const int j = tid + q * kK2Threads;
            const uint32_t taddr = tmem_thread + 32 * q;
            if (chain == 0) {
                const float2* x0s = nullptr;
                const float2* x1s = nullptr;
                if (FAST && q == 1) {
                    if (bulk) {
                        mbar_wait_parity(bar_a, 0);
                        if (KK_K2_BULK_X1) x1s = E + kK2Threads + tid;
                    } else {
                        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
                    }
                    x0s = S.A + tid;
                }
                k2_load_column_ab<FAST>(p, bi, S.rot, j, mA, mB, bnd, s1024, s16384, v, taddr, x0s, x1s);
                // the staged x1 of odd rows sits one slot right: the slot this
                // thread's row outputs overwrite belongs to the neighbour's input
                if (KK_K2_BULK_X1 && bulk && q == 1) __syncthreads();
                if (FAST && !bulk && q == 0) {
                    // the second column's x0 half (16 x 8 B per thread) is copied into
                    // the (still unused) A buffer while the first column is transformed
                    // (K2 11.83 -> 11.54 ms per 2^30 samples; issuing it before the first
                    // column's loads gained less, also staging x1 into the FFT buffer lost)
                    const float2* zq1 = p.z + (bi.base - p.z_index0) + tid + kK2Threads;
#pragma unroll
                    for (int r = 0; r < 16; ++r) {
                        const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(S.A + r * kK2Threads + tid));
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(zq1 + 1024 * r)
                                     : "memory");
                    }
                    asm volatile("cp.async.commit_group;\n" ::: "memory");
                }
            } else {
                float2 h0[8], h1[8];
                tmem_ld16(taddr, h0);
                tmem_ld16(taddr + 16, h1);
                tmem_wait_ld();
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    v[r] = h0[r];
                    v[8 + r] = h1[r];
                }
            }
            dft_reg<16, false>(v);
            // W16384^{j k1}; chain 1 also W32768^j: W32768^{j (2 k1 + 1)}
            const float2 s2 = tw.template w<kHopS>(j);
            float2 wr = s2;
            if (chain == 1) {
                wr = tw.template w<kNS>(j);
                v[0] = cmul(v[0], wr);
            }
#pragma unroll
            for (int k1 = 1; k1 < 16; ++k1) {
                if (chain == 1 || k1 > 1) wr = cmul(wr, s2);
                v[k1] = cmul(v[k1], wr);
            }
#pragma unroll
            for (int k1 = 0; k1 < 16; ++k1) E[k1 * kRowE + j] = v[k1];
        }
        __syncthreads();
        // ---- FFT16384 step 2: warp k1 transforms row k1 -> bin k1 + 16 k2 at [k1][k2] ----
        warp_fft1024<false>(E + warp * kRowE, lane, tw);
        __syncthreads();

        // ---- IFFT8192 step 1: column m2 = tid of the kept bins x H (stride 512) ----
        const float2* h = chain == 0 ? p.h_even : p.h_odd;
        float2 u[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int m = tid + 512 * r;
            const int k = r < 8 ? m : m + 8192;          // kept bins: low and high quarters
            u[r] = cmul(E[(k & 15) * kRowE + (k >> 4)], __ldg(h + m));
        }
        __syncthreads();
        dft_reg<16, true>(u);
        apply_twiddle_chain<16, true>(u, tw.template w<kNOut>(tid));
#pragma unroll
        for (int p1 = 0; p1 < 16; ++p1) E[p1 * kRowI + tid] = u[p1];
        __syncthreads();
        // ---- IFFT8192 step 2: warp p1 transforms row p1 -> sample p1 + 16 p2 ----
        if (chain == 0) {
            auto st_a = [&](int p2, float2 v) { S.A[padi(warp + 16 * p2)] = v; };
            warp_fft512<true>(E + warp * kRowI, lane, tw, st_a);
            __syncthreads();
        } else {
            const float sc = 0.5f / 16384.0f;
            auto st_o = [&](int p2, float2 v) {
                const int r = warp + 16 * p2;
                // W16384^{-r} B[r]
                const float2 bt = cmulc(v, tw.template w<kHopS>(r));
                S.A[padi(r)] = cscale(csub(S.A[padi(r)], bt), sc);
            };
            warp_fft512<true>(E + warp * kRowI, lane, tw, st_o);
            __syncthreads();
            float2* out = p.out + int64_t(bx) * kNOut;
#pragma unroll 4
            for (int i = tid; i < kNOut; i += kK2Threads) out[i] = S.A[padi(i)];
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base_sh), "n"(kTmemCols));
}

template <bool FAST>
__global__ void __launch_bounds__(kK2Threads, 1) static_blocks_kernel(K2Params p, const float2* __restrict__ tw_g) {
    k2_body<FAST>(blockIdx.x, gridDim.x, p, tw_g);
}

// Batched K2 (independent streams in one launch): blockIdx.y
// selects the job (a contiguous run of blocks of one stream)
constexpr int kK2BatchMax = 32;
struct K2Batch {
    K2Params job[kK2BatchMax];
    int n_blocks[kK2BatchMax];
};
template <bool FAST>
__global__ void __launch_bounds__(kK2Threads, 1) static_blocks_batch_kernel(const __grid_constant__ K2Batch b,
                                                                            const float2* __restrict__ tw_g) {
    const int nb = b.n_blocks[blockIdx.y];
    if (static_cast<int>(blockIdx.x) >= nb) return;
    k2_body<FAST>(blockIdx.x, nb, b.job[blockIdx.y], tw_g);
}

}  // namespace kk

namespace kk {
// the up-to-three launch ranges of one stream's blocks: the interior ones
// (inside [0, valid_end), <= 1 carrier boundary) take the FAST
// specialisation, the stream-edge ones the generic one
struct K2Range {
    bool fast;
    int64_t a, b;
};
static int k2_plan(const kk_k2_job& j, K2Params& p, K2Range (&r)[3]) {
    if (j.carrier && (j.seg_len <= 0 || !j.seg_mean)) return set_error(KK_ERR_PARAM, "carrier means missing");
    if (j.rot_q > 0 && !j.rot_tab) return set_error(KK_ERR_PARAM, "rotation table missing");
    if (j.rot_q > kRotMax) return set_error(KK_ERR_PARAM, "rotation denominator must be <= 1024");
    p.z = static_cast<const float2*>(j.z);
    p.z_index0 = j.z_index0;
    p.hb0 = j.hb0;
    p.valid_end = j.valid_end;
    p.seg_mean = static_cast<const float2*>(j.seg_mean);
    p.seg_index0 = j.seg_index0;
    p.seg_len = j.seg_len;
    p.carrier = j.carrier;
    p.rot_p = j.rot_p;
    p.rot_q = j.rot_q;
    p.rot_tab = static_cast<const float2*>(j.rot_tab);
    p.rot_step = j.rot_q > 0 ? 0ull : j.rot_step;
    p.mirror = j.mirror;
    p.h_even = static_cast<const float2*>(j.h_even);
    p.h_odd = static_cast<const float2*>(j.h_odd);
    p.out = static_cast<float2*>(j.out);
    p.prefetch_ahead = num_sms();
    const int64_t hb0 = j.hb0, hb1 = j.hb0 + j.n_blocks;
    int64_t lo = hb0, hi = hb1;
    if (!j.carrier || (j.seg_len >= kNS && j.seg_len % kHopS == 0)) {
        lo = std::max<int64_t>(hb0, 1);
        hi = std::min<int64_t>(hb1, j.valid_end / kHopS);
        if (hi < lo) { lo = hb0; hi = hb0; }
    } else {
        lo = hi = hb0;
    }
    r[0] = {false, hb0, lo};
    r[1] = {true, lo, hi};
    r[2] = {false, hi, hb1};
    return KK_OK;
}
static K2Params k2_sub(const K2Params& p, int64_t hb0, int64_t a) {
    K2Params q = p;
    q.hb0 = a;
    q.out = p.out + (a - hb0) * kNOut;
    return q;
}
static int k2_attrs() {
    const size_t smem = sizeof(K2Smem);
    if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(static_blocks_kernel<true>), smem, "K2 smem attr"))
        return rc;
    if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(static_blocks_kernel<false>), smem, "K2 smem attr"))
        return rc;
    if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(static_blocks_batch_kernel<true>), smem, "K2 smem attr"))
        return rc;
    return ensure_smem_attr(reinterpret_cast<const void*>(static_blocks_batch_kernel<false>), smem, "K2 smem attr");
}
}  // namespace kk

extern "C" int kk_static_blocks(const void* z, int64_t z_index0, int64_t hb0, int64_t n_blocks,
                                int64_t valid_end, const void* seg_mean, int64_t seg_index0, int seg_len,
                                int carrier, int rot_p, int rot_q, const void* rot_tab,
                                unsigned long long rot_step, int mirror, const void* h_even, const void* h_odd,
                                void* out, void* stream) {
    using namespace kk;
    clear_error();
    if (n_blocks <= 0) return KK_OK;
    const float2* tw = twiddle_table_device();
    if (!tw) return KK_ERR_CUDA;
    if (int rc = k2_attrs()) return rc;
    const kk_k2_job j = {z, z_index0, hb0, n_blocks, valid_end, seg_mean, seg_index0, seg_len, carrier, rot_p,
                         rot_q, rot_tab, rot_step, mirror, h_even, h_odd, out};
    K2Params p;
    K2Range r[3];
    if (int rc = k2_plan(j, p, r)) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t smem = sizeof(K2Smem);
    for (const K2Range& g : r) {
        if (g.b <= g.a) continue;
        const K2Params q = k2_sub(p, hb0, g.a);
        if (g.fast)
            static_blocks_kernel<true><<<static_cast<unsigned>(g.b - g.a), kK2Threads, smem, s>>>(q, tw);
        else
            static_blocks_kernel<false><<<static_cast<unsigned>(g.b - g.a), kK2Threads, smem, s>>>(q, tw);
        if (int rc = check_launch("static_blocks_kernel")) return rc;
    }
    return KK_OK;
}

extern "C" int kk_static_blocks_batch(const kk_k2_job* jobs, int n_jobs, void* stream) {
    using namespace kk;
    clear_error();
    if (n_jobs <= 0) return KK_OK;
    if (!jobs) return set_error(KK_ERR_PARAM, "jobs missing");
    const float2* tw = twiddle_table_device();
    if (!tw) return KK_ERR_CUDA;
    if (int rc = k2_attrs()) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t smem = sizeof(K2Smem);
    // all jobs' ranges, grouped by specialisation, kK2BatchMax per launch
    for (int fast = 0; fast < 2; ++fast) {
        K2Batch b;
        int m = 0;
        int64_t gx = 0;
        auto flush = [&]() -> int {
            if (m == 0) return KK_OK;
            if (fast)
                static_blocks_batch_kernel<true><<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(m)),
                                                    kK2Threads, smem, s>>>(b, tw);
            else
                static_blocks_batch_kernel<false><<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(m)),
                                                     kK2Threads, smem, s>>>(b, tw);
            m = 0;
            gx = 0;
            return check_launch("static_blocks_batch_kernel");
        };
        for (int i = 0; i < n_jobs; ++i) {
            if (jobs[i].n_blocks <= 0) continue;
            K2Params p;
            K2Range r[3];
            if (int rc = k2_plan(jobs[i], p, r)) return rc;
            for (const K2Range& g : r) {
                if (g.b <= g.a || g.fast != (fast == 1)) continue;
                if (g.b - g.a >= (int64_t(1) << 31)) return set_error(KK_ERR_PARAM, "too many blocks per job");
                b.job[m] = k2_sub(p, jobs[i].hb0, g.a);
                b.n_blocks[m] = static_cast<int>(g.b - g.a);
                gx = std::max<int64_t>(gx, g.b - g.a);
                if (++m == kK2BatchMax)
                    if (int rc = flush()) return rc;
            }
        }
        if (int rc = flush()) return rc;
    }
    return KK_OK;
}

// ---------------------------------------------------------------------------
// carrier means: mean over each aligned segment from the per-hop field sums
// (rxdsp.py:685-687).  seg s covers hops [s*hps, (s+1)*hps) of the hop-sum
// array; the last segment may be partial (flush) with `last_len` samples.
// ---------------------------------------------------------------------------
namespace kk {
__global__ void carrier_means_kernel(const float2* __restrict__ hop_sum, int64_t n_segs, int hops_per_seg,
                                     int64_t n_hops_avail, int64_t last_len, int seg_len, float2* __restrict__ mean) {
    // one warp per segment: lane-strided fp64 partial sums (all loads
    // independent), fixed shuffle tree -- a deterministic order that does not
    // depend on how the stream was chunked
    const int64_t s = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= n_segs) return;
    double re = 0.0, im = 0.0;
    const int64_t h0 = s * hops_per_seg;
    for (int i = lane; i < hops_per_seg; i += 32) {
        const int64_t h = h0 + i;
        if (h < n_hops_avail) {
            const float2 v = __ldg(hop_sum + h);
            re += v.x;
            im += v.y;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, o);
        im += __shfl_xor_sync(0xffffffffu, im, o);
    }
    if (lane == 0) {
        const double len = (s == n_segs - 1 && last_len > 0) ? static_cast<double>(last_len) : static_cast<double>(seg_len);
        mean[s] = make_float2(static_cast<float>(re / len), static_cast<float>(im / len));
    }
}
}  // namespace kk

extern "C" int kk_carrier_means(const void* hop_sum, int64_t n_segs, int hops_per_seg, int64_t n_hops_avail,
                                int64_t last_len, int seg_len, void* mean, void* stream) {
    using namespace kk;
    clear_error();
    if (n_segs <= 0) return KK_OK;
    const int th = 128;   // 4 segments per CTA (one warp each)
    carrier_means_kernel<<<static_cast<unsigned>((n_segs * 32 + th - 1) / th), th, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const float2*>(hop_sum), n_segs, hops_per_seg, n_hops_avail, last_len, seg_len,
        static_cast<float2*>(mean));
    return check_launch("carrier_means_kernel");
}
