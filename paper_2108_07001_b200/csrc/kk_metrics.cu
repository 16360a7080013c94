// Measurement kernels of the sweep/measure path:
//   * kk_bit_xcorr   -- frame_sync's bipolar cross-correlation of the received
//     and transmitted bit streams over ALL lags, with peak / sidelobe search
//     (reference: metrics.py `frame_sync` :69-112).  The reference evaluates
//     it with float64 FFTs (np.fft / scipy fftconvolve); so does this file,
//     with its own power-of-two Stockham FFT.  The correlation of two ±1
//     sequences is an integer, and the float64 transform error at these
//     sizes (~ eps * N * log2 N < 1e-5 for N = 2^31) is far below 0.5, so
//     every value is rounded to the exact integer before the search: the
//     peak index and the peak / sidelobe magnitudes are the exact ones.
//   * kk_label_bits        -- decided point labels -> per-bit uint8 stream
//     (rxdsp.py demap :548-567 bit order, MSB first).
//   * kk_bit_error_windows -- error count and per-window counts of two
//     aligned bit streams (harness/runner.py measure_point :104-137 with
//     metrics.py windowed_q :130-150 windows).
//   * kk_evm_sums          -- float64 sums of |soft - ref|^2 and |ref|^2
//     (metrics.py evm :169-179).
//
// FFT layout: N = 2^n complex float64 points (double2), n in [12, 31],
// out-of-place Stockham passes of radix R = 2^r (3 <= r <= 10, the passes of
// one transform as equal as possible).  One CTA owns 4096 points: TILE =
// 4096/R consecutive "columns" q, each with its R inputs q + m N/R (coalesced
// along q); it applies the pass twiddles w_{Ns R}^{(q mod Ns) m}, runs the
// R-point DFT in shared memory as radix-16/8/4/2 Stockham stages (one 16-
// value register butterfly set per thread per stage), and writes
// (q / Ns) Ns R + (q mod Ns) + m Ns.  Pass twiddles come from a two-level
// table w_N^e = lo[e mod 2^h] * hi[e >> h] (correctly rounded sincospi
// entries, both tables L2 resident); inner twiddles from a 1024-entry table.
// HBM: 32 B per point per pass (read + write), ceil(n / 10) passes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kk_internal.h"

namespace kk {
namespace xc {

constexpr int kThreads = 256;
constexpr int kTilePoints = 4096;   // points per CTA per pass
constexpr int kInner = 1024;        // inner twiddle table size

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

// cos / sin(2 pi i / 16), i < 16
__device__ constexpr double kC16[16] = {
    1.0, 0.92387953251128674, 0.70710678118654757, 0.38268343236508984, 0.0, -0.38268343236508984,
    -0.70710678118654757, -0.92387953251128674, -1.0, -0.92387953251128674, -0.70710678118654757,
    -0.38268343236508984, 0.0, 0.38268343236508984, 0.70710678118654757, 0.92387953251128674};
__device__ constexpr double kS16[16] = {
    0.0, 0.38268343236508978, 0.70710678118654746, 0.92387953251128674, 1.0, 0.92387953251128674,
    0.70710678118654746, 0.38268343236508978, 0.0, -0.38268343236508978, -0.70710678118654746,
    -0.92387953251128674, -1.0, -0.92387953251128674, -0.70710678118654746, -0.38268343236508978};

// a * exp(-2 pi i t / 16) with t a compile-time constant after unrolling
__device__ __forceinline__ double2 rot16(double2 a, int t) {
    t &= 15;
    if (t == 0) return a;
    if (t == 4) return make_double2(a.y, -a.x);
    if (t == 8) return make_double2(-a.x, -a.y);
    if (t == 12) return make_double2(-a.y, a.x);
    const double c = kC16[t], s = -kS16[t];
    return make_double2(fma(a.x, c, -a.y * s), fma(a.x, s, a.y * c));
}

// In-register DFT of R <= 16 points, natural order in and out (radix-2 DIF,
// then the bit-reversal permutation resolved at compile time).
template <int R>
__device__ __forceinline__ void dft(double2 (&v)[R]) {
#pragma unroll
    for (int half = R / 2; half >= 1; half >>= 1) {
#pragma unroll
        for (int st = 0; st < R; st += 2 * half) {
#pragma unroll
            for (int j = 0; j < half; ++j) {
                const double2 a = v[st + j], b = v[st + j + half];
                v[st + j] = cadd(a, b);
                v[st + j + half] = rot16(csub(a, b), j * (16 / (2 * half)));
            }
        }
    }
    double2 t[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
        int rev = 0;
#pragma unroll
        for (int b = 1, rb = R / 2; b < R; b <<= 1, rb >>= 1)
            if (i & b) rev |= rb;
        t[i] = v[rev];
    }
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = t[i];
}

struct Tables {
    const double2* lo;    // w_N^b, b < 2^h
    const double2* hi;    // w_N^(a 2^h)
    const double2* inner; // w_1024^x, x < 1024
    int h;
};

__device__ __forceinline__ double2 tw_n(const Tables& t, int64_t e) {
    const double2 a = t.lo[e & ((int64_t(1) << t.h) - 1)];
    if ((e >> t.h) == 0) return a;
    return cmul(a, t.hi[e >> t.h]);
}

__global__ void tables_kernel(double2* lo, double2* hi, double2* inner, int log_n, int h) {
    const int64_t n_lo = int64_t(1) << h, n_hi = int64_t(1) << (log_n - h);
    const double inv = 2.0 / double(int64_t(1) << log_n);   // exact power of two
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_lo + n_hi + kInner;
         i += int64_t(gridDim.x) * blockDim.x) {
        double s, c;
        if (i < n_lo) {
            sincospi(double(i) * inv, &s, &c);
            lo[i] = make_double2(c, -s);
        } else if (i < n_lo + n_hi) {
            const int64_t a = i - n_lo;
            sincospi(double(a << h) * inv, &s, &c);
            hi[a] = make_double2(c, -s);
        } else {
            const int64_t x = i - n_lo - n_hi;
            sincospi(double(x) * (2.0 / kInner), &s, &c);
            inner[x] = make_double2(c, -s);
        }
    }
}

// One inner Stockham stage of radix RS over TILE columns of length R held in
// shared memory (column stride R + 1 doubles2: conflict-free column walks).
template <int R, int RS>
__device__ __forceinline__ void inner_stage(double2* s, int ls, const double2* __restrict__ inner) {
    constexpr int TILE = kTilePoints / R;
    constexpr int BFLY = R / RS;            // butterflies per column
    constexpr int PER = 16 / RS;            // butterflies per thread
    static_assert(TILE * BFLY == kThreads * PER, "tile / thread mismatch");
    double2 v[PER][RS];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int g = threadIdx.x + kThreads * u;
        const int t = g / BFLY, b = g % BFLY;
        const int k = b % ls;
        const double2* col = s + t * (R + 1);
#pragma unroll
        for (int m = 0; m < RS; ++m) {
            double2 x = col[b + m * BFLY];
            if (m > 0 && k > 0) x = cmul(x, inner[(k * m * (kInner / (ls * RS))) & (kInner - 1)]);
            v[u][m] = x;
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        dft<RS>(v[u]);
        const int g = threadIdx.x + kThreads * u;
        const int t = g / BFLY, b = g % BFLY;
        const int j = b / ls, k = b % ls;
        double2* col = s + t * (R + 1);
#pragma unroll
        for (int m = 0; m < RS; ++m) col[j * RS * ls + m * ls + k] = v[u][m];
    }
    __syncthreads();
}

template <int LOGR>
__global__ void __launch_bounds__(kThreads) fft_pass_kernel(const double2* __restrict__ in, double2* __restrict__ out,
                                                            int log_n, int64_t ns, const Tables tb) {
    constexpr int R = 1 << LOGR;
    constexpr int TILE = kTilePoints / R;
    extern __shared__ double2 sm[];
    const int64_t n = int64_t(1) << log_n;
    const int64_t nr = n >> LOGR;
    const int64_t q0 = int64_t(blockIdx.x) * TILE;
    const int64_t tw_step = n / (ns * R);   // w_{Ns R} = w_N^(N / (Ns R))
    // load + pass twiddle, t fastest (coalesced along q)
#pragma unroll 4
    for (int i = 0; i < kTilePoints / kThreads; ++i) {
        const int e = threadIdx.x + kThreads * i;
        const int t = e % TILE, m = e / TILE;
        const int64_t q = q0 + t;
        double2 x = in[q + int64_t(m) * nr];
        const int64_t k = q & (ns - 1);
        if (k != 0 && m != 0) x = cmul(x, tw_n(tb, ((k * m) * tw_step) & (n - 1)));
        sm[t * (R + 1) + m] = x;
    }
    __syncthreads();
    // R-point DFTs of every column: radix-16 stages, then the remainder
    constexpr int N16 = LOGR / 4, REM = LOGR % 4;
    int ls = 1;
    if constexpr (N16 > 0) {
#pragma unroll
        for (int st = 0; st < N16; ++st) {
            inner_stage<R, 16>(sm, ls, tb.inner);
            ls *= 16;
        }
    }
    if constexpr (REM == 3) inner_stage<R, 8>(sm, ls, tb.inner);
    if constexpr (REM == 2) inner_stage<R, 4>(sm, ls, tb.inner);
    if constexpr (REM == 1) inner_stage<R, 2>(sm, ls, tb.inner);
    // store
    if (ns == 1) {
        // out[q R + m]: m fastest -> one contiguous TILE * R run
#pragma unroll 4
        for (int i = 0; i < kTilePoints / kThreads; ++i) {
            const int e = threadIdx.x + kThreads * i;
            const int t = e / R, m = e % R;
            out[(q0 + t) * R + m] = sm[t * (R + 1) + m];
        }
    } else {
#pragma unroll 4
        for (int i = 0; i < kTilePoints / kThreads; ++i) {
            const int e = threadIdx.x + kThreads * i;
            const int t = e % TILE, m = e / TILE;
            const int64_t q = q0 + t;
            out[(q / ns) * ns * R + (q & (ns - 1)) + int64_t(m) * ns] = sm[t * (R + 1) + m];
        }
    }
}

// z[i] = (2 rx[i] - 1) + j (2 tx[n_tx - 1 - i] - 1), zero padded
__global__ void pack_kernel(const uint8_t* __restrict__ rx, int64_t n_rx, const uint8_t* __restrict__ tx,
                            int64_t n_tx, double2* __restrict__ z, int64_t n) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const double a = i < n_rx ? (rx[i] ? 1.0 : -1.0) : 0.0;
        const double b = i < n_tx ? (tx[n_tx - 1 - i] ? 1.0 : -1.0) : 0.0;
        z[i] = make_double2(a, b);
    }
}

// Z = FFT(a + j b) -> conj(A B) in place (A, B the spectra of a and b), so a
// forward FFT of the result is conj(N * conv) and its real part is N * conv.
__global__ void product_kernel(double2* __restrict__ z, int64_t n) {
    for (int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; f <= n / 2;
         f += int64_t(gridDim.x) * blockDim.x) {
        const int64_t g = (n - f) & (n - 1);
        const double2 zf = z[f], zg = z[g];
        // A = (Zf + conj Zg) / 2, B = (Zf - conj Zg) / (2 j)
        const double2 a = make_double2(0.5 * (zf.x + zg.x), 0.5 * (zf.y - zg.y));
        const double2 d = make_double2(0.5 * (zf.x - zg.x), 0.5 * (zf.y + zg.y));
        const double2 b = make_double2(d.y, -d.x);
        const double2 p = cmul(a, b);
        z[f] = cconj(p);
        if (g != f) z[g] = p;   // P(-f) = conj P(f)
    }
}

__device__ __forceinline__ long long conv_at(const double2* __restrict__ y, int64_t j, double inv_n) {
    return llrint(y[j].x * inv_n);
}

// |correlation| at index i: linear (i < L) = |conv[i]|; circular (i < n) =
// |conv[n - 1 + i] + conv[i - 1]|
__device__ __forceinline__ long long corr_mag(const double2* __restrict__ y, int64_t i, int circular, int64_t n_c,
                                              double inv_n) {
    long long c;
    if (circular) {
        c = conv_at(y, n_c - 1 + i, inv_n);
        if (i >= 1) c += conv_at(y, i - 1, inv_n);
    } else {
        c = conv_at(y, i, inv_n);
    }
    return c < 0 ? -c : c;
}

// key = |c| << 32 | (2^32 - 1 - i): the max key is the largest magnitude at
// the smallest index (np.argmax's first-occurrence rule)
__global__ void peak_kernel(const double2* __restrict__ y, int64_t m, int circular, int64_t n_c, double inv_n,
                            unsigned long long* __restrict__ best) {
    unsigned long long kbest = 0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
        const unsigned long long mag = static_cast<unsigned long long>(corr_mag(y, i, circular, n_c, inv_n));
        const unsigned long long key = (mag << 32) | (0xFFFFFFFFull - static_cast<unsigned long long>(i));
        kbest = key > kbest ? key : kbest;
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, kbest, o);
        kbest = other > kbest ? other : kbest;
    }
    if ((threadIdx.x & 31) == 0 && kbest) atomicMax(best, kbest);
}

// max |c| outside [k - w, k + w]
__global__ void side_kernel(const double2* __restrict__ y, int64_t m, int circular, int64_t n_c, double inv_n,
                            const unsigned long long* __restrict__ best, int w,
                            unsigned long long* __restrict__ side) {
    const int64_t k = static_cast<int64_t>(0xFFFFFFFFull - (*best & 0xFFFFFFFFull));
    unsigned long long mx = 0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
        if (i >= k - w && i <= k + w) continue;
        const unsigned long long mag = static_cast<unsigned long long>(corr_mag(y, i, circular, n_c, inv_n));
        mx = mag > mx ? mag : mx;
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = other > mx ? other : mx;
    }
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(side, mx);
}

__global__ void xcorr_result_kernel(const unsigned long long* __restrict__ best,
                                    const unsigned long long* __restrict__ side, long long* __restrict__ out) {
    out[0] = static_cast<long long>(0xFFFFFFFFull - (*best & 0xFFFFFFFFull));
    out[1] = static_cast<long long>(*best >> 32);
    out[2] = static_cast<long long>(*side);
}

struct Plan {
    int log_n = 0, h = 0, npass = 0;
    int logr[4] = {0, 0, 0, 0};
    int64_t n = 0;
    size_t off_b = 0, off_lo = 0, off_hi = 0, off_inner = 0, off_red = 0, total = 0;
};

inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

inline bool make_plan(int64_t n_rx, int64_t n_tx, int circular, Plan& p) {
    const int64_t len = circular ? 2 * n_rx - 1 : n_rx + n_tx - 1;
    int log_n = 12;
    while ((int64_t(1) << log_n) < len) ++log_n;
    if (log_n > 31) return false;
    p.log_n = log_n;
    p.n = int64_t(1) << log_n;
    p.h = (log_n + 1) / 2;
    p.npass = (log_n + 9) / 10;
    for (int i = 0; i < p.npass; ++i) p.logr[i] = log_n / p.npass + (i < log_n % p.npass ? 1 : 0);
    const size_t buf = size_t(p.n) * sizeof(double2);
    p.off_b = al(buf);
    p.off_lo = p.off_b + al(buf);
    p.off_hi = p.off_lo + al((size_t(1) << p.h) * sizeof(double2));
    p.off_inner = p.off_hi + al((size_t(1) << (log_n - p.h)) * sizeof(double2));
    p.off_red = p.off_inner + al(kInner * sizeof(double2));
    p.total = p.off_red + 256;
    return true;
}

template <int LOGR>
int launch_pass(const double2* in, double2* out, const Plan& p, int64_t ns, const Tables& tb, cudaStream_t st) {
    constexpr int R = 1 << LOGR;
    const size_t smem = size_t(kTilePoints / R) * (R + 1) * sizeof(double2);
    if (ensure_smem_attr(reinterpret_cast<const void*>(&fft_pass_kernel<LOGR>), smem, "fft_pass_kernel") != KK_OK)
        return KK_ERR_CUDA;
    fft_pass_kernel<LOGR><<<static_cast<unsigned>(p.n / kTilePoints), kThreads, smem, st>>>(in, out, p.log_n, ns, tb);
    return check_launch("fft_pass_kernel");
}

// forward FFT of `a` (length p.n); returns the buffer holding the result
double2* fft(double2* a, double2* b, const Plan& p, const Tables& tb, cudaStream_t st, int* rc) {
    int64_t ns = 1;
    double2 *src = a, *dst = b;
    for (int i = 0; i < p.npass && *rc == KK_OK; ++i) {
        switch (p.logr[i]) {
            case 3: *rc = launch_pass<3>(src, dst, p, ns, tb, st); break;
            case 4: *rc = launch_pass<4>(src, dst, p, ns, tb, st); break;
            case 5: *rc = launch_pass<5>(src, dst, p, ns, tb, st); break;
            case 6: *rc = launch_pass<6>(src, dst, p, ns, tb, st); break;
            case 7: *rc = launch_pass<7>(src, dst, p, ns, tb, st); break;
            case 8: *rc = launch_pass<8>(src, dst, p, ns, tb, st); break;
            case 9: *rc = launch_pass<9>(src, dst, p, ns, tb, st); break;
            case 10: *rc = launch_pass<10>(src, dst, p, ns, tb, st); break;
            default: *rc = set_error(KK_ERR_PARAM, "fft: bad pass radix");
        }
        ns <<= p.logr[i];
        std::swap(src, dst);
    }
    return src;
}

inline unsigned grid_for(int64_t n, int th) {
    int64_t b = (n + th - 1) / th;
    const int64_t cap = int64_t(num_sms()) * 16;
    return static_cast<unsigned>(std::max<int64_t>(1, std::min(b, cap)));
}

}  // namespace xc

// ---------------------------------------------------------------------------
// labels -> bits, per-window error counts, EVM sums
// ---------------------------------------------------------------------------
struct LabelBits {
    uint8_t v[64];
};

__global__ void label_bits_kernel(const uint8_t* __restrict__ lab, int64_t n, const __grid_constant__ LabelBits pl,
                                  int k, uint8_t* __restrict__ out) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n * k;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t s = i / k;
        const int b = static_cast<int>(i - s * k);
        out[i] = (pl.v[lab[s] & 63] >> (k - 1 - b)) & 1;
    }
}

__global__ void bit_error_windows_kernel(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, int64_t n,
                                         int64_t bpw, int64_t n_win, unsigned long long* __restrict__ total,
                                         unsigned long long* __restrict__ win) {
    unsigned long long cnt = 0;
    for (int64_t i0 = int64_t(blockIdx.x) * blockDim.x; i0 < n; i0 += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        const bool e = i < n && a[i] != b[i];
        cnt += e ? 1 : 0;
        if (win) {
            const int64_t w = (i < n && bpw > 0) ? i / bpw : -1;
            const bool counted = e && w < n_win;
            // lanes of one window add once (windows are usually >> 32 bits)
            const unsigned grp = __match_any_sync(0xffffffffu, counted ? w : -1);
            const unsigned vote = __ballot_sync(0xffffffffu, counted) & grp;
            if (counted && (__ffs(vote) - 1) == (threadIdx.x & 31))
                atomicAdd(win + w, static_cast<unsigned long long>(__popc(vote)));
        }
    }
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(total, cnt);
}

__global__ void evm_sums_kernel(const float2* __restrict__ soft, const double2* __restrict__ ref, int64_t n,
                                double* __restrict__ sums) {
    double se = 0.0, sr = 0.0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const float2 s = soft[i];
        const double2 r = ref[i];
        const double dx = double(s.x) - r.x, dy = double(s.y) - r.y;
        se = fma(dx, dx, fma(dy, dy, se));
        sr = fma(r.x, r.x, fma(r.y, r.y, sr));
    }
    for (int o = 16; o; o >>= 1) {
        se += __shfl_xor_sync(0xffffffffu, se, o);
        sr += __shfl_xor_sync(0xffffffffu, sr, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(sums, se);
        atomicAdd(sums + 1, sr);
    }
}

}  // namespace kk

extern "C" size_t kk_bit_xcorr_workspace_bytes(int64_t n_rx, int64_t n_tx, int circular) {
    kk::xc::Plan p;
    if (n_rx <= 0 || n_tx <= 0 || !kk::xc::make_plan(n_rx, n_tx, circular, p)) return 0;
    return p.total;
}

extern "C" int kk_bit_xcorr(const uint8_t* rx, int64_t n_rx, const uint8_t* tx, int64_t n_tx, int circular, void* ws,
                            size_t ws_bytes, long long* out3, void* stream) {
    using namespace kk;
    using namespace kk::xc;
    clear_error();
    if (n_rx <= 0 || n_tx <= 0 || !rx || !tx || !out3) return set_error(KK_ERR_PARAM, "kk_bit_xcorr: bad arguments");
    if (circular && n_rx != n_tx) return set_error(KK_ERR_PARAM, "kk_bit_xcorr: circular needs equal lengths");
    Plan p;
    if (!make_plan(n_rx, n_tx, circular, p)) return set_error(KK_ERR_PARAM, "kk_bit_xcorr: streams too long");
    if (!ws || ws_bytes < p.total) return set_error(KK_ERR_PARAM, "kk_bit_xcorr: workspace too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    char* base = static_cast<char*>(ws);
    double2* a = reinterpret_cast<double2*>(base);
    double2* b = reinterpret_cast<double2*>(base + p.off_b);
    double2* lo = reinterpret_cast<double2*>(base + p.off_lo);
    double2* hi = reinterpret_cast<double2*>(base + p.off_hi);
    double2* inner = reinterpret_cast<double2*>(base + p.off_inner);
    unsigned long long* red = reinterpret_cast<unsigned long long*>(base + p.off_red);
    if (cudaMemsetAsync(red, 0, 2 * sizeof(unsigned long long), st) != cudaSuccess)
        return set_cuda_error("kk_bit_xcorr memset");
    const int64_t n_tab = (int64_t(1) << p.h) + (int64_t(1) << (p.log_n - p.h)) + kInner;
    tables_kernel<<<grid_for(n_tab, 256), 256, 0, st>>>(lo, hi, inner, p.log_n, p.h);
    int rc = check_launch("xcorr tables_kernel");
    if (rc != KK_OK) return rc;
    const Tables tb{lo, hi, inner, p.h};
    pack_kernel<<<grid_for(p.n, 256), 256, 0, st>>>(rx, n_rx, tx, n_tx, a, p.n);
    if ((rc = check_launch("xcorr pack_kernel")) != KK_OK) return rc;
    double2* z = fft(a, b, p, tb, st, &rc);
    if (rc != KK_OK) return rc;
    product_kernel<<<grid_for(p.n / 2 + 1, 256), 256, 0, st>>>(z, p.n);
    if ((rc = check_launch("xcorr product_kernel")) != KK_OK) return rc;
    double2* y = fft(z, z == a ? b : a, p, tb, st, &rc);
    if (rc != KK_OK) return rc;
    const int64_t m = circular ? n_rx : n_rx + n_tx - 1;
    const double inv_n = 1.0 / double(p.n);
    peak_kernel<<<grid_for(m, 256), 256, 0, st>>>(y, m, circular, n_rx, inv_n, red);
    if ((rc = check_launch("xcorr peak_kernel")) != KK_OK) return rc;
    side_kernel<<<grid_for(m, 256), 256, 0, st>>>(y, m, circular, n_rx, inv_n, red, circular ? 0 : 2, red + 1);
    if ((rc = check_launch("xcorr side_kernel")) != KK_OK) return rc;
    xcorr_result_kernel<<<1, 1, 0, st>>>(red, red + 1, out3);
    return check_launch("xcorr_result_kernel");
}

extern "C" int kk_label_bits(const uint8_t* labels, int64_t n, const uint8_t* point_label_host, int order,
                             int bits_per_symbol, uint8_t* out, void* stream) {
    using namespace kk;
    clear_error();
    if (bits_per_symbol < 1 || bits_per_symbol > 6 || order < 2 || order > 64 || !point_label_host)
        return set_error(KK_ERR_PARAM, "kk_label_bits: bits_per_symbol in [1, 6], order in [2, 64]");
    if (n <= 0) return KK_OK;
    LabelBits pl{};
    for (int i = 0; i < order; ++i) pl.v[i] = point_label_host[i];
    label_bits_kernel<<<xc::grid_for(n * bits_per_symbol, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        labels, n, pl, bits_per_symbol, out);
    return check_launch("label_bits_kernel");
}

extern "C" int kk_bit_error_windows(const uint8_t* a, const uint8_t* b, int64_t n, int64_t bits_per_window,
                                    unsigned long long* total, unsigned long long* win_counts, void* stream) {
    using namespace kk;
    clear_error();
    if (n < 0 || !total || (n > 0 && (!a || !b))) return set_error(KK_ERR_PARAM, "kk_bit_error_windows: bad arguments");
    if (n == 0) return KK_OK;
    const int64_t n_win = (win_counts && bits_per_window > 0) ? n / bits_per_window : 0;
    bit_error_windows_kernel<<<xc::grid_for(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        a, b, n, bits_per_window, n_win, total, n_win > 0 ? win_counts : nullptr);
    return check_launch("bit_error_windows_kernel");
}

extern "C" int kk_evm_sums(const void* soft, const void* ref, int64_t n, double* sums, void* stream) {
    using namespace kk;
    clear_error();
    if (n < 0 || !sums || (n > 0 && (!soft || !ref))) return set_error(KK_ERR_PARAM, "kk_evm_sums: bad arguments");
    if (n == 0) return KK_OK;
    evm_sums_kernel<<<xc::grid_for(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const float2*>(soft), static_cast<const double2*>(ref), n, sums);
    return check_launch("evm_sums_kernel");
}
