// Float64 complex FFTs of any length, and the split-step Fourier fiber span
// built on them -- the capture side of the path (the step
// before the receiver) and frame_sync's correlation (kk_metrics.cu).
//
// Power-of-two lengths N = 2^n (batched rows): out-of-place Stockham passes of
// radix R = 2^r (1 <= r <= 10, ceil(n / 10) passes as equal as possible).  One
// CTA owns 4096 points = TILE = 4096 / R consecutive columns Q of the batch
// (column Q = row * N/R + q), each with its R inputs q + m N/R (coalesced
// along q); it applies the pass twiddles w_{Ns R}^{(q mod Ns) m}, runs the
// R-point DFT in shared memory as radix-16/8/4/2 Stockham stages (16 register
// values per thread per stage), and writes (q / Ns) Ns R + (q mod Ns) + m Ns
// of its row.  Pass twiddles come from a two-level table w_N^e =
// lo[e mod 2^h] * hi[e >> h] (correctly rounded sincospi entries, L2
// resident); inner twiddles from a 1024-entry table.  32 B of HBM per point
// per pass (fp64 read + write).
//
// Other lengths: Bluestein's chirp-z on a power-of-two M >= 2n - 1:
// X[k] = w[k] sum_j (x[j] w[j]) conj(w[k - j]), w[j] = exp(-i pi j^2 / n), with
// j^2 reduced mod 2n in integers so the chirp phase is exact at any n.
//
// Inverse transforms: ifft(x) = conj(fft(conj x)) / n (numpy's normalisation).
//
// Reference: numpy.fft (pocketfft, float64) as called by kkmodem's channel
// (channel.py apply_cd :90-103, ssfm_span :124-158) and metrics (frame_sync
// :69-112).  Results agree to float64 rounding, not bit for bit.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kk_internal.h"

namespace kk {
namespace fft64 {

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

inline int half_bits(int log_n) { return (log_n + 1) / 2; }
inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

Tables tables_at(const void* mem, int log_n) {
    const int h = half_bits(log_n);
    const char* p = static_cast<const char*>(mem);
    Tables t;
    t.lo = reinterpret_cast<const double2*>(p);
    t.hi = reinterpret_cast<const double2*>(p + al((size_t(1) << h) * sizeof(double2)));
    t.inner = reinterpret_cast<const double2*>(p + al((size_t(1) << h) * sizeof(double2)) +
                                               al((size_t(1) << (log_n - h)) * sizeof(double2)));
    t.h = h;
    return t;
}

size_t table_bytes(int log_n) {
    const int h = half_bits(log_n);
    return al((size_t(1) << h) * sizeof(double2)) + al((size_t(1) << (log_n - h)) * sizeof(double2)) +
           al(kInner * sizeof(double2));
}

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

inline unsigned grid_for(int64_t n, int th) {
    const int64_t b = (n + th - 1) / th;
    const int64_t cap = int64_t(num_sms()) * 16;
    return static_cast<unsigned>(std::max<int64_t>(1, std::min(b, cap)));
}

int build_tables(void* mem, int log_n, cudaStream_t st) {
    const Tables t = tables_at(mem, log_n);
    const int64_t n_tab = (int64_t(1) << t.h) + (int64_t(1) << (log_n - t.h)) + kInner;
    tables_kernel<<<grid_for(n_tab, 256), 256, 0, st>>>(const_cast<double2*>(t.lo), const_cast<double2*>(t.hi),
                                                       const_cast<double2*>(t.inner), log_n, t.h);
    return check_launch("fft tables_kernel");
}

// One inner Stockham stage of radix RS over TILE columns of length R held in
// shared memory (column stride R + 1 double2: conflict-free column walks).
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

// One Stockham pass over `cols` = batch * N/R columns.
#ifndef KK_FFT_MINB
#define KK_FFT_MINB 2   // 2 CTAs/SM (<= 128 registers): measured 1.45x over 1 CTA at 140
#endif
#ifndef KK_FFT_UNROLL
#define KK_FFT_UNROLL 4
#endif
constexpr int kFftUnroll = KK_FFT_UNROLL;
template <int LOGR, bool FULL>   // FULL: cols is a multiple of TILE (no bounds tests)
__global__ void __launch_bounds__(kThreads, KK_FFT_MINB) fft_pass_kernel(const double2* __restrict__ in, double2* __restrict__ out,
                                                            int log_n, int64_t ns, int64_t cols, const Tables tb) {
    constexpr int R = 1 << LOGR;
    constexpr int TILE = kTilePoints / R;
    extern __shared__ double2 sm[];
    const int64_t n = int64_t(1) << log_n;
    const int lnr = log_n - LOGR;             // log2(N / R)
    const int64_t nr = int64_t(1) << lnr;
    const int64_t c0 = int64_t(blockIdx.x) * TILE;
    const int64_t tw_step = n / (ns * R);     // w_{Ns R} = w_N^(N / (Ns R))
    // load + pass twiddle, t fastest (coalesced along q).  For TILE <= the
    // thread count a thread keeps one column t for all its elements: the
    // column's address, twiddle exponent step and bounds test are hoisted.
    if constexpr (TILE <= kThreads) {
        constexpr int MS = kThreads / TILE;           // m step per element
        const int t = threadIdx.x % TILE, m0 = threadIdx.x / TILE;
        const int64_t c = c0 + t;
        const bool ok = FULL || c < cols;
        const int64_t q = c & (nr - 1);
        const double2* src = in + ((c >> lnr) << log_n) + q;
        const int64_t kstep = (q & (ns - 1)) * tw_step;   // exponent per unit of m
#pragma unroll kFftUnroll
        for (int i = 0; i < kTilePoints / kThreads; ++i) {
            const int m = m0 + MS * i;
            double2 x = make_double2(0.0, 0.0);
            if (ok) {
                x = src[int64_t(m) * nr];
                if (kstep != 0 && m != 0) x = cmul(x, tw_n(tb, (kstep * m) & (n - 1)));
            }
            sm[t * (R + 1) + m] = x;
        }
    } else {
#pragma unroll 4
        for (int i = 0; i < kTilePoints / kThreads; ++i) {
            const int e = threadIdx.x + kThreads * i;
            const int t = e % TILE, m = e / TILE;
            const int64_t c = c0 + t;
            double2 x = make_double2(0.0, 0.0);
            if (c < cols) {
                const int64_t row = c >> lnr, q = c & (nr - 1);
                x = in[(row << log_n) + q + int64_t(m) * nr];
                const int64_t k = q & (ns - 1);
                if (k != 0 && m != 0) x = cmul(x, tw_n(tb, ((k * m) * tw_step) & (n - 1)));
            }
            sm[t * (R + 1) + m] = x;
        }
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
        // out[row N + q R + m] = out[c R + m]: m fastest -> one contiguous run
#pragma unroll 4
        for (int i = 0; i < kTilePoints / kThreads; ++i) {
            const int e = threadIdx.x + kThreads * i;
            const int t = e / R, m = e % R;
            if (FULL || c0 + t < cols) out[(c0 + t) * R + m] = sm[t * (R + 1) + m];
        }
    } else if constexpr (TILE <= kThreads) {
        constexpr int MS = kThreads / TILE;
        const int t = threadIdx.x % TILE, m0 = threadIdx.x / TILE;
        const int64_t c = c0 + t;
        if (FULL || c < cols) {
            const int64_t q = c & (nr - 1);
            double2* dst = out + ((c >> lnr) << log_n) + (q / ns) * ns * R + (q & (ns - 1));
#pragma unroll kFftUnroll
            for (int i = 0; i < kTilePoints / kThreads; ++i) {
                const int m = m0 + MS * i;
                dst[int64_t(m) * ns] = sm[t * (R + 1) + m];
            }
        }
    } else {
#pragma unroll 4
        for (int i = 0; i < kTilePoints / kThreads; ++i) {
            const int e = threadIdx.x + kThreads * i;
            const int t = e % TILE, m = e / TILE;
            const int64_t c = c0 + t;
            if (c >= cols) continue;
            const int64_t row = c >> lnr, q = c & (nr - 1);
            out[(row << log_n) + (q / ns) * ns * R + (q & (ns - 1)) + int64_t(m) * ns] = sm[t * (R + 1) + m];
        }
    }
}

template <int LOGR>
int launch_pass(const double2* in, double2* out, int log_n, int64_t batch, int64_t ns, const Tables& tb,
                cudaStream_t st) {
    constexpr int R = 1 << LOGR;
    constexpr int TILE = kTilePoints / R;
    const size_t smem = size_t(TILE) * (R + 1) * sizeof(double2);
    const int64_t cols = batch << (log_n - LOGR);
    const int64_t blocks = (cols + TILE - 1) / TILE;
    if (blocks > 0x7FFFFFFFLL) return set_error(KK_ERR_PARAM, "fft: transform too large");
    if (cols % TILE == 0) {
        if (ensure_smem_attr(reinterpret_cast<const void*>(&fft_pass_kernel<LOGR, true>), smem, "fft_pass_kernel") !=
            KK_OK)
            return KK_ERR_CUDA;
        fft_pass_kernel<LOGR, true><<<static_cast<unsigned>(blocks), kThreads, smem, st>>>(in, out, log_n, ns, cols, tb);
    } else {
        if (ensure_smem_attr(reinterpret_cast<const void*>(&fft_pass_kernel<LOGR, false>), smem, "fft_pass_kernel") !=
            KK_OK)
            return KK_ERR_CUDA;
        fft_pass_kernel<LOGR, false><<<static_cast<unsigned>(blocks), kThreads, smem, st>>>(in, out, log_n, ns, cols,
                                                                                           tb);
    }
    return check_launch("fft_pass_kernel");
}

int forward_pow2(double2* a, double2* b, int log_n, int64_t batch, const void* tables, cudaStream_t st,
                 double2** result) {
    if (log_n < 1 || log_n > 31) return set_error(KK_ERR_PARAM, "fft: length must be 2^1 .. 2^31");
    const Tables tb = tables_at(tables, log_n);
    const int npass = (log_n + 9) / 10;
    int64_t ns = 1;
    double2 *src = a, *dst = b;
    int rc = KK_OK;
    for (int i = 0; i < npass && rc == KK_OK; ++i) {
        const int lr = log_n / npass + (i < log_n % npass ? 1 : 0);
        switch (lr) {
            case 1: rc = launch_pass<1>(src, dst, log_n, batch, ns, tb, st); break;
            case 2: rc = launch_pass<2>(src, dst, log_n, batch, ns, tb, st); break;
            case 3: rc = launch_pass<3>(src, dst, log_n, batch, ns, tb, st); break;
            case 4: rc = launch_pass<4>(src, dst, log_n, batch, ns, tb, st); break;
            case 5: rc = launch_pass<5>(src, dst, log_n, batch, ns, tb, st); break;
            case 6: rc = launch_pass<6>(src, dst, log_n, batch, ns, tb, st); break;
            case 7: rc = launch_pass<7>(src, dst, log_n, batch, ns, tb, st); break;
            case 8: rc = launch_pass<8>(src, dst, log_n, batch, ns, tb, st); break;
            case 9: rc = launch_pass<9>(src, dst, log_n, batch, ns, tb, st); break;
            case 10: rc = launch_pass<10>(src, dst, log_n, batch, ns, tb, st); break;
            default: rc = set_error(KK_ERR_PARAM, "fft: bad pass radix");
        }
        ns <<= lr;
        std::swap(src, dst);
    }
    *result = src;
    return rc;
}

// ---------------------------------------------------------------------------
// Any-length transforms (rows of n points, in place in `x`)
// ---------------------------------------------------------------------------
inline int log2_ceil(int64_t v) {
    int l = 0;
    while ((int64_t(1) << l) < v) ++l;
    return l;
}
inline bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

struct AnyPlan {
    int64_t n = 0, batch = 0, m = 0;   // m: power-of-two transform length
    int log_m = 0;
    bool blue = false;
    size_t off_a = 0, off_b = 0, off_chirp = 0, off_bspec = 0, off_tab = 0, total = 0;
};

inline AnyPlan plan_any(int64_t n, int64_t batch) {
    AnyPlan p;
    p.n = n;
    p.batch = batch;
    p.blue = !is_pow2(n) || n < 2;
    p.m = p.blue ? (int64_t(1) << std::max(1, log2_ceil(2 * n - 1))) : n;
    p.log_m = log2_ceil(p.m);
    const size_t rows = size_t(batch) * size_t(p.m) * sizeof(double2);
    p.off_a = 0;
    p.off_b = al(rows);
    p.off_chirp = p.off_b + al(rows);
    p.off_bspec = p.off_chirp + (p.blue ? al(size_t(n) * sizeof(double2)) : 0);
    p.off_tab = p.off_bspec + (p.blue ? al(size_t(p.m) * sizeof(double2)) : 0);
    p.total = p.off_tab + table_bytes(p.log_m);
    return p;
}

// dst[r][j] = (conj_in ? conj : id)(src[r][j]) * (chirp ? chirp[j] : 1), zero
// padded from n to m per row
__global__ void load_rows_kernel(const double2* __restrict__ src, double2* __restrict__ dst, int64_t n, int64_t m,
                                 int64_t batch, int conj_in, const double2* __restrict__ chirp) {
    const int64_t total = batch * m;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / m, j = i - r * m;
        double2 v = make_double2(0.0, 0.0);
        if (j < n) {
            v = src[r * n + j];
            if (conj_in) v = cconj(v);
            if (chirp) v = cmul(v, chirp[j]);
        }
        dst[i] = v;
    }
}

// dst[r][k] = post(src[r][k]) for k < n: optional chirp multiply, conj, scale
__global__ void store_rows_kernel(const double2* __restrict__ src, double2* __restrict__ dst, int64_t n, int64_t m,
                                  int64_t batch, const double2* __restrict__ chirp, int conj_out, double scale) {
    const int64_t total = batch * n;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / n, k = i - r * n;
        double2 v = src[r * m + k];
        if (chirp) v = cmul(v, chirp[k]);
        if (conj_out) v = cconj(v);
        dst[i] = make_double2(v.x * scale, v.y * scale);
    }
}

// w[j] = exp(-i pi (j^2 mod 2n) / n)
__global__ void chirp_kernel(double2* __restrict__ w, int64_t n) {
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x) {
        const unsigned long long jj = static_cast<unsigned long long>(j);
        const unsigned long long r = (jj * jj) % (2ull * static_cast<unsigned long long>(n));   // j < 2^31
        double s, c;
        sincospi(double(r) / double(n), &s, &c);
        w[j] = make_double2(c, -s);
    }
}

// b[j] = conj w[|j|] for |j| < n (wrapped mod m), 0 elsewhere
__global__ void bluestein_b_kernel(const double2* __restrict__ w, double2* __restrict__ b, int64_t n, int64_t m) {
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m; j += int64_t(gridDim.x) * blockDim.x) {
        double2 v = make_double2(0.0, 0.0);
        if (j < n) v = cconj(w[j]);
        else if (m - j < n) v = cconj(w[m - j]);
        b[j] = v;
    }
}

// a[r][k] = conj(a[r][k] * bspec[k])   (the next forward FFT is the inverse)
__global__ void spec_mul_conj_kernel(double2* __restrict__ a, const double2* __restrict__ bs, int64_t m,
                                     int64_t batch) {
    const int64_t total = batch * m;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x)
        a[i] = cconj(cmul(a[i], bs[i & (m - 1)]));
}

// Transform `batch` rows of n points from x into y (x == y allowed).
// prepared: the twiddle tables (and, for Bluestein lengths, the chirp and its
// spectrum) are already in ws from an earlier call with the same n (the
// split-step loop runs four transforms of one length per step).
int transform(const double2* x, double2* y, int64_t n, int64_t batch, bool inverse, void* ws, size_t ws_bytes,
              cudaStream_t st, bool prepared = false) {
    const AnyPlan p = plan_any(n, batch);
    if (p.log_m > 31) return set_error(KK_ERR_PARAM, "fft: length too large");
    if (!ws || ws_bytes < p.total) return set_error(KK_ERR_PARAM, "fft: workspace too small");
    char* base = static_cast<char*>(ws);
    double2* a = reinterpret_cast<double2*>(base + p.off_a);
    double2* b = reinterpret_cast<double2*>(base + p.off_b);
    void* tab = base + p.off_tab;
    int rc = prepared ? KK_OK : build_tables(tab, p.log_m, st);
    if (rc != KK_OK) return rc;
    const unsigned g = grid_for(p.batch * p.m, 256);
    double2* res = nullptr;
    if (!p.blue) {
        load_rows_kernel<<<g, 256, 0, st>>>(x, a, n, n, batch, inverse ? 1 : 0, nullptr);
        if ((rc = check_launch("fft load_rows_kernel")) != KK_OK) return rc;
        if ((rc = forward_pow2(a, b, p.log_m, batch, tab, st, &res)) != KK_OK) return rc;
        store_rows_kernel<<<g, 256, 0, st>>>(res, y, n, n, batch, nullptr, inverse ? 1 : 0,
                                             inverse ? 1.0 / double(n) : 1.0);
        return check_launch("fft store_rows_kernel");
    }
    double2* w = reinterpret_cast<double2*>(base + p.off_chirp);
    double2* bs = reinterpret_cast<double2*>(base + p.off_bspec);
    if (!prepared) {
        chirp_kernel<<<grid_for(n, 256), 256, 0, st>>>(w, n);
        if ((rc = check_launch("fft chirp_kernel")) != KK_OK) return rc;
        // chirp spectrum: one row in a, transformed into bs
        bluestein_b_kernel<<<grid_for(p.m, 256), 256, 0, st>>>(w, a, n, p.m);
        if ((rc = check_launch("fft bluestein_b_kernel")) != KK_OK) return rc;
        if ((rc = forward_pow2(a, b, p.log_m, 1, tab, st, &res)) != KK_OK) return rc;
        if (cudaMemcpyAsync(bs, res, size_t(p.m) * sizeof(double2), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return set_cuda_error("fft bluestein copy");
    }
    load_rows_kernel<<<g, 256, 0, st>>>(x, a, n, p.m, batch, inverse ? 1 : 0, w);
    if ((rc = check_launch("fft load_rows_kernel")) != KK_OK) return rc;
    if ((rc = forward_pow2(a, b, p.log_m, batch, tab, st, &res)) != KK_OK) return rc;
    spec_mul_conj_kernel<<<g, 256, 0, st>>>(res, bs, p.m, batch);
    if ((rc = check_launch("fft spec_mul_conj_kernel")) != KK_OK) return rc;
    double2* other = res == a ? b : a;
    if ((rc = forward_pow2(res, other, p.log_m, batch, tab, st, &res)) != KK_OK) return rc;
    // res = M * conj(conv); X = w * conv = w * conj(res) / M (inverse: conj(X) / n)
    store_rows_kernel<<<grid_for(p.batch * n, 256), 256, 0, st>>>(res, y, n, p.m, batch, nullptr, 1, 1.0);
    if ((rc = check_launch("fft store_rows_kernel")) != KK_OK) return rc;
    // y = conj(res); now the chirp, 1 / M (and the inverse's conj and 1 / n) in place
    store_rows_kernel<<<grid_for(p.batch * n, 256), 256, 0, st>>>(y, y, n, n, batch, w, inverse ? 1 : 0,
                                                                   (1.0 / double(p.m)) *
                                                                       (inverse ? 1.0 / double(n) : 1.0));
    return check_launch("fft store_rows_kernel");
}

// ---------------------------------------------------------------------------
// Split-step Fourier span (channel.py ssfm_span :124-158)
// ---------------------------------------------------------------------------
// lin[k] = exp(-1j * a_half * f * f), f = numpy.fft.fftfreq(n, 1 / fs)[k]
__global__ void ssfm_lin_kernel(double2* __restrict__ lin, int64_t n, double val, double a_half) {
    const int64_t npos = (n - 1) / 2 + 1;
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const double f = double(k < npos ? k : k - n) * val;
        const double th = (-a_half * f) * f;
        double s, c;
        sincos(th, &s, &c);
        lin[k] = make_double2(c, s);
    }
}

__global__ void cmul_inplace_kernel(double2* __restrict__ x, const double2* __restrict__ h, int64_t n) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x)
        x[k] = cmul(x[k], h[k]);
}

// x *= exp(1j * gamma * (|x|^2 * 1e-3) * l_eff)
__global__ void ssfm_nl_kernel(double2* __restrict__ x, int64_t n, double gamma, double l_eff) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const double2 v = x[k];
        const double a = hypot(v.x, v.y);
        const double th = (gamma * ((a * a) * 1e-3)) * l_eff;
        double s, c;
        sincos(th, &s, &c);
        x[k] = cmul(v, make_double2(c, s));
    }
}

__global__ void scale_kernel(double2* __restrict__ x, int64_t n, double s) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const double2 v = x[k];
        x[k] = make_double2(v.x * s, v.y * s);
    }
}

}  // namespace fft64
}  // namespace kk

extern "C" size_t kk_fft_workspace_bytes(int64_t n, int64_t batch) {
    if (n <= 0 || batch <= 0) return 0;
    const kk::fft64::AnyPlan p = kk::fft64::plan_any(n, batch);
    return p.log_m > 31 ? 0 : p.total;
}

extern "C" int kk_fft(const void* in, void* out, int64_t n, int64_t batch, int inverse, void* ws, size_t ws_bytes,
                      void* stream) {
    kk::clear_error();
    if (n <= 0 || batch <= 0 || !in || !out) return kk::set_error(KK_ERR_PARAM, "kk_fft: bad arguments");
    return kk::fft64::transform(static_cast<const double2*>(in), static_cast<double2*>(out), n, batch, inverse != 0,
                                ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

extern "C" size_t kk_ssfm_workspace_bytes(int64_t n) {
    if (n <= 0) return 0;
    const size_t f = kk_fft_workspace_bytes(n, 1);
    return f ? f + kk::fft64::al(size_t(n) * sizeof(double2)) : 0;
}

extern "C" int kk_ssfm_span(void* x, int64_t n, double sample_rate_hz, int n_steps, double a_half,
                            double gamma_per_w_km, double l_eff_km, double loss_amp, void* ws, size_t ws_bytes,
                            void* stream) {
    using namespace kk;
    using namespace kk::fft64;
    clear_error();
    if (n <= 0 || !x || n_steps < 1 || !(sample_rate_hz > 0))
        return set_error(KK_ERR_PARAM, "kk_ssfm_span: bad arguments");
    const size_t need = kk_ssfm_workspace_bytes(n);
    if (!need || !ws || ws_bytes < need) return set_error(KK_ERR_PARAM, "kk_ssfm_span: workspace too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    double2* lin = static_cast<double2*>(ws);
    char* fws = static_cast<char*>(ws) + al(size_t(n) * sizeof(double2));
    const size_t fbytes = ws_bytes - al(size_t(n) * sizeof(double2));
    double2* v = static_cast<double2*>(x);
    const unsigned g = grid_for(n, 256);
    // numpy.fft.fftfreq: k * (1 / (n * d)), d = 1 / fs
    const double val = 1.0 / (double(n) * (1.0 / sample_rate_hz));
    ssfm_lin_kernel<<<g, 256, 0, st>>>(lin, n, val, a_half);
    int rc = check_launch("ssfm_lin_kernel");
    for (int s = 0; s < n_steps && rc == KK_OK; ++s) {
        // the first transform prepares the tables / chirp in the workspace
        if ((rc = transform(v, v, n, 1, false, fws, fbytes, st, s > 0)) != KK_OK) break;
        cmul_inplace_kernel<<<g, 256, 0, st>>>(v, lin, n);
        if ((rc = check_launch("ssfm cmul_inplace_kernel")) != KK_OK) break;
        if ((rc = transform(v, v, n, 1, true, fws, fbytes, st, true)) != KK_OK) break;
        ssfm_nl_kernel<<<g, 256, 0, st>>>(v, n, gamma_per_w_km, l_eff_km);
        if ((rc = check_launch("ssfm_nl_kernel")) != KK_OK) break;
        if ((rc = transform(v, v, n, 1, false, fws, fbytes, st, true)) != KK_OK) break;
        cmul_inplace_kernel<<<g, 256, 0, st>>>(v, lin, n);
        if ((rc = check_launch("ssfm cmul_inplace_kernel")) != KK_OK) break;
        if ((rc = transform(v, v, n, 1, true, fws, fbytes, st, true)) != KK_OK) break;
        scale_kernel<<<g, 256, 0, st>>>(v, n, loss_amp);
        rc = check_launch("ssfm scale_kernel");
    }
    return rc;
}
