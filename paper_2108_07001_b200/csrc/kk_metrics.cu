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
// The correlation: z = (2rx - 1) + j reverse(2tx - 1), zero padded to N =
// 2^n >= the correlation length; Z = FFT(z) (kk_fft.cu's float64 Stockham
// passes); conj(A B) formed from Z(f), Z(-f) in one pass; a second forward
// FFT gives N * conv in the real parts; two reduction passes find the peak
// (first index of the max |c|) and the largest sidelobe.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kk_internal.h"

namespace kk {
namespace xc {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

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
    int log_n = 0;
    int64_t n = 0;
    size_t off_b = 0, off_tab = 0, off_red = 0, total = 0;
};

inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

inline bool make_plan(int64_t n_rx, int64_t n_tx, int circular, Plan& p) {
    const int64_t len = circular ? 2 * n_rx - 1 : n_rx + n_tx - 1;
    int log_n = 12;
    while ((int64_t(1) << log_n) < len) ++log_n;
    if (log_n > 31) return false;
    p.log_n = log_n;
    p.n = int64_t(1) << log_n;
    const size_t buf = size_t(p.n) * sizeof(double2);
    p.off_b = al(buf);
    p.off_tab = p.off_b + al(buf);
    p.off_red = p.off_tab + al(fft64::table_bytes(log_n));
    p.total = p.off_red + 256;
    return true;
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

// Deterministic two-stage sums (fixed grid, fixed combination order): the
// EVM of a run is bit-identical from run to run.
constexpr int kEvmBlocks = 512;

__global__ void evm_partials_kernel(const float2* __restrict__ soft, const double2* __restrict__ ref, int64_t n,
                                    double* __restrict__ part) {
    __shared__ double s_e[8], s_r[8];
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
        s_e[threadIdx.x >> 5] = se;
        s_r[threadIdx.x >> 5] = sr;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < 8; ++w) {
            a += s_e[w];
            b += s_r[w];
        }
        part[2 * blockIdx.x] = a;
        part[2 * blockIdx.x + 1] = b;
    }
}

__global__ void evm_final_kernel(const double* __restrict__ part, int nb, double* __restrict__ sums) {
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int i = 0; i < nb; ++i) {
            a += part[2 * i];
            b += part[2 * i + 1];
        }
        sums[0] += a;
        sums[1] += b;
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
    void* tab = base + p.off_tab;
    unsigned long long* red = reinterpret_cast<unsigned long long*>(base + p.off_red);
    if (cudaMemsetAsync(red, 0, 2 * sizeof(unsigned long long), st) != cudaSuccess)
        return set_cuda_error("kk_bit_xcorr memset");
    int rc = fft64::build_tables(tab, p.log_n, st);
    if (rc != KK_OK) return rc;
    pack_kernel<<<grid_for(p.n, 256), 256, 0, st>>>(rx, n_rx, tx, n_tx, a, p.n);
    if ((rc = check_launch("xcorr pack_kernel")) != KK_OK) return rc;
    double2* z = nullptr;
    if ((rc = fft64::forward_pow2(a, b, p.log_n, 1, tab, st, &z)) != KK_OK) return rc;
    product_kernel<<<grid_for(p.n / 2 + 1, 256), 256, 0, st>>>(z, p.n);
    if ((rc = check_launch("xcorr product_kernel")) != KK_OK) return rc;
    double2* y = nullptr;
    if ((rc = fft64::forward_pow2(z, z == a ? b : a, p.log_n, 1, tab, st, &y)) != KK_OK) return rc;
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

extern "C" int kk_evm_sums(const void* soft, const void* ref, int64_t n, double* sums, double* scratch,
                           void* stream) {
    using namespace kk;
    clear_error();
    if (n < 0 || !sums || (n > 0 && (!soft || !ref || !scratch)))
        return set_error(KK_ERR_PARAM, "kk_evm_sums: bad arguments");
    if (n == 0) return KK_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int nb = static_cast<int>(std::min<int64_t>(kEvmBlocks, (n + 255) / 256));
    evm_partials_kernel<<<nb, 256, 0, st>>>(static_cast<const float2*>(soft), static_cast<const double2*>(ref), n,
                                            scratch);
    int rc = check_launch("evm_partials_kernel");
    if (rc != KK_OK) return rc;
    evm_final_kernel<<<1, 32, 0, st>>>(scratch, nb, sums);
    return check_launch("evm_final_kernel");
}
