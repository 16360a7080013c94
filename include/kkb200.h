/*
 * kkb200.h -- C ABI of libkkb200.so, the B200 (sm_100a) Kramers-Kronig
 * receiver hot path.  Plain pointers, sizes and a cudaStream_t passed as
 * void*; no C++ or torch types cross this boundary; no exceptions.
 *
 * The reference (`kkmodem`, /root/reference/pkg/src/kkmodem) is pure Python
 * and has no FFI of its own: its plugin surface is the Python API of
 * kkmodem.rxdsp consumed by kkmodem/harness/runner.py:16-24.  Each entry
 * point below replaces one reference function (cited as rxdsp.py:line etc.);
 * paper_2108_07001_b200/rxdsp.py re-exposes the reference's Python surface
 * on top of these calls (ctypes), and INTEGRATION.md shows the binding a
 * kkmodem maintainer would add.
 *
 * Conventions
 *   - every entry point returns an int status: KK_OK, or KK_ERR_PARAM
 *     (-> ParameterError, sigcore.py:37), KK_ERR_SYNC (-> SyncError,
 *     rxdsp.py:63), KK_ERR_CUDA / KK_ERR_INTERNAL (-> RuntimeError);
 *     kk_last_error() returns the thread-local message of the last failure.
 *   - all array pointers are DEVICE pointers unless named *_host; complex
 *     arrays are interleaved float32 (re, im) = complex64.
 *   - the library owns only immutable per-device twiddle tables (built once,
 *     std::call_once); all streaming state lives in caller buffers.
 *   - entry points are reentrant across pipelines and devices; calls on one
 *     pipeline must be serialised by the caller (one stream).
 */
#ifndef KKB200_H
#define KKB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KK_ABI_VERSION 2

#define KK_OK 0
#define KK_ERR_PARAM 1
#define KK_ERR_SYNC 2
#define KK_ERR_CUDA 3
#define KK_ERR_INTERNAL 4

#define KK_DTYPE_I16 0 /* ADC codes; value = code * in_scale (odd half-LSB codes) */
#define KK_DTYPE_F32 1
#define KK_DTYPE_F64 2
/* packed 12-bit ADC codes c, two per 3 bytes little-endian (byte0 = c0[7:0],
 * byte1 = c0[11:8] | c1[3:0] << 4, byte2 = c1[11:4]); value = (2c + 1) *
 * in_scale (the int16 path's odd half-LSB code h = 2c + 1).  1.5 B/sample.
 * The buffer must be 4-byte aligned.  B200 addition (the reference's raw format is int16, sigcore.py:357) */
#define KK_DTYPE_P12 3
/* or-ed into in_dtype of kk_reconstruct_pairs: correctly rounded
 * logf/expf/sincosf instead of the SFU approximations (functional API) */
#define KK_DTYPE_PRECISE 0x100

const char *kk_last_error(void);
int kk_version(void);
int kk_device_sync(void);
/* number of kernels this library has launched (process-wide counter) */
unsigned long long kk_launch_count(void);
/* measured FP32 FFMA throughput of the current device (FLOP/s), for the
 * roofline of the FP32-bound FFT kernels */
int kk_fma_peak(double *flops_per_s_host, void *stream);
/* Stream-ordered host->device upload of a small host buffer through kernel
 * parameters (16 KB per launch): unlike a DMA copy it never queues behind
 * bulk host->device transfers already in flight.  The host buffer may be
 * reused on return.  (B200 addition; the reference has no device.) */
int kk_upload(void *dst_dev, const void *src_host, int64_t bytes, void *stream);

/*
 * K1 kk_fused -- replaces rxdsp.py:184-244 `kk_reconstruct` (+ the downshift
 * rxdsp.py:247-257 / :690-696 and the carrier segment sums rxdsp.py:685-687).
 * Processes n_hops hops of 512 ADC samples in pairs (hop 2p, 2p+1 of this
 * call).  State in/out = the reference state dict: u_tail[512] (float),
 * a_hist[256] (float), dead_hist[256] (uint8).  Output out[n_hops*512] is
 * the field, rotated by the downshift (sigcore.py frequency_shift :286-299 by
 * -tone) at global index g = n0_global + i, conjugated when mirror != 0:
 * rot_q > 0: exp(-2 pi i (rot_p*g mod rot_q)/rot_q) (tone/fs = rot_p/rot_q,
 * rot_q <= 1024, rot_tab[a] = exp(-2 pi i a/rot_q)); rot_q == 0 and
 * rot_step != 0: any tone, exp(-2 pi i (g*rot_step mod 2^64)/2^64) with
 * rot_step = tone/fs as a 64-bit fixed-point fraction; both 0: none.
 * hop_sum[n_hops]: per-hop sum of the (unrotated) field; hop_dead[n_hops];
 * clamped: += clamped-sample count.  clamp_rel: rxdsp.py:188 (1e-12).
 */
int kk_reconstruct_pairs(int in_dtype, const void *in, float in_scale, float clamp_rel, int64_t n_hops,
                         const float *st_u, const float *st_a, const uint8_t *st_dead,
                         float *new_u, float *new_a, uint8_t *new_dead, void *out,
                         void *hop_sum, uint8_t *hop_dead, unsigned long long *clamped,
                         int64_t n0_global, int rot_p, int rot_q, const void *rot_tab,
                         unsigned long long rot_step, int mirror, void *stream);

/*
 * Batched K1 (B200 addition): independent streams (sweep
 * points) in one launch; every job is one kk_reconstruct_pairs call (same
 * argument meaning), all with the same in_dtype.  The job array is host
 * memory (copied into the launch).
 */
typedef struct {
    const void *in;
    float in_scale;
    float clamp_rel;
    int64_t n_hops;
    const float *st_u;
    const float *st_a;
    const uint8_t *st_dead;
    float *new_u;
    float *new_a;
    uint8_t *new_dead;
    void *out;
    void *hop_sum;
    uint8_t *hop_dead;
    unsigned long long *clamped;
    int64_t n0_global;
    int rot_p;
    int rot_q;
    const void *rot_tab;
    unsigned long long rot_step;
    int mirror;
} kk_k1_job;
int kk_reconstruct_pairs_batch(int in_dtype, const kk_k1_job *jobs, int n_jobs, void *stream);

/*
 * Standalone downshift (downshift_dc rx:247-257 = frequency_shift
 * sigcore.py:286-299 by -tone), complex128 in/out (x == y allowed):
 * y[i] = x[i] exp(j ((two_pi_df (start_index + i)) / fs)), two_pi_df =
 * 2 pi delta_f as the caller forms it.
 */
int kk_frequency_shift(const void *x, void *y, int64_t n, double two_pi_df, double fs, int64_t start_index,
                       void *stream);

/* packed 12-bit codes (KK_DTYPE_P12 layout, n even) -> int16 odd codes h */
int kk_unpack12(const uint8_t *in, int64_t n, int16_t *out, void *stream);

/*
 * Carrier means -- replaces the per-segment np.mean of rxdsp.py:685-687.
 * mean[s] = sum(hop_sum[s*hps .. (s+1)*hps)) / len, len = seg_len, or
 * last_len for the final (flush-partial) segment when last_len > 0.
 */
int kk_carrier_means(const void *hop_sum, int64_t n_segs, int hops_per_seg, int64_t n_hops_avail,
                     int64_t last_len, int seg_len, void *mean, void *stream);

/*
 * K2 static_fused -- replaces rxdsp.py:698-720 `_run_static`
 * (== :414-453 `static_equalize_and_resample`) fused with the carrier
 * subtraction rxdsp.py:687.  Block hb (global static hop, 16384 samples)
 * reads s[16384(hb-1) .. 16384(hb+1)) where s = z - conj(mean*rot)
 * (mirror) and writes 8192 2-sps outputs.  h_even/h_odd: the response
 * _static_response (rxdsp.py:401-411) at even / odd kept indices.  The
 * rotation arguments mean what they mean for kk_reconstruct_pairs.
 */
int kk_static_blocks(const void *z, int64_t z_index0, int64_t hb0, int64_t n_blocks, int64_t valid_end,
                     const void *seg_mean, int64_t seg_index0, int seg_len, int carrier, int rot_p,
                     int rot_q, const void *rot_tab, unsigned long long rot_step, int mirror,
                     const void *h_even, const void *h_odd, void *out, void *stream);

/* Batched K2 (B200 addition): one job per stream, each a
 * kk_static_blocks call with the same argument meaning; host job array. */
typedef struct {
    const void *z;
    int64_t z_index0;
    int64_t hb0;
    int64_t n_blocks;
    int64_t valid_end;
    const void *seg_mean;
    int64_t seg_index0;
    int seg_len;
    int carrier;
    int rot_p;
    int rot_q;
    const void *rot_tab;
    unsigned long long rot_step;
    int mirror;
    const void *h_even;
    const void *h_odd;
    void *out;
} kk_k2_job;
int kk_static_blocks_batch(const kk_k2_job *jobs, int n_jobs, void *stream);

/*
 * K3 sync -- replaces rxdsp.py:574-601 `symbol_sync` and the eq_scale RMS of
 * rxdsp.py:734-737.  result_host[4] = {parity, k, peak-to-rms ratio,
 * rms(head[skip:])}; offset = 2k + parity.  Blocking (one stream sync).
 */
size_t kk_symbol_sync_scratch_bytes(int64_t n_head, int n_ref);
/* Non-blocking form: enqueues the same kernels on `stream`; the 4 result
 * doubles are written to result (device memory or UVA-mapped pinned host
 * memory) when they complete (B200 addition: the pipeline keeps the device
 * busy with the rest of the front end while the host waits for the sync). */
int kk_symbol_sync_enqueue(const void *head, int64_t n_head, const void *ref, int n_ref, int64_t skip,
                           double *result, void *scratch, size_t scratch_bytes, void *stream);
int kk_symbol_sync(const void *head, int64_t n_head, const void *ref, int n_ref, int64_t skip,
                   double *result_host, void *scratch, size_t scratch_bytes, void *stream);

/*
 * K4 sequential chain -- replaces rxdsp.py:460-499 `_ddlms_core` exactly
 * (complex form, fp32): used by the functional ddlms_wl API (rxdsp.py:510),
 * non-widely-linear mode and exact fallbacks.  wg[2*n_taps] complex = w, g;
 * fz[2] = {frozen, div_count}; both updated in place.  Constellation tables
 * are host arrays: pts_host[2*order] (re, im), grid_host[grid_m^2] maps
 * (i_re*m + i_im) -> point index for square QAM (grid_m = 0: brute force).
 */
int kk_ddlms_sequential(const void *x, int64_t n_out, float scale, int n_taps, const void *train,
                        int64_t n_train, void *wg, int *fz, int order, const float *pts_host,
                        const uint8_t *grid_host, int grid_m, float norm, float max_radius,
                        float guard_factor, int guard_run, float mu, int widely_linear,
                        uint8_t *labels, void *soft, void *dec, void *stream);

/*
 * K4 exact block-parallel WL DDLMS (4 taps) -- same results as the
 * sequential recurrence rxdsp.py:465-498 (speculative affine prefix scan to
 * the certified fixpoint).  T_init_host / T_final_host: float[16], the WL
 * taps in real 2x8 form.  stats_host[6] = {iterations, blocks re-run,
 * fallback (0 none, 1 guard exceeded -> caller re-runs sequentially,
 * 2 not converged -> chained), guard exceedances, changed blocks in the
 * last iteration, blocks, then for iterations 1..16: (changed blocks,
 * re-run blocks)}: the buffer must hold 38 int64.
 */
size_t kk_ddlms_workspace_bytes(int64_t nsym, int block);
int kk_ddlms_solve(const void *x, int64_t nsym, float scale, const void *train, int64_t n_train,
                   const float *T_init_host, int order, const float *pts_host, const uint8_t *grid_host,
                   int grid_m, float norm, float max_radius, float guard_factor, int guard_run,
                   float mu, int block, int max_iter, float soft_tol, uint8_t *labels, void *soft,
                   float *T_final_host, void *workspace, size_t ws_bytes, int64_t *stats_host,
                   void *stream);

/*
 * K4 asynchronous form of kk_ddlms_solve (B200 addition): everything is
 * enqueued on `stream`, nothing is read back, so the host can queue the next
 * frame / stream while this one runs.  The fixpoint loop runs as a CUDA-graph
 * WHILE node.  widely_linear = 0: the linear equaliser (rxdsp.py:491-497 with
 * g = 0; T keeps the form T1 = T0 M).  T_io: device float[16], the frame's start taps in, its end taps
 * out (real 2x8 form); state_io: device int[2] {frozen, div_count} in/out
 * (rxdsp.py:484-490 guard state); stats_out: device or mapped pinned host
 * int64[38] (layout of kk_ddlms_solve's stats; [2] = fallback taken: 1 exact
 * sequential chain on the device, 2 not converged -> chained), may be NULL.
 * The workspace must stay allocated until the enqueued work completes.
 * max_iter < 0: cap |max_iter|, and the loop runs as host-driven batches with
 * readbacks instead of a graph (blocks the calling thread; for worker threads
 * that solve frames while other streams stream input: instantiating a graph
 * allocates device memory, which serialises concurrent streams).
 */
int kk_ddlms_solve_async(const void *x, int64_t nsym, float scale, const void *train, int64_t n_train,
                         float *T_io, int *state_io, int order, const float *pts_host, const uint8_t *grid_host,
                         int grid_m, float norm, float max_radius, float guard_factor, int guard_run, float mu,
                         int widely_linear, int block, int max_iter, float soft_tol, uint8_t *labels, void *soft,
                         void *workspace, size_t ws_bytes, int64_t *stats_out, void *stream);

/*
 * K4 as a phased solver over one frame, so frames on different GPUs can be
 * chained exactly (superframe sharding): the host exchanges
 * frame maps (P, Q) -- T_end = T_start P + Q, map_host = float[64 + 16] --
 * between ranks.  kk_ddlms_create carves the caller's workspace
 * (kk_ddlms_workspace_bytes) and returns an opaque handle (NULL on error).
 *   train(T_start)      exact pure-training blocks -> training-end taps
 *   speculate(T_guess)  first pass of the decision-directed blocks -> map
 *   iterate(T_start)    exact frame-start taps: re-run blocks whose decision
 *                       margin the start move could cross (soft_pass: also
 *                       those whose soft outputs would move > soft_tol);
 *                       changed blocks -> map
 *   finish              labels / soft / end taps / guard exceedances
 * kk_ddlms_bind_outputs (optional, before the final iterate) makes the final
 * pass write labels / soft straight into the caller's device arrays; finish
 * then copies nothing when given the same pointers.
 */
void *kk_ddlms_create(const void *x, int64_t nsym, float scale, const void *train, int64_t n_train, int order,
                      const float *pts_host, const uint8_t *grid_host, int grid_m, float norm, float max_radius,
                      float guard_factor, float mu, int block, float soft_tol, void *workspace, size_t ws_bytes,
                      void *stream);
int kk_ddlms_train(void *solver, const float *T_start_host, float *T_train_end_host);
int kk_ddlms_speculate(void *solver, const float *T_guess_host, float *map_host);
int kk_ddlms_iterate(void *solver, const float *T_start_host, int soft_pass, int64_t *changed_blocks,
                     int64_t *rerun_blocks, float *map_host);
int kk_ddlms_bind_outputs(void *solver, uint8_t *labels, void *soft);
int kk_ddlms_finish(void *solver, uint8_t *labels, void *soft, float *T_final_host, int64_t *guard_exceed);
void kk_ddlms_destroy(void *solver);

/*
 * BER -- replaces demap (rxdsp.py:548-567) + the XOR count of
 * runner.py:360-362: total += popcount(label[lab[i]] ^ label[ref[i]]);
 * win[i / win_syms] += the same (win may be NULL when win_syms <= 0).
 * Symbols with (i + ex_phase) mod ex_period >= ex_period - ex_len are
 * skipped when ex_period > 0 (tile seams of a tiled capture);
 * n_counted (may be NULL) += symbols counted.
 */
int kk_bit_errors(const uint8_t *labels, const uint8_t *ref_idx, int64_t n, const uint8_t *point_label,
                  int64_t win_syms, unsigned long long *total, unsigned int *win, int64_t ex_period,
                  int64_t ex_len, int64_t ex_phase, unsigned long long *n_counted, void *stream);

/*
 * demap -- nearest constellation point of rxdsp.py:560-565 (first minimum
 * wins): idx[i] = point index; n_fallback += count of inputs that are not
 * exactly a constellation point.
 */
int kk_demap(const void *symbols, int64_t n, int order, const float *pts_host, uint8_t *idx,
             unsigned long long *n_fallback, void *stream);

/*
 * Receiver output bits -- decided labels demapped (rxdsp.py:548-567 bit
 * order) and packed MSB first (np.packbits layout): out[(n*k + 7) / 8].
 * Label 255 (training) takes train_idx[sym0 + i] when sym0 + i < n_train.
 */
int kk_pack_bits(const uint8_t *labels, int64_t n, int64_t sym0, const uint8_t *train_idx, int64_t n_train,
                 int bits_per_symbol, const uint8_t *point_label_host, int order, uint8_t *out, void *stream);

/*
 * frame_sync's bipolar cross-correlation (metrics.py frame_sync :69-112)
 * over all lags, on the device: rx / tx are 0/1 bytes.  Linear (circular=0):
 * c = conv(2rx-1, reverse(2tx-1)) of length n_rx + n_tx - 1 (scipy
 * fftconvolve "full" indexing); circular (circular=1, n_rx == n_tx): c[k] =
 * sum_i (2rx[i+k mod n]-1)(2tx[i]-1).  Evaluated with float64 FFTs rounded
 * to the exact integers.  out3 (device, int64[3]) = {k = first index of
 * max |c|, |c[k]|, max |c| outside [k-2, k+2] (linear) / outside k
 * (circular)}; the caller forms the peak ratio and the alignment as the
 * reference does.  ws: kk_bit_xcorr_workspace_bytes() bytes of device
 * memory (32 B per FFT point plus tables; 0 = unsupported size).
 */
size_t kk_bit_xcorr_workspace_bytes(int64_t n_rx, int64_t n_tx, int circular);
int kk_bit_xcorr(const uint8_t *rx, int64_t n_rx, const uint8_t *tx, int64_t n_tx, int circular, void *ws,
                 size_t ws_bytes, long long *out3, void *stream);

/*
 * Decided labels -> one byte per bit (rxdsp.py demap :548-567 bit order,
 * MSB first): out[i*k + b] = (point_label[labels[i]] >> (k-1-b)) & 1.
 */
int kk_label_bits(const uint8_t *labels, int64_t n, const uint8_t *point_label_host, int order,
                  int bits_per_symbol, uint8_t *out, void *stream);

/*
 * Bit errors of two aligned bit streams (runner.py measure_point :104-137):
 * total += count(a[i] != b[i]); win_counts[w] += the errors of bits
 * [w*bpw, (w+1)*bpw) for the n / bpw whole windows (metrics.py windowed_q
 * :130-150; win_counts may be NULL).  Counters are accumulated, not reset.
 */
int kk_bit_error_windows(const uint8_t *a, const uint8_t *b, int64_t n, int64_t bits_per_window,
                         unsigned long long *total, unsigned long long *win_counts, void *stream);

/*
 * EVM sums (metrics.py evm :169-179): sums[0] += sum |soft - ref|^2,
 * sums[1] += sum |ref|^2 in float64; soft complex64, ref complex128.
 * Deterministic (fixed reduction order); scratch: 1024 doubles of device
 * memory.
 */
int kk_evm_sums(const void *soft, const void *ref, int64_t n, double *sums, double *scratch, void *stream);

/*
 * Float64 complex FFT of any length (numpy.fft.fft / ifft semantics, the
 * transforms kkmodem's channel runs: channel.py apply_cd :90-103, ssfm_span
 * :124-158): `batch` contiguous rows of n complex128 values from in to out
 * (in == out allowed); inverse != 0 -> ifft with the 1/n normalisation.
 * Powers of two run as Stockham passes, other lengths as Bluestein's
 * chirp-z on a power-of-two length >= 2n - 1.  ws: kk_fft_workspace_bytes()
 * bytes of device memory (0 = unsupported size).
 */
size_t kk_fft_workspace_bytes(int64_t n, int64_t batch);
int kk_fft(const void *in, void *out, int64_t n, int64_t batch, int inverse, void *ws, size_t ws_bytes,
           void *stream);

/*
 * One fiber span by the symmetric split-step Fourier method, in place on n
 * complex128 field samples (replaces channel.py ssfm_span :124-158): n_steps
 * times { half-step dispersion exp(-1j a_half f^2) (f = fftfreq(n, 1/fs));
 * x *= exp(1j gamma (|x|^2 1e-3) l_eff); half-step dispersion; x *= loss_amp }.
 * The caller derives n_steps, a_half, l_eff and loss_amp from the span as
 * the reference does.  ws: kk_ssfm_workspace_bytes(n) bytes of device memory.
 */
size_t kk_ssfm_workspace_bytes(int64_t n);
int kk_ssfm_span(void *x, int64_t n, double sample_rate_hz, int n_steps, double a_half, double gamma_per_w_km,
                 double l_eff_km, double loss_amp, void *ws, size_t ws_bytes, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* KKB200_H */
