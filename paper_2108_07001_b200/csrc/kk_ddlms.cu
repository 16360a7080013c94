// K3 sync / K4 widely-linear DDLMS / BER kernels.
//
// Reference: rxdsp.py `_ddlms_core` :460-499, `ddlms_wl` :510-545,
// `symbol_sync` :574-601, `demap` :548-567; harness/runner.py
// `_accumulate_errors` :351-363.
//
// DDLMS, real form.  With X = [Re x0, Im x0, ..., Re x3, Im x3] (the 4-tap
// 2-sps window of symbol k) and the widely-linear taps written as a real 2x8
// matrix T (row 0 -> Re y, row 1 -> Im y), the reference recurrence
//     y = sum conj(w_i) x_i + conj(g_i) conj(x_i)
//     w_i += mu conj(d - y) x_i ;  g_i += mu conj(d - y) conj(x_i)
// is exactly  y = T X,  T <- T + 2 mu (D - T X) X^T   (D = [Re d, Im d]),
// i.e. T <- T A_k + c_k with A_k = I - 2 mu X X^T (real symmetric 8x8) and
// c_k = 2 mu D X^T.  With decisions fixed a block of B symbols is the affine
// map T -> T P_b + Q_b, P_b = A_0..A_{B-1} (decision independent), Q_b built
// from the decisions.
//
// Exact parallel solve (kk_ddlms_solve): P_b for all blocks; exact Q for the
// pure-training blocks; speculate every decision-directed block from the
// training-end taps; then iterate { deterministic multi-level prefix scan of
// (P, Q) -> block start taps; re-run every block whose start taps moved by
// more than its certified margin; count changed decisions } until no
// decision changes -- that fixpoint is the sequential recurrence's result.
// Guard trips, frozen state and non-convergence fall back to the exact
// sequential chain.
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "kk_common.cuh"
#include "kk_internal.h"

namespace kk {

// ---------------------------------------------------------------------------
// slicer (nearest constellation point, first minimum wins: rxdsp.py:476-483)
// ---------------------------------------------------------------------------
struct Slicer {
    int kind;          // 0 = square grid (separable), 1 = brute force
    int npts;
    int m;             // levels per axis (square)
    float norm;        // level value = (2i - (m-1)) / norm
    float thr;         // guard: divergence_factor * max_radius
    float2 pts[64];
    uint8_t grid[64];  // (i_re * m + i_im) -> point index (square)
    int sep;           // square grid whose points are exactly ((2 i_re - (m-1)) h, (2 i_im - (m-1)) h) in fp32
    float lev_h;
};

// returns point index, sets decision value and margin (distance to the
// nearest decision boundary)
__device__ __forceinline__ int slice(const Slicer& s, float yr, float yi, float& margin) {
    if (s.kind == 0) {
        const float h = 1.0f / s.norm;                       // half spacing
        const float fr = (yr * s.norm + (s.m - 1)) * 0.5f;
        const float fi = (yi * s.norm + (s.m - 1)) * 0.5f;
        int ir = __float2int_rn(fr), ii = __float2int_rn(fi);
        ir = min(max(ir, 0), s.m - 1);
        ii = min(max(ii, 0), s.m - 1);
        const float lr = (2 * ir - (s.m - 1)) * h, li = (2 * ii - (s.m - 1)) * h;
        float mr = 3.0e38f, mi = 3.0e38f;
        if (ir > 0) mr = yr - (lr - h);
        if (ir < s.m - 1) mr = fminf(mr, (lr + h) - yr);
        if (ii > 0) mi = yi - (li - h);
        if (ii < s.m - 1) mi = fminf(mi, (li + h) - yi);
        margin = fminf(mr, mi);
        return s.grid[ir * s.m + ii];
    }
    int best = 0;
    float bd = 3.0e38f;
    for (int p = 0; p < s.npts; ++p) {
        const float dr = yr - s.pts[p].x, di = yi - s.pts[p].y;
        const float d = dr * dr + di * di;
        if (d < bd) { bd = d; best = p; }
    }
    float mg = 3.0e38f;
    const float2 pb = s.pts[best];
    for (int p = 0; p < s.npts; ++p) {
        if (p == best) continue;
        const float dr = yr - s.pts[p].x, di = yi - s.pts[p].y;
        const float ex = pb.x - s.pts[p].x, ey = pb.y - s.pts[p].y;
        const float sep = sqrtf(ex * ex + ey * ey);
        mg = fminf(mg, ((dr * dr + di * di) - bd) / (2.0f * sep));
    }
    margin = mg;
    return best;
}

// ---------------------------------------------------------------------------
// sequential chain, complex form, exact reference semantics (fp32)
// (used by the functional ddlms_wl API, non-WL mode and fallbacks)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void seq_chain(const float2* __restrict__ x, int64_t n_out, float scale, int n_taps,
                                          const float2* __restrict__ train, int64_t n_train, float2 (&w)[16],
                                          float2 (&g)[16], int& frozen, int& div, const Slicer& sl, float mu, int wl,
                                          int guard_run, uint8_t* __restrict__ labels, float2* __restrict__ soft,
                                          float2* __restrict__ dec) {
    for (int64_t k = 0; k < n_out; ++k) {
        const float2* xk = x + 2 * k;
        float2 y = make_float2(0.f, 0.f);
        for (int i = 0; i < n_taps; ++i) {
            const float2 xi = cscale(xk[i], scale);
            y = cadd(y, cmul(cconj(w[i]), xi));
            if (wl) y = cadd(y, cmul(cconj(g[i]), cconj(xi)));
        }
        float2 d;
        int lab;
        if (k < n_train) {
            d = train[k];
            lab = 255;
        } else {
            float mg;
            lab = slice(sl, y.x, y.y, mg);
            d = sl.pts[lab];
        }
        if (sqrtf(y.x * y.x + y.y * y.y) > sl.thr) {
            div += 1;
            if (div >= guard_run) frozen = 1;
        } else {
            div = 0;
        }
        if (!frozen && mu != 0.0f) {
            const float2 ce = cconj(csub(d, y));
            const float2 mce = cscale(ce, mu);
            for (int i = 0; i < n_taps; ++i) {
                const float2 xi = cscale(xk[i], scale);
                w[i] = cadd(w[i], cmul(mce, xi));
                if (wl) g[i] = cadd(g[i], cmul(mce, cconj(xi)));
            }
        }
        if (labels) labels[k] = static_cast<uint8_t>(lab);
        if (soft) soft[k] = y;
        if (dec) dec[k] = d;
    }
}

__global__ void ddlms_seq_kernel(const float2* __restrict__ x, int64_t n_out, float scale, int n_taps,
                                 const float2* __restrict__ train, int64_t n_train, float2* __restrict__ wg,
                                 int* __restrict__ fz, Slicer sl, float mu, int wl, int guard_run,
                                 uint8_t* __restrict__ labels, float2* __restrict__ soft,
                                 float2* __restrict__ dec) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    float2 w[16], g[16];
    for (int i = 0; i < n_taps; ++i) { w[i] = wg[i]; g[i] = wg[n_taps + i]; }
    int frozen = fz[0];
    int div = fz[1];
    seq_chain(x, n_out, scale, n_taps, train, n_train, w, g, frozen, div, sl, mu, wl, guard_run, labels, soft, dec);
    for (int i = 0; i < n_taps; ++i) { wg[i] = w[i]; wg[n_taps + i] = g[i]; }
    fz[0] = frozen;
    fz[1] = div;
}

// WL taps (w, g; 4 taps) <-> real 2x8 form T (rxdsp._T_from_wg / _wg_from_T)
__device__ __forceinline__ void wg_from_T(const float* T, float inv, float2 (&w)[16], float2 (&g)[16]) {
    for (int i = 0; i < 4; ++i) {
        const float a = T[2 * i] * inv, b = T[2 * i + 1] * inv, c = T[8 + 2 * i] * inv, d = T[9 + 2 * i] * inv;
        w[i] = make_float2((a + d) * 0.5f, (b - c) * 0.5f);
        g[i] = make_float2((a - d) * 0.5f, -(b + c) * 0.5f);
    }
}
__device__ __forceinline__ void T_from_wg(const float2 (&w)[16], const float2 (&g)[16], float* T) {
    for (int i = 0; i < 4; ++i) {
        T[2 * i] = w[i].x + g[i].x;
        T[2 * i + 1] = w[i].y - g[i].y;
        T[8 + 2 * i] = -w[i].y - g[i].y;
        T[9 + 2 * i] = w[i].x - g[i].x;
    }
}

// ---------------------------------------------------------------------------
// block-parallel solve (WL, 4 taps)
// ---------------------------------------------------------------------------
struct SolveArgs {
    const float2* x;      // 2-sps input; symbol k uses x[2k .. 2k+3]
    int64_t nsym;
    float scale;
    const float2* train;  // training symbols, k < n_train
    int64_t n_train;
    float mu;
    int B;                // symbols per block
    int64_t nb;
    int guard_run = 100;  // divergence guard run length (rx:484-490)
    int lin = 0;          // linear (not widely-linear) equaliser
};

// symbol k's window x[2k .. 2k+3] (scaled); consecutive symbols share two
// samples, so the loops below slide the window and load 2 samples per symbol
__device__ __forceinline__ void load_pair(const SolveArgs& a, int64_t i, float& r0, float& i0, float& r1, float& i1) {
    const float2 v0 = __ldg(a.x + i), v1 = __ldg(a.x + i + 1);
    r0 = v0.x * a.scale; i0 = v0.y * a.scale; r1 = v1.x * a.scale; i1 = v1.y * a.scale;
}


struct RunOut {
    uint8_t* labels;
    float2* soft;
    float* Q;         // [nb][16]
    float* Tused;     // [nb][16] start taps of the block's latest run
    float* Twritten;  // [nb][16] start taps of its latest output-writing run (NaN: never)
    float* margin;    // [nb]
    float* Tend;      // [16] end taps of the last block
    int* over;        // [nb] guard exceedances in the block's latest run
    unsigned long long* hash;  // [nb] hash of the block's latest label sequence
    uint2* ties;               // [nb] recorded fp32-tie decisions (two slots per block)
    int2* grun;                // [nb] guard exceedance runs of the block's latest run:
                               //   x = leading run | trailing run << 16, y = (first in-block run
                               //   reaching guard_run) + 1 (0: none) | all-exceeded << 16
    unsigned long long* counters;  // [0] changed decisions, [1] blocks re-run
    unsigned int* first_changed;   // lowest block index whose decisions changed (atomicMin)
};

// Run blocks [b_lo, b_hi) starting from Tstart[b] (or chain them when chain != 0:
// one thread, block b+1 starts from block b's end taps).  Skip test: re-run a
// block only if |T_new - T_used|_F * max|X| >= min(margin, soft_tol).
struct ReadBack;
__device__ bool fallback_gate(const ReadBack* rb, int64_t& b_lo);

// linear-equaliser update of real-form taps (see ddlms_block_kernel<.., LIN>)
__device__ __forceinline__ void lin_update(float (&T)[16], const float (&X)[8], float el, float fl) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const float x0 = X[2 * u], x1 = X[2 * u + 1];
        const float d0 = fmaf(el, x0, fl * x1);
        const float d1 = fmaf(el, x1, -fl * x0);
        T[2 * u] += d0;
        T[2 * u + 1] += d1;
        T[8 + 2 * u] -= d1;
        T[9 + 2 * u] += d0;
    }
}

__global__ void ddlms_run_kernel(SolveArgs a, Slicer sl, const float* __restrict__ Tstart,
                                 const float* __restrict__ maxx2, RunOut o, int64_t b_lo, int64_t b_hi,
                                 int use_skip, float soft_tol, int chain, int first_run,
                                 const ReadBack* gate = nullptr) {
    // gate (asynchronous solve, fallback mode 2): run only then, from the
    // lowest block whose decisions changed in the last iteration
    if (gate && !fallback_gate(gate, b_lo)) return;
    int64_t b = b_lo + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (chain) {
        if (blockIdx.x != 0 || threadIdx.x != 0) return;
        b = b_lo;
    }
    if (b >= b_hi) return;
    float T[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) T[i] = Tstart[b * 16 + i];
    const float tm = 2.0f * a.mu;
    unsigned long long changed = 0, over = 0, reruns = 0;
    for (;;) {
        bool run = true;
        if (use_skip && !chain && !first_run) {
            float d2 = 0.f;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float d = T[i] - o.Tused[b * 16 + i];
                d2 = fmaf(d, d, d2);
            }
            const float bound = sqrtf(d2 * maxx2[b]);
            const float ok = fminf(o.margin[b], soft_tol);
            run = !(bound < ok) || (a.mu * maxx2[b] > 1.0f);
        }
        if (run) {
            ++reruns;
#pragma unroll
            for (int i = 0; i < 16; ++i) o.Tused[b * 16 + i] = T[i];
            float Q[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) Q[i] = 0.f;
            float mg = 3.0e38f;
            const int64_t k0 = b * a.B, k1 = min(k0 + a.B, a.nsym);
            float X[8];
            load_pair(a, 2 * k0, X[4], X[5], X[6], X[7]);
            for (int64_t k = k0; k < k1; ++k) {
                X[0] = X[4]; X[1] = X[5]; X[2] = X[6]; X[3] = X[7];
                load_pair(a, 2 * k + 2, X[4], X[5], X[6], X[7]);
                float yr = 0.f, yi = 0.f, qr = 0.f, qi = 0.f;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    yr = fmaf(T[j], X[j], yr);
                    yi = fmaf(T[8 + j], X[j], yi);
                    qr = fmaf(Q[j], X[j], qr);
                    qi = fmaf(Q[8 + j], X[j], qi);
                }
                float dr, di;
                int lab;
                if (k < a.n_train) {
                    const float2 t = __ldg(a.train + k);
                    dr = t.x; di = t.y;
                    lab = 255;
                } else {
                    float m;
                    lab = slice(sl, yr, yi, m);
                    mg = fminf(mg, m);
                    dr = sl.pts[lab].x; di = sl.pts[lab].y;
                }
                const float ay = sqrtf(yr * yr + yi * yi);
                if (ay > sl.thr) ++over;
                mg = fminf(mg, fabsf(ay - sl.thr));
                const float er = tm * (dr - yr), ei = tm * (di - yi);
                const float fr = tm * (dr - qr), fi = tm * (di - qi);
                if (a.lin) {
                    lin_update(T, X, 0.5f * er, 0.5f * ei);
                    lin_update(Q, X, 0.5f * fr, 0.5f * fi);
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        T[j] = fmaf(er, X[j], T[j]);
                        T[8 + j] = fmaf(ei, X[j], T[8 + j]);
                        Q[j] = fmaf(fr, X[j], Q[j]);
                        Q[8 + j] = fmaf(fi, X[j], Q[8 + j]);
                    }
                }
                const uint8_t old = o.labels[k];
                if (old != static_cast<uint8_t>(lab)) { o.labels[k] = static_cast<uint8_t>(lab); ++changed; }
                o.soft[k] = make_float2(yr, yi);
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) o.Q[b * 16 + i] = Q[i];
            o.margin[b] = mg;
            o.over[b] = static_cast<int>(over);
            over = 0;
            if (b == a.nb - 1) {
#pragma unroll
                for (int i = 0; i < 16; ++i) o.Tend[i] = T[i];
            }
        }
        if (!chain) break;
        ++b;
        if (b >= b_hi) break;
        if (!run) {
#pragma unroll
            for (int i = 0; i < 16; ++i) T[i] = Tstart[b * 16 + i];
        }
    }
    if (changed) atomicAdd(o.counters + 0, changed);
    if (reruns) atomicAdd(o.counters + 1, reruns);
}

__global__ void sum_int_kernel(const int* __restrict__ v, int64_t n, unsigned long long* __restrict__ out) {
    unsigned long long acc = 0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        acc += static_cast<unsigned long long>(v[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// Device-driven fixpoint iteration (kk_ddlms_solve): the pass mode lives in
// device memory, every kernel of an iteration reads it and a done frame's
// remaining (pre-queued) iterations return at once; the host reads the
// control block back once per batch of iterations instead of once per pass.
constexpr int kModeDecision = 0, kModeOutput = 1, kModeDone = 2;
#ifndef KK_CASCADE_FROM
#define KK_CASCADE_FROM 4   // first 0-based iteration that queues cascade steps
#endif
#ifndef KK_CASCADE_W
#define KK_CASCADE_W 8
#endif
#ifndef KK_LOOP_UNROLL
#define KK_LOOP_UNROLL 4
#endif
constexpr int kLoopUnroll = KK_LOOP_UNROLL;                    // fixpoint iterations per graph-loop trip
constexpr int kCascadeW = KK_CASCADE_W;                        // blocks the exact frontier advances per step set
constexpr unsigned long long kCascadeMaxChanged = 64; // "a cascade": at most this many changed blocks
constexpr int kMaxStatIters = 64;
struct ReadBack {
    unsigned long long ctr[4];   // [0] changed blocks, [1] blocks re-run, [2] guard sum, [3] list length
    int ctl[4];                  // [0] mode, [1] iterations run
    unsigned int first_changed;  // lowest changed block of the running iteration (~0: none)
    unsigned int last_first;     // the same for the last finished iteration
    unsigned long long it_stats[2 * kMaxStatIters];   // per iteration (changed, re-run)
    float Tend[16];              // end taps of the frame (scaled)
    float Tfz[16];               // frozen taps (scaled) of a guard freeze
    long long freeze_k;          // symbol whose exceedance run froze the taps (LLONG_MAX: none)
    int carry;                   // div_count at the frame end (exceedance run in progress)
};

__device__ __forceinline__ bool ctl_done(const int* ctl) { return ctl && *ctl == kModeDone; }

// Counter / control resets of the readback record in one launch (replaces
// 2-3 small memsets per frame step; each costs a launch slot on the stream).
enum : int {
    kRbCtr01 = 1, kRbCtr2 = 2, kRbCtr3 = 4, kRbFirst0 = 8, kRbFirst1 = 16, kRbCtl = 32, kRbAll = 64,
};
__global__ void rb_reset_kernel(ReadBack* __restrict__ rb, int what) {
    if (threadIdx.x != 0) return;
    if (what & kRbAll) {
        unsigned long long* w = reinterpret_cast<unsigned long long*>(rb);
        for (size_t i = 0; i < sizeof(ReadBack) / 8; ++i) w[i] = 0ull;
        rb->first_changed = ~0u;
        rb->last_first = ~0u;
        return;
    }
    if (what & kRbCtr01) rb->ctr[0] = rb->ctr[1] = 0ull;
    if (what & kRbCtr2) rb->ctr[2] = 0ull;
    if (what & kRbCtr3) rb->ctr[3] = 0ull;
    if (what & kRbFirst0) rb->first_changed = ~0u;
    if (what & kRbFirst1) rb->last_first = ~0u;
    if (what & kRbCtl) rb->ctl[0] = rb->ctl[1] = rb->ctl[2] = rb->ctl[3] = 0;
}
static_assert(sizeof(ReadBack) % 8 == 0, "ReadBack layout");



__device__ bool fallback_gate(const ReadBack* rb, int64_t& b_lo) {
    if (rb->ctl[3] != 2) return false;
    b_lo = rb->last_first;
    return true;
}

// end of one iteration: record its counts, pick the next pass (decision
// passes until nothing changes, then one output pass; an output pass that
// changes nothing ends the frame)
// With use_cond the kernel is the last node of the CUDA-graph while loop's
// body (kk_ddlms_solve_async): it also sets the loop condition (not done,
// fewer than max_iter iterations).
__global__ void ddlms_advance_kernel(ReadBack* rb, cudaGraphConditionalHandle loop, int use_cond, int max_iter) {
    const int mode = rb->ctl[0];
    if (mode != kModeDone) {
        const unsigned long long ch = rb->ctr[0], rr = rb->ctr[1];
        const int it = rb->ctl[1];
        if (it < kMaxStatIters) {
            rb->it_stats[2 * it] = ch;
            rb->it_stats[2 * it + 1] = rr;
        }
        rb->ctl[1] = it + 1;
        rb->ctl[0] = ch ? kModeDecision : (mode == kModeOutput ? kModeDone : kModeOutput);
        rb->last_first = rb->first_changed;
        rb->first_changed = 0xffffffffu;
        rb->ctr[0] = 0;
        rb->ctr[1] = 0;
        rb->ctr[3] = 0;
    }
    if (use_cond) {
        if (rb->ctl[0] != kModeDone && rb->ctl[1] >= max_iter) {
            rb->ctl[3] = 2;              // not converged: the frame takes the chained fallback
            rb->ctl[0] = kModeDone;      // (the unrolled iterations left in the body return at once)
        }
        cudaGraphSetConditional(loop, rb->ctl[0] != kModeDone ? 1u : 0u);
    }
}

// ---- asynchronous solve: frame begin / end on the device (no readback) ----
// frame start taps T_in (unscaled, device) -> Tinit (scaled).  Equalizer
// state {frozen, div_count} != 0 at the frame start: the affine maps assume
// live, guard-free taps, so the frame takes the exact sequential chain.
__global__ void frame_begin_kernel(const float* __restrict__ T_in, float scale, float* __restrict__ Tinit,
                                   const int* __restrict__ state, ReadBack* rb) {
    const int i = threadIdx.x;
    if (i < 16) Tinit[i] = T_in[i] * scale;
    if (i < 16) rb->Tfz[i] = T_in[i] * scale;
    if (i == 0) {
        rb->freeze_k = LLONG_MAX;
        rb->carry = 0;
        // taps frozen by an earlier frame: every decision of this frame is a
        // parallel map with constant taps (mode 3); the solver stands down
        if (state && state[0] != 0) {
            rb->ctl[0] = kModeDone;
            rb->ctl[3] = 3;
        }
    }
}

__global__ void copy16_kernel(float* __restrict__ dst, const float* __restrict__ src) {
    if (threadIdx.x < 16) dst[threadIdx.x] = src[threadIdx.x];
}

// after the loop (guard sum in ctr[2]): fallback mode ctl[3] = 0 none,
// 1 sequential chain from the frame start (guard exceedances / state),
// 2 not converged within max_iter -> output pass below the lowest changed
// block m, chain from m.  ctl[2] gates the mode-2 kernels (kModeOutput: run).
__global__ void frame_end_kernel(ReadBack* rb) {
    int fb = rb->ctl[3];
    if (fb == 0 && rb->ctl[0] != kModeDone) fb = 2;
    rb->ctl[3] = fb;
    rb->ctl[2] = (fb == 2 || fb == 4) ? kModeOutput : kModeDone;
    rb->ctr[3] = 0;
}

// Divergence guard (rx:484-490) at the converged fixpoint: the decisions are
// those of the live-tap recurrence, so they are exact up to the first symbol
// k* at which an exceedance run reaches guard_run (taps freeze there).  Runs
// cross blocks: a block's carry-in is the trailing run of the block before,
// extended through all-exceeded blocks (at most guard_run / B + 1 of them),
// starting from the frame-start div_count.  One thread per block holding an
// exceedance; the earliest freeze wins (atomicMin); the last block records
// the frame-end div_count.
__global__ void guard_scan_kernel(ReadBack* rb, const int2* __restrict__ grun, const int* __restrict__ over,
                                  int64_t nb, int B, int64_t nsym, int guard_run, const int* __restrict__ state,
                                  int final_pass) {
    // in the fixpoint loop (final_pass 0): only the certified prefix -- the
    // blocks below the lowest block whose decisions changed this iteration
    // ran from exact starts -- so a freeze found there is the
    // stream's; the blocks after it need no further iterations
    if (rb->ctl[3] != 0 || rb->ctr[2] == 0) return;
    if (!final_pass && rb->ctl[0] == kModeDone) return;
    const int64_t limit = final_pass ? nb : min(nb, static_cast<int64_t>(rb->first_changed));
    for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < nb; b += int64_t(gridDim.x) * blockDim.x) {
        const bool last = final_pass && b == nb - 1;
        if (b >= limit || (!over[b] && !last)) continue;
        int64_t c = 0;
        for (int64_t j = b - 1;; --j) {
            if (j < 0) {
                c += state ? state[1] : 0;
                break;
            }
            const int2 g = grun[j];
            if ((g.y >> 16) & 1) {                    // all exceeded: the run continues through it
                c += min(static_cast<int64_t>(B), nsym - j * B);
                if (c >= guard_run) break;
            } else {
                c += (g.x >> 16) & 0xffff;            // trailing run
                break;
            }
        }
        const int2 g = grun[b];
        const int pre = g.x & 0xffff, first1 = g.y & 0xffff;   // first in-block run + 1 (0: none)
        const int64_t k0 = b * B;
        if (over[b]) {
            long long cand = LLONG_MAX;
            if (c + pre >= guard_run) cand = k0 + (guard_run - c - 1);
            else if (first1 != 0) cand = k0 + first1 - 1;
            if (cand != LLONG_MAX) atomicMin(&rb->freeze_k, cand);
        }
        if (last)
            rb->carry = static_cast<int>(min(static_cast<int64_t>(guard_run),
                                             ((g.y >> 16) & 1) ? c + (nsym - k0) : ((g.x >> 16) & 0xffff)));
    }
}

// a certified freeze ends the fixpoint iteration (mode 4)
__global__ void guard_decide_kernel(ReadBack* rb) {
    if (rb->ctl[3] == 0 && rb->freeze_k != LLONG_MAX) {
        rb->ctl[3] = 4;
        rb->ctl[0] = kModeDone;
    }
}

// mode 4: the exact chain of the freezing block from its (exact) start taps
// up to the freezing symbol k* (which is decided with the taps it froze,
// without an update); the frozen taps -> rb->Tfz
__global__ void freeze_chain_kernel(SolveArgs a, Slicer sl, const float* __restrict__ Tstart, ReadBack* rb,
                                    uint8_t* __restrict__ labels, float2* __restrict__ soft) {
    if (threadIdx.x != 0 || blockIdx.x != 0 || rb->ctl[3] != 4) return;
    const int64_t ks = rb->freeze_k;
    const int64_t b = ks / a.B;
    float T[16];
    for (int i = 0; i < 16; ++i) T[i] = Tstart[b * 16 + i];
    const float tm = 2.0f * a.mu;
    for (int64_t k = b * a.B; k <= ks; ++k) {
        float X[8];
        for (int u = 0; u < 4; ++u) {
            const float2 v = a.x[2 * k + u];
            X[2 * u] = v.x;
            X[2 * u + 1] = v.y;
        }
        float yr = 0.f, yi = 0.f;
        for (int j = 0; j < 8; ++j) {
            yr = fmaf(T[j], X[j], yr);
            yi = fmaf(T[8 + j], X[j], yi);
        }
        float dr, di;
        int lab;
        if (k < a.n_train) {
            const float2 t = a.train[k];
            dr = t.x;
            di = t.y;
            lab = 255;
        } else {
            float m;
            lab = slice(sl, yr, yi, m);
            dr = sl.pts[lab].x;
            di = sl.pts[lab].y;
        }
        labels[k] = static_cast<uint8_t>(lab);
        soft[k] = make_float2(yr, yi);
        if (k == ks) break;                        // frozen: no update from here on
        const float er = tm * (dr - yr), ei = tm * (di - yi);
        if (a.lin) {
            lin_update(T, X, 0.5f * er, 0.5f * ei);
        } else {
            for (int j = 0; j < 8; ++j) {
                T[j] = fmaf(er, X[j], T[j]);
                T[8 + j] = fmaf(ei, X[j], T[8 + j]);
            }
        }
    }
    for (int i = 0; i < 16; ++i) rb->Tfz[i] = T[i];
}

// modes 3 / 4: decisions with frozen taps are independent of each other --
// a parallel map (rb->Tfz: the frame-start taps in mode 3)
__global__ void frozen_map_kernel(SolveArgs a, Slicer sl, const ReadBack* rb, uint8_t* __restrict__ labels,
                                  float2* __restrict__ soft) {
    const int mode = rb->ctl[3];
    if (mode != 3 && mode != 4) return;
    const int64_t k0 = mode == 3 ? 0 : rb->freeze_k + 1;
    __shared__ float Ts[16];
    if (threadIdx.x < 16) Ts[threadIdx.x] = rb->Tfz[threadIdx.x];
    __syncthreads();
    for (int64_t k = k0 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < a.nsym;
         k += int64_t(gridDim.x) * blockDim.x) {
        float yr = 0.f, yi = 0.f;
        for (int u = 0; u < 4; ++u) {
            const float2 v = __ldg(a.x + 2 * k + u);
            yr = fmaf(Ts[2 * u], v.x, fmaf(Ts[2 * u + 1], v.y, yr));
            yi = fmaf(Ts[8 + 2 * u], v.x, fmaf(Ts[9 + 2 * u], v.y, yi));
        }
        int lab = 255;
        if (k >= a.n_train) {
            float m;
            lab = slice(sl, yr, yi, m);
        }
        labels[k] = static_cast<uint8_t>(lab);
        soft[k] = make_float2(yr, yi);
    }
}

// modes 2 / 4: output pass over blocks [0, m) -- m the lowest block whose
// decisions changed in the last iteration (their starts are exact), or the
// freezing block
__global__ void fallback_list_kernel(ReadBack* rb, int* __restrict__ list, int64_t nb, int B) {
    const int mode = rb->ctl[3];
    if (mode != 2 && mode != 4) return;
    const int64_t m = mode == 4 ? min(static_cast<int64_t>(rb->freeze_k / B), nb)
                                : min(static_cast<int64_t>(rb->last_first), nb);
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x)
        list[i] = static_cast<int>(i);
    if (blockIdx.x == 0 && threadIdx.x == 0) rb->ctr[3] = static_cast<unsigned long long>(m > 0 ? m : 0);
}

// after the mode-2 chain: guard exceedances there -> mode 1
__global__ void frame_end2_kernel(ReadBack* rb) {
    if (rb->ctl[3] == 2 && rb->ctr[2] > 0) rb->ctl[3] = 1;
}

// mode 1: the exact sequential recurrence (rx:465-498, guard included) over
// the whole frame from its start taps and state
__global__ void seq_fallback_kernel(const float2* __restrict__ x, int64_t nsym, float scale,
                                    const float2* __restrict__ train, int64_t n_train, const float* __restrict__ Tinit,
                                    float* __restrict__ T_io, int* __restrict__ state_io, Slicer sl, float mu,
                                    int guard_run, int wl, uint8_t* __restrict__ labels, float2* __restrict__ soft,
                                    const ReadBack* rb) {
    if (threadIdx.x != 0 || blockIdx.x != 0 || rb->ctl[3] != 1) return;
    float2 w[16], g[16];
    wg_from_T(Tinit, 1.0f / scale, w, g);
    int frozen = state_io ? state_io[0] : 0, div = state_io ? state_io[1] : 0;
    seq_chain(x, nsym, scale, 4, train, n_train, w, g, frozen, div, sl, mu, wl, guard_run, labels, soft, nullptr);
    T_from_wg(w, g, T_io);
    if (state_io) {
        state_io[0] = frozen;
        state_io[1] = div;
    }
}

// modes 0 / 2: end taps (scaled Tend -> unscaled) and a clear state (no
// guard exceedance in the frame: div_count ends at 0, taps live)
__global__ void frame_final_kernel(const ReadBack* rb, float inv_scale, float* __restrict__ T_io,
                                   int* __restrict__ state_io) {
    const int mode = rb->ctl[3];
    if (mode == 1) return;                         // the sequential chain wrote them
    const bool frozen = mode == 3 || mode == 4;
    const int i = threadIdx.x;
    if (i < 16) T_io[i] = (frozen ? rb->Tfz[i] : rb->Tend[i]) * inv_scale;
    if (i == 0 && state_io) {
        state_io[0] = frozen ? 1 : 0;
        state_io[1] = frozen ? 0 : rb->carry;    // (a frozen state never unfreezes: div_count is moot)
    }
}

// statistics of the finished frame -> out[38] (device or mapped host):
// iterations, blocks run, fallback, guard exceedances, changed blocks in the
// last iteration, blocks, per-iteration (changed, re-run) for 1..16
__global__ void frame_stats_kernel(const ReadBack* rb, int64_t nb, int64_t pre_runs, int64_t* __restrict__ out) {
    if (threadIdx.x != 0) return;
    const int it = rb->ctl[1];
    int64_t runs = pre_runs;
    for (int i = 0; i < min(it, kMaxStatIters); ++i) runs += static_cast<int64_t>(rb->it_stats[2 * i + 1]);
    out[0] = it;
    out[1] = runs;
    out[2] = rb->ctl[3];
    out[3] = static_cast<int64_t>(rb->ctr[2]);
    out[4] = (it > 0 && it <= kMaxStatIters) ? static_cast<int64_t>(rb->it_stats[2 * (it - 1)]) : 0;
    out[5] = nb;
    for (int i = 0; i < 16; ++i) {
        out[6 + 2 * i] = i < it ? static_cast<int64_t>(rb->it_stats[2 * i]) : 0;
        out[7 + 2 * i] = i < it ? static_cast<int64_t>(rb->it_stats[2 * i + 1]) : 0;
    }
}

// Decision cascades (64-QAM): late iterations change a few blocks, one block
// further per iteration.  After an iteration's pass changed at most
// max_changed blocks, the lowest changed block m ran from its exact start, so
// the starts of m+1 .. m+W follow exactly from the maps of m .. m+W-1; W
// repetitions of {these starts -> re-run the W blocks} move the exact
// frontier W blocks ahead inside one iteration (step = repetition index).
__global__ void cascade_prep_kernel(ReadBack* rb, const float* __restrict__ Pb, const float* __restrict__ Qb,
                                    const float* __restrict__ Tused, float* __restrict__ Tstart, int* __restrict__ list,
                                    int64_t nb, int64_t ntb, int W, int step, unsigned long long max_changed,
                                    int from_iter) {
    if (threadIdx.x != 0) return;
    if (step == 0)
        rb->ctl[2] = (rb->ctl[0] != kModeDone && rb->ctl[1] >= from_iter && rb->ctr[0] > 0 &&
                      rb->ctr[0] <= max_changed) ? 1 : 0;
    rb->ctr[3] = 0;
    if (!rb->ctl[2]) return;
    const int64_t m = rb->first_changed;
    if (m < ntb || m + 1 >= nb) return;
    float T[16];
    for (int i = 0; i < 16; ++i) T[i] = Tused[m * 16 + i];
    int n = 0;
    for (int64_t b = m; b + 1 < nb && n < W; ++b) {
        const float* P = Pb + b * 64;
        const float* Q = Qb + b * 16;
        float U[16];
        for (int r = 0; r < 2; ++r)
            for (int j = 0; j < 8; ++j) {
                float acc = Q[r * 8 + j];
                for (int k = 0; k < 8; ++k) acc = fmaf(T[r * 8 + k], P[k * 8 + j], acc);
                U[r * 8 + j] = acc;
            }
        for (int i = 0; i < 16; ++i) {
            T[i] = U[i];
            Tstart[(b + 1) * 16 + i] = U[i];
        }
        list[n++] = static_cast<int>(b + 1);
    }
    rb->ctr[3] = static_cast<unsigned long long>(n);
}

struct Vec16 {
    float v[16];
};
__global__ void set16_kernel(float* __restrict__ dst, Vec16 v) {
    if (threadIdx.x < 16) dst[threadIdx.x] = v.v[threadIdx.x];
}

__global__ void fill_T_kernel(float* __restrict__ T, int64_t b0, int64_t b1, const float* __restrict__ src) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t n = (b1 - b0) * 16;
    if (i < n) T[b0 * 16 + i] = src[i & 15];
}

// Block-parallel DDLMS passes (ddlms_block_kernel below): one thread per
// block of B symbols, reading the 2-sps equalizer input in place (no
// transposition) through a per-thread cp.async ring, and writing the final
// soft / labels in natural order.
// ---------------------------------------------------------------------------
#ifndef KK_DD_MINB
#define KK_DD_MINB 4      // resident CTAs / SM of the decision passes
#endif
#ifndef KK_DD_MINB_P
#define KK_DD_MINB_P 4    // resident CTAs / SM of the P pass (4: 128 registers, 16 B spill, measured 8.33 -> 8.29 ms)
#endif
// per-symbol tap products / updates and the P_b rank-1 updates on the packed
// FP32 pipe (FFMA2: two lanes per instruction, same roundings as scalar)
#ifndef KK_DD_PACKED
#define KK_DD_PACKED 1
#endif
#ifndef KK_DD_SLICER_PACKED       // the square-grid slicer's pair arithmetic too
#define KK_DD_SLICER_PACKED KK_DD_PACKED
#endif
constexpr int kBlockThreads = 128;

__device__ __forceinline__ void cp_async16(void* smem, const void* g, int src_bytes) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async8z(void* smem, const void* g, int src_bytes) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(src_bytes) : "memory");
}
// predicated in PTX (-> SASS predicate, not a branch: a branch would make
// ptxas wait on every outstanding shared load at the reconvergence point)
__device__ __forceinline__ void cp_async8_if(bool pred, void* smem, const void* g) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p cp.async.ca.shared.global [%0], [%1], 8;\n}\n" ::"r"(sa),
        "l"(g), "r"(static_cast<int>(pred))
        : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }


struct TOut {
    float2* ST;       // [nsym] soft (final pass)
    uint8_t* LT;      // [nsym] labels (final pass)
};

// Block-parallel DDLMS pass, one thread per block of B symbols.  Lean
// per-symbol work: the input scale s is folded into the taps (T' = s T,
// mu' = mu s^2, so y = T' x_raw); Q_b is recovered once per block as
// T_end - T_start P_b; decision changes are detected with a 64-bit hash of
// the block's label sequence; the guard is tracked as max |y|^2 and the
// decision margin conservatively as the distance to the nearest interior
// boundary.  WITH_P (first pass) also accumulates P_b = prod (I - 2 mu' x x^T)
// and max |x|^2.  SQ > 0: separable square constellation with SQ levels per
// axis -- branch-free arithmetic slicer; SQ == 0: table / brute-force slicer.
//
// Input staging (the 2-sps input x is read in place): a warp's 32 lanes own
// 32 blocks; the warp loads chunks of 8 pair rows for all of them
// cooperatively with cp.async (8 lanes x 16 B = one 128 B run of one block
// per quarter warp), kChunks chunks in flight, into a swizzled smem ring
// [chunk][row][lane]; each lane then reads its own column (conflict-free).
// Register-destination prefetches were measured not to work here (ptxas
// folds them onto shared scoreboards and the chain waits on the newest load).
// TRAIN (launches covering blocks with training symbols): a per-thread
// cp.async ring of training symbols as well.  Outputs (final pass) are
// written per lane in 8-symbol runs (64 B soft, 8 B labels).
constexpr int kChunkRows = 8;
constexpr int kChunks = 3;
constexpr int kTrainRing = 32;   // >= kChunks * kChunkRows symbols in flight
constexpr size_t kWarpStage = size_t(kChunks) * kChunkRows * 32 * sizeof(float4);
constexpr size_t kStageSmem = kWarpStage * (kBlockThreads / 32);
constexpr size_t kTrainSmem = size_t(kTrainRing) * kBlockThreads * sizeof(float2);

__device__ __forceinline__ int stage_idx(int chunk, int row, int col) {
    return (chunk * kChunkRows + row) * 32 + (col ^ ((row * 4) & 31));
}

// normalised slicer units (level spacing 1): how far v lies outside level
// s's cell (negative inside; edge levels are open outwards)
__device__ __forceinline__ float cell_excess(float v, float s, float m1f) {
    const float up = s < m1f ? v - s : -3.0e38f;
    const float dn = s > 0.f ? s - v : -3.0e38f;
    return fmaxf(up, dn) - 0.5f;
}
#ifndef KK_TIE_EPS
#define KK_TIE_EPS 1e-5f
#endif
constexpr float kTieEps = KK_TIE_EPS;   // fp32 tie zone, normalised units (ties: DESIGN §4)

// fp32 ties (|margin| < kTieEps): a re-run from start taps that differ by
// rounding must not flip them back and forth.  The block's first decision at
// a tie is recorded (two slots per block: bit 31 valid, bits 16..23 grid
// cell ir * m + ii, bits 0..15 symbol within the block) and kept while y
// stays within kTieEps of that cell; the symbol's margin is then the
// distance to leaving that zone, not the rounding-level distance to the
// boundary.
__device__ __forceinline__ void tie_rule(int i, float vr, float vi, float m1f, int m, float& fr, float& fi,
                                         float& mg_s, unsigned& tie0, unsigned& tie1, bool& dirty) {
    const bool h0 = (tie0 >> 31) && (tie0 & 0xffffu) == static_cast<unsigned>(i);
    const bool h1 = (tie1 >> 31) && (tie1 & 0xffffu) == static_cast<unsigned>(i);
    if (h0 || h1) {
        const int g = ((h0 ? tie0 : tie1) >> 16) & 0xff;
        const float sr = static_cast<float>(g / m), si = static_cast<float>(g % m);
        const float e = fmaxf(cell_excess(vr, sr, m1f), cell_excess(vi, si, m1f));
        if (e < kTieEps) {
            fr = sr;
            fi = si;
            mg_s = kTieEps - e;
        }
    } else {
        const unsigned rec = 0x80000000u |
                             (static_cast<unsigned>(static_cast<int>(fr) * m + static_cast<int>(fi)) << 16) |
                             static_cast<unsigned>(i);
        if (!(tie0 >> 31)) {
            tie0 = rec;
            mg_s = kTieEps + mg_s;
            dirty = true;
        } else if (!(tie1 >> 31)) {
            tie1 = rec;
            mg_s = kTieEps + mg_s;
            dirty = true;
        }
    }
}

// LIN: the linear (not widely-linear) equaliser, rx:491-497 with g == 0.
// In the real 2x8 form T1 = T0 M (M = blockdiag [[0,1],[-1,0]]) stays true;
// the update is T0 += mu (e_r X + e_i JX) with JX = (x1, -x0) per tap (the
// real embedding of w += mu conj(e) x), i.e. the affine map
// A = I - mu (X X^T + JX JX^T), which commutes with M -- the same 2x8 scan.
template <bool WITH_P, int SQ, bool AL16, bool TRAIN, bool LIN>
__global__ void __launch_bounds__(kBlockThreads, WITH_P ? KK_DD_MINB_P : KK_DD_MINB)
ddlms_block_kernel(SolveArgs a, Slicer sl, const float* __restrict__ Tstart, float* __restrict__ Pb,
                   float* __restrict__ maxx2, RunOut o, TOut to, int64_t b_lo, int64_t b_hi, int use_skip,
                   float soft_tol, const int* __restrict__ list, const unsigned long long* __restrict__ list_n,
                   int write_out, const int* __restrict__ ctl) {
    // write_out: bit 0 = store the block's outputs (soft, labels, Twritten)
    // when it runs; bit 1 = also re-run blocks whose outputs are stale (start
    // moved > soft_tol since they were written: output passes)
    // (storing in decision passes too was measured not to pay: the first
    // decision pass moves nearly every block's start by more than soft_tol,
    // so the output pass re-ran 485 k of 524 k blocks anyway)
    if (ctl) {   // device-driven pass mode: only output passes store (and refresh)
        const int mode = *ctl;
        if (mode == kModeDone) return;
        if (WITH_P) {
            write_out = 0;
        } else {
            write_out = mode == kModeOutput ? 3 : 0;
            if (mode != kModeOutput) soft_tol = 3.0e38f;
        }
    }
    const bool refresh = (write_out & 2) != 0;
    __shared__ float2 pts[64];
    __shared__ uint8_t grid[64];
    extern __shared__ float4 dyn_sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 64) {
        pts[tid] = sl.pts[tid];
        grid[tid] = sl.grid[tid];
    }
    __syncthreads();
    const int m = SQ > 0 ? SQ : sl.m;
    const int m1 = m - 1;
    const float half_norm = 0.5f * sl.norm, off = 0.5f * (m - 1);
    const float thr2 = sl.thr * sl.thr;
    const float lev_h = sl.lev_h;
    const unsigned glab = SQ == 2 ? (unsigned(sl.grid[0]) | unsigned(sl.grid[1]) << 8 | unsigned(sl.grid[2]) << 16 |
                                     unsigned(sl.grid[3]) << 24)
                                  : 0u;

    int64_t b = b_lo + int64_t(blockIdx.x) * blockDim.x + tid;
    bool run;
    if (list) {   // compacted list of the blocks to re-run
        const int64_t t = int64_t(blockIdx.x) * blockDim.x + tid;
        run = t < static_cast<int64_t>(*list_n);
        b = run ? list[t] : 0;
    } else {
        run = b < b_hi;
    }
    float T[16];
    if (run) {
#pragma unroll
        for (int i = 0; i < 16; ++i) T[i] = Tstart[b * 16 + i];
        if (use_skip && !WITH_P) {
            float d2 = 0.f;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float d = T[i] - o.Tused[b * 16 + i];
                d2 = fmaf(d, d, d2);
            }
            const float bound = sqrtf(d2 * maxx2[b]);
            run = !(bound < fminf(o.margin[b], refresh ? 3.0e38f : soft_tol)) || (a.mu * maxx2[b] > 1.0f);
            if (refresh) {   // outputs valid within soft_tol since their last write?
                float w2 = 0.f;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const float d = T[i] - o.Twritten[b * 16 + i];
                    w2 = fmaf(d, d, w2);
                }
                run = run || !(sqrtf(w2 * maxx2[b]) < soft_tol);   // NaN (never written) -> run
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) T[i] = 0.f;
    }
    const unsigned act = __ballot_sync(0xffffffffu, run);
    if (!act) return;    // whole warp idle (no block-level barriers below)

    const int64_t k0 = b * a.B;
    const int nk = run ? static_cast<int>(min(static_cast<int64_t>(a.B), a.nsym - k0)) : 0;
    const int ntr = TRAIN ? static_cast<int>(max(static_cast<int64_t>(0), min(static_cast<int64_t>(nk), a.n_train - k0))) : 0;
    const int nk_w = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(nk));
    const int nchunks = (nk_w + kChunkRows - 1) / kChunkRows;
    const int bsh = run ? static_cast<int>(b) : -1;   // block index shared with the loader lanes

    float4* stage = dyn_sm + warp * (kWarpStage / sizeof(float4));
    // loader: rows 8c+1 .. 8c+8 of the warp's 32 blocks (row r of block q =
    // samples x[2(k0_q + r)], x[2(k0_q + r) + 1]; rows 1..nk_q are valid)
    const int lrow = lane & 7;
    auto load_chunk = [&](int c) {
        const int slot = c % kChunks;
        const int r = c * kChunkRows + 1 + lrow;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int col = q * 4 + (lane >> 3);
            const int bq = __shfl_sync(0xffffffffu, bsh, col);
            const int64_t kq = static_cast<int64_t>(bq) * a.B;
            const bool ok = bq >= 0 && r <= min(static_cast<int64_t>(a.B), a.nsym - kq);
            const float2* src = a.x + 2 * (ok ? kq + r : 0);
            float4* dst = stage + stage_idx(slot, lrow, col);
            if constexpr (AL16) {
                cp_async16(dst, src, ok ? 16 : 0);
            } else {
                cp_async8z(dst, src, ok ? 8 : 0);
                cp_async8z(reinterpret_cast<float2*>(dst) + 1, src + 1, ok ? 8 : 0);
            }
        }
    };
    // training ring (per thread): slot i & (kTrainRing-1) <- train[k0 + i]
    float2* trr = reinterpret_cast<float2*>(dyn_sm + kStageSmem / sizeof(float4)) + tid;
    const float2* tg = a.train + k0;
    auto load_train = [&](int i) {
        if constexpr (TRAIN) cp_async8_if(i < ntr, trr + (i & (kTrainRing - 1)) * kBlockThreads, tg + i);
    };
    // one commit group per chunk (training symbols of the chunk's 8 symbols ride along)
    auto issue = [&](int c) {
        load_chunk(c);
        if constexpr (TRAIN) {
#pragma unroll
            for (int j = 0; j < kChunkRows; ++j) load_train(c * kChunkRows + j);
        }
        cp_async_commit();
    };

    float P[WITH_P ? 64 : 1];
    if constexpr (WITH_P) {
#pragma unroll
        for (int i = 0; i < 64; ++i) P[i] = (i % 9 == 0) ? 1.f : 0.f;
    }
    const float tm = 2.0f * a.mu;      // mu' (scale folded in)
    float mgl = 3.0e38f, mgb = 3.0e38f, mx = 0.f, my2 = 0.f;
    // tie slots of the block (see the slicer below): bit 31 valid, bits
    // 16..23 grid cell (ir * SQ + ii), bits 0..15 symbol within the block
    unsigned tie0 = 0u, tie1 = 0u;
    bool ties_dirty = false;
    // divergence-guard runs (|y| > thr), tracked only at exceedances (a
    // warp vote per symbol; the slow path is rare): last exceeding symbol,
    // current run and its start, the leading run (from symbol 0) and the
    // first in-block run reaching guard_run
    int g_prev = -2, g_run = 0, g_start = 0, g_lead = 0, g_first = 0xffff;
    if constexpr (!WITH_P) {
        if (run) {
            const uint2 t = o.ties[b];
            tie0 = t.x;
            tie1 = t.y;
        }
    }
    unsigned long long hsh = 14695981039346656037ull;   // 64-bit FNV-1a of the block's labels
    float X[8];
    {
        float2 u0 = make_float2(0.f, 0.f), u1 = u0;
        if (run) {
            u0 = __ldg(a.x + 2 * k0);
            u1 = __ldg(a.x + 2 * k0 + 1);
        }
        X[4] = u0.x; X[5] = u0.y; X[6] = u1.x; X[7] = u1.y;
    }
    float2* sp = to.ST + k0;
    uint8_t* lp = to.LT + k0;

#pragma unroll 1
    for (int c = 0; c < kChunks - 1; ++c) issue(c);
#pragma unroll 1
    for (int c = 0; c < nchunks; ++c) {
        __syncwarp();                  // every lane is done with chunk c-1's slot
        issue(c + kChunks - 1);        // (empty groups past the end keep the count uniform)
        cp_async_wait<kChunks - 1>();  // this lane's copies of chunk c landed
        __syncwarp();                  // ... and every other lane's
        // decision passes preload the chunk's 8 rows (ILP); the P pass reads
        // each row when it is needed (32 fewer live registers: 4 CTAs / SM)
        float4 rows[WITH_P ? 1 : kChunkRows];
        if constexpr (!WITH_P) {
#pragma unroll
            for (int j = 0; j < kChunkRows; ++j) rows[j] = stage[stage_idx(c % kChunks, j, lane)];
        }
        float2 soft8[kChunkRows];
        unsigned lab8[2] = {0u, 0u};
#pragma unroll
        for (int j = 0; j < kChunkRows; ++j) {
            const int i = c * kChunkRows + j;
            const bool live = i < nk;
            X[0] = X[4]; X[1] = X[5]; X[2] = X[6]; X[3] = X[7];
            const float4 rw = WITH_P ? stage[stage_idx(c % kChunks, j, lane)] : rows[WITH_P ? 0 : j];
            X[4] = rw.x; X[5] = rw.y; X[6] = rw.z; X[7] = rw.w;
#if KK_DD_PACKED
            // (re, im) pairs (T[jj], T[8 + jj]) on the packed FP32 pipe: the
            // same fma sequence per lane as the scalar form
            float2 yza = make_float2(0.f, 0.f), yzb = make_float2(0.f, 0.f);
#pragma unroll
            for (int jj = 0; jj < 8; jj += 2) {
                yza = __ffma2_rn(make_float2(T[jj], T[8 + jj]), make_float2(X[jj], X[jj]), yza);
                yzb = __ffma2_rn(make_float2(T[jj + 1], T[9 + jj]), make_float2(X[jj + 1], X[jj + 1]), yzb);
            }
            const float2 yri = __fadd2_rn(yza, yzb);
            const float yr = yri.x, yi = yri.y;
#else
            float ya = 0.f, yb = 0.f, za = 0.f, zb = 0.f;
#pragma unroll
            for (int jj = 0; jj < 8; jj += 2) {
                ya = fmaf(T[jj], X[jj], ya);
                yb = fmaf(T[jj + 1], X[jj + 1], yb);
                za = fmaf(T[8 + jj], X[jj], za);
                zb = fmaf(T[9 + jj], X[jj + 1], zb);
            }
            const float yr = ya + yb, yi = za + zb;
#endif
            float dr, di;
            int lab;
            float2 tcur = make_float2(0.f, 0.f);
            if constexpr (TRAIN) tcur = trr[(i & (kTrainRing - 1)) * kBlockThreads];
            const bool trn = i < ntr;
            if constexpr (SQ > 0) {
                // branch-free: no F2I (MIO) and no control flow on the chain.
                // (v + 1.5*2^23) - 1.5*2^23 == rint(v) for |v| < 2^22.
                constexpr float kMagic = 12582912.0f;
                const float m1f = static_cast<float>(m1);
#if KK_DD_SLICER_PACKED
                const float2 v2 = __ffma2_rn(yri, make_float2(half_norm, half_norm), make_float2(off, off));
                const float vr = v2.x, vi = v2.y;
                const float2 vc2 = make_float2(fminf(fmaxf(vr, 0.f), m1f), fminf(fmaxf(vi, 0.f), m1f));
                const float2 f2 = __fadd2_rn(__fadd2_rn(vc2, make_float2(kMagic, kMagic)),
                                             make_float2(-kMagic, -kMagic));
                const float2 dv = __fadd2_rn(vc2, make_float2(-f2.x, -f2.y));
                float fr = f2.x, fi = f2.y;
                float mg_s = 0.5f - fmaxf(fabsf(dv.x), fabsf(dv.y));
#else
                const float vr = fmaf(yr, half_norm, off), vi = fmaf(yi, half_norm, off);
                // distance to the nearest decision boundary; an edge level has
                // none on its outer side, so v is clamped to the level range
                // first (margin 0.5 there: conservative)
                const float vcr = fminf(fmaxf(vr, 0.f), m1f), vci = fminf(fmaxf(vi, 0.f), m1f);
                float fr = (vcr + kMagic) - kMagic;
                float fi = (vci + kMagic) - kMagic;
                float mg_s = 0.5f - fmaxf(fabsf(vcr - fr), fabsf(vci - fi));
#endif
                if constexpr (!WITH_P) {
                    const bool near = live && !trn && mg_s < kTieEps;
                    if (__any_sync(0xffffffffu, near) && near)
                        tie_rule(i, vr, vi, m1f, SQ, fr, fi, mg_s, tie0, tie1, ties_dirty);
                }
                mgl = (live && !trn) ? fminf(mgl, mg_s) : mgl;
                const int ir = __float_as_int(fr + kMagic) - __float_as_int(kMagic);
                const int ii = __float_as_int(fi + kMagic) - __float_as_int(kMagic);
                // level value (2 i - (m-1)) * h: exact for the constellation
                // (checked on the host, Slicer::sep)
#if KK_DD_SLICER_PACKED
                const float2 lev = __fmul2_rn(__ffma2_rn(make_float2(2.0f, 2.0f), make_float2(fr, fi),
                                                         make_float2(-m1f, -m1f)),
                                              make_float2(lev_h, lev_h));
                dr = trn ? tcur.x : lev.x;
                di = trn ? tcur.y : lev.y;
#else
                dr = trn ? tcur.x : fmaf(2.0f, fr, -static_cast<float>(m1)) * lev_h;
                di = trn ? tcur.y : fmaf(2.0f, fi, -static_cast<float>(m1)) * lev_h;
#endif
                int sl_lab;
                if constexpr (SQ == 2) sl_lab = (glab >> (8 * (ir * 2 + ii))) & 0xff;
                else sl_lab = grid[ir * SQ + ii];
                lab = trn ? 255 : sl_lab;
            } else {
                // square grid whose points are not exactly the fp32 level
                // products (e.g. 16/64-QAM at unit power): table values.
                // (computed for every lane: the warp vote must be convergent)
                float vr = 0.f, vi = 0.f, fr = 0.f, fi = 0.f, mg_s = 3.0e38f;
                const float m1f = static_cast<float>(m1);
                if (sl.kind == 0) {
                    vr = fmaf(yr, half_norm, off);
                    vi = fmaf(yi, half_norm, off);
                    const float vcr = fminf(fmaxf(vr, 0.f), m1f), vci = fminf(fmaxf(vi, 0.f), m1f);
                    fr = rintf(vcr);
                    fi = rintf(vci);
                    mg_s = 0.5f - fmaxf(fabsf(vcr - fr), fabsf(vci - fi));
                    if constexpr (!WITH_P) {
                        const bool near = live && !trn && mg_s < kTieEps;
                        if (__any_sync(0xffffffffu, near) && near)
                            tie_rule(i, vr, vi, m1f, m, fr, fi, mg_s, tie0, tie1, ties_dirty);
                    }
                }
                if (trn) {
                    dr = tcur.x; di = tcur.y;
                    lab = 255;
                } else if (sl.kind == 0) {
                    if (live) mgl = fminf(mgl, mg_s);
                    const int ir = static_cast<int>(fr), ii = static_cast<int>(fi);
                    lab = grid[ir * m + ii];
                    const float2 pp = pts[lab];
                    dr = pp.x; di = pp.y;
                } else {
                    float m_;
                    lab = slice(sl, yr, yi, m_);
                    if (live) mgb = fminf(mgb, m_);
                    const float2 pp = pts[lab];
                    dr = pp.x; di = pp.y;
                }
            }
            {
                const float d2 = fmaf(yr, yr, yi * yi);
                my2 = live ? fmaxf(my2, d2) : my2;
                // every pass (the P pass too: a block not re-run later keeps these)
                const bool exc = live && d2 > thr2;
                if (__any_sync(0xffffffffu, exc) && exc) {
                    if (g_prev == i - 1) {
                        ++g_run;
                    } else {
                        g_run = 1;
                        g_start = i;
                    }
                    g_prev = i;
                    if (g_start == 0) g_lead = g_run;
                    else if (g_run == a.guard_run && g_first == 0xffff) g_first = i;
                }
            }
#if KK_DD_PACKED
            const float2 e2p = __fmul2_rn(make_float2(tm, tm), __fadd2_rn(make_float2(dr, di), make_float2(-yr, -yi)));
            const float er = live ? e2p.x : 0.f, ei = live ? e2p.y : 0.f;
#else
            const float er = live ? tm * (dr - yr) : 0.f, ei = live ? tm * (di - yi) : 0.f;
#endif
            if constexpr (WITH_P) {
                float n2 = 0.f;
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) n2 = fmaf(X[jj], X[jj], n2);
                mx = fmaxf(mx, n2);     // rows past nk are zero-filled
                if constexpr (LIN) {
                    // P <- P - mu (P X) X^T - mu (P JX) JX^T
                    float JX[8];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        JX[2 * u] = X[2 * u + 1];
                        JX[2 * u + 1] = -X[2 * u];
                    }
                    float v[8], w[8];
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        float sa = 0.f, sb = 0.f;
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) {
                            sa = fmaf(P[r * 8 + jj], X[jj], sa);
                            sb = fmaf(P[r * 8 + jj], JX[jj], sb);
                        }
                        v[r] = live ? sa * (0.5f * tm) : 0.f;
                        w[r] = live ? sb * (0.5f * tm) : 0.f;
                    }
#pragma unroll
                    for (int r = 0; r < 8; ++r)
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj)
                            P[r * 8 + jj] = fmaf(-w[r], JX[jj], fmaf(-v[r], X[jj], P[r * 8 + jj]));
                } else {
#if KK_DD_PACKED
                    // rows (2q, 2q + 1) as pairs: the scalar form's fma order per row
                    float2 nv[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        float2 sacc = make_float2(0.f, 0.f);
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj)
                            sacc = __ffma2_rn(make_float2(P[2 * q * 8 + jj], P[(2 * q + 1) * 8 + jj]),
                                              make_float2(X[jj], X[jj]), sacc);
                        nv[q] = live ? __fmul2_rn(sacc, make_float2(-tm, -tm)) : make_float2(0.f, 0.f);
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q)
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) {
                            const float2 np = __ffma2_rn(nv[q], make_float2(X[jj], X[jj]),
                                                         make_float2(P[2 * q * 8 + jj], P[(2 * q + 1) * 8 + jj]));
                            P[2 * q * 8 + jj] = np.x;
                            P[(2 * q + 1) * 8 + jj] = np.y;
                        }
#else
                    float v[8];
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        float sacc = 0.f;
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) sacc = fmaf(P[r * 8 + jj], X[jj], sacc);
                        v[r] = live ? sacc * tm : 0.f;
                    }
#pragma unroll
                    for (int r = 0; r < 8; ++r)
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) P[r * 8 + jj] = fmaf(-v[r], X[jj], P[r * 8 + jj]);
#endif
                }
            }
            if constexpr (LIN) {
                // T0 += mu (e_r X + e_i JX), T1 = T0 M
                const float el = 0.5f * er, fl = 0.5f * ei;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float x0 = X[2 * u], x1 = X[2 * u + 1];
                    const float d0 = fmaf(el, x0, fl * x1);
                    const float d1 = fmaf(el, x1, -fl * x0);
                    T[2 * u] += d0;
                    T[2 * u + 1] += d1;
                    T[8 + 2 * u] -= d1;
                    T[9 + 2 * u] += d0;
                }
            } else {
#if KK_DD_PACKED
                const float2 e2 = make_float2(er, ei);
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    const float2 nt = __ffma2_rn(e2, make_float2(X[jj], X[jj]), make_float2(T[jj], T[8 + jj]));
                    T[jj] = nt.x;
                    T[8 + jj] = nt.y;
                }
#else
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    T[jj] = fmaf(er, X[jj], T[jj]);
                    T[8 + jj] = fmaf(ei, X[jj], T[8 + jj]);
                }
#endif
            }
            hsh = live ? (hsh ^ static_cast<unsigned long long>(lab & 0xff)) * 1099511628211ull : hsh;
            soft8[j] = make_float2(yr, yi);
            lab8[j >> 2] |= static_cast<unsigned>(lab & 0xff) << (8 * (j & 3));
        }
        if (!WITH_P && (write_out & 1)) {   // outputs from output passes
            const int i0 = c * kChunkRows;
            // vector stores need 16 B (soft) / 8 B (labels) alignment of the
            // run: block starts k0 = b B are multiples of 8 when B is
            if ((a.B & 7) == 0 && i0 + kChunkRows <= nk) {
                float4* s4 = reinterpret_cast<float4*>(sp + i0);
#pragma unroll
                for (int j = 0; j < kChunkRows / 2; ++j)
                    s4[j] = make_float4(soft8[2 * j].x, soft8[2 * j].y, soft8[2 * j + 1].x, soft8[2 * j + 1].y);
                *reinterpret_cast<uint2*>(lp + i0) = make_uint2(lab8[0], lab8[1]);
            } else {
#pragma unroll
                for (int j = 0; j < kChunkRows; ++j)
                    if (i0 + j < nk) {
                        sp[i0 + j] = soft8[j];
                        lp[i0 + j] = static_cast<uint8_t>(lab8[j >> 2] >> (8 * (j & 3)));
                    }
            }
        }
    }
    cp_async_wait<0>();
    unsigned long long changed = 0;
    if (run) {
        changed = (o.hash[b] != hsh) ? 1ull : 0ull;
        o.hash[b] = hsh;
        // Q_b = T_end - T_start P_b
        const float* Pm = Pb + b * 64;
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                float acc = T[r * 8 + j];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    float pij;
                    if constexpr (WITH_P) pij = P[i * 8 + j];
                    else pij = __ldg(Pm + i * 8 + j);
                    acc = fmaf(-Tstart[b * 16 + r * 8 + i], pij, acc);
                }
                o.Q[b * 16 + r * 8 + j] = acc;
            }
#pragma unroll
        for (int i = 0; i < 16; ++i) o.Tused[b * 16 + i] = Tstart[b * 16 + i];
        if (!WITH_P && (write_out & 1)) {
#pragma unroll
            for (int i = 0; i < 16; ++i) o.Twritten[b * 16 + i] = Tstart[b * 16 + i];
        }
        if constexpr (!WITH_P) {
            if (ties_dirty) o.ties[b] = make_uint2(tie0, tie1);
        }
        const bool sq = SQ > 0 || sl.kind == 0;
        const float mg = sq ? fminf(mgl, 0.5f * 3.0e38f) * (2.0f / sl.norm) : mgb;
        // guard certificate: without exceedances the block maximum is the
        // closest to the threshold; a block with exceedances gets margin 0
        // (re-run whenever its start moves: rare, and exact)
        const float gm = my2 > thr2 ? 0.f : sl.thr - sqrtf(my2);
        o.margin[b] = fminf(mg, gm);
        o.over[b] = my2 > thr2 ? 1 : 0;
        {
            // first in-block run stored +1 (0: none), so a zeroed table means "no runs"
            const int full = g_lead >= nk ? 1 : 0;
            const int suf = g_prev == nk - 1 ? g_run : 0;
            o.grun[b] = make_int2((g_lead & 0xffff) | ((suf & 0xffff) << 16),
                                  ((g_first == 0xffff ? 0 : g_first + 1) & 0xffff) | (full << 16));
            if (!WITH_P && my2 > thr2) atomicMax(o.counters + 2, 1ull);   // an exceedance seen: guard checks from now on
        }
        if (b == a.nb - 1) {
#pragma unroll
            for (int i = 0; i < 16; ++i) o.Tend[i] = T[i];
        }
        if constexpr (WITH_P) {
#pragma unroll
            for (int i = 0; i < 64; ++i) Pb[b * 64 + i] = P[i];
            maxx2[b] = mx;
        }
    }
    unsigned long long rr = run ? 1ull : 0ull;
    const unsigned first = __reduce_min_sync(0xffffffffu, changed ? static_cast<unsigned>(b) : 0xffffffffu);
#pragma unroll
    for (int off_ = 16; off_ > 0; off_ >>= 1) {
        changed += __shfl_xor_sync(0xffffffffu, changed, off_);
        rr += __shfl_xor_sync(0xffffffffu, rr, off_);
    }
    if (lane == 0) {
        if (changed) {
            atomicAdd(o.counters + 0, changed);
            atomicMin(o.first_changed, first);
        }
        if (rr) atomicAdd(o.counters + 1, rr);
    }
}

// Which blocks must re-run: |T_new - T_used|_F * max|x| >= min(margin, tol)
// (decision / guard margin certificate, soft tolerance), compacted into a
// list (warp-aggregated append; block order inside a warp preserved).
// Output passes (Twritten != null): also re-run every block whose start moved
// by more than tol since its outputs were last written (or never were).
__global__ void ddlms_select_kernel(const float* __restrict__ Tstart, const float* __restrict__ Tused,
                                    const float* __restrict__ margin, const float* __restrict__ maxx2, float mu,
                                    int64_t b_lo, int64_t nb, float tol, const float* __restrict__ Twritten,
                                    int* __restrict__ list, unsigned long long* __restrict__ list_n,
                                    const int* __restrict__ ctl) {
    if (ctl) {   // device-driven pass mode: output passes check Twritten against tol
        const int mode = *ctl;
        if (mode == kModeDone) return;
        if (mode != kModeOutput) {
            Twritten = nullptr;
            tol = 3.0e38f;
        }
    }
    const int64_t b = b_lo + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    bool run = false;
    if (b < nb) {
        float d2 = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const float d = Tstart[b * 16 + i] - Tused[b * 16 + i];
            d2 = fmaf(d, d, d2);
        }
        const float bound = sqrtf(d2 * maxx2[b]);
        run = !(bound < fminf(margin[b], Twritten ? 3.0e38f : tol)) || (mu * maxx2[b] > 1.0f);
        if (Twritten) {
            float w2 = 0.f;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float d = Tstart[b * 16 + i] - Twritten[b * 16 + i];
                w2 = fmaf(d, d, w2);
            }
            run = run || !(sqrtf(w2 * maxx2[b]) < tol);
        }
    }
    const unsigned m = __ballot_sync(0xffffffffu, run);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(list_n, static_cast<unsigned long long>(__popc(m)));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (run) list[base + __popc(m & ((1u << lane) - 1u))] = static_cast<int>(b);
}

// fold groups of G (<= 32) consecutive maps:  (P, Q) <- (P P_c, Q P_c + Q_c)
// One warp per group.  The group's children (P_c, Q_c) are first staged in
// shared memory with all loads in flight, then folded serially from smem.
constexpr int kScanWarps = 2;

// Stage a group's nc children (P_c: 64 floats, Q_c: 16 floats each, both
// contiguous in global memory) into the warp's padded smem tiles with all
// loads issued up front (float4, coalesced): the per-child load loop this
// replaces serialised ~32 global latencies per group.
__device__ __forceinline__ void stage_children(const float* __restrict__ Pc, const float* __restrict__ Qc,
                                               int64_t c0, int nc, int l, float (*cP)[65], float (*cQ)[17]) {
    if (nc <= 0) return;
    const float4* p4 = reinterpret_cast<const float4*>(Pc + c0 * 64);
    const float4* q4 = reinterpret_cast<const float4*>(Qc + c0 * 16);
    float4 pv[16], qv[4];
    const int np4 = nc * 16, nq4 = nc * 4;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int e = l + 32 * k;
        pv[k] = e < np4 ? __ldg(p4 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int e = l + 32 * k;
        qv[k] = e < nq4 ? __ldg(q4 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int e = l + 32 * k;
        if (e < np4) {
            float* d = &cP[e >> 4][(e & 15) * 4];
            d[0] = pv[k].x; d[1] = pv[k].y; d[2] = pv[k].z; d[3] = pv[k].w;
        }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int e = l + 32 * k;
        if (e < nq4) {
            float* d = &cQ[e >> 2][(e & 3) * 4];
            d[0] = qv[k].x; d[1] = qv[k].y; d[2] = qv[k].z; d[3] = qv[k].w;
        }
    }
    __syncwarp();
}

__global__ void __launch_bounds__(32 * kScanWarps)
scan_fold_kernel(const float* __restrict__ Pc, const float* __restrict__ Qc, int64_t n_child, int G,
                 float* __restrict__ Pg, float* __restrict__ Qg, int64_t n_grp, int with_p,
                 const int* __restrict__ ctl) {
    if (ctl_done(ctl)) return;
    __shared__ float sP[kScanWarps][64];
    __shared__ float sQ[kScanWarps][16];
    __shared__ float cP[kScanWarps][32][65];
    __shared__ float cQ[kScanWarps][32][17];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int64_t g = int64_t(blockIdx.x) * kScanWarps + w;
    if (g >= n_grp) return;
    const int64_t c0 = g * G;
    const int nc = static_cast<int>(min(static_cast<int64_t>(G), n_child - c0));
    stage_children(Pc, Qc, c0, nc, l, cP[w], cQ[w]);
    float* P = sP[w];
    float* Q = sQ[w];
    P[2 * l] = ((2 * l) % 9 == 0) ? 1.f : 0.f;
    P[2 * l + 1] = ((2 * l + 1) % 9 == 0) ? 1.f : 0.f;
    if (l < 16) Q[l] = 0.f;
    __syncwarp();
    const int pi = (2 * l) >> 3, pj = (2 * l) & 7;   // P entries (pi, pj), (pi, pj+1)
    const int qr = l >> 3, qj = l & 7;               // Q entry (qr, qj) for l < 16
    for (int c = 0; c < nc; ++c) {
        const float* M = cP[w][c];
        float q = 0.f, p0 = 0.f, p1 = 0.f;
        if (l < 16) {
            q = cQ[w][c][l];
#pragma unroll
            for (int k = 0; k < 8; ++k) q = fmaf(Q[qr * 8 + k], M[k * 8 + qj], q);
        }
        if (with_p) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float a = P[pi * 8 + k];
                p0 = fmaf(a, M[k * 8 + pj], p0);
                p1 = fmaf(a, M[k * 8 + pj + 1], p1);
            }
        }
        __syncwarp();
        if (l < 16) Q[l] = q;
        if (with_p) { P[2 * l] = p0; P[2 * l + 1] = p1; }
        __syncwarp();
    }
    if (l < 16) Qg[g * 16 + l] = Q[l];
    if (with_p) { Pg[g * 64 + 2 * l] = P[2 * l]; Pg[g * 64 + 2 * l + 1] = P[2 * l + 1]; }
}

// down-sweep: children start taps from the group start taps, one warp per
// group (lanes 0..15 own T entries); children staged in smem first
__global__ void __launch_bounds__(32 * kScanWarps)
scan_down_kernel(const float* __restrict__ Pc, const float* __restrict__ Qc, int64_t n_child, int G,
                 const float* __restrict__ Tg, int64_t n_grp, float* __restrict__ Tc,
                 const int* __restrict__ ctl) {
    if (ctl_done(ctl)) return;
    __shared__ float sT[kScanWarps][16];
    __shared__ float cP[kScanWarps][32][65];
    __shared__ float cQ[kScanWarps][32][17];
    __shared__ float oT[kScanWarps][32][17];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int64_t g = int64_t(blockIdx.x) * kScanWarps + w;
    if (g >= n_grp) return;
    const int64_t c0 = g * G;
    const int nc = static_cast<int>(min(static_cast<int64_t>(G), n_child - c0));
    stage_children(Pc, Qc, c0, nc - 1, l, cP[w], cQ[w]);
    float* T = sT[w];
    if (l < 16) T[l] = Tg[g * 16 + l];
    __syncwarp();
    const int r = l >> 3, j = l & 7;
    for (int c = 0; c < nc; ++c) {
        if (l < 16) oT[w][c][l] = T[l];
        if (c + 1 == nc) break;
        const float* M = cP[w][c];
        float t = 0.f;
        if (l < 16) {
            t = cQ[w][c][l];
#pragma unroll
            for (int k = 0; k < 8; ++k) t = fmaf(T[r * 8 + k], M[k * 8 + j], t);
        }
        __syncwarp();
        if (l < 16) T[l] = t;
        __syncwarp();
    }
    __syncwarp();
    // the group's children are contiguous: one coalesced sweep
    for (int e = l; e < nc * 16; e += 32) Tc[c0 * 16 + e] = oT[w][e >> 4][e & 15];
}

// ---------------------------------------------------------------------------
// symbol sync (rxdsp.py:574-601): |xcorr| of both 2-sps parities with the
// reference, argmax, sidelobe RMS; plus the head RMS for eq_scale
// (rxdsp.py:734-737).  float64 accumulation.
// ---------------------------------------------------------------------------
__global__ void xcorr_kernel(const float2* __restrict__ head, int64_t n_head, const float2* __restrict__ ref,
                             int n_ref, int64_t n_lag0, int64_t n_lag1, double* __restrict__ mag) {
    extern __shared__ float2 sref[];
    for (int i = threadIdx.x; i < n_ref; i += blockDim.x) sref[i] = ref[i];
    __syncthreads();
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t tot = n_lag0 + n_lag1;
    if (t >= tot) return;
    const int parity = t < n_lag0 ? 0 : 1;
    const int64_t k = parity ? t - n_lag0 : t;
    float re[4] = {0.f, 0.f, 0.f, 0.f}, im[4] = {0.f, 0.f, 0.f, 0.f};
    const float2* zp = head + parity + 2 * k;
    int i = 0;
    for (; i + 4 <= n_ref; i += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float2 z = __ldg(zp + 2 * (i + u));
            const float2 r = sref[i + u];
            re[u] = fmaf(z.x, r.x, fmaf(z.y, r.y, re[u]));      // z * conj(r)
            im[u] = fmaf(z.y, r.x, fmaf(-z.x, r.y, im[u]));
        }
    }
    for (; i < n_ref; ++i) {
        const float2 z = __ldg(zp + 2 * i);
        const float2 r = sref[i];
        re[0] = fmaf(z.x, r.x, fmaf(z.y, r.y, re[0]));
        im[0] = fmaf(z.y, r.x, fmaf(-z.x, r.y, im[0]));
    }
    const double R = (static_cast<double>(re[0]) + re[1]) + (static_cast<double>(re[2]) + re[3]);
    const double I = (static_cast<double>(im[0]) + im[1]) + (static_cast<double>(im[2]) + im[3]);
    mag[t] = sqrt(R * R + I * I);
}

// Tiled form: a CTA owns kXcTile consecutive lags of one parity (thread t:
// lags t + 256 m, m < 4) and one kXcChunk-symbol segment of the reference
// (blockIdx.z), both staged in shared memory, so each head sample is read
// from L2 once per tile instead of once per lag (the per-lag kernel above
// re-read the window for every lag, ~2 GB of L1/L2 loads per stream head),
// and a 2^16-lag head gives 512 CTAs.  fp32 sums within a segment; the
// segments' float64 partials are combined in a fixed order (deterministic).
constexpr int kXcThreads = 256, kXcPer = 4, kXcTile = kXcThreads * kXcPer, kXcChunk = 512;
__global__ void __launch_bounds__(kXcThreads) xcorr_tiled_kernel(const float2* __restrict__ head, int64_t n_head,
                                                                 const float2* __restrict__ ref, int n_ref,
                                                                 int64_t n_lag0, int64_t n_lag1,
                                                                 double2* __restrict__ part) {
    __shared__ float2 sref[kXcChunk];
    __shared__ float2 sz[kXcTile + kXcChunk];
    const int parity = blockIdx.y;
    const int64_t nl = parity ? n_lag1 : n_lag0;
    const int64_t k0 = int64_t(blockIdx.x) * kXcTile;
    if (k0 >= nl) return;
    const int t = threadIdx.x;
    const int i0 = blockIdx.z * kXcChunk;
    const int nc = min(kXcChunk, n_ref - i0);
    for (int c = t; c < kXcChunk; c += kXcThreads) sref[c] = c < nc ? ref[i0 + c] : make_float2(0.f, 0.f);
    for (int j = t; j < kXcTile + kXcChunk; j += kXcThreads) {
        const int64_t si = parity + 2 * (k0 + i0 + j);
        sz[j] = si < n_head ? __ldg(head + si) : make_float2(0.f, 0.f);
    }
    __syncthreads();
    float re[kXcPer], im[kXcPer];
#pragma unroll
    for (int m = 0; m < kXcPer; ++m) re[m] = im[m] = 0.f;
#pragma unroll 8
    for (int c = 0; c < kXcChunk; ++c) {
        const float2 r = sref[c];
#pragma unroll
        for (int m = 0; m < kXcPer; ++m) {
            const float2 z = sz[t + kXcThreads * m + c];
            re[m] = fmaf(z.x, r.x, fmaf(z.y, r.y, re[m]));      // z * conj(r)
            im[m] = fmaf(z.y, r.x, fmaf(-z.x, r.y, im[m]));
        }
    }
    // part[segment][lag], lags of both parities concatenated (parity 1 at n_lag0)
    double2* out = part + int64_t(blockIdx.z) * (n_lag0 + n_lag1) + (parity ? n_lag0 : 0);
#pragma unroll
    for (int m = 0; m < kXcPer; ++m) {
        const int64_t k = k0 + t + kXcThreads * m;
        if (k < nl) out[k] = make_double2(re[m], im[m]);
    }
}

__global__ void xcorr_combine_kernel(const double2* __restrict__ part, int n_seg, int64_t n_lags,
                                     double* __restrict__ mag) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n_lags; k += int64_t(gridDim.x) * blockDim.x) {
        double R = 0.0, I = 0.0;
        for (int sgm = 0; sgm < n_seg; ++sgm) {
            const double2 v = part[int64_t(sgm) * n_lags + k];
            R += v.x;
            I += v.y;
        }
        mag[k] = sqrt(R * R + I * I);
    }
}

__global__ void sync_reduce_kernel(const double* __restrict__ mag, int64_t n_lag0, int64_t n_lag1,
                                   const float2* __restrict__ head, int64_t n_head, int64_t skip,
                                   double* __restrict__ res) {
    // res: [0] best parity, [1] k, [2] ratio, [3] rms of head[skip:]
    __shared__ double sd[1024];
    __shared__ long long si[1024];
    const int tid = threadIdx.x;
    double best_ratio = -1.0;
    long long best_k = -1;
    int best_p = -1;
    for (int parity = 0; parity < 2; ++parity) {
        const int64_t n = parity ? n_lag1 : n_lag0;
        if (n <= 0) continue;
        const double* m = mag + (parity ? n_lag0 : 0);
        double bv = -1.0;
        long long bi = 0;
        for (int64_t i = tid; i < n; i += blockDim.x)
            if (m[i] > bv) { bv = m[i]; bi = i; }
        sd[tid] = bv;
        si[tid] = bi;
        __syncthreads();
        for (int s = blockDim.x / 2; s > 0; s >>= 1) {
            if (tid < s) {
                const double ov = sd[tid + s];
                const long long oi = si[tid + s];
                if (ov > sd[tid] || (ov == sd[tid] && oi < si[tid])) { sd[tid] = ov; si[tid] = oi; }
            }
            __syncthreads();
        }
        const double peak = sd[0];
        const long long k = si[0];
        __syncthreads();
        double acc = 0.0;
        for (int64_t i = tid; i < n; i += blockDim.x)
            if (i < k - 2 || i > k + 2) acc += m[i] * m[i];
        sd[tid] = acc;
        __syncthreads();
        for (int s = blockDim.x / 2; s > 0; s >>= 1) {
            if (tid < s) sd[tid] += sd[tid + s];
            __syncthreads();
        }
        const long long lo = k - 2 < 0 ? 0 : k - 2;
        const long long hi = k + 3 > n ? n : k + 3;
        const long long n_side = n - (hi - lo);
        const double rms = n_side > 0 ? sqrt(sd[0] / static_cast<double>(n_side)) : 1e-30;
        const double ratio = peak / rms;
        if (ratio > best_ratio) { best_ratio = ratio; best_k = k; best_p = parity; }
        __syncthreads();
    }
    double acc = 0.0;
    for (int64_t i = skip + tid; i < n_head; i += blockDim.x) {
        const float2 v = head[i];
        acc += static_cast<double>(v.x) * v.x + static_cast<double>(v.y) * v.y;
    }
    sd[tid] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (tid < s) sd[tid] += sd[tid + s];
        __syncthreads();
    }
    if (tid == 0) {
        res[0] = best_p;
        res[1] = static_cast<double>(best_k);
        res[2] = best_ratio;
        const int64_t cnt = n_head - skip;
        res[3] = cnt > 0 ? sqrt(sd[0] / static_cast<double>(cnt)) : 0.0;
    }
}

// ---------------------------------------------------------------------------
// BER: bit errors between decided point indices and reference point indices
// (demap rxdsp.py:548-567 + XOR count runner.py:360-362), per-window counts
// ---------------------------------------------------------------------------
__global__ void bit_errors_kernel(const uint8_t* __restrict__ lab, const uint8_t* __restrict__ ref, int64_t n,
                                  const uint8_t* __restrict__ point_label, int64_t win_syms,
                                  unsigned long long* __restrict__ total, unsigned int* __restrict__ win,
                                  int64_t ex_period, int64_t ex_len, int64_t ex_phase,
                                  unsigned long long* __restrict__ n_counted) {
    __shared__ uint8_t pl[64];
    if (threadIdx.x < 64) pl[threadIdx.x] = point_label[threadIdx.x];
    __syncthreads();
    // each thread owns a contiguous run of 16 symbols (one uint4 of each
    // array); the seam phase is tracked incrementally (no 64-bit modulo)
    unsigned long long e = 0, cnt = 0;
    const int64_t n16 = n / 16;
    const uint4* L4 = reinterpret_cast<const uint4*>(lab);
    const uint4* R4 = reinterpret_cast<const uint4*>(ref);
    const bool aligned = ((reinterpret_cast<uintptr_t>(lab) | reinterpret_cast<uintptr_t>(ref)) & 15) == 0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    const int64_t t0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    // seam phase of the thread's first run, then advanced by 16 * stride
    // (mod period) per trip: one 64-bit modulo per thread, not per trip
    int64_t ph_run = ex_period > 0 ? (16 * t0 + ex_phase) % ex_period : 0;
    const int64_t ph_step = ex_period > 0 ? (16 * stride) % ex_period : 0;
    for (int64_t t = t0; t < (aligned ? n16 : 0); t += stride) {
        const uint4 a4 = L4[t], b4 = R4[t];
        const uint8_t* a = reinterpret_cast<const uint8_t*>(&a4);
        const uint8_t* b = reinterpret_cast<const uint8_t*>(&b4);
        int64_t ph = ph_run;
        if (ex_period > 0) {
            ph_run += ph_step;
            if (ph_run >= ex_period) ph_run -= ex_period;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const bool skip = ex_period > 0 && ph >= ex_period - ex_len;
            if (ex_period > 0 && ++ph == ex_period) ph = 0;
            if (skip) continue;
            ++cnt;
            const unsigned c = __popc(static_cast<unsigned>(pl[a[u] & 63] ^ pl[b[u] & 63]));
            e += c;
            if (win && c) atomicAdd(win + (16 * t + u) / win_syms, c);
        }
    }
    // tail (or the whole range when unaligned)
    for (int64_t i = (aligned ? n16 * 16 : 0) + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        if (ex_period > 0 && ((i + ex_phase) % ex_period) >= ex_period - ex_len) continue;
        ++cnt;
        const unsigned c = __popc(static_cast<unsigned>(pl[lab[i] & 63] ^ pl[ref[i] & 63]));
        e += c;
        if (win && c) atomicAdd(win + i / win_syms, c);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        e += __shfl_xor_sync(0xffffffffu, e, o);
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (e) atomicAdd(total, e);
        if (cnt && n_counted) atomicAdd(n_counted, cnt);
    }
}

// nearest point (first minimum wins) + fallback count (rxdsp.py:560-565)
__global__ void demap_kernel(const float2* __restrict__ sym, int64_t n, Slicer sl, uint8_t* __restrict__ idx,
                             unsigned long long* __restrict__ n_fallback) {
    unsigned long long fb = 0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const float2 y = sym[i];
        int best = 0;
        float bd = 3.0e38f;
        for (int p = 0; p < sl.npts; ++p) {
            const float dr = y.x - sl.pts[p].x, di = y.y - sl.pts[p].y;
            const float d = dr * dr + di * di;
            if (d < bd) { bd = d; best = p; }
        }
        idx[i] = static_cast<uint8_t>(best);
        if (bd > 1e-18f) ++fb;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) fb += __shfl_xor_sync(0xffffffffu, fb, o);
    if ((threadIdx.x & 31) == 0 && fb) atomicAdd(n_fallback, fb);
}

}  // namespace kk

// ===========================================================================
// C ABI
// ===========================================================================
using namespace kk;

static Slicer make_slicer(int order, const float* pts_ri, const uint8_t* grid, int grid_m, float norm,
                          float max_radius, float guard_factor) {
    Slicer s{};
    s.npts = order;
    s.kind = grid_m > 0 ? 0 : 1;
    s.m = grid_m;
    s.norm = norm;
    s.thr = guard_factor * max_radius;
    for (int i = 0; i < order && i < 64; ++i) s.pts[i] = make_float2(pts_ri[2 * i], pts_ri[2 * i + 1]);
    if (grid_m > 0)
        for (int i = 0; i < grid_m * grid_m && i < 64; ++i) s.grid[i] = grid[i];
    s.sep = 0;
    s.lev_h = 0.f;
    if (grid_m == 2 || grid_m == 4 || grid_m == 8) {
        // h = the first positive level (2 i - (m-1) == 1); every point must be
        // reproduced bit-exactly by the device formula
        const float h = s.pts[s.grid[(grid_m / 2) * grid_m]].x;
        bool ok = h > 0.f;
        for (int i = 0; i < grid_m; ++i)
            for (int j = 0; j < grid_m; ++j) {
                const float2 p = s.pts[s.grid[i * grid_m + j]];
                const volatile float lr = static_cast<float>(2 * i - (grid_m - 1)) * h;
                const volatile float li = static_cast<float>(2 * j - (grid_m - 1)) * h;
                ok = ok && p.x == lr && p.y == li;
            }
        s.sep = ok ? 1 : 0;
        s.lev_h = h;
    }
    return s;
}

extern "C" int kk_ddlms_sequential(const void* x, int64_t n_out, float scale, int n_taps, const void* train,
                                   int64_t n_train, void* wg, int* fz, int order, const float* pts_host,
                                   const uint8_t* grid_host, int grid_m, float norm, float max_radius,
                                   float guard_factor, int guard_run, float mu, int widely_linear,
                                   uint8_t* labels, void* soft, void* dec, void* stream) {
    clear_error();
    if (n_taps < 1 || n_taps > 16) return set_error(KK_ERR_PARAM, "n_taps must be in [1, 16]");
    if (order < 2 || order > 64) return set_error(KK_ERR_PARAM, "constellation order must be <= 64");
    if (n_out <= 0) return KK_OK;
    Slicer sl = make_slicer(order, pts_host, grid_host, grid_m, norm, max_radius, guard_factor);
    ddlms_seq_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const float2*>(x), n_out, scale, n_taps, static_cast<const float2*>(train), n_train,
        static_cast<float2*>(wg), fz, sl, mu, widely_linear, guard_run, labels, static_cast<float2*>(soft),
        static_cast<float2*>(dec));
    return check_launch("ddlms_seq_kernel");
}


// Small device->host reads through a per-thread pinned staging buffer (a
// copy to pageable memory goes through the driver's shared bounce buffer and
// stalls other host threads' CUDA calls while it waits on this stream).
// The copy is a kernel writing into mapped pinned memory, not a DMA: a
// DMA readback would queue behind bulk device->host transfers (the packed
// output bits of a streaming receive) on the copy engine, idling the solver
// between its passes.
__global__ void readback_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, int n16) {
    for (int i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
}

// Mapped pinned staging buffers for small readbacks, pooled process-wide:
// a call borrows one for its duration (threads never share one at a time),
// so the number allocated is bounded by the peak number of concurrent
// readers and no buffer is allocated per pipeline / worker thread.
namespace {
struct PinBuf {
    void* host = nullptr;
    void* dev = nullptr;
};
std::mutex g_pin_mu;
std::vector<PinBuf> g_pin_free;
constexpr size_t kPin = 64 << 10;

struct PinLease {
    PinBuf b;
    int rc = KK_OK;
    PinLease() {
        {
            std::lock_guard<std::mutex> lk(g_pin_mu);
            if (!g_pin_free.empty()) {
                b = g_pin_free.back();
                g_pin_free.pop_back();
                return;
            }
        }
        if (cudaHostAlloc(&b.host, kPin, cudaHostAllocMapped) != cudaSuccess ||
            cudaHostGetDevicePointer(&b.dev, b.host, 0) != cudaSuccess) {
            b = PinBuf{};
            rc = set_cuda_error("mapped pinned staging");
        }
    }
    ~PinLease() {
        if (b.host) {
            std::lock_guard<std::mutex> lk(g_pin_mu);
            g_pin_free.push_back(b);
        }
    }
};
}  // namespace

static int d2h_small(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes > kPin) return set_error(KK_ERR_PARAM, "d2h_small: too large");
    PinLease lease;
    if (lease.rc) return lease.rc;
    void* pin = lease.b.host;
    void* pin_dev = lease.b.dev;
    if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        const int n16 = static_cast<int>((bytes + 15) / 16);   // src regions are 256 B-aligned workspace slots
        readback_kernel<<<1, 256, 0, s>>>(static_cast<const uint4*>(src), static_cast<uint4*>(pin_dev), n16);
        if (int rc = check_launch("readback_kernel")) return rc;
    } else if (cudaMemcpyAsync(pin, src, bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess) {
        return set_cuda_error("device->host readback");
    }
    if (cudaStreamSynchronize(s) != cudaSuccess) return set_cuda_error("device->host readback");
    std::memcpy(dst, pin, bytes);
    return KK_OK;
}

namespace {
constexpr int kG = 32;   // scan fan-in

struct Level {
    int64_t n;
    float *P, *Q, *T;
};

size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

struct Layout {
    int64_t nb;
    std::vector<int64_t> n;  // entries per level (level 0 = blocks)
    size_t bytes;
};

Layout plan(int64_t nsym, int B) {
    Layout L;
    L.nb = (nsym + B - 1) / B;
    int64_t n = L.nb;
    L.n.push_back(n);
    while (n > kG) {
        n = (n + kG - 1) / kG;
        L.n.push_back(n);
    }
    size_t b = 0;
    for (size_t l = 0; l < L.n.size(); ++l) b += align_up(L.n[l] * 96 * sizeof(float));  // P64 + Q16 + T16
    b += align_up(L.nb * 16 * sizeof(float));   // Tused
    b += align_up(L.nb * 16 * sizeof(float));   // Twritten
    b += align_up(L.nb * sizeof(float)) * 2;    // margin, maxx2
    b += align_up(16 * sizeof(float));          // Tinit
    b += align_up(L.nb * sizeof(int));          // over
    b += align_up(L.nb * sizeof(unsigned long long));   // label hashes
    b += align_up(L.nb * sizeof(uint2));                 // tie slots
    b += align_up(L.nb * sizeof(int2));                  // guard runs
    b += align_up(size_t(nsym) * 8);                     // ST (soft, unless bound to the caller's)
    b += align_up(size_t(nsym));                         // LT (labels, idem)
    b += align_up(L.nb * sizeof(int));                   // re-run list
    b += align_up(sizeof(ReadBack));                     // counters, pass control, end taps
    L.bytes = b;
    return L;
}
}  // namespace

extern "C" size_t kk_ddlms_workspace_bytes(int64_t nsym, int block) {
    if (nsym <= 0 || block <= 0) return 0;
    return plan(nsym, block).bytes;
}

// ---------------------------------------------------------------------------
// DdlmsSolver: exact block-parallel WL DDLMS (4 taps) over one frame of nsym
// symbols, in phases so that frames on different GPUs can be chained by a
// host-side exchange of their composed affine maps (superframe / multirank):
//   train(T_start)      pure-training blocks (exact from any start) -> exact
//                       training-end taps
//   speculate(T_guess)  first pass of every decision-directed block from the
//                       guess, fused with the block maps P_b -> frame map
//   iterate(T_start)    exact frame start taps: scan, re-run blocks whose start
//                       moved beyond their certified margin, count changed
//                       blocks -> frame map
//   finish()            outputs (labels, soft), end taps, guard check
// A frame map (P, Q) means T_end = T_start P + Q (host float[64 + 16]).
// ---------------------------------------------------------------------------
namespace {
#ifndef KK_DD_TRAIN_FORK
#define KK_DD_TRAIN_FORK 1
#endif
// per-device non-blocking side stream for the training blocks' speculative
// pass (created once, never destroyed: process lifetime)
inline cudaStream_t train_side_stream() {
    static std::mutex mu;
    static cudaStream_t side[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if (!side[dev]) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if (cudaStreamCreateWithPriority(&side[dev], cudaStreamNonBlocking, hi) != cudaSuccess) side[dev] = nullptr;
    }
    return side[dev];
}

struct DdlmsSolver {
    cudaStream_t s;
    Layout L;
    std::vector<Level> lv;
    int top;
    Slicer sl;
    SolveArgs a;
    RunOut o;
    TOut to;
    float scale, soft_tol;
    float *Tused, *Twritten, *margin, *maxx2, *Tend, *Tinit_d;
    int* over;
    unsigned long long *hsh, *ctr;
    uint2* ties = nullptr;
    int2* grun = nullptr;
    float2* ST_own = nullptr;    // workspace soft / labels (outputs not bound)
    uint8_t* LT_own = nullptr;
    int* list;
    ReadBack* rb;
    const int* ctl_d = nullptr;   // device pass control while a device-driven loop is queued
    int64_t bt = 0;      // pure training blocks
    int64_t ntb = 0;     // blocks holding any training symbol
    bool speculated = false;
    bool speculated_async = false;   // solve_async: guard checks inside the loop
    int64_t iters = 0, reruns = 0, last_changed = 0;
    unsigned int last_first_changed = 0;   // lowest changed block of the last iteration (solve_loop)

    int scan_up(bool with_p) {
        const unsigned wblk = 32 * kScanWarps;
        for (int l = 1; l <= top; ++l) {
            const unsigned g = static_cast<unsigned>((lv[l].n + kScanWarps - 1) / kScanWarps);
            scan_fold_kernel<<<g, wblk, 0, s>>>(lv[l - 1].P, lv[l - 1].Q, lv[l - 1].n, kG, lv[l].P, lv[l].Q,
                                                lv[l].n, with_p ? 1 : 0, ctl_d);
            if (int rc = check_launch("scan_fold_kernel")) return rc;
        }
        return KK_OK;
    }
    int scan_down() {   // from Tinit_d (frame start, scaled)
        const unsigned wblk = 32 * kScanWarps;
        scan_down_kernel<<<1, wblk, 0, s>>>(lv[top].P, lv[top].Q, lv[top].n, static_cast<int>(lv[top].n), Tinit_d, 1,
                                            lv[top].T, ctl_d);
        if (int rc = check_launch("scan_down_kernel")) return rc;
        for (int l = top; l >= 1; --l) {
            const unsigned g = static_cast<unsigned>((lv[l].n + kScanWarps - 1) / kScanWarps);
            scan_down_kernel<<<g, wblk, 0, s>>>(lv[l - 1].P, lv[l - 1].Q, lv[l - 1].n, kG, lv[l].T, lv[l].n,
                                                lv[l - 1].T, ctl_d);
            if (int rc = check_launch("scan_down_kernel")) return rc;
        }
        return KK_OK;
    }
    // frame map from the top-level aggregates (host fold), unscaled Q
    int frame_map(float* agg) {
        if (!agg) return KK_OK;
        const int64_t n = lv[top].n;
        std::vector<float> P(n * 64), Q(n * 16);
        if (int rc = d2h_small(P.data(), lv[top].P, P.size() * 4, s)) return rc;
        if (int rc = d2h_small(Q.data(), lv[top].Q, Q.size() * 4, s)) return rc;
        double Pa[64], Qa[16];
        for (int i = 0; i < 64; ++i) Pa[i] = (i % 9 == 0) ? 1.0 : 0.0;
        for (int i = 0; i < 16; ++i) Qa[i] = 0.0;
        for (int64_t g = 0; g < n; ++g) {
            double nP[64], nQ[16];
            for (int r = 0; r < 8; ++r)
                for (int j = 0; j < 8; ++j) {
                    double acc = 0.0;
                    for (int k = 0; k < 8; ++k) acc += Pa[r * 8 + k] * P[g * 64 + k * 8 + j];
                    nP[r * 8 + j] = acc;
                }
            for (int r = 0; r < 2; ++r)
                for (int j = 0; j < 8; ++j) {
                    double acc = Q[g * 16 + r * 8 + j];
                    for (int k = 0; k < 8; ++k) acc += Qa[r * 8 + k] * P[g * 64 + k * 8 + j];
                    nQ[r * 8 + j] = acc;
                }
            for (int i = 0; i < 64; ++i) Pa[i] = nP[i];
            for (int i = 0; i < 16; ++i) Qa[i] = nQ[i];
        }
        for (int i = 0; i < 64; ++i) agg[i] = static_cast<float>(Pa[i]);
        for (int i = 0; i < 16; ++i) agg[64 + i] = static_cast<float>(Qa[i] / scale);
        return KK_OK;
    }
    // small host values go down as kernel arguments, not H2D copies: a copy
    // would queue behind the bulk input transfers of a streaming receive on
    // the (in-order) host->device copy engine
    int upload16(float* dst, const float* T_host) {
        Vec16 v;
        for (int i = 0; i < 16; ++i) v.v[i] = T_host[i] * scale;
        set16_kernel<<<1, 16, 0, s>>>(dst, v);
        return check_launch("set16_kernel");
    }
    int set_start(const float* T_host) { return upload16(Tinit_d, T_host); }
    int fill_T(int64_t b0, int64_t b1, const float* src_dev) {
        if (b1 <= b0) return KK_OK;
        fill_T_kernel<<<static_cast<unsigned>(((b1 - b0) * 16 + 127) / 128), 128, 0, s>>>(lv[0].T, b0, b1, src_dev);
        return check_launch("fill_T_kernel");
    }
    // Run blocks [b0, b1): the blocks holding training symbols (b < ntb) in a
    // TRAIN launch (range mode, in-kernel skip test), the rest in a plain
    // launch -- compacted into a re-run list first when use_skip.
    int run_blocks(bool with_p, int64_t b0, int64_t b1, int use_skip, float tol = 0.f, int write_out = 0,
                   const int* ext_list = nullptr) {
        if (b1 <= b0) return KK_OK;
        // kernel attributes once per device and process (ensure_smem_attr)
        {
            struct KS { const void* k; size_t smem; };
            const KS ks[] = {
#define KK_DD_K1(P_, S_, T_, L_) {reinterpret_cast<const void*>(ddlms_block_kernel<P_, S_, true, T_, L_>), T_ ? kStageSmem + kTrainSmem : kStageSmem}, \
                            {reinterpret_cast<const void*>(ddlms_block_kernel<P_, S_, false, T_, L_>), T_ ? kStageSmem + kTrainSmem : kStageSmem}
#define KK_DD_K(P_, S_, T_) KK_DD_K1(P_, S_, T_, false), KK_DD_K1(P_, S_, T_, true)
                KK_DD_K(true, 0, true), KK_DD_K(true, 2, true), KK_DD_K(true, 4, true), KK_DD_K(true, 8, true),
                KK_DD_K(false, 0, true), KK_DD_K(false, 2, true), KK_DD_K(false, 4, true), KK_DD_K(false, 8, true),
                KK_DD_K(true, 0, false), KK_DD_K(true, 2, false), KK_DD_K(true, 4, false), KK_DD_K(true, 8, false),
                KK_DD_K(false, 0, false), KK_DD_K(false, 2, false), KK_DD_K(false, 4, false), KK_DD_K(false, 8, false)
#undef KK_DD_K
#undef KK_DD_K1
            };
            for (const KS& k : ks)
                if (int rc = ensure_smem_attr(k.k, k.smem, "ddlms_block_kernel smem attribute")) return rc;
        }
        const int sq = sl.sep ? sl.m : 0;
        const bool al = (reinterpret_cast<uintptr_t>(a.x) & 15) == 0;
        auto launch = [&](bool train_blocks, int64_t lo, int64_t hi, int skip, const int* lst,
                          const unsigned long long* lst_n) {
            const unsigned g = static_cast<unsigned>((hi - lo + kBlockThreads - 1) / kBlockThreads);
            const size_t smem = train_blocks ? kStageSmem + kTrainSmem : kStageSmem;
            auto go = [&](auto kern) {
                kern<<<g, kBlockThreads, smem, s>>>(a, sl, lv[0].T, lv[0].P, maxx2, o, to, lo, hi, skip, tol, lst,
                                                    lst_n, write_out, ctl_d);
            };
#define KK_DD_GO4(P_, S_, T_, L_) (al ? go(ddlms_block_kernel<P_, S_, true, T_, L_>) : go(ddlms_block_kernel<P_, S_, false, T_, L_>))
#define KK_DD_GO3(P_, S_, T_) (a.lin ? KK_DD_GO4(P_, S_, T_, true) : KK_DD_GO4(P_, S_, T_, false))
#define KK_DD_GO(P_, S_) (train_blocks ? KK_DD_GO3(P_, S_, true) : KK_DD_GO3(P_, S_, false))
            if (with_p) {
                if (sq == 2) KK_DD_GO(true, 2);
                else if (sq == 4) KK_DD_GO(true, 4);
                else if (sq == 8) KK_DD_GO(true, 8);
                else KK_DD_GO(true, 0);
            } else {
                if (sq == 2) KK_DD_GO(false, 2);
                else if (sq == 4) KK_DD_GO(false, 4);
                else if (sq == 8) KK_DD_GO(false, 8);
                else KK_DD_GO(false, 0);
            }
#undef KK_DD_GO
#undef KK_DD_GO3
#undef KK_DD_GO4
            return check_launch("ddlms_block_kernel");
        };
        if (ext_list) return launch(false, b0, b1, 0, ext_list, ctr + 3);   // device-built list (cascades)
        const int64_t t1 = std::min(b1, ntb);
        const int64_t d0 = std::max(b0, ntb);
        // the speculative P pass's blocks holding training symbols (one CTA,
        // a sequential chain of ~170 us) run on a side stream next to the
        // main launch instead of before it (not while a graph is captured)
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        const bool fork = KK_DD_TRAIN_FORK && with_p && b0 < t1 && d0 < b1 &&
                          cudaStreamIsCapturing(s, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusNone;
        if (fork) {
            cudaStream_t side = train_side_stream();
            cudaEvent_t e0 = nullptr, e1 = nullptr;
            if (!side || cudaEventCreateWithFlags(&e0, cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&e1, cudaEventDisableTiming) != cudaSuccess)
                return set_cuda_error("train fork events");
            const cudaStream_t main_s = s;
            int rc = KK_OK;
            if (cudaEventRecord(e0, main_s) != cudaSuccess || cudaStreamWaitEvent(side, e0, 0) != cudaSuccess)
                rc = set_cuda_error("train fork");
            if (rc == KK_OK) {
                s = side;
                rc = launch(true, b0, t1, 0, nullptr, nullptr);
                s = main_s;
            }
            if (rc == KK_OK) rc = launch(false, d0, b1, 0, nullptr, nullptr);
            if (rc == KK_OK && (cudaEventRecord(e1, side) != cudaSuccess ||
                                cudaStreamWaitEvent(main_s, e1, 0) != cudaSuccess))
                rc = set_cuda_error("train join");
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            return rc;
        }
        if (b0 < t1)
            if (int rc = launch(true, b0, t1, (use_skip && !with_p) ? 1 : 0, nullptr, nullptr)) return rc;
        if (d0 >= b1) return KK_OK;
        if (use_skip && !with_p) {
            // compact the blocks to re-run so that warps only carry live chains
            const unsigned g = static_cast<unsigned>((b1 - d0 + 127) / 128);
            ddlms_select_kernel<<<g, 128, 0, s>>>(lv[0].T, Tused, margin, maxx2, a.mu, d0, b1, tol,
                                                  ((write_out & 2) || ctl_d) ? Twritten : nullptr, list, ctr + 3,
                                                  ctl_d);
            if (int rc = check_launch("ddlms_select_kernel")) return rc;
            return launch(false, d0, b1, 0, list, ctr + 3);
        }
        return launch(false, d0, b1, 0, nullptr, nullptr);
    }
    int read_ctr(unsigned long long (&h)[4]) {
        return d2h_small(h, ctr, sizeof(h), s);
    }

    int init(const void* x, int64_t nsym, float scale_, const void* train, int64_t n_train, Slicer sl_, float mu,
             int block, float soft_tol_, void* workspace, size_t ws_bytes, cudaStream_t s_) {
        s = s_;
        sl = sl_;
        scale = scale_;
        soft_tol = soft_tol_;
        L = plan(nsym, block);
        if (ws_bytes < L.bytes) return set_error(KK_ERR_PARAM, "workspace too small");
        char* w = static_cast<char*>(workspace);
        ws_base = workspace;
        lv.resize(L.n.size());
        for (size_t l = 0; l < L.n.size(); ++l) {
            lv[l].n = L.n[l];
            lv[l].P = reinterpret_cast<float*>(w);
            lv[l].Q = lv[l].P + L.n[l] * 64;
            lv[l].T = lv[l].Q + L.n[l] * 16;
            w += align_up(L.n[l] * 96 * sizeof(float));
        }
        top = static_cast<int>(lv.size()) - 1;
        Tused = reinterpret_cast<float*>(w); w += align_up(L.nb * 16 * sizeof(float));
        Twritten = reinterpret_cast<float*>(w); w += align_up(L.nb * 16 * sizeof(float));
        margin = reinterpret_cast<float*>(w); w += align_up(L.nb * sizeof(float));
        maxx2 = reinterpret_cast<float*>(w); w += align_up(L.nb * sizeof(float));
        Tinit_d = reinterpret_cast<float*>(w); w += align_up(16 * sizeof(float));
        over = reinterpret_cast<int*>(w); w += align_up(L.nb * sizeof(int));
        hsh = reinterpret_cast<unsigned long long*>(w); w += align_up(L.nb * 8);
        ties = reinterpret_cast<uint2*>(w); w += align_up(L.nb * sizeof(uint2));
        grun = reinterpret_cast<int2*>(w); w += align_up(L.nb * sizeof(int2));
        ST_own = reinterpret_cast<float2*>(w); w += align_up(size_t(nsym) * 8);
        LT_own = reinterpret_cast<uint8_t*>(w); w += align_up(size_t(nsym));
        to.ST = ST_own;
        to.LT = LT_own;
        list = reinterpret_cast<int*>(w); w += align_up(L.nb * sizeof(int));
        rb = reinterpret_cast<ReadBack*>(w);
        ctr = rb->ctr;
        Tend = rb->Tend;
        // the block kernels work on the raw input with the scale folded into
        // the taps: T' = s T, mu' = mu s^2 (y = T' x_raw == T (s x_raw))
        a.x = static_cast<const float2*>(x);
        a.nsym = nsym;
        a.scale = 1.0f;
        a.train = static_cast<const float2*>(train);
        a.n_train = n_train;
        a.mu = mu * scale * scale;
        a.B = block;
        a.nb = L.nb;
        o.labels = nullptr;
        o.soft = nullptr;
        o.Q = lv[0].Q;
        o.Tused = Tused;
        o.Twritten = Twritten;
        o.margin = margin;
        o.Tend = Tend;
        o.over = over;
        o.hash = hsh;
        o.ties = ties;
        o.grun = grun;
        o.counters = ctr;
        o.first_changed = &rb->first_changed;
        bt = std::min<int64_t>(n_train / block, L.nb);
        ntb = std::min<int64_t>((n_train + block - 1) / block, L.nb);
        // over, hsh, ties and grun are contiguous in the workspace: one memset
        const size_t zero_bytes = reinterpret_cast<char*>(grun + L.nb) - reinterpret_cast<char*>(over);
        if (cudaMemsetAsync(over, 0, zero_bytes, s) != cudaSuccess ||
            cudaMemsetAsync(Twritten, 0xFF, L.nb * 16 * sizeof(float), s) != cudaSuccess)   // NaN: never written
            return set_cuda_error("solver init");
        rb_reset_kernel<<<1, 32, 0, s>>>(rb, kRbCtr01 | kRbCtr2 | kRbCtr3 | kRbFirst0 | kRbFirst1 | kRbCtl);
        return check_launch("rb_reset_kernel");
    }

    // the final pass writes straight into the caller's arrays when bound
    // (8-symbol runs are stored as 16 B soft / 8 B label words: alignment)
    void bind_outputs(uint8_t* labels, float2* soft) {
        const bool ok = labels && soft && (reinterpret_cast<uintptr_t>(labels) & 7) == 0 &&
                        (reinterpret_cast<uintptr_t>(soft) & 15) == 0;
        to.LT = ok ? labels : LT_own;
        to.ST = ok ? soft : ST_own;
    }

    // pure-training blocks from T_start; writes the exact training-end taps
    int train(const float* T_start, float* T_train_end) {
        if (int rc = set_start(T_start)) return rc;
        if (int rc = fill_T(0, L.nb, Tinit_d)) return rc;
        if (bt > 0) {
            if (int rc = run_blocks(true, 0, bt, 0)) return rc;
            if (bt < L.nb &&
                cudaMemsetAsync(lv[0].Q + bt * 16, 0, (L.nb - bt) * 16 * sizeof(float), s) != cudaSuccess)
                return set_cuda_error("Q init");
            if (int rc = scan_up(true)) return rc;
            if (int rc = scan_down()) return rc;
        }
        if (T_train_end && bt == 0) {   // no training blocks: the start taps themselves
            for (int i = 0; i < 16; ++i) T_train_end[i] = T_start[i];
        } else if (T_train_end) {
            float Tt[16];
            if (bt < L.nb) {
                if (int rc = d2h_small(Tt, lv[0].T + bt * 16, sizeof(Tt), s)) return rc;
                for (int i = 0; i < 16; ++i) T_train_end[i] = Tt[i] / scale;
            } else {
                // training covers the frame: its end taps
                if (int rc = d2h_small(Tt, Tend, sizeof(Tt), s)) return rc;
                for (int i = 0; i < 16; ++i) T_train_end[i] = Tt[i] / scale;
            }
        }
        return KK_OK;
    }

    // first pass of the decision-directed blocks from T_guess (+ P_b)
    int speculate(const float* T_guess, float* agg) {
        if (int rc = upload16(Tend, T_guess)) return rc;
        if (int rc = fill_T(bt, L.nb, Tend)) return rc;
        if (int rc = run_blocks(true, bt, L.nb, 0)) return rc;
        reruns += L.nb;
        speculated = true;
        if (int rc = scan_up(true)) return rc;
        return frame_map(agg);
    }

    // exact frame start taps -> re-run; returns changed blocks.  A
    // decision pass re-runs only blocks whose certified decision margin the
    // start-tap move could cross; a soft pass also refreshes every block
    // whose soft outputs would move by more than soft_tol.
    int iterate(const float* T_start, int64_t* changed, int64_t* rerun, float* agg, bool soft_pass) {
        if (!speculated) return set_error(KK_ERR_PARAM, "speculate() must precede iterate()");
        if (int rc = set_start(T_start)) return rc;
        if (int rc = scan_down()) return rc;
        rb_reset_kernel<<<1, 32, 0, s>>>(rb, kRbCtr01 | kRbCtr3 | kRbFirst0);
        if (int rc = check_launch("rb_reset_kernel")) return rc;
        // decision pass: compacted re-run of the blocks whose certified margin
        // the start move could cross, no outputs; output pass: also the blocks
        // whose outputs are missing or were written from a start more than
        // soft_tol away (the first output pass of a frame runs every block; a
        // later one, after a late decision change, only its wake)
        if (int rc = soft_pass ? run_blocks(false, 0, L.nb, 1, soft_tol, 3)
                               : run_blocks(false, 0, L.nb, 1, 3.0e38f, 0))
            return rc;
        // decision cascades: as in solve_loop (rb->ctl[0] stays "decision" here)
        for (int step = 0; iters >= KK_CASCADE_FROM && step < kCascadeW; ++step) {
            cascade_prep_kernel<<<1, 32, 0, s>>>(rb, lv[0].P, lv[0].Q, Tused, lv[0].T, list, L.nb, ntb, kCascadeW,
                                                 step, kCascadeMaxChanged, 0);
            if (int rc = check_launch("cascade_prep_kernel")) return rc;
            if (int rc = run_blocks(false, 0, kCascadeW, 0, soft_pass ? soft_tol : 3.0e38f, soft_pass ? 3 : 0, list))
                return rc;
        }
        unsigned long long h[4];
        if (int rc = read_ctr(h)) return rc;
        ++iters;
        reruns += static_cast<int64_t>(h[1]);
        last_changed = static_cast<int64_t>(h[0]);
        if (changed) *changed = last_changed;
        if (rerun) *rerun = static_cast<int64_t>(h[1]);
        if (int rc = scan_up(false)) return rc;
        return frame_map(agg);
    }

    // Up to max_iter fixpoint iterations from the exact frame start taps,
    // queued in batches with the pass mode kept on the device (see
    // ddlms_advance_kernel): one host readback per batch, not per pass.  On
    // convergence the guard count and end taps come back in the same read.
    int solve_loop(const float* T_start, int max_iter, int64_t* it_stats, bool* converged, int64_t* guard,
                   float* T_final, bool reset = true) {
        if (!speculated) return set_error(KK_ERR_PARAM, "speculate() must precede solve_loop()");
        if (T_start)
            if (int rc = set_start(T_start)) return rc;
        if (reset) {
            rb_reset_kernel<<<1, 32, 0, s>>>(rb, kRbCtr01 | kRbCtr2 | kRbCtr3 | kRbCtl | kRbFirst0 | kRbFirst1);
            if (int rc = check_launch("rb_reset_kernel")) return rc;
        }
        *converged = false;
        ReadBack h;
        int queued = 0;
        int batch = 4;   // the bench streams converge in 4 iterations
        ctl_d = rb->ctl;
        while (queued < max_iter) {
            const int n = std::min(batch, max_iter - queued);
            int rc = KK_OK;
            for (int i = 0; i < n && rc == KK_OK; ++i) {
                rc = scan_down();
                if (rc == KK_OK) rc = run_blocks(false, 0, L.nb, 1, soft_tol, 3);
                // cascade window steps from the fifth iteration on (frames that
                // converge in four, the QPSK/16-QAM norm, never queue them)
                for (int step = 0; rc == KK_OK && queued + i >= KK_CASCADE_FROM && step < kCascadeW; ++step) {
                    cascade_prep_kernel<<<1, 32, 0, s>>>(rb, lv[0].P, lv[0].Q, Tused, lv[0].T, list, L.nb, ntb,
                                                         kCascadeW, step, kCascadeMaxChanged, 0);
                    rc = check_launch("cascade_prep_kernel");
                    if (rc == KK_OK) rc = run_blocks(false, 0, kCascadeW, 0, soft_tol, 3, list);
                }
                if (rc == KK_OK && ctl_d && speculated_async) rc = guard_check();
                if (rc == KK_OK) rc = scan_up(false);
                if (rc == KK_OK) {
                    ddlms_advance_kernel<<<1, 1, 0, s>>>(rb, cudaGraphConditionalHandle{}, 0, 0);
                    rc = check_launch("ddlms_advance_kernel");
                }
            }
            if (rc == KK_OK) {
                const int64_t gblocks = std::min<int64_t>((L.nb + 127) / 128, 148 * 8);
                if (cudaMemsetAsync(ctr + 2, 0, sizeof(unsigned long long), s) != cudaSuccess) {
                    rc = set_cuda_error("ctr");
                } else {
                    sum_int_kernel<<<static_cast<unsigned>(gblocks), 128, 0, s>>>(over, L.nb, ctr + 2);
                    rc = check_launch("sum_int_kernel");
                }
            }
            if (rc == KK_OK) rc = d2h_small(&h, rb, sizeof(h), s);
            if (rc != KK_OK) {
                ctl_d = nullptr;
                return rc;
            }
            queued += n;
            batch = std::min(2 * batch, 32);   // long decision cascades (64-QAM): fewer readbacks
            if (h.ctl[0] == kModeDone) break;
        }
        ctl_d = nullptr;
        const int it = h.ctl[1];
        iters += it;
        for (int i = 0; i < std::min(it, kMaxStatIters); ++i) {
            reruns += static_cast<int64_t>(h.it_stats[2 * i + 1]);
            if (it_stats && i < 16) {
                it_stats[2 * i] = static_cast<int64_t>(h.it_stats[2 * i]);
                it_stats[2 * i + 1] = static_cast<int64_t>(h.it_stats[2 * i + 1]);
            }
        }
        if (it > 0 && it <= kMaxStatIters) last_changed = static_cast<int64_t>(h.it_stats[2 * (it - 1)]);
        *converged = h.ctl[0] == kModeDone;
        last_first_changed = h.last_first;
        if (*converged) {
            if (guard) *guard = static_cast<int64_t>(h.ctr[2]);
            if (T_final)
                for (int i = 0; i < 16; ++i) T_final[i] = h.Tend[i] / scale;
        }
        return KK_OK;
    }

    // ---- asynchronous solve (kk_ddlms_solve_async): everything enqueued,
    // nothing read back; the fixpoint loop is a CUDA-graph WHILE node whose
    // condition the iteration's advance kernel sets (no pre-queued idle
    // iterations, no host round trip per batch) ----
    cudaGraphExec_t loop_exec = nullptr;
    bool loop_exec_cached = false;   // owned by the process-wide cache below
    void* ws_base = nullptr;

    static cudaStream_t capture_stream() {
        static thread_local cudaStream_t cs = nullptr;
        if (!cs && cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) cs = nullptr;
        return cs;
    }

    // one fixpoint iteration, as in solve_loop (mode from rb->ctl[0])
    int one_iteration(cudaGraphConditionalHandle h, int max_iter) {
        if (int rc = scan_down()) return rc;
        if (int rc = run_blocks(false, 0, L.nb, 1, soft_tol, 3)) return rc;
        for (int step = 0; step < kCascadeW; ++step) {
            cascade_prep_kernel<<<1, 32, 0, s>>>(rb, lv[0].P, lv[0].Q, Tused, lv[0].T, list, L.nb, ntb, kCascadeW,
                                                 step, kCascadeMaxChanged, KK_CASCADE_FROM);
            if (int rc = check_launch("cascade_prep_kernel")) return rc;
            if (int rc = run_blocks(false, 0, kCascadeW, 0, soft_tol, 3, list)) return rc;
        }
        if (int rc = guard_check()) return rc;
        if (int rc = scan_up(false)) return rc;
        ddlms_advance_kernel<<<1, 1, 0, s>>>(rb, h, 1, max_iter);
        return check_launch("ddlms_advance_kernel");
    }

    // a divergence-guard freeze in the certified prefix ends the iteration
    // (both kernels return at once unless an exceedance has been seen)
    int guard_check() {
        guard_scan_kernel<<<148 * 4, 128, 0, s>>>(rb, grun, over, L.nb, a.B, a.nsym, a.guard_run, nullptr, 0);
        if (int rc = check_launch("guard_scan_kernel")) return rc;
        guard_decide_kernel<<<1, 1, 0, s>>>(rb);
        return check_launch("guard_decide_kernel");
    }

    // Instantiated loop graphs are cached by everything their kernels' launch
    // parameters depend on (a repeated frame of the same shape on the same
    // workspace -- every step of a device-resident stream -- reuses its
    // graph): instantiation costs ~0.4 ms of host time and allocates device
    // memory, which serialises concurrent streams.
    std::vector<uint64_t> loop_key(int max_iter) const {
        auto f2u = [](float v) { uint32_t u; std::memcpy(&u, &v, 4); return static_cast<uint64_t>(u); };
        std::vector<uint64_t> k = {
            reinterpret_cast<uint64_t>(a.x), static_cast<uint64_t>(a.nsym), reinterpret_cast<uint64_t>(a.train),
            static_cast<uint64_t>(a.n_train), f2u(a.mu), f2u(a.scale), static_cast<uint64_t>(a.B),
            static_cast<uint64_t>(a.nb), reinterpret_cast<uint64_t>(ws_base), reinterpret_cast<uint64_t>(to.LT),
            reinterpret_cast<uint64_t>(to.ST), f2u(soft_tol), static_cast<uint64_t>(max_iter),
            static_cast<uint64_t>(ntb), static_cast<uint64_t>(bt), static_cast<uint64_t>(a.guard_run), static_cast<uint64_t>(a.lin),
            static_cast<uint64_t>(sl.kind), static_cast<uint64_t>(sl.npts), static_cast<uint64_t>(sl.m),
            f2u(sl.norm), f2u(sl.thr), static_cast<uint64_t>(sl.sep), f2u(sl.lev_h)};
        for (int i = 0; i < 64; ++i) k.push_back(f2u(sl.pts[i].x) << 32 | f2u(sl.pts[i].y));
        for (int i = 0; i < 64; i += 8) {
            uint64_t g = 0;
            for (int j = 0; j < 8; ++j) g |= static_cast<uint64_t>(sl.grid[i + j]) << (8 * j);
            k.push_back(g);
        }
        int dev = -1;
        cudaGetDevice(&dev);
        k.push_back(static_cast<uint64_t>(dev));
        return k;
    }

    int build_loop(int max_iter) {
        static std::mutex mu;
        static std::vector<std::pair<std::vector<uint64_t>, cudaGraphExec_t>> cache;   // most recent last
        const std::vector<uint64_t> key = loop_key(max_iter);
        {
            std::lock_guard<std::mutex> lk(mu);
            for (size_t i = 0; i < cache.size(); ++i)
                if (cache[i].first == key) {
                    loop_exec = cache[i].second;
                    loop_exec_cached = true;
                    std::rotate(cache.begin() + i, cache.begin() + i + 1, cache.end());
                    return KK_OK;
                }
        }
        if (int rc = instantiate_loop(max_iter)) return rc;
        std::lock_guard<std::mutex> lk(mu);
        if (cache.size() >= 16) {
            cudaGraphExecDestroy(cache.front().second);   // an in-flight launch completes first
            cache.erase(cache.begin());
        }
        cache.emplace_back(key, loop_exec);
        loop_exec_cached = true;
        return KK_OK;
    }

    int instantiate_loop(int max_iter) {
        cudaGraph_t g = nullptr;
        if (cudaGraphCreate(&g, 0) != cudaSuccess) return set_cuda_error("graph create");
        struct GraphGuard {
            cudaGraph_t g;
            ~GraphGuard() { if (g) cudaGraphDestroy(g); }
        } gg{g};
        cudaGraphConditionalHandle h;
        if (cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) != cudaSuccess)
            return set_cuda_error("graph conditional handle");
        cudaGraphNodeParams np = {};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = h;
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        cudaGraphNode_t node;
        if (cudaGraphAddNode(&node, g, nullptr, 0, &np) != cudaSuccess) return set_cuda_error("graph while node");
        cudaGraph_t body = np.conditional.phGraph_out[0];
        cudaStream_t cs = capture_stream();
        if (!cs) return set_cuda_error("capture stream");
        const cudaStream_t s_run = s;
        if (cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) != cudaSuccess)
            return set_cuda_error("begin capture");
        s = cs;
        // the body holds kLoopUnroll iterations: each trip of a graph WHILE
        // loop costs ~70 us of device-side scheduling (measured), each idle
        // unrolled iteration ~30 kernels that return at once (~1 us each)
        int rc = KK_OK;
        for (int u = 0; u < kLoopUnroll && rc == KK_OK; ++u) rc = one_iteration(h, max_iter);
        s = s_run;
        cudaGraph_t captured = nullptr;
        const cudaError_t ec = cudaStreamEndCapture(cs, &captured);
        if (rc) return rc;
        if (ec != cudaSuccess) return set_cuda_error("end capture");
        if (cudaGraphInstantiate(&loop_exec, g, 0) != cudaSuccess) {
            loop_exec = nullptr;
            return set_cuda_error("graph instantiate");
        }
        return KK_OK;
    }

    int solve_async(float* T_io, int* state_io, int max_iter, int guard_run, float mu_raw, int64_t* stats_out,
                    uint8_t* labels, float2* soft, bool use_graph, bool widely_linear) {
        a.guard_run = guard_run;
        a.lin = widely_linear ? 0 : 1;
        ctl_d = rb->ctl;
        rb_reset_kernel<<<1, 32, 0, s>>>(rb, kRbAll);
        if (int rc = check_launch("rb_reset_kernel")) return rc;
        frame_begin_kernel<<<1, 32, 0, s>>>(T_io, scale, Tinit_d, state_io, rb);
        if (int rc = check_launch("frame_begin_kernel")) return rc;
        // pure training blocks (exact from the frame start), then the first
        // pass of the decision-directed blocks from the training-end taps
        if (int rc = fill_T(0, L.nb, Tinit_d)) return rc;
        if (bt > 0) {
            if (int rc = run_blocks(true, 0, bt, 0)) return rc;
            if (bt < L.nb &&
                cudaMemsetAsync(lv[0].Q + bt * 16, 0, (L.nb - bt) * 16 * sizeof(float), s) != cudaSuccess)
                return set_cuda_error("Q init");
            if (int rc = scan_up(true)) return rc;
            if (int rc = scan_down()) return rc;
        }
        if (bt < L.nb) {
            copy16_kernel<<<1, 32, 0, s>>>(Tend, bt > 0 ? lv[0].T + bt * 16 : Tinit_d);
            if (int rc = check_launch("copy16_kernel")) return rc;
            if (int rc = fill_T(bt, L.nb, Tend)) return rc;
            if (int rc = run_blocks(true, bt, L.nb, 0)) return rc;
        }
        if (int rc = scan_up(true)) return rc;
        speculated = true;
        speculated_async = true;
        rb_reset_kernel<<<1, 32, 0, s>>>(rb, kRbCtr01 | kRbCtr2 | kRbCtr3 | kRbFirst0);
        if (int rc = check_launch("rb_reset_kernel")) return rc;
        if (!use_graph) {
            // host-driven batches with readbacks (blocks the calling thread):
            // for frames solved by a worker thread while other streams work --
            // instantiating a graph allocates device memory, which serialises
            // the other streams (measured: e2e 6.3 -> 4.3 GBaud)
            bool conv = false;
            if (int rc = solve_loop(nullptr, max_iter, nullptr, &conv, nullptr, nullptr, false)) return rc;
            ctl_d = rb->ctl;
        } else {
            static const bool trace = [] {
                const char* e = std::getenv("KK_DDLMS_TRACE");
                return e && e[0] == '1';
            }();
            const auto t0 = std::chrono::steady_clock::now();
            if (int rc = build_loop(max_iter)) return rc;
            const auto t1 = std::chrono::steady_clock::now();
            if (cudaGraphLaunch(loop_exec, s) != cudaSuccess) return set_cuda_error("graph launch");
            if (trace)
                std::fprintf(stderr, "[kk_ddlms_solve_async] nsym %lld: loop graph build %.3f ms, launch %.3f ms\n",
                             static_cast<long long>(a.nsym),
                             std::chrono::duration<double, std::milli>(t1 - t0).count(),
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count());
        }
        // epilogue: guard sum, fallback decision and the fallback paths (each
        // kernel returns at once unless its mode was chosen)
        const int64_t gblocks = std::min<int64_t>((L.nb + 127) / 128, 148 * 8);
        if (cudaMemsetAsync(ctr + 2, 0, sizeof(unsigned long long), s) != cudaSuccess)
            return set_cuda_error("ctr");
        sum_int_kernel<<<static_cast<unsigned>(gblocks), 128, 0, s>>>(over, L.nb, ctr + 2);
        if (int rc = check_launch("sum_int_kernel")) return rc;
        // guard exceedances in a converged frame: the first freeze, if any
        guard_scan_kernel<<<148 * 4, 128, 0, s>>>(rb, grun, over, L.nb, a.B, a.nsym, a.guard_run, state_io, 1);
        if (int rc = check_launch("guard_scan_kernel")) return rc;
        guard_decide_kernel<<<1, 1, 0, s>>>(rb);
        if (int rc = check_launch("guard_decide_kernel")) return rc;
        frame_end_kernel<<<1, 1, 0, s>>>(rb);
        if (int rc = check_launch("frame_end_kernel")) return rc;
        // modes 2 (not converged) / 4 (freeze): output pass of [0, m); mode 2: chain from m
        {
            const int* save = ctl_d;
            ctl_d = &rb->ctl[2];   // kModeOutput in mode 2, kModeDone otherwise
            fallback_list_kernel<<<static_cast<unsigned>(std::min<int64_t>((L.nb + 255) / 256, 1024)), 256, 0, s>>>(
                rb, list, L.nb, a.B);
            int rc = check_launch("fallback_list_kernel");
            if (rc == KK_OK) rc = scan_down();
            if (rc == KK_OK) rc = run_blocks(false, 0, L.nb, 0, soft_tol, 3, list);
            ctl_d = save;
            if (rc) return rc;
            o.labels = to.LT;
            o.soft = to.ST;
            ddlms_run_kernel<<<1, 1, 0, s>>>(a, sl, lv[0].T, maxx2, o, 0, L.nb, 0, soft_tol, 1, 1, rb);
            if (int rc2 = check_launch("ddlms_run_kernel chain")) return rc2;
            if (cudaMemsetAsync(ctr + 2, 0, sizeof(unsigned long long), s) != cudaSuccess)
                return set_cuda_error("ctr");
            sum_int_kernel<<<static_cast<unsigned>(gblocks), 128, 0, s>>>(over, L.nb, ctr + 2);
            if (int rc2 = check_launch("sum_int_kernel")) return rc2;
            frame_end2_kernel<<<1, 1, 0, s>>>(rb);
            if (int rc2 = check_launch("frame_end2_kernel")) return rc2;
        }
        // mode 1: the exact sequential chain over the frame
        seq_fallback_kernel<<<1, 1, 0, s>>>(a.x, a.nsym, scale, a.train, a.n_train, Tinit_d, T_io, state_io, sl,
                                            mu_raw, guard_run, a.lin ? 0 : 1, to.LT, to.ST, rb);
        if (int rc = check_launch("seq_fallback_kernel")) return rc;
        // mode 4: the freezing block's chain; modes 3 / 4: frozen-tap map
        freeze_chain_kernel<<<1, 1, 0, s>>>(a, sl, lv[0].T, rb, to.LT, to.ST);
        if (int rc = check_launch("freeze_chain_kernel")) return rc;
        frozen_map_kernel<<<static_cast<unsigned>(std::min<int64_t>((a.nsym + 255) / 256, 148 * 16)), 256, 0, s>>>(
            a, sl, rb, to.LT, to.ST);
        if (int rc = check_launch("frozen_map_kernel")) return rc;
        frame_final_kernel<<<1, 32, 0, s>>>(rb, 1.0f / scale, T_io, state_io);
        if (int rc = check_launch("frame_final_kernel")) return rc;
        if (stats_out) {
            frame_stats_kernel<<<1, 32, 0, s>>>(rb, L.nb, L.nb, stats_out);
            if (int rc = check_launch("frame_stats_kernel")) return rc;
        }
        ctl_d = nullptr;
        return copy_outputs(labels, soft);
    }

    ~DdlmsSolver() {
        if (loop_exec && !loop_exec_cached) cudaGraphExecDestroy(loop_exec);   // freed after an in-flight launch
    }

    int copy_outputs(uint8_t* labels, float2* soft) {
        if (labels && labels != to.LT &&
            cudaMemcpyAsync(labels, to.LT, size_t(a.nsym), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            return set_cuda_error("labels copy");
        if (soft && soft != to.ST &&
            cudaMemcpyAsync(soft, to.ST, size_t(a.nsym) * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            return set_cuda_error("soft copy");
        return KK_OK;
    }

    // chained exact fallback from block 0 (start taps already in lv[0].T[0])
    // Non-converged frame: blocks before the lowest block m whose decisions
    // changed in the last iteration ran from exact start taps with exact
    // decisions (induction from the exact frame start: none of them changed,
    // so the scan reproduces their starts).  They get an output pass from
    // those starts; the sequential chain covers [m, nb) only.
    int chain(uint8_t* labels, float2* soft, int64_t m = 0) {
        m = std::max<int64_t>(0, std::min<int64_t>(m, L.nb));
        o.labels = labels;
        o.soft = soft;
        if (int rc = scan_down()) return rc;
        if (m > 0) {
            if (int rc = run_blocks(false, 0, m, 1, soft_tol, 3)) return rc;
            const size_t n0 = static_cast<size_t>(std::min<int64_t>(m * a.B, a.nsym));
            if (labels && labels != to.LT &&
                cudaMemcpyAsync(labels, to.LT, n0, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
                return set_cuda_error("labels copy");
            if (soft && soft != to.ST &&
                cudaMemcpyAsync(soft, to.ST, n0 * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
                return set_cuda_error("soft copy");
        }
        if (m >= L.nb) return KK_OK;
        ddlms_run_kernel<<<1, 1, 0, s>>>(a, sl, lv[0].T, maxx2, o, m, L.nb, 0, soft_tol, 1, 1);
        return check_launch("ddlms_run_kernel chain");
    }

    int finish(uint8_t* labels, float2* soft, float* T_final, int64_t* guard) {
        if (int rc = copy_outputs(labels, soft)) return rc;
        return end_state(T_final, guard);
    }
    int end_state(float* T_final, int64_t* guard) {
        if (cudaMemsetAsync(ctr + 2, 0, sizeof(unsigned long long), s) != cudaSuccess) return set_cuda_error("ctr");
        const int64_t gblocks = std::min<int64_t>((L.nb + 127) / 128, 148 * 8);
        sum_int_kernel<<<static_cast<unsigned>(gblocks), 128, 0, s>>>(over, L.nb, ctr + 2);
        if (int rc = check_launch("sum_int_kernel")) return rc;
        unsigned long long h[4];
        if (int rc = read_ctr(h)) return rc;
        if (guard) *guard = static_cast<int64_t>(h[2]);
        if (T_final) {
            float Tt[16];
            if (int rc = d2h_small(Tt, Tend, sizeof(Tt), s)) return rc;
            for (int i = 0; i < 16; ++i) T_final[i] = Tt[i] / scale;
        }
        return KK_OK;
    }
};

int make_solver(DdlmsSolver& sv, const void* x, int64_t nsym, float scale, const void* train, int64_t n_train,
                int order, const float* pts_host, const uint8_t* grid_host, int grid_m, float norm, float max_radius,
                float guard_factor, float mu, int block, float soft_tol, void* workspace, size_t ws_bytes,
                cudaStream_t s) {
    if (nsym <= 0) return set_error(KK_ERR_PARAM, "nsym must be positive");
    if (block <= 0) return set_error(KK_ERR_PARAM, "block must be positive");
    if (order < 2 || order > 64) return set_error(KK_ERR_PARAM, "constellation order must be <= 64");
    if (!(scale > 0.0f)) return set_error(KK_ERR_PARAM, "scale must be positive");
    Slicer sl = make_slicer(order, pts_host, grid_host, grid_m, norm, max_radius, guard_factor);
    return sv.init(x, nsym, scale, train, n_train, sl, mu, block, soft_tol, workspace, ws_bytes, s);
}
}  // namespace

extern "C" void* kk_ddlms_create(const void* x, int64_t nsym, float scale, const void* train, int64_t n_train,
                                 int order, const float* pts_host, const uint8_t* grid_host, int grid_m, float norm,
                                 float max_radius, float guard_factor, float mu, int block, float soft_tol,
                                 void* workspace, size_t ws_bytes, void* stream) {
    clear_error();
    auto* sv = new DdlmsSolver();
    if (make_solver(*sv, x, nsym, scale, train, n_train, order, pts_host, grid_host, grid_m, norm, max_radius,
                    guard_factor, mu, block, soft_tol, workspace, ws_bytes, static_cast<cudaStream_t>(stream))) {
        delete sv;
        return nullptr;
    }
    return sv;
}

extern "C" int kk_ddlms_train(void* h, const float* T_start_host, float* T_train_end_host) {
    clear_error();
    if (!h) return set_error(KK_ERR_PARAM, "null solver");
    return static_cast<DdlmsSolver*>(h)->train(T_start_host, T_train_end_host);
}

extern "C" int kk_ddlms_speculate(void* h, const float* T_guess_host, float* map_host) {
    clear_error();
    if (!h) return set_error(KK_ERR_PARAM, "null solver");
    return static_cast<DdlmsSolver*>(h)->speculate(T_guess_host, map_host);
}

extern "C" int kk_ddlms_iterate(void* h, const float* T_start_host, int soft_pass, int64_t* changed, int64_t* rerun,
                                float* map_host) {
    clear_error();
    if (!h) return set_error(KK_ERR_PARAM, "null solver");
    return static_cast<DdlmsSolver*>(h)->iterate(T_start_host, changed, rerun, map_host, soft_pass != 0);
}

extern "C" int kk_ddlms_finish(void* h, uint8_t* labels, void* soft, float* T_final_host, int64_t* guard) {
    clear_error();
    if (!h) return set_error(KK_ERR_PARAM, "null solver");
    return static_cast<DdlmsSolver*>(h)->finish(labels, static_cast<float2*>(soft), T_final_host, guard);
}

extern "C" int kk_ddlms_bind_outputs(void* h, uint8_t* labels, void* soft) {
    clear_error();
    if (!h) return set_error(KK_ERR_PARAM, "null solver");
    static_cast<DdlmsSolver*>(h)->bind_outputs(labels, static_cast<float2*>(soft));
    return KK_OK;
}

extern "C" void kk_ddlms_destroy(void* h) { delete static_cast<DdlmsSolver*>(h); }

// Single-frame exact solve (T_init = exact frame start taps).  stats (host
// int64[38]): iterations, blocks re-run, fallback (0 none, 1 guard exceeded
// -> caller re-runs sequentially, 2 not converged -> chained), guard
// exceedances, changed blocks in the last iteration, blocks, then
// per-iteration (changed blocks, re-run blocks) for iterations 1..16.
extern "C" int kk_ddlms_solve(const void* x, int64_t nsym, float scale, const void* train, int64_t n_train,
                              const float* T_init, int order, const float* pts_host, const uint8_t* grid_host,
                              int grid_m, float norm, float max_radius, float guard_factor, int guard_run,
                              float mu, int block, int max_iter, float soft_tol, uint8_t* labels, void* soft,
                              float* T_final, void* workspace, size_t ws_bytes, int64_t* stats, void* stream) {
    clear_error();
    (void)guard_run;
    if (nsym <= 0) return KK_OK;
    // KK_DDLMS_TRACE=1: per-phase device times of each solve on stderr
    static const bool trace = [] {
        const char* e = std::getenv("KK_DDLMS_TRACE");
        return e && e[0] == '1';
    }();
    cudaEvent_t ev[5] = {};
    double host_ms[5] = {};
    const auto h0 = std::chrono::steady_clock::now();
    auto mark = [&](int i) {
        if (trace) {
            if (!ev[i]) cudaEventCreate(&ev[i]);
            cudaEventRecord(ev[i], static_cast<cudaStream_t>(stream));
            host_ms[i] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
        }
    };
    mark(0);
    DdlmsSolver sv;
    if (int rc = make_solver(sv, x, nsym, scale, train, n_train, order, pts_host, grid_host, grid_m, norm,
                             max_radius, guard_factor, mu, block, soft_tol, workspace, ws_bytes,
                             static_cast<cudaStream_t>(stream)))
        return rc;
    sv.bind_outputs(labels, static_cast<float2*>(soft));
    float Tg[16];
    if (int rc = sv.train(T_init, Tg)) return rc;
    mark(1);
    if (int rc = sv.speculate(sv.bt > 0 ? Tg : T_init, nullptr)) return rc;
    mark(2);
    int64_t st[6] = {0, 0, 0, 0, 0, sv.L.nb};
    bool converged = false;
    int64_t guard = 0;
    // decision passes until nothing changes, then one output pass (device-driven)
    if (int rc = sv.solve_loop(T_init, max_iter, stats ? stats + 6 : nullptr, &converged, &guard, T_final))
        return rc;
    mark(3);
    if (trace) {
        cudaEventSynchronize(ev[3]);
        float t[3];
        for (int i = 0; i < 3; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
        std::fprintf(stderr,
                     "[kk_ddlms_solve] nsym %lld B %d: device init+train %.3f ms, speculate %.3f ms, loop %.3f ms; "
                     "host marks %.3f %.3f %.3f %.3f ms\n",
                     static_cast<long long>(nsym), block, t[0], t[1], t[2], host_ms[0], host_ms[1], host_ms[2],
                     host_ms[3]);
        for (cudaEvent_t e : ev)
            if (e) cudaEventDestroy(e);
    }
    if (converged) {
        if (int rc = sv.copy_outputs(labels, static_cast<float2*>(soft))) return rc;
    } else {
        st[2] = 2;
        if (int rc = sv.chain(labels, static_cast<float2*>(soft), sv.last_first_changed)) return rc;
        if (int rc = sv.end_state(T_final, &guard)) return rc;
    }
    st[0] = sv.iters;
    st[1] = sv.reruns;
    st[3] = guard;
    st[4] = sv.last_changed;
    if (guard > 0 && st[2] == 0) st[2] = 1;   // guard exceedances: caller must re-run exactly
    if (stats)
        for (int i = 0; i < 6; ++i) stats[i] = st[i];
    return KK_OK;
}

// Asynchronous single-frame exact solve: enqueued on `stream`, nothing read
// back.  T_io (device float[16], unscaled real 2x8 form) holds the frame's
// start taps and receives its end taps; state_io (device int[2] = {frozen,
// div_count}) likewise; stats_out (device or mapped host int64[38], may be
// NULL) receives the statistics of kk_ddlms_solve.  Guard exceedances, a
// non-clear state at the frame start and non-convergence fall back to exact
// chains on the device.  The workspace must stay valid until the stream
// reaches the end of the enqueued work.
extern "C" int kk_ddlms_solve_async(const void* x, int64_t nsym, float scale, const void* train, int64_t n_train,
                                    float* T_io, int* state_io, int order, const float* pts_host,
                                    const uint8_t* grid_host, int grid_m, float norm, float max_radius,
                                    float guard_factor, int guard_run, float mu, int widely_linear, int block,
                                    int max_iter, float soft_tol, uint8_t* labels, void* soft, void* workspace,
                                    size_t ws_bytes, int64_t* stats_out, void* stream) {
    clear_error();
    if (nsym <= 0) return KK_OK;
    if (!T_io) return set_error(KK_ERR_PARAM, "T_io missing");
    if (max_iter == 0) return set_error(KK_ERR_PARAM, "max_iter must be nonzero");
    DdlmsSolver sv;
    if (int rc = make_solver(sv, x, nsym, scale, train, n_train, order, pts_host, grid_host, grid_m, norm,
                             max_radius, guard_factor, mu, block, soft_tol, workspace, ws_bytes,
                             static_cast<cudaStream_t>(stream)))
        return rc;
    sv.bind_outputs(labels, static_cast<float2*>(soft));
    const bool use_graph = max_iter > 0;
    return sv.solve_async(T_io, state_io, max_iter > 0 ? max_iter : -max_iter, guard_run, mu, stats_out, labels,
                          static_cast<float2*>(soft), use_graph, widely_linear != 0);
}

// enqueue the sync kernels; the 4 result doubles land in `res` (device or
// UVA-mapped pinned host memory)
// sync scratch (doubles): [mag: n_lags rounded to 32 | result: 32 | the
// tiled correlation's per-segment partials: n_seg * n_lags double2]
static inline int64_t sync_part_offset(int64_t n_lags) { return ((n_lags + 31) / 32) * 32 + 32; }
static inline size_t sync_scratch_bytes(int64_t n_lags, int n_ref) {
    const int64_t n_seg = n_ref > 0 ? (n_ref + kXcChunk - 1) / kXcChunk : 0;
    return static_cast<size_t>(sync_part_offset(n_lags) + 2 * n_seg * n_lags) * sizeof(double) + 256;
}

static int symbol_sync_launch(const void* head, int64_t n_head, const void* ref, int n_ref, int64_t skip,
                              double* res_out, void* scratch, size_t scratch_bytes, cudaStream_t s) {
    const int64_t l0 = (n_head + 1) / 2, l1 = n_head / 2;
    const int64_t nl0 = (ref && n_ref > 0 && l0 >= n_ref) ? l0 - n_ref + 1 : 0;
    const int64_t nl1 = (ref && n_ref > 0 && l1 >= n_ref) ? l1 - n_ref + 1 : 0;
    const size_t need = sync_scratch_bytes(nl0 + nl1, n_ref);
    if (scratch_bytes < need) return set_error(KK_ERR_PARAM, "sync scratch too small");
    double* mag = static_cast<double*>(scratch);
    if (nl0 + nl1 > 0) {
#ifndef KK_XCORR_TILED
#define KK_XCORR_TILED 1
#endif
        if (KK_XCORR_TILED) {
            const int n_seg = (n_ref + kXcChunk - 1) / kXcChunk;
            double2* part = reinterpret_cast<double2*>(mag + sync_part_offset(nl0 + nl1));
            const dim3 grid(static_cast<unsigned>((std::max(nl0, nl1) + kXcTile - 1) / kXcTile), 2,
                            static_cast<unsigned>(n_seg));
            xcorr_tiled_kernel<<<grid, kXcThreads, 0, s>>>(static_cast<const float2*>(head), n_head,
                                                           static_cast<const float2*>(ref), n_ref, nl0, nl1, part);
            if (int rc = check_launch("xcorr_tiled_kernel")) return rc;
            const int64_t nl = nl0 + nl1;
            xcorr_combine_kernel<<<static_cast<unsigned>(std::min<int64_t>((nl + 255) / 256, 1184)), 256, 0, s>>>(
                part, n_seg, nl, mag);
            if (int rc = check_launch("xcorr_combine_kernel")) return rc;
        } else {
            const int th = 256;
            const size_t sm = static_cast<size_t>(n_ref) * sizeof(float2);
            if (sm > 48 * 1024 &&
                cudaFuncSetAttribute(xcorr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(sm)) != cudaSuccess)
                return set_cuda_error("xcorr smem");
            xcorr_kernel<<<static_cast<unsigned>((nl0 + nl1 + th - 1) / th), th, sm, s>>>(
                static_cast<const float2*>(head), n_head, static_cast<const float2*>(ref), n_ref, nl0, nl1, mag);
            if (int rc = check_launch("xcorr_kernel")) return rc;
        }
    }
    sync_reduce_kernel<<<1, 1024, 0, s>>>(mag, nl0, nl1, static_cast<const float2*>(head), n_head, skip, res_out);
    return check_launch("sync_reduce_kernel");
}

extern "C" int kk_symbol_sync_enqueue(const void* head, int64_t n_head, const void* ref, int n_ref, int64_t skip,
                                      double* result, void* scratch, size_t scratch_bytes, void* stream) {
    clear_error();
    if (!result) return set_error(KK_ERR_PARAM, "result pointer missing");
    return symbol_sync_launch(head, n_head, ref, n_ref, skip, result, scratch, scratch_bytes,
                              static_cast<cudaStream_t>(stream));
}

extern "C" int kk_symbol_sync(const void* head, int64_t n_head, const void* ref, int n_ref, int64_t skip,
                              double* result, void* scratch, size_t scratch_bytes, void* stream) {
    clear_error();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t l0 = (n_head + 1) / 2, l1 = n_head / 2;
    const int64_t nl0 = (ref && n_ref > 0 && l0 >= n_ref) ? l0 - n_ref + 1 : 0;
    const int64_t nl1 = (ref && n_ref > 0 && l1 >= n_ref) ? l1 - n_ref + 1 : 0;
    double* res = static_cast<double*>(scratch) + ((nl0 + nl1 + 31) / 32) * 32;
    if (int rc = symbol_sync_launch(head, n_head, ref, n_ref, skip, res, scratch, scratch_bytes, s)) return rc;
    return d2h_small(result, res, 4 * sizeof(double), s);
}

extern "C" size_t kk_symbol_sync_scratch_bytes(int64_t n_head, int n_ref) {
    const int64_t l0 = (n_head + 1) / 2, l1 = n_head / 2;
    const int64_t nl0 = (n_ref > 0 && l0 >= n_ref) ? l0 - n_ref + 1 : 0;
    const int64_t nl1 = (n_ref > 0 && l1 >= n_ref) ? l1 - n_ref + 1 : 0;
    return sync_scratch_bytes(nl0 + nl1, n_ref);
}

extern "C" int kk_bit_errors(const uint8_t* labels, const uint8_t* ref_idx, int64_t n, const uint8_t* point_label,
                             int64_t win_syms, unsigned long long* total, unsigned int* win, int64_t ex_period,
                             int64_t ex_len, int64_t ex_phase, unsigned long long* n_counted, void* stream) {
    clear_error();
    if (n <= 0) return KK_OK;
    const int th = 256;
    int64_t blocks = (n + th - 1) / th;
    if (blocks > 148 * 16) blocks = 148 * 16;
    bit_errors_kernel<<<static_cast<unsigned>(blocks), th, 0, static_cast<cudaStream_t>(stream)>>>(
        labels, ref_idx, n, point_label, win_syms > 0 ? win_syms : 1, total, win_syms > 0 ? win : nullptr,
        ex_period, ex_len, ex_phase, n_counted);
    return check_launch("bit_errors_kernel");
}

extern "C" int kk_demap(const void* symbols, int64_t n, int order, const float* pts_host, uint8_t* idx,
                        unsigned long long* n_fallback, void* stream) {
    clear_error();
    if (order < 2 || order > 64) return set_error(KK_ERR_PARAM, "constellation order must be <= 64");
    if (n <= 0) return KK_OK;
    Slicer sl = make_slicer(order, pts_host, nullptr, 0, 1.0f, 1.0f, 1.0f);
    const int th = 256;
    int64_t blocks = (n + th - 1) / th;
    if (blocks > 148 * 16) blocks = 148 * 16;
    demap_kernel<<<static_cast<unsigned>(blocks), th, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const float2*>(symbols), n, sl, idx, n_fallback);
    return check_launch("demap_kernel");
}

// ---------------------------------------------------------------------------
// Decided labels -> demapped bit stream, packed MSB first (the receiver's
// output: rxdsp.py demap :548-567 bit order, np.packbits layout).  Label 255
// (training symbol) takes the training symbol's point index train_idx[k].
// One thread per output byte; bit b belongs to symbol b / k, bit k-1-(b % k).
// ---------------------------------------------------------------------------
namespace kk {
struct PointLabels {
    uint8_t v[64];
};
// One thread per group of 8 symbols: 8 k bits = exactly k output bytes (no
// per-byte divisions; the label table is read from the parameter bank).
__global__ void pack_bits_kernel(const uint8_t* __restrict__ lab, int64_t n, int64_t sym0,
                                 const uint8_t* __restrict__ train_idx, int64_t n_train,
                                 const __grid_constant__ PointLabels pl, int k, uint8_t* __restrict__ out,
                                 int64_t nbytes) {
    const int64_t ngroups = (n + 7) / 8;
    for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < ngroups;
         g += int64_t(gridDim.x) * blockDim.x) {
        unsigned long long bits = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t s = 8 * g + j;
            unsigned w = 0;
            if (s < n) {
                int li = lab[s];
                if (li == 255) li = (sym0 + s < n_train && train_idx) ? train_idx[sym0 + s] : 0;
                w = pl.v[li & 63];
            }
            bits = (bits << k) | w;
        }
        for (int b = 0; b < k; ++b) {
            const int64_t o = g * k + b;
            if (o < nbytes) out[o] = static_cast<uint8_t>(bits >> (8 * (k - 1 - b)));
        }
    }
}
}  // namespace kk

extern "C" int kk_pack_bits(const uint8_t* labels, int64_t n, int64_t sym0, const uint8_t* train_idx,
                            int64_t n_train, int bits_per_symbol, const uint8_t* point_label_host, int order,
                            uint8_t* out, void* stream) {
    using namespace kk;
    clear_error();
    if (bits_per_symbol < 1 || bits_per_symbol > 6 || order > 64 || order < 2)
        return set_error(KK_ERR_PARAM, "bits_per_symbol must be in [1, 6], order in [2, 64]");
    if (n <= 0) return KK_OK;
    PointLabels pl{};
    for (int i = 0; i < order; ++i) pl.v[i] = point_label_host[i];
    const int64_t nbytes = (n * bits_per_symbol + 7) / 8;
    const int th = 256;
    int64_t blocks = ((n + 7) / 8 + th - 1) / th;
#ifndef KK_PACK_CTAS
#define KK_PACK_CTAS (148 * 32)
#endif
    if (blocks > KK_PACK_CTAS) blocks = KK_PACK_CTAS;
    pack_bits_kernel<<<static_cast<unsigned>(blocks), th, 0, static_cast<cudaStream_t>(stream)>>>(
        labels, n, sym0, train_idx, n_train, pl, bits_per_symbol, out, nbytes);
    return check_launch("pack_bits_kernel");
}
