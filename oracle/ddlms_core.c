/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Never linked into or called by the
 * product path (paper_2108_07001_b200/).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library.
 *
 * Plain-C float64 restatement of the reference's sequential widely-linear
 * decision-directed LMS recurrence, `_ddlms_core` in
 * /root/reference/pkg/src/kkmodem/rxdsp.py:460-499 (numba-jitted at
 * rxdsp.py:502-507), called from `ddlms_wl` rxdsp.py:510-545.
 *
 * Per output symbol k (rxdsp.py:465-498):
 *   y   = sum_i conj(w_i) x[2k+i] + conj(g_i) conj(x[2k+i])       (WL)
 *   d   = train[k] if k < n_train else nearest point, first minimum wins
 *   guard: |y| > factor*max_radius for `run` consecutive symbols -> frozen
 *   if !frozen && mu != 0:  w_i += mu conj(d-y) x_i ; g_i += mu conj(d-y) conj(x_i)
 *
 * Complex arithmetic is spelled out in real arithmetic with the same
 * association order as the complex128 operations of the reference, and the
 * file is compiled with -ffp-contract=off so no FMA contraction changes the
 * rounding.  abs() of a complex is hypot(), as in numpy/numba.
 */
#include <math.h>
#include <stdint.h>

typedef struct { double re, im; } cplx;

static inline cplx c_add(cplx a, cplx b) { cplx r = {a.re + b.re, a.im + b.im}; return r; }
static inline cplx c_sub(cplx a, cplx b) { cplx r = {a.re - b.re, a.im - b.im}; return r; }
static inline cplx c_conj(cplx a) { cplx r = {a.re, -a.im}; return r; }
static inline cplx c_mul(cplx a, cplx b) {
    cplx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
    return r;
}
static inline cplx c_scale(double s, cplx a) {
    /* python `float * complex` promotes s to complex(s, 0) */
    cplx sc = {s, 0.0};
    return c_mul(sc, a);
}
static inline double c_abs(cplx a) { return hypot(a.re, a.im); }

/*
 * x: n_in complex (interleaved re,im); w,g: n_taps complex, updated in place;
 * points: n_pts complex; train: n_train complex; soft/dec: n_out complex out.
 * state[0] = frozen (0/1), state[1] = div_count; updated in place.
 * Returns 0.
 */
int oracle_ddlms_core(const double *x, int64_t n_in, double *w, double *g, int n_taps,
                      const double *points, int n_pts, const double *train, int64_t n_train,
                      double mu, int widely_linear, double max_radius, double guard_factor,
                      int64_t guard_run, int64_t *state, double *soft, double *dec,
                      int64_t n_out)
{
    (void)n_in;
    const cplx *X = (const cplx *)x;
    cplx *W = (cplx *)w;
    cplx *G = (cplx *)g;
    const cplx *P = (const cplx *)points;
    const cplx *TR = (const cplx *)train;
    cplx *S = (cplx *)soft;
    cplx *D = (cplx *)dec;
    int frozen = (int)state[0];
    int64_t div_count = state[1];
    const double thr = guard_factor * max_radius;
    for (int64_t k = 0; k < n_out; ++k) {
        const int64_t base = 2 * k;
        cplx y = {0.0, 0.0};
        for (int i = 0; i < n_taps; ++i) {
            cplx xi = X[base + i];
            y = c_add(y, c_mul(c_conj(W[i]), xi));
            if (widely_linear) y = c_add(y, c_mul(c_conj(G[i]), c_conj(xi)));
        }
        cplx d;
        if (k < n_train) {
            d = TR[k];
        } else {
            int best = 0;
            double bd = c_abs(c_sub(y, P[0]));
            for (int p = 1; p < n_pts; ++p) {
                double dp = c_abs(c_sub(y, P[p]));
                if (dp < bd) { bd = dp; best = p; }
            }
            d = P[best];
        }
        if (c_abs(y) > thr) {
            div_count += 1;
            if (div_count >= guard_run) frozen = 1;
        } else {
            div_count = 0;
        }
        if (!frozen && mu != 0.0) {
            cplx ce = c_conj(c_sub(d, y));
            for (int i = 0; i < n_taps; ++i) {
                cplx xi = X[base + i];
                /* w[i] + mu*ce*xi : (mu*ce)*xi, python left-to-right */
                W[i] = c_add(W[i], c_mul(c_scale(mu, ce), xi));
                if (widely_linear) G[i] = c_add(G[i], c_mul(c_scale(mu, ce), c_conj(xi)));
            }
        }
        S[k] = y;
        D[k] = d;
    }
    state[0] = frozen;
    state[1] = div_count;
    return 0;
}
