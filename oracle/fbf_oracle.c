/*
 * fbf_oracle.c -- TEST INFRASTRUCTURE ONLY (see fbf_oracle.h).
 *
 * fp64 restatement of the reference path.  Each function cites the reference
 * lines it restates and keeps the reference's evaluation order (ascending tap
 * index, ascending harmonic, row pass before column pass, left-to-right
 * products), so that with -ffp-contract=off the results are bit-identical to
 * the reference library compiled with the same flags.
 *
 * Row-range evaluation: an output row depends on the source rows within +-W
 * (after mirroring), and every per-pixel operation is position independent,
 * so computing rows [row0, row1) from just those source rows reproduces the
 * whole-image result bit for bit.  That is what makes the oracle usable on
 * strips of the 8192^2 config and lets it run multi-threaded.
 */
#include "fbf_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* image.hpp:34-40: half-sample symmetric reflection, period 2n. */
int fbo_mirror_index(int i, int n) {
    if (i >= 0 && i < n) return i;
    int period = 2 * n;
    int j = i % period;
    if (j < 0) j += period;
    return j < n ? j : period - 1 - j;
}

/* spatial.hpp:36-52 */
int fbo_spatial_gaussian(double sigma_s, double* profile, int* radius, double* w0) {
    if (!(sigma_s > 0.0)) return -1;
    int W = (int)ceil(3.0 * sigma_s);
    *radius = W;
    if (!profile) return 0;
    double total = 0.0;
    for (int j = -W; j <= W; ++j) {
        double e = exp(-((double)j * j) / (2.0 * sigma_s * sigma_s));
        profile[j + W] = e;
        total += e;
    }
    for (int k = 0; k < 2 * W + 1; ++k) profile[k] /= total;
    if (w0) *w0 = profile[W] * profile[W];
    return 0;
}

/* spatial.hpp:55-65 */
int fbo_spatial_box(int radius, double* profile, double* w0) {
    if (radius < 1) return -1;
    double tap = 1.0 / (2.0 * radius + 1.0);
    if (profile)
        for (int k = 0; k < 2 * radius + 1; ++k) profile[k] = tap;
    if (w0) *w0 = tap * tap;
    return 0;
}

/* kernels.hpp:79-96 */
double fbo_range_eval(int family, double sigma_r, double t) {
    double a = fabs(t);
    if (family == FBO_RANGE_EXPONENTIAL) return exp(-a / sigma_r);
    return exp(-(a * a) / (2.0 * sigma_r * sigma_r));
}

/* ------------------------------------------------------------------------ */
/* Least-squares cosine fit: kernel_approx.hpp:51-149 (QrState), :152-157,   */
/* :169-219 (progressive_fit).                                               */

typedef struct {
    int m;       /* grid rows T+1 */
    int k;       /* columns so far */
    int cap;
    double* b;   /* samples            [m]       */
    double* A;   /* raw columns        [cap][m]  */
    double* Qm;  /* orthonormal cols   [cap][m]  */
    double* R;   /* column j holds R[j][0..j]    */
    double* p;   /* projections Q^T b  [cap]     */
} qr_t;

static double dotv(const double* x, const double* y, int m) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += x[i] * y[i];
    return s;
}

static double normv(const double* x, int m) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += x[i] * x[i];
    return sqrt(s);
}

static void qr_init(qr_t* q, const double* samples, int m, int cap) {
    q->m = m;
    q->cap = cap;
    q->b = (double*)malloc(sizeof(double) * m);
    q->A = (double*)malloc(sizeof(double) * m * cap);
    q->Qm = (double*)malloc(sizeof(double) * m * cap);
    q->R = (double*)calloc((size_t)cap * cap, sizeof(double));
    q->p = (double*)malloc(sizeof(double) * cap);
    memcpy(q->b, samples, sizeof(double) * m);
    double nrm = sqrt((double)m);
    for (int t = 0; t < m; ++t) {
        q->A[t] = 1.0;
        q->Qm[t] = 1.0 / nrm;
    }
    q->p[0] = dotv(q->Qm, q->b, m);
    q->R[0] = nrm;
    q->k = 1;
}

static void qr_free(qr_t* q) {
    free(q->b); free(q->A); free(q->Qm); free(q->R); free(q->p);
}

/* Two-pass modified Gram-Schmidt; rejects when ||v|| < 1e-12 ||a||. */
static int qr_append(qr_t* q, const double* a) {
    int m = q->m, k = q->k;
    double* v = (double*)malloc(sizeof(double) * m);
    double* r = (double*)calloc((size_t)k + 1, sizeof(double));
    memcpy(v, a, sizeof(double) * m);
    for (int pass = 0; pass < 2; ++pass)
        for (int j = 0; j < k; ++j) {
            const double* qj = q->Qm + (size_t)j * m;
            double s = dotv(v, qj, m);
            for (int t = 0; t < m; ++t) v[t] += -s * qj[t];
            r[j] += s;
        }
    double rn = normv(v, m);
    if (rn < 1e-12 * normv(a, m)) { free(v); free(r); return 0; }
    for (int t = 0; t < m; ++t) v[t] /= rn;
    r[k] = rn;
    memcpy(q->A + (size_t)k * m, a, sizeof(double) * m);
    memcpy(q->Qm + (size_t)k * m, v, sizeof(double) * m);
    for (int i = 0; i <= k; ++i) q->R[(size_t)k * q->cap + i] = r[i];
    q->p[k] = dotv(v, q->b, m);
    q->k = k + 1;
    free(v); free(r);
    return 1;
}

static void qr_solve(const qr_t* q, double* d) {
    for (int i = q->k - 1; i >= 0; --i) {
        double s = q->p[i];
        for (int j = i + 1; j < q->k; ++j) s -= q->R[(size_t)j * q->cap + i] * d[j];
        d[i] = s / q->R[(size_t)i * q->cap + i];
    }
}

static double qr_residual(const qr_t* q, const double* d, double* max_abs) {
    double ss = 0.0, mx = 0.0;
    for (int t = 0; t < q->m; ++t) {
        double r = q->b[t];
        for (int j = 0; j < q->k; ++j) r -= q->A[(size_t)j * q->m + t] * d[j];
        ss += r * r;
        if (fabs(r) > mx) mx = fabs(r);
    }
    *max_abs = mx;
    return sqrt(ss);
}

static double* sample_range(int family, double sigma_r, int T) {
    double* b = (double*)malloc(sizeof(double) * (T + 1));
    for (int t = 0; t <= T; ++t) b[t] = fbo_range_eval(family, sigma_r, t);
    return b;
}

static void cosine_column(double* col, int n, double omega, int T) {
    for (int t = 0; t <= T; ++t) col[t] = cos(n * omega * t);
}

int fbo_fit_fixed(int family, double sigma_r, int T, int N, double* d, double* residual_norm,
                  double* max_pointwise_error) {
    if (T < 1 || N < 0 || N > T) return -1;
    const double pi = 3.14159265358979323846;
    double omega = pi / T;
    double* b = sample_range(family, sigma_r, T);
    double* col = (double*)malloc(sizeof(double) * (T + 1));
    qr_t q;
    qr_init(&q, b, T + 1, N + 1);
    int ok = 1;
    for (int n = 1; n <= N && ok; ++n) {
        cosine_column(col, n, omega, T);
        ok = qr_append(&q, col);
    }
    if (ok) {
        qr_solve(&q, d);
        double mx;
        double rn = qr_residual(&q, d, &mx);
        if (residual_norm) *residual_norm = rn;
        if (max_pointwise_error) *max_pointwise_error = mx;
    }
    qr_free(&q);
    free(col);
    free(b);
    return ok ? 0 : -1;
}

int fbo_progressive_fit(int family, double sigma_r, int T, double epsilon, double* d, int* N_out,
                        double* residual_norm, double* max_pointwise_error) {
    if (T < 1) return -1;
    if (!(epsilon > 0.0) || !(epsilon < sqrt((double)T + 1.0))) return -1;
    const double pi = 3.14159265358979323846;
    double omega = pi / T;
    double* b = sample_range(family, sigma_r, T);
    double* col = (double*)malloc(sizeof(double) * (T + 1));
    qr_t q;
    qr_init(&q, b, T + 1, T + 1);
    int N = 0, rc = 0;
    double mx;
    qr_solve(&q, d);
    double E = qr_residual(&q, d, &mx);
    while (E > epsilon) {
        if (N == T) { rc = -1; break; }
        int n = N + 1;
        cosine_column(col, n, omega, T);
        if (!qr_append(&q, col)) { rc = -1; break; }
        N = n;
        qr_solve(&q, d);
        E = qr_residual(&q, d, &mx);
    }
    *N_out = N;
    if (residual_norm) *residual_norm = E;
    if (max_pointwise_error) *max_pointwise_error = mx;
    qr_free(&q);
    free(col);
    free(b);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Separable direct convolution: spatial.hpp:74-112.                         */

/* One 1-D pass over a line of length n read with stride `in_stride`:
 * out[i] = sum_{j=-W..W} p[j+W] * line[mirror(i - j)], ascending j. */
static void fir_line(const double* line, long in_stride, int n, const double* p, int W,
                     double* pad, double* out, long out_stride) {
    for (int i = 0; i < n + 2 * W; ++i) pad[i] = line[(long)fbo_mirror_index(i - W, n) * in_stride];
    for (int i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int j = -W; j <= W; ++j) acc += p[j + W] * pad[i - j + W];
        out[(long)i * out_stride] = acc;
    }
}

void fbo_convolve(const double* in, double* out, int w, int h, const double* p, int W) {
    double* tmp = (double*)malloc(sizeof(double) * (size_t)w * h);
    int L = (w > h ? w : h) + 2 * W;
    double* pad = (double*)malloc(sizeof(double) * L);
    for (int y = 0; y < h; ++y) fir_line(in + (size_t)y * w, 1, w, p, W, pad, tmp + (size_t)y * w, 1);
    for (int x = 0; x < w; ++x) fir_line(tmp + x, w, h, p, W, pad, out + x, w);
    free(pad);
    free(tmp);
}

/* ------------------------------------------------------------------------ */
/* Fast shiftable filter: bilateral.hpp:109-160, rows [row0,row1).           */

typedef struct {
    const double* img; int w, h; const double* p; int W;
    const double* d; int N; double omega;
    int row0, row1;
    double* P; double* Q;   /* (row1-row0)*w, caller zeroed */
    int n_lo, n_hi;         /* harmonic range [n_lo, n_hi) */
} fast_job;

/* source rows needed by output rows [row0,row1): [lo, hi) */
static void needed_rows(int row0, int row1, int h, int W, int* lo, int* hi) {
    int a = h, b = -1;
    for (int y = row0; y < row1; ++y)
        for (int k = -W; k <= W; ++k) {
            int s = fbo_mirror_index(y + k, h);
            if (s < a) a = s;
            if (s > b) b = s;
        }
    *lo = a;
    *hi = b + 1;
}

static void* fast_worker(void* arg) {
    fast_job* J = (fast_job*)arg;
    const int w = J->w, h = J->h, W = J->W;
    int lo, hi;
    needed_rows(J->row0, J->row1, h, W, &lo, &hi);
    const int ns = hi - lo;
    size_t sz = (size_t)ns * w;
    /* modulated planes g = (cos, sin, f cos, f sin) on source rows, then row-passed */
    double* mod[4];
    double* rp[4];
    for (int k = 0; k < 4; ++k) {
        mod[k] = (double*)malloc(sizeof(double) * sz);
        rp[k] = (double*)malloc(sizeof(double) * sz);
    }
    int L = (w > h ? w : h) + 2 * W;
    double* pad = (double*)malloc(sizeof(double) * L);
    double conv[4];

    for (int n = J->n_lo; n < J->n_hi; ++n) {
        const double freq = J->omega * n;
        for (size_t i = 0; i < sz; ++i) {
            double f = J->img[(size_t)lo * w + i];
            double ph = freq * f;
            double c = cos(ph), s = sin(ph);
            mod[0][i] = c;
            mod[1][i] = s;
            mod[2][i] = c * f;
            mod[3][i] = s * f;
        }
        for (int k = 0; k < 4; ++k)
            for (int r = 0; r < ns; ++r)
                fir_line(mod[k] + (size_t)r * w, 1, w, J->p, W, pad, rp[k] + (size_t)r * w, 1);
        for (int y = J->row0; y < J->row1; ++y) {
            const size_t oi = (size_t)(y - J->row0) * w;
            for (int x = 0; x < w; ++x) {
                for (int k = 0; k < 4; ++k) {
                    /* column pass at (x, y), ascending j (transpose + convolve_rows) */
                    double acc = 0.0;
                    for (int j = -W; j <= W; ++j)
                        acc += J->p[j + W] * rp[k][(size_t)(fbo_mirror_index(y - j, h) - lo) * w + x];
                    conv[k] = acc;
                }
                double f = J->img[(size_t)y * w + x];
                double ph = freq * f;
                double c = cos(ph), s = sin(ph);
                const double dn = J->d[n];
                /* order as in bilateral.hpp:138-144: P uses (fcos_s, fsin_s), Q (cos_s, sin_s) */
                J->P[oi + x] += dn * (c * conv[2] + s * conv[3]);
                J->Q[oi + x] += dn * (c * conv[0] + s * conv[1]);
            }
        }
    }
    for (int k = 0; k < 4; ++k) { free(mod[k]); free(rp[k]); }
    free(pad);
    return NULL;
}

/* The numerator/denominator sums of bilateral.hpp:125-145 restricted to the
 * harmonics [n_lo, n_hi) (the decomposition the multi-GPU harmonic split
 * distributes): P and Q are (row1-row0)*w, overwritten. */
void fbo_partial_sums(const double* img, int w, int h, const double* p, int W, const double* d, int N,
                      double omega, int n_lo, int n_hi, int row0, int row1, double* P, double* Q) {
    const int no = row1 - row0;
    memset(P, 0, sizeof(double) * (size_t)no * w);
    memset(Q, 0, sizeof(double) * (size_t)no * w);
    fast_job J = {img, w, h, p, W, d, N, omega, row0, row1, P, Q, n_lo, n_hi};
    fast_worker(&J);
}

int fbo_bilateral_fast(const double* img, int w, int h, const double* p, int W, double w0,
                       const double* d, int N, double omega, double max_err, int check_eps,
                       int row0, int row1, int nthreads, double* out, long long* bad_index) {
    if (w <= 0 || h <= 0 || row0 < 0 || row1 > h || row0 >= row1) return 1;
    if (check_eps && !(max_err < w0)) return 1;
    const int no = row1 - row0;
    double* P = (double*)calloc((size_t)no * w, sizeof(double));
    double* Q = (double*)calloc((size_t)no * w, sizeof(double));
    if (nthreads < 1) nthreads = 1;
    if (nthreads > no) nthreads = no;
    fast_job* jobs = (fast_job*)malloc(sizeof(fast_job) * nthreads);
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
    for (int t = 0; t < nthreads; ++t) {
        int a = row0 + (int)((long)no * t / nthreads), b = row0 + (int)((long)no * (t + 1) / nthreads);
        fast_job J = {img, w, h, p, W, d, N, omega, a, b,
                      P + (size_t)(a - row0) * w, Q + (size_t)(a - row0) * w, 0, N + 1};
        jobs[t] = J;
        if (nthreads > 1) pthread_create(&th[t], NULL, fast_worker, &jobs[t]);
        else fast_worker(&jobs[t]);
    }
    if (nthreads > 1)
        for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    /* bilateral.hpp:147-158: first collapsed denominator in row-major order */
    const double q_floor = (w0 - max_err) / 2.0;
    int rc = 0;
    for (size_t i = 0; i < (size_t)no * w; ++i) {
        if (fabs(Q[i]) < q_floor) {
            if (bad_index) *bad_index = (long long)row0 * w + (long long)i;
            rc = 2;
            break;
        }
        out[i] = P[i] / Q[i];
    }
    free(P); free(Q); free(jobs); free(th);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Brute-force filter: bilateral.hpp:78-102.                                 */

typedef struct {
    const double* img; int w, h; const double* p; int W; int family; double sigma_r;
    int row0, row1; double* out;
} exact_job;

static void* exact_worker(void* arg) {
    exact_job* J = (exact_job*)arg;
    const int w = J->w, h = J->h, W = J->W;
    for (int y = J->row0; y < J->row1; ++y)
        for (int x = 0; x < w; ++x) {
            const double center = J->img[(size_t)y * w + x];
            double num = 0.0, den = 0.0;
            for (int dy = -W; dy <= W; ++dy) {
                const int sy = fbo_mirror_index(y - dy, h);
                for (int dx = -W; dx <= W; ++dx) {
                    const int sx = fbo_mirror_index(x - dx, w);
                    const double v = J->img[(size_t)sy * w + sx];
                    const double wgt =
                        (J->p[dx + W] * J->p[dy + W]) * fbo_range_eval(J->family, J->sigma_r, v - center);
                    num += wgt * v;
                    den += wgt;
                }
            }
            J->out[(size_t)y * w + x] = num / den;
        }
    return NULL;
}

void fbo_bilateral_exact(const double* img, int w, int h, const double* p, int W, int family,
                         double sigma_r, int row0, int row1, int nthreads, double* out) {
    const int no = row1 - row0;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > no) nthreads = no;
    exact_job* jobs = (exact_job*)malloc(sizeof(exact_job) * nthreads);
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
    double* base = out - (size_t)row0 * w; /* worker indexes by global row */
    for (int t = 0; t < nthreads; ++t) {
        int a = row0 + (int)((long)no * t / nthreads), b = row0 + (int)((long)no * (t + 1) / nthreads);
        exact_job J = {img, w, h, p, W, family, sigma_r, a, b, base};
        jobs[t] = J;
        if (nthreads > 1) pthread_create(&th[t], NULL, exact_worker, &jobs[t]);
        else exact_worker(&jobs[t]);
    }
    if (nthreads > 1)
        for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(jobs); free(th);
}

/* ------------------------------------------------------------------------ */
/* bilateral.hpp:21-74: ceil(max over pixels of windowed max - windowed min) */

int fbo_local_dynamic_range(const double* img, int w, int h, int W) {
    if (w <= 0 || h <= 0 || W < 1) return -1;
    size_t n = (size_t)w * h;
    double* hi = (double*)malloc(sizeof(double) * n);
    double* lo = (double*)malloc(sizeof(double) * n);
    double* hi2 = (double*)malloc(sizeof(double) * n);
    double* lo2 = (double*)malloc(sizeof(double) * n);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double a = -INFINITY, b = INFINITY;
            for (int k = -W; k <= W; ++k) {
                double v = img[(size_t)y * w + fbo_mirror_index(x + k, w)];
                if (v > a) a = v;
                if (v < b) b = v;
            }
            hi[(size_t)y * w + x] = a;
            lo[(size_t)y * w + x] = b;
        }
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double a = -INFINITY, b = INFINITY;
            for (int k = -W; k <= W; ++k) {
                size_t s = (size_t)fbo_mirror_index(y + k, h) * w + x;
                if (hi[s] > a) a = hi[s];
                if (lo[s] < b) b = lo[s];
            }
            hi2[(size_t)y * w + x] = a;
            lo2[(size_t)y * w + x] = b;
        }
    double spread = 0.0;
    for (size_t i = 0; i < n; ++i)
        if (hi2[i] - lo2[i] > spread) spread = hi2[i] - lo2[i];
    free(hi); free(lo); free(hi2); free(lo2);
    return (int)ceil(spread);
}

/* analysis.hpp:27-34 */
double fbo_error_bound(int T, double epsilon, double w0) {
    if (T < 0 || !(epsilon >= 0.0) || !(epsilon < w0)) return -1.0;
    return 2.0 * T * epsilon / (w0 - epsilon);
}
