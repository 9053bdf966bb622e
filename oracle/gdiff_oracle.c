/*
 * gdiff_oracle.c -- CPU restatement of the reference local-diffusion path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for bench.py; it is never linked into, loaded by, or
 * called from the product path (paper_2410_21634_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may use it.
 *
 * Every routine restates one function of the reference package
 * (/root/reference/pkg/src/graphdiff, cited as src/<file>:<line>) with the
 * same floating-point operation order so results are bit-identical:
 *   - no fused multiply-add (build with -ffp-contract=off; numba emits
 *     separate vmulsd/vaddsd),
 *   - numpy reductions (np.abs(v).sum()) use numpy's pairwise summation,
 *     restated in pw_sum() and pinned against numpy in tests/test_oracle.py.
 *
 * Parity is pinned against golden vectors produced by running the reference
 * itself (tests/golden/make_golden.py -> the .npz files in tests/golden).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* report container (library-owned arrays, freed by orc_report_free)        */
/* ------------------------------------------------------------------------ */

typedef struct {
    int32_t converged;
    int32_t diverged;
    int64_t sweeps;
    int64_t total_ops;
    double min_residual;
    int64_t support_size;
    int64_t n_logs;          /* entries in vol/gamma/sign/frontier_sizes */
    int64_t *vol_log;
    double *gamma_log;
    double *l1_log;          /* n_logs + 1 entries */
    int8_t *sign_log;
    int64_t *frontier_sizes;
    int64_t *trace;          /* concatenated frontiers (when recorded) */
    int64_t trace_len;
    double *l2_log;          /* global GD only: n_logs + 1 entries */
    int64_t cap, trace_cap;
} orc_report;

static void rep_init(orc_report *rep) {
    memset(rep, 0, sizeof(*rep));
    rep->converged = 1;
    rep->min_residual = INFINITY;
    rep->cap = 64;
    rep->vol_log = malloc(sizeof(int64_t) * rep->cap);
    rep->gamma_log = malloc(sizeof(double) * rep->cap);
    rep->l1_log = malloc(sizeof(double) * (rep->cap + 1));
    rep->l2_log = malloc(sizeof(double) * (rep->cap + 1));
    rep->sign_log = malloc(sizeof(int8_t) * rep->cap);
    rep->frontier_sizes = malloc(sizeof(int64_t) * rep->cap);
    rep->trace_cap = 0;
    rep->trace = NULL;
}

static void rep_grow(orc_report *rep) {
    if (rep->n_logs < rep->cap) return;
    rep->cap *= 2;
    rep->vol_log = realloc(rep->vol_log, sizeof(int64_t) * rep->cap);
    rep->gamma_log = realloc(rep->gamma_log, sizeof(double) * rep->cap);
    rep->l1_log = realloc(rep->l1_log, sizeof(double) * (rep->cap + 1));
    rep->l2_log = realloc(rep->l2_log, sizeof(double) * (rep->cap + 1));
    rep->sign_log = realloc(rep->sign_log, sizeof(int8_t) * rep->cap);
    rep->frontier_sizes = realloc(rep->frontier_sizes, sizeof(int64_t) * rep->cap);
}

static void rep_trace(orc_report *rep, const int64_t *f, int64_t cnt) {
    if (rep->trace_len + cnt > rep->trace_cap) {
        int64_t nc = rep->trace_cap ? rep->trace_cap : 256;
        while (nc < rep->trace_len + cnt) nc *= 2;
        rep->trace = realloc(rep->trace, sizeof(int64_t) * nc);
        rep->trace_cap = nc;
    }
    memcpy(rep->trace + rep->trace_len, f, sizeof(int64_t) * cnt);
    rep->trace_len += cnt;
}

void orc_report_free(orc_report *rep) {
    free(rep->vol_log);
    free(rep->gamma_log);
    free(rep->l1_log);
    free(rep->l2_log);
    free(rep->sign_log);
    free(rep->frontier_sizes);
    free(rep->trace);
    memset(rep, 0, sizeof(*rep));
}

int64_t orc_report_sizeof(void) { return (int64_t)sizeof(orc_report); }

/* ------------------------------------------------------------------------ */
/* numpy helpers                                                            */
/* ------------------------------------------------------------------------ */

/* numpy's pairwise summation (DOUBLE_pairwise_sum, PW_BLOCKSIZE 128) of
 * |a_i| (take_abs) or a_i: what float(np.abs(v).sum()) evaluates. */
static double pw_sum(const double *a, int64_t n, int take_abs) {
    if (n < 8) {
        double res = -0.0;
        for (int64_t i = 0; i < n; i++) res += take_abs ? fabs(a[i]) : a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int k = 0; k < 8; k++) r[k] = take_abs ? fabs(a[k]) : a[k];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; k++) r[k] += take_abs ? fabs(a[i + k]) : a[i + k];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += take_abs ? fabs(a[i]) : a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pw_sum(a, n2, take_abs) + pw_sum(a + n2, n - n2, take_abs);
    }
}

double orc_pairwise_sum(const double *a, int64_t n, int32_t take_abs) {
    return pw_sum(a, n, take_abs);
}

static double sumsq_pw(const double *a, int64_t n) {
    double *sq = malloc(sizeof(double) * (n ? n : 1));
    for (int64_t i = 0; i < n; i++) sq[i] = a[i] * a[i];
    double s = pw_sum(sq, n, 0);
    free(sq);
    return s;
}

/* src/local_solvers.py:353-361 */
static void l1_and_min(const double *r, int64_t n, double *l1, double *mn) {
    double s = 0.0, m = INFINITY;
    for (int64_t i = 0; i < n; i++) {
        s += fabs(r[i]);
        if (r[i] < m) m = r[i];
    }
    *l1 = s;
    *mn = m;
}

/* ------------------------------------------------------------------------ */
/* sweep-synchronous kernels: LocalGD / LocalCH                             */
/* ------------------------------------------------------------------------ */

/* src/local_solvers.py:267-292 (_apply_update_seq) */
static int64_t apply_update_seq(const int64_t *off, const int64_t *tgt, const double *w,
                                double *r, const int64_t *fr, int64_t fc, const double *vals,
                                uint8_t *cmark, int64_t *cand) {
    int64_t cc = 0;
    for (int64_t i = 0; i < fc; i++) {
        int64_t u = fr[i];
        r[u] -= vals[i];
        if (!cmark[u]) {
            cmark[u] = 1;
            cand[cc++] = u;
        }
    }
    for (int64_t i = 0; i < fc; i++) {
        int64_t u = fr[i];
        double val = vals[i];
        for (int64_t j = off[u]; j < off[u + 1]; j++) {
            int64_t v = tgt[j];
            r[v] += val * w[j];
            if (!cmark[v]) {
                cmark[v] = 1;
                cand[cc++] = v;
            }
        }
    }
    return cc;
}

/* src/local_solvers.py:336-350 (_filter_frontier) */
static int64_t filter_frontier(const double *r, const double *theta, const int64_t *cand,
                               int64_t cc, uint8_t *cmark, int64_t *out, int sgn) {
    int64_t fc = 0;
    for (int64_t i = 0; i < cc; i++) {
        int64_t u = cand[i];
        cmark[u] = 0;
        double ru = r[u];
        int act = sgn ? (fabs(ru) >= theta[u]) : (ru >= theta[u]);
        if (act) out[fc++] = u;
    }
    return fc;
}

typedef struct {
    int64_t n;
    const int64_t *off, *tgt;
    const double *w, *theta;
    double *x, *r;
    uint8_t *cmark;
    int64_t *cand, *fbuf, *front, fcount;
    int sgn;
} sweep_driver;

/* src/local_solvers.py:367-391 (_SweepDriver.__init__), x/r caller-owned */
static void drv_init(sweep_driver *d, int64_t n, const int64_t *off, const int64_t *tgt,
                     const double *w, const double *theta, const double *b, double *x,
                     double *r, int sgn, orc_report *rep) {
    d->n = n; d->off = off; d->tgt = tgt; d->w = w; d->theta = theta;
    d->x = x; d->r = r; d->sgn = sgn;
    memcpy(r, b, sizeof(double) * n);
    memset(x, 0, sizeof(double) * n);
    d->cmark = calloc(n ? n : 1, 1);
    d->cand = malloc(sizeof(int64_t) * (n ? n : 1));
    d->fbuf = malloc(sizeof(int64_t) * (n ? n : 1));
    d->front = malloc(sizeof(int64_t) * (n ? n : 1));
    int64_t ns = 0;
    for (int64_t i = 0; i < n; i++)   /* np.flatnonzero(sys.b) */
        if (b[i] != 0.0) d->cand[ns++] = i;
    d->fcount = filter_frontier(r, theta, d->cand, ns, d->cmark, d->fbuf, sgn);
    memcpy(d->front, d->fbuf, sizeof(int64_t) * d->fcount);
    double l1, mn;
    l1_and_min(r, n, &l1, &mn);
    rep->l1_log[0] = l1;
    rep->min_residual = mn;
}

static void drv_free(sweep_driver *d) {
    free(d->cmark); free(d->cand); free(d->fbuf); free(d->front);
}

/* src/local_solvers.py:393-415 (sequential branch) */
static void drv_apply(sweep_driver *d, const double *vals) {
    int64_t cc = apply_update_seq(d->off, d->tgt, d->w, d->r, d->front, d->fcount, vals,
                                  d->cmark, d->cand);
    d->fcount = filter_frontier(d->r, d->theta, d->cand, cc, d->cmark, d->fbuf, d->sgn);
    memcpy(d->front, d->fbuf, sizeof(int64_t) * d->fcount);
}

/* src/local_solvers.py:417-422 */
static void drv_log(sweep_driver *d, orc_report *rep, int64_t svol, double sgamma) {
    rep_grow(rep);
    int64_t t = rep->n_logs;
    double prev = rep->l1_log[t];
    rep->vol_log[t] = svol;
    rep->gamma_log[t] = prev > 0 ? sgamma / prev : 0.0;
    double l1, mn;
    l1_and_min(d->r, d->n, &l1, &mn);
    rep->l1_log[t + 1] = l1;
    if (mn < rep->min_residual) rep->min_residual = mn;
    rep->n_logs = t + 1;
}

static int64_t count_nonzero(const double *r, int64_t n) {
    int64_t c = 0;
    for (int64_t i = 0; i < n; i++) c += (r[i] != 0.0);
    return c;
}

/* src/local_solvers.py:428-470 (local_gd, parallel=False) */
int orc_local_gd(int64_t n, const int64_t *off, const int64_t *tgt, const double *w,
                 const double *theta, const double *b, double *x, double *r,
                 int64_t max_sweeps, int32_t record_trace, orc_report *rep) {
    rep_init(rep);
    sweep_driver d;
    drv_init(&d, n, off, tgt, w, theta, b, x, r, 0, rep);
    double *vals = malloc(sizeof(double) * (n ? n : 1));
    while (d.fcount) {
        if (rep->sweeps >= max_sweeps) { rep->converged = 0; break; }
        rep_grow(rep);
        rep->frontier_sizes[rep->n_logs] = d.fcount;
        if (record_trace) rep_trace(rep, d.front, d.fcount);
        int64_t svol = 0;
        for (int64_t i = 0; i < d.fcount; i++) {
            int64_t u = d.front[i];
            svol += off[u + 1] - off[u];
            vals[i] = r[u];
        }
        double sgamma = pw_sum(vals, d.fcount, 1);
        for (int64_t i = 0; i < d.fcount; i++) x[d.front[i]] += vals[i];
        drv_apply(&d, vals);
        drv_log(&d, rep, svol, sgamma);
        rep->total_ops += svol;
        rep->sweeps += 1;
    }
    rep->support_size = count_nonzero(r, n);
    free(vals);
    drv_free(&d);
    return 0;
}

/* Warm-started signed LocalGD: the reference
 * sweep loop (src/local_solvers.py:364-470: _SweepDriver, _apply_update_seq,
 * _filter_frontier with signed=True) started from a given pair (x = p,
 * r = s - Q p) instead of (0, b); S_0 = filter(flatnonzero(r)).  x and r
 * are read and updated in place. */
int orc_local_gd_warm(int64_t n, const int64_t *off, const int64_t *tgt, const double *w,
                      const double *theta, double *x, double *r, int32_t sgn,
                      int64_t max_sweeps, int32_t record_trace, orc_report *rep) {
    rep_init(rep);
    double *r0 = calloc(n ? n : 1, sizeof(double));
    double *x0 = calloc(n ? n : 1, sizeof(double));
    memcpy(r0, r, sizeof(double) * n);
    memcpy(x0, x, sizeof(double) * n);
    sweep_driver d;
    drv_init(&d, n, off, tgt, w, theta, r0, x, r, sgn, rep);
    memcpy(x, x0, sizeof(double) * n); /* drv_init zeroes x; warm start keeps p */
    double *vals = malloc(sizeof(double) * (n ? n : 1));
    while (d.fcount) {
        if (rep->sweeps >= max_sweeps) { rep->converged = 0; break; }
        rep_grow(rep);
        rep->frontier_sizes[rep->n_logs] = d.fcount;
        if (record_trace) rep_trace(rep, d.front, d.fcount);
        int64_t svol = 0;
        for (int64_t i = 0; i < d.fcount; i++) {
            int64_t u = d.front[i];
            svol += off[u + 1] - off[u];
            vals[i] = r[u];
        }
        double sgamma = pw_sum(vals, d.fcount, 1);
        for (int64_t i = 0; i < d.fcount; i++) x[d.front[i]] += vals[i];
        drv_apply(&d, vals);
        drv_log(&d, rep, svol, sgamma);
        rep->total_ops += svol;
        rep->sweeps += 1;
    }
    rep->support_size = count_nonzero(r, n);
    free(vals); free(r0); free(x0);
    drv_free(&d);
    return 0;
}

/* src/local_solvers.py:473-538 (local_ch); mu, L resolved by the caller via
 * the _cheby_bounds rule (src/local_solvers.py:541-558). */
static int local_momentum(int64_t n, const int64_t *off, const int64_t *tgt, const double *w,
                          const double *theta, const double *b, double *x, double *r, double mu,
                          double L, int64_t max_sweeps, int32_t record_trace, orc_report *rep,
                          int hb);

int orc_local_ch(int64_t n, const int64_t *off, const int64_t *tgt, const double *w,
                 const double *theta, const double *b, double *x, double *r, double mu,
                 double L, int64_t max_sweeps, int32_t record_trace, orc_report *rep) {
    return local_momentum(n, off, tgt, w, theta, b, x, r, mu, L, max_sweeps, record_trace, rep, 0);
}

/* LocalHB (heavy-ball momentum): NOT in the reference -- its momentum method
 * is local_ch.  Restated as local_ch (src/local_solvers.py:473-538) with
 * Polyak's stationary coefficients for eigenvalues in [mu, L] (the limit of
 * the Chebyshev recurrence): eta = 4/(sqrt(L)+sqrt(mu))^2, beta = ((sqrt(L)-
 * sqrt(mu))/(sqrt(L)+sqrt(mu)))^2; sweep 0 vals = eta r, then eta r + beta
 * prev.  Pinned to the reference's own _SweepDriver by tests/golden/hb.npz
 * (tests/golden/make_golden_hb.py). */
int orc_local_hb(int64_t n, const int64_t *off, const int64_t *tgt, const double *w,
                 const double *theta, const double *b, double *x, double *r, double mu,
                 double L, int64_t max_sweeps, int32_t record_trace, orc_report *rep) {
    return local_momentum(n, off, tgt, w, theta, b, x, r, mu, L, max_sweeps, record_trace, rep, 1);
}

static int local_momentum(int64_t n, const int64_t *off, const int64_t *tgt, const double *w,
                          const double *theta, const double *b, double *x, double *r, double mu,
                          double L, int64_t max_sweeps, int32_t record_trace, orc_report *rep,
                          int hb) {
    rep_init(rep);
    sweep_driver d;
    drv_init(&d, n, off, tgt, w, theta, b, x, r, 1, rep);
    double rho = (L - mu) / (L + mu);
    double step0 = 2.0 / (L + mu);
    double *mom = calloc(n ? n : 1, sizeof(double));
    int64_t *stamp = malloc(sizeof(int64_t) * (n ? n : 1));
    for (int64_t i = 0; i < n; i++) stamp[i] = -2;
    double b_l1 = pw_sum(b, n, 1);
    double *rvals = malloc(sizeof(double) * (n ? n : 1));
    double *vals = malloc(sizeof(double) * (n ? n : 1));
    double delta = rho;
    while (d.fcount) {
        if (rep->sweeps >= max_sweeps) { rep->converged = 0; break; }
        int64_t t = rep->sweeps;
        rep_grow(rep);
        rep->frontier_sizes[rep->n_logs] = d.fcount;
        if (record_trace) rep_trace(rep, d.front, d.fcount);
        int64_t svol = 0;
        for (int64_t i = 0; i < d.fcount; i++) {
            int64_t u = d.front[i];
            svol += off[u + 1] - off[u];
            rvals[i] = r[u];
        }
        double sgamma = pw_sum(rvals, d.fcount, 1);
        if (hb) {
            const double sq = sqrt(L), sm = sqrt(mu);
            const double eta = 4.0 / ((sq + sm) * (sq + sm));
            const double q = (sq - sm) / (sq + sm);
            const double beta = q * q;  /* (python ** 2 of a double: one product) */
            for (int64_t i = 0; i < d.fcount; i++) {
                int64_t u = d.front[i];
                if (t == 0) {
                    vals[i] = eta * rvals[i];
                } else {
                    double prev = (stamp[u] == t - 1) ? mom[u] : 0.0;
                    vals[i] = eta * rvals[i] + beta * prev;
                }
            }
        } else if (t == 0) {
            for (int64_t i = 0; i < d.fcount; i++) vals[i] = step0 * rvals[i];
        } else {
            double delta_next = 1.0 / (2.0 * (L + mu) / (L - mu) - delta);
            double coef_r = 4.0 * delta_next / (L - mu);
            double coef_m = delta * delta_next;
            for (int64_t i = 0; i < d.fcount; i++) {
                int64_t u = d.front[i];
                double prev = (stamp[u] == t - 1) ? mom[u] : 0.0;
                vals[i] = coef_r * rvals[i] + coef_m * prev;
            }
            delta = delta_next;
        }
        for (int64_t i = 0; i < d.fcount; i++) {
            int64_t u = d.front[i];
            x[u] += vals[i];
            mom[u] = vals[i];
            stamp[u] = t;
        }
        drv_apply(&d, vals);
        drv_log(&d, rep, svol, sgamma);
        rep->total_ops += svol;
        rep->sweeps += 1;
        if (rep->l1_log[rep->n_logs] > 10.0 * b_l1) {
            rep->converged = 0;
            rep->diverged = 1;
            break;
        }
    }
    rep->support_size = count_nonzero(r, n);
    free(mom); free(stamp); free(rvals); free(vals);
    drv_free(&d);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* FIFO push kernel: LocalGS / LocalSOR / dynamic repair                    */
/* ------------------------------------------------------------------------ */

/* src/local_solvers.py:48-188 (_push_kernel).  dim = len(theta). */
int orc_push_kernel(int64_t dim, const int64_t *off, const int64_t *tgt, const double *w,
                    const double *theta, double *x, double *r, const int64_t *seeds,
                    int64_t n_seeds, double omega, double x_gain, int32_t sgn,
                    int64_t max_sweeps, orc_report *rep) {
    rep_init(rep);
    const int64_t sent = dim, qcap = dim + 2;
    int64_t *queue = malloc(sizeof(int64_t) * qcap);
    uint8_t *qmark = calloc(dim ? dim : 1, 1);
    int64_t front = 0, rear = 0;
    for (int64_t i = 0; i < n_seeds; i++) {
        int64_t u = seeds[i];
        double ru = r[u];
        int act = sgn ? (fabs(ru) >= theta[u]) : (ru >= theta[u]);
        if (act && !qmark[u]) {
            queue[rear] = u;
            rear = (rear + 1) % qcap;
            qmark[u] = 1;
        }
    }
    double l1 = 0.0, min_r = INFINITY;
    for (int64_t i = 0; i < dim; i++) {
        l1 += fabs(r[i]);
        if (r[i] < min_r) min_r = r[i];
    }
    rep->l1_log[0] = l1;
    int64_t sweeps = 0, total_ops = 0;
    if (front == rear) goto done;
    queue[rear] = sent;
    rear = (rear + 1) % qcap;
    int64_t svol = 0;
    double sgamma = 0.0;
    int saw_pos = 0, saw_neg = 0;
    while (front != rear) {
        int64_t u = queue[front];
        front = (front + 1) % qcap;
        if (u == sent) {
            rep->n_logs = sweeps;
            rep_grow(rep);
            rep->vol_log[sweeps] = svol;
            rep->gamma_log[sweeps] = l1 > 0.0 ? sgamma / l1 : 0.0;
            rep->sign_log[sweeps] = (saw_pos && saw_neg) ? 2 : saw_pos ? 1 : saw_neg ? -1 : 0;
            total_ops += svol;
            sweeps += 1;
            l1 = 0.0;
            for (int64_t i = 0; i < dim; i++) {
                l1 += fabs(r[i]);
                if (r[i] < min_r) min_r = r[i];
            }
            rep->l1_log[sweeps] = l1;
            rep->n_logs = sweeps;
            if (front == rear) break;
            if (sweeps >= max_sweeps) { rep->converged = 0; break; }
            queue[rear] = sent;
            rear = (rear + 1) % qcap;
            svol = 0;
            sgamma = 0.0;
            saw_pos = saw_neg = 0;
            continue;
        }
        qmark[u] = 0;
        double ru = r[u];
        if (sgn ? (fabs(ru) < theta[u]) : (ru < theta[u])) continue;
        svol += off[u + 1] - off[u];
        sgamma += fabs(ru);
        if (ru > 0.0) saw_pos = 1;
        else if (ru < 0.0) saw_neg = 1;
        double res = omega * ru;
        x[u] += x_gain * res;
        r[u] = ru - res;
        for (int64_t j = off[u]; j < off[u + 1]; j++) {
            int64_t v = tgt[j];
            double rv = r[v] + res * w[j];
            r[v] = rv;
            if (!qmark[v]) {
                int act = sgn ? (fabs(rv) >= theta[v]) : (rv >= theta[v]);
                if (act) {
                    queue[rear] = v;
                    rear = (rear + 1) % qcap;
                    qmark[v] = 1;
                }
            }
        }
        if (!qmark[u]) {
            double ru2 = r[u];
            int act = sgn ? (fabs(ru2) >= theta[u]) : (ru2 >= theta[u]);
            if (act) {
                queue[rear] = u;
                rear = (rear + 1) % qcap;
                qmark[u] = 1;
            }
        }
    }
done:
    rep->sweeps = sweeps;
    rep->total_ops = total_ops;
    rep->min_residual = min_r;
    rep->support_size = count_nonzero(r, dim);
    free(queue);
    free(qmark);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* heat kernel: push on the stage-expanded system                           */
/* ------------------------------------------------------------------------ */

/* src/local_solvers.py:566-661 (_hk_push_kernel); v, r have (N+1)*n entries */
int orc_hk_push(int64_t n, int64_t n_stages, const int64_t *off, const int64_t *tgt,
                const double *base_w, const double *stage_w, const double *theta, double *v,
                double *r, int64_t seed, int64_t max_sweeps, orc_report *rep) {
    rep_init(rep);
    const int64_t dim = (n_stages + 1) * n, sent = dim, qcap = dim + 2;
    int64_t *queue = malloc(sizeof(int64_t) * qcap);
    uint8_t *qmark = calloc(dim ? dim : 1, 1);
    int64_t front = 0, rear = 0;
    if (r[seed] >= theta[seed]) {
        queue[rear++] = seed;
        qmark[seed] = 1;
    }
    double l1 = 0.0, min_r = INFINITY;
    for (int64_t i = 0; i < dim; i++) {
        l1 += fabs(r[i]);
        if (r[i] < min_r) min_r = r[i];
    }
    rep->l1_log[0] = l1;
    int64_t sweeps = 0, total_ops = 0;
    if (front == rear) goto done;
    queue[rear] = sent;
    rear = (rear + 1) % qcap;
    int64_t svol = 0;
    double sgamma = 0.0;
    while (front != rear) {
        int64_t idx = queue[front];
        front = (front + 1) % qcap;
        if (idx == sent) {
            rep->n_logs = sweeps;
            rep_grow(rep);
            rep->vol_log[sweeps] = svol;
            rep->gamma_log[sweeps] = l1 > 0.0 ? sgamma / l1 : 0.0;
            total_ops += svol;
            sweeps += 1;
            l1 = 0.0;
            for (int64_t i = 0; i < dim; i++) {
                l1 += fabs(r[i]);
                if (r[i] < min_r) min_r = r[i];
            }
            rep->l1_log[sweeps] = l1;
            rep->n_logs = sweeps;
            if (front == rear) break;
            if (sweeps >= max_sweeps) { rep->converged = 0; break; }
            queue[rear] = sent;
            rear = (rear + 1) % qcap;
            svol = 0;
            sgamma = 0.0;
            continue;
        }
        qmark[idx] = 0;
        double ri = r[idx];
        if (ri < theta[idx]) continue;
        int64_t k = idx / n, u = idx - k * n;
        svol += off[u + 1] - off[u];
        sgamma += fabs(ri);
        v[idx] += ri;
        r[idx] = 0.0;
        if (k < n_stages) {
            double wk = stage_w[k];
            int64_t base = k * n + n;
            for (int64_t j = off[u]; j < off[u + 1]; j++) {
                int64_t t = base + tgt[j];
                double rt = r[t] + ri * wk * base_w[j];
                r[t] = rt;
                if (!qmark[t] && rt >= theta[t]) {
                    queue[rear] = t;
                    rear = (rear + 1) % qcap;
                    qmark[t] = 1;
                }
            }
        }
    }
done:
    rep->sweeps = sweeps;
    rep->total_ops = total_ops;
    rep->min_residual = min_r;
    rep->support_size = count_nonzero(r, dim);
    free(queue);
    free(qmark);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* global gradient descent (reference point)                                */
/* ------------------------------------------------------------------------ */

/* src/global_solvers.py:41-47 */
static int any_active(const double *r, const double *theta, int64_t n, int sgn) {
    for (int64_t i = 0; i < n; i++) {
        double ri = sgn ? fabs(r[i]) : r[i];
        if (ri >= theta[i]) return 1;
    }
    return 0;
}

/* src/global_solvers.py:124-152 (gradient_descent) + _scatter_full :63-71.
 * l2_log uses sqrt(pairwise sum of squares) (np.linalg.norm goes through BLAS,
 * so l2 parity is by tolerance only). */
int orc_gradient_descent(int64_t n, const int64_t *off, const int64_t *tgt, const double *w,
                         const double *theta, const double *b, double *x, double *r,
                         int64_t max_sweeps, orc_report *rep) {
    rep_init(rep);
    memcpy(r, b, sizeof(double) * n);
    memset(x, 0, sizeof(double) * n);
    int64_t vol = off[n];
    rep->l1_log[0] = pw_sum(r, n, 1);
    rep->l2_log[0] = sqrt(sumsq_pw(r, n));
    double *nxt = malloc(sizeof(double) * (n ? n : 1));
    int conv = !any_active(r, theta, n, 0);
    while (!conv && rep->sweeps < max_sweeps) {
        for (int64_t i = 0; i < n; i++) x[i] += r[i];
        memset(nxt, 0, sizeof(double) * n);
        for (int64_t u = 0; u < n; u++) {
            double val = r[u];
            if (val == 0.0) continue;
            for (int64_t j = off[u]; j < off[u + 1]; j++) nxt[tgt[j]] += val * w[j];
        }
        memcpy(r, nxt, sizeof(double) * n);
        rep->n_logs = rep->sweeps;
        rep_grow(rep);
        rep->vol_log[rep->sweeps] = vol;
        rep->sweeps += 1;
        rep->total_ops += vol;
        rep->l1_log[rep->sweeps] = pw_sum(r, n, 1);
        rep->l2_log[rep->sweeps] = sqrt(sumsq_pw(r, n));
        rep->n_logs = rep->sweeps;
        conv = !any_active(r, theta, n, 0);
    }
    rep->converged = conv;
    free(nxt);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* per-seed parity of a GPU batch result against the reference x            */
/* ------------------------------------------------------------------------ */

/* The GPU batch returns x of seed i as (node, value) pairs:
 * nodes[off[i] .. off[i] + cnt[i]), caller ids.  Compared against the dense
 * reference x: l1 of the difference and of the reference (the l1 entry of
 * error_norms, src/metrics.py:157-171) and the top-k ranking. */
typedef struct {
    const int64_t *off, *cnt;
    const int32_t *nodes;
    const double *vals;
    double *l1d, *l1r;
    int32_t *topk; /* bit 0: top-k lists identical; bit 1: identical up to
                      swaps of entries whose reference values agree to 1e-12 */
    int32_t k;
} gpu_cmp;

typedef struct { int64_t node; double val; } kv;

static int kv_better(kv a, kv b) { return a.val > b.val || (a.val == b.val && a.node < b.node); }

/* min-heap of the k best: root = worst kept */
static void kv_sift(kv *h, int64_t n, int64_t i) {
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, w = i;
        if (l < n && kv_better(h[w], h[l])) w = l;
        if (r < n && kv_better(h[w], h[r])) w = r;
        if (w == i) return;
        kv t = h[i]; h[i] = h[w]; h[w] = t;
        i = w;
    }
}

static void kv_offer(kv *h, int64_t *n, int64_t k, kv c) {
    if (*n < k) {
        int64_t i = (*n)++;
        h[i] = c;
        while (i > 0) {  /* sift up: a parent must be worse than its children */
            int64_t p = (i - 1) / 2;
            if (!kv_better(h[p], h[i])) break;
            kv t = h[i]; h[i] = h[p]; h[p] = t;
            i = p;
        }
    } else if (k > 0 && kv_better(c, h[0])) {
        h[0] = c;
        kv_sift(h, *n, 0);
    }
}

static int kv_cmp_desc(const void *a, const void *b) {
    kv x = *(const kv *)a, y = *(const kv *)b;
    return kv_better(x, y) ? -1 : (kv_better(y, x) ? 1 : 0);
}

/* scratch: n zeroed doubles (left zeroed on return) */
static void cmp_seed(const gpu_cmp *C, int64_t i, const double *xr, int64_t n, double *scratch) {
    const int64_t a = C->off[i], c = C->cnt[i];
    for (int64_t j = 0; j < c; j++) scratch[C->nodes[a + j]] = C->vals[a + j];
    double d = 0.0, s = 0.0;
    for (int64_t u = 0; u < n; u++) {
        d += fabs(scratch[u] - xr[u]);
        s += fabs(xr[u]);
    }
    C->l1d[i] = d;
    C->l1r[i] = s;
    if (C->topk) {
        const int64_t k = C->k;
        kv *hr = malloc(sizeof(kv) * (k ? k : 1)), *hg = malloc(sizeof(kv) * (k ? k : 1));
        int64_t nr = 0, ng = 0;
        for (int64_t u = 0; u < n; u++)
            if (xr[u] != 0.0) kv_offer(hr, &nr, k, (kv){u, xr[u]});
        for (int64_t j = 0; j < c; j++)
            if (C->vals[a + j] != 0.0) kv_offer(hg, &ng, k, (kv){C->nodes[a + j], C->vals[a + j]});
        qsort(hr, nr, sizeof(kv), kv_cmp_desc);
        qsort(hg, ng, sizeof(kv), kv_cmp_desc);
        int strict = nr == ng, ties = nr == ng;
        for (int64_t j = 0; j < nr && j < ng; j++) {
            if (hr[j].node == hg[j].node) continue;
            strict = 0;
            const double va = xr[hr[j].node], vb = xr[hg[j].node];
            if (!(fabs(va - vb) <= 1e-12 * fabs(va))) ties = 0;
        }
        C->topk[i] = strict | (ties << 1);
        free(hr); free(hg);
    }
    for (int64_t j = 0; j < c; j++) scratch[C->nodes[a + j]] = 0.0;
}

/* ------------------------------------------------------------------------ */
/* batched CPU baseline: the reference's per-seed local_gd, many threads    */
/* ------------------------------------------------------------------------ */

typedef struct {
    int64_t n;
    const int64_t *off, *tgt;
    const double *w, *theta;
    double alpha;
    int32_t method;  /* 0 local_gd, 1 local_sor, 2 local_ch, 3 local_hb */
    double omega;
    double mu, L;    /* local_ch bounds */
    const int64_t *seeds;
    int64_t n_seeds, max_sweeps;
    int64_t *out_sweeps, *out_ops, *out_pushes;
    int32_t *out_conv;
    double *out_xsum;
    const gpu_cmp *cmp;  /* optional per-seed parity against a GPU result */
    int64_t next;
} batch_job;

/* One seed exactly as `local_gd(dataclasses.replace(sys, b=alpha*e_s))`
 * (src/local_solvers.py:428-470) or `local_sor(..., omega)` (:221-253) would
 * run it, including the per-solve O(n) allocations and per-sweep O(n) l1
 * scans of the reference.  The system's b is built once per thread and only
 * its spike moves from seed to seed: the reference CLI builds systems outside
 * its timed region (src/cli.py:152-156). */
static void *batch_worker(void *arg) {
    batch_job *J = arg;
    int64_t n = J->n;
    double *b = calloc(n ? n : 1, sizeof(double));
    double *scratch = J->cmp ? calloc(n ? n : 1, sizeof(double)) : NULL;
    for (;;) {
        int64_t i = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
        if (i >= J->n_seeds) break;
        double *x = malloc(sizeof(double) * (n ? n : 1));
        double *r = malloc(sizeof(double) * (n ? n : 1));
        b[J->seeds[i]] = J->alpha;
        orc_report rep;
        int64_t pushes = 0;
        if (J->method == 1) {
            /* local_sor (src/local_solvers.py:221-253): x = 0, r = b, seeds = [s] */
            memcpy(r, b, sizeof(double) * n);
            memset(x, 0, sizeof(double) * n);
            int64_t sd = J->seeds[i];
            orc_push_kernel(n, J->off, J->tgt, J->w, J->theta, x, r, &sd, 1, J->omega, 1.0,
                            J->omega > 1.0, J->max_sweeps, &rep);
            pushes = -1;
        } else if (J->method == 2 || J->method == 3) {
            /* local_ch (src/local_solvers.py:473-538) / its heavy-ball form on b = bval e_s */
            local_momentum(n, J->off, J->tgt, J->w, J->theta, b, x, r, J->mu, J->L, J->max_sweeps,
                           0, &rep, J->method == 3);
            pushes = 0;
            for (int64_t t = 0; t < rep.n_logs; t++) pushes += rep.frontier_sizes[t];
        } else {
            orc_local_gd(n, J->off, J->tgt, J->w, J->theta, b, x, r, J->max_sweeps, 0, &rep);
            for (int64_t t = 0; t < rep.n_logs; t++) pushes += rep.frontier_sizes[t];
        }
        b[J->seeds[i]] = 0.0;
        J->out_sweeps[i] = rep.sweeps;
        J->out_ops[i] = rep.total_ops;
        J->out_pushes[i] = pushes;
        J->out_conv[i] = rep.converged;
        if (J->out_xsum) J->out_xsum[i] = pw_sum(x, n, 0);
        if (J->cmp) cmp_seed(J->cmp, i, x, n, scratch);
        orc_report_free(&rep);
        free(x); free(r);
    }
    free(b);
    free(scratch);
    return NULL;
}

static void run_threads(void *(*fn)(void *), void *job, int32_t n_threads) {
    if (n_threads < 1) n_threads = 1;
    pthread_t *th = malloc(sizeof(pthread_t) * n_threads);
    for (int t = 0; t < n_threads; t++) pthread_create(&th[t], NULL, fn, job);
    for (int t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
    free(th);
}

/* Optional GPU comparison: g_off == NULL -> none.  topk_k == 0 -> l1 only. */
static gpu_cmp make_cmp(const int64_t *g_off, const int64_t *g_cnt, const int32_t *g_nodes,
                        const double *g_vals, double *out_l1d, double *out_l1r,
                        int32_t *out_topk, int32_t topk_k) {
    gpu_cmp c = {g_off, g_cnt, g_nodes, g_vals, out_l1d, out_l1r, topk_k > 0 ? out_topk : NULL,
                 topk_k};
    return c;
}

int orc_batch_local(int64_t n, const int64_t *off, const int64_t *tgt, const double *w,
                    const double *theta, double alpha, int32_t method, double omega,
                    const int64_t *seeds, int64_t n_seeds, int64_t max_sweeps, int32_t n_threads,
                    int64_t *out_sweeps, int64_t *out_ops, int64_t *out_pushes,
                    int32_t *out_conv, double *out_xsum, const int64_t *g_off,
                    const int64_t *g_cnt, const int32_t *g_nodes, const double *g_vals,
                    double *out_l1d, double *out_l1r, int32_t *out_topk, int32_t topk_k) {
    gpu_cmp C = make_cmp(g_off, g_cnt, g_nodes, g_vals, out_l1d, out_l1r, out_topk, topk_k);
    batch_job J = {n, off, tgt, w, theta, alpha, method, omega, 0.0, 0.0, seeds, n_seeds,
                   max_sweeps, out_sweeps, out_ops, out_pushes, out_conv, out_xsum,
                   g_off ? &C : NULL, 0};
    run_threads(batch_worker, &J, n_threads);
    return 0;
}

/* Per-seed local_ch over many threads: b = bval e_s (alpha for PPR, 1 for
 * Katz), operator given by the arc weights / thresholds. */
int orc_batch_local_ch(int64_t n, const int64_t *off, const int64_t *tgt, const double *w,
                       const double *theta, double bval, double mu, double L,
                       const int64_t *seeds, int64_t n_seeds, int64_t max_sweeps,
                       int32_t n_threads, int64_t *out_sweeps, int64_t *out_ops,
                       int32_t *out_conv, double *out_xsum, const int64_t *g_off,
                       const int64_t *g_cnt, const int32_t *g_nodes, const double *g_vals,
                       double *out_l1d, double *out_l1r, int32_t *out_topk, int32_t topk_k,
                       int32_t hb) {
    gpu_cmp C = make_cmp(g_off, g_cnt, g_nodes, g_vals, out_l1d, out_l1r, out_topk, topk_k);
    batch_job J = {n, off, tgt, w, theta, bval, hb ? 3 : 2, 1.0, mu, L, seeds, n_seeds, max_sweeps,
                   out_sweeps, out_ops, NULL, out_conv, out_xsum, g_off ? &C : NULL, 0};
    int64_t *pushes = malloc(sizeof(int64_t) * (n_seeds ? n_seeds : 1));
    J.out_pushes = pushes;
    run_threads(batch_worker, &J, n_threads);
    free(pushes);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* LocalGD-PPR at papers100M scale: rule weights, int32 targets             */
/* ------------------------------------------------------------------------ */

/* The same algorithm as orc_local_gd (src/local_solvers.py:428-470 with
 * _apply_update_seq :267-292 and _filter_frontier :336-350) for the PPR
 * system of make_ppr_system (src/systems.py:163-191), with the operator and
 * thresholds evaluated from their rules instead of stored arrays:
 *   arc_w[j] = fl(fl(1/d_u) * (1 - alpha))   (_gen_arc_weights "rw", :85-108)
 *   theta_u  = fl(fl(eps*alpha) * d_u), +inf at d_u = 0   (_theta_vec, :157-160)
 * which are the arrays' values bit for bit (tests/test_host.py).  Targets are
 * int32 (n < 2^31) and the per-thread dense state is allocated once and
 * reset over the nodes a seed wrote, so a 111 M-node graph needs ~3 GB per
 * thread instead of the reference's ~50 GB of per-solve arrays.  The l1 /
 * min-residual logs of the report are not produced (x, r, sweeps, ops and
 * pushes are).  A checker only: never a timed baseline. */
typedef struct {
    int64_t n;
    const int64_t *off;
    const int32_t *tgt;
    double alpha, beta, tcoeff;
    const int64_t *seeds;
    int64_t n_seeds, max_sweeps;
    int64_t *out_sweeps, *out_ops, *out_pushes;
    int32_t *out_conv;
    const gpu_cmp *cmp;
    int64_t next;
} rule_job;

static void *rule_worker(void *arg) {
    rule_job *J = arg;
    const int64_t n = J->n;
    const size_t nn = n ? (size_t)n : 1;
    double *x = calloc(nn, sizeof(double)), *r = calloc(nn, sizeof(double));
    double *vals = malloc(sizeof(double) * nn);
    uint8_t *cmark = calloc(nn, 1), *dmark = calloc(nn, 1);
    int32_t *cand = malloc(sizeof(int32_t) * nn), *front = malloc(sizeof(int32_t) * nn);
    int32_t *fbuf = malloc(sizeof(int32_t) * nn), *dirty = malloc(sizeof(int32_t) * nn);
    double *scratch = J->cmp ? calloc(nn, sizeof(double)) : NULL;
    for (;;) {
        int64_t i = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
        if (i >= J->n_seeds) break;
        const int32_t s = (int32_t)J->seeds[i];
        int64_t nd = 0;
        r[s] = J->alpha;
        dmark[s] = 1;
        dirty[nd++] = s;
        const int64_t ds = J->off[s + 1] - J->off[s];
        const double ths = ds > 0 ? J->tcoeff * (double)ds : INFINITY;
        int64_t fc = r[s] >= ths ? 1 : 0;
        front[0] = s;
        int64_t sweeps = 0, ops = 0, pushes = 0;
        int32_t conv = 1;
        while (fc) {
            if (sweeps >= J->max_sweeps) { conv = 0; break; }
            int64_t svol = 0;
            for (int64_t q = 0; q < fc; q++) {
                const int32_t u = front[q];
                svol += J->off[u + 1] - J->off[u];
                vals[q] = r[u];
            }
            for (int64_t q = 0; q < fc; q++) x[front[q]] += vals[q];
            /* _apply_update_seq */
            int64_t cc = 0;
            for (int64_t q = 0; q < fc; q++) {
                const int32_t u = front[q];
                r[u] -= vals[q];
                if (!cmark[u]) { cmark[u] = 1; cand[cc++] = u; }
            }
            for (int64_t q = 0; q < fc; q++) {
                const int32_t u = front[q];
                const double val = vals[q];
                const double wu = (1.0 / (double)(J->off[u + 1] - J->off[u])) * J->beta;
                for (int64_t j = J->off[u]; j < J->off[u + 1]; j++) {
                    const int32_t v = J->tgt[j];
                    r[v] += val * wu;
                    if (!dmark[v]) { dmark[v] = 1; dirty[nd++] = v; }
                    if (!cmark[v]) { cmark[v] = 1; cand[cc++] = v; }
                }
            }
            /* _filter_frontier */
            int64_t nf = 0;
            for (int64_t q = 0; q < cc; q++) {
                const int32_t u = cand[q];
                cmark[u] = 0;
                const int64_t du = J->off[u + 1] - J->off[u];
                const double th = du > 0 ? J->tcoeff * (double)du : INFINITY;
                if (r[u] >= th) fbuf[nf++] = u;
            }
            memcpy(front, fbuf, sizeof(int32_t) * nf);
            ops += svol;
            pushes += fc;
            sweeps += 1;
            fc = nf;
        }
        J->out_sweeps[i] = sweeps;
        J->out_ops[i] = ops;
        J->out_pushes[i] = pushes;
        J->out_conv[i] = conv;
        if (J->cmp) cmp_seed(J->cmp, i, x, n, scratch);
        for (int64_t q = 0; q < nd; q++) {
            const int32_t v = dirty[q];
            x[v] = 0.0; r[v] = 0.0; dmark[v] = 0;
        }
    }
    free(x); free(r); free(vals); free(cmark); free(dmark);
    free(cand); free(front); free(fbuf); free(dirty); free(scratch);
    return NULL;
}

int orc_batch_gd_rule(int64_t n, const int64_t *off, const int32_t *tgt, double alpha,
                      double eps, const int64_t *seeds, int64_t n_seeds, int64_t max_sweeps,
                      int32_t n_threads, int64_t *out_sweeps, int64_t *out_ops,
                      int64_t *out_pushes, int32_t *out_conv, const int64_t *g_off,
                      const int64_t *g_cnt, const int32_t *g_nodes, const double *g_vals,
                      double *out_l1d, double *out_l1r, int32_t *out_topk, int32_t topk_k) {
    gpu_cmp C = make_cmp(g_off, g_cnt, g_nodes, g_vals, out_l1d, out_l1r, out_topk, topk_k);
    rule_job J = {n, off, tgt, alpha, 1.0 - alpha, eps * alpha, seeds, n_seeds, max_sweeps,
                  out_sweeps, out_ops, out_pushes, out_conv, g_off ? &C : NULL, 0};
    run_threads(rule_worker, &J, n_threads);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* batched CPU baseline of the heat kernel: the reference's local_hk per   */
/* seed (src/local_solvers.py:664-696), one seed per thread, dense         */
/* (N+1) n state per thread as in the reference                            */
/* ------------------------------------------------------------------------ */

typedef struct {
    int64_t n, n_stages;
    const int64_t *off, *tgt;
    const double *base_w, *stage_w, *theta;
    double tau;
    const int64_t *seeds;
    int64_t n_seeds, max_sweeps;
    int64_t *out_sweeps, *out_ops;
    int32_t *out_conv;
    double *out_fsum;
    const gpu_cmp *cmp;  /* against f_hat */
    int64_t next;
} hk_job;

static void *hk_worker(void *arg) {
    hk_job *J = arg;
    const int64_t dim = (J->n_stages + 1) * J->n;
    double *v = malloc(sizeof(double) * (dim ? dim : 1));
    double *r = malloc(sizeof(double) * (dim ? dim : 1));
    double *f = (J->out_fsum || J->cmp) ? malloc(sizeof(double) * (J->n ? J->n : 1)) : NULL;
    double *scratch = J->cmp ? calloc(J->n ? J->n : 1, sizeof(double)) : NULL;
    for (;;) {
        int64_t i = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
        if (i >= J->n_seeds) break;
        memset(v, 0, sizeof(double) * dim);
        memset(r, 0, sizeof(double) * dim);
        r[J->seeds[i]] = 1.0; /* b = e_s at stage 0 */
        orc_report rep;
        orc_hk_push(J->n, J->n_stages, J->off, J->tgt, J->base_w, J->stage_w, J->theta, v, r,
                    J->seeds[i], J->max_sweeps, &rep);
        J->out_sweeps[i] = rep.sweeps;
        J->out_ops[i] = rep.total_ops;
        J->out_conv[i] = rep.converged;
        if (f) { /* f_hat = e^-tau * sum_k v_k (stage order per node, back_transform) */
            const double e = exp(-J->tau);
            double s = 0.0;
            for (int64_t u = 0; u < J->n; u++) {
                double acc = v[u];
                for (int64_t k = 1; k <= J->n_stages; k++) acc += v[k * J->n + u];
                f[u] = e * acc;
                s += f[u];
            }
            if (J->out_fsum) J->out_fsum[i] = s;
            if (J->cmp) cmp_seed(J->cmp, i, f, J->n, scratch);
        }
        orc_report_free(&rep);
    }
    free(v);
    free(r);
    free(f);
    free(scratch);
    return NULL;
}

int orc_batch_hk(int64_t n, int64_t n_stages, const int64_t *off, const int64_t *tgt,
                 const double *base_w, const double *stage_w, const double *theta, double tau,
                 const int64_t *seeds, int64_t n_seeds, int64_t max_sweeps, int32_t n_threads,
                 int64_t *out_sweeps, int64_t *out_ops, int32_t *out_conv, double *out_fsum,
                 const int64_t *g_off, const int64_t *g_cnt, const int32_t *g_nodes,
                 const double *g_vals, double *out_l1d, double *out_l1r, int32_t *out_topk,
                 int32_t topk_k) {
    gpu_cmp C = make_cmp(g_off, g_cnt, g_nodes, g_vals, out_l1d, out_l1r, out_topk, topk_k);
    hk_job J = {n, n_stages, off, tgt, base_w, stage_w, theta, tau, seeds, n_seeds, max_sweeps,
                out_sweeps, out_ops, out_conv, out_fsum, g_off ? &C : NULL, 0};
    run_threads(hk_worker, &J, n_threads);
    return 0;
}
