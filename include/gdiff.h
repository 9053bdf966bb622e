/*
 * gdiff.h -- C ABI of the B200 local-diffusion library (libgdiff.so).
 *
 * Drop-in boundary for the reference package's native layer: the numba
 * kernels of /root/reference/pkg/src/graphdiff (cited as src/<file>:<line>)
 * and the Python sweep drivers around them.  Array arguments follow the
 * numpy layouts those kernels take (int64 CSR offsets/targets, float64
 * vectors), plain pointers and sizes, no framework types; a ctypes binding
 * can pass numpy buffers straight through.
 *
 * Memory: functions named *_device take device pointers and a cudaStream_t
 * (passed as void*); every other pointer argument is host memory.  The
 * library keeps graphs resident in HBM (gd_graph) so repeated solves on one
 * graph do not re-upload it.
 *
 * Errors: every function returns GD_OK (0) or a negative code; the message
 * of the last failure on the calling thread is available from
 * gd_last_error().  Non-convergence is NOT an error: it is reported through
 * gd_report.converged, like the reference.
 *
 * Numerics: single-system solvers are bit-exact with the reference
 * (identical x, r, frontier traces, sweep/operation counts); see DESIGN.md.
 */
#ifndef GDIFF_H
#define GDIFF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GD_OK 0
#define GD_ERR_ARG (-1)
#define GD_ERR_CUDA (-2)
#define GD_ERR_OOM (-3)
#define GD_ERR_CAPACITY (-4)
#define GD_ERR_UNSUPPORTED (-5)

/* scatter-weight rules: replace OperatorQ.arc_weights (src/systems.py:43-108) */
#define GD_W_RW 0    /* w_j = fl(fl(1/d_u) * beta)  ("rw", and "gen" with b=0)  */
#define GD_W_CONST 1 /* w_j = beta                  ("adj", Katz)             */
#define GD_W_ARC 2   /* w_j = arc_w[j]              (any other operator)       */

/* threshold rules: replace DiffusionSystem.theta (src/systems.py:157-160) */
#define GD_T_DEGREE 0 /* theta_u = fl(coeff * d_u), +inf where d_u == 0 */
#define GD_T_ARRAY 1  /* theta_u = theta[u]                            */

typedef struct gd_graph gd_graph;

typedef struct {
    int32_t weight_rule;  /* GD_W_* */
    int32_t theta_rule;   /* GD_T_* */
    double beta;          /* operator damping (GD_W_RW / GD_W_CONST) */
    double theta_coeff;   /* GD_T_DEGREE */
    const double *arc_w;  /* GD_W_ARC: n_arcs entries (host) */
    const double *theta;  /* GD_T_ARRAY: dim entries (host) */
} gd_operator;

/* Run report: mirrors LocalReport / SolveReport (src/reports.py:25-79) plus
 * the frontier trace of SolverState (src/reports.py:14-22).  Arrays are
 * owned by the library; release them with gd_report_free. */
typedef struct {
    int32_t converged;
    int32_t diverged;        /* LocalCH abort (src/local_solvers.py:527-530) */
    int64_t sweeps;
    int64_t total_ops;       /* sum of vol(S_t) */
    int64_t pushes;          /* sum of |S_t| */
    double min_residual;
    int64_t support_size;    /* count_nonzero(r) */
    int64_t n_logs;          /* == sweeps */
    int64_t *vol_log;        /* n_logs */
    double *gamma_log;       /* n_logs */
    double *l1_log;          /* n_logs + 1 */
    int8_t *sign_log;        /* n_logs (FIFO solvers) */
    int64_t *frontier_sizes; /* n_logs (sweep-synchronous solvers) */
    int64_t *trace;          /* concatenated S_t when recorded */
    int64_t trace_len;
    double *l2_log;          /* n_logs + 1 (global GD) */
} gd_report;

/* ---- library ---------------------------------------------------------- */
const char *gd_last_error(void);
int gd_version(void);
void gd_report_free(gd_report *rep);

/* ---- graph (replaces CsrGraph arrays, src/graph.py:62-81) --------------- */
/* Upload host int64 offsets[n+1] / targets[n_arcs] (canonical symmetric CSR)
 * to HBM as int64 row_ptr + int32 col_idx + int32 degree. */
int gd_graph_create(int64_t n, const int64_t *offsets, const int64_t *targets,
                    int64_t n_arcs, int32_t device, gd_graph **out);
/* Same from device buffers (int64 row_ptr, int32 col_idx), e.g. a graph
 * generated on the GPU; the data is copied. */
int gd_graph_create_device(int64_t n, const int64_t *d_row_ptr, const int32_t *d_col,
                           int64_t n_arcs, int32_t device, gd_graph **out);
/* A new graph: g with an ordered batch of undirected edge events applied
 * (kinds[i] = 1 insert, 0 delete of (us[i], vs[i])), built on the device;
 * the same canonical CSR as apply_events (src/graph.py:235-258).  Errors
 * (GD_ERR_ARG) on an insert of a present / delete of a missing edge. */
int gd_graph_apply_events(const gd_graph *g, const int32_t *kinds, const int64_t *us,
                          const int64_t *vs, int64_t n_events, gd_graph **out);
/* Same, into an existing graph h != g whose device buffers are reused. */
int gd_graph_apply_events_into(const gd_graph *g, const int32_t *kinds, const int64_t *us,
                               const int64_t *vs, int64_t n_events, gd_graph *h);
/* Copy a device graph back in the reference layout (int64 n+1 offsets,
 * int64 n_arcs targets). */
int gd_graph_export(const gd_graph *g, int64_t *offsets, int64_t *targets);
int gd_graph_destroy(gd_graph *g);
int gd_graph_info(const gd_graph *g, int64_t *n, int64_t *n_arcs, int64_t *d_max);

/* ---- single-system solvers (host buffers in/out, bit-exact) ------------ */

/* LocalGD: replaces local_gd (src/local_solvers.py:428-470) with its kernels
 * _apply_update_seq :267-292, _filter_frontier :336-350, _l1_and_min :353-361.
 * b: dim source; x, r: dim outputs. */
int gd_local_gd(const gd_graph *g, const gd_operator *op, const double *b, double *x,
                double *r, int64_t max_sweeps, int32_t record_trace, gd_report *rep);

/* Warm-started (signed) LocalGD from a pair: x = p, r = s - Q p on entry,
 * updated in place; S_0 = filter(flatnonzero(r)).  The sweep loop of
 * local_gd (src/local_solvers.py:364-470) with _filter_frontier(signed)
 * :336-350, started from the event-adjusted pair of dynamic.py:110-128
 * (the LocalGD form of repair, config 5). */
int gd_local_gd_warm(const gd_graph *g, const gd_operator *op, double *x, double *r,
                     int32_t is_signed, int64_t max_sweeps, int32_t record_trace,
                     gd_report *rep);

/* LocalCH: replaces local_ch (src/local_solvers.py:473-538); mu, L already
 * resolved (the _cheby_bounds rule, :541-558). */
int gd_local_ch(const gd_graph *g, const gd_operator *op, const double *b, double *x,
                double *r, double mu, double L, int64_t max_sweeps, int32_t record_trace,
                gd_report *rep);
/* LocalHB (heavy-ball momentum, no reference counterpart): local_ch's loop with
 * eta = 4/(sqrt(L)+sqrt(mu))^2, beta = ((sqrt(L)-sqrt(mu))/(sqrt(L)+sqrt(mu)))^2;
 * bit-exact with the restatement oracle/ orc_local_hb. */
int gd_local_hb(const gd_graph *g, const gd_operator *op, const double *b, double *x,
                double *r, double mu, double L, int64_t max_sweeps, int32_t record_trace,
                gd_report *rep);

/* FIFO push: replaces _push_kernel (src/local_solvers.py:48-188); x, r are
 * updated in place (LocalGS/LocalSOR, dynamic repair). */
int gd_push_kernel(const gd_graph *g, const gd_operator *op, double *x, double *r,
                   const int64_t *seeds, int64_t n_seeds, double omega, double x_gain,
                   int32_t is_signed, int64_t max_sweeps, gd_report *rep);

/* Heat-kernel push: replaces _hk_push_kernel (src/local_solvers.py:566-661).
 * v, r: (n_stages+1)*n, in place; thresholds theta_coeff * d_u per stage
 * (src/systems.py:295-299); base weights fl(1/d_u). */
int gd_hk_push(const gd_graph *g, int64_t n_stages, const double *stage_w,
               double theta_coeff, double *v, double *r, int64_t seed, int64_t max_sweeps,
               gd_report *rep);

/* Global gradient descent (reference point): replaces gradient_descent +
 * _scatter_full + _any_active (src/global_solvers.py:41-71, :124-152). */
int gd_gradient_descent(const gd_graph *g, const gd_operator *op, const double *b,
                        double *x, double *r, int64_t max_sweeps, gd_report *rep);

/* Global Chebyshev (reference point): replaces chebyshev (src/global_solvers.py:
 * 155-204); mu < L resolved by the caller (cheby_bounds).  x, r: n doubles out;
 * rep: l1 and l2 per sweep. */
int gd_chebyshev(const gd_graph *g, const gd_operator *op, const double *b, double *x,
                 double *r, double mu, double L, int64_t max_sweeps, gd_report *rep);

/* Heat-kernel Taylor stages: replaces hk_taylor_global (src/global_solvers.py:
 * 207-235).  b0: stage-0 vector (n); v: (n_stages+1)*n out, v_{k+1} =
 * fl(stage_w[k] * P v_k) with P the bare 1/d_u column scatter. */
int gd_hk_taylor(const gd_graph *g, int64_t n_stages, const double *stage_w, const double *b0,
                 double *v);

/* Spectral norm estimate of A (Katz alpha / Chebyshev bounds): replaces
 * spectral_norm_estimate (src/graph.py:267-295), the shifted power iteration
 * on A + d_max I from the caller's start vector x0 (n entries); agrees with
 * the reference to rounding (its dot products go through BLAS). */
int gd_spectral_norm(const gd_graph *g, const double *x0, int64_t iters, double *lam_out);

/* ---- batched multi-seed solves (new; no reference counterpart) --------- */
/* A batch solves PPR systems (I - (1-alpha) A D^-1) x = alpha e_s for many
 * seeds s; the per-seed result equals local_gd(make_ppr_system(g, alpha, s,
 * eps)) (same frontier sets, sweeps and operation counts; x to rounding of
 * the atomic scatter order) for GD_M_LOCAL_GD, and local_sor(..., omega)
 * bit for bit for GD_M_LOCAL_SOR.  Per-seed state lives in `slots` dense
 * HBM vectors that are reset by walking what a seed touched. */
#define GD_M_LOCAL_GD 0  /* sweep-synchronous LocalGD (batch.cu)                 */
#define GD_M_LOCAL_SOR 1 /* FIFO LocalSOR / LocalGS, one warp per seed, bit-exact */
#define GD_M_LOCAL_CH 2  /* sweep-synchronous LocalCH, signed frontier
                            (batch_signed.cu): per seed local_ch(sys, mu, L)
                            with the same frontier sets, sweeps and operation
                            counts, x to rounding of the atomic scatter */

#define GD_M_LOCAL_HB 4  /* LocalHB: LocalCH's sweep loop with Polyak's heavy-ball
                            coefficients (no reference counterpart; restatement
                            oracle/ orc_local_hb), same frontier rule, momentum
                            stamps and divergence abort (batch_signed.cu) */
#define GD_M_HK 3        /* heat-kernel push on the stage-expanded system, run as
                            layered sweeps (batch.cu): per seed local_hk(g, tau,
                            s, eps) with the same sweeps and operation counts,
                            f_hat (x out, e^-tau applied) to rounding */

#define GD_P_PPR 0  /* (I - (1-alpha) A D^-1) x = alpha e_s, theta = eps alpha d */
#define GD_P_KATZ 1 /* (I - alpha A) x = e_s, theta = eps d (src/systems.py:194-219);
                       GD_M_LOCAL_CH only */

typedef struct gd_batch gd_batch;

#define GD_RESOLVE_FLAG 0
#define GD_RESOLVE_EXACT 1
#define GD_RESOLVE_ALL 2

typedef struct {
    int32_t method;      /* GD_M_* */
    int32_t slots;       /* seeds in flight on the device; 0 = auto */
    double alpha;
    double eps;
    int64_t max_sweeps;
    int64_t frontier_cap; /* max frontier entries per round; 0 = auto */
    int64_t out_cap;      /* max output (node, x) pairs per solve; 0 = auto */
    int32_t relabel;      /* 1: run on a degree-descending renumbering of the
                             graph (hubs contiguous: residual updates share
                             sectors / stay in L2); ids in and out are the
                             caller's.  Results are invariant. */
    int32_t problem;      /* GD_P_* (GD_P_KATZ with GD_M_LOCAL_CH only) */
    double omega;         /* GD_M_LOCAL_SOR: relaxation (1 = LocalGS, signed
                             frontier when > 1, src/local_solvers.py:238) */
    double mu, L;         /* GD_M_LOCAL_CH: eigenvalue bounds, mu < L (the
                             reference's cheby_bounds, src/local_solvers.py:541-558;
                             0, 0 = PPR defaults alpha, 2 - alpha) */
    /* GD_M_HK: the system of make_hk_system (src/systems.py:269-301): */
    double tau;
    int64_t n_stages;        /* N */
    const double *stage_w;   /* host, N entries: tau/(k+1) as the system stores them */
    double theta_coeff;      /* eps / (2 (N+1) vol); theta = fl(coeff * d) */
    int32_t want_r;          /* 1: also return each seed's final r as a sparse vector
                                (GD_M_LOCAL_GD / GD_M_LOCAL_CH / GD_M_LOCAL_SOR) */
    int32_t resolve;         /* near-threshold policy of the atomic-scatter batches
                                (LocalGD / LocalCH; see gd_batch_result.ambiguous):
                                GD_RESOLVE_FLAG (0): flag ambiguous seeds only;
                                GD_RESOLVE_EXACT (1): re-solve the flagged seeds on
                                the bit-exact path (their results are then the
                                reference's bit for bit);
                                GD_RESOLVE_ALL (2): re-solve every seed so. */
    int32_t log_sweeps;      /* LocalGD: > 0 = record per seed the first log_sweeps
                                sweeps' frontier size |S_t|, volume vol(S_t) and
                                sum |r_u| over S_t (the LocalReport logs,
                                src/reports.py:51-79; see gd_batch_logs) */
    int32_t reserved2;
} gd_batch_params;

typedef struct {
    /* per-seed, device arrays of n_seeds entries owned by the batch */
    int64_t *sweeps, *total_ops, *pushes, *support;
    int32_t *converged;
    int64_t *x_offset, *x_count;  /* segment of seed i in x_nodes/x_vals */
    int32_t *x_nodes;
    double *x_vals;
    int64_t x_total;              /* filled after synchronisation */
    int64_t kernel_launches;      /* kernels this solve launched */
    /* near-threshold detector of the atomic-scatter batches: ambiguous[i] = 1
       when one of seed i's batched updates landed within 2^-36 (relative) of
       its threshold, where the scatter order could decide frontier
       membership; such seeds were re-solved on the bit-exact path (their
       results above are the reference's bit for bit) */
    int32_t *ambiguous;           /* device, n_seeds entries */
    int64_t n_ambiguous;
} gd_batch_result;

int gd_batch_create(const gd_graph *g, const gd_batch_params *p, gd_batch **out);
int gd_batch_destroy(gd_batch *b);
/* d_seeds: device int64[n_seeds]; results stay on the device in *res.
 * stream: cudaStream_t (NULL = legacy default stream). */
int gd_batch_solve_device(gd_batch *b, const int64_t *d_seeds, int64_t n_seeds,
                          gd_batch_result *res, void *stream);
/* Host entry: seeds from host memory, per-seed stats and the sparse x
 * copied back into caller buffers (pinned memory recommended).  x buffers
 * hold x_cap pairs; GD_ERR_CAPACITY (with *x_total set) if too small.
 * In the wave (round-kernel) form each finished wave's (node, x) pairs are
 * copied into x_nodes / x_vals on a second stream while the next wave runs;
 * every copy has completed when the call returns. */
int gd_batch_solve_host(gd_batch *b, const int64_t *seeds, int64_t n_seeds,
                        int64_t *sweeps, int64_t *total_ops, int64_t *pushes,
                        int32_t *converged, int64_t *x_offset, int64_t *x_count,
                        int32_t *x_nodes, double *x_vals, int64_t x_cap, int64_t *x_total,
                        void *stream);
/* Copy the results of the last solve into host buffers again (e.g. after
 * GD_ERR_CAPACITY from gd_batch_solve_host) without re-solving. */
int gd_batch_fetch_host(gd_batch *b, int64_t n_seeds, int64_t *sweeps, int64_t *total_ops,
                        int64_t *pushes, int32_t *converged, int64_t *x_offset, int64_t *x_count,
                        int32_t *x_nodes, double *x_vals, int64_t x_cap, int64_t *x_total,
                        void *stream);
/* Sparse r of the last solve (want_r): device arrays owned by the batch
 * (r_offset / r_count per seed, then (node, value) pairs, caller ids). */
int gd_batch_r_device(const gd_batch *b, int64_t **r_offset, int64_t **r_count,
                      int32_t **r_nodes, double **r_vals, int64_t *r_total);
/* The same copied into host buffers; GD_ERR_CAPACITY with *r_total set when
 * r_cap is too small (fetch again with larger buffers). */
int gd_batch_fetch_r_host(gd_batch *b, int64_t n_seeds, int64_t *r_offset, int64_t *r_count,
                          int32_t *r_nodes, double *r_vals, int64_t r_cap, int64_t *r_total,
                          void *stream);
/* Per-seed sweep logs of the last solve (log_sweeps > 0): host arrays of
 * n_seeds * log_sweeps entries, row i = seed i, entry t = sweep t (rows hold
 * min(sweeps, log_sweeps) entries, the rest 0): |S_t|, vol(S_t) and the sum
 * of |r_u| pushed in sweep t (gamma_t = that / l1_t; for PPR l1_{t+1} =
 * l1_t - alpha * that).  Any pointer may be NULL. */
int gd_batch_logs(const gd_batch *b, int64_t n_seeds, int64_t *frontier_sizes, int64_t *vol_log,
                  double *pushed_mass);
/* Seeds of the last solve that the near-threshold detector flagged and the
 * bit-exact path re-solved (see gd_batch_result.ambiguous). */
int gd_batch_last_ambiguous(const gd_batch *b, int64_t *count);
/* The same count, how many of those seeds the exact re-solve changed
 * (sweeps / operation counts / pushes differed from the batch's), and the
 * host wall time (ms) the re-solves took. */
int gd_batch_resolve_stats(const gd_batch *b, int64_t *flagged, int64_t *changed, double *ms);
/* Change the near-threshold policy (GD_RESOLVE_*) of an existing batch. */
int gd_batch_set_resolve(gd_batch *b, int32_t mode);
/* Device time (ms) of the dominant kernel (the sweep loop) in the last
 * solve, measured with CUDA events on the launching stream. */
int gd_batch_last_kernel_ms(const gd_batch *b, double *ms);
/* Execution form chosen at creation: GD_BATCH_STREAM (the round kernel, slots
 * refilled in-kernel as seeds finish), GD_BATCH_ROUNDS (the wave round kernel,
 * k_rounds / k_signed_rounds), GD_BATCH_CTA (LocalGD on small graphs: one CTA
 * per seed, k_seed_cta) or GD_BATCH_FIFO (LocalSOR/GS, warp per seed); and
 * the number of seeds in flight. */
#define GD_BATCH_ROUNDS 0
#define GD_BATCH_CTA 1
#define GD_BATCH_FIFO 2
#define GD_BATCH_FIFO_WIN 3 /* LocalSOR/GS in exact windows, one CTA per seed */
#define GD_BATCH_STREAM 4   /* the round kernel with slots refilled in-kernel
                               (k_rounds streaming form: LocalGD without want_r) */
#define GD_BATCH_CTA_SMEM 5 /* GD_BATCH_CTA with each seed's whole state in shared
                               memory (k_seed_smem: graphs of up to ~6 K nodes) */
int gd_batch_info(const gd_batch *b, int32_t *mode, int64_t *slots);
/* Instrumentation of the last wave: per sweep round (F entries, P arcs,
 * device globaltimer ns) as 3*min(cap, rounds) int64 values. */
int gd_batch_round_log(const gd_batch *b, int64_t *out, int64_t cap, int64_t *rounds);
/* ... and the device ns at which each round's scatter phase began (cap/2
 * entries), then per round the slots whose seed finished (| refill << 32). */
int gd_batch_round_phase_log(const gd_batch *b, int64_t *out, int64_t cap);

/* ---- multi-column degree-generalized feature push (new) -------------- */
/* beta_push (src/dynamic.py:199-222) for every column of a source matrix:
 * per column a signed FIFO push (_push_kernel) from p = 0, r = source with
 * per-arc weights arc_w (n_arcs) and thresholds theta (n), x_gain = alpha;
 * one warp per column, each column bit-identical with beta_push.
 * source, p_out, r_out: n x ncols host arrays, row-major; the per-column
 * statistics may be NULL. */
int gd_feature_push(const gd_graph *g, const double *arc_w, const double *theta, double x_gain,
                    double omega, int64_t ncols, const double *source, int64_t max_sweeps,
                    double *p_out, double *r_out, int64_t *sweeps, int64_t *total_ops,
                    int64_t *pushes, int32_t *converged);

/* ---- resident PPR pairs on an evolving graph (config 5, batched) ------- */
/* K pairs (p_i, r_i) with r_i = alpha e_{s_i} - (I - (1-alpha) A D^-1) p_i
 * kept in HBM across snapshots.  Replaces, for K sources at once, the
 * reference's per-source loop of event_adjust + repair (src/dynamic.py:
 * 110-196): every event batch is applied to every pair in event order (the
 * O(1) endpoint corrections, bit-exact), then all pairs are repaired on the
 * new graph by one warm-started signed LocalGD solve (thresholds eps d_u,
 * src/dynamic.py:139-141).  Per-pair sweeps / total_ops / pushes equal the
 * single-pair warm LocalGD on the same state; p, r to rounding of the
 * atomic scatter. */
typedef struct gd_pairs gd_pairs;

/* Pairs start at (0, alpha e_s) and are solved on g (stats: k entries each,
 * any may be NULL).  frontier_cap / max_sweeps: 0 = auto. */
int gd_pairs_create(const gd_graph *g, double alpha, double eps, const int64_t *sources,
                    int64_t k, int64_t frontier_cap, int64_t max_sweeps, gd_pairs **out,
                    int64_t *sweeps, int64_t *total_ops, int64_t *pushes, int32_t *converged);
/* Repair method of a pool: GD_PAIRS_GD (default above) = warm-started signed
 * LocalGD, sweep-synchronous over all pairs (p, r to rounding); GD_PAIRS_PUSH =
 * the reference's own repair (src/dynamic.py:131-162: seeds flatnonzero(|r| >=
 * eps d), signed FIFO push _push_kernel with omega = 1), one warp per pair,
 * bit-identical p, r, sweeps and operation counts. */
#define GD_PAIRS_GD 0
#define GD_PAIRS_PUSH 1
int gd_pairs_create_ex(const gd_graph *g, double alpha, double eps, const int64_t *sources,
                       int64_t k, int64_t frontier_cap, int64_t max_sweeps, int32_t method,
                       gd_pairs **out, int64_t *sweeps, int64_t *total_ops, int64_t *pushes,
                       int32_t *converged);
int gd_pairs_destroy(gd_pairs *p);
/* g_new must be the previous graph with the events applied (checked on the
 * degrees); kinds[i] = 1 insert, 0 delete of edge (us[i], vs[i]). */
int gd_pairs_update(gd_pairs *p, const gd_graph *g_new, const int32_t *kinds, const int64_t *us,
                    const int64_t *vs, int64_t n_events, int64_t max_sweeps, int64_t *sweeps,
                    int64_t *total_ops, int64_t *pushes, int32_t *converged);
/* Dense host copies of pair i (n doubles each; either pointer may be NULL). */
int gd_pairs_get(const gd_pairs *p, int64_t i, double *p_out, double *r_out);
/* Device view: pair i's p at p[i*ld .. i*ld+n), r likewise. */
int gd_pairs_device(const gd_pairs *p, double **p_dev, double **r_dev, int64_t *ld);
/* Device time (ms) of the last repair's sweep loop (CUDA events). */
int gd_pairs_last_kernel_ms(const gd_pairs *p, double *ms);

/* ---- synthetic graphs -------------------------------------------------- */
/* R-MAT candidate edges [first, first+count) at `scale`, ids permuted and
 * encoded as key = min*n + max, or -1 when dropped (id >= n or self loop);
 * identical to paper_2410_21634_b200.synth.rmat_edges + permute_ids. */
int gd_rmat_keys_device(int32_t scale, int64_t n, int64_t first, int64_t count,
                        uint64_t seed, double a, double b, double c, int64_t *d_keys,
                        void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GDIFF_H */
