// feature_push.cu -- multi-column degree-generalized signed feature push.
//
// beta_push (src/dynamic.py:199-222) repairs ONE source column: a signed FIFO
// push (_push_kernel, src/local_solvers.py:48-188) from p = 0, r = source,
// with weights (1-alpha) / (d_u^(1-b) d_v^b), thresholds eps d_u^(1-b) and
// x_gain = alpha (the alpha-p convention).  Feature propagation (APPNP /
// InstantGNN style) runs it for every column of a
// feature matrix; the columns are independent, so one warp owns a column:
// its dense p and r columns are both the working state and the output.
// Per column the pops, the enqueue order and every fl() step are the
// reference's, so each column is bit-identical with beta_push on it.
#include "common.cuh"
#include "window.cuh"

namespace gd {
namespace {

constexpr int FP_THREADS = 128;
constexpr unsigned FPFULL = 0xffffffffu;

struct FpArgs {
    DevGraph g;
    const double *arc_w;  // n_arcs
    const double *theta;  // n
    double x_gain, omega;
    int64_t n, ncols, max_sweeps;
    double *p, *r;        // n x ncols, column-major (column c at c * n)
    int32_t *queue;       // per warp: n + 2
    uint32_t *qmark;      // per warp: qw words
    int64_t qw;
    int nwarps;
    unsigned long long *next_col;
    int64_t *sweeps, *ops, *pushes;
    int32_t *conv;
};

__device__ __forceinline__ unsigned fp_lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__global__ void __launch_bounds__(FP_THREADS) k_feature_push(FpArgs A) {
    const int lane = threadIdx.x & 31;
    const int wid = (int)((blockIdx.x * (int64_t)FP_THREADS + threadIdx.x) >> 5);
    if (wid >= A.nwarps) return;
    int32_t *queue = A.queue + (int64_t)wid * (A.n + 2);
    uint32_t *qmark = A.qmark + (int64_t)wid * A.qw;
    const int64_t sent = A.n, qcap = A.n + 2;
    for (;;) {
        unsigned long long ci = 0;
        if (lane == 0) ci = atomicAdd(A.next_col, 1ULL);
        ci = __shfl_sync(FPFULL, ci, 0);
        if ((int64_t)ci >= A.ncols) break;
        double *x = A.p + (int64_t)ci * A.n, *r = A.r + (int64_t)ci * A.n;
        // seeds = flatnonzero(|r| >= theta) in index order (dynamic.py:141),
        // enqueued in order (local_solvers.py:59-69): a warp-wide ordered scan
        int64_t rear = 0;
        for (int64_t b = 0; b < A.n; b += 32) {
            const int64_t u = b + lane;
            bool act = false;
            if (u < A.n) act = fabs(r[u]) >= A.theta[u];
            const unsigned bal = __ballot_sync(FPFULL, act);
            if (act) {
                queue[rear + __popc(bal & fp_lanemask_lt())] = (int32_t)u;
                atomicOr(qmark + (u >> 5), 1u << (u & 31));
            }
            rear += __popc(bal);
        }
        int64_t front = 0, sweeps = 0, ops = 0, pushes = 0;
        int conv = 1;
        if (rear > 0) {
            if (lane == 0) queue[rear] = (int32_t)sent;
            rear = rear + 1 == qcap ? 0 : rear + 1;
            int64_t svol = 0;
            __syncwarp();
            for (;;) {
                const int64_t u = queue[front];
                front = (front + 1 == qcap) ? 0 : front + 1;
                if (u == sent) {  // sweep boundary (:102-144)
                    ops += svol;
                    sweeps += 1;
                    if (front == rear) break;
                    if (sweeps >= A.max_sweeps) {
                        conv = 0;
                        break;
                    }
                    if (lane == 0) queue[rear] = (int32_t)sent;
                    rear = (rear + 1 == qcap) ? 0 : rear + 1;
                    svol = 0;
                    __syncwarp();
                    continue;
                }
                const double ru = r[u];
                const double th = A.theta[u];
                const int64_t rs = A.g.row[u];
                const int32_t d = A.g.deg[u];
                if (lane == 0) atomicAnd(qmark + (u >> 5), ~(1u << (u & 31)));
                if (fabs(ru) < th) {
                    __syncwarp();
                    continue;
                }
                svol += d;
                pushes += 1;
                const double res = __dmul_rn(A.omega, ru);
                if (lane == 0) {
                    x[u] = __dadd_rn(x[u], __dmul_rn(A.x_gain, res));
                    r[u] = __dsub_rn(ru, res);
                }
                for (int64_t base = 0; base < d; base += 32) {
                    const int64_t j = base + lane;
                    bool act = false;
                    int32_t v = 0;
                    if (j < d) {
                        v = A.g.col[rs + j];
                        const double old = r[v];
                        const double w = A.arc_w[rs + j];
                        const uint32_t qm = qmark[v >> 5];
                        const double tv = A.theta[v];
                        const double rv = __dadd_rn(old, __dmul_rn(res, w));
                        r[v] = rv;
                        act = !((qm >> (v & 31)) & 1u) && fabs(rv) >= tv;
                    }
                    const unsigned bal = __ballot_sync(FPFULL, act);
                    if (act) {
                        int64_t q = rear + __popc(bal & fp_lanemask_lt());
                        if (q >= qcap) q -= qcap;
                        queue[q] = v;
                        atomicOr(qmark + (v >> 5), 1u << (v & 31));
                    }
                    rear += __popc(bal);
                    if (rear >= qcap) rear -= qcap;
                }
                __syncwarp();
                const double ru2 = __dsub_rn(ru, res);  // self re-check (:176-185)
                if (fabs(ru2) >= th) {
                    if (lane == 0) {
                        queue[rear] = (int32_t)u;
                        atomicOr(qmark + (u >> 5), 1u << (u & 31));
                    }
                    rear = (rear + 1 == qcap) ? 0 : rear + 1;
                }
                __syncwarp();
            }
            if (!conv)  // marks of the nodes still queued
                for (int64_t w = lane; w < A.qw; w += 32) qmark[w] = 0u;
        }
        if (lane == 0) {
            A.sweeps[ci] = sweeps;
            A.ops[ci] = ops;
            A.pushes[ci] = pushes;
            A.conv[ci] = conv;
        }
        __syncwarp();
    }
}

// The same column solves in exact windows (window.cuh): one CTA per column at
// a time, persistent over the columns.
struct FwArgs {
    DevGraph g;
    DevOp op;
    double x_gain, omega;
    int64_t n, ncols, max_sweeps;
    double *p, *r;
    int32_t *queue;   // per CTA: n + 2
    uint32_t *qmark;  // per CTA: qw words
    int64_t qw;
    unsigned long long *next_col;
    int64_t *sweeps, *ops, *pushes;
    int32_t *conv;
};

__global__ void __launch_bounds__(win::WT, 1) k_feature_win(FwArgs A) {
    extern __shared__ __align__(16) unsigned char smraw[];
    win::Smem &S = *reinterpret_cast<win::Smem *>(smraw);
    __shared__ long long sh_col;
    __shared__ int64_t sh_sweeps, sh_ops;
    __shared__ int sh_done, sh_conv;
    win::init_smem(S);
    const int64_t qcap = A.n + 2;
    win::Sys Y{A.g, A.op, nullptr, nullptr, A.queue + (int64_t)blockIdx.x * qcap,
               A.qmark + (int64_t)blockIdx.x * A.qw, qcap, A.omega, A.x_gain, 1, 0};
    for (;;) {
        if (threadIdx.x == 0) sh_col = (long long)atomicAdd(A.next_col, 1ULL);
        __syncthreads();
        const int64_t ci = sh_col;
        if (ci >= A.ncols) break;
        Y.x = A.p + ci * A.n;
        Y.r = A.r + ci * A.n;
        // seeds = flatnonzero(|r| >= theta), enqueued in order (dynamic.py:141)
        const int64_t cnt = win::scan_enqueue(Y, S, A.n);
        if (threadIdx.x == 0) {
            S.front = 0;
            S.svol = S.pushes = 0;
            sh_sweeps = sh_ops = 0;
            sh_conv = 1;
            sh_done = cnt == 0;
            S.sentpos = cnt;
            S.rear = cnt + 1;
        }
        __syncthreads();
        while (!sh_done) {
            win::run_sweep(Y, S);
            if (threadIdx.x == 0) {
                sh_ops += S.svol;
                sh_sweeps += 1;
                S.front = S.sentpos + 1 == qcap ? 0 : S.sentpos + 1;
                if (S.front == S.rear) {
                    sh_done = 1;
                } else if (sh_sweeps >= A.max_sweeps) {
                    sh_conv = 0;
                    sh_done = 1;
                } else {
                    S.sentpos = S.rear;
                    S.rear = S.rear + 1 == qcap ? 0 : S.rear + 1;
                    S.svol = 0;
                }
            }
            __syncthreads();
        }
        if (!sh_conv)  // marks of the nodes still queued
            for (int64_t w = threadIdx.x; w < A.qw; w += win::WT) Y.qmark[w] = 0u;
        if (threadIdx.x == 0) {
            A.sweeps[ci] = sh_sweeps;
            A.ops[ci] = sh_ops;
            A.pushes[ci] = S.pushes;
            A.conv[ci] = sh_conv;
        }
        __syncthreads();
    }
}

// out (cols x rows) = in (rows x cols)^T, 32 x 32 tiles through shared memory.
__global__ void k_transpose(const double *__restrict__ in, double *__restrict__ out, int64_t rows,
                            int64_t cols) {
    __shared__ double tile[32][33];
    const int64_t tr = (rows + 31) / 32;  // tiles flattened into grid.x
    const int64_t r0 = ((int64_t)blockIdx.x % tr) * 32, c0 = ((int64_t)blockIdx.x / tr) * 32;
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int64_t rr = r0 + i, cc = c0 + threadIdx.x;
        if (rr < rows && cc < cols) tile[i][threadIdx.x] = in[rr * cols + cc];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int64_t cc = c0 + i, rr = r0 + threadIdx.x;
        if (rr < rows && cc < cols) out[cc * rows + rr] = tile[threadIdx.x][i];
    }
}

void transpose(const double *in, double *out, int64_t rows, int64_t cols) {
    const int64_t tiles = ((rows + 31) / 32) * ((cols + 31) / 32);
    k_transpose<<<(unsigned)tiles, dim3(32, 8)>>>(in, out, rows, cols);
    GD_LAUNCH_CHECK();
}

}  // namespace
}  // namespace gd

using namespace gd;

// Columns c = 0..ncols-1 of the host source matrix (n x ncols, row-major: the
// feature-matrix layout; transposed on the device so each column is
// contiguous while it is pushed)
// are pushed independently; p and r come back in the same layout.  arc_w /
// theta: the operator of beta_push (per arc / per node, host arrays).
extern "C" int gd_feature_push(const gd_graph *G, const double *arc_w, const double *theta,
                               double x_gain, double omega, int64_t ncols, const double *source,
                               int64_t max_sweeps, double *p_out, double *r_out, int64_t *sweeps,
                               int64_t *total_ops, int64_t *pushes, int32_t *converged) {
    return guarded([&] {
        GD_CHECK_ARG(G && arc_w && theta && source && p_out && r_out, "null pointer");
        GD_CHECK_ARG(ncols >= 0, "ncols must be >= 0");
        GD_CHECK_ARG(omega > 0.0 && omega <= 2.0, "omega must be in (0, 2]");
        GD_CUDA(cudaSetDevice(G->device));
        const int64_t n = G->n;
        if (ncols == 0 || n == 0) return;
        const size_t nc = (size_t)n * (size_t)ncols;
        DBuf<double> aw(G->n_arcs ? G->n_arcs : 1), th(n), p(nc), r(nc);
        GD_CUDA(cudaMemcpy(aw.p, arc_w, sizeof(double) * G->n_arcs, cudaMemcpyHostToDevice));
        GD_CUDA(cudaMemcpy(th.p, theta, sizeof(double) * n, cudaMemcpyHostToDevice));
        {
            DBuf<double> rowm(nc);
            GD_CUDA(cudaMemcpy(rowm.p, source, sizeof(double) * nc, cudaMemcpyHostToDevice));
            transpose(rowm.p, r.p, n, ncols);  // (n x C) -> (C x n)
        }
        GD_CUDA(cudaMemset(p.p, 0, sizeof(double) * nc));
        size_t fr = 0, tot = 0;
        GD_CUDA(cudaMemGetInfo(&fr, &tot));
        const int64_t qw = n / 32 + 1;
        const int64_t per = 4 * (n + 2) + 4 * qw;
        DBuf<int64_t> d_sw(ncols), d_ops(ncols), d_pu(ncols);
        DBuf<int32_t> d_cv(ncols);
        DBuf<unsigned long long> ctr(1);
        GD_CUDA(cudaMemset(ctr.p, 0, sizeof(unsigned long long)));
        static const bool warp_chain = [] {
            const char *e = getenv("GDIFF_FIFO");
            return e && e[0] == 'w';
        }();
        if (!warp_chain) {  // one CTA per column at a time
            int64_t nb = ncols < n_sms(G->device) ? ncols : n_sms(G->device);
            if (nb > (int64_t)(fr / 4) / per) nb = (int64_t)(fr / 4) / per;
            if (nb < 1) nb = 1;
            DBuf<int32_t> queue((size_t)nb * (n + 2));
            DBuf<uint32_t> qmark((size_t)nb * qw);
            GD_CUDA(cudaMemset(qmark.p, 0, sizeof(uint32_t) * (size_t)nb * qw));
            FwArgs A{};
            A.g = G->view();
            A.op.wrule = GD_W_ARC;
            A.op.trule = GD_T_ARRAY;
            A.op.arc_w = aw.p;
            A.op.theta = th.p;
            A.x_gain = x_gain;
            A.omega = omega;
            A.n = n;
            A.ncols = ncols;
            A.max_sweeps = max_sweeps > 0 ? max_sweeps : 1000000;
            A.p = p.p;
            A.r = r.p;
            A.queue = queue.p;
            A.qmark = qmark.p;
            A.qw = qw;
            A.next_col = ctr.p;
            A.sweeps = d_sw.p;
            A.ops = d_ops.p;
            A.pushes = d_pu.p;
            A.conv = d_cv.p;
            static bool attr = false;
            if (!attr) {
                GD_CUDA(cudaFuncSetAttribute(k_feature_win, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(win::Smem)));
                attr = true;
            }
            k_feature_win<<<(int)nb, win::WT, sizeof(win::Smem)>>>(A);
            GD_LAUNCH_CHECK();
            GD_CUDA(cudaDeviceSynchronize());
        } else {  // one warp per column
            int64_t nw = ncols;
            const int64_t resident = (int64_t)n_sms(G->device) * 64;
            if (nw > resident) nw = resident;
            if (nw > (int64_t)(fr / 4) / per) nw = (int64_t)(fr / 4) / per;
            if (nw < 1) nw = 1;
            DBuf<int32_t> queue((size_t)nw * (n + 2));
            DBuf<uint32_t> qmark((size_t)nw * qw);
            GD_CUDA(cudaMemset(qmark.p, 0, sizeof(uint32_t) * (size_t)nw * qw));
            FpArgs A{};
            A.g = G->view();
            A.arc_w = aw.p;
            A.theta = th.p;
            A.x_gain = x_gain;
            A.omega = omega;
            A.n = n;
            A.ncols = ncols;
            A.max_sweeps = max_sweeps > 0 ? max_sweeps : 1000000;
            A.p = p.p;
            A.r = r.p;
            A.queue = queue.p;
            A.qmark = qmark.p;
            A.qw = qw;
            A.nwarps = (int)nw;
            A.next_col = ctr.p;
            A.sweeps = d_sw.p;
            A.ops = d_ops.p;
            A.pushes = d_pu.p;
            A.conv = d_cv.p;
            k_feature_push<<<(int)((nw * 32 + FP_THREADS - 1) / FP_THREADS), FP_THREADS>>>(A);
            GD_LAUNCH_CHECK();
            GD_CUDA(cudaDeviceSynchronize());
        }
        {
            DBuf<double> rowm(nc);
            transpose(p.p, rowm.p, ncols, n);
            GD_CUDA(cudaMemcpy(p_out, rowm.p, sizeof(double) * nc, cudaMemcpyDeviceToHost));
            transpose(r.p, rowm.p, ncols, n);
            GD_CUDA(cudaMemcpy(r_out, rowm.p, sizeof(double) * nc, cudaMemcpyDeviceToHost));
        }
        if (sweeps) GD_CUDA(cudaMemcpy(sweeps, d_sw.p, 8 * ncols, cudaMemcpyDeviceToHost));
        if (total_ops) GD_CUDA(cudaMemcpy(total_ops, d_ops.p, 8 * ncols, cudaMemcpyDeviceToHost));
        if (pushes) GD_CUDA(cudaMemcpy(pushes, d_pu.p, 8 * ncols, cudaMemcpyDeviceToHost));
        if (converged) GD_CUDA(cudaMemcpy(converged, d_cv.p, 4 * ncols, cudaMemcpyDeviceToHost));
    });
}
