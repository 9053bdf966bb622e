// fifo.cu -- exact FIFO push (LocalGS / LocalSOR / dynamic repair), one
// warp per system.  (The heat-kernel push runs as layered sweeps, hk.cu.)
//
// The reference kernels (_push_kernel src/local_solvers.py:48-188 and
// _hk_push_kernel :566-661) are sequential Gauss-Seidel pushes: every pop
// reads residuals written by the previous one, so a system is inherently a
// single chain.  The chain runs in one warp; what parallelises is the arc
// loop of each push: 32 lanes take 32 consecutive arcs of the row, and the
// activation test's ballot + popc gives every newly active neighbour its
// queue slot in CSR order, which keeps the FIFO (and thus every later pop,
// the sweep boundaries and all logs) identical to the reference.  At each
// sentinel the whole CTA rescans the residual for the l1/min logs, as the
// reference does (:127-132).
#include <memory>

#include "common.cuh"
#include "window.cuh"

namespace gd {
namespace {

constexpr int FIFO_THREADS = 1024;

struct FifoArgs {
    DevGraph g;
    DevOp op;
    int64_t dim;           // coordinates (n)
    double *x, *r;
    int32_t *queue;        // ring of dim + 2 slots
    uint32_t *qmark;       // queued-node bit map (dim / 32 + 1 words, L2/L1-resident)
    const int32_t *seeds;
    int64_t n_seeds;
    double omega, x_gain;
    int sgn;
    int64_t max_sweeps;
    // logs
    int64_t log_cap;
    int64_t *vol_log;
    double *gamma_log, *l1_log;
    int8_t *sign_log;
    int64_t *out;          // sweeps, total_ops, converged, pushes
    double *out_min;
};

__device__ __forceinline__ bool qm_test(const uint32_t *q, int64_t v) {
    return (q[v >> 5] >> (v & 31)) & 1u;
}

// Block-wide l1 / min over r[0, dim): fixed-shape, deterministic.
__device__ void block_l1_min(const FifoArgs &A, double *s_s, double *s_m, double &l1,
                             double &mn) {
    double s = 0.0, m = __longlong_as_double(0x7ff0000000000000LL);
    for (int64_t i = threadIdx.x; i < A.dim; i += FIFO_THREADS) {
        double v = A.r[i];
        s += fabs(v);
        m = v < m ? v : m;
    }
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        double mo = __shfl_xor_sync(0xffffffffu, m, o);
        m = mo < m ? mo : m;
    }
    int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_s[w] = s;
        s_m[w] = m;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double ts = 0.0, tm = __longlong_as_double(0x7ff0000000000000LL);
        for (int k = 0; k < FIFO_THREADS / 32; k++) {
            ts += s_s[k];
            tm = s_m[k] < tm ? s_m[k] : tm;
        }
        s_s[0] = ts;
        s_m[0] = tm;
    }
    __syncthreads();
    l1 = s_s[0];
    mn = s_m[0];
    __syncthreads();
}

// One warp runs the pop chain; at each sentinel the whole block rescans r
// for the l1 / min logs (:127-132).  Per pop the next queue entry's r, x,
// degree, row and first 32 neighbours are prefetched while the current pop
// scatters (r is re-read if the scatter touched it; x is written only by a
// node's own pops), and each arc's r / mark / threshold loads issue together.
__global__ void __launch_bounds__(FIFO_THREADS, 1) k_fifo(FifoArgs A) {
    __shared__ double s_s[32], s_m[32];
    __shared__ int64_t sh_front, sh_rear, sh_sweeps, sh_ops, sh_pushes, sh_svol;
    __shared__ double sh_sgamma, sh_l1, sh_min;
    __shared__ int sh_pos, sh_neg, sh_cmd, sh_conv;
    const int64_t sent = A.dim, qcap = A.dim + 2;
    const int lane = threadIdx.x & 31;
    const bool w0 = threadIdx.x < 32;
    const unsigned FULLM = 0xffffffffu;

    if (threadIdx.x == 0) {  // seed enqueue, sequential (:59-69)
        int64_t rear = 0;
        for (int64_t i = 0; i < A.n_seeds; i++) {
            int32_t u = A.seeds[i];
            bool act = is_active(A.r[u], theta_of(A.op, u, A.g.deg[u]), A.sgn);
            if (act && !qm_test(A.qmark, u)) {
                A.queue[rear] = u;
                rear = (rear + 1) % qcap;
                A.qmark[u >> 5] |= 1u << (u & 31);
            }
        }
        sh_front = 0;
        sh_rear = rear;
        sh_sweeps = sh_ops = sh_pushes = sh_svol = 0;
        sh_sgamma = 0.0;
        sh_pos = sh_neg = 0;
        sh_conv = 1;
    }
    __syncthreads();
    double l1, mn;
    block_l1_min(A, s_s, s_m, l1, mn);
    if (threadIdx.x == 0) {
        sh_l1 = l1;
        sh_min = mn;
        A.l1_log[0] = l1;
        sh_cmd = (sh_front == sh_rear) ? 2 : 0;
        if (sh_cmd == 0) {
            A.queue[sh_rear] = (int32_t)sent;
            sh_rear = (sh_rear + 1) % qcap;
        }
    }
    __syncthreads();

    while (sh_cmd != 2) {
        if (w0) {
            int64_t front = sh_front, rear = sh_rear, svol = sh_svol, pushes = sh_pushes;
            double sgamma = sh_sgamma;
            int pos = sh_pos, neg = sh_neg;
            int64_t pu = -1, prs = 0;
            double pr = 0.0, px = 0.0;
            int32_t pd = 0, pcol = 0;
            for (;;) {
                const int64_t u = A.queue[front];
                front = (front + 1 == qcap) ? 0 : front + 1;
                if (u == sent) break;
                double ru, xu;
                int32_t d, c0;
                int64_t rs;
                if (u == pu) {
                    ru = pr;
                    d = pd;
                    rs = prs;
                    c0 = pcol;
                    xu = px;
                } else {
                    ru = A.r[u];
                    d = A.g.deg[u];
                    rs = A.g.row[u];
                    c0 = lane < d ? A.g.col[rs + lane] : 0;
                    xu = A.x[u];
                }
                pu = -1;
                if (lane == 0) atomicAnd(A.qmark + (u >> 5), ~(1u << (u & 31)));
                const double th = theta_of(A.op, u, d);
                if (!is_active(ru, th, A.sgn)) {
                    __syncwarp();
                    continue;
                }
                if (front != rear) {  // prefetch the next pop
                    const int64_t nx = A.queue[front];
                    if (nx != sent) {
                        pu = nx;
                        pr = A.r[nx];
                        pd = A.g.deg[nx];
                        prs = A.g.row[nx];
                        px = A.x[nx];
                        pcol = lane < pd ? A.g.col[prs + lane] : 0;
                    }
                }
                svol += d;
                sgamma += fabs(ru);
                pushes += 1;
                if (ru > 0.0) pos = 1;
                else if (ru < 0.0) neg = 1;
                const double res = __dmul_rn(A.omega, ru);
                if (lane == 0) {
                    A.x[u] = __dadd_rn(xu, __dmul_rn(A.x_gain, res));
                    A.r[u] = __dsub_rn(ru, res);
                }
                const double wn = node_weight(A.op, d);
                bool hit = false;
                for (int64_t base = 0; base < d; base += 32) {
                    const int64_t j = base + lane;
                    bool act = false;
                    int32_t t = 0;
                    if (j < d) {
                        t = base == 0 ? c0 : A.g.col[rs + j];
                        // the arc's loads, issued together
                        const double old = A.r[t];
                        const uint32_t qm = A.qmark[t >> 5];
                        const double tht = theta_of(A.op, t, A.g.deg[t]);
                        const double w = arc_weight(A.op, wn, rs + j);
                        const double rv = __dadd_rn(old, __dmul_rn(res, w));
                        A.r[t] = rv;
                        hit |= t == pu;
                        act = !((qm >> (t & 31)) & 1u) && is_active(rv, tht, A.sgn);
                    }
                    const unsigned bal = __ballot_sync(FULLM, act);
                    if (act) {
                        int64_t slot = rear + __popc(bal & ((1u << lane) - 1u));
                        if (slot >= qcap) slot -= qcap;
                        A.queue[slot] = t;
                        atomicOr(A.qmark + (t >> 5), 1u << (t & 31));
                    }
                    rear += __popc(bal);
                    if (rear >= qcap) rear -= qcap;
                }
                __syncwarp();
                if (__any_sync(FULLM, hit)) pr = A.r[pu];  // the scatter changed the next pop's r
                // self re-check (:176-185); the mark of u was cleared at pop
                const double ru2 = __dsub_rn(ru, res);
                if (is_active(ru2, th, A.sgn)) {
                    if (lane == 0) {
                        A.queue[rear] = (int32_t)u;
                        atomicOr(A.qmark + (u >> 5), 1u << (u & 31));
                    }
                    rear = (rear + 1 == qcap) ? 0 : rear + 1;
                }
                __syncwarp();
            }
            if (lane == 0) {  // sentinel: close the sweep (:102-126)
                int64_t t = sh_sweeps;
                if (t < A.log_cap) {
                    A.vol_log[t] = svol;
                    A.gamma_log[t] = sh_l1 > 0.0 ? sgamma / sh_l1 : 0.0;
                    A.sign_log[t] = (pos && neg) ? 2 : pos ? 1 : neg ? -1 : 0;
                }
                sh_ops += svol;
                sh_sweeps = t + 1;
                sh_front = front;
                sh_rear = rear;
                sh_pushes = pushes;
            }
        }
        __syncthreads();
        block_l1_min(A, s_s, s_m, l1, mn);
        if (threadIdx.x == 0) {
            int64_t t = sh_sweeps;
            if (t < A.log_cap) A.l1_log[t] = l1;
            sh_l1 = l1;
            if (mn < sh_min) sh_min = mn;
            if (sh_front == sh_rear) {
                sh_cmd = 2;
            } else if (t >= A.max_sweeps) {
                sh_conv = 0;
                sh_cmd = 2;
            } else {
                A.queue[sh_rear] = (int32_t)sent;
                sh_rear = (sh_rear + 1) % qcap;
                sh_svol = 0;
                sh_sgamma = 0.0;
                sh_pos = sh_neg = 0;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        A.out[0] = sh_sweeps;
        A.out[1] = sh_ops;
        A.out[2] = sh_conv;
        A.out[3] = sh_pushes;
        A.out_min[0] = sh_min;
    }
}

// The same solve with the pops taken in exact windows (window.cuh): one CTA,
// the sentinel / log handling of k_fifo around win::run_sweep.
__global__ void __launch_bounds__(FIFO_THREADS, 1) k_fifo_win(FifoArgs A) {
    extern __shared__ __align__(16) unsigned char smraw[];
    win::Smem &S = *reinterpret_cast<win::Smem *>(smraw);
    __shared__ double s_s[32], s_m[32];
    __shared__ double sh_l1, sh_min;
    __shared__ int64_t sh_sweeps, sh_ops;
    __shared__ int sh_cmd, sh_conv;
    static_assert(win::WT == FIFO_THREADS, "one CTA shape");
    const win::Sys Y{A.g, A.op, A.x, A.r, A.queue, A.qmark, A.dim + 2, A.omega, A.x_gain, A.sgn, 1};
    win::init_smem(S);
    if (threadIdx.x == 0) {  // seed enqueue, sequential (:59-69)
        int64_t rear = 0;
        for (int64_t i = 0; i < A.n_seeds; i++) {
            int32_t u = A.seeds[i];
            bool act = is_active(A.r[u], theta_of(A.op, u, A.g.deg[u]), A.sgn);
            if (act && !qm_test(A.qmark, u)) {
                A.queue[rear] = u;
                rear = rear + 1;
                A.qmark[u >> 5] |= 1u << (u & 31);
            }
        }
        S.front = 0;
        S.rear = rear;
        S.svol = S.pushes = 0;
        S.sgamma = 0.0;
        S.pos = S.neg = 0;
        sh_sweeps = sh_ops = 0;
        sh_conv = 1;
    }
    __syncthreads();
    double l1, mn;
    block_l1_min(A, s_s, s_m, l1, mn);
    if (threadIdx.x == 0) {
        sh_l1 = l1;
        sh_min = mn;
        A.l1_log[0] = l1;
        sh_cmd = (S.front == S.rear) ? 2 : 0;
        if (sh_cmd == 0) {
            S.sentpos = S.rear;
            S.rear = S.rear + 1;
        }
    }
    __syncthreads();
    const int64_t qcap = A.dim + 2;
    while (sh_cmd != 2) {
        win::run_sweep(Y, S);
        if (threadIdx.x == 0) {  // the sentinel: close the sweep (:102-126)
            const int64_t t = sh_sweeps;
            if (t < A.log_cap) {
                A.vol_log[t] = S.svol;
                A.gamma_log[t] = sh_l1 > 0.0 ? S.sgamma / sh_l1 : 0.0;
                A.sign_log[t] = (S.pos && S.neg) ? 2 : S.pos ? 1 : S.neg ? -1 : 0;
            }
            sh_ops += S.svol;
            sh_sweeps = t + 1;
            S.front = S.sentpos + 1 == qcap ? 0 : S.sentpos + 1;
        }
        __syncthreads();
        block_l1_min(A, s_s, s_m, l1, mn);
        if (threadIdx.x == 0) {
            const int64_t t = sh_sweeps;
            if (t < A.log_cap) A.l1_log[t] = l1;
            sh_l1 = l1;
            if (mn < sh_min) sh_min = mn;
            if (S.front == S.rear) {
                sh_cmd = 2;
            } else if (t >= A.max_sweeps) {
                sh_conv = 0;
                sh_cmd = 2;
            } else {
                S.sentpos = S.rear;
                S.rear = S.rear + 1 == qcap ? 0 : S.rear + 1;
                S.svol = 0;
                S.sgamma = 0.0;
                S.pos = S.neg = 0;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        A.out[0] = sh_sweeps;
        A.out[1] = sh_ops;
        A.out[2] = sh_conv;
        A.out[3] = S.pushes;
        A.out_min[0] = sh_min;
#ifdef GD_WIN_PROF
        printf("wprof windows=%llu", win::g_wprof[31]);
        for (int i = 0; i < 12; i++) printf(" p%d=%.1fus", i, win::g_wprof[i] / 1.9e3);
        printf("\n  windows=%llu pops/win=%.1f conflict=%llu arcbudget=%llu slice/win=%.1f arcs/win=%.1f sweepend=%llu big=%llu\n",
               win::g_wprof[20], (double)win::g_wprof[21] / win::g_wprof[20], win::g_wprof[22], win::g_wprof[23],
               (double)win::g_wprof[24] / win::g_wprof[20], (double)win::g_wprof[25] / win::g_wprof[20], win::g_wprof[26], win::g_wprof[27]);
        for (int i = 0; i < 32; i++) win::g_wprof[i] = 0;
#endif
    }
}

// Device buffers of a FIFO solve, kept across calls on the host thread.
struct FifoWS {
    DBuf<double> x, r, gam, l1, mn;
    DBuf<int32_t> queue, sd;
    DBuf<uint32_t> qmark;
    DBuf<int64_t> vol, out;
    DBuf<int8_t> sgn;
};

void run_fifo(const gd_graph *G, FifoArgs A, double *hx, double *hr,
              const int64_t *seeds, int64_t n_seeds, gd_report *rep) {
    const int64_t dim = A.dim;
    GD_CHECK_ARG(dim + 2 < (1LL << 31), "coordinate count must be < 2^31");
    thread_local std::unique_ptr<FifoWS> ws;
    if (!ws) ws.reset(new FifoWS());
    FifoWS &W = *ws;
    int64_t log_cap = A.max_sweeps < (1 << 20) ? A.max_sweeps + 1 : (1 << 20);
    W.x.ensure(dim ? dim : 1); W.r.ensure(dim ? dim : 1); W.queue.ensure(dim + 2);
    W.sd.ensure(n_seeds ? n_seeds : 1); W.qmark.ensure(dim / 32 + 1);
    W.vol.ensure(log_cap); W.out.ensure(4); W.gam.ensure(log_cap); W.l1.ensure(log_cap + 1);
    W.mn.ensure(1); W.sgn.ensure(log_cap);
    auto &x = W.x, &r = W.r, &gam = W.gam, &l1 = W.l1, &mn = W.mn;
    auto &queue = W.queue, &sd = W.sd;
    auto &qmark = W.qmark;
    auto &vol = W.vol, &out = W.out;
    auto &sgn = W.sgn;
    GD_CUDA(cudaMemcpy(x.p, hx, sizeof(double) * dim, cudaMemcpyHostToDevice));
    GD_CUDA(cudaMemcpy(r.p, hr, sizeof(double) * dim, cudaMemcpyHostToDevice));
    GD_CUDA(cudaMemset(qmark.p, 0, sizeof(uint32_t) * (dim / 32 + 1)));
    std::vector<int32_t> s32(n_seeds);
    for (int64_t i = 0; i < n_seeds; i++) {
        GD_CHECK_ARG(seeds[i] >= 0 && seeds[i] < dim, "seed out of range");
        s32[i] = (int32_t)seeds[i];
    }
    if (n_seeds)
        GD_CUDA(cudaMemcpy(sd.p, s32.data(), sizeof(int32_t) * n_seeds, cudaMemcpyHostToDevice));
    A.x = x.p; A.r = r.p; A.queue = queue.p; A.qmark = qmark.p; A.seeds = sd.p;
    A.n_seeds = n_seeds; A.log_cap = log_cap; A.vol_log = vol.p; A.gamma_log = gam.p;
    A.l1_log = l1.p; A.sign_log = sgn.p; A.out = out.p; A.out_min = mn.p;
    static const bool warp_chain = [] {
        const char *e = getenv("GDIFF_FIFO");
        return e && e[0] == 'w';
    }();
    if (warp_chain) {
        k_fifo<<<1, FIFO_THREADS>>>(A);
    } else {
        static bool attr = false;
        if (!attr) {
            GD_CUDA(cudaFuncSetAttribute(k_fifo_win, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(win::Smem)));
            attr = true;
        }
        k_fifo_win<<<1, FIFO_THREADS, sizeof(win::Smem)>>>(A);
    }
    GD_LAUNCH_CHECK();
    GD_CUDA(cudaDeviceSynchronize());
    int64_t o[4];
    GD_CUDA(cudaMemcpy(o, out.p, sizeof(o), cudaMemcpyDeviceToHost));
    int64_t cap = 64;
    report_alloc(rep, cap);
    int64_t nl = o[0] < log_cap ? o[0] : log_cap;
    std::vector<int64_t> hv(nl);
    std::vector<double> hg(nl), hl(nl + 1);
    std::vector<int8_t> hs(nl);
    if (nl) {
        GD_CUDA(cudaMemcpy(hv.data(), vol.p, sizeof(int64_t) * nl, cudaMemcpyDeviceToHost));
        GD_CUDA(cudaMemcpy(hg.data(), gam.p, sizeof(double) * nl, cudaMemcpyDeviceToHost));
        GD_CUDA(cudaMemcpy(hs.data(), sgn.p, nl, cudaMemcpyDeviceToHost));
    }
    GD_CUDA(cudaMemcpy(hl.data(), l1.p, sizeof(double) * (nl + 1), cudaMemcpyDeviceToHost));
    rep->l1_log[0] = hl[0];
    for (int64_t t = 0; t < nl; t++) report_push_log(rep, cap, hv[t], hg[t], hl[t + 1], hs[t], 0);
    rep->sweeps = o[0];
    rep->total_ops = o[1];
    rep->converged = (int32_t)o[2];
    rep->pushes = o[3];
    GD_CUDA(cudaMemcpy(&rep->min_residual, mn.p, sizeof(double), cudaMemcpyDeviceToHost));
    GD_CUDA(cudaMemcpy(hx, x.p, sizeof(double) * dim, cudaMemcpyDeviceToHost));
    GD_CUDA(cudaMemcpy(hr, r.p, sizeof(double) * dim, cudaMemcpyDeviceToHost));
    int64_t nz = 0;
    for (int64_t i = 0; i < dim; i++) nz += (hr[i] != 0.0);
    rep->support_size = nz;
}

}  // namespace
}  // namespace gd

using namespace gd;

extern "C" {

int gd_push_kernel(const gd_graph *G, const gd_operator *o, double *x, double *r,
                   const int64_t *seeds, int64_t n_seeds, double omega, double x_gain,
                   int32_t is_signed, int64_t max_sweeps, gd_report *rep) {
    return guarded([&] {
        GD_CHECK_ARG(G && o && x && r && rep && (seeds || n_seeds == 0), "null pointer");
        GD_CUDA(cudaSetDevice(G->device));
        HostOp op;
        upload_op(G, o, G->n, op, 0);
        FifoArgs A{};
        A.g = G->view();
        A.op = op.dev;
        A.dim = G->n;
        A.omega = omega;
        A.x_gain = x_gain;
        A.sgn = is_signed ? 1 : 0;
        A.max_sweeps = max_sweeps;
        run_fifo(G, A, x, r, seeds, n_seeds, rep);
    });
}

}  // extern "C"
