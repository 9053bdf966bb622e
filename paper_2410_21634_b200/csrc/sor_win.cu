// sor_win.cu -- batched LocalSOR / LocalGS-PPR in exact windows, one CTA per seed.
//
// Per seed s the run is local_sor(make_ppr_system(g, alpha, s, eps), omega)
// (src/local_solvers.py:191-259): _push_kernel from x = 0, r = alpha e_s,
// queue = [s] -- bit-identical, like fifo_batch.cu's warp-per-seed chain.
// Here the chain runs in window.cuh's exact windows (a CTA pops up to 128
// queued nodes at once, cut at the first forward conflict, ordered per-node
// folds, the reference's enqueue order), so one seed's pops overlap their
// memory round trips instead of paying them one pop at a time.  Persistent
// CTAs (one per SM: the window tables take ~210 KB of shared memory) pull
// seeds from a counter; a CTA's slot is a dense x / r pair, scanned once at
// the end of the seed (x != 0 -> output, caller ids are the graph's: the FIFO
// replay needs the caller's CSR order, no relabel) and returned to zero.
#include "common.cuh"
#include "window.cuh"

namespace gd {
namespace {

struct SwArgs {
    DevGraph g;
    DevOp op;
    double alpha, omega;
    int64_t n, ld, max_sweeps, qw;
    double *x, *r;        // per CTA: ld
    int32_t *queue;       // per CTA: n + 2
    uint32_t *qmark;      // per CTA: qw words
    const int64_t *seeds;
    int64_t n_seeds;
    unsigned long long *next_seed, *cursor;
    int64_t *sweeps, *ops, *pushes, *xoff, *xcnt;
    int32_t *conv, *xnodes;
    double *xvals;
    int64_t xcap;
};

__global__ void __launch_bounds__(win::WT, 1) k_sor_win(SwArgs A) {
    extern __shared__ __align__(16) unsigned char smraw[];
    win::Smem &S = *reinterpret_cast<win::Smem *>(smraw);
    __shared__ long long sh_seed;
    __shared__ int64_t sh_sweeps, sh_ops, sh_base;
    __shared__ int sh_done, sh_conv;
    __shared__ int sh_wc[win::WT / 32];
    win::init_smem(S);
    const int64_t qcap = A.n + 2;
    double *const x = A.x + (int64_t)blockIdx.x * A.ld;
    double *const r = A.r + (int64_t)blockIdx.x * A.ld;
    win::Sys Y{A.g, A.op, x, r, A.queue + (int64_t)blockIdx.x * qcap,
               A.qmark + (int64_t)blockIdx.x * A.qw, qcap, A.omega, 1.0, A.omega > 1.0 ? 1 : 0, 0};
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    for (;;) {
        if (t == 0) sh_seed = (long long)atomicAdd(A.next_seed, 1ULL);
        __syncthreads();
        const int64_t si = sh_seed;
        if (si >= A.n_seeds) break;
        const int32_t s = (int32_t)A.seeds[si];
        if (t == 0) {
            r[s] = A.alpha;
            const bool act = is_active(A.alpha, theta_of(A.op, s, A.g.deg[s]), Y.sgn);
            if (act) {
                Y.queue[0] = s;
                Y.qmark[s >> 5] |= 1u << (s & 31);
            }
            S.front = 0;
            S.svol = S.pushes = 0;
            sh_sweeps = sh_ops = 0;
            sh_conv = 1;
            sh_done = act ? 0 : 1;
            S.sentpos = act ? 1 : 0;
            S.rear = act ? 2 : 1;
            if (act) Y.queue[1] = (int32_t)A.n;  // the sweep's sentinel
        }
        __syncthreads();
        while (!sh_done) {
            win::run_sweep(Y, S);
            if (t == 0) {
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
            for (int64_t w = t; w < A.qw; w += win::WT) Y.qmark[w] = 0u;
        // x out: nonzero entries in node order; x and r back to zero
        int mine = 0;
        for (int64_t u = t; u < A.n; u += win::WT) mine += __double_as_longlong(x[u]) != 0;
        mine = __reduce_add_sync(0xffffffffu, mine);
        if (lane == 0) sh_wc[wid] = mine;
        __syncthreads();
        if (t == 0) {
            int tot = 0;
            for (int w = 0; w < win::WT / 32; ++w) tot += sh_wc[w];
            sh_base = (int64_t)atomicAdd(A.cursor, (unsigned long long)tot);
            A.sweeps[si] = sh_sweeps;
            A.ops[si] = sh_ops;
            A.pushes[si] = S.pushes;
            A.conv[si] = sh_conv;
            A.xcnt[si] = tot;
            A.xoff[si] = sh_base;
        }
        __syncthreads();
        int64_t pos = sh_base;
        for (int64_t b0 = 0; b0 < A.n; b0 += win::WT) {
            const int64_t u = b0 + t;
            double xv = 0.0;
            if (u < A.n) {
                xv = x[u];
                r[u] = 0.0;
            }
            const bool nz = __double_as_longlong(xv) != 0;
            const unsigned bal = __ballot_sync(0xffffffffu, nz);
            if (lane == 0) sh_wc[wid] = __popc(bal);
            __syncthreads();
            int off = 0, tot = 0;
            for (int w = 0; w < win::WT / 32; ++w) {
                const int c = sh_wc[w];
                off += w < wid ? c : 0;
                tot += c;
            }
            if (nz) {
                const int64_t p = pos + off + __popc(bal & win::lanemask_lt());
                if (p < A.xcap) {
                    A.xnodes[p] = (int32_t)u;
                    A.xvals[p] = xv;
                }
                x[u] = 0.0;
            }
            pos += tot;
            __syncthreads();
        }
    }
}

}  // namespace

struct SorWinState {
    int ctas = 0;
    int64_t ld = 0, qw = 0;
    DBuf<double> x, r;
    DBuf<int32_t> queue;
    DBuf<uint32_t> qmark;
    DBuf<unsigned long long> next;
};

SorWinState *sorwin_create(const gd_graph *G, int max_ctas) {
    SorWinState *W = new SorWinState();
    try {
        GD_CUDA(cudaFuncSetAttribute(k_sor_win, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(win::Smem)));
        int per_sm = 0;
        GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sor_win, win::WT,
                                                              sizeof(win::Smem)));
        GD_CHECK_ARG(per_sm > 0, "window kernel does not fit on an SM");
        int ctas = per_sm * n_sms(G->device);
        if (max_ctas > 0 && max_ctas < ctas) ctas = max_ctas;
        const int64_t n = G->n ? G->n : 1;
        W->ctas = ctas;
        W->ld = (n + 1) & ~1LL;
        W->qw = (n + 31) / 32;
        const size_t sn = (size_t)ctas * (size_t)W->ld;
        W->x.alloc(sn);
        W->r.alloc(sn);
        GD_CUDA(cudaMemset(W->x.p, 0, sizeof(double) * sn));
        GD_CUDA(cudaMemset(W->r.p, 0, sizeof(double) * sn));
        W->queue.alloc((size_t)ctas * (size_t)(n + 2));
        W->qmark.alloc((size_t)ctas * (size_t)W->qw);
        GD_CUDA(cudaMemset(W->qmark.p, 0, sizeof(uint32_t) * (size_t)ctas * (size_t)W->qw));
        W->next.alloc(1);
    } catch (...) {
        delete W;
        throw;
    }
    return W;
}

void sorwin_destroy(SorWinState *W) { delete W; }

void sorwin_run(SorWinState *W, const gd_graph *G, const gd_batch_params &p,
                const int64_t *d_seeds, int64_t n_seeds, int64_t *sweeps, int64_t *ops,
                int64_t *pushes, int32_t *conv, int64_t *xoff, int64_t *xcnt, int32_t *xnodes,
                double *xvals, int64_t xcap, unsigned long long *cursor, cudaStream_t st) {
    if (n_seeds == 0) return;
    SwArgs A{};
    A.g = G->view();
    A.op = DevOp{GD_W_RW, GD_T_DEGREE, 1.0 - p.alpha, p.eps * p.alpha, nullptr, nullptr};
    A.alpha = p.alpha;
    A.omega = p.omega;
    A.n = G->n;
    A.ld = W->ld;
    A.max_sweeps = p.max_sweeps > 0 ? p.max_sweeps : 1000000;
    A.qw = W->qw;
    A.x = W->x.p; A.r = W->r.p; A.queue = W->queue.p; A.qmark = W->qmark.p;
    A.seeds = d_seeds; A.n_seeds = n_seeds;
    A.next_seed = W->next.p; A.cursor = cursor;
    A.sweeps = sweeps; A.ops = ops; A.pushes = pushes; A.xoff = xoff; A.xcnt = xcnt;
    A.conv = conv; A.xnodes = xnodes; A.xvals = xvals; A.xcap = xcap;
    GD_CUDA(cudaMemsetAsync(W->next.p, 0, sizeof(unsigned long long), st));
    const int grid = (int)(n_seeds < W->ctas ? n_seeds : W->ctas);
    k_sor_win<<<grid, win::WT, sizeof(win::Smem), st>>>(A);
    GD_LAUNCH_CHECK();
}

}  // namespace gd
