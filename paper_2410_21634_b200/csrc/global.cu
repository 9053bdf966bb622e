// global.cu -- full-graph gradient descent (the "global GD on GPU" reference
// point of the north star), bit-exact with src/global_solvers.py:124-152.
//
// The reference scatter (_scatter_full :63-71) adds contributions to out[v]
// in ascending source order u.  The graph is symmetric and every row is
// sorted, so the *pull* form -- one thread per v folding over its sorted
// neighbour row -- performs the same additions in the same order without
// atomics: r_{t+1}[v] = fl(...fl(0 + fl(r_t[u1] w_u1)) + ...), u1 < u2 < ...
#include "common.cuh"

namespace gd {
namespace {

constexpr int TPB = 256;

__global__ void k_axpy(double *__restrict__ x, const double *__restrict__ r, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = __dadd_rn(x[i], r[i]);
}

__device__ __forceinline__ double pull_weight(const DevGraph &g, const DevOp &op, int32_t u,
                                              int64_t v) {
    if (op.wrule != GD_W_ARC) return node_weight(op, g.deg[u]);
    // weight of arc u -> v: locate v in u's sorted row
    int64_t lo = g.row[u], hi = g.row[u + 1];
    while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if (g.col[mid] <= v) lo = mid; else hi = mid;
    }
    return op.arc_w[lo];
}

// Ordered pull of row v by one warp: lanes form c_j = fl(src[u_j] w_j) for 32
// consecutive arcs (sources ascending: the reference's scatter order), lane 0
// adds the nonzero ones in order (zeros are skipped as _scatter_full does).
// Hub rows no longer serialise one thread for thousands of arcs.
__device__ __forceinline__ double warp_row_fold(const DevGraph &g, const DevOp &op,
                                                const double *__restrict__ src, int64_t v,
                                                int lane) {
    const int64_t rs = g.row[v], re = g.row[v + 1];
    double acc = 0.0;
    for (int64_t b = rs; b < re; b += 32) {
        const int64_t j = b + lane;
        double c = 0.0;
        bool nz = false;
        if (j < re) {
            const int32_t u = g.col[j];
            const double val = src[u];
            nz = val != 0.0;
            if (nz) c = __dmul_rn(val, pull_weight(g, op, u, v));
        }
        const unsigned m = __ballot_sync(0xffffffffu, nz);
        const int cnt = (int)min((int64_t)32, re - b);
        for (int l = 0; l < cnt; l++) {
            const double cl = __shfl_sync(0xffffffffu, c, l);
            if ((m >> l) & 1u) acc = __dadd_rn(acc, cl);
        }
    }
    return acc;  // (valid in every lane: all lanes run the same adds)
}

// r_next = beta P r (pull, warp per row), plus any-active flag and partial
// l1 / l2 sums.
__global__ void k_pull(DevGraph g, DevOp op, const double *__restrict__ r,
                       double *__restrict__ nxt, int *__restrict__ active,
                       double *__restrict__ part) {
    __shared__ double s1[TPB / 32], s2[TPB / 32];
    const int lane = threadIdx.x & 31;
    double a1 = 0.0, a2 = 0.0;
    int any = 0;
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < g.n;
         v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const double acc = warp_row_fold(g, op, r, v, lane);
        if (lane == 0) {
            nxt[v] = acc;
            a1 += fabs(acc);
            a2 += acc * acc;
            any |= acc >= theta_of(op, v, g.deg[v]);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    any = __any_sync(0xffffffffu, any);
    if (lane == 0) {
        s1[threadIdx.x >> 5] = a1;
        s2[threadIdx.x >> 5] = a2;
        if (any) atomicOr(active, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t1 = 0.0, t2 = 0.0;
        for (int k = 0; k < TPB / 32; k++) { t1 += s1[k]; t2 += s2[k]; }
        part[2 * blockIdx.x] = t1;
        part[2 * blockIdx.x + 1] = t2;
    }
}

__global__ void k_active0(DevGraph g, DevOp op, const double *__restrict__ r,
                          int *__restrict__ active, double *__restrict__ part) {
    double a1 = 0.0, a2 = 0.0;
    int any = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < g.n;
         v += (int64_t)gridDim.x * blockDim.x) {
        double val = r[v];
        a1 += fabs(val);
        a2 += val * val;
        any |= val >= theta_of(op, v, g.deg[v]);
    }
    __shared__ double s1[TPB / 32], s2[TPB / 32];
    for (int o = 16; o > 0; o >>= 1) {
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    any = __any_sync(0xffffffffu, any);
    if ((threadIdx.x & 31) == 0) {
        s1[threadIdx.x >> 5] = a1;
        s2[threadIdx.x >> 5] = a2;
        if (any) atomicOr(active, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t1 = 0.0, t2 = 0.0;
        for (int k = 0; k < TPB / 32; k++) { t1 += s1[k]; t2 += s2[k]; }
        part[2 * blockIdx.x] = t1;
        part[2 * blockIdx.x + 1] = t2;
    }
}

}  // namespace
}  // namespace gd

using namespace gd;

extern "C" int gd_gradient_descent(const gd_graph *G, const gd_operator *o, const double *b,
                                   double *hx, double *hr, int64_t max_sweeps, gd_report *rep) {
    return guarded([&] {
        GD_CHECK_ARG(G && o && b && hx && hr && rep, "null pointer");
        GD_CUDA(cudaSetDevice(G->device));
        HostOp op;
        upload_op(G, o, G->n, op, 0);
        const int64_t n = G->n;
        const int blocks = 16 * n_sms(G->device);  // (warp-per-row pulls)
        DevGraph g = G->view();
        DBuf<double> x(n ? n : 1), r(n ? n : 1), nx(n ? n : 1), part(2 * blocks);
        DBuf<int> act(1);
        GD_CUDA(cudaMemcpy(r.p, b, sizeof(double) * n, cudaMemcpyHostToDevice));
        GD_CUDA(cudaMemset(x.p, 0, sizeof(double) * (n ? n : 1)));
        std::vector<double> hp(2 * blocks);
        auto finish_sweep = [&](int *any, double *l1, double *l2) {
            GD_CUDA(cudaMemcpy(any, act.p, sizeof(int), cudaMemcpyDeviceToHost));
            GD_CUDA(cudaMemcpy(hp.data(), part.p, sizeof(double) * 2 * blocks,
                               cudaMemcpyDeviceToHost));
            double s1 = 0.0, s2 = 0.0;
            for (int k = 0; k < blocks; k++) { s1 += hp[2 * k]; s2 += hp[2 * k + 1]; }
            *l1 = s1;
            *l2 = sqrt(s2);
        };
        int64_t cap = 64;
        report_alloc(rep, cap);
        int any = 0;
        double l1, l2;
        GD_CUDA(cudaMemset(act.p, 0, sizeof(int)));
        k_active0<<<blocks, TPB>>>(g, op.dev, r.p, act.p, part.p);
        GD_LAUNCH_CHECK();
        finish_sweep(&any, &l1, &l2);
        rep->l1_log[0] = l1;
        rep->l2_log[0] = l2;
        const int64_t vol = G->n_arcs;
        while (any && rep->sweeps < max_sweeps) {
            k_axpy<<<blocks, TPB>>>(x.p, r.p, n);
            GD_CUDA(cudaMemset(act.p, 0, sizeof(int)));
            k_pull<<<blocks, TPB>>>(g, op.dev, r.p, nx.p, act.p, part.p);
            GD_LAUNCH_CHECK();
            std::swap(r.p, nx.p);
            finish_sweep(&any, &l1, &l2);
            report_push_log(rep, cap, vol, 0.0, l1, 0, 0);
            rep->l2_log[rep->n_logs] = l2;
            rep->sweeps += 1;
            rep->total_ops += vol;
        }
        rep->converged = any ? 0 : 1;
        GD_CUDA(cudaMemcpy(hx, x.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
        GD_CUDA(cudaMemcpy(hr, r.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
        int64_t nz = 0;
        for (int64_t i = 0; i < n; i++) nz += (hr[i] != 0.0);
        rep->support_size = nz;
    });
}

// ---------------------------------------------------------------------------
// Spectral norm estimate (Katz bounds): shifted power iteration on A + d_max I
// (src/graph.py:267-295), 200 SpMVs on the device instead of np.add.at on the
// host.  y = A x + d_max x (warp per row), lam = x.y, x <- y / ||y||.
// The dot products are tree reductions (the reference uses BLAS), so the
// estimate agrees to rounding, not bit for bit.
// ---------------------------------------------------------------------------
namespace gd {
namespace {

__global__ void k_shifted_spmv(DevGraph g, double dmax, const double *__restrict__ x,
                               double *__restrict__ y, double *__restrict__ part) {
    __shared__ double s1[TPB / 32], s2[TPB / 32];
    const int lane = threadIdx.x & 31;
    double dot = 0.0, nrm = 0.0;
    for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < g.n;
         u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        double acc = 0.0;
        for (int64_t j = g.row[u] + lane; j < g.row[u + 1]; j += 32) acc += x[g.col[j]];
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        const double yu = acc + dmax * x[u];
        if (lane == 0) {
            y[u] = yu;
            dot += x[u] * yu;
            nrm += yu * yu;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        dot += __shfl_xor_sync(0xffffffffu, dot, o);
        nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    }
    if (lane == 0) {
        s1[threadIdx.x >> 5] = dot;
        s2[threadIdx.x >> 5] = nrm;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int k = 0; k < TPB / 32; k++) { a += s1[k]; b += s2[k]; }
        part[2 * blockIdx.x] = a;
        part[2 * blockIdx.x + 1] = b;
    }
}

__global__ void k_scale(const double *__restrict__ y, double inv, double *__restrict__ x,
                        int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = y[i] * inv;
}

}  // namespace
}  // namespace gd

extern "C" int gd_spectral_norm(const gd_graph *G, const double *x0, int64_t iters,
                                double *lam_out) {
    using namespace gd;
    return guarded([&] {
        GD_CHECK_ARG(G && x0 && lam_out, "null pointer");
        GD_CHECK_ARG(iters >= 1, "iters must be >= 1");
        GD_CUDA(cudaSetDevice(G->device));
        const int64_t n = G->n;
        const double dmax = (double)G->d_max;
        if (n == 0 || dmax == 0.0) {
            *lam_out = 0.0;
            return;
        }
        const int blocks = 4 * n_sms(G->device);
        DBuf<double> x(n), y(n), part(2 * blocks);
        std::vector<double> hp(2 * blocks);
        GD_CUDA(cudaMemcpy(x.p, x0, sizeof(double) * n, cudaMemcpyHostToDevice));
        double lam = 0.0;
        for (int64_t it = 0; it < iters; ++it) {
            k_shifted_spmv<<<blocks, TPB>>>(G->view(), dmax, x.p, y.p, part.p);
            GD_LAUNCH_CHECK();
            GD_CUDA(cudaMemcpy(hp.data(), part.p, sizeof(double) * 2 * blocks,
                               cudaMemcpyDeviceToHost));
            double dot = 0.0, nrm2 = 0.0;
            for (int k = 0; k < blocks; k++) { dot += hp[2 * k]; nrm2 += hp[2 * k + 1]; }
            lam = dot;
            const double nrm = sqrt(nrm2);
            if (nrm == 0.0) break;
            k_scale<<<blocks, TPB>>>(y.p, 1.0 / nrm, x.p, n);
            GD_LAUNCH_CHECK();
        }
        *lam_out = (lam - dmax) < dmax ? (lam - dmax) : dmax;
    });
}

// ---------------------------------------------------------------------------
// Global Chebyshev (src/global_solvers.py:155-204) and the heat-kernel Taylor
// stages (:207-235), bit-exact: the same elementwise fl() sequence as the
// numpy expressions, and the scatter as the sorted-row pull (ascending source
// order, zeros skipped as _scatter_full does).
// ---------------------------------------------------------------------------
namespace gd {
namespace {

// out[v] = sum over u in N(v), ascending, of src[u] * w(u -> v); src[u] == 0 skipped
__global__ void k_pull_plain(DevGraph g, DevOp op, const double *__restrict__ src,
                             double *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < g.n;
         v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const double acc = warp_row_fold(g, op, src, v, lane);
        if (lane == 0) out[v] = acc;
    }
}

// inc = c0 r (first sweep) or fl(fl(c1 r) + fl(c2 prev)); x += inc
__global__ void k_cheb_inc(const double *__restrict__ r, const double *__restrict__ prev,
                           double *__restrict__ inc, double *__restrict__ x, int64_t n,
                           int first, double c0, double c1, double c2) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double v = first ? __dmul_rn(c0, r[i])
                               : __dadd_rn(__dmul_rn(c1, r[i]), __dmul_rn(c2, prev[i]));
        inc[i] = v;
        x[i] = __dadd_rn(x[i], v);
    }
}

// r += scat - inc; partial l1 / l2 sums and the signed activity flag
__global__ void k_cheb_r(DevGraph g, DevOp op, double *__restrict__ r,
                         const double *__restrict__ scat, const double *__restrict__ inc,
                         int *__restrict__ active, double *__restrict__ part) {
    __shared__ double s1[TPB / 32], s2[TPB / 32];
    double a1 = 0.0, a2 = 0.0;
    int any = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < g.n;
         v += (int64_t)gridDim.x * blockDim.x) {
        const double nv = __dadd_rn(r[v], __dsub_rn(scat[v], inc[v]));
        r[v] = nv;
        a1 += fabs(nv);
        a2 += nv * nv;
        any |= fabs(nv) >= theta_of(op, v, g.deg[v]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    any = __any_sync(0xffffffffu, any);
    if ((threadIdx.x & 31) == 0) {
        s1[threadIdx.x >> 5] = a1;
        s2[threadIdx.x >> 5] = a2;
        if (any) atomicOr(active, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t1 = 0.0, t2 = 0.0;
        for (int k = 0; k < TPB / 32; k++) { t1 += s1[k]; t2 += s2[k]; }
        part[2 * blockIdx.x] = t1;
        part[2 * blockIdx.x + 1] = t2;
    }
}

__global__ void k_active_signed(DevGraph g, DevOp op, const double *__restrict__ r,
                                int *__restrict__ active, double *__restrict__ part) {
    __shared__ double s1[TPB / 32], s2[TPB / 32];
    double a1 = 0.0, a2 = 0.0;
    int any = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < g.n;
         v += (int64_t)gridDim.x * blockDim.x) {
        const double val = r[v];
        a1 += fabs(val);
        a2 += val * val;
        any |= fabs(val) >= theta_of(op, v, g.deg[v]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    any = __any_sync(0xffffffffu, any);
    if ((threadIdx.x & 31) == 0) {
        s1[threadIdx.x >> 5] = a1;
        s2[threadIdx.x >> 5] = a2;
        if (any) atomicOr(active, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t1 = 0.0, t2 = 0.0;
        for (int k = 0; k < TPB / 32; k++) { t1 += s1[k]; t2 += s2[k]; }
        part[2 * blockIdx.x] = t1;
        part[2 * blockIdx.x + 1] = t2;
    }
}

__global__ void k_scale_into(const double *__restrict__ a, double w, double *__restrict__ o,
                             int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        o[i] = __dmul_rn(w, a[i]);
}

}  // namespace
}  // namespace gd

extern "C" int gd_chebyshev(const gd_graph *G, const gd_operator *o, const double *b, double *hx,
                            double *hr, double mu, double L, int64_t max_sweeps, gd_report *rep) {
    using namespace gd;
    return guarded([&] {
        GD_CHECK_ARG(G && o && b && hx && hr && rep, "null pointer");
        GD_CHECK_ARG(mu < L, "need mu < L");
        GD_CUDA(cudaSetDevice(G->device));
        HostOp op;
        upload_op(G, o, G->n, op, 0);
        const int64_t n = G->n;
        const size_t nn = n ? n : 1;
        const int blocks = 16 * n_sms(G->device);  // (warp-per-row pulls)
        DevGraph g = G->view();
        DBuf<double> x(nn), r(nn), inc(nn), prev(nn), scat(nn), part(2 * blocks);
        DBuf<int> act(1);
        GD_CUDA(cudaMemcpy(r.p, b, sizeof(double) * n, cudaMemcpyHostToDevice));
        GD_CUDA(cudaMemset(x.p, 0, sizeof(double) * nn));
        std::vector<double> hp(2 * blocks);
        auto finish = [&](int *any, double *l1, double *l2) {
            GD_CUDA(cudaMemcpy(any, act.p, sizeof(int), cudaMemcpyDeviceToHost));
            GD_CUDA(cudaMemcpy(hp.data(), part.p, sizeof(double) * 2 * blocks,
                               cudaMemcpyDeviceToHost));
            double s1 = 0.0, s2 = 0.0;
            for (int k = 0; k < blocks; k++) { s1 += hp[2 * k]; s2 += hp[2 * k + 1]; }
            *l1 = s1;
            *l2 = sqrt(s2);
        };
        int64_t cap = 64;
        report_alloc(rep, cap);
        int any = 0;
        double l1, l2;
        GD_CUDA(cudaMemset(act.p, 0, sizeof(int)));
        k_active_signed<<<blocks, TPB>>>(g, op.dev, r.p, act.p, part.p);
        GD_LAUNCH_CHECK();
        finish(&any, &l1, &l2);
        rep->l1_log[0] = l1;
        rep->l2_log[0] = l2;
        const int64_t vol = G->n_arcs;
        // the reference's coefficient recurrence, in Python float arithmetic
        double delta = (L - mu) / (L + mu);
        const double c0 = 2.0 / (L + mu);
        bool first = true;
        while (any && rep->sweeps < max_sweeps) {
            double c1 = 0.0, c2 = 0.0;
            if (!first) {
                const double dn = 1.0 / (2.0 * (L + mu) / (L - mu) - delta);
                c1 = 4.0 * dn / (L - mu);
                c2 = delta * dn;
                delta = dn;
            }
            k_cheb_inc<<<blocks, TPB>>>(r.p, prev.p, inc.p, x.p, n, first ? 1 : 0, c0, c1, c2);
            k_pull_plain<<<blocks, TPB>>>(g, op.dev, inc.p, scat.p);
            GD_CUDA(cudaMemset(act.p, 0, sizeof(int)));
            k_cheb_r<<<blocks, TPB>>>(g, op.dev, r.p, scat.p, inc.p, act.p, part.p);
            GD_LAUNCH_CHECK();
            std::swap(prev.p, inc.p);
            first = false;
            finish(&any, &l1, &l2);
            report_push_log(rep, cap, vol, 0.0, l1, 0, 0);
            rep->l2_log[rep->n_logs] = l2;
            rep->sweeps += 1;
            rep->total_ops += vol;
        }
        rep->converged = any ? 0 : 1;
        GD_CUDA(cudaMemcpy(hx, x.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
        GD_CUDA(cudaMemcpy(hr, r.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
        int64_t nz = 0;
        for (int64_t i = 0; i < n; i++) nz += (hr[i] != 0.0);
        rep->support_size = nz;
    });
}

extern "C" int gd_hk_taylor(const gd_graph *G, int64_t n_stages, const double *stage_w,
                            const double *b0, double *hv) {
    using namespace gd;
    return guarded([&] {
        GD_CHECK_ARG(G && b0 && hv && (stage_w || n_stages == 0), "null pointer");
        GD_CHECK_ARG(n_stages >= 0, "n_stages must be >= 0");
        GD_CUDA(cudaSetDevice(G->device));
        const int64_t n = G->n;
        const size_t nn = n ? n : 1;
        const int blocks = 16 * n_sms(G->device);  // (warp-per-row pulls)
        DevGraph g = G->view();
        const DevOp op{GD_W_RW, GD_T_DEGREE, 1.0, 0.0, nullptr, nullptr};  // bare 1/d_u
        DBuf<double> vk(nn), nxt(nn);
        GD_CUDA(cudaMemcpy(vk.p, b0, sizeof(double) * n, cudaMemcpyHostToDevice));
        memcpy(hv, b0, sizeof(double) * n);
        for (int64_t k = 0; k < n_stages; ++k) {
            k_pull_plain<<<blocks, TPB>>>(g, op, vk.p, nxt.p);
            k_scale_into<<<blocks, TPB>>>(nxt.p, stage_w[k], vk.p, n);
            GD_LAUNCH_CHECK();
            GD_CUDA(cudaMemcpy(hv + (k + 1) * n, vk.p, sizeof(double) * n,
                               cudaMemcpyDeviceToHost));
        }
    });
}
