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

// r_next = beta P r (pull), plus any-active flag and partial l1 / l2 sums.
__global__ void k_pull(DevGraph g, DevOp op, const double *__restrict__ r,
                       double *__restrict__ nxt, int *__restrict__ active,
                       double *__restrict__ part) {
    __shared__ double s1[TPB / 32], s2[TPB / 32];
    double a1 = 0.0, a2 = 0.0;
    int any = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < g.n;
         v += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int64_t j = g.row[v]; j < g.row[v + 1]; j++) {
            int32_t u = g.col[j];
            double val = r[u];
            if (val == 0.0) continue;
            acc = __dadd_rn(acc, __dmul_rn(val, pull_weight(g, op, u, v)));
        }
        nxt[v] = acc;
        a1 += fabs(acc);
        a2 += acc * acc;
        any |= acc >= theta_of(op, v, g.deg[v]);
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
        const int blocks = 4 * n_sms(G->device);
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
