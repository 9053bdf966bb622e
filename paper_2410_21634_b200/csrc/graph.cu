// graph.cu -- library glue: errors, reports, graph upload, operator upload.
#include <stdarg.h>

#include <new>

#include "common.cuh"

namespace gd {

static thread_local char g_err[1024] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

void report_alloc(gd_report *rep, int64_t cap) {
    memset(rep, 0, sizeof(*rep));
    rep->converged = 1;
    rep->min_residual = __builtin_inf();
    rep->vol_log = (int64_t *)malloc(sizeof(int64_t) * cap);
    rep->gamma_log = (double *)malloc(sizeof(double) * cap);
    rep->l1_log = (double *)malloc(sizeof(double) * (cap + 1));
    rep->l2_log = (double *)malloc(sizeof(double) * (cap + 1));
    rep->sign_log = (int8_t *)malloc(sizeof(int8_t) * cap);
    rep->frontier_sizes = (int64_t *)malloc(sizeof(int64_t) * cap);
    if (!rep->vol_log || !rep->gamma_log || !rep->l1_log || !rep->l2_log || !rep->sign_log ||
        !rep->frontier_sizes)
        throw std::bad_alloc();
}

static void *grow(void *p, size_t bytes) {
    void *q = realloc(p, bytes);
    if (!q) throw std::bad_alloc();
    return q;
}

// Append one sweep to the logs (l1 is the value *after* the sweep).
void report_push_log(gd_report *rep, int64_t &cap, int64_t vol, double gamma, double l1,
                     int8_t sign, int64_t fsize) {
    int64_t t = rep->n_logs;
    if (t >= cap) {
        cap *= 2;
        rep->vol_log = (int64_t *)grow(rep->vol_log, sizeof(int64_t) * cap);
        rep->gamma_log = (double *)grow(rep->gamma_log, sizeof(double) * cap);
        rep->l1_log = (double *)grow(rep->l1_log, sizeof(double) * (cap + 1));
        rep->l2_log = (double *)grow(rep->l2_log, sizeof(double) * (cap + 1));
        rep->sign_log = (int8_t *)grow(rep->sign_log, sizeof(int8_t) * cap);
        rep->frontier_sizes = (int64_t *)grow(rep->frontier_sizes, sizeof(int64_t) * cap);
    }
    rep->vol_log[t] = vol;
    rep->gamma_log[t] = gamma;
    rep->l1_log[t + 1] = l1;
    rep->sign_log[t] = sign;
    rep->frontier_sizes[t] = fsize;
    rep->n_logs = t + 1;
}

void report_trace(gd_report *rep, int64_t &tcap, const int64_t *f, int64_t cnt) {
    if (rep->trace_len + cnt > tcap) {
        int64_t nc = tcap ? tcap : 1024;
        while (nc < rep->trace_len + cnt) nc *= 2;
        rep->trace = (int64_t *)grow(rep->trace, sizeof(int64_t) * nc);
        tcap = nc;
    }
    memcpy(rep->trace + rep->trace_len, f, sizeof(int64_t) * cnt);
    rep->trace_len += cnt;
}

void upload_op(const gd_graph *g, const gd_operator *op, int64_t dim, HostOp &out,
               cudaStream_t s) {
    GD_CHECK_ARG(op != nullptr, "operator is NULL");
    GD_CHECK_ARG(op->weight_rule >= GD_W_RW && op->weight_rule <= GD_W_ARC, "weight_rule");
    GD_CHECK_ARG(op->theta_rule == GD_T_DEGREE || op->theta_rule == GD_T_ARRAY, "theta_rule");
    out.dev = DevOp{op->weight_rule, op->theta_rule, op->beta, op->theta_coeff, nullptr, nullptr};
    if (op->weight_rule == GD_W_ARC) {
        GD_CHECK_ARG(op->arc_w != nullptr, "arc_w is NULL for GD_W_ARC");
        out.arc_w.alloc(g->n_arcs);
        if (g->n_arcs)
            GD_CUDA(cudaMemcpyAsync(out.arc_w.p, op->arc_w, sizeof(double) * g->n_arcs,
                                    cudaMemcpyHostToDevice, s));
        out.dev.arc_w = out.arc_w.p;
    }
    if (op->theta_rule == GD_T_ARRAY) {
        GD_CHECK_ARG(op->theta != nullptr, "theta is NULL for GD_T_ARRAY");
        out.theta.alloc(dim);
        GD_CUDA(cudaMemcpyAsync(out.theta.p, op->theta, sizeof(double) * dim,
                                cudaMemcpyHostToDevice, s));
        out.dev.theta = out.theta.p;
    }
}

// int64 CSR (reference layout) -> int32 column ids + degrees, on the device.
__global__ void k_narrow_cols(const int64_t *__restrict__ tg, int32_t *__restrict__ col,
                              int64_t n_arcs) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_arcs;
         j += (int64_t)gridDim.x * blockDim.x)
        col[j] = (int32_t)tg[j];
}

__global__ void k_degrees(const int64_t *__restrict__ row, int32_t *__restrict__ deg, int64_t n,
                          unsigned long long *__restrict__ dmax) {
    int32_t local = 0;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
         u += (int64_t)gridDim.x * blockDim.x) {
        int32_t d = (int32_t)(row[u + 1] - row[u]);
        deg[u] = d;
        local = d > local ? d : local;
    }
    for (int o = 16; o > 0; o >>= 1) {
        int32_t v = __shfl_xor_sync(0xffffffffu, local, o);
        local = v > local ? v : local;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(dmax, (unsigned long long)local);
}

static void finish_graph(gd_graph *g) {
    DBuf<unsigned long long> dmax(1);
    GD_CUDA(cudaMemset(dmax.p, 0, sizeof(unsigned long long)));
    int blocks = 4 * n_sms(g->device);
    if (g->n) k_degrees<<<blocks, 256>>>(g->row.p, g->deg.p, g->n, dmax.p);
    GD_LAUNCH_CHECK();
    unsigned long long h = 0;
    GD_CUDA(cudaMemcpy(&h, dmax.p, sizeof(h), cudaMemcpyDeviceToHost));
    g->d_max = (int64_t)h;
}

}  // namespace gd

using namespace gd;

extern "C" {

const char *gd_last_error(void) { return g_err; }

int gd_version(void) { return 1; }

void gd_report_free(gd_report *rep) {
    if (!rep) return;
    free(rep->vol_log);
    free(rep->gamma_log);
    free(rep->l1_log);
    free(rep->l2_log);
    free(rep->sign_log);
    free(rep->frontier_sizes);
    free(rep->trace);
    memset(rep, 0, sizeof(*rep));
}

int gd_graph_create(int64_t n, const int64_t *offsets, const int64_t *targets, int64_t n_arcs,
                    int32_t device, gd_graph **out) {
    return guarded([&] {
        GD_CHECK_ARG(out && offsets && (targets || n_arcs == 0), "null pointer");
        GD_CHECK_ARG(n >= 0 && n < (1LL << 31), "n must be in [0, 2^31)");
        GD_CHECK_ARG(offsets[0] == 0 && offsets[n] == n_arcs, "offsets do not cover targets");
        GD_CUDA(cudaSetDevice(device));
        gd_graph *g = new gd_graph();
        g->device = device;
        g->n = n;
        g->n_arcs = n_arcs;
        try {
            g->row.alloc(n + 1);
            g->col.alloc(n_arcs ? n_arcs : 1);
            g->deg.alloc(n ? n : 1);
            GD_CUDA(cudaMemcpy(g->row.p, offsets, sizeof(int64_t) * (n + 1),
                               cudaMemcpyHostToDevice));
            // stage int64 targets through HBM in chunks, narrowing to int32
            const int64_t chunk = 1 << 26;
            DBuf<int64_t> stage(n_arcs < chunk ? (n_arcs ? n_arcs : 1) : chunk);
            for (int64_t s = 0; s < n_arcs; s += chunk) {
                int64_t c = n_arcs - s < chunk ? n_arcs - s : chunk;
                GD_CUDA(cudaMemcpy(stage.p, targets + s, sizeof(int64_t) * c,
                                   cudaMemcpyHostToDevice));
                k_narrow_cols<<<4 * n_sms(device), 256>>>(stage.p, g->col.p + s, c);
                GD_LAUNCH_CHECK();
            }
            finish_graph(g);
            GD_CUDA(cudaDeviceSynchronize());
        } catch (...) {
            delete g;
            throw;
        }
        *out = g;
    });
}

int gd_graph_create_device(int64_t n, const int64_t *d_row_ptr, const int32_t *d_col,
                           int64_t n_arcs, int32_t device, gd_graph **out) {
    return guarded([&] {
        GD_CHECK_ARG(out && d_row_ptr && (d_col || n_arcs == 0), "null pointer");
        GD_CHECK_ARG(n >= 0 && n < (1LL << 31), "n must be in [0, 2^31)");
        GD_CUDA(cudaSetDevice(device));
        gd_graph *g = new gd_graph();
        g->device = device;
        g->n = n;
        g->n_arcs = n_arcs;
        try {
            g->row.alloc(n + 1);
            g->col.alloc(n_arcs ? n_arcs : 1);
            g->deg.alloc(n ? n : 1);
            GD_CUDA(cudaMemcpy(g->row.p, d_row_ptr, sizeof(int64_t) * (n + 1),
                               cudaMemcpyDeviceToDevice));
            if (n_arcs)
                GD_CUDA(cudaMemcpy(g->col.p, d_col, sizeof(int32_t) * n_arcs,
                                   cudaMemcpyDeviceToDevice));
            finish_graph(g);
            GD_CUDA(cudaDeviceSynchronize());
        } catch (...) {
            delete g;
            throw;
        }
        *out = g;
    });
}

int gd_graph_destroy(gd_graph *g) {
    delete g;
    return GD_OK;
}

int gd_graph_info(const gd_graph *g, int64_t *n, int64_t *n_arcs, int64_t *d_max) {
    if (!g) return GD_ERR_ARG;
    if (n) *n = g->n;
    if (n_arcs) *n_arcs = g->n_arcs;
    if (d_max) *d_max = g->d_max;
    return GD_OK;
}

}  // extern "C"
