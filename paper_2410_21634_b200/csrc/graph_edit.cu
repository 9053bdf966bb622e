// graph_edit.cu -- edge-event batches applied to a device CSR graph, on the
// device: the same canonical CSR as apply_events (src/graph.py:235-258:
// rows sorted, no duplicates, symmetric), without a host round trip of the
// graph.  Used by the resident pair pool on streamed snapshots.
//
//   1. presence of every distinct event edge: binary search of hi in row lo
//   2. host: replay the event order per edge (validity, net add / drop),
//      directed change arcs sorted by (src, dst)  -- O(events)
//   3. device: new degrees, exclusive scan -> row offsets, then rows copied
//      (warp per row, coalesced) with the changed rows merged by one thread
//      each against their sorted change arcs.
#include <cub/cub.cuh>

#include <algorithm>
#include <memory>
#include <vector>

#include "common.cuh"

namespace gd {
namespace {

constexpr int ETPB = 256;

__global__ void k_edge_present(DevGraph g, const int64_t *__restrict__ keys, int64_t k,
                               int32_t *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = keys[i] / g.n, hi = keys[i] % g.n;
        int64_t a = g.row[lo], b = g.row[lo + 1];
        while (a < b) {
            const int64_t mid = (a + b) >> 1;
            if (g.col[mid] < hi) a = mid + 1; else b = mid;
        }
        out[i] = (a < g.row[lo + 1] && g.col[a] == hi) ? 1 : 0;
    }
}

// new degree (int64, for the scan) and row -> changed-row index map
__global__ void k_new_degrees(DevGraph g, int64_t *__restrict__ deg64,
                              int32_t *__restrict__ rowchg) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < g.n;
         u += (int64_t)gridDim.x * blockDim.x) {
        deg64[u] = g.deg[u];
        rowchg[u] = -1;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) deg64[g.n] = 0;
}

__global__ void k_apply_deltas(const int32_t *__restrict__ cnode, const int32_t *__restrict__ cdelta,
                               int64_t nc, int64_t *__restrict__ deg64,
                               int32_t *__restrict__ rowchg) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc;
         i += (int64_t)gridDim.x * blockDim.x) {
        deg64[cnode[i]] += cdelta[i];
        rowchg[cnode[i]] = (int32_t)i;
    }
}

__global__ void k_copy_rows(DevGraph g, const int64_t *__restrict__ row2,
                            const int32_t *__restrict__ rowchg, int32_t *__restrict__ col2,
                            int32_t *__restrict__ deg2, unsigned long long *__restrict__ dmax) {
    const int lane = threadIdx.x & 31;
    int64_t local = 0;
    for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < g.n;
         u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t d2 = row2[u + 1] - row2[u];
        if (lane == 0) deg2[u] = (int32_t)d2;
        local = d2 > local ? d2 : local;
        if (rowchg[u] >= 0) continue;  // merged by k_merge_rows
        const int64_t s = g.row[u], t = row2[u], d = g.row[u + 1] - s;
        for (int64_t j = lane; j < d; j += 32) col2[t + j] = g.col[s + j];
    }
    for (int o = 16; o > 0; o >>= 1) {
        const int64_t v = __shfl_xor_sync(0xffffffffu, local, o);
        local = v > local ? v : local;
    }
    if (lane == 0) atomicMax(dmax, (unsigned long long)local);
}

// changed row i: old row of cnode[i] merged with its change arcs
// [coff[i], coff[i+1]) (targets ascending; sign +1 add, -1 drop)
__global__ void k_merge_rows(DevGraph g, const int64_t *__restrict__ row2,
                             const int32_t *__restrict__ cnode, const int64_t *__restrict__ coff,
                             const int32_t *__restrict__ ctgt, const int32_t *__restrict__ csign,
                             int64_t nc, int32_t *__restrict__ col2) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t u = cnode[i];
        int64_t a = g.row[u];
        const int64_t ae = g.row[u + 1];
        int64_t c = coff[i];
        const int64_t ce = coff[i + 1];
        int64_t o = row2[u];
        while (a < ae || c < ce) {
            const int32_t va = a < ae ? g.col[a] : INT32_MAX;
            const int32_t vc = c < ce ? ctgt[c] : INT32_MAX;
            if (vc < va) {  // insertion (validated on the host)
                col2[o++] = vc;
                ++c;
            } else if (vc == va) {  // deletion of an existing arc
                ++a;
                ++c;
            } else {
                col2[o++] = va;
                ++a;
            }
        }
    }
}

}  // namespace
}  // namespace gd

using namespace gd;

extern "C" {

// Device scratch of the edit, kept per host thread (a snapshot stream must not
// pay n-sized cudaMalloc / cudaFree pairs per batch).
struct EditWS {
    DBuf<int64_t> deg64, dcoff, dk;
    DBuf<int32_t> rowchg, dnode, ddelta, dtgt, dsign, dp;
    DBuf<unsigned long long> dmax;
    DBuf<char> tmp;
};

static void apply_events_impl(const gd_graph *G, const int32_t *kinds, const int64_t *us,
                              const int64_t *vs, int64_t n_events, gd_graph *H) {
    thread_local std::unique_ptr<EditWS> wsp;
    if (!wsp) wsp.reset(new EditWS());
    EditWS &W = *wsp;
    {
        GD_CUDA(cudaSetDevice(G->device));
        const int64_t n = G->n;
        // 1. distinct event edges in event order per edge
        std::vector<int64_t> keys(n_events);
        for (int64_t i = 0; i < n_events; ++i) {
            GD_CHECK_ARG(us[i] >= 0 && vs[i] >= 0 && us[i] < n && vs[i] < n,
                         "event endpoint out of range");
            GD_CHECK_ARG(us[i] != vs[i], "self loop event");
            keys[i] = std::min(us[i], vs[i]) * n + std::max(us[i], vs[i]);
        }
        std::vector<int64_t> order(n_events);
        for (int64_t i = 0; i < n_events; ++i) order[i] = i;
        std::stable_sort(order.begin(), order.end(),
                         [&](int64_t a, int64_t b) { return keys[a] < keys[b]; });
        std::vector<int64_t> uk;
        std::vector<int64_t> first;
        for (int64_t j = 0; j < n_events; ++j)
            if (j == 0 || keys[order[j]] != keys[order[j - 1]]) {
                uk.push_back(keys[order[j]]);
                first.push_back(j);
            }
        const int64_t K = (int64_t)uk.size();
        std::vector<int32_t> was(K ? K : 1, 0);
        if (K) {
            W.dk.ensure(K);
            W.dp.ensure(K);
            GD_CUDA(cudaMemcpy(W.dk.p, uk.data(), 8 * K, cudaMemcpyHostToDevice));
            k_edge_present<<<(int)std::min<int64_t>((K + ETPB - 1) / ETPB, 4096), ETPB>>>(
                G->view(), W.dk.p, K, W.dp.p);
            GD_LAUNCH_CHECK();
            GD_CUDA(cudaMemcpy(was.data(), W.dp.p, 4 * K, cudaMemcpyDeviceToHost));
        }
        // 2. replay per edge; directed change arcs
        struct Arc {
            int32_t s, t, sign;
        };
        std::vector<Arc> arcs;
        for (int64_t q = 0; q < K; ++q) {
            const int64_t j1 = q + 1 < K ? first[q + 1] : n_events;
            bool present = was[q] != 0;
            for (int64_t j = first[q]; j < j1; ++j) {
                const bool ins = kinds[order[j]] != 0;
                if (ins && present) {
                    set_error("invalid argument: insert of existing edge (%lld, %lld)",
                              (long long)(uk[q] / n), (long long)(uk[q] % n));
                    throw Error{GD_ERR_ARG};
                }
                if (!ins && !present) {
                    set_error("invalid argument: delete of missing edge (%lld, %lld)",
                              (long long)(uk[q] / n), (long long)(uk[q] % n));
                    throw Error{GD_ERR_ARG};
                }
                present = ins;
            }
            if (present != (was[q] != 0)) {
                const int32_t lo = (int32_t)(uk[q] / n), hi = (int32_t)(uk[q] % n);
                const int32_t sg = present ? 1 : -1;
                arcs.push_back({lo, hi, sg});
                arcs.push_back({hi, lo, sg});
            }
        }
        std::sort(arcs.begin(), arcs.end(), [](const Arc &a, const Arc &b) {
            return a.s != b.s ? a.s < b.s : a.t < b.t;
        });
        std::vector<int32_t> cnode, cdelta, ctgt, csign;
        std::vector<int64_t> coff;
        for (size_t i = 0; i < arcs.size(); ++i) {
            if (i == 0 || arcs[i].s != arcs[i - 1].s) {
                cnode.push_back(arcs[i].s);
                cdelta.push_back(0);
                coff.push_back((int64_t)i);
            }
            cdelta.back() += arcs[i].sign;
            ctgt.push_back(arcs[i].t);
            csign.push_back(arcs[i].sign);
        }
        coff.push_back((int64_t)arcs.size());
        const int64_t nc = (int64_t)cnode.size();
        int64_t net = 0;
        for (int32_t d : cdelta) net += d;
        // 3. the new graph on the device (H's buffers reused when large enough)
        {
            H->device = G->device;
            H->n = n;
            H->n_arcs = G->n_arcs + net;
            H->row.ensure(n + 1);
            if (H->col.n < (size_t)(H->n_arcs ? H->n_arcs : 1))  // grow with slack: a stream of
                H->col.alloc((size_t)H->n_arcs + (size_t)H->n_arcs / 16 + 1);  // insertions
            H->deg.ensure(n ? n : 1);
            W.deg64.ensure(n + 1); W.dcoff.ensure(nc + 1); W.rowchg.ensure(n ? n : 1);
            W.dnode.ensure(nc ? nc : 1); W.ddelta.ensure(nc ? nc : 1);
            W.dtgt.ensure(arcs.empty() ? 1 : arcs.size()); W.dsign.ensure(arcs.empty() ? 1 : arcs.size());
            W.dmax.ensure(1);
            auto &deg64 = W.deg64, &dcoff = W.dcoff;
            auto &rowchg = W.rowchg, &dnode = W.dnode, &ddelta = W.ddelta, &dtgt = W.dtgt,
                 &dsign = W.dsign;
            auto &dmax = W.dmax;
            GD_CUDA(cudaMemset(dmax.p, 0, sizeof(unsigned long long)));
            if (nc) {
                GD_CUDA(cudaMemcpy(dnode.p, cnode.data(), 4 * nc, cudaMemcpyHostToDevice));
                GD_CUDA(cudaMemcpy(ddelta.p, cdelta.data(), 4 * nc, cudaMemcpyHostToDevice));
                GD_CUDA(cudaMemcpy(dcoff.p, coff.data(), 8 * (nc + 1), cudaMemcpyHostToDevice));
                GD_CUDA(cudaMemcpy(dtgt.p, ctgt.data(), 4 * arcs.size(), cudaMemcpyHostToDevice));
                GD_CUDA(cudaMemcpy(dsign.p, csign.data(), 4 * arcs.size(), cudaMemcpyHostToDevice));
            }
            const int blocks = 4 * n_sms(G->device);
            DevGraph g = G->view();
            k_new_degrees<<<blocks, ETPB>>>(g, deg64.p, rowchg.p);
            if (nc) k_apply_deltas<<<(int)((nc + ETPB - 1) / ETPB), ETPB>>>(dnode.p, ddelta.p, nc,
                                                                             deg64.p, rowchg.p);
            GD_LAUNCH_CHECK();
            size_t bytes = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, bytes, deg64.p, H->row.p, n + 1);
            W.tmp.ensure(bytes ? bytes : 1);
            cub::DeviceScan::ExclusiveSum(W.tmp.p, bytes, deg64.p, H->row.p, n + 1);
            if (n) k_copy_rows<<<blocks, ETPB>>>(g, H->row.p, rowchg.p, H->col.p, H->deg.p, dmax.p);
            if (nc) k_merge_rows<<<(int)((nc + ETPB - 1) / ETPB), ETPB>>>(
                g, H->row.p, dnode.p, dcoff.p, dtgt.p, dsign.p, nc, H->col.p);
            GD_LAUNCH_CHECK();
            unsigned long long h = 0;
            GD_CUDA(cudaMemcpy(&h, dmax.p, sizeof(h), cudaMemcpyDeviceToHost));
            H->d_max = (int64_t)h;
        }
    }
}

int gd_graph_apply_events(const gd_graph *G, const int32_t *kinds, const int64_t *us,
                          const int64_t *vs, int64_t n_events, gd_graph **out) {
    return guarded([&] {
        GD_CHECK_ARG(G && out && (n_events == 0 || (kinds && us && vs)), "null pointer");
        gd_graph *H = new gd_graph();
        try {
            apply_events_impl(G, kinds, us, vs, n_events, H);
        } catch (...) {
            delete H;
            throw;
        }
        *out = H;
    });
}

// As gd_graph_apply_events, writing into an existing graph H != G whose
// buffers are reused (a snapshot stream alternates two graphs).
int gd_graph_apply_events_into(const gd_graph *G, const int32_t *kinds, const int64_t *us,
                               const int64_t *vs, int64_t n_events, gd_graph *H) {
    return guarded([&] {
        GD_CHECK_ARG(G && H && (n_events == 0 || (kinds && us && vs)), "null pointer");
        GD_CHECK_ARG(G != H, "output graph must differ from the input graph");
        apply_events_impl(G, kinds, us, vs, n_events, H);
    });
}

// Copy a device graph back in the reference layout (int64 offsets / targets).
int gd_graph_export(const gd_graph *G, int64_t *offsets, int64_t *targets) {
    return guarded([&] {
        GD_CHECK_ARG(G && offsets && (targets || G->n_arcs == 0), "null pointer");
        GD_CUDA(cudaSetDevice(G->device));
        GD_CUDA(cudaMemcpy(offsets, G->row.p, 8 * (G->n + 1), cudaMemcpyDeviceToHost));
        if (G->n_arcs) {
            std::vector<int32_t> c(G->n_arcs);
            GD_CUDA(cudaMemcpy(c.data(), G->col.p, 4 * G->n_arcs, cudaMemcpyDeviceToHost));
            for (int64_t j = 0; j < G->n_arcs; ++j) targets[j] = c[j];
        }
    });
}

}  // extern "C"
