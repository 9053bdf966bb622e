// hk.cu -- bit-exact heat-kernel push (_hk_push_kernel, src/local_solvers.py:
// 566-661) as data-parallel layered sweeps.
//
// The reference runs a FIFO push on the stage-expanded system, coordinates
// (k, u) for stages k = 0..N.  A pop of (k, u) only scatters into stage k+1,
// and the queue starts with the seed at stage 0, so sweep s (the span between
// two sentinels) pops exactly the stage-(s-1) coordinates that crossed their
// threshold during sweep s-1, and a pop never changes another coordinate of
// its own sweep.  The FIFO order therefore matters in two places only:
//   * the fp order of the contributions into a stage-(k+1) residual: pop
//     order, then CSR order -- reproduced by a stable radix sort of
//     (target, arc position) and an ordered fold per target, and
//   * the queue order of the next sweep: the order of the contributions that
//     first lift a residual to its threshold (`not qmark[t] and rt >=
//     theta[t]`) -- reproduced by sorting the crossing targets by the arc
//     position of their crossing contribution.
// Everything else is elementwise, so each stage is one parallel sweep: the
// products are c = fl(fl(r * tau/(k+1)) * fl(1/d_u)) exactly as the
// reference forms `ri * w * base_w[j]`.
#include <cub/cub.cuh>

#include <memory>
#include <vector>

#include "common.cuh"

namespace gd {
namespace {

constexpr int HT = 256;

inline int hblocks(int64_t n, int cap = 1 << 20) {
    int64_t b = (n + HT - 1) / HT;
    if (b < 1) b = 1;
    return (int)(b < cap ? b : cap);
}

__device__ __forceinline__ double hk_theta(double coeff, int32_t d) {
    return d > 0 ? __dmul_rn(coeff, (double)d) : __longlong_as_double(0x7ff0000000000000LL);
}

// pops of one stage: v += r, r = 0; per-pop scatter value fl(r * w_k)
__global__ void k_hk_gather(const int32_t *__restrict__ F, int64_t f, double *__restrict__ rk,
                            double *__restrict__ vk, double *__restrict__ vals,
                            double *__restrict__ absv, double *__restrict__ wnode,
                            int64_t *__restrict__ fdeg, double wk, double coeff, DevGraph g) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < f;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t u = F[i];
        const double ri = rk[u];
        const int32_t d = g.deg[u];
        if (ri < hk_theta(coeff, d)) {  // (the reference re-checks at pop, :637-639)
            vals[i] = 0.0;
            absv[i] = 0.0;
            wnode[i] = 0.0;
            fdeg[i] = 0;
            continue;
        }
        vk[u] = __dadd_rn(vk[u], ri);
        rk[u] = 0.0;
        vals[i] = __dmul_rn(ri, wk);
        absv[i] = fabs(ri);
        wnode[i] = __ddiv_rn(1.0, (double)d);
        fdeg[i] = d;
    }
}

__device__ __forceinline__ int64_t hk_bsearch_le(const int64_t *a, int64_t cnt, int64_t p) {
    int64_t lo = 0, hi = cnt;
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] <= p) lo = mid; else hi = mid;
    }
    return lo;
}

__global__ void k_hk_expand(const int32_t *__restrict__ F, const int64_t *__restrict__ arcoff,
                            int64_t f, int64_t P, DevGraph g, uint32_t *__restrict__ keys,
                            uint32_t *__restrict__ pidx, int32_t *__restrict__ arc_i) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = hk_bsearch_le(arcoff, f, p);
        keys[p] = (uint32_t)g.col[g.row[F[i]] + (p - arcoff[i])];
        pidx[p] = (uint32_t)p;
        arc_i[p] = (int32_t)i;
    }
}

// ordered fold per target (warp per run of equal targets): r_{k+1}[v] =
// fl(...fl(r + c_1)...) in arc-position order; the first contribution after
// which r >= theta is the enqueue event -> (crossing position << 32 | v)
__global__ void k_hk_fold(const uint32_t *__restrict__ ukeys, const int64_t *__restrict__ segoff,
                          const int64_t *__restrict__ nseg_p, const uint32_t *__restrict__ sp,
                          const int32_t *__restrict__ arc_i, const double *__restrict__ vals,
                          const double *__restrict__ wnode, double *__restrict__ rn,
                          double coeff, DevGraph g, unsigned long long *__restrict__ cross,
                          unsigned long long *__restrict__ ncross) {
    const int lane = threadIdx.x & 31;
    const int64_t nseg = *nseg_p;
    for (int64_t sgi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; sgi < nseg;
         sgi += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t v = ukeys[sgi];
        const int64_t q0 = segoff[sgi], q1 = segoff[sgi + 1];
        const double th = hk_theta(coeff, g.deg[v]);
        double acc = rn[v];
        int64_t qx = -1;
        for (int64_t b = q0; b < q1; b += 32) {
            const int64_t q = b + lane;
            double c = 0.0;
            if (q < q1) {
                const int32_t i = arc_i[sp[q]];
                c = __dmul_rn(vals[i], wnode[i]);
            }
            const int cnt = (int)min((int64_t)32, q1 - b);
            for (int l = 0; l < cnt; l++) {
                acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, c, l));
                if (qx < 0 && acc >= th) qx = b + l;
            }
        }
        if (lane == 0) {
            rn[v] = acc;
            cross[sgi] = qx >= 0 ? ((unsigned long long)sp[qx] << 32) | v : ~0ULL;
            if (qx >= 0) atomicAdd(ncross, 1ULL);
        }
    }
}

__global__ void k_hk_low32(const unsigned long long *__restrict__ a, int64_t n,
                           int32_t *__restrict__ o) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        o[i] = (int32_t)(a[i] & 0xffffffffULL);
}

// fixed-shape sum / min over an n-vector (logs; tree order, 1e-12 of the
// reference's sequential sums)
constexpr int HRB = 256;
__global__ void k_hk_sum_min(const double *__restrict__ a, int64_t n, double *__restrict__ part) {
    __shared__ double ss[HT], sm[HT];
    double s = 0.0, m = __longlong_as_double(0x7ff0000000000000LL);
    for (int64_t i = blockIdx.x * (int64_t)HT + threadIdx.x; i < n; i += (int64_t)HRB * HT) {
        const double v = a[i];
        s += fabs(v);
        m = v < m ? v : m;
    }
    ss[threadIdx.x] = s;
    sm[threadIdx.x] = m;
    __syncthreads();
    for (int o = HT / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            ss[threadIdx.x] += ss[threadIdx.x + o];
            sm[threadIdx.x] = sm[threadIdx.x + o] < sm[threadIdx.x] ? sm[threadIdx.x + o]
                                                                    : sm[threadIdx.x];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = ss[0];
        part[2 * blockIdx.x + 1] = sm[0];
    }
}

struct HkSolver {
    DBuf<double> v, r, vals, absv, wnode, part;
    DBuf<int32_t> F, Fn, arc_i;
    DBuf<int64_t> fdeg, arcoff, segcnt, segoff, nseg, cnt;
    DBuf<uint32_t> keys, skeys, pidx, sp, ukeys;
    DBuf<unsigned long long> cross, csel, csorted, ncross;
    DBuf<char> tmp;
    std::vector<double> hpart;
    void tmp_need(size_t b) { tmp.ensure(b ? b : 1); }

    void sum_min(const double *a, int64_t n, double *s, double *m) {
        k_hk_sum_min<<<HRB, HT>>>(a, n, part.p);
        GD_LAUNCH_CHECK();
        hpart.resize(2 * HRB);
        GD_CUDA(cudaMemcpy(hpart.data(), part.p, sizeof(double) * 2 * HRB, cudaMemcpyDeviceToHost));
        double ts = 0.0, tm = __builtin_inf();
        for (int b = 0; b < HRB; ++b) {
            ts += hpart[2 * b];
            tm = hpart[2 * b + 1] < tm ? hpart[2 * b + 1] : tm;
        }
        *s = ts;
        *m = tm;
    }
};

}  // namespace
}  // namespace gd

using namespace gd;

extern "C" int gd_hk_push(const gd_graph *G, int64_t n_stages, const double *stage_w,
                          double theta_coeff, double *hv, double *hr, int64_t seed,
                          int64_t max_sweeps, gd_report *rep) {
    return guarded([&] {
        GD_CHECK_ARG(G && hv && hr && rep && (stage_w || n_stages == 0), "null pointer");
        GD_CHECK_ARG(n_stages >= 0, "n_stages must be >= 0");
        GD_CHECK_ARG(seed >= 0 && seed < G->n, "seed out of range");
        GD_CUDA(cudaSetDevice(G->device));
        const int64_t n = G->n, L = n_stages + 1, dim = L * n;
        GD_CHECK_ARG(n < (1LL << 31), "n must be < 2^31");
        thread_local std::unique_ptr<HkSolver> ws;
        if (!ws) ws.reset(new HkSolver());
        HkSolver &S = *ws;
        const DevGraph g = G->view();
        const size_t nn = n ? n : 1;
        S.v.ensure(dim); S.r.ensure(dim);
        S.vals.ensure(nn); S.absv.ensure(nn); S.wnode.ensure(nn); S.part.ensure(2 * HRB);
        S.F.ensure(nn); S.Fn.ensure(nn); S.fdeg.ensure(nn + 1); S.arcoff.ensure(nn + 1);
        S.cnt.ensure(2); S.ncross.ensure(1);
        GD_CUDA(cudaMemcpy(S.v.p, hv, sizeof(double) * dim, cudaMemcpyHostToDevice));
        GD_CUDA(cudaMemcpy(S.r.p, hr, sizeof(double) * dim, cudaMemcpyHostToDevice));
        int bits = 1;
        while ((1LL << bits) < n) ++bits;

        // sweep-0 logs from the caller's r, sequentially as the reference (:586-591)
        double l1 = 0.0, min_r = __builtin_inf();
        std::vector<double> layer_l1(L, 0.0);
        for (int64_t k = 0; k < L; ++k)
            for (int64_t i = 0; i < n; ++i) {
                const double x = hr[k * n + i];
                l1 += fabs(x);
                layer_l1[k] += fabs(x);
                if (x < min_r) min_r = x;
            }
        int64_t cap = 64;
        report_alloc(rep, cap);
        rep->l1_log[0] = l1;
        // untouched later layers keep their initial l1 in the rescans
        std::vector<double> rest(L + 1, 0.0);
        for (int64_t k = L - 1; k >= 0; --k) rest[k] = rest[k + 1] + layer_l1[k];

        int32_t d0 = 0;
        GD_CUDA(cudaMemcpy(&d0, G->deg.p + seed, sizeof(int32_t), cudaMemcpyDeviceToHost));
        const double th0 = d0 > 0 ? theta_coeff * (double)d0 : __builtin_inf();
        int64_t f = 0;
        if (hr[seed] >= th0) {  // (:576-579)
            const int32_t s32 = (int32_t)seed;
            GD_CUDA(cudaMemcpy(S.F.p, &s32, sizeof(int32_t), cudaMemcpyHostToDevice));
            f = 1;
        }
        int64_t pushes = 0;
        double left = 0.0;  // l1 of the finished stages (their residual is final)
        int32_t conv = 1;
        for (int64_t k = 0; f > 0; ++k) {
            if (rep->sweeps >= max_sweeps) {
                conv = 0;
                break;
            }
            double *rk = S.r.p + k * n, *vk = S.v.p + k * n;
            const bool scatter = k < n_stages;
            const double wk = scatter ? stage_w[k] : 0.0;
            k_hk_gather<<<hblocks(f), HT>>>(S.F.p, f, rk, vk, S.vals.p, S.absv.p, S.wnode.p,
                                            S.fdeg.p, wk, theta_coeff, g);
            GD_LAUNCH_CHECK();
            GD_CUDA(cudaMemsetAsync(S.fdeg.p + f, 0, sizeof(int64_t)));
            size_t bytes = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, bytes, S.fdeg.p, S.arcoff.p, f + 1);
            S.tmp_need(bytes);
            cub::DeviceScan::ExclusiveSum(S.tmp.p, bytes, S.fdeg.p, S.arcoff.p, f + 1);
            int64_t P = 0;
            GD_CUDA(cudaMemcpy(&P, S.arcoff.p + f, sizeof(int64_t), cudaMemcpyDeviceToHost));
            GD_CHECK_ARG(P < (1LL << 32), "stage volume exceeds 2^32 arcs");
            // sgamma: |r| of the pops (tree sum of the gathered values)
            double sg = 0.0, dummy = 0.0;
            S.sum_min(S.absv.p, f, &sg, &dummy);
            int64_t fnext = 0;
            if (scatter && P > 0) {
                double *rn = S.r.p + (k + 1) * n;
                S.keys.ensure(P); S.skeys.ensure(P); S.pidx.ensure(P); S.sp.ensure(P);
                S.arc_i.ensure(P); S.ukeys.ensure(P); S.segcnt.ensure(P + 1);
                S.segoff.ensure(P + 1); S.nseg.ensure(1); S.cross.ensure(P); S.csel.ensure(P);
                S.csorted.ensure(P);
                GD_CUDA(cudaMemset(S.ncross.p, 0, sizeof(unsigned long long)));
                k_hk_expand<<<hblocks(P), HT>>>(S.F.p, S.arcoff.p, f, P, g, S.keys.p, S.pidx.p,
                                                S.arc_i.p);
                GD_LAUNCH_CHECK();
                bytes = 0;
                cub::DeviceRadixSort::SortPairs(nullptr, bytes, S.keys.p, S.skeys.p, S.pidx.p,
                                                S.sp.p, (int64_t)P, 0, bits);
                S.tmp_need(bytes);
                cub::DeviceRadixSort::SortPairs(S.tmp.p, bytes, S.keys.p, S.skeys.p, S.pidx.p,
                                                S.sp.p, (int64_t)P, 0, bits);
                bytes = 0;
                cub::DeviceRunLengthEncode::Encode(nullptr, bytes, S.skeys.p, S.ukeys.p,
                                                   S.segcnt.p, S.nseg.p, (int64_t)P);
                S.tmp_need(bytes);
                cub::DeviceRunLengthEncode::Encode(S.tmp.p, bytes, S.skeys.p, S.ukeys.p,
                                                   S.segcnt.p, S.nseg.p, (int64_t)P);
                bytes = 0;
                cub::DeviceScan::ExclusiveSum(nullptr, bytes, S.segcnt.p, S.segoff.p, P + 1);
                S.tmp_need(bytes);
                cub::DeviceScan::ExclusiveSum(S.tmp.p, bytes, S.segcnt.p, S.segoff.p, P + 1);
                k_hk_fold<<<hblocks(32 * P, 1 << 16), HT>>>(S.ukeys.p, S.segoff.p, S.nseg.p,
                                                           S.sp.p, S.arc_i.p, S.vals.p,
                                                           S.wnode.p, rn, theta_coeff, g,
                                                           S.cross.p, S.ncross.p);
                GD_LAUNCH_CHECK();
                int64_t nseg = 0;
                GD_CUDA(cudaMemcpy(&nseg, S.nseg.p, sizeof(int64_t), cudaMemcpyDeviceToHost));
                // crossing targets in crossing order = the next sweep's queue
                bytes = 0;
                cub::DeviceRadixSort::SortKeys(nullptr, bytes, S.cross.p, S.csorted.p, nseg);
                S.tmp_need(bytes);
                cub::DeviceRadixSort::SortKeys(S.tmp.p, bytes, S.cross.p, S.csorted.p, nseg);
                unsigned long long nc = 0;  // crossing targets sort first (non-crossing = ~0)
                GD_CUDA(cudaMemcpy(&nc, S.ncross.p, sizeof(nc), cudaMemcpyDeviceToHost));
                fnext = (int64_t)nc;
                if (fnext) k_hk_low32<<<hblocks(fnext), HT>>>(S.csorted.p, fnext, S.Fn.p);
                GD_LAUNCH_CHECK();
            }
            // logs of the sweep (:602-621): l1 = finished stages + this stage's
            // leftover + the receiving stage + untouched later stages
            double sk = 0.0, mk = 0.0, sn = 0.0, mn = __builtin_inf();
            S.sum_min(rk, n, &sk, &mk);
            if (k + 1 < L) S.sum_min(S.r.p + (k + 1) * n, n, &sn, &mn);
            left += sk;
            const double prev_l1 = l1;
            l1 = left + sn + rest[k + 2 < L + 1 ? k + 2 : L];
            if (mk < min_r) min_r = mk;
            if (mn < min_r) min_r = mn;
            report_push_log(rep, cap, P, prev_l1 > 0.0 ? sg / prev_l1 : 0.0, l1, 0, f);
            rep->sweeps += 1;
            rep->total_ops += P;
            pushes += f;
            f = fnext;
            std::swap(S.F.p, S.Fn.p);
        }
        rep->converged = conv;
        rep->pushes = pushes;
        rep->min_residual = min_r;
        GD_CUDA(cudaMemcpy(hv, S.v.p, sizeof(double) * dim, cudaMemcpyDeviceToHost));
        GD_CUDA(cudaMemcpy(hr, S.r.p, sizeof(double) * dim, cudaMemcpyDeviceToHost));
        int64_t nz = 0;
        for (int64_t i = 0; i < dim; i++) nz += (hr[i] != 0.0);
        rep->support_size = nz;
    });
}
