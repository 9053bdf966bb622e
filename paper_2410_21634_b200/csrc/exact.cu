// exact.cu -- bit-exact sweep-synchronous LocalGD / LocalCH for one system.
//
// Reproduces src/local_solvers.py:364-538 bit for bit on the device:
//   * gather   : vals_i from r[S_t]; x[S_t] += vals; r[S_t] -= vals
//   * expand   : every arc (i, j) of the frontier gets its global position
//                p = arcoff[i] + j (frontier order, then CSR order)
//   * sort     : stable radix sort of (target v, p) pairs by v groups each
//                target's contributions in frontier-index order
//   * fold     : r[v] = fl(...fl(fl(r[v] + c_1) + c_2)...) in that order,
//                with c = fl(vals_i * w_j) (no FMA) -- the reference's
//                sequential arc loop (_apply_update_seq :282-291)
//   * frontier : S_{t+1} = [u in S_t, active] ++ [first-touch order of new
//                nodes, active] (_apply_update_seq + _filter_frontier), via
//                a head flag at each target's smallest arc position p and
//                two order-preserving compactions.
// The batched throughput path (batch.cu) trades the sort for fp64 atomics.
#include <cub/cub.cuh>

#include <chrono>
#include <memory>
#include <vector>

#include "common.cuh"

namespace gd {
namespace {

constexpr int TPB = 256;

inline int blocks_for(int64_t n, int cap = 1 << 20) {
    int64_t b = (n + TPB - 1) / TPB;
    if (b < 1) b = 1;
    return (int)(b < cap ? b : cap);
}

__device__ __forceinline__ int64_t bsearch_le(const int64_t *a, int64_t cnt, int64_t p) {
    // largest i in [0, cnt) with a[i] <= p (a[0] == 0 <= p)
    int64_t lo = 0, hi = cnt;
    while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] <= p) lo = mid; else hi = mid;
    }
    return lo;
}

// Node u of the solve's id space: the graph's node u % n1 (copy u / n1).  A
// re-solve of K seeds runs them on K disjoint copies of the graph at once
// (node j*n1 + v = node v of copy j): the reference's sweep order restricted
// to one copy is exactly that copy's single-seed order, so each copy's x, r
// and counts are the single solve's bit for bit, for the launches and host
// syncs of one solve.
__device__ __forceinline__ int64_t base_of(int64_t u, int64_t n1) { return u < n1 ? u : u % n1; }

}  // namespace

// Polyak's heavy-ball coefficients for eigenvalues in [mu, L] (the
// stationary limit of local_ch's Chebyshev recurrence), each rounding as the
// restatement writes it (oracle/gdiff_oracle.c orc_local_hb).
void hb_coefficients(double mu, double L, double *eta, double *beta) {
    const double sq = std::sqrt(L), sm = std::sqrt(mu);
    *eta = 4.0 / ((sq + sm) * (sq + sm));
    const double q = (sq - sm) / (sq + sm);
    *beta = q * q;
}

namespace {

// ---- seeds -> initial frontier flags (filter of flatnonzero(b), :383-386)
__global__ void k_flag_active_nodes(const int32_t *__restrict__ nodes, int64_t cnt,
                                    const double *__restrict__ r, DevGraph g, DevOp op,
                                    bool sgn, uint8_t *__restrict__ flag, int64_t n1) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t u = nodes[i];
        const int64_t ub = base_of(u, n1);
        flag[i] = is_active(r[u], theta_of(op, ub, g.deg[ub]), sgn) ? 1 : 0;
    }
}

// ---- gather (LocalGD): src/local_solvers.py:452-456 and the first loop of
// _apply_update_seq (:275-281)
__global__ void k_gather_gd(const int32_t *__restrict__ F, int64_t f, double *__restrict__ x,
                            double *__restrict__ r, double *__restrict__ vals,
                            double *__restrict__ absv, double *__restrict__ wnode,
                            int64_t *__restrict__ fdeg, int32_t *__restrict__ fstamp, int32_t t,
                            DevGraph g, DevOp op, int64_t n1) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < f;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t u = F[i];
        double val = r[u];
        vals[i] = val;
        absv[i] = fabs(val);
        x[u] = __dadd_rn(x[u], val);
        r[u] = __dsub_rn(r[u], val);
        int32_t d = g.deg[base_of(u, n1)];
        fdeg[i] = d;
        wnode[i] = node_weight(op, d);
        fstamp[u] = t;
    }
}

// ---- gather (LocalCH): src/local_solvers.py:507-522
__global__ void k_gather_ch(const int32_t *__restrict__ F, int64_t f, double *__restrict__ x,
                            double *__restrict__ r, double *__restrict__ vals,
                            double *__restrict__ absv, double *__restrict__ wnode,
                            int64_t *__restrict__ fdeg, int32_t *__restrict__ fstamp, int32_t t,
                            double *__restrict__ mom, int32_t *__restrict__ mstamp,
                            double step0, double coef_r, double coef_m, DevGraph g, DevOp op,
                            int64_t n1) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < f;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t u = F[i];
        double rv = r[u];
        absv[i] = fabs(rv);
        double v;
        if (t == 0) {
            v = __dmul_rn(step0, rv);
        } else {
            double prev = (mstamp[u] == t - 1) ? mom[u] : 0.0;
            v = __dadd_rn(__dmul_rn(coef_r, rv), __dmul_rn(coef_m, prev));
        }
        vals[i] = v;
        x[u] = __dadd_rn(x[u], v);
        mom[u] = v;
        mstamp[u] = t;
        r[u] = __dsub_rn(rv, v);
        int32_t d = g.deg[base_of(u, n1)];
        fdeg[i] = d;
        wnode[i] = node_weight(op, d);
        fstamp[u] = t;
    }
}

// ---- expand: arc position p -> (target key, p)
__global__ void k_expand(const int32_t *__restrict__ F, const int64_t *__restrict__ arcoff,
                         int64_t f, int64_t P, DevGraph g, uint32_t *__restrict__ keys,
                         uint32_t *__restrict__ pidx, int32_t *__restrict__ arc_i, int64_t n1) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = bsearch_le(arcoff, f, p);
        int32_t u = F[i];
        const int64_t ub = base_of(u, n1);
        keys[p] = (uint32_t)((u - ub) + g.col[g.row[ub] + (p - arcoff[i])]);
        pidx[p] = (uint32_t)p;
        arc_i[p] = (int32_t)i;
    }
}

// ---- ordered fold, one warp per target segment (second loop of
// _apply_update_seq, :282-291).  Segments come from a run-length encode of
// the sorted targets.  Lanes form the products c = fl(vals_i * w_j) of 32
// consecutive contributions in parallel; lane 0 then adds them in order
// (shuffles), so r[v] = fl(...fl(fl(r[v] + c_1) + c_2)...) exactly.
__global__ void k_fold(const uint32_t *__restrict__ ukeys, const int64_t *__restrict__ segoff,
                       const int64_t *__restrict__ nseg_p, const uint32_t *__restrict__ sp,
                       const int32_t *__restrict__ arc_i, const int64_t *__restrict__ arcoff,
                       const int32_t *__restrict__ F, const double *__restrict__ vals,
                       const double *__restrict__ wnode, DevGraph g, DevOp op,
                       double *__restrict__ r, const int32_t *__restrict__ fstamp, int32_t t,
                       uint8_t *__restrict__ head, int64_t n1) {
    const int lane = threadIdx.x & 31;
    const int64_t nseg = *nseg_p;
    for (int64_t sgi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; sgi < nseg;
         sgi += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t v = ukeys[sgi];
        const int64_t q0 = segoff[sgi], q1 = segoff[sgi + 1];
        double acc = r[v];
        for (int64_t b = q0; b < q1; b += 32) {
            const int64_t q = b + lane;
            double c = 0.0;
            if (q < q1) {
                const int64_t p = sp[q];
                const int32_t i = arc_i[p];
                double w = wnode[i];
                if (op.wrule == GD_W_ARC) w = op.arc_w[g.row[base_of(F[i], n1)] + (p - arcoff[i])];
                c = __dmul_rn(vals[i], w);
            }
            const int cnt = (int)min((int64_t)32, q1 - b);
            for (int l = 0; l < cnt; l++) {
                const double cl = __shfl_sync(0xffffffffu, c, l);
                acc = __dadd_rn(acc, cl);
            }
        }
        if (lane == 0) {
            r[v] = acc;
            if (fstamp[v] != t) head[sp[q0]] = 1;  // first touch of a node outside S_t
        }
    }
}

// ---- candidates that survive the filter (_filter_frontier :336-350)
__global__ void k_flag_heads(const uint32_t *__restrict__ keys, const uint8_t *__restrict__ head,
                             int64_t P, const double *__restrict__ r, DevGraph g, DevOp op,
                             bool sgn, uint8_t *__restrict__ flag, int64_t n1) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        uint8_t h = head[p];
        if (h) {
            uint32_t v = keys[p];
            const int64_t vb = base_of(v, n1);
            h = is_active(r[v], theta_of(op, vb, g.deg[vb]), sgn) ? 1 : 0;
        }
        flag[p] = h;
    }
}

// ---- deterministic l1 / min over r (_l1_and_min :353-361; fixed-shape tree)
constexpr int RED_BLOCKS = 512;
__global__ void k_l1_min_part(const double *__restrict__ r, int64_t n, double *__restrict__ ps,
                              double *__restrict__ pm) {
    __shared__ double ss[TPB], sm[TPB];
    double s = 0.0, m = __longlong_as_double(0x7ff0000000000000LL);
    for (int64_t i = blockIdx.x * (int64_t)TPB + threadIdx.x; i < n; i += (int64_t)RED_BLOCKS * TPB) {
        double v = r[i];
        s += fabs(v);
        m = v < m ? v : m;
    }
    ss[threadIdx.x] = s;
    sm[threadIdx.x] = m;
    __syncthreads();
    for (int o = TPB / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            ss[threadIdx.x] += ss[threadIdx.x + o];
            double b = sm[threadIdx.x + o];
            sm[threadIdx.x] = b < sm[threadIdx.x] ? b : sm[threadIdx.x];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ps[blockIdx.x] = ss[0];
        pm[blockIdx.x] = sm[0];
    }
}

__global__ void k_l1_min_final(const double *__restrict__ ps, const double *__restrict__ pm,
                               double *__restrict__ out) {
    __shared__ double ss[RED_BLOCKS], sm[RED_BLOCKS];
    for (int i = threadIdx.x; i < RED_BLOCKS; i += blockDim.x) {
        ss[i] = ps[i];
        sm[i] = pm[i];
    }
    __syncthreads();
    for (int o = RED_BLOCKS / 2; o > 0; o >>= 1) {
        for (int i = threadIdx.x; i < o; i += blockDim.x) {
            ss[i] += ss[i + o];
            sm[i] = sm[i + o] < sm[i] ? sm[i + o] : sm[i];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = ss[0];
        out[1] = sm[0];
    }
}

__global__ void k_sum_block(const double *__restrict__ a, int64_t n, double *__restrict__ out) {
    // single-block deterministic sum (frontier |vals| -> sgamma)
    __shared__ double ss[TPB];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += TPB) s += a[i];
    ss[threadIdx.x] = s;
    __syncthreads();
    for (int o = TPB / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) ss[threadIdx.x] += ss[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = ss[0];
}

// per-copy frontier statistics of a multi-seed re-solve: pushes, volume,
// last sweep with work
__global__ void k_copy_stats(const int32_t *__restrict__ F, int64_t f, int64_t n1, DevGraph g,
                             int32_t t, unsigned long long *__restrict__ pushes,
                             unsigned long long *__restrict__ ops, int32_t *__restrict__ last) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < f;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = F[i], j = u / n1;
        atomicAdd(pushes + j, 1ULL);
        atomicAdd(ops + j, (unsigned long long)g.deg[u - j * n1]);
        atomicMax(last + j, t);
    }
}

__global__ void k_set_seeds(double *__restrict__ r, int32_t *__restrict__ ids,
                            const int64_t *__restrict__ seeds, int K, int64_t n1, double val) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < K) {
        const int64_t u = j * n1 + seeds[j];
        r[u] = val;
        ids[j] = (int32_t)u;
    }
}

__global__ void k_to_i64(const int32_t *__restrict__ a, int64_t n, int64_t *__restrict__ o) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        o[i] = a[i];
}

// numpy pairwise sum of |b| (np.abs(sys.b).sum(), :496)
double pw_sum_abs(const double *a, int64_t n) {
    if (n < 8) {
        double res = -0.0;
        for (int64_t i = 0; i < n; i++) res += fabs(a[i]);
        return res;
    } else if (n <= 128) {
        double rr[8];
        int64_t i;
        for (int k = 0; k < 8; k++) rr[k] = fabs(a[k]);
        for (i = 8; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; k++) rr[k] += fabs(a[i + k]);
        double res = ((rr[0] + rr[1]) + (rr[2] + rr[3])) + ((rr[4] + rr[5]) + (rr[6] + rr[7]));
        for (; i < n; i++) res += fabs(a[i]);
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pw_sum_abs(a, n2) + pw_sum_abs(a + n2, n - n2);
}

struct SweepSolver {
    const gd_graph *G;
    DevGraph g;
    HostOp op;
    int64_t n;           // solve id space: copies * n1
    int64_t n1 = 0;      // graph nodes
    int64_t copies = 1;  // disjoint copies (multi-seed re-solve)
    bool sgn;
    cudaStream_t s = 0;
    DBuf<double> x, r, vals, absv, wnode, mom, red_ps, red_pm, scal;
    DBuf<int32_t> F, Fn, fstamp, mstamp, seeds;
    DBuf<int64_t> fdeg, arcoff, trace64, cnt;
    DBuf<uint32_t> keys, skeys, pidx, sp, ukeys;
    DBuf<int32_t> arc_i;
    DBuf<int64_t> segcnt, segoff, nseg;
    DBuf<uint8_t> head, flag;
    DBuf<char> tmp;
    int bits = 1;

    void tmp_need(size_t bytes) { tmp.ensure(bytes ? bytes : 1); }

    // Buffers are kept across calls (per host thread, grown on demand): a
    // drop-in call should not pay a dozen n-sized cudaMalloc/cudaFree pairs.
    void prepare(const gd_graph *G_, const gd_operator *o, bool sgn_, int64_t copies_ = 1) {
        G = G_;
        sgn = sgn_;
        g = G->view();
        n1 = G->n;
        copies = copies_;
        n = copies * n1;
        upload_op(G, o, n1, op, s);
        size_t nn = n ? n : 1;
        x.ensure(nn); r.ensure(nn); vals.ensure(nn); absv.ensure(nn); wnode.ensure(nn);
        F.ensure(nn); Fn.ensure(nn); fstamp.ensure(nn); seeds.ensure(nn);
        fdeg.ensure(nn + 1); arcoff.ensure(nn + 1); trace64.ensure(nn); cnt.ensure(4);
        red_ps.ensure(RED_BLOCKS); red_pm.ensure(RED_BLOCKS); scal.ensure(4);
        flag.ensure(nn);
        bits = 1;
        while ((1LL << bits) < n) ++bits;
        GD_CUDA(cudaMemsetAsync(fstamp.p, 0xFF, sizeof(int32_t) * nn, s));  // -1: never in S_t
    }

    void reduce_l1_min(double *host2) {
        k_l1_min_part<<<RED_BLOCKS, TPB, 0, s>>>(r.p, n, red_ps.p, red_pm.p);
        k_l1_min_final<<<1, 256, 0, s>>>(red_ps.p, red_pm.p, scal.p);
        GD_LAUNCH_CHECK();
        GD_CUDA(cudaMemcpyAsync(host2, scal.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
        GD_CUDA(cudaStreamSynchronize(s));
    }

    // S_0 = filter(flatnonzero(b)) in index order; x = x0 (zero unless warm)
    int64_t init(const double *b, const double *x0 = nullptr) {
        GD_CUDA(cudaMemcpy(r.p, b, sizeof(double) * n, cudaMemcpyHostToDevice));
        if (x0)
            GD_CUDA(cudaMemcpy(x.p, x0, sizeof(double) * n, cudaMemcpyHostToDevice));
        else
            GD_CUDA(cudaMemset(x.p, 0, sizeof(double) * (n ? n : 1)));
        std::vector<int32_t> nz;
        for (int64_t i = 0; i < n; i++)
            if (b[i] != 0.0) nz.push_back((int32_t)i);
        int64_t cnt0 = (int64_t)nz.size();
        if (!cnt0) return 0;
        GD_CUDA(cudaMemcpy(seeds.p, nz.data(), sizeof(int32_t) * cnt0, cudaMemcpyHostToDevice));
        k_flag_active_nodes<<<blocks_for(cnt0), TPB, 0, s>>>(seeds.p, cnt0, r.p, g, op.dev, sgn,
                                                             flag.p, n1);
        GD_LAUNCH_CHECK();
        size_t bytes = 0;
        cub::DeviceSelect::Flagged(nullptr, bytes, seeds.p, flag.p, F.p, cnt.p, cnt0, s);
        tmp_need(bytes);
        cub::DeviceSelect::Flagged(tmp.p, bytes, seeds.p, flag.p, F.p, cnt.p, cnt0, s);
        int64_t f = 0;
        GD_CUDA(cudaMemcpyAsync(&f, cnt.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        GD_CUDA(cudaStreamSynchronize(s));
        return f;
    }

    // S_0 for b = val e_seed: the same filter, state zeroed on the device
    int64_t init_spike(int64_t seed, double val) {
        GD_CUDA(cudaMemsetAsync(r.p, 0, sizeof(double) * (n ? n : 1), s));
        GD_CUDA(cudaMemsetAsync(x.p, 0, sizeof(double) * (n ? n : 1), s));
        GD_CUDA(cudaMemcpyAsync(r.p + seed, &val, sizeof(double), cudaMemcpyHostToDevice, s));
        const int32_t sd = (int32_t)seed;
        GD_CUDA(cudaMemcpyAsync(seeds.p, &sd, sizeof(int32_t), cudaMemcpyHostToDevice, s));
        k_flag_active_nodes<<<1, TPB, 0, s>>>(seeds.p, 1, r.p, g, op.dev, sgn, flag.p, n1);
        GD_LAUNCH_CHECK();
        uint8_t f = 0;
        GD_CUDA(cudaMemcpyAsync(&f, flag.p, 1, cudaMemcpyDeviceToHost, s));
        GD_CUDA(cudaStreamSynchronize(s));
        if (f) {
            GD_CUDA(cudaMemcpyAsync(F.p, &sd, sizeof(int32_t), cudaMemcpyHostToDevice, s));
            GD_CUDA(cudaStreamSynchronize(s));
        }
        return f ? 1 : 0;
    }

    // K seeds on K graph copies: r = val at node j*n1 + seeds[j] (device
    // seeds), S_0 = the active ones in id (= copy) order
    int64_t init_copies(const int64_t *d_seeds, int K, double val) {
        GD_CUDA(cudaMemsetAsync(r.p, 0, sizeof(double) * (n ? n : 1), s));
        GD_CUDA(cudaMemsetAsync(x.p, 0, sizeof(double) * (n ? n : 1), s));
        k_set_seeds<<<1, 64, 0, s>>>(r.p, seeds.p, d_seeds, K, n1, val);
        k_flag_active_nodes<<<1, TPB, 0, s>>>(seeds.p, K, r.p, g, op.dev, sgn, flag.p, n1);
        GD_LAUNCH_CHECK();
        size_t bytes = 0;
        cub::DeviceSelect::Flagged(nullptr, bytes, seeds.p, flag.p, F.p, cnt.p, K, s);
        tmp_need(bytes);
        cub::DeviceSelect::Flagged(tmp.p, bytes, seeds.p, flag.p, F.p, cnt.p, K, s);
        int64_t f = 0;
        GD_CUDA(cudaMemcpyAsync(&f, cnt.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        GD_CUDA(cudaStreamSynchronize(s));
        return f;
    }

    // one sweep after the gather kernel ran; returns |S_{t+1}| and P
    int64_t scatter_and_filter(int64_t f, int32_t t, int64_t *P_out, double *sgamma) {
        // arc offsets: exclusive scan of frontier degrees (fdeg[f] = 0 -> total)
        GD_CUDA(cudaMemsetAsync(fdeg.p + f, 0, sizeof(int64_t), s));
        size_t bytes = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, bytes, fdeg.p, arcoff.p, f + 1, s);
        tmp_need(bytes);
        cub::DeviceScan::ExclusiveSum(tmp.p, bytes, fdeg.p, arcoff.p, f + 1, s);
        k_sum_block<<<1, TPB, 0, s>>>(absv.p, f, scal.p + 2);
        GD_LAUNCH_CHECK();
        int64_t P = 0;
        GD_CUDA(cudaMemcpyAsync(&P, arcoff.p + f, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        GD_CUDA(cudaMemcpyAsync(sgamma, scal.p + 2, sizeof(double), cudaMemcpyDeviceToHost, s));
        GD_CUDA(cudaStreamSynchronize(s));
        GD_CHECK_ARG(P < (1LL << 32), "frontier volume exceeds 2^32 arcs");
        *P_out = P;
        if (P > 0) {
            keys.ensure(P); skeys.ensure(P); pidx.ensure(P); sp.ensure(P); arc_i.ensure(P);
            ukeys.ensure(P); segcnt.ensure(P + 1); segoff.ensure(P + 1); nseg.ensure(1);
            head.ensure(P);
            if (flag.n < (size_t)P) flag.alloc(P);
            GD_CUDA(cudaMemsetAsync(head.p, 0, P, s));
            k_expand<<<blocks_for(P), TPB, 0, s>>>(F.p, arcoff.p, f, P, g, keys.p, pidx.p, arc_i.p,
                                                   n1);
            GD_LAUNCH_CHECK();
            bytes = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, skeys.p, pidx.p, sp.p,
                                            (int64_t)P, 0, bits, s);
            tmp_need(bytes);
            cub::DeviceRadixSort::SortPairs(tmp.p, bytes, keys.p, skeys.p, pidx.p, sp.p,
                                            (int64_t)P, 0, bits, s);
            // target segments: (unique target, run length) -> offsets
            bytes = 0;
            cub::DeviceRunLengthEncode::Encode(nullptr, bytes, skeys.p, ukeys.p, segcnt.p, nseg.p,
                                               (int64_t)P, s);
            tmp_need(bytes);
            cub::DeviceRunLengthEncode::Encode(tmp.p, bytes, skeys.p, ukeys.p, segcnt.p, nseg.p,
                                               (int64_t)P, s);
            bytes = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, bytes, segcnt.p, segoff.p, P + 1, s);
            tmp_need(bytes);
            // (only offsets [0, nseg] are read: exact whatever follows the runs)
            cub::DeviceScan::ExclusiveSum(tmp.p, bytes, segcnt.p, segoff.p, P + 1, s);
            k_fold<<<blocks_for(32 * P, 1 << 16), TPB, 0, s>>>(ukeys.p, segoff.p, nseg.p, sp.p,
                                                               arc_i.p, arcoff.p, F.p, vals.p,
                                                               wnode.p, g, op.dev, r.p, fstamp.p,
                                                               t, head.p, n1);
            GD_LAUNCH_CHECK();
        }
        // 1) frontier members that stay active, in S_t order
        k_flag_active_nodes<<<blocks_for(f), TPB, 0, s>>>(F.p, f, r.p, g, op.dev, sgn, flag.p, n1);
        GD_LAUNCH_CHECK();
        bytes = 0;
        cub::DeviceSelect::Flagged(nullptr, bytes, F.p, flag.p, Fn.p, cnt.p, f, s);
        tmp_need(bytes);
        cub::DeviceSelect::Flagged(tmp.p, bytes, F.p, flag.p, Fn.p, cnt.p, f, s);
        int64_t c1 = 0;
        GD_CUDA(cudaMemcpyAsync(&c1, cnt.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        GD_CUDA(cudaStreamSynchronize(s));
        int64_t c2 = 0;
        if (P > 0) {
            k_flag_heads<<<blocks_for(P), TPB, 0, s>>>(keys.p, head.p, P, r.p, g, op.dev, sgn,
                                                       flag.p, n1);
            GD_LAUNCH_CHECK();
            bytes = 0;
            cub::DeviceSelect::Flagged(nullptr, bytes, (int32_t *)keys.p, flag.p, Fn.p + c1,
                                       cnt.p + 1, P, s);
            tmp_need(bytes);
            cub::DeviceSelect::Flagged(tmp.p, bytes, (int32_t *)keys.p, flag.p, Fn.p + c1,
                                       cnt.p + 1, P, s);
            GD_CUDA(cudaMemcpyAsync(&c2, cnt.p + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
            GD_CUDA(cudaStreamSynchronize(s));
        }
        std::swap(F.p, Fn.p);
        return c1 + c2;
    }

    void record(gd_report *rep, int64_t &tcap, int64_t f) {
        k_to_i64<<<blocks_for(f), TPB, 0, s>>>(F.p, f, trace64.p);
        GD_LAUNCH_CHECK();
        std::vector<int64_t> h(f);
        GD_CUDA(cudaMemcpyAsync(h.data(), trace64.p, sizeof(int64_t) * f, cudaMemcpyDeviceToHost, s));
        GD_CUDA(cudaStreamSynchronize(s));
        report_trace(rep, tcap, h.data(), f);
    }

    void finish(double *hx, double *hr, gd_report *rep) {
        GD_CUDA(cudaMemcpy(hx, x.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
        GD_CUDA(cudaMemcpy(hr, r.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
        int64_t nz = 0;
        for (int64_t i = 0; i < n; i++) nz += (hr[i] != 0.0);
        rep->support_size = nz;
    }
};

SweepSolver &solver_for(const gd_graph *G, const gd_operator *o, bool sgn) {
    thread_local std::unique_ptr<SweepSolver> cache;
    thread_local int device = -1;
    if (!cache || device != G->device) {
        cache.reset(new SweepSolver());
        device = G->device;
    }
    cache->prepare(G, o, sgn);
    return *cache;
}

}  // namespace

// A re-solve worker: its own solver buffers and a non-blocking stream, so
// several host threads can run exact seeds concurrently.
struct ExactWorker {
    SweepSolver S;
    // persistent small buffers (a cudaFree would synchronise the device and
    // serialise the workers): seeds, per-copy stats, caller scratch
    DBuf<int64_t> dseeds;
    DBuf<unsigned long long> st, scratch;
    DBuf<int32_t> last;
    ExactWorker() { GD_CUDA(cudaStreamCreateWithFlags(&S.s, cudaStreamNonBlocking)); }
    ~ExactWorker() {
        if (S.s) cudaStreamDestroy(S.s);
    }
};

ExactWorker *exact_worker_create() { return new ExactWorker(); }

// K LocalGD seeds at once on K disjoint graph copies (see base_of): one sweep
// loop, so the per-sweep launches and host syncs -- most of a single re-solve's
// cost -- are paid once for all K.  Per copy: bit-exact x, r, sweeps, ops,
// pushes and convergence of the single-seed solve.
ExactMulti exact_multi_solve(ExactWorker *W, const gd_graph *G, const gd_operator *o,
                             const int64_t *seeds, int K, double bval, int64_t max_sweeps) {
    SweepSolver &S = W->S;
    S.prepare(G, o, false, K);
    ExactMulti out;
    out.n1 = S.n1;
    out.K = K;
    W->dseeds.ensure(64);
    W->st.ensure(128);
    W->last.ensure(64);
    GD_CHECK_ARG(K <= 64, "at most 64 seeds per exact multi-solve");
    int64_t *dseeds = W->dseeds.p;
    unsigned long long *st = W->st.p;
    int32_t *last = W->last.p;
    GD_CUDA(cudaMemcpyAsync(dseeds, seeds, sizeof(int64_t) * K, cudaMemcpyHostToDevice, S.s));
    GD_CUDA(cudaMemsetAsync(st, 0, sizeof(unsigned long long) * 2 * K, S.s));
    GD_CUDA(cudaMemsetAsync(last, 0xFF, sizeof(int32_t) * K, S.s));
    int64_t f = S.init_copies(dseeds, K, bval);
    std::vector<int32_t> capped(K, 0);
    int32_t t = 0;
    while (f) {
        if (t >= max_sweeps) {  // copies with work left are not converged
            std::vector<int32_t> h(f);
            GD_CUDA(cudaMemcpy(h.data(), S.F.p, sizeof(int32_t) * f, cudaMemcpyDeviceToHost));
            for (int32_t u : h) capped[u / S.n1] = 1;
            break;
        }
        k_gather_gd<<<blocks_for(f), TPB, 0, S.s>>>(S.F.p, f, S.x.p, S.r.p, S.vals.p, S.absv.p,
                                                    S.wnode.p, S.fdeg.p, S.fstamp.p, t, S.g,
                                                    S.op.dev, S.n1);
        k_copy_stats<<<blocks_for(f), TPB, 0, S.s>>>(S.F.p, f, S.n1, S.g, t, st, st + K, last);
        GD_LAUNCH_CHECK();
        int64_t P = 0;
        double sgamma = 0.0;
        f = S.scatter_and_filter(f, t, &P, &sgamma);
        ++t;
    }
    std::vector<unsigned long long> hs(2 * K);
    std::vector<int32_t> hl(K);
    GD_CUDA(cudaMemcpyAsync(hs.data(), st, sizeof(unsigned long long) * 2 * K,
                            cudaMemcpyDeviceToHost, S.s));
    GD_CUDA(cudaMemcpyAsync(hl.data(), last, sizeof(int32_t) * K, cudaMemcpyDeviceToHost, S.s));
    GD_CUDA(cudaStreamSynchronize(S.s));
    for (int j = 0; j < K; ++j) {
        out.pushes.push_back((int64_t)hs[j]);
        out.ops.push_back((int64_t)hs[K + j]);
        out.sweeps.push_back((int64_t)hl[j] + 1);
        out.conv.push_back(capped[j] ? 0 : 1);
    }
    out.x = S.x.p;
    out.r = S.r.p;
    return out;
}
void exact_worker_destroy(ExactWorker *w) { delete w; }
cudaStream_t exact_worker_stream(ExactWorker *w) { return w->S.s; }
unsigned long long *exact_worker_scratch(ExactWorker *w) {
    w->scratch.ensure(4);
    return w->scratch.p;
}

// Bit-exact re-solve of one seed for the batched solvers (common.cuh): the
// sweep loops of local_gd_run / gd_local_ch below without the per-sweep
// logs (LocalCH keeps its l1 for the divergence abort, :527-530).
ExactSeed exact_seed_solve(ExactWorker *W, const gd_graph *G, const gd_operator *o,
                           int32_t method, int64_t seed, double bval, double mu, double L,
                           int64_t max_sweeps, bool sgn) {
    const bool ch = method == GD_M_LOCAL_CH || method == GD_M_LOCAL_HB;
    const bool hb = method == GD_M_LOCAL_HB;
    SweepSolver &S = W->S;
    S.prepare(G, o, ch || sgn);
    ExactSeed out{0, 0, 0, 1, 0, nullptr, nullptr, S.n};
    size_t nn = S.n ? S.n : 1;
    if (ch) {
        S.mom.ensure(nn);
        S.mstamp.ensure(nn);
        GD_CUDA(cudaMemsetAsync(S.mom.p, 0, sizeof(double) * nn, S.s));
        GD_CUDA(cudaMemsetAsync(S.mstamp.p, 0xFE, sizeof(int32_t) * nn, S.s));
    }
    int64_t f = S.init_spike(seed, bval);
    const double rho = ch ? (L - mu) / (L + mu) : 0.0, step0 = ch ? 2.0 / (L + mu) : 0.0;
    const double b_l1 = fabs(bval);
    double delta = rho;
    int32_t t = 0;
    while (f) {
        if (out.sweeps >= max_sweeps) { out.converged = 0; break; }
        if (ch) {
            double coef_r = 0.0, coef_m = 0.0, s0 = step0;
            if (hb) {
                hb_coefficients(mu, L, &s0, &coef_m);
                coef_r = s0;
            } else if (t > 0) {
                const double dn = 1.0 / (2.0 * (L + mu) / (L - mu) - delta);
                coef_r = 4.0 * dn / (L - mu);
                coef_m = delta * dn;
                delta = dn;
            }
            k_gather_ch<<<blocks_for(f), TPB, 0, S.s>>>(S.F.p, f, S.x.p, S.r.p, S.vals.p, S.absv.p,
                                                        S.wnode.p, S.fdeg.p, S.fstamp.p, t,
                                                        S.mom.p, S.mstamp.p, s0, coef_r, coef_m,
                                                        S.g, S.op.dev, S.n1);
        } else {
            k_gather_gd<<<blocks_for(f), TPB, 0, S.s>>>(S.F.p, f, S.x.p, S.r.p, S.vals.p, S.absv.p,
                                                        S.wnode.p, S.fdeg.p, S.fstamp.p, t, S.g,
                                                        S.op.dev, S.n1);
        }
        GD_LAUNCH_CHECK();
        int64_t P = 0;
        double sgamma = 0.0;
        const auto tt0 = std::chrono::steady_clock::now();
        const int64_t fnext = S.scatter_and_filter(f, t, &P, &sgamma);
        static const bool trace = getenv("GDIFF_EXACT_TRACE") != nullptr;  // (diagnostic)
        if (trace)
            fprintf(stderr, "exact sweep %d f=%lld P=%lld %.1f us\n", t, (long long)f, (long long)P,
                    std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tt0)
                        .count());
        out.ops += P;
        out.pushes += f;
        out.sweeps += 1;
        f = fnext;
        ++t;
        if (ch) {
            double lm[2];
            S.reduce_l1_min(lm);
            if (lm[0] > 10.0 * b_l1) {
                out.converged = 0;
                out.diverged = 1;
                break;
            }
        }
    }
    GD_CUDA(cudaStreamSynchronize(S.s));
    out.x = S.x.p;
    out.r = S.r.p;
    return out;
}

}  // namespace gd

using namespace gd;

extern "C" {

static void local_gd_run(const gd_graph *G, const gd_operator *o, const double *b,
                         const double *x0, bool sgn, double *x, double *r, int64_t max_sweeps,
                         int32_t record_trace, gd_report *rep) {
    {
        GD_CUDA(cudaSetDevice(G->device));
        int64_t cap = 64, tcap = 0;
        report_alloc(rep, cap);
        SweepSolver &S = solver_for(G, o, sgn);
        int64_t f = S.init(b, x0);
        double lm[2];
        S.reduce_l1_min(lm);
        rep->l1_log[0] = lm[0];
        rep->min_residual = lm[1];
        int32_t t = 0;
        while (f) {
            if (rep->sweeps >= max_sweeps) { rep->converged = 0; break; }
            if (record_trace) S.record(rep, tcap, f);
            k_gather_gd<<<blocks_for(f), TPB, 0, S.s>>>(S.F.p, f, S.x.p, S.r.p, S.vals.p, S.absv.p,
                                                        S.wnode.p, S.fdeg.p, S.fstamp.p, t, S.g,
                                                        S.op.dev, S.n1);
            GD_LAUNCH_CHECK();
            int64_t P = 0;
            double sgamma = 0.0;
            int64_t fnext = S.scatter_and_filter(f, t, &P, &sgamma);
            double prev = rep->l1_log[rep->n_logs];
            S.reduce_l1_min(lm);
            report_push_log(rep, cap, P, prev > 0 ? sgamma / prev : 0.0, lm[0], 0, f);
            if (lm[1] < rep->min_residual) rep->min_residual = lm[1];
            rep->total_ops += P;
            rep->pushes += f;
            rep->sweeps += 1;
            f = fnext;
            ++t;
        }
        S.finish(x, r, rep);
    }
}

int gd_local_gd(const gd_graph *G, const gd_operator *o, const double *b, double *x, double *r,
                int64_t max_sweeps, int32_t record_trace, gd_report *rep) {
    return guarded([&] {
        GD_CHECK_ARG(G && o && b && x && r && rep, "null pointer");
        local_gd_run(G, o, b, nullptr, false, x, r, max_sweeps, record_trace, rep);
    });
}

int gd_local_gd_warm(const gd_graph *G, const gd_operator *o, double *x, double *r,
                     int32_t is_signed, int64_t max_sweeps, int32_t record_trace,
                     gd_report *rep) {
    return guarded([&] {
        GD_CHECK_ARG(G && o && x && r && rep, "null pointer");
        std::vector<double> r0(r, r + G->n), x0(x, x + G->n);
        local_gd_run(G, o, r0.data(), x0.data(), is_signed != 0, x, r, max_sweeps, record_trace,
                     rep);
    });
}

static int local_momentum(const gd_graph *G, const gd_operator *o, const double *b, double *x,
                          double *r, double mu, double L, int64_t max_sweeps,
                          int32_t record_trace, gd_report *rep, bool hb);

int gd_local_ch(const gd_graph *G, const gd_operator *o, const double *b, double *x, double *r,
                double mu, double L, int64_t max_sweeps, int32_t record_trace, gd_report *rep) {
    return local_momentum(G, o, b, x, r, mu, L, max_sweeps, record_trace, rep, false);
}

// LocalHB: local_ch with Polyak's stationary heavy-ball coefficients (no
// reference counterpart; restatement in oracle/ orc_local_hb, golden
// tests/golden/hb.npz from the reference's own _SweepDriver).
int gd_local_hb(const gd_graph *G, const gd_operator *o, const double *b, double *x, double *r,
                double mu, double L, int64_t max_sweeps, int32_t record_trace, gd_report *rep) {
    return local_momentum(G, o, b, x, r, mu, L, max_sweeps, record_trace, rep, true);
}

static int local_momentum(const gd_graph *G, const gd_operator *o, const double *b, double *x,
                          double *r, double mu, double L, int64_t max_sweeps,
                          int32_t record_trace, gd_report *rep, bool hb) {
    return guarded([&] {
        GD_CHECK_ARG(G && o && b && x && r && rep, "null pointer");
        GD_CHECK_ARG(mu < L, "need mu < L");
        GD_CUDA(cudaSetDevice(G->device));
        int64_t cap = 64, tcap = 0;
        report_alloc(rep, cap);
        SweepSolver &S = solver_for(G, o, true);
        size_t nn = S.n ? S.n : 1;
        S.mom.ensure(nn);
        S.mstamp.ensure(nn);
        GD_CUDA(cudaMemset(S.mom.p, 0, sizeof(double) * nn));
        GD_CUDA(cudaMemset(S.mstamp.p, 0xFE, sizeof(int32_t) * nn));  // never t-1 >= -1
        int64_t f = S.init(b);
        double lm[2];
        S.reduce_l1_min(lm);
        rep->l1_log[0] = lm[0];
        rep->min_residual = lm[1];
        const double rho = (L - mu) / (L + mu);
        const double step0 = 2.0 / (L + mu);
        const double b_l1 = pw_sum_abs(b, S.n);
        double delta = rho;
        int32_t t = 0;
        while (f) {
            if (rep->sweeps >= max_sweeps) { rep->converged = 0; break; }
            if (record_trace) S.record(rep, tcap, f);
            double coef_r = 0.0, coef_m = 0.0, s0 = step0;
            if (hb) {  // eta r (+ beta prev): the gather's t == 0 branch uses step0 = eta
                hb_coefficients(mu, L, &s0, &coef_m);
                coef_r = s0;
            } else if (t > 0) {
                double delta_next = 1.0 / (2.0 * (L + mu) / (L - mu) - delta);
                coef_r = 4.0 * delta_next / (L - mu);
                coef_m = delta * delta_next;
                delta = delta_next;
            }
            k_gather_ch<<<blocks_for(f), TPB, 0, S.s>>>(S.F.p, f, S.x.p, S.r.p, S.vals.p, S.absv.p,
                                                        S.wnode.p, S.fdeg.p, S.fstamp.p, t,
                                                        S.mom.p, S.mstamp.p, s0, coef_r, coef_m,
                                                        S.g, S.op.dev, S.n1);
            GD_LAUNCH_CHECK();
            int64_t P = 0;
            double sgamma = 0.0;
            int64_t fnext = S.scatter_and_filter(f, t, &P, &sgamma);
            double prev = rep->l1_log[rep->n_logs];
            S.reduce_l1_min(lm);
            report_push_log(rep, cap, P, prev > 0 ? sgamma / prev : 0.0, lm[0], 0, f);
            if (lm[1] < rep->min_residual) rep->min_residual = lm[1];
            rep->total_ops += P;
            rep->pushes += f;
            rep->sweeps += 1;
            f = fnext;
            ++t;
            if (lm[0] > 10.0 * b_l1) {
                rep->converged = 0;
                rep->diverged = 1;
                break;
            }
        }
        S.finish(x, r, rep);
    });
}

}  // extern "C"
