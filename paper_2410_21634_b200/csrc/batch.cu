// batch.cu -- batched multi-seed LocalGD-PPR, the throughput path.
//
// Semantics: for every seed s the run equals local_gd(make_ppr_system(g,
// alpha, s, eps)) (src/local_solvers.py:428-470): the same frontier SETS
// S_t, hence the same sweeps, vol(S_t) and operation counts; x agrees to
// the rounding of the scatter order (atomics instead of the sequential
// fold; exact order is exact.cu's job).
//
// Design (B200):
//  * `slots` seeds run concurrently, each with dense x/r vectors in HBM
//    (slot-major, n doubles each).  They are never memset: every touched
//    coordinate is on a per-slot dirty list and is reset after extraction.
//  * One persistent cooperative kernel runs all sweeps of a wave of seeds;
//    sweeps of all slots advance together ("rounds"), with two grid
//    barriers per round:
//      phase A (one thread per frontier entry): vals = r[u]; x[u] += vals;
//              r[u] = -0.0 (a pushed node; +0.0 means "never touched");
//              c_u = fl(vals * fl(fl(1/d_u)*(1-alpha))) staged per entry.
//      phase B (arc-balanced: every warp owns an equal slice of the round's
//              concatenated arc space): r[v] += c_u with a returning fp64
//              atomic.  The returned old value decides, without any extra
//              memory traffic, (1) first touch (old == +0.0 -> dirty list)
//              and (2) frontier entry: residuals only grow inside a round
//              (all c_u > 0, pushed nodes restart from 0), so exactly one
//              arc observes old < theta_v <= old + c; that arc appends
//              (slot, v) to S_{t+1}.  No candidate list, no filter pass.
//  * Frontier appends reserve (entries, arcs) with ONE packed 64-bit
//    atomic per warp, so entry order and arc-offset order agree and the
//    next round's arc space is a prefix sum for free.
//  * Thresholds come from an L2-resident int32 degree array
//    (theta_v = fl(eps*alpha*d_v)), not a per-node double.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <vector>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace gd {
namespace {

constexpr int BT = 512;  // threads per block of the round kernel
constexpr int CNT_SHIFT = 36;
constexpr unsigned long long ARC_MASK = (1ULL << CNT_SHIFT) - 1ULL;
constexpr unsigned FULL = 0xffffffffu;

struct RoundArgs {
    DevGraph g;
    double beta;    // 1 - alpha
    double tcoeff;  // eps * alpha
    int64_t n;
    int64_t ld;     // slot stride (n rounded up to even: 16 B aligned slots)
    int64_t max_sweeps;
    int64_t fcap;
    double *x, *r;
    int32_t *dirty, *pushed;
    unsigned long long *dirty_cnt, *pushed_cnt;
    int64_t *fkey[2], *farc[2];
    int64_t *frow;
    double *fcval;
    unsigned long long *fctr;  // [2] packed (entries << 36 | arcs)
    unsigned long long *s_ops, *s_pushes, *s_negz;
    int32_t *s_last, *s_conv;
    int32_t *overflow;
    const int32_t *perm;  // caller id -> relabeled id (nullable)
};

__device__ __forceinline__ double theta_deg(double tc, int32_t d) {
    return d > 0 ? __dmul_rn(tc, (double)d) : __longlong_as_double(0x7ff0000000000000LL);
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Append `item` to the per-slot list k (warp-aggregated by slot).
__device__ __forceinline__ void slot_append(bool flag, int32_t k, int32_t item, int64_t n,
                                            int32_t *list, unsigned long long *cnt) {
    unsigned am = __ballot_sync(FULL, flag);
    if (!flag) return;
    unsigned peers = __match_any_sync(am, k);
    int leader = __ffs(peers) - 1;
    int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(cnt + k, (unsigned long long)__popc(peers));
    base = __shfl_sync(peers, base, leader);
    list[(int64_t)k * n + (int64_t)base + __popc(peers & lanemask_lt())] = item;
}

// Count `flag` lanes into the per-slot counter k (warp-aggregated).
__device__ __forceinline__ void slot_count(bool flag, int32_t k, unsigned long long *cnt) {
    unsigned am = __ballot_sync(FULL, flag);
    if (!flag) return;
    unsigned peers = __match_any_sync(am, k);
    if ((int)(threadIdx.x & 31) == __ffs(peers) - 1)
        atomicAdd(cnt + k, (unsigned long long)__popc(peers));
}

// Append (k, v) with degree d to the next frontier (warp-aggregated, one
// packed atomic reserving entry slots and arc range together).
__device__ __forceinline__ void frontier_append(bool flag, int32_t k, int32_t v, int32_t d,
                                                const RoundArgs &A, int nxt) {
    unsigned am = __ballot_sync(FULL, flag);
    if (am == 0) return;
    int lane = threadIdx.x & 31;
    unsigned long long incl = flag ? (unsigned long long)d : 0ULL;
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    unsigned long long total = __shfl_sync(FULL, incl, 31);
    unsigned long long old = 0;
    if (lane == 0)
        old = atomicAdd(A.fctr + nxt, ((unsigned long long)__popc(am) << CNT_SHIFT) + total);
    old = __shfl_sync(FULL, old, 0);
    if (flag) {
        int64_t idx = (int64_t)(old >> CNT_SHIFT) + __popc(am & lanemask_lt());
        if (idx < A.fcap) {
            A.fkey[nxt][idx] = ((int64_t)k << 32) | (uint32_t)v;
            A.farc[nxt][idx] = (int64_t)(old & ARC_MASK) + (int64_t)(incl - (unsigned long long)d);
        } else {
            A.overflow[0] = 1;
        }
    }
}

__global__ void __launch_bounds__(BT) k_rounds(RoundArgs A) {
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const int64_t gtid = blockIdx.x * (int64_t)BT + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * BT;
    const int64_t W = nthreads >> 5, wid = gtid >> 5;
    for (int32_t t = 0;; ++t) {
        const int cur = t & 1, nxt = cur ^ 1;
        const unsigned long long packed = *(volatile unsigned long long *)(A.fctr + cur);
        const int64_t F = (int64_t)(packed >> CNT_SHIFT);
        const int64_t P = (int64_t)(packed & ARC_MASK);
        if (F == 0) break;
        if (t >= A.max_sweeps || F > A.fcap) {
            for (int64_t e = gtid; e < F && e < A.fcap; e += nthreads)
                A.s_conv[A.fkey[cur][e] >> 32] = 0;
            break;
        }
        // ---------------- phase A: push the frontier entries ----------------
        if (gtid == 0) A.fctr[nxt] = 0ULL;
        const int64_t *fk = A.fkey[cur];
        for (int64_t e0 = gtid - lane; e0 < F; e0 += nthreads) {  // warp-uniform trip count
            const int64_t e = e0 + lane;
            const bool live = e < F;
            int32_t k = 0, u = 0, d = 0;
            if (live) {
                int64_t key = fk[e];
                k = (int32_t)(key >> 32);
                u = (int32_t)(key & 0xffffffffLL);
                int64_t idx = (int64_t)k * A.ld + u;
                double val = A.r[idx];
                double xo = A.x[idx];
                A.x[idx] = __dadd_rn(xo, val);
                A.r[idx] = -0.0;
                d = A.g.deg[u];
                A.frow[e] = A.g.row[u];
                A.fcval[e] = __dmul_rn(val, __dmul_rn(__ddiv_rn(1.0, (double)d), A.beta));
                u = __double_as_longlong(xo) == 0 ? u : -1;  // first push of u?
            }
            slot_append(live && u >= 0, k, u, A.ld, A.pushed, A.pushed_cnt);
            // per-slot counters, aggregated over lanes of the same slot
            unsigned am = __ballot_sync(FULL, live);
            if (live) {
                unsigned peers = __match_any_sync(am, k);
                unsigned sum = __reduce_add_sync(peers, (unsigned)d);
                if (lane == __ffs(peers) - 1) {
                    atomicAdd(A.s_ops + k, (unsigned long long)sum);
                    atomicAdd(A.s_pushes + k, (unsigned long long)__popc(peers));
                    A.s_last[k] = t;
                }
            }
        }
        grid.sync();
        // ---------------- phase B: arc-balanced scatter ----------------------
        const int64_t p0 = (int64_t)(((unsigned long long)P * (unsigned long long)wid) / W);
        const int64_t p1 = (int64_t)(((unsigned long long)P * (unsigned long long)(wid + 1)) / W);
        if (p0 < p1) {
            const int64_t *fa = A.farc[cur];
            // 32-ary search: entry e with fa[e] <= p0 < fa[e+1]
            int64_t lo = 0, hi = F;
            while (hi - lo > 32) {
                int64_t step = (hi - lo + 31) >> 5;
                int64_t i = lo + lane * step;
                unsigned b = __ballot_sync(FULL, i < hi && fa[i] <= p0);
                lo += (int64_t)(31 - __clz(b)) * step;
                hi = min(hi, lo + step);
            }
            int64_t e;
            {
                int64_t i = lo + lane;
                unsigned b = __ballot_sync(FULL, i < hi && fa[i] <= p0);
                e = lo + (31 - __clz(b));
            }
            for (int64_t base = p0; base < p1; base += 32) {
                const int64_t wi = e + 1 + lane;
                const int64_t st = wi < F ? fa[wi] : INT64_MAX;
                const int64_t pos = st - base;  // >= 1
                const unsigned starts = __reduce_or_sync(FULL, pos < 32 ? (1u << pos) : 0u);
                const unsigned upto = __ballot_sync(FULL, pos <= 32);
                const int64_t me = e + __popc(starts & ((2u << lane) - 1u));
                const int64_t p = base + lane;
                bool valid = p < p1;
                bool first = false, cross = false, negz = false;
                int32_t k = 0, v = 0, dv = 0;
                if (valid) {
                    const int64_t key = A.fkey[cur][me];
                    k = (int32_t)(key >> 32);
                    const double c = A.fcval[me];
                    v = A.g.col[A.frow[me] + (p - fa[me])];
                    dv = A.g.deg[v];
                    const double th = theta_deg(A.tcoeff, dv);
                    const double old = atomicAdd(A.r + (int64_t)k * A.ld + v, c);
                    const double nw = __dadd_rn(old, c);
                    first = __double_as_longlong(old) == 0;
                    negz = __double_as_longlong(old) == (long long)0x8000000000000000ULL;
                    cross = (old < th) && (nw >= th);
                }
                slot_append(first, k, v, A.ld, A.dirty, A.dirty_cnt);
                slot_count(negz, k, A.s_negz);
                frontier_append(cross, k, v, dv, A, nxt);
                e += __popc(upto);
            }
        }
        grid.sync();
    }
}

// Seeds -> slots: r[s] = alpha, dirty = {s}, S_0 = {s} if alpha >= theta_s.
__global__ void k_wave_init(RoundArgs A, const int64_t *__restrict__ seeds, int64_t m,
                            double alpha) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    int32_t s = (int32_t)seeds[k];
    if (A.perm) s = A.perm[s];
    A.r[k * A.ld + s] = alpha;
    A.dirty[k * A.ld] = s;
    A.dirty_cnt[k] = 1;
    A.pushed_cnt[k] = 0;
    A.s_ops[k] = 0;
    A.s_pushes[k] = 0;
    A.s_negz[k] = 0;
    A.s_last[k] = -1;
    A.s_conv[k] = 1;
    int32_t d = A.g.deg[s];
    if (alpha >= theta_deg(A.tcoeff, d)) {
        unsigned long long old = atomicAdd(A.fctr, (1ULL << CNT_SHIFT) + (unsigned long long)d);
        int64_t idx = (int64_t)(old >> CNT_SHIFT);
        if (idx < A.fcap) {
            A.fkey[0][idx] = (k << 32) | (uint32_t)s;
            A.farc[0][idx] = (int64_t)(old & ARC_MASK);
        }
    }
}

struct OutArgs {
    int64_t *sweeps, *ops, *pushes, *support, *xoff, *xcnt;
    int32_t *conv;
    int32_t *xnodes;
    double *xvals;
    int64_t xcap;
    unsigned long long *cursor;
    const int32_t *inv;  // relabeled id -> caller id (nullable)
};

// Per slot: extract x over the pushed list (and zero it), write the seed's
// counters.  support = |dirty| - |pushed nodes whose r is still -0.0|: every
// push writes -0.0, the first later contribution observes it (s_negz).
__global__ void k_wave_extract(RoundArgs A, OutArgs O, int64_t seed_base) {
    const int k = blockIdx.x;
    const int64_t off = (int64_t)k * A.ld;
    __shared__ unsigned long long s_base;
    const int64_t pc = (int64_t)A.pushed_cnt[k];
    if (threadIdx.x == 0) s_base = atomicAdd(O.cursor, (unsigned long long)pc);
    __syncthreads();
    const int64_t b = (int64_t)s_base;
    for (int64_t i = threadIdx.x; i < pc; i += blockDim.x) {
        int32_t u = A.pushed[off + i];
        double xv = A.x[off + u];
        A.x[off + u] = 0.0;
        if (b + i < O.xcap) {
            O.xnodes[b + i] = O.inv ? O.inv[u] : u;
            O.xvals[b + i] = xv;
        }
    }
    if (threadIdx.x == 0) {
        const int64_t si = seed_base + k;
        const int64_t pushes = (int64_t)A.s_pushes[k];
        O.sweeps[si] = (int64_t)A.s_last[k] + 1;
        O.ops[si] = (int64_t)A.s_ops[k];
        O.pushes[si] = pushes;
        O.conv[si] = A.s_conv[k];
        O.support[si] = (int64_t)A.dirty_cnt[k] - (pushes - (int64_t)A.s_negz[k]);
        O.xoff[si] = b;
        O.xcnt[si] = pc;
    }
}

// Reset r of every slot: a write-only stream of zeros over the slot when its
// touched set is large (a random 8 B reset costs a 32 B sector RMW), else a
// scatter over the dirty list.  grid = (RESET_CHUNKS, slots).
constexpr int RESET_CHUNKS = 32;
__global__ void k_wave_reset(RoundArgs A) {
    const int k = blockIdx.y;
    const int64_t off = (int64_t)k * A.ld;
    const int64_t dc = (int64_t)A.dirty_cnt[k];
    if (dc * 8 > A.ld) {
        double2 *r2 = reinterpret_cast<double2 *>(A.r + off);
        const int64_t h = A.ld >> 1;
        const int64_t per = (h + RESET_CHUNKS - 1) / RESET_CHUNKS;
        const int64_t lo = blockIdx.x * per, hi = min(h, lo + per);
        for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) r2[i] = make_double2(0.0, 0.0);
    } else {
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < dc;
             i += (int64_t)RESET_CHUNKS * blockDim.x)
            A.r[off + A.dirty[off + i]] = 0.0;
    }
}

// ---- degree relabeling (setup): new id = rank by descending degree ------
__global__ void k_iota(int32_t *ids, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        ids[i] = (int32_t)i;
}

__global__ void k_invert(const int32_t *__restrict__ inv, int32_t *__restrict__ perm,
                         const int32_t *__restrict__ dsorted, int64_t *__restrict__ deg64,
                         int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        perm[inv[i]] = (int32_t)i;
        deg64[i] = dsorted[i];
    }
}

__global__ void k_remap_rows(DevGraph g, const int32_t *__restrict__ inv,
                             const int32_t *__restrict__ perm, const int64_t *__restrict__ row2,
                             int32_t *__restrict__ col2) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < g.n;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int32_t o = inv[i];
        const int64_t rs = g.row[o], d = g.row[o + 1] - rs, rs2 = row2[i];
        for (int64_t j = lane; j < d; j += 32) col2[rs2 + j] = perm[g.col[rs + j]];
    }
}

}  // namespace
}  // namespace gd

using namespace gd;

struct gd_batch {
    const gd_graph *G;   // caller's graph
    gd_graph *R = nullptr;  // degree-relabeled copy (when p.relabel)
    DBuf<int32_t> perm, inv;
    gd_batch_params p;
    int slots;
    int grid;
    int64_t fcap, xcap;
    DBuf<double> x, r, fcval;
    DBuf<int32_t> dirty, pushed, s_last, s_conv, overflow;
    DBuf<unsigned long long> dirty_cnt, pushed_cnt, fctr, s_ops, s_pushes, s_negz, cursor;
    DBuf<int64_t> fkey0, fkey1, farc0, farc1, frow;
    // results
    DBuf<int64_t> sweeps, ops, pushes, support, xoff, xcnt;
    DBuf<int32_t> conv, xnodes;
    DBuf<double> xvals;
    std::vector<cudaEvent_t> ev;
    double last_ms = 0.0;
    int64_t last_launches = 0;

    const gd_graph *work() const { return R ? R : G; }

    RoundArgs args() {
        RoundArgs A{};
        A.g = work()->view();
        A.beta = 1.0 - p.alpha;
        A.tcoeff = p.eps * p.alpha;
        A.n = G->n;
        A.ld = (G->n + 1) & ~1LL;
        A.max_sweeps = p.max_sweeps;
        A.fcap = fcap;
        A.x = x.p; A.r = r.p; A.dirty = dirty.p; A.pushed = pushed.p;
        A.dirty_cnt = dirty_cnt.p; A.pushed_cnt = pushed_cnt.p;
        A.fkey[0] = fkey0.p; A.fkey[1] = fkey1.p; A.farc[0] = farc0.p; A.farc[1] = farc1.p;
        A.frow = frow.p; A.fcval = fcval.p; A.fctr = fctr.p;
        A.s_ops = s_ops.p; A.s_pushes = s_pushes.p; A.s_last = s_last.p; A.s_conv = s_conv.p;
        A.s_negz = s_negz.p;
        A.overflow = overflow.p;
        A.perm = R ? perm.p : nullptr;
        return A;
    }
    ~gd_batch() {
        for (auto e : ev) cudaEventDestroy(e);
        delete R;
    }
};

static void batch_run(gd_batch *B, const int64_t *d_seeds, int64_t n_seeds, cudaStream_t st) {
    const int64_t n = B->G->n;
    B->sweeps.ensure(n_seeds ? n_seeds : 1); B->ops.ensure(n_seeds ? n_seeds : 1);
    B->pushes.ensure(n_seeds ? n_seeds : 1); B->support.ensure(n_seeds ? n_seeds : 1);
    B->xoff.ensure(n_seeds ? n_seeds : 1); B->xcnt.ensure(n_seeds ? n_seeds : 1);
    B->conv.ensure(n_seeds ? n_seeds : 1);
    GD_CUDA(cudaMemsetAsync(B->cursor.p, 0, sizeof(unsigned long long), st));
    GD_CUDA(cudaMemsetAsync(B->overflow.p, 0, sizeof(int32_t), st));
    const int64_t waves = (n_seeds + B->slots - 1) / B->slots;
    while ((int64_t)B->ev.size() < 2 * waves) {
        cudaEvent_t e;
        GD_CUDA(cudaEventCreate(&e));
        B->ev.push_back(e);
    }
    OutArgs O{B->sweeps.p, B->ops.p, B->pushes.p, B->support.p, B->xoff.p, B->xcnt.p,
              B->conv.p, B->xnodes.p, B->xvals.p, B->xcap, B->cursor.p,
              B->R ? B->inv.p : nullptr};
    RoundArgs A = B->args();
    int64_t launches = 0;
    for (int64_t w = 0; w < waves; ++w) {
        const int64_t base = w * B->slots;
        const int64_t m = n_seeds - base < B->slots ? n_seeds - base : B->slots;
        GD_CUDA(cudaMemsetAsync(B->fctr.p, 0, 2 * sizeof(unsigned long long), st));
        k_wave_init<<<(int)((m + 255) / 256), 256, 0, st>>>(A, d_seeds + base, m, B->p.alpha);
        GD_LAUNCH_CHECK();
        GD_CUDA(cudaEventRecord(B->ev[2 * w], st));
        void *kargs[] = {&A};
        GD_CUDA(cudaLaunchCooperativeKernel((const void *)k_rounds, dim3(B->grid), dim3(BT), kargs,
                                            0, st));
        GD_CUDA(cudaEventRecord(B->ev[2 * w + 1], st));
        k_wave_extract<<<(int)m, 256, 0, st>>>(A, O, base);
        k_wave_reset<<<dim3(RESET_CHUNKS, (unsigned)m), 256, 0, st>>>(A);
        GD_LAUNCH_CHECK();
        launches += 4;
    }
    GD_CUDA(cudaStreamSynchronize(st));
    double ms = 0.0;
    for (int64_t w = 0; w < waves; ++w) {
        float f = 0.f;
        GD_CUDA(cudaEventElapsedTime(&f, B->ev[2 * w], B->ev[2 * w + 1]));
        ms += f;
    }
    B->last_ms = ms;
    B->last_launches = launches;
}

// Degree-descending renumbering of the graph on the device (one-time setup).
static void build_relabeled(gd_batch *B) {
    const gd_graph *G = B->G;
    const int64_t n = G->n;
    if (n == 0) return;
    DevGraph g = G->view();
    DBuf<int32_t> ids(n), dsorted(n);
    B->perm.alloc(n);
    B->inv.alloc(n);
    const int blocks = 4 * n_sms(G->device);
    k_iota<<<blocks, 256>>>(ids.p, n);
    GD_LAUNCH_CHECK();
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, g.deg, dsorted.p, ids.p, B->inv.p,
                                              (int64_t)n);
    DBuf<char> tmp(bytes ? bytes : 1);
    cub::DeviceRadixSort::SortPairsDescending(tmp.p, bytes, g.deg, dsorted.p, ids.p, B->inv.p,
                                              (int64_t)n);
    gd_graph *R = new gd_graph();
    B->R = R;
    R->device = G->device;
    R->n = n;
    R->n_arcs = G->n_arcs;
    R->d_max = G->d_max;
    R->row.alloc(n + 1);
    R->col.alloc(G->n_arcs ? G->n_arcs : 1);
    R->deg.alloc(n);
    DBuf<int64_t> deg64(n + 1);
    k_invert<<<blocks, 256>>>(B->inv.p, B->perm.p, dsorted.p, deg64.p, n);
    GD_LAUNCH_CHECK();
    GD_CUDA(cudaMemset(deg64.p + n, 0, sizeof(int64_t)));
    bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, deg64.p, R->row.p, n + 1);
    tmp.ensure(bytes ? bytes : 1);
    cub::DeviceScan::ExclusiveSum(tmp.p, bytes, deg64.p, R->row.p, n + 1);
    GD_CUDA(cudaMemcpy(R->deg.p, dsorted.p, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice));
    k_remap_rows<<<blocks, 256>>>(g, B->inv.p, B->perm.p, R->row.p, R->col.p);
    GD_LAUNCH_CHECK();
    GD_CUDA(cudaDeviceSynchronize());
}

extern "C" {

int gd_batch_create(const gd_graph *G, const gd_batch_params *p, gd_batch **out) {
    return guarded([&] {
        GD_CHECK_ARG(G && p && out, "null pointer");
        GD_CHECK_ARG(p->method == GD_M_LOCAL_GD, "only GD_M_LOCAL_GD is batched");
        GD_CHECK_ARG(p->alpha > 0.0 && p->alpha <= 1.0, "alpha must be in (0, 1]");
        GD_CHECK_ARG(p->eps > 0.0, "eps must be positive");
        GD_CHECK_ARG(G->n_arcs < (1LL << CNT_SHIFT), "too many arcs");
        GD_CUDA(cudaSetDevice(G->device));
        const int64_t n = G->n ? G->n : 1;
        gd_batch *B = new gd_batch();
        try {
            B->G = G;
            B->p = *p;
            if (p->relabel) build_relabeled(B);
            if (B->p.max_sweeps <= 0) B->p.max_sweeps = 1000000;
            int slots = p->slots;
            if (slots <= 0) {
                size_t fr = 0, tot = 0;
                GD_CUDA(cudaMemGetInfo(&fr, &tot));
                int64_t by_mem = (int64_t)(fr / 4) / (n * 24);
                slots = (int)(by_mem < 256 ? (by_mem < 1 ? 1 : by_mem) : 256);
            }
            B->slots = slots;
            int64_t fc = p->frontier_cap > 0 ? p->frontier_cap : (int64_t)slots * n;
            if (p->frontier_cap <= 0 && fc > (64LL << 20)) fc = 64LL << 20;
            B->fcap = fc;
            B->xcap = p->out_cap > 0 ? p->out_cap : (16LL << 20);
            const size_t sn = (size_t)slots * (size_t)((n + 1) & ~1LL);
            B->x.alloc(sn); B->r.alloc(sn);
            GD_CUDA(cudaMemset(B->x.p, 0, sizeof(double) * sn));
            GD_CUDA(cudaMemset(B->r.p, 0, sizeof(double) * sn));
            B->dirty.alloc(sn); B->pushed.alloc(sn);
            B->dirty_cnt.alloc(slots); B->pushed_cnt.alloc(slots);
            B->s_ops.alloc(slots); B->s_pushes.alloc(slots); B->s_negz.alloc(slots);
            B->s_last.alloc(slots); B->s_conv.alloc(slots);
            B->fctr.alloc(2); B->cursor.alloc(1); B->overflow.alloc(1);
            B->fkey0.alloc(fc); B->fkey1.alloc(fc); B->farc0.alloc(fc); B->farc1.alloc(fc);
            B->frow.alloc(fc); B->fcval.alloc(fc);
            B->xnodes.alloc(B->xcap); B->xvals.alloc(B->xcap);
            int per_sm = 0;
            GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rounds, BT, 0));
            GD_CHECK_ARG(per_sm > 0, "round kernel does not fit on an SM");
            B->grid = per_sm * n_sms(G->device);
        } catch (...) {
            delete B;
            throw;
        }
        *out = B;
    });
}

int gd_batch_destroy(gd_batch *b) {
    delete b;
    return GD_OK;
}

int gd_batch_solve_device(gd_batch *B, const int64_t *d_seeds, int64_t n_seeds,
                          gd_batch_result *res, void *stream) {
    return guarded([&] {
        GD_CHECK_ARG(B && res && (d_seeds || n_seeds == 0), "null pointer");
        GD_CUDA(cudaSetDevice(B->G->device));
        cudaStream_t st = (cudaStream_t)stream;
        for (int attempt = 0; attempt < 2; ++attempt) {
            batch_run(B, d_seeds, n_seeds, st);
            int32_t ovf = 0;
            unsigned long long used = 0;
            GD_CUDA(cudaMemcpy(&ovf, B->overflow.p, sizeof(ovf), cudaMemcpyDeviceToHost));
            GD_CUDA(cudaMemcpy(&used, B->cursor.p, sizeof(used), cudaMemcpyDeviceToHost));
            if (ovf) {
                set_error("frontier capacity %lld exceeded; raise frontier_cap",
                          (long long)B->fcap);
                throw Error{GD_ERR_CAPACITY};
            }
            res->x_total = (int64_t)used;
            if ((int64_t)used <= B->xcap) break;
            GD_CHECK_ARG(attempt == 0, "output pool sizing failed");
            B->xcap = (int64_t)used + (int64_t)used / 8 + 1024;  // grow and redo
            B->xnodes.alloc(B->xcap);
            B->xvals.alloc(B->xcap);
        }
        res->sweeps = B->sweeps.p; res->total_ops = B->ops.p; res->pushes = B->pushes.p;
        res->support = B->support.p; res->converged = B->conv.p; res->x_offset = B->xoff.p;
        res->x_count = B->xcnt.p; res->x_nodes = B->xnodes.p; res->x_vals = B->xvals.p;
        res->kernel_launches = B->last_launches;
    });
}

int gd_batch_solve_host(gd_batch *B, const int64_t *seeds, int64_t n_seeds, int64_t *sweeps,
                        int64_t *total_ops, int64_t *pushes, int32_t *converged,
                        int64_t *x_offset, int64_t *x_count, int32_t *x_nodes, double *x_vals,
                        int64_t x_cap, int64_t *x_total, void *stream) {
    return guarded([&] {
        GD_CHECK_ARG(B && (seeds || n_seeds == 0) && x_total, "null pointer");
        GD_CUDA(cudaSetDevice(B->G->device));
        cudaStream_t st = (cudaStream_t)stream;
        DBuf<int64_t> ds(n_seeds ? n_seeds : 1);
        GD_CUDA(cudaMemcpyAsync(ds.p, seeds, sizeof(int64_t) * n_seeds, cudaMemcpyHostToDevice, st));
        gd_batch_result res{};
        int rc = gd_batch_solve_device(B, ds.p, n_seeds, &res, stream);
        if (rc != GD_OK) throw Error{rc};
        *x_total = res.x_total;
        auto d2h = [&](void *dst, const void *src, size_t bytes) {
            if (dst && bytes) GD_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
        };
        d2h(sweeps, res.sweeps, sizeof(int64_t) * n_seeds);
        d2h(total_ops, res.total_ops, sizeof(int64_t) * n_seeds);
        d2h(pushes, res.pushes, sizeof(int64_t) * n_seeds);
        d2h(converged, res.converged, sizeof(int32_t) * n_seeds);
        d2h(x_offset, res.x_offset, sizeof(int64_t) * n_seeds);
        d2h(x_count, res.x_count, sizeof(int64_t) * n_seeds);
        if (res.x_total > x_cap) {
            GD_CUDA(cudaStreamSynchronize(st));
            set_error("x buffers hold %lld pairs, %lld needed", (long long)x_cap,
                      (long long)res.x_total);
            throw Error{GD_ERR_CAPACITY};
        }
        d2h(x_nodes, res.x_nodes, sizeof(int32_t) * res.x_total);
        d2h(x_vals, res.x_vals, sizeof(double) * res.x_total);
        GD_CUDA(cudaStreamSynchronize(st));
    });
}

int gd_batch_last_kernel_ms(const gd_batch *B, double *ms) {
    if (!B || !ms) return GD_ERR_ARG;
    *ms = B->last_ms;
    return GD_OK;
}

}  // extern "C"
