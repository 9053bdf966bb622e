// fifo_batch.cu -- batched LocalSOR / LocalGS-PPR: one warp per seed.
//
// Every seed is an independent replay of the reference FIFO push
// (_push_kernel src/local_solvers.py:48-188 via local_sor :221-253) on
// b = alpha e_s: same pops, same enqueue order (ballot + popc over 32
// consecutive arcs of the row keeps CSR order), same fl() sequence -- so x,
// the sweep count and the operation count are bit-identical with the
// reference, per seed.  A warp owns a slot (dense x / r, ring queue, queue
// marks, touched marks) and pulls seeds from a global counter until the
// batch is exhausted; the slot is cleaned by walking its touched list.
//
// Bound: latency of the per-pop dependent chain (a Gauss-Seidel push cannot
// start before the previous one finished); throughput comes from many
// warps, i.e. from slot count x SM residency, sized to HBM capacity.
#include "common.cuh"

namespace gd {
struct RPool {  // (batch.cu)
    int64_t *off, *cnt;
    int32_t *nodes;
    double *vals;
    int64_t cap;
    unsigned long long *cursor;
    unsigned long long *scratch;
};
namespace {

constexpr int FB_THREADS = 256;
constexpr unsigned FULL = 0xffffffffu;

struct FifoBatchArgs {
    DevGraph g;
    double alpha, beta, tcoeff, omega;
    int sgn;
    int64_t n, ld, max_sweeps, n_seeds, xcap;
    double *x, *r;
    int32_t *queue;        // ld + 2 per slot
    uint32_t *qmark;       // queued-node bit map per slot (qw words): L2-resident
    int64_t qw;
    int32_t *touched;      // touched list per slot (ld)
    int32_t *plist;        // pushed-node list per slot (ld): x support
    // optional sparse r out (want_r; r_off null = not wanted)
    int64_t *r_off, *r_cnt;
    int32_t *r_nodes;
    double *r_vals;
    int64_t rcap;
    unsigned long long *rcursor;
    const int64_t *seeds;
    unsigned long long *next_seed, *cursor;
    int64_t *sweeps, *ops, *pushes, *xoff, *xcnt;
    int32_t *conv;
    int32_t *xnodes;
    double *xvals;
    int nslots;
};

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ double theta_d(double tc, int32_t d) {
    return d > 0 ? __dmul_rn(tc, (double)d) : __longlong_as_double(0x7ff0000000000000LL);
}

__global__ void __launch_bounds__(FB_THREADS) k_fifo_batch(FifoBatchArgs A) {
    const int lane = threadIdx.x & 31;
    const int slot = (int)((blockIdx.x * (int64_t)FB_THREADS + threadIdx.x) >> 5);
    if (slot >= A.nslots) return;
    const int64_t off = (int64_t)slot * A.ld;
    double *x = A.x + off, *r = A.r + off;
    int32_t *queue = A.queue + (int64_t)slot * (A.ld + 2);
    uint32_t *qmark = A.qmark + (int64_t)slot * A.qw;
    int32_t *touched = A.touched + off;
    int32_t *plist = A.plist + off;
    const int64_t sent = A.n, qcap = A.n + 2;

    for (;;) {
        unsigned long long si = 0;
        if (lane == 0) si = atomicAdd(A.next_seed, 1ULL);
        si = __shfl_sync(FULL, si, 0);
        if ((int64_t)si >= A.n_seeds) break;
        const int32_t s = (int32_t)A.seeds[si];
        // b = alpha e_s, x = 0 (slot is clean); seed enqueue (:59-69).  A node
        // is "touched" once its r word is not +0.0: residuals that become
        // exactly zero are stored as -0.0, which adds like +0.0.
        int64_t ntouch = 1, npl = 0;
        if (lane == 0) {
            r[s] = A.alpha;
            touched[0] = s;
        }
        __syncwarp();
        int64_t front = 0, rear = 0;
        const double ths = theta_d(A.tcoeff, A.g.deg[s]);
        const bool act0 = A.sgn ? fabs(A.alpha) >= ths : A.alpha >= ths;
        int64_t sweeps = 0, ops = 0, pushes = 0;
        int conv = 1;
        if (act0) {
            if (lane == 0) {
                queue[0] = s;
                qmark[s >> 5] |= 1u << (s & 31);
                queue[1] = (int32_t)sent;
            }
            rear = 2;
            int64_t svol = 0;
            // software pipeline: the next pop's node, r, degree and row are
            // loaded while the current pop scatters (r re-read if it was hit)
            int64_t pu = -1, prs = 0;
            double pr = 0.0, px = 0.0;
            int32_t pd = 0, pcol = 0;  // (pcol: this lane's first neighbour of the next pop)
            __syncwarp();
            for (;;) {
                const int64_t u = queue[front];
                front = (front + 1 == qcap) ? 0 : front + 1;
                if (u == sent) {  // sweep boundary (:102-144)
                    ops += svol;
                    sweeps += 1;
                    pu = -1;
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
                double ru, xu;
                int32_t d, c0;
                int64_t rs;
                if (u == pu) {  // (x[u] is written only by u's own pops: px is exact)
                    ru = pr;
                    d = pd;
                    rs = prs;
                    c0 = pcol;
                    xu = px;
                } else {
                    ru = r[u];
                    d = A.g.deg[u];
                    rs = A.g.row[u];
                    c0 = lane < d ? A.g.col[rs + lane] : 0;
                    xu = x[u];
                }
                pu = -1;
                if (lane == 0) atomicAnd(qmark + (u >> 5), ~(1u << (u & 31)));
                const double th = theta_d(A.tcoeff, d);
                if (A.sgn ? fabs(ru) < th : ru < th) {
                    __syncwarp();
                    continue;
                }
                if (front != rear) {  // prefetch the next pop
                    const int64_t nx = queue[front];
                    if (nx != sent) {
                        pu = nx;
                        pr = r[nx];
                        pd = A.g.deg[nx];
                        prs = A.g.row[nx];
                        px = x[nx];
                        pcol = lane < pd ? A.g.col[prs + lane] : 0;
                    }
                }
                svol += d;
                pushes += 1;
                const double res = __dmul_rn(A.omega, ru);
                if (__double_as_longlong(xu) == 0) {  // first push of u (x never returns to +0.0)
                    if (lane == 0) plist[npl] = (int32_t)u;
                    ++npl;
                }
                if (lane == 0) {
                    const double xn = __dadd_rn(xu, res);  // x_gain = 1
                    x[u] = __double_as_longlong(xn) == 0 ? -0.0 : xn;
                    const double rn = __dsub_rn(ru, res);
                    r[u] = __double_as_longlong(rn) == 0 ? -0.0 : rn;
                }
                const double w = __dmul_rn(__ddiv_rn(1.0, (double)d), A.beta);
                bool hit = false;
                for (int64_t base = 0; base < d; base += 32) {
                    const int64_t j = base + lane;
                    bool act = false, fresh = false;
                    int32_t v = 0;
                    if (j < d) {
                        v = base == 0 ? c0 : A.g.col[rs + j];
                        // the three loads of the arc, issued together
                        const double old = r[v];
                        const uint32_t qm = qmark[v >> 5];
                        const int32_t dv = A.g.deg[v];
                        const double rv = __dadd_rn(old, __dmul_rn(res, w));
                        r[v] = __double_as_longlong(rv) == 0 ? -0.0 : rv;
                        fresh = __double_as_longlong(old) == 0;
                        hit |= v == pu;
                        if (!((qm >> (v & 31)) & 1u)) {
                            const double tv = theta_d(A.tcoeff, dv);
                            act = A.sgn ? fabs(rv) >= tv : rv >= tv;
                        }
                    }
                    const unsigned bal = __ballot_sync(FULL, act);
                    if (act) {
                        int64_t q = rear + __popc(bal & lanemask_lt());
                        if (q >= qcap) q -= qcap;
                        queue[q] = v;
                        atomicOr(qmark + (v >> 5), 1u << (v & 31));
                    }
                    rear += __popc(bal);
                    if (rear >= qcap) rear -= qcap;
                    const unsigned fb = __ballot_sync(FULL, fresh);
                    if (fresh) touched[ntouch + __popc(fb & lanemask_lt())] = v;
                    ntouch += __popc(fb);
                }
                __syncwarp();
                if (__any_sync(FULL, hit)) pr = r[pu];  // the scatter changed the next pop's r
                const double ru2 = __dsub_rn(ru, res);  // self re-check (:176-185)
                if (A.sgn ? fabs(ru2) >= th : ru2 >= th) {
                    if (lane == 0) {
                        queue[rear] = (int32_t)u;
                        atomicOr(qmark + (u >> 5), 1u << (u & 31));
                    }
                    rear = (rear + 1 == qcap) ? 0 : rear + 1;
                }
                __syncwarp();
            }
        }
        // outputs: x over the pushed nodes with x != 0; then r back to +0.0
        // over the touched nodes (stores only) and, after a sweep cap, the
        // marks of the nodes still queued
        int64_t nx = 0;
        for (int64_t i = lane; i < npl; i += 32) nx += x[plist[i]] != 0.0;
        for (int o = 16; o > 0; o >>= 1) nx += __shfl_xor_sync(FULL, nx, o);
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(A.cursor, (unsigned long long)nx);
        base = __shfl_sync(FULL, base, 0);
        if (A.r_off) {  // sparse r out over the touched nodes (count, reserve, emit)
            int64_t nr = 0;
            for (int64_t i = lane; i < ntouch; i += 32) nr += r[touched[i]] != 0.0;
            for (int o = 16; o > 0; o >>= 1) nr += __shfl_xor_sync(FULL, nr, o);
            unsigned long long rb = 0;
            if (lane == 0) rb = atomicAdd(A.rcursor, (unsigned long long)nr);
            rb = __shfl_sync(FULL, rb, 0);
            if (lane == 0) {
                A.r_off[si] = (int64_t)rb;
                A.r_cnt[si] = nr;
            }
            int64_t wr = (int64_t)rb;
            for (int64_t i0 = 0; i0 < ntouch; i0 += 32) {
                const int64_t i = i0 + lane;
                int32_t v = 0;
                double rv = 0.0;
                if (i < ntouch) {
                    v = touched[i];
                    rv = r[v];
                    r[v] = 0.0;
                }
                const unsigned nzb = __ballot_sync(FULL, rv != 0.0);
                if (rv != 0.0) {
                    const int64_t at = wr + __popc(nzb & lanemask_lt());
                    if (at < A.rcap) {
                        A.r_nodes[at] = v;
                        A.r_vals[at] = rv;
                    }
                }
                wr += __popc(nzb);
            }
        } else {
            for (int64_t i = lane; i < ntouch; i += 32) r[touched[i]] = 0.0;
        }
        if (!conv)
            for (int64_t w = lane; w < A.qw; w += 32) qmark[w] = 0u;
        int64_t w = (int64_t)base;
        for (int64_t i0 = 0; i0 < npl; i0 += 32) {
            const int64_t i = i0 + lane;
            int32_t v = 0;
            double xv = 0.0;
            if (i < npl) {
                v = plist[i];
                xv = x[v];
                x[v] = 0.0;
            }
            const unsigned nzb = __ballot_sync(FULL, xv != 0.0);
            if (xv != 0.0) {
                const int64_t pos = w + __popc(nzb & lanemask_lt());
                if (pos < A.xcap) {
                    A.xnodes[pos] = v;
                    A.xvals[pos] = xv;
                }
            }
            w += __popc(nzb);
        }
        if (lane == 0) {
            A.sweeps[si] = sweeps;
            A.ops[si] = ops;
            A.pushes[si] = pushes;
            A.conv[si] = conv;
            A.xoff[si] = (int64_t)base;
            A.xcnt[si] = nx;
        }
        __syncwarp();
    }
}

// ---- small graphs: the same replay with the seed's state in shared memory --
// k_fifo_smem: one warp per CTA and seed, x, r, the queue marks and the ring
// queue in shared memory (graphs of up to ~4 K nodes: cora), so every step of
// a pop's dependent chain except the CSR reads is a shared-memory access.  The
// pops, enqueue order and fl() sequence are k_fifo_batch's (the reference's);
// values are stored as computed.  Between seeds the arrays are zero-filled;
// x goes out in node order.
__host__ inline size_t fifo_smem_bytes(int64_t n) {
    const int64_t ld = (n + 1) & ~1LL;
    return (size_t)(16 * ld + 4 * (ld / 32 + 1) + 4 * (n + 2)) + 16;
}

__global__ void __launch_bounds__(32) k_fifo_smem(FifoBatchArgs A) {
    extern __shared__ __align__(16) unsigned char fsm[];
    const int lane = threadIdx.x & 31;
    const int64_t n = A.n, ld = (n + 1) & ~1LL, qw = ld / 32 + 1;
    double *const x = reinterpret_cast<double *>(fsm);
    double *const r = x + ld;
    uint32_t *const qmark = reinterpret_cast<uint32_t *>(r + ld);
    int32_t *const queue = reinterpret_cast<int32_t *>(qmark + qw);
    const int64_t sent = n, qcap = n + 2;
    for (;;) {
        unsigned long long si = 0;
        if (lane == 0) si = atomicAdd(A.next_seed, 1ULL);
        si = __shfl_sync(FULL, si, 0);
        if ((int64_t)si >= A.n_seeds) break;
        for (int64_t i = lane; i < ld; i += 32) {
            x[i] = 0.0;
            r[i] = 0.0;
        }
        for (int64_t i = lane; i < qw; i += 32) qmark[i] = 0u;
        __syncwarp();
        const int32_t s = (int32_t)A.seeds[si];
        if (lane == 0) r[s] = A.alpha;
        int64_t front = 0, rear = 0;
        const double ths = theta_d(A.tcoeff, A.g.deg[s]);
        const bool act0 = A.sgn ? fabs(A.alpha) >= ths : A.alpha >= ths;
        int64_t sweeps = 0, ops = 0, pushes = 0;
        int conv = 1;
        if (act0) {
            if (lane == 0) {
                queue[0] = s;
                qmark[s >> 5] |= 1u << (s & 31);
                queue[1] = (int32_t)sent;
            }
            rear = 2;
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
                const double ru = r[u], xu = x[u];
                const int32_t d = A.g.deg[u];
                const int64_t rs = A.g.row[u];
                __syncwarp();
                if (lane == 0) qmark[u >> 5] &= ~(1u << (u & 31));
                const double th = theta_d(A.tcoeff, d);
                if (A.sgn ? fabs(ru) < th : ru < th) {
                    __syncwarp();
                    continue;
                }
                svol += d;
                pushes += 1;
                const double res = __dmul_rn(A.omega, ru);
                if (lane == 0) {
                    x[u] = __dadd_rn(xu, res);  // x_gain = 1
                    r[u] = __dsub_rn(ru, res);
                }
                __syncwarp();
                const double w = __dmul_rn(__ddiv_rn(1.0, (double)d), A.beta);
                for (int64_t base = 0; base < d; base += 32) {
                    const int64_t j = base + lane;
                    bool act = false;
                    int32_t v = 0;
                    if (j < d) {
                        v = A.g.col[rs + j];
                        const double rv = __dadd_rn(r[v], __dmul_rn(res, w));
                        r[v] = rv;
                        if (!((qmark[v >> 5] >> (v & 31)) & 1u)) {
                            const double tv = theta_d(A.tcoeff, A.g.deg[v]);
                            act = A.sgn ? fabs(rv) >= tv : rv >= tv;
                        }
                    }
                    const unsigned bal = __ballot_sync(FULL, act);
                    if (act) {
                        int64_t q = rear + __popc(bal & lanemask_lt());
                        if (q >= qcap) q -= qcap;
                        queue[q] = v;
                        atomicOr(qmark + (v >> 5), 1u << (v & 31));
                    }
                    rear += __popc(bal);
                    if (rear >= qcap) rear -= qcap;
                    __syncwarp();
                }
                const double ru2 = __dsub_rn(ru, res);  // self re-check (:176-185)
                if (A.sgn ? fabs(ru2) >= th : ru2 >= th) {
                    if (lane == 0) {
                        queue[rear] = (int32_t)u;
                        qmark[u >> 5] |= 1u << (u & 31);
                    }
                    rear = (rear + 1 == qcap) ? 0 : rear + 1;
                }
                __syncwarp();
            }
        }
        // x out in node order
        int64_t nx = 0;
        for (int64_t i = lane; i < n; i += 32) nx += x[i] != 0.0;
        for (int o = 16; o > 0; o >>= 1) nx += __shfl_xor_sync(FULL, nx, o);
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(A.cursor, (unsigned long long)nx);
        base = __shfl_sync(FULL, base, 0);
        int64_t wpos = (int64_t)base;
        for (int64_t i0 = 0; i0 < n; i0 += 32) {
            const int64_t i = i0 + lane;
            const double xv = i < n ? x[i] : 0.0;
            const unsigned nzb = __ballot_sync(FULL, xv != 0.0);
            if (xv != 0.0) {
                const int64_t pos = wpos + __popc(nzb & lanemask_lt());
                if (pos < A.xcap) {
                    A.xnodes[pos] = (int32_t)i;
                    A.xvals[pos] = xv;
                }
            }
            wpos += __popc(nzb);
        }
        if (lane == 0) {
            A.sweeps[si] = sweeps;
            A.ops[si] = ops;
            A.pushes[si] = pushes;
            A.conv[si] = conv;
            A.xoff[si] = (int64_t)base;
            A.xcnt[si] = nx;
        }
        __syncwarp();
    }
}

// ---- the reference's repair for resident pairs ------------------------------
// dynamic.repair (src/dynamic.py:131-162) on every pair of a gd_pairs pool at
// once, one warp per pair: seeds = flatnonzero(|r| >= eps d) in index order
// (:141), then the signed FIFO push of _push_kernel (src/local_solvers.py:
// 48-188) with omega = 1, x_gain = 1 and weights fl(fl(1/d_u) (1 - alpha))
// on the new graph -- pop for pop and fl() for fl() the reference, so p, r,
// sweeps and operation counts are bit-identical with the per-pair loop.
// p and r stay resident (no reset): values are stored exactly as computed.
struct FifoPairsArgs {
    DevGraph g;
    double beta, tcoeff;
    int64_t n, ld, k, max_sweeps;
    double *p, *r;
    int32_t *queue;   // (n + 2) per pair
    uint32_t *qmark;  // qw words per pair (all clear between calls)
    int64_t qw;
    int64_t *sweeps, *ops, *pushes;
    int32_t *conv;
};

__global__ void __launch_bounds__(FB_THREADS) k_fifo_pairs(FifoPairsArgs A) {
    const int lane = threadIdx.x & 31;
    const int64_t pair = (blockIdx.x * (int64_t)FB_THREADS + threadIdx.x) >> 5;
    if (pair >= A.k) return;
    double *x = A.p + pair * A.ld, *r = A.r + pair * A.ld;
    int32_t *queue = A.queue + pair * (A.n + 2);
    uint32_t *qmark = A.qmark + pair * A.qw;
    const int64_t sent = A.n, qcap = A.n + 2;
    // seeds in index order (:141 + :59-69): ordered warp compaction
    int64_t rear = 0;
    for (int64_t v0 = 0; v0 < A.n; v0 += 32) {
        const int64_t v = v0 + lane;
        bool act = false;
        if (v < A.n) act = fabs(r[v]) >= theta_d(A.tcoeff, A.g.deg[v]);
        const unsigned bal = __ballot_sync(FULL, act);
        if (act) {
            queue[rear + __popc(bal & lanemask_lt())] = (int32_t)v;
            atomicOr(qmark + (v >> 5), 1u << (v & 31));
        }
        rear += __popc(bal);
    }
    int64_t front = 0, sweeps = 0, ops = 0, pushes = 0;
    int conv = 1;
    __syncwarp();
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
            const int32_t d = A.g.deg[u];
            const int64_t rs = A.g.row[u];
            if (lane == 0) atomicAnd(qmark + (u >> 5), ~(1u << (u & 31)));
            const double th = theta_d(A.tcoeff, d);
            if (fabs(ru) < th) {
                __syncwarp();
                continue;
            }
            svol += d;
            pushes += 1;
            const double res = ru;  // omega = 1
            if (lane == 0) {
                x[u] = __dadd_rn(x[u], res);  // x_gain = 1
                r[u] = __dsub_rn(ru, res);
            }
            __syncwarp();
            const double w = __dmul_rn(__ddiv_rn(1.0, (double)d), A.beta);
            for (int64_t base = 0; base < d; base += 32) {
                const int64_t j = base + lane;
                bool act = false;
                int32_t v = 0;
                if (j < d) {
                    v = A.g.col[rs + j];
                    const double rv = __dadd_rn(r[v], __dmul_rn(res, w));
                    r[v] = rv;
                    if (!((qmark[v >> 5] >> (v & 31)) & 1u))
                        act = fabs(rv) >= theta_d(A.tcoeff, A.g.deg[v]);
                }
                const unsigned bal = __ballot_sync(FULL, act);
                if (act) {
                    int64_t q = rear + __popc(bal & lanemask_lt());
                    if (q >= qcap) q -= qcap;
                    queue[q] = v;
                    atomicOr(qmark + (v >> 5), 1u << (v & 31));
                }
                rear += __popc(bal);
                if (rear >= qcap) rear -= qcap;
                __syncwarp();
            }
            const double ru2 = r[u];  // self re-check (:176-185)
            if (!((qmark[u >> 5] >> (u & 31)) & 1u) && fabs(ru2) >= th) {
                if (lane == 0) {
                    queue[rear] = (int32_t)u;
                    atomicOr(qmark + (u >> 5), 1u << (u & 31));
                }
                rear = (rear + 1 == qcap) ? 0 : rear + 1;
            }
            __syncwarp();
        }
    }
    if (!conv)  // a sweep cap left nodes queued: clear their marks
        for (int64_t w = lane; w < A.qw; w += 32) qmark[w] = 0u;
    if (lane == 0) {
        A.sweeps[pair] = sweeps;
        A.ops[pair] = ops;
        A.pushes[pair] = pushes;
        A.conv[pair] = conv;
    }
}

}  // namespace

// Host side, called from batch.cu for GD_M_LOCAL_SOR batches.
struct FifoBatchState {
    int nslots = 0;
    int64_t ld = 0;
    DBuf<double> x, r;
    DBuf<int32_t> queue, touched, plist;
    DBuf<uint32_t> qmark;
    int64_t qw = 0;
    DBuf<unsigned long long> ctr;  // next_seed
    bool smem = false;             // k_fifo_smem (small graphs)
    size_t smem_bytes = 0;
    int64_t smem_ctas = 0;
};

FifoBatchState *fifo_batch_create(const gd_graph *G, int slots) {
    const int64_t n = G->n ? G->n : 1;
    const int64_t ld = (n + 1) & ~1LL;
    if (slots <= 0) {
        size_t fr = 0, tot = 0;
        GD_CUDA(cudaMemGetInfo(&fr, &tot));
        const int64_t per = ld * (8 + 8 + 4 + 4 + 4) + ld / 8 + 16;
        int64_t by_mem = (int64_t)(fr / 3) / per;
        int64_t resident = (int64_t)n_sms(G->device) * 64;  // warps
        slots = (int)(by_mem < resident ? (by_mem < 1 ? 1 : by_mem) : resident);
    }
    FifoBatchState *F = new FifoBatchState();
    try {
        F->nslots = slots;
        F->ld = ld;
        const size_t sn = (size_t)slots * (size_t)ld;
        F->x.alloc(sn); F->r.alloc(sn); F->touched.alloc(sn); F->plist.alloc(sn);
        F->queue.alloc((size_t)slots * (size_t)(ld + 2));
        F->qw = ld / 32 + 1;
        F->qmark.alloc((size_t)slots * (size_t)F->qw);
        GD_CUDA(cudaMemset(F->x.p, 0, sizeof(double) * sn));
        GD_CUDA(cudaMemset(F->r.p, 0, sizeof(double) * sn));
        GD_CUDA(cudaMemset(F->qmark.p, 0, sizeof(uint32_t) * (size_t)slots * (size_t)F->qw));
        F->ctr.alloc(1);
        {   // shared-memory form when a seed's state fits (GDIFF_FIFO_SMEM=0: off)
            const char *e = getenv("GDIFF_FIFO_SMEM");
            const size_t need = fifo_smem_bytes(n);
            int maxo = 0;
            GD_CUDA(cudaDeviceGetAttribute(&maxo, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                                           G->device));
            if (!(e && atoi(e) == 0) && need <= (size_t)maxo && need <= (96u << 10)) {
                GD_CUDA(cudaFuncSetAttribute(k_fifo_smem,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need));
                int per_sm = 0;
                GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fifo_smem, 32, need));
                if (per_sm > 0) {
                    F->smem = true;
                    F->smem_bytes = need;
                    F->smem_ctas = (int64_t)per_sm * n_sms(G->device);
                }
            }
        }
    } catch (...) {
        delete F;
        throw;
    }
    return F;
}

void fifo_batch_destroy(FifoBatchState *F) { delete F; }

int fifo_batch_slots(const FifoBatchState *F) { return F->nslots; }
bool fifo_batch_smem(const FifoBatchState *F) { return F->smem; }

void fifo_batch_run(FifoBatchState *F, const gd_graph *G, const gd_batch_params &p,
                    const int64_t *d_seeds, int64_t n_seeds, int64_t *sweeps, int64_t *ops,
                    int64_t *pushes, int32_t *conv, int64_t *xoff, int64_t *xcnt, int32_t *xnodes,
                    double *xvals, int64_t xcap, unsigned long long *cursor, cudaStream_t st,
                    const RPool *rp) {
    FifoBatchArgs A{};
    A.g = G->view();
    A.alpha = p.alpha;
    A.beta = 1.0 - p.alpha;
    A.tcoeff = p.eps * p.alpha;
    A.omega = p.omega;
    A.sgn = p.omega > 1.0 ? 1 : 0;
    A.n = G->n;
    A.ld = F->ld;
    A.max_sweeps = p.max_sweeps > 0 ? p.max_sweeps : 1000000;
    A.n_seeds = n_seeds;
    A.xcap = xcap;
    A.x = F->x.p; A.r = F->r.p; A.queue = F->queue.p; A.qmark = F->qmark.p; A.qw = F->qw;
    A.touched = F->touched.p; A.plist = F->plist.p; A.seeds = d_seeds; A.next_seed = F->ctr.p; A.cursor = cursor;
    A.sweeps = sweeps; A.ops = ops; A.pushes = pushes; A.conv = conv; A.xoff = xoff;
    A.xcnt = xcnt; A.xnodes = xnodes; A.xvals = xvals; A.nslots = F->nslots;
    if (rp) {
        A.r_off = rp->off; A.r_cnt = rp->cnt; A.r_nodes = rp->nodes; A.r_vals = rp->vals;
        A.rcap = rp->cap; A.rcursor = rp->cursor;
    }
    GD_CUDA(cudaMemsetAsync(F->ctr.p, 0, sizeof(unsigned long long), st));
    if (F->smem && !rp) {  // small graph: the seed's state in shared memory
        const int64_t ctas = F->smem_ctas < n_seeds ? F->smem_ctas : (n_seeds ? n_seeds : 1);
        k_fifo_smem<<<(int)ctas, 32, F->smem_bytes, st>>>(A);
        GD_LAUNCH_CHECK();
        return;
    }
    const int64_t warps = F->nslots < n_seeds ? F->nslots : (n_seeds ? n_seeds : 1);
    const int blocks = (int)((warps * 32 + FB_THREADS - 1) / FB_THREADS);
    k_fifo_batch<<<blocks, FB_THREADS, 0, st>>>(A);
    GD_LAUNCH_CHECK();
}

void fifo_pairs_run(const gd_graph *G, double *p, double *r, int64_t ld, int64_t k, double alpha,
                    double eps, int64_t max_sweeps, int32_t *queue, uint32_t *qmark, int64_t qw,
                    int64_t *sweeps, int64_t *ops, int64_t *pushes, int32_t *conv, cudaStream_t st) {
    FifoPairsArgs A{};
    A.g = G->view();
    A.beta = 1.0 - alpha;
    A.tcoeff = eps;  // repair thresholds eps * d_u (src/dynamic.py:139-141)
    A.n = G->n;
    A.ld = ld;
    A.k = k;
    A.max_sweeps = max_sweeps;
    A.p = p; A.r = r; A.queue = queue; A.qmark = qmark; A.qw = qw;
    A.sweeps = sweeps; A.ops = ops; A.pushes = pushes; A.conv = conv;
    const int blocks = (int)((k * 32 + FB_THREADS - 1) / FB_THREADS);
    k_fifo_pairs<<<blocks, FB_THREADS, 0, st>>>(A);
    GD_LAUNCH_CHECK();
}

}  // namespace gd
