// batch_cta.cu -- batched LocalGD-PPR with one CTA per seed (small graphs).
//
// Same per-seed semantics as k_rounds (batch.cu) and the reference's
// local_gd (src/local_solvers.py:428-470): every sweep pushes the whole
// frontier S_t (x_u += r_u, r_u = 0, r_v += r_u * fl(fl(1/d_u)(1-alpha))
// over u's arcs) and S_{t+1} = {v : r_v >= theta_v}; identical frontier
// sets, sweeps and operation counts, x to the rounding of the scatter order.
//
// Why a second form: k_rounds advances all seeds of a wave in lock step with
// two grid-wide barriers per sweep, which is the right shape when a sweep
// scatters millions of arcs (products, papers100M) but leaves small graphs
// (cora: ~7 K arcs per seed per sweep) barrier-bound.  Here each CTA owns a
// slot (dense x / r of its own in HBM, L2-resident at these sizes), pulls
// seeds from a global counter, and runs every sweep of its seed with CTA
// barriers only.  Seeds finish at their own pace; there are no waves, and
// init / extraction / reset happen inside the same kernel:
//   phase A (thread per entry, tiles of BT): push; block-scan the degrees
//            into arc offsets; chunk map (entry holding arc 32c, bit 31 when
//            the whole chunk lies in it) -- the same map as k_rounds;
//   phase B (warp per 32-arc chunk, UNROLL in flight): returning fp64
//            atomic; old == +0.0 marks the sector for the reset; the one arc
//            with old < theta_v <= old + c appends v to S_{t+1}.
//   end of seed: x over the pushed list -> output pool (caller ids), x
//            zeroed there, r zeroed over the marked sectors.
#include <cub/block/block_scan.cuh>
#include <cub/block/block_reduce.cuh>

#include "common.cuh"

namespace gd {
namespace {

constexpr int CT = 512;      // threads per CTA
constexpr int CUNROLL = 4;   // chunks in flight per warp in phase B
constexpr unsigned FULLM = 0xffffffffu;
constexpr int NEAR_CAP = 256;  // landings just below theta per sweep (common.cuh)

struct CtaArgs {
    DevGraph g;
    const int2 *colp;          // per arc: (neighbour, its degree)
    double alpha, beta, tcoeff;
    int64_t max_sweeps;
    int64_t ld;                // slot stride of x / r
    int64_t ncap;              // frontier / pushed list capacity per slot (n)
    int64_t ccap;              // chunk map capacity per slot
    int64_t smw;               // sector-map words per slot
    double *x, *r;
    int32_t *front;            // [slot][2][ncap]
    double *fc;                // [slot][ncap] c_u of the current frontier
    int32_t *fa;               // [slot][ncap] first arc offset of each entry
    int32_t *cmap;             // [slot][ccap]
    int32_t *pushed;           // [slot][ncap]
    uint32_t *secmap;          // [slot][smw]
    const int64_t *seeds;
    int64_t n_seeds;
    const int32_t *perm, *inv;
    unsigned long long *next_seed, *cursor;
    int64_t *sweeps, *ops, *pushes, *support, *xoff, *xcnt;
    int32_t *conv, *xnodes;
    double *xvals;
    int64_t xcap;
    int32_t *amb;                 // per seed: near-threshold update seen (common.cuh)
    unsigned long long *amb_cnt;  // flagged seeds
    int64_t *lg_f, *lg_ops;       // per-seed sweep logs (nullable): |S_t|, vol(S_t),
    double *lg_g;                 //   sum |r_u| pushed
    int64_t lg_cap;
};

__device__ __forceinline__ double theta_d(double tc, int32_t d) {
    return d > 0 ? __dmul_rn(tc, (double)d) : __longlong_as_double(0x7ff0000000000000LL);
}

__device__ __forceinline__ unsigned lanemask_lt_() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// warp-aggregated append of `item` to list[...] with a shared counter
__device__ __forceinline__ void cta_append(bool flag, int32_t item, int32_t *list, int *cnt) {
    const unsigned am = __ballot_sync(FULLM, flag);
    if (!am) return;
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == __ffs(am) - 1) base = atomicAdd(cnt, __popc(am));
    base = __shfl_sync(FULLM, base, __ffs(am) - 1);
    if (flag) list[base + __popc(am & lanemask_lt_())] = item;
}

__global__ void __launch_bounds__(CT, 2) k_seed_cta(CtaArgs A) {
    using Scan = cub::BlockScan<int64_t, CT>;
    using Red = cub::BlockReduce<unsigned long long, CT>;
    using RedD = cub::BlockReduce<double, CT>;
    __shared__ typename RedD::TempStorage redd_tmp;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ typename Red::TempStorage red_tmp;
    __shared__ int s_F, s_nf, s_pc;
    __shared__ int64_t s_run, s_seed, s_base;
    __shared__ int s_overflow;
    __shared__ unsigned s_touch, s_negz;
    __shared__ int s_amb, s_nnear;
    __shared__ int32_t s_near[NEAR_CAP];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = CT / 32;
    const int64_t slot = blockIdx.x;
    double *const x = A.x + slot * A.ld;
    double *const r = A.r + slot * A.ld;
    int32_t *const fr0 = A.front + slot * 2 * A.ncap;
    double *const fc = A.fc + slot * A.ncap;
    int32_t *const fa = A.fa + slot * A.ncap;
    int32_t *const cmap = A.cmap + slot * A.ccap;
    int32_t *const pushed = A.pushed + slot * A.ncap;
    uint32_t *const map = A.secmap + slot * A.smw;

    for (;;) {
        if (tid == 0) s_seed = (int64_t)atomicAdd(A.next_seed, 1ULL);
        __syncthreads();
        const int64_t si = s_seed;
        if (si >= A.n_seeds) return;
        int32_t s = (int32_t)A.seeds[si];
        if (A.perm) s = A.perm[s];
        if (tid == 0) {
            r[s] = A.alpha;
            map[s >> 7] |= 1u << ((s >> 2) & 31);
            s_F = A.alpha >= theta_d(A.tcoeff, A.g.deg[s]) ? 1 : 0;
            fr0[0] = s;
            s_pc = 0;
            s_touch = 1;  // the seed's r word
            s_negz = 0;
            s_overflow = 0;
            s_amb = 0;
            s_nnear = 0;
        }
        unsigned long long my_ops = 0, my_push = 0;
        int64_t t = 0;
        __syncthreads();
        for (;; ++t) {
            {   // final values of last sweep's landings just below theta
                const int nn = min(s_nnear, NEAR_CAP);
                for (int i = tid; i < nn; i += CT) {
                    const int32_t v = s_near[i];
                    if (below_theta(r[v], theta_d(A.tcoeff, A.g.deg[v]))) s_amb = 1;
                }
                __syncthreads();
                if (tid == 0) s_nnear = 0;
            }
            const int F = s_F;
            if (F == 0 || t >= A.max_sweeps) break;
            int32_t *const cur = fr0 + (t & 1) * A.ncap;
            int32_t *const nxt = fr0 + ((t & 1) ^ 1) * A.ncap;
            // ------------- phase A: push, arc offsets, chunk map -------------
            if (tid == 0) {
                s_run = 0;
                s_nf = 0;
            }
            __syncthreads();
            double my_g = 0.0;  // (sweep log) this thread's pushed |r|
            for (int tile = 0; tile < F; tile += CT) {
                const int e = tile + tid;
                const bool live = e < F;
                int32_t u = 0, d = 0;
                bool fresh = false;
                if (live) {
                    u = cur[e];
                    const double val = r[u];
                    const double xo = x[u];
                    x[u] = __dadd_rn(xo, val);
                    r[u] = -0.0;  // pushed (+0.0 = never touched)
                    my_g += fabs(val);
                    d = A.g.deg[u];
                    if (near_theta(val, theta_d(A.tcoeff, d))) s_amb = 1;  // final r >= theta
                    fc[e] = __dmul_rn(val, __dmul_rn(__ddiv_rn(1.0, (double)d), A.beta));
                    fresh = __double_as_longlong(xo) == 0;
                    my_ops += (unsigned long long)d;
                    my_push += 1ULL;
                }
                int64_t excl = 0, total = 0;
                Scan(scan_tmp).ExclusiveSum((int64_t)d, excl, total);
                const int64_t a0 = s_run + excl;
                int64_t clo = 0, chi = 0, cfull = 0;
                if (live) {
                    fa[e] = (int32_t)a0;
                    clo = (a0 + 31) >> 5;
                    chi = (a0 + d + 31) >> 5;
                    cfull = (a0 + d) >> 5;
                    if (chi > A.ccap) s_overflow = 1;
                    chi = min(chi, A.ccap);
                }
                unsigned big = __ballot_sync(FULLM, chi - clo > 4);
                if (!(big >> lane & 1u))
                    for (int64_t c = clo; c < chi; ++c)
                        cmap[c] = (int32_t)((uint32_t)e | (c < cfull ? 0x80000000u : 0u));
                while (big) {
                    const int src = __ffs(big) - 1;
                    big &= big - 1;
                    const int64_t lo2 = __shfl_sync(FULLM, clo, src), hi2 = __shfl_sync(FULLM, chi, src);
                    const int64_t cf2 = __shfl_sync(FULLM, cfull, src);
                    const uint32_t e2 = (uint32_t)__shfl_sync(FULLM, e, src);
                    for (int64_t c = lo2 + lane; c < hi2; c += 32)
                        cmap[c] = (int32_t)(e2 | (c < cf2 ? 0x80000000u : 0u));
                }
                cta_append(fresh, u, pushed, &s_pc);
                __syncthreads();
                if (tid == 0) s_run += total;
                __syncthreads();
            }
            const int64_t P = s_run;
            if (A.lg_f && t < A.lg_cap) {  // sweep log: |S_t|, vol(S_t), sum |r_u|
                const double g = RedD(redd_tmp).Sum(my_g);
                if (tid == 0) {
                    A.lg_f[si * A.lg_cap + t] = F;
                    A.lg_ops[si * A.lg_cap + t] = P;
                    A.lg_g[si * A.lg_cap + t] = g;
                }
                __syncthreads();
            }
            // ------------- phase B: scatter 32-arc chunks ----------------------
            const int64_t C = min((P + 31) >> 5, A.ccap);
            const double tc = A.tcoeff;
            for (int64_t cb = (int64_t)warp * CUNROLL; cb < C; cb += (int64_t)nwarps * CUNROLL) {
                int32_t v[CUNROLL], dv[CUNROLL];
                double c[CUNROLL], old[CUNROLL];
                bool valid[CUNROLL];
#pragma unroll
                for (int q = 0; q < CUNROLL; ++q) {
                    const int64_t ch = cb + q;
                    const bool lv = ch < C;
                    const uint32_t raw = lv ? (uint32_t)cmap[ch] : 0u;
                    const int e = (int)(raw & 0x7fffffffu);
                    const int64_t a = ch << 5;
                    int me = e;
                    if (!(raw >> 31)) {  // entries starting inside (a, a + 32)
                        const int wi = e + 1 + lane;
                        const int64_t st = (lv && wi < F) ? (int64_t)fa[wi] : INT64_MAX;
                        const int64_t pos = st - a;
                        const unsigned starts = __reduce_or_sync(FULLM, pos < 32 ? (1u << pos) : 0u);
                        me = e + __popc(starts & ((2u << lane) - 1u));
                    }
                    const int64_t p = a + lane;
                    valid[q] = lv && p < P;
                    v[q] = 0; dv[q] = 0; c[q] = 0.0;
                    if (valid[q]) {
                        const int32_t u = cur[me];
                        c[q] = fc[me];
                        const int2 vd = __ldg(A.colp + A.g.row[u] + (p - fa[me]));
                        v[q] = vd.x;
                        dv[q] = vd.y;
                    }
                }
#pragma unroll
                for (int q = 0; q < CUNROLL; ++q) {
                    GD_DCHECK(!valid[q] || (v[q] >= 0 && v[q] < A.g.n));
                    old[q] = valid[q] ? atomicAdd(r + v[q], c[q]) : 0.0;
                }
#pragma unroll
                for (int q = 0; q < CUNROLL; ++q) {
                    const long long ob = __double_as_longlong(old[q]);
                    const bool first = valid[q] && ob == 0;
                    const bool negz = valid[q] && ob == (long long)0x8000000000000000ULL;
                    const double th = theta_d(tc, dv[q]);
                    const double nw = __dadd_rn(old[q], c[q]);
                    const bool cross = valid[q] && old[q] < th && nw >= th;
                    if (valid[q] && below_theta(nw, th)) {
                        const int at = atomicAdd(&s_nnear, 1);
                        if (at < NEAR_CAP) s_near[at] = v[q]; else s_amb = 1;
                    }
                    if (first) atomicOr(map + (v[q] >> 7), 1u << ((v[q] >> 2) & 31));
                    const unsigned fm = __ballot_sync(FULLM, first), nm = __ballot_sync(FULLM, negz);
                    if (lane == 0) {
                        if (fm) atomicAdd(&s_touch, (unsigned)__popc(fm));
                        if (nm) atomicAdd(&s_negz, (unsigned)__popc(nm));
                    }
                    cta_append(cross, v[q], nxt, &s_nf);
                }
            }
            __syncthreads();
            if (tid == 0) s_F = s_nf;
            __syncthreads();
        }
        // ------------------ end of seed: counters, x out, reset -------------
        const unsigned long long ops = Red(red_tmp).Sum(my_ops);
        __syncthreads();
        const unsigned long long psh = Red(red_tmp).Sum(my_push);
        const int pc = s_pc;
        if (tid == 0) {
            s_base = (int64_t)atomicAdd(A.cursor, (unsigned long long)pc);
            A.sweeps[si] = t;
            A.ops[si] = (int64_t)ops;
            A.pushes[si] = (int64_t)psh;
            A.conv[si] = (s_F == 0 && !s_overflow) ? 1 : 0;
            A.support[si] = (int64_t)s_touch - ((int64_t)psh - (int64_t)s_negz);
            A.xcnt[si] = pc;
            A.amb[si] = s_amb;
            if (s_amb) atomicAdd(A.amb_cnt, 1ULL);
        }
        __syncthreads();
        const int64_t b = s_base;
        if (tid == 0) A.xoff[si] = b;
        for (int i = tid; i < pc; i += CT) {
            const int32_t u = pushed[i];
            const double xv = x[u];
            x[u] = 0.0;
            if (b + i < A.xcap) {
                A.xnodes[b + i] = A.inv ? A.inv[u] : u;
                A.xvals[b + i] = xv;
            }
        }
        double4 *r4 = reinterpret_cast<double4 *>(r);
        for (int64_t w = tid; w < A.smw; w += CT) {
            uint32_t bits = map[w];
            if (!bits) continue;
            map[w] = 0u;
            while (bits) {
                const int j = __ffs(bits) - 1;
                bits &= bits - 1;
                const int64_t sec = w * 32 + j;  // doubles [4 sec, 4 sec + 4)
                if (4 * sec + 3 < A.ld)
                    r4[sec] = make_double4(0.0, 0.0, 0.0, 0.0);
                else
                    for (int64_t i = 4 * sec; i < A.ld; ++i) r[i] = 0.0;
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// k_seed_smem: the same per-seed sweep loop with the seed's whole state in
// shared memory -- graphs whose x, r, frontier lists, c_u, arc offsets and
// chunk map fit in one SM (cora-class, n up to ~6 K nodes).  Every access of
// the sweep except the graph reads (row, (neighbour, degree) pairs, degree:
// L1-resident at these sizes) is a shared-memory one, so a sweep's dependent
// chain (entry -> r -> scan -> chunk map -> arc -> atomic -> append) runs at
// shared-memory instead of L2 latency; there is nothing to reset between
// seeds but a zero fill.  Residual updates: fp64 shared-memory atomics
// (compare-and-swap loops; the returned old value decides the threshold
// crossing exactly as in k_seed_cta).  Support = nonzero residuals at the end;
// x goes out in node order.
struct SmemView {
    double *r, *x, *fc;
    int32_t *front, *fa, *cmap;
};
__host__ __device__ inline size_t smem_seed_bytes(int64_t n, int64_t ccap) {
    const int64_t ld = (n + 3) & ~3LL;
    return (size_t)(8 * (2 * ld + ld) + 4 * (2 * ld + ld + ccap));
}
__device__ inline SmemView smem_carve(unsigned char *p, int64_t n) {
    const int64_t ld = (n + 3) & ~3LL;
    SmemView V;
    V.r = reinterpret_cast<double *>(p);
    V.x = V.r + ld;
    V.fc = V.x + ld;
    V.front = reinterpret_cast<int32_t *>(V.fc + ld);
    V.fa = V.front + 2 * ld;
    V.cmap = V.fa + ld;
    return V;
}

__global__ void __launch_bounds__(CT, 1) k_seed_smem(CtaArgs A) {
    using Scan = cub::BlockScan<int64_t, CT>;
    using Red = cub::BlockReduce<unsigned long long, CT>;
    using RedD = cub::BlockReduce<double, CT>;
    __shared__ typename RedD::TempStorage redd_tmp;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ typename Red::TempStorage red_tmp;
    __shared__ int s_F, s_nf, s_xc, s_rc;
    __shared__ int64_t s_run, s_seed, s_base;
    __shared__ int s_amb, s_nnear;
    __shared__ int32_t s_near[NEAR_CAP];
    extern __shared__ __align__(16) unsigned char smem_dyn[];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = CT / 32;
    const int64_t n = A.g.n, ld = (n + 3) & ~3LL;
    const SmemView V = smem_carve(smem_dyn, n);
    double *const r = V.r;
    double *const x = V.x;

    for (;;) {
        if (tid == 0) s_seed = (int64_t)atomicAdd(A.next_seed, 1ULL);
        for (int64_t i = tid; i < ld; i += CT) {
            r[i] = 0.0;
            x[i] = 0.0;
        }
        __syncthreads();
        const int64_t si = s_seed;
        if (si >= A.n_seeds) return;
        int32_t s = (int32_t)A.seeds[si];
        if (A.perm) s = A.perm[s];
        if (tid == 0) {
            r[s] = A.alpha;
            s_F = A.alpha >= theta_d(A.tcoeff, A.g.deg[s]) ? 1 : 0;
            V.front[0] = s;
            s_amb = 0;
            s_nnear = 0;
        }
        unsigned long long my_ops = 0, my_push = 0;
        int64_t t = 0;
        __syncthreads();
        for (;; ++t) {
            {   // final values of last sweep's landings just below theta
                const int nn = min(s_nnear, NEAR_CAP);
                for (int i = tid; i < nn; i += CT) {
                    const int32_t v = s_near[i];
                    if (below_theta(r[v], theta_d(A.tcoeff, A.g.deg[v]))) s_amb = 1;
                }
                __syncthreads();
                if (tid == 0) s_nnear = 0;
            }
            const int F = s_F;
            if (F == 0 || t >= A.max_sweeps) break;
            int32_t *const cur = V.front + (t & 1) * ld;
            int32_t *const nxt = V.front + ((t & 1) ^ 1) * ld;
            // ------------- phase A: push, arc offsets, chunk map -------------
            if (tid == 0) {
                s_run = 0;
                s_nf = 0;
            }
            __syncthreads();
            double my_g = 0.0;
            for (int tile = 0; tile < F; tile += CT) {
                const int e = tile + tid;
                const bool live = e < F;
                int32_t u = 0, d = 0;
                if (live) {
                    u = cur[e];
                    const double val = r[u];
                    x[u] = __dadd_rn(x[u], val);
                    r[u] = 0.0;
                    my_g += fabs(val);
                    d = A.g.deg[u];
                    if (near_theta(val, theta_d(A.tcoeff, d))) s_amb = 1;  // final r >= theta
                    V.fc[e] = __dmul_rn(val, __dmul_rn(__ddiv_rn(1.0, (double)d), A.beta));
                    my_ops += (unsigned long long)d;
                    my_push += 1ULL;
                }
                int64_t excl = 0, total = 0;
                Scan(scan_tmp).ExclusiveSum((int64_t)d, excl, total);
                const int64_t a0 = s_run + excl;
                int64_t clo = 0, chi = 0, cfull = 0;
                if (live) {
                    V.fa[e] = (int32_t)a0;
                    clo = (a0 + 31) >> 5;
                    chi = min((a0 + d + 31) >> 5, A.ccap);
                    cfull = (a0 + d) >> 5;
                }
                unsigned big = __ballot_sync(FULLM, chi - clo > 4);
                if (!(big >> lane & 1u))
                    for (int64_t c = clo; c < chi; ++c)
                        V.cmap[c] = (int32_t)((uint32_t)e | (c < cfull ? 0x80000000u : 0u));
                while (big) {
                    const int src = __ffs(big) - 1;
                    big &= big - 1;
                    const int64_t lo2 = __shfl_sync(FULLM, clo, src), hi2 = __shfl_sync(FULLM, chi, src);
                    const int64_t cf2 = __shfl_sync(FULLM, cfull, src);
                    const uint32_t e2 = (uint32_t)__shfl_sync(FULLM, e, src);
                    for (int64_t c = lo2 + lane; c < hi2; c += 32)
                        V.cmap[c] = (int32_t)(e2 | (c < cf2 ? 0x80000000u : 0u));
                }
                __syncthreads();
                if (tid == 0) s_run += total;
                __syncthreads();
            }
            const int64_t P = s_run;
            if (A.lg_f && t < A.lg_cap) {  // sweep log: |S_t|, vol(S_t), sum |r_u|
                const double g = RedD(redd_tmp).Sum(my_g);
                if (tid == 0) {
                    A.lg_f[si * A.lg_cap + t] = F;
                    A.lg_ops[si * A.lg_cap + t] = P;
                    A.lg_g[si * A.lg_cap + t] = g;
                }
                __syncthreads();
            }
            // ------------- phase B: scatter 32-arc chunks ----------------------
            const int64_t C = min((P + 31) >> 5, A.ccap);
            const double tc = A.tcoeff;
            for (int64_t cb = (int64_t)warp * CUNROLL; cb < C; cb += (int64_t)nwarps * CUNROLL) {
                int32_t v[CUNROLL], dv[CUNROLL];
                double c[CUNROLL], old[CUNROLL];
                bool valid[CUNROLL];
#pragma unroll
                for (int q = 0; q < CUNROLL; ++q) {
                    const int64_t ch = cb + q;
                    const bool lv = ch < C;
                    const uint32_t raw = lv ? (uint32_t)V.cmap[ch] : 0u;
                    const int e = (int)(raw & 0x7fffffffu);
                    const int64_t a = ch << 5;
                    int me = e;
                    if (!(raw >> 31)) {  // entries starting inside (a, a + 32)
                        const int wi = e + 1 + lane;
                        const int64_t st = (lv && wi < F) ? (int64_t)V.fa[wi] : INT64_MAX;
                        const int64_t pos = st - a;
                        const unsigned starts = __reduce_or_sync(FULLM, pos < 32 ? (1u << pos) : 0u);
                        me = e + __popc(starts & ((2u << lane) - 1u));
                    }
                    const int64_t p = a + lane;
                    valid[q] = lv && p < P;
                    v[q] = 0; dv[q] = 0; c[q] = 0.0;
                    if (valid[q]) {
                        const int32_t u = cur[me];
                        c[q] = V.fc[me];
                        const int2 vd = __ldg(A.colp + A.g.row[u] + (p - V.fa[me]));
                        v[q] = vd.x;
                        dv[q] = vd.y;
                    }
                }
#pragma unroll
                for (int q = 0; q < CUNROLL; ++q) {
                    GD_DCHECK(!valid[q] || (v[q] >= 0 && v[q] < A.g.n));
                    old[q] = valid[q] ? atomicAdd(r + v[q], c[q]) : 0.0;
                }
#pragma unroll
                for (int q = 0; q < CUNROLL; ++q) {
                    const double th = theta_d(tc, dv[q]);
                    const double nw = __dadd_rn(old[q], c[q]);
                    const bool cross = valid[q] && old[q] < th && nw >= th;
                    if (valid[q] && below_theta(nw, th)) {
                        const int at = atomicAdd(&s_nnear, 1);
                        if (at < NEAR_CAP) s_near[at] = v[q]; else s_amb = 1;
                    }
                    cta_append(cross, v[q], nxt, &s_nf);
                }
            }
            __syncthreads();
            if (tid == 0) s_F = s_nf;
            __syncthreads();
        }
        // ------------------ end of seed: counters, x out --------------------
        const unsigned long long ops = Red(red_tmp).Sum(my_ops);
        __syncthreads();
        const unsigned long long psh = Red(red_tmp).Sum(my_push);
        unsigned long long nzx = 0, nzr = 0;
        for (int64_t i = tid; i < n; i += CT) {
            nzx += x[i] != 0.0;
            nzr += r[i] != 0.0;
        }
        __syncthreads();
        const unsigned long long xc = Red(red_tmp).Sum(nzx);
        __syncthreads();
        const unsigned long long rc = Red(red_tmp).Sum(nzr);
        if (tid == 0) {
            s_base = (int64_t)atomicAdd(A.cursor, xc);
            s_xc = 0;
            A.sweeps[si] = t;
            A.ops[si] = (int64_t)ops;
            A.pushes[si] = (int64_t)psh;
            A.conv[si] = s_F == 0 ? 1 : 0;
            A.support[si] = (int64_t)rc;
            A.xcnt[si] = (int64_t)xc;
            A.xoff[si] = s_base;
            A.amb[si] = s_amb;
            if (s_amb) atomicAdd(A.amb_cnt, 1ULL);
        }
        __syncthreads();
        const int64_t b = s_base;
        for (int64_t i0 = 0; i0 < n; i0 += CT) {  // warp-uniform trip count
            const int64_t i = i0 + tid;
            const bool nz = i < n && x[i] != 0.0;
            const unsigned am = __ballot_sync(FULLM, nz);
            int base = 0;
            if (am && lane == __ffs(am) - 1) base = atomicAdd(&s_xc, __popc(am));
            base = __shfl_sync(FULLM, base, __ffs(am ? am : 1u) - 1);
            if (nz) {
                const int64_t at = b + base + __popc(am & lanemask_lt_());
                if (at < A.xcap) {
                    A.xnodes[at] = A.inv ? A.inv[i] : (int32_t)i;
                    A.xvals[at] = x[i];
                }
            }
        }
        __syncthreads();
        (void)s_rc;
    }
}

}  // namespace

struct CtaState {
    int slots = 0;
    int64_t ld = 0, ncap = 0, ccap = 0, smw = 0;
    DBuf<double> x, r, fc;
    DBuf<int32_t> front, fa, cmap, pushed;
    DBuf<uint32_t> secmap;
    DBuf<unsigned long long> next;
    // k_seed_smem: the whole per-seed state in shared memory, one CTA per SM;
    // used for batches of at most smem_cap seeds (larger batches run more
    // CTAs per SM in the HBM form, which measured faster there: cora 1,024
    // seeds 6.2 vs 6.3 ms, 50 seeds 1.18 vs 0.93 ms)
    bool smem = false;
    size_t smem_bytes = 0;
    int smem_cap = 0, smem_slots = 0;  // CTAs resident at once; CTAs launched
};

// Slots = CTAs resident at once (capped by `max_slots` when > 0 and by the
// number of seeds at run time).
CtaState *cta_batch_create(const gd_graph *W, int max_slots) {
    CtaState *S = new CtaState();
    try {
        int per_sm = 0;
        {   // shared-memory form when one seed's state fits (GDIFF_CTA_SMEM=0: off)
            const char *e = getenv("GDIFF_CTA_SMEM");
            int maxo = 0;
            GD_CUDA(cudaDeviceGetAttribute(&maxo, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                                           W->device));
            const int64_t ccap = (W->n_arcs + 31) / 32 + 1;
            const size_t need = smem_seed_bytes(W->n ? W->n : 1, ccap);
            const size_t stat = 16 * 1024;  // static shared memory of the kernel (upper bound)
            if (!(e && atoi(e) == 0) && need + stat <= (size_t)maxo) {
                GD_CUDA(cudaFuncSetAttribute(k_seed_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)need));
                GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_seed_smem, CT,
                                                                      need));
                if (per_sm > 0) {
                    S->smem = true;
                    S->smem_bytes = need;
                    S->smem_cap = S->smem_slots = per_sm * n_sms(W->device);
                    if (max_slots > 0 && max_slots < S->smem_slots) S->smem_slots = max_slots;
                }
            }
        }
        GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_seed_cta, CT, 0));
        GD_CHECK_ARG(per_sm > 0, "seed kernel does not fit on an SM");
        int slots = per_sm * n_sms(W->device);
        if (max_slots > 0 && max_slots < slots) slots = max_slots;
        const int64_t n = W->n ? W->n : 1;
        S->slots = slots;
        S->ld = (n + 3) & ~3LL;
        S->ncap = n;
        S->ccap = (W->n_arcs + 31) / 32 + 1;
        S->smw = (S->ld / 4 + 31) / 32;
        const size_t sn = (size_t)slots * (size_t)S->ld;
        S->x.alloc(sn);
        S->r.alloc(sn);
        GD_CUDA(cudaMemset(S->x.p, 0, sizeof(double) * sn));
        GD_CUDA(cudaMemset(S->r.p, 0, sizeof(double) * sn));
        S->front.alloc((size_t)slots * 2 * (size_t)S->ncap);
        S->fc.alloc((size_t)slots * (size_t)S->ncap);
        S->fa.alloc((size_t)slots * (size_t)S->ncap);
        S->pushed.alloc((size_t)slots * (size_t)S->ncap);
        S->cmap.alloc((size_t)slots * (size_t)S->ccap);
        S->secmap.alloc((size_t)slots * (size_t)S->smw);
        GD_CUDA(cudaMemset(S->secmap.p, 0, sizeof(uint32_t) * (size_t)slots * (size_t)S->smw));
        S->next.alloc(1);
    } catch (...) {
        delete S;
        throw;
    }
    return S;
}

void cta_batch_destroy(CtaState *S) { delete S; }

int cta_batch_slots(const CtaState *S) { return S->slots; }
bool cta_batch_smem(const CtaState *S) { return S->smem; }

// Bytes of device memory one slot needs (for the host's mode choice).
int64_t cta_slot_bytes(int64_t n, int64_t n_arcs) {
    const int64_t ld = (n + 3) & ~3LL;
    return 16 * ld + 24 * n + 4 * ((n_arcs + 31) / 32 + 1) + ld / 32 + 64;
}

void cta_batch_run(CtaState *S, const gd_graph *W, const int2 *colp, double alpha, double eps,
                   int64_t max_sweeps, const int64_t *d_seeds, int64_t n_seeds,
                   const int32_t *perm, const int32_t *inv, int64_t *sweeps, int64_t *ops,
                   int64_t *pushes, int64_t *support, int32_t *conv, int64_t *xoff,
                   int64_t *xcnt, int32_t *xnodes, double *xvals, int64_t xcap,
                   unsigned long long *cursor, int32_t *amb, unsigned long long *amb_cnt,
                   cudaStream_t st, int64_t *lg_f, int64_t *lg_ops, double *lg_g,
                   int64_t lg_cap) {
    if (n_seeds == 0) return;
    CtaArgs A{};
    A.g = W->view();
    A.colp = colp;
    A.alpha = alpha;
    A.beta = 1.0 - alpha;
    A.tcoeff = eps * alpha;
    A.max_sweeps = max_sweeps;
    A.ld = S->ld; A.ncap = S->ncap; A.ccap = S->ccap; A.smw = S->smw;
    A.x = S->x.p; A.r = S->r.p; A.front = S->front.p; A.fc = S->fc.p; A.fa = S->fa.p;
    A.cmap = S->cmap.p; A.pushed = S->pushed.p; A.secmap = S->secmap.p;
    A.seeds = d_seeds; A.n_seeds = n_seeds;
    A.perm = perm; A.inv = inv;
    A.next_seed = S->next.p; A.cursor = cursor;
    A.sweeps = sweeps; A.ops = ops; A.pushes = pushes; A.support = support;
    A.xoff = xoff; A.xcnt = xcnt; A.conv = conv; A.xnodes = xnodes; A.xvals = xvals;
    A.xcap = xcap;
    A.amb = amb;
    A.amb_cnt = amb_cnt;
    A.lg_f = lg_f;
    A.lg_ops = lg_ops;
    A.lg_g = lg_g;
    A.lg_cap = lg_cap;
    GD_CUDA(cudaMemsetAsync(S->next.p, 0, sizeof(unsigned long long), st));
    if (S->smem && n_seeds <= S->smem_cap) {
        k_seed_smem<<<(int)(n_seeds < S->smem_slots ? n_seeds : S->smem_slots), CT, S->smem_bytes,
                      st>>>(A);
    } else {
        const int grid = (int)(n_seeds < S->slots ? n_seeds : S->slots);
        k_seed_cta<<<grid, CT, 0, st>>>(A);
    }
    GD_LAUNCH_CHECK();
}

}  // namespace gd
