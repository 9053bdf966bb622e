// batch_signed.cu -- batched sweep-synchronous solvers with SIGNED residuals:
//   * LocalCH (Chebyshev momentum, src/local_solvers.py:473-538) for many
//     seeds, PPR or Katz (gd_batch with GD_M_LOCAL_CH), and
//   * warm-started signed LocalGD over a pool of resident PPR pairs (p, r)
//     on an evolving graph (gd_pairs: config 5's incremental maintenance;
//     event adjustment src/dynamic.py:40-107, repair on the new graph).
//
// Per slot (one seed / pair): dense x, r (+ momentum value and stamp for
// CH).  Residuals change sign, so the unsigned kernel's "exactly one arc
// observes the threshold crossing" does not hold.  The frontier of round t
// is instead filtered from CANDIDATES: under momentum the previous frontier
// (whose r is r - vals, not 0), plus every node that received a
// contribution in round t-1 AND saw |r| >= theta right after one of its
// updates.  The reference filters every touched node (_apply_update_seq +
// _filter_frontier, signed test); the two sets agree on the active nodes
// because the last update of a node stores its final value.  A per-slot bit
// map per round parity deduplicates candidates (the old word returned by
// one atomicOr says whether the node is new this round).
//
// Round t:  phase A  candidates -> |r| >= theta ? push (x, r, momentum,
//                    l1 delta) and stage (slot, node, c_u) : skip;
//                    block flushes -> entries + arc offsets + chunk map
//           phase B  32-arc chunks: r[v] += c_u (returning atomic: l1
//                    delta, first touch -> sector map), candidate for t+1
// The per-slot l1 norm is tracked incrementally (|old + c| - |old| per
// update) for the LocalCH divergence abort (l1 > 10 ||b||_1, :527-530); it
// equals the reference's pairwise sum to rounding, which can only matter when
// l1 sits within rounding of the abort level.
#include <cooperative_groups.h>

#include <cub/block/block_scan.cuh>

#include <algorithm>
#include <cmath>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace gd {
struct RPool {  // (batch.cu)
    int64_t *off, *cnt;
    int32_t *nodes;
    double *vals;
    int64_t cap;
    unsigned long long *cursor;
    unsigned long long *scratch;
};
void r_extract_wave(uint32_t *secmap, int64_t smw, double *r, int64_t ld, int64_t m,
                    const int32_t *inv, int64_t seed_base, unsigned long long *cnt_scratch,
                    unsigned long long *cursor, int64_t *r_off, int64_t *r_cnt,
                    int32_t *r_nodes, double *r_vals, int64_t rcap, cudaStream_t st);
namespace {

constexpr int SBT = 512;
constexpr int SUNROLL = 4;
constexpr int SCNT_SHIFT = 36;
constexpr unsigned long long SARC_MASK = (1ULL << SCNT_SHIFT) - 1ULL;
constexpr unsigned SFULL = 0xffffffffu;
constexpr int SSTAGE = 4 * SBT;  // staged entries / candidates per block
constexpr int SCHUNKS = 32;
constexpr int SSUPER = 16;  // SUNROLL-chunk groups per block super-chunk (grouped mode)

struct SArgs {
    DevGraph g;
    DevOp op;        // weight rule (RW / CONST) and theta coefficient
    int method;      // 0 signed GD, 1 CH
    int64_t m, ld, max_sweeps, fcap, ccap, candcap;
    double *x, *r, *mom;
    int32_t *mstamp;  // round of the last momentum write; -1 = never pushed
    const double *coef_r, *coef_m;  // CH coefficients per sweep index
    double step0, l1cap;            // CH: first step, abort factor on ||b||_1
    int32_t *pushed;                // CH: per slot first-pushed nodes (x support)
    unsigned long long *pushed_cnt;
    uint32_t *cmark[2];             // per slot candidate bit maps (cmw words each)
    int64_t cmw;
    uint32_t *secmap;               // per slot touched 32 B sectors of r (nullable)
    int64_t smw;
    int64_t *cand[2];               // (slot << 32 | node)
    unsigned long long *candctr;    // [2]
    const int2 *colp;               // (neighbour, degree) per arc
    int grouped;                    // 1: entries regrouped by slot group before phase B
    int64_t sgroup;                 //    (slot vectors exceed L2; see batch.cu)
    int64_t group_min;              //    ... in rounds with at least this many candidates
    int64_t *ukey;                  //    unsorted entries of the round and their c_u
    double *ucval;
    unsigned long long *gcnt, *gfill;  // per slot group: packed (entries, arcs), fill
    int64_t *fkey, *farc, *frow;    // frontier of the current round
    double *fcval;
    int32_t *chunk_e;
    unsigned long long *fctr;       // packed (entries << 36 | arcs)
    unsigned long long *s_ops, *s_pushes;
    double *s_l1, *s_b1;
    int32_t *s_last, *s_conv;
    int32_t *s_amb;  // per slot: a final |r| within AMB_REL of theta (common.cuh)
    NearList nearl;  // landings just below theta, re-checked after the round
    int32_t *overflow;
    // CTA-local tail (k_s_tail): once a round has <= tail_f candidates past the
    // wave's peak (or after 16 rounds), block k finishes slot k alone; lists of n
    // entries per slot: candidates (two) and frontier entries, and their c
    int32_t *tail_list;
    double *tail_c;
    int64_t tail_f;
    int32_t tail_t;       // (or from this round on)
    int64_t *tail_state;  // round, candidates (-1: no tail)
};

__device__ __forceinline__ unsigned lanemask_lt_s() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

struct SStage {
    double *c;
    double *l1;                      // [m] per-slot l1 deltas of the block
    unsigned long long *gc;          // [m] per slot group (entries, arcs) of the block
    unsigned long long *gbase;       // [m] group offsets of the grouped frontier
    unsigned long long *ops, *push;  // [m]
    unsigned long long *scan;        // [SBT/32 + 2]
    unsigned long long *next;
    int32_t *k, *v, *d;
    int32_t *ck, *cv;  // staged candidates
    unsigned *cnt, *ccnt;
};

inline size_t sstage_bytes(int64_t m) {
    return (size_t)SSTAGE * 8 + (size_t)m * 40 + 8 * (SBT / 32 + 3) + (size_t)SSTAGE * 20 + 32;
}

__device__ SStage sstage_carve(void *base, int64_t m) {
    char *p = (char *)base;
    SStage s;
    s.c = (double *)p; p += 8 * SSTAGE;
    s.l1 = (double *)p; p += 8 * m;
    s.gc = (unsigned long long *)p; p += 8 * m;
    s.gbase = (unsigned long long *)p; p += 8 * m;
    s.ops = (unsigned long long *)p; p += 8 * m;
    s.push = (unsigned long long *)p; p += 8 * m;
    s.scan = (unsigned long long *)p; p += 8 * (SBT / 32 + 2);
    s.next = (unsigned long long *)p; p += 8;
    s.k = (int32_t *)p; p += 4 * SSTAGE;
    s.v = (int32_t *)p; p += 4 * SSTAGE;
    s.d = (int32_t *)p; p += 4 * SSTAGE;
    s.ck = (int32_t *)p; p += 4 * SSTAGE;
    s.cv = (int32_t *)p; p += 4 * SSTAGE;
    s.cnt = (unsigned *)p; p += 16;
    s.ccnt = (unsigned *)p;
    return s;
}

__device__ __forceinline__ void slot_add_u(bool flag, int32_t k, unsigned val,
                                           unsigned long long *cnt) {
    unsigned am = __ballot_sync(SFULL, flag);
    if (!flag) return;
    unsigned peers = __match_any_sync(am, k);
    unsigned sum = __reduce_add_sync(peers, val);
    if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(cnt + k, (unsigned long long)sum);
}

// per-slot double sum into shared memory; one atomic per warp when the
// warp's lanes share a slot (the common case: a chunk is one entry's arcs)
__device__ __forceinline__ void slot_add_d(bool flag, int32_t k, double val, double *acc) {
    const unsigned am = __ballot_sync(SFULL, flag);
    if (!am) return;
    const int32_t k0 = __shfl_sync(SFULL, k, __ffs(am) - 1);
    if (__all_sync(SFULL, !flag || k == k0)) {
        double s = flag ? val : 0.0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(SFULL, s, o);
        if ((threadIdx.x & 31) == 0 && s != 0.0) atomicAdd(acc + k0, s);
    } else if (flag) {
        atomicAdd(acc + k, val);
    }
}

__device__ void cand_append_global(bool flag, int32_t k, int32_t v, const SArgs &A, int par) {
    unsigned am = __ballot_sync(SFULL, flag);
    if (!am) return;
    const int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(A.candctr + par, (unsigned long long)__popc(am));
    base = __shfl_sync(SFULL, base, 0);
    if (flag) {
        const int64_t idx = (int64_t)base + __popc(am & lanemask_lt_s());
        if (idx < A.candcap) A.cand[par][idx] = ((int64_t)k << 32) | (uint32_t)v;
        else A.overflow[0] = 1;
    }
}

// stage a candidate in the block buffer (spill to the global list when full)
__device__ void cand_stage(bool flag, int32_t k, int32_t v, const SStage &S, const SArgs &A,
                           int par) {
    unsigned am = __ballot_sync(SFULL, flag);
    if (!am) return;
    const int lane = threadIdx.x & 31;
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(S.ccnt, (unsigned)__popc(am));
    base = __shfl_sync(SFULL, base, 0);
    const unsigned my = base + __popc(am & lanemask_lt_s());
    const bool spill = flag && my >= (unsigned)SSTAGE;
    if (flag && !spill) {
        S.ck[my] = k;
        S.cv[my] = v;
    }
    cand_append_global(spill, k, v, A, par);
}

__device__ void cand_flush(const SStage &S, const SArgs &A, int par) {
    __syncthreads();
    const unsigned cnt = min(*S.ccnt, (unsigned)SSTAGE);
    __shared__ unsigned long long base;
    if (threadIdx.x == 0) base = cnt ? atomicAdd(A.candctr + par, (unsigned long long)cnt) : 0ULL;
    __syncthreads();
    for (unsigned i = threadIdx.x; i < cnt; i += SBT) {
        const int64_t idx = (int64_t)base + i;
        if (idx < A.candcap) A.cand[par][idx] = ((int64_t)S.ck[i] << 32) | (uint32_t)S.cv[i];
        else A.overflow[0] = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) *S.ccnt = 0;
    __syncthreads();
}

// first mark of (k, v) in the candidate map of parity par?
__device__ __forceinline__ bool cand_mark(bool flag, int32_t k, int32_t v, const SArgs &A,
                                          int par) {
    if (!flag) return false;
    uint32_t *w = A.cmark[par] + (int64_t)k * A.cmw + (v >> 5);
    const uint32_t bit = 1u << (v & 31);
    return !(atomicOr(w, bit) & bit);
}

__device__ void entry_stage(bool flag, int32_t k, int32_t u, int32_t d, double c, const SStage &S) {
    unsigned am = __ballot_sync(SFULL, flag);
    if (!am) return;
    const int lane = threadIdx.x & 31;
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(S.cnt, (unsigned)__popc(am));
    base = __shfl_sync(SFULL, base, 0);
    const unsigned my = base + __popc(am & lanemask_lt_s());
    if (flag) {  // the caller flushes before the buffer can overflow
        S.k[my] = k;
        S.v[my] = u;
        S.d[my] = d;
        S.c[my] = c;
    }
}

// Block flush of staged frontier entries: one reservation, arc offsets by a
// block scan, entry arrays + chunk map written here (the entries are final).
__device__ void entry_flush(const SStage &S, const SArgs &A, bool grp) {
    __syncthreads();
    const unsigned cnt = *S.cnt;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const unsigned per = (cnt + SBT - 1) / SBT;
    const unsigned lo = min(cnt, tid * per), hi = min(cnt, lo + per);
    unsigned long long mine = 0;
    for (unsigned i = lo; i < hi; i++) mine += (unsigned long long)S.d[i];
    unsigned long long incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(SFULL, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) S.scan[w] = incl;
    __syncthreads();
    if (tid == 0) {
        unsigned long long run = 0;
        for (int i = 0; i < SBT / 32; i++) {
            unsigned long long x = S.scan[i];
            S.scan[i] = run;
            run += x;
        }
        unsigned long long old = 0;
        if (cnt) old = atomicAdd(A.fctr, ((unsigned long long)cnt << SCNT_SHIFT) + run);
        S.scan[SBT / 32] = old;
    }
    __syncthreads();
    const unsigned long long old = S.scan[SBT / 32];
    int64_t arc = (int64_t)(old & SARC_MASK) + (int64_t)(S.scan[w] + incl - mine);
    const int64_t ebase = (int64_t)(old >> SCNT_SHIFT);
    if (grp) {  // unsorted entries + per-group counts; placed after the barrier
        for (unsigned i = lo; i < hi; i++) {
            const int64_t e = ebase + i;
            if (e < A.fcap) {
                A.ukey[e] = ((int64_t)S.k[i] << 32) | (uint32_t)S.v[i];
                A.ucval[e] = S.c[i];
            } else {
                A.overflow[0] = 1;
            }
            atomicAdd(S.gc + S.k[i] / A.sgroup, (1ULL << SCNT_SHIFT) + (unsigned long long)S.d[i]);
        }
        __syncthreads();
        for (int64_t g = tid; g < A.m; g += SBT)
            if (S.gc[g]) {
                atomicAdd(A.gcnt + g, S.gc[g]);
                S.gc[g] = 0;
            }
        __syncthreads();
        if (tid == 0) *S.cnt = 0;
        __syncthreads();
        return;
    }
    for (unsigned i = lo; i < hi; i++) {
        const int64_t e = ebase + i;
        const int32_t u = S.v[i];
        if (e < A.fcap) {
            A.fkey[e] = ((int64_t)S.k[i] << 32) | (uint32_t)u;
            A.farc[e] = arc;
            A.frow[e] = A.g.row[u];
            A.fcval[e] = S.c[i];
            const int64_t c0 = (arc + 31) >> 5, c1 = min((arc + S.d[i] + 31) >> 5, A.ccap);
            for (int64_t c = c0; c < c1; ++c) A.chunk_e[c] = (int32_t)e;
        } else {
            A.overflow[0] = 1;
        }
        arc += S.d[i];
    }
    __syncthreads();
    if (tid == 0) *S.cnt = 0;
    __syncthreads();
}

// S.gbase[g] = sum over groups j < g of A.gcnt[j] (packed), per block.
__device__ void group_bases(const SStage &S, const SArgs &A) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t per = (A.m + SBT - 1) / SBT;
    const int64_t lo = min(A.m, tid * per), hi = min(A.m, lo + per);
    unsigned long long mine = 0;
    for (int64_t g = lo; g < hi; g++) mine += A.gcnt[g];
    unsigned long long incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(SFULL, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) S.scan[w] = incl;
    __syncthreads();
    if (tid == 0) {
        unsigned long long run = 0;
        for (int i = 0; i < SBT / 32; i++) {
            unsigned long long x = S.scan[i];
            S.scan[i] = run;
            run += x;
        }
    }
    __syncthreads();
    unsigned long long b = S.scan[w] + incl - mine;
    for (int64_t g = lo; g < hi; g++) {
        S.gbase[g] = b;
        b += A.gcnt[g];
    }
    __syncthreads();
}

__device__ __forceinline__ bool slot_diverged(const SArgs &A, int32_t k) {
    return A.method == 1 && A.s_l1[k] > A.l1cap * A.s_b1[k];
}

__global__ void __launch_bounds__(SBT) k_signed_rounds(SArgs A) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char sm_raw[];
    const SStage S = sstage_carve(sm_raw, A.m);
    const int lane = threadIdx.x & 31;
    const int64_t gtid = blockIdx.x * (int64_t)SBT + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * SBT;
    const bool ch = A.method == 1;
    for (int64_t k = threadIdx.x; k < A.m; k += SBT) {
        S.l1[k] = 0.0;
        S.ops[k] = S.push[k] = 0;
        S.gc[k] = 0;
    }
    if (threadIdx.x == 0) {
        *S.cnt = 0;
        *S.ccnt = 0;
        *S.next = 0;
    }
    __syncthreads();
    int64_t ncmax = 0;  // largest candidate round so far (the same in every block)
    for (int32_t t = 0;; ++t) {
        const int cur = t & 1, nxt = cur ^ 1;
        const int64_t NC = (int64_t)*(volatile unsigned long long *)(A.candctr + cur);
        {   // final |r| of last round's landings just below theta (common.cuh)
            const int64_t nn = min((int64_t)*(volatile unsigned long long *)(A.nearl.cnt[cur]),
                                   A.nearl.cap);
            for (int64_t i = gtid; i < nn; i += nthreads) {
                const int64_t key = A.nearl.key[cur][i];
                const int32_t k = (int32_t)(key >> 32), v = (int32_t)(key & 0xffffffffLL);
                if (below_theta(fabs(A.r[(int64_t)k * A.ld + v]), theta_of(A.op, v, A.g.deg[v])))
                    A.s_amb[k] = 1;
            }
        }
        if (NC == 0) break;
        ncmax = NC > ncmax ? NC : ncmax;
        if (A.tail_list && NC <= A.tail_f && (16 * NC <= ncmax || t >= A.tail_t)) {
            if (gtid == 0) {  // the rest of the wave in k_s_tail, one block per slot
                A.tail_state[0] = t;
                A.tail_state[1] = NC;
            }
            break;
        }
        if (NC > A.candcap) {
            if (gtid == 0) A.overflow[0] = 1;
            break;
        }
        // ---------------- phase A: filter candidates, push the frontier ------
        if (gtid == 0) {
            A.fctr[0] = 0ULL;
            A.candctr[nxt] = 0ULL;
            *A.nearl.cnt[nxt] = 0ULL;
        }
        grid.sync();  // counter resets visible before any reservation
        // group only rounds with enough work to pay for the placement pass and
        // its barrier (small rounds are barrier-bound, not L2-bound)
        const bool grp = A.grouped && NC >= A.group_min;
        const double cr = (ch && t > 0) ? A.coef_r[t] : 0.0;
        const double cm = (ch && t > 0) ? A.coef_m[t] : 0.0;
        for (int64_t base = blockIdx.x * (int64_t)SBT; base < NC; base += nthreads) {
            const int64_t ci = base + threadIdx.x;
            bool act = false, fresh = false;
            int32_t k = 0, u = 0, d = 0;
            double cval = 0.0, dl1 = 0.0;
            if (ci < NC) {
                const int64_t key = A.cand[cur][ci];
                k = (int32_t)(key >> 32);
                u = (int32_t)(key & 0xffffffffLL);
                atomicAnd(A.cmark[cur] + (int64_t)k * A.cmw + (u >> 5), ~(1u << (u & 31)));
                const int64_t idx = (int64_t)k * A.ld + u;
                GD_DCHECK(k >= 0 && k < A.m && u >= 0 && u < A.g.n);
                const double ru = A.r[idx];
                d = A.g.deg[u];
                const double th = theta_of(A.op, u, d);
                if (near_theta(fabs(ru), th)) A.s_amb[k] = 1;
                act = fabs(ru) >= th && !slot_diverged(A, k);
                if (act && t >= A.max_sweeps) {  // sweep cap reached with work left
                    A.s_conv[k] = 0;
                    act = false;
                }
                if (act) {
                    double v;
                    if (!ch) {
                        v = ru;
                    } else if (t == 0) {
                        v = __dmul_rn(A.step0, ru);
                    } else {
                        const double prev = (A.mstamp[idx] == t - 1) ? A.mom[idx] : 0.0;
                        v = __dadd_rn(__dmul_rn(cr, ru), __dmul_rn(cm, prev));
                    }
                    A.x[idx] = __dadd_rn(A.x[idx], v);
                    const double rn = __dsub_rn(ru, v);
                    A.r[idx] = rn;
                    if (ch) {
                        dl1 = fabs(rn) - fabs(ru);
                        fresh = A.mstamp[idx] == -1;
                        A.mom[idx] = v;
                        A.mstamp[idx] = t;
                    }
                    cval = __dmul_rn(v, node_weight(A.op, d));
                    A.s_last[k] = t;
                }
            }
            if (ch) {  // pushed-node list (x support; mstamp reset)
                unsigned am = __ballot_sync(SFULL, fresh);
                if (fresh) {
                    unsigned peers = __match_any_sync(am, k);
                    const int leader = __ffs(peers) - 1;
                    unsigned long long b = 0;
                    if (lane == leader)
                        b = atomicAdd(A.pushed_cnt + k, (unsigned long long)__popc(peers));
                    b = __shfl_sync(peers, b, leader);
                    A.pushed[(int64_t)k * A.ld + (int64_t)b + __popc(peers & lanemask_lt_s())] = u;
                }
                slot_add_d(act, k, dl1, S.l1);
            }
            slot_add_u(act, k, (unsigned)d, S.ops);
            slot_add_u(act, k, 1u, S.push);
            entry_stage(act, k, u, d, cval, S);
            // under momentum a pushed node keeps a residual: candidate again
            const bool again = cand_mark(ch && act, k, u, A, nxt);
            cand_stage(again, k, u, S, A, nxt);
            __syncthreads();
            if (*S.cnt > (unsigned)(SSTAGE - SBT)) entry_flush(S, A, grp);
        }
        entry_flush(S, A, grp);
        for (int64_t k = threadIdx.x; k < A.m; k += SBT) {
            if (S.ops[k]) { atomicAdd(A.s_ops + k, S.ops[k]); S.ops[k] = 0; }
            if (S.push[k]) { atomicAdd(A.s_pushes + k, S.push[k]); S.push[k] = 0; }
        }
        grid.sync();
        const unsigned long long pk = *(volatile unsigned long long *)A.fctr;
        const int64_t F = (int64_t)(pk >> SCNT_SHIFT), P = (int64_t)(pk & SARC_MASK);
        if (F > A.fcap || ((P + 31) >> 5) > A.ccap) {
            if (gtid == 0) A.overflow[0] = 1;
            break;
        }
        if (grp) {
            // ---------------- placement: frontier grouped by slot group -------
            group_bases(S, A);
            for (int64_t e0 = gtid - lane; e0 < F; e0 += nthreads) {
                const int64_t e = e0 + lane;
                const bool live = e < F;
                int64_t key = 0;
                int32_t k = 0, u = 0, d = 0;
                if (live) {
                    key = A.ukey[e];
                    k = (int32_t)(key >> 32);
                    u = (int32_t)(key & 0xffffffffLL);
                    d = A.g.deg[u];
                }
                const int32_t g = k / (int32_t)A.sgroup;
                const unsigned long long pv = live ? (1ULL << SCNT_SHIFT) + (unsigned long long)d : 0ULL;
                const unsigned peers = __match_any_sync(SFULL, live ? g : -1);
                unsigned long long pre = 0, tot = 0;
                for (int i = 0; i < 32; ++i) {
                    const unsigned long long vi = __shfl_sync(SFULL, pv, i);
                    if ((peers >> i) & 1u) {
                        tot += vi;
                        if (i < lane) pre += vi;
                    }
                }
                const int leader = __ffs(peers) - 1;
                unsigned long long o = 0;
                if (live && lane == leader) o = atomicAdd(A.gfill + g, tot);
                o = __shfl_sync(SFULL, o, leader);
                if (live) {
                    const unsigned long long b = S.gbase[g] + o + pre;
                    const int64_t pos = (int64_t)(b >> SCNT_SHIFT), a0 = (int64_t)(b & SARC_MASK);
                    A.fkey[pos] = key;
                    A.farc[pos] = a0;
                    A.frow[pos] = A.g.row[u];
                    A.fcval[pos] = A.ucval[e];
                    const int64_t c0 = (a0 + 31) >> 5, c1 = min((a0 + d + 31) >> 5, A.ccap);
                    for (int64_t c = c0; c < c1; ++c) A.chunk_e[c] = (int32_t)pos;
                }
            }
            grid.sync();
            for (int64_t g = gtid; g < A.m; g += nthreads) {  // (read by every block above)
                A.gcnt[g] = 0ULL;
                A.gfill[g] = 0ULL;
            }
        }
        // ---------------- phase B: arc chunks -------------------------------
        const int64_t C = (P + 31) >> 5;
        const int64_t bc0 = (int64_t)(((unsigned long long)C * blockIdx.x) / gridDim.x);
        const int64_t bc1 = (int64_t)(((unsigned long long)C * (blockIdx.x + 1)) / gridDim.x);
        for (;;) {
            unsigned long long claim = 0;
            if (lane == 0) claim = atomicAdd(S.next, 1ULL);
            const int64_t ci = (int64_t)__shfl_sync(SFULL, claim, 0);
            int64_t cb, cend;
            if (grp) {  // super-chunks b, b + G, ...: the grid advances together
                const int64_t sup = ci / SSUPER, within = ci - sup * SSUPER;
                cb = ((sup * gridDim.x + blockIdx.x) * SSUPER + within) * SUNROLL;
                cend = C;
            } else {  // this block's contiguous range
                cb = bc0 + ci * SUNROLL;
                cend = bc1;
            }
            if (cb >= cend) break;
            int32_t k[SUNROLL], v[SUNROLL], dv[SUNROLL];
            double c[SUNROLL], old[SUNROLL];
            bool valid[SUNROLL];
#pragma unroll
            for (int q = 0; q < SUNROLL; q++) {
                const int64_t chn = cb + q;
                const bool live = chn < cend;
                const int64_t e = live ? A.chunk_e[chn] : 0;
                const int64_t a = chn << 5;
                const int64_t wi = e + 1 + lane;
                const int64_t st = (live && wi < F) ? A.farc[wi] : INT64_MAX;
                const int64_t pos = st - a;
                const unsigned starts = __reduce_or_sync(SFULL, pos < 32 ? (1u << pos) : 0u);
                const int64_t me = e + __popc(starts & ((2u << lane) - 1u));
                const int64_t p = a + lane;
                valid[q] = live && p < P;
                k[q] = 0;
                v[q] = 0;
                c[q] = 0.0;
                dv[q] = 0;
                if (valid[q]) {
                    k[q] = (int32_t)(A.fkey[me] >> 32);
                    c[q] = A.fcval[me];
                    const int2 nd = A.colp[A.frow[me] + (p - A.farc[me])];
                    v[q] = nd.x;
                    dv[q] = nd.y;
                }
            }
#pragma unroll
            for (int q = 0; q < SUNROLL; q++) {
                GD_DCHECK(!valid[q] || (k[q] >= 0 && k[q] < A.m && v[q] >= 0 && v[q] < A.g.n));
                old[q] = valid[q] ? atomicAdd(A.r + (int64_t)k[q] * A.ld + v[q], c[q]) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < SUNROLL; q++) {
                // the value this atomic stored; the LAST update of a node in
                // the round stores its final value, so a node active at the
                // end of the round is marked by at least one of its updates
                const double nv = __dadd_rn(old[q], c[q]);
                if (ch) slot_add_d(valid[q], k[q], valid[q] ? fabs(nv) - fabs(old[q]) : 0.0, S.l1);
                if (A.secmap && valid[q] && __double_as_longlong(old[q]) == 0)
                    atomicOr(A.secmap + (int64_t)k[q] * A.smw + (v[q] >> 7),
                             1u << ((v[q] >> 2) & 31));
                const double th = theta_of(A.op, v[q], dv[q]);
                // mark on a cold -> hot transition only: an update that finds
                // |old| >= theta follows one that stored that hot value (and
                // marks, or has marked, the node) -- at the round start every
                // hot node is a frontier node already re-marked by phase A
                // ("again") or was filtered out as inactive (cap / divergence)
                const bool rise = valid[q] && fabs(nv) >= th && !(fabs(old[q]) >= th);
                // a node whose final |r| sits just below theta is never a
                // candidate: its landings there are re-read after the round
                if (valid[q] && below_theta(fabs(nv), th))
                    near_record(A.nearl, nxt, k[q], v[q], A.s_amb);
                const bool nw = cand_mark(rise, k[q], v[q], A, nxt);
                cand_stage(nw, k[q], v[q], S, A, nxt);
            }
        }
        cand_flush(S, A, nxt);
        if (threadIdx.x == 0) *S.next = 0;
        for (int64_t k = threadIdx.x; k < A.m; k += SBT)
            if (S.l1[k] != 0.0) {
                atomicAdd(A.s_l1 + k, S.l1[k]);
                S.l1[k] = 0.0;
            }
        grid.sync();
    }
}

// ---------------------------------------------------------------------------
// k_s_tail: the CTA-local tail of a signed wave (LocalCH / LocalHB), the
// counterpart of batch.cu's k_tail.  Katz waves on the products shape run ~100-
// 240 rounds of a few hundred arcs per seed, where the cooperative round
// kernel's three grid barriers per round are the whole cost.  Block k takes
// slot k's candidates of round t and runs the remaining sweeps alone with the
// same rules as k_signed_rounds: phase A filters candidates (|r| >= theta, not
// diverged, sweep cap) and pushes them with the Chebyshev / heavy-ball
// recurrence, keeping the momentum and the incremental l1; phase B scatters
// the entries' arcs (block-balanced: degrees block-scanned per segment, binary
// search per arc) with returning atomics, marks a candidate on a cold -> hot
// transition, the sector map on first touch, landings just below theta for the
// final check.  Sweeps stay numbered as rounds.
constexpr int STAIL_SEG = 1024;
constexpr int STAIL_NEAR = 256;
constexpr int SUNROLL_T = 4;

__global__ void __launch_bounds__(SBT, 1) k_s_tail(const __grid_constant__ SArgs A) {
    using Scan = cub::BlockScan<int, SBT>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ double tc[STAIL_SEG];
    __shared__ int64_t trow[STAIL_SEG];
    __shared__ int32_t toff[STAIL_SEG + 1], tnear[STAIL_NEAR];
    __shared__ int s_cur, s_nxt, s_ne, s_nn, s_amb;
    __shared__ unsigned long long c_ops, c_push;
    __shared__ double c_l1;
    const int64_t NC = A.tail_state[1];
    if (NC < 0) return;  // the wave ended in the round kernel
    int32_t t = (int32_t)A.tail_state[0];
    const int tid = threadIdx.x, lane = tid & 31;
    const int32_t k = (int32_t)blockIdx.x;
    const int64_t C = A.g.n;
    int32_t *const l0 = A.tail_list + (int64_t)k * 3 * C, *const l1 = l0 + C, *const eu = l1 + C;
    double *const ec = A.tail_c + (int64_t)k * C;
    const int64_t off = (int64_t)k * A.ld;
    double *const r = A.r + off;
    const bool ch = A.method == 1;
    if (tid == 0) {
        s_cur = s_nn = s_amb = 0;
    }
    __syncthreads();
    for (int64_t e0 = 0; e0 < NC; e0 += SBT) {  // this slot's candidates of round t
        const int64_t e = e0 + tid;
        const int64_t key = e < NC ? A.cand[t & 1][e] : -1;
        const bool mine = e < NC && (int32_t)(key >> 32) == k;
        const unsigned am = __ballot_sync(SFULL, mine);
        int base = 0;
        if (am && lane == __ffs(am) - 1) base = atomicAdd(&s_cur, __popc(am));
        base = __shfl_sync(SFULL, base, __ffs(am ? am : 1u) - 1);
        if (mine) l0[base + __popc(am & lanemask_lt_s())] = (int32_t)(key & 0xffffffffLL);
    }
    int cur = 0;
    __syncthreads();
    for (;; ++t) {
        const int par = t & 1, npar = par ^ 1;
        const int nn = min(s_nn, STAIL_NEAR);
        for (int i = tid; i < nn; i += SBT)
            if (below_theta(fabs(r[tnear[i]]), theta_of(A.op, tnear[i], A.g.deg[tnear[i]])))
                s_amb = 1;
        __syncthreads();
        const int Fc = s_cur;
        if (Fc == 0) break;
        if (tid == 0) {
            s_nn = 0;
            s_nxt = 0;
            s_ne = 0;
            c_ops = c_push = 0ULL;
            c_l1 = 0.0;
        }
        __syncthreads();
        int32_t *const cl = cur ? l1 : l0, *const nl = cur ? l0 : l1;
        const bool div = slot_diverged(A, k);
        const double cr = (ch && t > 0) ? A.coef_r[t] : 0.0;
        const double cm = (ch && t > 0) ? A.coef_m[t] : 0.0;
        // ---- phase A: candidates -> |r| >= theta ? push : skip
        double my_l1 = 0.0;
        for (int i0 = 0; i0 < Fc; i0 += SBT) {  // warp-uniform trips
            const int i = i0 + tid;
            const bool live = i < Fc;
            bool act = false, fresh = false;
            int32_t u = 0, d = 0;
            double c = 0.0;
            if (live) {
                u = cl[i];
                atomicAnd(A.cmark[par] + (int64_t)k * A.cmw + (u >> 5), ~(1u << (u & 31)));
                const int64_t idx = off + u;
                const double ru = A.r[idx];
                d = A.g.deg[u];
                const double th = theta_of(A.op, u, d);
                if (near_theta(fabs(ru), th)) s_amb = 1;
                act = fabs(ru) >= th && !div;
                if (act && t >= A.max_sweeps) {  // sweep cap reached with work left
                    A.s_conv[k] = 0;
                    act = false;
                }
                if (act) {
                    double v;
                    if (!ch) {
                        v = ru;
                    } else if (t == 0) {
                        v = __dmul_rn(A.step0, ru);
                    } else {
                        const double prev = (A.mstamp[idx] == t - 1) ? A.mom[idx] : 0.0;
                        v = __dadd_rn(__dmul_rn(cr, ru), __dmul_rn(cm, prev));
                    }
                    A.x[idx] = __dadd_rn(A.x[idx], v);
                    const double rn = __dsub_rn(ru, v);
                    A.r[idx] = rn;
                    if (ch) {
                        my_l1 += fabs(rn) - fabs(ru);
                        fresh = A.mstamp[idx] == -1;
                        A.mom[idx] = v;
                        A.mstamp[idx] = t;
                    }
                    c = __dmul_rn(v, node_weight(A.op, d));
                    A.s_last[k] = t;
                }
            }
            {   // pushed-node list (x support)
                const unsigned fm = __ballot_sync(SFULL, fresh);
                if (fm) {
                    unsigned long long b = 0;
                    if (lane == __ffs(fm) - 1)
                        b = atomicAdd(A.pushed_cnt + k, (unsigned long long)__popc(fm));
                    b = __shfl_sync(SFULL, b, __ffs(fm) - 1);
                    if (fresh) A.pushed[off + (int64_t)b + __popc(fm & lanemask_lt_s())] = u;
                }
            }
            {   // frontier entry (u, c) and the counters
                const unsigned am = __ballot_sync(SFULL, act);
                if (am) {
                    int b = 0;
                    if (lane == __ffs(am) - 1) b = atomicAdd(&s_ne, __popc(am));
                    b = __shfl_sync(SFULL, b, __ffs(am) - 1);
                    if (act) {
                        const int at = b + __popc(am & lanemask_lt_s());
                        eu[at] = u;
                        ec[at] = c;
                    }
                    const unsigned ds = __reduce_add_sync(SFULL, act ? (unsigned)d : 0u);
                    if (lane == __ffs(am) - 1) {
                        atomicAdd(&c_ops, (unsigned long long)ds);
                        atomicAdd(&c_push, (unsigned long long)__popc(am));
                    }
                }
            }
            {   // under momentum a pushed node keeps a residual: candidate again
                const bool again = cand_mark(ch && act, k, u, A, npar);
                const unsigned gm = __ballot_sync(SFULL, again);
                if (gm) {
                    int b = 0;
                    if (lane == __ffs(gm) - 1) b = atomicAdd(&s_nxt, __popc(gm));
                    b = __shfl_sync(SFULL, b, __ffs(gm) - 1);
                    if (again) nl[b + __popc(gm & lanemask_lt_s())] = u;
                }
            }
        }
        __syncthreads();
        // ---- phase B: the entries' arcs
        const int Fe = s_ne;
        for (int seg0 = 0; seg0 < Fe; seg0 += STAIL_SEG) {
            const int ns = min(STAIL_SEG, Fe - seg0);
            constexpr int PER = STAIL_SEG / SBT;
            int dd[PER];
            int mine = 0;
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const int i = tid * PER + j;
                dd[j] = 0;
                if (i < ns) {
                    const int32_t u = eu[seg0 + i];
                    dd[j] = A.g.deg[u];
                    trow[i] = A.g.row[u];
                    tc[i] = ec[seg0 + i];
                }
                mine += dd[j];
            }
            int excl = 0, tot = 0;
            Scan(scan_tmp).ExclusiveSum(mine, excl, tot);
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const int i = tid * PER + j;
                if (i < ns) toff[i] = excl;
                excl += dd[j];
            }
            if (tid == 0) toff[ns] = tot;
            __syncthreads();
            const int P = tot;
            for (int p0 = tid; p0 - tid < P; p0 += SBT * SUNROLL_T) {  // warp-uniform trips
                int32_t v[SUNROLL_T], dv[SUNROLL_T];
                double c[SUNROLL_T], old[SUNROLL_T];
                bool valid[SUNROLL_T];
#pragma unroll
                for (int q = 0; q < SUNROLL_T; ++q) {
                    const int p = p0 + q * SBT;
                    valid[q] = p < P;
                    v[q] = 0; dv[q] = 0; c[q] = 0.0;
                    if (valid[q]) {
                        int lo = 0, hi = ns - 1;  // last entry with toff <= p
                        while (lo < hi) {
                            const int mid = (lo + hi + 1) >> 1;
                            if (toff[mid] <= p) lo = mid; else hi = mid - 1;
                        }
                        c[q] = tc[lo];
                        const int2 nd = A.colp[trow[lo] + (p - toff[lo])];
                        v[q] = nd.x;
                        dv[q] = nd.y;
                    }
                }
#pragma unroll
                for (int q = 0; q < SUNROLL_T; ++q) {
                    GD_DCHECK(!valid[q] || (v[q] >= 0 && v[q] < A.g.n));
                    old[q] = valid[q] ? atomicAdd(r + v[q], c[q]) : 0.0;
                }
#pragma unroll
                for (int q = 0; q < SUNROLL_T; ++q) {
                    const double nv = __dadd_rn(old[q], c[q]);
                    if (ch && valid[q]) my_l1 += fabs(nv) - fabs(old[q]);
                    if (A.secmap && valid[q] && __double_as_longlong(old[q]) == 0)
                        atomicOr(A.secmap + (int64_t)k * A.smw + (v[q] >> 7), 1u << ((v[q] >> 2) & 31));
                    const double th = theta_of(A.op, v[q], dv[q]);
                    const bool rise = valid[q] && fabs(nv) >= th && !(fabs(old[q]) >= th);
                    if (valid[q] && below_theta(fabs(nv), th)) {
                        const int at = atomicAdd(&s_nn, 1);
                        if (at < STAIL_NEAR) tnear[at] = v[q]; else s_amb = 1;
                    }
                    const bool nw = cand_mark(rise, k, v[q], A, npar);
                    const unsigned gm = __ballot_sync(SFULL, nw);
                    if (gm) {
                        int b = 0;
                        if (lane == __ffs(gm) - 1) b = atomicAdd(&s_nxt, __popc(gm));
                        b = __shfl_sync(SFULL, b, __ffs(gm) - 1);
                        if (nw) nl[b + __popc(gm & lanemask_lt_s())] = v[q];
                    }
                }
            }
            __syncthreads();
        }
        if (ch) {
            for (int o = 16; o > 0; o >>= 1) my_l1 += __shfl_xor_sync(SFULL, my_l1, o);
            if (lane == 0 && my_l1 != 0.0) atomicAdd(&c_l1, my_l1);
        }
        __syncthreads();
        if (tid == 0) {
            A.s_ops[k] += c_ops;
            A.s_pushes[k] += c_push;
            if (ch) A.s_l1[k] += c_l1;
            s_cur = s_nxt;
        }
        cur ^= 1;
        __syncthreads();
    }
    if (tid == 0 && s_amb) A.s_amb[k] = 1;
}

__global__ void k_s_pack_cols(DevGraph g, int2 *__restrict__ colp) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < g.n_arcs;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = g.col[j];
        colp[j] = make_int2(v, g.deg[v]);
    }
}

// ---- cold waves (gd_batch, GD_M_LOCAL_CH) ---------------------------------

// seeds -> slots: r[s] = b_s, the seed is the only round-0 candidate
__global__ void k_s_init(SArgs A, const int64_t *__restrict__ seeds, const int32_t *perm,
                         double bval) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k == 0) {
        A.candctr[0] = (unsigned long long)A.m;
        A.candctr[1] = 0ULL;
    }
    if (k >= A.m) return;
    int32_t s = (int32_t)seeds[k];
    if (perm) s = perm[s];
    A.r[k * A.ld + s] = bval;
    A.secmap[k * A.smw + (s >> 7)] |= 1u << ((s >> 2) & 31);
    A.cmark[0][k * A.cmw + (s >> 5)] |= 1u << (s & 31);
    A.cand[0][k] = (k << 32) | (uint32_t)s;
    A.pushed_cnt[k] = 0;
    A.s_ops[k] = 0;
    A.s_pushes[k] = 0;
    A.s_l1[k] = fabs(bval);
    A.s_b1[k] = fabs(bval);
    A.s_last[k] = -1;
    A.s_conv[k] = 1;
    A.s_amb[k] = 0;
}

__global__ void k_s_reserve(SArgs A, unsigned long long *cursor, int64_t *slot_base) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < A.m) slot_base[k] = (int64_t)atomicAdd(cursor, A.pushed_cnt[k]);
}

struct SOut {
    int64_t *sweeps, *ops, *pushes, *support, *xoff, *xcnt;
    int32_t *conv;
    int32_t *xnodes;
    double *xvals;
    int64_t xcap;
    const int32_t *inv;
    const int64_t *slot_base;
    int32_t *amb;
    unsigned long long *amb_cnt;
};

// grid (SCHUNKS, slots): x over the pushed list out (caller ids); x, mstamp
// back to their idle values; block (0, k) writes the seed's counters.
__global__ void k_s_extract(SArgs A, SOut O, int64_t seed_base) {
    const int k = blockIdx.y;
    const int64_t off = (int64_t)k * A.ld;
    const int64_t pc = (int64_t)A.pushed_cnt[k];
    const int64_t b = O.slot_base[k];
    // XU entries per thread, every load before any store (as k_wave_extract)
    constexpr int XU = 4;
    const int64_t stride = (int64_t)SCHUNKS * blockDim.x;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < pc; i0 += XU * stride) {
        int32_t u[XU], id[XU];
        double xv[XU];
#pragma unroll
        for (int j = 0; j < XU; ++j) {
            const int64_t i = i0 + j * stride;
            u[j] = i < pc ? __ldg(A.pushed + off + i) : -1;
        }
#pragma unroll
        for (int j = 0; j < XU; ++j) {
            xv[j] = u[j] >= 0 ? A.x[off + u[j]] : 0.0;
            id[j] = (u[j] >= 0 && O.inv) ? __ldg(O.inv + u[j]) : u[j];
        }
#pragma unroll
        for (int j = 0; j < XU; ++j) {
            const int64_t i = i0 + j * stride;
            if (u[j] < 0) continue;
            A.x[off + u[j]] = 0.0;
            A.mstamp[off + u[j]] = -1;
            if (b + i < O.xcap) {
                O.xnodes[b + i] = id[j];
                O.xvals[b + i] = xv[j];
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t si = seed_base + k;
        O.sweeps[si] = (int64_t)A.s_last[k] + 1;
        O.ops[si] = (int64_t)A.s_ops[k];
        O.pushes[si] = (int64_t)A.s_pushes[k];
        O.conv[si] = (A.s_conv[k] && !slot_diverged(A, k)) ? 1 : 0;
        O.support[si] = -1;  // not tracked for signed solves
        O.xoff[si] = b;
        O.xcnt[si] = pc;
        O.amb[si] = A.s_amb[k];
        if (A.s_amb[k]) atomicAdd(O.amb_cnt, 1ULL);
    }
}

// grid (SCHUNKS, slots): zero exactly the 32 B sectors of r a slot wrote; a
// warp clears one map word (1 KB of r) per step with one store per lane.
__global__ void k_s_reset(SArgs A) {
    const int k = blockIdx.y;
    const int64_t per = (A.smw + gridDim.x - 1) / gridDim.x;  // gridDim.x scales with the map
    const int64_t lo = blockIdx.x * per, hi = min(A.smw, lo + per);
    reset_sector_words(A.secmap + (int64_t)k * A.smw, A.r + (int64_t)k * A.ld, A.ld, lo, hi);
}

// ---- resident pairs (gd_pairs) ------------------------------------------

struct PairEvent {
    int32_t u, v, du, dv;  // endpoints and their degrees before the event
    int32_t step;          // +1 insert, -1 delete
};

// Endpoint a of edge (a, b), degree d0 -> d1 (src/dynamic.py:70-98), with
// numpy's evaluation order: p*(d1/d0), (1-alpha)*p/d1 = fl(fl(q p) / d1).
__device__ __forceinline__ void pair_endpoint(double *p, double *r, double q, int32_t a,
                                              int32_t b, int32_t d0, int32_t d1) {
    const double fd0 = (double)d0, fd1 = (double)d1;
    if (d1 > d0) {
        if (d0 > 0) {
            p[a] = __dmul_rn(p[a], __ddiv_rn(fd1, fd0));
            r[a] = __dsub_rn(r[a], __ddiv_rn(p[a], fd1));
        }
        r[b] = __dadd_rn(r[b], __ddiv_rn(__dmul_rn(q, p[a]), fd1));
    } else {
        const double ratio = __ddiv_rn(p[a], fd0);
        if (d1 > 0) {
            p[a] = __dmul_rn(p[a], __ddiv_rn(fd1, fd0));
            r[a] = __dadd_rn(r[a], __ddiv_rn(p[a], fd1));
        } else {
            r[a] = __dadd_rn(r[a], p[a]);
            p[a] = 0.0;
        }
        r[b] = __dsub_rn(r[b], __dmul_rn(q, ratio));
    }
}

// One dependency level of the event batch: the events of a level share no
// node, so thread (event, pair) applies one event to one pair and the
// per-node order of operations -- hence every bit -- is the sequential
// reference's.  Endpoints become round-0 candidates of the repair.
__global__ void k_pair_events(SArgs A, const PairEvent *__restrict__ ev, int64_t n_ev, double q) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_ev * A.m) return;
    const int64_t k = t % A.m, i = t / A.m;
    double *p = A.x + k * A.ld, *r = A.r + k * A.ld;
    const PairEvent e = ev[i];
    pair_endpoint(p, r, q, e.u, e.v, e.du, e.du + e.step);
    pair_endpoint(p, r, q, e.v, e.u, e.dv, e.dv + e.step);
    const int32_t ends[2] = {e.u, e.v};
    for (int j = 0; j < 2; ++j) {
        const int32_t a = ends[j];
        const uint32_t bit = 1u << (a & 31);
        if (!(atomicOr(A.cmark[0] + k * A.cmw + (a >> 5), bit) & bit)) {
            const unsigned long long at = atomicAdd(A.candctr, 1ULL);
            if ((int64_t)at < A.candcap) A.cand[0][at] = (k << 32) | (uint32_t)a;
            else A.overflow[0] = 1;
        }
    }
}

// every active node of every pair as a round-0 candidate (pool creation,
// or after a repair that stopped at max_sweeps)
__global__ void k_pair_scan(SArgs A) {
    const int64_t total = A.m * A.ld;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = i / A.ld, u = i - k * A.ld;
        if (u >= A.g.n) continue;
        const double ru = A.r[i];
        if (ru == 0.0 || !(fabs(ru) >= theta_of(A.op, u, A.g.deg[u]))) continue;
        uint32_t *w = A.cmark[0] + k * A.cmw + (u >> 5);
        const uint32_t bit = 1u << (u & 31);
        if (atomicOr(w, bit) & bit) continue;
        const unsigned long long at = atomicAdd(A.candctr, 1ULL);
        if ((int64_t)at < A.candcap) A.cand[0][at] = (k << 32) | (uint32_t)u;
        else A.overflow[0] = 1;
    }
}

__global__ void k_gather_deg(DevGraph g, const int32_t *__restrict__ nodes, int64_t c,
                             int32_t *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < c) out[i] = g.deg[nodes[i]];
}

__global__ void k_pair_stats_reset(SArgs A) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= A.m) return;
    A.s_ops[k] = 0;
    A.s_pushes[k] = 0;
    A.s_last[k] = -1;
    A.s_conv[k] = 1;
}

}  // namespace

// ---------------------------------------------------------------------------
// Shared state of both drivers.
// ---------------------------------------------------------------------------
struct SignedState {
    int device = 0;
    int method = 0;
    int slots = 0, grid = 0;
    int64_t n = 0, ld = 0, fcap = 0, ccap = 0, candcap = 0, cmw = 0, smw = 0, max_sweeps = 0;
    DevOp op{};
    double step0 = 0.0, l1cap = 10.0;
    DBuf<double> coef_r, coef_m;
    DBuf<double> x, r, mom, fcval, s_l1, s_b1;
    DBuf<int32_t> mstamp, pushed, chunk_e, s_last, s_conv, s_amb, overflow;
    DBuf<int64_t> nearkey;
    DBuf<unsigned long long> nearcnt;
    static constexpr int64_t NEAR_CAP = 1 << 16;
    DBuf<uint32_t> cm0, cm1, secmap;
    DBuf<int64_t> cand0, cand1, fkey, farc, frow, slot_base;
    DBuf<int2> colp;
    int grouped = 0;
    int64_t sgroup = 1, group_min = 1 << 16;
    DBuf<int64_t> ukey;
    DBuf<double> ucval;
    DBuf<unsigned long long> gcnt, gfill;
    DBuf<unsigned long long> candctr, fctr, s_ops, s_pushes, pushed_cnt;
    bool dirty = false;  // an aborted run left marks behind: full clear next time
    size_t smem = 0;
    // CTA-local tails (k_s_tail, cold LocalCH / LocalHB waves): 3 x n int32 + n
    // doubles per slot, when that costs <= 4 GB (GDIFF_TAIL=0: off)
    DBuf<int32_t> tail_list;
    DBuf<double> tail_c;
    DBuf<int64_t> tail_state;
    int64_t tail_f = 1 << 13;
    int32_t tail_t = 16;
    bool tail_on = false;

    void alloc(const gd_graph *W, int method_, int slots_, int64_t fcap_, bool cold) {
        device = W->device;
        method = method_;
        slots = slots_;
        n = W->n;
        ld = ((n ? n : 1) + 3) & ~3LL;
        cmw = (ld + 31) / 32;
        smw = (ld / 4 + 31) / 32;
        const size_t sn = (size_t)slots * (size_t)ld;
        x.alloc(sn); r.alloc(sn);
        GD_CUDA(cudaMemset(x.p, 0, sizeof(double) * sn));
        GD_CUDA(cudaMemset(r.p, 0, sizeof(double) * sn));
        if (method == 1) {
            mom.alloc(sn);
            mstamp.alloc(sn);
            pushed.alloc(sn);
            GD_CUDA(cudaMemset(mstamp.p, 0xFF, sizeof(int32_t) * sn));  // -1: never pushed
        }
        cm0.alloc((size_t)slots * cmw); cm1.alloc((size_t)slots * cmw);
        GD_CUDA(cudaMemset(cm0.p, 0, sizeof(uint32_t) * (size_t)slots * cmw));
        GD_CUDA(cudaMemset(cm1.p, 0, sizeof(uint32_t) * (size_t)slots * cmw));
        if (cold) {
            secmap.alloc((size_t)slots * smw);
            GD_CUDA(cudaMemset(secmap.p, 0, sizeof(uint32_t) * (size_t)slots * smw));
        }
        fcap = fcap_;
        ccap = fcap_;
        candcap = fcap_;
        cand0.alloc(candcap); cand1.alloc(candcap);
        fkey.alloc(fcap); farc.alloc(fcap); frow.alloc(fcap); fcval.alloc(fcap);
        {  // slot groups of ~96 MB of residual vectors; one group = ungrouped mode
            int64_t gsz = (96LL << 20) / (ld * 8);
            if (const char *e = getenv("GDIFF_SLOT_GROUP")) gsz = atoll(e);  // experiments
            sgroup = gsz < 1 ? 1 : (gsz > slots ? slots : gsz);
            grouped = sgroup < slots ? 1 : 0;
            if (const char *e = getenv("GDIFF_GROUP_MIN")) group_min = atoll(e);  // (tests)
        }
        if (grouped) {
            ukey.alloc(fcap); ucval.alloc(fcap);
        }
        gcnt.alloc(slots); gfill.alloc(slots);
        GD_CUDA(cudaMemset(gcnt.p, 0, sizeof(unsigned long long) * slots));
        GD_CUDA(cudaMemset(gfill.p, 0, sizeof(unsigned long long) * slots));
        chunk_e.alloc(ccap);
        candctr.alloc(2); fctr.alloc(1); overflow.alloc(1);
        s_ops.alloc(slots); s_pushes.alloc(slots); pushed_cnt.alloc(slots);
        s_l1.alloc(slots); s_b1.alloc(slots); s_last.alloc(slots); s_conv.alloc(slots);
        s_amb.alloc(slots);
        GD_CUDA(cudaMemset(s_amb.p, 0, sizeof(int32_t) * slots));
        nearkey.alloc(2 * NEAR_CAP);
        nearcnt.alloc(2);
        GD_CUDA(cudaMemset(nearcnt.p, 0, 2 * sizeof(unsigned long long)));
        slot_base.alloc(slots);
        GD_CUDA(cudaMemset(s_l1.p, 0, sizeof(double) * slots));
        GD_CUDA(cudaMemset(s_b1.p, 0, sizeof(double) * slots));
        smem = sstage_bytes(slots);
        GD_CUDA(cudaFuncSetAttribute(k_signed_rounds, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        int per_sm = 0;
        GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_signed_rounds, SBT, smem));
        GD_CHECK_ARG(per_sm > 0, "signed round kernel does not fit on an SM");
        grid = per_sm * n_sms(device);
    }

    // (neighbour, degree) per arc of the graph the next solves run on
    void pack(const gd_graph *W, cudaStream_t st) {
        colp.ensure(W->n_arcs ? W->n_arcs : 1);
        if (W->n_arcs) k_s_pack_cols<<<4 * n_sms(device), 256, 0, st>>>(W->view(), colp.p);
        GD_LAUNCH_CHECK();
    }

    // LocalHB: constant heavy-ball coefficients (eta r + beta prev; sweep 0 eta r)
    void set_hb(double mu, double L, int64_t max_sweeps_) {
        max_sweeps = max_sweeps_;
        double eta = 0.0, beta = 0.0;
        hb_coefficients(mu, L, &eta, &beta);
        step0 = eta;
        const int64_t T = max_sweeps + 1;
        std::vector<double> cr(T, eta), cmv(T, beta);
        coef_r.alloc(T);
        coef_m.alloc(T);
        GD_CUDA(cudaMemcpy(coef_r.p, cr.data(), sizeof(double) * T, cudaMemcpyHostToDevice));
        GD_CUDA(cudaMemcpy(coef_m.p, cmv.data(), sizeof(double) * T, cudaMemcpyHostToDevice));
    }

    void set_ch(double mu, double L, int64_t max_sweeps_) {
        max_sweeps = max_sweeps_;
        step0 = 2.0 / (L + mu);
        // delta recurrence of src/local_solvers.py:508-520, per sweep index
        const int64_t T = max_sweeps + 1;
        std::vector<double> cr(T, 0.0), cmv(T, 0.0);
        double delta = (L - mu) / (L + mu);
        for (int64_t t = 1; t < T; ++t) {
            const double dn = 1.0 / (2.0 * (L + mu) / (L - mu) - delta);
            cr[t] = 4.0 * dn / (L - mu);
            cmv[t] = delta * dn;
            delta = dn;
        }
        coef_r.alloc(T);
        coef_m.alloc(T);
        GD_CUDA(cudaMemcpy(coef_r.p, cr.data(), sizeof(double) * T, cudaMemcpyHostToDevice));
        GD_CUDA(cudaMemcpy(coef_m.p, cmv.data(), sizeof(double) * T, cudaMemcpyHostToDevice));
    }

    SArgs args(const gd_graph *W, int64_t m) {
        SArgs A{};
        A.g = W->view();
        A.op = op;
        A.method = method;
        A.m = m;
        A.ld = ld;
        A.max_sweeps = max_sweeps;
        A.fcap = fcap; A.ccap = ccap; A.candcap = candcap;
        A.x = x.p; A.r = r.p; A.mom = mom.p; A.mstamp = mstamp.p;
        A.coef_r = coef_r.p; A.coef_m = coef_m.p;
        A.step0 = step0; A.l1cap = l1cap;
        A.pushed = pushed.p; A.pushed_cnt = pushed_cnt.p;
        A.cmark[0] = cm0.p; A.cmark[1] = cm1.p; A.cmw = cmw;
        A.secmap = secmap.p; A.smw = smw;
        A.cand[0] = cand0.p; A.cand[1] = cand1.p; A.candctr = candctr.p;
        A.colp = colp.p;
        A.grouped = grouped; A.sgroup = sgroup; A.ukey = ukey.p; A.ucval = ucval.p;
        A.group_min = group_min;
        A.gcnt = gcnt.p; A.gfill = gfill.p;
        A.fkey = fkey.p; A.farc = farc.p; A.frow = frow.p; A.fcval = fcval.p;
        A.chunk_e = chunk_e.p; A.fctr = fctr.p;
        A.s_ops = s_ops.p; A.s_pushes = s_pushes.p; A.s_l1 = s_l1.p; A.s_b1 = s_b1.p;
        A.s_last = s_last.p; A.s_conv = s_conv.p; A.s_amb = s_amb.p;
        A.nearl = NearList{{nearkey.p, nearkey.p + NEAR_CAP}, {nearcnt.p, nearcnt.p + 1}, NEAR_CAP};
        A.overflow = overflow.p;
        if (tail_on) {
            A.tail_list = tail_list.p;
            A.tail_c = tail_c.p;
            A.tail_f = tail_f;
            A.tail_t = tail_t;
            A.tail_state = tail_state.p;
        }
        return A;
    }

    void clear_marks(cudaStream_t st) {
        GD_CUDA(cudaMemsetAsync(cm0.p, 0, sizeof(uint32_t) * (size_t)slots * cmw, st));
        GD_CUDA(cudaMemsetAsync(cm1.p, 0, sizeof(uint32_t) * (size_t)slots * cmw, st));
    }

    void rounds(SArgs &A, cudaStream_t st) {
        GD_CUDA(cudaMemsetAsync(nearcnt.p, 0, 2 * sizeof(unsigned long long), st));
        void *kargs[] = {&A};
        GD_CUDA(cudaLaunchCooperativeKernel((const void *)k_signed_rounds, dim3(grid), dim3(SBT),
                                            kargs, smem, st));
    }

    void check_overflow(cudaStream_t st) {
        int32_t ovf = 0;
        GD_CUDA(cudaMemcpyAsync(&ovf, overflow.p, sizeof(ovf), cudaMemcpyDeviceToHost, st));
        GD_CUDA(cudaStreamSynchronize(st));
        if (ovf) {
            dirty = true;
            set_error("signed batch capacity %lld (frontier entries, arc chunks or candidates "
                      "per round) exceeded; raise frontier_cap",
                      (long long)fcap);
            throw Error{GD_ERR_CAPACITY};
        }
    }
};

// ---- cold waves -----------------------------------------------------------

SignedState *signed_batch_create(const gd_graph *W, const gd_batch_params &p, int slots) {
    SignedState *S = new SignedState();
    try {
        const int64_t n = W->n ? W->n : 1;
        int64_t fc = p.frontier_cap > 0 ? p.frontier_cap : (int64_t)slots * n;
        if (p.frontier_cap <= 0 && fc > (64LL << 20)) fc = 64LL << 20;
        S->alloc(W, 1, slots, fc, true);
        S->pack(W, 0);
        // operator: PPR  w = fl(1/d)(1-alpha), b = alpha e_s, theta = eps alpha d
        //           Katz w = alpha,            b = e_s,       theta = eps d
        S->op.wrule = p.problem == GD_P_KATZ ? GD_W_CONST : GD_W_RW;
        S->op.trule = GD_T_DEGREE;
        S->op.beta = p.problem == GD_P_KATZ ? p.alpha : 1.0 - p.alpha;
        S->op.tcoeff = p.problem == GD_P_KATZ ? p.eps : p.eps * p.alpha;
        if (p.method == GD_M_LOCAL_HB)
            S->set_hb(p.mu, p.L, p.max_sweeps);
        else
            S->set_ch(p.mu, p.L, p.max_sweeps);
        {
            const char *e = getenv("GDIFF_TAIL");
            const size_t per = (size_t)slots * (size_t)n;
            size_t fr = 0, tot = 0;  // lists cost at most a quarter of the free HBM
            GD_CUDA(cudaMemGetInfo(&fr, &tot));
            size_t cap = std::max<size_t>(4ULL << 30, fr / 4);
            if (const char *v = getenv("GDIFF_TAIL_MEM_GB")) cap = (size_t)atoll(v) << 30;  // (A/B)
            if (!(e && atoi(e) == 0) && per * 20 <= cap) {
                S->tail_list.alloc(3 * per);
                S->tail_c.alloc(per);
                S->tail_state.alloc(2);
                S->tail_on = true;
                S->tail_f = std::max<int64_t>(1 << 13, 128LL * slots);  // (~128 per slot)
                if (const char *v = getenv("GDIFF_TAIL_F")) S->tail_f = atoll(v);  // (A/B)
                if (const char *v = getenv("GDIFF_TAIL_T")) S->tail_t = atoi(v);
            }
        }
    } catch (...) {
        delete S;
        throw;
    }
    return S;
}

void signed_batch_destroy(SignedState *S) { delete S; }
int signed_batch_slots(const SignedState *S) { return S->slots; }

void signed_batch_run(SignedState *S, const gd_graph *W, const gd_batch_params &p,
                      const int64_t *d_seeds, int64_t n_seeds, const int32_t *perm,
                      const int32_t *inv, int64_t *sweeps, int64_t *ops, int64_t *pushes,
                      int64_t *support, int32_t *conv, int64_t *xoff, int64_t *xcnt,
                      int32_t *xnodes, double *xvals, int64_t xcap, unsigned long long *cursor,
                      std::vector<cudaEvent_t> &ev, double *ms, int64_t *launches,
                      cudaStream_t st, const RPool *rp, int32_t *amb,
                      unsigned long long *amb_cnt) {
    if (S->dirty) {  // a capacity abort left marks / residuals behind
        S->clear_marks(st);
        const size_t sn = (size_t)S->slots * (size_t)S->ld;
        GD_CUDA(cudaMemsetAsync(S->x.p, 0, sizeof(double) * sn, st));
        GD_CUDA(cudaMemsetAsync(S->r.p, 0, sizeof(double) * sn, st));
        GD_CUDA(cudaMemsetAsync(S->mstamp.p, 0xFF, sizeof(int32_t) * sn, st));
        GD_CUDA(cudaMemsetAsync(S->secmap.p, 0, sizeof(uint32_t) * (size_t)S->slots * S->smw, st));
        S->dirty = false;
    }
    GD_CUDA(cudaMemsetAsync(S->overflow.p, 0, sizeof(int32_t), st));
    const double bval = p.problem == GD_P_KATZ ? 1.0 : p.alpha;
    const int64_t waves = (n_seeds + S->slots - 1) / S->slots;
    while ((int64_t)ev.size() < 2 * waves) {
        cudaEvent_t e;
        GD_CUDA(cudaEventCreate(&e));
        ev.push_back(e);
    }
    SOut O{sweeps, ops, pushes, support, xoff, xcnt, conv, xnodes, xvals, xcap, inv,
           S->slot_base.p, amb, amb_cnt};
    int64_t nl = 0;
    for (int64_t w = 0; w < waves; ++w) {
        const int64_t base = w * S->slots;
        const int64_t m = n_seeds - base < S->slots ? n_seeds - base : S->slots;
        SArgs A = S->args(W, m);
        k_s_init<<<(int)((m + 255) / 256), 256, 0, st>>>(A, d_seeds + base, perm, bval);
        GD_LAUNCH_CHECK();
        if (S->tail_on)  // (-1: no tail handed over)
            GD_CUDA(cudaMemsetAsync(S->tail_state.p, 0xFF, 2 * sizeof(int64_t), st));
        GD_CUDA(cudaEventRecord(ev[2 * w], st));
        S->rounds(A, st);
        if (S->tail_on) {
            k_s_tail<<<(unsigned)m, SBT, 0, st>>>(A);
            nl += 1;
        }
        GD_CUDA(cudaEventRecord(ev[2 * w + 1], st));
        k_s_reserve<<<(int)((m + 255) / 256), 256, 0, st>>>(A, cursor, S->slot_base.p);
        k_s_extract<<<dim3(SCHUNKS, (unsigned)m), 256, 0, st>>>(A, O, base);
        if (rp) {  // sparse r out; zeroes the slots' r itself
            r_extract_wave(A.secmap, A.smw, A.r, A.ld, m, inv, base, rp->scratch, rp->cursor,
                           rp->off, rp->cnt, rp->nodes, rp->vals, rp->cap, st);
        } else {
            const int64_t rc = (S->smw + 2047) / 2048;  // ~2,048 map words per block
            k_s_reset<<<dim3((unsigned)(rc < SCHUNKS ? SCHUNKS : (rc > 4096 ? 4096 : rc)),
                             (unsigned)m), 256, 0, st>>>(A);
        }
        GD_LAUNCH_CHECK();
        nl += 5;
    }
    S->check_overflow(st);
    double tot = 0.0;
    for (int64_t w = 0; w < waves; ++w) {
        float f = 0.f;
        GD_CUDA(cudaEventElapsedTime(&f, ev[2 * w], ev[2 * w + 1]));
        tot += f;
    }
    *ms = tot;
    *launches = nl;
}

}  // namespace gd

using namespace gd;

// ---------------------------------------------------------------------------
// gd_pairs: K resident PPR pairs on an evolving graph.
// ---------------------------------------------------------------------------
namespace gd {
void fifo_pairs_run(const gd_graph *G, double *p, double *r, int64_t ld, int64_t k, double alpha,
                    double eps, int64_t max_sweeps, int32_t *queue, uint32_t *qmark, int64_t qw,
                    int64_t *sweeps, int64_t *ops, int64_t *pushes, int32_t *conv, cudaStream_t st);
}

struct gd_pairs {
    SignedState S;
    double alpha = 0.0, eps = 0.0;
    int64_t k = 0;
    int32_t method = GD_PAIRS_GD;      // repair: warm signed LocalGD or the reference FIFO push
    DBuf<int32_t> fq;                  // (push) per-pair FIFO queue
    DBuf<uint32_t> fqm;                // (push) per-pair queued marks
    int64_t fqw = 0;
    DBuf<int64_t> fst;                 // (push) sweeps, ops, pushes per pair
    DBuf<int32_t> fconv;
    std::vector<int32_t> deg;  // host copy of the current degrees (event bookkeeping)
    int64_t n_arcs = 0;
    DBuf<int32_t> gnodes, gdeg;
    DBuf<PairEvent> dev_events;
    bool all_converged = true;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    double last_ms = 0.0;
    ~gd_pairs() {
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
    }
};

static void pairs_repair(gd_pairs *P, const gd_graph *G, bool scan, int64_t max_sweeps,
                         const PairEvent *dev_ev, const std::vector<int64_t> &lvl_off,
                         int64_t *sweeps, int64_t *ops, int64_t *pushes, int32_t *conv) {
    SignedState &S = P->S;
    cudaStream_t st = 0;
    if (S.dirty) {
        S.clear_marks(st);
        S.dirty = false;
        scan = true;
    }
    S.max_sweeps = max_sweeps;
    S.pack(G, st);  // the graph changes per snapshot
    SArgs A = S.args(G, P->k);
    GD_CUDA(cudaMemsetAsync(S.overflow.p, 0, sizeof(int32_t), st));
    GD_CUDA(cudaMemsetAsync(S.candctr.p, 0, 2 * sizeof(unsigned long long), st));
    k_pair_stats_reset<<<(int)((P->k + 255) / 256), 256, 0, st>>>(A);
    for (size_t l = 0; l + 1 < lvl_off.size(); ++l) {  // dependency levels, in order
        const int64_t e0 = lvl_off[l], ne = lvl_off[l + 1] - e0;
        const int64_t threads = ne * P->k;
        k_pair_events<<<(int)((threads + 255) / 256), 256, 0, st>>>(A, dev_ev + e0, ne,
                                                                    1.0 - P->alpha);
    }
    const int64_t K = P->k;
    if (P->method == GD_PAIRS_PUSH) {  // the reference's repair: signed FIFO push per pair
        GD_LAUNCH_CHECK();
        const int64_t n = G->n ? G->n : 1;
        if (!P->fq.p) {
            P->fq.alloc((size_t)K * (size_t)(n + 2));
            P->fqw = n / 32 + 1;
            P->fqm.alloc((size_t)K * (size_t)P->fqw);
            GD_CUDA(cudaMemset(P->fqm.p, 0, sizeof(uint32_t) * (size_t)K * (size_t)P->fqw));
            P->fst.alloc(3 * (size_t)K);
            P->fconv.alloc((size_t)K);
        }
        GD_CUDA(cudaEventRecord(P->e0, st));
        fifo_pairs_run(G, S.x.p, S.r.p, S.ld, K, P->alpha, P->eps, max_sweeps, P->fq.p, P->fqm.p,
                       P->fqw, P->fst.p, P->fst.p + K, P->fst.p + 2 * K, P->fconv.p, st);
        GD_CUDA(cudaEventRecord(P->e1, st));
        GD_CUDA(cudaStreamSynchronize(st));
        float f = 0.f;
        GD_CUDA(cudaEventElapsedTime(&f, P->e0, P->e1));
        P->last_ms = f;
        std::vector<int64_t> h(3 * K);
        std::vector<int32_t> cv(K);
        GD_CUDA(cudaMemcpy(h.data(), P->fst.p, 8 * 3 * K, cudaMemcpyDeviceToHost));
        GD_CUDA(cudaMemcpy(cv.data(), P->fconv.p, 4 * K, cudaMemcpyDeviceToHost));
        P->all_converged = true;
        for (int64_t i = 0; i < K; ++i) {
            if (sweeps) sweeps[i] = h[i];
            if (ops) ops[i] = h[K + i];
            if (pushes) pushes[i] = h[2 * K + i];
            if (conv) conv[i] = cv[i];
            P->all_converged = P->all_converged && cv[i];
        }
        return;
    }
    if (scan) k_pair_scan<<<4 * n_sms(S.device), 256, 0, st>>>(A);
    GD_LAUNCH_CHECK();
    GD_CUDA(cudaEventRecord(P->e0, st));
    S.rounds(A, st);
    GD_CUDA(cudaEventRecord(P->e1, st));
    S.check_overflow(st);
    float f = 0.f;
    GD_CUDA(cudaEventElapsedTime(&f, P->e0, P->e1));
    P->last_ms = f;
    std::vector<int32_t> last(K), cv(K);
    std::vector<unsigned long long> o(K), pu(K);
    GD_CUDA(cudaMemcpy(last.data(), S.s_last.p, 4 * K, cudaMemcpyDeviceToHost));
    GD_CUDA(cudaMemcpy(cv.data(), S.s_conv.p, 4 * K, cudaMemcpyDeviceToHost));
    GD_CUDA(cudaMemcpy(o.data(), S.s_ops.p, 8 * K, cudaMemcpyDeviceToHost));
    GD_CUDA(cudaMemcpy(pu.data(), S.s_pushes.p, 8 * K, cudaMemcpyDeviceToHost));
    P->all_converged = true;
    for (int64_t i = 0; i < K; ++i) {
        if (sweeps) sweeps[i] = (int64_t)last[i] + 1;
        if (ops) ops[i] = (int64_t)o[i];
        if (pushes) pushes[i] = (int64_t)pu[i];
        if (conv) conv[i] = cv[i];
        P->all_converged = P->all_converged && cv[i];
    }
}

extern "C" {

int gd_pairs_create(const gd_graph *G, double alpha, double eps, const int64_t *sources,
                    int64_t k, int64_t frontier_cap, int64_t max_sweeps, gd_pairs **out,
                    int64_t *sweeps, int64_t *total_ops, int64_t *pushes, int32_t *converged) {
    return gd_pairs_create_ex(G, alpha, eps, sources, k, frontier_cap, max_sweeps, GD_PAIRS_GD, out,
                              sweeps, total_ops, pushes, converged);
}

int gd_pairs_create_ex(const gd_graph *G, double alpha, double eps, const int64_t *sources,
                       int64_t k, int64_t frontier_cap, int64_t max_sweeps, int32_t method,
                       gd_pairs **out, int64_t *sweeps, int64_t *total_ops, int64_t *pushes,
                       int32_t *converged) {
    return guarded([&] {
        GD_CHECK_ARG(method == GD_PAIRS_GD || method == GD_PAIRS_PUSH, "unknown pair repair method");
        GD_CHECK_ARG(G && sources && out, "null pointer");
        GD_CHECK_ARG(k >= 1 && k <= 4096, "pair count must be in [1, 4096]");
        GD_CHECK_ARG(alpha > 0.0 && alpha < 1.0, "alpha must be in (0, 1)");
        GD_CHECK_ARG(eps > 0.0, "eps must be positive");
        GD_CUDA(cudaSetDevice(G->device));
        gd_pairs *P = new gd_pairs();
        try {
            P->alpha = alpha;
            P->eps = eps;
            P->k = k;
            P->method = method;
            P->deg.resize(G->n);
            P->n_arcs = G->n_arcs;
            if (G->n)
                GD_CUDA(cudaMemcpy(P->deg.data(), G->deg.p, 4 * G->n, cudaMemcpyDeviceToHost));
            for (int64_t i = 0; i < k; ++i) {
                GD_CHECK_ARG(sources[i] >= 0 && sources[i] < G->n, "source out of range");
                GD_CHECK_ARG(P->deg[sources[i]] >= 1, "source must have at least one neighbor");
            }
            const int64_t n = G->n ? G->n : 1;
            int64_t fc = frontier_cap > 0 ? frontier_cap : k * n;
            if (frontier_cap <= 0 && fc > (64LL << 20)) fc = 64LL << 20;
            P->S.alloc(G, 0, (int)k, fc, false);
            P->S.op.wrule = GD_W_RW;
            P->S.op.trule = GD_T_DEGREE;
            P->S.op.beta = 1.0 - alpha;
            P->S.op.tcoeff = eps;  // repair thresholds eps * d_u (src/dynamic.py:139-141)
            for (int64_t i = 0; i < k; ++i)
                GD_CUDA(cudaMemcpy(P->S.r.p + i * P->S.ld + sources[i], &alpha, sizeof(double),
                                   cudaMemcpyHostToDevice));
            GD_CUDA(cudaEventCreate(&P->e0));
            GD_CUDA(cudaEventCreate(&P->e1));
            pairs_repair(P, G, true, max_sweeps > 0 ? max_sweeps : 1000000, nullptr,
                         std::vector<int64_t>(), sweeps, total_ops, pushes, converged);
        } catch (...) {
            delete P;
            throw;
        }
        *out = P;
    });
}

int gd_pairs_destroy(gd_pairs *P) {
    delete P;
    return GD_OK;
}

int gd_pairs_update(gd_pairs *P, const gd_graph *G_new, const int32_t *kinds, const int64_t *us,
                    const int64_t *vs, int64_t n_events, int64_t max_sweeps, int64_t *sweeps,
                    int64_t *total_ops, int64_t *pushes, int32_t *converged) {
    return guarded([&] {
        GD_CHECK_ARG(P && G_new && (n_events == 0 || (kinds && us && vs)), "null pointer");
        GD_CHECK_ARG(G_new->n == (int64_t)P->deg.size(), "node count changed");
        GD_CUDA(cudaSetDevice(G_new->device));
        // degrees evolve event by event (event_adjust_many semantics); only the
        // endpoints change, so they are tracked in a map and committed at the end
        std::vector<PairEvent> ev(n_events);
        std::unordered_map<int32_t, int32_t> nd;
        auto cur = [&](int64_t x) {
            auto it = nd.find((int32_t)x);
            return it == nd.end() ? P->deg[x] : it->second;
        };
        int64_t net = 0;
        for (int64_t i = 0; i < n_events; ++i) {
            const int64_t u = us[i], v = vs[i];
            GD_CHECK_ARG(u >= 0 && v >= 0 && u < G_new->n && v < G_new->n && u != v,
                         "bad event endpoints");
            const int32_t step = kinds[i] ? 1 : -1;
            const int32_t du = cur(u), dv = cur(v);
            GD_CHECK_ARG(du + step >= 0 && dv + step >= 0, "delete would make a degree negative");
            ev[i] = PairEvent{(int32_t)u, (int32_t)v, du, dv, step};
            nd[(int32_t)u] = du + step;
            nd[(int32_t)v] = dv + step;
            net += 2 * step;
        }
        // G_new must be the old graph with these events: arc count and the
        // endpoints' degrees (gathered on the device)
        GD_CHECK_ARG(G_new->n_arcs == P->n_arcs + net,
                     "G_new is not the old graph with these events applied");
        if (!nd.empty()) {
            std::vector<int32_t> nodes, want;
            for (auto &kv : nd) {
                nodes.push_back(kv.first);
                want.push_back(kv.second);
            }
            const int64_t c = (int64_t)nodes.size();
            P->gnodes.ensure(c);
            P->gdeg.ensure(c);
            GD_CUDA(cudaMemcpy(P->gnodes.p, nodes.data(), 4 * c, cudaMemcpyHostToDevice));
            k_gather_deg<<<(int)((c + 255) / 256), 256>>>(G_new->view(), P->gnodes.p, c,
                                                          P->gdeg.p);
            GD_LAUNCH_CHECK();
            std::vector<int32_t> got(c);
            GD_CUDA(cudaMemcpy(got.data(), P->gdeg.p, 4 * c, cudaMemcpyDeviceToHost));
            GD_CHECK_ARG(got == want, "G_new is not the old graph with these events applied");
        }
        // dependency levels: an event waits for the latest earlier event that
        // shares one of its nodes (a stable sort by level keeps event order
        // inside a level; per-node order is preserved exactly)
        std::vector<int32_t> level(n_events);
        std::unordered_map<int32_t, int32_t> last;
        int32_t nlev = 0;
        for (int64_t i = 0; i < n_events; ++i) {
            int32_t l = 0;
            auto a = last.find(ev[i].u), b = last.find(ev[i].v);
            if (a != last.end()) l = std::max(l, a->second + 1);
            if (b != last.end()) l = std::max(l, b->second + 1);
            level[i] = l;
            last[ev[i].u] = l;
            last[ev[i].v] = l;
            nlev = std::max(nlev, l + 1);
        }
        std::vector<int64_t> lvl_off(nlev + 1, 0);
        for (int64_t i = 0; i < n_events; ++i) lvl_off[level[i] + 1]++;
        for (int32_t l = 0; l < nlev; ++l) lvl_off[l + 1] += lvl_off[l];
        std::vector<PairEvent> sorted(n_events);
        {
            std::vector<int64_t> fill(lvl_off.begin(), lvl_off.end() - 1);
            for (int64_t i = 0; i < n_events; ++i) sorted[fill[level[i]]++] = ev[i];
        }
        P->dev_events.ensure(n_events ? n_events : 1);
        if (n_events)
            GD_CUDA(cudaMemcpy(P->dev_events.p, sorted.data(), sizeof(PairEvent) * n_events,
                               cudaMemcpyHostToDevice));
        pairs_repair(P, G_new, !P->all_converged, max_sweeps > 0 ? max_sweeps : 1000000,
                     P->dev_events.p, lvl_off, sweeps, total_ops, pushes, converged);
        for (auto &kv : nd) P->deg[kv.first] = kv.second;
        P->n_arcs = G_new->n_arcs;
    });
}

// Dense copies of pair i (p, r: n doubles each; either may be NULL).
int gd_pairs_get(const gd_pairs *P, int64_t i, double *p, double *r) {
    return guarded([&] {
        GD_CHECK_ARG(P, "null pointer");
        GD_CHECK_ARG(i >= 0 && i < P->k, "pair index out of range");
        const size_t n = P->deg.size();
        if (p) GD_CUDA(cudaMemcpy(p, P->S.x.p + i * P->S.ld, 8 * n, cudaMemcpyDeviceToHost));
        if (r) GD_CUDA(cudaMemcpy(r, P->S.r.p + i * P->S.ld, 8 * n, cudaMemcpyDeviceToHost));
    });
}

// Device view of the pool: pair i's p at p[i * ld], r at r[i * ld].
int gd_pairs_device(const gd_pairs *P, double **p, double **r, int64_t *ld) {
    if (!P || !p || !r || !ld) return GD_ERR_ARG;
    *p = P->S.x.p;
    *r = P->S.r.p;
    *ld = P->S.ld;
    return GD_OK;
}

int gd_pairs_last_kernel_ms(const gd_pairs *P, double *ms) {
    if (!P || !ms) return GD_ERR_ARG;
    *ms = P->last_ms;
    return GD_OK;
}

}  // extern "C"
