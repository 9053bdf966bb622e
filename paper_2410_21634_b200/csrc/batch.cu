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
//    (slot-major).  Between waves a slot is reset by zeroing exactly the
//    32 B sectors of r it wrote (sector bit map set on first touch, cleared
//    warp-cooperatively in coalesced 1 KB runs) and x over its pushed-node
//    list -- never by a memset of the whole slot.
//  * The graph is renumbered once by descending degree with sorted rows:
//    hubs, which receive most residual updates, form a contiguous block, so
//    a warp's 32 atomics land in few sectors and stay L2 resident.
//  * One persistent cooperative kernel runs all sweeps of a wave; sweeps of
//    all slots advance together ("rounds"), two grid barriers per round:
//      phase A (thread per frontier entry): vals = r[u]; x[u] += vals;
//              r[u] = -0.0 (pushed; +0.0 means "never touched");
//              c_u = fl(vals * fl(fl(1/d_u)*(1-alpha))) staged per entry.
//      phase B (arc-balanced: every warp owns an equal slice of the round's
//              concatenated arc space, 4 chunks of 32 arcs in flight per
//              lane): r[v] += c_u with a returning fp64 atomic.  The old
//              value decides, with no extra memory traffic, (1) first touch
//              (old == +0.0, counted) and (2) frontier entry: residuals only
//              grow inside a round, so exactly one arc observes
//              old < theta_v <= old + c and appends (slot, v) to S_{t+1}.
//  * Frontier appends reserve (entries, arcs) with ONE packed 64-bit atomic
//    per warp, so entry order and arc-offset order agree and the next
//    round's arc space is a prefix sum for free.
//  * Thresholds come from the L2-resident int32 degree array
//    (theta_v = fl(eps*alpha*d_v)), not a per-node double.
#include <cooperative_groups.h>

#include <cub/cub.cuh>
#include <atomic>
#include <chrono>
#include <mutex>
#include <string>
#include <thread>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace gd {  // fifo_batch.cu
// optional sparse r output of a solve (want_r); null pointer = not wanted
struct RPool {
    int64_t *off, *cnt;          // per seed
    int32_t *nodes;
    double *vals;
    int64_t cap;
    unsigned long long *cursor;  // pairs used
    unsigned long long *scratch; // per (slot, chunk) counts
};
void r_extract_wave(uint32_t *secmap, int64_t smw, double *r, int64_t ld, int64_t m,
                    const int32_t *inv, int64_t seed_base, unsigned long long *cnt_scratch,
                    unsigned long long *cursor, int64_t *r_off, int64_t *r_cnt,
                    int32_t *r_nodes, double *r_vals, int64_t rcap, cudaStream_t st);
int r_extract_chunks(int64_t smw);
struct FifoBatchState;
FifoBatchState *fifo_batch_create(const gd_graph *G, int slots);
void fifo_batch_destroy(FifoBatchState *F);
struct SignedState;
SignedState *signed_batch_create(const gd_graph *W, const gd_batch_params &p, int slots);
void signed_batch_destroy(SignedState *S);
void signed_batch_run(SignedState *S, const gd_graph *W, const gd_batch_params &p,
                      const int64_t *d_seeds, int64_t n_seeds, const int32_t *perm,
                      const int32_t *inv, int64_t *sweeps, int64_t *ops, int64_t *pushes,
                      int64_t *support, int32_t *conv, int64_t *xoff, int64_t *xcnt,
                      int32_t *xnodes, double *xvals, int64_t xcap, unsigned long long *cursor,
                      std::vector<cudaEvent_t> &ev, double *ms, int64_t *launches,
                      cudaStream_t st, const RPool *rp, int32_t *amb,
                      unsigned long long *amb_cnt);
int fifo_batch_slots(const FifoBatchState *F);
struct SorWinState;  // sor_win.cu: LocalSOR/GS seeds in exact windows, one CTA per seed
SorWinState *sorwin_create(const gd_graph *G, int max_ctas);
void sorwin_destroy(SorWinState *W);
void sorwin_run(SorWinState *W, const gd_graph *G, const gd_batch_params &p,
                const int64_t *d_seeds, int64_t n_seeds, int64_t *sweeps, int64_t *ops,
                int64_t *pushes, int32_t *conv, int64_t *xoff, int64_t *xcnt, int32_t *xnodes,
                double *xvals, int64_t xcap, unsigned long long *cursor, cudaStream_t st);
struct CtaState;  // batch_cta.cu: one CTA per seed (small graphs)
CtaState *cta_batch_create(const gd_graph *W, int max_slots);
void cta_batch_destroy(CtaState *S);
int cta_batch_slots(const CtaState *S);
bool cta_batch_smem(const CtaState *S);
int64_t cta_slot_bytes(int64_t n, int64_t n_arcs);
void cta_batch_run(CtaState *S, const gd_graph *W, const int2 *colp, double alpha, double eps,
                   int64_t max_sweeps, const int64_t *d_seeds, int64_t n_seeds,
                   const int32_t *perm, const int32_t *inv, int64_t *sweeps, int64_t *ops,
                   int64_t *pushes, int64_t *support, int32_t *conv, int64_t *xoff,
                   int64_t *xcnt, int32_t *xnodes, double *xvals, int64_t xcap,
                   unsigned long long *cursor, int32_t *amb, unsigned long long *amb_cnt,
                   cudaStream_t st, int64_t *lg_f, int64_t *lg_ops, double *lg_g,
                   int64_t lg_cap);
bool fifo_batch_smem(const FifoBatchState *F);
void fifo_batch_run(FifoBatchState *F, const gd_graph *G, const gd_batch_params &p,
                    const int64_t *d_seeds, int64_t n_seeds, int64_t *sweeps, int64_t *ops,
                    int64_t *pushes, int32_t *conv, int64_t *xoff, int64_t *xcnt, int32_t *xnodes,
                    double *xvals, int64_t xcap, unsigned long long *cursor, cudaStream_t st,
                    const RPool *rp);
}  // namespace gd

namespace gd {
namespace {

constexpr int BT = 512;   // threads per block of the round kernel
#ifndef GD_KR_MINB
#define GD_KR_MINB 2  // resident round-kernel blocks per SM (register budget)
#endif
#ifndef GD_KR_MINB_HK
#define GD_KR_MINB_HK 1  // (heat kernel: one block per SM, registers for the pull's HKC sums)
#endif
#ifndef GD_HKC
#define GD_HKC 14
#endif
constexpr int UNROLL = 4; // 32-arc chunks in flight per warp in phase B
constexpr int SUPER = 16; // UNROLL-chunk groups per block super-chunk in phase B
constexpr int CNT_SHIFT = 36;
constexpr unsigned long long ARC_MASK = (1ULL << CNT_SHIFT) - 1ULL;
constexpr unsigned FULL = 0xffffffffu;
constexpr int CHUNKS = 32;  // blocks per slot in the extract / reset kernels
constexpr int64_t CTA_MAX_N = 1LL << 18;  // one-CTA-per-seed mode up to this many nodes

struct RoundArgs {
    DevGraph g;
    double beta;    // 1 - alpha
    double tcoeff;  // eps * alpha
    int64_t n;
    int64_t ld;     // slot stride (n rounded up to 4: 32 B aligned slots)
    int64_t max_sweeps;
    int64_t fcap;
    int64_t m;      // slots in use this wave
    double *x, *r;
    double *r2;              // heat kernel: second residual layer (stages alternate)
    uint32_t *secmap2;       // heat kernel: sector map of r2
    const double *stage_w;   // heat kernel: tau/(k+1) per stage (device)
    int64_t n_stages;        // heat kernel: N (stage N is absorbing)
    int32_t *pushed;
    int32_t *seed;  // per slot: seed in working ids
    unsigned long long *touched, *pushed_cnt;
    int64_t *ukey;        // next frontier as appended: (slot << 32 | node), any order
    int64_t *uarc;        // its first arc offsets in append order (ungrouped mode)
    int64_t group_min;    // (rounds with fewer frontier arcs stay ungrouped)
    int grouped;          // 1: phase A regroups the frontier by slot group and phase B
                          //    walks it with a grid-wide window (slot vectors > L2);
                          // 0: append order, contiguous per-block ranges (L2 holds
                          //    every slot; spreading blocks over slots avoids
                          //    same-word atomic contention)
    int64_t *skey, *sarc; // current frontier grouped by slot: key, first arc offset
    unsigned long long *scnt[2];  // per slot, per round parity: packed (entries << 36 | arcs)
    unsigned long long *sfill;    // per slot group: fill of the grouped frontier (phase A)
    int64_t sgroup;               // slots per group: the frontier copy is grouped by
                                  // k / sgroup (L2-sized groups; slots inside a group
                                  // interleave, spreading same-word atomics)
    unsigned long long *cctr;     // phase-B chunk claim counter
    int64_t *frow;
    double *fcval;
    const int2 *colp;     // per arc (neighbour, its degree): one 8 B load gives theta
    int32_t *chunk_e;     // entry holding arc 32c of the round (phase A -> B)
    int64_t ccap;         // chunk_e capacity
    unsigned long long *fctr;  // [2] packed (entries << 36 | arcs)
    unsigned long long *s_ops, *s_pushes, *s_negz, *s_pvol;
    int32_t *s_last, *s_conv;
    int32_t *s_amb;       // per slot: a final residual within AMB_REL of theta (common.cuh)
    NearList nearl;       // landings just below theta, re-checked after the round
    int32_t *overflow;
    const int32_t *perm;  // caller id -> working id (nullable)
    unsigned long long *cursor;  // output pool allocation
    int64_t *slot_base;
    uint32_t *secmap;   // per slot: bit per 32 B sector of r ever written (reset map)
    int64_t smw;        // words per slot in secmap
    int64_t *lg_f, *lg_ops;  // per-seed sweep logs (log_sweeps > 0; else null):
    double *lg_g;            //   |S_t|, vol(S_t), sum |r_u| -- row (seed_base + k)
    int64_t lg_cap, seed_base;
    int64_t *rlog;      // per round: F, P, globaltimer ns (3 entries), debug
    int64_t rlog_cap;   // rounds recorded
    // streaming form (k_rounds<false, true>): slots refilled inside the kernel
    const int64_t *seeds;         // the solve's seeds (caller ids)
    int64_t n_seeds;
    double alpha;
    unsigned long long *seed_ctr; // next seed index to start
    unsigned long long *done_ctr; // seeds finished since the solve began
    int64_t seg_done;             // leave at a round start once done_ctr >= seg_done
    int32_t *t_state;             // round to resume from (kept across launches)
    int32_t *s_idx;               // per slot: seed index, -1 = idle
    int32_t *s_t0;                // per slot: round of the seed's first push
    unsigned long long *sn[2];    // per slot: entries in the frontier, per round parity
    int64_t *drain_cnt;           // per slot: pushed count of the finished seed
    int64_t reset_units;          // sector-map reset work units per finished slot
    int32_t dbg;                  // (experiments) 1: skip x extract, 2: skip r reset
    int64_t cohort;               // refill only once this many slots are free (they
                                  // then start together: see k_rounds)
    // CTA-local tail (k_tail): once a round past the wave's peak has <=
    // tail_p arcs and <= tail_f entries, k_rounds leaves (t, F) in tail_state
    // and k_tail finishes slot k in block k; frontier lists in tail_list
    // (2 x n per slot), c_u in tail_c (n per slot)
    int64_t tail_p, tail_f, tail_cap;
    int32_t *tail_list;
    // heat kernel, dense stages (hk_pull_*): c_u per (node, slot), node-major
    // (n x m), and the prefix of nodes with >= HEAVY_DEG arcs (degree-sorted ids)
    double *cn;
    int tma;               //   stage the pull's arc records with bulk async copies
    int64_t heavy, mid;    //   mid: nodes with >= MEDIUM_DEG arcs (heavy included)
    const int64_t *hitem;  // heavy-row segments: (node << 20) | segment
    int64_t hitems;
    double *hacc;          // heavy (node, slot) partial sums, node-major
    double *tail_c;
    int64_t *tail_state;
};

__device__ __forceinline__ int64_t globaltimer() {
    int64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ double theta_deg(double tc, int32_t d) {
    return d > 0 ? __dmul_rn(tc, (double)d) : __longlong_as_double(0x7ff0000000000000LL);
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Append `item` to the per-slot list k (warp-aggregated by slot).
__device__ __forceinline__ void slot_append(bool flag, int32_t k, int32_t item, int64_t ld,
                                            int32_t *list, unsigned long long *cnt) {
    unsigned am = __ballot_sync(FULL, flag);
    if (!flag) return;
    unsigned peers = __match_any_sync(am, k);
    int leader = __ffs(peers) - 1;
    int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(cnt + k, (unsigned long long)__popc(peers));
    base = __shfl_sync(peers, base, leader);
    list[(int64_t)k * ld + (int64_t)base + __popc(peers & lanemask_lt())] = item;
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
            A.ukey[idx] = ((int64_t)k << 32) | (uint32_t)v;
            A.uarc[idx] = (int64_t)(old & ARC_MASK) + (int64_t)(incl - (unsigned long long)d);
        } else {
            A.overflow[0] = 1;
        }
    }
    if (A.grouped) {  // per slot group (entries, arcs): one atomic per group present
        const int32_t g = flag ? k / (int32_t)A.sgroup : -1;
        const unsigned peers = __match_any_sync(FULL, g);
        unsigned long long pv = flag ? (1ULL << CNT_SHIFT) + (unsigned long long)d : 0ULL;
        unsigned long long sum = 0;
        for (int i = 0; i < 32; ++i) {
            const unsigned long long vi = __shfl_sync(FULL, pv, i);
            if ((peers >> i) & 1u) sum += vi;
        }
        if (flag && lane == __ffs(peers) - 1) atomicAdd(A.scnt[nxt] + g, sum);
    }
}

// Block-level staging (shared memory): per-slot counters of the block and a
// buffer of the block's next-frontier entries.  Flushed once per phase, so
// global atomics on the shared frontier counter drop from one per warp with
// a crossing to one per block per round.
constexpr int STAGE_CAP = 3072;  // staged frontier entries per block per round

struct Stage {
    unsigned long long *ops, *pvol;      // [S]
    unsigned long long *scnt;            // [S] packed entries/arcs staged for the next round
    unsigned long long *sbase;           // [S] slot offsets of the grouped frontier
    unsigned *push, *touch, *negz;       // [S]
    int32_t *fk, *fv, *fd;               // [STAGE_CAP]
    unsigned *fcnt;                      // [1]
    unsigned long long *next;            // [1] phase-B chunk claim counter
    unsigned long long *scan;            // [BT/32 + 2]
    unsigned *nf;                        // [S] next-frontier entries per slot (streaming)
    int32_t *fin;                        // [S] slots whose seed finished (streaming)
    unsigned *nfin;                      // [2] finished, idle slots
    int32_t *idle;                       // [S] idle slots (streaming)
    double *gsum;                        // [S] pushed |r| of the round (sweep logs)
};

__host__ __device__ inline size_t stage_bytes(int S) {
    return (size_t)S * (8 + 8 + 8 + 8 + 4 + 4 + 4 + 4 + 4 + 4 + 8) + (size_t)STAGE_CAP * 12 + 16 +
           8 * (BT / 32 + 3) + 16 + 64;
}

__device__ Stage stage_carve(void *base, int S) {
    char *p = (char *)base;
    Stage st;
    st.gsum = (double *)p; p += 8 * S;
    st.ops = (unsigned long long *)p; p += 8 * S;
    st.pvol = (unsigned long long *)p; p += 8 * S;
    st.scnt = (unsigned long long *)p; p += 8 * S;
    st.sbase = (unsigned long long *)p; p += 8 * S;
    st.scan = (unsigned long long *)p; p += 8 * (BT / 32 + 2);
    st.next = (unsigned long long *)p; p += 8;
    st.push = (unsigned *)p; p += 4 * S;
    st.touch = (unsigned *)p; p += 4 * S;
    st.negz = (unsigned *)p; p += 4 * S;
    st.fcnt = (unsigned *)p; p += 16;
    st.fk = (int32_t *)p; p += 4 * STAGE_CAP;
    st.fv = (int32_t *)p; p += 4 * STAGE_CAP;
    st.fd = (int32_t *)p; p += 4 * STAGE_CAP;
    st.nf = (unsigned *)p; p += 4 * S;
    st.fin = (int32_t *)p; p += 4 * S;
    st.idle = (int32_t *)p; p += 4 * S;
    st.nfin = (unsigned *)p;
    return st;
}

// Warp-aggregated add of `val` over flagged lanes into counter array cnt[k]
// (shared-memory counters: cheap, no global contention).
template <class T>
__device__ __forceinline__ void block_count(bool flag, int32_t k, unsigned val, T *cnt) {
    unsigned am = __ballot_sync(FULL, flag);
    if (!flag) return;
    unsigned peers = __match_any_sync(am, k);
    unsigned sum = __reduce_add_sync(peers, val);
    if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(cnt + k, (T)sum);
}

// Stage (k, v, d) in the block buffer; lanes beyond its capacity append
// straight to the global frontier.
__device__ __forceinline__ void stage_append(bool flag, int32_t k, int32_t v, int32_t d,
                                             const Stage &S, const RoundArgs &A, int nxt) {
    unsigned am = __ballot_sync(FULL, flag);
    if (am == 0) return;
    if (A.sn[0]) block_count(flag, k, 1u, S.nf);  // streaming: entries per slot
    const int lane = threadIdx.x & 31;
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(S.fcnt, (unsigned)__popc(am));
    base = __shfl_sync(FULL, base, 0);
    const unsigned my = base + __popc(am & lanemask_lt());
    const bool spill = flag && my >= (unsigned)STAGE_CAP;
    const bool staged = flag && !spill;
    if (staged) {
        S.fk[my] = k;
        S.fv[my] = v;
        S.fd[my] = d;
    }
    // grouped mode: per slot group (entries, arcs) of the staged lanes, one
    // shared atomic per group present in the warp (usually one)
    if (A.grouped) {
        const unsigned sm = __ballot_sync(FULL, staged);
        if (sm) {
            const int32_t g = k / (int32_t)A.sgroup;
            const int32_t g0 = __shfl_sync(FULL, g, __ffs(sm) - 1);
            if (__all_sync(FULL, !staged || g == g0)) {
                const unsigned dsum = __reduce_add_sync(FULL, staged ? (unsigned)d : 0u);
                if (lane == 0)
                    atomicAdd(S.scnt + g0, ((unsigned long long)__popc(sm) << CNT_SHIFT) + dsum);
            } else if (staged) {
                const unsigned peers = __match_any_sync(sm, g);
                const unsigned dsum = __reduce_add_sync(peers, (unsigned)d);
                if (lane == __ffs(peers) - 1)
                    atomicAdd(S.scnt + g, ((unsigned long long)__popc(peers) << CNT_SHIFT) + dsum);
            }
        }
    }
    frontier_append(spill, k, v, d, A, nxt);
}

// Block-wide: move the staged entries to the global next frontier with ONE
// reservation (entries and the arc total), and add the block's per-slot
// entry / arc counts (the next round groups the frontier by slot).
__device__ void stage_flush(const Stage &S, const RoundArgs &A, int nxt) {
    __syncthreads();
    const unsigned cnt = min(*S.fcnt, (unsigned)STAGE_CAP);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const unsigned per = (cnt + BT - 1) / BT;
    const unsigned lo = min(cnt, tid * per), hi = min(cnt, lo + per);
    unsigned long long mine = 0;
    for (unsigned i = lo; i < hi; i++) mine += (unsigned long long)S.fd[i];
    unsigned long long incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) S.scan[w] = incl;
    __syncthreads();
    if (tid == 0) {
        unsigned long long run = 0;
        for (int i = 0; i < BT / 32; i++) {
            unsigned long long x = S.scan[i];
            S.scan[i] = run;
            run += x;
        }
        unsigned long long old = 0;
        if (cnt) old = atomicAdd(A.fctr + nxt, ((unsigned long long)cnt << CNT_SHIFT) + run);
        S.scan[BT / 32] = old;
    }
    __syncthreads();
    const unsigned long long old = S.scan[BT / 32];
    const int64_t ebase = (int64_t)(old >> CNT_SHIFT);
    int64_t arc = (int64_t)(old & ARC_MASK) + (int64_t)(S.scan[w] + incl - mine);
    for (unsigned i = lo; i < hi; i++) {
        const int64_t idx = ebase + i;
        if (idx < A.fcap) {
            A.ukey[idx] = ((int64_t)S.fk[i] << 32) | (uint32_t)S.fv[i];
            A.uarc[idx] = arc;  // (read in the ungrouped mode only)
        } else {
            A.overflow[0] = 1;
        }
        arc += S.fd[i];
    }
    if (A.grouped)
        for (int64_t k = tid; k < A.m; k += BT) {
            const unsigned long long v = S.scnt[k];
            if (v) {
                atomicAdd(A.scnt[nxt] + k, v);
                S.scnt[k] = 0;
            }
        }
    if (A.sn[0])
        for (int64_t k = tid; k < A.m; k += BT) {
            const unsigned v = S.nf[k];
            if (v) {
                atomicAdd(A.sn[nxt] + k, (unsigned long long)v);
                S.nf[k] = 0;
            }
        }
    __syncthreads();
    if (tid == 0) *S.fcnt = 0;
}

// S.sbase[g] = sum over slot groups j < g of A.scnt[cur][j] (packed: entries
// and arcs together), computed by every block for itself.
__device__ void slot_bases(const Stage &S, const RoundArgs &A, int cur) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t per = (A.m + BT - 1) / BT;
    const int64_t lo = min(A.m, tid * per), hi = min(A.m, lo + per);
    unsigned long long mine = 0;
    for (int64_t k = lo; k < hi; k++) mine += A.scnt[cur][k];
    unsigned long long incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) S.scan[w] = incl;
    __syncthreads();
    if (tid == 0) {
        unsigned long long run = 0;
        for (int i = 0; i < BT / 32; i++) {
            unsigned long long x = S.scan[i];
            S.scan[i] = run;
            run += x;
        }
    }
    __syncthreads();
    unsigned long long b = S.scan[w] + incl - mine;
    for (int64_t k = lo; k < hi; k++) {
        S.sbase[k] = b;
        b += A.scnt[cur][k];
    }
    __syncthreads();
}

template <class T>
__device__ void counters_flush(T *sc, unsigned long long *g, int64_t m) {
    for (int64_t k = threadIdx.x; k < m; k += BT) {
        const T v = sc[k];
        if (v) {
            atomicAdd(g + k, (unsigned long long)v);
            sc[k] = 0;
        }
    }
}

struct OutArgs {
    int64_t *sweeps, *ops, *pushes, *support, *xoff, *xcnt;
    int32_t *conv;
    int32_t *xnodes;
    double *xvals;
    int64_t xcap;
    const int32_t *inv;  // working id -> caller id (nullable)
    double xscale;       // x out = fl(xscale * x) (heat kernel: e^-tau; else 1)
    int hk;
    int32_t *amb;                 // per seed: near-threshold flag
    unsigned long long *amb_cnt;  // flagged seeds
};

//
// STREAM = true (LocalGD without sparse r): the slots are refilled inside the
// kernel instead of running in synchronous waves.  A slot whose seed had no
// frontier entries in a round (sn == 0) finished in the round before; in
// that round every block lists it (same data, read after the barrier), and
//   phase A: one thread reserves the seed's output segment and writes its
//            counters; warps zero the slot's touched r sectors (sector map);
//   phase B: warps copy x over its pushed list out (and zero it); one thread
//            writes the near-threshold flag, takes the next seed from a
//            counter (r[s] = alpha, counters reset) and appends it to the
//            next frontier.
// So a slot idles for one round between seeds, no round waits for the
// slowest seed of a wave, and there are no extract / reset launches.  The
// kernel leaves at a round start once `seg_done` seeds have finished (the
// host copies their x out while the next launch runs) and resumes there.
// ---------------------------------------------------------------------------
// CTA-local tail of a wave (k_tail).  The last rounds of a wave carry a few
// hundred arcs but each costs the round kernel two grid barriers and a dozen
// dependent global accesses (~10-15 us; ~8 % of a products wave).  Once a
// round past the wave's peak is small (<= tail_p arcs, <= tail_f entries;
// every block sees the same F and P), k_rounds stops and leaves (t, F) in
// tail_state; k_tail then runs one block per slot: block k takes slot k's
// entries of round t and runs the remaining sweeps of that seed alone with
// block barriers only -- the same push, threshold-crossing, first-touch and
// near-threshold rules as k_rounds, the whole frontier pushed before any
// scatter, arcs block-balanced (entries in segments of TAIL_SEG, degrees
// block-scanned, UNROLL_T arcs in flight per thread, entry found by binary
// search in shared memory), the next frontier in the slot's own list.  Sweeps
// stay numbered as rounds, so sweeps, ops and frontier sets are unchanged.  A
// separate kernel rather than a branch of k_rounds: inlined there it cost the
// round loop ~3 % through register allocation.
constexpr int TAIL_SEG = 1024;
constexpr int TAIL_NEAR = 256;
constexpr int UNROLL_T = 4;

__global__ void __launch_bounds__(BT, 2) k_tail(const __grid_constant__ RoundArgs A) {
    using Scan = cub::BlockScan<int, BT>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ double tc[TAIL_SEG];
    __shared__ int64_t trow[TAIL_SEG];
    __shared__ int32_t toff[TAIL_SEG + 1], tnear[TAIL_NEAR];
    __shared__ unsigned long long c_ops[1], c_pvol[1];
    __shared__ unsigned c_push[1], c_touch[1], c_negz[1];
    __shared__ double c_g;
    __shared__ int s_cur, s_nxt, s_nn, s_amb, s_ovf;
    const int64_t F = A.tail_state[1];
    if (F < 0) return;  // the wave ended in the round kernel
    int32_t t = (int32_t)A.tail_state[0];
    const int tid = threadIdx.x, lane = tid & 31;
    const int32_t k = (int32_t)blockIdx.x;
    const int64_t n = A.n;
    const int64_t C = A.tail_cap;  // list capacity per slot (n, or less on huge graphs)
    int32_t *const l0 = A.tail_list + (int64_t)k * 2 * C, *const l1 = l0 + C;
    double *const cval = A.tail_c + (int64_t)k * C;  // c_u of the sweep's entries
    if (tid == 0) {
        s_cur = s_nn = s_amb = s_ovf = 0;
        c_ops[0] = c_pvol[0] = 0;
        c_push[0] = c_touch[0] = c_negz[0] = 0;
        c_g = 0.0;
    }
    __syncthreads();
    for (int64_t e0 = 0; e0 < F; e0 += BT) {  // this slot's entries of round t
        const int64_t e = e0 + tid;
        const int64_t key = e < F ? A.ukey[e] : -1;
        const bool mine = e < F && (int32_t)(key >> 32) == k;
        const unsigned am = __ballot_sync(FULL, mine);
        int base = 0;
        if (am && lane == __ffs(am) - 1) base = atomicAdd(&s_cur, __popc(am));
        base = __shfl_sync(FULL, base, __ffs(am ? am : 1u) - 1);
        const int at = base + __popc(am & lanemask_lt());
        if (mine && at < C) l0[at] = (int32_t)(key & 0xffffffffLL);
    }
    double *const r = A.r + (int64_t)k * A.ld;
    double *const x = A.x + (int64_t)k * A.ld;
    uint32_t *const map = A.secmap + (int64_t)k * A.smw;
    const double tcf = A.tcoeff;
    int cur = 0;
    __syncthreads();
    if (s_cur > C) {  // (see the list overflow below)
        if (tid == 0) A.overflow[0] = 2;
        s_cur = 0;  // (every thread writes the same)
    }
    __syncthreads();
    for (;; ++t) {
        const int nn = min(s_nn, TAIL_NEAR);
        for (int i = tid; i < nn; i += BT)
            if (below_theta(r[tnear[i]], theta_deg(tcf, A.g.deg[tnear[i]]))) s_amb = 1;
        __syncthreads();
        const int Fc = s_cur;
        if (Fc == 0) break;
        if (t >= A.max_sweeps) {
            if (tid == 0) A.s_conv[k] = 0;
            break;
        }
        int32_t *const cl = cur ? l1 : l0, *const nl = cur ? l0 : l1;
        // push every entry of the sweep before any scatter (the reference reads
        // r over the whole frontier first): x += r, r = -0, c_u kept per entry
        double my_g = 0.0;
        for (int i0 = 0; i0 < Fc; i0 += BT) {  // warp-uniform trips
            const int i = i0 + tid;
            const bool live = i < Fc;
            int32_t u = 0, d = 0;
            bool fresh = false;
            if (live) {
                u = cl[i];
                d = A.g.deg[u];
                const double val = r[u];
                const double xo = x[u];
                x[u] = __dadd_rn(xo, val);
                r[u] = -0.0;
                my_g += fabs(val);
                if (near_theta(val, theta_deg(tcf, d))) s_amb = 1;  // final r >= theta
                cval[i] = __dmul_rn(val, __dmul_rn(__ddiv_rn(1.0, (double)d), A.beta));
                fresh = __double_as_longlong(xo) == 0;
            }
            slot_append(fresh, k, u, A.ld, A.pushed, A.pushed_cnt);
            block_count(fresh, 0, (unsigned)d, c_pvol);
            block_count(live, 0, (unsigned)d, c_ops);
            block_count(live, 0, 1u, c_push);
        }
        if (A.lg_f) atomicAdd(&c_g, my_g);
        if (tid == 0) {
            s_nn = 0;
            s_nxt = 0;
            A.s_last[k] = t;
        }
        __syncthreads();
        // scatter, TAIL_SEG entries at a time, arcs block-balanced
        for (int seg0 = 0; seg0 < Fc; seg0 += TAIL_SEG) {
            const int ns = min(TAIL_SEG, Fc - seg0);
            constexpr int PER = TAIL_SEG / BT;
            int dd[PER];
            int mine = 0;
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const int i = tid * PER + j;
                dd[j] = 0;
                if (i < ns) {
                    const int32_t u = cl[seg0 + i];
                    dd[j] = A.g.deg[u];
                    trow[i] = A.g.row[u];
                    tc[i] = cval[seg0 + i];
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
            for (int p0 = tid; p0 - tid < P; p0 += BT * UNROLL_T) {  // warp-uniform trips
                int32_t v[UNROLL_T], dv[UNROLL_T];
                double c[UNROLL_T], old[UNROLL_T];
                bool valid[UNROLL_T];
#pragma unroll
                for (int q = 0; q < UNROLL_T; ++q) {
                    const int p = p0 + q * BT;
                    valid[q] = p < P;
                    v[q] = 0; dv[q] = 0; c[q] = 0.0;
                    if (valid[q]) {
                        int lo = 0, hi = ns - 1;  // last entry with toff <= p
                        while (lo < hi) {
                            const int mid = (lo + hi + 1) >> 1;
                            if (toff[mid] <= p) lo = mid; else hi = mid - 1;
                        }
                        c[q] = tc[lo];
                        const int2 vd = __ldg(A.colp + trow[lo] + (p - toff[lo]));
                        v[q] = vd.x;
                        dv[q] = vd.y;
                    }
                }
#pragma unroll
                for (int q = 0; q < UNROLL_T; ++q) {
                    GD_DCHECK(!valid[q] || (v[q] >= 0 && v[q] < A.n));
                    old[q] = valid[q] ? atomicAdd(r + v[q], c[q]) : 0.0;
                }
#pragma unroll
                for (int q = 0; q < UNROLL_T; ++q) {
                    const long long ob = __double_as_longlong(old[q]);
                    const double th = theta_deg(tcf, dv[q]);
                    const bool first = valid[q] && ob == 0;
                    const bool negz = valid[q] && ob == (long long)0x8000000000000000ULL;
                    const double nw = __dadd_rn(old[q], c[q]);
                    const bool cross = valid[q] && old[q] < th && nw >= th;
                    if (valid[q] && below_theta(nw, th)) {
                        const int at = atomicAdd(&s_nn, 1);
                        if (at < TAIL_NEAR) tnear[at] = v[q]; else s_amb = 1;
                    }
                    block_count(first, 0, 1u, c_touch);
                    if (first) atomicOr(map + (v[q] >> 7), 1u << ((v[q] >> 2) & 31));
                    block_count(negz, 0, 1u, c_negz);
                    const unsigned am = __ballot_sync(FULL, cross);
                    int base = 0;
                    if (am && lane == __ffs(am) - 1) base = atomicAdd(&s_nxt, __popc(am));
                    base = __shfl_sync(FULL, base, __ffs(am ? am : 1u) - 1);
                    if (cross) {
                        const int at = base + __popc(am & lanemask_lt());
                        if (at < C) nl[at] = v[q]; else s_ovf = 1;
                    }
                }
            }
            __syncthreads();
        }
        if (tid == 0) {
            if (A.lg_f && t < A.lg_cap) {
                const int64_t at = (A.seed_base + k) * A.lg_cap + t;
                atomicAdd((unsigned long long *)A.lg_f + at, (unsigned long long)c_push[0]);
                atomicAdd((unsigned long long *)A.lg_ops + at, c_ops[0]);
                atomicAdd(A.lg_g + at, c_g);
            }
            A.s_ops[k] += c_ops[0];
            A.s_pvol[k] += c_pvol[0];
            A.s_pushes[k] += c_push[0];
            A.touched[k] += c_touch[0];
            A.s_negz[k] += c_negz[0];
            c_ops[0] = c_pvol[0] = 0;
            c_push[0] = c_touch[0] = c_negz[0] = 0;
            c_g = 0.0;
            s_cur = s_nxt;
            if (s_ovf) A.overflow[0] = 2;  // list capacity: the host redoes the solve
        }                                  // without tails
        cur ^= 1;
        __syncthreads();
        if (s_ovf) break;
    }
    if (tid == 0) {
        if (s_amb) A.s_amb[k] = 1;
        A.slot_base[k] = (int64_t)atomicAdd(A.cursor, A.pushed_cnt[k]);  // (final here)
    }
}

// ---------------------------------------------------------------------------
// Heat kernel, dense stages.  At tau = 10 on the products shape every stage
// after the third covers all of every slot's arcs (profiles: 3.46 G arcs per
// round for 28 slots); the push then does 3.46 G returning atomics per stage.
// A dense stage instead (a) pushes every active (slot, node) -- r >= theta in
// the stage layer, the same test the frontier entries passed -- and writes
// c_u = fl(fl(r tau/(k+1)) fl(1/d_u)) (0 when inactive) into a node-major
// n x m array, then (b) PULLS: r_next[k][v] = sum over the arcs (v, u) of
// c[u][k], the m slots of a row in chunks of HKC registers, warp per node for
// the degree-sorted heavy prefix, lane per node after it; the row sum is the
// final value, so the threshold test, the near-threshold check and the next
// frontier need no atomics.  Same c values as the push, summed in another
// order (x to rounding; integer work identical up to the near-threshold
// detector, as for the atomic scatter).
constexpr int HKC = GD_HKC;     // slots per accumulator chunk
constexpr int HEAVY_DEG = 256;  // rows split into segments at or above this degree
constexpr int HSEG = 2048;      // arcs per heavy-row segment (HSEG_TMA when staged:
constexpr int HSEG_TMA = 1024;  //  a segment fits a warp's TMA buffer)
constexpr int MEDIUM_DEG = 32;  // warp per node at or above this degree

// Bulk asynchronous copy (the TMA engine, cp.async.bulk) of the arc records
// [a0, a1) of the pull into this warp's shared-memory buffer, completion on the
// warp's mbarrier; returns the first staged index (a0 rounded down to 16 B).
// The buffer holds TBUF records: every range passed here is shorter (light
// warps: 32 rows of < MEDIUM_DEG arcs; medium rows < HEAVY_DEG; heavy segments
// HSEG_TMA).  Records stay in shared memory for all the stage's slot chunks.
constexpr int TBUF = 1026;       // int2 records per warp buffer (8 KB + 16 B)
__host__ __device__ inline size_t tma_bytes() { return 16 + (BT / 32) * (8 + (size_t)TBUF * 8); }
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ int64_t tma_stage(const int2 *colp, int64_t a0, int64_t a1, int2 *buf,
                                             uint64_t *bar, uint32_t &ph) {
    const int64_t s0 = a0 & ~1LL;
    if (a1 <= a0) return s0;  // (warp-uniform: nothing to copy, no phase)
    if (a1 - s0 + 1 > TBUF) return -1;  // (does not fit: the caller reads global memory)
    const uint32_t bytes = (uint32_t)((((a1 - s0) * 8) + 15) & ~15LL);
    __syncwarp();  // every lane is done with the previous contents
    if ((threadIdx.x & 31) == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
                     "[%0], [%1], %2, [%3];"
                     :: "r"(smem_u32(buf)), "l"(colp + s0), "r"(bytes), "r"(smem_u32(bar))
                     : "memory");
    }
    uint32_t ok = 0;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                     "selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(smem_u32(bar)), "r"(ph) : "memory");
    } while (!ok);
    ph ^= 1;
    return s0;
}

__device__ __forceinline__ void hk_dense_push(const RoundArgs &A, const Stage &S, double *rc,
                                              int32_t t) {
    const int64_t gtid = blockIdx.x * (int64_t)BT + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * BT;
    const int lane = threadIdx.x & 31;
    const double w = t < A.n_stages ? A.stage_w[t] : 0.0;  // (the last stage absorbs)
    for (int64_t u0 = gtid - lane; u0 < A.n; u0 += nthreads) {  // lane = node (warp-uniform trips)
        const int32_t u = (int32_t)(u0 + lane);
        const bool live = u < A.n;
        const int32_t d = live ? A.g.deg[u] : 0;
        const double th = theta_deg(A.tcoeff, d);
        for (int32_t k = 0; k < (int32_t)A.m; ++k) {
            const int64_t idx = (int64_t)k * A.ld + u;
            const double val = live ? rc[idx] : 0.0;
            const bool act = live && val >= th;
            bool fresh = false;
            double c = 0.0;
            if (act) {
                const double xo = A.x[idx];
                A.x[idx] = __dadd_rn(xo, val);
                rc[idx] = 0.0;
                if (near_theta(val, th)) A.s_amb[k] = 1;  // final r >= theta
                c = __dmul_rn(__dmul_rn(val, w), __ddiv_rn(1.0, (double)d));
                fresh = __double_as_longlong(xo) == 0;
                A.s_last[k] = t;
            }
            if (live) A.cn[(int64_t)u * A.m + k] = c;
            // (k is the same in every lane: plain warp reductions, no slot matching)
            const unsigned am = __ballot_sync(FULL, act);
            if (am) {
                const unsigned ds = __reduce_add_sync(FULL, act ? (unsigned)d : 0u);
                if (lane == 0) {
                    atomicAdd(S.ops + k, (unsigned long long)ds);
                    atomicAdd(S.push + k, (unsigned)__popc(am));
                }
            }
            const unsigned fm = __ballot_sync(FULL, fresh);
            if (fm) {
                unsigned long long b = 0;
                if (lane == 0) b = atomicAdd(A.pushed_cnt + k, (unsigned long long)__popc(fm));
                b = __shfl_sync(FULL, b, 0);
                if (fresh) A.pushed[(int64_t)k * A.ld + (int64_t)b + __popc(fm & lanemask_lt())] = u;
            }
        }
    }
}

// (slot k, node v) of a dense stage: its final value val of layer t+1
// same_word: all lanes hold the same slot and 32 consecutive nodes of one
// 128-node block, so the sector marks of the warp go into one map word
// append: write the next frontier's entries; else only count them (entries,
// arcs) in cnt[0..1] (shared): the next stage then runs densely without a list
__device__ __forceinline__ void hk_pull_finish(bool live, int32_t k, int32_t v, int32_t dv,
                                               double val, const RoundArgs &A, const Stage &S,
                                               double *rn, uint32_t *mapn, int nxt,
                                               bool same_word, bool append,
                                               unsigned long long *cnt) {
    const double th = theta_deg(A.tcoeff, dv);
    const bool nz = live && val != 0.0;
    if (nz) {
        rn[(int64_t)k * A.ld + v] = val;  // (the layer is zero here)
        if (below_theta(val, th)) A.s_amb[k] = 1;
    }
    if (same_word) {
        const unsigned bits = __reduce_or_sync(FULL, nz ? 1u << ((v >> 2) & 31) : 0u);
        const unsigned any = __ballot_sync(FULL, nz);
        if (bits && (threadIdx.x & 31) == __ffs(any) - 1)
            atomicOr(mapn + (int64_t)k * A.smw + (v >> 7), bits);
    } else if (nz) {
        atomicOr(mapn + (int64_t)k * A.smw + (v >> 7), 1u << ((v >> 2) & 31));
    }
    const bool cross = nz && val >= th;
    if (append) {
        stage_append(cross, k, v, dv, S, A, nxt);
    } else {
        const unsigned cm = __ballot_sync(FULL, cross);
        const unsigned long long ds = __reduce_add_sync(FULL, cross ? (unsigned)dv : 0u);
        if (cm && (threadIdx.x & 31) == 0) {
            atomicAdd(cnt, (unsigned long long)__popc(cm));
            atomicAdd(cnt + 1, ds);
        }
    }
}

__device__ void hk_pull(const RoundArgs &A, const Stage &S, double *rn, uint32_t *mapn, int nxt,
                        int64_t swarp, int64_t nwarps, bool append, int2 *tbuf, uint64_t *tbar,
                        uint32_t &tph) {
    __shared__ unsigned long long cnt[2];
    if (threadIdx.x < 2) cnt[threadIdx.x] = 0ULL;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t m = A.m;
    // heavy prefix: rows cut into segments of HSEG arcs, one warp per segment,
    // lanes split it; the warp-reduced partial sums go into hacc (node, slot)
    // with fp64 adds; after a grid barrier every heavy (node, slot) is finished
    // from hacc (which is cleared for the next dense stage)
    for (int64_t it = swarp; it < A.hitems; it += nwarps) {
        const int64_t key = A.hitem[it];
        const int64_t v = key >> 20, sg = key & 0xfffff;
        const int64_t row = A.g.row[v];
        const int32_t d = A.g.deg[v];
        const int32_t hs = A.tma ? HSEG_TMA : HSEG;
        const int32_t j0 = (int32_t)(sg * hs), j1 = min(d, (int32_t)(j0 + hs));
        const int64_t sb = A.tma ? tma_stage(A.colp, row + j0, row + j1, tbuf, tbar, tph) : -1;
        for (int64_t k0 = 0; k0 < m; k0 += HKC) {
            double acc[HKC];
#pragma unroll
            for (int q = 0; q < HKC; ++q) acc[q] = 0.0;
            for (int32_t j = j0 + lane; j < j1; j += 32) {
                const int32_t u = sb >= 0 ? tbuf[row + j - sb].x : __ldg(A.colp + row + j).x;
                const double *cu = A.cn + (int64_t)u * m + k0;
#pragma unroll
                for (int q = 0; q < HKC; ++q)
                    if (k0 + q < m) acc[q] += cu[q];
            }
#pragma unroll
            for (int q = 0; q < HKC; ++q)
                for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(FULL, acc[q], o);
            double mine = 0.0;
#pragma unroll
            for (int q = 0; q < HKC; ++q)
                if (lane == q) mine = acc[q];
            if (lane < HKC && k0 + lane < m && mine != 0.0)
                atomicAdd(A.hacc + v * m + k0 + lane, mine);
        }
    }
    // medium nodes (>= MEDIUM_DEG arcs) and the few up to the next multiple of 32:
    // one warp per node; light nodes: one lane per node (32 consecutive ids,
    // similar degrees) -- so no lane walks a row of more than MEDIUM_DEG arcs
    const int64_t lo = (A.mid + 31) & ~31LL;
    for (int64_t v = A.heavy + swarp; v < lo && v < A.n; v += nwarps) {
        const int64_t row = A.g.row[v];
        const int32_t d = A.g.deg[v];
        const int64_t sb = A.tma ? tma_stage(A.colp, row, row + d, tbuf, tbar, tph) : -1;
        for (int64_t k0 = 0; k0 < m; k0 += HKC) {
            double acc[HKC];
#pragma unroll
            for (int q = 0; q < HKC; ++q) acc[q] = 0.0;
            for (int32_t j = lane; j < d; j += 32) {
                const int32_t u = sb >= 0 ? tbuf[row + j - sb].x : __ldg(A.colp + row + j).x;
                const double *cu = A.cn + (int64_t)u * m + k0;
#pragma unroll
                for (int q = 0; q < HKC; ++q)
                    if (k0 + q < m) acc[q] += cu[q];
            }
#pragma unroll
            for (int q = 0; q < HKC; ++q)
                for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(FULL, acc[q], o);
            double mine = 0.0;
#pragma unroll
            for (int q = 0; q < HKC; ++q)
                if (lane == q) mine = acc[q];
            hk_pull_finish(lane < HKC && k0 + lane < m, (int32_t)(k0 + lane), (int32_t)v, d,
                           mine, A, S, rn, mapn, nxt, false, append, cnt);
        }
    }
    for (int64_t v0 = lo + swarp * 32; v0 < A.n; v0 += nwarps * 32) {
        const int64_t v = v0 + lane;
        const bool live = v < A.n;
        const int64_t row = live ? A.g.row[v] : 0;
        const int32_t d = live ? A.g.deg[v] : 0;
        // the 32 nodes' rows are one contiguous range of arc records
        const int64_t sb = A.tma ? tma_stage(A.colp, A.g.row[v0], A.g.row[min(v0 + 32, A.n)], tbuf,
                                             tbar, tph)
                                 : -1;
        for (int64_t k0 = 0; k0 < m; k0 += HKC) {
            double acc[HKC];
#pragma unroll
            for (int q = 0; q < HKC; ++q) acc[q] = 0.0;
            for (int32_t j = 0; j < d; ++j) {
                const int32_t u = sb >= 0 ? tbuf[row + j - sb].x : __ldg(A.colp + row + j).x;
                const double *cu = A.cn + (int64_t)u * m + k0;
#pragma unroll
                for (int q = 0; q < HKC; ++q)
                    if (k0 + q < m) acc[q] += cu[q];
            }
#pragma unroll
            for (int q = 0; q < HKC; ++q)
                hk_pull_finish(live && k0 + q < m, (int32_t)(k0 + q), (int32_t)v, d, acc[q], A, S,
                               rn, mapn, nxt, true, append, cnt);
        }
    }
    cg::this_grid().sync();  // (every heavy partial sum is in hacc)
    const int64_t gtid = blockIdx.x * (int64_t)BT + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * BT;
    const int64_t hm = A.heavy * m;
    for (int64_t i0 = gtid - lane; i0 < hm; i0 += nthreads) {  // (warp-uniform trips)
        const int64_t i = i0 + lane;
        const bool live = i < hm;
        const int64_t v = live ? i / m : 0;
        const int32_t k = live ? (int32_t)(i - v * m) : 0;
        double val = 0.0;
        if (live) {
            val = A.hacc[i];
            A.hacc[i] = 0.0;
        }
        hk_pull_finish(live, k, (int32_t)v, live ? A.g.deg[v] : 0, val, A, S, rn, mapn, nxt,
                       false, append, cnt);
    }
    __syncthreads();
    if (threadIdx.x == 0 && cnt[0])  // (counted, not listed: the next stage is dense)
        atomicAdd(A.fctr + nxt, (cnt[0] << CNT_SHIFT) + cnt[1]);
}

template <bool HK, bool STREAM = false>
__global__ void __launch_bounds__(BT, HK ? GD_KR_MINB_HK : GD_KR_MINB)
    k_rounds(const __grid_constant__ RoundArgs A, const __grid_constant__ OutArgs O) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Stage S = stage_carve(smem_raw, (int)A.m);
    // (heat kernel, A.tma) per warp: an mbarrier and a buffer for the pull's arc records
    uint64_t *const tbars = reinterpret_cast<uint64_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + stage_bytes((int)A.m) + 15) & ~(uintptr_t)15);
    int2 *const tbuf = reinterpret_cast<int2 *>(tbars + BT / 32) + (size_t)(threadIdx.x >> 5) * TBUF;
    uint64_t *const tbar = tbars + (threadIdx.x >> 5);
    uint32_t tph = 0;
    if (HK && A.tma && (threadIdx.x & 31) == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(tbar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const int lane = threadIdx.x & 31;
    const int64_t gtid = blockIdx.x * (int64_t)BT + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * BT;
    const int64_t nwarps = nthreads >> 5;
    // warp index that walks the blocks first: consecutive work units land on
    // different SMs (the finishing work of a few slots must use them all)
    const int64_t swarp = (int64_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x;
    for (int64_t k = threadIdx.x; k < A.m; k += BT) {
        S.ops[k] = S.pvol[k] = S.scnt[k] = 0;
        S.push[k] = S.touch[k] = S.negz[k] = 0;
        S.nf[k] = 0;
        S.gsum[k] = 0.0;
    }
    if (threadIdx.x == 0) {
        *S.fcnt = 0;
        *S.next = 0;
        S.nfin[0] = S.nfin[1] = 0;
    }
    __syncthreads();

    bool tail = false;
    bool nolist = false;  // (heat kernel) the current stage's frontier was only counted
    int64_t pmax = 0;  // largest round so far (the same in every block)
    for (int32_t t = STREAM ? *A.t_state : 0;; ++t) {
        const int cur = t & 1, nxt = cur ^ 1;
        const unsigned long long packed = *(volatile unsigned long long *)(A.fctr + cur);
        const int64_t F = (int64_t)(packed >> CNT_SHIFT);
        const int64_t P = (int64_t)(packed & ARC_MASK);
        if (gtid == 0 && t < A.rlog_cap) {
            A.rlog[3 * t] = F;
            A.rlog[3 * t + 1] = P;
            A.rlog[3 * t + 2] = globaltimer();
            A.rlog[3 * A.rlog_cap] = t + 1;
        }
        int64_t nn = 0;
        {   // final values of last round's landings just below theta (common.cuh)
            double *const rl = (HK && (t & 1)) ? A.r2 : A.r;
            nn = min((int64_t)*(volatile unsigned long long *)(A.nearl.cnt[cur]), A.nearl.cap);
            for (int64_t i = gtid; i < nn; i += nthreads) {
                const int64_t key = A.nearl.key[cur][i];
                const int32_t k = (int32_t)(key >> 32), v = (int32_t)(key & 0xffffffffLL);
                if (below_theta(rl[(int64_t)k * A.ld + v], theta_deg(A.tcoeff, A.g.deg[v])))
                    A.s_amb[k] = 1;
            }
        }
        unsigned nfin = 0, nidle = 0;
        bool refill = false;
        if (STREAM) {
            // seeds that finished: running slots without entries this round,
            // listed in slot order (every block must see the same list: the
            // work units below are split across blocks by position in it)
            if (threadIdx.x < 32) {
                unsigned cnt = 0, ci = 0;
                for (int64_t k0 = 0; k0 < A.m; k0 += 32) {
                    const int64_t k = k0 + lane;
                    const int32_t si = k < A.m ? A.s_idx[k] : 0;
                    const bool f = k < A.m && si >= 0 &&
                                   *(volatile unsigned long long *)(A.sn[cur] + k) == 0ULL;
                    const bool id = k < A.m && si < 0;
                    const unsigned b = __ballot_sync(FULL, f), bi = __ballot_sync(FULL, id);
                    if (f) S.fin[cnt + __popc(b & lanemask_lt())] = (int32_t)k;
                    if (id) S.idle[ci + __popc(bi & lanemask_lt())] = (int32_t)k;
                    cnt += __popc(b);
                    ci += __popc(bi);
                }
                if (lane == 0) {
                    S.nfin[0] = cnt;
                    S.nfin[1] = ci;
                }
            }
            __syncthreads();
            nfin = S.nfin[0];
            nidle = S.nfin[1];
            // cohorts: free slots take new seeds only once `cohort` of them are
            // free (or nothing else runs), so seeds start -- and reach their
            // big rounds -- together
            const bool left =
                *(volatile unsigned long long *)A.seed_ctr < (unsigned long long)A.n_seeds;
            refill = left && (nfin + nidle >= (unsigned)A.cohort || nfin + nidle == (unsigned)A.m);
            const unsigned long long done = *(volatile unsigned long long *)A.done_ctr;
            if ((F == 0 && nfin == 0 && !refill) || (int64_t)done >= A.seg_done) {
                if (gtid == 0) *A.t_state = t;
                break;
            }
            if (nn > 0) grid.sync();  // (the reset below must not overtake those reads)
        } else if (F == 0) {
            break;
        }
        pmax = P > pmax ? P : pmax;
        if (!HK && !STREAM && A.tail_list && P <= A.tail_p && F <= A.tail_f && 16 * P <= pmax) {
            // the rest of the wave (past its peak) in k_tail, one block per slot
            if (gtid == 0) {
                A.tail_state[0] = t;
                A.tail_state[1] = F;
            }
            tail = true;
            break;
        }
        if (((P + 31) >> 5) > A.ccap) {  // arc-chunk map too small: report, stop
            if (gtid == 0) A.overflow[0] = 1;
            break;
        }
        if (STREAM && F > A.fcap) {  // (per-slot sweep caps below)
            if (gtid == 0) A.overflow[0] = 1;
            break;
        }
        if (!STREAM && (t >= A.max_sweeps || F > A.fcap)) {
            for (int64_t e = gtid; e < F && e < A.fcap; e += nthreads)
                A.s_conv[A.ukey[e] >> 32] = 0;
            break;
        }
        // ---------------- phase A: push the frontier entries ----------------
        // Entries arrive in append order; each is also placed into a copy of
        // the frontier grouped by slot (per-slot packed reservation gives its
        // position and first arc), so phase B walks the arcs slot by slot and
        // the residual words it updates at any moment belong to a few slots
        // (an L2-sized working set instead of all slots' vectors).
        if (gtid == 0) {
            A.fctr[nxt] = 0ULL;
            A.cctr[0] = 0ULL;
            *A.nearl.cnt[nxt] = 0ULL;  // (last read two barriers ago)
        }
        for (int64_t k = gtid; k < A.m; k += nthreads) {
            A.scnt[nxt][k] = 0ULL;
            if (STREAM) A.sn[nxt][k] = 0ULL;
        }
        double *const rc = (HK && (t & 1)) ? A.r2 : A.r;        // layer t
        double *const rn = (HK && !(t & 1)) ? A.r2 : A.r;       // layer t+1 (HK)
        uint32_t *const mapn = (HK && !(t & 1)) ? A.secmap2 : A.secmap;
        if (HK && t >= 1 && t < A.n_stages) {
            // layer t+1 reuses layer t-1's array: zero its touched sectors
            const int64_t total = A.m * A.smw;
            const int64_t gw = gtid >> 5, nw = nthreads >> 5;
            for (int64_t w0 = gw * 32; w0 < total; w0 += nw * 32) {
                const uint32_t mine = (w0 + lane < total) ? mapn[w0 + lane] : 0u;
                unsigned any = __ballot_sync(FULL, mine != 0u);
                while (any) {
                    const int src = __ffs(any) - 1;
                    any &= any - 1;
                    const uint32_t wb = __shfl_sync(FULL, mine, src);
                    if ((wb >> lane) & 1u) {
                        const int64_t w = w0 + src, kk = w / A.smw;
                        const int64_t sec = (w - kk * A.smw) * 32 + lane;
                        double *base = rn + kk * A.ld;
                        if (4 * sec + 3 < A.ld)
                            reinterpret_cast<double4 *>(base)[sec] = make_double4(0.0, 0.0, 0.0, 0.0);
                        else
                            for (int64_t i = 4 * sec; i < A.ld; ++i) base[i] = 0.0;
                    }
                }
                if (mine) mapn[w0 + lane] = 0u;
            }
        }
        // group this round only when it is large enough to be L2-bound (small
        // rounds are barrier-bound and keep the append order)
        // heat kernel: a stage whose frontier covers at least half of every slot's
        // arcs is run densely -- push every active (slot, node) here, then a PULL
        // SpMM over all nodes in phase B (no atomics; see hk_pull_node)
        // (nolist: the previous dense stage only counted its crossings, so this one
        // is dense too; a dense stage lists them only below 3/4 density)
        const bool dense = HK && A.cn && (nolist || (t < A.n_stages && 2 * P >= A.m * A.g.n_arcs));
        const bool dense_pull = dense && t < A.n_stages;
        const bool list_next = !(dense_pull && 4 * P >= 3 * A.m * A.g.n_arcs);
        const bool grp = !dense && A.grouped && P >= A.group_min;
        if (grp) slot_bases(S, A, cur);
        if (dense) hk_dense_push(A, S, rc, t);
        for (int64_t e0 = gtid - lane; e0 < (dense ? 0 : F); e0 += nthreads) {  // warp-uniform
            const int64_t e = e0 + lane;
            const bool live = e < F;
            int32_t k = 0, u = 0, d = 0;
            bool fresh = false;
            int64_t clo = 0, chi = 0, cfull = 0, pos = 0;
            int64_t key = 0;
            double val = 0.0, xo = 0.0;
            bool capped = false;  // (streaming) the seed's sweep cap: not pushed
            if (live) {
                key = A.ukey[e];
                k = (int32_t)(key >> 32);
                u = (int32_t)(key & 0xffffffffLL);
                const int64_t idx = (int64_t)k * A.ld + u;
                GD_DCHECK(k >= 0 && k < A.m && u >= 0 && u < A.n);
                d = A.g.deg[u];
                capped = STREAM && (int64_t)(t - A.s_t0[k]) >= A.max_sweeps;
                if (!capped) {
                    val = rc[idx];
                    xo = A.x[idx];
                    A.x[idx] = __dadd_rn(xo, val);
                    rc[idx] = HK ? 0.0 : -0.0;
                    if (near_theta(val, theta_deg(A.tcoeff, d))) A.s_amb[k] = 1;  // final r >= theta
                } else {
                    A.s_conv[k] = 0;
                    xo = 1.0;  // (not a first push)
                }
            }
            // group-sorted position: one packed reservation per (warp, slot group);
            // ungrouped: the entry keeps its append position and arc offset
            unsigned long long b = 0;
            if (!grp) {
                if (live) b = ((unsigned long long)e << CNT_SHIFT) | (unsigned long long)A.uarc[e];
            } else {
                const int32_t kg = k / (int32_t)A.sgroup;
                const unsigned long long pv = live ? (1ULL << CNT_SHIFT) + (unsigned long long)d : 0ULL;
                const unsigned peers = __match_any_sync(FULL, live ? kg : -1);
                unsigned long long pre = 0, tot = 0;
                for (int i = 0; i < 32; ++i) {
                    const unsigned long long vi = __shfl_sync(FULL, pv, i);
                    if ((peers >> i) & 1u) {
                        tot += vi;
                        if (i < lane) pre += vi;
                    }
                }
                const int leader = __ffs(peers) - 1;
                unsigned long long old = 0;
                if (live && lane == leader) old = atomicAdd(A.sfill + kg, tot);
                old = __shfl_sync(FULL, old, leader);
                if (live) b = S.sbase[kg] + old + pre;
            }
            if (live) {
                pos = (int64_t)(b >> CNT_SHIFT);
                const int64_t a0 = (int64_t)(b & ARC_MASK);
                A.skey[pos] = key;
                A.sarc[pos] = a0;
                A.frow[pos] = A.g.row[u];
                A.fcval[pos] =
                    capped ? 0.0  // (phase B skips c == 0)
                    : HK ? __dmul_rn(__dmul_rn(val, A.stage_w[t < A.n_stages ? t : 0]),
                                     __ddiv_rn(1.0, (double)d))
                         : __dmul_rn(val, __dmul_rn(__ddiv_rn(1.0, (double)d), A.beta));
                fresh = __double_as_longlong(xo) == 0;  // first push of u
                // chunks (32 arcs) whose first arc lies in this entry: [clo, chi)
                clo = (a0 + 31) >> 5;
                chi = min((a0 + d + 31) >> 5, A.ccap);
                cfull = (a0 + d) >> 5;  // chunks below this one lie entirely in the entry
            }
            // hubs own thousands of chunks, so the warp writes them together;
            // bit 31 marks a chunk whose 32 arcs all belong to this entry
            unsigned big = __ballot_sync(FULL, chi - clo > 4);
            if (!(big >> lane & 1u))
                for (int64_t c = clo; c < chi; ++c)
                    A.chunk_e[c] = (int32_t)((uint32_t)pos | (c < cfull ? 0x80000000u : 0u));
            while (big) {
                const int src = __ffs(big) - 1;
                big &= big - 1;
                const int64_t lo2 = __shfl_sync(FULL, clo, src), hi2 = __shfl_sync(FULL, chi, src);
                const int64_t cf2 = __shfl_sync(FULL, cfull, src);
                const uint32_t e2 = (uint32_t)__shfl_sync(FULL, pos, src);
                for (int64_t c = lo2 + lane; c < hi2; c += 32)
                    A.chunk_e[c] = (int32_t)(e2 | (c < cf2 ? 0x80000000u : 0u));
            }
            const bool pushed = live && !capped;
            if (A.lg_f && pushed) atomicAdd(S.gsum + k, fabs(val));
            slot_append(fresh, k, u, A.ld, A.pushed, A.pushed_cnt);
            block_count(fresh, k, (unsigned)d, S.pvol);
            block_count(pushed, k, (unsigned)d, S.ops);
            block_count(pushed, k, 1u, S.push);
            if (pushed) A.s_last[k] = t;
        }
        if (STREAM && nfin) {
            // finished seeds: output segment + counters (one thread each) ...
            for (int64_t j = gtid; j < nfin; j += nthreads) {
                const int32_t k = S.fin[j];
                const int64_t si = A.s_idx[k];
                const unsigned long long pc = A.pushed_cnt[k];
                const int64_t b = (int64_t)atomicAdd(A.cursor, pc);
                A.slot_base[k] = b;
                A.drain_cnt[k] = (int64_t)pc;
                const int64_t pushes = (int64_t)A.s_pushes[k];
                O.sweeps[si] = (int64_t)(A.s_last[k] - A.s_t0[k]) + 1;
                O.ops[si] = (int64_t)A.s_ops[k];
                O.pushes[si] = pushes;
                O.conv[si] = A.s_conv[k];
                O.support[si] = (int64_t)A.touched[k] - (pushes - (int64_t)A.s_negz[k]);
                O.xoff[si] = b;
                O.xcnt[si] = (int64_t)pc;
            }
            // ... and their r back to +0.0: zero the marked sectors, clear the map
            const int64_t units = (int64_t)nfin * A.reset_units;
            const int64_t per = (A.smw + A.reset_units - 1) / A.reset_units;
            for (int64_t u = swarp; u < units && !(A.dbg & 2); u += nwarps) {
                const int32_t k = S.fin[u / A.reset_units];
                const int64_t lo = (u % A.reset_units) * per, hi = min(A.smw, lo + per);
                uint32_t *map = A.secmap + (int64_t)k * A.smw;
                double *rk = A.r + (int64_t)k * A.ld;
                for (int64_t w0 = lo; w0 < hi; w0 += 32) {
                    const uint32_t mine = (w0 + lane < hi) ? map[w0 + lane] : 0u;
                    unsigned any = __ballot_sync(FULL, mine != 0u);
                    while (any) {
                        const int src = __ffs(any) - 1;
                        any &= any - 1;
                        const uint32_t wb = __shfl_sync(FULL, mine, src);
                        if ((wb >> lane) & 1u) {
                            const int64_t sec = (w0 + src) * 32 + lane;
                            if (4 * sec + 3 < A.ld)
                                reinterpret_cast<double4 *>(rk)[sec] = make_double4(0.0, 0.0, 0.0, 0.0);
                            else
                                for (int64_t i = 4 * sec; i < A.ld; ++i) rk[i] = 0.0;
                        }
                    }
                    if (mine) map[w0 + lane] = 0u;
                }
            }
        }
        __syncthreads();
        if (A.lg_f && !STREAM && t < A.lg_cap)  // per-seed sweep logs (waves: t = sweep)
            for (int64_t k = threadIdx.x; k < A.m; k += BT) {
                if (S.push[k]) {
                    const int64_t at = (A.seed_base + k) * A.lg_cap + t;
                    atomicAdd((unsigned long long *)A.lg_f + at, (unsigned long long)S.push[k]);
                    atomicAdd((unsigned long long *)A.lg_ops + at, S.ops[k]);
                    atomicAdd(A.lg_g + at, S.gsum[k]);
                }
                S.gsum[k] = 0.0;
            }
        counters_flush(S.ops, A.s_ops, A.m);
        counters_flush(S.pvol, A.s_pvol, A.m);
        counters_flush(S.push, A.s_pushes, A.m);
        grid.sync();
        if (gtid == 0 && t < A.rlog_cap) {
            A.rlog[3 * A.rlog_cap + 1 + t] = globaltimer();
            A.rlog[4 * A.rlog_cap + 1 + t] = (int64_t)nfin | ((int64_t)refill << 32);
        }
        // ---------------- phase B: arc-balanced scatter ----------------------
        // chunk c = arcs [32c, 32c+32) of the slot-grouped frontier.  Warp w
        // takes chunk groups w, w + W, w + 2W, ... (UNROLL chunks, each lane
        // one atomic in flight per chunk), so the whole grid sweeps the arc
        // space front to back, slot by slot, without a claim counter.
        for (int64_t k = gtid; k < A.m; k += nthreads) A.sfill[k] = 0ULL;  // for the next round
        if (STREAM && (nfin || refill)) {
            // finished seeds: x over the pushed list out (caller ids), zeroed.
            // Work-balanced: the finished slots' pushed lists are one
            // concatenated index space (prefix in shared memory, same in every
            // block), walked 256 entries per warp step with all 8 gathers of a
            // lane in flight before any store
            if (threadIdx.x < 32) {
                unsigned long long run = 0;
                for (unsigned j0 = 0; j0 < nfin; j0 += 32) {
                    const unsigned j = j0 + lane;
                    const unsigned long long c = j < nfin ? (unsigned long long)A.drain_cnt[S.fin[j]] : 0ULL;
                    unsigned long long incl = c;
                    for (int o = 1; o < 32; o <<= 1) {
                        const unsigned long long y = __shfl_up_sync(FULL, incl, o);
                        if (lane >= o) incl += y;
                    }
                    if (j < nfin) S.sbase[j] = run + incl - c;
                    run += __shfl_sync(FULL, incl, 31);
                }
                if (lane == 0) S.scan[0] = run;
            }
            __syncthreads();
            const int64_t total = (int64_t)S.scan[0];
            constexpr int XQ = 8;
            for (int64_t e0 = swarp * 32 * XQ; e0 < total && !(A.dbg & 1); e0 += nwarps * 32 * XQ) {
                int32_t v[XQ], id[XQ];
                int64_t at[XQ], xo[XQ];
                double xv[XQ];
#pragma unroll
                for (int q = 0; q < XQ; ++q) {
                    const int64_t e = e0 + q * 32 + lane;
                    v[q] = -1;
                    if (e < total) {
                        unsigned lo = 0, hi = nfin;  // last j with prefix[j] <= e
                        while (hi - lo > 1) {
                            const unsigned mid = (lo + hi) >> 1;
                            if ((int64_t)S.sbase[mid] <= e) lo = mid; else hi = mid;
                        }
                        const int32_t k = S.fin[lo];
                        const int64_t i = e - (int64_t)S.sbase[lo];
                        xo[q] = (int64_t)k * A.ld;
                        at[q] = A.slot_base[k] + i;
                        v[q] = A.pushed[xo[q] + i];
                    }
                }
#pragma unroll
                for (int q = 0; q < XQ; ++q) {
                    if (v[q] < 0) continue;
                    xv[q] = A.x[xo[q] + v[q]];
                    id[q] = O.inv ? __ldg(O.inv + v[q]) : v[q];
                }
#pragma unroll
                for (int q = 0; q < XQ; ++q) {
                    if (v[q] < 0) continue;
                    A.x[xo[q] + v[q]] = 0.0;
                    if (at[q] < O.xcap) {
                        O.xnodes[at[q]] = id[q];
                        O.xvals[at[q]] = xv[q];
                    }
                }
            }
            // the near-threshold flag (final now), then -- once the cohort is
            // complete -- the free slots' next seeds
            const unsigned nfree = refill ? nfin + nidle : nfin;
            for (int64_t j0 = swarp * 32; j0 < nfree; j0 += nwarps * 32) {
                const int64_t j = j0 + lane;
                bool act = false;
                int32_t k = 0, s = 0, d = 0;
                if (j < nfree) {
                    k = j < nfin ? S.fin[j] : S.idle[j - nfin];
                    if (j < nfin) {
                        const int64_t si = A.s_idx[k];
                        O.amb[si] = A.s_amb[k];
                        if (A.s_amb[k]) atomicAdd(O.amb_cnt, 1ULL);
                        // (counted here, not in phase A: every block reads the
                        // counter at the next round start, after the barrier)
                        atomicAdd(A.done_ctr, 1ULL);
                    }
                    const unsigned long long i = refill ? atomicAdd(A.seed_ctr, 1ULL)
                                                        : (unsigned long long)A.n_seeds;
                    if ((int64_t)i < A.n_seeds) {
                        s = (int32_t)A.seeds[i];
                        if (A.perm) s = A.perm[s];
                        A.s_idx[k] = (int32_t)i;
                        A.s_t0[k] = t + 1;
                        A.s_last[k] = t;  // (sweeps = s_last - t0 + 1)
                        A.r[(int64_t)k * A.ld + s] = A.alpha;
                        A.secmap[(int64_t)k * A.smw + (s >> 7)] |= 1u << ((s >> 2) & 31);
                        A.touched[k] = 1;
                        A.pushed_cnt[k] = 0;
                        A.s_ops[k] = A.s_pushes[k] = A.s_negz[k] = A.s_pvol[k] = 0;
                        A.s_conv[k] = 1;
                        A.s_amb[k] = 0;
                        d = A.g.deg[s];
                        act = A.alpha >= theta_deg(A.tcoeff, d);
                    } else {
                        A.s_idx[k] = -1;  // no seeds left: idle
                    }
                }
                stage_append(act, k, s, d, S, A, nxt);
            }
        }
        const int64_t C = (P + 31) >> 5;
        const int64_t *fa = A.sarc;
        if (dense_pull) hk_pull(A, S, rn, mapn, nxt, swarp, nwarps, list_next, tbuf, tbar, tph);
        else if (!dense && (!HK || t < A.n_stages)) {  // (the last heat-kernel stage is absorbing)
            const int64_t c1 = C;
          for (;;) {
            // block b owns super-chunks b, b + G, b + 2G, ... (SUPER groups of
            // UNROLL chunks each); its warps claim groups in order from a
            // shared counter, so the grid advances through the arc space
            // together while latency differences between warps even out
            unsigned long long claim = 0;
            if (lane == 0) claim = atomicAdd(S.next, 1ULL);
            const int64_t i = (int64_t)__shfl_sync(FULL, claim, 0);
            int64_t cb, cend;
            if (grp) {
                const int64_t sup = i / SUPER, within = i - sup * SUPER;
                cb = ((sup * gridDim.x + blockIdx.x) * SUPER + within) * UNROLL;
                cend = c1;
            } else {  // this block's contiguous range
                cb = (int64_t)(((unsigned long long)C * blockIdx.x) / gridDim.x) + i * UNROLL;
                cend = (int64_t)(((unsigned long long)C * (blockIdx.x + 1)) / gridDim.x);
            }
            if (cb >= cend) break;
            int32_t k[UNROLL], v[UNROLL], dv[UNROLL];
            double c[UNROLL], old[UNROLL];
            bool valid[UNROLL];
            // stage 1: every load of all UNROLL chunks, before any atomic, so
            // the chunks' dependent-load chains overlap
#pragma unroll
            for (int q = 0; q < UNROLL; q++) {
                const int64_t ch = cb + q;
                const bool live = ch < cend;
                GD_DCHECK(!live || ch < A.ccap);
                const uint32_t raw = live ? (uint32_t)A.chunk_e[ch] : 0u;  // same for all lanes
                const int64_t e = raw & 0x7fffffffu;
                const int64_t a = ch << 5;
                int64_t me = e;
                if (!(raw >> 31)) {
                    // entries starting inside (a, a+32): one bit per start offset
                    const int64_t wi = e + 1 + lane;
                    const int64_t st = (live && wi < F) ? fa[wi] : INT64_MAX;
                    const int64_t pos = st - a;
                    const unsigned starts = __reduce_or_sync(FULL, pos < 32 ? (1u << pos) : 0u);
                    me = e + __popc(starts & ((2u << lane) - 1u));
                }
                const int64_t p = a + lane;
                valid[q] = live && p < P;
                k[q] = 0; v[q] = 0; dv[q] = 0; c[q] = 0.0;
                if (valid[q]) {
                    GD_DCHECK(me >= 0 && me < F && fa[me] <= p && p < fa[me] + A.g.n_arcs);
                    k[q] = (int32_t)(A.skey[me] >> 32);
                    c[q] = A.fcval[me];
                    GD_DCHECK(A.frow[me] + (p - fa[me]) < A.g.n_arcs);
                    const int2 vd = __ldg(A.colp + A.frow[me] + (p - fa[me]));
                    v[q] = vd.x;
                    dv[q] = vd.y;
                    if (STREAM) valid[q] = c[q] != 0.0;  // (an entry past its seed's sweep cap)
                }
            }
            // stage 2: the atomics, back to back (UNROLL in flight per lane)
#pragma unroll
            for (int q = 0; q < UNROLL; q++) {
                GD_DCHECK(!valid[q] || (k[q] >= 0 && k[q] < A.m && v[q] >= 0 && v[q] < A.n));
                old[q] = valid[q] ? atomicAdd(rn + (int64_t)k[q] * A.ld + v[q], c[q]) : 0.0;
            }
            // stage 3: first touch / re-touch of a pushed node / frontier entry
#pragma unroll
            for (int q = 0; q < UNROLL; q++) {
                const long long ob = __double_as_longlong(old[q]);
                const double th = theta_deg(A.tcoeff, dv[q]);
                const bool first = valid[q] && ob == 0;
                const bool negz = valid[q] && ob == (long long)0x8000000000000000ULL;
                const double nw = __dadd_rn(old[q], c[q]);
                const bool cross = valid[q] && old[q] < th && nw >= th;
                if (valid[q] && below_theta(nw, th)) near_record(A.nearl, nxt, k[q], v[q], A.s_amb);
                block_count(first, k[q], 1u, S.touch);
                if (first)  // first write of this r word: remember its 32 B sector
                    atomicOr(mapn + (int64_t)k[q] * A.smw + (v[q] >> 7), 1u << ((v[q] >> 2) & 31));
                block_count(negz, k[q], 1u, S.negz);
                stage_append(cross, k[q], v[q], dv[q], S, A, nxt);
            }
          }
        }
        stage_flush(S, A, nxt);  // (its barriers also order the claim counter reset)
        nolist = dense_pull && !list_next;
        if (threadIdx.x == 0) *S.next = 0;
        counters_flush(S.touch, A.touched, A.m);
        counters_flush(S.negz, A.s_negz, A.m);
        grid.sync();
    }
    // reserve each slot's output segment (pushed counts are final here; after
    // a tail handed to k_tail, it reserves them)
    if (!STREAM && !tail && blockIdx.x == 0)
        for (int64_t k = threadIdx.x; k < A.m; k += BT)
            A.slot_base[k] = (int64_t)atomicAdd(A.cursor, A.pushed_cnt[k]);
}

// Seeds -> slots: r[s] = alpha, S_0 = {s} if alpha >= theta_s.
// One block (zero_ctrs, m <= blockDim.x * 8): also zeroes the wave's round
// counters first -- the frontier counters, per-group counts, near-list counters
// and the tail hand-over -- instead of four memset launches per wave.
__device__ void wave_init_slot(const RoundArgs &A, const int64_t *__restrict__ seeds,
                               double alpha, int64_t k);
__global__ void k_wave_init(RoundArgs A, const int64_t *__restrict__ seeds, double alpha,
                            int zero_ctrs, int64_t scnt_n) {
    if (zero_ctrs) {
        for (int64_t i = threadIdx.x; i < scnt_n; i += blockDim.x) A.scnt[0][i] = 0ULL;
        if (threadIdx.x < 2) {
            A.fctr[threadIdx.x] = 0ULL;
            *A.nearl.cnt[threadIdx.x] = 0ULL;
            if (A.tail_state) A.tail_state[threadIdx.x] = -1;
        }
        __syncthreads();
        for (int64_t k = threadIdx.x; k < A.m; k += blockDim.x) wave_init_slot(A, seeds, alpha, k);
        return;
    }
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= A.m) return;
    wave_init_slot(A, seeds, alpha, k);
}

__device__ void wave_init_slot(const RoundArgs &A, const int64_t *__restrict__ seeds,
                               double alpha, int64_t k) {
    int32_t s = (int32_t)seeds[k];
    if (A.perm) s = A.perm[s];
    A.seed[k] = s;
    A.r[k * A.ld + s] = alpha;
    A.touched[k] = 1;
    A.secmap[k * A.smw + (s >> 7)] |= 1u << ((s >> 2) & 31);
    A.pushed_cnt[k] = 0;
    A.s_ops[k] = 0;
    A.s_pushes[k] = 0;
    A.s_negz[k] = 0;
    A.s_pvol[k] = 0;
    A.s_last[k] = -1;
    A.s_conv[k] = 1;
    A.s_amb[k] = 0;
    int32_t d = A.g.deg[s];
    A.sfill[k] = 0ULL;
    const bool act = alpha >= theta_deg(A.tcoeff, d);
    if (A.s_idx) {  // streaming form: slot k starts seed k; the rest follow in-kernel
        A.s_idx[k] = (int32_t)k;
        A.s_t0[k] = 0;
        A.sn[0][k] = act ? 1ULL : 0ULL;
        A.sn[1][k] = 0ULL;
        if (k == 0) {
            *A.seed_ctr = (unsigned long long)A.m;
            *A.done_ctr = 0ULL;
            *A.t_state = 0;
        }
    }
    if (act) {
        unsigned long long old = atomicAdd(A.fctr, (1ULL << CNT_SHIFT) + (unsigned long long)d);
        int64_t idx = (int64_t)(old >> CNT_SHIFT);
        if (idx < A.fcap) {
            A.ukey[idx] = (k << 32) | (uint32_t)s;
            A.uarc[idx] = (int64_t)(old & ARC_MASK);
        }
        if (A.grouped)  // (zeroed by the host before this kernel)
            atomicAdd(A.scnt[0] + k / A.sgroup, (1ULL << CNT_SHIFT) + (unsigned long long)d);
    }
}


// grid (CHUNKS, slots): copy x over the pushed list out (caller ids) and zero
// x and r there; block (0, k) writes the seed's counters.
// support = touched - (pushes - negz): every push writes -0.0 into r[u] and
// the first later contribution observes it, so the pushed nodes still at
// zero are pushes - negz.
__global__ void k_wave_extract(RoundArgs A, OutArgs O, int64_t seed_base) {
    const int k = blockIdx.y;
    const int64_t off = (int64_t)k * A.ld;
    const int64_t pc = (int64_t)A.pushed_cnt[k];
    const int64_t b = A.slot_base[k];
    // XU entries per thread with every load issued before any store (the x
    // stores would otherwise order each gather behind the previous one)
    constexpr int XU = 4;
    const int64_t stride = (int64_t)CHUNKS * blockDim.x;
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
            if (b + i < O.xcap) {
                O.xnodes[b + i] = id[j];
                O.xvals[b + i] = __dmul_rn(O.xscale, xv[j]);
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t si = seed_base + k;
        const int64_t pushes = (int64_t)A.s_pushes[k];
        O.sweeps[si] = (int64_t)A.s_last[k] + 1;
        O.ops[si] = (int64_t)A.s_ops[k];
        O.pushes[si] = pushes;
        O.conv[si] = A.s_conv[k];
        O.support[si] = O.hk ? -1 : (int64_t)A.touched[k] - (pushes - (int64_t)A.s_negz[k]);
        O.xoff[si] = b;
        O.xcnt[si] = pc;
        O.amb[si] = A.s_amb[k];
        if (A.s_amb[k]) atomicAdd(O.amb_cnt, 1ULL);
        if (pc == 0) A.r[off + A.seed[k]] = 0.0;  // an inactive seed keeps r = alpha
    }
}

// Work-balanced form of k_wave_extract: the wave's pushed lists are treated
// as one concatenated index space (per-slot prefix of pushed_cnt in shared
// memory, slot found by binary search), so every thread of a full-GPU grid
// has XB independent gathers in flight whatever the slots' sizes -- the
// per-slot grid leaves most warps with one or two entries and the kernel
// waits on the longest dependent chain (pushed -> x / inv -> store) per block
// wave.  Per-seed counters: threads k < m of block 0.
constexpr int XB = 8;
constexpr int EXB_MAX_SLOTS = 1024;
__global__ void __launch_bounds__(256) k_wave_extract_bal(RoundArgs A, OutArgs O, int64_t seed_base) {
    __shared__ int64_t pre[EXB_MAX_SLOTS + 1];
    const int m = (int)A.m;
    if (threadIdx.x == 0) {
        int64_t run = 0;
        for (int k = 0; k < m; ++k) {
            pre[k] = run;
            run += (int64_t)A.pushed_cnt[k];
        }
        pre[m] = run;
    }
    __syncthreads();
    const int64_t total = pre[m];
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t g0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g0 < total; g0 += XB * nth) {
        int32_t u[XB], id[XB];
        int64_t at[XB], xo[XB];
        double xv[XB];
#pragma unroll
        for (int j = 0; j < XB; ++j) {
            const int64_t g = g0 + j * nth;
            u[j] = -1;
            if (g < total) {
                int lo = 0, hi = m - 1;  // last k with pre[k] <= g
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (pre[mid] <= g) lo = mid; else hi = mid - 1;
                }
                const int64_t i = g - pre[lo];
                xo[j] = (int64_t)lo * A.ld;
                at[j] = A.slot_base[lo] + i;
                u[j] = __ldg(A.pushed + (int64_t)lo * A.ld + i);
            }
        }
#pragma unroll
        for (int j = 0; j < XB; ++j) {
            xv[j] = u[j] >= 0 ? A.x[xo[j] + u[j]] : 0.0;
            id[j] = (u[j] >= 0 && O.inv) ? __ldg(O.inv + u[j]) : u[j];
        }
#pragma unroll
        for (int j = 0; j < XB; ++j) {
            if (u[j] < 0) continue;
            A.x[xo[j] + u[j]] = 0.0;
            if (at[j] < O.xcap) {
                O.xnodes[at[j]] = id[j];
                O.xvals[at[j]] = __dmul_rn(O.xscale, xv[j]);
            }
        }
    }
    if (blockIdx.x == 0) {
        for (int k = threadIdx.x; k < m; k += blockDim.x) {
            const int64_t si = seed_base + k;
            const int64_t pushes = (int64_t)A.s_pushes[k];
            const int64_t pc = pre[k + 1] - pre[k];
            O.sweeps[si] = (int64_t)A.s_last[k] + 1;
            O.ops[si] = (int64_t)A.s_ops[k];
            O.pushes[si] = pushes;
            O.conv[si] = A.s_conv[k];
            O.support[si] = O.hk ? -1 : (int64_t)A.touched[k] - (pushes - (int64_t)A.s_negz[k]);
            O.xoff[si] = A.slot_base[k];
            O.xcnt[si] = pc;
            O.amb[si] = A.s_amb[k];
            if (A.s_amb[k]) atomicAdd(O.amb_cnt, 1ULL);
            if (pc == 0) A.r[(int64_t)k * A.ld + A.seed[k]] = 0.0;  // inactive seed: r = alpha
        }
    }
}

// grid (CHUNKS, slots): return r of every slot to +0.0 -- zero exactly the
// 32 B sectors this slot ever wrote (sector map set on first touch) and clear
// the map (reset_sector_words, common.cuh).
__global__ void k_wave_reset(RoundArgs A) {
    const int k = blockIdx.y;
    const int64_t per = (A.smw + gridDim.x - 1) / gridDim.x;  // gridDim.x scales with the map
    const int64_t lo = blockIdx.x * per, hi = min(A.smw, lo + per);
    reset_sector_words(A.secmap + (int64_t)k * A.smw, A.r + (int64_t)k * A.ld, A.ld, lo, hi);
}

static void wave_reset(const RoundArgs &A, unsigned chunks, cudaStream_t st) {
    k_wave_reset<<<dim3(chunks, (unsigned)A.m), 256, 0, st>>>(A);
}

// (neighbour, degree) per arc, for the threshold test without a second load
__global__ void k_pack_cols(DevGraph g, int2 *__restrict__ colp) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < g.n_arcs;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = g.col[j];
        colp[j] = make_int2(v, g.deg[v]);
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

// ---- optional sparse r out (gd_batch_params.want_r) ----------------------
// r of a slot is nonzero only inside its touched 32 B sectors (sector map),
// so the reset walk doubles as the extraction: count the nonzero entries per
// (slot, chunk), reserve each slot's segment of the r pool, then emit (node,
// value) pairs and zero the sectors / clear the map in one more walk.
__global__ void k_r_count(const uint32_t *__restrict__ secmap, int64_t smw,
                          const double *__restrict__ r, int64_t ld,
                          unsigned long long *__restrict__ cnt) {
    __shared__ unsigned long long bsum;
    const int k = blockIdx.y;
    const int64_t per = (smw + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * per, hi = min(smw, lo + per);
    const uint32_t *map = secmap + (int64_t)k * smw;
    const double *rk = r + (int64_t)k * ld;
    if (threadIdx.x == 0) bsum = 0;
    __syncthreads();
    unsigned long long c = 0;
    for (int64_t w = lo + threadIdx.x; w < hi; w += blockDim.x) {
        uint32_t bits = map[w];
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int64_t i0 = (w * 32 + b) * 4;
            for (int q = 0; q < 4 && i0 + q < ld; ++q) c += rk[i0 + q] != 0.0;
        }
    }
    atomicAdd(&bsum, c);
    __syncthreads();
    if (threadIdx.x == 0) cnt[(int64_t)k * gridDim.x + blockIdx.x] = bsum;
}

// one thread per slot: chunk offsets (exclusive, in place) and the slot's
// segment of the pool
__global__ void k_r_reserve(int64_t m, int chunks, unsigned long long *__restrict__ cnt,
                            unsigned long long *__restrict__ cursor, int64_t seed_base,
                            int64_t *__restrict__ r_off, int64_t *__restrict__ r_cnt) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    unsigned long long run = 0;
    for (int c = 0; c < chunks; ++c) {
        const unsigned long long x = cnt[k * chunks + c];
        cnt[k * chunks + c] = run;
        run += x;
    }
    const unsigned long long base = atomicAdd(cursor, run);
    for (int c = 0; c < chunks; ++c) cnt[k * chunks + c] += base;
    r_off[seed_base + k] = (int64_t)base;
    r_cnt[seed_base + k] = (int64_t)run;
}

__global__ void k_r_emit(uint32_t *__restrict__ secmap, int64_t smw, double *__restrict__ r,
                         int64_t ld, const unsigned long long *__restrict__ cnt,
                         const int32_t *__restrict__ inv, int32_t *__restrict__ r_nodes,
                         double *__restrict__ r_vals, int64_t rcap) {
    __shared__ unsigned long long bpos;
    const int k = blockIdx.y;
    const int64_t per = (smw + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * per, hi = min(smw, lo + per);
    uint32_t *map = secmap + (int64_t)k * smw;
    double *rk = r + (int64_t)k * ld;
    if (threadIdx.x == 0) bpos = cnt[(int64_t)k * gridDim.x + blockIdx.x];
    __syncthreads();
    for (int64_t w = lo + threadIdx.x; w < hi; w += blockDim.x) {
        uint32_t bits = map[w];
        if (!bits) continue;
        map[w] = 0u;
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int64_t i0 = (w * 32 + b) * 4;
            for (int q = 0; q < 4 && i0 + q < ld; ++q) {
                const double v = rk[i0 + q];
                rk[i0 + q] = 0.0;
                if (v != 0.0) {
                    const unsigned long long at = atomicAdd(&bpos, 1ULL);
                    if ((int64_t)at < rcap) {
                        r_nodes[at] = inv ? inv[i0 + q] : (int32_t)(i0 + q);
                        r_vals[at] = v;
                    }
                }
            }
        }
    }
}

}  // namespace

// Sparse r of the m slots of a wave into the pool (and the slots' r back to
// +0.0, sector map cleared): replaces the reset of that wave.
void r_extract_wave(uint32_t *secmap, int64_t smw, double *r, int64_t ld, int64_t m,
                    const int32_t *inv, int64_t seed_base, unsigned long long *cnt_scratch,
                    unsigned long long *cursor, int64_t *r_off, int64_t *r_cnt,
                    int32_t *r_nodes, double *r_vals, int64_t rcap, cudaStream_t st) {
    const int64_t c = (smw + 2047) / 2048;
    const int chunks = (int)(c < 32 ? 32 : (c > 4096 ? 4096 : c));
    k_r_count<<<dim3(chunks, (unsigned)m), 256, 0, st>>>(secmap, smw, r, ld, cnt_scratch);
    k_r_reserve<<<(int)((m + 127) / 128), 128, 0, st>>>(m, chunks, cnt_scratch, cursor, seed_base,
                                                         r_off, r_cnt);
    k_r_emit<<<dim3(chunks, (unsigned)m), 256, 0, st>>>(secmap, smw, r, ld, cnt_scratch, inv,
                                                        r_nodes, r_vals, rcap);
    GD_LAUNCH_CHECK();
}

int r_extract_chunks(int64_t smw) {
    const int64_t c = (smw + 2047) / 2048;
    return (int)(c < 32 ? 32 : (c > 4096 ? 4096 : c));
}

}  // namespace gd

using namespace gd;

struct gd_batch {
    const gd_graph *G;      // caller's graph
    FifoBatchState *fifo = nullptr;  // GD_M_LOCAL_SOR state
    SignedState *sgn = nullptr;      // GD_M_LOCAL_CH state
    CtaState *cta = nullptr;         // GD_M_LOCAL_GD, small graphs: one CTA per seed
    SorWinState *sorwin = nullptr;   // GD_M_LOCAL_SOR in exact windows, one CTA per seed
    gd_graph *R = nullptr;  // degree-relabeled copy (when p.relabel)
    DBuf<int32_t> perm, inv;
    gd_batch_params p;
    int slots;
    int grid;
    int64_t fcap, xcap;
    DBuf<double> x, r, fcval;
    DBuf<int32_t> pushed, seed, s_last, s_conv, s_amb, overflow;
    DBuf<int32_t> amb;               // per seed: near-threshold flag of the last solve
    // streaming form of the round kernel (k_rounds<false, true>)
    bool stream = false;
    int sgrid = 0;                   // its cooperative grid
    int64_t cohort = 0;              // free slots that start new seeds together (0 = all)
    int32_t dbg = 0;                 // (experiments, GDIFF_DBG)
    int32_t resolve_workers = (int32_t)RESOLVE_WORKERS;
    bool host_stream = true;         // host entry copies finished waves' x during the solve
    DBuf<int32_t> s_idx, s_t0, t_state;
    DBuf<unsigned long long> sn, sctr;  // per slot entries [2][slots]; seed / done counters
    DBuf<int64_t> drain_cnt;
    DBuf<int64_t> nearkey;           // near list: 2 x NEAR_CAP keys + 2 counters
    DBuf<unsigned long long> nearcnt;
    static constexpr int64_t NEAR_CAP = 1 << 16;
    DBuf<unsigned long long> amb_cnt;
    int64_t last_amb = 0;            // seeds re-solved on the exact path
    DBuf<int64_t> lg_f, lg_ops;      // per-seed sweep logs (p.log_sweeps > 0)
    DBuf<double> lg_g;
    bool logs_on() const { return p.log_sweeps > 0 && p.method == GD_M_LOCAL_GD && !stream; }
    static constexpr size_t RESOLVE_WORKERS = 8;
    std::vector<ExactWorker *> workers;  // exact re-solve workers (created on demand)
    int64_t last_changed = 0;        // ... whose integer work the re-solve changed
    double last_resolve_ms = 0.0;    // host wall time of the re-solves
    DBuf<unsigned long long> touched, pushed_cnt, fctr, s_ops, s_pushes, s_negz, s_pvol, cursor;
    DBuf<int64_t> ukey, uarc, skey, sarc, frow, slot_base;
    DBuf<unsigned long long> scnt, sfill, cctr;
    int64_t sgroup = 1, group_min = 1 << 22;
    DBuf<int32_t> chunk_e;
    DBuf<int2> colp;
    int64_t ccap = 0;
    DBuf<int64_t> rlog;
    static constexpr int64_t RLOG_CAP = 4096;
    DBuf<uint32_t> secmap;
    int64_t smw = 0;
    bool hk = false;           // GD_M_HK: layered stage sweeps
    // optional sparse r output (want_r)
    DBuf<int64_t> roff, rcnt;
    DBuf<int32_t> rnodes;
    DBuf<double> rvals;
    DBuf<unsigned long long> rcursor, rscratch;
    int64_t rcap = 0, last_r_total = 0;
    bool want_r() const { return p.want_r != 0 && !hk; }
    RPool rpool() {
        return RPool{roff.p, rcnt.p, rnodes.p, rvals.p, rcap, rcursor.p, rscratch.p};
    }
    DBuf<double> r2, stage_w;  // (heat kernel) second residual layer, tau/(k+1)
    DBuf<double> cn;           // (heat kernel) dense stages: c per (node, slot)
    bool tma_on = false;       //   the pull stages its arc records by bulk async copy
    size_t kr_smem = 0;        // dynamic shared memory of the round kernel
    bool kr_tma() const { return hk && cn.p && tma_on; }
    int64_t heavy = 0;         //   nodes with >= HEAVY_DEG arcs (degree-sorted prefix)
    int64_t mid = 0;           //   ... with >= MEDIUM_DEG arcs
    DBuf<int64_t> hitem;       //   their row segments
    int64_t hitems = 0;
    DBuf<double> hacc;         //   partial sums per (heavy node, slot)
    DBuf<uint32_t> secmap2;
    // results
    DBuf<int64_t> sweeps, ops, pushes, support, xoff, xcnt;
    DBuf<int32_t> conv, xnodes;
    DBuf<double> xvals;
    std::vector<cudaEvent_t> ev;
    double last_ms = 0.0;
    int64_t last_launches = 0;
    int64_t last_x_total = 0;
    DBuf<int64_t> dseeds;  // host-entry staging of the seed list
    // Host entry (gd_batch_solve_host): the sparse x of wave w is copied to the
    // caller's buffers on a copy stream while wave w+1 runs (rounds mode).
    struct HostStream {
        int32_t *nodes = nullptr;
        double *vals = nullptr;
        int64_t cap = 0;        // caller's pairs
        int64_t streamed = 0;   // pairs [0, streamed) already queued on `cs`
        cudaStream_t cs = nullptr;
        unsigned long long *curh = nullptr;  // pinned: pool cursor after each wave
        int64_t curh_n = 0;
        std::vector<cudaEvent_t> wev;
    } hs;
    bool hs_on = false;

    const gd_graph *work() const { return R ? R : G; }
    // blocks per slot of the reset: ~2,048 map words (256 KB of r) per block
    unsigned reset_chunks() const {
        const int64_t c = (smw + 2047) / 2048;
        return (unsigned)(c < CHUNKS ? CHUNKS : (c > 4096 ? 4096 : c));
    }

    RoundArgs args() {
        RoundArgs A{};
        A.g = work()->view();
        A.beta = 1.0 - p.alpha;
        A.tcoeff = hk ? p.theta_coeff : p.eps * p.alpha;
        A.r2 = r2.p; A.secmap2 = secmap2.p; A.stage_w = stage_w.p;
        A.n_stages = hk ? p.n_stages : 0;
        A.n = G->n;
        A.ld = (G->n + 3) & ~3LL;
        A.max_sweeps = p.max_sweeps;
        A.fcap = fcap;
        A.x = x.p; A.r = r.p; A.pushed = pushed.p; A.seed = seed.p;
        A.touched = touched.p; A.pushed_cnt = pushed_cnt.p;
        A.ukey = ukey.p; A.skey = skey.p; A.sarc = sarc.p;
        A.scnt[0] = scnt.p; A.scnt[1] = scnt.p + slots; A.sfill = sfill.p; A.cctr = cctr.p;
        A.sgroup = sgroup;
        A.uarc = uarc.p;
        A.grouped = sgroup < slots ? 1 : 0;
        A.group_min = group_min;
        A.frow = frow.p; A.fcval = fcval.p; A.fctr = fctr.p;
        A.chunk_e = chunk_e.p; A.ccap = ccap;
        A.colp = colp.p;
        A.rlog = rlog.p; A.rlog_cap = RLOG_CAP;
        A.secmap = secmap.p; A.smw = smw;
        A.s_ops = s_ops.p; A.s_pushes = s_pushes.p; A.s_negz = s_negz.p; A.s_pvol = s_pvol.p;
        A.s_last = s_last.p; A.s_conv = s_conv.p; A.s_amb = s_amb.p;
        A.nearl = NearList{{nearkey.p, nearkey.p + NEAR_CAP}, {nearcnt.p, nearcnt.p + 1}, NEAR_CAP};
        if (logs_on()) {
            A.lg_f = lg_f.p; A.lg_ops = lg_ops.p; A.lg_g = lg_g.p; A.lg_cap = p.log_sweeps;
        }
        if (stream) {
            A.alpha = p.alpha;
            A.seed_ctr = sctr.p;
            A.done_ctr = sctr.p + 1;
            A.t_state = t_state.p;
            A.s_idx = s_idx.p;
            A.s_t0 = s_t0.p;
            A.sn[0] = sn.p;
            A.sn[1] = sn.p + slots;
            A.drain_cnt = drain_cnt.p;
            A.cohort = cohort > 0 ? cohort : slots;
            A.dbg = dbg;
            {   // sector-map reset units per finished slot: ~64 map words each
                const int64_t u = (smw + 63) / 64;
                A.reset_units = u < 256 ? 256 : (u > 16384 ? 16384 : u);
            }
        }
        A.dbg = dbg;
        A.cn = cn.p;
        A.tma = kr_tma() ? 1 : 0;
        A.heavy = heavy;
        A.mid = mid;
        A.hitem = hitem.p;
        A.hitems = hitems;
        A.hacc = hacc.p;
        if (tail_list.p && tail_on) {
            A.tail_list = tail_list.p;
            A.tail_cap = tail_cap;
            A.tail_c = tail_c.p;
            A.tail_state = tail_state.p;
            A.tail_p = tail_p;
            A.tail_f = tail_f;
        }
        A.overflow = overflow.p;
        A.perm = R ? perm.p : nullptr;
        A.cursor = cursor.p;
        A.slot_base = slot_base.p;
        return A;
    }
    // Queue the copy of wave w's pairs [cursor after w-1, cursor after w).
    void hs_drain(int64_t w) {
        GD_CUDA(cudaEventSynchronize(hs.wev[w]));
        int64_t end = (int64_t)hs.curh[w];
        const int64_t lim = hs.cap < xcap ? hs.cap : xcap;
        if (end > lim) end = lim;
        if (end > hs.streamed) {
            const int64_t k = end - hs.streamed;
            GD_CUDA(cudaMemcpyAsync(hs.nodes + hs.streamed, xnodes.p + hs.streamed,
                                    sizeof(int32_t) * k, cudaMemcpyDeviceToHost, hs.cs));
            GD_CUDA(cudaMemcpyAsync(hs.vals + hs.streamed, xvals.p + hs.streamed,
                                    sizeof(double) * k, cudaMemcpyDeviceToHost, hs.cs));
            hs.streamed = end;
        }
    }
    // Called after wave w is enqueued on st: record its cursor, drain wave w-1
    // (the GPU already holds wave w, so the host wait does not idle it).
    void hs_wave(int64_t w, int64_t waves, cudaStream_t st) {
        if (!hs_on) return;
        if (hs.curh_n < waves) {
            if (hs.curh) cudaFreeHost(hs.curh);
            GD_CUDA(cudaMallocHost(&hs.curh, sizeof(unsigned long long) * waves));
            hs.curh_n = waves;
        }
        while ((int64_t)hs.wev.size() < waves) {
            cudaEvent_t e;
            GD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            hs.wev.push_back(e);
        }
        GD_CUDA(cudaMemcpyAsync(hs.curh + w, cursor.p, sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, st));
        GD_CUDA(cudaEventRecord(hs.wev[w], st));
        if (w >= 1) hs_drain(w - 1);
        if (w == waves - 1) hs_drain(w);
    }
    // CTA-local wave tails (tail_sweeps): 2 x n int32 frontier lists and n c_u
    // per slot, allocated when they cost at most 4 GB (GDIFF_TAIL=0: off)
    DBuf<int32_t> tail_list;
    DBuf<double> tail_c;
    DBuf<int64_t> tail_state;
    int64_t tail_p = 1 << 14, tail_f = 1 << 13, tail_cap = 0;
    bool tail_on = false;            // (off for good after a list overflow)
    // two residual sets (see batch_run): r / secmap and r_alt / secmap_alt
    bool dbuf = false;
    DBuf<double> r_alt;
    DBuf<uint32_t> secmap_alt;
    cudaEvent_t ev_rs[2] = {nullptr, nullptr};  // set s reset on the second stream
    bool trace = false;              // GDIFF_WAVE_TRACE: per-wave timeline to stderr
    bool serial = false;             // GDIFF_WAVE_SERIAL: no second stream
    bool ext_bal = false;            // work-balanced x extraction
    int ext_blocks = 0;
    std::vector<cudaEvent_t> tev;
    cudaStream_t aux = nullptr;      // second stream of the wave transitions
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    ~gd_batch() {
        for (auto e : tev) cudaEventDestroy(e);
        if (ev_fork) cudaEventDestroy(ev_fork);
        for (auto e : ev_rs) if (e) cudaEventDestroy(e);
        if (ev_join) cudaEventDestroy(ev_join);
        if (aux) cudaStreamDestroy(aux);
        for (auto w : workers) exact_worker_destroy(w);
        if (hs.curh) cudaFreeHost(hs.curh);
        for (auto e : hs.wev) cudaEventDestroy(e);
        if (hs.cs) cudaStreamDestroy(hs.cs);
        for (auto e : ev) cudaEventDestroy(e);
        delete R;
        if (fifo) fifo_batch_destroy(fifo);
        if (sgn) signed_batch_destroy(sgn);
        if (cta) cta_batch_destroy(cta);
        if (sorwin) sorwin_destroy(sorwin);
    }
};

static void batch_run(gd_batch *B, const int64_t *d_seeds, int64_t n_seeds, cudaStream_t st) {
    const size_t ns = n_seeds ? (size_t)n_seeds : 1;
    B->sweeps.ensure(ns); B->ops.ensure(ns); B->pushes.ensure(ns); B->support.ensure(ns);
    B->xoff.ensure(ns); B->xcnt.ensure(ns); B->conv.ensure(ns); B->amb.ensure(ns);
    GD_CUDA(cudaMemsetAsync(B->cursor.p, 0, sizeof(unsigned long long), st));
    GD_CUDA(cudaMemsetAsync(B->amb_cnt.p, 0, sizeof(unsigned long long), st));
    if (B->logs_on()) {
        const size_t cells = ns * (size_t)B->p.log_sweeps;
        B->lg_f.ensure(cells); B->lg_ops.ensure(cells); B->lg_g.ensure(cells);
        GD_CUDA(cudaMemsetAsync(B->lg_f.p, 0, sizeof(int64_t) * cells, st));
        GD_CUDA(cudaMemsetAsync(B->lg_ops.p, 0, sizeof(int64_t) * cells, st));
        GD_CUDA(cudaMemsetAsync(B->lg_g.p, 0, sizeof(double) * cells, st));
    }
    B->hs.streamed = 0;
    RPool rp{};
    if (B->want_r()) {
        B->roff.ensure(ns); B->rcnt.ensure(ns);
        GD_CUDA(cudaMemsetAsync(B->rcursor.p, 0, sizeof(unsigned long long), st));
        rp = B->rpool();
    }
    const RPool *rpp = B->want_r() ? &rp : nullptr;
    GD_CUDA(cudaMemsetAsync(B->overflow.p, 0, sizeof(int32_t), st));
    if (B->fifo) {  // FIFO methods: one persistent launch, warps pull seeds
        if (B->ev.empty()) {
            cudaEvent_t e0, e1;
            GD_CUDA(cudaEventCreate(&e0));
            GD_CUDA(cudaEventCreate(&e1));
            B->ev.push_back(e0);
            B->ev.push_back(e1);
        }
        GD_CUDA(cudaMemsetAsync(B->support.p, 0xFF, sizeof(int64_t) * ns, st));  // not tracked
        // the FIFO replay is bit-exact: nothing is ever ambiguous
        GD_CUDA(cudaMemsetAsync(B->amb.p, 0, sizeof(int32_t) * ns, st));
        GD_CUDA(cudaEventRecord(B->ev[0], st));
        if (n_seeds && B->sorwin && !rpp)
            sorwin_run(B->sorwin, B->G, B->p, d_seeds, n_seeds, B->sweeps.p, B->ops.p,
                       B->pushes.p, B->conv.p, B->xoff.p, B->xcnt.p, B->xnodes.p, B->xvals.p,
                       B->xcap, B->cursor.p, st);
        else if (n_seeds)
            fifo_batch_run(B->fifo, B->G, B->p, d_seeds, n_seeds, B->sweeps.p, B->ops.p,
                           B->pushes.p, B->conv.p, B->xoff.p, B->xcnt.p, B->xnodes.p,
                           B->xvals.p, B->xcap, B->cursor.p, st, rpp);
        GD_CUDA(cudaEventRecord(B->ev[1], st));
        GD_CUDA(cudaStreamSynchronize(st));
        float f = 0.f;
        GD_CUDA(cudaEventElapsedTime(&f, B->ev[0], B->ev[1]));
        B->last_ms = f;
        B->last_launches = n_seeds ? 1 : 0;
        return;
    }
    if (B->cta) {  // one CTA per seed (batch_cta.cu): no waves, no grid barriers
        if (B->ev.size() < 2) {
            for (size_t i = B->ev.size(); i < 2; ++i) {
                cudaEvent_t e;
                GD_CUDA(cudaEventCreate(&e));
                B->ev.push_back(e);
            }
        }
        GD_CUDA(cudaEventRecord(B->ev[0], st));
        cta_batch_run(B->cta, B->work(), B->colp.p, B->p.alpha, B->p.eps, B->p.max_sweeps, d_seeds,
                      n_seeds, B->R ? B->perm.p : nullptr, B->R ? B->inv.p : nullptr, B->sweeps.p,
                      B->ops.p, B->pushes.p, B->support.p, B->conv.p, B->xoff.p, B->xcnt.p,
                      B->xnodes.p, B->xvals.p, B->xcap, B->cursor.p, B->amb.p, B->amb_cnt.p, st,
                      B->logs_on() ? B->lg_f.p : nullptr, B->lg_ops.p, B->lg_g.p,
                      B->p.log_sweeps);
        GD_CUDA(cudaEventRecord(B->ev[1], st));
        GD_CUDA(cudaStreamSynchronize(st));
        float f = 0.f;
        GD_CUDA(cudaEventElapsedTime(&f, B->ev[0], B->ev[1]));
        B->last_ms = f;
        B->last_launches = n_seeds ? 1 : 0;
        return;
    }
    if (B->sgn) {  // signed sweep-synchronous waves (batch_signed.cu)
        if (n_seeds == 0) {
            B->last_ms = 0.0;
            B->last_launches = 0;
            return;
        }
        signed_batch_run(B->sgn, B->work(), B->p, d_seeds, n_seeds, B->R ? B->perm.p : nullptr,
                         B->R ? B->inv.p : nullptr, B->sweeps.p, B->ops.p, B->pushes.p,
                         B->support.p, B->conv.p, B->xoff.p, B->xcnt.p, B->xnodes.p, B->xvals.p,
                         B->xcap, B->cursor.p, B->ev, &B->last_ms, &B->last_launches, st, rpp,
                         B->amb.p, B->amb_cnt.p);
        return;
    }
    const int64_t waves = (n_seeds + B->slots - 1) / B->slots;
    while ((int64_t)B->ev.size() < 2 * waves) {
        cudaEvent_t e;
        GD_CUDA(cudaEventCreate(&e));
        B->ev.push_back(e);
    }
    OutArgs O{B->sweeps.p, B->ops.p, B->pushes.p, B->support.p, B->xoff.p, B->xcnt.p,
              B->conv.p, B->xnodes.p, B->xvals.p, B->xcap, B->R ? B->inv.p : nullptr,
              B->hk ? std::exp(-B->p.tau) : 1.0, B->hk ? 1 : 0, B->amb.p, B->amb_cnt.p};
    int64_t launches = 0;
    if (B->stream && n_seeds > 0) {
        // one state for the whole solve; a launch per `slots` finished seeds
        RoundArgs A = B->args();
        A.m = n_seeds < B->slots ? n_seeds : B->slots;
        A.seeds = d_seeds;
        A.n_seeds = n_seeds;
        GD_CUDA(cudaMemsetAsync(B->fctr.p, 0, 2 * sizeof(unsigned long long), st));
        GD_CUDA(cudaMemsetAsync(B->scnt.p, 0, 2 * sizeof(unsigned long long) * B->slots, st));
        GD_CUDA(cudaMemsetAsync(B->nearcnt.p, 0, 2 * sizeof(unsigned long long), st));
        k_wave_init<<<(int)((A.m + 255) / 256), 256, 0, st>>>(A, d_seeds, B->p.alpha, 0, 0);
        GD_LAUNCH_CHECK();
        launches += 1;
        for (int64_t w = 0; w < waves; ++w) {
            A.seg_done = (w + 1) * B->slots < n_seeds ? (w + 1) * B->slots : n_seeds;
            GD_CUDA(cudaEventRecord(B->ev[2 * w], st));
            void *kargs[] = {&A, &O};
            GD_CUDA(cudaLaunchCooperativeKernel((const void *)k_rounds<false, true>,
                                                dim3(B->sgrid), dim3(BT), kargs,
                                                stage_bytes(B->slots), st));
            GD_CUDA(cudaEventRecord(B->ev[2 * w + 1], st));
            launches += 1;
            B->hs_wave(w, waves, st);
        }
    }
    if (!B->ext_blocks) {
        int per = 0;
        GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_wave_extract_bal, 256, 0));
        B->ext_blocks = std::max(1, per) * n_sms(B->G->device);
    }
    while (B->trace && (int64_t)B->tev.size() < 2 * waves) {
        cudaEvent_t e;
        GD_CUDA(cudaEventCreate(&e));
        B->tev.push_back(e);
    }
    if (!B->aux && !B->stream && waves > 0) {
        GD_CUDA(cudaStreamCreateWithFlags(&B->aux, cudaStreamNonBlocking));
        GD_CUDA(cudaEventCreateWithFlags(&B->ev_fork, cudaEventDisableTiming));
        GD_CUDA(cudaEventCreateWithFlags(&B->ev_join, cudaEventDisableTiming));
        GD_CUDA(cudaEventCreateWithFlags(&B->ev_rs[0], cudaEventDisableTiming));
        GD_CUDA(cudaEventCreateWithFlags(&B->ev_rs[1], cudaEventDisableTiming));
    }
    // two residual sets (dbuf): wave w runs on set w & 1 while wave w-1's set
    // is reset on the second stream beside wave w's CTA-local tail and x
    // extraction -- the part of a wave that leaves most SMs idle (the
    // cooperative round kernel itself leaves no room for another kernel)
    const bool dbuf = B->dbuf && !rpp && !B->hk && !B->stream;
    int64_t m_prev = 0;
    for (int64_t w = 0; w < waves && !B->stream; ++w) {
        const int64_t base = w * B->slots;
        RoundArgs A = B->args();
        A.m = n_seeds - base < B->slots ? n_seeds - base : B->slots;
        A.seed_base = base;
        const int set = dbuf ? (int)(w & 1) : 0;
        if (dbuf) {
            A.r = set ? B->r_alt.p : B->r.p;
            A.secmap = set ? B->secmap_alt.p : B->secmap.p;
            if (w >= 2) GD_CUDA(cudaStreamWaitEvent(st, B->ev_rs[set], 0));  // set is clean
        }
        const bool one = A.m <= 8 * 1024;  // init + counter zeroing in one block
        if (!one) {
            GD_CUDA(cudaMemsetAsync(B->fctr.p, 0, 2 * sizeof(unsigned long long), st));
            GD_CUDA(cudaMemsetAsync(B->scnt.p, 0, 2 * sizeof(unsigned long long) * B->slots, st));
            GD_CUDA(cudaMemsetAsync(B->nearcnt.p, 0, 2 * sizeof(unsigned long long), st));
            if (B->tail_on && !B->hk)  // (-1: no tail handed over)
                GD_CUDA(cudaMemsetAsync(B->tail_state.p, 0xFF, 2 * sizeof(int64_t), st));
        }
        A.tail_state = (B->tail_on && !B->hk) ? B->tail_state.p : nullptr;
        k_wave_init<<<one ? 1 : (int)((A.m + 255) / 256), 256, 0, st>>>(
            A, d_seeds + base, B->hk ? 1.0 : B->p.alpha, one ? 1 : 0, 2 * (int64_t)B->slots);
        GD_LAUNCH_CHECK();
        GD_CUDA(cudaEventRecord(B->ev[2 * w], st));
        void *kargs[] = {&A, &O};
        const void *kfn = B->hk ? (const void *)k_rounds<true> : (const void *)k_rounds<false>;
        GD_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(B->grid), dim3(BT), kargs, B->kr_smem, st));
        if (dbuf && w >= 1) {  // wave w-1's set, beside this wave's tail and extraction
            RoundArgs Ap = A;
            Ap.r = set ? B->r.p : B->r_alt.p;
            Ap.secmap = set ? B->secmap.p : B->secmap_alt.p;
            Ap.m = m_prev;
            GD_CUDA(cudaEventRecord(B->ev_fork, st));
            GD_CUDA(cudaStreamWaitEvent(B->aux, B->ev_fork, 0));
            wave_reset(Ap, B->reset_chunks(), B->aux);
            GD_CUDA(cudaEventRecord(B->ev_rs[set ^ 1], B->aux));
            launches += 1;
        }
        if (B->tail_on && !B->hk) {
            k_tail<<<(unsigned)A.m, BT, 0, st>>>(A);
            launches += 1;
        }
        GD_CUDA(cudaEventRecord(B->ev[2 * w + 1], st));
        // x extraction (random gathers: latency-bound) on st.  Without a second
        // residual set the r reset (sector stores: bandwidth-bound) runs beside
        // it on the second stream (disjoint data) and the next wave waits for
        // both; with one (dbuf) this set is reset during the next wave's tail.
        const cudaStream_t tst = B->serial ? st : B->aux;
        if (!dbuf) {
        GD_CUDA(cudaEventRecord(B->ev_fork, st));
        GD_CUDA(cudaStreamWaitEvent(tst, B->ev_fork, 0));
        if (rpp)  // the r extraction zeroes the slots' r itself
            r_extract_wave(A.secmap, A.smw, A.r, A.ld, A.m, B->R ? B->inv.p : nullptr, base,
                           rp.scratch, rp.cursor, rp.off, rp.cnt, rp.nodes, rp.vals, rp.cap,
                           tst);
        else
            wave_reset(A, B->reset_chunks(), tst);
        if (B->hk) {  // the other residual layer
            RoundArgs A2 = A;
            A2.r = A.r2;
            A2.secmap = A.secmap2;
            wave_reset(A2, B->reset_chunks(), tst);
        }
        }
        if (B->trace && B->serial) GD_CUDA(cudaEventRecord(B->tev[2 * w + 1], st));
        if (B->ext_bal && A.m <= EXB_MAX_SLOTS)
            k_wave_extract_bal<<<B->ext_blocks, 256, 0, st>>>(A, O, base);
        else
            k_wave_extract<<<dim3(CHUNKS, (unsigned)A.m), 256, 0, st>>>(A, O, base);
        if (B->trace) {
            GD_CUDA(cudaEventRecord(B->tev[2 * w], st));
            if (!B->serial) GD_CUDA(cudaEventRecord(B->tev[2 * w + 1], tst));
        }
        if (!dbuf) {
            GD_CUDA(cudaEventRecord(B->ev_join, tst));
            GD_CUDA(cudaStreamWaitEvent(st, B->ev_join, 0));
        }
        GD_LAUNCH_CHECK();
        launches += B->hk ? 5 : (dbuf ? 3 : 4);
        B->hs_wave(w, waves, st);
        m_prev = A.m;
    }
    if (dbuf && waves > 0) {  // both sets clean on return: the last wave's here,
        RoundArgs A = B->args();  // the one before on the second stream
        const int set = (int)((waves - 1) & 1);
        A.r = set ? B->r_alt.p : B->r.p;
        A.secmap = set ? B->secmap_alt.p : B->secmap.p;
        A.m = m_prev;
        wave_reset(A, B->reset_chunks(), st);
        if (waves >= 2) GD_CUDA(cudaStreamWaitEvent(st, B->ev_rs[set ^ 1], 0));
        GD_LAUNCH_CHECK();
        launches += 1;
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
    if (B->trace && !B->stream) {
        for (int64_t w = 0; w < waves; ++w) {
            float f = 0.f, g = 0.f, ex = 0.f, rs = 0.f;
            GD_CUDA(cudaEventElapsedTime(&f, B->ev[2 * w], B->ev[2 * w + 1]));
            GD_CUDA(cudaEventElapsedTime(&ex, B->ev[2 * w + 1], B->tev[2 * w]));
            GD_CUDA(cudaEventElapsedTime(&rs, B->ev[2 * w + 1], B->tev[2 * w + 1]));
            if (w + 1 < waves) GD_CUDA(cudaEventElapsedTime(&g, B->ev[2 * w + 1], B->ev[2 * w + 2]));
            fprintf(stderr, "wave %lld kernel %.1f us, extract done +%.1f, reset done +%.1f, next "
                    "wave +%.1f us\n", (long long)w, 1e3 * f, 1e3 * ex, 1e3 * rs, 1e3 * g);
        }
    }
}

struct RebaseOp {
    int64_t base;
    __host__ __device__ int64_t operator()(int64_t v) const { return v - base; }
};
using RebaseIt = cub::TransformInputIterator<int64_t, RebaseOp, const int64_t *>;

// Degree-descending renumbering with sorted rows, on the device (setup).
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
    DBuf<int32_t> unsorted(G->n_arcs ? G->n_arcs : 1);
    k_remap_rows<<<blocks, 256>>>(g, B->inv.p, B->perm.p, R->row.p, unsorted.p);
    GD_LAUNCH_CHECK();
    // sort every row by new id: a warp's 32 consecutive arcs then target
    // nearby residual words (hubs are contiguous), so its atomics share
    // sectors.  CUB's segmented sort counts items in int: sort groups of
    // whole rows holding <= 2^30 arcs each, offsets rebased per group.
    std::vector<int64_t> hrow(n + 1);
    GD_CUDA(cudaMemcpy(hrow.data(), R->row.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost));
    const int64_t LIMIT = 1LL << 30;
    for (int64_t r0 = 0; r0 < n;) {
        int64_t r1 = r0 + 1;
        {  // largest r1 with arcs(r0, r1) <= LIMIT (at least one row)
            int64_t lo = r0 + 1, hi = n;
            while (lo < hi) {
                const int64_t mid = (lo + hi + 1) / 2;
                if (hrow[mid] - hrow[r0] <= LIMIT) lo = mid; else hi = mid - 1;
            }
            r1 = lo;
        }
        const int64_t base = hrow[r0], items = hrow[r1] - base;
        if (items > 0) {
            RebaseIt begin(R->row.p + r0, RebaseOp{base}), end(R->row.p + r0 + 1, RebaseOp{base});
            bytes = 0;
            cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, unsorted.p + base, R->col.p + base,
                                               (int)items, (int)(r1 - r0), begin, end);
            tmp.ensure(bytes ? bytes : 1);
            cub::DeviceSegmentedSort::SortKeys(tmp.p, bytes, unsorted.p + base, R->col.p + base,
                                               (int)items, (int)(r1 - r0), begin, end);
        }
        r0 = r1;
    }
    GD_CUDA(cudaDeviceSynchronize());
}

// ---- re-solve of ambiguous seeds on the bit-exact path --------------------
namespace gd {
namespace {

__global__ void k_count_nz(const double *__restrict__ v, int64_t n, unsigned long long *cnt) {
    unsigned long long c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        c += v[i] != 0.0;
    c = __reduce_add_sync(FULL, (unsigned)c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

// (node, scale * v) for every nonzero of v, appended at *cursor (any order)
__global__ void k_emit_nz(const double *__restrict__ v, int64_t n, double scale,
                          int32_t *__restrict__ nodes, double *__restrict__ vals,
                          unsigned long long *cursor) {
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        const double x = i < n ? v[i] : 0.0;
        const bool nz = x != 0.0;
        const unsigned am = __ballot_sync(FULL, nz);
        if (!am) continue;
        const int lane = threadIdx.x & 31;
        unsigned long long b = 0;
        if (lane == __ffs(am) - 1) b = atomicAdd(cursor, (unsigned long long)__popc(am));
        b = __shfl_sync(FULL, b, __ffs(am) - 1);
        if (nz) {
            const unsigned long long at = b + __popc(am & lanemask_lt());
            nodes[at] = (int32_t)i;
            vals[at] = __dmul_rn(scale, x);
        }
    }
}

}  // namespace

// grow a device pool to `cap` entries keeping its first `used`
template <class T>
static void grow_keep(DBuf<T> &b, size_t cap, size_t used) {
    GD_CUDA(cudaDeviceSynchronize());  // (emits of other workers into the old pool)
    DBuf<T> nb(cap);
    if (used) GD_CUDA(cudaMemcpy(nb.p, b.p, used * sizeof(T), cudaMemcpyDeviceToDevice));
    std::swap(b.p, nb.p);
    std::swap(b.n, nb.n);
}

}  // namespace gd

// The sweep-synchronous batches flag every seed with an update that landed
// within AMB_REL of its threshold (common.cuh): there the atomic scatter
// order could round the residual to the other side of theta than the
// reference's sequential fold.  Each flagged seed is solved again on the
// bit-exact path (exact.cu, the reference's own frontier order) and its
// per-seed results and sparse x / r segments are replaced -- so every seed's
// frontier sets, sweeps and operation counts are the reference's.
static void resolve_ambiguous(gd_batch *B, const int64_t *d_seeds, int64_t n_seeds,
                              cudaStream_t st) {
    unsigned long long cnt = 0;
    GD_CUDA(cudaMemcpy(&cnt, B->amb_cnt.p, sizeof(cnt), cudaMemcpyDeviceToHost));
    B->last_amb = (int64_t)cnt;
    B->last_changed = 0;
    B->last_resolve_ms = 0.0;
    const bool all = B->p.resolve == GD_RESOLVE_ALL;
    if (B->p.resolve == GD_RESOLVE_FLAG || (!cnt && !all) || B->hk || B->fifo)
        return;  // (heat kernel: reported, not re-solved)
    const auto t0 = std::chrono::steady_clock::now();
    GD_CUDA(cudaStreamSynchronize(st));
    std::vector<int32_t> amb(n_seeds);
    std::vector<int64_t> seeds(n_seeds), before(3 * n_seeds);
    GD_CUDA(cudaMemcpy(amb.data(), B->amb.p, sizeof(int32_t) * n_seeds, cudaMemcpyDeviceToHost));
    GD_CUDA(cudaMemcpy(seeds.data(), d_seeds, sizeof(int64_t) * n_seeds, cudaMemcpyDeviceToHost));
    GD_CUDA(cudaMemcpy(before.data(), B->sweeps.p, 8 * n_seeds, cudaMemcpyDeviceToHost));
    GD_CUDA(cudaMemcpy(before.data() + n_seeds, B->ops.p, 8 * n_seeds, cudaMemcpyDeviceToHost));
    GD_CUDA(cudaMemcpy(before.data() + 2 * n_seeds, B->pushes.p, 8 * n_seeds,
                       cudaMemcpyDeviceToHost));
    std::vector<int64_t> todo;
    for (int64_t i = 0; i < n_seeds; ++i)
        if (amb[i] || all) todo.push_back(i);
    const bool ch = B->p.method == GD_M_LOCAL_CH || B->p.method == GD_M_LOCAL_HB;
    const bool katz = B->p.problem == GD_P_KATZ;
    gd_operator op{};
    op.weight_rule = katz ? GD_W_CONST : GD_W_RW;
    op.theta_rule = GD_T_DEGREE;
    op.beta = katz ? B->p.alpha : 1.0 - B->p.alpha;
    op.theta_coeff = katz ? B->p.eps : B->p.eps * B->p.alpha;
    const double bval = katz ? 1.0 : B->p.alpha;
    const int64_t n = B->G->n;
    const int nb = 4 * n_sms(B->G->device);
    if (B->hs_on) GD_CUDA(cudaStreamSynchronize(B->hs.cs));  // pools may move
    // Work items: LocalGD seeds in chunks of K solved together on K graph
    // copies (exact_multi_solve: one sweep loop, the per-sweep launch and
    // sync overhead paid once per chunk); LocalCH seeds one at a time (its
    // divergence abort is per seed).  Items run on up to resolve_workers
    // workers (own buffers and stream each), overlapping on the device.
    // Workers and K are bounded by free HBM (a graph copy needs ~112 B per
    // node plus frontier-sized sort scratch); an out-of-memory failure frees
    // the workers' buffers and retries the unfinished seeds with half the
    // workers (then half the copies), down to one seed on one worker.
    const size_t per_copy = 112 * (size_t)(n ? n : 1);  // solver arrays per graph copy
    size_t fr = 0, hbm = 0;
    GD_CUDA(cudaMemGetInfo(&fr, &hbm));
    size_t K = 1, Tcap = (size_t)B->resolve_workers;
    if (!ch) {
        const size_t want = (todo.size() + Tcap - 1) / Tcap;
        K = std::min<size_t>(64, std::max<size_t>(16, want));
        const size_t by_mem = (fr / 2) / (per_copy * Tcap);
        K = std::min(K, std::max<size_t>(1, by_mem));
        K = std::min<size_t>(K, (size_t)((1LL << 31) - 1) / (size_t)(n ? n : 1));
        K = std::max<size_t>(1, std::min(K, todo.size()));
    }
    Tcap = std::min(Tcap, std::max<size_t>(1, (fr / 2) / (per_copy * K)));
    std::vector<char> done(todo.size(), 0), chg(todo.size(), 0);
    std::vector<size_t> pend;
    std::atomic<size_t> next{0};
    std::mutex mu;  // output pools, cursor and per-seed records
    std::atomic<int> err{GD_OK};
    std::string errmsg;
    size_t items = 0;
    auto work = [&](size_t w) {
        try {
            GD_CUDA(cudaSetDevice(B->G->device));
            ExactWorker *W = B->workers[w];
            const cudaStream_t ws = exact_worker_stream(W);
            struct { unsigned long long *p; } cnts{exact_worker_scratch(W)};
            for (;;) {
                const size_t it = next.fetch_add(1);
                if (it >= items || err.load() != GD_OK) break;
                const size_t j0 = it * K, j1 = std::min(pend.size(), j0 + K);
                // solve the item: copy c of the result = seed todo[pend[j0 + c]]
                std::vector<int64_t> sd, sw, op_, pu;
                std::vector<int32_t> cvv;
                const double *xb = nullptr, *rb = nullptr;
                for (size_t j = j0; j < j1; ++j) sd.push_back(seeds[todo[pend[j]]]);
                if (ch) {
                    const ExactSeed e = exact_seed_solve(W, B->G, &op, B->p.method, sd[0], bval,
                                                         B->p.mu, B->p.L, B->p.max_sweeps, false);
                    xb = e.x; rb = e.r;
                    sw.push_back(e.sweeps); op_.push_back(e.ops); pu.push_back(e.pushes);
                    cvv.push_back(e.converged);
                } else {
                    const ExactMulti e = exact_multi_solve(W, B->G, &op, sd.data(), (int)sd.size(),
                                                           bval, B->p.max_sweeps);
                    xb = e.x; rb = e.r;
                    sw = e.sweeps; op_ = e.ops; pu = e.pushes; cvv = e.conv;
                }
                for (size_t c = 0; c < sd.size(); ++c) {
                    const size_t q = pend[j0 + c];
                    const int64_t i = todo[q];
                    const double *ex = xb + (int64_t)c * n, *er = rb + (int64_t)c * n;
                    chg[q] = before[i] != sw[c] || before[n_seeds + i] != op_[c] ||
                             (!ch && before[2 * n_seeds + i] != pu[c]);
                    unsigned long long nz[2] = {0, 0};
                    GD_CUDA(cudaMemsetAsync(cnts.p, 0, 2 * sizeof(unsigned long long), ws));
                    k_count_nz<<<nb, 256, 0, ws>>>(ex, n, cnts.p);
                    k_count_nz<<<nb, 256, 0, ws>>>(er, n, cnts.p + 1);
                    GD_LAUNCH_CHECK();
                    GD_CUDA(cudaMemcpyAsync(nz, cnts.p, sizeof(nz), cudaMemcpyDeviceToHost, ws));
                    GD_CUDA(cudaStreamSynchronize(ws));
                    std::lock_guard<std::mutex> lk(mu);
                    const int64_t xb0 = B->last_x_total, xc = (int64_t)nz[0], sup = (int64_t)nz[1];
                    if (xb0 + xc > B->xcap) {
                        const int64_t cap = 2 * (xb0 + xc);
                        grow_keep(B->xnodes, (size_t)cap, (size_t)xb0);
                        grow_keep(B->xvals, (size_t)cap, (size_t)xb0);
                        B->xcap = cap;
                    }
                    unsigned long long c0 = (unsigned long long)xb0;
                    GD_CUDA(cudaMemcpyAsync(cnts.p, &c0, sizeof(c0), cudaMemcpyHostToDevice, ws));
                    k_emit_nz<<<nb, 256, 0, ws>>>(ex, n, 1.0, B->xnodes.p, B->xvals.p, cnts.p);
                    GD_LAUNCH_CHECK();
                    B->last_x_total = xb0 + xc;
                    const int64_t rec[6] = {sw[c], op_[c], pu[c], sup, xb0, xc};
                    const int32_t cv = cvv[c];
                    GD_CUDA(cudaMemcpyAsync(B->sweeps.p + i, &rec[0], 8, cudaMemcpyHostToDevice, ws));
                    GD_CUDA(cudaMemcpyAsync(B->ops.p + i, &rec[1], 8, cudaMemcpyHostToDevice, ws));
                    GD_CUDA(cudaMemcpyAsync(B->pushes.p + i, &rec[2], 8, cudaMemcpyHostToDevice, ws));
                    GD_CUDA(cudaMemcpyAsync(B->support.p + i, &rec[3], 8, cudaMemcpyHostToDevice, ws));
                    GD_CUDA(cudaMemcpyAsync(B->xoff.p + i, &rec[4], 8, cudaMemcpyHostToDevice, ws));
                    GD_CUDA(cudaMemcpyAsync(B->xcnt.p + i, &rec[5], 8, cudaMemcpyHostToDevice, ws));
                    GD_CUDA(cudaMemcpyAsync(B->conv.p + i, &cv, 4, cudaMemcpyHostToDevice, ws));
                    int64_t rr[2] = {0, 0};
                    if (B->want_r()) {
                        const int64_t rb0 = B->last_r_total;
                        if (rb0 + sup > B->rcap) {
                            const int64_t cap = 2 * (rb0 + sup);
                            grow_keep(B->rnodes, (size_t)cap, (size_t)rb0);
                            grow_keep(B->rvals, (size_t)cap, (size_t)rb0);
                            B->rcap = cap;
                        }
                        unsigned long long r0 = (unsigned long long)rb0;
                        GD_CUDA(cudaMemcpyAsync(cnts.p + 1, &r0, sizeof(r0), cudaMemcpyHostToDevice, ws));
                        k_emit_nz<<<nb, 256, 0, ws>>>(er, n, 1.0, B->rnodes.p, B->rvals.p, cnts.p + 1);
                        GD_LAUNCH_CHECK();
                        B->last_r_total = rb0 + sup;
                        rr[0] = rb0;
                        rr[1] = sup;
                        GD_CUDA(cudaMemcpyAsync(B->roff.p + i, &rr[0], 8, cudaMemcpyHostToDevice, ws));
                        GD_CUDA(cudaMemcpyAsync(B->rcnt.p + i, &rr[1], 8, cudaMemcpyHostToDevice, ws));
                    }
                    GD_CUDA(cudaStreamSynchronize(ws));  // (host records above go out of scope)
                    done[q] = 1;
                }
            }
        } catch (const Error &e) {
            std::lock_guard<std::mutex> lk(mu);
            errmsg = gd_last_error();
            err = e.code;
        } catch (...) {
            err = GD_ERR_CUDA;
        }
    };
    for (;;) {
        pend.clear();
        for (size_t q = 0; q < todo.size(); ++q)
            if (!done[q]) pend.push_back(q);
        if (pend.empty()) break;
        K = std::min(K, pend.size());
        items = (pend.size() + K - 1) / K;
        const size_t T = std::min(items, Tcap);
        while (B->workers.size() < T) B->workers.push_back(exact_worker_create());
        next = 0;
        err = GD_OK;
        std::vector<std::thread> th;
        for (size_t w = 1; w < T; ++w) th.emplace_back(work, w);
        work(0);
        for (auto &x : th) x.join();
        if (err.load() == GD_OK) continue;
        if (err.load() != GD_ERR_OOM || (T == 1 && K == 1)) {
            set_error("exact re-solve failed: %s", errmsg.c_str());
            throw Error{err.load()};
        }
        for (auto w : B->workers) exact_worker_destroy(w);  // free their buffers
        B->workers.clear();
        cudaGetLastError();
        if (T > 1) Tcap = T / 2;
        else K = std::max<size_t>(1, K / 2);
    }
    int64_t changed = 0;
    for (char c : chg) changed += c;
    B->last_changed = changed;
    const unsigned long long tot = (unsigned long long)B->last_x_total;
    GD_CUDA(cudaMemcpy(B->cursor.p, &tot, sizeof(tot), cudaMemcpyHostToDevice));
    B->last_resolve_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

extern "C" {

static int batch_create_once(const gd_graph *G, const gd_batch_params *p, gd_batch **out);

// Creation with an out-of-memory fallback: the slot count chosen from free
// HBM can still be too many once the other allocations are made (another
// solver, NCCL buffers, torch's cache); then halve the slots and retry.
int gd_batch_create(const gd_graph *G, const gd_batch_params *p, gd_batch **out) {
    int rc = batch_create_once(G, p, out);
    if (rc != GD_ERR_OOM || !p || !out) return rc;
    gd_batch_params q = *p;
    int slots = p->slots;
    if (slots <= 0) slots = 64;  // (the automatic choice is at most 64)
    for (slots /= 2; rc == GD_ERR_OOM && slots >= 1; slots /= 2) {
        cudaGetLastError();  // (clear the sticky-free allocation error)
        q.slots = slots;
        rc = batch_create_once(G, &q, out);
    }
    return rc;
}

static int batch_create_once(const gd_graph *G, const gd_batch_params *p, gd_batch **out) {
    return guarded([&] {
        GD_CHECK_ARG(G && p && out, "null pointer");
        GD_CHECK_ARG(p->method == GD_M_LOCAL_GD || p->method == GD_M_LOCAL_SOR ||
                         p->method == GD_M_LOCAL_CH || p->method == GD_M_LOCAL_HB ||
                         p->method == GD_M_HK,
                     "unknown batch method");
        GD_CHECK_ARG(p->method != GD_M_HK ||
                         (p->n_stages >= 0 && (p->stage_w || p->n_stages == 0) &&
                          p->theta_coeff > 0.0 && p->tau >= 0.0),
                     "heat kernel batches need tau >= 0, n_stages, stage_w, theta_coeff > 0");
        GD_CHECK_ARG(p->problem == GD_P_PPR ||
                         (p->problem == GD_P_KATZ &&
                          (p->method == GD_M_LOCAL_CH || p->method == GD_M_LOCAL_HB)),
                     "Katz batches need GD_M_LOCAL_CH or GD_M_LOCAL_HB");
        GD_CHECK_ARG(p->method != GD_M_LOCAL_SOR || (p->omega > 0.0 && p->omega <= 2.0),
                     "omega must be in (0, 2]");
        GD_CHECK_ARG(p->method == GD_M_HK ||
                         (p->alpha > 0.0 && (p->problem == GD_P_KATZ || p->alpha <= 1.0)),
                     "alpha must be in (0, 1]");
        GD_CHECK_ARG(p->method == GD_M_HK || p->eps > 0.0, "eps must be positive");
        GD_CHECK_ARG(G->n_arcs < (1LL << CNT_SHIFT), "too many arcs");
        GD_CUDA(cudaSetDevice(G->device));
        const int64_t n = G->n ? G->n : 1;
        const int64_t ld = (n + 3) & ~3LL;
        gd_batch *B = new gd_batch();
        try {
            B->G = G;
            B->p = *p;
            if (const char *e = getenv("GDIFF_RESOLVE_WORKERS"))  // (experiments)
                B->resolve_workers = atoi(e) < 1 ? 1 : atoi(e);
            B->host_stream = getenv("GDIFF_NO_STREAM") == nullptr;  // (A/B, read once)
            if (B->p.max_sweeps <= 0) B->p.max_sweeps = 1000000;
            if (p->want_r && p->method != GD_M_HK) {  // sparse r pool (per-slot scratch below)
                B->rcap = p->out_cap > 0 ? p->out_cap : (64LL << 20);
                B->rnodes.alloc(B->rcap);
                B->rvals.alloc(B->rcap);
                B->rcursor.alloc(1);
            }
            if (p->method == GD_M_LOCAL_SOR) {
                // exact FIFO replay needs the caller's CSR order: no relabeling
                B->fifo = fifo_batch_create(G, p->slots);
                B->slots = fifo_batch_slots(B->fifo);
                // exact windows, one CTA per seed (sor_win.cu), for the unsigned
                // push (omega <= 1): windows of ~80 pops beat the one-pop-at-a-time
                // warp chain (arxiv LocalGS eps=1e-6: 38.4 -> 24.0 ms per 1,024
                // seeds, cora 39.8 -> 11.0 ms per 50).  Signed SOR (omega > 1)
                // keeps adjacent nodes queued together, windows shrink to ~10 pops
                // and the warp chain wins (arxiv 214 vs 740 ms).  GDIFF_SOR_MODE=
                // win|warp forces either; not with want_r.
                // (the warp chain runs with the seed's state in shared memory when it
                // fits, k_fifo_smem: cora SOR(omega*) 15.2 -> 8.3 ms per 50 seeds;
                // for LocalGS the windows stay ahead, 11.1 vs 22.7 ms)
                bool use_win = p->omega <= 1.0;
                if (const char *e = getenv("GDIFF_SOR_MODE"))
                    use_win = strcmp(e, "win") == 0 ? true : (strcmp(e, "warp") == 0 ? false : use_win);
                if (use_win && !p->want_r) B->sorwin = sorwin_create(G, p->slots);
                B->cursor.alloc(1); B->overflow.alloc(1); B->amb_cnt.alloc(1);
                B->xcap = p->out_cap > 0 ? p->out_cap : (16LL << 20);
                B->xnodes.alloc(B->xcap); B->xvals.alloc(B->xcap);
                *out = B;
                return;
            }
            B->hk = p->method == GD_M_HK;
            if (p->relabel) build_relabeled(B);
            if (p->method == GD_M_LOCAL_CH || p->method == GD_M_LOCAL_HB) {
                if (B->p.mu == 0.0 && B->p.L == 0.0) {
                    GD_CHECK_ARG(p->problem == GD_P_PPR, "Katz batches need mu, L");
                    B->p.mu = p->alpha;
                    B->p.L = 2.0 - p->alpha;
                }
                GD_CHECK_ARG(B->p.mu < B->p.L, "need mu < L");
                if (p->max_sweeps <= 0) {  // the reference default (src/local_solvers.py:500)
                    const double gap = B->p.mu > 1e-12 ? B->p.mu : 1e-12;
                    const double inv = 1.0 / (p->eps > 1e-300 ? p->eps : 1e-300);
                    const int64_t d =
                        (int64_t)(10.0 * std::log(inv > 2.0 ? inv : 2.0) / gap);
                    B->p.max_sweeps = d > 1000 ? d : 1000;
                }
                int slots = p->slots;
                if (slots <= 0) {
                    size_t fr = 0, tot = 0;
                    GD_CUDA(cudaMemGetInfo(&fr, &tot));
                    const int64_t by_mem = (int64_t)(fr / 4) / (ld * 33);
                    // Katz seeds (alpha < 1/lambda) do little work each (products:
                    // ~26 K operations over ~110 sweeps), so a wave is bound by its
                    // slowest seed's sweep chain: more seeds per wave (products Katz
                    // 64 -> 512 slots: 8.4 K -> 10.8 K solves/s); PPR keeps 64
                    const int64_t cap = p->problem == GD_P_KATZ ? 512 : 64;
                    slots = (int)(by_mem < cap ? (by_mem < 1 ? 1 : by_mem) : cap);
                }
                if (slots > 2048) slots = 2048;
                B->slots = slots;
                { const int64_t ldr = (n + 3) & ~3LL, smwr = (ldr / 4 + 31) / 32;  // r extraction scratch
                  if (B->rcap) B->rscratch.alloc((size_t)B->slots * (size_t)r_extract_chunks(smwr)); }
                B->xcap = p->out_cap > 0 ? p->out_cap : (64LL << 20);
                B->cursor.alloc(1); B->overflow.alloc(1); B->amb_cnt.alloc(1);
                B->xnodes.alloc(B->xcap); B->xvals.alloc(B->xcap);
                B->sgn = signed_batch_create(B->work(), B->p, slots);
                *out = B;
                return;
            }
            B->colp.alloc(G->n_arcs + 2);  // (+2: bulk copies round their size up to 16 B)
            k_pack_cols<<<4 * n_sms(G->device), 256>>>(B->work()->view(), B->colp.p);
            GD_LAUNCH_CHECK();
            GD_CUDA(cudaDeviceSynchronize());
            if (B->R) B->R->col.release();  // the batch reads (neighbour, degree) pairs only
            int slots = p->slots;
            if (slots <= 0) {
                size_t fr = 0, tot = 0;
                GD_CUDA(cudaMemGetInfo(&fr, &tot));
                // 64 in flight measured best on the products shape (L2 reuse of
                // the hub block vs. barrier amortisation); fewer if memory-bound
                double frac = 0.7;  // share of free HBM for the slot vectors (papers100M:
                                    // 13 -> 29 slots, eps=1e-6 50.9 K -> 65.6 K solves/s)
                if (const char *e = getenv("GDIFF_SLOT_MEM")) frac = atof(e);  // experiments
                int64_t budget = (int64_t)((double)fr * frac);
                // what is allocated after this sizing, explicitly: frontier
                // arrays (6 x 8 B per entry, 64 M entries at most), chunk map
                // (4 B), the x pool and -- with want_r -- the r pool (12 B per
                // pair, 64 M at first); plus headroom for pool growth, the
                // exact re-solve workers and a multi-GPU gather on rank 0
                const int64_t fc_est = 64LL << 20;
                const int64_t fixed = fc_est * (48 + 4) + (64LL << 20) * 12 * (p->want_r ? 2 : 1);
                const int64_t keep = fixed + std::max<int64_t>(8LL << 30, (int64_t)(0.1 * (double)fr));
                if (budget > (int64_t)fr - keep) budget = (int64_t)fr - keep;
                if (budget < 0) budget = 0;
                int64_t by_mem = budget / (ld * (B->hk ? 28 : 20));
                // the heat kernel at large tau is effectively global: a stage's
                // frontier approaches n per seed, so bound slots * n as well
                if (B->hk && by_mem > (64LL << 20) / n) by_mem = (64LL << 20) / n;
                slots = (int)(by_mem < 64 ? (by_mem < 1 ? 1 : by_mem) : 64);
            }
            if (slots > 2048) slots = 2048;  // per-block slot counters live in shared memory
            B->slots = slots;
            { const int64_t ldr = (n + 3) & ~3LL, smwr = (ldr / 4 + 31) / 32;  // r extraction scratch
              if (B->rcap) B->rscratch.alloc((size_t)B->slots * (size_t)r_extract_chunks(smwr)); }
            int64_t fc = p->frontier_cap > 0 ? p->frontier_cap : (int64_t)slots * n;
            if (p->frontier_cap <= 0 && fc > (64LL << 20) && !B->hk) fc = 64LL << 20;
            B->fcap = fc;
            B->xcap = p->out_cap > 0 ? p->out_cap : (64LL << 20);
            const size_t sn = (size_t)slots * (size_t)ld;
            B->x.alloc(sn); B->r.alloc(sn);
            GD_CUDA(cudaMemset(B->x.p, 0, sizeof(double) * sn));
            GD_CUDA(cudaMemset(B->r.p, 0, sizeof(double) * sn));
            B->pushed.alloc(sn);
            B->seed.alloc(slots); B->touched.alloc(slots); B->pushed_cnt.alloc(slots);
            B->s_ops.alloc(slots); B->s_pushes.alloc(slots); B->s_negz.alloc(slots);
            B->s_pvol.alloc(slots); B->s_last.alloc(slots); B->s_conv.alloc(slots);
            B->s_amb.alloc(slots); B->amb_cnt.alloc(1);
            B->nearkey.alloc(2 * gd_batch::NEAR_CAP); B->nearcnt.alloc(2);
            B->slot_base.alloc(slots);
            B->fctr.alloc(2); B->cursor.alloc(1); B->overflow.alloc(1);
            B->ukey.alloc(fc); B->uarc.alloc(fc); B->skey.alloc(fc); B->sarc.alloc(fc);
            B->scnt.alloc(2 * (size_t)slots); B->sfill.alloc(slots); B->cctr.alloc(1);
            {  // slot groups of about 96 MB of residual vectors (see RoundArgs::sgroup,
               // ::grouped): all slots in one group = the ungrouped mode
                int64_t gsz = (96LL << 20) / (ld * 8);
                if (const char *e = getenv("GDIFF_SLOT_GROUP")) gsz = atoll(e);  // experiments
                B->sgroup = gsz < 1 ? 1 : (gsz > slots ? slots : gsz);
                if (const char *e = getenv("GDIFF_GROUP_MIN")) B->group_min = atoll(e);  // (tests)
            }
            B->frow.alloc(fc); B->fcval.alloc(fc);
            B->ccap = fc;  // chunks of 32 arcs per round: P/32 <= entries * avg degree / 32
            if (B->hk && p->frontier_cap <= 0) {  // global stages: up to slots * 2m arcs
                const int64_t cc = ((int64_t)slots * G->n_arcs + 31) / 32 + slots;
                if (cc > B->ccap) B->ccap = cc;
            }
            B->chunk_e.alloc(B->ccap);
            B->rlog.alloc(5 * gd_batch::RLOG_CAP + 1);  // (F, P, t0) per round, count, tB, nfin
            B->smw = (ld / 4 + 31) / 32;  // one bit per 4 doubles (32 B sector)
            B->secmap.alloc((size_t)slots * (size_t)B->smw);
            GD_CUDA(cudaMemset(B->secmap.p, 0, sizeof(uint32_t) * (size_t)slots * (size_t)B->smw));
            {   // second residual set: when it costs no slots (slots not bound by
                // memory) and 8 GB stay free (GDIFF_DBUF=0: off)
                const char *e = getenv("GDIFF_DBUF");
                bool want = !B->hk && !p->want_r && !(e && atoi(e) == 0);
                if (want && p->slots <= 0 && slots < 64) want = false;
                size_t fr = 0, tot = 0;
                GD_CUDA(cudaMemGetInfo(&fr, &tot));
                const size_t need = sn * sizeof(double) + (size_t)slots * B->smw * 4;
                if (want && fr > need + (8ULL << 30)) {
                    B->r_alt.alloc(sn);
                    GD_CUDA(cudaMemset(B->r_alt.p, 0, sizeof(double) * sn));
                    B->secmap_alt.alloc((size_t)slots * (size_t)B->smw);
                    GD_CUDA(cudaMemset(B->secmap_alt.p, 0,
                                       sizeof(uint32_t) * (size_t)slots * (size_t)B->smw));
                    B->dbuf = true;
                }
            }
            if (B->hk) {
                // dense stages (hk_pull): c per (node, slot), when it fits (GDIFF_HK_PULL=0: off)
                const char *e = getenv("GDIFF_HK_PULL");
                size_t fr = 0, tot = 0;
                GD_CUDA(cudaMemGetInfo(&fr, &tot));
                if (!(e && atoi(e) == 0) && fr > sn * 8 + (8ULL << 30)) {
                    B->cn.alloc(sn);
                    const char *tm = getenv("GDIFF_HK_TMA");  // (A/B: 0 = plain loads)
                    // staging pays when a stage re-reads the records for >= 3 slot chunks
                    // (arxiv, 64 slots: +2 %; products, 28 slots in 2 chunks: -1 %)
                    const bool reuse = (slots + HKC - 1) / HKC >= 3;
                    B->tma_on = (tm ? atoi(tm) != 0 : reuse) && B->R;  // (degree-sorted ids)
                    // heavy prefix: nodes with >= HEAVY_DEG arcs (ids sorted by degree
                    // when relabeled; otherwise none: lane per node everywhere)
                    if (B->R) {
                        std::vector<int32_t> deg((size_t)n);
                        GD_CUDA(cudaMemcpy(deg.data(), B->work()->view().deg, sizeof(int32_t) * n,
                                           cudaMemcpyDeviceToHost));
                        int64_t h = 0;
                        while (h < n && deg[(size_t)h] >= HEAVY_DEG) ++h;
                        B->heavy = h;
                        int64_t md = h;
                        while (md < n && deg[(size_t)md] >= MEDIUM_DEG) ++md;
                        B->mid = md;
                        std::vector<int64_t> items;
                        for (int64_t v = 0; v < h; ++v)
                            for (int64_t sg = 0; sg * (B->tma_on ? HSEG_TMA : HSEG) < deg[(size_t)v];
                                 ++sg)
                                items.push_back((v << 20) | sg);
                        B->hitem.alloc(items.size() ? items.size() : 1);
                        if (!items.empty())
                            GD_CUDA(cudaMemcpy(B->hitem.p, items.data(), 8 * items.size(),
                                               cudaMemcpyHostToDevice));
                        B->hitems = (int64_t)items.size();
                        B->hacc.alloc((size_t)(h ? h : 1) * (size_t)slots);
                        GD_CUDA(cudaMemset(B->hacc.p, 0, sizeof(double) * (size_t)(h ? h : 1) *
                                                             (size_t)slots));
                    }
                }
                B->r2.alloc(sn);
                GD_CUDA(cudaMemset(B->r2.p, 0, sizeof(double) * sn));
                B->secmap2.alloc((size_t)slots * (size_t)B->smw);
                GD_CUDA(cudaMemset(B->secmap2.p, 0,
                                   sizeof(uint32_t) * (size_t)slots * (size_t)B->smw));
                B->stage_w.alloc(p->n_stages ? p->n_stages : 1);
                if (p->n_stages)
                    GD_CUDA(cudaMemcpy(B->stage_w.p, p->stage_w, sizeof(double) * p->n_stages,
                                       cudaMemcpyHostToDevice));
                B->p.stage_w = nullptr;  // (the caller's array is not kept)
            }
            B->xnodes.alloc(B->xcap); B->xvals.alloc(B->xcap);
            {
                const char *e = getenv("GDIFF_TAIL");
                // lists of n entries per slot (a tail frontier can never exceed
                // them) when that costs <= 4 GB, else 1 M (huge graphs: a tail
                // frontier that outgrows them makes the solve rerun without tails)
                int64_t cap = (int64_t)n;
                if ((size_t)slots * (size_t)n * 16 > (4ULL << 30)) cap = std::min<int64_t>(n, 1 << 20);
                if (const char *v = getenv("GDIFF_TAIL_CAP")) cap = atoll(v);  // (tests)
                if (!B->hk && !(e && atoi(e) == 0) && cap > 0) {
                    B->tail_cap = cap;
                    B->tail_list.alloc(2 * (size_t)slots * (size_t)cap);
                    B->tail_c.alloc((size_t)slots * (size_t)cap);
                    B->tail_state.alloc(2);
                    B->tail_on = true;
                    if (const char *v = getenv("GDIFF_TAIL_P")) B->tail_p = atoll(v);  // (A/B)
                    if (const char *v = getenv("GDIFF_TAIL_F")) B->tail_f = atoll(v);
                }
            }
            const size_t smem = stage_bytes(slots) + (B->kr_tma() ? tma_bytes() : 0);
            B->kr_smem = smem;
            const void *kfn = B->hk ? (const void *)k_rounds<true> : (const void *)k_rounds<false>;
            GD_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
            int per_sm = 0;
            GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, BT, smem));
            GD_CHECK_ARG(per_sm > 0, "round kernel does not fit on an SM");
            B->grid = per_sm * n_sms(G->device);
            // streaming form (slots refilled in-kernel, LocalGD without sparse
            // r) only on request (GDIFF_STREAM=1, read here once): measured on
            // the products shape it loses to the synchronous waves (33.0 vs
            // 26.5 + 4.3 ms per 1,024 seeds) -- a wave's seeds reach their big
            // round together, and that round (~100 M arcs) keeps each slot's
            // residual sectors hot in L2 far better than streamed rounds of
            // ~8 M arcs do
            B->stream = false;
            if (const char *e = getenv("GDIFF_STREAM"))
                B->stream = !B->hk && !B->want_r() && atoi(e) != 0;
            if (const char *e = getenv("GDIFF_COHORT")) B->cohort = atoll(e);  // (A/B)
            B->trace = getenv("GDIFF_WAVE_TRACE") != nullptr;   // (diagnostics: per-wave timeline)
            B->serial = getenv("GDIFF_WAVE_SERIAL") != nullptr; // (A/B: reset after extract on st)
            {   // GDIFF_EXTRACT_BAL=0: the per-slot extraction grid (A/B)
                const char *e = getenv("GDIFF_EXTRACT_BAL");
                B->ext_bal = !(e && atoi(e) == 0);
            }
            if (const char *e = getenv("GDIFF_DBG")) B->dbg = atoi(e);        // (experiments)
            if (B->stream) {
                const void *sfn = (const void *)k_rounds<false, true>;
                GD_CUDA(cudaFuncSetAttribute(sfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem));
                int ps = 0;
                GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, sfn, BT, smem));
                GD_CHECK_ARG(ps > 0, "streaming round kernel does not fit on an SM");
                B->sgrid = ps * n_sms(G->device);
                B->s_idx.alloc(slots); B->s_t0.alloc(slots); B->t_state.alloc(1);
                B->sn.alloc(2 * (size_t)slots); B->sctr.alloc(2); B->drain_cnt.alloc(slots);
            }
            if (!B->hk && !B->want_r() && p->frontier_cap <= 0) {
                // small graphs: sweeps scatter too few arcs to amortise two grid
                // barriers, so each seed runs in a CTA of its own (batch_cta.cu)
                bool use_cta = G->n <= CTA_MAX_N;
                if (const char *e = getenv("GDIFF_BATCH_MODE"))  // (tests, A/B)
                    use_cta = strcmp(e, "cta") == 0 ? true : (strcmp(e, "rounds") == 0 ? false : use_cta);
                if (use_cta) {
                    size_t fr = 0, tot = 0;
                    GD_CUDA(cudaMemGetInfo(&fr, &tot));
                    const int64_t per = cta_slot_bytes(G->n, G->n_arcs);
                    int64_t cap = (int64_t)(fr / 4) / per;
                    if (p->slots > 0 && p->slots < cap) cap = p->slots;
                    if (cap >= 1) B->cta = cta_batch_create(B->work(), (int)(cap < (1 << 20) ? cap : (1 << 20)));
                    if (B->cta) B->stream = false;  // (the round kernel is not used)
                }
            }
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
            if (ovf == 2 && B->tail_on) {  // a CTA-local tail outgrew its list: redo
                B->tail_on = false;        // the solve (the slots were reset) without
                if (B->hs_on) GD_CUDA(cudaStreamSynchronize(B->hs.cs));  // tails
                --attempt;
                continue;
            }
            if (ovf) {
                set_error("frontier capacity %lld (entries or arc chunks per round) exceeded; "
                          "raise frontier_cap",
                          (long long)B->fcap);
                throw Error{GD_ERR_CAPACITY};
            }
            res->x_total = (int64_t)used;
            B->last_x_total = (int64_t)used;
            unsigned long long rused = 0;
            if (B->want_r())
                GD_CUDA(cudaMemcpy(&rused, B->rcursor.p, sizeof(rused), cudaMemcpyDeviceToHost));
            B->last_r_total = (int64_t)rused;
            if ((int64_t)used <= B->xcap && (int64_t)rused <= B->rcap) break;
            GD_CHECK_ARG(attempt == 0, "output pool sizing failed");
            // grow (doubling, so a growing workload redoes at most log times) and redo;
            // host-entry copies still reading the old pool finish first
            if (B->hs_on) GD_CUDA(cudaStreamSynchronize(B->hs.cs));
            // new pools are allocated before the old ones go, and the
            // capacities change only once both exist: a failed grow (OOM)
            // leaves the handle consistent
            if ((int64_t)used > B->xcap) {
                const int64_t cap = 2 * (int64_t)used;
                DBuf<int32_t> nn(cap);
                DBuf<double> nv(cap);
                std::swap(B->xnodes.p, nn.p); std::swap(B->xnodes.n, nn.n);
                std::swap(B->xvals.p, nv.p); std::swap(B->xvals.n, nv.n);
                B->xcap = cap;
            }
            if ((int64_t)rused > B->rcap) {
                const int64_t cap = 2 * (int64_t)rused;
                DBuf<int32_t> nn(cap);
                DBuf<double> nv(cap);
                std::swap(B->rnodes.p, nn.p); std::swap(B->rnodes.n, nn.n);
                std::swap(B->rvals.p, nv.p); std::swap(B->rvals.n, nv.n);
                B->rcap = cap;
            }
        }
        resolve_ambiguous(B, d_seeds, n_seeds, st);
        res->x_total = B->last_x_total;
        res->sweeps = B->sweeps.p; res->total_ops = B->ops.p; res->pushes = B->pushes.p;
        res->support = B->support.p; res->converged = B->conv.p; res->x_offset = B->xoff.p;
        res->x_count = B->xcnt.p; res->x_nodes = B->xnodes.p; res->x_vals = B->xvals.p;
        res->kernel_launches = B->last_launches;
        res->ambiguous = B->amb.p;
        res->n_ambiguous = B->last_amb;
    });
}

// Copy the results of the last solve (still on the device) into host
// buffers; GD_ERR_CAPACITY with *x_total set when x_cap is too small, in
// which case the caller can grow its buffers and fetch again (no re-solve).
int gd_batch_fetch_host(gd_batch *B, int64_t n_seeds, int64_t *sweeps, int64_t *total_ops,
                        int64_t *pushes, int32_t *converged, int64_t *x_offset, int64_t *x_count,
                        int32_t *x_nodes, double *x_vals, int64_t x_cap, int64_t *x_total,
                        void *stream) {
    return guarded([&] {
        GD_CHECK_ARG(B && x_total, "null pointer");
        GD_CUDA(cudaSetDevice(B->G->device));
        cudaStream_t st = (cudaStream_t)stream;
        *x_total = B->last_x_total;
        auto d2h = [&](void *dst, const void *src, size_t bytes) {
            if (dst && bytes) GD_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
        };
        d2h(sweeps, B->sweeps.p, sizeof(int64_t) * n_seeds);
        d2h(total_ops, B->ops.p, sizeof(int64_t) * n_seeds);
        d2h(pushes, B->pushes.p, sizeof(int64_t) * n_seeds);
        d2h(converged, B->conv.p, sizeof(int32_t) * n_seeds);
        d2h(x_offset, B->xoff.p, sizeof(int64_t) * n_seeds);
        d2h(x_count, B->xcnt.p, sizeof(int64_t) * n_seeds);
        if (B->last_x_total > x_cap) {
            GD_CUDA(cudaStreamSynchronize(st));
            set_error("x buffers hold %lld pairs, %lld needed", (long long)x_cap,
                      (long long)B->last_x_total);
            throw Error{GD_ERR_CAPACITY};
        }
        // pairs the wave loop already queued on the copy stream (host entry)
        int64_t done = 0;
        if (B->hs_on && B->hs.nodes == x_nodes && B->hs.vals == x_vals) done = B->hs.streamed;
        if (done > B->last_x_total) done = B->last_x_total;
        d2h(x_nodes + done, B->xnodes.p + done, sizeof(int32_t) * (B->last_x_total - done));
        d2h(x_vals + done, B->xvals.p + done, sizeof(double) * (B->last_x_total - done));
        GD_CUDA(cudaStreamSynchronize(st));
        if (done) GD_CUDA(cudaStreamSynchronize(B->hs.cs));
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
        B->dseeds.ensure(n_seeds ? n_seeds : 1);
        GD_CUDA(cudaMemcpyAsync(B->dseeds.p, seeds, sizeof(int64_t) * n_seeds,
                                cudaMemcpyHostToDevice, st));
        gd_batch_result res{};
        if (x_nodes && x_vals && x_cap > 0 && B->host_stream) {  // stream finished waves' x to the host
            if (!B->hs.cs) GD_CUDA(cudaStreamCreateWithFlags(&B->hs.cs, cudaStreamNonBlocking));
            B->hs.nodes = x_nodes;
            B->hs.vals = x_vals;
            B->hs.cap = x_cap;
            B->hs_on = true;
        }
        int rc = gd_batch_solve_device(B, B->dseeds.p, n_seeds, &res, stream);
        if (rc == GD_OK)
            rc = gd_batch_fetch_host(B, n_seeds, sweeps, total_ops, pushes, converged, x_offset,
                                     x_count, x_nodes, x_vals, x_cap, x_total, stream);
        if (B->hs_on) {
            cudaStreamSynchronize(B->hs.cs);  // no copy may outlive the call
            B->hs_on = false;
            B->hs.nodes = nullptr;
            B->hs.vals = nullptr;
        }
        if (rc != GD_OK) throw Error{rc};
    });
}

int gd_batch_round_phase_log(const gd_batch *B, int64_t *out, int64_t cap) {
    return guarded([&] {
        GD_CHECK_ARG(B && out, "null pointer");
        GD_CHECK_ARG(B->rlog.p, "no round kernel");
        // cap entries of scatter-phase start ns, then cap of (streaming)
        // finished slots | refill << 32
        const int64_t k = cap / 2 < gd_batch::RLOG_CAP ? cap / 2 : gd_batch::RLOG_CAP;
        GD_CUDA(cudaMemcpy(out, B->rlog.p + 3 * gd_batch::RLOG_CAP + 1, sizeof(int64_t) * k,
                           cudaMemcpyDeviceToHost));
        GD_CUDA(cudaMemcpy(out + k, B->rlog.p + 4 * gd_batch::RLOG_CAP + 1, sizeof(int64_t) * k,
                           cudaMemcpyDeviceToHost));
    });
}

int gd_batch_round_log(const gd_batch *B, int64_t *out, int64_t cap, int64_t *rounds) {
    return guarded([&] {
        GD_CHECK_ARG(B && out && rounds, "null pointer");
        int64_t cnt = 0;
        GD_CUDA(cudaMemcpy(&cnt, B->rlog.p + 3 * gd_batch::RLOG_CAP, sizeof(int64_t),
                           cudaMemcpyDeviceToHost));
        *rounds = cnt;
        int64_t k = cnt < cap ? cnt : cap;
        if (k) GD_CUDA(cudaMemcpy(out, B->rlog.p, sizeof(int64_t) * 3 * k, cudaMemcpyDeviceToHost));
    });
}

int gd_batch_r_device(const gd_batch *B, int64_t **r_offset, int64_t **r_count, int32_t **r_nodes,
                      double **r_vals, int64_t *r_total) {
    if (!B || !r_offset || !r_count || !r_nodes || !r_vals || !r_total) return GD_ERR_ARG;
    if (!B->want_r()) {
        set_error("the batch was created without want_r");
        return GD_ERR_ARG;
    }
    *r_offset = B->roff.p;
    *r_count = B->rcnt.p;
    *r_nodes = B->rnodes.p;
    *r_vals = B->rvals.p;
    *r_total = B->last_r_total;
    return GD_OK;
}

int gd_batch_fetch_r_host(gd_batch *B, int64_t n_seeds, int64_t *r_offset, int64_t *r_count,
                          int32_t *r_nodes, double *r_vals, int64_t r_cap, int64_t *r_total,
                          void *stream) {
    return guarded([&] {
        GD_CHECK_ARG(B && r_total, "null pointer");
        GD_CHECK_ARG(B->want_r(), "the batch was created without want_r");
        GD_CUDA(cudaSetDevice(B->G->device));
        cudaStream_t st = (cudaStream_t)stream;
        *r_total = B->last_r_total;
        auto d2h = [&](void *dst, const void *src, size_t bytes) {
            if (dst && bytes) GD_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
        };
        d2h(r_offset, B->roff.p, sizeof(int64_t) * n_seeds);
        d2h(r_count, B->rcnt.p, sizeof(int64_t) * n_seeds);
        if (B->last_r_total > r_cap) {
            GD_CUDA(cudaStreamSynchronize(st));
            set_error("r buffers hold %lld pairs, %lld needed", (long long)r_cap,
                      (long long)B->last_r_total);
            throw Error{GD_ERR_CAPACITY};
        }
        d2h(r_nodes, B->rnodes.p, sizeof(int32_t) * B->last_r_total);
        d2h(r_vals, B->rvals.p, sizeof(double) * B->last_r_total);
        GD_CUDA(cudaStreamSynchronize(st));
    });
}

int gd_batch_last_ambiguous(const gd_batch *B, int64_t *count) {
    if (!B || !count) return GD_ERR_ARG;
    *count = B->last_amb;
    return GD_OK;
}

int gd_batch_logs(const gd_batch *B, int64_t n_seeds, int64_t *frontier_sizes, int64_t *vol_log,
                  double *pushed_mass) {
    return guarded([&] {
        GD_CHECK_ARG(B, "null pointer");
        GD_CHECK_ARG(B->logs_on(), "the batch records no sweep logs (log_sweeps, LocalGD)");
        const size_t cells = (size_t)n_seeds * (size_t)B->p.log_sweeps;
        GD_CHECK_ARG(cells <= B->lg_f.n, "n_seeds exceeds the last solve");
        if (frontier_sizes)
            GD_CUDA(cudaMemcpy(frontier_sizes, B->lg_f.p, 8 * cells, cudaMemcpyDeviceToHost));
        if (vol_log) GD_CUDA(cudaMemcpy(vol_log, B->lg_ops.p, 8 * cells, cudaMemcpyDeviceToHost));
        if (pushed_mass)
            GD_CUDA(cudaMemcpy(pushed_mass, B->lg_g.p, 8 * cells, cudaMemcpyDeviceToHost));
    });
}

int gd_batch_set_resolve(gd_batch *B, int32_t mode) {
    if (!B || mode < GD_RESOLVE_FLAG || mode > GD_RESOLVE_ALL) return GD_ERR_ARG;
    B->p.resolve = mode;
    return GD_OK;
}

int gd_batch_resolve_stats(const gd_batch *B, int64_t *flagged, int64_t *changed, double *ms) {
    if (!B || !flagged || !changed || !ms) return GD_ERR_ARG;
    *flagged = B->last_amb;
    *changed = B->last_changed;
    *ms = B->last_resolve_ms;
    return GD_OK;
}

int gd_batch_last_kernel_ms(const gd_batch *B, double *ms) {
    if (!B || !ms) return GD_ERR_ARG;
    *ms = B->last_ms;
    return GD_OK;
}

int gd_batch_info(const gd_batch *B, int32_t *mode, int64_t *slots) {
    if (!B || !mode || !slots) return GD_ERR_ARG;
    *mode = B->cta ? (cta_batch_smem(B->cta) ? GD_BATCH_CTA_SMEM : GD_BATCH_CTA)
                   : (B->sorwin ? GD_BATCH_FIFO_WIN
                                : (B->fifo ? GD_BATCH_FIFO
                                           : (B->stream ? GD_BATCH_STREAM : GD_BATCH_ROUNDS)));
    *slots = B->cta ? (int64_t)cta_batch_slots(B->cta) : (int64_t)B->slots;
    return GD_OK;
}

}  // extern "C"
