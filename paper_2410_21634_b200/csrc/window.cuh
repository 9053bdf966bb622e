// window.cuh -- exact FIFO push in windows, one CTA per system.
//
// The reference push (_push_kernel, src/local_solvers.py:48-188) pops one
// node at a time; a warp-per-system chain (fifo.cu's k_fifo) pays several
// dependent memory round trips per pop.  Here a CTA pops a WINDOW of queued
// nodes at once and still reproduces the sequential chain bit for bit:
//
//  * slice: up to WMAX queue entries from the front, never past the sweep's
//    sentinel, so every entry was queued before the window started;
//  * cut: pop i can join only if no earlier ACTIVE pop of the window pushes
//    to u_i (then r[u_i] at window start is exactly the r the sequential pop
//    would read).  Pops after the first such i wait for the next window;
//  * ordered fold: a node touched by several pops of the window receives its
//    contributions in pop order (records are placed per node by the rank of
//    the pop among the node's contributors, a bit mask per node), one thread
//    per node, with fl(r + fl(res * w)) exactly as the reference;
//  * enqueue order: each newly active node's queue slot comes from the key
//    (pop, arc position) of the contribution that first made it active --
//    the reference's enqueue order -- and a pop's self re-check (:176-185)
//    follows its own arcs.
// A pop whose row alone exceeds the window's arc budget runs as a window of
// one over the whole CTA.  Nodes that are popped and later pushed to inside
// the same window (a later pop reaching back) start their fold from the
// post-pop value, as the sequential chain sees them.
#pragma once

#include "common.cuh"

namespace gd {
namespace win {
namespace {

constexpr int WT = 1024;              // threads per system
constexpr int WMAX = 128;             // pops per window
constexpr int ACAP = 3072;            // arcs per window
constexpr int SCAP = ACAP + WMAX;     // distinct nodes per window
constexpr int HBITS = 13;
constexpr int HS = 1 << HBITS;        // hash entries
constexpr int KW = (SCAP + 31) / 32;  // enqueue-key bitmap words
constexpr int RPT = ACAP / WT;        // records per thread
constexpr int SPT = (SCAP + WT - 1) / WT;
constexpr int MW = WMAX / 32;         // contributor mask words per node
constexpr unsigned FULL = 0xffffffffu;

#ifdef GD_WIN_PROF
__device__ unsigned long long g_wprof[32];
#define WPROF(i)                                              \
    do {                                                      \
        if (threadIdx.x == 0) {                               \
            const long long now_ = clock64();                 \
            g_wprof[i] += (unsigned long long)(now_ - wlast); \
            wlast = now_;                                     \
        }                                                     \
    } while (0)
#else
#define WPROF(i) \
    do {         \
    } while (0)
#endif
static_assert(ACAP % WT == 0, "records per thread");

struct Smem {
    int32_t hk[HS];          // node id, -1 = empty
    int16_t hs[HS];          // slot of the entry
    uint8_t hpos[HS];        // slice position, 0xff = not in the slice
    int32_t slot_node[SCAP];
    int16_t slot_h[SCAP];
    int16_t slot_base[SCAP];
    uint32_t mask[SCAP][MW]; // contributing pops
    double delta[ACAP];      // fl(res_j * w) per record
    int16_t list[ACAP];      // records grouped per node, pop order
    uint8_t rec_j[ACAP];
    int32_t keynode[SCAP];
    uint32_t keybits[KW];
    uint32_t keypre[KW];
    double pr[WMAX], pth[WMAX], px[WMAX], pw[WMAX];
    int64_t prow[WMAX];
    int32_t pu[WMAX], pdeg[WMAX], pre[WMAX + 1], cpre[WMAX + 1];
    uint8_t pact[WMAX];
    int32_t wsum[WT / 32];
    int64_t front, rear, sentpos, svol, pushes;
    double sgamma;
    int nslice, jlim, cut, nslots, alloc, nenq, pos, neg;
};

struct Sys {
    DevGraph g;
    DevOp op;
    double *x, *r;
    int32_t *queue;
    uint32_t *qmark;
    int64_t qcap;
    double omega, gain;
    int sgn;
    int stats;  // accumulate sgamma / sign flags (the logs)
};

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Hash insert; *isnew when this call created the entry (its slot is given
// out by slot_alloc, warp-aggregated, after the probe loop reconverges).
__device__ __forceinline__ int h_insert(Smem &S, int32_t v, bool *isnew) {
    uint32_t h = ((uint32_t)v * 0x9E3779B1u) >> (32 - HBITS);
    for (;;) {
        const int32_t prev = atomicCAS(&S.hk[h], -1, v);
        if (prev == -1 || prev == v) {
            *isnew = prev == -1;
            return (int)h;
        }
        h = (h + 1) & (HS - 1);
    }
}

// Every lane of the warp calls; lanes with isnew get consecutive slots.
__device__ __forceinline__ void slot_alloc(Smem &S, bool isnew, int h, int32_t v) {
    const unsigned b = __ballot_sync(FULL, isnew);
    if (!b) return;
    const int lead = __ffs(b) - 1;
    int base = 0;
    if ((int)(threadIdx.x & 31) == lead) base = atomicAdd(&S.nslots, __popc(b));
    base = __shfl_sync(FULL, base, lead);
    if (isnew) {
        const int s = base + __popc(b & lanemask_lt());
        S.hs[h] = (int16_t)s;
        S.slot_node[s] = v;
        S.slot_h[s] = (int16_t)h;
    }
}

// One-time init of the shared tables (before the first window).
__device__ void init_smem(Smem &S) {
    for (int i = threadIdx.x; i < HS; i += WT) {
        S.hk[i] = -1;
        S.hpos[i] = 0xff;
    }
    for (int i = threadIdx.x; i < SCAP * MW; i += WT) (&S.mask[0][0])[i] = 0u;
    for (int i = threadIdx.x; i < KW; i += WT) S.keybits[i] = 0u;
}

__device__ __forceinline__ void pop_stats(const Sys &Y, Smem &S, int j) {
    const double ru = S.pr[j];
    S.svol += S.pdeg[j];
    S.pushes += 1;
    if (Y.stats) {
        S.sgamma = __dadd_rn(S.sgamma, fabs(ru));
        if (ru > 0.0) S.pos = 1;
        else if (ru < 0.0) S.neg = 1;
    }
}

// Thread 0: the next window's slice length and fresh per-window counters.
__device__ __forceinline__ void next_window(const Sys &Y, Smem &S) {
    const int64_t av = S.sentpos >= S.front ? S.sentpos - S.front : S.sentpos + Y.qcap - S.front;
    S.nslice = av < WMAX ? (int)av : WMAX;
    S.cut = WMAX;
    S.nslots = 0;
    S.alloc = 0;
}

// Slice entry 0 is active and its row exceeds ACAP: a window of one pop,
// its arcs in CTA-wide chunks, enqueue order by a CTA prefix over the chunk.
__device__ void big_pop(const Sys &Y, Smem &S) {
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int32_t u = S.pu[0];
    const double ru = S.pr[0];
    const double res = __dmul_rn(Y.omega, ru);
    const int32_t d = S.pdeg[0];
    const int64_t rs = S.prow[0];
    const int nslots = S.nslots;  // (thread 0 resets it at the end)
    if (t == 0) {
        atomicAnd(Y.qmark + (u >> 5), ~(1u << (u & 31)));
        Y.r[u] = __dsub_rn(ru, res);
        Y.x[u] = __dadd_rn(S.px[0], __dmul_rn(Y.gain, res));
        pop_stats(Y, S, 0);
    }
    __syncthreads();
    int64_t rear = S.rear;
    for (int64_t b = 0; b < d; b += WT) {
        const int64_t k = b + t;
        bool act = false;
        int32_t v = 0;
        if (k < d) {
            const int64_t a = rs + k;
            v = Y.g.col[a];
            const double w = arc_weight(Y.op, S.pw[0], a);
            const double old = Y.r[v];
            const uint32_t qm = Y.qmark[v >> 5];
            const double th = theta_of(Y.op, v, Y.g.deg[v]);
            const double rv = __dadd_rn(old, __dmul_rn(res, w));
            Y.r[v] = rv;
            act = !((qm >> (v & 31)) & 1u) && is_active(rv, th, Y.sgn);
        }
        const unsigned bal = __ballot_sync(FULL, act);
        if (lane == 0) S.wsum[wid] = __popc(bal);
        __syncthreads();
        int off = 0, tot = 0;
        for (int w2 = 0; w2 < WT / 32; w2++) {
            const int c = S.wsum[w2];
            off += w2 < wid ? c : 0;
            tot += c;
        }
        if (act) {
            int64_t p = rear + off + __popc(bal & lanemask_lt());
            if (p >= Y.qcap) p -= Y.qcap;
            Y.queue[p] = v;
            atomicOr(Y.qmark + (v >> 5), 1u << (v & 31));
        }
        rear += tot;
        if (rear >= Y.qcap) rear -= Y.qcap;
        __syncthreads();
    }
    for (int s = t; s < nslots; s += WT) {
        const int h = S.slot_h[s];
        S.hk[h] = -1;
        S.hpos[h] = 0xff;
    }
    if (t == 0) {
        const double ru2 = __dsub_rn(ru, res);
        if (is_active(ru2, S.pth[0], Y.sgn)) {
            Y.queue[rear] = u;
            atomicOr(Y.qmark + (u >> 5), 1u << (u & 31));
            rear = rear + 1 == Y.qcap ? 0 : rear + 1;
        }
        S.rear = rear;
        S.front = S.front + 1 == Y.qcap ? 0 : S.front + 1;
        next_window(Y, S);
    }
    __syncthreads();
}

// Warp-redundant prefix over the slice: lane l holds entries 4l..4l+3 (arcs
// of active pops, capped at ACAP + 1, and active-pop counts).  Returns jlim,
// the first pop whose arcs overflow the budget (or nslice).
__device__ __forceinline__ int slice_prefix(const Smem &S, int nslice, int lane, int (&pa)[4],
                                            int (&pc)[4], int &ta, int &tc) {
    int la[4], lc[4], sa = 0, sc = 0;
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int i = lane * 4 + q;
        const bool act = i < nslice && S.pact[i];
        const int l = act ? S.pdeg[i] : 0;
        la[q] = l > ACAP ? ACAP + 1 : l;
        lc[q] = act ? 1 : 0;
        sa += la[q];
        sc += lc[q];
    }
    int ia = sa, ic = sc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int ya = __shfl_up_sync(FULL, ia, o), yc = __shfl_up_sync(FULL, ic, o);
        if (lane >= o) {
            ia += ya;
            ic += yc;
        }
    }
    ta = __shfl_sync(FULL, ia, 31);
    tc = __shfl_sync(FULL, ic, 31);
    int ea = ia - sa, ec = ic - sc, first = WMAX;
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int i = lane * 4 + q;
        pa[q] = ea;
        pc[q] = ec;
        if (i < nslice && ea + la[q] > ACAP && first == WMAX) first = i;
        ea += la[q];
        ec += lc[q];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int y = __shfl_xor_sync(FULL, first, o);
        first = y < first ? y : first;
    }
    return first < nslice ? first : nslice;
}

// Pops every queue entry before the sweep's sentinel (S.sentpos), in windows.
// Entry: S.front / S.rear / S.sentpos set and visible to the CTA.
__device__ void run_sweep(const Sys &Y, Smem &S) {
    static_assert(WMAX == 128, "slice_prefix holds 4 entries per lane");
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int wbase = t & ~31;
#ifdef GD_WIN_PROF
    long long wlast = clock64();
    if (t == 0) g_wprof[31] += 1;
#endif
    if (t == 0) next_window(Y, S);
    __syncthreads();
    for (;;) {
        WPROF(0);
        const int nslice = S.nslice;
        if (nslice == 0) break;
        // ---- slice: the entries and their state at window start
        if (t < KW) S.keybits[t] = 0u;
        if (t < WMAX) {  // whole warps (slot_alloc)
            bool isnew = false;
            int h = 0;
            int32_t u = 0;
            if (t < nslice) {
                int64_t qi = S.front + t;
                if (qi >= Y.qcap) qi -= Y.qcap;
                u = Y.queue[qi];
                const double ru = Y.r[u];
                const int32_t d = Y.g.deg[u];
                const int64_t rs = Y.g.row[u];
                const double xu = Y.x[u];
                const double th = theta_of(Y.op, u, d);
                S.pu[t] = u;
                S.pr[t] = ru;
                S.pdeg[t] = d;
                S.prow[t] = rs;
                S.px[t] = xu;
                S.pth[t] = th;
                S.pw[t] = node_weight(Y.op, d);
                S.pact[t] = is_active(ru, th, Y.sgn) ? 1 : 0;
                h = h_insert(S, u, &isnew);
                S.hpos[h] = (uint8_t)t;
            }
            slot_alloc(S, isnew, h, u);
        }
        __syncthreads();
        WPROF(1);
        // ---- arc prefix (every warp computes it); the arc budget bounds the
        //      window; record -> pop map, warp w filling pops w, w+32, ...
        int pa[4], pc[4], ta, tc;
        const int jlim = slice_prefix(S, nslice, lane, pa, pc, ta, tc);
        if (jlim == 0) {
            big_pop(Y, S);
            continue;
        }
        if (wid == 0) {
#pragma unroll
            for (int q = 0; q < 4; q++) {
                S.pre[lane * 4 + q] = pa[q];
                S.cpre[lane * 4 + q] = pc[q];
            }
            if (lane == 0) {
                S.pre[WMAX] = ta;
                S.cpre[WMAX] = tc;
            }
        }
#pragma unroll
        for (int q4 = 0; q4 < 4; q4++) {  // pops j = wid + 32 q4; lane j / 4 holds pre[j]
            const int j = wid + 32 * q4, j1 = j + 1;
            int b = 0, e = ta;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const int v = __shfl_sync(FULL, pa[q], j >> 2);
                const int v1 = __shfl_sync(FULL, pa[q], (j1 >> 2) & 31);
                if (q == (j & 3)) b = v;
                if (j1 < WMAX && q == (j1 & 3)) e = v1;
            }
            if (j < jlim)
                for (int k = b + lane; k < e; k += 32) S.rec_j[k] = (uint8_t)j;
        }
        const int64_t rear = S.rear;  // (thread 0 moves it in the last phase)
        __syncthreads();
        WPROF(2);
        // ---- records: every arc of the pops before jlim; a pop is cut when
        //      an earlier active pop pushes to it
        const int narcs = S.pre[jlim];
        int32_t rv[RPT];
        double rw[RPT];
        int rh[RPT], rj[RPT];
#pragma unroll
        for (int q = 0; q < RPT; q++) {
            const int k = t + q * WT;
            rj[q] = -1;
            rv[q] = 0;
            if (k < narcs) {
                const int j = S.rec_j[k];
                const int64_t a = S.prow[j] + (k - S.pre[j]);
                rj[q] = j;
                rv[q] = Y.g.col[a];
                rw[q] = arc_weight(Y.op, S.pw[j], a);
            }
        }
#pragma unroll
        for (int q = 0; q < RPT; q++) {
            if (wbase + q * WT >= narcs) break;
            bool isnew = false;
            int h = 0;
            if (rj[q] >= 0) {
                h = h_insert(S, rv[q], &isnew);
                rh[q] = h;
                const int hp = S.hpos[h];
                if (hp != 0xff && hp > rj[q]) atomicMin(&S.cut, hp);
            }
            slot_alloc(S, isnew, h, rv[q]);
        }
        __syncthreads();
        WPROF(3);
        const int cut = S.cut < jlim ? S.cut : jlim;
        const int nvalid = S.pre[cut];
#ifdef GD_WIN_PROF
        if (t == 0) {
            g_wprof[20] += 1;
            g_wprof[21] += cut;
            g_wprof[22] += S.cut < jlim;          // conflict
            g_wprof[23] += jlim < nslice && S.cut >= jlim;  // arc budget
            g_wprof[24] += nslice;
            g_wprof[25] += nvalid;
        }
#endif
        const int nslots = S.nslots;
        // ---- contributor masks and deltas; each node's state at window start
#pragma unroll
        for (int q = 0; q < RPT; q++) {
            const int k = t + q * WT;
            if (k >= nvalid) continue;
            const int j = rj[q];
            const int s = S.hs[rh[q]];
            rh[q] = s;
            atomicOr(&S.mask[s][j >> 5], 1u << (j & 31));
            S.delta[k] = __dmul_rn(__dmul_rn(Y.omega, S.pr[j]), rw[q]);
        }
        double sval[SPT], sth[SPT];
        int sinfo[SPT];  // bit 0 marked, bits 8.. slice position (0xff none)
#pragma unroll
        for (int q = 0; q < SPT; q++) {
            const int s = t + q * WT;
            sinfo[q] = 0xff << 8;
            if (s >= nslots) continue;
            const int32_t v = S.slot_node[s];
            const int hp = S.hpos[S.slot_h[s]];
            if (hp == 0xff) {
                sval[q] = Y.r[v];
                sth[q] = theta_of(Y.op, v, Y.g.deg[v]);
                sinfo[q] = (int)((Y.qmark[v >> 5] >> (v & 31)) & 1u) | (0xff << 8);
            } else if (hp < cut) {  // popped: the post-pop value, mark cleared
                const double ru = S.pr[hp];
                sval[q] = S.pact[hp] ? __dsub_rn(ru, __dmul_rn(Y.omega, ru)) : ru;
                sth[q] = S.pth[hp];
                sinfo[q] = hp << 8;
            } else {                // still queued
                sval[q] = S.pr[hp];
                sth[q] = S.pth[hp];
                sinfo[q] = 1 | (hp << 8);
            }
        }
        __syncthreads();
        WPROF(4);
        // ---- per-node record ranges (warp-aggregated allocation)
        int scnt[SPT], sbase[SPT];
#pragma unroll
        for (int q = 0; q < SPT; q++) {
            scnt[q] = 0;
            sbase[q] = 0;
        }
#pragma unroll
        for (int q = 0; q < SPT; q++) {
            if (wbase + q * WT >= nslots) break;
            const int s = t + q * WT;
            int c = 0;
            if (s < nslots) {
#pragma unroll
                for (int w2 = 0; w2 < MW; w2++) c += __popc(S.mask[s][w2]);
            }
            scnt[q] = c;
            int inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(FULL, inc, o);
                if (lane >= o) inc += y;
            }
            int base = 0;
            if (lane == 31 && inc) base = atomicAdd(&S.alloc, inc);
            base = __shfl_sync(FULL, base, 31);
            sbase[q] = base + inc - c;
            if (c) S.slot_base[s] = (int16_t)sbase[q];
        }
        __syncthreads();
        WPROF(5);
#pragma unroll
        for (int q = 0; q < RPT; q++) {
            const int k = t + q * WT;
            if (k >= nvalid) continue;
            const int j = rj[q], s = rh[q];
            int below = __popc(S.mask[s][j >> 5] & ((1u << (j & 31)) - 1u));
#pragma unroll
            for (int w2 = 0; w2 < MW; w2++) below += w2 < (j >> 5) ? __popc(S.mask[s][w2]) : 0;
            S.list[S.slot_base[s] + below] = (int16_t)k;
        }
        __syncthreads();
        WPROF(6);
        // ---- ordered folds, write-back, first crossings
#pragma unroll
        for (int q = 0; q < SPT; q++) {
            const int s = t + q * WT;
            if (s >= nslots) continue;
            const int hp = sinfo[q] >> 8;
            const bool popped = hp < cut;
            const int c = scnt[q];
            if (!c && !popped) continue;
            const int32_t v = S.slot_node[s];
            const double th = sth[q];
            const int base = sbase[q];
            double val = sval[q];
            bool mark = sinfo[q] & 1;
            int i = 0;
            if (popped && S.pact[hp]) {
                // the pop's own arcs (a self loop: its record is the node's
                // first) precede its re-check (:176-185); later pops follow it
                if (c && ((S.mask[s][hp >> 5] >> (hp & 31)) & 1u)) {
                    const int k = S.list[base];
                    val = __dadd_rn(val, S.delta[k]);
                    if (is_active(val, th, Y.sgn)) {
                        mark = true;
                        const int key = k + hp;
                        atomicOr(&S.keybits[key >> 5], 1u << (key & 31));
                        S.keynode[key] = v;
                    }
                    i = 1;
                }
                if (is_active(sval[q], th, Y.sgn)) {
                    mark = true;
                    const int key = S.pre[hp + 1] + hp;
                    atomicOr(&S.keybits[key >> 5], 1u << (key & 31));
                    S.keynode[key] = v;
                }
            }
            for (; i < c; i++) {
                const int k = S.list[base + i];
                val = __dadd_rn(val, S.delta[k]);
                if (!mark && is_active(val, th, Y.sgn)) {
                    mark = true;
                    const int key = k + S.rec_j[k];
                    atomicOr(&S.keybits[key >> 5], 1u << (key & 31));
                    S.keynode[key] = v;
                }
            }
            if (c || (popped && S.pact[hp])) Y.r[v] = val;
            if (popped) {
                if (!mark) atomicAnd(Y.qmark + (v >> 5), ~(1u << (v & 31)));
            } else if (mark && !(sinfo[q] & 1)) {
                atomicOr(Y.qmark + (v >> 5), 1u << (v & 31));
            }
        }
        if (t < cut && S.pact[t]) {
            const double ru = S.pr[t];
            Y.x[S.pu[t]] = __dadd_rn(S.px[t], __dmul_rn(Y.gain, __dmul_rn(Y.omega, ru)));
            if (Y.stats) {
                if (ru > 0.0) S.pos = 1;
                else if (ru < 0.0) S.neg = 1;
            }
        }
        if (Y.stats && t == WT - 1) {  // the logs' ordered sum of |r| over the pushes
            double g = S.sgamma;
            for (int j = 0; j < cut; j++) g = __dadd_rn(g, S.pact[j] ? fabs(S.pr[j]) : 0.0);
            S.sgamma = g;
        }
        __syncthreads();
        WPROF(7);
        // ---- queue slots of the new entries: every warp scans the key bitmap
        //      (lane l holds words l, l + 32, ...; warp w places words w + 32 i)
        const int nkeys = nvalid + cut;
        const int nkw = (nkeys + 31) >> 5;
        constexpr int PER = (KW + 31) / 32;
        int kpre[PER];
        int run = 0;
#pragma unroll
        for (int q = 0; q < PER; q++) {
            const int w2 = q * 32 + lane;
            const int c = w2 < nkw ? __popc(S.keybits[w2]) : 0;
            int inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(FULL, inc, o);
                if (lane >= o) inc += y;
            }
            kpre[q] = run + inc - c;
            run += __shfl_sync(FULL, inc, 31);
        }
#pragma unroll
        for (int q = 0; q < PER; q++) {
            const int w2 = q * 32 + wid;  // this warp's word in block q
            const int wpre = __shfl_sync(FULL, kpre[q], wid);
            if (w2 >= nkw) continue;
            const uint32_t bits = S.keybits[w2];
            if (!((bits >> lane) & 1u)) continue;
            int64_t p = rear + wpre + __popc(bits & lanemask_lt());
            if (p >= Y.qcap) p -= Y.qcap;
            Y.queue[p] = S.keynode[w2 * 32 + lane];
        }
        for (int s = t; s < nslots; s += WT) {
            const int h = S.slot_h[s];
            S.hk[h] = -1;
            S.hpos[h] = 0xff;
#pragma unroll
            for (int w2 = 0; w2 < MW; w2++) S.mask[s][w2] = 0u;
        }
        if (t == 0) {
            int64_t r2 = rear + run;
            if (r2 >= Y.qcap) r2 -= Y.qcap;
            S.rear = r2;
            int64_t f2 = S.front + cut;
            if (f2 >= Y.qcap) f2 -= Y.qcap;
            S.front = f2;
            S.svol += nvalid;
            S.pushes += S.cpre[cut];
            next_window(Y, S);
        }
        __syncthreads();
    }
}

// CTA-ordered enqueue of the nodes u in [0, n) with is_active(r[u]) in index
// order (the reference's seeds = flatnonzero(...) path); returns the count.
__device__ int64_t scan_enqueue(const Sys &Y, Smem &S, int64_t n) {
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    int64_t rear = 0;
    for (int64_t b = 0; b < n; b += WT) {
        const int64_t u = b + t;
        bool act = false;
        if (u < n) act = is_active(Y.r[u], theta_of(Y.op, u, Y.g.deg[u]), Y.sgn);
        const unsigned bal = __ballot_sync(FULL, act);
        if (lane == 0) S.wsum[wid] = __popc(bal);
        __syncthreads();
        int off = 0, tot = 0;
        for (int w2 = 0; w2 < WT / 32; w2++) {
            const int c = S.wsum[w2];
            off += w2 < wid ? c : 0;
            tot += c;
        }
        if (act) {
            Y.queue[rear + off + __popc(bal & lanemask_lt())] = (int32_t)u;
            atomicOr(Y.qmark + (u >> 5), 1u << (u & 31));
        }
        rear += tot;
        __syncthreads();
    }
    return rear;
}

}  // namespace
}  // namespace win
}  // namespace gd
