// common.cuh -- shared device/host helpers of libgdiff (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <vector>
#include <new>

#include "../../include/gdiff.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libgdiff is built for sm_100a only"
#endif

namespace gd {

// ---------------------------------------------------------------- errors --
void set_error(const char *fmt, ...);

struct Error {
    int code;
};

#define GD_CUDA(call)                                                               \
    do {                                                                            \
        cudaError_t e_ = (call);                                                    \
        if (e_ != cudaSuccess) {                                                    \
            ::gd::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,             \
                            cudaGetErrorString(e_));                                \
            throw ::gd::Error{e_ == cudaErrorMemoryAllocation ? GD_ERR_OOM         \
                                                               : GD_ERR_CUDA};      \
        }                                                                           \
    } while (0)

#define GD_CHECK_ARG(cond, msg)                                                     \
    do {                                                                            \
        if (!(cond)) {                                                              \
            ::gd::set_error("invalid argument: %s", msg);                          \
            throw ::gd::Error{GD_ERR_ARG};                                          \
        }                                                                           \
    } while (0)

#define GD_LAUNCH_CHECK() GD_CUDA(cudaGetLastError())

// Run a C-ABI body, mapping exceptions to return codes.
template <class F>
int guarded(F &&f) {
    try {
        f();
        return GD_OK;
    } catch (const Error &e) {
        return e.code;
    } catch (const std::bad_alloc &) {
        set_error("host allocation failed");
        return GD_ERR_OOM;
    } catch (...) {
        set_error("unexpected exception");
        return GD_ERR_CUDA;
    }
}

// ----------------------------------------------------------- device memory --
template <class T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    ~DBuf() { release(); }
    void alloc(size_t count) {
        release();
        if (count) GD_CUDA(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void ensure(size_t count) {
        if (count > n) alloc(count);
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

// ------------------------------------------------------------------ graph --
// HBM layout: int64 row_ptr[n+1], int32 col[n_arcs] (n < 2^31), int32 deg[n].
// The degree array (4 B/node, 9.5 MB on the products shape) stays L2
// resident and serves every per-arc threshold test without touching row_ptr.
struct DevGraph {
    int64_t n;
    int64_t n_arcs;
    const int64_t *row;
    const int32_t *col;
    const int32_t *deg;
};

}  // namespace gd

struct gd_graph {
    int device;
    int64_t n, n_arcs, d_max;
    gd::DBuf<int64_t> row;
    gd::DBuf<int32_t> col;
    gd::DBuf<int32_t> deg;
    gd::DevGraph view() const { return gd::DevGraph{n, n_arcs, row.p, col.p, deg.p}; }
};

namespace gd {

// --------------------------------------------------------- operator rules --
// Device form of gd_operator (arrays already in HBM).
struct DevOp {
    int32_t wrule, trule;
    double beta, tcoeff;
    const double *arc_w;  // GD_W_ARC
    const double *theta;  // GD_T_ARRAY
};

// w for the arcs of node u with degree d (per-node rules).  Both roundings
// are explicit: fl(fl(1/d) * beta), exactly what src/systems.py:85-108 stores.
__device__ __forceinline__ double node_weight(const DevOp &op, int32_t d) {
    if (op.wrule == GD_W_CONST) return op.beta;
    return __dmul_rn(__ddiv_rn(1.0, (double)d), op.beta);
}

__device__ __forceinline__ double arc_weight(const DevOp &op, double wnode, int64_t j) {
    return op.wrule == GD_W_ARC ? op.arc_w[j] : wnode;
}

// theta_u = fl(coeff * d_u) for d_u > 0, +inf otherwise (src/systems.py:157-160).
__device__ __forceinline__ double theta_of(const DevOp &op, int64_t u, int32_t d) {
    if (op.trule == GD_T_ARRAY) return op.theta[u];
    return d > 0 ? __dmul_rn(op.tcoeff, (double)d) : __longlong_as_double(0x7ff0000000000000LL);
}

__device__ __forceinline__ bool is_active(double ru, double th, bool sgn) {
    return sgn ? (fabs(ru) >= th) : (ru >= th);
}

// ------------------------------------------------------------- host glue --
struct HostOp {
    DevOp dev;
    DBuf<double> arc_w, theta;
};
void upload_op(const gd_graph *g, const gd_operator *op, int64_t dim, HostOp &out,
               cudaStream_t s);

void report_alloc(gd_report *rep, int64_t cap);
void report_push_log(gd_report *rep, int64_t &cap, int64_t vol, double gamma, double l1,
                     int8_t sign, int64_t fsize);
void report_trace(gd_report *rep, int64_t &tcap, const int64_t *f, int64_t cnt);

// ------------------------------------------------------- checked builds --
// `python -m paper_2410_21634_b200.build --checked` compiles with
// -DGD_CHECKED into libgdiff_checked.so: every GD_DCHECK traps with a message
// on a failed index / state invariant (the bounds checks this pool allows in
// place of compute-sanitizer); the product build compiles them out.
#ifdef GD_CHECKED
#define GD_DCHECK(cond)                                                              \
    do {                                                                             \
        if (!(cond)) {                                                               \
            printf("GD_DCHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
            __trap();                                                                \
        }                                                                            \
    } while (0)
#else
#define GD_DCHECK(cond) \
    do {                \
    } while (0)
#endif

// ------------------------------------------------- near-threshold detector --
// Batched sweep-synchronous solvers scatter with fp64 atomics, so a residual
// is summed in another order than the reference's sequential fold
// (src/local_solvers.py:282-291) and may differ from it in the last bits.
// Frontier membership (r_v >= theta_v, :336-350) can then differ only when a
// residual lands within that rounding of its threshold.  Every batched update
// whose result lies within a relative AMB_REL of theta_v flags its seed
// "ambiguous"; flagged seeds are re-solved on the bit-exact path (exact.cu),
// so the batch's frontier sets, sweeps and operation counts are the
// reference's.  AMB_REL = 2^-36 (1.46e-11) covers the forward-error bound
// 2 k u (u = 2^-53) of k <= 2^16 reordered additions into one residual.
constexpr double AMB_REL = 1.4551915228366852e-11;  // 2^-36

// Sector-map reset of one slot's residual over map words [lo, hi): every set
// bit b of word w marks the 32 B sector of doubles [4(32w+b), 4(32w+b)+4)
// written since the last reset; zero those sectors and clear the words.  A
// dense word (>= 8 sectors) is stored by the whole warp, lane j taking bit j,
// so its stores are one coalesced run; a sparse word's few sectors are stored
// by its own lane (a warp-serial walk of sparse words would spend a warp
// iteration per word on one or two stores).
__device__ __forceinline__ void reset_sector_words(uint32_t *map, double *r, int64_t ld,
                                                   int64_t lo, int64_t hi) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double4 *r4 = reinterpret_cast<double4 *>(r);
    auto zero = [&](int64_t sec) {
        if (4 * sec + 3 < ld) {
            r4[sec] = make_double4(0.0, 0.0, 0.0, 0.0);
        } else {
            for (int64_t i = 4 * sec; i < ld; ++i) r[i] = 0.0;
        }
    };
    for (int64_t w0 = lo + warp * 32; w0 < hi; w0 += nw * 32) {
        const uint32_t mine = (w0 + lane < hi) ? map[w0 + lane] : 0u;
        const bool dense = __popc(mine) >= 8;
        unsigned any = __ballot_sync(0xffffffffu, dense);
        while (any) {
            const int src = __ffs(any) - 1;
            any &= any - 1;
            const uint32_t wb = __shfl_sync(0xffffffffu, mine, src);
            if ((wb >> lane) & 1u) zero((w0 + src) * 32 + lane);
        }
        if (!dense) {
            uint32_t b = mine;
            while (b) {
                const int j = __ffs(b) - 1;
                b &= b - 1;
                zero((w0 + lane) * 32 + j);
            }
        }
        if (mine) map[w0 + lane] = 0u;
    }
}

__device__ __forceinline__ bool near_theta(double v, double th) {
    return fabs(__dsub_rn(v, th)) <= AMB_REL * th;
}

// Only a residual's FINAL value of a round decides membership, and partial
// sums of a hub pass near theta all the time, so the detector tests final
// values: the frontier entries of the next round (final r >= theta) in their
// push phase, and -- for final values just below theta -- every update that
// lands in [theta (1 - AMB_REL), theta) is recorded as (slot, node) and
// re-read once the round is over (a later update may have moved it on).
struct NearList {
    int64_t *key[2];              // (slot << 32 | node), per round parity
    unsigned long long *cnt[2];
    int64_t cap;
};

__device__ __forceinline__ bool below_theta(double v, double th) {
    return v < th && near_theta(v, th);
}

__device__ __forceinline__ void near_record(const NearList &L, int par, int32_t k, int32_t v,
                                            int32_t *s_amb) {
    const unsigned long long i = atomicAdd(L.cnt[par], 1ULL);
    if (i < (unsigned long long)L.cap)
        L.key[par][i] = ((int64_t)k << 32) | (uint32_t)v;
    else
        s_amb[k] = 1;  // list full: flag conservatively
}

// Bit-exact single-seed solve on the device (exact.cu): LocalGD (method
// GD_M_LOCAL_GD, b = bval e_seed, frontier signed when sgn) or LocalCH
// (GD_M_LOCAL_CH, bounds mu < L), on a worker (own buffers, own non-blocking
// stream; one host thread per worker at a time).  x and r are left in the
// worker's device buffers (valid until its next solve), the stream idle.
struct ExactSeed {
    int64_t sweeps, ops, pushes;
    int32_t converged, diverged;
    const double *x, *r;
    int64_t n;
};
// Polyak heavy-ball coefficients (LocalHB; exact.cu)
void hb_coefficients(double mu, double L, double *eta, double *beta);

struct ExactWorker;
ExactWorker *exact_worker_create();
void exact_worker_destroy(ExactWorker *w);
cudaStream_t exact_worker_stream(ExactWorker *w);
unsigned long long *exact_worker_scratch(ExactWorker *w);  // 4 device words
ExactSeed exact_seed_solve(ExactWorker *w, const gd_graph *G, const gd_operator *op,
                           int32_t method, int64_t seed, double bval, double mu, double L,
                           int64_t max_sweeps, bool sgn);
// K LocalGD seeds (host array) in one bit-exact sweep loop over K disjoint
// copies of the graph: copy j's x, r at [j*n1, (j+1)*n1) of the worker's
// buffers, per-copy counts below.
struct ExactMulti {
    int64_t n1 = 0;
    int K = 0;
    const double *x = nullptr, *r = nullptr;
    std::vector<int64_t> sweeps, ops, pushes;
    std::vector<int32_t> conv;
};
ExactMulti exact_multi_solve(ExactWorker *w, const gd_graph *G, const gd_operator *op,
                             const int64_t *seeds, int K, double bval, int64_t max_sweeps);

inline int n_sms(int device) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    return v > 0 ? v : 148;
}

}  // namespace gd
