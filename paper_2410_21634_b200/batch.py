"""Batched multi-seed local diffusion (new API; no reference counterpart).

A seed batch in the reference is a loop of ``local_gd`` calls, one system per
seed (src/cli.py:150-190).  ``BatchSolver`` solves thousands of PPR systems
per call on one GPU; per seed it returns what the reference's report holds
for integer work (sweeps, total_ops, pushes, converged, support size) plus x
as a sparse vector over the pushed nodes (x is zero elsewhere).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as gdl
from .device import DeviceGraph, device_graph

__all__ = ["BatchSolver", "BatchOutput", "local_gd_batch", "local_sor_batch", "local_ch_batch",
           "local_hb_batch", "local_hk_batch"]


def _host_array(count: int, dtype, pinned: bool) -> np.ndarray:
    """Host buffer; page-locked (via torch) when pinned, so copies are async DMA."""
    if not pinned:
        return np.empty(count, dtype)
    import torch

    tdt = {np.dtype(np.int64): torch.int64, np.dtype(np.int32): torch.int32,
           np.dtype(np.float64): torch.float64}[np.dtype(dtype)]
    return torch.empty(max(count, 1), dtype=tdt, pin_memory=True).numpy()[:count]


class _CudaView:
    """Expose a raw device pointer to torch via __cuda_array_interface__."""

    def __init__(self, ptr: int, shape: tuple, typestr: str):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


@dataclass
class BatchOutput:
    sweeps: np.ndarray
    total_ops: np.ndarray
    pushes: np.ndarray
    converged: np.ndarray
    x_offset: np.ndarray
    x_count: np.ndarray
    x_nodes: np.ndarray
    x_vals: np.ndarray
    r_offset: np.ndarray | None = None  # (want_r) final residual, sparse per seed
    r_count: np.ndarray | None = None
    r_nodes: np.ndarray | None = None
    r_vals: np.ndarray | None = None
    # (log_sweeps) per seed and sweep: |S_t|, vol(S_t), sum of pushed |r_u|
    frontier_sizes: np.ndarray | None = None
    vol_log: np.ndarray | None = None
    pushed_mass: np.ndarray | None = None
    alpha: float = 0.0
    eps: float = 0.0

    def report(self, i: int):
        """Seed i's LocalReport (src/reports.py:51-79) from the sweep logs:
        vol_log, gamma_log (pushed |r| / l1 before the sweep), the l1 trace
        (PPR: l1_0 = alpha, l1_{t+1} = l1_t - alpha * pushed |r|; the reference
        sums |r| over all nodes -- equal to rounding) and frontier_sizes in
        notes, as local_gd reports them (src/local_solvers.py:459-467)."""
        from .reports import LocalReport

        if self.frontier_sizes is None:
            raise ValueError("the solver was created without log_sweeps")
        k = int(self.sweeps[i])
        if k > self.frontier_sizes.shape[1]:
            raise ValueError(f"seed {i} ran {k} sweeps, only {self.frontier_sizes.shape[1]} logged")
        mass = self.pushed_mass[i, :k]
        l1 = [self.alpha]
        for g in mass:
            l1.append(l1[-1] - self.alpha * float(g))
        gamma = [float(g) / l if l > 0 else 0.0 for g, l in zip(mass, l1)]
        return LocalReport(
            method="local-gd", problem="ppr", converged=bool(self.converged[i]), sweeps=k,
            total_ops=int(self.total_ops[i]), eps=self.eps, residual_l1_trace=l1,
            gamma_log=gamma, vol_log=[int(v) for v in self.vol_log[i, :k]],
            notes={"parallel": False, "frontier_sizes": [int(v) for v in self.frontier_sizes[i, :k]],
                   "batched": True})

    def r_sparse(self, i: int) -> tuple[np.ndarray, np.ndarray]:
        if self.r_offset is None:
            raise ValueError("the solver was created without want_r")
        a, c = int(self.r_offset[i]), int(self.r_count[i])
        return self.r_nodes[a:a + c], self.r_vals[a:a + c]

    def r_dense(self, i: int, n: int) -> np.ndarray:
        r = np.zeros(n)
        nodes, vals = self.r_sparse(i)
        r[nodes] = vals
        return r

    def x_sparse(self, i: int) -> tuple[np.ndarray, np.ndarray]:
        a, c = int(self.x_offset[i]), int(self.x_count[i])
        return self.x_nodes[a:a + c], self.x_vals[a:a + c]

    def x_dense(self, i: int, n: int) -> np.ndarray:
        x = np.zeros(n)
        nodes, vals = self.x_sparse(i)
        x[nodes] = vals
        return x


class BatchSolver:
    """Solve (I - (1-alpha) A D^-1) x = alpha e_s for many seeds s.

    method "local-gd": sweep-synchronous LocalGD (frontier sets, sweeps and
    operation counts identical to the reference, x to 1e-9);
    method "local-sor": FIFO LocalSOR with relaxation omega (omega = 1:
    LocalGS), one warp per seed, bit-identical with the reference;
    method "local-ch": LocalCH (Chebyshev momentum, signed frontier) for
    problem "ppr" or "katz" ((I - alpha A) x = e_s; needs mu, L), frontier
    sets, sweeps and operation counts identical to the reference's
    local_ch(sys, mu, L), x to 1e-9.  ``support`` is not tracked for it."""

    def __init__(self, g, alpha: float, eps: float, slots: int = 0,
                 max_sweeps: int = 1_000_000, frontier_cap: int = 0, out_cap: int = 0,
                 device: int = 0, relabel: bool = True, method: str = "local-gd",
                 omega: float = 1.0, problem: str = "ppr", mu: float | None = None,
                 L: float | None = None, hk: dict | None = None, want_r: bool = False,
                 resolve: str = "flag", log_sweeps: int = 0):
        if method not in ("local-gd", "local-sor", "local-ch", "local-hb", "local-hk"):
            raise ValueError(f"unknown batch method {method!r}")
        if problem not in ("ppr", "katz") or (problem == "katz" and method not in ("local-ch", "local-hb")):
            raise ValueError("problem must be 'ppr', or 'katz' with method 'local-ch' / 'local-hb'")
        if resolve not in ("flag", "exact", "all"):
            raise ValueError("resolve must be 'flag', 'exact' or 'all'")
        if method == "local-hk" and not hk:
            raise ValueError("local-hk needs hk={tau, n_stages, stage_w, theta_coeff}")
        if method != "local-hk" and problem == "ppr" and not 0.0 < alpha <= 1.0:
            raise ValueError("alpha must be in (0, 1]")
        if problem == "katz" and not alpha > 0.0:
            raise ValueError("alpha must be positive")
        if method == "local-sor" and not 0.0 < omega <= 2.0:
            raise ValueError("omega must be in (0, 2]")
        if method in ("local-ch", "local-hb"):
            if (mu is None) != (L is None):
                raise ValueError("give both mu and L, or neither")
            if mu is None and problem == "katz":
                raise ValueError("Katz batches need mu, L (see local_ch_batch)")
            if mu is not None and not mu < L:
                raise ValueError(f"need mu < L, got mu={mu}, L={L}")
        self.method = method
        self.lib = gdl.load()
        self.graph = g if isinstance(g, DeviceGraph) else device_graph(g, device)
        self.alpha, self.eps = float(alpha), float(eps)
        mcode = {"local-gd": gdl.GD_M_LOCAL_GD, "local-sor": gdl.GD_M_LOCAL_SOR,
                 "local-ch": gdl.GD_M_LOCAL_CH, "local-hb": gdl.GD_M_LOCAL_HB,
                 "local-hk": gdl.GD_M_HK}[method]
        hk = hk or {}
        sw = np.ascontiguousarray(hk.get("stage_w", np.zeros(1)), dtype=np.float64)
        p = gdl.BatchParams(method=mcode, slots=int(slots), alpha=self.alpha, eps=self.eps,
                            max_sweeps=int(max_sweeps), frontier_cap=int(frontier_cap),
                            out_cap=int(out_cap), relabel=int(bool(relabel)),
                            problem=gdl.GD_P_KATZ if problem == "katz" else gdl.GD_P_PPR,
                            omega=float(omega), mu=float(mu or 0.0), L=float(L or 0.0),
                            tau=float(hk.get("tau", 0.0)), n_stages=int(hk.get("n_stages", 0)),
                            stage_w=gdl.ptr(sw), theta_coeff=float(hk.get("theta_coeff", 0.0)),
                            want_r=int(bool(want_r) and method != "local-hk"),
                            resolve={"flag": 0, "exact": 1, "all": 2}[resolve],
                            log_sweeps=int(log_sweeps) if method == "local-gd" else 0)
        self.log_sweeps = int(log_sweeps) if method == "local-gd" else 0
        self.want_r = bool(want_r) and method != "local-hk"
        h = C.c_void_p()
        gdl.check(self.lib.gd_batch_create(self.graph.handle, C.byref(p), C.byref(h)))
        self.handle = h
        self._last_total = 0

    def close(self):
        if self.handle and self.handle.value:
            self.lib.gd_batch_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def last_kernel_ms(self) -> float:
        ms = C.c_double()
        gdl.check(self.lib.gd_batch_last_kernel_ms(self.handle, C.byref(ms)))
        return ms.value

    @property
    def last_ambiguous(self) -> int:
        """Seeds of the last solve flagged by the near-threshold detector (an
        update within 2^-36 of its threshold) and re-solved bit-exactly."""
        c = C.c_int64()
        gdl.check(self.lib.gd_batch_last_ambiguous(self.handle, C.byref(c)))
        return int(c.value)

    def set_resolve(self, resolve: str) -> None:
        """Near-threshold policy for the next solves: "flag", "exact", "all"."""
        if resolve not in ("flag", "exact", "all"):
            raise ValueError("resolve must be 'flag', 'exact' or 'all'")
        gdl.check(self.lib.gd_batch_set_resolve(self.handle, {"flag": 0, "exact": 1, "all": 2}[resolve]))

    def resolve_stats(self) -> dict:
        """Near-threshold re-solves of the last solve: seeds flagged, seeds
        whose integer work the bit-exact re-solve changed, host ms spent."""
        f, c, ms = C.c_int64(), C.c_int64(), C.c_double()
        gdl.check(self.lib.gd_batch_resolve_stats(self.handle, C.byref(f), C.byref(c), C.byref(ms)))
        return {"flagged": int(f.value), "changed": int(c.value), "ms": float(ms.value)}

    @property
    def mode(self) -> str:
        """Execution form: "stream" (round kernel, slots refilled in-kernel:
        LocalGD without want_r), "rounds" (wave round kernel), "cta" (one CTA per
        seed, LocalGD on small graphs), "cta-smem" (the same with each seed's
        state in shared memory, graphs of up to ~6 K nodes), "fifo" (LocalSOR/GS,
        warp per seed) or "fifo-win" (LocalSOR/GS in exact windows, CTA per seed)."""
        m, s = C.c_int32(), C.c_int64()
        gdl.check(self.lib.gd_batch_info(self.handle, C.byref(m), C.byref(s)))
        return ("rounds", "cta", "fifo", "fifo-win", "stream", "cta-smem")[m.value]

    @property
    def slots(self) -> int:
        """Seeds in flight per wave (chosen from free HBM when slots=0)."""
        m, s = C.c_int32(), C.c_int64()
        gdl.check(self.lib.gd_batch_info(self.handle, C.byref(m), C.byref(s)))
        return int(s.value)

    def round_log(self) -> np.ndarray:
        """(rounds, 5) int64: frontier entries, arcs, device ns at round start
        and at the start of its scatter phase, finished slots (| refill << 32),
        for the last wave (streaming
        form: the whole solve) of the last solve (instrumentation)."""
        buf = np.zeros(3 * 4096, np.int64)
        cnt = C.c_int64()
        gdl.check(self.lib.gd_batch_round_log(self.handle, gdl.ptr(buf, C.c_int64), 4096,
                                              C.byref(cnt)))
        k = min(cnt.value, 4096)
        tb = np.zeros(2 * 4096, np.int64)
        gdl.check(self.lib.gd_batch_round_phase_log(self.handle, gdl.ptr(tb, C.c_int64), 2 * 4096))
        return np.concatenate([buf[:3 * k].reshape(-1, 3), tb[:k, None], tb[4096:4096 + k, None]],
                              axis=1)

    def solve_device(self, seeds, stream=None) -> dict:
        """seeds: CUDA int64 tensor.  Returns torch CUDA tensors (views of the
        solver's buffers, valid until the next solve)."""
        import torch

        seeds = seeds.to(dtype=torch.int64).contiguous()
        k = int(seeds.numel())
        res = gdl.BatchResult()
        st = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
        gdl.check(self.lib.gd_batch_solve_device(self.handle, C.c_void_p(seeds.data_ptr()), k,
                                                 C.byref(res), C.c_void_p(st)))

        def view(p, cnt, typestr):
            addr = C.cast(p, C.c_void_p).value
            return torch.as_tensor(_CudaView(addr, (cnt,), typestr), device="cuda")

        tot = int(res.x_total)
        return {
            "sweeps": view(res.sweeps, k, "<i8"), "total_ops": view(res.total_ops, k, "<i8"),
            "pushes": view(res.pushes, k, "<i8"), "support": view(res.support, k, "<i8"),
            "converged": view(res.converged, k, "<i4"), "x_offset": view(res.x_offset, k, "<i8"),
            "x_count": view(res.x_count, k, "<i8"), "x_nodes": view(res.x_nodes, max(tot, 1), "<i4")[:tot],
            "x_vals": view(res.x_vals, max(tot, 1), "<f8")[:tot], "x_total": tot,
            "kernel_launches": int(res.kernel_launches),
            "ambiguous": view(res.ambiguous, k, "<i4"), "n_ambiguous": int(res.n_ambiguous),
        }

    def solve(self, seeds, x_cap: int | None = None, stream=None, out: dict | None = None) -> BatchOutput:
        """Host path: seeds from host memory, results copied back to host.

        ``out`` may hold preallocated (pinned) numpy buffers to reuse."""
        sd = np.ascontiguousarray(seeds, dtype=np.int64)
        k = sd.shape[0]
        out = {} if out is None else out
        pinned = bool(out.get("pinned", False))
        if "sweeps" not in out or out["sweeps"].shape[0] < k:
            for name, dt in (("sweeps", np.int64), ("total_ops", np.int64), ("pushes", np.int64),
                             ("converged", np.int32), ("x_offset", np.int64), ("x_count", np.int64)):
                out[name] = _host_array(k, dt, pinned)
        # host x buffers: reused while they hold the previous solve's pairs; a new
        # (pinned: slow to allocate) pair of buffers gets 1.5x headroom
        have = out["x_nodes"].shape[0] if "x_nodes" in out else 0
        if x_cap is not None:
            cap = x_cap
        elif have >= self._last_total + 1024:
            cap = have
        else:
            cap = int(1.5 * self._last_total) + 1024
        st = 0
        if stream is not None:
            st = stream.cuda_stream

        def bufs():
            return (gdl.ptr(out["sweeps"], C.c_int64), gdl.ptr(out["total_ops"], C.c_int64),
                    gdl.ptr(out["pushes"], C.c_int64), gdl.ptr(out["converged"], C.c_int32),
                    gdl.ptr(out["x_offset"], C.c_int64), gdl.ptr(out["x_count"], C.c_int64),
                    gdl.ptr(out["x_nodes"], C.c_int32), gdl.ptr(out["x_vals"]),
                    int(out["x_nodes"].shape[0]))

        if "x_nodes" not in out or out["x_nodes"].shape[0] < cap:
            out["x_nodes"] = _host_array(cap, np.int32, pinned)
            out["x_vals"] = _host_array(cap, np.float64, pinned)
        tot = C.c_int64()
        rc = self.lib.gd_batch_solve_host(self.handle, gdl.ptr(sd, C.c_int64), k, *bufs(),
                                          C.byref(tot), C.c_void_p(st))
        if rc == gdl.GD_ERR_CAPACITY and tot.value > out["x_nodes"].shape[0]:
            # results are still on the device: grow the host buffers, fetch again
            cap = int(tot.value * 1.5) + 1024  # (pinned allocations are slow: grow ahead)
            out["x_nodes"] = _host_array(cap, np.int32, pinned)
            out["x_vals"] = _host_array(cap, np.float64, pinned)
            rc = self.lib.gd_batch_fetch_host(self.handle, k, *bufs(), C.byref(tot), C.c_void_p(st))
        gdl.check(rc)
        t = int(tot.value)
        self._last_total = t
        res = BatchOutput(out["sweeps"][:k], out["total_ops"][:k], out["pushes"][:k],
                          out["converged"][:k].astype(bool), out["x_offset"][:k],
                          out["x_count"][:k], out["x_nodes"][:t], out["x_vals"][:t])
        if self.log_sweeps:
            L = self.log_sweeps
            res.frontier_sizes = np.zeros((k, L), np.int64)
            res.vol_log = np.zeros((k, L), np.int64)
            res.pushed_mass = np.zeros((k, L))
            if k:
                gdl.check(self.lib.gd_batch_logs(self.handle, k, gdl.ptr(res.frontier_sizes, C.c_int64),
                                                 gdl.ptr(res.vol_log, C.c_int64),
                                                 gdl.ptr(res.pushed_mass)))
            res.alpha, res.eps = self.alpha, self.eps
        if self.want_r:
            roff, rcnt = np.empty(k, np.int64), np.empty(k, np.int64)
            rt = C.c_int64()
            cap = max(int(1.25 * getattr(self, "_last_rtotal", 0)) + 1024, 1024)
            for _ in range(2):
                rn, rv = np.empty(cap, np.int32), np.empty(cap)
                rc = self.lib.gd_batch_fetch_r_host(self.handle, k, gdl.ptr(roff, C.c_int64),
                                                    gdl.ptr(rcnt, C.c_int64), gdl.ptr(rn, C.c_int32),
                                                    gdl.ptr(rv), cap, C.byref(rt), C.c_void_p(st))
                if rc != gdl.GD_ERR_CAPACITY:
                    break
                cap = int(rt.value) + 1024
            gdl.check(rc)
            self._last_rtotal = int(rt.value)
            res.r_offset, res.r_count = roff, rcnt
            res.r_nodes, res.r_vals = rn[:rt.value], rv[:rt.value]
        return res



def _check_seeds(g, seeds) -> np.ndarray:
    deg = np.asarray(g.degrees)
    sd = np.asarray(seeds, dtype=np.int64)
    if sd.size and (sd.min() < 0 or sd.max() >= g.n):
        raise ValueError("seed out of range")
    if sd.size and np.any(deg[sd] < 1):
        raise ValueError("source must have at least one neighbor")
    return sd


def local_gd_batch(g, seeds, alpha: float, eps: float, slots: int = 0,
                   max_sweeps: int = 1_000_000, relabel: bool = True) -> BatchOutput:
    """Batched LocalGD-PPR over `seeds` (host in, host out)."""
    sd = _check_seeds(g, seeds)
    solver = BatchSolver(g, alpha, eps, slots=slots, max_sweeps=max_sweeps, relabel=relabel)
    try:
        return solver.solve(sd)
    finally:
        solver.close()


def local_sor_batch(g, seeds, alpha: float, eps: float, omega: float = 1.0, slots: int = 0,
                    max_sweeps: int = 1_000_000) -> BatchOutput:
    """Batched LocalSOR-PPR (omega = 1: LocalGS), bit-identical per seed with
    local_sor(make_ppr_system(g, alpha, s, eps), omega)."""
    sd = _check_seeds(g, seeds)
    solver = BatchSolver(g, alpha, eps, slots=slots, max_sweeps=max_sweeps, method="local-sor",
                         omega=omega)
    try:
        return solver.solve(sd)
    finally:
        solver.close()


def local_ch_batch(g, seeds, alpha: float, eps: float, problem: str = "ppr",
                   mu: float | None = None, L: float | None = None,
                   lam_hat: float | None = None, max_sweeps: int | None = None, slots: int = 0,
                   relabel: bool = True, method: str = "local-ch") -> BatchOutput:
    """Batched LocalCH over `seeds`: per seed the reference's
    local_ch(make_ppr_system(g, alpha, s, eps)) or, for problem "katz",
    local_ch(make_katz_system(g, alpha, s, eps)) with its default bounds
    (cheby_bounds, src/local_solvers.py:541-558; Katz from lam_hat, the
    spectral norm estimate, computed on the host when not given)."""
    import math

    sd = _check_seeds(g, seeds)
    if mu is None or L is None:
        if problem == "ppr":
            mu, L = alpha, 2.0 - alpha
        else:
            if lam_hat is None:
                from .graph import spectral_norm_estimate
                lam_hat = spectral_norm_estimate(g, iters=200, seed=0)
            lam = min(max(lam_hat, 1e-12), float(g.d_max))
            mu, L = 1.0 - alpha * lam, 1.0 + alpha * lam
    if max_sweeps is None:  # the reference default (src/local_solvers.py:500)
        gap = max(mu, 1e-12)
        max_sweeps = max(1000, int(10 * math.log(max(1.0 / max(eps, 1e-300), 2.0)) / gap))
    solver = BatchSolver(g, alpha, eps, slots=slots, max_sweeps=max_sweeps, method=method,
                         problem=problem, mu=mu, L=L, relabel=relabel)
    try:
        return solver.solve(sd)
    finally:
        solver.close()


def local_hb_batch(g, seeds, alpha: float, eps: float, **kw) -> BatchOutput:
    """Batched LocalHB (heavy-ball momentum: local_ch's loop with Polyak's
    stationary coefficients; no reference counterpart, restated in oracle/
    orc_local_hb): the arguments of local_ch_batch."""
    return local_ch_batch(g, seeds, alpha, eps, method="local-hb", **kw)


def hk_params(g, tau: float, eps: float, s: int = 0) -> dict:
    """Seed-independent part of make_hk_system (src/systems.py:269-301)."""
    from .systems import make_hk_system

    sys = make_hk_system(g, tau, int(s), eps)
    N = int(sys.op.stage_count)
    return {"tau": float(tau), "n_stages": N,
            "stage_w": np.asarray(sys.op.stage_weights if N else np.zeros(1), dtype=np.float64),
            "theta_coeff": float(sys.theta_coeff)}


def local_hk_batch(g, seeds, tau: float, eps: float, slots: int = 0, relabel: bool = True,
                   max_sweeps: int = 1_000_000) -> BatchOutput:
    """Batched heat kernel: per seed the reference's local_hk(g, tau, s, eps)
    (same sweeps and operation counts; x = f_hat to rounding), as layered
    stage sweeps over many seeds at once."""
    sd = _check_seeds(g, seeds)
    hk = hk_params(g, tau, eps, int(sd[0]) if sd.size else 0)
    solver = BatchSolver(g, 1.0, eps, slots=slots, max_sweeps=max_sweeps, method="local-hk",
                         relabel=relabel, hk=hk)
    try:
        return solver.solve(sd)
    finally:
        solver.close()
