"""Device-resident graphs and operator descriptions for the C ABI."""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _lib as L

__all__ = ["DeviceGraph", "device_graph", "operator_for", "report_arrays"]


class DeviceGraph:
    """A gd_graph handle (int64 row_ptr + int32 col + int32 degree in HBM)."""

    def __init__(self, handle: int, n: int, n_arcs: int, d_max: int, device: int):
        self.handle = C.c_void_p(handle)
        self.n, self.n_arcs, self.d_max, self.device = n, n_arcs, d_max, device

    @classmethod
    def from_host(cls, g, device: int = 0) -> "DeviceGraph":
        lib = L.load()
        off = np.ascontiguousarray(g.offsets, dtype=np.int64)
        tg = np.ascontiguousarray(g.targets, dtype=np.int64)
        h = C.c_void_p()
        L.check(lib.gd_graph_create(int(g.n), L.ptr(off, C.c_int64), L.ptr(tg, C.c_int64),
                                    int(tg.shape[0]), device, C.byref(h)))
        return cls._wrap(h, device)

    @classmethod
    def from_device(cls, n: int, row_ptr, col, device: int = 0) -> "DeviceGraph":
        """From torch CUDA tensors (int64 row_ptr[n+1], int32 col[arcs])."""
        lib = L.load()
        h = C.c_void_p()
        L.check(lib.gd_graph_create_device(int(n), C.c_void_p(row_ptr.data_ptr()),
                                           C.c_void_p(col.data_ptr()), int(col.numel()), device,
                                           C.byref(h)))
        return cls._wrap(h, device)

    @classmethod
    def _wrap(cls, h, device):
        lib = L.load()
        n, a, d = C.c_int64(), C.c_int64(), C.c_int64()
        L.check(lib.gd_graph_info(h, C.byref(n), C.byref(a), C.byref(d)))
        return cls(h.value, n.value, a.value, d.value, device)

    def apply_events(self, events, out: "DeviceGraph | None" = None) -> "DeviceGraph":
        """Device graph with the event batch applied in order (on the device;
        same CSR as graph.apply_events).  ``out`` (a different graph) is
        overwritten in place, reusing its device buffers."""
        lib = L.load()
        kinds = np.array([1 if e.kind == "insert" else 0 for e in events], np.int32)
        us = np.array([e.u for e in events], np.int64)
        vs = np.array([e.v for e in events], np.int64)
        if out is not None:
            L.check(lib.gd_graph_apply_events_into(self.handle, L.ptr(kinds, C.c_int32),
                                                   L.ptr(us, C.c_int64), L.ptr(vs, C.c_int64),
                                                   len(events), out.handle))
            n, a, d = C.c_int64(), C.c_int64(), C.c_int64()
            L.check(lib.gd_graph_info(out.handle, C.byref(n), C.byref(a), C.byref(d)))
            out.n, out.n_arcs, out.d_max = n.value, a.value, d.value
            return out
        h = C.c_void_p()
        L.check(lib.gd_graph_apply_events(self.handle, L.ptr(kinds, C.c_int32), L.ptr(us, C.c_int64),
                                          L.ptr(vs, C.c_int64), len(events), C.byref(h)))
        return DeviceGraph._wrap(h, self.device)

    def to_host(self):
        """The graph in the reference layout (CsrGraph)."""
        from .graph import CsrGraph

        off = np.empty(self.n + 1, np.int64)
        tg = np.empty(self.n_arcs, np.int64)
        L.check(L.load().gd_graph_export(self.handle, L.ptr(off, C.c_int64), L.ptr(tg, C.c_int64)))
        return CsrGraph(n=self.n, offsets=off, targets=tg)

    def close(self):
        if self.handle and self.handle.value:
            L.load(require_gpu=False).gd_graph_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_cache: dict[int, DeviceGraph] = {}


def device_graph(g, device: int = 0) -> DeviceGraph:
    """Upload g once and keep it resident while g is alive."""
    if isinstance(g, DeviceGraph):
        return g
    key = id(g)
    dg = _cache.get(key)
    if dg is None or dg.n != g.n:
        dg = DeviceGraph.from_host(g, device)
        _cache[key] = dg
        weakref.finalize(g, _cache.pop, key, None)
    return dg


def operator_for(sys) -> tuple[L.Operator, list]:
    """gd_operator for a DiffusionSystem (ours or the reference's).

    Per-node rules are used whenever they reproduce the system's per-arc
    weights / thresholds bit for bit; otherwise the arrays are passed.
    """
    op = sys.op
    keep = []
    o = L.Operator()
    beta = float(op.beta)
    b_exp = float(getattr(op, "b_exp", getattr(sys, "beta_exp", 0.0)) or 0.0)
    if op.pkind == "adj":
        o.weight_rule, o.beta = L.GD_W_CONST, beta
    elif op.pkind == "rw" or (op.pkind == "gen" and b_exp == 0.0):
        o.weight_rule, o.beta = L.GD_W_RW, beta
    else:
        w = np.ascontiguousarray(op.arc_weights, dtype=np.float64)
        keep.append(w)
        o.weight_rule, o.arc_w = L.GD_W_ARC, L.ptr(w)
    if "arc_weights" in getattr(op, "__dataclass_fields__", {}) and o.weight_rule != L.GD_W_ARC:
        # a reference OperatorQ with a materialised array: use the rule only
        # if it is bitwise what the array holds
        g = sys.graph
        d = np.repeat(np.asarray(g.degrees, dtype=np.float64), np.asarray(g.degrees))
        rule = np.full(d.shape, beta) if o.weight_rule == L.GD_W_CONST else (1.0 / np.where(d > 0, d, 1.0)) * beta
        if not np.array_equal(np.asarray(op.arc_weights), rule):
            w = np.ascontiguousarray(op.arc_weights, dtype=np.float64)
            keep.append(w)
            o.weight_rule, o.arc_w = L.GD_W_ARC, L.ptr(w)
    coeff = getattr(sys, "theta_coeff", None)
    if coeff is not None and getattr(sys, "theta_power", 1.0) == 1.0 and sys.problem != "hk":
        o.theta_rule, o.theta_coeff = L.GD_T_DEGREE, float(coeff)
    else:
        th = np.ascontiguousarray(sys.theta, dtype=np.float64)
        keep.append(th)
        o.theta_rule, o.theta = L.GD_T_ARRAY, L.ptr(th)
    return o, keep


def report_arrays(rep: L.Report, with_trace: bool = False) -> dict:
    """Copy a gd_report into numpy arrays and free it."""
    k = int(rep.n_logs)

    def arr(p, cnt, dt):
        return np.ctypeslib.as_array(p, (cnt,)).astype(dt, copy=True) if cnt else np.empty(0, dt)

    out = {
        "converged": bool(rep.converged), "diverged": bool(rep.diverged),
        "sweeps": int(rep.sweeps), "total_ops": int(rep.total_ops), "pushes": int(rep.pushes),
        "min_residual": float(rep.min_residual), "support_size": int(rep.support_size),
        "vol_log": arr(rep.vol_log, k, np.int64), "gamma_log": arr(rep.gamma_log, k, np.float64),
        "l1_log": arr(rep.l1_log, k + 1, np.float64), "sign_log": arr(rep.sign_log, k, np.int8),
        "frontier_sizes": arr(rep.frontier_sizes, k, np.int64),
        "l2_log": arr(rep.l2_log, k + 1, np.float64),
    }
    if with_trace:
        flat = arr(rep.trace, int(rep.trace_len), np.int64)
        out["frontier_trace"] = np.split(flat, np.cumsum(out["frontier_sizes"])[:-1]) if k else []
    L.load(require_gpu=False).gd_report_free(C.byref(rep))
    return out
