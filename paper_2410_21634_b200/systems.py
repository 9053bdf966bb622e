"""Diffusion systems Q x = b (host side).

Restates the reference's problem builders (src/systems.py:43-322) with one
B200-driven change: the scatter operator is described by *rule*, not by a
materialised per-arc array.  For the operators the local solvers use,

  pkind "rw"  (PPR, heat kernel, dynamic pair): w_j = fl(fl(1/d_u) * beta)
  pkind "adj" (Katz):                           w_j = beta
  pkind "gen" with b_exp = 0:                   same as "rw"

every arc of node u carries the same weight, so the device computes it from
the degree (8 B per push instead of 8 B per arc, and no 990 MB array on the
products shape).  ``OperatorQ.arc_weights`` still materialises the
reference's array on demand, bit-identical to src/systems.py:85-108, for
oracles, dense checks and the general "sym"/"gen" operators.  Thresholds
follow the same idea: theta_u = fl(coeff * d_u) (inf at degree 0) is a rule
(`theta_coeff`), with the dense vector available as ``theta``.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "OperatorQ", "DiffusionSystem", "SystemError", "make_ppr_system",
    "make_katz_system", "default_katz_alpha", "make_hk_system",
    "make_generalized_system", "hk_stage_count", "hk_tail_bound",
    "hk_paper_bound", "dense_solve", "series_oracle", "theta_vector",
    "arc_weights_for",
]

_DENSE_GUARD = 2000


class SystemError(ValueError):
    """Invalid system construction or oracle precondition."""


def arc_weights_for(g, beta: float, pkind: str, b_exp: float = 0.0) -> np.ndarray:
    """Per-arc beta*P[t_j, src_j] exactly as the reference materialises it."""
    if pkind == "adj":
        return np.full(g.targets.shape[0], beta)
    expo = {"rw": 0.0, "sym": 0.5, "gen": b_exp}[pkind]
    d = g.degrees.astype(np.float64)
    d = np.where(d > 0, d, 1.0)
    src = np.repeat(np.arange(g.n, dtype=np.int64), g.degrees)
    w = 1.0 / (d[src] ** (1.0 - expo) * d[g.targets] ** expo)
    w = 1.0 * w
    w *= beta
    return w


def _p_max(g, pkind: str, b_exp: float) -> float:
    if pkind == "adj":
        return float(g.d_max)
    if g.n == 0:
        return 0.0
    expo = {"rw": 0.0, "sym": 0.5, "gen": b_exp}[pkind]
    if expo == 0.0:
        # column mass of A D^-1 is exactly d_u * (1/d_u)
        d = g.degrees.astype(np.float64)
        inv = np.where(d > 0, 1.0 / np.where(d > 0, d, 1.0), 0.0)
        colsum = np.zeros(g.n)
        np.add.at(colsum, np.repeat(np.arange(g.n), g.degrees), np.repeat(inv, g.degrees))
        return float(colsum.max())
    w = arc_weights_for(g, 1.0, pkind, b_exp)
    colsum = np.zeros(g.n)
    np.add.at(colsum, np.repeat(np.arange(g.n), g.degrees), w)
    return float(colsum.max())


@dataclass(frozen=True, eq=False)
class OperatorQ:
    """Q = I - beta * P, P given by ``pkind`` (rw | adj | sym | gen)."""

    graph: object
    beta: float
    pkind: str
    b_exp: float = 0.0
    stage_count: int = 0
    stage_weights: np.ndarray = field(default=None)
    _p_max: float | None = field(default=None, repr=False)
    _arc_cache: list = field(default_factory=list, repr=False)

    @property
    def node_rule(self) -> str | None:
        """'rw' / 'adj' when every arc of a node has one weight, else None."""
        if self.pkind == "adj":
            return "adj"
        if self.pkind == "rw" or (self.pkind == "gen" and self.b_exp == 0.0):
            return "rw"
        return None

    @property
    def arc_weights(self) -> np.ndarray:
        if not self._arc_cache:
            self._arc_cache.append(arc_weights_for(self.graph, self.beta, self.pkind, self.b_exp))
        return self._arc_cache[0]

    @property
    def p_max(self) -> float:
        if self._p_max is None:
            object.__setattr__(self, "_p_max", _p_max(self.graph, self.pkind, self.b_exp))
        return self._p_max

    @property
    def contraction_ok(self) -> bool:
        return bool(self.beta * self.p_max < 1.0)

    def propagate(self, x: np.ndarray) -> np.ndarray:
        g = self.graph
        src = np.repeat(np.arange(g.n, dtype=np.int64), g.degrees)
        out = np.zeros(g.n)
        np.add.at(out, g.targets, self.arc_weights * x[src])
        return out

    def apply(self, x: np.ndarray) -> np.ndarray:
        return x - self.propagate(x)

    def dense_matrix(self) -> np.ndarray:
        g = self.graph
        if g.n > _DENSE_GUARD:
            raise SystemError(f"dense matrix guard: n={g.n} > {_DENSE_GUARD}")
        q = np.eye(g.n)
        src = np.repeat(np.arange(g.n, dtype=np.int64), g.degrees)
        np.subtract.at(q, (g.targets, src), self.arc_weights)
        return q


def theta_vector(g, coeff: float, power: float = 1.0) -> np.ndarray:
    d = g.degrees.astype(np.float64)
    return np.where(d > 0, coeff * np.power(np.maximum(d, 1.0), power), np.inf)


@dataclass(frozen=True, eq=False)
class DiffusionSystem:
    """Q x = b with per-coordinate thresholds (theta rule: coeff * d^power)."""

    op: OperatorQ
    b: np.ndarray
    theta_coeff: float
    problem: str
    alpha: float = 0.0
    tau: float = 0.0
    eps: float = 0.0
    beta_exp: float = 0.0
    symmetrized: bool = False
    regime: str = "nonneg"
    source: int = -1
    theta_power: float = 1.0
    _theta: list = field(default_factory=list, repr=False)

    @property
    def graph(self):
        return self.op.graph

    @property
    def dim(self) -> int:
        return int(self.b.shape[0])

    @property
    def theta(self) -> np.ndarray:
        if not self._theta:
            t = theta_vector(self.graph, self.theta_coeff, self.theta_power)
            if self.problem == "hk":
                t = np.tile(t, self.op.stage_count + 1)
            self._theta.append(t)
        return self._theta[0]

    def with_source(self, s: int) -> "DiffusionSystem":
        """Same system with b moved to node s (the per-seed swap of a batch)."""
        b = np.zeros_like(self.b)
        b[s] = self.b[self.source] if self.source >= 0 else 1.0
        return DiffusionSystem(op=self.op, b=b, theta_coeff=self.theta_coeff,
                               problem=self.problem, alpha=self.alpha, tau=self.tau,
                               eps=self.eps, beta_exp=self.beta_exp,
                               symmetrized=self.symmetrized, regime=self.regime,
                               source=s, theta_power=self.theta_power, _theta=self._theta)

    def residual(self, x: np.ndarray) -> np.ndarray:
        if self.problem == "hk":
            return self.b - _hk_apply(self, x)
        return self.b - self.op.apply(x)

    def back_transform(self, x: np.ndarray) -> np.ndarray:
        if self.problem in ("ppr", "gen"):
            return x.copy()
        if self.problem == "katz":
            return x - self.b
        if self.problem == "hk":
            st = x.reshape(self.op.stage_count + 1, self.graph.n)
            return math.exp(-self.tau) * st.sum(axis=0)
        raise SystemError(f"unknown problem {self.problem}")


def _check_source(g, s: int) -> None:
    if not 0 <= s < g.n:
        raise SystemError("source out of range")
    if g.degrees[s] < 1:
        raise SystemError("source must have at least one neighbor")


def make_ppr_system(g, alpha: float, s: int, eps: float,
                    symmetrized: bool = False) -> DiffusionSystem:
    """(I - (1-alpha) A D^-1) x = alpha e_s, theta_u = (eps*alpha) d_u
    (src/systems.py:163-191)."""
    if not 0.0 < alpha <= 1.0:
        raise SystemError("alpha must be in (0, 1]")
    _check_source(g, s)
    if not 0.0 < eps <= 1.0 / g.degrees[s]:
        warnings.warn(f"eps={eps} outside (0, 1/d_s]; runtime guarantees may not apply",
                      stacklevel=2)
    op = OperatorQ(graph=g, beta=1.0 - alpha, pkind="rw")
    b = np.zeros(g.n)
    b[s] = alpha
    return DiffusionSystem(op=op, b=b, theta_coeff=eps * alpha, problem="ppr",
                           alpha=alpha, eps=eps, symmetrized=symmetrized, source=s)


def make_katz_system(g, alpha: float, s: int, eps: float,
                     lam_hat: float | None = None) -> DiffusionSystem:
    """(I - alpha A) x = e_s, theta_u = eps d_u (src/systems.py:194-219)."""
    _check_source(g, s)
    if lam_hat is None:
        from .graph import spectral_norm_estimate
        lam_hat = spectral_norm_estimate(g, iters=200, seed=0)
    if alpha <= 0.0 or (lam_hat > 0 and alpha >= 1.0 / lam_hat):
        raise SystemError(f"alpha={alpha} not in (0, 1/lam_hat)")
    op = OperatorQ(graph=g, beta=alpha, pkind="adj")
    b = np.zeros(g.n)
    b[s] = 1.0
    return DiffusionSystem(op=op, b=b, theta_coeff=eps, problem="katz", alpha=alpha,
                           eps=eps, regime="nonneg" if alpha * g.d_max < 1.0 else "spectral",
                           source=s)


def default_katz_alpha(g, lam_hat: float | None = None) -> float:
    if lam_hat is None:
        from .graph import spectral_norm_estimate
        lam_hat = spectral_norm_estimate(g, iters=200, seed=0)
    return 1.0 / (lam_hat + 1.0)


def hk_tail_bound(tau: float, n_stages: int) -> float:
    """e^-tau * sum_{k>N} tau^k/k!, summed forward until it stops changing."""
    term = 1.0
    for k in range(1, n_stages + 1):
        term *= tau / k
    tail, k = 0.0, n_stages
    while True:
        k += 1
        term *= tau / k
        nxt = tail + term
        if nxt == tail:
            break
        tail = nxt
        if k > n_stages + 500:
            break
    return math.exp(-tau) * tail


def hk_paper_bound(n_stages: int) -> float:
    return math.inf if n_stages < 1 else 1.0 / (math.factorial(n_stages) * n_stages)


def hk_stage_count(tau: float, eps: float) -> int:
    cap = int(2 * tau + 40)
    for k in range(cap + 1):
        if hk_tail_bound(tau, k) <= eps / 2.0:
            return k
    return cap


def make_hk_system(g, tau: float, s: int, eps: float) -> DiffusionSystem:
    """Stage-expanded heat kernel over (N+1) n coordinates (src/systems.py:269-301)."""
    if tau <= 0.0:
        raise SystemError("tau must be positive")
    _check_source(g, s)
    N = hk_stage_count(tau, eps)
    stage_w = tau / np.arange(1.0, N + 1.0) if N else np.empty(0)
    op = OperatorQ(graph=g, beta=1.0, pkind="rw", stage_count=N, stage_weights=stage_w)
    b = np.zeros((N + 1) * g.n)
    b[s] = 1.0
    vol = float(g.degrees.sum())
    return DiffusionSystem(op=op, b=b, theta_coeff=eps / (2.0 * (N + 1) * vol),
                           problem="hk", tau=tau, eps=eps, source=s)


def make_generalized_system(g, alpha: float, source: np.ndarray, eps: float,
                            beta_exp: float) -> DiffusionSystem:
    if not 0.0 < alpha < 1.0:
        raise SystemError("alpha must be in (0, 1)")
    if not 0.0 <= beta_exp <= 1.0:
        raise SystemError("beta_exp must be in [0, 1]")
    source = np.asarray(source, dtype=np.float64)
    if source.shape != (g.n,):
        raise SystemError("source must be a length-n vector")
    op = OperatorQ(graph=g, beta=1.0 - alpha, pkind="gen", b_exp=beta_exp)
    return DiffusionSystem(op=op, b=alpha * source, theta_coeff=eps * alpha,
                           theta_power=1.0 - beta_exp, problem="gen", alpha=alpha,
                           eps=eps, beta_exp=beta_exp)


def _hk_apply(sys: DiffusionSystem, v: np.ndarray) -> np.ndarray:
    n, N = sys.graph.n, sys.op.stage_count
    st = v.reshape(N + 1, n)
    out = st.copy()
    for k in range(N):
        out[k + 1] -= sys.op.stage_weights[k] * sys.op.propagate(st[k])
    return out.reshape(-1)


def dense_solve(sys: DiffusionSystem) -> np.ndarray:
    """Dense direct solution (n <= 2000), back-transformed (src/systems.py:336-364)."""
    import scipy.linalg

    g = sys.graph
    if g.n > _DENSE_GUARD:
        raise SystemError(f"dense solve guard: n={g.n} > {_DENSE_GUARD}")
    if sys.problem == "hk":
        m = np.eye(g.n) - sys.op.dense_matrix()
        N = sys.op.stage_count
        v = np.zeros((N + 1, g.n))
        v[0] = sys.b[:g.n]
        for k in range(N):
            v[k + 1] = sys.op.stage_weights[k] * (m @ v[k])
        return sys.back_transform(v.reshape(-1))
    if sys.symmetrized:
        dq = np.sqrt(np.maximum(g.degrees.astype(np.float64), 1.0))
        qs = (sys.op.dense_matrix() * dq[np.newaxis, :]) / dq[:, np.newaxis]
        xs = scipy.linalg.solve(qs, sys.b / dq, assume_a="sym")
        return sys.back_transform(dq * xs)
    try:
        x = scipy.linalg.solve(sys.op.dense_matrix(), sys.b)
    except scipy.linalg.LinAlgError as exc:
        raise SystemError("singular operator") from exc
    return sys.back_transform(x)


def series_oracle(sys: DiffusionSystem, terms: int) -> np.ndarray:
    """Truncated power series sum_k c_k M^k s (src/systems.py:367-408)."""
    if terms < 0:
        raise SystemError("terms must be >= 0")
    g = sys.graph
    if sys.problem in ("ppr", "gen"):
        vk, coeff, ratio = sys.b / sys.alpha, sys.alpha, 1.0 - sys.alpha
    elif sys.problem == "katz":
        vk, coeff, ratio = sys.b.copy(), 1.0, sys.alpha
    elif sys.problem == "hk":
        vk = np.zeros(g.n)
        vk[sys.source] = 1.0
        coeff, ratio = math.exp(-sys.tau), None
    else:
        raise SystemError(f"unknown problem {sys.problem}")
    bare = sys.op.arc_weights / sys.op.beta if sys.op.beta else sys.op.arc_weights
    src = np.repeat(np.arange(g.n, dtype=np.int64), g.degrees)
    total = coeff * vk
    for k in range(1, terms + 1):
        nxt = np.zeros(g.n)
        np.add.at(nxt, g.targets, bare * vk[src])
        vk = nxt
        coeff = coeff * ratio if ratio is not None else coeff * sys.tau / k
        total += coeff * vk
    if sys.problem == "katz":
        total -= sys.b
    return total
