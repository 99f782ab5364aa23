"""Collision integrals on the device (replaces kbesolve/collision.py).

``collision_frontier`` runs the history-streaming ``collision_kernel``
(K2) over the packed Sigma and G triangles and reduces its partial sums into
the reference's ``CollisionSlice`` (collision.py:165-176).  The quadrature
weights are closed-form in-kernel; the host functions below exist for API
parity (collision.py:31-78).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import require_cuda, stream_ptr, to_host
from .engine import Schedule
from .errors import ConfigError
from .state import _is_device_state, pack_history

LIMIT_MODES = ("as-printed", "langreth")
QUAD_KINDS = ("trapezoid", "simpson")
DEVICE_LIMIT_MODES = ("as-printed", "langreth")


def quadrature_weights(n: int, dt: float, kind: str = "trapezoid") -> np.ndarray:
    """Trapezoid / Simpson (odd n: first interval trapezoid) weights (collision.py:31-61)."""
    if n < 0:
        raise ValueError(f"interval count must be >= 0, got {n}")
    if n == 0:
        return np.zeros(0)
    if kind == "trapezoid":
        w = np.full(n + 1, dt)
        w[0] = w[-1] = 0.5 * dt
        return w
    if kind != "simpson":
        raise ConfigError(f"quadrature kind must be 'trapezoid' or 'simpson', got {kind!r}")
    w = np.zeros(n + 1)
    start = 0
    if n % 2 == 1:
        w[0] += 0.5 * dt
        w[1] += 0.5 * dt
        start = 1
        if n == 1:
            return w
    m = n - start
    ws = np.full(m + 1, 2.0)
    ws[1::2] = 4.0
    ws[0] = ws[-1] = 1.0
    w[start:] += ws * (dt / 3.0)
    return w


@dataclass(frozen=True)
class QuadratureRule:
    kind: str = "trapezoid"

    def weights(self, n: int, dt: float) -> np.ndarray:
        return quadrature_weights(n, dt, self.kind)


def weight_matrix(limits, n_rows: int, dt: float, rule: QuadratureRule) -> np.ndarray:
    """Column c holds the padded weights for interval count limits[c] (collision.py:72-78)."""
    out = np.zeros((n_rows, len(limits)))
    for c, lim in enumerate(limits):
        w = rule.weights(lim, dt)
        out[: len(w), c] = w
    return out


def collision_row(dg_first, g_first, s_like, s_other, w1, w2) -> np.ndarray:
    """Row-slice contraction (collision.py:141-162) on the device: ``collision_row_kernel``.

    s_like, s_other: (k,2,2,T,P) over history x pair columns; dg_first: (k,2,2,len(w1));
    g_first: (k,2,2,len(w2)) for a shared limit, or (k,2,2,T) with a (T,P) per-column
    w2 -- the reference's einsum shapes.  Returns term1 + term2, shape (k,2,2,P)."""
    from ._device import as_device_c128, as_device_f64
    dev = require_cuda()
    dg, g = as_device_c128(dg_first, dev), as_device_c128(g_first, dev)
    sl, so = as_device_c128(s_like, dev), as_device_c128(s_other, dev)
    w1a, w2a = np.asarray(w1, dtype=float).reshape(-1), np.asarray(w2, dtype=float)
    if sl.dim() != 5 or sl.shape != so.shape or tuple(sl.shape[1:3]) != (2, 2):
        raise ValueError(f"collision_row: s_like/s_other must be (k,2,2,T,P), got {tuple(sl.shape)} / {tuple(so.shape)}")
    nk, T, P = int(sl.shape[0]), int(sl.shape[3]), int(sl.shape[4])
    T1 = int(w1a.shape[0])
    T2 = T if w2a.ndim == 2 else int(w2a.shape[0])
    if w2a.ndim == 2 and w2a.shape != (T, P):
        raise ValueError(f"collision_row: w2 matrix must be {(T, P)}, got {w2a.shape}")
    if T1 > T or T2 > T or tuple(dg.shape) != (nk, 2, 2, T1) or tuple(g.shape) != (nk, 2, 2, T2):
        raise ValueError(f"collision_row: operands could not be broadcast together: dg {tuple(dg.shape)}, "
                         f"g {tuple(g.shape)}, s {tuple(sl.shape)}, w1 ({T1},), w2 {w2a.shape}")
    w1d, w2d = as_device_f64(w1a, dev), as_device_f64(w2a.reshape(-1), dev)
    out = torch.empty((nk, 2, 2, P), dtype=torch.complex128, device=dev)
    _lib.check(_lib.lib().kbe_collision_row(
        nk, T, P, T1, T2, int(w2a.ndim == 2), dg.data_ptr(), g.data_ptr(), sl.data_ptr(), so.data_ptr(),
        w1d.data_ptr(), w2d.data_ptr(), out.data_ptr(), stream_ptr()), "kbe_collision_row")
    return to_host(out)


@dataclass
class CollisionSlice:
    """I components on the step-n frontier (collision.py:165-176)."""

    lesser_row: np.ndarray
    greater_row: np.ndarray
    lesser_col: np.ndarray
    greater_col: np.ndarray


def validate_rule(kind: str, limit_mode: str) -> tuple[int, int]:
    if limit_mode not in LIMIT_MODES:
        raise ConfigError(f"limit_mode must be one of {LIMIT_MODES}, got {limit_mode!r}")
    if kind not in QUAD_KINDS:
        raise ConfigError(f"quadrature kind must be 'trapezoid' or 'simpson', got {kind!r}")
    if limit_mode not in DEVICE_LIMIT_MODES:
        raise ConfigError(f"limit_mode {limit_mode!r} is not implemented on the B200 device path yet")
    return QUAD_KINDS.index(kind), LIMIT_MODES.index(limit_mode)


def collision_frontier(state, sigma, n: int, rule: QuadratureRule = QuadratureRule(),
                       schedule: Schedule | None = None, limit_mode: str = "as-printed",
                       pool=None) -> CollisionSlice:
    """Both components on all frontier pairs of step n, one K2 launch (collision.py:228-277).

    Device states are read in place; reference-layout host arrays are packed
    into temporary device histories first.
    """
    quad, limit = validate_rule(rule.kind, limit_mode)
    if schedule is not None:
        schedule.validate(state.n_k_local)
    from .propagator import _Workspace
    dev = require_cuda()
    if _is_device_state(state) and isinstance(getattr(sigma, "hist", None), torch.Tensor):
        g_hist, s_hist, n_steps = state.hist, sigma.hist, state.n_steps
    else:
        lesser = np.asarray(state.lesser)
        n_steps = lesser.shape[-1] - 1
        g_hist = pack_history(lesser, state.greater, n_steps, n)
        s_hist = pack_history(sigma.greater, sigma.lesser, n_steps, n)
    nk = g_hist.shape[0]
    ws = _Workspace.for_collision(nk, n_steps, float(state.dt), quad, g_hist, s_hist, dev, limit)
    st = stream_ptr()
    L = _lib.lib()
    _lib.check(L.kbe_collision_frontier(ws.problem_ptr(), n, 0, st), "kbe_collision_frontier")
    lr = torch.empty((nk, 2, 2, n + 1), dtype=torch.complex128, device=dev)
    gr = torch.empty_like(lr)
    lc = torch.empty((nk, 2, 2, n), dtype=torch.complex128, device=dev)
    gc = torch.empty_like(lc)
    _lib.check(L.kbe_collision_slice(ws.problem_ptr(), n, lr.data_ptr(), gr.data_ptr(), lc.data_ptr(),
                                     gc.data_ptr(), st), "kbe_collision_slice")
    return CollisionSlice(to_host(lr), to_host(gr), to_host(lc), to_host(gc))


def collision_lesser(state, sigma, k: int, i: int, l: int, rule: QuadratureRule = QuadratureRule(),
                     limit_mode: str = "as-printed") -> np.ndarray:
    """Per-pair I<(k; t_i, t'_l) (collision.py:115-126): a row pair of frontier i
    when i >= l, else a column pair of frontier l."""
    if i >= l:
        return collision_frontier(state, sigma, i, rule, None, limit_mode).lesser_row[k, :, :, l]
    return collision_frontier(state, sigma, l, rule, None, limit_mode).lesser_col[k, :, :, i]


def collision_greater(state, sigma, k: int, i: int, l: int, rule: QuadratureRule = QuadratureRule(),
                      limit_mode: str = "as-printed") -> np.ndarray:
    """Per-pair I>(k; t_i, t'_l) (collision.py:129-138)."""
    if i >= l:
        return collision_frontier(state, sigma, i, rule, None, limit_mode).greater_row[k, :, :, l]
    return collision_frontier(state, sigma, l, rule, None, limit_mode).greater_col[k, :, :, i]
