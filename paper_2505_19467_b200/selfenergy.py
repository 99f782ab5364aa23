"""Second-Born self-energy on the device (replaces kbesolve/selfenergy.py).

Kernel-level functions keep the reference signatures and batch-last slice
layout ``(n_k, 2, 2[, nb])`` (selfenergy.py:55-56); each call runs the
sm_100a ``sigma_slice_kernel`` through the C ABI (``kbe_sigma_slice``).  The
driver path uses the fused ``kbe_sigma_frontier`` launch instead, which reads
the G frontier slice straight from the packed history and writes Sigma slice n.

Sigma^2 is evaluated in the factorised form of SURVEY finding 4 -- two
circular correlations, X(d) = sum_q B(d+q) C(q), Sigma^2(k) = sum_k' A(k') X(k'-k)
-- which is algebraically identical to the reference's O(n_k^3) triple sum
(selfenergy.py:139-203) and O(n_k^2) per pair.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import as_device_c128, as_device_f64, ptr, require_cuda, stream_ptr, to_host
from .engine import Schedule
from .kgrid import KGrid
from .state import _is_device_state, unpack_history


def _batched(x: np.ndarray) -> tuple[np.ndarray, bool]:
    x = np.asarray(x)
    return (x[..., None], True) if x.ndim == 3 else (x, False)


def _check_lookup(schedule, tables) -> None:
    if schedule is not None and schedule.index_mode == "lookup" and tables is None:
        raise ValueError("lookup index mode requires prebuilt tables")   # selfenergy.py:49-50


def _u_vector(u, nb: int) -> np.ndarray:
    u = np.asarray(u, dtype=float)
    return np.broadcast_to(u, (nb,)).astype(float) if u.ndim == 0 else u.reshape(nb).astype(float)


def _run_slice(gp, gr, u1, u2, n_k, k_range, pol_in=None, want=("sigma",)):
    gp, squeeze = _batched(gp)
    gr, _ = _batched(gr)
    if gp.shape != gr.shape:
        raise ValueError(f"slice shapes differ: {gp.shape} vs {gr.shape}")
    nb = gp.shape[-1]
    lo, hi = (0, n_k) if k_range is None else (int(k_range[0]), int(k_range[1]))
    dev = require_cuda()
    d_gp = as_device_c128(gp, dev)
    d_gr = as_device_c128(gr, dev)
    d_u1 = as_device_f64(_u_vector(u1, nb), dev)
    d_u2 = as_device_f64(_u_vector(u2, nb), dev)
    d_pol_in = None
    if pol_in is not None:
        p, _ = _batched(pol_in)
        d_pol_in = as_device_c128(p, dev)
    outs = {}
    shape_all = (n_k, 2, 2, nb)
    shape_loc = (hi - lo, 2, 2, nb)
    for name in want:
        outs[name] = torch.empty(shape_all if name == "pol" else shape_loc, dtype=torch.complex128, device=dev)
    _lib.check(_lib.lib().kbe_sigma_slice(
        n_k, nb, d_gp.data_ptr(), d_gr.data_ptr(), d_u1.data_ptr(), d_u2.data_ptr(), lo, hi,
        ptr(d_pol_in), ptr(outs.get("pol")), ptr(outs.get("s1")), ptr(outs.get("s2")),
        ptr(outs.get("sigma")), stream_ptr()), "kbe_sigma_slice")
    res = {k: to_host(v) for k, v in outs.items()}
    if squeeze:
        res = {k: v[..., 0] for k, v in res.items()}
    return res


def polarizability(g_less, g_greater_rev, grid: KGrid, schedule: Schedule | None = None, tables=None):
    """P_jm(q) = sum_k' G<_jm(k'+q) G>_mj(k') over the full k range (selfenergy.py:59-94)."""
    _check_lookup(schedule, tables)
    return _run_slice(g_less, g_greater_rev, 0.0, 0.0, grid.n_k, None, want=("pol",))["pol"]


def sigma_first(pol, g_less, u_t, u_tp, grid: KGrid, k_range=None, schedule: Schedule | None = None,
                tables=None):
    """First (polarizability) term on the local k range (selfenergy.py:104-136)."""
    _check_lookup(schedule, tables)
    g = np.asarray(g_less)
    return _run_slice(g, g, u_t, u_tp, grid.n_k, k_range, pol_in=pol, want=("s1",))["s1"]


def sigma_second(g_less, g_greater_rev, u_t, u_tp, grid: KGrid, k_range=None,
                 schedule: Schedule | None = None, tables=None, pool=None, scratch=None):
    """Second (exchange) term on the local k range (selfenergy.py:139-203)."""
    _check_lookup(schedule, tables)
    return _run_slice(g_less, g_greater_rev, u_t, u_tp, grid.n_k, k_range, want=("s2",))["s2"]


def assemble_sigma(sigma1, sigma2):
    """Full slice: first term minus second term (selfenergy.py:206-208)."""
    return sigma1 - sigma2


def sigma_slice(g_primary, g_reversed, u1, u2, grid: KGrid, k_range=None, schedule: Schedule | None = None,
                tables=None, pool=None, scratch=None, pol=None):
    """Complete pipeline for one component (selfenergy.py:211-236), one device launch."""
    _check_lookup(schedule, tables)
    return _run_slice(g_primary, g_reversed, u1, u2, grid.n_k, k_range, pol_in=pol, want=("sigma",))["sigma"]


class SigmaHistory:
    """Sigma components on the device, packed like G (selfenergy.py:239-244).

    Lower triangle = S> (rows, selfenergy.py:318), upper = S< (columns, 317).
    ``lesser`` / ``greater`` rebuild the reference layout on demand.
    """

    def __init__(self, hist: torch.Tensor, n_steps: int):
        self.hist = hist
        self.n_steps = n_steps

    def lesser_device(self) -> torch.Tensor:
        return unpack_history(self.hist, self.n_steps, 1)

    def greater_device(self) -> torch.Tensor:
        return unpack_history(self.hist, self.n_steps, 0)

    @property
    def lesser(self) -> np.ndarray:
        return to_host(self.lesser_device())

    @property
    def greater(self) -> np.ndarray:
        return to_host(self.greater_device())


def init_sigma_history(n_k: int, n_steps: int) -> SigmaHistory:
    """Zeroed device history (selfenergy.py:247-252)."""
    dev = require_cuda()
    hist = torch.zeros((n_k, _lib.tri_size(n_steps)), dtype=torch.complex128, device=dev)
    return SigmaHistory(hist, n_steps)


def evaluate_sigma_batched(state, sigma, n: int, grid: KGrid, u_table, schedule: Schedule | None = None,
                           tables=None, pool=None, scratch=None) -> None:
    """Both components on the step-n frontier in one batched pass (selfenergy.py:261-325).

    Device state + device SigmaHistory: one fused ``kbe_sigma_frontier`` launch
    that writes Sigma slice n of the packed history.  Reference-layout host
    arrays are also accepted (kernel-level parity): the two components run as
    ``kbe_sigma_slice`` launches and are written back with their mirrors.
    """
    _check_lookup(schedule, tables)
    if schedule is not None:
        schedule.validate(grid.n_k)
    u_table = np.asarray(u_table, dtype=float)
    if _is_device_state(state) and isinstance(sigma, SigmaHistory):
        from .propagator import _Workspace   # local import: propagator builds on this module
        ws = _Workspace.for_kernel_call(grid, state, sigma, u_table)
        _lib.check(_lib.lib().kbe_sigma_frontier(ws.problem_ptr(), n, 0, stream_ptr()), "kbe_sigma_frontier")
        torch.cuda.current_stream().synchronize()
        return
    gl = state.lesser if not _is_device_state(state) else state.lesser
    gg = state.greater if not _is_device_state(state) else state.greater
    gl_col = gl[:, :, :, 0: n + 1, n]
    gg_row = gg[:, :, :, n, 0: n + 1]
    lesser_col = sigma_slice(gl_col, gg_row, u_table[0: n + 1], float(u_table[n]), grid)
    greater_row = sigma_slice(gg_row, gl_col, float(u_table[n]), u_table[0: n + 1], grid)
    sigma.lesser[:, :, :, 0: n + 1, n] = lesser_col
    sigma.greater[:, :, :, n, 0: n + 1] = greater_row
    if n > 0:
        sigma.lesser[:, :, :, n, 0:n] = -np.conj(np.swapaxes(lesser_col[..., 0:n], 1, 2))
        sigma.greater[:, :, :, 0:n, n] = -np.conj(np.swapaxes(greater_row[..., 0:n], 1, 2))
