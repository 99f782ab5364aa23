"""Two-time state on the device: packed, time-sliced history of G< and G>.

Replaces kbesolve/state.py.  The reference keeps two full
(n_k, 2, 2, N+1, N+1) tensors and mirrors the redundant triangle after every
step (state.py:95-109).  Here each function is ONE packed history per k
(include/kbe200.h): slice s holds the row block G<(t_s, t_b) and the column
block G>(t_b, t_s) for b = 0..s, so a step appends exactly one contiguous
slice and the mirror is never materialised -- G(t', t) = -G(t, t')^dagger is
applied on read.  This halves the reference's memory and reproduces its
arrays bitwise (SURVEY probe P12).  ``lesser`` / ``greater`` rebuild the
reference layout on demand (device unpack kernel, then a host copy).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import as_device_c128, require_cuda, stream_ptr, to_host
from .errors import CapacityError
from .kgrid import KGrid

DEFAULT_MEMORY_BUDGET = 2 * 1024**3   # state.py:24
_COMPLEX_BYTES = 16


def state_bytes(n_k: int, n_steps: int) -> int:
    """Footprint of the reference's two G tensors (state.py:51-53); used for the
    same CapacityError rules as the reference."""
    return 2 * n_k * 4 * (n_steps + 1) ** 2 * _COMPLEX_BYTES


def packed_bytes(n_k: int, n_steps: int) -> int:
    """Device footprint of one packed history (both triangles of one function pair)."""
    return n_k * _lib.tri_size(n_steps) * _COMPLEX_BYTES


def unpack_history(hist: torch.Tensor, n_steps: int, which: int, frontier: int | None = None) -> torch.Tensor:
    """Reference layout (k_local, 2, 2, N+1, N+1) from a packed history (device)."""
    k_local = hist.shape[0]
    out = torch.empty((k_local, 2, 2, n_steps + 1, n_steps + 1), dtype=torch.complex128, device=hist.device)
    fr = n_steps if frontier is None else frontier
    _lib.check(_lib.lib().kbe_unpack(hist.data_ptr(), hist.shape[1], k_local, n_steps, fr, which,
                                     out.data_ptr(), stream_ptr()), "kbe_unpack")
    return out


def pack_history(lower, upper, n_steps: int, frontier: int, hist: torch.Tensor | None = None) -> torch.Tensor:
    """Packed history from reference-layout (lower-stored, upper-stored) arrays."""
    lo = as_device_c128(lower)
    up = as_device_c128(upper)
    k_local = lo.shape[0]
    tri = _lib.tri_size(n_steps)
    if hist is None:
        hist = torch.zeros((k_local, tri), dtype=torch.complex128, device=lo.device)
    _lib.check(_lib.lib().kbe_pack(lo.data_ptr(), up.data_ptr(), k_local, n_steps, frontier, tri,
                                   hist.data_ptr(), stream_ptr()), "kbe_pack")
    return hist


class TwoTimeGF:
    """G< / G> for a (possibly local) k-range, device-resident and packed.

    Same attributes as kbesolve.TwoTimeGF (state.py:29-39).  ``lesser`` and
    ``greater`` return fresh host arrays in the reference layout; writing into
    them does not change the device state (use ``from_arrays`` to upload).
    """

    def __init__(self, n_k_local: int, k_offset: int, n_steps: int, dt: float,
                 hist: torch.Tensor, frontier: int = 0):
        self.n_k_local = n_k_local
        self.k_offset = k_offset
        self.n_steps = n_steps
        self.dt = dt
        self.hist = hist            # (k_local, tri) complex128, CUDA
        self.frontier = frontier

    # --- reference-layout accessors -------------------------------------------------
    def lesser_device(self) -> torch.Tensor:
        return unpack_history(self.hist, self.n_steps, 0)

    def greater_device(self) -> torch.Tensor:
        return unpack_history(self.hist, self.n_steps, 1)

    @property
    def lesser(self) -> np.ndarray:
        return to_host(self.lesser_device())

    @property
    def greater(self) -> np.ndarray:
        return to_host(self.greater_device())

    def retarded_device(self, theta0: float = 1.0) -> torch.Tensor:
        """G^R(t,t') = theta(t - t') [G>(t,t') - G<(t,t')] in the reference layout, on the
        device (kbe_unpack_retarded), theta(0) = theta0 on the equal-time diagonal
        (default 1: the t -> t'+ limit, G^R(t,t) = -i).  A derived accessor (SURVEY
        finding 2: the reference has none); its parity follows from G< / G> parity."""
        n1 = self.n_steps + 1
        out = torch.empty((self.n_k_local, 2, 2, n1, n1), dtype=torch.complex128, device=self.hist.device)
        _lib.check(_lib.lib().kbe_unpack_retarded(self.hist.data_ptr(), self.hist.shape[1], self.n_k_local,
                                                  self.n_steps, self.n_steps, float(theta0), out.data_ptr(),
                                                  stream_ptr()), "kbe_unpack_retarded")
        return out

    def retarded(self, theta0: float = 1.0) -> np.ndarray:
        """Host copy of retarded_device(theta0)."""
        return to_host(self.retarded_device(theta0))

    # --- frontier slices (device, no host round trip) ----------------------------------
    def slice_view(self, s: int) -> torch.Tensor:
        """(k_local, 8, s+1) device copy of slice s: planes 0..3 G<(t_s,t_b), 4..7 G>(t_b,t_s).
        The slice is stored as blocks of 8 planes x 32 points (include/kbe200.h)."""
        off = _lib.slice_offset(s)
        pl = _lib.plane_len(s)
        blk = self.hist[:, off: off + 8 * pl].view(self.n_k_local, pl // 32, 8, 32)
        return blk.permute(0, 2, 1, 3).reshape(self.n_k_local, 8, pl)[:, :, : s + 1]

    @classmethod
    def from_arrays(cls, lesser, greater, dt: float, frontier: int | None = None, k_offset: int = 0):
        lesser = np.asarray(lesser)
        n_steps = lesser.shape[-1] - 1
        fr = n_steps if frontier is None else frontier
        hist = pack_history(lesser, greater, n_steps, fr)
        return cls(lesser.shape[0], k_offset, n_steps, dt, hist, 0 if frontier is None else frontier)


@dataclass
class Observables:
    """Per-k occupations and the k-averaged density at one time (state.py:42-48)."""

    n_v: np.ndarray
    n_c: np.ndarray
    density: float


def _ground_state(hist: torch.Tensor) -> None:
    """Slice 0 in the packed layout: entry (plane c, point 0) is at slice_offset(0) + c*32."""
    hist.zero_()
    s0 = _lib.slice_offset(0)
    hist[:, s0 + 0 * 32] = 1.0j     # plane 0 = G<(0,0)_00 = i   (state.py:85)
    hist[:, s0 + 7 * 32] = -1.0j    # plane 7 = G>(0,0)_11 = -i  (state.py:86)


def init_state(grid: KGrid, n_steps: int, dt: float, memory_budget: int = DEFAULT_MEMORY_BUDGET,
               n_k_local: int | None = None, k_offset: int = 0) -> TwoTimeGF:
    """Allocate the device history and set the ground state (state.py:56-87)."""
    if n_steps < 1:
        raise CapacityError(f"n_steps must be >= 1, got {n_steps}")
    if dt <= 0:
        raise CapacityError(f"dt must be > 0, got {dt}")
    nk = grid.n_k if n_k_local is None else n_k_local
    needed = state_bytes(nk, n_steps)
    if needed > memory_budget:
        raise CapacityError(
            f"state needs {needed} bytes for n_k={nk}, n_steps={n_steps}; budget is {memory_budget}"
        )
    dev = require_cuda()
    hist = torch.empty((nk, _lib.tri_size(n_steps)), dtype=torch.complex128, device=dev)
    _ground_state(hist)
    return TwoTimeGF(nk, k_offset, n_steps, dt, hist)


def _is_device_state(state) -> bool:
    return isinstance(getattr(state, "hist", None), torch.Tensor)


def mirror_frontier(state, n: int | None = None) -> None:
    """Populate the redundant triangle of frontier n (state.py:95-109).

    A no-op for device states (the packed layout applies the symmetry on
    read); applied in place for reference-layout host arrays.
    """
    if _is_device_state(state):
        return
    if n is None:
        n = state.frontier
    if n == 0:
        return
    row_l = state.lesser[:, :, :, n, 0:n]
    state.lesser[:, :, :, 0:n, n] = -np.conj(np.swapaxes(row_l, 1, 2))
    col_g = state.greater[:, :, :, 0:n, n]
    state.greater[:, :, :, n, 0:n] = -np.conj(np.swapaxes(col_g, 1, 2))


def _diag_blocks(state, i: int):
    """(k, 2, 2) host copies of G<(t_i,t_i) and G>(t_i,t_i)."""
    if _is_device_state(state):
        sl = state.slice_view(i)[:, :, i]            # (k, 8)
        h = to_host(sl)
        return h[:, 0:4].reshape(-1, 2, 2), h[:, 4:8].reshape(-1, 2, 2)
    return state.lesser[:, :, :, i, i], state.greater[:, :, :, i, i]


def symmetry_residual(state, n: int | None = None) -> float:
    """Max deviation from conjugate symmetry on the frontier slices (state.py:112-122)."""
    if n is None:
        n = state.frontier
    if _is_device_state(state):
        # off-diagonal entries are symmetric by construction; only the diagonal can deviate
        gl, gg = _diag_blocks(state, n)
        res = 0.0
        for g in (gl, gg):
            res = max(res, float(np.abs(g + np.conj(np.swapaxes(g, 1, 2))).max()))
        return res
    res = 0.0
    for g in (state.lesser, state.greater):
        row = g[:, :, :, n, 0: n + 1]
        col = g[:, :, :, 0: n + 1, n]
        res = max(res, float(np.abs(col + np.conj(np.swapaxes(row, 1, 2))).max()))
    return res


def diagonal_blocks(state, n0: int, n1: int) -> tuple[np.ndarray, np.ndarray]:
    """G<(t_s,t_s) and G>(t_s,t_s) for s = n0..n1, all local k, as host (steps, k, 2, 2)
    arrays: one device gather over the packed history (no per-step host round trip)."""
    steps = np.arange(n0, n1 + 1)
    if not _is_device_state(state):
        gl = np.moveaxis(state.lesser[:, :, :, steps, steps], -1, 0)
        gg = np.moveaxis(state.greater[:, :, :, steps, steps], -1, 0)
        return gl, gg
    tri = state.hist.shape[1]
    offs = np.array([_lib.slice_offset(int(t)) for t in steps], dtype=np.int64)
    blk = (steps // 32) * 256 + steps % 32                      # point s of slice s
    planes = np.arange(8, dtype=np.int64) * 32
    idx = (np.arange(state.n_k_local, dtype=np.int64)[None, :, None] * tri
           + (offs + blk)[:, None, None] + planes[None, None, :])  # (steps, k, 8)
    vals = torch.take(state.hist, torch.from_numpy(idx).to(state.hist.device))
    h = to_host(vals)
    return h[..., 0:4].reshape(len(steps), -1, 2, 2), h[..., 4:8].reshape(len(steps), -1, 2, 2)


def observables_at(state, i: int) -> Observables:
    """n_b(k, t_i) = Im G<_bb(k; t_i, t_i) and the density (state.py:125-130)."""
    gl, _ = _diag_blocks(state, i)
    n_v = np.imag(gl[:, 0, 0]).copy()
    n_c = np.imag(gl[:, 1, 1]).copy()
    return Observables(n_v=n_v, n_c=n_c, density=float(np.mean(n_v + n_c)))


def anticommutation_drift(state, i: int) -> float:
    """max |G>(t,t) - G<(t,t) + i Id| at t_i (state.py:133-137)."""
    gl, gg = _diag_blocks(state, i)
    diff = gg - gl + 1.0j * np.eye(2)[None, :, :]
    return float(np.abs(diff).max())


def rho(state, i: int) -> np.ndarray:
    """Density matrix rho = -i G<(t_i, t_i) per k (propagator.py:272-273)."""
    gl, _ = _diag_blocks(state, i)
    return -1j * gl


def scatter(state: TwoTimeGF, n_shards: int) -> list:
    """Split into contiguous per-shard k-ranges (state.py:140-160)."""
    if state.n_k_local % n_shards != 0:
        raise ValueError(f"{n_shards} shards do not divide n_k={state.n_k_local}")
    my = state.n_k_local // n_shards
    return [TwoTimeGF(my, state.k_offset + s * my, state.n_steps, state.dt,
                      state.hist[s * my:(s + 1) * my].clone(), state.frontier) for s in range(n_shards)]


def gather(shards: list) -> TwoTimeGF:
    """Concatenate per-shard states ordered by k (state.py:163-181)."""
    ordered = sorted(shards, key=lambda s: s.k_offset)
    base = ordered[0]
    expect = base.k_offset
    for sh in ordered:
        if sh.k_offset != expect:
            raise ValueError(f"shards not contiguous at k-offset {sh.k_offset}")
        if sh.n_steps != base.n_steps or sh.dt != base.dt or sh.frontier != base.frontier:
            raise ValueError("shards disagree on grid or frontier metadata")
        expect = sh.k_offset + sh.n_k_local
    hist = torch.cat([s.hist for s in ordered], dim=0)
    return TwoTimeGF(expect - base.k_offset, base.k_offset, base.n_steps, base.dt, hist, base.frontier)
