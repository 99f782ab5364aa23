"""Two-time stepping driver on one B200 per rank (replaces kbesolve/propagator.py).

``PropagationDriver`` keeps the reference constructor, ``step()``, ``run()``,
``state`` and ``sigma`` (propagator.py:229-392).  One step is the
reference's Algorithm 1 (propagator.py:316-382) as a fixed launch sequence
on one CUDA stream:

    K1 Sigma(n-1) -> K2 I(n-1) -> K3 predict(n)
    -> max_iter x [K1 Sigma(n) -> K2 I(n) -> K3 correct(n)] -> K4 finish(n)

Convergence is decided on the device: K3 max-reduces the residual into a
control block and every later launch of the step becomes a no-op once a
residual <= eps is recorded, so the host never synchronises inside a
step.  ``run()`` without an observer launches all steps back to back and
reads the StepReports once at the end.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._device import as_device_f64, require_cuda, stream_ptr, to_host
from .collision import validate_rule
from .engine import Schedule, WorkerPool, shard_range
from .errors import CapacityError, ConfigError, PoisonedStateError
from .kgrid import KGrid
from .model import ModelConfig, band_energies, step_tables, u_values
from .selfenergy import SigmaHistory
from .state import DEFAULT_MEMORY_BUDGET, TwoTimeGF, _ground_state, state_bytes


@dataclass
class StepConfig:
    """Same fields, defaults and validation as propagator.py:44-62."""

    dt: float
    n_steps: int
    eps: float = 1e-9
    max_iter: int = 6
    quadrature: str = "trapezoid"
    limit_mode: str = "as-printed"
    memory_budget: int = DEFAULT_MEMORY_BUDGET

    def validate(self) -> None:
        if self.dt <= 0:
            raise ConfigError(f"dt must be > 0, got {self.dt}")
        if self.n_steps < 0:
            raise ConfigError(f"n_steps must be >= 0, got {self.n_steps}")
        if self.eps <= 0:
            raise ConfigError(f"eps must be > 0, got {self.eps}")
        if self.max_iter < 1:
            raise ConfigError(f"max_iter must be >= 1, got {self.max_iter}")


@dataclass
class StepReport:
    """Per-step report (propagator.py:65-74)."""

    step: int
    iterations: int
    residual: float
    converged: bool
    anticommutation_drift: float
    density: float
    residual_history: list = field(default_factory=list)
    timings: dict = field(default_factory=dict)
    # one-body energy (1/n_k) sum_k Tr[h(k; t_n) rho(k; t_n)] with h = build_h at the grid
    # point t_n (model.py:123-152) and rho = -i G<(t_n, t_n) (propagator.py:272-273).  Not a
    # reference field (the reference has no energy observable, SURVEY finding 2); appended
    # with a default so the reference's positional fields are unchanged.
    energy: float = 0.0


def cayley_propagator(h: np.ndarray, dt: float) -> np.ndarray:
    """(1 + i dt h/2)^-1 (1 - i dt h/2) per k (propagator.py:77-94).

    API parity only; the device path builds Phi inside the update kernel.
    """
    a = 0.5j * dt * np.asarray(h)
    m00, m01, m10, m11 = 1.0 + a[:, 0, 0], a[:, 0, 1], a[:, 1, 0], 1.0 + a[:, 1, 1]
    n00, n01, n10, n11 = 1.0 - a[:, 0, 0], -a[:, 0, 1], -a[:, 1, 0], 1.0 - a[:, 1, 1]
    det = m00 * m11 - m01 * m10
    phi = np.empty_like(a)
    phi[:, 0, 0] = (m11 * n00 - m01 * n10) / det
    phi[:, 0, 1] = (m11 * n01 - m01 * n11) / det
    phi[:, 1, 0] = (m00 * n10 - m10 * n00) / det
    phi[:, 1, 1] = (m00 * n11 - m10 * n01) / det
    return phi


def _backend() -> str:
    import torch.distributed as dist
    return dist.get_backend() if dist.is_initialized() else "none"


def all_gather_device(out: torch.Tensor, inp: torch.Tensor) -> None:
    """out = concat over ranks of inp (rank order = k order).  NCCL moves device
    memory directly (NVLink); other backends (gloo, for tests) stage through the host."""
    import torch.distributed as dist
    o = torch.view_as_real(out) if out.is_complex() else out
    i = torch.view_as_real(inp) if inp.is_complex() else inp
    if _backend() == "nccl":
        dist.all_gather_into_tensor(o.reshape(-1), i.reshape(-1))
        return
    parts = [torch.empty(i.numel(), dtype=i.dtype) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, i.reshape(-1).cpu())
    o.reshape(-1).copy_(torch.cat(parts).to(o.device))


def all_reduce_device(t: torch.Tensor, op) -> None:
    import torch.distributed as dist
    if _backend() == "nccl":
        dist.all_reduce(t, op=op)
        return
    c = t.cpu()
    dist.all_reduce(c, op=op)
    t.copy_(c.to(t.device))


def all_gather_list(t: torch.Tensor, world: int) -> list:
    import torch.distributed as dist
    if _backend() == "nccl":
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return parts
    parts = [torch.empty_like(t, device="cpu") for _ in range(world)]
    dist.all_gather(parts, t.cpu())
    return parts


def combine_reports(stacked: np.ndarray) -> np.ndarray:
    """Per-rank StepReport rows (world, steps, W) -> global rows: drift is a max over
    k, the density column a sum over k, the non-finite flag an OR; iteration counts
    and residuals are already global (all-reduced every iteration)."""
    out = stacked[0].copy()
    out[:, 4] = stacked[:, :, 4].max(axis=0)
    out[:, 5] = stacked[:, :, 5].sum(axis=0)
    out[:, 6] = stacked[:, :, 6].max(axis=0)
    out[:, 7] = stacked[:, :, 7].sum(axis=0)                       # energy k-sum
    r0 = 8 + _lib.MAX_ITER
    out[:, r0: r0 + 4] = stacked[:, :, r0: r0 + 4].sum(axis=0)     # rho k-sums
    return out


class _Workspace:
    """Device buffers + the ``kbe_problem`` struct handed to the C ABI.

    Allocated once per driver (paper section IV-C: no allocation inside the
    step loop); the partial-sum buffers are the K2 -> K3 hand-off.
    """

    def __init__(self, *, n_k, k_lo, k_hi, n_steps, dt, eps, max_iter, quad, limit_mode, hf,
                 interacting, dipole, eps_v, eps_c, u_table, u_mid, amp, g_hist, s_hist, device,
                 multi_rank=False, incremental=False):
        N1 = n_steps + 1
        kl = k_hi - k_lo
        self.nbb = -(-N1 // _lib.TILE_B)
        self.nsb = -(-N1 // _lib.COL_CHUNK)
        c128 = dict(dtype=torch.complex128, device=device)
        self.g_hist, self.s_hist = g_hist, s_hist
        self.row_part = torch.zeros((kl, N1, self.nbb, 4), **c128)
        self.col_part = torch.zeros((kl, N1, self.nsb, 4), **c128)
        self.gc_part = torch.zeros((kl, N1, self.nbb, 4), **c128)
        self.lr_old = torch.zeros((kl, N1, 4), **c128)
        self.col_old = torch.zeros((kl, N1, 4), **c128)
        self.ctl = torch.zeros(int(_lib.lib().kbe_ctl_bytes()), dtype=torch.uint8, device=device)
        self.reports = torch.zeros((N1, _lib.REPORT_W), dtype=torch.float64, device=device)
        self.phi = torch.zeros((N1, kl, 4), **c128)
        self.fcol_part = torch.zeros((kl, N1, 4), **c128)
        # K3a -> K3b hand-off of the split update (as-printed, many local k)
        # [0]: the sums K3b reads; [1]: incremental problems' base sums of the last full
        # evaluation (reduce_kernel)
        self.i_red = torch.zeros((2, kl, N1, 4), **c128)
        self.g_red = torch.zeros((2, kl, N1, 4), **c128)
        # incremental collision evaluations (as-printed): complex64 shadows of the final
        # history slices and the frontier the last evaluation used (include/kbe200.h)
        self.g_sh = self.s_sh = self.v_prev = None
        if incremental and not limit_mode:
            self.g_sh = torch.zeros_like(g_hist, dtype=torch.complex64)
            self.s_sh = torch.zeros_like(s_hist, dtype=torch.complex64)
            self.v_prev = torch.zeros((kl, 2, 8 * _lib.plane_len(n_steps)), **c128)
            # delta slots: complex64 (FP32 sums, stored exactly; kbe200.cu st_keep_f)
            self.deltas = [torch.zeros(t.shape, dtype=torch.complex64, device=device)
                           for t in (self.row_part, self.col_part, self.gc_part)]
        self.lang = None
        if limit_mode:   # langreth: I> rows and I< columns kept separately, both directions
            shapes = (self.nbb, self.nsb, self.nbb, self.nsb, self.nsb)   # row_g, col_g, lc, gc_c, lc_c
            self.lang = [torch.zeros((kl, nb, N1, 4), **c128) for nb in shapes]
        self.eps_v = as_device_f64(eps_v, device)
        self.eps_c = as_device_f64(eps_c, device)
        self.u_table = as_device_f64(u_table, device)
        self.u_mid = as_device_f64(u_mid, device)
        self.amp = as_device_f64(amp, device)
        self.front_send = self.front_all = None
        if multi_rank:
            # one all-gather chunk per rank: [k_local][capacity slice] + control tail
            # (residual bits and non-finite flags; include/kbe200.h)
            chunk = kl * 8 * _lib.plane_len(n_steps) + _lib.TAIL_CPLX
            self.front_send = torch.zeros(chunk, **c128)
            self.front_all = torch.zeros((n_k // kl, chunk), **c128)
        p = _lib.KbeProblem()
        p.n_k, p.k_lo, p.k_hi, p.n_steps = n_k, k_lo, k_hi, n_steps
        p.quad, p.limit_mode, p.hf, p.max_iter = quad, limit_mode, int(hf), max_iter
        p.interacting, p.nbb, p.nsb = int(interacting), self.nbb, self.nsb
        p.dt, p.eps = float(dt), float(eps)
        p.dipole_re, p.dipole_im = float(np.real(dipole)), float(np.imag(dipole))
        p.tri = int(g_hist.shape[1])
        p.g_hist, p.s_hist = g_hist.data_ptr(), s_hist.data_ptr()
        p.eps_v, p.eps_c = self.eps_v.data_ptr(), self.eps_c.data_ptr()
        p.u_table, p.u_mid, p.amp = self.u_table.data_ptr(), self.u_mid.data_ptr(), self.amp.data_ptr()
        p.row_part, p.col_part, p.gc_part = (self.row_part.data_ptr(), self.col_part.data_ptr(),
                                             self.gc_part.data_ptr())
        p.lr_old, p.col_old = self.lr_old.data_ptr(), self.col_old.data_ptr()
        p.front_send = self.front_send.data_ptr() if self.front_send is not None else None
        p.front_all = self.front_all.data_ptr() if self.front_all is not None else None
        p.ctl, p.reports = self.ctl.data_ptr(), self.reports.data_ptr()
        p.phi = self.phi.data_ptr()
        if self.lang is not None:
            (p.row_part_g, p.col_part_g, p.lc_part, p.gc_part_c, p.lc_part_c) = [t.data_ptr() for t in self.lang]
        p.fcol_part = self.fcol_part.data_ptr()
        p.i_red, p.g_red = self.i_red.data_ptr(), self.g_red.data_ptr()
        if self.g_sh is not None:
            p.g_sh, p.s_sh, p.v_prev = self.g_sh.data_ptr(), self.s_sh.data_ptr(), self.v_prev.data_ptr()
            p.row_delta, p.col_delta, p.gc_delta = [t.data_ptr() for t in self.deltas]
        self.problem = p

    def problem_ptr(self) -> int:
        return ctypes.addressof(self.problem)

    # --- small workspaces for the kernel-level API ------------------------------------
    @classmethod
    def for_collision(cls, n_k, n_steps, dt, quad, g_hist, s_hist, device, limit_mode=0):
        z = np.zeros(max(n_k, n_steps + 1))
        return cls(n_k=n_k, k_lo=0, k_hi=n_k, n_steps=n_steps, dt=dt, eps=1e-9, max_iter=1, quad=quad,
                   limit_mode=limit_mode, hf=False, interacting=True, dipole=0.0, eps_v=z[:n_k], eps_c=z[:n_k],
                   u_table=z[: n_steps + 1], u_mid=z[: n_steps + 1], amp=z[: n_steps + 1],
                   g_hist=g_hist, s_hist=s_hist, device=device)

    @classmethod
    def for_kernel_call(cls, grid: KGrid, state: TwoTimeGF, sigma: SigmaHistory, u_table):
        n_k = state.n_k_local
        z = np.zeros(max(n_k, state.n_steps + 1))
        return cls(n_k=grid.n_k, k_lo=0, k_hi=n_k, n_steps=state.n_steps, dt=state.dt, eps=1e-9, max_iter=1,
                   quad=0, limit_mode=0, hf=False, interacting=True, dipole=0.0, eps_v=z[:n_k], eps_c=z[:n_k],
                   u_table=np.asarray(u_table, dtype=float)[: state.n_steps + 1],
                   u_mid=z[: state.n_steps + 1], amp=z[: state.n_steps + 1],
                   g_hist=state.hist, s_hist=sigma.hist, device=state.hist.device)


class _PeerExchange:
    """Peer-to-peer frontier exchange for k-sharded ranks (kbe_p2p_* in include/kbe200.h).

    Every rank cudaMallocs one exchange buffer, the IPC handles are all-gathered over
    torch.distributed, and each rank maps every peer's buffer.  The update kernel then
    stores its new slice and control tail straight into all peers' buffers (NVLink) and
    flags an epoch, replacing the per-iteration NCCL all-gather.  Used when every rank
    can map every peer (KBE_P2P=0 forces the NCCL path); the decision is collective."""

    def __init__(self, local, peers, rank):
        self.local, self.peers, self.rank = local, peers, rank

    @classmethod
    def setup(cls, ws, rank: int, world: int):
        import torch.distributed as dist
        if os.environ.get("KBE_P2P", "1") == "0" or world > _lib.MAX_RANKS:
            return None
        L, p = _lib.lib(), ws.problem
        nbytes = int(L.kbe_p2p_bytes(ws.problem_ptr(), world))
        local, handle = ctypes.c_void_p(), ctypes.create_string_buffer(64)
        ok = L.kbe_p2p_alloc(nbytes, ctypes.byref(local), handle) == 0
        handles = [None] * world
        dist.all_gather_object(handles, handle.raw if ok else None)
        peers = []
        if all(h is not None for h in handles):
            for r, h in enumerate(handles):
                if r == rank:
                    peers.append(local.value)
                    continue
                ptr = ctypes.c_void_p()
                if L.kbe_p2p_open(h, ctypes.byref(ptr)) != 0:
                    ok = False
                    break
                peers.append(ptr.value)
        flags = [None] * world
        dist.all_gather_object(flags, bool(ok and len(peers) == world))
        ex = cls(local.value if local.value else None, peers, rank)
        ex.nbytes = nbytes
        if not all(flags):       # every rank falls back to NCCL together
            dist.barrier()
            ex.close()
            return None
        p.p2p_world, p.p2p_rank, p.p2p_local = world, rank, local.value
        for r, ptr in enumerate(peers):
            p.p2p_peers[r] = ptr
        return ex

    def check(self, nbytes: int) -> None:
        """Raise if a peer wait timed out on this rank (the watchdog word after the epoch)."""
        if self.local is None:
            return
        word = torch.empty(1, dtype=torch.int64)
        import ctypes as _ct
        cuda = torch.cuda
        cuda.synchronize()
        src = self.local + nbytes - 8
        _lib.check(_lib.lib().kbe_p2p_read_u64(src, _ct.c_void_p(word.data_ptr())), "kbe_p2p_read_u64")
        # share the watchdog words so that every rank raises together: a rank whose own
        # wait did not time out would otherwise block in the next collective (_reports)
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            words = [torch.zeros(1, dtype=torch.int64) for _ in range(dist.get_world_size())]
            dist.all_gather(words, word) if dist.get_backend() == "gloo" else self._gather_words(words, word)
            hit = [(r, int(w[0])) for r, w in enumerate(words) if int(w[0]) != 0]
        else:
            hit = [(self.rank, int(word[0]))] if int(word[0]) != 0 else []
        if hit:
            r, w = hit[0]
            raise RuntimeError(f"peer-to-peer exchange timed out on rank {r} waiting for rank {w - 1}")

    @staticmethod
    def _gather_words(words, word):
        """all_gather of the 8-byte watchdog words on a device backend (NCCL)."""
        import torch.distributed as dist
        dev = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in words]
        dist.all_gather(dev, word.to("cuda"))
        for w, d in zip(words, dev):
            w.copy_(d.cpu())

    def close(self, free_local: bool = True) -> None:
        """Unmap the peers' buffers (after this rank's stream is idle).  The local buffer
        is freed only when every rank is known to be done with it (free_local, after a
        barrier); otherwise it is left allocated rather than risk a peer's late store."""
        if self.local is None:
            return
        L = _lib.lib()
        torch.cuda.synchronize()
        for r, ptr in enumerate(self.peers):
            if r != self.rank and ptr:
                L.kbe_p2p_close(ptr)
        if free_local:
            L.kbe_p2p_free(self.local)
        self.local, self.peers = None, []


def _incremental_default(n_k: int) -> bool:
    """Incremental collision evaluations (collision_kernel): KBE_INCR=1/0 forces them on /
    off; by default on for n_k >= 8.  With their complex64 arithmetic they pay from
    n_k = 16 up (profiles/r01/incr_ab_v23.jsonl: cfg2 +5.5 %, cfg3 +9 %, cfg5 +4.5 %);
    at n_k = 2 the snapshot and shadow writes cost more than they save (cfg1 -8 %)."""
    env = os.environ.get("KBE_INCR")
    if env in ("0", "1"):
        return env == "1"
    return n_k >= 8


_SIGMA_VARIANTS = {"auto": 0, "fft": 1, "dft": 2, "direct": 3}


def _sigma_variant_from_env() -> None:
    """KBE_SIGMA = auto | fft | dft | direct selects the K1 kernel (kbe_set_sigma_variant):
    by default FFT for power-of-two n_k > 2, the correlations at n_k = 2 and DMMA DFT GEMMs
    otherwise."""
    env = os.environ.get("KBE_SIGMA", "auto")
    if env not in _SIGMA_VARIANTS:
        raise ConfigError(f"KBE_SIGMA must be one of {sorted(_SIGMA_VARIANTS)}, got {env!r}")
    _lib.lib().kbe_set_sigma_variant(_SIGMA_VARIANTS[env])


def _dist_info(schedule: Schedule):
    """(rank, world) of the k-shard group: torch.distributed when initialised."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


class PropagationDriver:
    """Owns the device state and Sigma history and advances them (propagator.py:229-392)."""

    def __init__(self, grid: KGrid, model: ModelConfig, step_cfg: StepConfig,
                 schedule: Schedule | None = None, pool: WorkerPool | None = None, timings: bool | None = None):
        model.validate()
        step_cfg.validate()
        self.grid = grid
        self.model = model
        self.cfg = step_cfg
        self.schedule = schedule if schedule is not None else Schedule()
        self.schedule.validate(grid.n_k)
        self.pool = pool
        quad, limit = validate_rule(step_cfg.quadrature, step_cfg.limit_mode)
        if grid.n_k > _lib.MAX_NK:   # checked before any device allocation
            raise ConfigError(f"n_k must be <= {_lib.MAX_NK} on the device path, got {grid.n_k}")
        if step_cfg.max_iter > _lib.MAX_ITER:
            raise ConfigError(f"max_iter must be <= {_lib.MAX_ITER} on the device path, got {step_cfg.max_iter}")
        capacity = max(step_cfg.n_steps, 1)
        if 2 * state_bytes(grid.n_k, capacity) > step_cfg.memory_budget:   # propagator.py:253-259
            raise CapacityError(
                f"run needs {2 * state_bytes(grid.n_k, capacity)} bytes "
                f"(n_k={grid.n_k}, n_steps={capacity}); budget is {step_cfg.memory_budget}"
            )
        self.capacity = capacity
        self.u_table = u_values(model, capacity)
        self.interactions_on = bool(np.any(self.u_table != 0.0))
        eps_v, eps_c = band_energies(model, grid)
        u_mid, amp = step_tables(model, self.u_table, capacity, step_cfg.dt)

        self.rank, self.world = _dist_info(self.schedule)
        self.k_lo, self.k_hi = shard_range(grid.n_k, self.rank, self.world)
        dev = require_cuda()
        self.device = dev
        _sigma_variant_from_env()
        tri = _lib.tri_size(capacity)
        nkl = self.k_hi - self.k_lo
        g_hist = torch.empty((nkl, tri), dtype=torch.complex128, device=dev)
        s_hist = torch.empty((nkl, tri), dtype=torch.complex128, device=dev)
        self.ws = _Workspace(
            n_k=grid.n_k, k_lo=self.k_lo, k_hi=self.k_hi, n_steps=capacity, dt=step_cfg.dt,
            eps=step_cfg.eps, max_iter=step_cfg.max_iter, quad=quad, limit_mode=limit,
            hf=model.hf_mode == "on", interacting=self.interactions_on, dipole=complex(model.dipole),
            eps_v=eps_v, eps_c=eps_c, u_table=self.u_table, u_mid=u_mid, amp=amp,
            g_hist=g_hist, s_hist=s_hist, device=dev, multi_rank=self.world > 1,
            incremental=_incremental_default(grid.n_k))
        self.p2p = None
        if self.world > 1:
            self.p2p = _PeerExchange.setup(self.ws, self.rank, self.world)
        _lib.check(_lib.lib().kbe_init_history(self.ws.problem_ptr(), stream_ptr()), "kbe_init_history")
        self.state = TwoTimeGF(nkl, self.k_lo, capacity, step_cfg.dt, g_hist, frontier=0)
        self.sigma = SigmaHistory(s_hist, capacity)
        self._poisoned = None
        # one rank: KBE_GRAPH=1 replays kbe_run's step graph (corrector iterations behind
        # conditional nodes).  Off by default: on B200 the conditional nodes cost more
        # than the no-op launches they remove (profiles/r01/launch_modes.jsonl).
        self.use_graph = 1 if os.environ.get("KBE_GRAPH", "0") == "1" else 0
        # StepReport.timings (the reference's KernelTimers: sigma / collision / update,
        # propagator.py:328-381) from CUDA events around every launch class.  Off by
        # default: the events break the programmatic-launch overlap of the step kernels.
        self.timings_enabled = (os.environ.get("KBE_TIMINGS", "0") == "1") if timings is None else bool(timings)
        if self.world > 1:
            self.publish_initial()

    # ------------------------------------------------------------------ multi-rank plumbing
    def _gather_frontier(self) -> None:
        """All-gather the new G slice (local k) into the all-k frontier buffer (NCCL path;
        with the peer-to-peer exchange the update kernel has already stored it)."""
        if self.p2p is None:
            all_gather_device(self.ws.front_all, self.ws.front_send)

    def publish_initial(self) -> None:
        """Slice 0 (written by kbe_init_history) to every rank."""
        if self.p2p is not None:
            _lib.check(_lib.lib().kbe_p2p_publish(self.ws.problem_ptr(), stream_ptr()), "kbe_p2p_publish")
        else:
            all_gather_device(self.ws.front_all, self.ws.front_send)

    def _allreduce_hf(self) -> None:
        import torch.distributed as dist
        off = int(_lib.lib().kbe_ctl_hf_sum_offset())   # offsetof(kbe_ctl, hf_sum) from the library
        all_reduce_device(self.ws.ctl[off: off + 64].view(torch.float64), dist.ReduceOp.SUM)

    # ------------------------------------------------------------------ speculative iteration counts
    SPEC_CHUNK = 32

    def _speculative(self) -> bool:
        """Device-sequenced stream launches: launch only as many corrector iterations as the steps
        so far needed and roll back the rare step that needs more (kbe_run_iters).  The
        no-op launches of converged iterations cost ~4 % of a cfg2 step; KBE_SPECULATE=0
        launches all max_iter iterations every step."""
        # (k-sharded peer-to-peer ranks too: every rank's finish kernel sees the same merged
        # residuals, so all ranks stop, resume and continue at the same step)
        return (self._device_sequenced() and not (self.world == 1 and self.use_graph)
                and self.cfg.max_iter > 1 and os.environ.get("KBE_SPECULATE", "1") != "0")

    def _run_speculative(self, n0: int, n1: int) -> None:
        """Chunks of steps with m iterations each; the host reads each chunk's needs_more
        word one chunk behind (the GPU keeps the next chunk), and on a hit resumes that step
        with its remaining iterations (kbe_resume_step), raises m and continues after it.
        Every step's result is bitwise the full-iteration result (same kernels, same order)."""
        import collections
        L, P, sp = _lib.lib(), self.ws.problem_ptr(), stream_ptr()
        stream = torch.cuda.current_stream()
        off = int(L.kbe_ctl_needs_more_offset())
        word = self.ws.ctl[off: off + 4].view(torch.int32)
        m = max(1, min(self.cfg.max_iter, getattr(self, "_spec_m", 2)))
        # kernels per evaluation (K1, K2, [hf], [K3a], K3) for the launch count the bench reports
        per_eval = int(L.kbe_launches_per_eval(P))
        self.spec_launches = 0
        pending = collections.deque()
        n = n0
        while n <= n1 or pending:
            if n <= n1 and len(pending) < 2:
                b = min(n + self.SPEC_CHUNK - 1, n1)
                _lib.check(L.kbe_run_iters(P, n, b, m, sp), "kbe_run_iters")
                self.spec_launches += (b - n + 1) * ((1 + m) * per_eval + 1)
                buf = torch.empty(1, dtype=torch.int32, pin_memory=True)
                buf.copy_(word, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
                pending.append((m, ev, buf))
                n = b + 1
                continue
            mm, ev, buf = pending.popleft()
            ev.synchronize()
            hit = int(buf[0])
            if hit:
                stream.synchronize()          # the chunks after the hit were no-ops
                pending.clear()
                _lib.check(L.kbe_resume_step(P, hit, mm, sp), "kbe_resume_step")
                self.spec_launches += (self.cfg.max_iter - mm) * per_eval + 1
                m = min(self.cfg.max_iter, mm + 1)
                n = hit + 1
        self._spec_m = m

    def _device_sequenced(self) -> bool:
        """One rank, or peer-to-peer shards without hf: the whole step is one C call."""
        return self.world == 1 or (self.p2p is not None and self.model.hf_mode != "on")

    def _launch_step(self, n: int) -> None:
        L, P, st = _lib.lib(), self.ws.problem_ptr(), stream_ptr()
        if self._device_sequenced():
            _lib.check(L.kbe_run(P, n, n, self.use_graph if self.world == 1 else 0, st), "kbe_run")
            return
        # k-sharded step: same launch sequence, with one NCCL all-gather after every
        # update.  It carries the new G slice (the Sigma input needs all k) and each
        # rank's convergence record, which every kernel max-reduces over ranks itself.
        chk = _lib.check
        nold = n - 1
        if self.interactions_on:
            chk(L.kbe_sigma_frontier(P, nold, 0, st), "kbe_sigma_frontier")
        chk(L.kbe_collision_frontier(P, nold, 0, st), "kbe_collision_frontier")
        if self.model.hf_mode == "on":
            chk(L.kbe_hf_mean(P, n, 0, 0, st), "kbe_hf_mean")
            self._allreduce_hf()
            chk(L.kbe_build_phi(P, n, 0, st), "kbe_build_phi")
        chk(L.kbe_update(P, n, 0, 0, st), "kbe_update")
        self._gather_frontier()
        for it in range(self.cfg.max_iter):
            if self.interactions_on:
                chk(L.kbe_sigma_frontier(P, n, it, st), "kbe_sigma_frontier")
            chk(L.kbe_collision_frontier(P, n, it, st), "kbe_collision_frontier")
            if self.model.hf_mode == "on":
                chk(L.kbe_hf_mean(P, n, 1, it, st), "kbe_hf_mean")
                self._allreduce_hf()
                chk(L.kbe_build_phi(P, n, it, st), "kbe_build_phi")
            chk(L.kbe_update(P, n, 1, it, st), "kbe_update")
            self._gather_frontier()
        chk(L.kbe_finish_step(P, n, st), "kbe_finish_step")

    def _launch_step_timed(self, n: int) -> list:
        """The step's launches host-sequenced (kbe_step's order) with a CUDA event before
        each class -- Sigma, collision, update ([hf] + [K3a] + K3) -- and after the last;
        the finish kernel is timed into the last update.  Returns, per evaluation
        ci = 0 (predictor, frontier n-1) .. max_iter, the event tuple."""
        L, P, st = _lib.lib(), self.ws.problem_ptr(), stream_ptr()
        stream = torch.cuda.current_stream()
        chk = _lib.check

        def ev():
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            return e
        out = []
        calls = [(n - 1, 0, 0)] + [(n, 1, it) for it in range(self.cfg.max_iter)]
        for ci, (nf, phase, it) in enumerate(calls):
            e0 = ev()
            if self.interactions_on:
                chk(L.kbe_sigma_frontier(P, nf, it, st), "kbe_sigma_frontier")
            e1 = ev()
            chk(L.kbe_collision_frontier(P, nf, it, st), "kbe_collision_frontier")
            e2 = ev()
            if self.model.hf_mode == "on":
                chk(L.kbe_hf_mean(P, n, phase, it, st), "kbe_hf_mean")
                if self.world > 1:
                    self._allreduce_hf()
                    chk(L.kbe_build_phi(P, n, it, st), "kbe_build_phi")
            chk(L.kbe_update(P, n, phase, it, st), "kbe_update")
            if self.world > 1:
                self._gather_frontier()
            if ci == len(calls) - 1:
                chk(L.kbe_finish_step(P, n, st), "kbe_finish_step")
            out.append((e0, e1, e2, ev()))
        return out

    @staticmethod
    def _fill_timings(reports: list, events: list) -> None:
        """Seconds per class over the evaluations that did work (the predictor's and the
        corrector iterations up to the step's count; later launches were no-ops)."""
        torch.cuda.synchronize()
        for rep, evs in zip(reports, events):
            t = {"sigma": 0.0, "collision": 0.0, "update": 0.0}
            for ci, (e0, e1, e2, e3) in enumerate(evs):
                if ci > rep.iterations and ci < len(evs) - 1:
                    continue
                if ci <= rep.iterations:
                    t["sigma"] += e0.elapsed_time(e1) * 1e-3
                    t["collision"] += e1.elapsed_time(e2) * 1e-3
                    t["update"] += e2.elapsed_time(e3) * 1e-3
                else:   # the last (no-op) evaluation: only its finish kernel counts
                    t["update"] += e2.elapsed_time(e3) * 1e-3
            rep.timings = t

    # ------------------------------------------------------------------ reports
    def _reports(self, n0: int, n1: int) -> np.ndarray:
        rows = self.ws.reports[n0: n1 + 1].contiguous()
        if self.world > 1:
            parts = all_gather_list(rows, self.world)
            return combine_reports(np.stack([to_host(p) for p in parts]))
        return to_host(rows)

    def _to_report(self, row: np.ndarray) -> StepReport:
        it = int(row[1])
        return StepReport(
            step=int(row[0]), iterations=it, residual=float(row[2]), converged=bool(row[3]),
            anticommutation_drift=float(row[4]), density=float(row[5]) / self.grid.n_k,
            residual_history=[float(x) for x in row[8: 8 + it]], timings={},
            energy=self._energy(row),
        )

    def _energy(self, row: np.ndarray) -> float:
        """Report row -> energy: the device's k-sum of Re Tr[h0 rho] plus, with
        hf_mode="on", n_k Tr[hf m] for m the k-mean of rho (hartree_fock, model.py:106-120:
        hf is the same for every k, so its energy only needs m)."""
        nk = self.grid.n_k
        e = float(row[7])
        if self.model.hf_mode == "on":
            r0 = 8 + _lib.MAX_ITER
            m00, m11 = row[r0] / nk, row[r0 + 1] / nk
            m01 = complex(row[r0 + 2], row[r0 + 3]) / nk
            u = float(self.u_table[int(row[0])])
            # Tr[hf m] = u m11 m00 - u m01 m10 - u m10 m01 + u m00 m11, m10 = conj(m01)
            e += nk * float((u * m11 * m00 - u * m01 * np.conj(m01) - u * np.conj(m01) * m01 + u * m00 * m11).real)
        return e / nk

    def _precheck(self, n: int) -> None:
        if n > self.capacity:
            raise CapacityError(f"step {n} exceeds allocated capacity n_steps={self.capacity}")
        if self._poisoned is not None:
            raise PoisonedStateError(f"non-finite values on the frontier at step {self.state.frontier}")

    # ------------------------------------------------------------------ API
    def step(self) -> StepReport:
        """One time step (propagator.py:316-382); synchronises to return its report."""
        n = self.state.frontier + 1
        self._precheck(n)
        events = [self._launch_step_timed(n)] if self.timings_enabled else None
        if events is None:
            self._launch_step(n)
        row = self._reports(n, n)[0]
        self.state.frontier = n
        if row[6] != 0.0:
            self._poisoned = n
            raise PoisonedStateError(f"non-finite values produced at step {n}")
        rep = self._to_report(row)
        if events is not None:
            self._fill_timings([rep], events)
        return rep

    def run(self, observer=None) -> list:
        """Advance n_steps steps (propagator.py:384-392).

        Without an observer all steps are launched back to back and the
        reports are read once; with one, each step synchronises so the
        observer sees the live state (as in the reference).
        """
        if observer is not None:
            reports = []
            for _ in range(self.cfg.n_steps):
                rep = self.step()
                reports.append(rep)
                observer(self.state, rep)
            return reports
        n0 = self.state.frontier + 1
        last = self.state.frontier + self.cfg.n_steps
        if self.cfg.n_steps == 0:
            return []
        self._precheck(n0)
        n1 = min(last, self.capacity)
        events = None
        if self.timings_enabled:
            events = [self._launch_step_timed(n) for n in range(n0, n1 + 1)]
        elif self._speculative():
            self._run_speculative(n0, n1)
        elif self._device_sequenced():
            _lib.check(_lib.lib().kbe_run(self.ws.problem_ptr(), n0, n1, self.use_graph if self.world == 1 else 0,
                                          stream_ptr()), "kbe_run")
        else:
            for n in range(n0, n1 + 1):
                self._launch_step(n)
        if self.p2p is not None:
            self.p2p.check(self.p2p.nbytes)
        rows = self._reports(n0, n1)
        reports = []
        for row in rows:
            n = int(round(row[0])) if row[0] else None
            if n is None:      # step never ran (device poisoned earlier)
                break
            if row[6] != 0.0:
                self.state.frontier = n
                self._poisoned = n
                raise PoisonedStateError(f"non-finite values produced at step {n}")
            reports.append(self._to_report(row))
        if events is not None:
            self._fill_timings(reports, events)
        self.state.frontier = n1
        if last > self.capacity:
            raise CapacityError(f"step {self.capacity + 1} exceeds allocated capacity n_steps={self.capacity}")
        return reports

    def synchronize(self) -> None:
        torch.cuda.current_stream().synchronize()

    def close(self) -> None:
        """Release the peer-exchange mappings once every rank is done with them
        (collective when k-sharded)."""
        if getattr(self, "p2p", None) is None:
            return
        import torch.distributed as dist
        torch.cuda.synchronize()
        if dist.is_initialized():
            dist.barrier()
        self.p2p.close()
        self.p2p = None

    def __del__(self):
        if getattr(self, "p2p", None) is not None:
            self.p2p.close(free_local=False)   # no collective here: see close()
        ws = getattr(self, "ws", None)
        if ws is not None and getattr(self, "use_graph", 0):
            try:
                _lib.lib().kbe_release(ws.problem_ptr())
            except Exception:
                pass


def run(grid: KGrid, model: ModelConfig, step_cfg: StepConfig, schedule: Schedule | None = None,
        pool: WorkerPool | None = None, observer=None):
    """Propagate a fresh state for step_cfg.n_steps steps (propagator.py:395-406)."""
    driver = PropagationDriver(grid, model, step_cfg, schedule, pool)
    reports = driver.run(observer=observer)
    driver.close()
    return driver.state, reports
