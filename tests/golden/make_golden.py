"""Generate golden vectors by running the REAL reference (kbesolve 0.1.0).

Run in the build container (the reference sources are at /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

or on any host that has the unmodified reference installed, e.g. the GPU box's 16
cores with the driver's offline install (long runs; this is how the 120-step cfg5
fixture was made, profiles/r02/cfg5_golden_gpubox.log):

    KBE_REFERENCE_SRC=$PWD/baseline/_ref KBE_GOLDEN_OUT=gpurun_out KBE_GOLDEN_WORKERS=16 \
        KBE_GOLDEN_SHARDS=1 python tests/golden/make_golden.py cfg5

Runs longer than one call are chained (long_fixture's checkpoint/resume): each call runs
until a deadline and saves the reference driver's state on the box's /tmp, the next call
(on the same box, started within minutes) resumes from it:

    KBE_GOLDEN_CKPT=/tmp/kbe_cfg3_ckpt KBE_GOLDEN_DEADLINE=3000 KBE_GOLDEN_WORKERS=16 \
        KBE_GOLDEN_SHARDS=16 KBE_REFERENCE_SRC=$PWD/baseline/_ref python tests/golden/make_golden.py cfg3

Writes ``tests/golden/*.npz``.  Every fixture stores its inputs alongside
the reference outputs, so tests never need the reference (or a particular
numpy RNG) at run time.  The reference is deterministic bitwise (SURVEY
probe P5), so re-running this script reproduces the same bytes.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("KBE_REFERENCE_SRC", "/root/reference/pkg/src"))

import kbesolve as kb  # noqa: E402
from kbesolve.state import mirror_frontier  # noqa: E402


def _save(name, **arrays):
    # KBE_GOLDEN_OUT: write somewhere else (a long checkpointed run must not overwrite
    # a longer committed prefix with its first checkpoints)
    out_dir = os.environ.get("KBE_GOLDEN_OUT", HERE)
    os.makedirs(out_dir, exist_ok=True)
    path = os.path.join(out_dir, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


def sigma_fixture():
    out = {}
    for n_k in (2, 4, 8, 16, 32, 64):
        grid = kb.build_kgrid(n_k)
        rng = np.random.default_rng(100 + n_k)
        shape = (n_k, 2, 2, 5)
        gl = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        gg = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        u1 = np.linspace(0.4, 1.2, 5)
        u2 = 0.7
        pol = kb.polarizability(gl, gg, grid)
        s1 = kb.sigma_first(pol, gl, u1, u2, grid)
        s2 = kb.sigma_second(gl, gg, u1, u2, grid)
        out[f"gl_{n_k}"] = gl
        out[f"gg_{n_k}"] = gg
        out[f"u1_{n_k}"] = u1
        out[f"u2_{n_k}"] = np.array(u2)
        out[f"pol_{n_k}"] = pol
        out[f"s1_{n_k}"] = s1
        out[f"s2_{n_k}"] = s2
        out[f"sigma_{n_k}"] = kb.sigma_slice(gl, gg, u1, u2, grid)
        # k-range (shard) evaluation
        out[f"sigma_shard_{n_k}"] = kb.sigma_slice(gl, gg, u1, u2, grid, (n_k // 2, n_k))
    _save("sigma.npz", **out)


def _random_history(n_k, cap, frontier, seed, dt):
    """Random G and Sigma histories with the reference's mirror structure."""
    grid = kb.build_kgrid(n_k)
    rng = np.random.default_rng(seed)
    state = kb.init_state(grid, cap, dt)
    shape = state.lesser.shape
    state.lesser[:] = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    state.greater[:] = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    state.frontier = frontier
    for n in range(frontier + 1):
        mirror_frontier(state, n)
    sigma = kb.init_sigma_history(n_k, cap)
    sigma.lesser[:] = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    sigma.greater[:] = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    for n in range(1, frontier + 1):
        # evaluate_sigma_batched stores Sigma< on columns, Sigma> on rows and
        # mirrors the rest (selfenergy.py:317-325)
        sigma.lesser[:, :, :, n, :n] = -np.conj(np.swapaxes(sigma.lesser[:, :, :, :n, n], 1, 2))
        sigma.greater[:, :, :, :n, n] = -np.conj(np.swapaxes(sigma.greater[:, :, :, n, :n], 1, 2))
    return grid, state, sigma


def collision_fixture():
    out = {}
    n_k, cap, frontier, dt = 4, 9, 8, 0.05
    grid, state, sigma = _random_history(n_k, cap, frontier, 200, dt)
    out["GL"] = state.lesser
    out["GG"] = state.greater
    out["SL"] = sigma.lesser
    out["SG"] = sigma.greater
    out["dt"] = np.array(dt)
    for kind in ("trapezoid", "simpson"):
        for mode in ("as-printed", "langreth"):
            for n in (0, 1, 2, 5, 8):
                c = kb.collision_frontier(state, sigma, n, kb.QuadratureRule(kind), None, mode)
                tag = f"{kind}_{mode}_{n}"
                out[f"lr_{tag}"] = c.lesser_row
                out[f"gr_{tag}"] = c.greater_row
                out[f"lc_{tag}"] = c.lesser_col
                out[f"gc_{tag}"] = c.greater_col
    # per-pair oracle entries (collision.py:115-138)
    out["pair_lesser_k1_i5_l2"] = kb.collision_lesser(state, sigma, 1, 5, 2)
    out["pair_greater_k2_i3_l6"] = kb.collision_greater(state, sigma, 2, 3, 6)
    for n in (0, 3, 8):
        w = kb.quadrature_weights(n, dt, "simpson")
        out[f"wsimp_{n}"] = w
        out[f"wtrap_{n}"] = kb.quadrature_weights(n, dt, "trapezoid")
    for n in (1, 2, 7, 10):
        out[f"wsimp_{n}"] = kb.quadrature_weights(n, dt, "simpson")
        out[f"wtrap_{n}"] = kb.quadrature_weights(n, dt, "trapezoid")
    _save("collision.npz", **out)


def sigma_batched_fixture():
    out = {}
    n_k, cap, frontier, dt = 8, 7, 6, 0.05
    grid, state, _ = _random_history(n_k, cap, frontier, 300, dt)
    u = np.linspace(0.4, 0.9, cap + 1)
    out["GL"] = state.lesser
    out["GG"] = state.greater
    out["u"] = u
    for n in (0, 3, 6):
        sig = kb.init_sigma_history(n_k, cap)
        kb.evaluate_sigma_batched(state, sig, n, grid, u)
        out[f"SL_{n}"] = sig.lesser
        out[f"SG_{n}"] = sig.greater
    _save("sigma_batched.npz", **out)


def _run_fixture(name, n_k, model, step_cfg, full=False, rows_every=None, schedule=None):
    grid = kb.build_kgrid(n_k)
    t0 = time.time()
    drv = kb.PropagationDriver(grid, model, step_cfg, schedule)
    reps = drv.run()
    el = time.time() - t0
    N = step_cfg.n_steps
    st = drv.state
    idx = np.arange(N + 1)
    out = {
        "n_k": np.array(n_k),
        "dt": np.array(step_cfg.dt),
        "n_steps": np.array(N),
        "eps": np.array(step_cfg.eps),
        "max_iter": np.array(step_cfg.max_iter),
        "quadrature": np.array(step_cfg.quadrature),
        "limit_mode": np.array(step_cfg.limit_mode),
        "band_gap": np.array(model.band_gap),
        "hopping": np.array(model.hopping),
        "u_protocol": np.asarray(model.u_protocol, dtype=float),
        "pulse_intensity": np.array(model.pulse_intensity),
        "pulse_center": np.array(model.pulse_center),
        "dipole": np.array(complex(model.dipole)),
        "hf_mode": np.array(model.hf_mode),
        "iterations": np.array([r.iterations for r in reps]),
        "residual": np.array([r.residual for r in reps]),
        "converged": np.array([r.converged for r in reps]),
        "drift": np.array([r.anticommutation_drift for r in reps]),
        "density": np.array([r.density for r in reps]),
        "diag_lesser": st.lesser[:, :, :, idx, idx],
        "diag_greater": st.greater[:, :, :, idx, idx],
        "final_row_lesser": st.lesser[:, :, :, N, :],
        "final_col_greater": st.greater[:, :, :, :, N],
        "ref_seconds": np.array(el),
    }
    if model.eps_c_table is not None:
        out["eps_c_table"] = np.asarray(model.eps_c_table)
        out["eps_v_table"] = np.asarray(model.eps_v_table)
    if full:
        out["GL"] = st.lesser
        out["GG"] = st.greater
        out["SL"] = drv.sigma.lesser
        out["SG"] = drv.sigma.greater
    if rows_every:
        steps = np.arange(0, N + 1, rows_every)
        out["row_steps"] = steps
        out["rows_lesser"] = np.stack([st.lesser[:, :, :, s, :] for s in steps])
        out["cols_greater"] = np.stack([st.greater[:, :, :, :, s] for s in steps])
    _save(name, **out)
    print(f"  {name}: reference run {el:.1f}s, iterations {np.bincount(out['iterations'])}")


def trajectory_fixtures():
    # cfg1: the Hubbard dimer exactly as BASELINE.json names it
    _run_fixture(
        "traj_dimer.npz", 2,
        kb.ModelConfig(u_protocol=1.0, pulse_intensity=0.2, pulse_center=0.5),
        kb.StepConfig(dt=0.02, n_steps=200), rows_every=25,
    )
    # small full-history run with an early pulse (every stored array pinned)
    _run_fixture(
        "traj_nk4_full.npz", 4,
        kb.ModelConfig(u_protocol=1.0, pulse_intensity=0.2, pulse_center=0.1),
        kb.StepConfig(dt=0.02, n_steps=30), full=True,
    )
    # options: Hartree-Fock, Simpson, Langreth limit, time-dependent U
    u_ramp = np.linspace(0.5, 1.5, 21)
    _run_fixture(
        "traj_hf.npz", 4,
        kb.ModelConfig(u_protocol=1.0, pulse_intensity=0.3, pulse_center=0.1, hf_mode="on"),
        kb.StepConfig(dt=0.02, n_steps=20), full=True,
    )
    _run_fixture(
        "traj_simpson.npz", 4,
        kb.ModelConfig(u_protocol=u_ramp, pulse_intensity=0.3, pulse_center=0.1),
        kb.StepConfig(dt=0.02, n_steps=20, quadrature="simpson"), full=True,
    )
    _run_fixture(
        "traj_langreth.npz", 4,
        kb.ModelConfig(u_protocol=1.0, pulse_intensity=0.3, pulse_center=0.1, dipole=0.8 + 0.3j),
        kb.StepConfig(dt=0.02, n_steps=20, limit_mode="langreth"), full=True,
    )
    # cfg2 prefix (n_k=16), past the pulse at step 25
    _run_fixture(
        "traj_nk16.npz", 16,
        kb.ModelConfig(u_protocol=1.0, pulse_intensity=0.2, pulse_center=0.5),
        kb.StepConfig(dt=0.02, n_steps=40), rows_every=10,
    )
    # cfg3 synthetic tables, prefix with the pulse moved early
    rng = np.random.default_rng(7)
    eps_c = 1.0 + rng.uniform(0.0, 1.0, 64)
    u_tab = 1.0 + 0.1 * rng.standard_normal(1001)
    _run_fixture(
        "traj_nk64_synth.npz", 64,
        kb.ModelConfig(u_protocol=u_tab, pulse_intensity=0.2, pulse_center=0.1,
                       eps_c_table=eps_c, eps_v_table=-eps_c),
        kb.StepConfig(dt=0.02, n_steps=12, memory_budget=4 * 1024**3), rows_every=4,
        schedule=kb.Schedule(n_shards=8),
    )
    # free evolution (U = 0, no pulse): analytic known answer
    _run_fixture(
        "traj_free.npz", 16, kb.ModelConfig(),
        kb.StepConfig(dt=0.02, n_steps=100), rows_every=50,
    )


def cfg2_full_fixture():
    """The bench workload itself (BASELINE configs[1]) run by the REAL reference:
    n_k=16, 1000 steps, U=0.5 (U=1 diverges at step 667 in the reference's own
    scheme), pulse 0.2 at t=0.5.  k-sharded over 6 worker threads
    (bitwise identical to 1 shard, SURVEY probe P5).  Stores the final row/column,
    the equal-time diagonals and the per-step observables."""
    n_k, N = 16, 1000
    grid = kb.build_kgrid(n_k)
    model = kb.ModelConfig(u_protocol=0.5, pulse_intensity=0.2, pulse_center=0.5)
    cfg = kb.StepConfig(dt=0.02, n_steps=N, memory_budget=8 * 1024**3)
    workers = int(os.environ.get("KBE_GOLDEN_WORKERS", "6"))
    shards = 8 if workers >= 8 else (4 if workers >= 4 else 1)
    pool = kb.WorkerPool(workers)
    t0 = time.time()
    drv = kb.PropagationDriver(grid, model, cfg, kb.Schedule(n_shards=shards, workers=workers), pool)
    reps = []
    for n in range(1, N + 1):
        reps.append(drv.step())
        if n % 50 == 0:
            print(f"  cfg2 step {n} {time.time() - t0:.0f}s", flush=True)
    st = drv.state
    idx = np.arange(N + 1)
    _save("traj_cfg2_full.npz",
          n_k=np.array(n_k), n_steps=np.array(N), dt=np.array(0.02), u=np.array(0.5),
          pulse_intensity=np.array(0.2), pulse_center=np.array(0.5),
          iterations=np.array([r.iterations for r in reps]),
          drift=np.array([r.anticommutation_drift for r in reps]),
          density=np.array([r.density for r in reps]),
          diag_lesser=st.lesser[:, :, :, idx, idx],
          final_row_lesser=st.lesser[:, :, :, N, :],
          final_col_greater=st.greater[:, :, :, :, N],
          ref_seconds=np.array(time.time() - t0))


def _synth_tables(n_k, n_steps, u):
    """cfg3's synthetic system, the same draws as bench.model_kwargs:
    eps_c = 1 + U(0,1), eps_v = -eps_c, U(t) = u (1 + 0.1 N(0,1)), default_rng(7)."""
    rng = np.random.default_rng(7)
    eps_c = 1.0 + rng.uniform(0.0, 1.0, n_k)
    u_tab = u * (1.0 + 0.1 * rng.standard_normal(n_steps + 1))
    return eps_c, u_tab


# Long reference runs at the bench workloads' sizes.  name -> (file, n_k, N, model kwargs,
# rows_k, rows_every).  U per workload as bench.WORKLOADS states it: cfg3's
# tables at scale 0.75 (scale 1.0 diverges at step 868, 0.9 at step 987), cfg4 U = 0.2
# (its 4000-step workload; 0.25 diverges at 3778), cfg5 U = 1.0 (finite for 500 steps).
LONG_RUNS = {
    "cfg3": ("traj_cfg3_full.npz", 64, 1000, "synth", 0.75),
    "cfg4": ("traj_cfg4_prefix.npz", 32, 400, "plain", 0.2),
    "cfg5": ("traj_cfg5_prefix.npz", 128, 120, "plain", 1.0),
}


def _ckpt_save(ck, drv, n, acc):
    """Resumable state of the reference driver after step n: the filled [0..n] blocks of
    G<, G>, Sigma<, Sigma> (everything PropagationDriver.step reads from earlier steps,
    propagator.py:316-382; its ScratchPool only holds overwritten buffers) and the
    fixture's accumulators.  Written to a temp dir, then renamed (atomic)."""
    import shutil
    tmp = ck + ".tmp"
    shutil.rmtree(tmp, ignore_errors=True)
    os.makedirs(tmp)
    for name, arr in (("GL", drv.state.lesser), ("GG", drv.state.greater),
                      ("SL", drv.sigma.lesser), ("SG", drv.sigma.greater)):
        np.save(os.path.join(tmp, name + ".npy"), arr[..., : n + 1, : n + 1])
    extra = {f"acc_{k}": np.asarray(v) for k, v in acc.items() if not k.startswith("rc_")}
    for k, v in acc.items():
        if k.startswith("rc_"):
            extra[k] = v
    np.savez(os.path.join(tmp, "acc.npz"), n=np.array(n), **extra)
    shutil.rmtree(ck, ignore_errors=True)
    os.rename(tmp, ck)
    print(f"  checkpoint at step {n} -> {ck}", flush=True)


def _ckpt_load(ck, drv):
    """Restore _ckpt_save's state into a fresh driver; returns (n, accumulators)."""
    d = np.load(os.path.join(ck, "acc.npz"))
    n = int(d["n"])
    for name, arr in (("GL", drv.state.lesser), ("GG", drv.state.greater),
                      ("SL", drv.sigma.lesser), ("SG", drv.sigma.greater)):
        arr[..., : n + 1, : n + 1] = np.load(os.path.join(ck, name + ".npy"))
    drv.state.frontier = n
    acc = {k[4:]: list(d[k]) for k in d.files if k.startswith("acc_")}
    acc.update({k: d[k] for k in d.files if k.startswith("rc_")})
    return n, acc


def long_fixture(which):
    """A bench workload run by the REAL reference, checkpointed: every
    KBE_GOLDEN_SAVE_EVERY steps (default 50) the prefix computed so far is written,
    so an interrupted run still leaves a usable golden.  Stores the per-step
    observables, the equal-time diagonals, the final row G<(t_s, .) and column
    G>(., t_s), and rows/columns of a few k every 100 steps.

    Resumable (runs longer than one session or one GPU-box call): with
    KBE_GOLDEN_CKPT=<dir> the driver state is saved there when KBE_GOLDEN_DEADLINE
    seconds have passed (or at step KBE_GOLDEN_STOP_AT) and the run exits; a later run
    with the same directory continues from it.  The continuation is bitwise the
    uninterrupted run (tests/golden/make_golden.py resume_check)."""
    fname, n_k, N, kind, u = LONG_RUNS[which]
    N = int(os.environ.get("KBE_GOLDEN_STEPS", N))
    if which not in LONG_RUNS_TARGET:
        LONG_RUNS_TARGET[which] = LONG_RUNS[which][2]
    grid = kb.build_kgrid(n_k)
    kw = dict(pulse_intensity=0.2, pulse_center=0.5)
    if kind == "synth":
        eps_c, u_tab = _synth_tables(n_k, LONG_RUNS[which][2], u)
        kw.update(u_protocol=u_tab, eps_c_table=eps_c, eps_v_table=-eps_c)
    else:
        kw.update(u_protocol=u)
    model = kb.ModelConfig(**kw)
    cfg = kb.StepConfig(dt=0.02, n_steps=N, memory_budget=1 << 40)
    workers = int(os.environ.get("KBE_GOLDEN_WORKERS", "6"))
    shards = max(d for d in range(1, min(workers, n_k) + 1) if n_k % d == 0)
    # KBE_GOLDEN_SHARDS: fewer shards replicate less work per step (each shard
    # recomputes the polarizability, selfenergy.py:292); the results are bitwise
    # independent of the shard count (SURVEY probe P5)
    shards = int(os.environ.get("KBE_GOLDEN_SHARDS", shards))
    pool = kb.WorkerPool(workers)
    every = int(os.environ.get("KBE_GOLDEN_SAVE_EVERY", "50"))
    ck = os.environ.get("KBE_GOLDEN_CKPT")
    deadline = float(os.environ.get("KBE_GOLDEN_DEADLINE", "inf"))
    stop_at = int(os.environ.get("KBE_GOLDEN_STOP_AT", "0"))
    rows_k = np.arange(0, n_k, max(1, n_k // 4))
    t0 = time.time()
    drv = kb.PropagationDriver(grid, model, cfg, kb.Schedule(n_shards=shards, workers=workers), pool)
    acc = dict(iterations=[], residual=[], drift=[], density=[], row_steps=[], seconds=[0.0])
    n0 = 0
    if ck and not os.path.exists(os.path.join(ck, "acc.npz")) and os.path.exists(os.path.join(ck + ".tmp", "acc.npz")):
        os.rename(ck + ".tmp", ck)   # killed between the (complete) temp write and the rename
    if ck and os.path.exists(os.path.join(ck, "acc.npz")):
        n0, acc = _ckpt_load(ck, drv)
        print(f"  resumed {which} at step {n0}", flush=True)
    rows = [acc[f"rc_rows_{s}"] for s in acc["row_steps"]]
    cols = [acc[f"rc_cols_{s}"] for s in acc["row_steps"]]
    sec0 = float(acc["seconds"][0])
    for n in range(n0 + 1, N + 1):
        r = drv.step()
        acc["iterations"].append(r.iterations)
        acc["residual"].append(r.residual)
        acc["drift"].append(r.anticommutation_drift)
        acc["density"].append(r.density)
        st = drv.state
        if n % 100 == 0:
            acc["row_steps"].append(n)
            rows.append(st.lesser[rows_k, :, :, n, : n + 1].copy())
            cols.append(st.greater[rows_k, :, :, : n + 1, n].copy())
        stop = n < N and ((time.time() - t0) > deadline or n == stop_at)
        if n % every == 0 or n == N or stop:
            idx = np.arange(n + 1)
            out = dict(
                n_k=np.array(n_k), n_steps=np.array(n), target_steps=np.array(LONG_RUNS[which][2]),
                dt=np.array(0.02), u=np.array(u), pulse_intensity=np.array(0.2), pulse_center=np.array(0.5),
                u_protocol=np.asarray(model.u_protocol, dtype=float),
                iterations=np.array(acc["iterations"]),
                residual=np.array(acc["residual"]),
                drift=np.array(acc["drift"]),
                density=np.array(acc["density"]),
                diag_lesser=st.lesser[:, :, :, idx, idx],
                diag_greater=st.greater[:, :, :, idx, idx],
                final_row_lesser=st.lesser[:, :, :, n, : n + 1],
                final_col_greater=st.greater[:, :, :, : n + 1, n],
                rows_k=rows_k, row_steps=np.array(acc["row_steps"], dtype=int),
                ref_seconds=np.array(sec0 + time.time() - t0), workers=np.array(workers), shards=np.array(shards),
            )
            for s_, r_, c_ in zip(acc["row_steps"], rows, cols):
                out[f"rows_lesser_{s_}"] = r_
                out[f"cols_greater_{s_}"] = c_
            if kind == "synth":
                out["eps_c_table"] = np.asarray(model.eps_c_table)
            _save(fname, **out)
            print(f"  {which} step {n} {sec0 + time.time() - t0:.0f}s", flush=True)
        if stop and ck:
            acc["seconds"] = [sec0 + time.time() - t0]
            for s_, r_, c_ in zip(acc["row_steps"], rows, cols):
                acc[f"rc_rows_{s_}"] = r_
                acc[f"rc_cols_{s_}"] = c_
            _ckpt_save(ck, drv, n, acc)
            return


LONG_RUNS_TARGET = {}


def resume_check_fixture():
    """Bitwise check of the checkpoint/resume path on a small workload: n_k = 4, 210 steps
    straight vs 117 + resume + 93, across the 100-step row snapshots (raises on any difference)."""
    import shutil
    import tempfile
    LONG_RUNS["_rc"] = ("_resume_check.npz", 4, 210, "plain", 1.0)
    base = tempfile.mkdtemp()
    os.environ["KBE_GOLDEN_OUT"] = os.path.join(base, "a")
    long_fixture("_rc")
    os.environ["KBE_GOLDEN_OUT"] = os.path.join(base, "b")
    os.environ["KBE_GOLDEN_CKPT"] = os.path.join(base, "ck")
    os.environ["KBE_GOLDEN_STOP_AT"] = "117"
    long_fixture("_rc")
    os.environ.pop("KBE_GOLDEN_STOP_AT")
    long_fixture("_rc")
    a = np.load(os.path.join(base, "a", "_resume_check.npz"))
    b = np.load(os.path.join(base, "b", "_resume_check.npz"))
    for k in a.files:
        if k in ("ref_seconds",):
            continue
        if not np.array_equal(a[k], b[k]):
            raise AssertionError(f"resume differs in {k}")
    print("resume_check: bitwise identical over", list(a.files))
    shutil.rmtree(base)


def cfg3_fixture():
    long_fixture("cfg3")


def cfg4_fixture():
    long_fixture("cfg4")


def cfg5_fixture():
    long_fixture("cfg5")


def energy_fixture():
    """One-body energy E(t_n) = (1/n_k) sum_k Re Tr[h(k; t_n) rho(k; t_n)] of the stored
    reference trajectories, with the REFERENCE's own build_h (model.py:123-152, hf term
    included) at every grid point and rho = -i G<(t_n, t_n) from the golden diagonals
    (propagator.py:272-273).  The reference has no energy observable (SURVEY finding 2);
    this pins the derived one to its Hamiltonian."""
    out = {}
    names = ["traj_dimer.npz", "traj_hf.npz", "traj_langreth.npz", "traj_nk64_synth.npz", "traj_simpson.npz",
             "traj_nk4_full.npz", "traj_cfg2_full.npz"]
    for name in names:
        z = np.load(os.path.join(HERE, name))
        n_k, N = int(z["n_k"]), int(z["n_steps"])
        if "band_gap" in z:
            kw = dict(band_gap=float(z["band_gap"]), hopping=float(z["hopping"]),
                      u_protocol=(np.asarray(z["u_protocol"]) if np.asarray(z["u_protocol"]).ndim
                                  else float(z["u_protocol"])),
                      pulse_intensity=float(z["pulse_intensity"]), pulse_center=float(z["pulse_center"]),
                      dipole=complex(z["dipole"]), hf_mode=str(z["hf_mode"]))
            if "eps_c_table" in z:
                kw.update(eps_c_table=np.asarray(z["eps_c_table"]), eps_v_table=np.asarray(z["eps_v_table"]))
        else:   # traj_cfg2_full: model defaults + u, pulse
            kw = dict(u_protocol=float(z["u"]), pulse_intensity=float(z["pulse_intensity"]),
                      pulse_center=float(z["pulse_center"]))
        model = kb.ModelConfig(**kw)
        dt = float(z["dt"])
        grid = kb.build_kgrid(n_k)
        table = kb.u_values(model, N)
        gl = np.asarray(z["diag_lesser"])                  # (n_k, 2, 2, N+1)
        e = np.empty(N + 1)
        for n in range(N + 1):
            rho = -1j * gl[:, :, :, n]
            h = kb.build_h(grid, model, n * dt, rho, dt, table)
            e[n] = float(np.mean(np.einsum("kab,kba->k", h, rho).real))
        out[name.replace(".npz", "")] = e
    _save("energy.npz", **out)


def collision_row_fixture():
    """collision.collision_row (collision.py:141-162) on random inputs: vector and
    (T, P) matrix second-term weights, first-term weights shorter than T."""
    from kbesolve.collision import collision_row
    rng = np.random.default_rng(41)
    out = {}
    for tag, (n_k, T, P) in {"a": (2, 7, 3), "b": (4, 33, 5), "c": (16, 129, 2)}.items():
        def c(*shape):
            return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        # the t axis of dg_first / g_first is the weight length (reference einsum shapes)
        w1 = kb.quadrature_weights(T - 2, 0.02)            # length T-1 < T
        w2v = kb.quadrature_weights(T - 3, 0.02, "simpson")  # length T-2
        w2m = rng.uniform(0.0, 0.02, (T, P))
        dg, gv, gm = c(n_k, 2, 2, T - 1), c(n_k, 2, 2, T - 2), c(n_k, 2, 2, T)
        sl, so = c(n_k, 2, 2, T, P), c(n_k, 2, 2, T, P)
        for k, v in dict(dg=dg, gv=gv, gm=gm, sl=sl, so=so, w1=w1, w2v=w2v, w2m=w2m).items():
            out[f"{k}_{tag}"] = v
        out[f"vec_{tag}"] = collision_row(dg, gv, sl, so, w1, w2v)
        out[f"mat_{tag}"] = collision_row(dg, gm, sl, so, w1, w2m)
    _save("collision_row.npz", **out)


def reducers_fixture():
    """engine.chunk_partial_sums / tree_reduce / sequential_reduce (engine.py:141-202)."""
    from kbesolve import engine as E
    rng = np.random.default_rng(43)
    out = {}
    for tag, (shape, axis, bs) in {"a": ((3, 1000), -1, 128), "b": ((7, 5, 33), 1, 4), "c": ((300,), 0, 7)}.items():
        x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        out[f"x_{tag}"] = x
        out[f"meta_{tag}"] = np.array([axis, bs])
        out[f"chunks_{tag}"] = E.chunk_partial_sums(x, bs, axis)
        out[f"tree_{tag}"], rounds = E.tree_reduce(x, axis, return_rounds=True)
        out[f"rounds_{tag}"] = np.array(rounds)
        out[f"seq_{tag}"] = E.sequential_reduce(x, axis)
    _save("reducers.npz", **out)


CLI_CONFIG = {"n_k": 4, "dt": 0.02, "n_steps": 30, "u": 1.0, "pulse_intensity": 0.2, "pulse_center": 0.1}


CLI_CONFIG_OPTS = {"n_k": 4, "dt": 0.02, "n_steps": 24, "u": [1.0 + 0.01 * i for i in range(25)],
                   "pulse_intensity": 0.3, "pulse_center": 0.1, "hf_mode": "on", "quadrature": "simpson",
                   "limit_mode": "langreth", "dipole": [0.8, 0.2], "eps_v_table": [-1.0, -1.2, -1.1, -0.9],
                   "eps_c_table": [1.0, 1.2, 1.1, 0.9], "max_iter": 8}


def cli_opts_fixture():
    """`kbesolve run` with every non-default physics option (hf, Simpson, langreth,
    tabulated U(t) and bands, complex dipole): observables and report tables."""
    import json
    import shutil
    import tempfile
    from kbesolve import cli
    d = tempfile.mkdtemp()
    try:
        cfg = dict(CLI_CONFIG_OPTS, observables_path=os.path.join(d, "obs.csv"),
                   report_path=os.path.join(d, "rep.csv"), trajectory_path=os.path.join(d, "t.kbe"))
        with open(os.path.join(d, "run.json"), "w") as fh:
            json.dump(cfg, fh)
        assert cli.main(["run", "--config", os.path.join(d, "run.json")]) == 0
        shutil.copy(os.path.join(d, "obs.csv"), os.path.join(HERE, "cli_opts_observables.csv"))
        shutil.copy(os.path.join(d, "rep.csv"), os.path.join(HERE, "cli_opts_report.csv"))
        shutil.copy(os.path.join(d, "t.kbe"), os.path.join(HERE, "cli_opts.kbe"))
        with open(os.path.join(HERE, "cli_opts_config.json"), "w") as fh:
            json.dump(CLI_CONFIG_OPTS, fh, indent=1)
        print("wrote cli_opts.* fixtures")
    finally:
        shutil.rmtree(d)


def cli_fixture():
    """`kbesolve run` on a small config: the KBE1 trajectory bytes, the observables and
    report tables (cli.py:42-87, trajio.py:27-36), and `inspect` output."""
    import contextlib
    import io
    import json
    import shutil
    import tempfile
    from kbesolve import cli
    d = tempfile.mkdtemp()
    try:
        cfg = dict(CLI_CONFIG, trajectory_path=os.path.join(d, "t.kbe"),
                   observables_path=os.path.join(d, "obs.csv"), report_path=os.path.join(d, "rep.csv"))
        with open(os.path.join(d, "run.json"), "w") as fh:
            json.dump(cfg, fh)
        assert cli.main(["run", "--config", os.path.join(d, "run.json")]) == 0
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            assert cli.main(["inspect", os.path.join(d, "t.kbe")]) == 0
        shutil.copy(os.path.join(d, "t.kbe"), os.path.join(HERE, "cli_run.kbe"))
        shutil.copy(os.path.join(d, "obs.csv"), os.path.join(HERE, "cli_run_observables.csv"))
        shutil.copy(os.path.join(d, "rep.csv"), os.path.join(HERE, "cli_run_report.csv"))
        with open(os.path.join(HERE, "cli_run_inspect.txt"), "w") as fh:
            fh.write(buf.getvalue())
        with open(os.path.join(HERE, "cli_run_config.json"), "w") as fh:
            json.dump(CLI_CONFIG, fh, indent=1)
        print("wrote cli_run.* fixtures")
    finally:
        shutil.rmtree(d)


def config_fixture():
    """validate_config (config.py:76-163) on valid and invalid inputs: the exception type
    and message, or the resolved fields."""
    import json
    from kbesolve.config import validate_config
    cases = json.load(open(os.path.join(HERE, "config_cases.json")))["cases"]
    results = []
    for c in cases:
        try:
            r = validate_config(c)
            results.append({"ok": [r.n_k, r.step.dt, r.step.n_steps, r.step.memory_budget, r.step.max_iter,
                                   r.step.quadrature, r.step.limit_mode, r.schedule.n_shards, r.schedule.workers,
                                   [r.model.dipole.real, r.model.dipole.imag], r.model.hf_mode, r.seed]})
        except Exception as e:  # noqa: BLE001
            results.append({"error": type(e).__name__, "message": str(e)})
    json.dump({"cases": cases, "results": results}, open(os.path.join(HERE, "config_cases.json"), "w"), indent=0)
    print(f"wrote config_cases.json ({len(cases)} cases)")


if __name__ == "__main__":
    which = sys.argv[1:] or ["sigma", "collision", "sigma_batched", "trajectory"]
    for w in which:
        globals()[f"{w}_fixture" if w != "trajectory" else "trajectory_fixtures"]()
    # also: collision_row, cli, config (python make_golden.py collision_row cli config)

