"""Late-time per-step parity of the full cfg3 propagation against the REAL reference.

The committed cfg3 golden (traj_cfg3_full.npz) is the reference run from the ground
state; it covers the prefix the chained GPU-box calls reached (661 of 1000 steps, ~2.5 h
of 16 host cores; the full run needs ~6 h).  This script covers the rest of the
north_star target the other way round: the GPU path propagates the bench's exact cfg3
workload (n_k = 64, 1000 steps, seeded tables, bench.model_kwargs) and at a few late
frontiers m hands its whole state -- the filled [0..m] blocks of G<, G>, Sigma<, Sigma>,
which is everything the reference's PropagationDriver.step reads from earlier steps
(propagator.py:316-382; the same state make_golden.py's checkpoint/resume restores,
bitwise-checked by `make_golden.py resume_check`) -- to the unmodified reference
(kbesolve 0.1.0 from baseline/_ref), which then takes K steps on the host cores.  Both
sides' steps m+1..m+K are compared: G< row / G> column and Sigma> row / Sigma< column of
every k at every step, densities, residuals and iteration counts.  The last window
ends at step 1000.

Test infrastructure only (runs where baseline/_ref and a GPU exist, i.e. the GPU box):

    KBE_REFERENCE_SRC=$PWD/baseline/_ref python tests/golden/late_windows.py \
        > gpurun_out/late_windows.jsonl

KBE_WINDOWS (default "745,870,995") and KBE_WINDOW_STEPS (default 5) choose the windows;
KBE_WORKLOAD another bench workload (e.g. cfg1 with KBE_WINDOWS=150 for a quick check);
KBE_STEP_OPTS / KBE_MODEL_OPTS (JSON) the non-default physics, e.g.
KBE_STEP_OPTS='{"quadrature": "simpson"}'.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402  (the workload definition: tables, U, pulse)
import paper_2505_19467_b200 as kb  # noqa: E402
from paper_2505_19467_b200.state import TwoTimeGF, unpack_history  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def reference():
    """The unmodified reference (kbesolve 0.1.0): KBE_REFERENCE_SRC, else the driver's
    offline install baseline/_ref.  ImportError when neither is there."""
    src = os.environ.get("KBE_REFERENCE_SRC", os.path.join(ROOT, "baseline", "_ref"))
    if src not in sys.path:
        sys.path.insert(0, src)
    import kbesolve
    return kbesolve


def run_windows(workload, windows, K, workers=None, emit=None, step_opts=None, model_opts=None):
    """Returns (per-step records, worst-case summary); emit(record) is called as they come.
    step_opts / model_opts: extra StepConfig / ModelConfig fields for both sides (the
    non-default physics: quadrature="simpson", limit_mode="langreth", hf_mode="on")."""
    step_opts, model_opts = dict(step_opts or {}), dict(model_opts or {})
    ref = reference()
    emit = emit or (lambda rec: None)
    cfg = dict(bench.WORKLOADS[workload])
    n_k, N, dt = cfg["n_k"], cfg["n_steps"], cfg["dt"]
    kw = bench.model_kwargs(cfg)
    kw.update(model_opts)
    workers = workers or int(os.environ.get("KBE_REF_WORKERS", str(os.cpu_count() or 8)))
    shards = max(d for d in range(1, min(workers, n_k) + 1) if n_k % d == 0)

    windows = sorted(min(m, N - K) for m in windows)
    # the reference's capacity ends with the last window (u_values / u_at read the U table
    # only up to the step being taken, model.py:46-68, so the steps are unchanged) --
    # keeps its four dense (n_k, 2, 2, N+1, N+1) arrays in host memory for cfg4's sizes
    n_ref = max(windows) + K
    torch.cuda.set_device(0)
    gdrv = kb.PropagationDriver(kb.build_kgrid(n_k), kb.ModelConfig(**kw),
                                kb.StepConfig(dt=dt, n_steps=N, memory_budget=1 << 40, **step_opts))
    sig = TwoTimeGF(n_k, 0, N, dt, gdrv.sigma.hist)          # Sigma history, same packing
    rdrv = ref.PropagationDriver(ref.build_kgrid(n_k), ref.ModelConfig(**kw),
                                 ref.StepConfig(dt=dt, n_steps=n_ref, memory_budget=1 << 44, **step_opts),
                                 ref.Schedule(n_shards=shards, workers=workers), ref.WorkerPool(workers))
    emit({"workload": cfg["workload"], "step_opts": step_opts, "model_opts": model_opts, "windows": windows, "steps_per_window": K,
          "ref_capacity": n_ref, "ref_workers": workers, "ref_shards": shards,
          "incremental": gdrv.ws.g_sh is not None})
    worst, records = {"iteration_flips": 0}, []
    for m in windows:
        while gdrv.state.frontier < m:
            gdrv.step()
        t0 = time.time()
        # hand the GPU state at frontier m to the reference: the (m+1)^2 prefix of each
        # array, unpacked on the device one at a time (the packed layout does not depend
        # on the capacity); the reference's arrays are zero beyond the frontier
        for hist, which, ref_arr in ((gdrv.state.hist, 0, rdrv.state.lesser),
                                     (gdrv.state.hist, 1, rdrv.state.greater),
                                     (gdrv.sigma.hist, 1, rdrv.sigma.lesser),
                                     (gdrv.sigma.hist, 0, rdrv.sigma.greater)):
            a = unpack_history(hist, m, which).cpu().numpy()
            ref_arr[...] = 0
            ref_arr[..., : m + 1, : m + 1] = a
            del a
            torch.cuda.empty_cache()
        rdrv.state.frontier = m
        t_load = time.time() - t0
        gpu = []
        for _ in range(K):
            r = gdrv.step()
            n = gdrv.state.frontier
            g = gdrv.state.slice_view(n).cpu().numpy()
            s = sig.slice_view(n).cpu().numpy()
            gpu.append((n, r, g, s))
        for n, gr, g, s in gpu:
            t1 = time.time()
            rr = rdrv.step()
            st, sg = rdrv.state, rdrv.sigma
            rec = {
                "step": n, "window_start": m,
                "row_lesser": rel(g[:, 0:4].reshape(n_k, 2, 2, n + 1), st.lesser[:, :, :, n, : n + 1]),
                "col_greater": rel(g[:, 4:8].reshape(n_k, 2, 2, n + 1), st.greater[:, :, :, : n + 1, n]),
                "sigma_row_greater": rel(s[:, 0:4].reshape(n_k, 2, 2, n + 1), sg.greater[:, :, :, n, : n + 1]),
                "sigma_col_lesser": rel(s[:, 4:8].reshape(n_k, 2, 2, n + 1), sg.lesser[:, :, :, : n + 1, n]),
                "density_abs": abs(gr.density - rr.density),
                "drift_abs": abs(gr.anticommutation_drift - rr.anticommutation_drift),
                "residual_gpu": gr.residual, "residual_ref": rr.residual,
                "iterations_gpu": gr.iterations, "iterations_ref": rr.iterations,
                "ref_step_seconds": round(time.time() - t1, 1),
            }
            if n == gpu[0][0]:
                rec["state_handoff_seconds"] = round(t_load, 1)
            worst["iteration_flips"] += int(gr.iterations != rr.iterations)
            for k_ in ("row_lesser", "col_greater", "sigma_row_greater", "sigma_col_lesser",
                       "density_abs", "drift_abs"):
                worst[k_] = max(worst.get(k_, 0.0), rec[k_])
            records.append(rec)
            emit(rec)
    summary = {"summary": "max over all window steps", **worst, "final_step": gdrv.state.frontier}
    emit(summary)
    return records, summary


def main():
    windows = [int(x) for x in os.environ.get("KBE_WINDOWS", "745,870,995").split(",")]
    run_windows(os.environ.get("KBE_WORKLOAD", "cfg3"), windows, int(os.environ.get("KBE_WINDOW_STEPS", "5")),
                emit=lambda rec: print(json.dumps(rec), flush=True),
                step_opts=json.loads(os.environ.get("KBE_STEP_OPTS", "{}")),
                model_opts=json.loads(os.environ.get("KBE_MODEL_OPTS", "{}")))


if __name__ == "__main__":
    main()
