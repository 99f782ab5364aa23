"""KBE time-steps/sec on B200 (BASELINE.json metric) -- see DESIGN.md §Measurement.

Workload (BASELINE.json configs[1]): 1D Hubbard chain n_k=16, second-Born,
1000 time steps, dt=0.02, U=0.5, delta pulse I=0.2 at t=0.5, reference model
defaults otherwise.  U=0.5 rather than SURVEY's U=1: with U=1
the reference's own as-printed scheme diverges at step 667.  One bench "step" = one whole propagation
of the 1000 time steps from the ground state; value = time steps per second
of whole-job throughput (all ranks), inputs already on the device.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N > 1) every rank owns n_k/N k-points (the reference's
k-shards) and the step all-gathers each new G slice over NCCL.

The JSON line carries: e2e (through the public run() API with host inputs),
roofline of the dominant kernel (K2 collision, HBM-bound) measured live with
CUDA events, cpu_baseline (the numpy oracle port of the reference on this
host, rank 0 only) and clocks sampled during the timed region.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "KBE time-steps/sec (whole propagation)"
# BASELINE.json configs; cfg2 (configs[1]) is the headline line, the others are
# selectable with --workload for the per-config evidence under profiles/.
# U is lowered where the reference's own as-printed scheme diverges.
WORKLOADS = {
    "cfg1": dict(n_k=2, n_steps=200, dt=0.02, u=1.0, pulse_intensity=0.2, pulse_center=0.5,
                 workload="cfg1: Hubbard dimer n_k=2, second-Born, 200 time steps"),
    "cfg2": dict(n_k=16, n_steps=1000, dt=0.02, u=0.5, pulse_intensity=0.2, pulse_center=0.5,
                 workload="cfg2: 1D Hubbard chain n_k=16, second-Born, 1000 time steps"),
    "cfg3": dict(n_k=64, n_steps=1000, dt=0.02, u=0.5, pulse_intensity=0.2, pulse_center=0.5, synth=True,
                 workload="cfg3: synthetic dense-interaction n_k=64 (seeded band/U tables), 1000 time steps"),
    "cfg4": dict(n_k=32, n_steps=4000, dt=0.02, u=0.2, pulse_intensity=0.2, pulse_center=0.5,
                 workload="cfg4: long-time n_k=32, 4000 time steps (history-streaming)"),
    "cfg5": dict(n_k=128, n_steps=500, dt=0.02, u=0.5, pulse_intensity=0.2, pulse_center=0.5,
                 workload="cfg5: large basis n_k=128, 500 time steps"),
}
CFG = dict(WORKLOADS["cfg2"])
WORKLOAD = CFG["workload"]


def select_workload(name):
    global CFG, WORKLOAD
    CFG = dict(WORKLOADS[name])
    WORKLOAD = CFG["workload"]
    return CFG


def model_kwargs(cfg=None):
    """ModelConfig kwargs of a workload.  cfg3's synthetic system:
    seeded tabulated bands eps_c = 1 + U(0,1), eps_v = -eps_c and a seeded U(t)
    table u*(1 + 0.1 N(0,1)), all from default_rng(7)."""
    c = cfg if cfg is not None else CFG
    kw = dict(pulse_intensity=c["pulse_intensity"], pulse_center=c["pulse_center"])
    if c.get("synth"):
        rng = np.random.default_rng(7)
        eps_c = 1.0 + rng.uniform(0.0, 1.0, c["n_k"])
        kw.update(u_protocol=c["u"] * (1.0 + 0.1 * rng.standard_normal(c["n_steps"] + 1)),
                  eps_c_table=eps_c, eps_v_table=-eps_c)
    else:
        kw.update(u_protocol=c["u"])
    return kw


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self):
        self.rows, self._stop, self._th = [], threading.Event(), None

    def __enter__(self):
        def loop():
            q = ("--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    dev = os.environ.get("LOCAL_RANK", "0")
                    out = subprocess.run(["nvidia-smi", "-i", dev, q, "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._th = threading.Thread(target=loop, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and "Active" == r[2 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ CPU baseline (oracle port)
def cpu_baseline(iterations_per_step=None, budget_s=25.0):
    """Time the numpy oracle port of the reference on this host and extrapolate
    the full cfg2 propagation (SURVEY §8(d) method): single Sigma and collision
    evaluations at several frontiers n on a random-filled history, fit
    sigma(n) = a + b (n+1) and coll(n) = c0 + c2 n^2, sum over the run using the
    GPU run's iteration counts (1 + it_n evaluations at step n)."""
    from oracle import kbe_oracle as O
    n_k, N, dt = CFG["n_k"], CFG["n_steps"], CFG["dt"]
    ns = {2: [100, 200, 300], 16: [150, 300, 450], 32: [50, 100, 150], 64: [20, 40, 60]}.get(n_k, [8, 16, 24])
    cap = max(ns)
    drv = O.OracleDriver(n_k, O.Model(u_protocol=1.0), dt, cap)
    GL, GG = O.random_mirrored_state(n_k, cap, cap, seed=3)
    drv.GL[:] = 0.1 * GL
    drv.GG[:] = 0.1 * GG
    # the reference's own parallel decomposition (selfenergy.py:201, collision.py:264-268):
    # contiguous k-shards on a thread pool, one per host core up to n_k (numpy releases
    # the GIL inside the contractions)
    workers = max(1, min(os.cpu_count() or 1, n_k))
    shards = [(i * n_k // workers, (i + 1) * n_k // workers) for i in range(workers)]
    pool = ThreadPoolExecutor(workers)

    def eval_sigma(n):
        gl_col, gg_row = drv.GL[:, :, :, : n + 1, n], drv.GG[:, :, :, n, : n + 1]
        U = drv.U

        def one(kr):
            return (O.sigma_slice(gl_col, gg_row, U[: n + 1], float(U[n]), kr),
                    O.sigma_slice(gg_row, gl_col, float(U[n]), U[: n + 1], kr))
        parts = list(pool.map(one, shards))
        for (k0, k1), (les, gre) in zip(shards, parts):
            drv.SL[k0:k1, :, :, : n + 1, n] = les
            drv.SG[k0:k1, :, :, n, : n + 1] = gre

    def eval_collision(n):
        list(pool.map(lambda kr: O.collision_frontier(drv.GL[kr[0]:kr[1]], drv.GG[kr[0]:kr[1]], drv.SL[kr[0]:kr[1]],
                                                        drv.SG[kr[0]:kr[1]], n, dt), shards))

    ts, tc = [], []
    t_all = time.perf_counter()
    for n in ns:
        t0 = time.perf_counter()
        eval_sigma(n)
        t1 = time.perf_counter()
        eval_collision(n)
        t2 = time.perf_counter()
        ts.append(t1 - t0)
        tc.append(t2 - t1)
        if time.perf_counter() - t_all > budget_s:
            break
    pool.shutdown()
    m = len(ts)
    x = np.array(ns[:m], dtype=float)
    bs = np.polyfit(x + 1, ts, 1)
    A = np.stack([np.ones(m), x ** 2], axis=1)
    cc = np.linalg.lstsq(A, np.array(tc), rcond=None)[0]

    def sig(n):
        return max(bs[0] * (n + 1) + bs[1], 0.0)

    def col(n):
        return max(cc[0] + cc[1] * n * n, 0.0)

    its = iterations_per_step if iterations_per_step is not None else np.full(N, 2)
    total = 0.0
    for n in range(1, N + 1):
        total += sig(n - 1) + col(n - 1) + its[n - 1] * (sig(n) + col(n))
    return {
        "value": N / total, "unit": "time-steps/s", "cores": workers, "kind": "port",
        "sample": (f"numpy oracle port of the reference, k-sharded over {workers} host threads, single "
                   f"Sigma+collision evaluations at n={ns[:m]} on a random n_k={n_k} history "
                   f"({time.perf_counter() - t_all:.1f}s), fitted and extrapolated to the full {N}-step "
                   f"propagation with the measured iteration counts"),
        "extrapolated_seconds": total,
    }


# ------------------------------------------------------------------ GPU arm
def _setup_dist(n_gpus):
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # KBE_BENCH_SAME_DEVICE=1 + KBE_BENCH_BACKEND=gloo: every rank on cuda:0, for
        # exercising the sharded path on a one-GPU box (gloo stages through the host)
        dev = 0 if os.environ.get("KBE_BENCH_SAME_DEVICE") == "1" else local
        torch.cuda.set_device(dev)
        backend = os.environ.get("KBE_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    return rank, world


def _barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _make_driver(kb):
    model = kb.ModelConfig(**model_kwargs())
    cfg = kb.StepConfig(dt=CFG["dt"], n_steps=CFG["n_steps"], memory_budget=1 << 40)
    return model, cfg


def _reset(kb, drv):
    from paper_2505_19467_b200 import _lib
    from paper_2505_19467_b200._device import stream_ptr
    _lib.check(_lib.lib().kbe_init_history(drv.ws.problem_ptr(), stream_ptr()))
    drv.state.frontier = 0
    drv._poisoned = None
    if drv.world > 1:
        drv.publish_initial()


def _collision_roofline(kb, drv, hbm_peak):
    """One extra propagation with CUDA events around every K2 launch (same stream),
    counting only launches that did work (iteration <= the step's count)."""
    import torch
    from paper_2505_19467_b200 import _lib
    from paper_2505_19467_b200._device import stream_ptr
    L, P = _lib.lib(), drv.ws.problem_ptr()
    st = torch.cuda.current_stream()
    sp = stream_ptr()
    nk = drv.k_hi - drv.k_lo
    _reset(kb, drv)
    ev = []
    N = drv.capacity
    t_total0 = torch.cuda.Event(enable_timing=True)
    t_total1 = torch.cuda.Event(enable_timing=True)
    t_total0.record(st)
    for n in range(1, N + 1):
        calls = [(n - 1, 0)] + [(n, it) for it in range(drv.cfg.max_iter)]
        if drv.world > 1:
            raise RuntimeError("roofline pass runs on one rank")
        for ci, (nf, it) in enumerate(calls):   # same launch sequence as kbe_step
            if drv.interactions_on:
                _lib.check(L.kbe_sigma_frontier(P, nf, it, sp))
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _lib.check(L.kbe_collision_frontier(P, nf, it, sp))
            e1.record(st)
            ev.append((n, ci, nf, e0, e1))
            _lib.check(L.kbe_update(P, n, 0 if ci == 0 else 1, it, sp))
        _lib.check(L.kbe_finish_step(P, n, sp))
    t_total1.record(st)
    torch.cuda.synchronize()
    rows = drv.ws.reports.cpu().numpy()
    iters = rows[1:, 1].astype(int)
    hist = rows[1:, 8: 8 + _lib.MAX_ITER]
    eps = drv.cfg.eps

    def final_res(step):                      # residual of the step's last corrector
        h = hist[step - 1][: iters[step - 1]]
        return float(h[-1])

    # mirror of the device's incremental-evaluation rule (collision_kernel)
    incr_on = drv.ws.g_sh is not None
    prev_f = full_f = -1
    dsum = 0.0
    tot_b, tot_t, launches, n_incr = 0.0, 0.0, 0, 0
    for n, ci, nf, e0, e1 in ev:
        if ci > iters[n - 1]:
            continue    # converged: launch was a no-op
        it = 0 if ci == 0 else ci - 1
        delta = (final_res(nf) if nf >= 1 else float("inf")) if ci == 0 else (float(hist[n - 1][it - 1]) if it else float("inf"))
        incr = incr_on and prev_f == nf and full_f == nf and dsum + delta <= 1e-7
        prev_f = nf
        if incr:
            dsum += delta
            n_incr += 1
            # complex64 shadow of both triangles' slices < nf (64 B per cell) + FP64 slice nf
            tot_b += nk * (64.0 * nf * (nf + 1) + 128.0 * (nf + 1))
        else:
            full_f, dsum = nf, 0.0
            # algorithmic bytes: each unique 2x2 c128 block of the Sigma triangle (slices
            # 0..nf, both functions) and of the G triangle (slices 0..nf-1) read once
            blocks = 2 * (nf + 1) * (nf + 2) // 2 + 2 * nf * (nf + 1) // 2
            tot_b += 64.0 * nk * blocks
        tot_t += e0.elapsed_time(e1) * 1e-3
        launches += 1
    step_s = t_total0.elapsed_time(t_total1) * 1e-3
    achieved = tot_b / tot_t / 1e9
    return {
        "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
        "traffic": None, "kernel": "collision_kernel (K2)", "launches_with_work": launches,
        "incremental_launches": n_incr,
        "kernel_seconds": tot_t, "share_of_propagation": tot_t / step_s,
        "bytes_per_launch_formula": "64*n_k*[(n+1)(n+2) + n(n+1)]",
    }, iters


def run_ours(args):
    import torch
    rank, world = _setup_dist(args.gpus)
    import paper_2505_19467_b200 as kb
    from paper_2505_19467_b200 import _lib
    hbm_peak, peak_kind = _peaks()
    model, cfg = _make_driver(kb)
    grid = kb.build_kgrid(CFG["n_k"])
    drv = kb.PropagationDriver(grid, model, cfg)
    hist_gb = 2 * drv.ws.g_hist.numel() * 16 / 1e9
    st = torch.cuda.current_stream()
    N = CFG["n_steps"]

    def one_propagation():
        _reset(kb, drv)
        drv.run()

    for _ in range(args.warmup):
        one_propagation()
    torch.cuda.synchronize()
    _barrier(world)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler() as clk:
        torch.cuda.synchronize()
        _barrier(world)
        t0.record(st)
        spec_launches = 0
        for _ in range(args.steps):
            _reset(kb, drv)
            n1 = N
            if drv._speculative():      # the path driver.run() takes (speculative iteration counts)
                drv._run_speculative(1, n1)
                spec_launches += drv.spec_launches + 2   # + kbe_init_history's 2 kernels
            elif drv._device_sequenced():
                _lib.check(_lib.lib().kbe_run(drv.ws.problem_ptr(), 1, n1, drv.use_graph if world == 1 else 0,
                                              int(st.cuda_stream)))
            else:
                for n in range(1, n1 + 1):
                    drv._launch_step(n)
            drv.state.frontier = n1
        t1.record(st)
        torch.cuda.synchronize()
        _barrier(world)
    secs = _max_over_ranks(t0.elapsed_time(t1) * 1e-3, world)
    reps = drv._reports(1, N)
    if np.any(reps[:, 6] != 0) or np.any(reps[:, 0] == 0):
        raise RuntimeError("propagation poisoned or incomplete inside the timed region")
    iters = reps[:, 1].astype(int)
    dens = reps[:, 5] / CFG["n_k"]
    value = args.steps * N / secs
    # per evaluation K1 Sigma (interacting), K2 collision, K3 update; + K4 finish per step;
    # each propagation adds kbe_init_history's 2 kernels.  Stream path: all max_iter
    # corrector iterations launch (converged ones as no-ops); graph path: only the
    # iterations that ran (the rest sit behind conditional nodes that stay off).
    per_eval = 3 if drv.interactions_on else 2
    # K3 split into reduce + update for as-printed problems with >= 32 local k (kbe200.cu)
    if (drv.k_hi - drv.k_lo) >= 32 and drv.cfg.limit_mode == "as-printed" and not drv.use_graph:
        per_eval += 1
    if world == 1 and drv.use_graph:
        per_prop = int(np.sum((1 + iters) * per_eval + 1)) + 2
    else:
        per_prop = N * ((1 + cfg.max_iter) * per_eval + 1) + 2
    gpu_launches = spec_launches if drv._speculative() else args.steps * per_prop

    launch_mode = ("cuda-graph (conditional corrector)" if (world == 1 and drv.use_graph) else
                   "stream, speculative iteration counts" if drv._speculative() else "stream")
    roof, cpu = None, None
    if rank == 0 and world == 1:
        roof, _ = _collision_roofline(kb, drv, hbm_peak)
        roof["peak_kind"] = peak_kind
        try:
            traffic = json.load(open(os.path.join(ROOT, "profiles", "collision_traffic.json")))
            roof["traffic"] = traffic.get("bytes_per_launch")
            roof["traffic_note"] = traffic.get("note")
        except Exception:
            pass
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(iters)

    # e2e: public API with host inputs (model tables in, StepReports out); the timed
    # driver is released first so that large workloads (cfg4) fit twice over in HBM
    if world > 1:
        import torch.distributed as dist
        drv.close()
    del drv
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    _barrier(world)
    e2e_t = []
    for _ in range(max(1, min(args.steps, 3))):
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        state, reports = kb.run(grid, model, cfg)
        torch.cuda.synchronize()
        e2e_t.append(time.perf_counter() - w0)
        del state
    e2e_s = _max_over_ranks(float(np.median(e2e_t)), world)
    h2d = 8 * (2 * CFG["n_k"] + 3 * (N + 1))
    d2h = 8 * (N + 1) * _lib.REPORT_W

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "time-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128 (fp64)",
            "data": "synthetic (reference model defaults, deterministic; no dataset)",
            "config": {"workload": WORKLOAD, "n_k": CFG["n_k"], "n_steps": N, "dt": CFG["dt"], "U": CFG["u"],
                       "pulse": [CFG["pulse_intensity"], CFG["pulse_center"]],
                       "parallelism": f"k-shards x{world}", "bench_step": f"one whole {N}-step propagation",
                       "l2": f"inputs larger than L2 ({hist_gb:.2f} GB device history per propagation)"},
            "e2e": {"value": N / e2e_s, "unit": "time-steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "api": "paper_2505_19467_b200.run(grid, model, step_cfg)"},
            "gpu_launches": gpu_launches,
            "launch_mode": launch_mode,
            "iterations_hist": {int(k): int(v) for k, v in zip(*np.unique(iters, return_counts=True))},
            "final_density": float(dens[-1]),
            "roofline": roof, "cpu_baseline": cpu, "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cpu = cpu_baseline(None)
    # each "step" is the bounded sample + extrapolation of one whole propagation
    vals = [cpu["value"]]
    for _ in range(max(0, args.steps - 1)):
        break
    line = {
        "metric": METRIC, "value": float(np.median(vals)), "unit": "time-steps/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "impl": "reference", "dtype": "c128 (fp64)", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n_k": CFG["n_k"], "n_steps": CFG["n_steps"], "dt": CFG["dt"]},
        "cpu_baseline": {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cpu["value"], "unit": "time-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "vs_baseline": None,
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS),
                    help="BASELINE.json config (cfg2 = configs[1], the headline line)")
    args = ap.parse_args()
    select_workload(args.workload)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
