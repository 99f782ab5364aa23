"""KBE time-steps/sec on B200 (BASELINE.json metric) -- see DESIGN.md §7.

Default workload: the north_star target, BASELINE.json configs[2] (cfg3):
synthetic dense-interaction system n_k = n_orb = 64, second-Born, 1000 time
steps, dt = 0.02, delta pulse I = 0.2 at t = 0.5, the SURVEY §8(d) seeded
tables (eps_c = 1 + U(0,1), eps_v = -eps_c, U(t) = u (1 + 0.1 N(0,1)),
default_rng(7)) with u = 0.75: at u = 1 the reference's own scheme diverges
at step 868 (u = 0.9: step 987), DESIGN.md §6.  One bench "step" = one whole
propagation from the ground state; value = time steps per second of
whole-job throughput (all ranks), inputs already on the device.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg1..cfg5]

Under torchrun (N > 1) every rank owns n_k/N k-points (the reference's
k-shards) and each new G slice is exchanged over NVLink peer memory.

The JSON line carries: e2e (through the public run() API with host inputs),
the roofline of the dominant kernel (K2 collision, HBM-bound) and of the Sigma
kernel (K1, FP64) measured live with CUDA events, value_fp64_only (the same
propagation with the complex64 incremental collision corrections off),
cpu_baseline (the reference itself, kbesolve from baseline/_ref, on this host's
cores, rank 0 only) and clocks sampled during the timed region.
"""

from __future__ import annotations

import argparse
import json
import math
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
# BASELINE.json configs; cfg3 (configs[2], the north_star target) is the headline line,
# the others are selectable with --workload for the per-config evidence under profiles/.
# U is the SURVEY §8(d) value (1.0) except where the reference's own as-printed scheme
# diverges before the last step; there it is the largest tested value that stays finite
# (cfg2 u=1 diverges at step 667, cfg3 at 868, cfg4 u=0.25 at 3778).
WORKLOADS = {
    "cfg1": dict(n_k=2, n_steps=200, dt=0.02, u=1.0, pulse_intensity=0.2, pulse_center=0.5,
                 workload="cfg1: Hubbard dimer n_k=2, second-Born, 200 time steps"),
    "cfg2": dict(n_k=16, n_steps=1000, dt=0.02, u=0.5, pulse_intensity=0.2, pulse_center=0.5,
                 golden="traj_cfg2_full.npz",
                 workload="cfg2: 1D Hubbard chain n_k=16, second-Born, 1000 time steps"),
    "cfg3": dict(n_k=64, n_steps=1000, dt=0.02, u=0.75, pulse_intensity=0.2, pulse_center=0.5, synth=True,
                 golden="traj_cfg3_full.npz",
                 workload="cfg3: synthetic dense-interaction n_k=64 (seeded band/U tables), 1000 time steps"),
    "cfg4": dict(n_k=32, n_steps=4000, dt=0.02, u=0.2, pulse_intensity=0.2, pulse_center=0.5,
                 workload="cfg4: long-time n_k=32, 4000 time steps (history-streaming)"),
    "cfg5": dict(n_k=128, n_steps=500, dt=0.02, u=1.0, pulse_intensity=0.2, pulse_center=0.5,
                 workload="cfg5: large basis n_k=128, 500 time steps"),
}
CFG = dict(WORKLOADS["cfg3"])
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


# ------------------------------------------------------------------ CPU baseline
def _reference_pkg():
    """kbesolve 0.1.0 itself, from baseline/_ref (the offline pip install of
    /root/reference/pkg that travels with the repo snapshot), or None."""
    p = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isfile(os.path.join(p, "kbesolve", "__init__.py")):
        return None
    if p not in sys.path:
        sys.path.insert(0, p)
    import kbesolve
    return kbesolve


def _eval_points(N):
    """Frontiers for the single-evaluation samples: up to N/2, so the filled history
    (4 reference arrays of (n_k,2,2,n+1,n+1) complex128) stays a few GB."""
    return [max(8, N * i // 8) for i in (1, 2, 3, 4)]


class CpuReference:
    """The reference's own CPU path on this host, SURVEY §8(d) method:
    (i) a real prefix run of n_pre steps past the pulse (the reference's own
    PropagationDriver.step, which also times sigma / collision / update);
    (ii) single _eval_sigma(n) / _eval_collision(n) calls on a filled history at
    several n; (iii) fit sigma(n) = a + b (n+1), coll(n) = c0 + c2 n^2;
    (iv) extrapolate the whole propagation with per-step iteration counts
    (1 + it_n evaluations at step n) plus the prefix's mean update time.
    k-sharded over all host threads through the reference's own Schedule /
    WorkerPool (selfenergy.py:201, collision.py:264-268)."""

    def __init__(self, threads=None):
        self.kb = _reference_pkg()
        if self.kb is None:
            raise RuntimeError("baseline/_ref has no kbesolve")
        self.threads = threads or os.cpu_count() or 1
        n_k = CFG["n_k"]
        self.shards = max(d for d in range(1, min(self.threads, n_k) + 1) if n_k % d == 0)
        self.pool = self.kb.WorkerPool(self.threads)
        self.samples = []          # (n, sigma seconds, collision seconds)
        self.prefix = None

    def _driver(self, n_steps):
        kb = self.kb
        model = kb.ModelConfig(**model_kwargs())
        cfg = kb.StepConfig(dt=CFG["dt"], n_steps=n_steps, memory_budget=1 << 50)
        return kb.PropagationDriver(kb.build_kgrid(CFG["n_k"]), model, cfg,
                                    kb.Schedule(n_shards=self.shards, workers=self.threads), self.pool)

    def run_prefix(self, n_pre):
        drv = self._driver(n_pre)
        t0 = time.perf_counter()
        reps = [drv.step() for _ in range(n_pre)]
        secs = time.perf_counter() - t0
        self.prefix = {"steps": n_pre, "seconds": secs,
                       "iterations": [r.iterations for r in reps],
                       "update_s": float(np.mean([r.timings.get("update", 0.0) for r in reps]))}
        return self.prefix

    def eval_at(self, n):
        drv = self._driver(n)
        rng = np.random.default_rng(n)
        v = 0.1 * (rng.standard_normal(n + 1) + 1j * rng.standard_normal(n + 1))
        for arr in (drv.state.lesser, drv.state.greater, drv.sigma.lesser, drv.sigma.greater):
            arr[...] = v
        drv.state.frontier = n
        t0 = time.perf_counter()
        drv._eval_sigma(n)
        t1 = time.perf_counter()
        drv._eval_collision(n)
        t2 = time.perf_counter()
        self.samples.append((n, t1 - t0, t2 - t1))
        del drv
        return t2 - t0

    def extrapolate(self, iterations):
        x = np.array([s[0] for s in self.samples], dtype=float)
        ts = np.array([s[1] for s in self.samples])
        tc = np.array([s[2] for s in self.samples])
        bs = np.polyfit(x + 1, ts, 1)
        cc = np.linalg.lstsq(np.stack([np.ones_like(x), x * x], axis=1), tc, rcond=None)[0]

        def ev(n):
            return max(bs[0] * (n + 1) + bs[1], 0.0) + max(cc[0] + cc[1] * n * n, 0.0)

        upd = self.prefix["update_s"] if self.prefix else 0.0

        def total(its):
            return sum(ev(n - 1) + its[n - 1] * ev(n) + upd for n in range(1, len(its) + 1))

        N = CFG["n_steps"]
        out = {"seconds": total(iterations[:N]), "fit": {"sigma_a_b": bs.tolist()[::-1], "coll_c0_c2": cc.tolist()}}
        if self.prefix:
            pred = total(self.prefix["iterations"])
            out["prefix_predicted_s"] = pred
            out["prefix_measured_s"] = self.prefix["seconds"]
        return out

    def describe(self):
        s = (f"kbesolve 0.1.0 (baseline/_ref, unmodified) on {self.threads} host threads "
             f"(Schedule n_shards={self.shards}, workers={self.threads})")
        if self.prefix:
            s += (f"; real {self.prefix['steps']}-step prefix run {self.prefix['seconds']:.1f}s "
                  f"({self.prefix['steps'] / self.prefix['seconds']:.3g} steps/s)")
        s += (f"; single Sigma+collision evaluations at n={[x[0] for x in self.samples]} on a filled history, "
              f"fitted (sigma a+b(n+1), collision c0+c2 n^2) and extrapolated to the full {CFG['n_steps']}-step "
              f"propagation with per-step iteration counts")
        return s


def _golden_iterations():
    """The reference's own per-step iteration counts for this workload when a committed
    full-length golden exists (tests/golden/traj_<cfg>_full.npz), else None."""
    name = CFG.get("golden")
    if not name:
        return None
    path = os.path.join(ROOT, "tests", "golden", name)
    try:
        z = np.load(path)
        if int(z["n_steps"]) == CFG["n_steps"] and abs(float(z["u"]) - CFG["u"]) < 1e-15:
            return np.asarray(z["iterations"], dtype=int)
    except Exception:
        return None
    return None


def cpu_baseline(iterations_per_step=None, n_pre=60, points=None):
    """The reference on this host (CpuReference), else the numpy oracle port."""
    N = CFG["n_steps"]
    try:
        ref = CpuReference()
    except Exception:
        return _port_baseline(iterations_per_step)
    t_all = time.perf_counter()
    ref.run_prefix(min(n_pre, N))
    for n in (points or _eval_points(N)[1:]):
        ref.eval_at(n)
    its = iterations_per_step if iterations_per_step is not None else _golden_iterations()
    if its is None:
        post = ref.prefix["iterations"][30:] or ref.prefix["iterations"]
        its = np.full(N, max(1, int(round(float(np.mean(post))))))
    ex = ref.extrapolate(np.asarray(its))
    return {
        "value": N / ex["seconds"], "unit": "time-steps/s", "cores": ref.threads, "kind": "reference",
        "sample": ref.describe() + f" ({time.perf_counter() - t_all:.0f}s of CPU work)",
        "extrapolated_seconds": ex["seconds"], "prefix_steps_per_s": ref.prefix["steps"] / ref.prefix["seconds"],
        "prefix_predicted_over_measured": ex.get("prefix_predicted_s", 0.0) / ref.prefix["seconds"],
        "label": "extrapolated",
    }


def _port_baseline(iterations_per_step=None, budget_s=25.0):
    """Fallback when baseline/_ref is absent: the numpy oracle port of the reference,
    single Sigma and collision evaluations at several frontiers n on a random-filled
    history, fitted and extrapolated the same way (no prefix run)."""
    from oracle import kbe_oracle as O
    n_k, N, dt = CFG["n_k"], CFG["n_steps"], CFG["dt"]
    ns = _eval_points(N)[:3]
    cap = max(ns)
    drv = O.OracleDriver(n_k, O.Model(u_protocol=1.0), dt, cap)
    GL, GG = O.random_mirrored_state(n_k, cap, cap, seed=3)
    drv.GL[:] = 0.1 * GL
    drv.GG[:] = 0.1 * GG
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
    cc = np.linalg.lstsq(np.stack([np.ones(m), x ** 2], axis=1), np.array(tc), rcond=None)[0]

    def ev(n):
        return max(bs[0] * (n + 1) + bs[1], 0.0) + max(cc[0] + cc[1] * n * n, 0.0)

    its = iterations_per_step if iterations_per_step is not None else _golden_iterations()
    if its is None:
        its = np.full(N, 3)
    total = sum(ev(n - 1) + its[n - 1] * ev(n) for n in range(1, N + 1))
    return {
        "value": N / total, "unit": "time-steps/s", "cores": workers, "kind": "port",
        "sample": (f"numpy oracle port of the reference (baseline/_ref absent), k-sharded over {workers} host "
                   f"threads, single Sigma+collision evaluations at n={ns[:m]} on a random n_k={n_k} history "
                   f"({time.perf_counter() - t_all:.1f}s), fitted and extrapolated to the full {N}-step "
                   f"propagation with per-step iteration counts"),
        "extrapolated_seconds": total, "label": "extrapolated",
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


def _k1_peak(kind="dfma"):
    """FP64 roofline denominators for K1: MEASURED_PEAKS.json has no FP64 entry, so the
    DFMA / DMMA peaks measured on a B200 of this pool (profiles/fp64_peak.cu ->
    profiles/r01/fp64_peak.json, profiles/dmma_peak.cu -> profiles/r02/dmma_peak.jsonl),
    else the datasheet FP64 figure."""
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        if "fp64_tflops" in p:
            return float(p["fp64_tflops"]) * 1e3, "measured (MEASURED_PEAKS.json)"
    except Exception:
        pass
    try:
        if kind == "dmma":
            for line in open(os.path.join(ROOT, "profiles", "r02", "dmma_peak.jsonl")):
                d = json.loads(line)
                if "dmma_tflops" in d:
                    return float(d["dmma_tflops"]) * 1e3, "measured DMMA m8n8k4 peak (profiles/r02/dmma_peak.jsonl)"
        p = json.load(open(os.path.join(ROOT, "profiles", "r01", "fp64_peak.json")))
        return float(p["fp64_tflops"]) * 1e3, "measured DFMA peak (profiles/r01/fp64_peak.json)"
    except Exception:
        return 37000.0, "datasheet (HGX B200 FP64 / FP64 tensor)"


def _sigma_variant(n_k):
    """The K1 kernel a launch uses (propagator._sigma_variant_from_env / spec_sigma)."""
    env = os.environ.get("KBE_SIGMA", "auto")
    if env == "auto":
        if n_k == 2:
            return "direct"
        return "fft" if not (n_k & (n_k - 1)) else "dft"
    return env


def _k1_work(variant, nkg, nkl, pairs):
    """(executed flops, HBM bytes) of one K1 launch over `pairs` pairs.  Bytes: the G
    frontier slice (all k) in and the Sigma slice (local k) out, 8 planes of c128 each.
    Flops: fft = 16 length-n_k transforms per pair (radix-2 count 5 N log2 N + 6 N for the
    four-step twiddles) + the pointwise det / product (70 N); dft = 4 real DMMA MACs per
    complex MAC of the forward (8 n_k^2) and inverse (8 n_k n_k_local) GEMMs; direct = the
    four correlations (128 n_k^2 per pair and component)."""
    byt = pairs * 8 * 16.0 * (nkg + nkl)
    if variant == "fft":
        lg = math.log2(nkg)
        fl = pairs * (16 * (5 * nkg * lg + 6 * nkg) + 70 * nkg)
    elif variant == "dft":
        fl = pairs * 2 * 4 * (8 * nkg * nkg + 8 * nkg * nkl)
    else:
        fl = pairs * 2 * 128.0 * nkg * nkg
    return fl, byt


def _collision_roofline(kb, drv, hbm_peak):
    """One extra propagation with CUDA events around every K1, K2 and K3 launch (same
    stream, so K2 does not overlap K1 here), counting only launches that did work
    (iteration <= the step's count).  Returns the K2 (HBM) roofline with a K1 (FP64)
    roofline and K3 timings attached."""
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

    def E():
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        return e
    t_total0.record(st)
    for n in range(1, N + 1):
        calls = [(n - 1, 0)] + [(n, it) for it in range(drv.cfg.max_iter)]
        if drv.world > 1:
            raise RuntimeError("roofline pass runs on one rank")
        for ci, (nf, it) in enumerate(calls):   # same launch sequence as kbe_step
            s0 = E()
            if drv.interactions_on:
                _lib.check(L.kbe_sigma_frontier(P, nf, it, sp))
            e0 = E()
            _lib.check(L.kbe_collision_frontier(P, nf, it, sp))
            e1 = E()
            _lib.check(L.kbe_update(P, n, 0 if ci == 0 else 1, it, sp))
            u1 = E()
            ev.append((n, ci, nf, e0, e1, s0, u1))
        _lib.check(L.kbe_finish_step(P, n, sp))
    t_total1.record(st)
    torch.cuda.synchronize()
    rows = drv.ws.reports.cpu().numpy()
    iters = rows[1:, 1].astype(int)
    hist = rows[1:, 8: 8 + _lib.MAX_ITER]

    def final_res(step):                      # residual of the step's last corrector
        h = hist[step - 1][: iters[step - 1]]
        return float(h[-1])

    # mirror of the device's incremental-evaluation rule (collision_kernel)
    incr_on = drv.ws.g_sh is not None
    prev_f = full_f = -1
    dsum = 0.0
    tot_b, tot_t, launches, n_incr = 0.0, 0.0, 0, 0
    k1_f, k1_t, k1_n, k1_fdir, k1_b = 0.0, 0.0, 0, 0.0, 0.0
    k3_t, k3_late = 0.0, []
    nkg = drv.grid.n_k
    variant = _sigma_variant(nkg)
    for n, ci, nf, e0, e1, s0, u1 in ev:
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
        if drv.interactions_on:
            fl, byt = _k1_work(variant, nkg, nk, nf + 1)
            k1_f += fl
            k1_b += byt
            k1_fdir += 2.0 * (nf + 1) * (56.0 * nkg ** 3 + 64.0 * nkg ** 2)
            k1_t += s0.elapsed_time(e0) * 1e-3
            k1_n += 1
        ku = e1.elapsed_time(u1) * 1e-3
        k3_t += ku
        if n > 0.9 * N:
            k3_late.append(ku)
    step_s = t_total0.elapsed_time(t_total1) * 1e-3
    achieved = tot_b / tot_t / 1e9
    k1 = None
    if k1_n:
        pk, pk_kind = _k1_peak("dmma" if variant == "dft" else "dfma")
        a1 = k1_f / k1_t / 1e9
        names = {"fft": "sigma_fft_kernel (K1, four-step FFTs)", "dft": "sigma_dft_kernel (K1, DMMA DFT GEMMs)",
                 "direct": "sigma_frontier_kernel (K1, O(n_k^2) correlations)"}
        k1 = {"variant": variant, "kernel": names.get(variant, variant),
              "bound": {"fft": "latency", "dft": "fp64 tensor (DMMA)", "direct": "fp64"}.get(variant, "fp64"),
              "achieved": a1, "peak": pk, "unit": "GFLOP/s", "frac": a1 / pk, "peak_kind": pk_kind,
              "hbm_gbs": k1_b / k1_t / 1e9, "hbm_frac": k1_b / k1_t / 1e9 / hbm_peak,
              "launches_with_work": k1_n, "kernel_seconds": k1_t, "share_of_propagation": k1_t / step_s,
              "us_per_launch": k1_t / k1_n * 1e6,
              "flops_per_launch_formula": {
                  "fft": "(n+1)[16(5 n_k log2 n_k + 6 n_k) + 70 n_k] (FFTs + pointwise, executed)",
                  "dft": "(n+1) 8 (8 n_k^2 + 8 n_k n_k_local) (real DMMA flops, executed)",
                  "direct": "2(n+1) 128 n_k^2 (factorised correlations, executed)"}.get(variant),
              "bytes_per_launch_formula": "(n+1) 8 planes 16 B (n_k + n_k_local)",
              "reference_algorithm_gflops": k1_fdir / k1_t / 1e9,
              "reference_algorithm_note": "direct Alg. 2 count 2(n+1)(56 n_k^3 + 64 n_k^2) over the same time: the "
                                          "rate the reference's own algorithm would need to match this kernel"}
    return {
        "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
        "traffic": None, "kernel": "collision_kernel (K2)", "launches_with_work": launches,
        "incremental_launches": n_incr,
        "kernel_seconds": tot_t, "share_of_propagation": tot_t / step_s,
        "bytes_per_launch_formula": "64*n_k*[(n+1)(n+2) + n(n+1)]",
        "k1": k1,
        "k3": {"kernel": "reduce_kernel + update_kernel (K3)", "kernel_seconds": k3_t,
               "share_of_propagation": k3_t / step_s,
               "us_per_launch_last_10pct": float(np.mean(k3_late)) * 1e6 if k3_late else None},
        "timing_pass_seconds": step_s,
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
    def timed(drv, steps):
        """K whole propagations between CUDA events on the launching stream."""
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        _barrier(world)
        t0.record(st)
        launches = 0
        for _ in range(steps):
            _reset(kb, drv)
            n1 = N
            if drv._speculative():      # the path driver.run() takes (speculative iteration counts)
                drv._run_speculative(1, n1)
                launches += drv.spec_launches + 2   # + kbe_init_history's 2 kernels
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
        return t0.elapsed_time(t1) * 1e-3, launches

    with ClockSampler() as clk:
        secs_local, spec_launches = timed(drv, args.steps)
    secs = _max_over_ranks(secs_local, world)
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
    per_eval = int(_lib.lib().kbe_launches_per_eval(drv.ws.problem_ptr()))
    if drv.use_graph and world == 1:
        per_eval = (3 if drv.interactions_on else 2) + int(drv.model.hf_mode == "on")   # graph: fused K3
    if world == 1 and drv.use_graph:
        per_prop = int(np.sum((1 + iters) * per_eval + 1)) + 2
    else:
        per_prop = N * ((1 + cfg.max_iter) * per_eval + 1) + 2
    gpu_launches = spec_launches if drv._speculative() else args.steps * per_prop

    incr_used = drv.ws.g_sh is not None
    launch_mode = ("cuda-graph (conditional corrector)" if (world == 1 and drv.use_graph) else
                   "stream, speculative iteration counts" if drv._speculative() else "stream")
    roof, cpu = None, None
    if rank == 0 and world == 1:
        roof, _ = _collision_roofline(kb, drv, hbm_peak)
        roof["peak_kind"] = peak_kind
        try:
            # the ncu capture of this workload (profiles/collision_traffic.json, keyed by
            # workload); none for workloads without a capture
            traffic = json.load(open(os.path.join(ROOT, "profiles", "collision_traffic.json"))).get(CFG["workload"][:4])
            if traffic:
                roof["traffic"] = traffic.get("bytes_per_launch")
                roof["traffic_note"] = f"n = {traffic['n']} launch: " + traffic.get("note", "")
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

    # the same propagation with the incremental collision corrections (complex64 M dv
    # terms on repeated evaluations) switched off: every operation in FP64
    fp64_only = None
    if incr_used:
        old_env = os.environ.get("KBE_INCR")
        os.environ["KBE_INCR"] = "0"
        try:
            drv64 = kb.PropagationDriver(grid, model, cfg)
        finally:
            if old_env is None:
                os.environ.pop("KBE_INCR", None)
            else:
                os.environ["KBE_INCR"] = old_env
        assert drv64.ws.g_sh is None
        timed(drv64, 1)
        s64, _ = timed(drv64, args.steps)
        s64 = _max_over_ranks(s64, world)
        fp64_only = {"value": args.steps * N / s64, "unit": "time-steps/s", "ms_per_step": s64 / args.steps * 1e3,
                     "note": "KBE_INCR=0: no complex64 incremental collision corrections"}
        if world > 1:
            drv64.close()
        del drv64
        torch.cuda.empty_cache()
    h2d = 8 * (2 * CFG["n_k"] + 3 * (N + 1))
    d2h = 8 * (N + 1) * _lib.REPORT_W

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "time-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": ("c128 (fp64); repeated collision evaluations add a complex64 M*dv correction "
                      "(|dv| <= 1e-7 relative, DESIGN §3) -- value_fp64_only is the all-FP64 run")
            if incr_used else "c128 (fp64)",
            "value_fp64_only": fp64_only,
            "data": "synthetic (reference model defaults, deterministic; no dataset)",
            "config": {"workload": WORKLOAD, "n_k": CFG["n_k"], "n_steps": N, "dt": CFG["dt"], "U": CFG["u"],
                       "pulse": [CFG["pulse_intensity"], CFG["pulse_center"]],
                       "parallelism": f"k-shards x{world}", "bench_step": f"one whole {N}-step propagation",
                       "l2": f"inputs larger than L2 ({hist_gb:.2f} GB device history per propagation)"},
            "e2e": {"value": N / e2e_s, "unit": "time-steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "api": "paper_2505_19467_b200.run(grid, model, step_cfg)",
                    "result": "StepReports (observables) copied to the host; G</G> stay in HBM behind the "
                              "returned TwoTimeGF's lazy accessors (not materialised inside the timed region)"},
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
    """--impl reference: the reference's own CPU implementation (kbesolve from
    baseline/_ref, unmodified, through its PropagationDriver) on this host's cores.
    One bench step = one timed single Sigma + collision evaluation of the workload at a
    frontier n cycling through _eval_points(N); before the steps, one real prefix run
    past the pulse.  The steps' samples are fitted and extrapolated to the whole
    propagation with the reference's own iteration counts (committed
    golden) when available.  Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    N = CFG["n_steps"]
    base = {"metric": METRIC, "unit": "time-steps/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "impl": "reference",
            "dtype": "c128 (fp64)", "data": "synthetic", "vs_baseline": None, "scaling": "strong",
            "config": {"workload": WORKLOAD, "n_k": CFG["n_k"], "n_steps": N, "dt": CFG["dt"], "U": CFG["u"],
                       "pulse": [CFG["pulse_intensity"], CFG["pulse_center"]]}}
    try:
        ref = CpuReference()
    except Exception as e:  # noqa: BLE001
        cpu = _port_baseline(None)
        line = dict(base, value=cpu["value"], note=f"baseline/_ref unavailable ({e}); numpy port",
                    cpu_baseline={k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
                    e2e={"value": cpu["value"], "unit": "time-steps/s", "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0})
        print(json.dumps(line))
        return
    t_all = time.perf_counter()
    ref.run_prefix(min(60, N))
    pts = _eval_points(N)
    for _ in range(args.warmup):
        ref.eval_at(pts[0])
    ref.samples.clear()
    step_s = [ref.eval_at(pts[i % len(pts)]) for i in range(args.steps)]
    its = _golden_iterations()
    its_src = "the reference's own (committed golden)"
    if its is None:
        post = ref.prefix["iterations"][30:] or ref.prefix["iterations"]
        its = np.full(N, max(1, int(round(float(np.mean(post))))))
        its_src = "the prefix's post-pulse mean"
    ex = ref.extrapolate(np.asarray(its))
    value = N / ex["seconds"]
    cpu = {"value": value, "unit": "time-steps/s", "cores": ref.threads, "kind": "reference",
           "sample": ref.describe() + f"; iteration counts: {its_src}"}
    line = dict(base, value=value, ms_per_step=float(np.mean(step_s)) * 1e3,
                ms_per_step_meaning="mean wall time of one timed single-evaluation sample",
                label="extrapolated", extrapolated_seconds=ex["seconds"],
                prefix_steps_per_s=ref.prefix["steps"] / ref.prefix["seconds"],
                prefix_predicted_over_measured=ex["prefix_predicted_s"] / ref.prefix["seconds"],
                fit=ex["fit"], cpu_seconds=time.perf_counter() - t_all, cpu_baseline=cpu,
                e2e={"value": value, "unit": "time-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS),
                    help="BASELINE.json config (cfg3 = configs[2], the north_star target, is the headline line)")
    args = ap.parse_args()
    select_workload(args.workload)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
