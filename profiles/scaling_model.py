"""k-shard scaling model of one propagation from measured per-kernel times.

    python profiles/scaling_model.py [--workload cfg3] [--ranks 1 2 4 8] [--reps 10]

Every GPU call in this environment has ONE B200, so the N-GPU throughput of the
k-sharded path cannot be timed directly.  This tool measures, on one GPU, what one rank
of an R-rank run executes per corrector iteration at frontier n:

  * K2 (collision, full and incremental evaluations), K3 (reduce + update) and K4
    (finish) on n_k / R local k-points -- they are purely per-k, so a 1-rank problem with
    n_k / R k-points runs exactly rank 0's kernels (its band tables = rank 0's slice);
  * K1 (Sigma) on the full n_k: every rank transforms the gathered G slice of all k.

Times are CUDA events over back-to-back launches on a history filled with random values
(timing only), at several frontiers n, interpolated (K2 ~ a + b n + c n^2, the others
~ a + b n) and integrated over the workload's evaluation schedule: per step, the
evaluation count and the incremental share of the 1-GPU bench run (--evals, --incr).
The per-iteration exchange of an R-rank run adds the update kernel's peer stores of the
local G slice to R-1 peers (NVLink, --link-gbs) plus one flag round trip (--sync-us).
Prints one JSON line per R with the modelled propagation time, speed-up and efficiency.
"""

from __future__ import annotations

import argparse
import json
import os
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def measure(cfgw, nkl, ns, reps):
    import paper_2505_19467_b200 as kb
    from paper_2505_19467_b200 import _lib
    from paper_2505_19467_b200._device import stream_ptr

    kw = bench.model_kwargs(cfgw)
    if "eps_c_table" in kw:   # rank 0's slice of the band tables
        kw["eps_c_table"] = kw["eps_c_table"][:nkl]
        kw["eps_v_table"] = kw["eps_v_table"][:nkl]
    model = kb.ModelConfig(**kw)
    cfg = kb.StepConfig(dt=cfgw["dt"], n_steps=cfgw["n_steps"], memory_budget=1 << 40)
    drv = kb.PropagationDriver(kb.build_kgrid(nkl), model, cfg)
    L, P, sp = _lib.lib(), drv.ws.problem_ptr(), stream_ptr()
    st = torch.cuda.current_stream()
    g = torch.Generator(device="cuda").manual_seed(7)
    for h in (drv.ws.g_hist, drv.ws.s_hist):
        torch.view_as_real(h).normal_(0.0, 0.1, generator=g)
    res = drv.ws.ctl[0: 8 * _lib.MAX_ITER].view(torch.int64)

    def timed(fn):
        for _ in range(2):
            _lib.check(fn())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            _lib.check(fn())
        e1.record(st)
        torch.cuda.synchronize()
        return 1e3 * e0.elapsed_time(e1) / reps

    out = []
    for n in ns:
        # one full evaluation at n (snapshot + shadow state), then the forced-residual timings
        for f, it, ph in ((n - 1, 0, 0), (n, 0, 1)):
            _lib.check(L.kbe_sigma_frontier(P, f, it, sp))
            _lib.check(L.kbe_collision_frontier(P, f, it, sp))
            _lib.check(L.kbe_update(P, n, ph, 0, sp))
        torch.cuda.synchronize()
        row = {"n": n}
        for name, r0 in (("k2_full_us", 1e-3), ("k2_incr_us", 2e-9)):
            res[0] = struct.unpack("<q", struct.pack("<d", r0))[0]
            row[name] = timed(lambda: L.kbe_collision_frontier(P, n, 1, sp))
        res[0] = struct.unpack("<q", struct.pack("<d", 1e-3))[0]
        row["k3_us"] = timed(lambda: L.kbe_update(P, n, 1, 0, sp))
        row["k1_us"] = timed(lambda: L.kbe_sigma_frontier(P, n, 0, sp))
        row["k4_us"] = timed(lambda: L.kbe_finish_step(P, n, sp))
        out.append(row)
    del drv
    torch.cuda.empty_cache()
    return out


def fit(ns, ys, deg):
    return np.polyfit(np.asarray(ns, float), np.asarray(ys, float), deg)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--evals", type=float, default=3.849, help="K1/K2/K3 evaluations per step (1-GPU bench)")
    ap.add_argument("--incr", type=float, default=1768 / 3849, help="incremental share of K2 evaluations")
    ap.add_argument("--link-gbs", type=float, default=600.0, help="effective NVLink peer-store GB/s per rank")
    ap.add_argument("--sync-us", type=float, default=3.0, help="flag round trip per iteration (P2P epochs)")
    args = ap.parse_args()
    cfgw = bench.select_workload(args.workload)
    torch.cuda.set_device(0)
    nk, N = cfgw["n_k"], cfgw["n_steps"]
    ns = sorted(set([max(8, N // 10), N // 4, N // 2, (3 * N) // 4, N - 1]))
    full = measure(cfgw, nk, ns, args.reps)   # K1 on all n_k: replicated on every rank
    k1fit = fit(ns, [r["k1_us"] for r in full], 1)
    steps = np.arange(1, N + 1, dtype=float)
    base = None
    for R in args.ranks:
        if nk % R:
            continue
        rows = full if R == 1 else measure(cfgw, nk // R, ns, args.reps)
        f2 = fit(ns, [r["k2_full_us"] for r in rows], 2)
        i2 = fit(ns, [r["k2_incr_us"] for r in rows], 2)
        k3 = fit(ns, [r["k3_us"] for r in rows], 1)
        k4 = fit(ns, [r["k4_us"] for r in rows], 1)
        k2 = (1 - args.incr) * np.polyval(f2, steps) + args.incr * np.polyval(i2, steps)
        per_eval = k2 + np.polyval(k3, steps) + np.polyval(k1fit, steps)
        exch = 0.0 * steps
        if R > 1:
            byts = (steps + 1) * 8 * 16.0 * (nk // R) * (R - 1)
            exch = byts / (args.link_gbs * 1e3) + args.sync_us   # us per iteration
        t_us = np.sum(args.evals * (per_eval + exch) + np.polyval(k4, steps))
        t = t_us * 1e-6
        if base is None:
            base = t
        k1_share = float(np.sum(args.evals * np.polyval(k1fit, steps)) * 1e-6 / t)
        print(json.dumps({"workload": args.workload, "ranks": R, "n_k_local": nk // R, "model_seconds": t,
                          "steps_per_s": N / t, "speedup": base / t, "efficiency": base / t / R,
                          "k1_replicated_share": k1_share, "samples": rows,
                          "k1_full_samples_us": [r["k1_us"] for r in full]}))


if __name__ == "__main__":
    main()
