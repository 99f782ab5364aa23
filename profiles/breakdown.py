"""Per-kernel time breakdown of one whole propagation (CUDA events around every launch).

    python profiles/breakdown.py [--workload cfg2] [--ncu-step N0]

Replays kbe_step's launch sequence (include/kbe200.h) from Python with a CUDA
event pair around every launch on the launching stream, and reports per kernel
class: launches that did work, converged no-op launches, summed device time.
The events serialise the stream (no PDL overlap), so the sum is slightly above
the bench's ms_per_step; the SHARES are what this is for.

--ncu-step N0: run steps 1..N0-1 unprofiled, then bracket step N0 with
cudaProfilerStart/Stop, for `ncu --profile-from-start off` captures of one late
step (the launch lists and --set full captures under profiles/ come from this).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--ncu-step", type=int, default=0)
    ap.add_argument("--n-steps", type=int, default=0, help="override the workload's step count")
    ap.add_argument("--max-iter", type=int, default=6, help="StepConfig.max_iter (no-op launch cost A/B)")
    args = ap.parse_args()
    cfgw = bench.select_workload(args.workload)
    if args.n_steps:
        cfgw["n_steps"] = args.n_steps
    import paper_2505_19467_b200 as kb
    from paper_2505_19467_b200 import _lib
    from paper_2505_19467_b200._device import stream_ptr

    torch.cuda.set_device(0)
    model = kb.ModelConfig(**bench.model_kwargs(cfgw))
    cfg = kb.StepConfig(dt=cfgw["dt"], n_steps=cfgw["n_steps"], memory_budget=1 << 40, max_iter=args.max_iter)
    drv = kb.PropagationDriver(kb.build_kgrid(cfgw["n_k"]), model, cfg)
    L, P, sp = _lib.lib(), drv.ws.problem_ptr(), stream_ptr()
    st = torch.cuda.current_stream()
    N = drv.capacity

    if args.ncu_step:
        n0 = args.ncu_step
        _lib.check(L.kbe_run(P, 1, n0 - 1, 0, sp))
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        _lib.check(L.kbe_step(P, n0, sp))
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        print(json.dumps({"ncu_step": n0, "workload": args.workload}))
        return

    # warm-up propagation (module load, attributes), then reset
    _lib.check(L.kbe_run(P, 1, min(N, 50), 0, sp))
    torch.cuda.synchronize()
    bench._reset(kb, drv)
    t_plain0, t_plain1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_plain0.record(st)
    _lib.check(L.kbe_run(P, 1, N, 0, sp))
    t_plain1.record(st)
    torch.cuda.synchronize()
    plain_s = t_plain0.elapsed_time(t_plain1) * 1e-3
    bench._reset(kb, drv)

    ev = []

    def timed(name, n, it, fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        _lib.check(fn(), name)
        e1.record(st)
        ev.append((name, n, it, e0, e1))

    for n in range(1, N + 1):
        if drv.interactions_on:
            timed("sigma", n, -1, lambda: L.kbe_sigma_frontier(P, n - 1, 0, sp))
        timed("collision", n, -1, lambda: L.kbe_collision_frontier(P, n - 1, 0, sp))
        timed("update", n, -1, lambda: L.kbe_update(P, n, 0, 0, sp))
        for it in range(cfg.max_iter):
            if drv.interactions_on:
                timed("sigma", n, it, lambda: L.kbe_sigma_frontier(P, n, it, sp))
            timed("collision", n, it, lambda: L.kbe_collision_frontier(P, n, it, sp))
            timed("update", n, it, lambda: L.kbe_update(P, n, 1, it, sp))
        timed("finish", n, -1, lambda: L.kbe_finish_step(P, n, sp))
    torch.cuda.synchronize()
    rows = drv.ws.reports.cpu().numpy()
    iters = rows[1:, 1].astype(int)
    agg = {}
    for name, n, it, e0, e1 in ev:
        work = it < iters[n - 1]   # it == -1: predictor-side launches always work
        key = (name, "work" if work else "noop")
        t = e0.elapsed_time(e1) * 1e-3
        a = agg.setdefault(key, [0, 0.0])
        a[0] += 1
        a[1] += t
    total = sum(v[1] for v in agg.values())
    out = {"workload": args.workload, "n_steps": N, "plain_propagation_s": plain_s,
           "evented_sum_s": total, "iterations_hist": {int(k): int(v) for k, v in zip(*np.unique(iters, return_counts=True))},
           "kernels": {f"{k[0]}:{k[1]}": {"launches": v[0], "seconds": v[1], "us_avg": 1e6 * v[1] / v[0],
                                           "share": v[1] / total} for k, v in sorted(agg.items())}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
