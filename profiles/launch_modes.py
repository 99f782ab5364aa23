"""A/B of the step launch modes on whole propagations (device time, CUDA events).

    python profiles/launch_modes.py [--workloads cfg1,cfg2] [--reps 3]

Modes: "stream" (kbe_step per step, converged iterations as no-op launches, PDL),
"graph" (kbe_run's step graph with programmatic edges), "graph-nopdl"
(KBE_GRAPH_PDL=0: full dependencies between graph kernel nodes).  Also reports
the host time spent inside kbe_run, to show whether a mode is host-bound.
Each mode runs in its own subprocess (the library reads the env once).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(workload: str, reps: int) -> dict:
    import numpy as np
    import torch

    import bench
    cfgw = bench.select_workload(workload)
    import paper_2505_19467_b200 as kb
    from paper_2505_19467_b200 import _lib

    torch.cuda.set_device(0)
    model = kb.ModelConfig(**bench.model_kwargs(cfgw))
    cfg = kb.StepConfig(dt=cfgw["dt"], n_steps=cfgw["n_steps"], memory_budget=1 << 40)
    drv = kb.PropagationDriver(kb.build_kgrid(cfgw["n_k"]), model, cfg)
    st = torch.cuda.current_stream()
    N = cfgw["n_steps"]
    dev, host = [], []
    for r in range(reps + 2):
        bench._reset(kb, drv)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        h0 = time.perf_counter()
        _lib.check(_lib.lib().kbe_run(drv.ws.problem_ptr(), 1, N, drv.use_graph, int(st.cuda_stream)))
        h1 = time.perf_counter()
        e1.record(st)
        torch.cuda.synchronize()
        if r >= 2:
            dev.append(e0.elapsed_time(e1) * 1e-3)
            host.append(h1 - h0)
    rows = drv.ws.reports.cpu().numpy()[1:]
    its = rows[:, 1].astype(int)
    return {"workload": workload, "steps_per_s": N / float(np.median(dev)), "device_s": float(np.median(dev)),
            "host_submit_s": float(np.median(host)), "us_per_step": float(np.median(dev)) / N * 1e6,
            "mean_iterations": float(its.mean())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="cfg1,cfg2")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--child", default=None)
    args = ap.parse_args()
    if args.child:
        print(json.dumps(one(args.child, args.reps)))
        return
    modes = {"stream": {"KBE_GRAPH": "0"}, "graph": {"KBE_GRAPH": "1", "KBE_GRAPH_PDL": "1"},
             "graph-nopdl": {"KBE_GRAPH": "1", "KBE_GRAPH_PDL": "0"}}
    out = []
    for w in args.workloads.split(","):
        for m, env in modes.items():
            r = subprocess.run([sys.executable, __file__, "--child", w, "--reps", str(args.reps)],
                               env={**os.environ, **env}, capture_output=True, text=True)
            if r.returncode != 0:
                print(r.stderr[-2000:], file=sys.stderr)
                continue
            d = json.loads(r.stdout.strip().splitlines()[-1])
            d["mode"] = m
            out.append(d)
            print(json.dumps(d), flush=True)


if __name__ == "__main__":
    main()
