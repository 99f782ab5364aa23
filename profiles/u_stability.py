"""Where does the reference scheme diverge?  Runs bench workloads at several U
scales on the GPU path (which tracks the reference step for step) and
prints, per run, the poisoned step (or None), the iteration histogram and the
anticommutation drift at every 100th step.

    python profiles/u_stability.py cfg3:1.0 cfg3:0.75 cfg5:1.0 > gpurun_out/u.jsonl
"""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2505_19467_b200 as kb  # noqa: E402


def one(name, u):
    cfg = dict(bench.WORKLOADS[name])
    cfg["u"] = u
    model = kb.ModelConfig(**bench.model_kwargs(cfg))
    step = kb.StepConfig(dt=cfg["dt"], n_steps=cfg["n_steps"], memory_budget=1 << 40)
    drv = kb.PropagationDriver(kb.build_kgrid(cfg["n_k"]), model, step)
    reps, poisoned = [], None
    t0 = time.time()
    # chunks of 50 so a poisoned run still reports the steps before it
    while drv.state.frontier < cfg["n_steps"]:
        chunk = min(50, cfg["n_steps"] - drv.state.frontier)
        drv.cfg = kb.StepConfig(dt=cfg["dt"], n_steps=chunk, memory_budget=1 << 40)
        try:
            reps += drv.run()
        except kb.PoisonedStateError as e:
            poisoned = str(e)
            break
    drift = [float(r.anticommutation_drift) for r in reps]
    its = [r.iterations for r in reps]
    drv.close()
    return {"workload": name, "u": u, "n_k": cfg["n_k"], "n_steps": cfg["n_steps"],
            "steps_done": len(reps), "poisoned": poisoned,
            "iterations": np.bincount(its).tolist() if its else [],
            "drift_every_100": [drift[i] for i in range(99, len(drift), 100)],
            "max_drift": max(drift) if drift else None, "seconds": round(time.time() - t0, 2)}


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        name, u = arg.split(":")
        print(json.dumps(one(name, float(u))), flush=True)
