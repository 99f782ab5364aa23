"""Whole-run A/B of two builds of libkbe200.so on one box: bitwise comparison of the final
device histories and the time of a whole propagation (A/B tool for kernel changes).

    python profiles/lib_ab.py [--workload cfg3] [--steps N] [--reps 3] A B ...

A, B, ...: a built library (``*.so``: this tree's package with KBE_LIB=that file) or the
root of another source tree (its own package and library, e.g. an exported older commit,
when the host-side buffers changed too).  Each runs in its own process, propagates the workload for --steps
steps (default: the full length), and reports its device time per propagation (CUDA
events, best of --reps after one warm-up), the iteration histogram, and a SHA-256 of the
packed G and Sigma histories; the parent prints, per library, the max relative
difference of the final G< row / G> column against the first library.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(workload, steps, reps, out, root):
    sys.path.insert(0, root)
    import numpy as np
    import torch

    import bench
    import paper_2505_19467_b200 as kb

    cfgw = dict(bench.WORKLOADS[workload])
    N = steps or cfgw["n_steps"]
    model = kb.ModelConfig(**bench.model_kwargs(cfgw))
    cfg = kb.StepConfig(dt=cfgw["dt"], n_steps=N, memory_budget=1 << 40)
    torch.cuda.set_device(0)
    times = []
    for r in range(reps + 1):
        drv = kb.PropagationDriver(kb.build_kgrid(cfgw["n_k"]), model, cfg)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps_ = drv.run()
        e1.record()
        torch.cuda.synchronize()
        if r:
            times.append(e0.elapsed_time(e1) / 1e3)
        if r < reps:
            drv.close()
            del drv
    sl = drv.state.slice_view(N).cpu().numpy()
    np.save(out, sl)
    h = hashlib.sha256()
    h.update(drv.state.hist.cpu().numpy().tobytes())
    h.update(drv.sigma.hist.cpu().numpy().tobytes())
    its = [r.iterations for r in reps_]
    print(json.dumps({"lib": os.environ.get("KBE_LIB") or kb.__file__, "workload": workload, "steps": N,
                      "seconds_best": min(times), "seconds_all": times, "steps_per_s": N / min(times),
                      "iterations_hist": np.bincount(its).tolist(), "sha256": h.hexdigest()}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--steps", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--child", default=None)
    ap.add_argument("--root", default=ROOT)
    ap.add_argument("libs", nargs="*")
    a = ap.parse_args()
    if a.child:
        child(a.workload, a.steps, a.reps, a.child, a.root)
        return
    import numpy as np
    outs = []
    for i, lib in enumerate(a.libs):
        out = f"/tmp/lib_ab_{i}.npy"
        env, root = dict(os.environ), ROOT
        env.pop("KBE_LIB", None)
        if lib.endswith(".so"):
            env["KBE_LIB"] = os.path.abspath(lib)
        else:
            root = os.path.abspath(lib)
        subprocess.run([sys.executable, os.path.abspath(__file__), "--workload", a.workload, "--steps", str(a.steps),
                        "--reps", str(a.reps), "--child", out, "--root", root], env=env, check=True, cwd=root)
        outs.append(np.load(out))
    for lib, o in zip(a.libs, outs):
        d = float(np.abs(o - outs[0]).max() / np.abs(outs[0]).max())
        print(json.dumps({"lib": lib, "final_slice_rel_diff_vs_first": d, "bitwise_equal_first": bool(np.array_equal(o, outs[0]))}))


if __name__ == "__main__":
    main()
