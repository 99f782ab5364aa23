"""Collision kernel (K2) time and bandwidth as a function of the frontier n.

    python profiles/coll_sweep.py [--workload cfg2] [--every 50] [--reps 10]

Random finite history (timing only), one driver, every n in range(every, N+1, every):
average device time of `reps` back-to-back K2 launches (CUDA events on the launching
stream) and algorithmic GB/s.  With the measured iteration histogram this says where
a whole propagation loses its HBM roofline fraction (small n: launch/latency bound).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--every", type=int, default=50)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    cfgw = bench.select_workload(args.workload)
    import paper_2505_19467_b200 as kb
    from paper_2505_19467_b200 import _lib
    from paper_2505_19467_b200._device import stream_ptr

    torch.cuda.set_device(0)
    model = kb.ModelConfig(**bench.model_kwargs(cfgw))
    cfg = kb.StepConfig(dt=cfgw["dt"], n_steps=cfgw["n_steps"], memory_budget=1 << 40)
    drv = kb.PropagationDriver(kb.build_kgrid(cfgw["n_k"]), model, cfg)
    L, P, sp = _lib.lib(), drv.ws.problem_ptr(), stream_ptr()
    st = torch.cuda.current_stream()
    g = torch.Generator(device="cuda").manual_seed(7)
    for h in (drv.ws.g_hist, drv.ws.s_hist):
        torch.view_as_real(h).normal_(0.0, 0.1, generator=g)
    nk = cfgw["n_k"]
    out = []
    for n in list(range(args.every, cfgw["n_steps"] + 1, args.every)):
        for _ in range(2):
            _lib.check(L.kbe_collision_frontier(P, n, 0, sp))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(args.reps):
            _lib.check(L.kbe_collision_frontier(P, n, 0, sp))
        e1.record(st)
        torch.cuda.synchronize()
        us = 1e3 * e0.elapsed_time(e1) / args.reps
        blocks = 2 * (n + 1) * (n + 2) // 2 + 2 * n * (n + 1) // 2
        gbs = 64.0 * nk * blocks / (us * 1e-6) / 1e9
        out.append({"n": n, "us": round(us, 2), "gbs": round(gbs, 1)})
    print(json.dumps({"workload": args.workload, "lib": os.environ.get("KBE_LIB", "product"), "sweep": out}))


if __name__ == "__main__":
    main()
