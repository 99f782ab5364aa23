"""Isolated per-kernel timings at one late frontier (A/B tool for kernel changes).

    python profiles/kernel_ab.py [--workload cfg2] [--n 900] [--reps 50]

Propagates to step n-1, runs step n's predictor and first corrector once, then
re-launches each step kernel `reps` times back to back at that frontier and
reports the average device time per launch (CUDA events on the launching
stream).  Re-launching the corrector update of iteration 0 is idempotent up to
the residual, so every launch does the full work.
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
    ap.add_argument("--n", type=int, default=900)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--random", action="store_true",
                    help="fill the history with random values instead of propagating to n-1 (timing-only "
                         "library variants whose results are wrong)")
    ap.add_argument("--ncu", action="store_true",
                    help="after the set-up, run each step kernel once between cudaProfilerStart/Stop and exit "
                         "(for ncu --profile-from-start off)")
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
    n = args.n
    if args.random:
        g = torch.Generator(device="cuda").manual_seed(7)
        for h in (drv.ws.g_hist, drv.ws.s_hist):
            torch.view_as_real(h).normal_(0.0, 0.1, generator=g)
    else:
        _lib.check(L.kbe_run(P, 1, n - 1, 0, sp))
    _lib.check(L.kbe_sigma_frontier(P, n - 1, 0, sp))
    _lib.check(L.kbe_collision_frontier(P, n - 1, 0, sp))
    _lib.check(L.kbe_update(P, n, 0, 0, sp))
    _lib.check(L.kbe_sigma_frontier(P, n, 0, sp))
    _lib.check(L.kbe_collision_frontier(P, n, 0, sp))
    _lib.check(L.kbe_update(P, n, 1, 0, sp))
    torch.cuda.synchronize()

    if args.ncu:
        torch.cuda.profiler.start()
        _lib.check(L.kbe_sigma_frontier(P, n, 0, sp))
        _lib.check(L.kbe_collision_frontier(P, n, 0, sp))
        _lib.check(L.kbe_update(P, n, 1, 0, sp))
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return

    def bench_fn(fn):
        for _ in range(3):
            _lib.check(fn())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(args.reps):
            _lib.check(fn())
        e1.record(st)
        torch.cuda.synchronize()
        return 1e3 * e0.elapsed_time(e1) / args.reps

    out = {"workload": args.workload, "n": n, "random": args.random,
           "env": {k: v for k, v in os.environ.items() if k.startswith("KBE_")}}
    out["collision_us"] = bench_fn(lambda: L.kbe_collision_frontier(P, n, 0, sp))
    out["update_us"] = bench_fn(lambda: L.kbe_update(P, n, 1, 0, sp))
    out["sigma_frontier_us"] = bench_fn(lambda: L.kbe_sigma_frontier(P, n, 0, sp))
    out["finish_us"] = bench_fn(lambda: L.kbe_finish_step(P, n, sp))
    blocks = 2 * (n + 1) * (n + 2) // 2 + 2 * n * (n + 1) // 2
    out["collision_gbs"] = 64.0 * cfgw["n_k"] * blocks / (out["collision_us"] * 1e-6) / 1e9
    nk = cfgw["n_k"]
    out["sigma_gflop"] = 256.0 * nk * nk * (n + 1) / 1e9
    out["sigma_tflops"] = out["sigma_gflop"] / (out["sigma_frontier_us"] * 1e-6) / 1e3
    print(json.dumps(out))


if __name__ == "__main__":
    main()
