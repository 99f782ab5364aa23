"""Worker functions for the multi-process tests (importable by spawned processes)."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _init(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def comm_worker(rank, world, port, outdir):
    """CPU: the collective helpers the k-sharded driver uses, on gloo."""
    import torch
    import torch.distributed as dist
    from paper_2505_19467_b200.engine import shard_range
    from paper_2505_19467_b200.propagator import all_gather_device, all_gather_list, all_reduce_device, combine_reports
    _init(rank, world, port)
    lo, hi = shard_range(8, rank, world)
    send = torch.arange(lo * 6, hi * 6, dtype=torch.float64).reshape(hi - lo, 3, 2)
    send = torch.view_as_complex(send.contiguous())                      # (k_local, 3) complex
    out = torch.zeros((8, 3), dtype=torch.complex128)
    all_gather_device(out, send)
    bits = torch.tensor([rank * 10, 5, 7 - rank], dtype=torch.int64)
    all_reduce_device(bits, dist.ReduceOp.MAX)
    hf = torch.tensor([1.5 * (rank + 1)], dtype=torch.float64)
    all_reduce_device(hf, dist.ReduceOp.SUM)
    rows = torch.zeros((3, 24), dtype=torch.float64)
    rows[:, 0] = torch.arange(1, 4)
    rows[:, 4] = rank + 0.5
    rows[:, 5] = 10.0 * (rank + 1)
    rows[:, 6] = float(rank == 1)
    comb = combine_reports(np.stack([p.numpy() for p in all_gather_list(rows, world)]))
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), out=out.numpy(), bits=bits.numpy(), hf=hf.numpy(), comb=comb)
    dist.destroy_process_group()


def driver_worker(rank, world, port, outdir, n_k, n_steps):
    """GPU: a k-sharded PropagationDriver (2 ranks sharing cuda:0 over gloo staging)."""
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    _init(rank, world, port)
    import paper_2505_19467_b200 as kb
    model = kb.ModelConfig(u_protocol=1.0, pulse_intensity=0.3, pulse_center=0.1, hf_mode=os.environ.get("KBE_HF", "off"))
    drv = kb.PropagationDriver(kb.build_kgrid(n_k), model,
                               kb.StepConfig(dt=0.02, n_steps=n_steps, memory_budget=1 << 40),
                               kb.Schedule(n_shards=world))
    reps = drv.run()
    np.savez(os.path.join(outdir, f"drv{rank}.npz"), hist=drv.state.hist.cpu().numpy(),
             sig=drv.sigma.hist.cpu().numpy(), k_lo=drv.k_lo,
             its=np.array([r.iterations for r in reps]), dens=np.array([r.density for r in reps]),
             drift=np.array([r.anticommutation_drift for r in reps]), p2p=drv.p2p is not None)
    drv.close()
    dist.destroy_process_group()
