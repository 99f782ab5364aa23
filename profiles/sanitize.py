"""Small propagations for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool memcheck python profiles/sanitize.py single
    compute-sanitizer --tool racecheck --target-processes all python profiles/sanitize.py p2p

single  : n_k = 8, 40 steps, pulse at step 5 -- the production path: K2 starting before
          K1 finishes (early start), incremental complex64 evaluations and their delta
          slots, split K3 (K3a + K3b), speculative iteration counts with rollbacks
options : n_k = 4, 20 steps each with hf_mode="on", Simpson + U(t) ramp, langreth limits
          (fused K3, langreth K2, hf k-mean kernel), plus the kernel-level operators
variants: the K1 kernels (round 2): four-step FFT at n_k = 16 and 128, DMMA DFT GEMMs at
          n_k = 8 (KBE_SIGMA=dft) and n_k = 12 (the default there), direct correlations
p2p     : 2 ranks sharing cuda:0, k-sharded, the update kernels storing each new slice
          into the peer's buffer (CUDA IPC) with epoch flags, 12 steps
"""

import os
import socket
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def single():
    import torch
    import paper_2505_19467_b200 as kb
    torch.cuda.set_device(0)
    os.environ["KBE_INCR"] = "1"
    model = kb.ModelConfig(u_protocol=1.0, pulse_intensity=0.2, pulse_center=0.1)
    drv = kb.PropagationDriver(kb.build_kgrid(8), model, kb.StepConfig(dt=0.02, n_steps=40))
    assert drv.ws.g_sh is not None
    reps = drv.run()
    print("single", len(reps), np.bincount([r.iterations for r in reps]).tolist(), reps[-1].density)


def options():
    import torch
    import paper_2505_19467_b200 as kb
    torch.cuda.set_device(0)
    grid = kb.build_kgrid(4)
    runs = [
        (kb.ModelConfig(u_protocol=1.0, pulse_intensity=0.3, pulse_center=0.1, hf_mode="on"),
         kb.StepConfig(dt=0.02, n_steps=20)),
        (kb.ModelConfig(u_protocol=np.linspace(0.5, 1.5, 21), pulse_intensity=0.3, pulse_center=0.1),
         kb.StepConfig(dt=0.02, n_steps=20, quadrature="simpson")),
        (kb.ModelConfig(u_protocol=1.0, pulse_intensity=0.3, pulse_center=0.1, dipole=0.8 + 0.3j),
         kb.StepConfig(dt=0.02, n_steps=20, limit_mode="langreth")),
    ]
    for model, cfg in runs:
        st, reps = kb.run(grid, model, cfg)
        _ = st.lesser, st.greater, st.retarded()
        print("options", cfg.quadrature, cfg.limit_mode, model.hf_mode, len(reps), reps[-1].density)
    rng = np.random.default_rng(1)
    gl = rng.standard_normal((8, 2, 2, 5)) + 1j * rng.standard_normal((8, 2, 2, 5))
    gg = rng.standard_normal((8, 2, 2, 5)) + 1j * rng.standard_normal((8, 2, 2, 5))
    kb.sigma_slice(gl, gg, np.linspace(0.4, 1.2, 5), 0.7, kb.build_kgrid(8))


def variants():
    import torch
    import paper_2505_19467_b200 as kb
    torch.cuda.set_device(0)
    model = kb.ModelConfig(u_protocol=1.0, pulse_intensity=0.2, pulse_center=0.1)
    for n_k, sig, steps in ((16, "fft", 30), (128, "fft", 8), (8, "dft", 30), (12, "auto", 30), (8, "direct", 20)):
        os.environ["KBE_SIGMA"] = sig
        drv = kb.PropagationDriver(kb.build_kgrid(n_k), model, kb.StepConfig(dt=0.02, n_steps=steps))
        reps = drv.run()
        print("variant", n_k, sig, len(reps), reps[-1].density)
        drv.close()


def _p2p_worker(rank, world, port):
    import torch
    import torch.distributed as dist
    import paper_2505_19467_b200 as kb
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["KBE_P2P"] = "1"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    model = kb.ModelConfig(u_protocol=1.0, pulse_intensity=0.2, pulse_center=0.1)
    drv = kb.PropagationDriver(kb.build_kgrid(8), model, kb.StepConfig(dt=0.02, n_steps=12))
    assert drv.p2p is not None
    reps = drv.run()
    drv.close()
    if rank == 0:
        print("p2p", len(reps), reps[-1].density)
    dist.destroy_process_group()


def p2p():
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_p2p_worker, args=(2, port), nprocs=2, join=True)


if __name__ == "__main__":
    {"single": single, "options": options, "variants": variants, "p2p": p2p}[sys.argv[1]]()
