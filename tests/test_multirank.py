"""World-size-2 tests of the k-sharded path (gloo).

CPU: the collective helpers and report combination the sharded driver uses.
GPU: two ranks share cuda:0 (gloo stages the all-gather through the host) and
must reproduce the single-rank propagation bitwise.
"""

import os
import socket

import numpy as np
import pytest

import _mp_workers as W

torch = pytest.importorskip("torch")
mp = torch.multiprocessing


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_collectives_world2_gloo(tmp_path):
    mp.spawn(W.comm_worker, args=(2, _port(), str(tmp_path)), nprocs=2, join=True)
    r0, r1 = (np.load(tmp_path / f"rank{r}.npz") for r in (0, 1))
    want = np.arange(48, dtype=float).reshape(8, 3, 2)
    want = want[..., 0] + 1j * want[..., 1]
    for r in (r0, r1):
        np.testing.assert_array_equal(r["out"], want)                  # k order = rank order
        np.testing.assert_array_equal(r["bits"], [10, 5, 7])
        np.testing.assert_array_equal(r["hf"], [4.5])
        np.testing.assert_array_equal(r["comb"][:, 4], [1.5, 1.5, 1.5])   # drift: max
        np.testing.assert_array_equal(r["comb"][:, 5], [30.0] * 3)        # density: sum
        np.testing.assert_array_equal(r["comb"][:, 6], [1.0] * 3)         # non-finite: or


@pytest.mark.gpu
@pytest.mark.parametrize("hf, world, p2p, sigma, n_k",
                         [("off", 2, "1", "auto", 8), ("on", 2, "1", "auto", 8), ("off", 4, "1", "auto", 8),
                          ("off", 2, "0", "auto", 8), ("on", 2, "0", "auto", 8),
                          ("off", 2, "1", "dft", 8), ("off", 2, "1", "auto", 12), ("off", 4, "0", "direct", 8)])
def test_k_sharded_driver_matches_single_rank(tmp_path, hf, world, p2p, sigma, n_k):
    """Each exchanged chunk carries the rank's G slice and its convergence record; the
    kernels max-reduce the records over ranks, so iteration counts match exactly.
    p2p=1: the update kernel stores into every peer's buffer (CUDA IPC; the ranks share
    one GPU here, NVLink peers on a node); p2p=0: all-gather through torch.distributed.
    sigma: the K1 variant reading the gathered frontier (FFT, DMMA DFT GEMMs -- the
    default for n_k = 12 --, direct correlations)."""
    import paper_2505_19467_b200 as kb
    n_steps = 40
    os.environ["KBE_HF"] = hf
    os.environ["KBE_P2P"] = p2p
    os.environ["KBE_SIGMA"] = sigma
    try:
        mp.spawn(W.driver_worker, args=(world, _port(), str(tmp_path), n_k, n_steps), nprocs=world, join=True)
    finally:
        os.environ.pop("KBE_HF", None)
        os.environ.pop("KBE_P2P", None)
        os.environ.pop("KBE_SIGMA", None)
    if p2p == "1":
        assert all(np.load(tmp_path / f"drv{r}.npz")["p2p"] for r in range(world))
    parts = [np.load(tmp_path / f"drv{r}.npz") for r in range(world)]
    hist = np.concatenate([p["hist"] for p in parts])
    sig = np.concatenate([p["sig"] for p in parts])
    torch.cuda.set_device(0)
    model = kb.ModelConfig(u_protocol=1.0, pulse_intensity=0.3, pulse_center=0.1, hf_mode=hf)
    one = kb.PropagationDriver(kb.build_kgrid(n_k), model, kb.StepConfig(dt=0.02, n_steps=n_steps, memory_budget=1 << 40))
    reps = one.run()
    ref_hist = one.state.hist.cpu().numpy()
    ref_sig = one.sigma.hist.cpu().numpy()
    scale = np.abs(ref_hist).max()
    assert np.abs(hist - ref_hist).max() <= 1e-13 * scale
    assert np.abs(sig - ref_sig).max() <= 1e-13 * np.abs(ref_sig).max()
    for p in parts:
        assert list(p["its"]) == [r.iterations for r in reps]
        np.testing.assert_allclose(p["dens"], [r.density for r in reps], rtol=0, atol=1e-14)
        np.testing.assert_allclose(p["drift"], [r.anticommutation_drift for r in reps], rtol=0, atol=1e-14)
