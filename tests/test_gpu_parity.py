"""Parity of the CUDA path (through the C ABI) with the oracle and the reference goldens.

Tolerances: kernel level <= 1e-12 relative (SURVEY §8(c) protocol 1),
trajectories <= 1e-10 relative (BASELINE.json north_star), densities 1e-12 abs.
"""

import numpy as np
import pytest

from conftest import load_golden, rel_err
from oracle import kbe_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_19467_b200 as kb  # noqa: E402


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


# ------------------------------------------------------------------ Sigma (kernel level)
@pytest.mark.parametrize("n_k", [2, 4, 8, 16, 32, 64])
def test_sigma_slice_matches_reference_golden(n_k):
    g = load_golden("sigma.npz")
    grid = kb.build_kgrid(n_k)
    gl, gg = g[f"gl_{n_k}"], g[f"gg_{n_k}"]
    u1, u2 = g[f"u1_{n_k}"], float(g[f"u2_{n_k}"])
    pol = kb.polarizability(gl, gg, grid)
    assert rel_err(pol, g[f"pol_{n_k}"]) <= 1e-12
    assert rel_err(kb.sigma_first(g[f"pol_{n_k}"], gl, u1, u2, grid), g[f"s1_{n_k}"]) <= 1e-12
    assert rel_err(kb.sigma_second(gl, gg, u1, u2, grid), g[f"s2_{n_k}"]) <= 1e-12
    assert rel_err(kb.sigma_slice(gl, gg, u1, u2, grid), g[f"sigma_{n_k}"]) <= 1e-12
    shard = kb.sigma_slice(gl, gg, u1, u2, grid, (n_k // 2, n_k))
    assert rel_err(shard, g[f"sigma_shard_{n_k}"]) <= 1e-12


@pytest.mark.parametrize("n_k", [2, 16, 128])
def test_sigma_slice_matches_oracle_random(n_k):
    rng = np.random.default_rng(n_k)
    shape = (n_k, 2, 2, 7)
    gl = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    gg = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    u1 = rng.uniform(0.5, 1.5, 7)
    grid = kb.build_kgrid(n_k)
    got = kb.sigma_slice(gl, gg, u1, 0.8, grid)
    want = O.sigma_slice(gl, gg, u1, 0.8)
    assert rel_err(got, want) <= 1e-12
    # 3-D input squeezes back (selfenergy.py:55-56)
    one = kb.sigma_slice(gl[..., 0], gg[..., 0], 1.0, 1.0, grid)
    assert one.shape == (n_k, 2, 2)


def test_sigma_batched_matches_reference_golden():
    g = load_golden("sigma_batched.npz")
    GL, GG, u = g["GL"], g["GG"], g["u"]
    n_k, cap = GL.shape[0], GL.shape[-1] - 1
    grid = kb.build_kgrid(n_k)
    for n in (0, 3, 6):
        state = kb.TwoTimeGF.from_arrays(GL, GG, dt=0.05, frontier=cap)
        sigma = kb.init_sigma_history(n_k, cap)
        kb.evaluate_sigma_batched(state, sigma, n, grid, u)
        assert rel_err(sigma.lesser, g[f"SL_{n}"]) <= 1e-12
        assert rel_err(sigma.greater, g[f"SG_{n}"]) <= 1e-12


# ------------------------------------------------------------------ collision (kernel level)
class _Arrays:
    def __init__(self, lesser, greater, dt=0.05):
        self.lesser, self.greater, self.dt = lesser, greater, dt
        self.n_k_local = lesser.shape[0]


@pytest.mark.parametrize("kind", ["trapezoid", "simpson"])
@pytest.mark.parametrize("mode", ["as-printed", "langreth"])
@pytest.mark.parametrize("n", [0, 1, 2, 5, 8])
def test_collision_matches_reference_golden(kind, mode, n):
    g = load_golden("collision.npz")
    state = _Arrays(g["GL"], g["GG"], float(g["dt"]))
    sigma = _Arrays(g["SL"], g["SG"])
    c = kb.collision_frontier(state, sigma, n, kb.QuadratureRule(kind), limit_mode=mode)
    tag = f"{kind}_{mode}_{n}"
    for name, got in (("lr", c.lesser_row), ("gr", c.greater_row), ("lc", c.lesser_col), ("gc", c.greater_col)):
        want = g[f"{name}_{tag}"]
        assert got.shape == want.shape
        if want.size:
            assert rel_err(got, want) <= 1e-12, name


def test_collision_pair_matches_reference_golden():
    g = load_golden("collision.npz")
    state = _Arrays(g["GL"], g["GG"], float(g["dt"]))
    sigma = _Arrays(g["SL"], g["SG"])
    assert rel_err(kb.collision_lesser(state, sigma, 1, 5, 2), g["pair_lesser_k1_i5_l2"]) <= 1e-12
    assert rel_err(kb.collision_greater(state, sigma, 2, 3, 6), g["pair_greater_k2_i3_l6"]) <= 1e-12


def _random_sym_history(n_k, cap, seed):
    GL, GG = O.random_mirrored_state(n_k, cap, cap, seed)
    rng = np.random.default_rng(seed + 1)
    shape = GL.shape
    SL = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    SG = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    for n in range(1, cap + 1):
        SL[:, :, :, n, :n] = -np.conj(np.swapaxes(SL[:, :, :, :n, n], 1, 2))
        SG[:, :, :, :n, n] = -np.conj(np.swapaxes(SG[:, :, :, n, :n], 1, 2))
    return GL, GG, SL, SG


@pytest.mark.parametrize("kind", ["trapezoid", "simpson"])
@pytest.mark.parametrize("mode", ["as-printed", "langreth"])
@pytest.mark.parametrize("n", [31, 32, 33, 63, 64, 65, 127, 128, 200, 301])
def test_collision_multi_tile_matches_oracle(kind, mode, n):
    """Task edges of K2 (32 slices x 32 points per warp) against the oracle."""
    n_k = 2
    GL, GG, SL, SG = _random_sym_history(n_k, n, seed=n)
    c = kb.collision_frontier(_Arrays(GL, GG), _Arrays(SL, SG), n, kb.QuadratureRule(kind), limit_mode=mode)
    want = O.collision_frontier(GL, GG, SL, SG, n, 0.05, kind, mode)
    assert rel_err(c.lesser_row, want.lesser_row) <= 1e-12
    assert rel_err(c.greater_row, want.greater_row) <= 1e-12
    assert rel_err(c.lesser_col, want.lesser_col) <= 1e-12
    assert rel_err(c.greater_col, want.greater_col) <= 1e-12


def test_back_to_back_collision_launches_are_ordered():
    """kbe_collision_frontier launched twice in a row (no Sigma launch between) must not
    overlap the two grids (they share the task queue): the second evaluation equals a
    lone one."""
    from paper_2505_19467_b200 import _lib
    from paper_2505_19467_b200._device import stream_ptr
    from paper_2505_19467_b200.propagator import _Workspace
    from paper_2505_19467_b200.state import pack_history

    n_k, n = 4, 300
    GL, GG, SL, SG = _random_sym_history(n_k, n, seed=5)
    dev = torch.device("cuda:0")
    ws = _Workspace.for_collision(n_k, n, 0.05, 0, pack_history(GL, GG, n, n).to(dev),
                                  pack_history(SG, SL, n, n).to(dev), dev)
    L, P, st = _lib.lib(), ws.problem_ptr(), stream_ptr()

    def rows(seq):
        for m in seq:
            _lib.check(L.kbe_collision_frontier(P, m, 0, st))
        f = seq[-1]
        out = [torch.empty((n_k, 2, 2, f + 1), dtype=torch.complex128, device=dev) for _ in range(2)]
        out += [torch.empty((n_k, 2, 2, f), dtype=torch.complex128, device=dev) for _ in range(2)]
        _lib.check(L.kbe_collision_slice(P, f, *[t.data_ptr() for t in out], st))
        torch.cuda.synchronize()
        return [t.cpu().numpy() for t in out]

    for f in (n, n - 40):
        lone = rows([f])
        for _ in range(3):
            for a, b in zip(rows([n, n - 40, n, f]), lone):
                assert np.array_equal(a, b)


def test_unknown_limit_mode_is_rejected():
    g = load_golden("collision.npz")
    with pytest.raises(kb.ConfigError):
        kb.collision_frontier(_Arrays(g["GL"], g["GG"]), _Arrays(g["SL"], g["SG"]), 3, limit_mode="retarded")


# ------------------------------------------------------------------ trajectories (reference goldens)
def _driver_from_fixture(g):
    model = kb.ModelConfig(
        band_gap=float(g["band_gap"]), hopping=float(g["hopping"]),
        u_protocol=(float(g["u_protocol"]) if g["u_protocol"].ndim == 0 else g["u_protocol"]),
        pulse_intensity=float(g["pulse_intensity"]), pulse_center=float(g["pulse_center"]),
        dipole=complex(g["dipole"]), hf_mode=str(g["hf_mode"]),
        eps_c_table=g["eps_c_table"] if "eps_c_table" in g else None,
        eps_v_table=g["eps_v_table"] if "eps_v_table" in g else None,
    )
    cfg = kb.StepConfig(dt=float(g["dt"]), n_steps=int(g["n_steps"]), eps=float(g["eps"]),
                        max_iter=int(g["max_iter"]), quadrature=str(g["quadrature"]),
                        limit_mode=str(g["limit_mode"]), memory_budget=1 << 40)
    return kb.PropagationDriver(kb.build_kgrid(int(g["n_k"])), model, cfg)


TRAJ = ["traj_nk4_full.npz", "traj_hf.npz", "traj_simpson.npz", "traj_langreth.npz", "traj_nk64_synth.npz",
        "traj_dimer.npz", "traj_free.npz", "traj_nk16.npz"]


@pytest.mark.parametrize("name", TRAJ)
def test_trajectory_matches_reference_golden(name):
    g = load_golden(name)
    drv = _driver_from_fixture(g)
    reps = drv.run()
    N = int(g["n_steps"])
    GL, GG = drv.state.lesser, drv.state.greater
    idx = np.arange(N + 1)
    assert rel_err(GL[:, :, :, idx, idx], g["diag_lesser"]) <= 1e-10
    assert rel_err(GG[:, :, :, idx, idx], g["diag_greater"]) <= 1e-10
    assert rel_err(GL[:, :, :, N, :], g["final_row_lesser"]) <= 1e-10
    assert rel_err(GG[:, :, :, :, N], g["final_col_greater"]) <= 1e-10
    np.testing.assert_allclose([r.density for r in reps], g["density"], rtol=0, atol=1e-12)
    np.testing.assert_allclose([r.anticommutation_drift for r in reps], g["drift"], rtol=0, atol=1e-10)
    flips = np.sum(np.array([r.iterations for r in reps]) != g["iterations"])
    assert flips <= max(1, N // 50)
    if "GL" in g:
        assert rel_err(GL, g["GL"]) <= 1e-10
        assert rel_err(GG, g["GG"]) <= 1e-10
        assert rel_err(drv.sigma.lesser, g["SL"]) <= 1e-10
        assert rel_err(drv.sigma.greater, g["SG"]) <= 1e-10
    if "rows_lesser" in g:
        for s, row, col in zip(g["row_steps"], g["rows_lesser"], g["cols_greater"]):
            assert rel_err(GL[:, :, :, s, :], row) <= 1e-10
            assert rel_err(GG[:, :, :, :, s], col) <= 1e-10


def test_step_by_step_equals_batched_run():
    g = load_golden("traj_nk4_full.npz")
    a = _driver_from_fixture(g)
    ra = a.run()
    b = _driver_from_fixture(g)
    rb = [b.step() for _ in range(int(g["n_steps"]))]
    assert [r.iterations for r in ra] == [r.iterations for r in rb]
    assert torch.equal(a.state.hist, b.state.hist)       # bitwise determinism
    assert torch.equal(a.sigma.hist, b.sigma.hist)


def test_poisoned_state_raises():
    model = kb.ModelConfig(u_protocol=1.0, pulse_intensity=0.2, pulse_center=0.1)
    drv = kb.PropagationDriver(kb.build_kgrid(4), model, kb.StepConfig(dt=0.02, n_steps=10))
    drv.step()
    drv.state.hist[0, kb_slice_entry(1)] = complex(float("nan"), 0.0)
    with pytest.raises(kb.PoisonedStateError):
        drv.run()


@pytest.mark.parametrize("n_k,n_steps", [(2, 3), (4, 40), (16, 33)])
def test_init_state_is_the_reference_ground_state(n_k, n_steps):
    """init_state (ref state.py:56-87): G<(0,0)_00 = i, G>(0,0)_11 = -i for every k, zero
    elsewhere, in the packed layout's slice 0 -- and the same history kbe_init_history
    gives the driver."""
    st = kb.init_state(kb.build_kgrid(n_k), n_steps, 0.02)
    want_l = np.zeros((n_k, 2, 2, n_steps + 1, n_steps + 1), dtype=complex)
    want_g = np.zeros_like(want_l)
    want_l[:, 0, 0, 0, 0] = 1.0j
    want_g[:, 1, 1, 0, 0] = -1.0j
    assert np.array_equal(st.lesser, want_l)
    assert np.array_equal(st.greater, want_g)
    drv = kb.PropagationDriver(kb.build_kgrid(n_k), kb.ModelConfig(u_protocol=1.0),
                               kb.StepConfig(dt=0.02, n_steps=n_steps))
    assert torch.equal(drv.state.slice_view(0), st.slice_view(0))
    assert kb.anticommutation_drift(st, 0) == 0.0


def kb_slice_entry(s):
    from paper_2505_19467_b200 import _lib
    return _lib.slice_offset(s)


def test_capacity_errors():
    model = kb.ModelConfig(u_protocol=1.0)
    with pytest.raises(kb.CapacityError):
        kb.PropagationDriver(kb.build_kgrid(16), model, kb.StepConfig(dt=0.02, n_steps=1000))
    drv = kb.PropagationDriver(kb.build_kgrid(2), model, kb.StepConfig(dt=0.02, n_steps=2))
    drv.run()
    with pytest.raises(kb.CapacityError):
        drv.step()


# ------------------------------------------------------------------ the bench workload, full length
def test_cfg2_full_propagation_matches_reference_golden():
    """BASELINE configs[1] (n_k=16, 1000 steps, U=0.5) against the REAL reference run
    in full (tests/golden/make_golden.py cfg2_full): final row/column, equal-time
    diagonals and per-step observables <= 1e-10."""
    import os
    from conftest import GOLDEN
    path = os.path.join(GOLDEN, "traj_cfg2_full.npz")
    if not os.path.exists(path):
        pytest.skip("traj_cfg2_full.npz not generated")
    g = np.load(path)
    N = int(g["n_steps"])
    model = kb.ModelConfig(u_protocol=float(g["u"]), pulse_intensity=float(g["pulse_intensity"]),
                           pulse_center=float(g["pulse_center"]))
    drv = kb.PropagationDriver(kb.build_kgrid(int(g["n_k"])), model,
                               kb.StepConfig(dt=float(g["dt"]), n_steps=N, memory_budget=1 << 40))
    reps = drv.run()
    sl = drv.state.slice_view(N).cpu().numpy()           # (k, 8, N+1): row G<(N, b), column G>(b, N)
    row = sl[:, 0:4, :].reshape(-1, 2, 2, N + 1)
    col = sl[:, 4:8, :].reshape(-1, 2, 2, N + 1)
    assert rel_err(row, g["final_row_lesser"]) <= 1e-10
    assert rel_err(col, g["final_col_greater"]) <= 1e-10
    diag = np.stack([drv.state.slice_view(s)[:, 0:4, s].cpu().numpy() for s in range(N + 1)], axis=-1)
    assert rel_err(diag.reshape(-1, 2, 2, N + 1), g["diag_lesser"]) <= 1e-10
    np.testing.assert_allclose([r.density for r in reps], g["density"], rtol=0, atol=1e-12)
    np.testing.assert_allclose([r.anticommutation_drift for r in reps], g["drift"], rtol=0, atol=1e-10)
    flips = np.sum(np.array([r.iterations for r in reps]) != g["iterations"])
    assert flips <= N // 50


def test_large_run_is_deterministic():
    """Two propagations through the TMA pipeline and the work queue are bitwise equal."""
    model = kb.ModelConfig(u_protocol=0.5, pulse_intensity=0.2, pulse_center=0.5)
    cfg = kb.StepConfig(dt=0.02, n_steps=400, memory_budget=1 << 40)
    a = kb.PropagationDriver(kb.build_kgrid(16), model, cfg)
    ra = a.run()
    b = kb.PropagationDriver(kb.build_kgrid(16), model, cfg)
    rb = b.run()
    assert [r.iterations for r in ra] == [r.iterations for r in rb]
    assert torch.equal(a.state.hist, b.state.hist)
    assert torch.equal(a.sigma.hist, b.sigma.hist)


@pytest.mark.parametrize("name", ["traj_nk4_full.npz", "traj_hf.npz", "traj_langreth.npz", "traj_free.npz"])
def test_graph_path_equals_stream_path(name, monkeypatch):
    """kbe_run's step graph (corrector iterations behind conditional nodes) is bitwise
    identical to the plain stream sequence in which converged iterations are no-ops."""
    g = load_golden(name)
    monkeypatch.setenv("KBE_GRAPH", "0")
    a = _driver_from_fixture(g)
    assert a.use_graph == 0
    ra = a.run()
    monkeypatch.setenv("KBE_GRAPH", "1")
    b = _driver_from_fixture(g)
    assert b.use_graph == 1
    rb = b.run()
    assert [r.iterations for r in ra] == [r.iterations for r in rb]
    assert [r.residual_history for r in ra] == [r.residual_history for r in rb]
    assert torch.equal(a.state.hist, b.state.hist)
    assert torch.equal(a.sigma.hist, b.sigma.hist)
    # the same graph replayed after a reset of the history
    c = _driver_from_fixture(g)
    rc = [c.step() for _ in range(int(g["n_steps"]))]
    assert [r.iterations for r in rc] == [r.iterations for r in rb]
    assert torch.equal(c.state.hist, b.state.hist)


@pytest.mark.parametrize("name", ["traj_nk16.npz", "traj_simpson.npz", "traj_nk64_synth.npz"])
def test_incremental_evaluations_match_full_evaluations(name, monkeypatch):
    """Repeated collision evaluations at one frontier with |dv| <= 1e-7 add M_fp32 dv to
    the previous partials (collision_kernel, incremental mode); the trajectory equals the
    all-FP64 one to 1e-13 with the same iteration counts."""
    g = load_golden(name)
    monkeypatch.setenv("KBE_INCR", "0")
    a = _driver_from_fixture(g)
    assert a.ws.g_sh is None
    ra = a.run()
    monkeypatch.setenv("KBE_INCR", "1")
    b = _driver_from_fixture(g)
    assert b.ws.g_sh is not None
    rb = b.run()
    assert [r.iterations for r in ra] == [r.iterations for r in rb]
    scale = float(a.state.hist.abs().max())
    assert float((a.state.hist - b.state.hist).abs().max()) <= 1e-13 * scale
    assert float((a.sigma.hist - b.sigma.hist).abs().max()) <= 1e-13 * float(a.sigma.hist.abs().max())


@pytest.mark.parametrize("quadrature", ["trapezoid", "simpson"])
def test_incremental_evaluations_match_full_evaluations_long(quadrature, monkeypatch):
    """The same over 300 steps at n_k = 8: the complex64 off-diagonal loops (blocks with
    wb0 + 32 <= s0, per-task parity weights) and taller tasks run from n = 64 on."""
    n_k, n_steps = 8, 300
    model = kb.ModelConfig(u_protocol=0.5, pulse_intensity=0.2, pulse_center=0.5)
    cfg = kb.StepConfig(dt=0.02, n_steps=n_steps, quadrature=quadrature, memory_budget=1 << 34)
    runs = []
    for incr in ("0", "1"):
        monkeypatch.setenv("KBE_INCR", incr)
        d = kb.PropagationDriver(kb.build_kgrid(n_k), model, cfg)
        assert (d.ws.g_sh is not None) == (incr == "1")
        runs.append((d, d.run()))
    (a, ra), (b, rb) = runs
    assert [r.iterations for r in ra] == [r.iterations for r in rb]
    scale = float(a.state.hist.abs().max())
    assert float((a.state.hist - b.state.hist).abs().max()) <= 1e-12 * scale
    assert float((a.sigma.hist - b.sigma.hist).abs().max()) <= 1e-12 * float(a.sigma.hist.abs().max())


@pytest.mark.parametrize("name", ["traj_nk16.npz", "traj_hf.npz", "traj_langreth.npz", "traj_dimer.npz"])
def test_speculative_iteration_counts_equal_full_launches(name, monkeypatch):
    """run() launches only as many corrector iterations as earlier steps needed and
    resumes a step that needs more (kbe_run_iters / kbe_resume_step); the result is
    bitwise the all-max_iter run, reports included."""
    g = load_golden(name)
    monkeypatch.setenv("KBE_SPECULATE", "0")
    a = _driver_from_fixture(g)
    ra = a.run()
    monkeypatch.setenv("KBE_SPECULATE", "1")
    b = _driver_from_fixture(g)
    assert b._speculative()
    b._spec_m = 1                      # force rollbacks at every increase
    rb = b.run()
    assert [r.iterations for r in ra] == [r.iterations for r in rb]
    assert [r.residual_history for r in ra] == [r.residual_history for r in rb]
    assert [r.density for r in ra] == [r.density for r in rb]
    assert torch.equal(a.state.hist, b.state.hist) and torch.equal(a.sigma.hist, b.sigma.hist)


# ------------------------------------------------------------------ derived observables
ENERGY = ["traj_dimer", "traj_hf", "traj_langreth", "traj_nk64_synth", "traj_simpson", "traj_nk4_full"]


@pytest.mark.parametrize("name", ENERGY)
def test_energy_matches_reference_build_h(name):
    """StepReport.energy (finish_kernel k-sums + the host hf term) against the energy of
    the reference trajectory computed with the reference's own build_h
    (tests/golden/energy.npz)."""
    g = load_golden(name + ".npz")
    e_ref = load_golden("energy.npz")[name]
    reps = _driver_from_fixture(g).run()
    e = np.array([r.energy for r in reps])
    assert rel_err(e, e_ref[1:]) <= 1e-10


def test_energy_of_cfg2_full_run():
    import os
    from conftest import GOLDEN
    if not os.path.exists(os.path.join(GOLDEN, "traj_cfg2_full.npz")):
        pytest.skip("traj_cfg2_full.npz not generated")
    g = load_golden("traj_cfg2_full.npz")
    model = kb.ModelConfig(u_protocol=float(g["u"]), pulse_intensity=float(g["pulse_intensity"]),
                           pulse_center=float(g["pulse_center"]))
    reps = kb.PropagationDriver(kb.build_kgrid(int(g["n_k"])), model,
                                kb.StepConfig(dt=float(g["dt"]), n_steps=int(g["n_steps"]),
                                              memory_budget=1 << 40)).run()
    assert rel_err([r.energy for r in reps], load_golden("energy.npz")["traj_cfg2_full"][1:]) <= 1e-10


@pytest.mark.parametrize("theta0", [1.0, 0.5])
def test_retarded_accessor_on_device(theta0):
    """G^R = theta(t - t') (G> - G<) from the device unpack equals the same formula on the
    reference's full arrays (traj_nk4_full.npz) and has G^R(t,t) = -i theta0 up to the
    anticommutation drift."""
    g = load_golden("traj_nk4_full.npz")
    drv = _driver_from_fixture(g)
    reps = drv.run()
    gr = drv.state.retarded(theta0)
    n1 = int(g["n_steps"]) + 1
    theta = np.tril(np.ones((n1, n1)), -1) + theta0 * np.eye(n1)
    ref = (g["GG"] - g["GL"]) * theta
    assert rel_err(gr, ref) <= 1e-10
    # bitwise the same formula applied to the device's own unpacked arrays
    np.testing.assert_array_equal(gr, (drv.state.greater - drv.state.lesser) * theta)
    idx = np.arange(n1)
    diag = gr[:, :, :, idx, idx]
    drift = max(r.anticommutation_drift for r in reps)
    assert np.abs(diag - (-1j * theta0) * np.eye(2)[None, :, :, None]).max() <= theta0 * drift + 1e-15


def test_step_timings_from_cuda_events():
    """StepReport.timings (sigma / collision / update seconds, the reference's KernelTimers)
    are filled when enabled, and timing changes no result."""
    g = load_golden("traj_nk16.npz")
    plain = _driver_from_fixture(g).run()
    drv = _driver_from_fixture(g)
    drv.timings_enabled = True
    timed = drv.run()
    for a, b in zip(plain, timed):
        assert a.density == b.density and a.iterations == b.iterations and a.residual == b.residual
        assert set(b.timings) == {"sigma", "collision", "update"}
        assert all(v > 0.0 for v in b.timings.values())
    assert plain[0].timings == {}
    one = _driver_from_fixture(g)
    one.timings_enabled = True
    rep = one.step()
    assert rep.timings["collision"] > 0.0 and rep.density == plain[0].density


# ------------------------------------------------------------------ K1 variants
@pytest.mark.parametrize("n_k,variant", [(6, "auto"), (10, "auto"), (12, "auto"), (24, "auto"), (2, "dft"),
                                         (8, "dft"), (16, "dft"), (32, "dft"), (6, "direct"), (2, "fft"),
                                         (4, "fft"), (8, "fft"), (16, "fft"), (32, "fft"), (128, "fft"),
                                         (128, "dft")])
def test_sigma_variant_trajectory_matches_oracle(n_k, variant, monkeypatch):
    """K1 as FFTs (power-of-two n_k), as DMMA DFT GEMMs (any even n_k; the default when n_k
    is not a power of two) and as the direct correlations all reproduce the oracle's
    trajectory, G and Sigma, to 1e-10 (selfenergy.py:59-325)."""
    monkeypatch.setenv("KBE_SIGMA", variant)
    n_steps = 25
    model = kb.ModelConfig(u_protocol=1.0, pulse_intensity=0.2, pulse_center=0.1)
    drv = kb.PropagationDriver(kb.build_kgrid(n_k), model, kb.StepConfig(dt=0.02, n_steps=n_steps))
    reps = drv.run()
    ref = O.OracleDriver(n_k, O.Model(u_protocol=1.0, pulse_intensity=0.2, pulse_center=0.1), 0.02, n_steps)
    ref_reps = ref.run()
    assert rel_err(drv.state.lesser, ref.GL) <= 1e-10
    assert rel_err(drv.state.greater, ref.GG) <= 1e-10
    assert rel_err(drv.sigma.lesser, ref.SL) <= 1e-10
    assert rel_err(drv.sigma.greater, ref.SG) <= 1e-10
    np.testing.assert_allclose([r.density for r in reps], [r.density for r in ref_reps], rtol=0, atol=1e-12)


@pytest.mark.parametrize("variant", ["fft", "dft", "direct"])
def test_sigma_variants_on_nk64_golden(variant, monkeypatch):
    """The n_k = 64 synthetic golden (the reference's own run) with each K1 variant."""
    monkeypatch.setenv("KBE_SIGMA", variant)
    g = load_golden("traj_nk64_synth.npz")
    drv = _driver_from_fixture(g)
    drv.run()
    N = int(g["n_steps"])
    assert rel_err(drv.state.lesser[:, :, :, N, :], g["final_row_lesser"]) <= 1e-10
    assert rel_err(drv.state.greater[:, :, :, :, N], g["final_col_greater"]) <= 1e-10


def test_sigma_variant_setter_rejects_unknown(monkeypatch):
    from paper_2505_19467_b200 import _lib
    assert _lib.lib().kbe_set_sigma_variant(7) == -1
    monkeypatch.setenv("KBE_SIGMA", "bogus")
    with pytest.raises(kb.ConfigError):
        kb.PropagationDriver(kb.build_kgrid(4), kb.ModelConfig(), kb.StepConfig(dt=0.02, n_steps=2))
