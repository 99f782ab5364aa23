"""KBE1 trajectory I/O, JSON config, CLI verbs, host reducers.

Pinned to fixtures produced by the real reference (tests/golden/make_golden.py
collision_row cli config reducers): the reference's KBE1 file of a 30-step
n_k=4 run, its observables/report tables and `inspect` output, its
validate_config results on 39 valid/invalid inputs, and its reducers.
CPU tests need no GPU; the `gpu` ones run the device path and compare.
"""

import contextlib
import io
import json
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, rel_err

import paper_2505_19467_b200 as kb  # noqa: E402
from paper_2505_19467_b200 import cli, trajio  # noqa: E402
from paper_2505_19467_b200.config import validate_config  # noqa: E402

REF_KBE = os.path.join(GOLDEN, "cli_run.kbe")


# ------------------------------------------------------------------ config (CPU)
def test_validate_config_matches_reference_on_all_cases():
    data = json.load(open(os.path.join(GOLDEN, "config_cases.json")))
    assert len(data["cases"]) == len(data["results"]) >= 39
    for case, want in zip(data["cases"], data["results"]):
        try:
            r = validate_config(case)
            got = {"ok": [r.n_k, r.step.dt, r.step.n_steps, r.step.memory_budget, r.step.max_iter,
                          r.step.quadrature, r.step.limit_mode, r.schedule.n_shards, r.schedule.workers,
                          [r.model.dipole.real, r.model.dipole.imag], r.model.hf_mode, r.seed]}
        except Exception as e:  # noqa: BLE001
            got = {"error": type(e).__name__, "message": str(e)}
        assert got == want, case


def test_workers_env_override(monkeypatch):
    base = {"n_k": 4, "dt": 0.02, "n_steps": 3}
    monkeypatch.setenv("KBESOLVE_WORKERS", "5")
    assert validate_config(base).schedule.workers == 5
    monkeypatch.setenv("KBESOLVE_WORKERS", "many")
    with pytest.raises(kb.ConfigError, match="KBESOLVE_WORKERS"):
        validate_config(base)


# ------------------------------------------------------------------ reducers (CPU host utilities)
def test_reducers_match_reference_bitwise():
    g = load_golden("reducers.npz")
    for tag in "abc":
        x, (axis, bs) = g[f"x_{tag}"], g[f"meta_{tag}"]
        assert np.array_equal(kb.chunk_partial_sums(x, int(bs), int(axis)), g[f"chunks_{tag}"])
        tot, rounds = kb.tree_reduce(x, int(axis), return_rounds=True)
        assert np.array_equal(tot, g[f"tree_{tag}"]) and rounds == int(g[f"rounds_{tag}"])
        assert np.array_equal(kb.sequential_reduce(x, int(axis)), g[f"seq_{tag}"])
    with pytest.raises(ValueError):
        kb.tree_reduce(np.zeros((3, 0)))


# ------------------------------------------------------------------ KBE1 (CPU)
def test_read_header_of_reference_file():
    h = trajio.read_header(REF_KBE)
    assert h == {"magic": "KBE1", "version": 1, "n_k": 4, "n_steps": 30, "dt": 0.02, "bands": 2, "flags": 0}


class _HostState:
    def __init__(self, lesser, greater, dt):
        self.lesser, self.greater, self.dt = lesser, greater, dt
        self.n_k_local, self.frontier = lesser.shape[0], lesser.shape[-1] - 1


def test_host_write_reproduces_reference_bytes(tmp_path):
    hdr, gl, gg = trajio.read_arrays(REF_KBE)
    assert gl.shape == (4, 2, 2, 31, 31) and gl.dtype == np.complex128
    out = tmp_path / "w.kbe"
    trajio.write_trajectory(str(out), _HostState(gl, gg, hdr["dt"]))
    assert out.read_bytes() == open(REF_KBE, "rb").read()


@pytest.mark.parametrize("mutate, msg", [
    (lambda b: b[:10], "truncated header"),
    (lambda b: b"XBE1" + b[4:], "bad magic"),
    (lambda b: b[:4] + (2).to_bytes(2, "little") + b[6:], "unsupported version"),
    (lambda b: b[:22] + bytes([3]) + b[23:], "unsupported band count"),
    (lambda b: b[:-16], "body has"),
])
def test_malformed_files_raise(tmp_path, mutate, msg):
    p = tmp_path / "bad.kbe"
    p.write_bytes(mutate(open(REF_KBE, "rb").read()))
    with pytest.raises(kb.TrajectoryFormatError, match=msg):
        trajio.read_arrays(str(p))


def test_cli_inspect_and_exit_codes(tmp_path):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        assert cli.main(["inspect", REF_KBE]) == cli.EXIT_OK
    assert buf.getvalue() == open(os.path.join(GOLDEN, "cli_run_inspect.txt")).read()
    bad = tmp_path / "bad.json"
    bad.write_text('{"n_k": 4, "dt": 0.02}')
    assert cli.main(["run", "--config", str(bad)]) == cli.EXIT_CONFIG
    bad.write_text("{not json")
    assert cli.main(["run", "--config", str(bad)]) == cli.EXIT_CONFIG
    assert cli.main(["inspect", str(tmp_path / "missing.kbe")]) == cli.EXIT_IO
    (tmp_path / "junk.kbe").write_bytes(b"KBE2" + bytes(40))
    assert cli.main(["inspect", str(tmp_path / "junk.kbe")]) == cli.EXIT_IO
    assert cli.main(["bench", "--kernel", "nope"]) == cli.EXIT_CONFIG
    assert cli.main(["scaling", "--mode", "diagonal"]) == cli.EXIT_CONFIG


# ------------------------------------------------------------------ device path
def _parse_table(path):
    """CSV -> float matrix; accepts the reference's numpy-2 'np.float64(x)' reprs."""
    lines = open(path).read().strip().splitlines()
    rows = [[float(c.replace("np.float64(", "").rstrip(")")) for c in ln.split(",")] for ln in lines[1:]]
    return lines[0], np.array(rows)


@pytest.mark.gpu
def test_collision_row_matches_reference_golden():
    g = load_golden("collision_row.npz")
    for tag in "abc":
        a = [g[f"{k}_{tag}"] for k in ("sl", "so")]
        vec = kb.collision_row(g[f"dg_{tag}"], g[f"gv_{tag}"], *a, g[f"w1_{tag}"], g[f"w2v_{tag}"])
        mat = kb.collision_row(g[f"dg_{tag}"], g[f"gm_{tag}"], *a, g[f"w1_{tag}"], g[f"w2m_{tag}"])
        assert rel_err(vec, g[f"vec_{tag}"]) <= 1e-12
        assert rel_err(mat, g[f"mat_{tag}"]) <= 1e-12
    with pytest.raises(ValueError):
        kb.collision_row(g["dg_a"], g["gm_a"], g["sl_a"], g["so_a"], g["w1_a"], g["w2v_a"])


@pytest.mark.gpu
def test_cli_run_matches_reference_tables_and_trajectory(tmp_path):
    cfg = json.load(open(os.path.join(GOLDEN, "cli_run_config.json")))
    cfg.update(trajectory_path=str(tmp_path / "t.kbe"), observables_path=str(tmp_path / "obs.csv"),
               report_path=str(tmp_path / "rep.csv"))
    (tmp_path / "run.json").write_text(json.dumps(cfg))
    assert cli.main(["run", "--config", str(tmp_path / "run.json")]) == cli.EXIT_OK
    h1, ours = _parse_table(tmp_path / "obs.csv")
    h2, ref = _parse_table(os.path.join(GOLDEN, "cli_run_observables.csv"))
    assert h1 == h2 and ours.shape == ref.shape
    np.testing.assert_allclose(ours[:, :4], ref[:, :4], rtol=0, atol=1e-12)     # t, n_v, n_c, density
    np.testing.assert_allclose(ours[:, 4], ref[:, 4], rtol=0, atol=1e-9)        # residuals (<= eps)
    h1, ours = _parse_table(tmp_path / "rep.csv")
    h2, ref = _parse_table(os.path.join(GOLDEN, "cli_run_report.csv"))
    assert h1 == h2 and ours.shape == ref.shape
    np.testing.assert_array_equal(ours[:, 0], ref[:, 0])
    assert np.sum(ours[:, 1] != ref[:, 1]) <= 1                                  # iteration counts
    np.testing.assert_allclose(ours[:, 4:6], ref[:, 4:6], rtol=0, atol=1e-10)    # drift, density
    assert np.all(ours[:, 7] > 0) and np.all(ours[:, 8] > 0)                      # t_collision, t_update (events)
    # trajectory: same header bytes, values within the trajectory tolerance
    ob, rb = open(tmp_path / "t.kbe", "rb").read(), open(REF_KBE, "rb").read()
    assert ob[:24] == rb[:24] and len(ob) == len(rb)
    _, gl, gg = trajio.read_arrays(str(tmp_path / "t.kbe"))
    _, rl, rg = trajio.read_arrays(REF_KBE)
    assert rel_err(gl, rl) <= 1e-10 and rel_err(gg, rg) <= 1e-10


@pytest.mark.gpu
def test_device_trajectory_round_trip_is_bitwise(tmp_path):
    model = kb.ModelConfig(u_protocol=1.0, pulse_intensity=0.2, pulse_center=0.1)
    drv = kb.PropagationDriver(kb.build_kgrid(4), model, kb.StepConfig(dt=0.02, n_steps=40))
    drv.run()
    drv.state.frontier = 25            # a partial block: only [0..25]^2 is written
    p = str(tmp_path / "x.kbe")
    kb.write_trajectory(p, drv.state)
    back = kb.read_trajectory(p)
    assert back.frontier == back.n_steps == 25
    want_l = drv.state.lesser[:, :, :, :26, :26]
    want_g = drv.state.greater[:, :, :, :26, :26]
    assert np.array_equal(back.lesser, want_l) and np.array_equal(back.greater, want_g)
    kb.write_trajectory(str(tmp_path / "y.kbe"), back)
    assert open(p, "rb").read() == open(tmp_path / "y.kbe", "rb").read()


@pytest.mark.gpu
def test_cli_bench_sweep_scaling_tables(tmp_path):
    for argv, header in [
        (["bench", "--kernel", "sigma", "--n-k", "8,16", "--reps", "2", "--warmup", "1"], cli.BENCH_HEADER),
        (["bench", "--kernel", "ci", "--n-k", "8", "--history", "64", "--reps", "2", "--warmup", "1"], cli.BENCH_HEADER),
        (["sweep", "--block-sizes", "64,128", "--n-k", "16", "--reps", "2", "--warmup", "1"], cli.BENCH_HEADER),
        (["scaling", "--mode", "weak", "--shards", "1,2", "--history", "32", "--reps", "2", "--warmup", "1"],
         cli.SCALING_HEADER),
        (["scaling", "--mode", "strong", "--shards", "1,2", "--n-k", "16", "--reps", "2", "--warmup", "1"],
         cli.SCALING_HEADER),
    ]:
        out = tmp_path / "t.csv"
        assert cli.main(argv + ["--out", str(out)]) == cli.EXIT_OK
        lines = out.read_text().strip().splitlines()
        assert lines[0] == header and len(lines) >= 2
        assert all(len(ln.split(",")) == len(header.split(",")) for ln in lines)


@pytest.mark.gpu
def test_cli_run_all_options_matches_reference(tmp_path):
    """hf_mode=on, Simpson, langreth, tabulated U(t) and bands, complex dipole, max_iter 8:
    the `run` tables and the trajectory against the reference CLI's own output."""
    cfg = json.load(open(os.path.join(GOLDEN, "cli_opts_config.json")))
    cfg.update(trajectory_path=str(tmp_path / "t.kbe"), observables_path=str(tmp_path / "obs.csv"),
               report_path=str(tmp_path / "rep.csv"))
    (tmp_path / "run.json").write_text(json.dumps(cfg))
    assert cli.main(["run", "--config", str(tmp_path / "run.json")]) == cli.EXIT_OK
    _, ours = _parse_table(tmp_path / "obs.csv")
    _, ref = _parse_table(os.path.join(GOLDEN, "cli_opts_observables.csv"))
    assert ours.shape == ref.shape
    np.testing.assert_allclose(ours[:, :4], ref[:, :4], rtol=0, atol=1e-12)
    _, ours = _parse_table(tmp_path / "rep.csv")
    _, ref = _parse_table(os.path.join(GOLDEN, "cli_opts_report.csv"))
    np.testing.assert_array_equal(ours[:, 0], ref[:, 0])
    assert np.sum(ours[:, 1] != ref[:, 1]) <= 1
    np.testing.assert_allclose(ours[:, 4:6], ref[:, 4:6], rtol=0, atol=1e-10)
    _, gl, gg = trajio.read_arrays(str(tmp_path / "t.kbe"))
    _, rl, rg = trajio.read_arrays(os.path.join(GOLDEN, "cli_opts.kbe"))
    assert rel_err(gl, rl) <= 1e-10 and rel_err(gg, rg) <= 1e-10
