"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
layout helpers, and the host-side setup logic (no GPU compute)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden
from oracle import kbe_oracle as O

import paper_2505_19467_b200 as kb
from paper_2505_19467_b200 import _lib
from paper_2505_19467_b200.model import step_tables


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "kbe200.h")).read()
    return sorted(set(re.findall(r"\b(kbe_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    handle = ctypes.CDLL(_lib.LIB_PATH)
    declared = _declared_symbols()
    assert len(declared) >= 18
    for name in declared:
        assert hasattr(handle, name), name
        assert name in _lib.SIGNATURES, name


def test_abi_struct_and_layout():
    L = _lib.lib()
    assert L.kbe_sizeof_problem() == ctypes.sizeof(_lib.KbeProblem)
    acc = 0
    for s in range(300):
        assert L.kbe_slice_offset(s) == acc == _lib.slice_offset(s)
        assert L.kbe_plane_len(s) % 32 == 0 and s + 1 <= L.kbe_plane_len(s) <= s + 32
        acc += 8 * L.kbe_plane_len(s)
    assert L.kbe_tri_size(1000) == _lib.slice_offset(1001)
    # inside a slice: 4 KB blocks of 8 planes x 32 points, every (plane, point) exactly once
    pl = _lib.plane_len(100)
    idx = sorted(_lib.slice_index(c, b) for c in range(8) for b in range(pl))
    assert idx == list(range(8 * pl))
    assert _lib.slice_index(3, 37) == 256 + 3 * 32 + 5


def test_step_tables_match_oracle_model():
    for center in (0.5, 0.1, 0.33):
        model = kb.ModelConfig(u_protocol=np.linspace(0.5, 1.5, 201), pulse_intensity=0.2, pulse_center=center)
        om = O.Model(u_protocol=model.u_protocol, pulse_intensity=0.2, pulse_center=center)
        table = kb.u_values(model, 200)
        u_mid, amp = step_tables(model, table, 200, 0.02)
        for n in range(1, 201):
            t = (n - 0.5) * 0.02
            assert u_mid[n] == O.u_at(O.u_table(om, 200), t, 0.02)
            assert amp[n] == O.pulse(t, om, 0.02)
        assert np.count_nonzero(amp) == 1


def test_quadrature_weights_match_golden():
    g = load_golden("collision.npz")
    for n in (0, 1, 2, 3, 7, 8, 10):
        np.testing.assert_array_equal(kb.quadrature_weights(n, float(g["dt"]), "simpson"), g[f"wsimp_{n}"])
        np.testing.assert_array_equal(kb.quadrature_weights(n, float(g["dt"]), "trapezoid"), g[f"wtrap_{n}"])


def test_config_validation_matches_reference():
    with pytest.raises(kb.ConfigError):
        kb.build_kgrid(3)
    with pytest.raises(kb.ConfigError):
        kb.StepConfig(dt=0.0, n_steps=1).validate()
    with pytest.raises(kb.ConfigError):
        kb.Schedule(n_shards=3).validate(16)
    with pytest.raises(kb.ConfigError):
        kb.ModelConfig(hf_mode="maybe").validate()
    with pytest.raises(kb.ConfigError):
        kb.quadrature_weights(3, 0.1, "gauss")
    assert issubclass(kb.ConfigError, ValueError)


def test_public_names_cover_reference_api():
    names = """CollisionSlice QuadratureRule collision_frontier collision_greater collision_lesser
    quadrature_weights Schedule WorkerPool combine_shards execute plan CapacityError ConfigError
    PoisonedStateError TrajectoryFormatError IndexTables KGrid build_index_tables build_kgrid
    index_of_diff index_of_sum ModelConfig band_energies build_h pulse_amplitude u_values
    PropagationDriver StepConfig StepReport cayley_propagator run SigmaHistory assemble_sigma
    evaluate_sigma_batched init_sigma_history polarizability sigma_first sigma_second sigma_slice
    Observables TwoTimeGF anticommutation_drift gather init_state mirror_frontier observables_at
    scatter symmetry_residual""".split()
    missing = [n for n in names if not hasattr(kb, n)]
    assert not missing


def test_index_helpers_match_tables():
    for n_k in (2, 4, 16):
        t = kb.build_index_tables(kb.build_kgrid(n_k))
        for a in range(1, n_k + 1):
            for b in range(1, n_k + 1):
                assert kb.index_of_sum(a, b, n_k) == t.sum_table[a - 1, b - 1]
                assert kb.index_of_diff(a, b, n_k) == t.diff_table[a - 1, b - 1]


def test_ops_fail_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError, match="CUDA"):
        kb.PropagationDriver(kb.build_kgrid(2), kb.ModelConfig(), kb.StepConfig(dt=0.02, n_steps=2))
