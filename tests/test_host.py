"""Host-side logic of the drop-in layer (no GPU): configs, partitions, grid decode, synthesis."""

import json

import numpy as np
import pytest

import paper_1805_01759_b200 as tb
from oracle import tomo_oracle as O
from paper_1805_01759_b200.solver import block_ranges
from paper_1805_01759_b200.synth import make_config


def test_solver_config_mirrors_reference(tmp_path):
    with pytest.raises(tb.ConfigurationError):
        tb.SolverConfig(tol=0.0)
    with pytest.raises(tb.ConfigurationError):
        tb.SolverConfig(c_alpha=1.0)
    with pytest.raises(tb.ConfigurationError):
        tb.SolverConfig(num_blocks=0)
    with pytest.raises(tb.ConfigurationError):
        tb.SolverConfig(lambda_reg=-1.0)
    with pytest.raises(tb.ConfigurationError):
        tb.SolverConfig(theta_schedule="1/k")
    with pytest.raises(tb.ConfigurationError):
        tb.SolverConfig(fixed_iters=0)
    cfg = tb.SolverConfig(lambda_reg=0.3, num_blocks=4, seed=9)
    path = tmp_path / "solver.json"
    path.write_text(json.dumps(cfg.to_dict()))
    assert tb.SolverConfig.from_json(path) == cfg
    with pytest.raises(tb.ConfigurationError):
        tb.SolverConfig.from_dict({"momentum": 0.9})
    schema = tb.config_schema()
    assert set(schema) == set(tb.SolverConfig().to_dict())
    assert schema["c_alpha"]["default"] == 0.5
    c = tb.SolverConfig(fixed_iters=37, max_iters=10).to_c()
    assert c.fixed_iters == 37 and c.max_iters == 10 and c.backtrack_cap == 50


def test_pipeline_config_and_estimates():
    with pytest.raises(tb.ConfigurationError):
        tb.PipelineConfig(backend="nope")
    with pytest.raises(tb.ConfigurationError):
        tb.PipelineConfig(k_max=0)
    with pytest.raises(tb.ConfigurationError):
        tb.PipelineConfig(wiener_mu=-1)
    assert tb.PipelineConfig().backend == "rbpg" and tb.PipelineConfig().k_max == 2
    with pytest.raises(tb.EstimationError):
        tb.ScattererEstimates(1, np.zeros(0), np.zeros((0, 0)), np.zeros(0), np.zeros(0), np.zeros(0))
    est = tb.ScattererEstimates(1, np.array([0.5]), np.zeros((1, 0)), np.array([1 + 2j]), np.zeros(2), np.array([7]))
    rec = tb.estimates_to_record(3, est)
    assert rec == {"pixel_id": 3, "model_order": 1, "elevations_m": [0.5], "motion_params": [[]], "amplitudes": [[1.0, 2.0]], "support": [7]}


@pytest.mark.parametrize("m,j", [(4, 2), (10, 3), (13, 5), (200, 8), (300, 8), (1, 1), (160000, 8)])
def test_block_ranges_match_oracle(m, j):
    assert list(block_ranges(m, j)) == O.block_ranges(m, j)


def test_block_partition_probabilities():
    part = tb.BlockPartition(blocks=((0, 1), (1, 2)), lipschitz=np.array([1.0, 3.0]))
    np.testing.assert_allclose(part.probabilities, [0.25, 0.75])
    with pytest.raises(tb.ConfigurationError):
        tb.BlockPartition(blocks=((0, 1), (2, 3)), lipschitz=np.array([1.0, 1.0]))
    with pytest.raises(tb.ConfigurationError):
        block_ranges(3, 4)


def test_objective_validation():
    with pytest.raises(tb.ConfigurationError):
        tb.Objective(dictionary=np.eye(3), measurement=np.zeros(2), lambda_reg=1.0)
    with pytest.raises(tb.ConfigurationError):
        tb.Objective(dictionary=np.eye(2), measurement=np.zeros(2), lambda_reg=-0.1)
    obj = tb.Objective(dictionary=np.eye(2), measurement=[1, 2], lambda_reg=0.1)
    assert obj.dictionary.dtype == np.complex128 and obj.shape == (2, 2)


def test_grid_decode_matches_numpy():
    g = tb.ParameterGrid.uniform((0, 4), 5, (("linear", 0, 1, 3), ("seasonal", 0, 2, 4)))
    assert g.shape == (5, 3, 4) and g.flat_size == 60 and g.inner_size == 12
    for flat in (0, 7, 33, 59):
        idx = np.unravel_index(flat, g.shape)
        s, p = g.values_at(flat)
        assert s == g.elevation[idx[0]]
        assert p == (g.motion_axes[0][idx[1]], g.motion_axes[1][idx[2]])
    with pytest.raises(tb.GridError):
        g.flat_to_multi(60)
    with pytest.raises(tb.GridError):
        tb.ParameterGrid(elevation=np.array([0.0, 1.0, 3.0]))


def test_synthetic_configs_are_deterministic_and_prefix_stable():
    a = make_config(1, num_pixels=64)
    b = make_config(1)
    assert a.pixels.dtype == np.complex64 and a.dictionary.dtype == np.complex64
    assert a.dictionary.shape == (25, 200) and b.pixels.shape == (1024, 25)
    np.testing.assert_array_equal(a.pixels, b.pixels[:64])
    np.testing.assert_array_equal(make_config(1, num_pixels=64).pixels, a.pixels)
    c3 = make_config(3, num_pixels=8)
    assert c3.dictionary.shape == (50, 512)
    # every cfg1 pixel has 0-2 scatterers at distinct bins
    assert all(len(s) == len(set(s)) <= 2 for s in a.truth_support)


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(tb.NumericalError):
        tb.Dictionary(np.eye(3, dtype=np.complex64))


def test_stack_format_roundtrip_and_errors(tmp_path):
    from paper_1805_01759_b200.exceptions import StackFormatError
    from paper_1805_01759_b200.stack import Geometry, read_stack, write_stack

    g = Geometry(np.linspace(-100, 100, 5), np.linspace(0, 1, 5), 0.031, 6e5)
    px = (np.arange(15) + 1j * np.arange(15)).reshape(3, 5).astype(np.complex64)
    p = tmp_path / "x.tstk"
    write_stack(p, g, px)
    g2, px2 = read_stack(p)
    np.testing.assert_array_equal(px2, px)
    p.write_bytes(p.read_bytes()[:-3])
    with pytest.raises(StackFormatError):
        read_stack(p)
