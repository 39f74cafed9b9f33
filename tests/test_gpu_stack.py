"""The batched `tomobpdn solve` driver (TSTK1 in, ordered JSONL/CSV out) against the REAL reference
CLI output on the same stack (tests/golden/make_golden.py runs `tomobpdn solve`)."""

import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tb():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1805_01759_b200 as tb

    return tb


@pytest.mark.parametrize("gname,backend", [("g1", "rbpg"), ("g1", "fista"), ("g2", "rbpg")])
def test_solve_stack_matches_reference_cli(tb, golden, tmp_path, gname, backend):
    from paper_1805_01759_b200.stack import read_stack, solve_stack

    spath = tmp_path / "s.tstk"
    spath.write_bytes(golden["cli/stack"].tobytes())
    geom, px = read_stack(spath)
    assert px.shape == (25, 29)
    cfg = json.loads(str(golden["cli/config"]))
    pc = tb.PipelineConfig(solver=tb.SolverConfig.from_dict(cfg), backend=backend, k_max=2)
    out = tmp_path / "o.jsonl"
    recs = solve_stack(spath, json.loads(str(golden[f"cli/{gname}"])), pc, out_jsonl=out, out_csv=tmp_path / "o.csv")
    ref = [json.loads(line) for line in str(golden[f"cli/{gname}_{backend}_jsonl"]).splitlines()]
    assert [json.loads(line) for line in out.read_text().splitlines()] == recs
    assert len(recs) == len(ref)
    for r, q in zip(recs, ref):
        assert r["pixel_id"] == q["pixel_id"]
        assert r["model_order"] == q["model_order"], (r, q)
        assert r["support"] == q["support"]
        assert r["elevations_m"] == q["elevations_m"]
        assert r["motion_params"] == q["motion_params"]
        np.testing.assert_allclose(np.array(r["amplitudes"]).reshape(-1), np.array(q["amplitudes"]).reshape(-1), rtol=1e-5, atol=1e-6)
    assert (tmp_path / "o.jsonl.manifest.json").exists()
