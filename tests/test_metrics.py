"""Validation metrics (reference walldist/metrics.py) against
goldens made by the reference itself (tests/golden/make_metrics_golden.py)."""
import numpy as np
import pytest

import paper_2111_09859_b200 as W
from paper_2111_09859_b200 import metrics as M

from goldens import load


def test_percentage_errors_and_histogram():
    z = load("metrics")
    pe = M.percentage_errors(z["pe_phi"], z["pe_exact"], exclude=z["pe_excl"])
    assert np.array_equal(pe, z["pe_out"])
    h = M.error_histogram_from_exact(z["pe_phi"], z["pe_exact"], 0.5, exclude=z["pe_excl"])
    assert h.total == pe.size and int(h.counts.sum()) == pe.size
    assert h.mean_pct == float(np.mean(pe))
    assert 0.0 <= h.fraction_within(-1.0, 1.0) <= 1.0


def test_timing_probe_needs_100_iterations():
    from paper_2111_09859_b200.errors import TooFewIterationsError
    rep = W.SolveReport(phi=np.zeros(3), iters=50, residual_history=np.zeros(50),
                        wall_seconds=np.linspace(0, 1, 50), converged=False)
    with pytest.raises(TooFewIterationsError):
        M.timing_probe(rep)


@pytest.mark.gpu
@pytest.mark.parametrize("d", [2, 3])
def test_sampled_wall_distance_bitwise(d):
    z = load("metrics")
    out = M.sampled_wall_distance(z[f"sw{d}_pts"], z[f"sw{d}_wall"])
    assert np.array_equal(out, z[f"sw{d}_out"])


@pytest.mark.gpu
def test_l2_norm_matches_reference():
    z = load("metrics")
    g = W.build_bump_grid(65, 33, W.BumpParams(), "E4")
    assert np.allclose(g.jacobian, z["l2_jac"], rtol=1e-13, atol=0)
    v = M.l2_norm(z["l2_phi"], z["l2_ex"], g)
    # deterministic GPU tree vs numpy's pairwise sum: round-off only
    assert abs(v - float(z["l2_out"])) <= 1e-13 * float(z["l2_out"])


@pytest.mark.gpu
@pytest.mark.parametrize("scheme", ["E4", "C6"])
def test_gradient_magnitude_bitwise(scheme):
    z = load("metrics")
    g = W.build_bump_grid(65, 33, W.BumpParams(), scheme)
    out = M.gradient_magnitude(z[f"gm_{scheme}_in"], g, scheme)
    assert np.array_equal(out, z[f"gm_{scheme}_out"])


@pytest.mark.gpu
def test_solve_l2_history():
    """solve_steady(exact=..., l2_every=5) samples the same L2 errors."""
    z = load("metrics")
    g = W.build_cartesian(41, 21, Lx=2.0, Ly=1.0)
    faces = {"imin": "farfield", "imax": "farfield", "jmin": "wall", "jmax": "farfield"}
    cfg = W.SolveConfig(formulation=W.FormulationConfig(kind="hj"), scheme="E4",
                        filter_config=W.FilterConfig(0.49), tol=1e-12, max_iters=40, l2_every=5,
                        arith="exact")
    rep = W.solve_steady(g, W.BoundarySpec(faces), cfg, exact=g.y.copy())
    h = np.asarray(rep.l2_history)
    assert h.shape == z["l2h"].shape
    assert np.array_equal(h[:, 0], z["l2h"][:, 0])
    assert np.allclose(h[:, 1], z["l2h"][:, 1], rtol=1e-12, atol=0)
