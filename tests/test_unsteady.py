"""Moving-body loop (solve_unsteady / MotionSpec, reference solver.py:296-410)
against goldens made by the reference itself (tests/golden/make_unsteady_golden.py)."""
import numpy as np
import pytest

import paper_2111_09859_b200 as W
from paper_2111_09859_b200.errors import BodyOutsideDomainError

from goldens import load

CASES = ["piston_hj_UW", "cube_hj_UW"]


def _setup(z):
    ni, nj = (int(v) for v in z["dims"])
    lx, ly = (float(v) for v in z["extents"])
    g = W.build_cartesian(ni, nj, Lx=lx, Ly=ly)
    motion = W.MotionSpec(kind=str(z["motion_kind"]), physical_dt=float(z["physical_dt"]))
    af = float(z["alpha_f"])
    cfg = W.SolveConfig(formulation=W.FormulationConfig(kind=str(z["kind"])),
                        scheme=str(z["scheme"]),
                        filter_config=None if np.isnan(af) else W.FilterConfig(af), cfl=0.5,
                        tol=float(z["tol"]), max_iters=int(z["max_iters"]), arith="exact")
    return g, motion, cfg


@pytest.mark.parametrize("case", CASES)
def test_body_masks_match_reference(case):
    """Host-side motion law and mask quantisation are bit-identical."""
    z = load("unsteady_" + case)
    g, motion, _ = _setup(z)
    for s in range(int(z["n_steps"])):
        t = s * motion.physical_dt
        assert t == float(z["times"][s])
        assert np.array_equal(motion.body_mask(g, t), z[f"mask_{s}"])


def test_motion_validation_and_faces():
    with pytest.raises(ValueError):
        W.MotionSpec(kind="spinning")
    with pytest.raises(ValueError):
        W.MotionSpec(physical_dt=0.0)
    assert set(W.MotionSpec(kind="piston_sinusoid").default_faces(2).values()) == {"wall"}
    f = W.MotionSpec(kind="bouncing_cube").default_faces(2)
    assert f["jmin"] == f["jmax"] == "wall" and f["imin"] == f["imax"] == "farfield"
    assert W.MotionSpec(kind="none").body_mask(W.build_cartesian(5, 5), 0.0) is None
    m = W.MotionSpec(kind="piston_sinusoid", x0=0.95, amplitude=0.2)
    with pytest.raises(BodyOutsideDomainError):
        m.body_mask(W.build_cartesian(11, 11), 0.25)
    # the cube parks on the floor once the rebound apex is negligible
    c = W.MotionSpec(kind="bouncing_cube")
    assert c.cube_center_y(1e3, 0.0) == 0.5 * c.size


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_solve_unsteady_matches_reference(case):
    """Every physical step: iteration count, residual history and field
    bit-identical to the reference's warm-started re-solves."""
    z = load("unsteady_" + case)
    g, motion, cfg = _setup(z)
    reps = W.solve_unsteady(g, motion, cfg, int(z["n_steps"]))
    assert [r.iters for r in reps] == z["iters"].tolist()
    for s, r in enumerate(reps):
        assert r.time == float(z["times"][s])
        assert np.array_equal(r.residual_history, z[f"res_{s}"])
        assert np.array_equal(r.phi, z[f"phi_{s}"])
