"""Level-set burnback application (reference walldist/levelset.py; SURVEY
8(f)-3) against goldens made by the reference (tests/golden/make_levelset_golden.py)."""
import numpy as np
import pytest

import paper_2111_09859_b200 as W
from paper_2111_09859_b200 import levelset as LS
from paper_2111_09859_b200.errors import CflViolationError, InvalidPolygonError

from goldens import load


def _grid():
    return W.build_cartesian(49, 49, Lx=2.0, Ly=2.0)


def test_geometry_matches_reference():
    z = load("levelset")
    star = LS.GrainShape.star(n_legs=6, center=(1.0, 1.0))
    assert np.array_equal(star.polygon, z["star_poly"])
    g = _grid()
    inside = LS.point_in_polygon(g.coords.reshape(2, -1).T, star.polygon).reshape(g.dims)
    assert np.array_equal(inside, z["inside"])


def test_polygon_validation():
    with pytest.raises(InvalidPolygonError):
        LS.GrainShape(np.array([[0.0, 0.0], [1.0, 0.0]]))
    with pytest.raises(InvalidPolygonError):
        LS.GrainShape(np.array([[0.0, 0.0], [1.0, 1.0], [1.0, 0.0], [0.0, 1.0]]))  # bow tie
    with pytest.raises(InvalidPolygonError):
        LS.GrainShape.star(port_radius=0.3, fin_length=0.35)
    with pytest.raises(ValueError):
        LS.chamber_pressure(1.0, 1.0, 1.2, 1.0, 2.0, 1.0, 1.0)
    assert LS.chamber_pressure(2.0, 0.5, 0.0, 1.0, 3.0, 1.0, 1.0) == 2.0


def test_isolines_and_perimeter_match_reference():
    """Marching squares on the reference's own signed-distance field."""
    z = load("levelset")
    sdf = LS.SignedDistanceField(values=z["sdf0"], grid=_grid())
    lines = LS.extract_isolines(sdf, 0.0)
    assert len(lines) == int(z["iso_n"])
    for q, ln in enumerate(lines):
        assert np.array_equal(ln, z[f"iso_{q}"])
    assert LS.perimeter(lines) == float(z["iso_perim"])
    assert LS.extract_isolines(sdf, 1e3) == []


@pytest.mark.gpu
def test_init_and_steps_bitwise():
    z = load("levelset")
    g = _grid()
    star = LS.GrainShape.star(n_legs=6, center=(1.0, 1.0))
    sdf = LS.init_signed_distance(g, star)
    assert np.array_equal(sdf.values, z["sdf0"])
    s = sdf
    for k in range(3):
        s = LS.levelset_step(s, 0.3, 0.01, scheme="UW")
        assert np.array_equal(s.values, z[f"step{k + 1}"]), k
    aw = LS.levelset_step(sdf, 0.3, 0.01, scheme="E4", mode="as_written")
    assert np.array_equal(aw.values, z["step_aw"])
    with pytest.raises(CflViolationError):
        LS.levelset_step(sdf, 10.0, 1.0)


@pytest.mark.gpu
def test_burnback_run_matches_reference():
    z = load("levelset")
    res = LS.burnback_run(_grid(), LS.GrainShape.circle(0.5, center=(1.0, 1.0)), n_steps=4,
                          tracked_levels=(0.0, 0.05))
    assert np.array_equal(res.times, z["bb_times"])
    assert np.array_equal(res.perimeters[0.0], z["bb_p0"])
    assert np.array_equal(res.perimeters[0.05], z["bb_p5"])
    assert np.array_equal(res.grad_drift, z["bb_drift"])
