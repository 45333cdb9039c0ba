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


def _canon_set(lines):
    out = [LS.canonical_polyline(ln) for ln in lines]
    return sorted(out, key=lambda p: (len(p), p[0, 0], p[0, 1]))


@pytest.mark.gpu
def test_isolines_and_perimeter_match_reference():
    """Marching squares (GPU cell kernel + host linking) on the reference's
    own signed-distance field: the same polylines vertex for vertex (bitwise
    coordinates) up to start vertex and direction; perimeter to round-off
    (hypot instead of the reference's sqrt of squares, another sum order)."""
    z = load("levelset")
    sdf = LS.SignedDistanceField(values=z["sdf0"], grid=_grid())
    lines = LS.extract_isolines(sdf, 0.0)
    ref = [z[f"iso_{q}"] for q in range(int(z["iso_n"]))]
    assert len(lines) == len(ref)
    for got, want in zip(_canon_set(lines), _canon_set(ref)):
        assert np.array_equal(got, want)
    assert LS.perimeter(lines) == pytest.approx(float(z["iso_perim"]), rel=1e-13)
    assert LS.extract_isolines(sdf, 1e3) == []


def test_linking_open_and_closed_chains():
    """Host linking alone: a closed square and an open 3-segment path given
    as shuffled segments come back as one ring and one open polyline."""
    sq = [(10, 11), (12, 11), (12, 13), (10, 13)]          # ring through ids 10..13
    op = [(1, 2), (3, 2), (3, 4)]                           # open 1-2-3-4
    ids = np.array(sq + op, dtype=np.int64)
    pts = ids[:, :, None].astype(float) * np.array([1.0, -1.0])
    lines = LS._link(ids, pts)
    assert sorted(len(ln) for ln in lines) == [4, 5]
    ring = next(ln for ln in lines if len(ln) == 5)
    assert np.array_equal(ring[0], ring[-1])
    assert sorted(ring[:-1, 0]) == [10.0, 11.0, 12.0, 13.0]
    path = next(ln for ln in lines if len(ln) == 4)
    assert list(LS.canonical_polyline(path)[:, 0]) == [1.0, 2.0, 3.0, 4.0]


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
    # perimeters: same vertices, lengths summed with hypot in another order
    assert np.allclose(res.perimeters[0.0], z["bb_p0"], rtol=1e-13, atol=0.0)
    assert np.allclose(res.perimeters[0.05], z["bb_p5"], rtol=1e-13, atol=0.0)
    assert np.array_equal(res.grad_drift, z["bb_drift"])
