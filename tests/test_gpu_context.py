"""Context reuse: the library's parked-context pool (wd_create / wd_destroy)
and the Python-level cache of the operator entry points must never change a
result -- reused contexts against fresh ones, after tolerance / max_iters
changes (captured graphs invalidated) and after a grid's metrics change."""
import dataclasses

import numpy as np
import pytest

from helpers import same

pytestmark = pytest.mark.gpu
W = pytest.importorskip("paper_2111_09859_b200")

PLATE = {"imin": "farfield", "imax": "farfield", "jmin": "wall", "jmax": "farfield"}


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_parked_context_reuse_is_invisible(monkeypatch):
    g = W.build_cartesian(41, 21, Lx=2.0, Ly=1.0)
    cfg = W.SolveConfig(formulation=W.FormulationConfig(kind="hj"), scheme="E4",
                        filter_config=W.FilterConfig(0.49), tol=1e-12, max_iters=30, arith="exact")
    monkeypatch.setenv("WD_NO_CTX_POOL", "1")
    fresh = W.solve_steady(g, W.BoundarySpec(PLATE), cfg)
    fresh20 = W.solve_steady(g, W.BoundarySpec(PLATE), dataclasses.replace(cfg, max_iters=20))
    monkeypatch.delenv("WD_NO_CTX_POOL")
    a = W.solve_steady(g, W.BoundarySpec(PLATE), cfg)
    b = W.solve_steady(g, W.BoundarySpec(PLATE), cfg)                       # parked context
    c = W.solve_steady(g, W.BoundarySpec(PLATE), dataclasses.replace(cfg, max_iters=20))
    d = W.solve_steady(g, W.BoundarySpec(PLATE), dataclasses.replace(cfg, tol=1e-3))
    for rep in (a, b):
        assert rep.iters == 30 and same(rep.phi, fresh.phi)
        assert same(rep.residual_history, fresh.residual_history)
    assert c.iters == 20 and same(c.phi, fresh20.phi)
    # a looser tolerance stops where the history first drops below it
    h = fresh.residual_history
    stop = int(np.argmax(h <= 1e-3)) + 1 if np.any(h <= 1e-3) else 30
    assert d.iters == stop and same(d.residual_history, h[:stop])


def test_operator_cache_follows_the_grid():
    from paper_2111_09859_b200 import formulations as F, _context
    g = W.build_sinusoidal_bump(33, 17, scheme="E4")
    fc = W.FormulationConfig(kind="hj")
    phi = np.random.default_rng(0).random(g.dims)
    k1 = F.tendency(phi, g, "E4", fc)
    n_ctx = len(_context._CACHE)
    k2 = F.tendency(phi, g, "E4", fc)          # cached context
    assert len(_context._CACHE) == n_ctx and same(k1, k2)
    # new metrics on the same grid object: the cached context must not be used
    g.metrics = 2.0 * g.metrics
    k3 = F.tendency(phi, g, "E4", fc)
    _context.drop_cached()
    k4 = F.tendency(phi, g, "E4", fc)          # fresh context, same answer
    assert same(k3, k4) and not same(k3, k1)
    _context.drop_cached()


def test_default_arithmetic_is_auto():
    """SolveConfig.arith defaults to "auto": fast arithmetic for the
    round-off-stable formulations (hj, poisson), exact for the chaotic ones."""
    mk = lambda kind: W.SolveConfig(formulation=W.FormulationConfig(kind=kind))  # noqa: E731
    assert mk("hj").arith == "auto"
    assert mk("hj").resolved_arith() == "fast" and mk("poisson").resolved_arith() == "fast"
    for kind in ("eikonal", "hj_lad", "hj_curvature"):
        assert mk(kind).resolved_arith() == "exact"
    import dataclasses
    assert dataclasses.replace(mk("hj"), arith="exact").resolved_arith() == "exact"
    with pytest.raises(ValueError):
        W.SolveConfig(arith="sloppy")
