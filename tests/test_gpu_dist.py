"""Slab-decomposed solve (dist.py) with P logical ranks on one GPU against
the single-GPU fused solve: bit-identical state and residual history with
the transposed axis-0 filter; round-off-level agreement with the
partitioned one (fast arithmetic)."""
import numpy as np
import pytest

from helpers import same

pytestmark = pytest.mark.gpu
W = pytest.importorskip("paper_2111_09859_b200")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


FACES = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "wall",
         "kmin": "periodic", "kmax": "periodic"}


def _run(P, arith, filter0, n0=32, overlap=True):
    from paper_2111_09859_b200 import dist
    dims = (n0, 48, 64)
    sp = (1.0 / n0, 1.0 / 47, 1.0 / 64)
    g = W.build_cartesian(*dims, Lx=1.0, Ly=1.0, Lz=1.0, periodic=(True, False, True))
    fc = W.FormulationConfig(kind="hj")
    filt = W.FilterConfig(0.49)
    steps = 6
    cfg = W.SolveConfig(formulation=fc, scheme="E6", filter_config=filt, tol=1e-15,
                        max_iters=steps, arith=arith)
    rng = np.random.default_rng(5)
    y = np.linspace(0.0, 1.0, dims[1])
    phi0 = np.broadcast_to(np.minimum(y, 1 - y)[None, :, None], dims).copy()
    phi0 += 1e-3 * rng.standard_normal(dims)
    ref = W.solve_steady(g, W.BoundarySpec(FACES), cfg, phi0=phi0)
    comm = dist.LocalComm(P)
    ds = dist.DistributedSolve(dims, sp, FACES, "E6", fc, filt, 0.5, 1e-15, steps, arith, comm,
                               list(range(P)), filter0=filter0, overlap=overlap)
    assert ds.overlap == (overlap and n0 // P >= 22)
    n = dims[0] // P
    # the single-GPU path applies the BCs to phi0 first; mirror it
    import torch
    phi_bc = phi0.copy()
    phi_bc[:, 0, :] = 0.0
    phi_bc[:, -1, :] = 0.0
    ds.set_state([phi_bc[r * n:(r + 1) * n] for r in range(P)])
    for _ in range(steps):
        ds.step()
    got = np.concatenate([s.cpu().numpy() for s in ds.state()], axis=0)
    hist = ds.history(0)
    ds.close()
    return got, hist, ref


@pytest.mark.parametrize("P,arith", [(1, "exact"), (2, "exact"), (4, "exact"), (2, "fast")])
def test_decomposed_equals_single(P, arith):
    got, hist, ref = _run(P, arith, "transpose")
    assert same(hist, ref.residual_history)
    assert same(got, ref.phi)


@pytest.mark.parametrize("P", [1, 2, 4])
def test_partitioned_axis0_filter(P):
    """Fast arithmetic with the axis-0 filter solved across the ranks
    (two per-line carry all_gathers instead of two slab transposes)."""
    got, hist, ref = _run(P, "fast", "partitioned")
    scale = float(np.max(np.abs(ref.phi)))
    assert np.max(np.abs(got - ref.phi)) <= 1e-12 * scale
    assert np.allclose(hist, ref.residual_history, rtol=1e-9, atol=1e-15)


def test_slab_checks():
    from paper_2111_09859_b200 import dist
    with pytest.raises(ValueError):
        dist.Slab(30, 4, 0).check(48)
    with pytest.raises(ValueError):
        dist.Slab(32, 4, 0).check(30)


@pytest.mark.parametrize("P,arith,filter0", [(2, "exact", "transpose"), (2, "fast", "transpose"),
                                             (4, "fast", "partitioned")])
def test_overlapped_ghost_exchange(P, arith, filter0):
    """Stage kernels split into ghost-free interior planes (launched while
    the ghost planes are in flight) and the boundary planes: same results."""
    got, hist, ref = _run(P, arith, filter0, n0=32 * P)
    if filter0 == "transpose":
        assert same(hist, ref.residual_history)
        assert same(got, ref.phi)
    else:
        scale = float(np.max(np.abs(ref.phi)))
        assert np.max(np.abs(got - ref.phi)) <= 1e-12 * scale
