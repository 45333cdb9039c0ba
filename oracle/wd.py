"""numpy restatement of the reference wall-distance hot path (+ extensions).

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  The product package
never imports this module.

Every function names the reference lines it restates.  The arithmetic is
written to reproduce the reference's IEEE-754 operation order exactly
(left-to-right Python ``sum``, ``(0.5*a)*(...)`` constant folding, true
divisions, the LAPACK ``dgtsv`` elimination order with its row
interchanges), so that on non-extension paths the result is bit-identical
to the reference; ``tests/test_oracle_vs_reference.py`` checks that.

Data layout (as the reference, grid.py:5-11): fields are C-order
``(ni, nj[, nk])``; axis 0 = xi.  ``metrics[l, m] = d xi_l / d x_m``.

EXTENSIONS (no reference counterpart; documented in DESIGN.md sec. 3):
  * scheme "E6": interior 6th-order central difference
    ``(3/4)(w1-w-1) - (3/20)(w2-w-2) + (1/60)(w3-w-3)``, with the E4
    one-sided closures at rows 0, 1, n-2, n-1 and the E4 central relation at
    rows 2 and n-3;
  * periodic axes: explicit stencils, the 4th derivative, one-sided UW
    differences and the filter wrap around; compact derivatives and the
    filter solve the cyclic system by Sherman-Morrison on top of the
    dgtsv-order solve; boundary conditions skip periodic faces;
    coordinates may jump by a constant period vector across the wrap.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# --------------------------------------------------------------------------
# errors (reference errors.py:8-44).  The oracle raises plain classes with
# the reference's names; tests compare by name.


class OracleError(Exception):
    pass


class LineTooShortError(OracleError, ValueError):
    pass


class ZeroPivotError(OracleError, ValueError):
    pass


class SingularMetricError(OracleError, ValueError):
    pass


class DivergenceError(OracleError, RuntimeError):
    pass


class NegativeRadicandError(OracleError, ValueError):
    pass


# --------------------------------------------------------------------------
# scheme tables (operators.py:24-36)

#            alpha,      a,           b            (unit spacing)
SCHEME_TABLE = {
    "E2": (0.0, 1.0, 0.0),
    "E4": (0.0, 4.0 / 3.0, -1.0 / 3.0),
    "C4": (0.25, 1.5, 0.0),
    "C6": (1.0 / 3.0, 14.0 / 9.0, 1.0 / 9.0),
}
# EXTENSION: E6 interior a, b, c of
#   d_i = (a/2)(w_{i+1}-w_{i-1}) + (b/4)(w_{i+2}-w_{i-2}) + (c/6)(w_{i+3}-w_{i-3})
E6_ABC = (1.5, -0.6, 0.1)

MIN_LINE = {"UW": 3, "E2": 3, "E4": 5, "E6": 7, "C4": 7, "C6": 7}
SCHEMES = ("UW", "E2", "E4", "E6", "C4", "C6")
HALF_WIDTH = {"E2": 1, "E4": 2, "E6": 3, "C4": 1, "C6": 2, "UW": 1}


def _lines(v, axis):
    """View with the operated axis last."""
    return np.moveaxis(np.asarray(v, dtype=float), axis, -1)


def _unlines(w, axis):
    return np.ascontiguousarray(np.moveaxis(w, -1, axis))


def _need(n, k, what):
    if n < k:
        raise LineTooShortError(f"{what} needs at least {k} points, got {n}")


def _wrapped(w, j, offset):
    """w[..., j] for any integer j on a periodic line whose values jump by
    ``offset`` per period (coordinates of a periodic direction).  EXTENSION."""
    n = w.shape[-1]
    q, r = divmod(j, n)
    if q == 0 or offset == 0.0:
        return w[..., r]
    return w[..., r] + q * offset


# --------------------------------------------------------------------------
# LAPACK dgtsv restated (third-party routine behind operators.py:75-76:
# scipy.linalg.solve_banded((1,1)) -> ?gtsv; LAPACK 3.x dgtsv.f, partial
# pivoting with the |d_i| >= |dl_i| no-swap test, NRHS-independent
# arithmetic).  The factor is field-independent, so it is computed once per
# (matrix) and applied to every grid line.


@dataclass
class GtsvFactor:
    n: int
    swap: np.ndarray      # (n-1,) bool: rows i, i+1 interchanged at step i
    fact: np.ndarray      # (n-1,) elimination multipliers
    d: np.ndarray         # (n,)  U diagonal
    du: np.ndarray        # (n-1,) U first superdiagonal
    du2: np.ndarray       # (n-2,) U second superdiagonal (0 where no swap)


def gtsv_factor(lower, diag, upper) -> GtsvFactor:
    """Factor the tridiagonal whose row i is lower[i] x[i-1] + diag[i] x[i]
    + upper[i] x[i+1] (operators.py:56-58 convention)."""
    d = np.array(diag, dtype=float)
    n = d.shape[0]
    dl = np.array(lower, dtype=float)[1:].copy()
    du = np.array(upper, dtype=float)[:-1].copy()
    swap = np.zeros(max(n - 1, 0), dtype=bool)
    fact = np.zeros(max(n - 1, 0))
    for i in range(n - 1):
        if abs(d[i]) >= abs(dl[i]):
            if d[i] == 0.0:
                raise ZeroPivotError(f"zero pivot at row {i + 1}")
            f = dl[i] / d[i]
            d[i + 1] = d[i + 1] - f * du[i]
            dl[i] = 0.0
        else:
            f = d[i] / dl[i]
            d[i] = dl[i]
            t = d[i + 1]
            d[i + 1] = du[i] - f * t
            if i < n - 2:
                dl[i] = du[i + 1]
                du[i + 1] = -f * dl[i]
            du[i] = t
            swap[i] = True
        fact[i] = f
    if n and d[n - 1] == 0.0:
        raise ZeroPivotError(f"zero pivot at row {n}")
    du2 = dl[: max(n - 2, 0)].copy()
    return GtsvFactor(n, swap, fact, d, du, du2)


def gtsv_apply(fac: GtsvFactor, b):
    """Solve for every line: b has the system axis LAST (..., n)."""
    x = np.array(b, dtype=float, copy=True)
    n = fac.n
    if n == 1:
        return x / fac.d[0]
    for i in range(n - 1):
        f = fac.fact[i]
        if fac.swap[i]:
            t = x[..., i].copy()
            x[..., i] = x[..., i + 1]
            x[..., i + 1] = t - f * x[..., i + 1]
        else:
            x[..., i + 1] = x[..., i + 1] - f * x[..., i]
    x[..., n - 1] = x[..., n - 1] / fac.d[n - 1]
    x[..., n - 2] = (x[..., n - 2] - fac.du[n - 2] * x[..., n - 1]) / fac.d[n - 2]
    for i in range(n - 3, -1, -1):
        r = x[..., i] - fac.du[i] * x[..., i + 1]
        if fac.du2[i] != 0.0:
            r = r - fac.du2[i] * x[..., i + 2]
        x[..., i] = r / fac.d[i]
    return x


def solve_tridiagonal(lower, diag, upper, rhs):
    """operators.py:53-78: rhs (n,) or (n, m) with the system axis FIRST."""
    diag = np.asarray(diag, dtype=float)
    rhs = np.asarray(rhs, dtype=float)
    if diag.shape[0] == 1:
        if diag[0] == 0.0:
            raise ZeroPivotError("1x1 tridiagonal system with zero diagonal")
        return rhs / diag[0]
    fac = gtsv_factor(lower, diag, upper)
    return np.moveaxis(gtsv_apply(fac, np.moveaxis(rhs, 0, -1)), -1, 0)


# EXTENSION: cyclic (periodic) constant-coefficient tridiagonal
#   alpha x_{i-1} + x_i + alpha x_{i+1} = r_i  (indices mod n)
# by Sherman-Morrison: A = B + u v^T with gamma = -1,
#   B = A without corners, B00 = 1 - gamma, B_{n-1,n-1} = 1 - alpha^2/gamma
#   u = (gamma, 0.., 0, alpha), v = (1, 0.., 0, alpha/gamma)
#   x = y - f z,  B y = r, B z = u,  f = (v . y) / denom,
#   denom = 1 + (z0 + vn z_{n-1}).
# B is symmetric, so v . y = v . B^-1 r = h . r with h = B^-1 v: f is
# accumulated from the right-hand side, h_0 r_0 + h_1 r_1 + ... in row order,
# which lets a single back substitution apply the correction.


@dataclass
class CyclicFactor:
    n: int
    alpha: float
    base: GtsvFactor
    z: np.ndarray
    h: np.ndarray
    vn: float
    denom: float


def cyclic_factor(alpha: float, n: int) -> CyclicFactor:
    gamma = -1.0
    lower = np.full(n, alpha)
    upper = np.full(n, alpha)
    diag = np.ones(n)
    lower[0] = 0.0
    upper[-1] = 0.0
    diag[0] = 1.0 - gamma
    diag[-1] = 1.0 - alpha * alpha / gamma
    base = gtsv_factor(lower, diag, upper)
    u = np.zeros(n)
    u[0] = gamma
    u[-1] = alpha
    z = gtsv_apply(base, u)
    vn = alpha / gamma
    v = np.zeros(n)
    v[0] = 1.0
    v[-1] = vn
    h = gtsv_apply(base, v)
    denom = 1.0 + (z[0] + vn * z[n - 1])
    if denom == 0.0:
        raise ZeroPivotError("singular cyclic system")
    return CyclicFactor(n, alpha, base, z, h, vn, denom)


def cyclic_apply(cf: CyclicFactor, b):
    b = np.asarray(b, dtype=float)
    s = 0.0
    for i in range(cf.n):
        s = s + cf.h[i] * b[..., i]
    f = s / cf.denom
    y = gtsv_apply(cf.base, b)
    return y - np.asarray(f)[..., None] * cf.z


# --------------------------------------------------------------------------
# first derivative (operators.py:94-148) + EXTENSIONS E6 / periodic


def _explicit_rhs_interior(w, i, coeffs, get):
    """(0.5 a)(w+1 - w-1) + (0.25 b)(w+2 - w-2) [+ (c/6)(w+3 - w-3)]."""
    ca, cb, cc = coeffs
    r = ca * (get(i + 1) - get(i - 1))
    if cb is not None:
        r = r + cb * (get(i + 2) - get(i - 2))
    if cc is not None:
        r = r + cc * (get(i + 3) - get(i - 3))
    return r


def _interior_coeffs(scheme):
    if scheme == "E6":
        a, b, c = E6_ABC
        return (0.5 * a, 0.25 * b, c / 6.0)
    _, a, b = SCHEME_TABLE[scheme]
    return (0.5 * a, 0.25 * b if b != 0.0 else None, None)


def _e4_closures(w):
    """operators.py:119-127 (rows 0, 1, n-2, n-1)."""
    r0 = (-25.0 * w[..., 0] + 48.0 * w[..., 1] - 36.0 * w[..., 2]
          + 16.0 * w[..., 3] - 3.0 * w[..., 4]) / 12.0
    r1 = (-3.0 * w[..., 0] - 10.0 * w[..., 1] + 18.0 * w[..., 2]
          - 6.0 * w[..., 3] + w[..., 4]) / 12.0
    rm1 = (25.0 * w[..., -1] - 48.0 * w[..., -2] + 36.0 * w[..., -3]
           - 16.0 * w[..., -4] + 3.0 * w[..., -5]) / 12.0
    rm2 = (3.0 * w[..., -1] + 10.0 * w[..., -2] - 18.0 * w[..., -3]
           + 6.0 * w[..., -4] - w[..., -5]) / 12.0
    return r0, r1, rm2, rm1


def _compact_matrix(scheme, n):
    """operators.py:132-145."""
    alpha, _, b = SCHEME_TABLE[scheme]
    lower = np.full(n, alpha)
    diag = np.ones(n)
    upper = np.full(n, alpha)
    lower[0] = 0.0
    upper[0] = 3.0
    upper[-1] = 0.0
    lower[-1] = 3.0
    if b != 0.0:
        lower[1] = upper[1] = 0.25
        lower[-2] = upper[-2] = 0.25
    return lower, diag, upper


_FACTOR_CACHE: dict = {}


def compact_factor(scheme, n):
    key = ("compact", scheme, n)
    if key not in _FACTOR_CACHE:
        _FACTOR_CACHE[key] = gtsv_factor(*_compact_matrix(scheme, n))
    return _FACTOR_CACHE[key]


def compact_cyclic_factor(scheme, n):
    key = ("ccyc", scheme, n)
    if key not in _FACTOR_CACHE:
        _FACTOR_CACHE[key] = cyclic_factor(SCHEME_TABLE[scheme][0], n)
    return _FACTOR_CACHE[key]


def deriv(values, scheme, axis=0, periodic=False, offset=0.0):
    """First derivative along ``axis`` (unit spacing).

    Restates operators.py:94-148 for E2/E4/C4/C6 on non-periodic lines;
    EXTENSION for E6 and periodic lines (``offset`` = coordinate jump per
    period, used only for coordinate differencing in compute_metrics).
    """
    if scheme not in SCHEMES or scheme == "UW":
        raise ValueError(f"bad central scheme {scheme!r}")
    w = _lines(values, axis)
    n = w.shape[-1]
    coeffs = _interior_coeffs(scheme)
    compact = scheme in ("C4", "C6")
    if periodic:
        _need(n, 5, f"periodic {scheme} derivative")
        get = lambda j: _wrapped(w, j, offset)  # noqa: E731
        rhs = np.empty_like(w)
        for i in range(n):
            rhs[..., i] = _explicit_rhs_interior(w, i, coeffs, get)
        if compact:
            rhs = cyclic_apply(compact_cyclic_factor(scheme, n), rhs)
        return _unlines(rhs, axis)

    _need(n, MIN_LINE[scheme], f"{scheme} derivative")
    get = lambda j: w[..., j]  # noqa: E731
    rhs = np.empty_like(w)
    hw = HALF_WIDTH[scheme] if not compact else (2 if scheme == "C6" else 1)
    # vectorised interior (same per-element operation order as the loop)
    ca, cb, cc = coeffs
    lo, hi = hw, n - hw
    r = ca * (w[..., lo + 1:hi + 1] - w[..., lo - 1:hi - 1])
    if cb is not None:
        r = r + cb * (w[..., lo + 2:hi + 2 if hi + 2 <= n else None]
                      - w[..., lo - 2:hi - 2])
    if cc is not None:
        r = r + cc * (w[..., lo + 3:hi + 3 if hi + 3 <= n else None]
                      - w[..., lo - 3:hi - 3])
    rhs[..., lo:hi] = r
    if scheme == "E2":
        rhs[..., 0] = -1.5 * w[..., 0] + 2.0 * w[..., 1] - 0.5 * w[..., 2]
        rhs[..., -1] = 1.5 * w[..., -1] - 2.0 * w[..., -2] + 0.5 * w[..., -3]
        return _unlines(rhs, axis)
    if scheme in ("E4", "E6"):
        r0, r1, rm2, rm1 = _e4_closures(w)
        rhs[..., 0], rhs[..., 1], rhs[..., -2], rhs[..., -1] = r0, r1, rm2, rm1
        if scheme == "E6":  # EXTENSION: E4 central relation at rows 2, n-3
            c4a, c4b, _ = _interior_coeffs("E4")
            for i in (2, n - 3):
                rhs[..., i] = (c4a * (w[..., i + 1] - w[..., i - 1])
                               + c4b * (w[..., i + 2] - w[..., i - 2]))
        return _unlines(rhs, axis)
    # compact closures (operators.py:136-145)
    rhs[..., 0] = (-17.0 * w[..., 0] + 9.0 * w[..., 1] + 9.0 * w[..., 2]
                   - w[..., 3]) / 6.0
    rhs[..., -1] = (17.0 * w[..., -1] - 9.0 * w[..., -2] - 9.0 * w[..., -3]
                    + w[..., -4]) / 6.0
    if scheme == "C6":
        rhs[..., 1] = 0.75 * (w[..., 2] - w[..., 0])
        rhs[..., -2] = 0.75 * (w[..., -1] - w[..., -3])
    out = gtsv_apply(compact_factor(scheme, n), rhs)
    return _unlines(out, axis)


# --------------------------------------------------------------------------
# fourth derivative (operators.py:236-250) + periodic EXTENSION


def d4(values, axis=0, periodic=False):
    w = _lines(values, axis)
    n = w.shape[-1]
    _need(n, 5, "fourth derivative")
    out = np.empty_like(w)
    if periodic:
        g = lambda j: w[..., j % n]  # noqa: E731
        for i in range(n):
            out[..., i] = (g(i - 2) - 4.0 * g(i - 1) + 6.0 * g(i)
                           - 4.0 * g(i + 1) + g(i + 2))
        return _unlines(out, axis)
    out[..., 2:-2] = (w[..., :-4] - 4.0 * w[..., 1:-3] + 6.0 * w[..., 2:-2]
                      - 4.0 * w[..., 3:-1] + w[..., 4:])
    out[..., 0] = out[..., 2]
    out[..., 1] = out[..., 2]
    out[..., -1] = out[..., -3]
    out[..., -2] = out[..., -3]
    return _unlines(out, axis)


# --------------------------------------------------------------------------
# implicit filter (operators.py:253-352) + periodic EXTENSION


def filter_coeffs(half: int, af: float):
    """operators.py:269-295 (identical expressions, identical rounding)."""
    if half == 1:
        return (0.5 + af, 0.5 + af)
    if half == 2:
        return ((5.0 + 6.0 * af) / 8.0, (1.0 + 2.0 * af) / 2.0,
                (-1.0 + 2.0 * af) / 8.0)
    if half == 3:
        return ((11.0 + 10.0 * af) / 16.0, (15.0 + 34.0 * af) / 32.0,
                (-3.0 + 6.0 * af) / 16.0, (1.0 - 2.0 * af) / 32.0)
    if half == 4:
        return ((93.0 + 70.0 * af) / 128.0, (7.0 + 18.0 * af) / 16.0,
                (-7.0 + 14.0 * af) / 32.0, (1.0 - 2.0 * af) / 16.0,
                (-1.0 + 2.0 * af) / 128.0)
    if half == 5:
        return ((193.0 + 126.0 * af) / 256.0, (105.0 + 302.0 * af) / 256.0,
                (-15.0 + 30.0 * af) / 64.0, (45.0 - 90.0 * af) / 512.0,
                (-5.0 + 10.0 * af) / 256.0, (1.0 - 2.0 * af) / 512.0)
    raise ValueError(f"no filter of half-order {half}")


def _filter_row(get, i, coeffs):
    """operators.py:298-302: c0 w_i + sum_k (0.5 c_k)(w_{i+k} + w_{i-k})."""
    r = coeffs[0] * get(i)
    for k in range(1, len(coeffs)):
        r = r + (0.5 * coeffs[k]) * (get(i + k) + get(i - k))
    return r


def filter_factor(af, n):
    key = ("filt", af, n)
    if key not in _FACTOR_CACHE:
        lower = np.full(n, af)
        diag = np.ones(n)
        upper = np.full(n, af)
        upper[0] = 0.0
        lower[-1] = 0.0
        _FACTOR_CACHE[key] = gtsv_factor(lower, diag, upper)
    return _FACTOR_CACHE[key]


def filter_cyclic_factor(af, n):
    key = ("fcyc", af, n)
    if key not in _FACTOR_CACHE:
        _FACTOR_CACHE[key] = cyclic_factor(af, n)
    return _FACTOR_CACHE[key]


def apply_filter(values, axis, af, pinned=None, periodic=False):
    """operators.py:305-352 (non-periodic); periodic = EXTENSION (all rows
    10th order, cyclic solve; requires af < 0.5)."""
    v = np.asarray(values, dtype=float)
    w = _lines(v, axis)
    n = w.shape[-1]
    if n < 3 and not periodic:
        out = v.copy()
        if pinned is not None:
            out[pinned] = v[pinned]
        return out
    rhs = np.empty_like(w)
    if periodic:
        if af >= 0.5:
            raise ValueError("periodic filter needs alpha_f < 0.5")
        full = filter_coeffs(5, af)
        g = lambda j: w[..., j % n]  # noqa: E731
        for i in range(n):
            rhs[..., i] = _filter_row(g, i, full)
        sol = cyclic_apply(filter_cyclic_factor(af, n), rhs)
    else:
        g = lambda j: w[..., j]  # noqa: E731
        rhs[..., 0] = w[..., 0]
        rhs[..., -1] = w[..., -1]
        if n >= 12:
            full = filter_coeffs(5, af)
            r = full[0] * w[..., 5:n - 5]
            for k in range(1, 6):
                r = r + (0.5 * full[k]) * (w[..., 5 + k:n - 5 + k]
                                           + w[..., 5 - k:n - 5 - k])
            rhs[..., 5:n - 5] = r
            near = list(range(1, 5)) + list(range(n - 5, n - 1))
        else:
            near = list(range(1, n - 1))
        for i in near:
            half = min(i, n - 1 - i, 5)
            rhs[..., i] = _filter_row(g, i, filter_coeffs(half, af))
        sol = gtsv_apply(filter_factor(af, n), rhs)
    out = _unlines(sol, axis)
    if pinned is not None:
        out[pinned] = v[pinned]
    return out


# --------------------------------------------------------------------------
# UW helpers (operators.py:151-233) + periodic EXTENSION


def one_sided(values, axis=0, periodic=False):
    w = _lines(values, axis)
    n = w.shape[-1]
    _need(n, 3, "one-sided differences")
    B = np.empty_like(w)
    F = np.empty_like(w)
    B[..., 1:] = w[..., 1:] - w[..., :-1]
    F[..., :-1] = B[..., 1:]
    if periodic:
        B[..., 0] = w[..., 0] - w[..., -1]
        F[..., -1] = B[..., 0]
    else:
        B[..., 0] = F[..., 0]
        F[..., -1] = B[..., -1]
    return _unlines(B, axis), _unlines(F, axis)


def _sign1(x):
    return np.where(x >= 0.0, 1.0, -1.0)


def front_derivative(B, F):
    s_fb = _sign1(F + B)
    n_im1 = 0.25 * (1.0 + s_fb) * (1.0 + _sign1(B))
    n_ip1 = 0.25 * (1.0 - s_fb) * (1.0 - _sign1(F))
    return n_im1 * B + n_ip1 * F


def upwind_flux(u_hat, B, F):
    au = np.abs(u_hat)
    return 0.5 * ((u_hat + au) * B + (u_hat - au) * F)


# --------------------------------------------------------------------------
# grid (grid.py:27-217) + EXTENSIONS (periodic metrics, config generators)


@dataclass
class Grid:
    coords: np.ndarray
    metrics: np.ndarray | None = None
    jacobian: np.ndarray | None = None
    ref_length: float = 1.0
    periodic: tuple = ()
    periods: np.ndarray | None = None   # (d, d): periods[l, m] coord jump

    @property
    def ndim(self):
        return self.coords.shape[0]

    @property
    def dims(self):
        return tuple(self.coords.shape[1:])

    def is_periodic(self, l):
        return bool(self.periodic) and bool(self.periodic[l])

    def row_sumsq(self, l):
        """grid.py:60-63: sum over m of metrics[l, m]^2 (in m order)."""
        s = self.metrics[l, 0] * self.metrics[l, 0]
        for m in range(1, self.ndim):
            s = s + self.metrics[l, m] * self.metrics[l, m]
        return s

    def min_spacing(self):
        """grid.py:65-73."""
        sp = [1.0 / np.sqrt(self.row_sumsq(l)) for l in range(self.ndim)]
        return np.min(np.stack(sp), axis=0)


def cartesian(ni, nj, nk=None, Lx=1.0, Ly=1.0, Lz=None, origin=(0.0, 0.0, 0.0),
              ref_length=1.0, periodic=None):
    """grid.py:93-122.  EXTENSION: ``periodic`` axes use spacing L/n (no
    duplicated end node) instead of L/(n-1)."""
    dims = (ni, nj) if nk is None else (ni, nj, nk)
    ext = (Lx, Ly) if nk is None else (Lx, Ly, 1.0 if Lz is None else Lz)
    nd = len(dims)
    per = tuple(bool(p) for p in (periodic or (False,) * nd))
    axes = []
    spacing = []
    for d in range(nd):
        if per[d]:
            h = ext[d] / dims[d]
            axes.append(origin[d] + h * np.arange(dims[d]))
        else:
            h = ext[d] / (dims[d] - 1)
            axes.append(np.linspace(origin[d], origin[d] + ext[d], dims[d]))
        spacing.append(h)
    coords = np.stack(np.meshgrid(*axes, indexing="ij"))
    metrics = np.zeros((nd, nd) + dims)
    for d in range(nd):
        metrics[d, d] = 1.0 / spacing[d]
    jac = np.full(dims, float(np.prod([1.0 / s for s in spacing])))
    periods = np.zeros((nd, nd))
    for d in range(nd):
        if per[d]:
            periods[d, d] = ext[d]
    return Grid(coords, metrics, jac, ref_length, per, periods)


def compute_metrics(grid: Grid, scheme="E2"):
    """grid.py:180-217.  3-D uses the closed-form cofactor inverse
    (the reference's np.linalg.inv/det agree to round-off, not bitwise)."""
    nd = grid.ndim
    dims = grid.dims
    csch = "E2" if scheme == "UW" else scheme
    fwd = np.empty((nd, nd) + dims)
    for m in range(nd):
        for l in range(nd):
            off = 0.0
            if grid.periods is not None:
                off = float(grid.periods[l, m])
            fwd[m, l] = deriv(grid.coords[m], csch, axis=l,
                              periodic=grid.is_periodic(l), offset=off)
    metrics = np.empty((nd, nd) + dims)
    if nd == 2:
        det = fwd[0, 0] * fwd[1, 1] - fwd[0, 1] * fwd[1, 0]
        if np.any(np.abs(det) < 1e-14):
            raise SingularMetricError("metric matrix is singular at a node")
        inv_det = 1.0 / det
        metrics[0, 0] = fwd[1, 1] * inv_det
        metrics[0, 1] = -fwd[0, 1] * inv_det
        metrics[1, 0] = -fwd[1, 0] * inv_det
        metrics[1, 1] = fwd[0, 0] * inv_det
    else:
        a = fwd
        c00 = a[1, 1] * a[2, 2] - a[1, 2] * a[2, 1]
        c01 = a[1, 2] * a[2, 0] - a[1, 0] * a[2, 2]
        c02 = a[1, 0] * a[2, 1] - a[1, 1] * a[2, 0]
        det = a[0, 0] * c00 + a[0, 1] * c01 + a[0, 2] * c02
        if np.any(np.abs(det) < 1e-14):
            raise SingularMetricError("metric matrix is singular at a node")
        inv_det = 1.0 / det
        # inverse of a (a[m, l] = dx_m/dxi_l): metrics[l, m] = (a^-1)[l, m]
        metrics[0, 0] = c00 * inv_det
        metrics[1, 0] = c01 * inv_det
        metrics[2, 0] = c02 * inv_det
        metrics[0, 1] = (a[0, 2] * a[2, 1] - a[0, 1] * a[2, 2]) * inv_det
        metrics[1, 1] = (a[0, 0] * a[2, 2] - a[0, 2] * a[2, 0]) * inv_det
        metrics[2, 1] = (a[0, 1] * a[2, 0] - a[0, 0] * a[2, 1]) * inv_det
        metrics[0, 2] = (a[0, 1] * a[1, 2] - a[0, 2] * a[1, 1]) * inv_det
        metrics[1, 2] = (a[0, 2] * a[1, 0] - a[0, 0] * a[1, 2]) * inv_det
        metrics[2, 2] = (a[0, 0] * a[1, 1] - a[0, 1] * a[1, 0]) * inv_det
    grid.metrics = metrics
    grid.jacobian = inv_det
    return grid


def tanh_stretch(n, beta):
    """t in [0,1], clustered at 0: t = 1 + tanh(beta (s-1)) / tanh(beta)."""
    s = np.linspace(0.0, 1.0, n)
    return 1.0 + np.tanh(beta * (s - 1.0)) / np.tanh(beta)


def sinusoidal_bump(ni, nj, beta=1.069082, amp=0.1, length=4.0, top=1.0,
                    scheme="E2"):
    """EXTENSION (BASELINE config 3): y_w = amp sin(2 pi x / 1) on [0, length],
    wall-normal tanh stretching, flat top."""
    x = np.linspace(0.0, length, ni)
    yw = amp * np.sin(2.0 * np.pi * x)
    t = tanh_stretch(nj, beta)
    X = np.repeat(x[:, None], nj, axis=1)
    Y = yw[:, None] * (1.0 - t[None, :]) + top * t[None, :]
    g = Grid(np.stack([X, Y]), periodic=(False, False))
    return compute_metrics(g, scheme)


def annulus(ntheta, nr, r0=0.5, r1=5.0, beta=3.041018, scheme="E2"):
    """EXTENSION (BASELINE config 2): clockwise theta (J > 0), periodic."""
    th = -2.0 * np.pi * np.arange(ntheta) / ntheta
    r = r0 + (r1 - r0) * tanh_stretch(nr, beta)
    T, R = np.meshgrid(th, r, indexing="ij")
    g = Grid(np.stack([R * np.cos(T), R * np.sin(T)]), periodic=(True, False),
             periods=np.zeros((2, 2)))
    return compute_metrics(g, scheme)


def cylinder(ntheta, nr, nz, r0=0.5, r1=10.0, lz=4.0, beta=2.643022,
             scheme="E2"):
    """EXTENSION (BASELINE config 5): (theta periodic, r, z periodic)."""
    th = -2.0 * np.pi * np.arange(ntheta) / ntheta
    r = r0 + (r1 - r0) * tanh_stretch(nr, beta)
    z = lz * np.arange(nz) / nz
    T, R, Z = np.meshgrid(th, r, z, indexing="ij")
    periods = np.zeros((3, 3))
    periods[2, 2] = lz
    g = Grid(np.stack([R * np.cos(T), R * np.sin(T), Z]),
             periodic=(True, False, True), periods=periods)
    return compute_metrics(g, scheme)


# --------------------------------------------------------------------------
# boundary conditions (solver.py:32-110) + periodic EXTENSION

FACES = ("imin", "imax", "jmin", "jmax", "kmin", "kmax")


@dataclass
class Boundary:
    faces: dict
    solid_mask: np.ndarray | None = None

    def has_wall(self):
        if any(k == "wall" for k in self.faces.values()):
            return True
        return self.solid_mask is not None and bool(np.any(self.solid_mask))

    def pinned(self, dims):
        p = np.zeros(dims, dtype=bool)
        nd = len(dims)
        for ax in range(nd):
            if self.faces.get(FACES[2 * ax]) == "wall":
                p[_face(nd, ax, 0)] = True
            if self.faces.get(FACES[2 * ax + 1]) == "wall":
                p[_face(nd, ax, -1)] = True
        if self.solid_mask is not None:
            p |= self.solid_mask
        return p


def _face(nd, ax, pos):
    idx = [slice(None)] * nd
    idx[ax] = pos
    return tuple(idx)


def apply_bc(phi, bnd: Boundary):
    """solver.py:87-110: far-field copies (axis order), then walls, then mask."""
    nd = phi.ndim
    for ax in range(nd):
        if bnd.faces.get(FACES[2 * ax]) == "farfield":
            phi[_face(nd, ax, 0)] = phi[_face(nd, ax, 1)]
        if bnd.faces.get(FACES[2 * ax + 1]) == "farfield":
            phi[_face(nd, ax, -1)] = phi[_face(nd, ax, -2)]
    for ax in range(nd):
        if bnd.faces.get(FACES[2 * ax]) == "wall":
            phi[_face(nd, ax, 0)] = 0.0
        if bnd.faces.get(FACES[2 * ax + 1]) == "wall":
            phi[_face(nd, ax, -1)] = 0.0
    if bnd.solid_mask is not None:
        phi[bnd.solid_mask] = 0.0
    return phi


# --------------------------------------------------------------------------
# formulations (formulations.py:75-270)


@dataclass(frozen=True)
class Formulation:
    kind: str = "eikonal"
    epsilon: float = 0.2
    lad_c: float = 0.1
    eps0: float | None = None


def _pysum(terms):
    """Python ``sum`` order: ((0 + t0) + t1) + ..."""
    acc = 0
    for t in terms:
        acc = acc + t
    return acc


def _dphi(phi, grid, scheme):
    nd = grid.ndim
    if scheme == "UW":
        bf = tuple(one_sided(phi, l, grid.is_periodic(l)) for l in range(nd))
        return tuple(front_derivative(B, F) for B, F in bf), bf
    return tuple(deriv(phi, scheme, l, grid.is_periodic(l))
                 for l in range(nd)), None


def cartesian_components(dphi, grid):
    """formulations.py:87-91."""
    nd = grid.ndim
    return tuple(_pysum(grid.metrics[l, m] * dphi[l] for l in range(nd))
                 for m in range(nd))


def contravariant(U, grid):
    """formulations.py:94-98."""
    nd = grid.ndim
    return tuple(_pysum(grid.metrics[l, m] * U[m] for m in range(nd))
                 for l in range(nd))


def grad_vel(phi, grid, scheme):
    """formulations.py:101-111 -> (dphi, U, Uhat, bf)."""
    dphi, bf = _dphi(phi, grid, scheme)
    U = cartesian_components(dphi, grid)
    return dphi, U, contravariant(U, grid), bf


def advection(dphi, Uhat, bf, grid, scheme):
    """formulations.py:114-121."""
    if scheme == "UW":
        return _pysum(upwind_flux(Uhat[l], *bf[l]) for l in range(grid.ndim))
    return _pysum(Uhat[l] * dphi[l] for l in range(grid.ndim))


def lap_scheme(scheme):
    return "E2" if scheme == "UW" else scheme


def central_grad(phi, grid, scheme):
    """formulations.py:128-132."""
    cs = lap_scheme(scheme)
    d = tuple(deriv(phi, cs, l, grid.is_periodic(l)) for l in range(grid.ndim))
    return cartesian_components(d, grid), cs


def divergence(V, grid, cs):
    """formulations.py:135-143: m-outer, l-inner, from 0.0."""
    out = 0.0
    for m in range(grid.ndim):
        for l in range(grid.ndim):
            out = out + grid.metrics[l, m] * deriv(V[m], cs, l,
                                                   grid.is_periodic(l))
    return out


def gamma_std(phi, eps):
    return eps * np.asarray(phi, dtype=float)


def gamma_lad(phi, grid, eps, c):
    """formulations.py:164-176."""
    sensor = 0.0
    for l in range(grid.ndim):
        sensor = sensor + np.sqrt(grid.row_sumsq(l)) * d4(
            phi, l, grid.is_periodic(l))
    return np.minimum(eps * np.asarray(phi, dtype=float), c * np.abs(sensor))


def residual(phi, grid, scheme, fc: Formulation):
    """formulations.py:153-241."""
    if fc.kind == "eikonal":
        dphi, U, Uh, bf = grad_vel(phi, grid, scheme)
        return 1.0 - advection(dphi, Uh, bf, grid, scheme)
    if fc.kind in ("hj", "hj_lad"):
        dphi, U, Uh, bf = grad_vel(phi, grid, scheme)
        if fc.kind == "hj_lad":
            gam = gamma_lad(phi, grid, fc.epsilon, fc.lad_c)
        else:
            gam = gamma_std(phi, fc.epsilon)
        if scheme == "UW":
            Ul, cs = central_grad(phi, grid, scheme)
        else:
            Ul, cs = U, scheme
        lap = divergence(Ul, grid, cs)
        return 1.0 + gam * lap - advection(dphi, Uh, bf, grid, scheme)
    if fc.kind == "hj_curvature":
        dphi, U, Uh, bf = grad_vel(phi, grid, scheme)
        if scheme == "UW":
            Ul, cs = central_grad(phi, grid, scheme)
        else:
            Ul, cs = U, scheme
        lap = divergence(Ul, grid, cs)
        gmag = np.sqrt(_pysum(u * u for u in Ul))
        eps0 = fc.eps0 if fc.eps0 is not None else 1e-12 / grid.ref_length
        normal = tuple(u / (gmag + eps0) for u in Ul)
        kappa = divergence(normal, grid, cs)
        nu = 0.001 * (1.0 - gmag) ** 2
        gam = fc.epsilon * np.asarray(phi, dtype=float) + nu
        corr = lap - np.maximum(0.0, gmag * kappa)
        return 1.0 + gam * corr - advection(dphi, Uh, bf, grid, scheme)
    if fc.kind == "poisson":
        Ul, cs = central_grad(phi, grid, scheme)
        return -1.0 - divergence(Ul, grid, cs)
    raise ValueError(fc.kind)


def tendency(phi, grid, scheme, fc):
    """formulations.py:244-252."""
    r = residual(phi, grid, scheme, fc)
    return -r if fc.kind == "poisson" else r


def poisson_post(pp, grid, scheme):
    """formulations.py:255-270."""
    pp = np.asarray(pp, dtype=float)
    pp = np.where((pp < 0.0) & (pp > -1e-12), 0.0, pp)
    U, _ = central_grad(pp, grid, scheme)
    gsq = _pysum(u * u for u in U)
    rad = gsq + 2.0 * pp
    if np.any(rad < -1e-12):
        raise NegativeRadicandError(f"min radicand {np.min(rad):.3e}")
    rad = np.maximum(rad, 0.0)
    return -np.sqrt(gsq) + np.sqrt(rad)


# --------------------------------------------------------------------------
# driver (solver.py:113-286)

DT_GUARD = 1e-30


@dataclass
class Config:
    formulation: Formulation = field(default_factory=Formulation)
    scheme: str = "UW"
    alpha_f: float | None = None
    cfl: float = 0.5
    tol: float = 1e-5
    max_iters: int = 50000

    def uses_filter(self):
        return self.alpha_f is not None and self.scheme != "UW"


def local_timestep(phi, grid, fc, cfl, scheme):
    """solver.py:160-180."""
    sum_S = _pysum(grid.row_sumsq(l) for l in range(grid.ndim))
    if fc.kind == "poisson":
        return cfl / (2.0 * sum_S)
    _, _, Uh, _ = grad_vel(phi, grid, scheme)
    denom = _pysum(np.abs(u) for u in Uh)
    if fc.kind in ("hj", "hj_curvature"):
        denom = denom + 2.0 * gamma_std(phi, fc.epsilon) * sum_S
    elif fc.kind == "hj_lad":
        denom = denom + 2.0 * gamma_lad(phi, grid, fc.epsilon, fc.lad_c) * sum_S
    dt = cfl / (denom + DT_GUARD)
    return np.minimum(dt, cfl * grid.min_spacing())


def rk4_step(phi, grid, cfg: Config, dt, bnd: Boundary):
    """solver.py:183-218."""
    fc, sch = cfg.formulation, cfg.scheme

    def rate(p):
        return tendency(p, grid, sch, fc)

    k1 = rate(phi)
    p1 = apply_bc(phi + 0.5 * dt * k1, bnd)
    k2 = rate(p1)
    p2 = apply_bc(phi + 0.5 * dt * k2, bnd)
    k3 = rate(p2)
    p3 = apply_bc(phi + dt * k3, bnd)
    k4 = rate(p3)
    out = phi + (dt / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
    apply_bc(out, bnd)
    if cfg.uses_filter():
        pin = bnd.pinned(grid.dims)
        for ax in range(grid.ndim):
            out = apply_filter(out, ax, cfg.alpha_f, pinned=pin,
                               periodic=grid.is_periodic(ax))
        apply_bc(out, bnd)
    limit = 1e6 * grid.ref_length
    if not np.all(np.isfinite(out)) or np.max(np.abs(out)) > limit:
        raise DivergenceError(f"diverged (max |phi| > {limit:g})")
    return out


@dataclass
class Report:
    phi: np.ndarray
    iters: int
    residual_history: np.ndarray
    converged: bool
    phi_prime: np.ndarray | None = None
    diverged_at: int | None = None


def solve(grid, bnd: Boundary, cfg: Config, phi0=None, max_iters=None,
          raise_on_divergence=True):
    """solver.py:221-286 without the wall-clock bookkeeping."""
    if not bnd.has_wall():
        raise ValueError("boundary spec pins no wall nodes")
    lref = grid.ref_length
    fc = cfg.formulation
    phi = np.zeros(grid.dims) if phi0 is None else np.array(phi0, dtype=float)
    apply_bc(phi, bnd)
    active = None if bnd.solid_mask is None else ~bnd.solid_mask
    cap = cfg.max_iters if max_iters is None else min(max_iters, cfg.max_iters)
    hist = []
    converged = False
    it = 0
    while it < cap:
        dt = local_timestep(phi, grid, fc, cfg.cfl, cfg.scheme)
        try:
            new = rk4_step(phi, grid, cfg, dt, bnd)
        except DivergenceError:
            if raise_on_divergence:
                raise
            return Report(phi, it, np.asarray(hist), False, diverged_at=it + 1)
        delta = np.abs(new - phi)
        if active is not None:
            delta = delta[active]
        change = float(np.max(delta)) / lref
        if not math.isfinite(change):
            raise DivergenceError("non-finite residual")
        phi = new
        hist.append(change)
        it += 1
        if change <= cfg.tol:
            converged = True
            break
    rep = Report(phi, it, np.asarray(hist), converged)
    if fc.kind == "poisson":
        rep.phi_prime = phi
        rep.phi = apply_bc(poisson_post(phi, grid, cfg.scheme), bnd)
    return rep
