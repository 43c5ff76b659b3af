"""Exact finite-difference weights: the host-side weight provider of the kernels.

The reference builds its weights with a Fornberg recursion in rational
arithmetic (/root/reference/pkg/src/fdroof/stencils.py:71-105) and the kernel
casts them through float64 to float32 at use (kernel.py:185, 199, 202).  The
weights are unique, so here they come from two independent derivations that
must agree exactly:

* closed forms for the centred first and second derivatives (the acoustic and
  TTI kernels), and
* a general exact Taylor-moment solve on arbitrary offsets (used for the
  half-integer staggered grid of the elastic kernel, which the reference's
  integer-offset recursion cannot produce, stencils.py:78-79).

`acoustic_weights_f32` reproduces the exact float32 values the reference
multiplies with, including the centre weight rounded as f32(3.0*w0) rather
than 3*f32(w0) (kernel.py:199; these differ at orders 20, 30 and 32).
"""

from fractions import Fraction
from functools import lru_cache
from math import factorial

import numpy as np

from .errors import ValidationError

MIN_ORDER = 2
MAX_ORDER = 32


def _check_order(order: int) -> int:
    if order % 2 != 0 or not MIN_ORDER <= order <= MAX_ORDER:
        raise ValidationError(
            f"accuracy order must be even and within [{MIN_ORDER}, {MAX_ORDER}], got {order}"
        )
    return order // 2


@lru_cache(maxsize=None)
def second_derivative_weights(order: int) -> tuple:
    """Exact weights for d2/dx2 on offsets -r..r (r = order/2), as Fractions.

    w_j = 2 (-1)^(j+1) (r!)^2 / (j^2 (r-j)! (r+j)!) for j >= 1 and
    w_0 = -2 sum_j w_j; index i of the tuple is offset i - r, matching the
    layout of FDWeights.weights in the reference (stencils.py:28-52).
    """
    r = _check_order(order)
    rf2 = factorial(r) ** 2
    side = [
        Fraction(2 * (-1) ** (j + 1) * rf2, j * j * factorial(r - j) * factorial(r + j))
        for j in range(1, r + 1)
    ]
    centre = -2 * sum(side, Fraction(0))
    return tuple(reversed(side)) + (centre,) + tuple(side)


@lru_cache(maxsize=None)
def first_derivative_weights(order: int) -> tuple:
    """Exact centred d/dx weights on offsets -r..r: w_j = (-1)^(j+1)(r!)^2/(j(r-j)!(r+j)!)."""
    r = _check_order(order)
    rf2 = factorial(r) ** 2
    side = [
        Fraction((-1) ** (j + 1) * rf2, j * factorial(r - j) * factorial(r + j))
        for j in range(1, r + 1)
    ]
    return tuple(-w for w in reversed(side)) + (Fraction(0),) + tuple(side)


def taylor_weights(offsets, deriv: int) -> tuple:
    """Exact weights w_i with sum_i w_i x_i^p = deriv! * [p == deriv], p < len(offsets).

    Gauss-Jordan elimination over Fractions; offsets may be any rationals
    (e.g. half-integers for staggered grids).
    """
    xs = [Fraction(x) for x in offsets]
    n = len(xs)
    if deriv >= n:
        raise ValidationError("need more points than the derivative order")
    rows = [[x ** p for x in xs] + [Fraction(factorial(deriv) if p == deriv else 0)]
            for p in range(n)]
    for col in range(n):
        piv = next(i for i in range(col, n) if rows[i][col] != 0)
        rows[col], rows[piv] = rows[piv], rows[col]
        inv = 1 / rows[col][col]
        rows[col] = [v * inv for v in rows[col]]
        for i in range(n):
            if i != col and rows[i][col] != 0:
                f = rows[i][col]
                rows[i] = [a - f * b for a, b in zip(rows[i], rows[col])]
    return tuple(rows[i][n] for i in range(n))


@lru_cache(maxsize=None)
def staggered_first_derivative_weights(order: int) -> tuple:
    """Exact d/dx weights c_1..c_r on the staggered offsets +-(k - 1/2).

    Derivative at x from samples at x + (k-1/2)h and x - (k-1/2)h:
    d/dx f ~ sum_k c_k (f(x+(k-1/2)h) - f(x-(k-1/2)h)) / h.
    """
    r = _check_order(order)
    offs = [Fraction(2 * k - 1, 2) for k in range(1, r + 1)]
    full = taylor_weights([-o for o in reversed(offs)] + offs, 1)
    return tuple(full[r:])


def abs_sum(weights) -> Fraction:
    return sum((abs(w) for w in weights), Fraction(0))


def a2_sum(order: int, dims: int = 3) -> float:
    """CFL weight sum a2 = dims * sum|w| of the 1D second derivative (stencils.py:108-113)."""
    if dims < 1:
        raise ValidationError(f"dims must be >= 1, got {dims}")
    return float(dims * abs_sum(second_derivative_weights(order)))


def acoustic_weights_f32(order: int) -> np.ndarray:
    """The float32 constants the reference kernel multiplies with, length r+1.

    [0] = f32(3.0 * float(w_0)), [j] = f32(float(w_j)) for j = 1..r
    (kernel.py:185, 199, 202: Fraction -> float64 -> float32).
    """
    r = order // 2
    w = [float(x) for x in second_derivative_weights(order)]
    out = np.empty(r + 1, dtype=np.float32)
    out[0] = np.float32(3.0 * w[r])
    for j in range(1, r + 1):
        out[j] = np.float32(w[r + j])
    return out
