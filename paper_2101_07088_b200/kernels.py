"""Host-side closed forms of the Gaussian-charge Ewald split.

Used by the planner (``tune_cutoff`` root-finds on the point gradient
kernel) and to derive the scalar constants the device kernels take as
arguments.  The pair sums themselves run on the GPU
(``csrc/nearfield.cu``), which evaluates the same expressions
(reference: ``slabewald/kernels.py:17-151``).

Convention: bare Coulomb pair potential q1 q2 / (4 pi eps r); every charge
is a normalised Gaussian of standard deviation ``g_w``; the screening
Gaussian has standard deviation ``1/(2 xi)``.
"""

import math

import numpy as np
from scipy.special import erf

FOUR_PI = 4.0 * np.pi
TWO_OVER_SQRTPI = 2.0 / np.sqrt(np.pi)

# Below these fractions of the kernel width the closed forms are replaced
# by their limits / Taylor series (reference kernels.py:46,65).
ERF_SMALL = 1e-10
DERF_SMALL = 1e-2


def split_widths(xi, g_w):
    """Total far-field width g_t = sqrt(g_w^2 + 1/(4 xi^2))."""
    if np.isinf(xi):
        return float(g_w)
    return float(np.hypot(0.5 / xi, g_w))


def point_width(g_w, xi):
    """c such that erf(r/c)/r is the pointwise screened potential."""
    if np.isinf(xi):
        return math.sqrt(2.0) * g_w
    if xi == 0.0:
        return np.inf
    return np.sqrt(2.0 * g_w**2 + 1.0 / xi**2)


# name used by the reference (kernels.py:29)
combined_width = point_width


def avg_width(g_w, xi):
    """c such that erf(r/c)/r is the Gaussian-averaged screened potential."""
    if np.isinf(xi):
        return 2.0 * g_w
    if xi == 0.0:
        return np.inf
    return np.sqrt(4.0 * g_w**2 + 1.0 / xi**2)


def erf_over_r(r, c):
    """erf(r/c)/r with the r -> 0 limit 2/(sqrt(pi) c)."""
    r = np.asarray(r, dtype=float)
    if np.isinf(c):
        return np.zeros_like(r)
    if c == 0.0:
        safe = np.where(r > 0, r, 1.0)
        return np.where(r > 0, 1.0 / safe, np.inf)
    tiny = r < ERF_SMALL * c
    rr = np.where(tiny, 1.0, r)
    return np.where(tiny, TWO_OVER_SQRTPI / c, erf(rr / c) / rr)


def d_erf_over_r(r, c):
    """Radial derivative of erf(r/c)/r (Taylor series for r < 0.01 c)."""
    r = np.asarray(r, dtype=float)
    if np.isinf(c):
        return np.zeros_like(r)
    if c == 0.0:
        safe = np.where(r > 0, r, 1.0)
        return np.where(r > 0, -1.0 / safe**2, -np.inf)
    tiny = r < DERF_SMALL * c
    rr = np.where(tiny, c, r)
    x = rr / c
    closed = TWO_OVER_SQRTPI * np.exp(-x * x) / (c * rr) - erf(x) / rr**2
    u = (r / c) ** 2
    taylor = TWO_OVER_SQRTPI / c**2 * (r / c) * (
        -2.0 / 3.0 + u * (2.0 / 5.0 + u * (-1.0 / 7.0 + u / 27.0)))
    return np.where(tiny, taylor, closed)


def near_potential_point(r, g_w, xi, eps=1.0):
    return (erf_over_r(r, math.sqrt(2.0) * g_w)
            - erf_over_r(r, point_width(g_w, xi))) / (FOUR_PI * eps)


def near_gradient_point(r, g_w, xi, eps=1.0):
    return (d_erf_over_r(r, math.sqrt(2.0) * g_w)
            - d_erf_over_r(r, point_width(g_w, xi))) / (FOUR_PI * eps)


def near_potential_avg(r, g_w, xi, eps=1.0):
    return (erf_over_r(r, 2.0 * g_w)
            - erf_over_r(r, avg_width(g_w, xi))) / (FOUR_PI * eps)


def near_gradient_avg(r, g_w, xi, eps=1.0):
    return (d_erf_over_r(r, 2.0 * g_w)
            - d_erf_over_r(r, avg_width(g_w, xi))) / (FOUR_PI * eps)


def self_potential_avg(g_w, xi, eps=1.0, subtract_unsplit=False):
    """Averaged near kernel at r = 0; optionally minus the unsplit
    self-energy q/(4 pi^1.5 eps g_w)."""
    c2 = avg_width(g_w, xi)
    if subtract_unsplit:
        return -TWO_OVER_SQRTPI / c2 / (FOUR_PI * eps)
    return TWO_OVER_SQRTPI * (0.5 / g_w - 1.0 / c2) / (FOUR_PI * eps)


def smoothed_pair_potential(r, g_w, eps=1.0):
    return erf_over_r(r, 2.0 * g_w) / (FOUR_PI * eps)


def far_potential_avg(r, g_w, xi, eps=1.0):
    return erf_over_r(r, 2.0 * split_widths(xi, g_w)) / (FOUR_PI * eps)
