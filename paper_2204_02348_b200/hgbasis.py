"""Host-side modal-basis bookkeeping (holopipe/hgbasis.py).

The HG profiles themselves are generated and int16-quantised by the C ABI
(hpg_plan_create, fp64); this module keeps the small index helpers and the
HG->LG transform matrix the engine applies after the overlap.
"""

import math

import numpy as np

from . import constants as C
from .errors import ErrorCode, HoloError


def mode_indices(group_count):
    """(m, n) pairs, group-major, m descending (hgbasis.py:17-27)."""
    return [(g - n, n) for g in range(group_count) for n in range(g + 1)]


def mode_count(group_count):
    return group_count * (group_count + 1) // 2


def mode_group_of_index(idx):
    return int((math.isqrt(8 * idx + 1) - 1) // 2)


def _binom_poly(n, m, k):
    # coefficient of t^k in (1-t)^n (1+t)^m
    return sum((-1) ** j * math.comb(n, j) * math.comb(m, k - j)
               for j in range(max(0, k - m), min(n, k) + 1))


def hg_to_lg_transform(group_count):
    """Unitary block-diagonal HG->LG matrix (hgbasis.py:126-175)."""
    if group_count > C.LG_GROUP_MAX:
        raise HoloError(ErrorCode.INVALIDARGUMENT, f"LG basis supports at most {C.LG_GROUP_MAX} groups")
    total = mode_count(group_count)
    T = np.zeros((total, total), np.complex128)
    base = 0
    for N in range(group_count):
        fac = [math.factorial(i) for i in range(N + 1)]
        for row in range(N + 1):
            n, m = row, N - row
            sgn = -1.0 if min(n, m) % 2 else 1.0
            den = fac[n] * fac[m] * (2 ** N)
            for k in range(N + 1):
                T[base + row, base + k] = sgn * (1j ** k) * math.sqrt(fac[N - k] * fac[k] / den) \
                    * _binom_poly(n, m, k)
        base += N + 1
    return T
