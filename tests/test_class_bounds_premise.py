"""CPU: the premise of the degree-class bounds (solver.cu k_class_bounds,
DESIGN.md section 5), checked on the oracle's restatement of the reference's
H2 priority (priorities.cpp:43-67, oracle/tcmis_oracle.c
orc_h2_priority_value):

  * for a fixed degree k, p(k, eps) is non-decreasing in eps over
    [0, 1 - 2^-53] (hash_to_unit's range), so every vertex of degree k has
    h2(k, 0) <= p <= h2(k, eps_max);
  * both ends are non-increasing in k.

With these, "h2(j, 0) > h2(k, eps_max)" proves that every vertex of degree j
out-ranks every vertex of degree k -- the hi bound -- and "h2(j, eps_max) <
h2(k, 0)" the reverse -- the lo bound.  The checks sweep the floor / clamp
corners (tiny averages, the 1/1024 denominator floor, scale_bits 8..30) and
eps values next to 0, 1 and the binary fractions where the subtraction
rounds."""
import ctypes as C
import math

import numpy as np
import pytest

import oracle as O

EPS_MAX = (2 ** 53 - 1) * 2.0 ** -53


def h2(avg, deg, eps, sb):
    return O.lib().orc_h2_priority_value(C.c_double(avg), deg, C.c_double(eps), sb)


def _eps_samples(rng):
    base = [0.0, 2.0 ** -53, 2.0 ** -30, 0.25, 0.5 - 2 ** -40, 0.5, 0.5 + 2 ** -40, 0.75,
            1 - 2 ** -30, EPS_MAX - 2 ** -52, EPS_MAX]
    return sorted(set(base + [float(x) for x in (rng.integers(0, 2 ** 53, 40) * 2.0 ** -53)]))


@pytest.mark.parametrize("sb", [8, 11, 20, 30])
@pytest.mark.parametrize("avg", [0.001, 0.75, 2.0, 3.0, 16.0, 31.347, 1000.5])
def test_h2_monotone_in_eps_and_degree(sb, avg):
    rng = np.random.default_rng(sb * 1000 + int(avg * 10))
    eps = _eps_samples(rng)
    degs = sorted(set([1, 2, 3, 4, 5, 7, 8, 15, 16, 31, 32, 100, 1000, 4095, 4096, 65535,
                       1 << 20, (1 << 31) - 1] + rng.integers(1, 5000, 30).tolist()))
    lo_prev = hi_prev = None
    for k in degs:
        vals = [h2(avg, k, e, sb) for e in eps]
        assert vals == sorted(vals), (k, "non-decreasing in eps")
        lo, hi = h2(avg, k, 0.0, sb), h2(avg, k, EPS_MAX, sb)
        assert lo == vals[0] and hi == vals[-1]
        if lo_prev is not None:
            assert lo <= lo_prev and hi <= hi_prev, (k, "ends non-increasing in degree")
        lo_prev, hi_prev = lo, hi


def test_bounds_separate_degrees_on_a_real_graph():
    """On an R-MAT graph's actual priorities: whenever the bounds say degree j
    out-ranks degree k, every vertex pair does (and p ties never cross)."""
    g = O.gen("rmat", 12, 16, 3)
    deg = np.diff(g.off).astype(np.int64)
    avg = 2.0 * (int(g.off[-1]) // 2) / g.n
    for sb in (8, 20):
        p = O.priorities(g, "h2", 5, sb).astype(np.int64)
        ks = np.unique(deg[deg > 0])
        lo = {int(k): h2(avg, int(k), 0.0, sb) for k in ks}
        hi = {int(k): h2(avg, int(k), EPS_MAX, sb) for k in ks}
        pmin = {int(k): int(p[deg == k].min()) for k in ks}
        pmax = {int(k): int(p[deg == k].max()) for k in ks}
        for k in ks:
            k = int(k)
            assert lo[k] <= pmin[k] and pmax[k] <= hi[k], k
        for j in ks:
            for k in ks:
                j, k = int(j), int(k)
                if lo[j] > hi[k]:
                    assert pmin[j] > pmax[k], (j, k)
                if hi[j] < lo[k]:
                    assert pmax[j] < pmin[k], (j, k)
        assert math.isfinite(avg)
