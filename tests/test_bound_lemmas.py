"""CPU checks of the floating-point lemmas the K1 lower bounds rest on; the kernels use them
only to skip work, so a violated lemma would show as a pruned-vs-literal mismatch on the GPU -- these
tests pin the inequalities themselves, with exact rational arithmetic as the reference.

* the RN sum of M copies of t >= 0 (user order, from 0.0) is >= RD(RD(M t) (1 - (M - 1) 2^-53))
  (the equal-deadline kernel's per-n~ bound);
* RD(phi RD(1 / x)) <= RN(phi / x) for phi >= 0, x > 0 (the batch-coupled bound's f_e floor g_p).
"""
import math
import random
from fractions import Fraction

import pytest


def rd(exact: Fraction) -> float:
    """The largest double <= exact (exact >= 0, below the overflow threshold)."""
    r = float(exact)                     # round to nearest
    if Fraction(r) > exact:
        r = math.nextafter(r, -math.inf)
    return r


def rd_mul(a: float, b: float) -> float:
    return rd(Fraction(a) * Fraction(b))


def rd_recip(x: float) -> float:
    return rd(1 / Fraction(x))


def samples(rng, n):
    out = [0.0, 5e-324, 2.2250738585072014e-308, 1.0, 1.0 - 2 ** -53, 1.5, 3.0, 1e300 / 64]
    for _ in range(n):
        e = rng.choice([rng.uniform(-1074, -1020), rng.uniform(-300, 300), rng.uniform(-30, 30)])
        out.append(min(2.0 ** e * rng.uniform(1, 2), 1e306))
    return out


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_rn_sum_of_equal_terms_bound(seed):
    rng = random.Random(seed)
    for t in samples(rng, 400):
        for M in (1, 2, 3, 7, 10, 16, 20, 31, 32):
            s = 0.0
            for _ in range(M):
                s = s + t
            lb = rd_mul(rd_mul(float(M), t), 1.0 - (M - 1) * 2.0 ** -53)
            assert lb <= s, (t, M, lb, s)


def test_rn_sum_bound_is_tight_enough():
    """The bound loses at most about M ulps: it is not vacuous (pruning relies on it being close)."""
    rng = random.Random(7)
    for t in samples(rng, 200):
        if t < 1e-300:
            continue
        for M in (2, 10, 32):
            s = 0.0
            for _ in range(M):
                s = s + t
            lb = rd_mul(rd_mul(float(M), t), 1.0 - (M - 1) * 2.0 ** -53)
            assert s - lb <= 4 * M * math.ulp(s), (t, M)


@pytest.mark.parametrize("seed", [4, 5])
def test_rd_reciprocal_product_below_quotient(seed):
    rng = random.Random(seed)
    xs = samples(rng, 150)
    for phi in samples(rng, 60):
        for x in xs:
            if x == 0.0 or x < 1e-300:
                continue
            q = phi / x
            if math.isinf(q):
                continue
            g = rd_mul(phi, rd_recip(x))
            assert g <= q, (phi, x, g, q)


def test_recip_rd_algorithm_equals_rd():
    """The kernels' recip_rd: q = RN(1/x), stepped to its predecessor when q x - 1 > 0 exactly (the sign of
    the fma residual) -- equal to RD(1/x) (jdob_dev.cuh)."""
    rng = random.Random(11)
    for x in samples(rng, 3000):
        if x == 0.0 or x < 1e-300:
            continue
        q = 1.0 / x
        alg = math.nextafter(q, -math.inf) if Fraction(q) * Fraction(x) - 1 > 0 else q
        assert alg == rd_recip(x), x


def rd_add(a: float, b: float) -> float:
    return rd(Fraction(a) + Fraction(b))


@pytest.mark.parametrize("seed", [8, 9])
def test_rn_sum_any_order_vs_rd_sum_bound(seed):
    """The differing-deadline kernel's bounds: for non-negative terms t_m, the RN sum in any order is
    >= RD(RD-sum of the terms (any order) x (1 - (M - 1) 2^-53)); also with some terms replaced by a
    smaller common value em (RD(k em) + RD-sum of the rest)."""
    rng = random.Random(seed)
    pool = samples(rng, 300)
    for _ in range(400):
        M = rng.choice([1, 2, 5, 10, 17, 32])
        ts = [rng.choice(pool) for _ in range(M)]
        s = 0.0
        for t in ts:
            s = s + t
        c = 1.0 - (M - 1) * 2.0 ** -53
        r = 0.0
        for t in sorted(ts):                  # a different order for the RD sum
            r = rd_add(r, t)
        assert rd_mul(r, c) <= s, (ts,)
        k = rng.randrange(0, M + 1)          # the first k terms bounded below by em = min of them
        em = min(ts[:k]) if k else 0.0
        r2 = 0.0
        for t in ts[k:]:
            r2 = rd_add(r2, t)
        lb = rd_mul(rd_add(rd_mul(float(k), em), r2), c)
        assert lb <= s, (ts, k)
