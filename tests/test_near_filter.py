"""The single-precision level-2 filter of k_near (build_kernels.cu,
MPAP_NEAR_F32; DESIGN.md §7 "Exact culling") must be conservative: it may
keep pairs without an edge, never drop one with c* < r (Near, P:206-212,
reading R7).  This restates the filter's float arithmetic in numpy float32
(IEEE round-to-nearest, the operation order of the kernel, no contraction)
and checks it against the oracle's exact cost on random double-integrator
pairs and on adversarial pairs whose c* sits just below r, including pairs
far from the origin and with near-zero velocity sums.  The kernel's own
decisions are covered by the CSR digests of the GPU tests."""
import numpy as np
import pytest

f32 = np.float32


def _tables(r):
    t = []
    for lvl, nseg in ((0, 1), (1, 4), (2, 16)):
        row = []
        for jj in range(nseg):
            ta = r * jj / nseg
            tb = r * (jj + 1) / nseg
            row.append((f32(ta), f32(tb), f32(1.0 / tb), f32(1.0 / (tb * tb * tb))))
        t.append(row)
    return t


def _round_up_f32(x):
    y = f32(x)
    return y if float(y) >= x else np.nextafter(y, f32(np.inf))


def near_filter_keeps(su, sv, d, ru, r):
    """k_near's level 1 (double) and level 2 (float) for one ordered pair."""
    v02 = 0.0
    for j in range(d):
        v02 += su[d + j] * su[d + j]
    bp = (np.sqrt(v02) * r + r * r / np.sqrt(3.0 * ru)) * (1.0 + 1e-9)
    bv = (r / (2.0 * np.sqrt(ru))) * (1.0 + 1e-9)
    dp2 = dv2 = 0.0
    for j in range(d):
        a = sv[j] - su[j]
        e = sv[d + j] - su[d + j]
        dp2 += a * a
        dv2 += e * e
    if dp2 > bp * bp or dv2 > bv * bv:
        return False
    ss = asum = 0.0
    for j in range(d):
        e = sv[d + j] + su[d + j]
        a = sv[j] - su[j]
        ss += e * e
        asum += a * e
    dp2f, asf, ssf, dv2f = f32(dp2), f32(asum), f32(ss), f32(dv2)
    ruf, rf = f32(ru), _round_up_f32(r)
    ss_ok = ssf > f32(1e-30) or ss == 0.0
    tvf = f32(f32(2.0) * asf) / ssf if ssf > f32(1e-30) else f32(0.0)
    tab = _tables(r)

    def possible(lvl, jj):
        ta, tb, k2, k3 = tab[lvl][jj]
        tq = min(max(tvf, ta), tb)
        t1 = f32(tq * asf)
        t2 = f32(f32(f32(tq * tq) * ssf) * f32(0.25))
        g2 = f32(f32(dp2f - t1) + t2)
        m = f32(f32(dp2f + abs(t1)) + t2)
        g2lo = max(f32(g2 - f32(f32(1e-6) * m)), f32(0.0))
        inner = f32(f32(f32(f32(12.0) * g2lo) * k3) + f32(dv2f * k2))
        L = f32(ta + f32(ruf * inner))
        return (not ss_ok) or f32(L * f32(f32(1.0) - f32(1e-6))) < rf

    if not possible(0, 0):
        return False
    for q in range(4):
        if not possible(1, q):
            continue
        for jj in range(4 * q, 4 * q + 4):
            if possible(2, jj):
                return True
    return False


def _pairs(rng, n, d, lo, hi, vmax):
    p = rng.uniform(lo, hi, size=(n, 2, d))
    v = rng.uniform(-vmax, vmax, size=(n, 2, d))
    return np.concatenate([p, v], axis=2)


@pytest.mark.parametrize("ru", [1.0, 0.05])
def test_f32_filter_keeps_every_edge_random(orc, ru):
    rng = np.random.default_rng(7)
    d, r = 3, 4.5
    st = _pairs(rng, 6000, d, np.array([0.0, 0.0, 0.0]), np.array([3.0, 3.0, 3.0]), 1.0)
    edges = 0
    for su, sv in st:
        cs = orc.cost_di(su, sv, d, ru, r)
        if cs is not None and cs[0] < r:
            edges += 1
            assert near_filter_keeps(su, sv, d, ru, r), (su, sv, cs)
    assert edges > 400


@pytest.mark.parametrize("offset", [0.0, 900.0])
def test_f32_filter_keeps_edges_at_the_boundary(orc, offset):
    """c* just below r: r = c* (1 + 1e-9), so every pair has an edge; far
    from the origin (offset) the float conversions of the positions lose
    the most relative precision of their difference."""
    rng = np.random.default_rng(11)
    d, ru = 3, 1.0
    st = _pairs(rng, 3000, d, np.full(3, offset), np.full(3, offset + 3.0), 1.0)
    # near-cancelling velocity sums (s ~ 0) and near-parallel a, s
    st[:500, 1, d:] = -st[:500, 0, d:] + rng.normal(0, 1e-7, size=(500, d))
    st[500:1000, 1, :d] = st[500:1000, 0, :d] + 0.5 * (st[500:1000, 0, d:] + st[500:1000, 1, d:]) * 1.3
    checked = 0
    for su, sv in st:
        cs = orc.cost_di(su, sv, d, ru, 1e3)
        if cs is None:
            continue
        r = cs[0] * (1.0 + 1e-9)
        if not (cs[1] <= r):
            continue
        again = orc.cost_di(su, sv, d, ru, r)
        if again is None or not again[0] < r:
            continue
        checked += 1
        assert near_filter_keeps(su, sv, d, ru, r), (su, sv, cs, r)
    assert checked > 1000


def test_f32_bound_never_exceeds_the_exact_bound():
    """The margin itself: on every interval, the float bound after its
    margins is at most the exact (rational) lower bound of c on that
    interval, including inputs where |a - s tau / 2|^2 cancels to ~0 (a
    parallel to s with tau* inside the interval) and far-from-origin
    magnitudes.  A margin that is too small fails here."""
    from fractions import Fraction as Fr
    rng = np.random.default_rng(5)
    r, ru = 4.5, 1.0
    tab = _tables(r)
    ruf = f32(ru)
    worst = -np.inf
    for it in range(6000):
        scale = 10.0 ** rng.uniform(-2, 2)
        s = rng.normal(size=3) * rng.uniform(0.01, 2.0)
        tau0 = rng.uniform(0, r)
        a = 0.5 * s * tau0 + (rng.normal(size=3) * scale * 1e-6 if it % 2 else rng.normal(size=3) * scale)
        e = rng.normal(size=3) * rng.uniform(0, 2.0)
        dp2 = float(a @ a)
        asum = float(a @ s)
        ss = float(s @ s)
        dv2 = float(e @ e)
        dp2f, asf, ssf, dv2f = f32(dp2), f32(asum), f32(ss), f32(dv2)
        tvf = f32(f32(2.0) * asf) / ssf
        for lvl, nseg in ((0, 1), (1, 4), (2, 16)):
            for jj in range(nseg):
                ta, tb, k2, k3 = tab[lvl][jj]
                tq = min(max(tvf, ta), tb)
                t1 = f32(tq * asf)
                t2 = f32(f32(f32(tq * tq) * ssf) * f32(0.25))
                g2 = f32(f32(dp2f - t1) + t2)
                m = f32(f32(dp2f + abs(t1)) + t2)
                g2lo = max(f32(g2 - f32(f32(1e-6) * m)), f32(0.0))
                inner = f32(f32(f32(f32(12.0) * g2lo) * k3) + f32(dv2f * k2))
                Lf = f32(f32(ta + f32(ruf * inner)) * f32(f32(1.0) - f32(1e-6)))
                # exact: min over [ta, tb] of the convex quadratic (real interval ends)
                Ta, Tb = Fr(r) * jj / nseg, Fr(r) * (jj + 1) / nseg
                A, S, SS = Fr(dp2), Fr(asum), Fr(ss)
                tv = 2 * S / SS
                tqe = min(max(tv, Ta), Tb)
                ge = max(A - tqe * S + tqe * tqe * SS / 4, Fr(0))
                Le = Ta + Fr(ru) * (12 * ge / (Tb ** 3) + Fr(dv2) / Tb)
                worst = max(worst, float((Fr(float(Lf)) - Le) / Le) if Le > 0 else -1.0)
                assert Fr(float(Lf)) <= Le, (it, lvl, jj, float(Lf), float(Le))
    assert worst < 0.0
