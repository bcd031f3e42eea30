"""The kernels evaluate Eq. 14 in a nested clamp form; this
CPU test checks that form, written out in numpy, against the oracle's literal
truncated-power Eq. 14 -- in FP64 (algebraic identity) and in FP32 (the
stability claim: error <= a few 1e-7 of the peak even as C -> 0, where the
literal form in FP32 fails)."""
import numpy as np

import oracle as O


def clamp_form(x, A, B, C, dtype):
    """M(x) = [ (clamp(z11,0,B) - clamp(z21,0,B)) + C/2 (t11^2 - t12^2 - t21^2 + t22^2) ] / (A B)
    with z11 = x + (A - C)/2 + B/2, z21 = z11 - A, t = sat(z/C + 1), t12/t22 via w1 = 1 - B/C."""
    x, A, B, C = (np.asarray(v, dtype=dtype) for v in (x, A, B, C))
    one = dtype(1)
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        invC = one / C
        z11 = x + (A - C) * dtype(0.5) + B * dtype(0.5)
        z21 = z11 - A
        w1 = one - B * invC
        sat = lambda u: np.nan_to_num(np.clip(u, 0, 1), nan=0.0).astype(dtype)
        t11, t12 = sat(z11 * invC + one), sat(z11 * invC + w1)
        t21, t22 = sat(z21 * invC + one), sat(z21 * invC + w1)
        T = (t11 * t11 - t12 * t12) - (t21 * t21 - t22 * t22)
        M2 = np.minimum(np.maximum(z11, 0), B) - np.minimum(np.maximum(z21, 0), B)
        num = M2 + C * dtype(0.5) * T
        return (num / (A * B)).astype(np.float64)


def literal32(x, A, B, C):
    """Eq. 14 as 8 truncated powers, evaluated in FP32 (what NOT to do)."""
    x, A, B, C = (np.float32(v) for v in (x, A, B, C))
    s = (A + B + C) * np.float32(0.5)
    tot = np.float32(0)
    for ma in (0, 1):
        for mb in (0, 1):
            for mc in (0, 1):
                u = x + s - ma * A - mb * B - mc * C
                sgn = -1 if (ma + mb + mc) % 2 else 1
                tot += np.float32(sgn) * np.float32(max(u, 0)) ** 2
    return float(tot / (np.float32(2) * A * B * C))


def _cases(rng, n, cmin):
    for _ in range(n):
        A = rng.uniform(0.7, 1.0)
        C = A * 10 ** rng.uniform(np.log10(cmin), 0)
        C = min(C, A)
        B = rng.uniform(0.05, 2.0)
        x = rng.uniform(-1.0, 1.0) * (A + B + C) / 2
        yield x, A, B, C


def test_clamp_form_fp64_equals_eq14():
    rng = np.random.default_rng(0)
    for x, A, B, C in _cases(rng, 3000, 1e-3):
        ref = O.box_spline([A, B, C], x)
        assert abs(clamp_form(x, A, B, C, np.float64) - ref) <= 1e-12 * (1 + ref)


def test_clamp_form_degenerate_c():
    # C == 0 (an axis-aligned ray): the delta direction is eliminated
    rng = np.random.default_rng(1)
    for _ in range(500):
        A, B = rng.uniform(0.7, 1.0), rng.uniform(0.05, 2.0)
        x = rng.uniform(-1, 1) * (A + B) / 2
        ref = O.box_spline([A, B], x)
        for dt in (np.float64, np.float32):
            got = clamp_form(x, A, B, 0.0, dt)
            assert abs(got - ref) <= (1e-12 if dt is np.float64 else 6e-7) * max(1.0, 1 / A)


def test_clamp_form_fp32_stable_where_literal_fails():
    # B = tau' ranges over [0.05, 2] A here; the configs have tau'/A in ~[0.3, 1.6]
    rng = np.random.default_rng(2)
    worst_nested, worst_real, worst_literal = 0.0, 0.0, 0.0
    for x, A, B, C in _cases(rng, 4000, 1e-8):
        ref = O.box_spline([A, B, C], x) if C >= 1e-6 * A else O.box_spline([A, B], x)
        peak = 1.0 / A
        err = abs(clamp_form(x, A, B, C, np.float32) - ref) / peak
        worst_nested = max(worst_nested, err)
        if B >= 0.3:
            worst_real = max(worst_real, err)
        worst_literal = max(worst_literal, abs(literal32(x, A, B, C) - ref) / peak)
    assert worst_real <= 5e-7
    assert worst_nested <= 1.2e-6
    assert worst_literal > 1e-2  # the reason the kernels do not use the literal form


def test_outside_support_residue_is_rounding_level():
    # the kernels do not mask |x| >= sigma: the residue there must be O(eps)
    rng = np.random.default_rng(3)
    for _ in range(2000):
        A, B = rng.uniform(0.7, 1.0), rng.uniform(0.05, 2.0)
        C = rng.uniform(0, A)
        s = (A + B + C) / 2
        x = np.sign(rng.uniform(-1, 1)) * rng.uniform(s, s + 3 * A)
        assert abs(clamp_form(x, A, B, C, np.float32)) <= 4e-7 * (s + 3 * A) / (A * B)


def precise_form(x, A, B, Cz):
    """The kernels' precise mode (cbp_common.cuh cnsf_prec) in
    numpy: s' = x and A in FP64; b = max(tau', C), c = min(tau', C) (the
    smallest width innermost); the four knot arguments formed in FP64 and
    rounded once to FP32; everything else FP32.  Returns M."""
    f32 = np.float32
    B, Cz = f32(B), f32(Cz)
    b, c = max(B, Cz), min(B, Cz)
    D = float(x) + 0.5 * (float(A) + float(f32(b - c)))
    k = [f32(D), f32(D - float(b)), f32(D - A), f32((D - A) - float(b))]
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        ic = f32(1) / c if c > 0 else f32(np.inf)
        t = [f32(0) if np.isnan(u) else f32(min(max(u, f32(0)), f32(1)))
             for u in (f32(kk * ic + f32(1)) for kk in k)]
    T = f32(f32(f32(t[0] * t[0]) - f32(t[1] * t[1])) - f32(f32(t[2] * t[2]) - f32(t[3] * t[3])))
    trap = max(f32(0), min(k[0], min(f32(A), b), -k[3]))
    num = f32(trap + f32(f32(0.5) * c) * T)
    return float(num / b) / A


def _near_knot_cases(rng, n, brel):
    """x within a ramp width of one of the 8 knots +-A/2 +-B/2 +-C/2 (where a
    position error matters), C from 0 to A."""
    for _ in range(n):
        A = rng.uniform(0.7, 1.0)
        C = A * rng.choice([0.0, 1e-3, 1e-2, 0.1, 0.5, 1.0]) * rng.uniform(0, 1)
        B = A * brel * rng.uniform(0.5, 1.0)
        knots = [sa * A / 2 + sb * B / 2 + sc * C / 2 for sa in (-1, 1) for sb in (-1, 1) for sc in (-1, 1)]
        x = rng.choice(knots) + rng.uniform(-1, 1) * 0.5 * max(B, C)
        yield x, A, B, C


def test_precise_form_holds_for_narrow_bins():
    # <= 2e-7 of the peak from tau'/A = 3 down to 1e-4 (cbp_validate's floor)
    rng = np.random.default_rng(11)
    for brel in (3.0, 0.3, 1e-2, 1e-3, 1e-4):
        worst = 0.0
        for x, A, B, C in _near_knot_cases(rng, 1500, brel):
            ref = O.box_spline([A, B, C], x) if C >= 1e-6 * A else O.box_spline([A, B], x)
            worst = max(worst, abs(precise_form(x, A, B, C) - ref) * A)
        assert worst <= 2.5e-7, (brel, worst)


def test_fp32_position_limits_the_standard_form():
    # the reason for the precise mode: the standard form fed an FP32 s' (one
    # rounding, the best an FP32 position can do) errs ~1e-7 A / tau' near knots
    rng = np.random.default_rng(12)
    worst = 0.0
    for x, A, B, C in _near_knot_cases(rng, 1500, 1e-2):
        ref = O.box_spline([A, B, C], x) if C >= 1e-6 * A else O.box_spline([A, B], x)
        worst = max(worst, abs(clamp_form(np.float32(x), A, B, C, np.float32) - ref) * A)
    assert worst > 5e-6
