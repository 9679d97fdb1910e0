"""The K3 quantizer's rounding thresholds (mkv_common.cuh quantize_group16) restated in
numpy and checked against the reference's per-value arithmetic (quantizer.cpp:40-50:
code = clamp(round_half_away(fl(fl(v - lo) / scale)), 0, 3)) on adversarial inputs:
values on, one ulp below and one ulp above every rounding boundary, over scales from
subnormal to huge.  CPU only."""
import numpy as np

F = np.float32


def thresholds(sc):
    T = []
    for k in range(3):
        c = F(k + 0.5)
        m = 0.5 * (float(np.nextafter(c, F(0))) + float(c))  # exact in double
        prod = m * float(sc)                                  # exact: 25 x 24 bits
        x = F(prod)                                           # round to nearest
        if float(x) < prod:
            x = np.nextafter(x, F(np.inf))
        T.append(x)
    return T


def ref_code(dv, sc):
    q = F(dv / sc)  # IEEE float32 division (numpy rounds the float32 quotient correctly)
    r = np.floor(q)  # std::round: half away from zero (q >= 0 here; q - floor(q) is exact)
    if q - r >= F(0.5):
        r += 1
    return int(min(max(r, 0.0), 3.0))


def test_thresholds_match_division_at_every_boundary():
    rng = np.random.default_rng(0)
    scales = np.concatenate([F(10.0) ** rng.uniform(-40, 37, 400).astype(F), np.array([1e-45, 1.4e-45, 3e-39, 1.0,
                             0.1, 1 / 3, 3.4e38 / 3], F)]).astype(F)
    checked = 0
    for sc in scales:
        if not (np.isfinite(sc) and sc > 0):
            continue
        T = thresholds(sc)
        cands = []
        for c in (0.5, 1.5, 2.5):
            p = F(F(c) * sc)
            cands += [p, np.nextafter(p, F(0)), np.nextafter(p, F(np.inf)),
                      np.nextafter(np.nextafter(p, F(0)), F(0)), np.nextafter(np.nextafter(p, F(np.inf)), F(np.inf))]
        cands += [F(0), F(3) * sc, np.nextafter(F(3) * sc, F(0)), *rng.uniform(0, 3 * float(sc), 20).astype(F)]
        for dv in cands:
            if not np.isfinite(dv) or dv < 0:
                continue
            got = int(dv >= T[0]) + int(dv >= T[1]) + int(dv >= T[2])
            assert got == ref_code(dv, sc), (sc, dv, T)
            checked += 1
    assert checked > 5000


def thresholds_fp32(sc):
    """The device's FP64-free form (mkv_common.cuh group_thresholds, scales in [2^-100, 2^100]):
    ds = sc * d_k, y = fma(c_k, sc, -ds), r = fma(-c_k, sc, y), T_k = y if r >= -ds else nextup(y).
    Both fma's are evaluated exactly in float64 here (c_k * sc needs <= 27 bits and ds sits
    <= 26 bits below it, so every pre-rounding value fits in 53 bits), then rounded once."""
    T = []
    for c, d in ((0.5, 2.0 ** -26), (1.5, 2.0 ** -24), (2.5, 2.0 ** -23)):
        ds = F(sc * F(d))
        y = F(c * float(sc) - float(ds))
        r = F(float(y) - c * float(sc))
        T.append(y if r >= -ds else np.nextafter(y, F(np.inf)))
    return T


def test_fp32_thresholds_equal_double_thresholds():
    """Sampled restatement of tools/threshold_fp32_check.c (which covers every fp32 scale in
    [2^-100, 2^100] exhaustively): binade edges, their neighbours and random scales."""
    rng = np.random.default_rng(5)
    scales = [F(2.0 ** e) for e in range(-100, 101)]
    scales += [np.nextafter(s, F(0)) for s in scales] + [np.nextafter(s, F(np.inf)) for s in scales]
    scales += list((rng.random(3000) * 2.0 ** rng.integers(-100, 100, 3000)).astype(F))
    scales += [F(1) / F(3), F(65504) / F(3), F(2.0 ** -24) / F(3)]
    n = 0
    for sc in scales:
        if not (F(2.0 ** -100) <= sc <= F(2.0 ** 100)):
            continue
        a, b = thresholds(sc), thresholds_fp32(sc)
        for x, y in zip(a, b):
            assert np.float32(x).view(np.uint32) == np.float32(y).view(np.uint32), (sc, a, b)
        n += 1
    assert n > 3000
