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
