"""H2O comparison baseline (harness.cpp:83-150) on the B200 vs the oracle.

The device kernel (csrc/h2o.cu) keeps the reference's arithmetic order (sequential fp32 dot,
scale * dot, max, correctly rounded exp, sequential fp32 sum, IEEE division, double score
accumulation), so the kept set after every step must equal the C restatement's (itself pinned
to the unmodified reference by tests/test_oracle_vs_reference.py) exactly.
"""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mkv():
    import paper_2411_18077_b200 as m
    return m


def _dev(*arrs):
    return [torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda() for a in arrs]


def _run(mkv, pk, sc, qs, ks, hh, rw, scale):
    t = mkv.h2o_dynamic_baseline(*_dev(pk, sc, qs, ks), hh, rw, scale)
    return t.kept_per_step


def test_h2o_random_configs_match_oracle(mkv):
    P = oracle.port()
    rng = np.random.default_rng(5)
    for _ in range(30):
        l = int(rng.integers(1, 400))
        d = int(rng.choice([2, 8, 16, 64, 128]))
        steps = int(rng.integers(0, 64))
        hh, rw = int(rng.integers(0, 256)), int(rng.integers(0, 64))
        hh = max(hh, 1 - rw)
        pk = rng.standard_normal((l, d)).astype(np.float32)
        sc = rng.random(l).astype(np.float32)
        qs = rng.standard_normal((steps, d)).astype(np.float32)
        ks = rng.standard_normal((steps, d)).astype(np.float32)
        scale = float(1 / np.sqrt(d))
        assert _run(mkv, pk, sc, qs, ks, hh, rw, scale) == P.h2o_dynamic_baseline(pk, sc, qs, ks, hh, rw, scale)


def test_h2o_long_prompt_against_reference(mkv):
    """A 4K prompt evicted to a 20% budget, 128 decode steps (acceptance-criterion scale x 32)."""
    P = oracle.port()
    rng = np.random.default_rng(9)
    l, d, steps = 4096, 128, 128
    pk = rng.standard_normal((l, d)).astype(np.float32)
    sc = (rng.pareto(1.5, l) + 1).astype(np.float32)  # heavy-tailed A_cumul-like scores
    qs = rng.standard_normal((steps, d)).astype(np.float32)
    ks = rng.standard_normal((steps, d)).astype(np.float32)
    got = _run(mkv, pk, sc, qs, ks, 409, 409, float(1 / np.sqrt(d)))
    assert got == P.h2o_dynamic_baseline(pk, sc, qs, ks, 409, 409, float(1 / np.sqrt(d)))
    assert all(len(k) == 818 for k in got)


def test_h2o_reference_cases(mkv):
    # test_harness.cpp:95-105: an oversized budget never evicts
    rng = np.random.default_rng(1)
    pk = rng.standard_normal((16, 8)).astype(np.float32)
    sc = rng.random(16).astype(np.float32)
    qs = rng.standard_normal((10, 8)).astype(np.float32)
    ks = rng.standard_normal((10, 8)).astype(np.float32)
    t = _run(mkv, pk, sc, qs, ks, 100, 0, float(1 / np.sqrt(8)))
    assert [len(k) for k in t] == [16 + s for s in range(11)]
    # test_harness.cpp:107-125: two slots keep the dominant token plus the newest
    l, d, steps = 4, 2, 6
    pk = np.zeros((l, d), np.float32)
    pk[0, 0] = 1.0
    pk[1:, 0] = -1.0
    sc = np.array([4.0, 0.3, 0.2, 0.1], np.float32)
    qs = np.tile(np.array([10.0, 0.0], np.float32), (steps, 1))
    ks = np.tile(np.array([-1.0, 0.0], np.float32), (steps, 1))
    t = _run(mkv, pk, sc, qs, ks, 1, 1, 1.0)
    for step in range(1, len(t)):
        assert len(t[step]) == 2 and 0 in t[step] and (l + step - 1) in t[step]
    # zero budget is rejected like the reference (harness.cpp:117-119)
    with pytest.raises(mkv.InvalidArgument):
        _run(mkv, pk, sc, qs, ks, 0, 0, 1.0)


def test_persistence_on_device_trace(mkv):
    """test_harness.cpp:144-177 on a device trace: 1 at full budget, 0 when disjoint,
    bounded and non-increasing fractions, empty heavy-hitter set rejected."""
    rng = np.random.default_rng(11)
    l, d, steps = 128, 16, 48
    pk = rng.standard_normal((l, d)).astype(np.float32)
    sc = (rng.pareto(1.2, l) + 1).astype(np.float32)
    qs = rng.standard_normal((steps, d)).astype(np.float32)
    ks = rng.standard_normal((steps, d)).astype(np.float32)
    full = mkv.h2o_dynamic_baseline(*_dev(pk, sc, qs, ks), l + steps, 0, float(1 / np.sqrt(d)))
    sel_hh = [int(x) for x in oracle.port().select_token_counts(sc, 48, 16)[0][:48]]
    assert all(f == 1.0 for f in mkv.persistence_analysis(full, sel_hh).fractions)
    assert all(f == 0.0 for f in mkv.persistence_analysis(full, [9999]).fractions)
    with pytest.raises(RuntimeError):
        mkv.persistence_analysis(full, [])
    t = mkv.h2o_dynamic_baseline(*_dev(pk, sc, qs, ks), 48, 16, float(1 / np.sqrt(d)))
    rep = mkv.persistence_analysis(t, sel_hh)
    prev = 1.0
    for f in rep.fractions:
        assert 0.0 <= f <= 1.0 and f <= prev + 1e-7
        prev = f
    assert rep.final_fraction == rep.fractions[-1]
