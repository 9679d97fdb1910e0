"""K4 fused 2-bit decode attention on the B200 vs the oracle.

Oracle (GQA composition): per unit one decode_append
(cache_engine.cpp:79-90), then for each q-head decode_attention over
[dequant(stored) ; residual] -- bit-identical to decode_step for G = 1 --
with the stored (scale, zero) rounded to fp16 as the device stores them.
Tolerance (stated in BASELINE/SURVEY 8(d)): max |t_O - oracle| <= 5e-3.
"""
import numpy as np
import pytest
import torch

import oracle
from tests.gpu_util import SEED, f32, max_abs, synth_np

pytestmark = pytest.mark.gpu
TOL = 5e-3


@pytest.fixture(scope="module")
def mkv():
    import paper_2411_18077_b200 as m
    return m


def run_decode(mkv, n_units, G, L, hh, rw, steps, n_r=128, seed=SEED, check_every=1, hh_per_unit=None):
    d = 128
    scale = 1.0 / np.sqrt(d)
    k = np.stack([synth_np(seed, oracle.stream_id(oracle.KIND_K, u), (L, d)) for u in range(n_units)])
    v = np.stack([synth_np(seed, oracle.stream_id(oracle.KIND_V, u), (L, d)) for u in range(n_units)])
    rng = np.random.default_rng(seed + L)
    a = rng.random((n_units, L)).astype(np.float32)
    hh_u = hh_per_unit or [hh] * n_units
    caps = [min(h + rw, L) for h in hh_u]
    cache = mkv.KVCache(n_units, caps, max_decode_tokens=steps + n_r, n_r=n_r)
    cache.prefill(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), torch.from_numpy(a).cuda(), hh_u, rw)
    P = oracle.port()
    ocs = []
    for u in range(n_units):
        oc = P.cache(d=d, n_r=n_r)
        oc.prefill(f32(k[u]), f32(v[u]), a[u], hh_u[u], rw)
        ocs.append(oc)
    worst = 0.0
    for s in range(steps):
        q = np.stack([synth_np(seed, oracle.stream_id(oracle.KIND_QDEC, u, s + 1), (G, d)) for u in range(n_units)])
        tk = np.stack([synth_np(seed, oracle.stream_id(oracle.KIND_KDEC, u, s + 1), (d,)) for u in range(n_units)])
        tv = np.stack([synth_np(seed, oracle.stream_id(oracle.KIND_VDEC, u, s + 1), (d,)) for u in range(n_units)])
        out = cache.decode_step(torch.from_numpy(q).cuda(), torch.from_numpy(tk).cuda(),
                                torch.from_numpy(tv).cuda(), scale)
        out = out.float().cpu().numpy()
        for u in range(n_units):
            ocs[u].append(f32(tk[u]), f32(tv[u]))
            if s % check_every == 0 or s == steps - 1:
                for h in range(G):
                    exp = ocs[u].attend(f32(q[u, h]), scale, param_fp16=True)
                    worst = max(worst, max_abs(out[u, h], exp))
    cache.check()
    return worst


@pytest.mark.parametrize("G", [1, 4, 8])
def test_decode_gqa_small(mkv, G):
    assert run_decode(mkv, n_units=3, G=G, L=400, hh=40, rw=40, steps=20) <= TOL


def test_decode_through_flush(mkv):
    # 818 kept (config-1 budget at L=4096 scaled down: partial last prefill page) and a flush at step 128
    worst = run_decode(mkv, n_units=2, G=4, L=1000, hh=91, rw=100, steps=140, check_every=7)
    assert worst <= TOL


def test_decode_partial_pages_and_tiny_units(mkv):
    # units with fewer than 16 kept tokens (one partial page) and ragged pyramid budgets
    worst = run_decode(mkv, n_units=5, G=4, L=300, hh=0, rw=3, steps=10, hh_per_unit=[0, 5, 13, 60, 200])
    assert worst <= TOL


def test_decode_many_units_split(mkv):
    # enough pages that units are split across several warps (split-K merge path)
    worst = run_decode(mkv, n_units=16, G=4, L=6000, hh=1500, rw=600, steps=3)
    assert worst <= TOL


def test_decode_more_units_than_sms(mkv):
    # more units per call than SMs: the default finish step is the split form (persistent
    # residual kernel + merge kernel on per-unit arrival counters), through a flush (n_r = 16)
    worst = run_decode(mkv, n_units=300, G=4, L=700, hh=160, rw=64, steps=20, n_r=16, check_every=6)
    assert worst <= TOL


def test_decode_small_n_r(mkv):
    worst = run_decode(mkv, n_units=2, G=2, L=200, hh=20, rw=20, steps=70, n_r=32, check_every=5)
    assert worst <= TOL


def test_decode_residual_only_unit(mkv):
    """A unit whose cache is only residual rows (no pages) is finished by the residual kernel."""
    d = 128
    cache = mkv.KVCache(1, 16, max_decode_tokens=64)
    P = oracle.port()
    oc = P.cache()
    rng = np.random.default_rng(3)
    # first append without attention, then decode steps (decode_step needs a non-empty cache)
    tk = rng.standard_normal((1, d)).astype(np.float16)
    tv = rng.standard_normal((1, d)).astype(np.float16)
    cache.append(torch.from_numpy(tk).cuda(), torch.from_numpy(tv).cuda())
    oc.append(f32(tk[0]), f32(tv[0]))
    for s in range(5):
        q = rng.standard_normal((1, 1, d)).astype(np.float16)
        tk = rng.standard_normal((1, d)).astype(np.float16)
        tv = rng.standard_normal((1, d)).astype(np.float16)
        out = cache.decode_step(torch.from_numpy(q).cuda(), torch.from_numpy(tk).cuda(),
                                torch.from_numpy(tv).cuda(), 0.1).float().cpu().numpy()
        exp = oc.decode_step(f32(q[0, 0]), f32(tk[0]), f32(tv[0]), 0.1, param_fp16=True)
        assert max_abs(out[0, 0], exp) <= TOL


def test_decode_residual_tiles_split_across_warps(mkv):
    # tiny prefill blocks and long residuals: one unit's fp16 residual tiles are spread over
    # several warps (residual partials + the arrival-counter merge), appends land in every tile
    worst = run_decode(mkv, n_units=40, G=4, L=64, hh=8, rw=8, steps=100, check_every=9)
    assert worst <= TOL


def test_decode_attend_only_is_idempotent(mkv):
    """k_new = None attends without appending: repeated calls give identical outputs."""
    d, n, G = 128, 6, 4
    rng = np.random.default_rng(5)
    L = 500
    k = torch.from_numpy(rng.standard_normal((n, L, d)).astype(np.float16)).cuda()
    v = torch.from_numpy(rng.standard_normal((n, L, d)).astype(np.float16)).cuda()
    a = torch.from_numpy(rng.random((n, L)).astype(np.float32)).cuda()
    cache = mkv.KVCache(n, 200, max_decode_tokens=64)
    cache.prefill(k, v, a, 100, 100)
    for s in range(20):
        tk = torch.from_numpy(rng.standard_normal((n, d)).astype(np.float16)).cuda()
        cache.append(tk, tk)
    q = torch.from_numpy(rng.standard_normal((n, G, d)).astype(np.float16)).cuda()
    o1 = cache.decode_step(q, None, None, 0.09).clone()
    o2 = cache.decode_step(q, None, None, 0.09)
    assert torch.equal(o1, o2)
    assert [cache.unit_info(u)["tokens_residual"] for u in range(n)] == [20] * n
    rk, rv = cache.export_residual(0)
    assert rk.shape == (20, d)


def test_append_only_cache_blocks_export_bit_exact(mkv):
    """A cache that never had a prefill: every quantized block is an n_r flush block
    (1000 appends -> 7 blocks + 104 residual rows, test_cache_engine.cpp:116-128), and
    the export matches the oracle's QuantizedTensor stream bit for bit."""
    d = 128
    rng = np.random.default_rng(21)
    cache = mkv.KVCache(1, 0, max_decode_tokens=1100, keep_fp32_params=True)
    oc = oracle.port().cache()
    for _ in range(1000):
        t = rng.standard_normal((1, d)).astype(np.float16)
        u = rng.standard_normal((1, d)).astype(np.float16)
        cache.append(torch.from_numpy(t).cuda(), torch.from_numpy(u).cuda())
        oc.append(f32(t[0]), f32(u[0]))
    cache.check()
    info = cache.unit_info(0)
    assert info["tokens_quantized"] == 7 * 128 and info["tokens_residual"] == 104 and info["n_blocks"] == 7
    for which in (0, 1):
        w, p, br = cache.export_reference(0, which)
        ew, ep, ebr = oc.export(which)
        assert np.array_equal(w, ew) and np.array_equal(p.reshape(-1), ep.reshape(-1)) and list(br) == list(ebr)


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_decode_randomized_configs(mkv, seed):
    """Randomized parity sweep: unit count, GQA group, n_r, per-unit budgets and step count
    drawn at random (partial pages, flushes, residual-only stretches), every output checked."""
    rng = np.random.default_rng(seed)
    n_units = int(rng.integers(1, 24))
    G = int(rng.choice([1, 2, 4, 8]))
    n_r = int(rng.choice([16, 32, 64, 128]))
    L = int(rng.integers(20, 900))
    rw = int(rng.integers(0, L // 4 + 1))
    hh = [int(rng.integers(0 if rw else 1, L // 3 + 2)) for _ in range(n_units)]
    steps = int(rng.integers(1, 2 * n_r + 5))
    worst = run_decode(mkv, n_units=n_units, G=G, L=L, hh=0, rw=rw, steps=steps, n_r=n_r,
                       check_every=max(1, steps // 12), hh_per_unit=hh, seed=seed)
    assert worst <= TOL, (n_units, G, n_r, L, rw, steps, worst)


def padded(x):
    """x [L, n, ...] as a view whose layers are NOT back to back (layer stride n + 1 rows): the
    per-layer form of mkv_decode_step_layers, which does not coalesce such layers."""
    big = torch.empty((x.shape[0], x.shape[1] + 1) + tuple(x.shape[2:]), dtype=x.dtype, device=x.device)
    big[:, :x.shape[1]] = x
    return big[:, :x.shape[1]]


def layers_forms(caches, q, tk, tv, scale, n):
    """One step through the three forms of a multi-layer decode step, on caches[0..3]:
      0  mkv_decode_step_layers, layers not back to back -> per-layer page/finish passes with the
         cross-layer overlap (bit-identical to 1);
      1  one mkv_decode_step per layer;
      2  mkv_decode_step_layers on one [L, n] array -> coalesced into a single pass over every
         layer's units (bit-identical to 3; MKV_LAYERS_SPLIT=1 turns coalescing off -> to 1);
      3  one mkv_decode_step over all L * n units."""
    import os
    layers = q.shape[0]
    lay = caches[0].decode_step_layers(padded(q), padded(tk), padded(tv), scale, out=torch.empty_like(q))
    per = torch.stack([caches[1].decode_step(q[l], tk[l], tv[l], scale, unit_begin=l * n) for l in range(layers)])
    co = caches[2].decode_step_layers(q, tk, tv, scale)
    flat = caches[3].decode_step(q.reshape(layers * n, *q.shape[2:]), tk.reshape(layers * n, -1),
                                 tv.reshape(layers * n, -1), scale).view_as(q)
    assert torch.equal(lay, per), f"per-layer form: max diff {(lay.float() - per.float()).abs().max()}"
    exp = per if os.environ.get("MKV_LAYERS_SPLIT") else flat
    assert torch.equal(co, exp), f"coalesced form: max diff {(co.float() - exp.float()).abs().max()}"
    # a different split-K partition of the same units: equal up to fp32 merge rounding
    assert (co.float() - per.float()).abs().max().item() <= 2e-3


def test_decode_step_layers_matches_per_layer_calls(mkv):
    """mkv_decode_step_layers in both of its forms (layers_forms): per-layer passes that overlap
    layer l's finish kernel with layer l+1's page pass (q of later layers read before
    griddepcontrol.wait, partial buffers shared by all layers) are bit-identical to one
    mkv_decode_step per layer; back-to-back layers are one pass, bit-identical to one
    mkv_decode_step over all their units -- through a flush and with very uneven layer sizes
    (partials of consecutive layers land in the same slots)."""
    d, n, G, L, layers, n_r = 128, 12, 4, 2000, 6, 32
    rng = np.random.default_rng(21)
    budgets = [1500, 40, 900, 16, 1200, 300]  # hh per layer: long, tiny, long, ...
    caps = [budgets[l] + 64 for l in range(layers) for _ in range(n)]
    k = torch.from_numpy(rng.standard_normal((layers * n, L, d)).astype(np.float16)).cuda()
    v = torch.from_numpy(rng.standard_normal((layers * n, L, d)).astype(np.float16)).cuda()
    a = torch.from_numpy(rng.random((layers * n, L)).astype(np.float32)).cuda()
    caches = []
    for _ in range(4):
        c = mkv.KVCache(layers * n, caps, max_decode_tokens=80, n_r=n_r)
        for l in range(layers):
            c.prefill(k[l * n:(l + 1) * n], v[l * n:(l + 1) * n], a[l * n:(l + 1) * n], budgets[l], 64,
                      unit_begin=l * n)
        caches.append(c)
    scale = 1.0 / np.sqrt(d)
    for s in range(40):  # n_r = 32: one flush at step 31
        q = torch.from_numpy(rng.standard_normal((layers, n, G, d)).astype(np.float16)).cuda()
        tk = torch.from_numpy(rng.standard_normal((layers, n, d)).astype(np.float16)).cuda()
        tv = torch.from_numpy(rng.standard_normal((layers, n, d)).astype(np.float16)).cuda()
        layers_forms(caches, q, tk, tv, scale, n)
    for c in caches:
        c.check()
    for c in caches[1:]:
        assert caches[0].unit_info(0) == c.unit_info(0)


def test_decode_step_layers_partial_flush_matches_per_layer_calls(mkv):
    """The fused flush path of the per-layer form (one append launch for every layer, plans built
    on the device) and the coalesced form's single append, with only some layers' units reaching
    n_r in a step: bit-identical as in layers_forms."""
    d, n, G, L, layers, n_r = 128, 8, 4, 700, 4, 16
    rng = np.random.default_rng(33)
    budgets = [300, 30, 200, 90]
    caps = [budgets[l] + 32 for l in range(layers) for _ in range(n)]
    k = torch.from_numpy(rng.standard_normal((layers * n, L, d)).astype(np.float16)).cuda()
    v = torch.from_numpy(rng.standard_normal((layers * n, L, d)).astype(np.float16)).cuda()
    a = torch.from_numpy(rng.random((layers * n, L)).astype(np.float32)).cuda()
    caches = []
    for _ in range(4):
        c = mkv.KVCache(layers * n, caps, max_decode_tokens=96, n_r=n_r)
        for l in range(layers):
            c.prefill(k[l * n:(l + 1) * n], v[l * n:(l + 1) * n], a[l * n:(l + 1) * n], budgets[l], 32,
                      unit_begin=l * n)
        # stagger the residual counts: layer l starts with 3 l extra tokens
        for l in range(layers):
            for t in range(3 * l):
                c.append(*(2 * [torch.full((n, d), 0.01 * (t + 1), dtype=torch.float16, device="cuda")]),
                         unit_begin=l * n)
        caches.append(c)
    scale = 1.0 / np.sqrt(d)
    for s in range(40):  # flushes hit different layers at different steps
        q = torch.from_numpy(rng.standard_normal((layers, n, G, d)).astype(np.float16)).cuda()
        tk = torch.from_numpy(rng.standard_normal((layers, n, d)).astype(np.float16)).cuda()
        tv = torch.from_numpy(rng.standard_normal((layers, n, d)).astype(np.float16)).cuda()
        layers_forms(caches, q, tk, tv, scale, n)
    for c in caches:
        c.check()
    for u in range(0, layers * n, n):
        for c in caches[1:]:
            assert caches[0].unit_info(u) == c.unit_info(u)


def test_decode_step_layers_overlapping_ranges_match_per_layer_calls(mkv):
    """mkv_decode_step_layers is n_layers consecutive decode_step calls: with overlapping but
    non-identical unit ranges (units appended twice in one call) a layer may not start its page
    pass early, and the result must equal the consecutive per-range calls bit for bit, through
    flushes (early flag only for ranges disjoint from every earlier one)."""
    from paper_2411_18077_b200 import _capi
    d, G, L, n_r = 128, 4, 600, 16
    ranges = [(0, 8), (4, 8), (10, 6), (2, 3)]  # overlapping, none identical
    n_units = 16
    rng = np.random.default_rng(44)
    caps = [200 + 40 for _ in range(n_units)]
    k = torch.from_numpy(rng.standard_normal((n_units, L, d)).astype(np.float16)).cuda()
    v = torch.from_numpy(rng.standard_normal((n_units, L, d)).astype(np.float16)).cuda()
    a = torch.from_numpy(rng.random((n_units, L)).astype(np.float32)).cuda()
    caches = []
    for _ in range(2):
        c = mkv.KVCache(n_units, caps, max_decode_tokens=160, n_r=n_r)
        c.prefill(k, v, a, [150 + 3 * u for u in range(n_units)], 40)
        caches.append(c)
    scale = 1.0 / np.sqrt(d)
    for s in range(24):
        qs = [torch.from_numpy(rng.standard_normal((n, G, d)).astype(np.float16)).cuda() for _, n in ranges]
        tks = [torch.from_numpy(rng.standard_normal((n, d)).astype(np.float16)).cuda() for _, n in ranges]
        tvs = [torch.from_numpy(rng.standard_normal((n, d)).astype(np.float16)).cuda() for _, n in ranges]
        outs = [torch.empty_like(q) for q in qs]
        args = (_capi.DecodeArgs * len(ranges))()
        for l, (ub, n) in enumerate(ranges):
            args[l] = _capi.DecodeArgs(ub, n, G, qs[l].data_ptr(), tks[l].data_ptr(), tvs[l].data_ptr(),
                                       outs[l].data_ptr(), float(scale))
        _capi.check(_capi.lib().mkv_decode_step_layers(caches[0].h, len(ranges), args,
                                                       int(torch.cuda.current_stream().cuda_stream)), "layers")
        refs = [caches[1].decode_step(qs[l], tks[l], tvs[l], scale, unit_begin=ub) for l, (ub, n) in enumerate(ranges)]
        for l in range(len(ranges)):
            assert torch.equal(outs[l], refs[l]), f"step {s} range {l}"
    for c in caches:
        c.check()
    for u in range(n_units):
        assert caches[0].unit_info(u) == caches[1].unit_info(u)


def test_decode_headline_shape_parity(mkv):
    """configs[1]'s real per-unit shape through the headline API: 32K context, the pyramid budgets
    hh 6084 -> 468 (+ rw 3276), 32 layers x 4 units, G = 4, every step through
    mkv_decode_step_layers (cross-layer overlap, device-built plans on the fused flush step),
    131 steps so the n_r = 128 flush happens inside; outputs checked against the oracle per
    q-head (GQA composition, fp16-rounded params) before, at and after the flush."""
    from tests.gpu_util import f32
    d, G, L, NL, U, n_r = 128, 4, 32768, 32, 4, 128
    P = oracle.port()
    x, rw = int(0.10 * L), int(0.10 * L)
    hh = [int(h) for h in P.allocate_pyramid(x, NL, 7, True)]
    assert hh[0] == 6084 and hh[-1] == 468 and rw == 3276
    n_units = NL * U
    caps = [hh[u // U] + rw for u in range(n_units)]
    cache = mkv.KVCache(n_units, caps, max_decode_tokens=256, n_r=n_r)
    ocs = []
    for l in range(NL):
        k = mkv.synth_fp16((U, L * d), SEED, (2 << 48) | ((l * U) << 16), 1 << 16).view(U, L, d)
        v = mkv.synth_fp16((U, L * d), SEED, (3 << 48) | ((l * U) << 16), 1 << 16).view(U, L, d)
        a = mkv.synth_uniform((U, L), SEED, (7 << 48) | ((l * U) << 16), 1 << 16)
        cache.prefill(k, v, a, [hh[l]] * U, rw, unit_begin=l * U)
        kh, vh, ah = k.cpu().numpy(), v.cpu().numpy(), a.cpu().numpy()
        for j in range(U):
            oc = P.cache(d=d, n_r=n_r)
            oc.prefill(f32(kh[j]), f32(vh[j]), ah[j], hh[l], rw)
            ocs.append(oc)
    scale = 1.0 / np.sqrt(d)
    steps = 131
    check = {0, 64, 126, 127, 128, 130}
    worst = 0.0
    for s in range(steps):
        q = mkv.synth_fp16((n_units, G * d), SEED, (4 << 48) | (s + 1), 1 << 16).view(NL, U, G, d)
        tk = mkv.synth_fp16((n_units, d), SEED, (5 << 48) | (s + 1), 1 << 16).view(NL, U, d)
        tv = mkv.synth_fp16((n_units, d), SEED, (6 << 48) | (s + 1), 1 << 16).view(NL, U, d)
        out = cache.decode_step_layers(q, tk, tv, scale).float().cpu().numpy().reshape(n_units, G, d)
        qh = q.cpu().numpy().reshape(n_units, G, d)
        tkh, tvh = tk.cpu().numpy().reshape(n_units, d), tv.cpu().numpy().reshape(n_units, d)
        for u in range(n_units):
            ocs[u].append(f32(tkh[u]), f32(tvh[u]))
            if s in check:
                for h in range(G):
                    exp = ocs[u].attend(f32(qh[u, h]), scale, param_fp16=True)
                    worst = max(worst, max_abs(out[u, h], exp))
    cache.check()
    info = cache.unit_info(0)
    assert info["tokens_residual"] == (steps % n_r) and info["n_blocks"] == 2
    assert worst <= TOL, worst


@pytest.mark.parametrize("env", [{"MKV_PAGES_IMPL": "tc"}, {"MKV_FLUSH": "fused"}, {"MKV_LAYERS_SPLIT": "1"},
                                 {"MKV_MERGE": "split"}, {"MKV_MERGE": "finish"}, {"MKV_STEPS": "off"}],
                         ids=["tcgen05-page-pass", "fused-flush", "layers-split", "split-finish", "one-kernel-finish",
                              "per-step-decode-steps"])
def test_decode_variant_parity(env):
    """The decode variants kept as measured A/Bs pass the same oracle parity tests (G = 1 / 4 / 8,
    flushes, partial pages, split units, the headline shape, bit-identity of the multi-layer
    call): MKV_PAGES_IMPL=tc -- the tcgen05 page pass (decode_tc.cu: codes -> TMEM,
    tcgen05.mma with per-page scaled B operands); MKV_FLUSH=fused -- the residual flush done by
    the finish kernel of the step that fills the block (pages built there, the block attended
    dequantized, the next plan uploaded off the critical path); MKV_MERGE=split / finish -- the
    finish step forced into its two-kernel form (persistent residual kernel + merge kernel on
    per-unit arrival counters) or its one-kernel form for every call size (the default picks by
    unit count, so the small suite cases would otherwise only see the one-kernel form)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", os.path.join(root, "tests", "test_gpu_decode.py"),
                        "-k", "not variant"], cwd=root, env=dict(os.environ, **env), capture_output=True, text=True,
                       timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_decode_256k_mha_units_parity(mkv):
    """configs[4]'s decode units (LWM-Text-7B MHA, 256K context, G = 1) at the pyramid's extreme
    layers (hh 48683 and 3745, rw 26214: ~4.7K and ~1.9K pages per unit), through a flush, against
    the oracle per head."""
    from tests.gpu_util import f32
    d, G, L, n_r = 128, 1, 262144, 128
    P = oracle.port()
    hh_all = [int(h) for h in P.allocate_pyramid(int(0.10 * L), 32, 7, True)]
    rw = int(0.10 * L)
    hh = [hh_all[0], hh_all[-1]]
    n = 2
    k = mkv.synth_fp16((n, L * d), SEED, 2 << 48, 1 << 16).view(n, L, d)
    v = mkv.synth_fp16((n, L * d), SEED, 3 << 48, 1 << 16).view(n, L, d)
    a = mkv.synth_uniform((n, L), SEED, 7 << 48, 1 << 16)
    cache = mkv.KVCache(n, [h + rw for h in hh], max_decode_tokens=256, n_r=n_r)
    cache.prefill(k, v, a, hh, rw)
    kh, vh, ah = k.cpu().numpy(), v.cpu().numpy(), a.cpu().numpy()
    ocs = []
    for u in range(n):
        oc = P.cache(d=d, n_r=n_r)
        oc.prefill(f32(kh[u]), f32(vh[u]), ah[u], hh[u], rw)
        ocs.append(oc)
    scale = 1.0 / np.sqrt(d)
    worst = 0.0
    for s in range(130):
        q = mkv.synth_fp16((n, G * d), SEED, (4 << 48) | (s + 1), 1 << 16).view(n, G, d)
        tk = mkv.synth_fp16((n, d), SEED, (5 << 48) | (s + 1), 1 << 16)
        tv = mkv.synth_fp16((n, d), SEED, (6 << 48) | (s + 1), 1 << 16)
        out = cache.decode_step(q, tk, tv, scale).float().cpu().numpy()
        qh, tkh, tvh = q.cpu().numpy(), tk.cpu().numpy(), tv.cpu().numpy()
        for u in range(n):
            ocs[u].append(f32(tkh[u]), f32(tvh[u]))
            if s in (0, 126, 127, 129):
                worst = max(worst, max_abs(out[u, 0], ocs[u].attend(f32(qh[u, 0]), scale, param_fp16=True)))
    cache.check()
    assert worst <= TOL, worst


@pytest.mark.parametrize("append", [True, False])
def test_decode_steps_matches_per_step_calls(mkv, append):
    """mkv_decode_steps (one FFI crossing for a prepared token stream, the reference's decode loop
    minikv_cli.cpp:180-201) against the same steps as mkv_decode_step calls, across two residual
    flushes (n_r = 32) and on a strided output: bit for bit on the per-step kernels
    (MKV_STEPS=off); on the unit-resident steps kernel (the default for these few short units)
    equal up to the fp32 accumulation order of a different split of the pages, with the same
    cache state (exported codes / params / residual bit-exact) and within tolerance of the
    oracle's decode at every step."""
    import os
    from tests.gpu_util import f32
    d, G, n, L, hh, rw, S, n_r = 128, 4, 3, 700, 60, 50, 70, 32
    scale = 1.0 / np.sqrt(d)
    k = torch.from_numpy(np.stack([synth_np(SEED, oracle.stream_id(oracle.KIND_K, u), (L, d)) for u in range(n)])).cuda()
    v = torch.from_numpy(np.stack([synth_np(SEED, oracle.stream_id(oracle.KIND_V, u), (L, d)) for u in range(n)])).cuda()
    a = torch.rand((n, L), generator=torch.Generator().manual_seed(3)).cuda()
    q = mkv.synth_fp16((S, n, G, d), SEED, 11 << 48, 1 << 16)
    tk = mkv.synth_fp16((S, n, d), SEED, 12 << 48, 1 << 16)
    tv = mkv.synth_fp16((S, n, d), SEED, 13 << 48, 1 << 16)
    caches = [mkv.KVCache(n, hh + rw, max_decode_tokens=S + n_r, n_r=n_r) for _ in range(2)]
    for c in caches:
        c.prefill(k, v, a, hh, rw)
    ref = torch.empty((S, n, G, d), dtype=torch.float16, device="cuda")
    for s in range(S):
        caches[0].decode_step(q[s], tk[s] if append else None, tv[s] if append else None, scale, out=ref[s])
    big = torch.zeros((S, 2, n, G, d), dtype=torch.float16, device="cuda")
    got = big[:, 1]  # step stride 2 n G d: exercises out_step != n G d
    caches[1].decode_steps(q, tk if append else None, tv if append else None, scale, out=got)
    torch.cuda.synchronize()
    if os.environ.get("MKV_STEPS") == "off":
        assert torch.equal(got, ref)
    else:
        assert (got.float() - ref.float()).abs().max().item() <= 2e-3
        for u in range(n):
            assert caches[0].unit_info(u) == caches[1].unit_info(u)
            for which in (0, 1):
                e0, e1 = caches[0].export_reference(u, which), caches[1].export_reference(u, which)
                for x0, x1 in zip(e0, e1):
                    assert np.array_equal(np.asarray(x0), np.asarray(x1))
            r0, r1 = caches[0].export_residual(u), caches[1].export_residual(u)
            for x0, x1 in zip(r0, r1):
                assert np.array_equal(np.asarray(x0), np.asarray(x1))
        # the oracle's decode of the same stream (fp16-rounded params), every step
        P = oracle.port()
        kn, vn, qn = k.cpu().numpy(), v.cpu().numpy(), q.cpu().numpy()
        tkn, tvn, gn = tk.cpu().numpy(), tv.cpu().numpy(), got.float().cpu().numpy()
        a_n = a.cpu().numpy()
        worst = 0.0
        for u in range(n):
            oc = P.cache(d=d, n_r=n_r)
            oc.prefill(f32(kn[u]), f32(vn[u]), a_n[u], hh, rw)
            for s in range(S):
                if append:
                    oc.append(f32(tkn[s, u]), f32(tvn[s, u]))
                for h in range(G):
                    exp = oc.attend(f32(qn[s, u, h]), scale, param_fp16=True)
                    worst = max(worst, max_abs(gn[s, u, h], exp))
        assert worst <= TOL, worst
    for c in caches:
        c.check()
        c.close()


@pytest.mark.parametrize("G,n_r,append", [(1, 16, True), (8, 16, True), (4, 128, True), (2, 32, False)])
def test_decode_steps_kernel_vs_oracle(mkv, G, n_r, append):
    """The unit-resident steps kernel (mkv_decode_steps for few short units) against the oracle's
    decode at every step: G = 1 / 2 / 4 / 8, flushes every 16 steps (n_r = 16), a partially
    filled residual block carried in (n_r = 128), attend-only steps, a partial last prefill page."""
    from tests.gpu_util import f32
    d, n, L, hh, rw, S = 128, 5, 500, 70, 37, 40
    scale = 1.0 / np.sqrt(d)
    k = np.stack([synth_np(SEED, oracle.stream_id(oracle.KIND_K, u), (L, d)) for u in range(n)])
    v = np.stack([synth_np(SEED, oracle.stream_id(oracle.KIND_V, u), (L, d)) for u in range(n)])
    a = np.random.default_rng(SEED + G).random((n, L)).astype(np.float32)
    q = mkv.synth_fp16((S, n, G, d), SEED, (21 << 48) | G, 1 << 16)
    tk = mkv.synth_fp16((S, n, d), SEED, 22 << 48, 1 << 16)
    tv = mkv.synth_fp16((S, n, d), SEED, 23 << 48, 1 << 16)
    cache = mkv.KVCache(n, hh + rw, max_decode_tokens=S + 2 * n_r, n_r=n_r)
    cache.prefill(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), torch.from_numpy(a).cuda(), hh, rw)
    P = oracle.port()
    ocs = []
    for u in range(n):
        oc = P.cache(d=d, n_r=n_r)
        oc.prefill(f32(k[u]), f32(v[u]), a[u], hh, rw)
        ocs.append(oc)
    pre = 5 if append else 0  # residual rows carried into the call (per-step path)
    for s in range(pre):
        qq = mkv.synth_fp16((n, G, d), SEED, (24 << 48) | s, 1 << 16)
        kk = mkv.synth_fp16((n, d), SEED, (25 << 48) | s, 1 << 16)
        vv = mkv.synth_fp16((n, d), SEED, (26 << 48) | s, 1 << 16)
        cache.decode_step(qq, kk, vv, scale)
        kn, vn = kk.cpu().numpy(), vv.cpu().numpy()
        for u in range(n):
            ocs[u].append(f32(kn[u]), f32(vn[u]))
    out = cache.decode_steps(q, tk if append else None, tv if append else None, scale)
    torch.cuda.synchronize()
    got, qn, tkn, tvn = out.float().cpu().numpy(), q.cpu().numpy(), tk.cpu().numpy(), tv.cpu().numpy()
    worst = 0.0
    for s in range(S):
        for u in range(n):
            if append:
                ocs[u].append(f32(tkn[s, u]), f32(tvn[s, u]))
            for h in range(G):
                exp = ocs[u].attend(f32(qn[s, u, h]), scale, param_fp16=True)
                worst = max(worst, max_abs(got[s, u, h], exp))
    cache.check()
    info = cache.unit_info(0)
    assert info["tokens_residual"] == ((pre + S) % n_r if append else 0)
    assert worst <= TOL, worst
    cache.close()
