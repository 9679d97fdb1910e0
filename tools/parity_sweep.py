"""Extended randomized parity sweep on the B200 (beyond the seeds the test suite pins):
decode (random unit counts, GQA groups, n_r, budgets, step counts), K2 selection on random
and tie-heavy scores, K3 codes/params through the reference-format export, all against the
oracle.  Prints one line per family with the case count and the worst deviation.

usage: python tools/parity_sweep.py [n_decode] [n_select] [n_pack] [n_prefill]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2411_18077_b200 as mkv  # noqa: E402
from tests.test_gpu_decode import TOL, run_decode  # noqa: E402
from tests.test_gpu_prefill import TOL_A_ABS, TOL_A_REL, TOL_LSE, TOL_O, make_inputs  # noqa: E402
from tests.gpu_util import f32  # noqa: E402

nd = int(sys.argv[1]) if len(sys.argv) > 1 else 60
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 300
npk = int(sys.argv[3]) if len(sys.argv) > 3 else 100
npf = int(sys.argv[4]) if len(sys.argv) > 4 else 40
P = oracle.port()

# ---- K4 decode ----
worst, fails = 0.0, 0
for seed in range(1000, 1000 + nd):
    rng = np.random.default_rng(seed)
    n_units = int(rng.integers(1, 24))
    G = int(rng.choice([1, 2, 4, 8]))
    n_r = int(rng.choice([16, 32, 64, 128]))
    L = int(rng.integers(20, 900))
    rw = int(rng.integers(0, L // 4 + 1))
    hh = [int(rng.integers(0 if rw else 1, L // 3 + 2)) for _ in range(n_units)]
    steps = int(rng.integers(1, 2 * n_r + 5))
    w = run_decode(mkv, n_units=n_units, G=G, L=L, hh=0, rw=rw, steps=steps, n_r=n_r,
                   check_every=max(1, steps // 12), hh_per_unit=hh, seed=seed)
    worst = max(worst, w)
    fails += w > TOL
print(f"K4 decode: {nd} random configs, worst max|t_O - oracle| = {worst:.3e} (tolerance {TOL}), failures {fails}")

# ---- K2 selection (bit-exact indices) ----
fails = 0
for seed in range(ns):
    rng = np.random.default_rng(50000 + seed)
    L = int(rng.integers(1, 20000))
    kind = seed % 3
    if kind == 0:
        a = rng.random(L).astype(np.float32)
    elif kind == 1:  # heavy ties
        a = rng.integers(0, 4, L).astype(np.float32)
    else:  # +-0 and denormal-ish mixes
        a = (rng.random(L) * (rng.random(L) < 0.5)).astype(np.float32) * np.float32(1e-38)
    hh, rw = int(rng.integers(0, L + 1)), int(rng.integers(0, L // 2 + 1))
    kept, nk = mkv.select_token_counts(torch.from_numpy(a).cuda()[None], hh, rw)
    got = kept[0, :int(nk[0])].cpu().numpy().astype(np.int64)
    exp, _ = P.select_token_counts(a, hh, rw)
    fails += not np.array_equal(got, exp)
print(f"K2 select: {ns} random cases (uniform / tie-heavy / tiny values), index mismatches {fails}")

# ---- K3 quantize + pack (bit-exact codes and fp32 params through the reference stream) ----
fails = 0
for seed in range(npk):
    rng = np.random.default_rng(90000 + seed)
    L = int(rng.integers(1, 1500))
    rw = int(rng.integers(0, L // 3 + 1))
    hh = int(rng.integers(0 if rw else 1, L // 2 + 1))
    scale = float(10.0 ** rng.uniform(-3, 2))
    k = (rng.standard_normal((1, L, 128)) * scale).astype(np.float16)
    v = (rng.standard_normal((1, L, 128)) * scale).astype(np.float16)
    a = rng.random((1, L)).astype(np.float32)
    cache = mkv.KVCache(1, min(hh + rw, L), 0, keep_fp32_params=True)
    cache.prefill(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), torch.from_numpy(a).cuda(), hh, rw)
    oc = P.cache()
    oc.prefill(k[0].astype(np.float32), v[0].astype(np.float32), a[0], hh, rw)
    for which in (0, 1):
        w, par, br = cache.export_reference(0, which)
        ow, opar, obr = oc.export(which)
        fails += not (np.array_equal(w, ow) and np.array_equal(par, opar) and np.array_equal(br, obr))
    cache.close()
print(f"K3 pack: {npk} random prefills (scales 1e-3..1e2), K and V streams compared, mismatches {fails}")

# ---- K1 prefill (X_O, LSE, A_cumul within the suite's tolerances) ----
import math  # noqa: E402
worst = {"o": 0.0, "lse": 0.0, "a_excess": 0.0}
fails = 0
for seed in range(npf):
    rng = np.random.default_rng(70000 + seed)
    B, Hkv, G = int(rng.integers(1, 3)), int(rng.integers(1, 3)), int(rng.choice([1, 2, 4]))
    causal = bool(rng.integers(0, 2))
    lq = int(rng.integers(1, 700))
    lk = lq + int(rng.integers(0, 300)) if causal else int(rng.integers(1, 1000))
    q, k, v = make_inputs(B, Hkv * G, Hkv, lq, lk, seed=7 + seed)
    scale = 1.0 / math.sqrt(128)
    r = mkv.selective_flash_attn(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(),
                                 scale, causal)
    out, lse, ac = r.output.float().cpu().numpy(), r.lse.cpu().numpy(), r.a_cumul.cpu().numpy()
    ok = True
    for b in range(B):
        for hk in range(Hkv):
            acc = None
            for g in range(G):
                h = hk * G + g
                ref = P.selective_flash_attn(f32(q[b, h]), f32(k[b, hk]), f32(v[b, hk]), scale, causal, 64, 64)
                eo = float(np.max(np.abs(out[b, h] - ref.output)))
                el = float(np.max(np.abs(lse[b, h] - ref.lse)))
                worst["o"], worst["lse"] = max(worst["o"], eo), max(worst["lse"], el)
                ok &= eo <= TOL_O and el <= TOL_LSE
                acc = ref.a_cumul.copy() if acc is None else acc + ref.a_cumul
            ex = float(np.max(np.abs(ac[b, hk] - acc) - (TOL_A_ABS + TOL_A_REL * np.abs(acc))))
            worst["a_excess"] = max(worst["a_excess"], ex) if worst["a_excess"] else ex
            ok &= ex <= 0
    fails += not ok
print(f"K1 prefill: {npf} random shapes (B, GQA group, causal / not, lq <= lk), worst |X_O| {worst['o']:.2e} "
      f"(tol {TOL_O}), |LSE| {worst['lse']:.2e} (tol {TOL_LSE}), A_cumul max(err - tol) {worst['a_excess']:.2e} "
      f"(<= 0 passes), failures {fails}")
