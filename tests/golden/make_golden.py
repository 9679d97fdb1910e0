"""Generate tests/golden/minikv_golden.npz by running the REFERENCE itself.

Inputs are seeded numpy arrays (stored in the fixture); outputs come from
oracle/_ref/libminikv_ref.so, i.e. the unmodified reference sources in
/root/reference/proj/core/src compiled by oracle/Makefile.  Run in the build
container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

The fixture is what pins the C restatement (oracle/minikv_oracle.c) on boxes
where the reference sources are absent (tests/test_oracle_golden.py).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "minikv_golden.npz")


def main():
    R = oracle.ref()
    rng = np.random.default_rng(20241127)
    g = {}
    # attention.cpp:29-117 -- shapes mirror test_attention.cpp:47-135
    att_cases = [(64, 64, 16, 1, 16, 16), (64, 64, 16, 1, 8, 32), (4, 8, 8, 1, 4, 4),
                 (32, 32, 16, 1, 8, 8), (1, 1, 4, 1, 4, 4), (50, 77, 8, 0, 7, 13), (96, 96, 128, 1, 64, 64)]
    for i, (lq, lk, d, causal, bm, bn) in enumerate(att_cases):
        q = rng.standard_normal((lq, d)).astype(np.float32)
        k = rng.standard_normal((lk, d)).astype(np.float32)
        v = rng.standard_normal((lk, d)).astype(np.float32)
        r = R.selective_flash_attn(q, k, v, 1.0 / np.sqrt(d), bool(causal), bm, bn)
        g[f"att{i}_shape"] = np.array([lq, lk, d, causal, bm, bn])
        g[f"att{i}_q"], g[f"att{i}_k"], g[f"att{i}_v"] = q, k, v
        g[f"att{i}_out"], g[f"att{i}_lse"], g[f"att{i}_acumul"] = r.output, r.lse, r.a_cumul
    # decode_attention, attention.cpp:119-143
    q = rng.standard_normal(8).astype(np.float32)
    keys = rng.standard_normal((16, 8)).astype(np.float32)
    vals = rng.standard_normal((16, 8)).astype(np.float32)
    o, a = R.decode_attention(q, keys, vals, 1.0 / np.sqrt(8))
    g.update(dec_q=q, dec_k=keys, dec_v=vals, dec_out=o, dec_attn=a)
    # quantize_matrix, quantizer.cpp:102-151 (short final group: 20 rows, test_quantizer.cpp:189-202)
    for i, (rows, cols) in enumerate([(20, 4), (37, 40), (128, 64), (1, 32), (16, 1)]):
        m = (rng.standard_normal((rows, cols)) * 3.0).astype(np.float32)
        g[f"qm{i}_m"] = m
        for axis in (0, 1):
            w, p = R.quantize_matrix(m, axis)
            g[f"qm{i}_ax{axis}_words"], g[f"qm{i}_ax{axis}_params"] = w, p
            g[f"qm{i}_ax{axis}_deq"] = R.quant_dequant_matrix(m, axis)
    # select_token_counts, selection.cpp:10-33
    for i, (L, hh, rw, levels) in enumerate([(256, 64, 64, 0), (1000, 100, 100, 5), (100, 95, 10, 0),
                                             (6, 2, 1, 1), (4096, 409, 409, 11)]):
        a = rng.random(L).astype(np.float32) if levels == 0 else \
            (rng.integers(0, levels, L).astype(np.float32) * np.float32(0.5))
        kept, cl = R.select_token_counts(a, hh, rw)
        g[f"sel{i}_a"], g[f"sel{i}_args"], g[f"sel{i}_kept"], g[f"sel{i}_clamped"] = \
            a, np.array([hh, rw]), kept, np.array([cl])
    # allocate_pyramid, selection.cpp:61-83
    for i, (x, layers, depth, bh) in enumerate([(70, 8, 7, 1), (70, 8, 7, 0), (3276, 32, 7, 1),
                                                (26214, 32, 7, 1), (100, 8, 1, 1), (5, 3, 9, 1)]):
        g[f"pyr{i}_args"] = np.array([x, layers, depth, bh])
        g[f"pyr{i}_out"] = R.allocate_pyramid(x, layers, depth, bool(bh))
    # cache engine: prefill + 150 decode steps through a flush (cache_engine.cpp:56-138)
    L, d, hh, rw = 300, 128, 37, 30
    k = rng.standard_normal((L, d)).astype(np.float32)
    v = rng.standard_normal((L, d)).astype(np.float32)
    a = rng.random(L).astype(np.float32)
    c = R.cache_prefill(k, v, a, hh, rw)
    steps = 150
    tq = rng.standard_normal((steps, d)).astype(np.float32)
    tk = rng.standard_normal((steps, d)).astype(np.float32)
    tv = rng.standard_normal((steps, d)).astype(np.float32)
    outs = np.stack([c.decode_step(tq[s], tk[s], tv[s], 1.0 / np.sqrt(d)) for s in range(steps)])
    g.update(cache_k=k, cache_v=v, cache_a=a, cache_args=np.array([hh, rw]), cache_tq=tq, cache_tk=tk,
             cache_tv=tv, cache_out=outs)
    for which in (0, 1):
        w, p, br = c.export(which)
        g[f"cache_ex{which}_words"], g[f"cache_ex{which}_params"], g[f"cache_ex{which}_blocks"] = w, p, br
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
