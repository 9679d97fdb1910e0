"""K1 two-pass selective flash-attention prefill (tcgen05) vs the oracle.

Oracle: selective_flash_attn (attention.cpp:29-117) per q-head on the same
fp16 inputs widened to fp32; A_cumul per kv-head = fp32 sum over its G q-heads
(the build-defined GQA contract).
Tolerances: X_O max abs <= 5e-3; LSE abs <= 1e-3;
A_cumul |d| <= 1e-3 + 2e-3 |ref|; sum_j A_cumul = G * lq within 1e-3 relative.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from tests.gpu_util import SEED, f32, synth_np

pytestmark = pytest.mark.gpu

TOL_O, TOL_LSE, TOL_A_ABS, TOL_A_REL = 5e-3, 1e-3, 1e-3, 2e-3


@pytest.fixture(scope="module")
def mkv():
    import paper_2411_18077_b200 as m
    return m


def make_inputs(B, Hq, Hkv, lq, lk, seed=SEED):
    d = 128
    q = np.stack([np.stack([synth_np(seed, oracle.stream_id(oracle.KIND_Q, b * Hq + h), (lq, d)) for h in range(Hq)])
                  for b in range(B)])
    k = np.stack([np.stack([synth_np(seed, oracle.stream_id(oracle.KIND_K, b * Hkv + h), (lk, d)) for h in range(Hkv)])
                  for b in range(B)])
    v = np.stack([np.stack([synth_np(seed, oracle.stream_id(oracle.KIND_V, b * Hkv + h), (lk, d)) for h in range(Hkv)])
                  for b in range(B)])
    return q, k, v


def run_case(mkv, B, Hq, Hkv, lq, lk, causal, scale_mult=1.0):
    q, k, v = make_inputs(B, Hq, Hkv, lq, lk)
    if scale_mult != 1.0:
        q = (q.astype(np.float32) * scale_mult).astype(np.float16)
    scale = 1.0 / math.sqrt(128)
    r = mkv.selective_flash_attn(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(),
                                 scale, causal)
    out = r.output.float().cpu().numpy()
    lse = r.lse.cpu().numpy()
    ac = r.a_cumul.cpu().numpy()
    P = oracle.port()
    G = Hq // Hkv
    worst = {"o": 0.0, "lse": 0.0, "a": 0.0}
    for b in range(B):
        for hk in range(Hkv):
            acc = np.zeros(lk, np.float32)
            for g in range(G):
                h = hk * G + g
                ref = P.selective_flash_attn(f32(q[b, h]), f32(k[b, hk]), f32(v[b, hk]), scale, causal, 64, 64)
                worst["o"] = max(worst["o"], float(np.max(np.abs(out[b, h] - ref.output))))
                worst["lse"] = max(worst["lse"], float(np.max(np.abs(lse[b, h] - ref.lse))))
                acc = acc + ref.a_cumul if g else ref.a_cumul.copy()
            err = np.abs(ac[b, hk] - acc)
            assert np.all(err <= TOL_A_ABS + TOL_A_REL * np.abs(acc)), (b, hk, float(err.max()))
            worst["a"] = max(worst["a"], float(err.max()))
            total = float(np.sum(ac[b, hk], dtype=np.float64))
            assert abs(total - G * lq) <= 1e-3 * G * lq, (total, G * lq)
    assert worst["o"] <= TOL_O, worst
    assert worst["lse"] <= TOL_LSE, worst
    return worst


@pytest.mark.parametrize("lq,lk,causal", [(128, 128, True), (256, 256, True), (300, 300, True), (77, 77, True),
                                          (200, 333, True), (256, 256, False), (130, 500, False), (1, 1, True),
                                          (1, 64, True)])
def test_prefill_small(mkv, lq, lk, causal):
    run_case(mkv, 1, 2, 1, lq, lk, causal)


def test_prefill_gqa_batch(mkv):
    run_case(mkv, 2, 8, 2, 640, 640, True)


def test_prefill_sharp_softmax(mkv):
    # larger logits exercise the lazy-rescale path (max grows by > 2^8 across tiles)
    run_case(mkv, 1, 2, 2, 512, 512, True, scale_mult=6.0)


def test_prefill_long_invariants(mkv):
    """L = 8K: A_cumul column sums = G * lq, sampled rows of X_O vs single-query oracle."""
    B, Hq, Hkv, L = 1, 4, 1, 8192
    q, k, v = make_inputs(B, Hq, Hkv, L, L)
    scale = 1.0 / math.sqrt(128)
    r = mkv.selective_flash_attn(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(),
                                 scale, True)
    ac = r.a_cumul.cpu().numpy()
    assert abs(float(ac.sum(dtype=np.float64)) - Hq * L) <= 1e-3 * Hq * L
    assert np.all(ac >= 0)
    out = r.output.float().cpu().numpy()
    P = oracle.port()
    for h in range(Hq):
        for i in (0, 1, 127, 128, 4095, 8191):
            o, _ = P.decode_attention(f32(q[0, h, i]), f32(k[0, 0, :i + 1]), f32(v[0, 0, :i + 1]), scale)
            assert float(np.max(np.abs(out[0, h, i] - o))) <= TOL_O


def test_prefill_errors(mkv):
    x = torch.zeros((1, 1, 8, 128), dtype=torch.float16, device="cuda")
    y = torch.zeros((1, 1, 4, 128), dtype=torch.float16, device="cuda")
    with pytest.raises(mkv.InvalidArgument):  # causal requires lq <= lk (attention.cpp:22-24)
        mkv.selective_flash_attn(x, y, y, 0.1, True)
    with pytest.raises(mkv.InvalidArgument):
        mkv.selective_flash_attn(x[:, :, :0], y, y, 0.1, False)


def test_prefill_128k_sampled_rows_and_columns(mkv):
    """configs[3] shape (Mistral-7B layer, 32 q / 8 kv heads, 128K causal): sampled X_O / LSE rows
    against the reference's single-query attention over the row's visible keys
    (attention.cpp:119-143 = row i of selective_flash_attn), and sampled A_cumul COLUMNS against an
    fp64 host recomputation of pass 2 (attention.cpp:101-115) from Q, k_j and the device LSE
    (itself checked on the sampled rows) -- the A_cumul that drives selection at this shape,
    column by column.  Also the global invariant sum A_cumul = G * lq."""
    import bench
    Hq, Hkv, L, d = 32, 8, 131072, 128
    q = mkv.synth_fp16((1, Hq, L, d), SEED, 1 << 48, 1 << 16)
    k = mkv.synth_fp16((1, Hkv, L, d), SEED, 2 << 48, 1 << 16)
    v = mkv.synth_fp16((1, Hkv, L, d), SEED, 3 << 48, 1 << 16)
    scale = 1.0 / math.sqrt(d)
    r = mkv.selective_flash_attn(q, k, v, scale, True)
    torch.cuda.synchronize()
    ac_sum = float(r.a_cumul.double().sum().item())
    assert abs(ac_sum - Hq * L) <= 1e-3 * Hq * L
    res = bench.prefill_parity(q, k, v, r, Hq, Hkv, L, d, scale,
                               rows=(0, 1, 127, 128, 65537, L - 129, L - 1),
                               cols=[0, 1, 2, 63, 64, 4097, L // 3, L // 2 + 1, L - 200, L - 128, L - 2, L - 1])
    assert res["x_o_max_abs"] <= TOL_O, res
    assert res["lse_max_abs"] <= TOL_LSE, res
    assert res["a_cumul_excess_over_rel_tol"] <= TOL_A_ABS, res


def test_prefill_256k_mha_sampled_rows_and_columns(mkv):
    """configs[4]'s prefill layer (LWM-Text-7B: 32 MHA heads, 256K causal): sampled X_O / LSE rows
    and A_cumul columns against the reference (as the 128K test), plus sum A_cumul = lq per head."""
    import bench
    Hq = Hkv = 32
    L, d = 262144, 128
    q = mkv.synth_fp16((1, Hq, L, d), SEED, 1 << 48, 1 << 16)
    k = mkv.synth_fp16((1, Hkv, L, d), SEED, 2 << 48, 1 << 16)
    v = mkv.synth_fp16((1, Hkv, L, d), SEED, 3 << 48, 1 << 16)
    scale = 1.0 / math.sqrt(d)
    r = mkv.selective_flash_attn(q, k, v, scale, True)
    torch.cuda.synchronize()
    sums = r.a_cumul[0].double().sum(-1)
    assert float((sums - L).abs().max()) <= 1e-3 * L
    res = bench.prefill_parity(q, k, v, r, Hq, Hkv, L, d, scale, rows=(0, 131071, L - 1),
                               cols=[0, 5, L // 2, L - 3, L - 1])
    assert res["x_o_max_abs"] <= TOL_O, res
    assert res["lse_max_abs"] <= TOL_LSE, res
    assert res["a_cumul_excess_over_rel_tol"] <= TOL_A_ABS, res
