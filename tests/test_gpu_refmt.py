"""The exact-fp32 reference-format device entries (csrc/refmt.cu) vs the reference.

They back the value-type reference signatures through the drop-in (any head dim, any group
size).  Checked here against the compiled reference (oracle/_ref) and the C restatement:
  * quantize / append_block: packed words and (scale, zero) params BIT-EXACT, including
    blocks appended at unaligned stream offsets, short final groups, +-0, constant groups,
    rounding ties, gathered rows (prefill's gather_rows + append_block);
  * dequantize_matrix: bit-exact (fl(fl(code * scale) + zero), no FMA);
  * decode_attention: scores bit-exact by construction, outputs within 1e-6;
  * selective_flash_attn fp32: X_O / A_cumul within 1e-5, LSE within 1e-5 (the reference's
    own suite demands 1e-4 / 1e-5).
"""
import math

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mkv():
    import paper_2411_18077_b200 as m
    return m


def _ref():
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    return oracle.ref()


def _matrix(rng, rows, cols, kind):
    if kind == "gauss":
        return rng.standard_normal((rows, cols)).astype(np.float32)
    if kind == "grid":  # values on the quantization grid and exact midpoints (rounding ties)
        return (rng.integers(0, 7, (rows, cols)) * 0.5).astype(np.float32)
    if kind == "zeros":  # signed zeros and constant groups
        m = np.zeros((rows, cols), np.float32)
        m[rng.random((rows, cols)) < 0.5] = -0.0
        return m
    return (rng.standard_normal((rows, cols)) * 10 ** rng.uniform(-3, 3)).astype(np.float32)


@pytest.mark.parametrize("kind", ["gauss", "grid", "zeros", "scaled"])
def test_quantize_matrix_bit_exact(mkv, kind):
    R = _ref()
    rng = np.random.default_rng(5)
    for trial in range(25):
        rows, cols = int(rng.integers(1, 70)), int(rng.integers(1, 40))
        gs = int(rng.choice([1, 2, 3, 4, 5, 16, 17]))
        axis = int(trial % 2)
        m = _matrix(rng, rows, cols, kind)
        w, p = mkv.quantize_block(torch.from_numpy(m).cuda(), axis, gs)
        rw, rp = R.quantize_matrix(m, axis, gs)
        assert np.array_equal(w.cpu().numpy().view(np.uint32), rw), (rows, cols, gs, axis)
        gp = p.cpu().numpy()
        assert np.array_equal(gp.view(np.uint32), rp.view(np.uint32)), (rows, cols, gs, axis)
        back = mkv.dequantize(w, p, [rows], cols, axis, gs).cpu().numpy()
        assert np.array_equal(back, R.quant_dequant_matrix(m, axis, gs)), (rows, cols, gs, axis)


def test_append_blocks_at_unaligned_offsets(mkv):
    """Blocks appended to a stream whose length is not a multiple of 16 codes: the device keeps
    the existing low codes of the partial word and continues the stream (quantizer.cpp:9-17)."""
    P = oracle.port()
    rng = np.random.default_rng(7)
    for axis in (0, 1):
        cols, gs = 5, 4
        blocks = [rng.standard_normal((r, cols)).astype(np.float32) for r in (3, 1, 7, 2, 16, 9)]
        words = np.zeros(0, np.uint32)
        params = np.zeros((0, 2), np.float32)
        off = 0
        for b in blocks:
            first = int(words[-1]) if off % 16 else 0
            w, p = mkv.quantize_block(torch.from_numpy(b).cuda(), axis, gs, code_offset=off, first_word=first)
            w = w.cpu().numpy().view(np.uint32)
            words = np.concatenate([words[:off // 16], w])
            params = np.concatenate([params, p.cpu().numpy()])
            off += b.size
        # reference stream: codes of every block, in order, packed continuously
        codes, ref_params = [], []
        for b in blocks:
            c, pp = P.quantize_block(b, axis, gs)
            codes.append(np.asarray(c, np.uint8))
            ref_params.append(np.asarray(pp, np.float32).reshape(-1, 2))
        ref_words = P.pack_codes(np.concatenate(codes))
        assert np.array_equal(words, ref_words)
        assert np.array_equal(params.view(np.uint32), np.concatenate(ref_params).view(np.uint32))
        back = mkv.dequantize(torch.from_numpy(words.view(np.int32)).cuda(), torch.from_numpy(params).cuda(),
                              [b.shape[0] for b in blocks], cols, axis, gs).cpu().numpy()
        exp = np.concatenate([P.dequantize_block(c, pp, b.shape[0], cols, axis, gs)
                              for c, pp, b in zip(codes, ref_params, blocks)])
        assert np.array_equal(back, exp)


def test_gathered_rows_equal_gather_then_quantize(mkv):
    """prefill's gather_rows + append_block (cache_engine.cpp:71-74) in one device pass."""
    R = _ref()
    rng = np.random.default_rng(9)
    k = rng.standard_normal((300, 24)).astype(np.float32)
    idx = np.sort(rng.choice(300, 77, replace=False)).astype(np.int32)
    for axis in (0, 1):
        w, p = mkv.quantize_block(torch.from_numpy(k).cuda(), axis, 16, row_idx=torch.from_numpy(idx).cuda())
        rw, rp = R.quantize_matrix(k[idx], axis, 16)
        assert np.array_equal(w.cpu().numpy().view(np.uint32), rw)
        assert np.array_equal(p.cpu().numpy().view(np.uint32), rp.view(np.uint32))


def test_quantize_rejects_non_finite(mkv):
    m = torch.ones((4, 16), dtype=torch.float32, device="cuda")
    m[2, 3] = float("nan")
    with pytest.raises(mkv.DomainError):
        mkv.quantize_block(m, 0, 16)
    m[2, 3] = float("inf")
    with pytest.raises(mkv.DomainError):
        mkv.quantize_block(m, 1, 16)


@pytest.mark.parametrize("n,d,dv", [(1, 2, 2), (2, 8, 8), (37, 16, 16), (1000, 64, 48), (5000, 128, 128)])
def test_decode_attention_vs_reference(mkv, n, d, dv):
    P = oracle.port()
    rng = np.random.default_rng(n + d)
    q = rng.standard_normal(d).astype(np.float32)
    k = rng.standard_normal((n, d)).astype(np.float32)
    v = rng.standard_normal((n, dv)).astype(np.float32)
    scale = 1.0 / math.sqrt(d)
    out, attn = mkv.decode_attention(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(),
                                     torch.from_numpy(v).cuda(), scale)
    eo, ea = P.decode_attention(q, k, v, scale)
    assert np.max(np.abs(attn.cpu().numpy() - ea)) <= 1e-6
    assert np.max(np.abs(out.cpu().numpy() - eo)) <= 1e-6
    if n == 1:
        assert float(attn[0]) == 1.0 and np.array_equal(out.cpu().numpy(), v[0])


@pytest.mark.parametrize("lq,lk,d,dv,causal", [(1, 1, 4, 4, True), (8, 8, 16, 16, True), (4, 8, 8, 8, True),
                                               (64, 64, 16, 16, True), (37, 100, 8, 12, False),
                                               (300, 513, 128, 128, True), (1024, 1024, 16, 16, True)])
def test_attention_f32_vs_reference(mkv, lq, lk, d, dv, causal):
    P = oracle.port()
    rng = np.random.default_rng(lq * 7 + lk)
    q = rng.standard_normal((lq, d)).astype(np.float32)
    k = rng.standard_normal((lk, d)).astype(np.float32)
    v = rng.standard_normal((lk, dv)).astype(np.float32)
    scale = 1.0 / math.sqrt(d)
    r = mkv.selective_flash_attn_f32(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(),
                                     torch.from_numpy(v).cuda(), scale, causal)
    e = P.selective_flash_attn(q, k, v, scale, causal)
    assert np.max(np.abs(r.output.cpu().numpy() - e.output)) <= 1e-5
    assert np.max(np.abs(r.a_cumul.cpu().numpy() - e.a_cumul)) <= 1e-5
    assert np.max(np.abs(r.lse.cpu().numpy() - e.lse)) <= 1e-5
    if lq == 1 and lk == 1:
        assert float(r.a_cumul[0]) == 1.0  # test_attention.cpp:24-33


def test_attention_f32_errors(mkv):
    x = torch.zeros((8, 16), device="cuda")
    y = torch.zeros((4, 16), device="cuda")
    with pytest.raises(mkv.InvalidArgument):  # causal requires lq <= lk
        mkv.selective_flash_attn_f32(x, y, y, 0.1, True)
    with pytest.raises(mkv.InvalidArgument):
        mkv.decode_attention(torch.zeros(16, device="cuda"), torch.zeros((0, 16), device="cuda"),
                             torch.zeros((0, 16), device="cuda"), 1.0)
