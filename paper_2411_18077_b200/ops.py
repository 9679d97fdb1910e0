"""Host-side mirror of the reference operator interface for the hot path.

Same names, argument meaning and error behaviour as the reference C++ API in
``/root/reference/proj/core/include/minikv`` (attention.hpp, selection.hpp,
quantizer.hpp, cache_engine.hpp), batched for B200: tensors are torch CUDA
tensors (PyTorch is only the device-memory / stream plumbing), every compute
call goes through the C ABI (``include/minikv_b200.h``) to the sm_100a kernels.
There is no CPU fallback.

Reference error classes map to Python exceptions (``_capi``):
std::invalid_argument -> InvalidArgument (a ValueError), std::domain_error ->
DomainError, std::runtime_error -> RuntimeFailure, std::out_of_range -> OutOfRange.
"""
from __future__ import annotations

import ctypes as C
import os
import math
from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch

from . import _capi
from ._capi import check, lib


def _stream_ptr(stream: Optional[torch.cuda.Stream] = None) -> int:
    if stream is not None:
        return int(stream.cuda_stream)
    # the raw handle of the current stream without building a torch.cuda.Stream object (a few
    # us per call: it is on every decode call's host path)
    return _raw_stream(torch.cuda.current_device())


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None) or \
    (lambda dev: int(torch.cuda.current_stream(dev).cuda_stream))


def default_scale(d_head: int) -> float:
    """attention.hpp:26-28."""
    return float(1.0 / math.sqrt(float(d_head)))


# ---------------------------------------------------------------------------
# K1  selective_flash_attn  (attention.hpp:38-39)
# ---------------------------------------------------------------------------
@dataclass
class AttentionResult:
    output: torch.Tensor   # fp16 [B, Hq, Lq, d]
    lse: torch.Tensor      # fp32 [B, Hq, Lq]
    a_cumul: torch.Tensor  # fp32 [B, Hkv, Lk], summed over each kv-head's q-heads


def selective_flash_attn(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, scale: float,
                         causal: bool = True, tiles=None, stream=None) -> AttentionResult:
    """Two-pass selective flash attention -> (X_O, LSE, A_cumul).

    Mirrors ``selective_flash_attn(q, k, v, scale, causal, TileConfig)``
    (attention.cpp:29-117).  Accepts [L, d] (one head, as the reference) or
    [B, H, L, d].  ``tiles`` is accepted for signature parity and ignored: the
    device tiling is fixed by the kernel, and A_cumul's per-column accumulation
    order does not depend on it in the reference either (attention.cpp:101-115).
    """
    squeeze = q.dim() == 2
    if squeeze:
        q, k, v = q[None, None], k[None, None], v[None, None]
    if q.dim() != 4 or k.dim() != 4 or v.dim() != 4:
        raise _capi.InvalidArgument("attention: expected [B, H, L, d] tensors")
    B, Hq, Lq, d = q.shape
    _, Hkv, Lk, dk = k.shape
    if Lq == 0 or Lk == 0:
        raise _capi.InvalidArgument("attention: zero-length sequence")
    if dk != d:
        raise _capi.InvalidArgument("attention: q/k head dimension mismatch")
    if v.shape[2] != Lk:
        raise _capi.InvalidArgument("attention: k/v token count mismatch")
    if causal and Lq > Lk:
        raise _capi.InvalidArgument("attention: causal requires l_query <= l_key")
    for t in (q, k, v):
        if t.dtype != torch.float16 or not t.is_cuda or t.stride(-1) != 1:
            raise _capi.InvalidArgument("attention: fp16 CUDA tensors with unit channel stride")
    out = torch.empty((B, Hq, Lq, v.shape[3]), dtype=torch.float16, device=q.device)
    lse = torch.empty((B, Hq, Lq), dtype=torch.float32, device=q.device)
    ac = torch.empty((B, Hkv, Lk), dtype=torch.float32, device=q.device)
    a = _capi.PrefillArgs(
        q.data_ptr(), q.stride(0), q.stride(1), q.stride(2),
        k.data_ptr(), k.stride(0), k.stride(1), k.stride(2),
        v.data_ptr(), v.stride(0), v.stride(1), v.stride(2),
        out.data_ptr(), out.stride(0), out.stride(1), out.stride(2),
        lse.data_ptr(), ac.data_ptr(), B, Hq, Hkv, Lq, Lk, d, float(scale), int(bool(causal)))
    check(lib().mkv_prefill_attn(C.byref(a), _stream_ptr(stream)), "selective_flash_attn")
    if squeeze:
        return AttentionResult(out[0, 0], lse[0, 0], ac[0, 0])
    return AttentionResult(out, lse, ac)


# ---------------------------------------------------------------------------
# K2  selection  (selection.hpp:30-57)
# ---------------------------------------------------------------------------
def select_token_counts(a_cumul: torch.Tensor, hh_count, rw_count: int, stream=None):
    """Rectified top-k selection (selection.cpp:10-33) for one or many units.

    ``a_cumul`` is fp32 [L] or [n_units, L]; ``hh_count`` an int or one int per
    unit.  Returns (kept int32 [n_units, max_kept] on device, n_kept list), where
    row u holds sort(HH) ++ RW in its first n_kept[u] entries.
    """
    single = a_cumul.dim() == 1
    a2 = a_cumul[None] if single else a_cumul
    if a2.dtype != torch.float32 or not a2.is_cuda or a2.stride(-1) != 1:
        raise _capi.InvalidArgument("select: a_cumul must be an fp32 CUDA tensor")
    n, L = a2.shape
    hh = [int(hh_count)] * n if isinstance(hh_count, int) else [int(x) for x in hh_count]
    if rw_count < 0 or any(h < 0 for h in hh):
        raise _capi.InvalidArgument("select_tokens: negative budget")
    n_kept = [min(h + rw_count, L) for h in hh]
    kept = torch.empty((n, max(L, 1)), dtype=torch.int32, device=a2.device)
    hh_arr = (C.c_int32 * n)(*hh)
    args = _capi.SelectArgs(a2.data_ptr(), a2.stride(0), n, L, hh_arr, int(rw_count),
                            kept.data_ptr(), kept.stride(0), None)
    check(lib().mkv_select(C.byref(args), _stream_ptr(stream)), "select_token_counts")
    if single:
        return kept[0, :n_kept[0]], n_kept[0]
    return kept, n_kept


def select_tokens(a_cumul: torch.Tensor, alpha_hh: float, alpha_rw: float, l_prompt: int, stream=None):
    """selection.cpp:35-46: floor(alpha * l) counts."""
    if a_cumul.shape[-1] != l_prompt:
        raise _capi.InvalidArgument("select_tokens: a_cumul length != l_prompt")
    if alpha_hh < 0 or alpha_rw < 0:
        raise _capi.InvalidArgument("select_tokens: negative budget")
    hh = int(math.floor(alpha_hh * float(l_prompt)))
    rw = int(math.floor(alpha_rw * float(l_prompt)))
    n = 1 if a_cumul.dim() == 1 else a_cumul.shape[0]
    return select_token_counts(a_cumul, hh if a_cumul.dim() == 1 else [hh] * n, rw, stream)


def allocate_pyramid(mean_budget_x: int, layers: int, depth: int = 7, bottom_heavy: bool = True):
    """selection.cpp:61-83 (host arithmetic in the C ABI)."""
    out = (C.c_int64 * max(layers, 1))()
    check(lib().mkv_allocate_pyramid(mean_budget_x, layers, depth, int(bottom_heavy), out),
          "allocate_pyramid")
    return [int(x) for x in out[:layers]]


class VarianceMode:
    """selection.hpp VarianceMode: shares proportional (Prop) or inverse (Inv) to variance."""
    Prop = 0
    Inv = 1


def allocate_variance(per_layer_variance: Sequence[float], total_hh: int, mode: int = VarianceMode.Prop):
    """selection.cpp:85-128 (host arithmetic in the C ABI, bit-exact).  Returns
    (per_layer_hh, uniform_fallback)."""
    v = (C.c_float * max(len(per_layer_variance), 1))(*[float(x) for x in per_layer_variance])
    out = (C.c_int64 * max(len(per_layer_variance), 1))()
    fb = C.c_int(0)
    check(lib().mkv_allocate_variance(v, len(per_layer_variance), int(total_hh), int(mode), out, C.byref(fb)),
          "allocate_variance")
    return [int(x) for x in out[:len(per_layer_variance)]], bool(fb.value)


def layer_score_variance(a_cumul: torch.Tensor, stream=None) -> torch.Tensor:
    """selection.cpp:130-146 on the device: population variance of each row of an fp32
    CUDA tensor [L] or [n, L] (fp64 two-pass) -> fp32 tensor [] or [n]."""
    single = a_cumul.dim() == 1
    a2 = a_cumul[None] if single else a_cumul
    if a2.dtype != torch.float32 or not a2.is_cuda or a2.stride(-1) != 1:
        raise _capi.InvalidArgument("layer_score_variance: a_cumul must be an fp32 CUDA tensor")
    n, L = a2.shape
    out = torch.empty(n, dtype=torch.float32, device=a2.device)
    check(lib().mkv_score_variance(a2.data_ptr(), a2.stride(0), n, L, out.data_ptr(), _stream_ptr(stream)),
          "layer_score_variance")
    return out[0] if single else out


def allocate_uniform(total_hh: int, layers: int):
    """selection.cpp:48-59."""
    out = (C.c_int64 * max(layers, 1))()
    check(lib().mkv_allocate_uniform(total_hh, layers, out), "allocate_uniform")
    return [int(x) for x in out[:layers]]


# ---------------------------------------------------------------------------
# H2O comparison baseline + persistence (harness.hpp:33-52, harness.cpp:83-169)
# ---------------------------------------------------------------------------
@dataclass
class H2OBaselineTrace:
    """harness.hpp:35-38: kept_per_step[0] is the post-prefill set, one entry per decode step
    follows; each entry is the ascending list of original token positions kept."""
    kept_per_step: List[List[int]]


@dataclass
class PersistenceReport:
    """harness.hpp:45-48."""
    fractions: List[float]
    final_fraction: float


def h2o_dynamic_baseline(prompt_k: torch.Tensor, prompt_scores: torch.Tensor, decode_qs: torch.Tensor,
                         decode_ks: torch.Tensor, hh_budget: int, rw_budget: int, scale: float,
                         stream=None) -> H2OBaselineTrace:
    """h2o_dynamic_baseline (harness.cpp:108-150) on the device: fp32 CUDA tensors prompt_k
    [L, d], prompt_scores [L], decode_qs / decode_ks [steps, d].  Kept sets are bit-identical to
    the reference (same arithmetic order, see csrc/h2o.cu)."""
    L = prompt_k.shape[0]
    d = prompt_k.shape[1] if prompt_k.dim() == 2 else decode_qs.shape[-1]
    if prompt_scores.numel() != L:
        raise _capi.InvalidArgument("h2o_dynamic_baseline: prompt score length mismatch")
    if decode_qs.shape[0] != decode_ks.shape[0]:
        raise _capi.InvalidArgument("h2o_dynamic_baseline: decode stream length mismatch")
    steps = decode_qs.shape[0]
    if steps and (decode_qs.shape[1] != d or decode_ks.shape[1] != d):
        raise _capi.InvalidArgument("append_row: width mismatch")
    for t in (prompt_k, prompt_scores, decode_qs, decode_ks):
        if t.numel() and (t.dtype != torch.float32 or not t.is_cuda or t.stride(-1) != 1):
            raise _capi.InvalidArgument("h2o_dynamic_baseline: fp32 CUDA tensors with unit stride expected")
    qs, ks = decode_qs.contiguous(), decode_ks.contiguous()
    stride = max(1, min(L + steps, hh_budget + rw_budget))
    kept = torch.empty((steps + 1, stride), dtype=torch.int32, device=prompt_scores.device)
    count = torch.empty(steps + 1, dtype=torch.int32, device=prompt_scores.device)
    args = _capi.H2OArgs(prompt_k.data_ptr() if L else None, prompt_k.stride(0) if L else d,
                         prompt_scores.data_ptr() if L else None, qs.data_ptr() if steps else None,
                         ks.data_ptr() if steps else None, L, d, steps, int(hh_budget), int(rw_budget),
                         float(scale), kept.data_ptr(), stride, count.data_ptr())
    check(lib().mkv_h2o_dynamic_baseline(C.byref(args), _stream_ptr(stream)), "h2o_dynamic_baseline")
    kh, ch = kept.cpu().tolist(), count.cpu().tolist()
    return H2OBaselineTrace([kh[s][:ch[s]] for s in range(steps + 1)])


def persistence_analysis(trace: H2OBaselineTrace, prefill_hh: Sequence[int]) -> PersistenceReport:
    """persistence_analysis (harness.cpp:152-169): per trace entry, the fraction of the prefill
    heavy hitters still kept (host arithmetic on the device-produced kept sets)."""
    if len(prefill_hh) == 0:
        raise _capi.RuntimeFailure("persistence_analysis: empty prefill heavy-hitter set")
    import bisect

    import numpy as np
    fr = []
    for kept in trace.kept_per_step:
        hit = 0
        for idx in prefill_hh:
            j = bisect.bisect_left(kept, idx)
            hit += 1 if j < len(kept) and kept[j] == idx else 0
        fr.append(float(np.float32(hit) / np.float32(len(prefill_hh))))  # float / float as the reference
    return PersistenceReport(fr, fr[-1])


# ---------------------------------------------------------------------------
# Device cache  (cache_engine.hpp:19-67)
# ---------------------------------------------------------------------------
class KVCache:
    """n_units independent KVCacheLayer's (one per (seq, layer, kv-head)).

    Mirrors make_cache / prefill / decode_append / decode_step
    (cache_engine.cpp:9-138) batched over units; unit order is the caller's
    (the bench uses u = (layer * B + b) * Hkv + h, so one layer is a
    contiguous unit range).
    """

    def __init__(self, n_units: int, prefill_capacity: Sequence[int] | int, max_decode_tokens: int,
                 d: int = 128, n_r: int = 128, group_size: int = 16, keep_fp32_params: bool = False):
        caps = [int(prefill_capacity)] * n_units if isinstance(prefill_capacity, int) else \
            [int(x) for x in prefill_capacity]
        self._caps = (C.c_int32 * n_units)(*caps)
        cfg = _capi.CacheConfig(n_units, d, n_r, group_size, self._caps, int(max_decode_tokens),
                                int(bool(keep_fp32_params)))
        h = C.c_void_p()
        check(lib().mkv_cache_create(C.byref(cfg), C.byref(h)), "make_cache")
        self.h = h
        self.n_units, self.d, self.n_r, self.group_size = n_units, d, n_r, group_size

    def close(self):
        if getattr(self, "h", None):
            lib().mkv_cache_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # prefill: select -> gather -> quantize (cache_engine.cpp:56-77)
    def prefill(self, k: torch.Tensor, v: torch.Tensor, a_cumul: torch.Tensor, hh_count, rw_count: int,
                unit_begin: int = 0, stream=None):
        """k, v fp16 [n, L, d]; a_cumul fp32 [n, L]; hh_count int or per-unit list."""
        if k.dim() == 2:
            k, v, a_cumul = k[None], v[None], a_cumul[None]
        n, L, d = k.shape
        if v.shape != k.shape or a_cumul.shape != (n, L):
            raise _capi.InvalidArgument("prefill: k/v/a_cumul length mismatch")
        hh = [int(hh_count)] * n if isinstance(hh_count, int) else [int(x) for x in hh_count]
        hh_arr = (C.c_int32 * n)(*hh)
        args = _capi.PrefillSelectArgs(unit_begin, n, L, a_cumul.data_ptr(), a_cumul.stride(0), hh_arr,
                                       int(rw_count), k.data_ptr(), k.stride(0), k.stride(1),
                                       v.data_ptr(), v.stride(0), v.stride(1))
        check(lib().mkv_cache_prefill_select(self.h, C.byref(args), _stream_ptr(stream)), "prefill")

    def prefill_kept(self, k: torch.Tensor, v: torch.Tensor, kept: torch.Tensor, n_kept: Sequence[int],
                     unit_begin: int = 0, stream=None):
        """Quantize already-selected tokens (kept int32 [n, >= n_kept], ascending)."""
        n = k.shape[0]
        nk = (C.c_int32 * n)(*[int(x) for x in n_kept])
        args = _capi.CachePrefillArgs(unit_begin, n, k.data_ptr(), k.stride(0), k.stride(1),
                                      v.data_ptr(), v.stride(0), v.stride(1), kept.data_ptr(),
                                      kept.stride(0), nk)
        check(lib().mkv_cache_prefill(self.h, C.byref(args), _stream_ptr(stream)), "prefill")

    def decode_step(self, q: torch.Tensor, k_new: Optional[torch.Tensor], v_new: Optional[torch.Tensor],
                    scale: float, unit_begin: int = 0, out: Optional[torch.Tensor] = None, stream=None):
        """q fp16 [n, G, d]; k_new/v_new fp16 [n, d] (None: attend without append)."""
        n, G, d = q.shape
        if out is None:
            out = torch.empty_like(q)
        args = _capi.DecodeArgs(unit_begin, n, G, q.data_ptr(),
                                k_new.data_ptr() if k_new is not None else None,
                                v_new.data_ptr() if v_new is not None else None,
                                out.data_ptr(), float(scale))
        check(lib().mkv_decode_step(self.h, C.byref(args), _stream_ptr(stream)), "decode_step")
        return out

    def decode_step_layers(self, q: torch.Tensor, k_new: Optional[torch.Tensor], v_new: Optional[torch.Tensor],
                           scale: float, unit_begin: int = 0, out: Optional[torch.Tensor] = None, stream=None):
        """All layers of one decode step in one call: q fp16 [L, n, G, d], k_new/v_new fp16 [L, n, d]
        (None: attend only); layer l owns units unit_begin + l*n .. + n.  Every q must be written
        before the call.  Layers laid out back to back (contiguous q / out / k_new / v_new) are
        one pass over all L * n units; otherwise layers after the first start their page pass
        while the previous layer's finish kernel is still merging (mkv_decode_step_layers)."""
        L, n, G, d = q.shape
        if out is None:
            out = torch.empty_like(q)
        args = (_capi.DecodeArgs * L)()
        for l in range(L):
            args[l] = _capi.DecodeArgs(unit_begin + l * n, n, G, q[l].data_ptr(),
                                       k_new[l].data_ptr() if k_new is not None else None,
                                       v_new[l].data_ptr() if v_new is not None else None,
                                       out[l].data_ptr(), float(scale))
        check(lib().mkv_decode_step_layers(self.h, L, args, _stream_ptr(stream)), "decode_step_layers")
        return out

    def decode_steps(self, q: torch.Tensor, k_new: Optional[torch.Tensor], v_new: Optional[torch.Tensor],
                     scale: float, unit_begin: int = 0, out: Optional[torch.Tensor] = None, stream=None):
        """S consecutive decode steps over a prepared token stream in one call (mkv_decode_steps):
        q fp16 [S, n, G, d], k_new / v_new fp16 [S, n, d] (None: attend only); out [S, n, G, d].
        Few short units run as one launch (a cluster of CTAs per unit for all S steps): the cache state is
        that of S decode_step calls bit for bit, outputs equal them up to fp32 accumulation
        order; other calls run the per-step kernels (bit-identical; MKV_STEPS=off forces them)."""
        S, n, G, d = q.shape
        if out is None:
            out = torch.empty_like(q)
        for t in (q, out) + ((k_new, v_new) if k_new is not None else ()):
            if not t[0].is_contiguous():
                raise _capi.InvalidArgument("decode_steps: each step's slice must be contiguous")
        args = _capi.DecodeStepsArgs(unit_begin, n, G, S, q.data_ptr(), q.stride(0),
                                     k_new.data_ptr() if k_new is not None else None,
                                     v_new.data_ptr() if v_new is not None else None,
                                     k_new.stride(0) if k_new is not None else 0,
                                     out.data_ptr(), out.stride(0), float(scale))
        if k_new is not None and v_new.stride(0) != k_new.stride(0):
            raise _capi.InvalidArgument("decode_steps: k_new / v_new step strides differ")
        check(lib().mkv_decode_steps(self.h, C.byref(args), _stream_ptr(stream)), "decode_steps")
        return out

    def append(self, k_new: torch.Tensor, v_new: torch.Tensor, unit_begin: int = 0, stream=None):
        """decode_append (cache_engine.cpp:79-90)."""
        check(lib().mkv_cache_append(self.h, unit_begin, k_new.shape[0], k_new.data_ptr(), v_new.data_ptr(),
                                     _stream_ptr(stream)), "decode_append")

    def check(self):
        """Synchronise and surface device-side faults (non-finite quantizer input)."""
        check(lib().mkv_cache_check(self.h), "cache")

    def unit_info(self, unit: int):
        vals = [C.c_int64() for _ in range(4)]
        check(lib().mkv_cache_unit_info(self.h, unit, *[C.byref(x) for x in vals]), "unit_info")
        tq, tr, npg, nb = (int(x.value) for x in vals)
        return {"tokens_quantized": tq, "tokens_residual": tr, "n_pages": npg, "n_blocks": nb}

    def bytes(self):
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib().mkv_cache_bytes(self.h, C.byref(a), C.byref(b), C.byref(c)), "bytes")
        return {"pages": a.value, "residual": b.value, "total": c.value}

    def export_reference(self, unit: int, which: int):
        """(packed_words u32, params f32 [n, 2], block_rows) as quantizer.hpp:30-42."""
        import numpy as np
        nw, npar, nb = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().mkv_cache_export_sizes(self.h, unit, which, C.byref(nw), C.byref(npar), C.byref(nb)),
              "export")
        words = np.zeros(max(nw.value, 1), np.uint32)
        params = np.zeros(max(2 * npar.value, 2), np.float32)
        br = np.zeros(max(nb.value, 1), np.int64)
        check(lib().mkv_cache_export_reference(self.h, unit, which, words.ctypes.data, params.ctypes.data,
                                               br.ctypes.data), "export")
        return words[:nw.value], params[:2 * npar.value].reshape(-1, 2), br[:nb.value]

    def save_mkvc(self, unit: int, path: str):
        """save_cache (snapshot.cpp:71-198): the unit as a reference MKVC v1 file."""
        check(lib().mkv_cache_save_mkvc(self.h, unit, os.fsencode(path)), "save_cache")

    def load_mkvc(self, unit: int, path: str):
        """load_cache (snapshot.cpp:159-198) into unit `unit` (pages rebuilt on the device)."""
        check(lib().mkv_cache_load_mkvc(self.h, unit, os.fsencode(path)), "load_cache")

    def export_residual(self, unit: int):
        import numpy as np
        info = self.unit_info(unit)
        n = info["tokens_residual"]
        rk = np.zeros((max(n, 1), self.d), np.uint16)
        rv = np.zeros((max(n, 1), self.d), np.uint16)
        check(lib().mkv_cache_export_residual(self.h, unit, rk.ctypes.data, rv.ctypes.data), "export")
        return rk[:n].view(np.float16), rv[:n].view(np.float16)


# ---------------------------------------------------------------------------
# synthetic inputs (bit-identical to oracle/minikv_oracle.c's generator)
# ---------------------------------------------------------------------------
def synth_fp16(shape, seed: int, stream_base: int, stream_step: int = 1, device="cuda", stream=None):
    """fp16 tensor; row r of the flattened [rows, shape[-1]] view uses stream
    stream_base + r * stream_step."""
    t = torch.empty(shape, dtype=torch.float16, device=device)
    row_len = shape[-1]
    rows = t.numel() // row_len if row_len else 0
    check(lib().mkv_synth_fp16_rows(t.data_ptr(), rows, row_len, row_len, seed, stream_base, stream_step,
                                    _stream_ptr(stream)), "synth")
    return t


def synth_uniform(shape, seed: int, stream_base: int, stream_step: int = 1, device="cuda", stream=None):
    t = torch.empty(shape, dtype=torch.float32, device=device)
    row_len = shape[-1]
    rows = t.numel() // row_len if row_len else 0
    check(lib().mkv_synth_uniform_f32(t.data_ptr(), rows, row_len, row_len, seed, stream_base, stream_step,
                                      _stream_ptr(stream)), "synth")
    return t


# ---------------------------------------------------------------------------
# exact-fp32 reference-format entries (refmt.cu): any head dim / group size
# ---------------------------------------------------------------------------
def _f32_cuda(x: torch.Tensor, what: str) -> torch.Tensor:
    if x.dtype != torch.float32 or not x.is_cuda:
        raise _capi.InvalidArgument(f"{what}: fp32 CUDA tensor expected")
    return x.contiguous()


def selective_flash_attn_f32(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, scale: float, causal: bool = True,
                             stream=None) -> AttentionResult:
    """selective_flash_attn (attention.cpp:29-117) on fp32 [L, d] matrices, any d, in the
    reference's dot-product / A_cumul accumulation order (mkv_attention_f32)."""
    q, k, v = _f32_cuda(q, "attention"), _f32_cuda(k, "attention"), _f32_cuda(v, "attention")
    lq, d = q.shape
    lk, dv = v.shape
    out = torch.empty((lq, dv), dtype=torch.float32, device=q.device)
    lse = torch.empty(lq, dtype=torch.float32, device=q.device)
    ac = torch.empty(lk, dtype=torch.float32, device=q.device)
    a = _capi.AttnF32Args(q.data_ptr(), d, k.data_ptr(), k.shape[1], v.data_ptr(), dv, out.data_ptr(), dv,
                          lse.data_ptr(), ac.data_ptr(), lq, lk, k.shape[1] if k.shape[1] == d else -1, dv,
                          float(scale), int(bool(causal)))
    check(lib().mkv_attention_f32(C.byref(a), _stream_ptr(stream)), "selective_flash_attn_f32")
    return AttentionResult(out, lse, ac)


def decode_attention(q: torch.Tensor, keys: torch.Tensor, values: torch.Tensor, scale: float, stream=None):
    """decode_attention (attention.cpp:119-143): (output row [dv], attention row [n]) on fp32."""
    q, keys, values = _f32_cuda(q, "decode_attention"), _f32_cuda(keys, "decode_attention"), \
        _f32_cuda(values, "decode_attention")
    n, d = keys.shape
    dv = values.shape[1]
    if q.numel() != d:
        raise _capi.InvalidArgument("decode_attention: query dimension mismatch")
    out = torch.empty(dv, dtype=torch.float32, device=q.device)
    attn = torch.empty(max(n, 1), dtype=torch.float32, device=q.device)
    check(lib().mkv_decode_attention_f32(q.data_ptr(), keys.data_ptr(), d, values.data_ptr(), dv, n, d, dv,
                                         float(scale), out.data_ptr(), attn.data_ptr(), _stream_ptr(stream)),
          "decode_attention")
    return out, attn[:n]


def quantize_block(block: torch.Tensor, axis: int, group_size: int = 16, code_offset: int = 0, first_word: int = 0,
                   row_idx: Optional[torch.Tensor] = None, stream=None):
    """append_block / quantize_matrix (quantizer.cpp:102-151) of an fp32 [rows, cols] block (rows
    gathered through int32 row_idx when given): (words int32-viewed u32 covering stream words
    [code_offset // 16, ...), params fp32 [n_groups, 2]).  axis 0 PerChannel, 1 PerToken."""
    block = _f32_cuda(block, "quantize")
    rows = row_idx.numel() if row_idx is not None else block.shape[0]
    cols = block.shape[1]
    n = rows * cols
    nw = (code_offset + n + 15) // 16 - code_offset // 16
    per = (rows + group_size - 1) // group_size if axis == 0 else (cols + group_size - 1) // group_size
    ng = (cols if axis == 0 else rows) * per
    words = torch.empty(max(nw, 1), dtype=torch.int32, device=block.device)
    params = torch.empty((max(ng, 1), 2), dtype=torch.float32, device=block.device)
    check(lib().mkv_quantize_block_f32(block.data_ptr(), cols, row_idx.data_ptr() if row_idx is not None else None,
                                       rows, cols, group_size, axis, code_offset, first_word & 0xFFFFFFFF,
                                       words.data_ptr(), params.data_ptr(), _stream_ptr(stream)), "quantize_block")
    return words[:nw], params[:ng]


def dequantize(words: torch.Tensor, params: torch.Tensor, block_rows: Sequence[int], cols: int, axis: int,
               group_size: int = 16, stream=None) -> torch.Tensor:
    """dequantize_matrix (quantizer.cpp:153-195) of a device stream -> fp32 [sum(block_rows), cols]."""
    rows = int(sum(block_rows))
    out = torch.empty((rows, cols), dtype=torch.float32, device=words.device)
    br = (C.c_int64 * max(len(block_rows), 1))(*[int(r) for r in block_rows])
    check(lib().mkv_dequantize_f32(words.data_ptr(), params.data_ptr(), br, len(block_rows), cols, group_size, axis,
                                   out.data_ptr(), cols, _stream_ptr(stream)), "dequantize_matrix")
    return out
