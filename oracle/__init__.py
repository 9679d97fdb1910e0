"""CPU parity oracle for the MiniKV attention hot path -- TEST INFRASTRUCTURE ONLY.

Two interchangeable backends with one numpy API:

* ``port()``  -- ``oracle/liboracle.so``, the plain-C restatement in
  ``minikv_oracle.c`` (each function cites the reference file:line it follows).
* ``ref()``   -- ``oracle/_ref/libminikv_ref.so``, the unmodified reference
  sources compiled in place by ``oracle/Makefile`` (only buildable where
  ``/root/reference`` exists; the built .so travels to the GPU box).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package.  The product package
``paper_2411_18077_b200`` never does.

Status codes map to the reference's exception classes.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libminikv_ref.so")

STATUS = {1: ValueError, 2: ArithmeticError, 3: RuntimeError, 4: IndexError}
STATUS_NAME = {1: "std::invalid_argument", 2: "std::domain_error", 3: "std::runtime_error",
               4: "std::out_of_range"}

# Synthetic stream ids: kind << 48 | unit << 16 | step.
KIND_Q, KIND_K, KIND_V, KIND_QDEC, KIND_KDEC, KIND_VDEC, KIND_ACUMUL = 1, 2, 3, 4, 5, 6, 7


def stream_id(kind: int, unit: int, step: int = 0) -> int:
    return (kind << 48) | (unit << 16) | step


class OracleError(Exception):
    pass


def _check(st: int, what: str):
    if st:
        exc = STATUS.get(st, OracleError)
        raise exc(f"{what}: {STATUS_NAME.get(st, 'error')} (status {st})")


_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_sz = C.c_size_t


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


@dataclass
class AttnResult:
    output: np.ndarray
    lse: np.ndarray
    a_cumul: np.ndarray
    aux_elements: int


class _Lib:
    """Common numpy API over either backend; prefix 'mko_' (port) or 'mkr_' (ref)."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library not built: {path} (run make -C oracle)")
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.path = path
        L, p = self.lib, prefix
        fa = getattr(L, p + "selective_flash_attn")
        fa.argtypes = [_f32p, _f32p, _f32p, _sz, _sz, _sz, _sz, C.c_float, C.c_int, _sz, _sz,
                       _f32p, _f32p, _f32p, C.POINTER(_sz)]
        da = getattr(L, p + "decode_attention")
        da.argtypes = [_f32p, _f32p, _f32p, _sz, _sz, _sz, C.c_float, _f32p, _f32p]
        qg = getattr(L, p + "quantize_group")
        qg.argtypes = [_f32p, _sz, _u8p, C.POINTER(C.c_float), C.POINTER(C.c_float)]
        pc = getattr(L, p + "pack_codes")
        pc.argtypes = [_u8p, _sz, _u32p]
        sel = getattr(L, p + "select_token_counts")
        if prefix == "mko_":
            sel.argtypes = [_f32p, _sz, _sz, _sz, _i64p, C.POINTER(_sz), C.c_void_p, C.c_void_p,
                            C.c_void_p, C.c_void_p, C.POINTER(C.c_int)]
        else:
            sel.argtypes = [_f32p, _sz, _sz, _sz, _i64p, C.POINTER(_sz), C.POINTER(C.c_int)]
        ap = getattr(L, p + "allocate_pyramid")
        ap.argtypes = [_sz, _sz, _sz, C.c_int, _i64p]
        au = getattr(L, p + "allocate_uniform")
        au.argtypes = [_sz, _sz, _i64p]
        av = getattr(L, p + "allocate_variance")
        av.argtypes = [_f32p, _sz, _sz, C.c_int, _i64p, C.POINTER(C.c_int)]
        lv = getattr(L, p + "layer_score_variance")
        lv.argtypes = [_f32p, _sz, C.POINTER(C.c_float)]
        h2 = getattr(L, p + "h2o_dynamic_baseline")
        h2.argtypes = [_f32p, _sz, _sz, _f32p, _f32p, _f32p, _sz, _sz, _sz, C.c_float,
                       np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS"), _sz,
                       np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")]

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)

    # attention.cpp:29-117
    def selective_flash_attn(self, q, k, v, scale, causal, block_m=64, block_n=64) -> AttnResult:
        q, k, v = _f32(q), _f32(k), _f32(v)
        lq, d = q.shape
        lk, dv = v.shape
        if k.shape[0] != lk or k.shape[1] != d:
            raise ValueError("shape mismatch")
        out = np.zeros((lq, dv), np.float32)
        lse = np.zeros(lq, np.float32)
        ac = np.zeros(lk, np.float32)
        aux = _sz(0)
        _check(self.fn("selective_flash_attn")(q, k, v, lq, lk, d, dv, scale, int(causal), block_m,
                                               block_n, out, lse, ac, C.byref(aux)),
               "selective_flash_attn")
        return AttnResult(out, lse, ac, aux.value)

    # attention.cpp:119-143
    def decode_attention(self, q, keys, values, scale):
        q, keys, values = _f32(q), _f32(keys), _f32(values)
        n, d = keys.shape
        dv = values.shape[1]
        out = np.zeros(dv, np.float32)
        attn = np.zeros(max(n, 1), np.float32)
        _check(self.fn("decode_attention")(q, keys, values, n, d, dv, scale, out, attn),
               "decode_attention")
        return out, attn[:n]

    # quantizer.cpp:28-53
    def quantize_group(self, values):
        values = _f32(values)
        codes = np.zeros(max(len(values), 1), np.uint8)
        sc, zp = C.c_float(), C.c_float()
        _check(self.fn("quantize_group")(values, len(values), codes, C.byref(sc), C.byref(zp)),
               "quantize_group")
        return codes[:len(values)], np.float32(sc.value), np.float32(zp.value)

    # quantizer.cpp:67-77
    def pack_codes(self, codes):
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        words = np.zeros(max((len(codes) + 15) // 16, 1), np.uint32)
        _check(self.fn("pack_codes")(codes, len(codes), words), "pack_codes")
        return words[:(len(codes) + 15) // 16]

    # selection.cpp:10-33
    def select_token_counts(self, a_cumul, hh, rw):
        a = _f32(a_cumul)
        kept = np.zeros(max(len(a), 1), np.int64)
        nk = _sz(0)
        cl = C.c_int(0)
        if self.prefix == "mko_":
            st = self.fn("select_token_counts")(a, len(a), hh, rw, kept, C.byref(nk), None, None,
                                                 None, None, C.byref(cl))
        else:
            st = self.fn("select_token_counts")(a, len(a), hh, rw, kept, C.byref(nk), C.byref(cl))
        _check(st, "select_token_counts")
        return kept[:nk.value].copy(), bool(cl.value)

    # selection.cpp:61-83
    def allocate_pyramid(self, x, layers, depth=7, bottom_heavy=True):
        out = np.zeros(max(layers, 1), np.int64)
        _check(self.fn("allocate_pyramid")(x, layers, depth, int(bottom_heavy), out),
               "allocate_pyramid")
        return out[:layers]

    # selection.cpp:85-128 (inverse: VarianceMode::Inv)
    def allocate_variance(self, variances, total, inverse=False):
        v = _f32(np.asarray(variances, np.float32))
        out = np.zeros(max(len(v), 1), np.int64)
        fb = C.c_int(0)
        _check(self.fn("allocate_variance")(v, len(v), total, int(inverse), out, C.byref(fb)), "allocate_variance")
        return out[:len(v)], bool(fb.value)

    # selection.cpp:130-146
    def layer_score_variance(self, a):
        a = _f32(np.asarray(a, np.float32))
        r = C.c_float(0)
        _check(self.fn("layer_score_variance")(a, len(a), C.byref(r)), "layer_score_variance")
        return r.value

    # harness.cpp:108-150 -> list of kept position lists (post-prefill set first)
    def h2o_dynamic_baseline(self, prompt_k, prompt_scores, qs, ks, hh, rw, scale):
        pk, sc = _f32(prompt_k), _f32(np.asarray(prompt_scores, np.float32))
        qs, ks = _f32(qs), _f32(ks)
        l, d = pk.shape
        steps = qs.shape[0]
        stride = max(1, min(l + steps, hh + rw))
        kept = np.zeros((steps + 1) * stride, np.int32)
        cnt = np.zeros(steps + 1, np.int32)
        _check(self.fn("h2o_dynamic_baseline")(pk, l, d, sc, qs.reshape(-1) if steps else np.zeros(1, np.float32),
                                               ks.reshape(-1) if steps else np.zeros(1, np.float32), steps, hh, rw,
                                               scale, kept, stride, cnt), "h2o_dynamic_baseline")
        kept = kept.reshape(steps + 1, stride)
        return [kept[s, :cnt[s]].tolist() for s in range(steps + 1)]

    # selection.cpp:48-59
    def allocate_uniform(self, total, layers):
        out = np.zeros(max(layers, 1), np.int64)
        _check(self.fn("allocate_uniform")(total, layers, out), "allocate_uniform")
        return out[:layers]


class PortOracle(_Lib):
    """The C restatement (minikv_oracle.c)."""

    def __init__(self):
        super().__init__(PORT_SO, "mko_")
        L = self.lib
        L.mko_quantize_block.argtypes = [_f32p, _sz, _sz, C.c_int, _sz, _u8p, _f32p, C.POINTER(_sz)]
        L.mko_dequantize_block.argtypes = [_u8p, _f32p, _sz, _sz, C.c_int, _sz, C.c_int, _f32p]
        L.mko_cache_create.argtypes = [_sz, _sz, _sz, C.POINTER(C.c_void_p)]
        L.mko_cache_destroy.argtypes = [C.c_void_p]
        L.mko_cache_prefill.argtypes = [C.c_void_p, _f32p, _f32p, _f32p, _sz, _sz, _sz]
        L.mko_cache_append.argtypes = [C.c_void_p, _f32p, _f32p]
        L.mko_cache_decode_step.argtypes = [C.c_void_p, _f32p, _f32p, _f32p, C.c_float, C.c_int, _f32p]
        L.mko_cache_attend.argtypes = [C.c_void_p, _f32p, C.c_float, C.c_int, _f32p]
        for n in ("tokens_quantized", "tokens_residual", "n_blocks"):
            f = getattr(L, "mko_cache_" + n)
            f.argtypes = [C.c_void_p]
            f.restype = _sz
        for n in ("total_codes", "n_params"):
            f = getattr(L, "mko_cache_" + n)
            f.argtypes = [C.c_void_p, C.c_int]
            f.restype = _sz
        L.mko_cache_export.argtypes = [C.c_void_p, C.c_int, _u32p, _f32p, _i64p]
        L.mko_cache_residual.argtypes = [C.c_void_p, _f32p, _f32p]
        L.mko_synth_fp16.argtypes = [C.c_uint64, C.c_uint64, _sz, _u16p]
        L.mko_synth_mix.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.mko_synth_mix.restype = C.c_uint64
        L.mko_round_fp16.argtypes = [C.c_float]
        L.mko_round_fp16.restype = C.c_float

    # append_block (quantizer.cpp:102-136) for one block: stream-order codes + params.
    def quantize_block(self, block, axis, group_size=16):
        block = _f32(block)
        rows, cols = block.shape
        codes = np.zeros(max(rows * cols, 1), np.uint8)
        ng_max = (cols * ((rows + group_size - 1) // group_size) if axis == 0
                  else rows * ((cols + group_size - 1) // group_size))
        params = np.zeros(max(2 * ng_max, 2), np.float32)
        ng = _sz(0)
        _check(self.lib.mko_quantize_block(block, rows, cols, axis, group_size, codes, params,
                                           C.byref(ng)), "quantize_block")
        return codes[:rows * cols], params[:2 * ng.value].reshape(-1, 2)

    def dequantize_block(self, codes, params, rows, cols, axis, group_size=16, param_fp16=False):
        out = np.zeros((rows, cols), np.float32)
        _check(self.lib.mko_dequantize_block(np.ascontiguousarray(codes, np.uint8),
                                             _f32(params).reshape(-1), rows, cols, axis,
                                             group_size, int(param_fp16), out), "dequantize_block")
        return out

    def synth_fp16(self, seed: int, stream: int, n: int) -> np.ndarray:
        """Synthetic approx-N(0,1) fp16 values (as np.float16)."""
        out = np.zeros(max(n, 1), np.uint16)
        self.lib.mko_synth_fp16(seed, stream, n, out)
        return out[:n].view(np.float16)

    def synth_uniform(self, seed: int, stream: int, n: int) -> np.ndarray:
        """Synthetic uniform [0,1) fp32 values (the a_cumul stand-in)."""
        mix = np.array([self.lib.mko_synth_mix(seed, stream, i) for i in range(n)], np.uint64)
        return ((mix >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0))

    def cache(self, d=128, n_r=128, group_size=16) -> "OracleCache":
        return OracleCache(self, d, n_r, group_size)


class OracleCache:
    """One (seq, layer, kv-head) KVCacheLayer (cache_engine.cpp) on the C port."""

    def __init__(self, port: PortOracle, d, n_r, gs):
        self.port, self.d, self.n_r, self.gs = port, d, n_r, gs
        h = C.c_void_p()
        _check(port.lib.mko_cache_create(d, n_r, gs, C.byref(h)), "make_cache")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.port.lib.mko_cache_destroy(self.h)
            self.h = None

    def prefill(self, k, v, a_cumul, hh, rw):
        k, v, a = _f32(k), _f32(v), _f32(a_cumul)
        _check(self.port.lib.mko_cache_prefill(self.h, k, v, a, len(a), hh, rw), "prefill")

    def append(self, tk, tv):
        _check(self.port.lib.mko_cache_append(self.h, _f32(tk), _f32(tv)), "decode_append")

    def decode_step(self, tq, tk, tv, scale, param_fp16=False):
        out = np.zeros(self.d, np.float32)
        _check(self.port.lib.mko_cache_decode_step(self.h, _f32(tq), _f32(tk), _f32(tv), scale,
                                                   int(param_fp16), out), "decode_step")
        return out

    def attend(self, tq, scale, param_fp16=False):
        out = np.zeros(self.d, np.float32)
        _check(self.port.lib.mko_cache_attend(self.h, _f32(tq), scale, int(param_fp16), out),
               "attend")
        return out

    @property
    def tokens_quantized(self):
        return self.port.lib.mko_cache_tokens_quantized(self.h)

    @property
    def tokens_residual(self):
        return self.port.lib.mko_cache_tokens_residual(self.h)

    def export(self, which: int):
        """Reference QuantizedTensor view: (packed_words, params[n,2], block_rows)."""
        L = self.port.lib
        nc = L.mko_cache_total_codes(self.h, which)
        npar = L.mko_cache_n_params(self.h, which)
        nb = L.mko_cache_n_blocks(self.h)
        words = np.zeros(max((nc + 15) // 16, 1), np.uint32)
        params = np.zeros(max(2 * npar, 2), np.float32)
        br = np.zeros(max(nb, 1), np.int64)
        L.mko_cache_export(self.h, which, words, params, br)
        return words[:(nc + 15) // 16], params[:2 * npar].reshape(-1, 2), br[:nb]

    def residual(self):
        n = self.tokens_residual
        rk = np.zeros((max(n, 1), self.d), np.float32)
        rv = np.zeros((max(n, 1), self.d), np.float32)
        self.port.lib.mko_cache_residual(self.h, rk, rv)
        return rk[:n], rv[:n]


class RefOracle(_Lib):
    """The unmodified reference, compiled in place (oracle/_ref/libminikv_ref.so)."""

    def __init__(self):
        super().__init__(REF_SO, "mkr_")
        L = self.lib
        L.mkr_quantize_matrix.argtypes = [_f32p, _sz, _sz, C.c_int, _sz, _u32p, C.POINTER(_sz),
                                          _f32p, C.POINTER(_sz)]
        L.mkr_quant_dequant_matrix.argtypes = [_f32p, _sz, _sz, C.c_int, _sz, _f32p]
        L.mkr_cache_prefill.argtypes = [_f32p, _f32p, _f32p, _sz, _sz, _sz, _sz, _sz, _sz,
                                        C.POINTER(C.c_void_p)]
        L.mkr_cache_destroy.argtypes = [C.c_void_p]
        L.mkr_cache_append.argtypes = [C.c_void_p, _f32p, _f32p]
        L.mkr_cache_decode_step.argtypes = [C.c_void_p, _f32p, _f32p, _f32p, C.c_float, _f32p]
        for n in ("tokens_quantized", "tokens_residual", "n_blocks"):
            f = getattr(L, "mkr_cache_" + n)
            f.argtypes = [C.c_void_p]
            f.restype = _sz
        for n in ("n_words", "n_params"):
            f = getattr(L, "mkr_cache_" + n)
            f.argtypes = [C.c_void_p, C.c_int]
            f.restype = _sz
        L.mkr_cache_export.argtypes = [C.c_void_p, C.c_int, _u32p, _f32p, _i64p]
        L.mkr_cache_save.argtypes = [C.c_void_p, C.c_char_p]
        L.mkr_cache_load.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.mkr_decode_set_create.argtypes = [_sz, _sz, _sz, _sz, _i64p, _sz, _sz, _sz, C.c_uint64,
                                            np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS"),
                                            C.c_int, C.POINTER(C.c_void_p)]
        L.mkr_decode_set_destroy.argtypes = [C.c_void_p]
        L.mkr_decode_set_append.argtypes = [C.c_void_p, _f32p, _f32p, C.c_int]
        L.mkr_pipeline_run.argtypes = [_sz, _sz, _sz, _sz, _sz, _sz, _sz, _sz, _sz, C.c_uint64, C.c_int,
                                       C.c_void_p, C.c_void_p, _sz, C.c_void_p, C.c_void_p,
                                       C.POINTER(C.c_double)]
        L.mkr_decode_set_step.argtypes = [C.c_void_p, _f32p, _f32p, _f32p, C.c_float, _f32p, C.c_int,
                                          C.POINTER(C.c_double)]
        L.mkr_prefill_heads.argtypes = [_sz, _sz, _sz, _sz, C.c_uint64, C.c_int,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]

    def quantize_matrix(self, m, axis, group_size=16):
        m = _f32(m)
        rows, cols = m.shape
        nmax = rows * cols
        words = np.zeros(max((nmax + 15) // 16, 1), np.uint32)
        ng_max = (cols * ((rows + group_size - 1) // group_size) if axis == 0
                  else rows * ((cols + group_size - 1) // group_size))
        params = np.zeros(max(2 * ng_max, 2), np.float32)
        nw, ng = _sz(0), _sz(0)
        _check(self.lib.mkr_quantize_matrix(m, rows, cols, axis, group_size, words, C.byref(nw),
                                            params, C.byref(ng)), "quantize_matrix")
        return words[:nw.value], params[:2 * ng.value].reshape(-1, 2)

    def quant_dequant_matrix(self, m, axis, group_size=16):
        m = _f32(m)
        out = np.zeros_like(m)
        _check(self.lib.mkr_quant_dequant_matrix(m, m.shape[0], m.shape[1], axis, group_size, out),
               "quantize/dequantize")
        return out

    def pipeline_run(self, n_kv, g, l, d, hh, rw, steps, seed, threads, n_r=128, gs=16, want_xo=False):
        """The reference's single-layer chain per kv-head unit (ref_capi.cpp mkr_pipeline_run):
        selective_flash_attn -> prefill -> `steps` decode steps, on `threads` host threads."""
        out = np.zeros((max(steps, 1), n_kv * g, d), np.float32)
        ks = max(min(hh + rw, l), 1)
        kept = np.zeros((n_kv, ks), np.int64)
        nk = np.zeros(n_kv, np.int64)
        xo = np.zeros((n_kv * g, l, d), np.float32) if want_xo else None
        secs = (C.c_double * 4)()
        _check(self.lib.mkr_pipeline_run(n_kv, g, l, d, hh, rw, n_r, gs, steps, seed, threads,
                                          out.ctypes.data, kept.ctypes.data, ks, nk.ctypes.data,
                                          xo.ctypes.data if xo is not None else None, secs), "pipeline_run")
        return {"out": out[:steps], "kept": kept, "n_kept": nk, "x_o": xo, "wall_s": secs[0],
                "attn_thread_s": secs[1], "prefill_thread_s": secs[2], "decode_thread_s": secs[3]}

    def cache_prefill(self, k, v, a_cumul, hh, rw, n_r=128, gs=16) -> "RefCache":
        k, v, a = _f32(k), _f32(v), _f32(a_cumul)
        h = C.c_void_p()
        _check(self.lib.mkr_cache_prefill(k, v, a, len(a), k.shape[1], hh, rw, n_r, gs,
                                          C.byref(h)), "prefill")
        return RefCache(self, h, k.shape[1])

    def load_cache(self, path, d=128) -> "RefCache":
        """load_cache (snapshot.cpp:159-198)."""
        h = C.c_void_p()
        _check(self.lib.mkr_cache_load(os.fsencode(path), C.byref(h)), "load_cache")
        return RefCache(self, h, d)


class RefCache:
    def __init__(self, ref: RefOracle, h, d):
        self.ref, self.h, self.d = ref, h, d

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.mkr_cache_destroy(self.h)
            self.h = None

    def append(self, tk, tv):
        _check(self.ref.lib.mkr_cache_append(self.h, _f32(tk), _f32(tv)), "decode_append")

    def decode_step(self, tq, tk, tv, scale):
        out = np.zeros(self.d, np.float32)
        _check(self.ref.lib.mkr_cache_decode_step(self.h, _f32(tq), _f32(tk), _f32(tv), scale, out),
               "decode_step")
        return out

    @property
    def tokens_quantized(self):
        return self.ref.lib.mkr_cache_tokens_quantized(self.h)

    @property
    def tokens_residual(self):
        return self.ref.lib.mkr_cache_tokens_residual(self.h)

    def save(self, path):
        """save_cache (snapshot.cpp:71-157)."""
        _check(self.ref.lib.mkr_cache_save(self.h, os.fsencode(path)), "save_cache")

    def export(self, which: int):
        L = self.ref.lib
        nw, npar, nb = L.mkr_cache_n_words(self.h, which), L.mkr_cache_n_params(self.h, which), \
            L.mkr_cache_n_blocks(self.h)
        words = np.zeros(max(nw, 1), np.uint32)
        params = np.zeros(max(2 * npar, 2), np.float32)
        br = np.zeros(max(nb, 1), np.int64)
        L.mkr_cache_export(self.h, which, words, params, br)
        return words[:nw], params[:2 * npar].reshape(-1, 2), br[:nb]


_PORT = None
_REF = None


def port() -> PortOracle:
    global _PORT
    if _PORT is None:
        _PORT = PortOracle()
    return _PORT


def ref() -> RefOracle:
    global _REF
    if _REF is None:
        _REF = RefOracle()
    return _REF


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def build():
    """Compile the checkers (C port always; the reference when /root/reference exists)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", HERE], check=True)
