"""Toy end-to-end MiniKV pipeline on the B200 path.

Restates run_model (pipeline.cpp:65-235) with every hot-path step on the device:
per layer the q/k/v projections (cuBLAS fp32), K1 selective flash attention
(X_O feeds the next layer, A_cumul drives selection), the per-layer A_cumul
variance (device), the budget policy (uniform / pyramid / variance-proportional /
variance-inverse, selection.cpp:48-128), K2 + K3 prefill compression; then `steps`
decode iterations through K4 with each layer's output feeding the next, while a
full-precision keep-all pipeline runs side by side from the same tokens -- the
deviation trace of pipeline.cpp:166-230.  The keep-all side is the reference's fp32
decode_attention (pipeline.cpp:205) on the device (refmt.cu), per head.  mode =
"identity" (QuantMode::Identity, cache_engine.hpp:13-15) keeps the selected rows in
fp32 and decodes them with the same kernel: with a keep-all budget it reproduces the
full-precision pipeline exactly (acceptance criterion 7's identity check).

The reference's own pipeline driver (pipeline.cpp run_from_config, its seeded Rng stream)
runs on these kernels through the drop-in adapter: tests/test_reference_suites.py
(test_cache_engine's run_model cases and acceptance criterion 7).

Differences from the reference pipeline, by design: the device head dimension is
128 (d = 128 * n_heads), activations enter the kernels rounded to fp16, and the
seeded weights / tokens come from torch generators (statistically the reference's
N(0, 1/d) initialisation, not its bit stream).  The analytic deviation bound of
pipeline.cpp:209-219 is evaluated once, after decode, from the exported caches.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List

import numpy as np
import torch

from . import ops

HEAD_DIM = 128


@dataclass
class RunConfig:  # pipeline.hpp:16-35
    seed: int = 0
    layers: int = 4
    n_heads: int = 1
    l_prompt: int = 256
    steps: int = 32
    alpha_hh: float = 0.25
    alpha_rw: float = 0.25
    policy: str = "uniform"  # uniform | pyramid | var_prop | var_inv
    pyramid_depth: int = 7
    bottom_heavy: bool = True
    n_r: int = 128
    group_size: int = 16
    mode: str = "two_bit"  # two_bit | identity (QuantMode, cache_engine.hpp:13-15)

    @property
    def d(self) -> int:
        return HEAD_DIM * self.n_heads

    def validate(self):
        if self.layers < 1 or self.n_heads < 1 or self.l_prompt < 1 or self.steps < 0:
            raise ValueError("RunConfig: layers, n_heads, l_prompt must be >= 1")
        if self.alpha_hh < 0 or self.alpha_rw < 0:
            raise ValueError("RunConfig: negative budget")
        if self.policy not in ("uniform", "pyramid", "var_prop", "var_inv"):
            raise ValueError(f"RunConfig: unknown policy {self.policy}")
        if self.mode not in ("two_bit", "identity"):
            raise ValueError(f"RunConfig: unknown mode {self.mode}")


@dataclass
class RunTrace:  # pipeline.hpp:37-62
    config: RunConfig
    layers: List[dict] = field(default_factory=list)
    decode: List[dict] = field(default_factory=list)
    per_layer_a_cumul: List[np.ndarray] = field(default_factory=list)
    per_layer_hh: List[int] = field(default_factory=list)
    total_bytes_before: int = 0
    total_bytes_after: int = 0
    max_abs_dev: float = 0.0
    analytic_dev_bound: float = 0.0


def toy_model(seed: int, layers: int, d: int, device="cuda"):
    """ToyModel::seeded (harness.cpp:47-71): w_q, w_k, w_v ~ N(0, 1/d) per layer."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    std = 1.0 / math.sqrt(d)
    return [tuple((torch.randn(d, d, generator=g) * std).to(device) for _ in range(3)) for _ in range(layers)]


def _heads(x: torch.Tensor, n_heads: int) -> torch.Tensor:  # [l, d] -> [1, H, l, 128] fp16
    return x.view(x.shape[0], n_heads, HEAD_DIM).permute(1, 0, 2).contiguous().half()[None]


def _measured_bytes(cache: ops.KVCache, unit: int) -> int:  # accounting.cpp:101-114
    total = 0
    for which in (0, 1):
        w, p, _ = cache.export_reference(unit, which)
        total += 4 * len(w) + 4 * len(p)
    return total + cache.unit_info(unit)["tokens_residual"] * HEAD_DIM * 4


def run_model(weights, prompt: torch.Tensor, cfg: RunConfig) -> RunTrace:
    """pipeline.cpp:65-235 on the device.  prompt: fp32 [l_prompt, d] on cuda."""
    cfg.validate()
    L, H, d, l = cfg.layers, cfg.n_heads, cfg.d, cfg.l_prompt
    if len(weights) != L or prompt.shape != (l, d):
        raise ValueError("run_model: model/config dimension mismatch")
    scale = ops.default_scale(HEAD_DIM)
    trace = RunTrace(config=cfg)
    # ---- prefill forward: attention for every layer first (variance policies need all) ----
    ks, vs, acs, layer_vars = [], [], [], []
    x = prompt.float()
    for (wq, wk, wv) in weights:
        q, k, v = _heads(x @ wq, H), _heads(x @ wk, H), _heads(x @ wv, H)
        r = ops.selective_flash_attn(q, k, v, scale, True)  # K1
        ac = r.a_cumul[0]                                    # [H, l]
        layer_vars.append(float(ops.layer_score_variance(ac).double().mean()))
        trace.per_layer_a_cumul.append(ac.float().mean(0).cpu().numpy())
        ks.append(k[0])
        vs.append(v[0])
        acs.append(ac.contiguous())
        x = r.output[0].permute(1, 0, 2).reshape(l, d).float()
    # ---- budgets (pipeline.cpp:119-138) ----
    mean_hh = int(math.floor(cfg.alpha_hh * l))
    rw = int(math.floor(cfg.alpha_rw * l))
    if cfg.policy == "uniform":
        hh = ops.allocate_uniform(mean_hh * L, L)
    elif cfg.policy == "pyramid":
        hh = ops.allocate_pyramid(mean_hh, L, cfg.pyramid_depth, cfg.bottom_heavy)
    else:
        mode = ops.VarianceMode.Prop if cfg.policy == "var_prop" else ops.VarianceMode.Inv
        hh, _ = ops.allocate_variance(layer_vars, mean_hh * L, mode)
    trace.per_layer_hh = list(hh)
    caps = [min(hh[i] + rw, l) for i in range(L) for _ in range(H)]
    identity = cfg.mode == "identity"
    cache = ops.KVCache(L * H, caps, max_decode_tokens=cfg.steps + cfg.n_r, n_r=cfg.n_r,
                        group_size=cfg.group_size, keep_fp32_params=True)
    id_k, id_v = [], []  # identity mode: the selected rows in fp32 per layer [H][n, 128]
    for i in range(L):  # K2 + K3 per layer (cache_engine.cpp:56-77)
        cache.prefill(ks[i], vs[i], acs[i], hh[i], rw, unit_begin=i * H)
        if identity:
            kept_idx, nk = ops.select_token_counts(acs[i], [hh[i]] * H, rw)
            id_k.append([ks[i][h, kept_idx[h, :nk[h]].long()].float() for h in range(H)])
            id_v.append([vs[i][h, kept_idx[h, :nk[h]].long()].float() for h in range(H)])
    cache.check()
    for i in range(L):
        kept = min(hh[i] + rw, l)
        before = H * 4 * l * HEAD_DIM
        after = (sum(2 * (t.numel() + u.numel()) for t, u in zip(id_k[i], id_v[i])) if identity
                 else sum(_measured_bytes(cache, i * H + h) for h in range(H)))
        trace.layers.append({"layer": i, "kept_tokens": H * kept, "hh_tokens": H * (kept - min(rw, l)),
                             "rw_tokens": H * min(rw, l), "bytes_before": before, "bytes_after": after})
        trace.total_bytes_before += before
        trace.total_bytes_after += after
    # ---- decode: compressed (K4) and full-precision keep-all pipelines side by side ----
    ref_k = [k.float().clone() for k in ks]  # [H, l, 128] growing
    ref_v = [v.float().clone() for v in vs]
    g = torch.Generator(device="cpu").manual_seed(cfg.seed * 1000003 + 0xD0)
    l1q = torch.zeros(L, H, device="cuda")  # max |t_q|_1 per (layer, head) over the steps
    for s in range(cfg.steps):
        token = torch.randn(d, generator=g).cuda()
        xc, xr = token, token
        step_dev = 0.0
        for i, (wq, wk, wv) in enumerate(weights):
            qc, kc, vc = (xc @ wq).view(H, HEAD_DIM), (xc @ wk).view(H, HEAD_DIM), (xc @ wv).view(H, HEAD_DIM)
            if identity:  # fp32 stores + the device decode_attention over [stored ; new token]
                oc = torch.empty(H, HEAD_DIM, device="cuda")
                for h in range(H):
                    id_k[i][h] = torch.cat([id_k[i][h], kc[h][None]], 0)
                    id_v[i][h] = torch.cat([id_v[i][h], vc[h][None]], 0)
                    oc[h] = ops.decode_attention(qc[h].contiguous(), id_k[i][h], id_v[i][h], scale)[0]
            else:
                out_c = cache.decode_step(qc.half()[:, None, :], kc.half(), vc.half(), scale, unit_begin=i * H)
                oc = out_c[:, 0, :].float()
            l1q[i] = torch.maximum(l1q[i], qc.abs().sum(-1))
            qr, kr, vr = (xr @ wq).view(H, HEAD_DIM), (xr @ wk).view(H, HEAD_DIM), (xr @ wv).view(H, HEAD_DIM)
            ref_k[i] = torch.cat([ref_k[i], kr[:, None, :]], 1)
            ref_v[i] = torch.cat([ref_v[i], vr[:, None, :]], 1)
            # the reference keep-all decode: decode_attention per head (pipeline.cpp:205), on the device
            out_r = torch.stack([ops.decode_attention(qr[h].contiguous(), ref_k[i][h].contiguous(),
                                                      ref_v[i][h].contiguous(), scale)[0] for h in range(H)])
            step_dev = max(step_dev, float((oc - out_r).abs().max()))
            xc, xr = oc.reshape(d), out_r.reshape(d)
        trace.decode.append({"step": s, "max_abs_dev": step_dev})
        trace.max_abs_dev = max(trace.max_abs_dev, step_dev)
    cache.check()
    # ---- first-order deviation bound (pipeline.cpp:209-219), from the final caches ----
    bound = 0.0
    for u in range(L * H):
        _, pk, _ = cache.export_reference(u, 0)
        _, pv, _ = cache.export_reference(u, 1)
        dk = float(np.max(pk[:, 0])) / 2 if len(pk) else 0.0
        dv = float(np.max(pv[:, 0])) / 2 if len(pv) else 0.0
        rk, rv = cache.export_residual(u)
        vmax = max(float(np.max(np.abs(pv[:, 1]) + 3 * pv[:, 0])) if len(pv) else 0.0,
                   float(np.max(np.abs(rv.astype(np.float32)))) if len(rv) else 0.0)
        bound = max(bound, 2.0 * scale * float(l1q[u // H, u % H]) * dk * vmax + dv)
    trace.analytic_dev_bound = bound
    cache.close()
    return trace


def run_from_config(cfg: RunConfig) -> RunTrace:
    """run_from_config (pipeline.cpp:237-245): seeded model and prompt."""
    cfg.validate()
    weights = toy_model(cfg.seed, cfg.layers, cfg.d)
    g = torch.Generator(device="cpu").manual_seed(cfg.seed * 7919 + 0xA0)
    prompt = torch.randn(cfg.l_prompt, cfg.d, generator=g).cuda()
    return run_model(weights, prompt, cfg)
