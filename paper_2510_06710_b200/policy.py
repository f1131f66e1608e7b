"""The fused action-token kernel as a standalone operator: PolicyNet::evaluate_chunk
(policy/policy_net.cpp:333-357) + aggregate_logprob (core/granularity.cpp:83-113) over
current-policy logits rows; and the softmax-backward seam, the per-position logits gradient of
PolicyNet::accumulate_chunk_gradient (policy/policy_net.cpp:431-456)."""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .core import _ptr, stream_ptr


def evaluate_chunks(logits: torch.Tensor, tokens: torch.Tensor, valid=None, stream=None):
    """logits [..., C, M, V] (f32/bf16), tokens [..., C, M] -> dict of token log-probs and
    entropies [..., C, M] (f32), action log-probs [..., C] and chunk log-probs [...] (f64,
    canonical summation order), and entropy at action / chunk granularity (f64: per slot the
    sum of its token entropies, per chunk the sum of its slots', over the `valid` [..., C]
    slots (bool / u8; default all), 0 elsewhere)."""
    *lead, Cn, M, V = logits.shape
    n = 1
    for d in lead:
        n *= d
    dev = logits.device
    lp = torch.empty((*lead, Cn, M), dtype=torch.float32, device=dev)
    ent = torch.empty_like(lp)
    act = torch.empty((*lead, Cn), dtype=torch.float64, device=dev)
    chk = torch.empty(tuple(lead), dtype=torch.float64, device=dev)
    aent = torch.empty_like(act)
    cent = torch.empty_like(chk)
    mask = None if valid is None else valid.to(device=dev, dtype=torch.uint8).contiguous()
    ld = _lib.DTYPE_BF16 if logits.dtype == torch.bfloat16 else _lib.DTYPE_F32
    td = _lib.DTYPE_U8 if tokens.dtype == torch.uint8 else _lib.DTYPE_I32
    tokens = tokens.contiguous() if tokens.dtype in (torch.uint8, torch.int32) else tokens.to(torch.int32).contiguous()
    _lib.check(_lib.lib().ckrl_token_stats(n, Cn, M, V, ld, _ptr(logits.contiguous()), td,
                                           _ptr(tokens), _ptr(lp), _ptr(ent), _ptr(act), _ptr(chk),
                                           _ptr(mask), _ptr(aent), _ptr(cent), stream_ptr(stream)))
    return {"token_logprob": lp, "token_entropy": ent, "action_logprob": act, "chunk_logprob": chk,
            "action_entropy": aent, "chunk_entropy": cent}


def project_token_stats(feature: torch.Tensor, w_pol: torch.Tensor, b_pol, tokens: torch.Tensor,
                        rows_out=None, want_logits=None, stream=None, rows_only: bool = False):
    """Row N2: the policy head PolicyNet::logits_from_feature (policy/policy_net.cpp:265-274,
    logits = W_pol h + b_pol) on the tensor cores, fused with evaluate_chunk's per-position
    log-prob / entropy (:333-357). feature [..., H] bf16 (H a multiple of 64), w_pol [256, H]
    bf16, b_pol [256] f32 or None, tokens [...]. Returns {"token_rows": [..., 2] f64 (the
    16-byte ckrl_token_row per position: PolicyOutputs(token_rows=...) feeds the losses),
    "token_logprob": [...] f64, "token_entropy": [...] f32, "logits": [..., 256] (only with
    want_logits = torch.float32 / torch.bfloat16)}; rows_only skips the separate lp / entropy
    arrays (the rows carry both)."""
    *lead, H = feature.shape
    rows = 1
    for d in lead:
        rows *= d
    dev = feature.device
    feature = feature.contiguous()
    w_pol = w_pol.contiguous()
    if feature.dtype != torch.bfloat16 or w_pol.dtype != torch.bfloat16:
        raise TypeError("feature and w_pol must be bfloat16")
    if w_pol.dim() != 2 or w_pol.shape[1] != H:
        raise ValueError(f"w_pol must be [vocab, {H}], got {tuple(w_pol.shape)}")
    V = w_pol.shape[0]
    if tokens.shape != tuple(lead):
        raise ValueError(f"tokens must have shape {tuple(lead)}, got {tuple(tokens.shape)}")
    b = None if b_pol is None else b_pol.to(device=dev, dtype=torch.float32).contiguous()
    if b is not None and b.numel() != V:
        raise ValueError(f"b_pol must have {V} entries")
    if rows_out is None:
        rows_out = torch.empty((*lead, 2), dtype=torch.float64, device=dev)
    elif (rows_out.dtype != torch.float64 or tuple(rows_out.shape) != (*lead, 2)
          or not rows_out.is_contiguous() or rows_out.device != dev):
        raise ValueError("rows_out must be a contiguous float64 [..., 2] tensor on the features' device")
    lp = None if rows_only else torch.empty(tuple(lead), dtype=torch.float64, device=dev)
    ent = None if rows_only else torch.empty(tuple(lead), dtype=torch.float32, device=dev)
    logits = None
    ld = _lib.DTYPE_F32
    if want_logits is not None:
        logits = torch.empty((*lead, V), dtype=want_logits, device=dev)
        ld = _lib.DTYPE_BF16 if want_logits == torch.bfloat16 else _lib.DTYPE_F32
    td = _lib.DTYPE_U8 if tokens.dtype == torch.uint8 else _lib.DTYPE_I32
    tokens = tokens.contiguous() if tokens.dtype in (torch.uint8, torch.int32) else tokens.to(torch.int32).contiguous()
    head = _lib.PolicyHead(H, V, _ptr(feature), _ptr(w_pol), _ptr(b))
    _lib.check(_lib.lib().ckrl_project_token_stats(rows, C.byref(head), td, _ptr(tokens), _ptr(rows_out),
                                                   _ptr(lp), _ptr(ent), ld, _ptr(logits), stream_ptr(stream)))
    return {"token_rows": rows_out, "token_logprob": lp, "token_entropy": ent, "logits": logits}


def logits_grad(logits: torch.Tensor, tokens: torch.Tensor, coeff_logprob: torch.Tensor,
                coeff_entropy=None, out=None, out_dtype=None, status=None, stream=None,
                check: bool = True) -> torch.Tensor:
    """dlogits[..., v] = coeff_lp * ([v == tok] - p_v) + coeff_ent * (-p_v * (ls_v + H)) per
    position (policy/policy_net.cpp:431-456). logits [..., V] (f32/bf16), tokens / coefficients
    [...] (the loss outputs). `out` may be `logits` itself (in place). With check=True the call
    synchronises and raises NonFinite like the reference (:437-438); otherwise pass a zeroed
    int32 `status` tensor and read it later with `_lib.read_status`."""
    V = logits.shape[-1]
    rows = logits.numel() // V
    if out is None:
        out = torch.empty(logits.shape, dtype=out_dtype or logits.dtype, device=logits.device)
    ld = _lib.DTYPE_BF16 if logits.dtype == torch.bfloat16 else _lib.DTYPE_F32
    od = _lib.DTYPE_BF16 if out.dtype == torch.bfloat16 else _lib.DTYPE_F32
    td = _lib.DTYPE_U8 if tokens.dtype == torch.uint8 else _lib.DTYPE_I32
    tokens = tokens.contiguous() if tokens.dtype in (torch.uint8, torch.int32) else tokens.to(torch.int32).contiguous()
    klp = coeff_logprob.contiguous().float()
    kent = coeff_entropy.contiguous().float() if coeff_entropy is not None else None
    if status is None and check:
        status = torch.zeros(1, dtype=torch.int32, device=logits.device)
    _lib.check(_lib.lib().ckrl_logits_grad(rows, V, ld, _ptr(logits.contiguous()), td, _ptr(tokens),
                                           _ptr(klp), _ptr(kent), od, _ptr(out), _ptr(status),
                                           stream_ptr(stream)))
    if check:
        _lib.check(_lib.lib().ckrl_read_status(_ptr(status), stream_ptr(stream)))
    return out
