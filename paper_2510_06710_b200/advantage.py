"""Advantage operators (chunkrl::advantage) on the B200: GAE, PPO batch assembly and
GRPO group assembly. Same names and argument meaning as advantage/gae.hpp,
advantage/grpo.hpp and advantage/assembler.hpp; inputs/outputs are device tensors."""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import _lib
from .core import (EpisodeTable, GaeParams, GranularitySpec, GrpoAssemblyOptions, GrpoBatch,
                   Level, PpoAssemblyOptions, PpoBatch, RolloutBuffer, Workspace, _ptr,
                   stream_ptr)
from .errors import LengthMismatch


def compute_gae(rewards, values, bootstrap, terminated, truncated, params: GaeParams = GaeParams(),
                stream=None):
    """compute_gae (advantage/gae.cpp:7-37) over one flat unit sequence, per-unit bootstrap.
    Accepts a float `bootstrap` for the convenience overload (gae.cpp:39-46). fp64 on device."""
    dev = torch.device("cuda")
    r = torch.as_tensor(rewards, dtype=torch.float64).to(dev)
    n = r.numel()
    if isinstance(bootstrap, (int, float)):
        b = torch.zeros(n, dtype=torch.float64, device=dev)
        if n:
            b[-1] = float(bootstrap)
    else:
        b = torch.as_tensor(bootstrap, dtype=torch.float64).to(dev)
    v = torch.as_tensor(values, dtype=torch.float64).to(dev)
    te = torch.as_tensor(terminated, dtype=torch.bool).to(dev)
    tr = torch.as_tensor(truncated, dtype=torch.bool).to(dev)
    if not (v.numel() == b.numel() == te.numel() == tr.numel() == n):
        raise LengthMismatch("compute_gae: input lengths differ")
    flags = (te.to(torch.uint8) * _lib.FLAG_TERMINATED + tr.to(torch.uint8) * _lib.FLAG_TRUNCATED).contiguous()
    adv = torch.empty(n, dtype=torch.float64, device=dev)
    ret = torch.empty(n, dtype=torch.float64, device=dev)
    if n == 0:
        return adv, ret
    offs = torch.tensor([0, n], dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().ckrl_compute_gae(1, _ptr(offs), _ptr(r.contiguous()), _ptr(v.contiguous()),
                                           _ptr(b.contiguous()), _ptr(flags), C.byref(params.c()),
                                           _ptr(adv), _ptr(ret), stream_ptr(stream)))
    return adv, ret


def compute_gae_batched(seq_offsets, rewards, values, bootstrap, flags, params: GaeParams = GaeParams(),
                        stream=None):
    """Many independent sequences packed back to back (one warp each)."""
    n = rewards.numel()
    adv = torch.empty(n, dtype=torch.float64, device=rewards.device)
    ret = torch.empty_like(adv)
    _lib.check(_lib.lib().ckrl_compute_gae(seq_offsets.numel() - 1, _ptr(seq_offsets), _ptr(rewards),
                                           _ptr(values), _ptr(bootstrap), _ptr(flags),
                                           C.byref(params.c()), _ptr(adv), _ptr(ret),
                                           stream_ptr(stream)))
    return adv, ret


def assemble_ppo_batch(rollout: RolloutBuffer, options: PpoAssemblyOptions,
                       workspace: Optional[Workspace] = None, out: Optional[PpoBatch] = None,
                       stream=None) -> PpoBatch:
    """assemble_ppo_batch (advantage/assembler.cpp:78-195). `rollout.bootstrap` must hold
    the snapshot value of post_obs for the advantage-level head."""
    E, Tc, Cn, M = rollout.shape
    spec = options.spec
    if out is None:
        dev = rollout.tokens.device
        shape = (E, Tc) if spec.advantage_level == Level.Chunk else (E, Tc, Cn)
        ws = workspace or Workspace(E, 1, dev)
        out = PpoBatch(spec=spec, counted=torch.empty((E, Tc, Cn), dtype=torch.uint8, device=dev),
                       advantages=torch.empty(shape, dtype=torch.float32, device=dev),
                       returns=torch.empty(shape, dtype=torch.float32, device=dev), workspace=ws)
    bc = out.c()
    _lib.check(_lib.lib().ckrl_assemble_ppo_batch(C.byref(rollout.c()), C.byref(options.gae.c()),
                                                  C.byref(spec.c()), C.byref(bc), out.workspace.ptr,
                                                  out.workspace.bytes, stream_ptr(stream)))
    return out


def assemble_grpo_batch(rollout: RolloutBuffer, episodes: EpisodeTable,
                        options: GrpoAssemblyOptions = GrpoAssemblyOptions(),
                        workspace: Optional[Workspace] = None, out: Optional[GrpoBatch] = None,
                        stream=None) -> GrpoBatch:
    """assemble_grpo_batch (advantage/assembler.cpp:197-267)."""
    E = rollout.shape[0]
    if out is None:
        ws = workspace or Workspace(E, 1, rollout.tokens.device)
        out = GrpoBatch.allocate(rollout, options.spec, ws)
    bc = out.c()
    _lib.check(_lib.lib().ckrl_assemble_grpo_batch(
        C.byref(rollout.c()), C.byref(episodes.c()), C.byref(options.spec.c()),
        C.byref(options.c()), C.byref(bc), out.workspace.ptr, out.workspace.bytes,
        stream_ptr(stream)))
    return out
