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
                       advantages=torch.empty(shape, dtype=torch.float64, device=dev),
                       returns=torch.empty(shape, dtype=torch.float64, device=dev), workspace=ws)
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


# ---- per-group / per-episode GRPO helpers (advantage/grpo.hpp:32-53), batched ---------------
def _segments(seqs, dtype):
    """list of per-group / per-episode sequences -> (flat device tensor, offsets)."""
    dev = torch.device("cuda")
    lens = [len(s) for s in seqs]
    offs = [0]
    for n in lens:
        offs.append(offs[-1] + n)
    flat = torch.tensor([x for s in seqs for x in s], dtype=dtype).to(dev)
    return flat, offs


def grpo_group_advantage(groups, eps_std: float, stream=None):
    """grpo_group_advantage (grpo.cpp:9-28) for every group at once. `groups`: list of
    per-group total-reward lists (GroupBatch::total_rewards). Returns a list of per-group
    advantage lists; raises DegenerateGroup like the reference."""
    R, offs = _segments(groups, torch.float64)
    dev = R.device
    o = torch.tensor(offs, dtype=torch.int32, device=dev)
    adv = torch.empty_like(R)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().ckrl_grpo_group_advantage(len(groups), _ptr(o), _ptr(R), C.c_double(eps_std),
                                                    _ptr(adv), _ptr(status), stream_ptr(stream)))
    st = int(status.item())
    if st:
        from . import errors
        raise errors.from_status(st, "GRPO group needs >= 2 trajectories with non-zero std or eps_std > 0")
    a = adv.cpu().tolist()
    return [a[offs[g]:offs[g + 1]] for g in range(len(groups))]


def group_mean_return(groups, stream=None):
    R, offs = _segments(groups, torch.float64)
    o = torch.tensor(offs, dtype=torch.int32, device=R.device)
    mean = torch.empty(len(groups), dtype=torch.float64, device=R.device)
    _lib.check(_lib.lib().ckrl_success_rate_filter(len(groups), _ptr(o), _ptr(R), C.c_double(0.0),
                                                   C.c_double(0.0), None, _ptr(mean), stream_ptr(stream)))
    return mean.cpu().tolist()


def success_rate_filter(groups, lower: float = 0.0, upper: float = 1.0, stream=None):
    """success_rate_filter (grpo.cpp:37-46): indices of the groups kept (strict bounds)."""
    R, offs = _segments(groups, torch.float64)
    o = torch.tensor(offs, dtype=torch.int32, device=R.device)
    keep = torch.empty(len(groups), dtype=torch.uint8, device=R.device)
    _lib.check(_lib.lib().ckrl_success_rate_filter(len(groups), _ptr(o), _ptr(R), C.c_double(lower),
                                                   C.c_double(upper), _ptr(keep), None, stream_ptr(stream)))
    return [g for g, k in enumerate(keep.cpu().tolist()) if k]


def _episode_args(episodes):
    dev = torch.device("cuda")
    offs = [0]
    for length, _, _ in episodes:
        offs.append(offs[-1] + int(length))
    o = torch.tensor(offs, dtype=torch.int64, device=dev)
    succ = torch.tensor([int(bool(s)) for _, s, _ in episodes], dtype=torch.uint8, device=dev)
    fs = torch.tensor([int(f) for _, _, f in episodes], dtype=torch.int64, device=dev)
    return offs, o, succ, fs


def valid_action_mask(episodes, stream=None):
    """valid_action_mask (grpo.cpp:48-55) for [(length, success, first_success_step), ...]."""
    offs, o, succ, fs = _episode_args(episodes)
    mask = torch.empty(offs[-1], dtype=torch.uint8, device=o.device)
    _lib.check(_lib.lib().ckrl_valid_action_mask(len(episodes), _ptr(o), _ptr(succ), _ptr(fs), _ptr(mask),
                                                 stream_ptr(stream)))
    m = [bool(x) for x in mask.cpu().tolist()]
    return [m[offs[i]:offs[i + 1]] for i in range(len(episodes))]


def length_norm_weights(episodes, length_normalized: bool, stream=None):
    """length_norm_weights (grpo.cpp:57-79) for [(length, success, first_success_step), ...]."""
    offs, o, succ, fs = _episode_args(episodes)
    w = torch.empty(offs[-1], dtype=torch.float64, device=o.device)
    _lib.check(_lib.lib().ckrl_length_norm_weights(len(episodes), _ptr(o), _ptr(succ), _ptr(fs),
                                                   int(bool(length_normalized)), _ptr(w),
                                                   stream_ptr(stream)))
    x = w.cpu().tolist()
    return [x[offs[i]:offs[i + 1]] for i in range(len(episodes))]


def slab_success_rate(episodes: EpisodeTable, stream=None) -> float:
    """slab_success_rate (assembler.cpp:269-278) over the device episode table."""
    out = torch.empty(1, dtype=torch.float64, device=episodes.env_id.device)
    _lib.check(_lib.lib().ckrl_slab_success_rate(C.byref(episodes.c()), _ptr(out), stream_ptr(stream)))
    return float(out.item())
