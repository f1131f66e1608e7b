"""Domain types mirroring chunkrl/core (granularity.hpp, gae.hpp, losses.hpp, assembler.hpp)
and the device-resident SoA rollout buffer that replaces TrajectorySlab (types.hpp:89-104).

All tensors live on the CUDA device; these classes only own device memory and build
the ckrl.h structures. Compute happens in libckrl.so.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import Optional

import torch

from . import _lib


class Level(enum.IntEnum):
    """core/granularity.hpp:8"""
    Chunk = _lib.LEVEL_CHUNK
    Action = _lib.LEVEL_ACTION
    Token = _lib.LEVEL_TOKEN

    @staticmethod
    def from_name(name: str) -> "Level":
        # core/granularity.cpp:22-30
        n = name.replace("_level", "")
        if n not in ("chunk", "action", "token"):
            from .errors import ConfigError
            raise ConfigError(f"unknown granularity level: {name}")
        return {"chunk": Level.Chunk, "action": Level.Action, "token": Level.Token}[n]


@dataclass(frozen=True)
class GranularitySpec:
    """core/granularity.hpp:21-27"""
    advantage_level: Level = Level.Chunk
    logprob_level: Level = Level.Chunk
    value_level: Level = Level.Chunk

    def c(self) -> _lib.Granularity:
        return _lib.Granularity(int(self.advantage_level), int(self.logprob_level),
                                int(self.value_level))


def validate_granularity(spec: GranularitySpec) -> None:
    """core/granularity.cpp:47-60"""
    _lib.check(_lib.lib().ckrl_validate_granularity(C.byref(spec.c())))


@dataclass(frozen=True)
class GaeParams:
    """advantage/gae.hpp:8-13"""
    gamma: float = 0.99
    lam: float = 0.95

    def c(self):
        return _lib.GaeParams(self.gamma, self.lam)


@dataclass(frozen=True)
class PpoParams:
    """optim/losses.hpp:12-21 (optimizer fields are out of scope of the hot path)."""
    clip_eps: float = 0.2
    value_loss_coef: float = 0.5
    entropy_coef: float = 0.0
    advantage_normalization: bool = True

    def c(self):
        return _lib.PpoParams(self.clip_eps, self.value_loss_coef, self.entropy_coef,
                              int(self.advantage_normalization))


@dataclass(frozen=True)
class GrpoParams:
    """optim/losses.hpp:23-29"""
    clip_eps: float = 0.2

    def c(self):
        return _lib.GrpoParams(self.clip_eps)


@dataclass(frozen=True)
class FilterBounds:
    """advantage/grpo.hpp:20-25"""
    lower: float = 0.0
    upper: float = 1.0


@dataclass(frozen=True)
class GrpoAssemblyOptions:
    """advantage/assembler.hpp:76-83"""
    spec: GranularitySpec = GranularitySpec()
    eps_std: float = 1e-8
    apply_filter: bool = True
    filter_bounds: FilterBounds = FilterBounds()
    length_normalized: bool = True
    min_group_size: int = 2

    def c(self):
        return _lib.GrpoOptions(self.eps_std, int(self.apply_filter), self.filter_bounds.lower,
                                self.filter_bounds.upper, int(self.length_normalized),
                                self.min_group_size)


@dataclass(frozen=True)
class PpoAssemblyOptions:
    """advantage/assembler.hpp:64-67"""
    gae: GaeParams = GaeParams()
    spec: GranularitySpec = GranularitySpec()


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _dev(t, dtype, device):
    return torch.as_tensor(t).to(device=device, dtype=dtype).contiguous()


@dataclass
class RolloutBuffer:
    """The SoA rollout buffer in HBM (include/ckrl.h layout). Replaces the AoS
    TrajectorySlab::records[env][chunk] of StepRecord (core/types.hpp:54-104)."""
    tokens: torch.Tensor        # [E][Tc][C][M] u8 (V<=256) or i32
    old_logprob: torch.Tensor   # [E][Tc][C][M] f32
    reward: torch.Tensor        # [E][Tc][C] f32
    flags: torch.Tensor         # [E][Tc][C] u8
    episode_id: torch.Tensor    # [E][Tc][C] i32
    value_scalar: torch.Tensor  # [E][Tc] f32
    value_vector: torch.Tensor  # [E][Tc][C] f32
    bootstrap: torch.Tensor     # [E][Tc][C] f32
    vocab: int

    @property
    def shape(self):
        E, Tc, Cn, M = self.tokens.shape
        return E, Tc, Cn, M

    def c(self) -> _lib.Rollout:
        E, Tc, Cn, M = self.shape
        tok_dtype = _lib.DTYPE_U8 if self.tokens.dtype == torch.uint8 else _lib.DTYPE_I32
        r = _lib.Rollout(E, Tc, Cn, M, self.vocab, tok_dtype, *[_ptr(t) for t in (
            self.tokens, self.old_logprob, self.reward, self.flags, self.episode_id,
            self.value_scalar, self.value_vector, self.bootstrap)])
        return r

    @classmethod
    def from_arrays(cls, d: dict, bootstrap, vocab: int, device="cuda") -> "RolloutBuffer":
        tok_dtype = torch.uint8 if vocab <= 256 else torch.int32
        return cls(tokens=_dev(d["tokens"], tok_dtype, device),
                   old_logprob=_dev(d["old_logprob"], torch.float32, device),
                   reward=_dev(d["reward"], torch.float32, device),
                   flags=_dev(d["flags"], torch.uint8, device),
                   episode_id=_dev(d["episode_id"], torch.int32, device),
                   value_scalar=_dev(d["value_scalar"], torch.float32, device),
                   value_vector=_dev(d["value_vector"], torch.float32, device),
                   bootstrap=_dev(bootstrap, torch.float32, device), vocab=vocab)


@dataclass
class EpisodeTable:
    """EpisodeInfo table (core/types.hpp:72-85) as SoA device tensors."""
    env_id: torch.Tensor
    episode_id: torch.Tensor
    start_step: torch.Tensor
    length: torch.Tensor
    total_reward: torch.Tensor  # f64
    first_success: torch.Tensor
    complete: torch.Tensor
    task_id: torch.Tensor
    reset_state_id: torch.Tensor

    def c(self) -> _lib.Episodes:
        return _lib.Episodes(int(self.env_id.numel()), *[_ptr(t) for t in (
            self.env_id, self.episode_id, self.start_step, self.length, self.total_reward,
            self.first_success, self.complete, self.task_id, self.reset_state_id)])

    @classmethod
    def from_arrays(cls, d: dict, device="cuda") -> "EpisodeTable":
        i32 = torch.int32
        return cls(env_id=_dev(d["ep_env_id"], i32, device),
                   episode_id=_dev(d["ep_episode_id"], i32, device),
                   start_step=_dev(d["ep_start"], i32, device),
                   length=_dev(d["ep_length"], i32, device),
                   total_reward=_dev(d["ep_total_reward"], torch.float64, device),
                   first_success=_dev(d["ep_first_success"], i32, device),
                   complete=_dev(d["ep_complete"], torch.uint8, device),
                   task_id=_dev(d["ep_task"], i32, device),
                   reset_state_id=_dev(d["ep_reset_id"], i32, device))


@dataclass
class PolicyOutputs:
    """Current-policy outputs the loss consumes (what ppo_loss recomputes through
    PolicyNet::evaluate_chunk / value, optim/losses.cpp:115, 196)."""
    logits: Optional[torch.Tensor]        # [E][Tc][C][M][V] f32 or bf16
    values: Optional[torch.Tensor] = None  # [E][Tc] or [E][Tc][C] f32
    # or, in place of logits, the policy head already reduced on the tensor cores:
    # [E][Tc][C][M] ckrl_token_row as a [..., 2] f64 tensor (policy.project_token_stats)
    token_rows: Optional[torch.Tensor] = None

    def c(self) -> _lib.PolicyOutputs:
        if self.token_rows is not None:
            t = self.token_rows
            if t.dtype != torch.float64 or t.shape[-1] != 2 or not t.is_contiguous():
                raise ValueError("token_rows must be a contiguous float64 [E][Tc][C][M][2] tensor "
                                 "(one 16-byte ckrl_token_row per position)")
            return _lib.PolicyOutputs(_lib.DTYPE_TOKEN_ROWS, _ptr(t), _ptr(self.values))
        dt = _lib.DTYPE_BF16 if self.logits.dtype == torch.bfloat16 else _lib.DTYPE_F32
        return _lib.PolicyOutputs(dt, _ptr(self.logits), _ptr(self.values))


class Workspace:
    """Caller-owned device scratch (allocated once, reused by every hot call)."""

    def __init__(self, num_envs: int, world: int = 1, device="cuda"):
        n = _lib.lib().ckrl_workspace_bytes(num_envs, 0, 1, 1, world)
        self.tensor = torch.zeros(int(n), dtype=torch.uint8, device=device)
        self.bytes = int(n)
        self.num_envs = num_envs
        self.world = world

    @property
    def ptr(self):
        return C.c_void_p(self.tensor.data_ptr())


@dataclass
class LossOutputs:
    """Optional per-position outputs of the loss (device tensors or None)."""
    coeff_logprob: Optional[torch.Tensor] = None
    coeff_entropy: Optional[torch.Tensor] = None
    coeff_value: Optional[torch.Tensor] = None
    token_logprob: Optional[torch.Tensor] = None
    token_entropy: Optional[torch.Tensor] = None
    dlogits: Optional[torch.Tensor] = None  # fused softmax-backward seam, logits' shape and dtype
    action_entropy: Optional[torch.Tensor] = None  # [E][Tc][C] f64, unit-active slots
    chunk_entropy: Optional[torch.Tensor] = None   # [E][Tc] f64

    def c(self) -> _lib.LossOutputs:
        return _lib.LossOutputs(*[_ptr(t) for t in (
            self.coeff_logprob, self.coeff_entropy, self.coeff_value, self.token_logprob,
            self.token_entropy, self.dlogits, self.action_entropy, self.chunk_entropy)])

    @classmethod
    def allocate(cls, rollout: RolloutBuffer, value_level: Level, tokens: bool = False,
                 entropy: bool = False):
        E, Tc, Cn, M = rollout.shape
        dev = rollout.tokens.device
        f = dict(dtype=torch.float32, device=dev)
        vshape = (E, Tc) if value_level == Level.Chunk else (E, Tc, Cn)
        return cls(coeff_logprob=torch.empty((E, Tc, Cn, M), **f),
                   coeff_entropy=torch.empty((E, Tc, Cn, M), **f),
                   coeff_value=torch.empty(vshape, **f),
                   token_logprob=torch.empty((E, Tc, Cn, M), **f) if tokens else None,
                   token_entropy=torch.empty((E, Tc, Cn, M), **f) if tokens else None,
                   action_entropy=torch.empty((E, Tc, Cn), dtype=torch.float64, device=dev) if entropy else None,
                   chunk_entropy=torch.empty((E, Tc), dtype=torch.float64, device=dev) if entropy else None)


def stream_ptr(stream: Optional[torch.cuda.Stream] = None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def diagnostics_dict(host) -> dict:
    return {k: float(host[i]) for i, k in enumerate(_lib.DIAG_NAMES)}


def read_diagnostics(diag: torch.Tensor, stream=None) -> dict:
    """Copies device diagnostics to the host (synchronises) and raises the reference's
    exceptions (SkipUpdate, DegenerateGroup, NonFinite)."""
    host = (C.c_double * _lib.DIAG_COUNT)()
    _lib.check(_lib.lib().ckrl_read_diagnostics(C.c_void_p(diag.data_ptr()), host,
                                                stream_ptr(stream)))
    d = diagnostics_dict(host)
    d["units"] = int(d["units"])
    d.pop("status")
    return d


@dataclass
class PpoBatch:
    """PpoBatch (advantage/assembler.hpp:31-37) as device SoA + its workspace."""
    spec: GranularitySpec
    counted: torch.Tensor
    advantages: torch.Tensor
    returns: torch.Tensor
    workspace: Workspace

    def c(self):
        if self.advantages.dtype != torch.float64 or self.returns.dtype != torch.float64:
            raise TypeError("PpoBatch advantages / returns are float64 (the reference's PpoBatch)")
        return _lib.PpoBatchC(_ptr(self.counted), _ptr(self.advantages), _ptr(self.returns))

    def advantage_unit_count(self) -> int:
        """assembler.cpp:161-177 (host sync)."""
        if self.spec.advantage_level == Level.Chunk:
            return int(self.counted.any(dim=-1).sum().item())
        return int(self.counted.sum().item())


@dataclass
class GrpoBatch:
    """GrpoBatch (advantage/assembler.hpp:58-62) as device SoA: per env its retained
    trajectory (group ordinal, member index, episode, advantage, group size) and per slot
    the trajectory membership and step weight."""
    spec: GranularitySpec
    env_group: torch.Tensor
    env_member: torch.Tensor
    env_episode: torch.Tensor
    env_advantage: torch.Tensor
    env_group_size: torch.Tensor
    slot_weight: torch.Tensor
    slot_member: torch.Tensor
    group_counts: torch.Tensor
    workspace: Workspace

    def c(self):
        return _lib.GrpoBatchC(*[_ptr(t) for t in (
            self.env_group, self.env_member, self.env_episode, self.env_advantage,
            self.env_group_size, self.slot_weight, self.slot_member, self.group_counts)])

    @property
    def groups_total(self) -> int:
        return int(self.group_counts[0].item())

    @property
    def groups_retained(self) -> int:
        return int(self.group_counts[1].item())

    @classmethod
    def allocate(cls, rollout: RolloutBuffer, spec: GranularitySpec, workspace: Workspace):
        E, Tc, Cn, M = rollout.shape
        dev = rollout.tokens.device
        i32 = dict(dtype=torch.int32, device=dev)
        return cls(spec=spec, env_group=torch.empty(E, **i32), env_member=torch.empty(E, **i32),
                   env_episode=torch.empty(E, **i32),
                   env_advantage=torch.empty(E, dtype=torch.float64, device=dev),
                   env_group_size=torch.empty(E, **i32),
                   slot_weight=torch.empty((E, Tc, Cn), dtype=torch.float64, device=dev),
                   slot_member=torch.empty((E, Tc, Cn), dtype=torch.uint8, device=dev),
                   group_counts=torch.zeros(2, **i32), workspace=workspace)

