"""(e) The rollout pipeline on the GPU: k env partitions, gen/sim kernels on two CUDA
streams with per-stage events (csrc/rollout.cu).

Mirrors the reference's rollout API — `placement::RolloutSpec` (rollout.hpp:16-22), the
`StageSim` / `StageGen` pair and `merge_stages` (rollout.cpp:11-109) as driven by
`RealBackend::run_rollout_epoch` (real_backend.cpp:59-138) — and returns the epoch as the
device-resident `RolloutBuffer` + `EpisodeTable` the advantage/loss path consumes, so one
epoch is rollout -> assemble -> loss without leaving HBM.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import torch

from . import _lib
from .core import EpisodeTable, Level, RolloutBuffer, _ptr

TOY_REACH, SCRIPTED = 0, 1


@dataclass
class EnvConfig:
    """envsim::VecEnvConfig (vec_env.hpp:16-35) + RolloutSpec::reset_mode."""
    kind: int = TOY_REACH
    num_envs: int = 4
    max_episode_steps: int = 8
    auto_reset: bool = True
    ignore_terminations: bool = False
    use_fixed_reset_state_ids: bool = False
    chunk_len: int = 2
    grid_size: int = 5
    reward_shaping: bool = False
    num_reset_states: int = 64
    success_step: int = 5
    deferred_reset: bool = False
    seed: int = 0

    @property
    def obs_dim(self) -> int:
        return 6 if self.kind == TOY_REACH else 2

    def c(self) -> _lib.EnvConfig:
        return _lib.EnvConfig(self.kind, self.num_envs, self.max_episode_steps,
                              int(self.auto_reset), int(self.ignore_terminations),
                              int(self.use_fixed_reset_state_ids), self.chunk_len,
                              self.grid_size, int(self.reward_shaping), self.num_reset_states,
                              self.success_step, int(self.deferred_reset), self.seed)


@dataclass
class PolicyDescriptor:
    """policy::PolicyDescriptor (policy_net.hpp:15-26)."""
    obs_dim: int
    hidden: int = 16
    trunk_layers: int = 1
    value_hidden: int = 16
    vocab: int = 16
    chunk_len: int = 2
    tokens_per_action: int = 2

    def c(self) -> _lib.PolicyDesc:
        return _lib.PolicyDesc(self.obs_dim, self.hidden, self.trunk_layers, self.value_hidden,
                               self.vocab, self.chunk_len, self.tokens_per_action)

    def num_params(self) -> int:
        return int(_lib.lib().ckrl_policy_num_params(C.byref(self.c())))


def random_params(desc: PolicyDescriptor, seed: int = 0, scale: float = 0.3,
                  device="cuda") -> torch.Tensor:
    """Synthetic f64 policy parameters in the reference's flat layout (random-init: the
    bench has no checkpoint)."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    return (torch.randn(desc.num_params(), generator=g, dtype=torch.float64) * scale).to(device)


@dataclass
class RolloutEpoch:
    """One epoch's outputs: the SoA slab (f32 + f64 copies) and the episode table."""
    t: dict
    episodes: EpisodeTable
    vocab: int

    def buffer(self, advantage_level: int = Level.Chunk) -> RolloutBuffer:
        """The slab as the loss path's RolloutBuffer; the bootstrap column follows
        assembler.cpp:98-104 (scalar head for chunk-level advantages, vector head [0] else)."""
        t = self.t
        boot = t["boot_scalar"] if int(advantage_level) == int(Level.Chunk) else t["boot_vector0"]
        return RolloutBuffer(tokens=t["tokens"], old_logprob=t["old_logprob"],
                             reward=t["reward"], flags=t["flags"], episode_id=t["episode_id"],
                             value_scalar=t["value_scalar"], value_vector=t["value_vector"],
                             bootstrap=boot, vocab=self.vocab)


SAMPLER_REFERENCE, SAMPLER_PARALLEL = _lib.SAMPLER_REFERENCE, _lib.SAMPLER_PARALLEL
COLOCATED, DISAGGREGATED, HYBRID = (_lib.PLACEMENT_COLOCATED, _lib.PLACEMENT_DISAGGREGATED,
                                    _lib.PLACEMENT_HYBRID)


def derive_mode(num_slots: int, env_slots, rollout_slots, actor_slots, pipeline_stage_num: int = 1) -> int:
    """placement::derive_mode after validate_plan (placement/plan.cpp:49-68) on inclusive slot
    ranges ("0-3" strings or (begin, end) pairs): COLOCATED / DISAGGREGATED / HYBRID; raises
    InvalidPlan like the reference."""
    def rng(r):
        if isinstance(r, str):
            b, _, e = r.partition("-")
            return int(b), int(e or b)
        return int(r[0]), int(r[1])
    (eb, ee), (rb, re_), (ab, ae) = rng(env_slots), rng(rollout_slots), rng(actor_slots)
    st = C.c_int32(0)
    m = _lib.lib().ckrl_placement_mode(num_slots, eb, ee, rb, re_, ab, ae, pipeline_stage_num, C.byref(st))
    _lib.check(st.value)
    return int(m)


class RolloutPipeline:
    """RealBackend::run_rollout_epoch with `stages` pipeline partitions. gen_device=None is
    the colocated placement (env and generation kernels on `device`); an int places the
    generation role on that device (hybrid / disaggregated: obs and action batches cross
    between the devices every chunk; it may equal `device`). `sampler` picks the reference-
    order serial sampler (bit-exact with sample_chunk) or the warp-parallel one."""

    def __init__(self, env: EnvConfig, policy: PolicyDescriptor, num_chunks: int,
                 stages: int = 1, sample_seed: int = 0,
                 reset_state_ids: Optional[torch.Tensor] = None, device="cuda",
                 keep_logits: bool = False, sampler: int = SAMPLER_REFERENCE,
                 gen_device: Optional[int] = None):
        self.env, self.policy, self.num_chunks, self.stages = env, policy, num_chunks, stages
        self.sample_seed = sample_seed
        self.device = torch.device(device)
        self.reset_ids = (None if reset_state_ids is None else
                          torch.as_tensor(reset_state_ids, dtype=torch.int32).to(self.device))
        self.spec = _lib.PipelineSpec(env.c(), policy.c(), num_chunks, stages, sample_seed,
                                      _ptr(self.reset_ids), int(sampler), int(gen_device is not None),
                                      0 if gen_device is None else int(gen_device), None, 0)
        self._lib = _lib.lib()
        nbytes = int(self._lib.ckrl_pipeline_workspace_bytes(C.byref(self.spec)))
        if nbytes == 0:  # invalid spec: re-run validation to raise the reference's exception
            _lib.check(self._lib.ckrl_pipeline_run(C.byref(self.spec), None, None, None, 0, None))
        self.gen_ws = None
        if gen_device is not None:
            gb = int(self._lib.ckrl_pipeline_gen_workspace_bytes(C.byref(self.spec)))
            self.gen_ws = torch.empty(gb, dtype=torch.uint8, device=torch.device("cuda", int(gen_device)))
            self.spec.gen_workspace = _ptr(self.gen_ws)
            self.spec.gen_workspace_bytes = gb
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.keep_logits = keep_logits
        self.out = self._alloc()
        self.c_out = _lib.PipelineOutputs(*[_ptr(self.out[n])
                                            for n in _lib.PIPELINE_OUTPUT_FIELDS])

    def _alloc(self) -> dict:
        E, T, Cn, M = self.env.num_envs, self.num_chunks, self.env.chunk_len, \
            self.policy.tokens_per_action
        cap = E * (T * Cn + 1)
        dev = self.device
        f32, f64, i32, u8 = torch.float32, torch.float64, torch.int32, torch.uint8

        def z(shape, dt):
            return torch.zeros(shape, dtype=dt, device=dev)
        o = dict(tokens=z((E, T, Cn, M), i32), old_logprob=z((E, T, Cn, M), f32),
                 old_logprob_f64=z((E, T, Cn, M), f64), reward=z((E, T, Cn), f32),
                 reward_f64=z((E, T, Cn), f64), flags=z((E, T, Cn), u8),
                 episode_id=z((E, T, Cn), i32), value_scalar=z((E, T), f32),
                 value_scalar_f64=z((E, T), f64))
        for n in ("value_vector", "boot_scalar", "boot_vector0"):
            o[n] = z((E, T, Cn), f32)
            o[n + "_f64"] = z((E, T, Cn), f64)
        o.update(episode_count=z(1, i32), ep_env_id=z(cap, i32), ep_episode_id=z(cap, i32),
                 ep_start=z(cap, i32), ep_length=z(cap, i32), ep_total_reward=z(cap, f64),
                 ep_first_success=z(cap, i32), ep_complete=z(cap, u8), ep_task=z(cap, i32),
                 ep_reset_id=z(cap, i32), status=z(1, i32))
        o["logits"] = (torch.empty((E, T, Cn, M, self.policy.vocab), dtype=f32, device=dev)
                       if self.keep_logits else None)
        return o

    def launch(self, params: torch.Tensor, stream: Optional[torch.cuda.Stream] = None):
        """Enqueue one epoch (no host sync). `params`: f64 device vector."""
        assert params.dtype == torch.float64 and params.is_cuda
        assert params.numel() == self.policy.num_params(), "parameter count mismatch"
        s = stream or torch.cuda.current_stream(self.device)
        _lib.check(self._lib.ckrl_pipeline_run(C.byref(self.spec), _ptr(params),
                                               C.byref(self.c_out), _ptr(self.ws),
                                               self.ws.numel(), C.c_void_p(s.cuda_stream)))

    def run(self, params: torch.Tensor) -> RolloutEpoch:
        """One epoch; syncs once to size the episode table and to raise BadResetId."""
        self.launch(params)
        st = int(self.out["status"].item())
        if st:
            from . import errors
            raise errors.from_status(st, "reset state id out of range / missing (vec_env.cpp:74-90)")
        n = int(self.out["episode_count"].item())
        o = self.out
        eps = EpisodeTable(env_id=o["ep_env_id"][:n], episode_id=o["ep_episode_id"][:n],
                           start_step=o["ep_start"][:n], length=o["ep_length"][:n],
                           total_reward=o["ep_total_reward"][:n],
                           first_success=o["ep_first_success"][:n],
                           complete=o["ep_complete"][:n], task_id=o["ep_task"][:n],
                           reset_state_id=o["ep_reset_id"][:n])
        return RolloutEpoch(t=dict(o), episodes=eps, vocab=self.policy.vocab)
