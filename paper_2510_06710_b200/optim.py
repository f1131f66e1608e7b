"""Loss operators (chunkrl::optim) on the B200: whitening, fused PPO / GRPO loss and the
whole advantage->loss step. Names and argument meaning follow optim/update.hpp and
optim/losses.hpp; the one unavoidable change is that the loss consumes the current
policy's outputs (logits, values) instead of re-running a PolicyNet."""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import _lib
from .core import (EpisodeTable, GaeParams, GranularitySpec, GrpoAssemblyOptions, GrpoBatch,
                   GrpoParams, Level, LossOutputs, PolicyOutputs, PpoBatch, PpoParams,
                   RolloutBuffer, Workspace, read_diagnostics, stream_ptr)


def _diag_buffer(device):
    return torch.zeros(_lib.DIAG_COUNT, dtype=torch.float64, device=device)


def normalize_advantages(rollout: RolloutBuffer, batch: PpoBatch, stream=None) -> None:
    """normalize_advantages (optim/update.cpp:14-45), in place on batch.advantages."""
    bc = batch.c()
    _lib.check(_lib.lib().ckrl_normalize_advantages(C.byref(rollout.c()), C.byref(batch.spec.c()),
                                                    C.byref(bc), batch.workspace.ptr,
                                                    batch.workspace.bytes, stream_ptr(stream)))


def ppo_loss(rollout: RolloutBuffer, policy: PolicyOutputs, batch: PpoBatch,
             params: PpoParams = PpoParams(), outputs: Optional[LossOutputs] = None,
             diag: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """ppo_loss (optim/losses.cpp:62-232) over every record. Whitening (update.cpp:66-67)
    is applied on the fly when params.advantage_normalization. Returns the device
    diagnostics vector; read it with core.read_diagnostics()."""
    diag = diag if diag is not None else _diag_buffer(rollout.tokens.device)
    bc = batch.c()
    oc = outputs.c() if outputs is not None else None
    _lib.check(_lib.lib().ckrl_ppo_loss(C.byref(rollout.c()), C.byref(bc), C.byref(policy.c()),
                                        C.byref(batch.spec.c()), C.byref(params.c()),
                                        C.byref(oc) if oc is not None else None,
                                        C.c_void_p(diag.data_ptr()), batch.workspace.ptr,
                                        batch.workspace.bytes, stream_ptr(stream)))
    return diag


def grpo_loss(rollout: RolloutBuffer, policy: PolicyOutputs, batch: GrpoBatch,
              params: GrpoParams = GrpoParams(), outputs: Optional[LossOutputs] = None,
              diag: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """grpo_loss (optim/losses.cpp:234-331) over every retained group."""
    diag = diag if diag is not None else _diag_buffer(rollout.tokens.device)
    bc = batch.c()
    oc = outputs.c() if outputs is not None else None
    _lib.check(_lib.lib().ckrl_grpo_loss(C.byref(rollout.c()), C.byref(bc), C.byref(policy.c()),
                                         C.byref(batch.spec.c()), C.byref(params.c()),
                                         C.byref(oc) if oc is not None else None,
                                         C.c_void_p(diag.data_ptr()), batch.workspace.ptr,
                                         batch.workspace.bytes, stream_ptr(stream)))
    return diag


class PpoStep:
    """The measured hot path: assemble_ppo_batch -> [NCCL stats all-gather] -> fused loss.
    Buffers are allocated once; __call__ only launches kernels (2 per step on 1 GPU)."""

    def __init__(self, rollout: RolloutBuffer, gae: GaeParams, spec: GranularitySpec,
                 params: PpoParams, outputs: bool = True, comm=None):
        E, Tc, Cn, M = rollout.shape
        dev = rollout.tokens.device
        world = comm.world if comm is not None else 1
        self.ws = Workspace(E, world, dev)
        shape = (E, Tc) if spec.advantage_level == Level.Chunk else (E, Tc, Cn)
        self.batch = PpoBatch(spec=spec,
                              counted=torch.empty((E, Tc, Cn), dtype=torch.uint8, device=dev),
                              advantages=torch.empty(shape, dtype=torch.float32, device=dev),
                              returns=torch.empty(shape, dtype=torch.float32, device=dev),
                              workspace=self.ws)
        self.outputs = LossOutputs.allocate(rollout, spec.value_level) if outputs else None
        self.diag = _diag_buffer(dev)
        self.gae, self.spec, self.params, self.comm = gae.c(), spec.c(), params.c(), comm
        self._bc = self.batch.c()
        self._oc = self.outputs.c() if outputs else None

    def __call__(self, rollout: RolloutBuffer, policy: PolicyOutputs, stream=None):
        _lib.check(_lib.lib().ckrl_ppo_step(
            C.byref(rollout.c()), C.byref(policy.c()), C.byref(self.gae), C.byref(self.spec),
            C.byref(self.params), C.byref(self._bc),
            C.byref(self._oc) if self._oc is not None else None, C.c_void_p(self.diag.data_ptr()),
            self.ws.ptr, self.ws.bytes, self.comm.handle if self.comm is not None else None,
            stream_ptr(stream)))
        return self.diag

    def diagnostics(self, stream=None) -> dict:
        return read_diagnostics(self.diag, stream)


class GrpoStep:
    """assemble_grpo_batch -> [NCCL stats all-gather] -> fused GRPO loss (3 launches)."""

    def __init__(self, rollout: RolloutBuffer, options: GrpoAssemblyOptions, params: GrpoParams,
                 outputs: bool = True, comm=None):
        E = rollout.shape[0]
        dev = rollout.tokens.device
        world = comm.world if comm is not None else 1
        self.ws = Workspace(E, world, dev)
        self.batch = GrpoBatch.allocate(rollout, options.spec, self.ws)
        self.outputs = LossOutputs.allocate(rollout, Level.Chunk) if outputs else None
        self.diag = _diag_buffer(dev)
        self.options, self.params, self.comm = options, params.c(), comm
        self._opt = options.c()
        self._spec = options.spec.c()
        self._bc = self.batch.c()
        self._oc = self.outputs.c() if outputs else None

    def __call__(self, rollout: RolloutBuffer, episodes: EpisodeTable, policy: PolicyOutputs,
                 stream=None):
        _lib.check(_lib.lib().ckrl_grpo_step(
            C.byref(rollout.c()), C.byref(episodes.c()), C.byref(policy.c()),
            C.byref(self._spec), C.byref(self._opt), C.byref(self.params), C.byref(self._bc),
            C.byref(self._oc) if self._oc is not None else None, C.c_void_p(self.diag.data_ptr()),
            self.ws.ptr, self.ws.bytes, self.comm.handle if self.comm is not None else None,
            stream_ptr(stream)))
        return self.diag

    def diagnostics(self, stream=None) -> dict:
        return read_diagnostics(self.diag, stream)
