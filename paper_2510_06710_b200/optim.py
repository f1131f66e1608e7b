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


def ppo_loss_minibatch(rollout: RolloutBuffer, policy: PolicyOutputs, batch: PpoBatch,
                       record_indices, params: PpoParams = PpoParams(), stream=None) -> dict:
    """ppo_loss (losses.cpp:62-232) over `record_indices` (record = env * Tc + chunk), the
    minibatch form update_ppo drives (update.cpp:83-99). Like the reference, the batch's
    advantages are used as they are: whiten them once beforehand with
    normalize_advantages (update.cpp:66-67). Returns the host diagnostics."""
    E, Tc, Cn, M = rollout.shape
    dev = rollout.tokens.device
    idx = torch.as_tensor(record_indices, dtype=torch.int64).to(dev).contiguous()
    n = idx.numel()
    V = rollout.vocab
    spec = batch.spec
    ulen = Cn if spec.advantage_level == Level.Action else 1
    vlen = Cn if spec.value_level == Level.Action else 1
    f32 = dict(dtype=torch.float32, device=dev)
    sub = RolloutBuffer(tokens=torch.empty((n, 1, Cn, M), dtype=rollout.tokens.dtype, device=dev),
                        old_logprob=torch.empty((n, 1, Cn, M), **f32),
                        reward=torch.empty((n, 1, Cn), **f32),
                        flags=torch.empty((n, 1, Cn), dtype=torch.uint8, device=dev),
                        episode_id=torch.empty((n, 1, Cn), dtype=torch.int32, device=dev),
                        value_scalar=torch.empty((n, 1), **f32),
                        value_vector=torch.empty((n, 1, Cn), **f32),
                        bootstrap=torch.empty((n, 1, Cn), **f32), vocab=V)
    ws = Workspace(n, 1, dev)
    sb = PpoBatch(spec=spec, counted=torch.empty((n, 1, Cn), dtype=torch.uint8, device=dev),
                  advantages=torch.empty((n, 1, ulen) if ulen > 1 else (n, 1), dtype=torch.float64, device=dev),
                  returns=torch.empty((n, 1, ulen) if ulen > 1 else (n, 1), dtype=torch.float64, device=dev),
                  workspace=ws)
    sp = PolicyOutputs(torch.empty((n, 1, Cn, M, V), dtype=policy.logits.dtype, device=dev),
                       torch.empty((n, 1, vlen) if vlen > 1 else (n, 1), **f32)
                       if policy.values is not None else None)
    _lib.check(_lib.lib().ckrl_select_records(
        C.byref(rollout.c()), C.byref(batch.c()), C.byref(policy.c()), C.byref(spec.c()), n,
        C.c_void_p(idx.data_ptr()), C.byref(sub.c()), C.byref(sb.c()), C.byref(sp.c()), ws.ptr,
        ws.bytes, stream_ptr(stream)))
    p = PpoParams(params.clip_eps, params.value_loss_coef, params.entropy_coef, False)
    return read_diagnostics(ppo_loss(sub, sp, sb, p, stream=stream), stream)


def grpo_loss_minibatch(rollout: RolloutBuffer, policy: PolicyOutputs, batch: GrpoBatch,
                        group_indices, params: GrpoParams = GrpoParams(), stream=None) -> dict:
    """grpo_loss (losses.cpp:234-331) over `group_indices` (retained-group ordinals in
    GroupKey order), the minibatch form of update_grpo (update.cpp:123-160). Raises
    SkipUpdate on an empty selection like the reference."""
    from .errors import SkipUpdate
    dev = rollout.tokens.device
    sel = torch.as_tensor(group_indices, dtype=torch.int32).to(dev).contiguous()
    if sel.numel() == 0:
        raise SkipUpdate("grpo_loss: no groups selected")
    ws = Workspace(batch.workspace.num_envs, 1, dev)
    ws.tensor.copy_(batch.workspace.tensor)
    env_group = torch.empty_like(batch.env_group)
    E = batch.env_group.numel()
    _lib.check(_lib.lib().ckrl_select_groups(E, C.c_void_p(batch.env_group.data_ptr()),
                                             C.c_void_p(env_group.data_ptr()), sel.numel(),
                                             C.c_void_p(sel.data_ptr()), ws.ptr, ws.bytes,
                                             stream_ptr(stream)))
    sub = GrpoBatch(spec=batch.spec, env_group=env_group, env_member=batch.env_member,
                    env_episode=batch.env_episode, env_advantage=batch.env_advantage,
                    env_group_size=batch.env_group_size, slot_weight=batch.slot_weight,
                    slot_member=batch.slot_member, group_counts=batch.group_counts, workspace=ws)
    return read_diagnostics(grpo_loss(rollout, policy, sub, params, stream=stream), stream)


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
                              advantages=torch.empty(shape, dtype=torch.float64, device=dev),
                              returns=torch.empty(shape, dtype=torch.float64, device=dev),
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

    # the two halves (ckrl_ppo_step_assemble / _loss) for pipelining batches across streams
    def assemble(self, rollout: RolloutBuffer, stream=None):
        _lib.check(_lib.lib().ckrl_ppo_step_assemble(
            C.byref(rollout.c()), C.byref(self.gae), C.byref(self.spec), C.byref(self._bc), self.ws.ptr,
            self.ws.bytes, self.comm.handle if self.comm is not None else None, stream_ptr(stream)))

    def loss(self, rollout: RolloutBuffer, policy: PolicyOutputs, stream=None):
        _lib.check(_lib.lib().ckrl_ppo_step_loss(
            C.byref(rollout.c()), C.byref(policy.c()), C.byref(self.spec), C.byref(self.params),
            C.byref(self._bc), C.byref(self._oc) if self._oc is not None else None,
            C.c_void_p(self.diag.data_ptr()), self.ws.ptr, self.ws.bytes,
            self.comm.handle if self.comm is not None else None, stream_ptr(stream)))
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

    # the two halves (ckrl_grpo_step_assemble / _loss) for pipelining batches across streams
    def assemble(self, rollout: RolloutBuffer, episodes: EpisodeTable, stream=None):
        _lib.check(_lib.lib().ckrl_grpo_step_assemble(
            C.byref(rollout.c()), C.byref(episodes.c()), C.byref(self._spec), C.byref(self._opt),
            C.byref(self._bc), self.ws.ptr, self.ws.bytes,
            self.comm.handle if self.comm is not None else None, stream_ptr(stream)))

    def loss(self, rollout: RolloutBuffer, policy: PolicyOutputs, stream=None):
        _lib.check(_lib.lib().ckrl_grpo_step_loss(
            C.byref(rollout.c()), C.byref(policy.c()), C.byref(self._spec), C.byref(self.params),
            C.byref(self._bc), C.byref(self._oc) if self._oc is not None else None,
            C.c_void_p(self.diag.data_ptr()), self.ws.ptr, self.ws.bytes,
            self.comm.handle if self.comm is not None else None, stream_ptr(stream)))
        return self.diag

    def diagnostics(self, stream=None) -> dict:
        return read_diagnostics(self.diag, stream)


class Pipelined:
    """Steps over a stream of batches with batch i+1's assembly on a side stream overlapping
    batch i's loss (the two halves of PpoStep / GrpoStep, one step object per in-flight batch
    slot: its workspace and batch buffers). Every batch still gets its full assembly and loss;
    only their placement in time changes. `issue(K, args_of)` enqueues K batches on the
    current stream (graph-capturable); batch i uses steps[i % len(steps)] and
    args_of(i) -> (assemble args, loss args)."""

    def __init__(self, steps, loss_streams: int = 3):
        """loss_streams = n > 1 rotates the losses over the current stream and n - 1 more, so
        batch i+1's loss depends only on its own assembly (not on batch i's loss): its CTAs
        start and run their unit phases while batch i's last CTAs finish (with the library's
        capped loss grids, side by side on disjoint SMs). Default 3: measured 1-3 % faster than 2
        for cfg3 / cfg2 and 10 % for cfg3 bf16 (with the 8..12-tiles-per-SM grid cap)."""
        import torch
        self.steps = steps
        self.alts = [torch.cuda.Stream() for _ in range(max(1, loss_streams) - 1)]
        # across ranks the exchange holds two batches in flight: an assembly may only start
        # once the loss two batches back has completed (ckrl.h, ckrl_ppo_step_assemble)
        self.multi_rank = any(getattr(st, "comm", None) is not None and st.comm.world > 1 for st in steps)
        self.side = torch.cuda.Stream()
        n = len(steps)
        self.ev_asm = [torch.cuda.Event() for _ in range(n)]
        self.ev_loss = [torch.cuda.Event() for _ in range(n)]

    def issue(self, K: int, args_of, loss_events=None):
        import torch
        n = len(self.steps)
        main = torch.cuda.current_stream()
        side = self.side
        side.wait_stream(main)

        def asm(j):
            a_args, _ = args_of(j)
            # slot reuse: loss j - n done; exchange: at most one batch ahead (loss j - 2 done)
            for back in ((n, 2) if self.multi_rank else (n,)):
                if j >= back:
                    side.wait_event(self.ev_loss[(j - back) % n])
            self.steps[j % n].assemble(*a_args, stream=side)
            self.ev_asm[j % n].record(side)

        for st in self.alts:
            st.wait_stream(main)
        with torch.cuda.stream(side):
            asm(0)
        for i in range(K):
            if i + 1 < K:
                with torch.cuda.stream(side):
                    asm(i + 1)
            _, l_args = args_of(i)
            q = i % (len(self.alts) + 1)
            ls = main if q == 0 else self.alts[q - 1]
            ls.wait_event(self.ev_asm[i % n])
            if loss_events is not None:  # (start, end) timing events around each loss launch
                loss_events[i][0].record(ls)
            with torch.cuda.stream(ls):
                self.steps[i % n].loss(*l_args, stream=ls)
            if loss_events is not None:
                loss_events[i][1].record(ls)
            self.ev_loss[i % n].record(ls)
        main.wait_stream(side)
        for st in self.alts:
            main.wait_stream(st)


class AdamParamsC(C.Structure):
    _fields_ = [("learning_rate", C.c_double), ("max_grad_norm", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("eps", C.c_double)]


class Adam:
    """optim::Adam (optim/adam.hpp:10-27): plain Adam with optional global gradient-norm
    clipping, on device tensors. step(params, grad) clips grad in place when
    max_grad_norm > 0, updates params, and returns the pre-clip gradient norm (a host float,
    like the reference; raises NonFinite without modifying anything when it is not finite).
    step_async leaves the norm / status on the device (no host sync). State dtype follows the
    parameters: float32, or float64 for the reference's precision. With `comm` (parameters
    sharded across ranks) ||g||^2 is all-reduced over NCCL."""

    def __init__(self, num_params: int, learning_rate: float, max_grad_norm: float = 0.0,
                 beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8, device="cuda",
                 dtype=torch.float32, comm=None):
        self.m = torch.zeros(num_params, dtype=dtype, device=device)
        self.v = torch.zeros(num_params, dtype=dtype, device=device)
        self.t = 0
        self.params = AdamParamsC(learning_rate, max_grad_norm, beta1, beta2, eps)
        nb = _lib.lib().ckrl_adam_workspace_bytes()
        self.ws = torch.zeros(int(nb), dtype=torch.uint8, device=device)
        self.norm = torch.zeros(1, dtype=torch.float64, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self.comm = comm

    def step_async(self, params: torch.Tensor, grad: torch.Tensor, stream=None) -> None:
        n = self.m.numel()
        if params.numel() != n or grad.numel() != n:
            from .errors import LengthMismatch
            raise LengthMismatch("Adam buffer size mismatch")
        if params.dtype != self.m.dtype or grad.dtype != self.m.dtype:
            raise TypeError("params / grad dtype must match the optimizer state")
        dt = _lib.DTYPE_F64 if self.m.dtype == torch.float64 else _lib.DTYPE_F32
        _lib.check(_lib.lib().ckrl_adam_step(
            dt, n, C.c_void_p(params.data_ptr()), C.c_void_p(grad.data_ptr()),
            C.c_void_p(self.m.data_ptr()), C.c_void_p(self.v.data_ptr()), C.byref(self.params),
            self.t + 1, C.c_void_p(self.norm.data_ptr()), C.c_void_p(self.status.data_ptr()),
            C.c_void_p(self.ws.data_ptr()), self.ws.numel(),
            self.comm.handle if self.comm is not None else None, stream_ptr(stream)))
        self.t += 1

    def step(self, params: torch.Tensor, grad: torch.Tensor, stream=None) -> float:
        self.status.zero_()
        self.step_async(params, grad, stream)
        st = _lib.lib().ckrl_read_status(C.c_void_p(self.status.data_ptr()), stream_ptr(stream))
        if st:
            self.t -= 1  # the reference throws before ++t_ (adam.cpp:21-28)
            _lib.check(st)
        return float(self.norm.item())
