"""Row f3: wire and on-disk formats of the SoA slab and the policy parameters (host side of
the C ABI; no device needed): the reference's trajectories dump (core/types.cpp:9-28) and its
CKRL checkpoint (policy/checkpoint.cpp:37-83)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def _np(a, dtype):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    return np.ascontiguousarray(a, dtype=dtype)


def dump_slab(tokens, reward_f64, flags, episode_id, first_env_id: int = 0) -> str:
    """dump_slab text of an SoA slab: tokens [E][Tc][C][M] (u8/i32), f64 rewards [E][Tc][C]
    (e.g. the pipeline's reward_f64), flags, episode ids (uid & 0xffffffff, -1 frozen);
    uids are (first_env_id + row) << 32 | id (a VecEnv partition / rank shard starting at
    global env first_env_id, vec_env.cpp:94). Tensors are read from wherever they live
    (device tensors are downloaded)."""
    tk = tokens.detach().cpu().numpy() if hasattr(tokens, "detach") else np.asarray(tokens)
    E, Tc, Cn, M = tk.shape
    td = _lib.DTYPE_U8 if tk.dtype == np.uint8 else _lib.DTYPE_I32
    tk = np.ascontiguousarray(tk, np.uint8 if td == _lib.DTYPE_U8 else np.int32)
    rw, fl, ids = _np(reward_f64, np.float64), _np(flags, np.uint8), _np(episode_id, np.int32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    n = C.c_size_t(0)
    f = _lib.lib().ckrl_dump_slab
    _lib.check(f(E, Tc, Cn, M, td, p(tk), p(rw), p(fl), p(ids), first_env_id, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _lib.check(f(E, Tc, Cn, M, td, p(tk), p(rw), p(fl), p(ids), first_env_id, buf, n.value + 1,
                 C.byref(n)))
    return buf.raw[:n.value].decode()


def save_checkpoint(desc, params, path: str) -> None:
    """save_checkpoint: `desc` a pipeline.PolicyDescriptor, params its flat f64 vector."""
    pr = _np(params, np.float64)
    _lib.check(_lib.lib().ckrl_save_checkpoint(C.byref(desc.c()), pr.ctypes.data_as(C.c_void_p),
                                               path.encode()))


def load_checkpoint(path: str):
    """load_checkpoint -> (PolicyDescriptor, f64 params); raises the reference's Error cases."""
    from .pipeline import PolicyDescriptor
    d = _lib.PolicyDesc()
    cnt = C.c_int64(0)
    _lib.check(_lib.lib().ckrl_load_checkpoint(path.encode(), C.byref(d), None, 0, C.byref(cnt)))
    params = np.zeros(cnt.value)
    _lib.check(_lib.lib().ckrl_load_checkpoint(path.encode(), C.byref(d), params.ctypes.data_as(C.c_void_p),
                                               cnt.value, C.byref(cnt)))
    desc = PolicyDescriptor(obs_dim=d.obs_dim, hidden=d.hidden, trunk_layers=d.trunk_layers,
                            value_hidden=d.value_hidden, vocab=d.vocab, chunk_len=d.chunk_len,
                            tokens_per_action=d.tokens_per_action)
    return desc, params
