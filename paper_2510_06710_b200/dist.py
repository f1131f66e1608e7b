"""Multi-GPU plumbing: env / group sharding and the NCCL communicator used by the step.

The path shards by environment (GAE segments never cross envs, assembler.cpp:108-193)
and, for GRPO, by whole groups (GroupKey, assembler.cpp:207-226). The only exchanges are
the 64-byte per-rank stats record before the loss (whitening moments + normalisers or the
retained-group count) and the loss scalars after it — both inside the step's two kernels,
as NVLink stores into every rank's exchange buffer (csrc/common.cuh ExSlot). torch.distributed
only bootstraps the communicator: it all-gathers the buffers' CUDA IPC handles (and, for a
sharded Adam step, broadcasts an NCCL unique id).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError


def env_shard(num_envs: int, world: int, rank: int, group_size: int = 1) -> range:
    """Contiguous env range of `rank`; GRPO groups (group_size consecutive envs sharing a
    reset id, train.cpp:92-101) are never split across ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError("bad world/rank")
    if num_envs % group_size:
        raise ConfigError("num_envs must be a multiple of group_size")
    groups = num_envs // group_size
    base, extra = divmod(groups, world)
    g0 = rank * base + min(rank, extra)
    g1 = g0 + base + (1 if rank < extra else 0)
    return range(g0 * group_size, g1 * group_size)


def key_shard(env_keys, world: int):
    """Shard envs by GRPO GroupKey (task_id, reset_state_id; assembler.cpp:207-226): every key's
    envs land on one rank, so each rank's std::map grouping is the global grouping restricted
    to its keys and only the retained-group count crosses ranks. `env_keys` is one key per env
    (its grouped episode's key; envs drawing reset ids with replacement share keys across
    non-adjacent envs, train.cpp:92-101). Keys are placed largest first on the least-loaded
    rank (ties: lower rank, then key order), deterministic. Returns one ascending env-index
    array per rank."""
    if world < 1:
        raise ConfigError("bad world")
    keys = [tuple(np.atleast_1d(k).tolist()) for k in env_keys]
    members = {}
    for e, k in enumerate(keys):
        members.setdefault(k, []).append(e)
    load = [0] * world
    parts = [[] for _ in range(world)]
    for k in sorted(members, key=lambda q: (-len(members[q]), q)):
        r = min(range(world), key=lambda i: (load[i], i))
        parts[r].extend(members[k])
        load[r] += len(members[k])
    return [np.array(sorted(p), dtype=np.int64) for p in parts]


def check_group_sharding(env_of_episode, key_of_episode, world: int, shard_of_env) -> None:
    """Raises ConfigError if any GroupKey (task, reset id) has members on two ranks: the
    rank-local grouping would then differ from the reference's global std::map grouping."""
    owner = {}
    for e, k in zip(np.asarray(env_of_episode).tolist(), [tuple(x) for x in np.asarray(key_of_episode).tolist()]):
        r = shard_of_env(e)
        if owner.setdefault(k, r) != r:
            raise ConfigError(f"group key {k} spans ranks {owner[k]} and {r}")


@dataclass
class StatsRecord:
    """Host view of the 64-byte record ranks all-gather (csrc/common.cuh StatsRecord):
    the advantage-unit moments (mean, M2 = sum of squared deviations) and the normalisers."""
    mean: float = 0.0
    m2: float = 0.0
    flags: int = 0
    n_adv: int = 0
    n_val: int = 0
    n_pos: int = 0
    groups_retained: int = 0
    status: int = 0

    DTYPE = np.dtype([("mean", "<f8"), ("m2", "<f8"), ("flags", "<i8"), ("n_adv", "<i8"),
                      ("n_val", "<i8"), ("n_pos", "<i8"), ("groups_retained", "<i8"),
                      ("status", "<i8")])

    def to_bytes(self) -> bytes:
        a = np.zeros(1, self.DTYPE)
        for k in self.DTYPE.names:
            a[k] = getattr(self, k)
        return a.tobytes()

    @classmethod
    def from_bytes(cls, raw: bytes) -> "StatsRecord":
        a = np.frombuffer(raw, cls.DTYPE, count=1)[0]
        return cls(*(a[k].item() for k in cls.DTYPE.names))

    @classmethod
    def from_units(cls, adv_units, n_val, n_pos, groups=0):
        a = np.asarray(adv_units, dtype=np.float64)
        n = a.size
        mean = float(a.mean()) if n else 0.0
        return cls(mean, float(((a - mean) ** 2).sum()) if n else 0.0, 0, n, int(n_val), int(n_pos),
                   int(groups), 0)


def merge_stats(records) -> dict:
    """Merges per-rank records in rank order with the same code the device uses
    (ckrl_merge_stats_host: Chan's pairwise moment update in rank order, then mean /
    population std + 1e-8)."""
    raw = b"".join(r.to_bytes() if isinstance(r, StatsRecord) else bytes(r) for r in records)
    assert _lib.lib().ckrl_stats_record_bytes() == StatsRecord.DTYPE.itemsize
    buf = C.create_string_buffer(raw, len(raw))
    mean, denom = C.c_double(), C.c_double()
    counts = (C.c_int64 * 4)()
    _lib.check(_lib.lib().ckrl_merge_stats_host(buf, len(records), C.byref(mean), C.byref(denom),
                                                counts))
    return {"mean": mean.value, "denom": denom.value, "n_adv": counts[0], "n_val": counts[1],
            "n_pos": counts[2], "groups_retained": counts[3]}


class Comm:
    """One rank's ckrl_comm: its exchange buffer (peer-mapped into every rank) and, when
    `unique_id` is given, an NCCL communicator for the sharded Adam step."""

    def __init__(self, world: int, rank: int, unique_id: bytes | None = None):
        self.world, self.rank = world, rank
        h = C.c_void_p()
        uid = C.create_string_buffer(unique_id, 128) if unique_id is not None else None
        _lib.check(_lib.lib().ckrl_comm_create(world, rank, uid, C.byref(h)))
        self.handle = h

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _lib.check(_lib.lib().ckrl_comm_unique_id(buf))
        return buf.raw

    def ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(IPC_HANDLE_BYTES)
        _lib.check(_lib.lib().ckrl_comm_ipc_handle(self.handle, buf))
        return buf.raw

    def open_peers(self, handles) -> None:
        """Maps every other rank's exchange buffer (CUDA IPC handles in rank order)."""
        if len(handles) != self.world or any(len(h) != IPC_HANDLE_BYTES for h in handles):
            raise ConfigError("need one IPC handle per rank")
        raw = b"".join(handles)
        _lib.check(_lib.lib().ckrl_comm_open_peers(self.handle, C.create_string_buffer(raw, len(raw))))

    def set_peers(self, comms) -> None:
        arr = (C.c_void_p * self.world)(*[c.handle.value for c in comms])
        _lib.check(_lib.lib().ckrl_comm_set_peers(self.handle, arr))

    @classmethod
    def from_torch(cls, nccl: bool = False) -> "Comm":
        """Collective over the default torch.distributed group: creates this rank's comm and
        maps every rank's exchange buffer."""
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        uid = None
        if nccl:
            obj = [cls.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        c = cls(world, rank, uid)
        if world > 1:
            handles = [None] * world
            dist.all_gather_object(handles, c.ipc_handle())
            c.open_peers(handles)
        return c

    @classmethod
    def local_group(cls, world: int, devices=None) -> list:
        """`world` ranks driven by this one process (one per device in `devices`, or all on
        the current device): the exchange runs through the same kernels as across processes."""
        import torch
        cur = torch.cuda.current_device()
        comms = []
        for r in range(world):
            torch.cuda.set_device(devices[r] if devices else cur)
            comms.append(cls(world, r))
        for r, c in enumerate(comms):
            torch.cuda.set_device(devices[r] if devices else cur)
            c.set_peers(comms)
        torch.cuda.set_device(cur)
        return comms

    def close(self):
        if self.handle:
            _lib.lib().ckrl_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


IPC_HANDLE_BYTES = 64
