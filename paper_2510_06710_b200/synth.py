"""Deterministic synthetic rollouts in the SoA layout, for the bench and for
parity tests at BASELINE sizes.

The episode process restates the reference env's bookkeeping (envsim/vec_env.cpp:137-288)
without its dynamics: per-step Bernoulli terminations (or a drawn success step for GRPO),
truncation at max_episode_steps, and the three rollout modes of harness/config.cpp:219-237:

  partial reset  auto_reset, immediate mode: the fresh episode takes the chunk's
                 remaining slots (new uid mid-chunk)
  deferred       auto_reset, deferred mode: frozen (valid=0, uid=-1, flags latched)
                 until the chunk ends, then reset
  mask           auto_reset off: frozen until the rollout ends
  fixed length   ignore_terminations: only truncations end episodes

Every draw comes from the reference's generator, chunkrl::Rng (core/rng.hpp:11-57: splitmix64,
next_double = (u64 >> 11) * 2^-53, next_below = u64 % n, next_normal = Box-Muller on two
doubles), with per-purpose seeds from its mix_seed (rng.hpp:60-65). splitmix64 is a counter
generator — the k-th draw of a stream is mix(seed + k * gamma) — so a stream of n draws is
vectorised (`Rng`, numpy, host) or generated on the device (`_device_draws`, torch int64
arithmetic) with the same values, and a rank's shard of the per-token tensors skips to its
offset in the full-batch stream (shard r's logits are rows of the full batch's). Structural
arrays are built with numpy (vectorised over envs, looping over time); the large per-token
tensors (logits, tokens, old log-probs) are drawn directly on the device.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

TERM, TRUNC, VALID = 1, 2, 4

_U64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15
_M1, _M2 = 0xBF58476D1CE4E5B9, 0x94D049BB133111EB


def _mix_np(z):
    z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
    return z ^ (z >> np.uint64(31))


def mix_seed(a: int, b: int) -> int:
    """chunkrl::mix_seed (core/rng.hpp:60-65)."""
    z = np.array([(a + _GAMMA * (b + 1)) & _U64], dtype=np.uint64)
    return int(_mix_np(z)[0])


class Rng:
    """chunkrl::Rng (core/rng.hpp:11-57), n draws of the sequential stream at a time."""

    def __init__(self, seed: int):
        self.state = seed & _U64
        self.u64(2)  # the constructor's two decorrelating draws

    def u64(self, n: int) -> np.ndarray:
        k = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(self.state) + k * np.uint64(_GAMMA)  # wraps mod 2^64
        self.state = (self.state + n * _GAMMA) & _U64
        return _mix_np(z)

    def double(self, n: int) -> np.ndarray:
        return (self.u64(n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53

    def below(self, n: int, bound: int) -> np.ndarray:
        return (self.u64(n) % np.uint64(bound)).astype(np.int64)

    def normal(self, n: int) -> np.ndarray:
        d = self.double(2 * n)
        u1, u2 = d[0::2], d[1::2]
        # next_normal redraws u1 == 0 (probability 2^-53 per draw); a vectorised stream cannot
        # shift its later positions, so such a seed is rejected instead
        if not np.all(u1 > 0.0):
            raise ValueError("Rng.normal: u1 == 0 drawn; pick another seed")
        return np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586476925287 * u2)


def _as_i64(u: int) -> int:
    return u - (1 << 64) if u >= (1 << 63) else u


def _srl(z: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64-held uint64 bits."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def _device_draws(seed: int, first: int, n: int, device) -> torch.Tensor:
    """u64 draws first+1 .. first+n (1-based after the constructor's two) of Rng(seed), as
    int64 bit patterns on `device` (int64 multiplies wrap mod 2^64 like the uint64 ones)."""
    k = torch.arange(first + 3, first + n + 3, dtype=torch.int64, device=device)
    z = k * _as_i64(_GAMMA) + _as_i64(seed & _U64)
    z = (z ^ _srl(z, 30)) * _as_i64(_M1)
    z = (z ^ _srl(z, 27)) * _as_i64(_M2)
    return z ^ _srl(z, 31)


def _device_doubles(seed, first, n, device):
    return _srl(_device_draws(seed, first, n, device), 11).to(torch.float64) * 2.0 ** -53


def _device_normals(seed: int, first: int, n: int, device) -> torch.Tensor:
    """next_normal draws first .. first+n-1 of Rng(seed) (two doubles each), f64."""
    d = _device_doubles(seed, 2 * first, 2 * n, device).view(n, 2)
    u1, u2 = d[:, 0], d[:, 1]
    if not bool((u1 > 0.0).all()):
        raise ValueError("next_normal: u1 == 0 drawn; pick another seed")
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(6.283185307179586476925287 * u2)


@dataclass
class SynthConfig:
    num_envs: int = 64
    num_chunks: int = 80
    chunk_len: int = 1
    tokens_per_action: int = 7
    vocab: int = 256
    algo: str = "ppo"                 # "ppo" | "grpo"
    mode: str = "partial"            # partial | deferred | mask | fixed
    max_episode_steps: int = 50
    p_terminate: float = 0.02        # PPO: Bernoulli terminations per atomic step
    p_success: float = 0.5           # GRPO: an episode succeeds with this probability
    group_size: int = 8
    logit_std: float = 2.0
    old_lp_noise: float = 0.05
    seed: int = 4


# Named configs of BASELINE.json
CONFIGS = {
    "cfg1": SynthConfig(num_envs=64, num_chunks=80, chunk_len=1, algo="ppo", mode="partial"),
    "cfg2": SynthConfig(num_envs=256, num_chunks=80, chunk_len=1, algo="grpo", mode="mask",
                        max_episode_steps=80),
    "cfg3": SynthConfig(num_envs=256, num_chunks=10, chunk_len=8, algo="ppo", mode="partial"),
    "cfg4": SynthConfig(num_envs=512, num_chunks=64, chunk_len=8, algo="grpo", mode="fixed",
                        max_episode_steps=512),
}
# (advantage, logprob, value) levels per config
SPECS = {"cfg1": (1, 2, 1), "cfg2": (0, 1, 0), "cfg3": (0, 0, 0), "cfg4": (0, 2, 0)}


def episodes_numpy(cfg: SynthConfig, env_offset: int = 0) -> dict:
    """Structural SoA arrays + episode table (numpy, host)."""
    E, Tc, C = cfg.num_envs, cfg.num_chunks, cfg.chunk_len
    T = Tc * C
    rng = Rng(mix_seed(cfg.seed, 1_000_003 + env_offset))
    reward = np.zeros((E, T), np.float64)
    flags = np.zeros((E, T), np.uint8)
    epi = np.full((E, T), -1, np.int32)

    ep_idx = np.zeros(E, np.int64)        # per-env episode counter (uid low bits)
    ep_step = np.zeros(E, np.int64)       # steps in current episode
    ep_start = np.zeros(E, np.int64)
    ep_rew = np.zeros(E)
    ep_fs = np.full(E, -1, np.int64)
    frozen = np.zeros(E, bool)
    latched = np.zeros(E, np.uint8)
    # GRPO: success step per (env, episode) drawn lazily at episode start
    p_draw = rng.double(E)
    succ_at = np.where(p_draw < cfg.p_success, rng.below(E, T), -1)
    table = []

    def close(e, complete):
        table.append((e + env_offset, int(ep_idx[e]), int(ep_start[e]), int(ep_step[e]),
                      float(ep_rew[e]), int(ep_fs[e]), int(complete)))

    for t in range(T):
        j = t % C
        if cfg.mode == "deferred" and j == 0:
            # reset frozen envs at the chunk boundary
            for e in np.nonzero(frozen)[0]:
                frozen[e] = False
                ep_idx[e] += 1
                ep_step[e] = 0
                ep_start[e] = t
                ep_rew[e] = 0.0
                ep_fs[e] = -1
        act = ~frozen
        # frozen slots: latched flags, invalid, uid -1
        flags[frozen, t] = latched[frozen]
        if not act.any():
            continue
        ae = np.nonzero(act)[0]
        epi[ae, t] = ep_idx[ae]
        if cfg.algo == "ppo":
            r = rng.normal(len(ae))
            term = rng.double(len(ae)) < cfg.p_terminate
        else:
            hit = (succ_at[ae] == t)
            r = hit.astype(np.float64)
            term = hit & (cfg.mode != "fixed")
        if cfg.mode == "fixed":
            term = np.zeros(len(ae), bool)
        reward[ae, t] = r
        ep_rew[ae] += r
        if cfg.algo == "grpo":
            newly = (r > 0) & (ep_fs[ae] < 0)
            ep_fs[ae[newly]] = ep_step[ae[newly]]
        ep_step[ae] += 1
        trunc = (ep_step[ae] >= cfg.max_episode_steps) & ~term
        fl = VALID | np.where(term, TERM, 0) | np.where(trunc, TRUNC, 0)
        flags[ae, t] = fl
        done = term | trunc
        for e, d, tm in zip(ae[done], term[done], trunc[done]):
            close(e, True)
            latched[e] = (TERM if d else 0) | (TRUNC if tm else 0)
            if cfg.mode in ("partial", "fixed"):
                ep_idx[e] += 1
                ep_step[e] = 0
                ep_start[e] = t + 1
                ep_rew[e] = 0.0
                ep_fs[e] = -1
            else:
                frozen[e] = True
    for e in range(E):
        if not frozen[e] and ep_step[e] > 0:
            close(e, False)
    table.sort(key=lambda x: (x[0], x[2]))
    tab = np.array(table, dtype=np.float64).reshape(-1, 7)
    out = dict(reward=reward.reshape(E, Tc, C), flags=flags.reshape(E, Tc, C),
               episode_id=epi.reshape(E, Tc, C),
               ep_env_id=tab[:, 0].astype(np.int32), ep_episode_id=tab[:, 1].astype(np.int32),
               ep_start=tab[:, 2].astype(np.int64), ep_length=tab[:, 3].astype(np.int64),
               ep_total_reward=tab[:, 4], ep_first_success=tab[:, 5].astype(np.int64),
               ep_complete=tab[:, 6].astype(np.uint8))
    n = len(tab)
    out["ep_task"] = np.zeros(n, np.int32)
    # unique reset id per group of G envs: groups never merge by key
    out["ep_reset_id"] = (out["ep_env_id"] // cfg.group_size).astype(np.int32)
    out["value_scalar"] = rng.normal(int(np.prod((E, Tc)))).reshape((E, Tc))
    out["value_vector"] = rng.normal(int(np.prod((E, Tc, C)))).reshape((E, Tc, C))
    out["boot_scalar"] = rng.normal(int(np.prod((E, Tc, C)))).reshape((E, Tc, C))
    out["boot_vector0"] = rng.normal(int(np.prod((E, Tc, C)))).reshape((E, Tc, C))
    out["new_value_scalar"] = rng.normal(int(np.prod((E, Tc)))).reshape((E, Tc))
    out["new_value_vector"] = rng.normal(int(np.prod((E, Tc, C)))).reshape((E, Tc, C))
    return out


def token_tensors(cfg: SynthConfig, device="cuda", dtype=torch.float32, env_offset: int = 0):
    """Logits ~ N(0, logit_std^2), tokens ~ U[0, V), old log-probs = current log-prob of the
    token + N(0, old_lp_noise^2) so ratios straddle the clip band. Drawn on `device` from three
    reference Rng streams (mix_seed(seed, 5 / 6 / 7)); env_offset skips each stream to the
    shard's first env, so a shard's tensors are the full batch's rows."""
    E, Tc, C, M, V = cfg.num_envs, cfg.num_chunks, cfg.chunk_len, cfg.tokens_per_action, cfg.vocab
    per_env = Tc * C * M
    s_logit, s_tok, s_noise = (mix_seed(cfg.seed, k) for k in (5, 6, 7))
    logits = torch.empty((E, Tc, C, M, V), dtype=torch.float32, device=device)
    flat = logits.view(-1)
    first = env_offset * per_env * V
    step = 1 << 24
    for i in range(0, flat.numel(), step):
        n = min(step, flat.numel() - i)
        flat[i:i + n] = (_device_normals(s_logit, first + i, n, device) * cfg.logit_std).float()
    logits = logits.to(dtype)
    n_tok = E * per_env
    u = _device_draws(s_tok, env_offset * per_env, n_tok, device)
    # next_below(V) = u64 % V as unsigned arithmetic: ((u >> 1) % V * 2 + (u & 1)) % V
    tokens = ((_srl(u, 1) % V) * 2 + (u & 1)) % V
    tokens = tokens.view(E, Tc, C, M)
    # old log-prob from the (possibly bf16-rounded) logits, chunked to bound memory
    lp = torch.empty((E, Tc, C, M), dtype=torch.float32, device=device)
    flat_l = logits.view(-1, V)
    flat_t = tokens.view(-1)
    flat_o = lp.view(-1)
    step = 1 << 20
    for i in range(0, flat_t.numel(), step):
        ls = torch.log_softmax(flat_l[i:i + step].double(), dim=-1)
        flat_o[i:i + step] = ls.gather(1, flat_t[i:i + step, None]).squeeze(1).float()
    noise = (_device_normals(s_noise, env_offset * per_env, n_tok, device) * cfg.old_lp_noise).float().view_as(lp)
    old_lp = lp + noise
    tok_dtype = torch.uint8 if V <= 256 else torch.int32
    return logits, tokens.to(tok_dtype), old_lp
