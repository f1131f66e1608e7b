"""Multi-rank host logic on CPU (gloo, world_size 2): env / group sharding, the 64-byte
stats-record exchange that precedes the loss, and the loss-scalar sum after it — the same
two exchanges ckrl_ppo_step / ckrl_grpo_step issue over NCCL on B200s. Per-rank compute is
the oracle on each shard; the merge uses the library's own ckrl_merge_stats_host. The
result must equal the single-process full-batch reference semantics."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def make_ppo(E=8, seed=3):
    from paper_2510_06710_b200 import synth
    cfg = synth.SynthConfig(num_envs=E, num_chunks=6, chunk_len=4, tokens_per_action=3, vocab=16,
                            algo="ppo", mode="partial", max_episode_steps=7, p_terminate=0.1,
                            seed=seed)
    d = synth.episodes_numpy(cfg)
    rng = np.random.default_rng(seed)
    d["tokens"] = rng.integers(0, 16, (E, 6, 4, 3)).astype(np.int32)
    d["logits"] = 2.0 * rng.standard_normal((E, 6, 4, 3, 16))
    d["old_logprob"] = -np.log(16) + 0.3 * rng.standard_normal((E, 6, 4, 3))
    d["V"] = 16
    return d


def make_grpo(E=16, G=4, seed=5):
    from paper_2510_06710_b200 import synth
    cfg = synth.SynthConfig(num_envs=E, num_chunks=5, chunk_len=2, tokens_per_action=3, vocab=16,
                            algo="grpo", mode="mask", max_episode_steps=10, group_size=G, seed=seed)
    d = synth.episodes_numpy(cfg)
    rng = np.random.default_rng(seed)
    d["tokens"] = rng.integers(0, 16, (E, 5, 2, 3)).astype(np.int32)
    d["logits"] = 2.0 * rng.standard_normal((E, 5, 2, 3, 16))
    d["old_logprob"] = -np.log(16) + 0.3 * rng.standard_normal((E, 5, 2, 3))
    d["V"] = 16
    return d


def shard(d, envs):
    out = {}
    e0, e1 = envs.start, envs.stop
    for k, v in d.items():
        if k == "V":
            out[k] = v
        elif k.startswith("ep_"):
            continue
        else:
            out[k] = v[e0:e1]
    if "ep_env_id" in d:
        m = (d["ep_env_id"] >= e0) & (d["ep_env_id"] < e1)
        for k in d:
            if k.startswith("ep_"):
                out[k] = d[k][m]
        out["ep_env_id"] = out["ep_env_id"] - e0
    return out


def adv_units(counted, adv, level):
    if level == 0:
        return adv[counted.any(-1)]
    return adv[counted.astype(bool)]


def ppo_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.bindings import Oracle
    from paper_2510_06710_b200.dist import StatsRecord, env_shard, merge_stats
    orc = Oracle()
    d = make_ppo()
    out = {}
    for spec in [(0, 0, 0), (0, 2, 0), (1, 2, 1)]:
        s = shard(d, env_shard(8, world, rank))
        st, counted, adv, ret = orc.assemble_ppo(s, spec, 0.99, 0.95)
        units = adv_units(counted, adv, spec[0])
        M = s["tokens"].shape[-1]
        rec = StatsRecord.from_units(units, n_val=len(units), n_pos=int(counted.sum()) * M)
        mine = torch.frombuffer(bytearray(rec.to_bytes()), dtype=torch.uint8)
        allr = [torch.zeros(64, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(allr, mine)
        g = merge_stats([bytes(t.numpy().tobytes()) for t in allr])
        # whiten with the global stats (update.cpp:66-67), then the rank-local loss
        a = adv.copy()
        if spec[0] == 0:
            m = counted.any(-1)
        else:
            m = counted.astype(bool)
        a[m] = (a[m] - g["mean"]) / g["denom"]
        nv = s["new_value_scalar"] if spec[2] == 0 else s["new_value_vector"]
        st, diag, *_ = orc.ppo_loss(s, spec, counted, a, ret, s["logits"], nv, 0.2, 0.5, 0.01)
        n_adv_l = len(units)
        n_pos_l = int(counted.sum()) * M
        raw = torch.tensor([-diag[1] * n_adv_l, diag[2] * n_adv_l, diag[3] * n_pos_l,
                            diag[5] * diag[6], diag[4] * diag[6], diag[6]], dtype=torch.float64)
        dist.all_reduce(raw)  # the post-loss scalar all-reduce
        surr = -raw[0].item() / g["n_adv"]
        vl = raw[1].item() / g["n_val"]
        ent = raw[2].item() / g["n_pos"]
        out[spec] = dict(loss=surr + 0.5 * vl - 0.01 * ent, surrogate=surr, value_loss=vl,
                         entropy=ent, clip_frac=raw[4].item() / raw[5].item(),
                         approx_kl=raw[3].item() / raw[5].item(), units=raw[5].item())
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


def test_ppo_two_ranks_match_full_batch(oracle):
    world, port = 2, free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=ppo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    d = make_ppo()
    for spec, g in got.items():
        st, counted, adv, ret = oracle.assemble_ppo(d, spec, 0.99, 0.95)
        advn = oracle.normalize_advantages(counted, adv, spec[0])
        nv = d["new_value_scalar"] if spec[2] == 0 else d["new_value_vector"]
        st, diag, *_ = oracle.ppo_loss(d, spec, counted, advn, ret, d["logits"], nv, 0.2, 0.5, 0.01)
        want = dict(zip(["loss", "surrogate", "value_loss", "entropy", "clip_frac", "approx_kl", "units"], diag))
        for k, v in want.items():
            assert g[k] == pytest.approx(v, rel=1e-10, abs=1e-12), (spec, k)


def grpo_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.bindings import Oracle
    from paper_2510_06710_b200.dist import env_shard
    orc = Oracle()
    d = make_grpo()
    out = {}
    for spec in [(0, 0, 0), (0, 2, 0)]:
        s = shard(d, env_shard(16, world, rank, group_size=4))  # whole groups per rank
        st, a = orc.assemble_grpo(s, spec)
        groups = torch.tensor([a["groups_retained"]], dtype=torch.int64)
        dist.all_reduce(groups)  # part of the stats-record exchange
        if a["groups_retained"]:
            st, diag, _ = orc.grpo_loss(s, spec[1], a, s["logits"], 0.2)
            raw = torch.tensor([-diag[1] * a["groups_retained"], diag[5] * diag[6], diag[4] * diag[6], diag[6]],
                               dtype=torch.float64)
        else:
            raw = torch.zeros(4, dtype=torch.float64)
        dist.all_reduce(raw)
        out[spec] = dict(loss=-raw[0].item() / groups.item(), clip_frac=raw[2].item() / raw[3].item(),
                         approx_kl=raw[1].item() / raw[3].item(), units=raw[3].item())
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


def test_grpo_two_ranks_match_full_batch(oracle):
    world, port = 2, free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=grpo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    d = make_grpo()
    for spec, g in got.items():
        st, a = oracle.assemble_grpo(d, spec)
        st, diag, _ = oracle.grpo_loss(d, spec[1], a, d["logits"], 0.2)
        assert g["loss"] == pytest.approx(diag[0], rel=1e-10, abs=1e-12)
        assert g["clip_frac"] == pytest.approx(diag[4], rel=1e-12)
        assert g["approx_kl"] == pytest.approx(diag[5], rel=1e-10)
        assert g["units"] == diag[6]


def test_env_shard_keeps_groups_whole():
    from paper_2510_06710_b200.dist import check_group_sharding, env_shard
    from paper_2510_06710_b200.errors import ConfigError
    parts = [env_shard(512, 8, r, group_size=8) for r in range(8)]
    assert [len(p) for p in parts] == [64] * 8
    assert sum(len(p) for p in parts) == 512 and parts[-1].stop == 512
    owner = lambda e: next(r for r, p in enumerate(parts) if e in p)  # noqa: E731
    envs = np.arange(512)
    check_group_sharding(envs, np.stack([np.zeros(512), envs // 8], 1), 8, owner)
    with pytest.raises(ConfigError):  # keys drawn with replacement can span ranks
        check_group_sharding(envs, np.stack([np.zeros(512), envs % 8], 1), 8, owner)
    with pytest.raises(ConfigError):
        env_shard(10, 2, 0, group_size=4)


def gather_envs(d, envs):
    """The shard of envs `envs` (ascending, any subset): slab rows and their episodes, env ids
    renumbered 0..len-1 in the same order."""
    envs = np.asarray(envs)
    out = {}
    for k, v in d.items():
        if k == "V":
            out[k] = v
        elif not k.startswith("ep_"):
            out[k] = v[envs]
    m = np.isin(d["ep_env_id"], envs)
    for k in d:
        if k.startswith("ep_"):
            out[k] = d[k][m]
    remap = {int(e): i for i, e in enumerate(envs)}
    out["ep_env_id"] = np.array([remap[int(e)] for e in out["ep_env_id"]], dtype=d["ep_env_id"].dtype)
    return out


def make_grpo_merged(E=16, seed=9):
    """Reset ids drawn with replacement (train.cpp:92-101): equal GroupKeys on non-adjacent envs."""
    d = make_grpo(E=E, G=4, seed=seed)
    rng = np.random.default_rng(seed)
    ids = rng.integers(0, 5, E).astype(d["ep_reset_id"].dtype)
    d["ep_reset_id"] = ids[d["ep_env_id"]]
    return d


def key_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.bindings import Oracle
    from paper_2510_06710_b200.dist import key_shard
    orc = Oracle()
    d = make_grpo_merged()
    first = {}
    for e, t, r in zip(d["ep_env_id"], d["ep_task"], d["ep_reset_id"]):
        first.setdefault(int(e), (int(t), int(r)))
    parts = key_shard([first[e] for e in range(16)], world)
    s = gather_envs(d, parts[rank])
    out = {}
    for spec in [(0, 0, 0), (0, 2, 0)]:
        st, a = orc.assemble_grpo(s, spec)
        groups = torch.tensor([a["groups_retained"]], dtype=torch.int64)
        dist.all_reduce(groups)
        if a["groups_retained"]:
            st, diag, _ = orc.grpo_loss(s, spec[1], a, s["logits"], 0.2)
            raw = torch.tensor([-diag[1] * a["groups_retained"], diag[5] * diag[6], diag[4] * diag[6], diag[6]],
                               dtype=torch.float64)
        else:
            raw = torch.zeros(4, dtype=torch.float64)
        dist.all_reduce(raw)
        out[spec] = dict(loss=-raw[0].item() / groups.item(), clip_frac=raw[2].item() / raw[3].item(),
                         approx_kl=raw[1].item() / raw[3].item(), units=raw[3].item(), groups=groups.item())
    if rank == 0:
        q.put((out, [p.tolist() for p in parts]))
    dist.destroy_process_group()


def test_grpo_key_sharded_two_ranks_match_full_batch(oracle):
    """Merged GroupKeys on non-adjacent envs: key_shard keeps every key on one rank, and the
    two ranks' losses (retained-group count exchanged) equal the full batch's."""
    world, port = 2, free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=key_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got, parts = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(sum(parts, [])) == list(range(16)) and all(parts)
    assert any(np.any(np.diff(p) > 1) for p in parts), "the shards should be non-contiguous here"
    d = make_grpo_merged()
    for spec, g in got.items():
        st, a = oracle.assemble_grpo(d, spec)
        st, diag, _ = oracle.grpo_loss(d, spec[1], a, d["logits"], 0.2)
        assert g["groups"] == a["groups_retained"]
        assert g["loss"] == pytest.approx(diag[0], rel=1e-10, abs=1e-12)
        assert g["clip_frac"] == pytest.approx(diag[4], rel=1e-12)
        assert g["approx_kl"] == pytest.approx(diag[5], rel=1e-10)
        assert g["units"] == diag[6]


def test_key_shard_balanced_and_whole():
    from paper_2510_06710_b200.dist import key_shard
    keys = [(0, i % 5) for i in range(37)]
    parts = key_shard(keys, 3)
    assert sorted(np.concatenate(parts).tolist()) == list(range(37))
    owner = {}
    for r, p in enumerate(parts):
        for e in p:
            assert owner.setdefault(keys[e], r) == r
    sizes = sorted(len(p) for p in parts)
    assert sizes[-1] - sizes[0] <= 8
