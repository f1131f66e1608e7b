"""The multi-rank CUDA path (comm->world > 1) on one B200.

K logical ranks, each with its own env shard (PPO: contiguous envs; GRPO: whole groups),
workspace, stream and communicator, exchange their stats records and raw loss sums through
the same kernels and exchange buffers a K-GPU job uses (csrc/common.cuh ExSlot: the
assembly's last CTA stores the rank's record into every rank's buffer, the loss kernel
waits for all of them before its unit phases and its last CTA all-reduces the raw sums).
Every rank must then report the diagnostics of the FULL batch — the reference's
single-process semantics (optim/update.cpp:14-45 whitening over all units,
optim/losses.cpp:75-87 / 221-227 normalisers and sums) — and its shard of the masks,
advantages and coefficients must equal the full-batch oracle's. Several steps run back to
back so both exchange parities and the epoch counter are exercised.

The cross-process variant maps the exchange buffers with CUDA IPC (ckrl_comm_open_peers), as
bench.py / torchrun ranks do; with one GPU both processes share it.
"""
import os
import socket

import numpy as np
import pytest
import torch

from conftest import assert_close
from test_multirank import shard

pytestmark = pytest.mark.gpu

import paper_2510_06710_b200 as ck  # noqa: E402
from paper_2510_06710_b200 import optim, synth  # noqa: E402
from paper_2510_06710_b200.core import (EpisodeTable, GaeParams, GranularitySpec,  # noqa: E402
                                        GrpoAssemblyOptions, GrpoParams, Level, PolicyOutputs,
                                        PpoParams, RolloutBuffer)
from paper_2510_06710_b200.dist import Comm, env_shard  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-5
DIAG = ("loss", "surrogate", "value_loss", "entropy", "clip_frac", "approx_kl", "units")


def f32(x):
    return np.asarray(x, np.float32).astype(np.float64)


def rounded(d):
    r = dict(d)
    for k in ("old_logprob", "reward", "value_scalar", "value_vector", "boot_scalar",
              "boot_vector0", "logits", "new_value_scalar", "new_value_vector"):
        if k in r:
            r[k] = f32(d[k])
    return r


def assert_diag_close(got, want, what, rel=1e-11):
    assert got.keys() == want.keys(), what
    for k in want:
        if k == "units":
            assert got[k] == want[k], (what, k)
        else:
            assert abs(got[k] - want[k]) <= rel * max(abs(want[k]), 1e-300) + 1e-18, (what, k, got[k], want[k])


def case(cfg_name, envs, seed=11):
    cfg = synth.SynthConfig(**{**synth.CONFIGS[cfg_name].__dict__, "num_envs": envs, "seed": seed})
    d = synth.episodes_numpy(cfg)
    logits, tokens, old = synth.token_tensors(cfg, "cuda", torch.float32)
    d["tokens"], d["old_logprob"] = tokens.cpu().numpy(), old.cpu().numpy()
    return cfg, d, logits


def run_ranks(steps, calls, iters):
    """Issues every rank's step on its own stream, `iters` times, and returns each
    iteration's per-rank diagnostics."""
    streams = [torch.cuda.Stream() for _ in steps]
    out = []
    for _ in range(iters):
        for st, call, s in zip(steps, calls, streams):
            call(s)
        torch.cuda.synchronize()
        out.append([st.diagnostics() for st in steps])
    return out


@pytest.fixture(scope="module", autouse=True)
def _device():
    assert torch.cuda.is_available()
    ck.lib()


@pytest.mark.parametrize("world", [2, 4])
def test_ppo_step_k_ranks_match_full_batch(world, oracle):
    cfg, d, logits = case("cfg3", 64)
    a, l, v = synth.SPECS["cfg3"]
    spec = GranularitySpec(Level(a), Level(l), Level(v))
    E = cfg.num_envs
    comms = Comm.local_group(world)
    steps, calls, parts = [], [], []
    for r in range(world):
        envs = env_shard(E, world, r)
        s = shard(d, envs)
        ro = RolloutBuffer.from_arrays(s, s["boot_scalar"], cfg.vocab)
        pol = PolicyOutputs(logits[envs.start:envs.stop],
                            torch.tensor(s["new_value_scalar"], dtype=torch.float32, device="cuda"))
        st = optim.PpoStep(ro, GaeParams(0.99, 0.95), spec, PpoParams(0.2, 0.5, 0.01, True),
                           comm=comms[r])
        steps.append(st)
        calls.append(lambda stream, st=st, ro=ro, pol=pol: st(ro, pol, stream=stream))
        parts.append(envs)
    runs = run_ranks(steps, calls, 3)

    r = rounded({**d, "logits": logits.cpu().numpy()})
    _, c_o, a_o, r_o = oracle.assemble_ppo(r, (a, l, v), 0.99, 0.95)
    a_n = oracle.normalize_advantages(c_o, a_o, a)
    _, want, clp, cent, cval = oracle.ppo_loss(r, (a, l, v), c_o, a_n, r_o, r["logits"],
                                               f32(d["new_value_scalar"]), 0.2, 0.5, 0.01)
    for it, diags in enumerate(runs):
        vecs = [np.array([dd[k] for k in DIAG]) for dd in diags]
        for q in range(1, world):  # the same rank-order sums on every rank: bitwise equal
            np.testing.assert_array_equal(vecs[q], vecs[0], err_msg=f"rank {q} iter {it}")
        assert vecs[0][6] == want[6]
        assert_close(vecs[0][:6], want[:6], TOL, f"ppo world={world} iter {it} diag")
    for st, envs in zip(steps, parts):
        sl = slice(envs.start, envs.stop)
        np.testing.assert_array_equal(st.batch.counted.cpu().numpy(), c_o[sl])
        assert_close(st.batch.advantages.cpu().numpy(), a_o[sl], TOL, f"ppo world={world} adv")
        assert_close(st.batch.returns.cpu().numpy(), r_o[sl], TOL, f"ppo world={world} ret")
        # coefficients carry the GLOBAL normalisers and whitening
        assert_close(st.outputs.coeff_entropy.cpu().numpy(), cent[sl], TOL, f"ppo world={world} coeff_ent")
        assert_close(st.outputs.coeff_value.cpu().numpy(), cval[sl], TOL, f"ppo world={world} coeff_val")
    got_clp = np.concatenate([st.outputs.coeff_logprob.cpu().numpy() for st in steps])
    lp_o, _ = oracle.token_stats(r["logits"].reshape(-1, cfg.vocab), d["tokens"].reshape(-1))
    from test_gpu_parity import away_from_clip
    keep = away_from_clip(lp_o, r["old_logprob"], c_o, l, cfg.chunk_len, cfg.tokens_per_action, 0.2)
    assert_close(got_clp.ravel(), clp.ravel(), TOL, f"ppo world={world} coeff_lp", mask=keep)
    for c in comms:
        c.close()


@pytest.mark.parametrize("world", [2, 4])
def test_grpo_step_k_ranks_match_full_batch(world, oracle):
    cfg, d, logits = case("cfg4", 64)  # 8 groups of 8 envs; whole groups per rank
    a, l, v = synth.SPECS["cfg4"]
    spec = GranularitySpec(Level(a), Level(l), Level(v))
    E = cfg.num_envs
    comms = Comm.local_group(world)
    steps, calls, parts = [], [], []
    for r in range(world):
        envs = env_shard(E, world, r, group_size=cfg.group_size)
        s = shard(d, envs)
        ro = RolloutBuffer.from_arrays(s, s["boot_scalar"], cfg.vocab)
        ept = EpisodeTable.from_arrays(s)
        pol = PolicyOutputs(logits[envs.start:envs.stop])
        st = optim.GrpoStep(ro, GrpoAssemblyOptions(spec), GrpoParams(0.2), comm=comms[r])
        steps.append(st)
        calls.append(lambda stream, st=st, ro=ro, ept=ept, pol=pol: st(ro, ept, pol, stream=stream))
        parts.append(envs)
    runs = run_ranks(steps, calls, 3)
    r = rounded({**d, "logits": logits.cpu().numpy()})
    st0, asm = oracle.assemble_grpo(r, (a, l, v))
    assert st0 == 0
    _, want, coeff = oracle.grpo_loss(r, l, asm, r["logits"], 0.2)
    for it, diags in enumerate(runs):
        vecs = [np.array([dd[k] for k in DIAG]) for dd in diags]
        for q in range(1, world):
            np.testing.assert_array_equal(vecs[q], vecs[0], err_msg=f"rank {q} iter {it}")
        assert vecs[0][6] == want[6]
        assert_close(vecs[0][:6], want[:6], TOL, f"grpo world={world} iter {it} diag")
    lp_o, _ = oracle.token_stats(r["logits"].reshape(-1, cfg.vocab), d["tokens"].reshape(-1))
    got = np.concatenate([st.outputs.coeff_logprob.cpu().numpy() for st in steps])
    from test_gpu_parity import away_from_clip
    active = (asm["slot_member"] != 0) & (asm["slot_weight"] != 0) & (asm["env_group"][:, None, None] >= 0)
    keep = away_from_clip(lp_o, r["old_logprob"], active, l, cfg.chunk_len, cfg.tokens_per_action, 0.2)
    assert_close(got.ravel(), coeff.ravel(), TOL, f"grpo world={world} coeff_lp", mask=keep)
    for st, envs in zip(steps, parts):
        sl = slice(envs.start, envs.stop)
        np.testing.assert_array_equal(st.batch.slot_weight.cpu().numpy(), asm["slot_weight"][sl])
    for c in comms:
        c.close()


def test_step_refuses_unopened_comm():
    from paper_2510_06710_b200 import errors
    cfg, d, logits = case("cfg3", 8)
    a, l, v = synth.SPECS["cfg3"]
    ro = RolloutBuffer.from_arrays(d, d["boot_scalar"], cfg.vocab)
    pol = PolicyOutputs(logits, torch.tensor(d["new_value_scalar"], dtype=torch.float32, device="cuda"))
    c = Comm(2, 0)  # peers never opened
    st = optim.PpoStep(ro, GaeParams(0.99, 0.95), GranularitySpec(Level(a), Level(l), Level(v)),
                       PpoParams(0.2, 0.5, 0.01, True), comm=c)
    with pytest.raises(errors.Error):
        st(ro, pol)
    c.close()


# ------------------------------------------------------------------ two processes, CUDA IPC
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = Comm.from_torch()
        cfg, d, logits = case("cfg3", 32)
        a, l, v = synth.SPECS["cfg3"]
        envs = env_shard(cfg.num_envs, world, rank)
        s = shard(d, envs)
        ro = RolloutBuffer.from_arrays(s, s["boot_scalar"], cfg.vocab)
        pol = PolicyOutputs(logits[envs.start:envs.stop].contiguous(),
                            torch.tensor(s["new_value_scalar"], dtype=torch.float32, device="cuda"))
        st = optim.PpoStep(ro, GaeParams(0.99, 0.95), GranularitySpec(Level(a), Level(l), Level(v)),
                           PpoParams(0.2, 0.5, 0.01, True), comm=comm)
        res = []
        for _ in range(2):
            st(ro, pol)
            res.append(st.diagnostics())
        q.put((rank, res))
        dist.barrier()
        comm.close()
    except Exception as e:  # report to the parent instead of hanging it
        q.put((rank, repr(e)))
    dist.destroy_process_group()


def test_two_processes_cuda_ipc(oracle):
    import torch.multiprocessing as mp
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_ipc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = {}
    try:
        for _ in range(world):
            rank, res = q.get(timeout=240)
            got[rank] = res
    finally:
        for p in ps:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for rank, res in got.items():
        assert not isinstance(res, str), f"rank {rank}: {res}"
    cfg, d, logits = case("cfg3", 32)
    a, l, v = synth.SPECS["cfg3"]
    r = rounded({**d, "logits": logits.cpu().numpy()})
    _, c_o, a_o, r_o = oracle.assemble_ppo(r, (a, l, v), 0.99, 0.95)
    a_n = oracle.normalize_advantages(c_o, a_o, a)
    _, want, *_ = oracle.ppo_loss(r, (a, l, v), c_o, a_n, r_o, r["logits"],
                                  f32(d["new_value_scalar"]), 0.2, 0.5, 0.01)
    for rank, res in got.items():
        for dd in res:
            vec = np.array([dd[k] for k in DIAG])
            assert vec[6] == want[6]
            assert_close(vec[:6], want[:6], TOL, f"ipc rank {rank} diag")


@pytest.mark.parametrize("world", [1, 2])
def test_pipelined_batches_match_plain_steps(world):
    """optim.Pipelined (batch i+1's assembly on a side stream overlapping batch i's loss, the
    ckrl_*_step_assemble / _loss halves) gives every batch the same diagnostics and masks as
    one ckrl_ppo_step per batch — single rank and across ranks (the exchange epoch travels in
    each batch's workspace, so a later batch's assembly may publish before an earlier loss)."""
    a, l, v = synth.SPECS["cfg3"]
    spec = GranularitySpec(Level(a), Level(l), Level(v))
    R, n_batches = 3, 7
    data = [case("cfg3", 32, seed=20 + r) for r in range(R)]
    comms = Comm.local_group(world) if world > 1 else [None]

    def rank_inputs(r, rep):
        cfg, d, logits = data[rep]
        envs = env_shard(cfg.num_envs, world, r)
        s = shard(d, envs)
        ro = RolloutBuffer.from_arrays(s, s["boot_scalar"], cfg.vocab)
        pol = PolicyOutputs(logits[envs.start:envs.stop],
                            torch.tensor(s["new_value_scalar"], dtype=torch.float32, device="cuda"))
        return ro, pol

    inputs = [[rank_inputs(r, rep) for rep in range(R)] for r in range(world)]
    params = PpoParams(0.2, 0.5, 0.01, True)
    mk = lambda r, rep: optim.PpoStep(inputs[r][rep][0], GaeParams(0.99, 0.95), spec, params,  # noqa: E731
                                      comm=comms[r])
    # reference: plain steps, batch i on replica i mod R
    plain = [[mk(r, rep) for rep in range(R)] for r in range(world)]
    streams = [torch.cuda.Stream() for _ in range(world)]
    want = {}
    for i in range(n_batches):
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                plain[r][i % R](*inputs[r][i % R], stream=streams[r])
        torch.cuda.synchronize()
        want[i] = [plain[r][i % R].diagnostics() for r in range(world)]
    # pipelined
    pipes = [optim.Pipelined([mk(r, rep) for rep in range(R)]) for r in range(world)]
    for r in range(world):
        with torch.cuda.stream(streams[r]):
            pipes[r].issue(n_batches, lambda i, r=r: ((inputs[r][i % R][0],), inputs[r][i % R]))
    torch.cuda.synchronize()
    for r in range(world):
        for rep in range(R):
            last = max(i for i in range(n_batches) if i % R == rep)
            got = pipes[r].steps[rep].diagnostics()
            # the pipelined losses may run on fewer CTAs (launch policy, csrc/abi.cu): the same
            # sums in another CTA grouping, so the fp64 diagnostics agree to rounding
            assert_diag_close(got, want[last][r], (r, rep))
            assert torch.equal(pipes[r].steps[rep].batch.counted, plain[r][rep].batch.counted)
    for c in comms:
        if c is not None:
            c.close()


@pytest.mark.parametrize("algo", ["ppo", "grpo"])
def test_pipelined_graph_matches_plain_steps(algo):
    """The bench's form of the pipelined step: optim.Pipelined captured in one CUDA graph (the
    losses chained as programmatic dependents, the assemblies on a side stream) and replayed;
    every batch's diagnostics and masks equal one plain step per batch (single rank, PPO cfg3
    and GRPO cfg2 shapes)."""
    cfg_name = "cfg3" if algo == "ppo" else "cfg2"
    a, l, v = synth.SPECS[cfg_name]
    spec = GranularitySpec(Level(a), Level(l), Level(v))
    R, n_batches = 3, 8
    data = [case(cfg_name, 64, seed=40 + r) for r in range(R)]
    inputs = []
    for cfg, d, logits in data:
        ro = RolloutBuffer.from_arrays(d, d["boot_scalar"], cfg.vocab)
        nv = torch.tensor(d["new_value_scalar"], dtype=torch.float32, device="cuda")
        ept = EpisodeTable.from_arrays(d) if algo == "grpo" else None
        inputs.append((ro, PolicyOutputs(logits, nv), ept))

    def mk(rep):
        ro = inputs[rep][0]
        if algo == "ppo":
            return optim.PpoStep(ro, GaeParams(0.99, 0.95), spec, PpoParams(0.2, 0.5, 0.01, True))
        return optim.GrpoStep(ro, GrpoAssemblyOptions(spec), GrpoParams(0.2))

    def args_of(i):
        ro, pol, ept = inputs[i % R]
        return ((ro,), (ro, pol)) if algo == "ppo" else ((ro, ept), (ro, pol))

    plain = [mk(rep) for rep in range(R)]
    want = {}
    for i in range(n_batches):
        ro, pol, ept = inputs[i % R]
        plain[i % R](ro, pol) if algo == "ppo" else plain[i % R](ro, ept, pol)
        torch.cuda.synchronize()
        want[i] = plain[i % R].diagnostics()
    pipe = optim.Pipelined([mk(rep) for rep in range(R)])
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        pipe.issue(1, args_of)  # warm-up outside the capture
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        pipe.issue(n_batches, args_of)
    for _ in range(2):  # replays are idempotent: every batch recomputes from its inputs
        g.replay()
        torch.cuda.synchronize()
        for rep in range(R):
            last = max(i for i in range(n_batches) if i % R == rep)
            assert_diag_close(pipe.steps[rep].diagnostics(), want[last], rep)
            if algo == "ppo":
                assert torch.equal(pipe.steps[rep].batch.counted, plain[rep].batch.counted)
            else:
                assert torch.equal(pipe.steps[rep].batch.env_group, plain[rep].batch.env_group)


@pytest.mark.parametrize("world", [2, 3])
def test_grpo_step_key_sharded_ranks_match_full_batch(world, oracle):
    """GroupKeys merged across non-adjacent envs (reset ids drawn with replacement,
    train.cpp:92-101), sharded by key (dist.key_shard: every key on one rank, non-contiguous env
    sets): the K ranks' CUDA steps, exchanging only the retained-group count and the raw loss
    sums, report the full batch's diagnostics; each rank's weights equal the oracle's rows."""
    from test_multirank import gather_envs
    from paper_2510_06710_b200.dist import key_shard
    cfg, d, logits = case("cfg2", 48, seed=17)
    rng = np.random.default_rng(17)
    ids = rng.integers(0, 9, cfg.num_envs).astype(d["ep_reset_id"].dtype)
    d["ep_reset_id"] = ids[d["ep_env_id"]]
    a, l, v = synth.SPECS["cfg2"]
    spec = GranularitySpec(Level(a), Level(l), Level(v))
    first = {}
    for e, t, rid in zip(d["ep_env_id"], d["ep_task"], d["ep_reset_id"]):
        first.setdefault(int(e), (int(t), int(rid)))
    parts = key_shard([first[e] for e in range(cfg.num_envs)], world)
    assert any(np.any(np.diff(p) > 1) for p in parts)
    comms = Comm.local_group(world)
    steps, calls = [], []
    lg = logits.cpu()
    for r in range(world):
        s = gather_envs(d, parts[r])
        ro = RolloutBuffer.from_arrays(s, s["boot_scalar"], cfg.vocab)
        ept = EpisodeTable.from_arrays(s)
        pol = PolicyOutputs(lg[torch.as_tensor(parts[r])].contiguous().cuda())
        st = optim.GrpoStep(ro, GrpoAssemblyOptions(spec), GrpoParams(0.2), comm=comms[r])
        steps.append(st)
        calls.append(lambda stream, st=st, ro=ro, ept=ept, pol=pol: st(ro, ept, pol, stream=stream))
    runs = run_ranks(steps, calls, 2)
    r = rounded({**d, "logits": logits.cpu().numpy()})
    st0, asm = oracle.assemble_grpo(r, (a, l, v))
    assert st0 == 0 and asm["groups_retained"] > 1
    _, want, coeff = oracle.grpo_loss(r, l, asm, r["logits"], 0.2)
    for it, diags in enumerate(runs):
        vecs = [np.array([dd[k] for k in DIAG]) for dd in diags]
        for q in range(1, world):
            np.testing.assert_array_equal(vecs[q], vecs[0], err_msg=f"rank {q} iter {it}")
        assert vecs[0][6] == want[6]
        # a signed sum of cancelling group terms, summed per rank then across ranks: 1e-5 of
        # the terms' L1 mass (sum |coeff_lp| at this lp level)
        mass = float(np.abs(coeff).sum())
        assert_close(vecs[0][:2], want[:2], TOL, f"grpo keys world={world} loss", floor=mass)
        assert_close(vecs[0][2:6], want[2:6], TOL, f"grpo keys world={world} diag")
    for st, envs in zip(steps, parts):
        np.testing.assert_array_equal(st.batch.slot_weight.cpu().numpy(), asm["slot_weight"][envs])
        np.testing.assert_array_equal(st.batch.env_advantage.cpu().numpy(), asm["env_adv"][envs])
    for c in comms:
        c.close()
