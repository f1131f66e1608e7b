"""(e) / §8 a13: the GPU rollout pipeline (csrc/rollout.cu) vs the UNMODIFIED reference.

The reference rolls out through its own StageSim / StageGen / merge_stages
(oracle/_ref/libchunkrl_ref.so, built from /root/reference by oracle/Makefile and carried
to the GPU box with the snapshot); the CUDA pipeline replays the same spec from the same
seeds and the same snapshot parameters. Checked:

* tokens, flags, episode ids, rewards, the merged episode table: bit-exact;
* old log-probs, values, bootstrap values (f64 copies): within 1e-12 relative (device
  exp/log/tanh vs glibc differ by <= 1 ulp);
* scheduling invariance (the reference's acceptance.cpp:245-311 contract): every output is
  bit-identical for pipeline depth k = 1, 2, 4;
* the slab feeds the PPO / GRPO path unchanged: diagnostics equal the reference's
  assemble -> loss on its own slab.
"""
import numpy as np
import pytest
import torch

from conftest import assert_close

pytestmark = pytest.mark.gpu

import paper_2510_06710_b200 as ck  # noqa: E402
from paper_2510_06710_b200 import advantage, errors, optim  # noqa: E402
from paper_2510_06710_b200.core import (EpisodeTable, FilterBounds, GaeParams,  # noqa: E402
                                        GranularitySpec, GrpoAssemblyOptions, GrpoParams,
                                        Level, LossOutputs, PolicyOutputs, PpoAssemblyOptions,
                                        PpoParams, read_diagnostics)
from paper_2510_06710_b200.pipeline import (SAMPLER_PARALLEL, SAMPLER_REFERENCE,  # noqa: E402
                                            EnvConfig, PolicyDescriptor, RolloutPipeline)

bindings = pytest.importorskip("oracle.bindings")
if not bindings.ref_available():
    pytest.skip("oracle/_ref/libchunkrl_ref.so not built", allow_module_level=True)

SCENARIOS = {
    "toyreach_immediate": dict(),
    "toyreach_shaped_long": dict(num_envs=16, num_chunks=6, max_episode_steps=5,
                                 reward_shaping=1, grid_size=4, hidden=12, value_hidden=6),
    "scripted_deferred": dict(env_kind=1, deferred_reset=1, num_envs=8, max_episode_steps=6,
                              success_step=3, chunk_length=3, num_chunks=5),
    "scripted_ignore_term": dict(env_kind=1, ignore_terminations=1, num_envs=4, chunk_length=4,
                                 max_episode_steps=7, success_step=2, num_chunks=3),
    "toyreach_fixed_ids": dict(use_fixed_reset_state_ids=1, group_size=2,
                               ids_with_replacement=1, num_envs=8, num_reset_states=5,
                               num_chunks=5),
    "toyreach_no_autoreset": dict(auto_reset=0, num_envs=4, num_chunks=6, max_episode_steps=4),
    "v256_m7": dict(vocab=256, tokens_per_action=7, hidden=32, trunk_layers=2, value_hidden=16,
                    num_envs=8, chunk_length=4, num_chunks=3, max_episode_steps=6,
                    grid_size=6),
    "deep_trunk_l0": dict(trunk_layers=0, hidden=40, vocab=37, tokens_per_action=3,
                          num_envs=4, num_chunks=4, deferred_reset=1),
}


def specs_of(kw):
    cfg = dict(bindings.REF_DEFAULTS)
    cfg.update(kw)
    env = EnvConfig(kind=cfg["env_kind"], num_envs=cfg["num_envs"],
                    max_episode_steps=cfg["max_episode_steps"], auto_reset=bool(cfg["auto_reset"]),
                    ignore_terminations=bool(cfg["ignore_terminations"]),
                    use_fixed_reset_state_ids=bool(cfg["use_fixed_reset_state_ids"]),
                    chunk_len=cfg["chunk_length"], grid_size=cfg["grid_size"],
                    reward_shaping=bool(cfg["reward_shaping"]),
                    num_reset_states=cfg["num_reset_states"], success_step=cfg["success_step"],
                    deferred_reset=bool(cfg["deferred_reset"]), seed=cfg["env_seed"])
    pol = PolicyDescriptor(obs_dim=env.obs_dim, hidden=cfg["hidden"],
                           trunk_layers=cfg["trunk_layers"], value_hidden=cfg["value_hidden"],
                           vocab=cfg["vocab"], chunk_len=cfg["chunk_length"],
                           tokens_per_action=cfg["tokens_per_action"])
    return cfg, env, pol


@pytest.fixture(scope="module")
def ref_cache():
    cache = {}

    def get(name):
        if name not in cache:
            sc = bindings.RefScenario(**SCENARIOS[name])
            d = sc.export(with_logits=True)
            p, ids = sc.params()
            cache[name] = (sc, d, p, ids)
        return cache[name]
    return get


def run_pipeline(name, stages, p, ids, sampler=SAMPLER_REFERENCE, gen_device=None, keep_logits=False):
    cfg, env, pol = specs_of(SCENARIOS[name])
    assert pol.num_params() == p.size
    pipe = RolloutPipeline(env, pol, cfg["num_chunks"], stages=stages,
                           sample_seed=cfg["sample_seed"],
                           reset_state_ids=None if ids is None else torch.tensor(ids),
                           sampler=sampler, gen_device=gen_device, keep_logits=keep_logits)
    ep = pipe.run(torch.tensor(p, dtype=torch.float64, device="cuda"))
    torch.cuda.synchronize()
    host = {k: v.cpu().numpy() for k, v in ep.t.items() if v is not None}
    n = int(host["episode_count"][0])
    for k in [k for k in host if k.startswith("ep_")]:
        host[k] = host[k][:n]
    return ep, host


EXACT = ("tokens", "flags", "episode_id", "reward_f64")
CLOSE = (("old_logprob_f64", "old_logprob"), ("value_scalar_f64", "value_scalar"),
         ("value_vector_f64", "value_vector"), ("boot_scalar_f64", "boot_scalar"),
         ("boot_vector0_f64", "boot_vector0"))
EPISODE = ("ep_env_id", "ep_episode_id", "ep_start", "ep_length", "ep_total_reward",
           "ep_first_success", "ep_complete", "ep_task", "ep_reset_id")


@pytest.mark.parametrize("name", sorted(SCENARIOS))
def test_pipeline_vs_reference_rollout(name, ref_cache):
    _, d, p, ids = ref_cache(name)
    _, g = run_pipeline(name, 1, p, ids)
    np.testing.assert_array_equal(g["tokens"], d["tokens"], err_msg="tokens")
    np.testing.assert_array_equal(g["flags"], d["flags"], err_msg="flags")
    np.testing.assert_array_equal(g["episode_id"], d["episode_id"], err_msg="episode ids")
    np.testing.assert_array_equal(g["reward_f64"], d["reward"], err_msg="rewards")
    np.testing.assert_array_equal(g["reward"], d["reward"].astype(np.float32))
    for mine, ref in CLOSE:
        np.testing.assert_allclose(g[mine], d[ref], rtol=1e-12, atol=1e-12, err_msg=mine)
        np.testing.assert_array_equal(g[ref], g[mine].astype(np.float32), err_msg=ref)
    assert g["ep_env_id"].size == d["ep_env_id"].size, "episode count"
    for k in EPISODE:
        np.testing.assert_array_equal(g[k], d[k].astype(g[k].dtype), err_msg=k)


def test_pipeline_logits_output(ref_cache):
    """keep_logits: the sampled tokens' log-softmax over the stored logits is the old lp."""
    name = "v256_m7"
    _, d, p, ids = ref_cache(name)
    cfg, env, pol = specs_of(SCENARIOS[name])
    pipe = RolloutPipeline(env, pol, cfg["num_chunks"], sample_seed=cfg["sample_seed"],
                           keep_logits=True)
    ep = pipe.run(torch.tensor(p, dtype=torch.float64, device="cuda"))
    lg = ep.t["logits"].double()
    lp = torch.log_softmax(lg, -1).gather(-1, ep.t["tokens"].long().unsqueeze(-1)).squeeze(-1)
    assert_close(lp.cpu().numpy(), d["old_logprob"], 1e-5, "lp from stored logits")


@pytest.mark.parametrize("name", sorted(SCENARIOS))
def test_pipeline_dump_is_the_references_trajectories_text(name, ref_cache):
    """Row f3: the CUDA rollout's slab, written in the reference's trajectories.txt format
    (ckrl_dump_slab), is byte-identical to the reference's own dump_slab of its rollout."""
    from paper_2510_06710_b200 import formats
    sc, _, p, ids = ref_cache(name)
    _, g = run_pipeline(name, 2 if specs_of(SCENARIOS[name])[0]["num_envs"] % 2 == 0 else 1, p, ids)
    assert formats.dump_slab(g["tokens"], g["reward_f64"], g["flags"], g["episode_id"]) == sc.dump_slab()


@pytest.mark.parametrize("name", sorted(SCENARIOS))
def test_pipeline_scheduling_invariance(name, ref_cache):
    _, _, p, ids = ref_cache(name)
    E = specs_of(SCENARIOS[name])[0]["num_envs"]
    _, base = run_pipeline(name, 1, p, ids)
    for k in (2, 4, E):
        if E % k or k == 1:
            continue
        _, g = run_pipeline(name, k, p, ids)
        for key in base:
            np.testing.assert_array_equal(g[key], base[key], err_msg=f"k={k} {key}")


@pytest.mark.parametrize("name", sorted(SCENARIOS))
def test_pipeline_placement_invariance(name, ref_cache):
    """a13 placements: the generation role placed on its own device (here the same B200, so
    the obs / action hand-offs run as device copies through the generation side's staging)
    gives the colocated slab bit-for-bit for every k, for both samplers, and with the
    reference sampler it is the reference's own rollout (tests/acceptance.cpp:245-311,
    real_backend.cpp:59-138)."""
    _, d, p, ids = ref_cache(name)
    E = specs_of(SCENARIOS[name])[0]["num_envs"]
    for sampler in (SAMPLER_REFERENCE, SAMPLER_PARALLEL):
        _, base = run_pipeline(name, 1, p, ids, sampler=sampler, keep_logits=True)
        for k in (1, 2, 4):
            if E % k:
                continue
            _, g = run_pipeline(name, k, p, ids, sampler=sampler, gen_device=0, keep_logits=True)
            for key in base:
                np.testing.assert_array_equal(g[key], base[key], err_msg=f"placed k={k} sampler={sampler} {key}")
        if sampler == SAMPLER_REFERENCE:
            np.testing.assert_array_equal(base["tokens"], d["tokens"])


@pytest.mark.parametrize("name", ["v256_m7", "toyreach_shaped_long", "deep_trunk_l0"])
def test_parallel_sampler_vs_reference(name, ref_cache):
    """The warp-parallel sampler reorders only the log-sum-exp and CDF sums: its tokens are
    the reference's (a differing draw needs u within an ulp of a CDF boundary) and its old
    log-probs match the reference's to 1e-12; invariance across k holds exactly."""
    _, d, p, ids = ref_cache(name)
    _, g = run_pipeline(name, 1, p, ids, sampler=SAMPLER_PARALLEL)
    np.testing.assert_array_equal(g["tokens"], d["tokens"], err_msg="tokens")
    np.testing.assert_array_equal(g["flags"], d["flags"], err_msg="flags")
    np.testing.assert_allclose(g["old_logprob_f64"], d["old_logprob"], rtol=1e-12, atol=1e-12)
    E = specs_of(SCENARIOS[name])[0]["num_envs"]
    for k in (2, 4):
        if E % k == 0:
            _, h = run_pipeline(name, k, p, ids, sampler=SAMPLER_PARALLEL)
            for key in g:
                np.testing.assert_array_equal(h[key], g[key], err_msg=f"k={k} {key}")


def test_pipeline_config_errors():
    env = EnvConfig(num_envs=6)
    pol = PolicyDescriptor(obs_dim=6, chunk_len=2)
    with pytest.raises(errors.ConfigError):
        RolloutPipeline(env, pol, 3, stages=4)  # k must divide num_envs (vec_env.cpp:324-327)
    with pytest.raises(errors.LengthMismatch):
        RolloutPipeline(env, PolicyDescriptor(obs_dim=2, chunk_len=2), 3)
    fixed = EnvConfig(num_envs=4, use_fixed_reset_state_ids=True, num_reset_states=3)
    with pytest.raises(errors.BadResetId):
        RolloutPipeline(fixed, pol, 2)  # fixed ids without ids
    pipe = RolloutPipeline(fixed, pol, 2, reset_state_ids=torch.tensor([0, 1, 2, 3]))
    with pytest.raises(errors.BadResetId):  # id 3 >= num_reset_states
        pipe.run(torch.zeros(pol.num_params(), dtype=torch.float64, device="cuda"))


def test_pipeline_feeds_ppo(ref_cache):
    """rollout (GPU) -> assemble -> loss equals the reference's whole chain."""
    name = "toyreach_shaped_long"
    sc, d, p, ids = ref_cache(name)
    ep, _ = run_pipeline(name, 2, p, ids)
    for tspec in ((0, 0, 0), (0, 2, 0), (1, 1, 1), (1, 2, 1)):
        spec = GranularitySpec(*(Level(x) for x in tspec))
        ro = ep.buffer(spec.advantage_level)
        batch = advantage.assemble_ppo_batch(ro, PpoAssemblyOptions(GaeParams(0.99, 0.95), spec))
        nv = d["new_value_scalar"] if tspec[2] == 0 else d["new_value_vector"]
        pol = PolicyOutputs(torch.tensor(d["logits"], dtype=torch.float32, device="cuda"),
                            torch.tensor(nv, dtype=torch.float32, device="cuda"))
        outs = LossOutputs.allocate(ro, spec.value_level)
        diag = read_diagnostics(optim.ppo_loss(ro, pol, batch, PpoParams(0.2, 0.5, 0.01, True),
                                               outs))
        want = sc.ppo(tspec)["diag"]
        got = np.array([diag[k] for k in ("loss", "surrogate", "value_loss", "entropy",
                                          "clip_frac", "approx_kl", "units")])
        assert got[6] == want[6]
        assert_close(got[:6], want[:6], 1e-5, f"{tspec} diag")


def test_pipeline_feeds_grpo(ref_cache):
    name = "toyreach_fixed_ids"
    sc, d, p, ids = ref_cache(name)
    ep, _ = run_pipeline(name, 4, p, ids)
    spec = GranularitySpec(Level.Chunk, Level.Token, Level.Chunk)
    opts = GrpoAssemblyOptions(spec, 1e-8, False, FilterBounds(0.0, 1.0), True, 2)
    ro = ep.buffer(Level.Chunk)
    try:
        b = advantage.assemble_grpo_batch(ro, ep.episodes, opts)
        pol = PolicyOutputs(torch.tensor(d["logits"], dtype=torch.float32, device="cuda"))
        outs = LossOutputs.allocate(ro, Level.Chunk)
        diag = read_diagnostics(optim.grpo_loss(ro, pol, b, GrpoParams(0.2), outs))
    except errors.Error:  # DegenerateGroup / SkipUpdate must match the reference's
        diag = None
    want = sc.grpo((0, 2, 0), eps_std=1e-8, apply_filter=False, length_normalized=True,
                   min_group_size=2)
    if diag is not None:
        assert want["status"] == 0
        got = np.array([diag[k] for k in ("loss", "surrogate", "value_loss", "entropy",
                                          "clip_frac", "approx_kl", "units")])
        assert got[6] == want["diag"][6]
        assert_close(got[:6], want["diag"][:6], 1e-5, "grpo diag")
    else:
        assert want["status"] != 0
