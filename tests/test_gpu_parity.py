"""CUDA path (libckrl.so via its C ABI) vs the reference and the oracle.

* golden fixtures (outputs of the unmodified reference, tests/golden): every PPO / GRPO
  granularity spec, the fused token kernel, masks / episode ids / group assignment
  bit-exact, floats within the north-star tolerance 1e-5 (fp32 accumulate) under the
  rule |x - ref| <= 1e-5 * max(|ref|, rms(ref));
* synthetic rollouts at the BASELINE shapes (V=256, M=7) vs the oracle run on the
  same (f32-rounded) inputs.
"""
import numpy as np
import pytest
import torch

from conftest import assert_close, golden_files, load_golden

pytestmark = pytest.mark.gpu

import paper_2510_06710_b200 as ck  # noqa: E402
from paper_2510_06710_b200 import advantage, errors, optim, policy  # noqa: E402
from paper_2510_06710_b200.core import (EpisodeTable, GaeParams, GranularitySpec,  # noqa: E402
                                        GrpoAssemblyOptions, FilterBounds, Level, LossOutputs,
                                        PolicyOutputs, PpoAssemblyOptions, PpoParams,
                                        GrpoParams, RolloutBuffer, read_diagnostics)

TOL = 1e-5
PPO = golden_files("ppo_")
GRPO = golden_files("grpo_")


def f32(x):
    return np.asarray(x, np.float32).astype(np.float64)


def rounded(d):
    """The fixture as the device sees it: every float rounded to f32."""
    r = dict(d)
    for k in ("old_logprob", "reward", "value_scalar", "value_vector", "boot_scalar",
              "boot_vector0", "logits", "new_value_scalar", "new_value_vector"):
        r[k] = f32(d[k])
    return r


def spec_of(key):
    a, l, v = (int(x) for x in key.split("_")[:3])
    return GranularitySpec(Level(a), Level(l), Level(v)), (a, l, v)


def away_from_clip(lp_cur, old, active, lp_level, C, M, clip, thr=1e-6):
    """Per-position mask of the lp units whose ratio is not within `thr` of a clip edge 1 +- eps
    (SURVEY §7 hard part 2): there an O(1e-7) log-prob difference legitimately flips
    clipped_surrogate's branch (losses.cpp:32-46) and the coefficient jumps between A*rho and
    0. `active` marks the positions that enter a unit (counted / weighted slots)."""
    lp_cur = np.asarray(lp_cur, np.float64).ravel()
    old = np.asarray(old, np.float64).ravel()
    act = np.broadcast_to(np.asarray(active, bool).reshape(-1, 1), (lp_cur.size // M, M)).ravel()
    pos = np.arange(lp_cur.size)
    unit = pos if lp_level == 2 else (pos // M if lp_level == 1 else pos // (C * M))
    d = np.bincount(unit[act], (lp_cur - old)[act], minlength=unit.max() + 1)
    rho = np.exp(d)
    near = np.minimum(np.abs(rho - (1 - clip)), np.abs(rho - (1 + clip))) < thr
    keep = ~near[unit]
    assert near.mean() < 0.01, f"{near.sum()} of {near.size} units sit on a clip edge"
    return keep


def diag_vec(dd):
    return np.array([dd[k] for k in ("loss", "surrogate", "value_loss", "entropy", "clip_frac",
                                     "approx_kl", "units")], dtype=np.float64)


@pytest.fixture(scope="module", autouse=True)
def _device():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    ck.lib()


@pytest.mark.parametrize("name", PPO)
def test_token_kernel_vs_reference(name):
    d = load_golden(name)
    logits = torch.tensor(d["logits"], dtype=torch.float32, device="cuda")
    tokens = torch.tensor(d["tokens"], dtype=torch.int32, device="cuda")
    out = policy.evaluate_chunks(logits, tokens)
    assert_close(out["token_logprob"].cpu().numpy(), d["lp_cur"], TOL, "token lp")
    assert_close(out["token_entropy"].cpu().numpy(), d["ent_cur"], TOL, "token entropy")
    # canonical aggregation (core/granularity.cpp:83-113): action = sum_j, chunk = sum_i
    act = d["lp_cur"].sum(-1)
    assert_close(out["action_logprob"].cpu().numpy(), act, TOL, "action lp")
    assert_close(out["chunk_logprob"].cpu().numpy(), act.sum(-1), TOL, "chunk lp")
    # u8 tokens and bf16 logits paths (oracle on the bf16-rounded logits)
    if d["dims"][4] <= 256:
        out8 = policy.evaluate_chunks(logits, tokens.to(torch.uint8))
        assert torch.equal(out8["token_logprob"], out["token_logprob"])


@pytest.mark.parametrize("name", PPO)
def test_ppo_pipeline_vs_reference(name, oracle):
    d = load_golden(name)
    r = rounded(d)
    gamma, lam, clip, vcoef, ecoef = d["ppo_params"]
    V = int(d["dims"][4])
    keys = sorted({k.split("/")[1] for k in d if k.startswith("ppo/")})
    for key in keys:
        spec, tspec = spec_of(key)
        boot = d["boot_scalar"] if tspec[0] == 0 else d["boot_vector0"]
        ro = RolloutBuffer.from_arrays(d, boot, V)
        batch = advantage.assemble_ppo_batch(ro, PpoAssemblyOptions(GaeParams(gamma, lam), spec))
        counted = batch.counted.cpu().numpy()
        np.testing.assert_array_equal(counted, d[f"ppo/{key}/counted"], err_msg=key)
        assert_close(batch.advantages.cpu().numpy(), d[f"ppo/{key}/adv_raw"], TOL, f"{key} adv")
        assert_close(batch.returns.cpu().numpy(), d[f"ppo/{key}/ret"], TOL, f"{key} ret")
        nv = d["new_value_scalar"] if tspec[2] == 0 else d["new_value_vector"]
        pol = PolicyOutputs(torch.tensor(d["logits"], dtype=torch.float32, device="cuda"),
                            torch.tensor(nv, dtype=torch.float32, device="cuda"))
        outs = LossOutputs.allocate(ro, spec.value_level, tokens=True)
        diag = optim.ppo_loss(ro, pol, batch, PpoParams(clip, vcoef, ecoef, True), outs)
        got = diag_vec(read_diagnostics(diag))
        want = d[f"ppo/{key}/diag"]
        assert got[6] == want[6], f"{key}: units"
        assert_close(got[:6], want[:6], TOL, f"{key} diag")
        # coefficients vs the oracle on the device-rounded inputs (whitened adv from oracle)
        st, c_o, a_o, r_o = oracle.assemble_ppo(r, tspec, gamma, lam)
        a_n = oracle.normalize_advantages(c_o, a_o, tspec[0])
        st, odiag, clp, cent, cval = oracle.ppo_loss(r, tspec, c_o, a_n, r_o, r["logits"],
                                                     r["new_value_scalar"] if tspec[2] == 0 else r["new_value_vector"],
                                                     clip, vcoef, ecoef)
        lp_o, _ = oracle.token_stats(r["logits"].reshape(-1, V), d["tokens"].reshape(-1))
        keep = away_from_clip(lp_o, r["old_logprob"], c_o, tspec[1], r["reward"].shape[2],
                              d["tokens"].shape[-1], clip)
        assert_close(outs.coeff_logprob.cpu().numpy().ravel(), clp.ravel(), TOL, f"{key} coeff_lp", mask=keep)
        assert_close(outs.coeff_entropy.cpu().numpy(), cent, TOL, f"{key} coeff_ent")
        assert_close(outs.coeff_value.cpu().numpy(), cval, TOL, f"{key} coeff_val")
        # materialised whitening (normalize_advantages) vs the reference, no floor
        optim.normalize_advantages(ro, batch)
        units = d[f"ppo/{key}/adv_raw"][c_o.any(-1) if tspec[0] == 0 else c_o != 0]
        if units.size >= 2 and units.std() == 0.0:
            # all-equal batch (the scripted env): the reference returns (a - mean) / 1e-8 with
            # `mean` its sequential sum's round-off, i.e. +-n ulp(a) / 1e-8; the device's
            # moments keep mean == a exactly and return 0. Both are round-off: bound them by
            # n * ulp(|a|) / 1e-8 (update.cpp:33-43).
            lim = units.size * np.spacing(np.abs(units).max()) / 1e-8
            assert np.abs(batch.advantages.cpu().numpy()).max() <= lim
            assert np.abs(d[f"ppo/{key}/adv_norm"]).max() <= lim
        else:
            assert_close(batch.advantages.cpu().numpy(), d[f"ppo/{key}/adv_norm"], TOL, f"{key} adv_norm")
        # ... and the reference's call order normalize_advantages -> ppo_loss (update.cpp:66-80):
        # the loss takes the whitened advantages as they are (no second whitening)
        diag2 = optim.ppo_loss(ro, pol, batch, PpoParams(clip, vcoef, ecoef, True), outs)
        assert_close(diag_vec(read_diagnostics(diag2))[:6], want[:6], TOL, f"{key} diag after normalize")


@pytest.mark.parametrize("name", GRPO)
def test_grpo_pipeline_vs_reference(name):
    d = load_golden(name)
    lower, upper, clip, min_g = d["grpo_params"]
    V = int(d["dims"][4])
    ro = RolloutBuffer.from_arrays(d, d["boot_scalar"], V)
    eps_tab = EpisodeTable.from_arrays(d)
    pol = PolicyOutputs(torch.tensor(d["logits"], dtype=torch.float32, device="cuda"))
    keys = sorted({k.split("/")[1] for k in d if k.startswith("grpo/")})
    for key in keys:
        spec, tspec = spec_of(key)
        parts = key.split("_")
        ln, eps, af = int(parts[3][2:]), (1e-8 if parts[4] == "eps1" else 0.0), int(parts[5][1:])
        opts = GrpoAssemblyOptions(spec, eps, bool(af), FilterBounds(lower, upper), bool(ln), int(min_g))
        b = advantage.assemble_grpo_batch(ro, eps_tab, opts)
        status = int(d[f"grpo/{key}/status"])
        gt, gr = (int(x) for x in d[f"grpo/{key}/groups"])
        if status != 7:  # the reference throws DegenerateGroup before reporting counts
            assert (b.groups_total, b.groups_retained) == (gt, gr), key
        outs = LossOutputs.allocate(ro, Level.Chunk)
        diag = optim.grpo_loss(ro, pol, b, GrpoParams(clip), outs)
        if status != 0:
            exc = {7: errors.DegenerateGroup, 8: errors.SkipUpdate}[status]
            with pytest.raises(exc):
                read_diagnostics(diag)
            continue
        for k, attr in (("env_group", "env_group"), ("env_member", "env_member"),
                        ("env_episode", "env_episode"), ("env_group_size", "env_group_size"),
                        ("slot_member", "slot_member")):
            np.testing.assert_array_equal(getattr(b, attr).cpu().numpy(), d[f"grpo/{key}/{k}"],
                                          err_msg=f"{key}:{k}")
        # fp64 group statistics: bit-exact with grpo.cpp:9-28
        np.testing.assert_array_equal(b.env_advantage.cpu().numpy(), d[f"grpo/{key}/env_adv"])
        # fp64 weights 1 / T (grpo.cpp:57-79): bit-exact
        np.testing.assert_array_equal(b.slot_weight.cpu().numpy(), d[f"grpo/{key}/slot_weight"], err_msg=key)
        got = diag_vec(read_diagnostics(diag))
        want = d[f"grpo/{key}/diag"]
        assert got[6] == want[6], f"{key}: units"
        assert_close(got[:6], want[:6], TOL, f"{key} diag")


# ----------------------------------------------------------------- synthetic, BASELINE shapes
def synth_case(cfg_name, scale_envs=None, seed=4, dtype=torch.float32):
    from paper_2510_06710_b200 import synth
    cfg = synth.CONFIGS[cfg_name]
    if scale_envs:
        cfg = synth.SynthConfig(**{**cfg.__dict__, "num_envs": scale_envs, "seed": seed})
    d = synth.episodes_numpy(cfg)
    logits, tokens, old_lp = synth.token_tensors(cfg, "cuda", dtype)
    d["tokens"] = tokens.cpu().numpy()
    d["old_logprob"] = old_lp.cpu().numpy()
    return cfg, d, logits, tokens


@pytest.mark.parametrize("cfg_name,envs", [("cfg1", None), ("cfg3", 64), ("cfg3", None)])
def test_ppo_synthetic_vs_oracle(cfg_name, envs, oracle):
    from paper_2510_06710_b200 import synth
    cfg, d, logits, tokens = synth_case(cfg_name, envs)
    a, l, v = synth.SPECS[cfg_name]
    spec = GranularitySpec(Level(a), Level(l), Level(v))
    boot = d["boot_scalar"] if a == 0 else d["boot_vector0"]
    nv = d["new_value_scalar"] if v == 0 else d["new_value_vector"]
    ro = RolloutBuffer.from_arrays(d, boot, cfg.vocab)
    pol = PolicyOutputs(logits, torch.tensor(nv, dtype=torch.float32, device="cuda"))
    params = PpoParams(0.2, 0.5, 0.01, True)
    step = optim.PpoStep(ro, GaeParams(0.99, 0.95), spec, params)
    step(ro, pol)
    got = diag_vec(step.diagnostics())
    r = rounded({**d, "logits": logits.cpu().numpy()})
    st, c_o, a_o, r_o = oracle.assemble_ppo(r, (a, l, v), 0.99, 0.95)
    np.testing.assert_array_equal(step.batch.counted.cpu().numpy(), c_o)
    assert_close(step.batch.advantages.cpu().numpy(), a_o, TOL, "adv")
    a_n = oracle.normalize_advantages(c_o, a_o, a)
    st, want, clp, cent, cval = oracle.ppo_loss(r, (a, l, v), c_o, a_n, r_o, r["logits"],
                                                f32(nv), 0.2, 0.5, 0.01)
    assert got[6] == want[6]
    assert_close(got[:6], want[:6], TOL, f"{cfg_name}/{envs} ppo diag")
    assert_close(step.batch.returns.cpu().numpy(), r_o, TOL, f"{cfg_name}/{envs} returns")
    lp_o, _ = oracle.token_stats(r["logits"].reshape(-1, cfg.vocab), d["tokens"].reshape(-1))
    keep = away_from_clip(lp_o, r["old_logprob"], c_o, l, cfg.chunk_len, cfg.tokens_per_action, 0.2)
    assert_close(step.outputs.coeff_logprob.cpu().numpy().ravel(), clp.ravel(), TOL,
                 f"{cfg_name}/{envs} ppo coeff_lp", mask=keep)
    assert_close(step.outputs.coeff_entropy.cpu().numpy(), cent, TOL, f"{cfg_name}/{envs} ppo coeff_ent")
    assert_close(step.outputs.coeff_value.cpu().numpy(), cval, TOL, f"{cfg_name}/{envs} ppo coeff_val")
    # determinism: a second run is bitwise identical
    first = step.diag.clone()
    step(ro, pol)
    torch.cuda.synchronize()
    assert torch.equal(first, step.diag)


@pytest.mark.parametrize("cfg_name,envs", [("cfg2", None), ("cfg4", 64), ("cfg4", None)])
def test_grpo_synthetic_vs_oracle(cfg_name, envs, oracle):
    from paper_2510_06710_b200 import synth
    cfg, d, logits, tokens = synth_case(cfg_name, envs)
    a, l, v = synth.SPECS[cfg_name]
    spec = GranularitySpec(Level(a), Level(l), Level(v))
    ro = RolloutBuffer.from_arrays(d, d["boot_scalar"], cfg.vocab)
    ept = EpisodeTable.from_arrays(d)
    pol = PolicyOutputs(logits)
    opts = GrpoAssemblyOptions(spec)
    step = optim.GrpoStep(ro, opts, GrpoParams(0.2))
    step(ro, ept, pol)
    got = diag_vec(step.diagnostics())
    r = rounded({**d, "logits": logits.cpu().numpy()})
    st, asm = oracle.assemble_grpo(r, (a, l, v))
    assert st == 0
    assert (step.batch.groups_total, step.batch.groups_retained) == (asm["groups_total"], asm["groups_retained"])
    np.testing.assert_array_equal(step.batch.env_group.cpu().numpy(), asm["env_group"])
    np.testing.assert_array_equal(step.batch.slot_member.cpu().numpy(), asm["slot_member"])
    st, want, coeff = oracle.grpo_loss(r, l, asm, r["logits"], 0.2)
    assert got[6] == want[6]
    # The GRPO loss is a signed sum whose terms cancel (group-relative advantages sum to ~0;
    # |loss| ~ 1e-3 of sum|terms| at the full cfg4 size): checked at 1e-5 of |loss| itself.
    assert_close(got[:2], want[:2], TOL, f"{cfg_name}/{envs} grpo loss / surrogate")
    assert_close(got[2:6], want[2:6], TOL, f"{cfg_name}/{envs} grpo diag")
    lp_o, _ = oracle.token_stats(r["logits"].reshape(-1, cfg.vocab), d["tokens"].reshape(-1))
    np.testing.assert_array_equal(step.batch.slot_weight.cpu().numpy(), asm["slot_weight"])
    active = (asm["slot_member"] != 0) & (asm["slot_weight"] != 0) & (asm["env_group"][:, None, None] >= 0)
    keep = away_from_clip(lp_o, r["old_logprob"], active, l, cfg.chunk_len, cfg.tokens_per_action, 0.2)
    assert_close(step.outputs.coeff_logprob.cpu().numpy().ravel(), coeff.ravel(), TOL,
                 f"{cfg_name}/{envs} grpo coeff_lp", mask=keep)


def test_bf16_logits_path(oracle):
    cfg, d, logits, tokens = synth_case("cfg3", 32, dtype=torch.bfloat16)
    out = policy.evaluate_chunks(logits, tokens)
    lp, ent = oracle.token_stats(logits.float().cpu().numpy(), tokens.cpu().numpy())
    assert_close(out["token_logprob"].cpu().numpy().ravel(), lp, TOL, "bf16 lp")
    assert_close(out["token_entropy"].cpu().numpy().ravel(), ent, TOL, "bf16 ent")


def test_compute_gae_known_answers():
    # test_advantage.cpp:16-25, 36-49
    adv, ret = advantage.compute_gae([0.0, 0.0, 1.0], [0.0] * 3, 0.0, [0, 0, 1], [0, 0, 0], GaeParams(1.0, 1.0))
    assert adv.cpu().tolist() == [1.0, 1.0, 1.0] and ret.cpu().tolist() == [1.0, 1.0, 1.0]
    adv, _ = advantage.compute_gae([1.0, 1.0], [0.5, 0.5], 0.5, [0, 0], [0, 0], GaeParams(0.5, 0.5))
    assert adv.cpu().tolist() == pytest.approx([0.9375, 0.75], rel=1e-12)
    with pytest.raises(errors.LengthMismatch):
        advantage.compute_gae([1.0, 2.0], [0.0], 0.0, [0, 0], [0, 0], GaeParams(0.9, 0.9))


def test_compute_gae_random_vs_oracle(oracle):
    rng = np.random.default_rng(0)
    for n in (1, 5, 31, 32, 33, 100, 1000):
        r, v, b = rng.standard_normal(n), rng.standard_normal(n), rng.standard_normal(n)
        u = rng.random(n)
        te, tr = u < 0.15, (u >= 0.15) & (u < 0.3)
        adv, ret = advantage.compute_gae(r, v, b, te, tr, GaeParams(0.97, 0.9))
        oa, orr = oracle.compute_gae(r, v, b, te, tr, 0.97, 0.9)
        np.testing.assert_allclose(adv.cpu().numpy(), oa, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(ret.cpu().numpy(), orr, rtol=1e-12, atol=1e-12)


def test_grpo_beyond_shared_memory_sort(oracle):
    """More eligible episodes than the group kernel's shared-memory sort holds (8192): the
    GroupKey sort runs in the workspace's sort region. Reset ids drawn with replacement
    (train.cpp:92-101) leave the keys unordered, so the bitonic sort really runs; group
    assignment, membership and the fp64 advantages must equal the oracle's bit-for-bit."""
    from paper_2510_06710_b200 import synth
    E = 9216
    cfg = synth.SynthConfig(num_envs=E, num_chunks=6, chunk_len=1, tokens_per_action=2, vocab=16,
                            algo="grpo", mode="mask", max_episode_steps=6, group_size=8, seed=21)
    d = synth.episodes_numpy(cfg)
    rng = np.random.default_rng(21)
    ids = rng.integers(0, E // 6, E).astype(d["ep_reset_id"].dtype)
    d["ep_reset_id"] = ids[d["ep_env_id"]]
    logits, tokens, old = synth.token_tensors(cfg)
    d["tokens"], d["old_logprob"] = tokens.cpu().numpy(), old.cpu().numpy()
    spec = GranularitySpec(Level(0), Level(1), Level(0))
    ro = RolloutBuffer.from_arrays(d, d["boot_scalar"], cfg.vocab)
    ept = EpisodeTable.from_arrays(d)
    step = optim.GrpoStep(ro, GrpoAssemblyOptions(spec), GrpoParams(0.2))
    step(ro, ept, PolicyOutputs(logits))
    got = diag_vec(step.diagnostics())
    r = rounded({**d, "logits": logits.cpu().numpy()})
    st, asm = oracle.assemble_grpo(r, (0, 1, 0))
    assert st == 0 and int((np.asarray(d["ep_complete"]) != 0).sum()) > 8192
    assert (step.batch.groups_total, step.batch.groups_retained) == (asm["groups_total"], asm["groups_retained"])
    np.testing.assert_array_equal(step.batch.env_group.cpu().numpy(), asm["env_group"])
    np.testing.assert_array_equal(step.batch.env_advantage.cpu().numpy(), asm["env_adv"])
    np.testing.assert_array_equal(step.batch.slot_member.cpu().numpy(), asm["slot_member"])
    st, want, _ = oracle.grpo_loss(r, 1, asm, r["logits"], 0.2)
    assert got[6] == want[6]
    assert_close(got[:6], want[:6], TOL, "grpo 9216 envs diag")
