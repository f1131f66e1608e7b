"""Row f1, the softmax-backward seam: ckrl_logits_grad (CUDA, via the C ABI) vs the oracle's
restatement of PolicyNet::accumulate_chunk_gradient's per-position logits gradient
(policy/policy_net.cpp:431-456). The oracle itself is pinned to the reference in
tests/test_ref_live.py (its row sums are the reference's b_pol gradient bit-for-bit).

Tolerance: f32 arithmetic on f32 (or bf16-rounded) inputs against the double oracle on the
same rounded inputs, |x - ref| <= 1e-5 * max(|ref|, rms(ref row)) per position row.
"""
import numpy as np
import pytest
import torch

from conftest import golden_files, load_golden

pytestmark = pytest.mark.gpu

import paper_2510_06710_b200 as ck  # noqa: E402
from paper_2510_06710_b200 import advantage, errors, optim, policy, synth  # noqa: E402
from paper_2510_06710_b200.core import (GaeParams, GranularitySpec, Level, LossOutputs,  # noqa: E402
                                        PolicyOutputs, PpoAssemblyOptions, PpoParams,
                                        RolloutBuffer)

TOL = 1e-5


def f32(x):
    return np.asarray(x, np.float32).astype(np.float64)


def assert_rows_close(got, want, rel=TOL, what=""):
    got = np.asarray(got, np.float64).reshape(-1, want.shape[-1])
    want = np.asarray(want, np.float64).reshape(-1, want.shape[-1])
    rms = np.sqrt(np.mean(want * want, axis=1, keepdims=True))
    bound = rel * np.maximum(np.abs(want), rms) + 1e-300
    err = np.abs(got - want)
    bad = err > bound
    assert not bad.any(), (f"{what}: {int(bad.sum())}/{want.size} outside tol; worst "
                           f"{float((err / bound).max()):.3g}x")


@pytest.fixture(scope="module", autouse=True)
def _device():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    ck.lib()


def _ppo_coeffs(cfg_name, envs):
    cfg = synth.SynthConfig(**{**synth.CONFIGS[cfg_name].__dict__, "num_envs": envs})
    d = synth.episodes_numpy(cfg)
    logits, tokens, old = synth.token_tensors(cfg)
    d["tokens"], d["old_logprob"] = tokens.cpu().numpy(), old.cpu().numpy()
    a, l, v = synth.SPECS[cfg_name]
    ro = RolloutBuffer.from_arrays(d, d["boot_scalar"] if a == 0 else d["boot_vector0"], cfg.vocab)
    nv = d["new_value_scalar"] if v == 0 else d["new_value_vector"]
    pol = PolicyOutputs(logits, torch.tensor(nv, dtype=torch.float32, device="cuda"))
    step = optim.PpoStep(ro, GaeParams(0.99, 0.95), GranularitySpec(Level(a), Level(l), Level(v)),
                         PpoParams(0.2, 0.5, 0.01, True))
    step(ro, pol)
    torch.cuda.synchronize()
    return logits, tokens, step.outputs.coeff_logprob, step.outputs.coeff_entropy


@pytest.mark.parametrize("cfg_name,envs", [("cfg3", 32), ("cfg1", 16)])
def test_logits_grad_vs_oracle_from_ppo_step(cfg_name, envs, oracle):
    logits, tokens, klp, kent = _ppo_coeffs(cfg_name, envs)
    assert (klp != 0).any() and (kent != 0).any()
    got = policy.logits_grad(logits, tokens, klp, kent)
    st, want = oracle.logits_grad(logits.double().cpu().numpy(), tokens.cpu().numpy(),
                                  f32(klp.cpu().numpy()), f32(kent.cpu().numpy()))
    assert st == 0
    assert_rows_close(got.cpu().numpy(), want, what=f"{cfg_name} dlogits")
    # positions the loss did not evaluate (both coefficients 0) are zero rows
    skip = ((klp == 0) & (kent == 0)).reshape(-1)
    assert torch.count_nonzero(got.reshape(-1, 256)[skip]) == 0
    # bf16 output of the same gradient; in-place over a copy of the logits
    got16 = policy.logits_grad(logits, tokens, klp, kent, out_dtype=torch.bfloat16)
    assert_rows_close(got16.float().cpu().numpy(), got.cpu().numpy(), rel=1e-2, what="bf16 out")
    buf = logits.clone()
    policy.logits_grad(buf, tokens, klp, kent, out=buf)
    assert torch.equal(buf, got)


def test_logits_grad_bf16_logits(oracle):
    logits, tokens, klp, kent = _ppo_coeffs("cfg3", 16)
    lb = logits.to(torch.bfloat16)
    got = policy.logits_grad(lb, tokens, klp, kent, out_dtype=torch.float32)
    st, want = oracle.logits_grad(lb.double().cpu().numpy(), tokens.cpu().numpy(),
                                  f32(klp.cpu().numpy()), f32(kent.cpu().numpy()))
    assert st == 0
    assert_rows_close(got.cpu().numpy(), want, what="bf16 logits")


@pytest.mark.parametrize("name", golden_files("ppo_"))
def test_logits_grad_on_reference_fixtures(name, oracle):
    """Reference forward_logits rows and the oracle's ppo_loss coefficients (bit-exact vs the
    reference) for every PPO spec of the fixture."""
    d = load_golden(name)
    gamma, lam, clip, vcoef, ecoef = d["ppo_params"]
    r = {k: (f32(v) if np.asarray(v).dtype.kind == "f" else v) for k, v in d.items()}
    lg = torch.tensor(d["logits"], dtype=torch.float32, device="cuda")
    tk = torch.tensor(d["tokens"], dtype=torch.int32, device="cuda")
    for key in sorted({k.split("/")[1] for k in d if k.startswith("ppo/")}):
        tspec = tuple(int(x) for x in key.split("_")[:3])
        st, c, a, R = oracle.assemble_ppo(r, tspec, gamma, lam)
        a = oracle.normalize_advantages(c, a, tspec[0])
        nv = r["new_value_scalar"] if tspec[2] == 0 else r["new_value_vector"]
        st, _, clp, cent, _ = oracle.ppo_loss(r, tspec, c, a, R, r["logits"], nv, clip, vcoef, ecoef)
        klp, kent = f32(clp), f32(cent)
        got = policy.logits_grad(lg, tk, torch.tensor(klp, dtype=torch.float32, device="cuda"),
                                 torch.tensor(kent, dtype=torch.float32, device="cuda"))
        st, want = oracle.logits_grad(r["logits"], d["tokens"], klp, kent)
        assert st == 0
        assert_rows_close(got.cpu().numpy(), want, what=f"{name} {key}")


@pytest.mark.parametrize("V,tok_dtype", [(100, torch.int32), (300, torch.int32), (256, torch.uint8)])
def test_logits_grad_generic_vocab_and_grpo_style(V, tok_dtype, oracle):
    g = torch.Generator(device="cuda").manual_seed(V)
    rows = 777
    logits = torch.randn(rows, V, device="cuda", generator=g) * 3
    tokens = torch.randint(0, V, (rows,), device="cuda", generator=g).to(tok_dtype)
    klp = torch.randn(rows, device="cuda", generator=g)
    klp[::5] = 0.0  # skipped positions
    got = policy.logits_grad(logits, tokens, klp)  # GRPO: no entropy coefficient
    st, want = oracle.logits_grad(logits.double().cpu().numpy(), tokens.cpu().numpy(),
                                  f32(klp.cpu().numpy()), np.zeros(rows))
    assert st == 0
    assert_rows_close(got.cpu().numpy(), want, what=f"V={V}")
    assert torch.count_nonzero(got[::5]) == 0


def test_logits_grad_non_finite_coefficient_is_nonfinite():
    logits = torch.randn(64, 256, device="cuda")
    tokens = torch.zeros(64, dtype=torch.uint8, device="cuda")
    klp = torch.ones(64, device="cuda")
    klp[7] = float("nan")
    with pytest.raises(errors.NonFinite):
        policy.logits_grad(logits, tokens, klp)
    out = policy.logits_grad(logits, tokens, torch.zeros(64, device="cuda"))
    assert torch.count_nonzero(out) == 0
    assert policy.logits_grad(logits[:0], tokens[:0], klp[:0]).numel() == 0


@pytest.mark.parametrize("cfg_name,envs,dtype", [("cfg3", 32, torch.float32), ("cfg1", 16, torch.float32),
                                                 ("cfg3", 16, torch.bfloat16)])
def test_fused_dlogits_in_the_ppo_step(cfg_name, envs, dtype, oracle):
    """The seam fused into the loss launch (LossOutputs.dlogits): same rows as the oracle on
    the step's own coefficients."""
    cfg = synth.SynthConfig(**{**synth.CONFIGS[cfg_name].__dict__, "num_envs": envs})
    d = synth.episodes_numpy(cfg)
    logits, tokens, old = synth.token_tensors(cfg, dtype=dtype)
    d["tokens"], d["old_logprob"] = tokens.cpu().numpy(), old.cpu().numpy()
    a, l, v = synth.SPECS[cfg_name]
    ro = RolloutBuffer.from_arrays(d, d["boot_scalar"] if a == 0 else d["boot_vector0"], cfg.vocab)
    nv = d["new_value_scalar"] if v == 0 else d["new_value_vector"]
    pol = PolicyOutputs(logits, torch.tensor(nv, dtype=torch.float32, device="cuda"))
    step = optim.PpoStep(ro, GaeParams(0.99, 0.95), GranularitySpec(Level(a), Level(l), Level(v)),
                         PpoParams(0.2, 0.5, 0.01, True))
    step.outputs.dlogits = torch.full_like(logits, float("nan"))
    step._oc = step.outputs.c()
    step(ro, pol)
    torch.cuda.synchronize()
    klp, kent = step.outputs.coeff_logprob, step.outputs.coeff_entropy
    st, want = oracle.logits_grad(logits.double().cpu().numpy(), tokens.cpu().numpy(),
                                  f32(klp.cpu().numpy()), f32(kent.cpu().numpy()))
    assert st == 0
    got = step.outputs.dlogits.float().cpu().numpy()
    assert np.isfinite(got).all(), "every row written"
    assert_rows_close(got, want, rel=TOL if dtype == torch.float32 else 1e-2, what=f"fused {cfg_name}")


def test_fused_dlogits_in_the_grpo_step(oracle):
    from paper_2510_06710_b200.core import EpisodeTable, GrpoAssemblyOptions, GrpoParams
    cfg = synth.SynthConfig(**{**synth.CONFIGS["cfg4"].__dict__, "num_envs": 16, "num_chunks": 8,
                               "max_episode_steps": 64})
    d = synth.episodes_numpy(cfg)
    logits, tokens, old = synth.token_tensors(cfg)
    d["tokens"], d["old_logprob"] = tokens.cpu().numpy(), old.cpu().numpy()
    a, l, v = synth.SPECS["cfg4"]
    ro = RolloutBuffer.from_arrays(d, d["boot_scalar"], cfg.vocab)
    step = optim.GrpoStep(ro, GrpoAssemblyOptions(GranularitySpec(Level(a), Level(l), Level(v)), apply_filter=False),
                          GrpoParams(0.2))
    step.outputs.dlogits = torch.full_like(logits, float("nan"))
    step._oc = step.outputs.c()
    step(ro, EpisodeTable.from_arrays(d), PolicyOutputs(logits))
    torch.cuda.synchronize()
    klp = step.outputs.coeff_logprob
    st, want = oracle.logits_grad(logits.double().cpu().numpy(), tokens.cpu().numpy(),
                                  f32(klp.cpu().numpy()), np.zeros(klp.numel()))
    assert st == 0
    got = step.outputs.dlogits.cpu().numpy()
    assert np.isfinite(got).all()
    assert_rows_close(got, want, what="fused grpo")
