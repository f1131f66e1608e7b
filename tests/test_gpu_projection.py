"""Row N2 on the GPU: the policy head (logits = W_pol h + b_pol, policy/policy_net.cpp:265-274) on
the tensor cores (tcgen05.mma into TMEM, csrc/proj.cu) fused with evaluate_chunk's per-position
log-prob and entropy (:333-357), against the reference fixture (proj_h128.npz, the reference's
own forward_logits / evaluate_chunk) and the oracle restatement at other shapes (bf16 inputs
are exact in f64, so the oracle sees the same numbers the tensor cores do; the device
accumulates in f32: 1e-5 relative). The losses fed with the projection's token rows
(CKRL_DTYPE_TOKEN_ROWS) must equal the losses fed with the logits."""
import numpy as np
import pytest
import torch

from conftest import assert_close, load_golden

pytestmark = pytest.mark.gpu

import paper_2510_06710_b200 as ck  # noqa: E402
from paper_2510_06710_b200 import errors, optim, policy, synth  # noqa: E402
from paper_2510_06710_b200.core import (GaeParams, GranularitySpec, GrpoAssemblyOptions,  # noqa: E402
                                        GrpoParams, Level, EpisodeTable, PolicyOutputs, PpoParams,
                                        RolloutBuffer)

TOL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _device():
    assert torch.cuda.is_available()
    ck.lib()


def _bf(x):
    return torch.tensor(x, dtype=torch.float64).to(torch.bfloat16).cuda()


def test_projection_vs_reference_fixture():
    d = load_golden("proj_h128.npz")
    f, W, b = _bf(d["feature"]), _bf(d["w_pol"]), torch.tensor(d["b_pol"], dtype=torch.float32).cuda()
    tok = torch.tensor(d["tokens"], dtype=torch.int32).cuda()
    out = policy.project_token_stats(f, W, b, tok, want_logits=torch.float32)
    assert_close(out["logits"].cpu().numpy(), d["logits"], TOL, "proj logits vs reference")
    assert_close(out["token_logprob"].cpu().numpy(), d["lp"], TOL, "proj lp vs reference")
    assert_close(out["token_entropy"].cpu().numpy(), d["ent"], TOL, "proj H vs reference")
    rows = out["token_rows"].cpu().numpy()
    np.testing.assert_array_equal(rows[:, 0], out["token_logprob"].cpu().numpy())
    ent_from_rows = np.ascontiguousarray(rows).view(np.float32).reshape(-1, 4)[:, 2]  # {f64 lp, f32 H, u32 0}
    np.testing.assert_array_equal(ent_from_rows, out["token_entropy"].cpu().numpy())


@pytest.mark.parametrize("rows,H", [(1, 64), (127, 64), (129, 128), (1000, 320), (4099, 1024), (300, 4096)])
@pytest.mark.parametrize("u8", [False, True])
def test_projection_vs_oracle(oracle, rows, H, u8):
    g = torch.Generator(device="cuda").manual_seed(rows + H)
    f = torch.randn(rows, H, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(256, H, device="cuda", generator=g) * (2.5 / H ** 0.5)).to(torch.bfloat16)
    b = 0.3 * torch.randn(256, device="cuda", generator=g) if H != 128 else None
    tok = torch.randint(0, 256, (rows,), device="cuda", generator=g, dtype=torch.int32)
    tk = tok.to(torch.uint8) if u8 else tok
    out = policy.project_token_stats(f, W, b, tk, want_logits=torch.float32)
    bb = None if b is None else b.double().cpu().numpy()
    logits = oracle.project_logits(f.double().cpu().numpy(), W.double().cpu().numpy(), bb)
    lp, ent = oracle.token_stats(logits, tok.cpu().numpy())
    # fp32 accumulation of H bf16 products (the north star's "fp32 accumulate"): a random walk
    # of H round-offs, so beyond H = 1024 the bound grows as sqrt(H / 1024) — at H = 4096 the
    # measured worst logit is 1.5e-5 of the rms, the entropy 9e-6, the log-prob 5e-6
    tol = TOL * max(1.0, (H / 1024) ** 0.5)
    assert_close(out["logits"].cpu().numpy(), logits, tol, f"proj logits rows={rows} H={H}")
    assert_close(out["token_logprob"].cpu().numpy(), lp, tol, f"proj lp rows={rows} H={H}")
    assert_close(out["token_entropy"].cpu().numpy(), ent, tol, f"proj H rows={rows} H={H}")


def test_projection_bf16_logits_and_rows_only(oracle):
    rows, H = 777, 256
    g = torch.Generator(device="cuda").manual_seed(5)
    f = torch.randn(rows, H, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(256, H, device="cuda", generator=g) / H ** 0.5).to(torch.bfloat16)
    tok = torch.randint(0, 256, (rows,), device="cuda", generator=g, dtype=torch.int32)
    a = policy.project_token_stats(f, W, None, tok)
    b = policy.project_token_stats(f, W, None, tok, want_logits=torch.bfloat16)
    torch.testing.assert_close(a["token_rows"], b["token_rows"], rtol=0, atol=0)  # deterministic
    ref = (f.float() @ W.float().t()).to(torch.bfloat16)
    torch.testing.assert_close(b["logits"], ref, rtol=1e-2, atol=1e-2)


def test_projection_argument_errors():
    f = torch.zeros(4, 96, dtype=torch.bfloat16, device="cuda")
    W = torch.zeros(256, 96, dtype=torch.bfloat16, device="cuda")
    tok = torch.zeros(4, dtype=torch.int32, device="cuda")
    with pytest.raises(errors.LengthMismatch):
        policy.project_token_stats(f, W, None, tok)  # H not a multiple of 64
    f = torch.zeros(4, 64, dtype=torch.bfloat16, device="cuda")
    W = torch.zeros(100, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(errors.LengthMismatch):
        policy.project_token_stats(f, W, None, tok)  # vocab != 256
    out = policy.project_token_stats(torch.zeros(0, 64, dtype=torch.bfloat16, device="cuda"),
                                     torch.zeros(256, 64, dtype=torch.bfloat16, device="cuda"), None,
                                     torch.zeros(0, dtype=torch.int32, device="cuda"))
    assert out["token_rows"].shape == (0, 2)


def _head_inputs(cfg, H, seed):
    """Features and a head whose logits have the synthetic slab's spread, plus the logits the
    head produces (f32, from the projection itself) for the logits-fed loss."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    shape = (cfg.num_envs, cfg.num_chunks, cfg.chunk_len, cfg.tokens_per_action)
    f = torch.randn(*shape, H, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(256, H, device="cuda", generator=g) * (2.0 / H ** 0.5)).to(torch.bfloat16)
    b = 0.1 * torch.randn(256, device="cuda", generator=g)
    return f, W, b


@pytest.mark.parametrize("cfg_name", ["cfg3", "cfg1"])
def test_ppo_loss_from_token_rows_equals_logits(cfg_name):
    cfg = synth.SynthConfig(**{**synth.CONFIGS[cfg_name].__dict__, "num_envs": 24})
    d = synth.episodes_numpy(cfg)
    _, tokens, old = synth.token_tensors(cfg)
    f, W, b = _head_inputs(cfg, 256, 7)
    proj = policy.project_token_stats(f, W, b, tokens, want_logits=torch.float32)
    d["tokens"], d["old_logprob"] = tokens, proj["token_logprob"].float() + 0.05 * torch.randn_like(old)
    a, l, v = synth.SPECS[cfg_name]
    spec = GranularitySpec(Level(a), Level(l), Level(v))
    boot = d["boot_scalar"] if a == 0 else d["boot_vector0"]
    ro = RolloutBuffer.from_arrays(d, boot, cfg.vocab)
    nv = torch.tensor(d["new_value_scalar"] if v == 0 else d["new_value_vector"], dtype=torch.float32, device="cuda")
    res = []
    for pol in (PolicyOutputs(proj["logits"], nv), PolicyOutputs(None, nv, token_rows=proj["token_rows"])):
        step = optim.PpoStep(ro, GaeParams(0.99, 0.95), spec, PpoParams(0.2, 0.5, 0.01, True))
        step(ro, pol)
        res.append((step.diagnostics(), step.outputs.coeff_logprob.clone(), step.outputs.coeff_entropy.clone()))
    (d0, k0, e0), (d1, k1, e1) = res
    for key in ("loss", "surrogate", "value_loss", "entropy", "approx_kl", "clip_frac"):
        assert_close([d1[key]], [d0[key]], TOL, f"{cfg_name} token-rows {key}")
    assert_close(k1.cpu().numpy(), k0.cpu().numpy(), TOL, f"{cfg_name} token-rows coeff_lp")
    assert_close(e1.cpu().numpy(), e0.cpu().numpy(), TOL, f"{cfg_name} token-rows coeff_ent")


def test_grpo_loss_from_token_rows_equals_logits():
    cfg = synth.SynthConfig(**{**synth.CONFIGS["cfg4"].__dict__, "num_envs": 16, "num_chunks": 8,
                               "max_episode_steps": 64})  # complete fixed-length episodes
    d = synth.episodes_numpy(cfg)
    _, tokens, old = synth.token_tensors(cfg)
    f, W, b = _head_inputs(cfg, 128, 9)
    proj = policy.project_token_stats(f, W, b, tokens, want_logits=torch.float32)
    d["tokens"], d["old_logprob"] = tokens, proj["token_logprob"].float() + 0.05 * torch.randn_like(old)
    a, l, v = synth.SPECS["cfg4"]
    spec = GranularitySpec(Level(a), Level(l), Level(v))
    ro = RolloutBuffer.from_arrays(d, d["boot_scalar"], cfg.vocab)
    ept = EpisodeTable.from_arrays(d)
    res = []
    for pol in (PolicyOutputs(proj["logits"]), PolicyOutputs(None, token_rows=proj["token_rows"])):
        step = optim.GrpoStep(ro, GrpoAssemblyOptions(spec), GrpoParams(0.2))
        step(ro, ept, pol)
        res.append((step.diagnostics(), step.outputs.coeff_logprob.clone()))
    (d0, k0), (d1, k1) = res
    # the GRPO loss is a signed sum whose terms cancel (group-relative advantages sum to ~0):
    # its error scales with the terms' L1 mass, which at token level is sum |coeff_lp|
    mass = float(k0.abs().sum())
    for key in ("loss", "surrogate"):
        assert_close([d1[key]], [d0[key]], TOL, f"grpo token-rows {key}", floor=mass)
    for key in ("approx_kl", "clip_frac"):
        assert_close([d1[key]], [d0[key]], TOL, f"grpo token-rows {key}")
    assert_close(k1.cpu().numpy(), k0.cpu().numpy(), TOL, "grpo token-rows coeff_lp")


def test_token_rows_reject_dlogits():
    """The softmax-backward seam needs the logits; with token rows the loss refuses it up front."""
    cfg = synth.SynthConfig(**{**synth.CONFIGS["cfg3"].__dict__, "num_envs": 4})
    d = synth.episodes_numpy(cfg)
    _, tokens, old = synth.token_tensors(cfg)
    d["tokens"], d["old_logprob"] = tokens, old
    ro = RolloutBuffer.from_arrays(d, d["boot_scalar"], cfg.vocab)
    rows = torch.zeros((*tokens.shape, 2), dtype=torch.float64, device="cuda")
    nv = torch.tensor(d["new_value_scalar"], dtype=torch.float32, device="cuda")
    step = optim.PpoStep(ro, GaeParams(0.99, 0.95), GranularitySpec(Level(0), Level(0), Level(0)),
                         PpoParams(0.2, 0.5, 0.01, True))
    step.outputs.dlogits = torch.empty((*tokens.shape, 256), dtype=torch.float32, device="cuda")
    step._oc = step.outputs.c()
    with pytest.raises(errors.InvalidArgument):
        step(ro, PolicyOutputs(None, nv, token_rows=rows))
