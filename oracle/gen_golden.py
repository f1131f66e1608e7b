"""TEST INFRASTRUCTURE — generates tests/golden/*.npz from the UNMODIFIED reference.

Run here (where /root/reference exists and `make -C oracle` built oracle/_ref):

    python oracle/gen_golden.py

Each fixture is one rollout produced by the reference's own StageSim/StageGen
(placement/rollout.cpp:11-109) with a reference PolicyNet of the stated (vocab, M),
exported in the SoA layout of include/ckrl.h (inputs, in float64), together with
the reference's outputs for every granularity spec:

  ppo/<a>_<l>_<v>/{counted, adv_raw, ret, adv_norm, diag}   assemble_ppo_batch ->
        normalize_advantages -> ppo_loss          (assembler.cpp:78-195, update.cpp:14-45,
                                                   losses.cpp:62-232)
  grpo/<a>_<l>_<v>_ln<0|1>/{env_*, slot_weight, slot_member, diag, groups_*, status}
        assemble_grpo_batch -> grpo_loss           (assembler.cpp:197-267, losses.cpp:234-331)
  lp_cur / ent_cur                                  PolicyNet::evaluate_chunk (policy_net.cpp:333-357)

The GPU box has no /root/reference; these committed fixtures are what the GPU
parity tests check against there.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.bindings import RefScenario  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

PPO_SPECS = [(0, 0, 0), (0, 1, 0), (0, 2, 0), (1, 1, 1), (1, 2, 1)]
GRPO_SPECS = [(0, 0, 0), (0, 1, 0), (0, 2, 0)]
PPO_PARAMS = dict(gamma=0.99, lam=0.95, normalize=True, clip=0.2, vcoef=0.5, ecoef=0.01)

SCENARIOS = {
    # partial reset, immediate mode: post-reset tail slots inside chunks, truncations
    "ppo_toyreach_immediate": dict(kind="ppo", num_envs=6, num_chunks=6, chunk_length=3,
                                   max_episode_steps=7, auto_reset=1, env_seed=101),
    # deferred reset with auto_reset: frozen slots mid-chunk, reset at chunk end
    "ppo_scripted_deferred": dict(kind="ppo", env_kind=1, success_step=3, num_envs=4,
                                  num_chunks=5, chunk_length=4, max_episode_steps=6,
                                  auto_reset=1, deferred_reset=1, env_seed=102),
    # fixed-length episodes (ignore_terminations): truncation bootstraps only
    "ppo_toyreach_fixedlen": dict(kind="ppo", num_envs=4, num_chunks=5, chunk_length=2,
                                  max_episode_steps=4, auto_reset=1, ignore_terminations=1,
                                  env_seed=103),
    # the OpenVLA action space: 256 bins x 7 tokens
    "ppo_v256_m7": dict(kind="ppo", vocab=256, tokens_per_action=7, num_envs=3, num_chunks=6,
                        chunk_length=2, max_episode_steps=5, env_seed=104, hidden=4),
    # GRPO valid-action-mask mode (auto_reset=false, deferred freeze), binary returns
    "grpo_toyreach_mask": dict(kind="grpo", num_envs=16, group_size=4,
                               use_fixed_reset_state_ids=1, auto_reset=0, deferred_reset=1,
                               max_episode_steps=8, num_chunks=4, chunk_length=2, env_seed=105),
    # shaped (non-binary) returns through the same filter
    "grpo_toyreach_shaped": dict(kind="grpo", num_envs=16, group_size=4,
                                 use_fixed_reset_state_ids=1, auto_reset=0, deferred_reset=1,
                                 max_episode_steps=8, num_chunks=4, chunk_length=2,
                                 reward_shaping=1, env_seed=106),
    # fixed-length + reset ids drawn with replacement (groups merge by key), no filter
    "grpo_fixedlen_merged": dict(kind="grpo", num_envs=16, group_size=4,
                                 use_fixed_reset_state_ids=1, ignore_terminations=1,
                                 auto_reset=0, deferred_reset=1, max_episode_steps=8,
                                 num_chunks=2, chunk_length=4, ids_with_replacement=1,
                                 num_reset_states=3, env_seed=107, apply_filter=0),
    # all-success scripted groups: filter drops all; unfiltered with eps 0 -> DegenerateGroup
    "grpo_scripted_degenerate": dict(kind="grpo", env_kind=1, success_step=3, num_envs=8,
                                     group_size=4, use_fixed_reset_state_ids=1, auto_reset=0,
                                     deferred_reset=1, max_episode_steps=6, num_chunks=3,
                                     chunk_length=2, env_seed=108),
    "grpo_v256_m7": dict(kind="grpo", vocab=256, tokens_per_action=7, num_envs=8, group_size=4,
                         use_fixed_reset_state_ids=1, auto_reset=0, deferred_reset=1,
                         max_episode_steps=6, num_chunks=3, chunk_length=2, env_seed=109,
                         hidden=4),
}


def spec_key(spec):
    return "_".join(str(x) for x in spec)


def generate(name: str, cfg: dict) -> dict:
    cfg = dict(cfg)
    kind = cfg.pop("kind")
    apply_filter = cfg.pop("apply_filter", 1)
    sc = RefScenario(**cfg)
    d = sc.export()
    out = {k: v for k, v in d.items() if k != "V"}
    out["dims"] = np.array([sc.E, sc.Tc, sc.C, sc.M, sc.V], np.int64)
    if kind == "ppo":
        for spec in PPO_SPECS:
            r = sc.ppo(spec, **PPO_PARAMS)
            for k in ("counted", "adv_raw", "ret", "adv_norm", "diag"):
                out[f"ppo/{spec_key(spec)}/{k}"] = r[k]
            out[f"ppo/{spec_key(spec)}/status"] = np.array(r["status"])
        out["ppo_params"] = np.array([PPO_PARAMS[k] for k in ("gamma", "lam", "clip", "vcoef", "ecoef")])
    else:
        variants = [(1e-8, 1), (1e-8, 0)]
        if name == "grpo_scripted_degenerate":
            variants += [(0.0, 1)]
        for spec in GRPO_SPECS:
            for eps, ln in variants:
                for af in ((apply_filter,) if name != "grpo_scripted_degenerate" else (1, 0)):
                    r = sc.grpo(spec, eps_std=eps, apply_filter=bool(af), length_normalized=bool(ln))
                    key = f"grpo/{spec_key(spec)}_ln{ln}_eps{0 if eps == 0 else 1}_f{af}"
                    for k in ("env_group", "env_member", "env_episode", "env_adv", "env_group_size",
                              "slot_weight", "slot_member", "diag"):
                        out[f"{key}/{k}"] = r[k]
                    out[f"{key}/status"] = np.array(r["status"])
                    out[f"{key}/groups"] = np.array([r["groups_total"], r["groups_retained"]])
        out["grpo_params"] = np.array([0.0, 1.0, 0.2, 2])  # lower, upper, clip, min_group_size
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, cfg in SCENARIOS.items():
        data = generate(name, cfg)
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **data)
        print(f"{path}: {os.path.getsize(path) / 1024:.1f} KiB")


def dump_fixture():
    """dump_toyreach.npz: a reference rollout's SoA slab + the reference's own dump_slab text
    (core/types.cpp:9-28), for tests/test_formats.py / test_gpu_pipeline.py on the GPU box."""
    sc = RefScenario(num_envs=4, num_chunks=5, chunk_length=3, max_episode_steps=5, reward_shaping=1,
                     env_seed=21, sample_seed=22, net_seed=23)
    d = sc.export(with_logits=False)
    text = sc.dump_slab()
    path = os.path.join(OUT, "dump_toyreach.npz")
    np.savez_compressed(path, tokens=d["tokens"], reward=d["reward"], flags=d["flags"],
                        episode_id=d["episode_id"], text=np.frombuffer(text.encode(), np.uint8))
    print("wrote", path, len(text), "bytes of dump text")


def proj_fixture():
    """proj_h128.npz: the reference's own policy head (forward_logits + evaluate_chunk on a
    head-only PolicyNet, ref_shim.cpp refx_project_token_stats) over bf16-representable
    features / W_pol / b_pol, for tests/test_gpu_projection.py on the GPU box (row N2)."""
    import torch
    from oracle.bindings import ref_project_token_stats
    g = torch.Generator().manual_seed(31)
    rows, H, V = 200, 128, 256
    f = torch.randn(rows, H, generator=g).to(torch.bfloat16).double().numpy()
    W = (torch.randn(V, H, generator=g) * (2.0 / H ** 0.5)).to(torch.bfloat16).double().numpy()
    b = (0.5 * torch.randn(V, generator=g)).to(torch.bfloat16).double().numpy()
    tok = torch.randint(0, V, (rows,), generator=g).numpy().astype(np.int32)
    logits, lp, ent = ref_project_token_stats(f, W, b, tok)
    path = os.path.join(OUT, "proj_h128.npz")
    np.savez_compressed(path, feature=f, w_pol=W, b_pol=b, tokens=tok, logits=logits, lp=lp, ent=ent)
    print("wrote", path)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "dump":
        dump_fixture()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "proj":
        proj_fixture()
        sys.exit(0)
    main()
