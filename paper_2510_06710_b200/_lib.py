"""ctypes binding of include/ckrl.h (the C ABI of libckrl.so).

The structures below mirror ckrl.h field for field. Loading fails loudly when the
library is missing: there is no Python / CPU fallback for the hot path.
"""
from __future__ import annotations

import ctypes as C
import os

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CKRL_LIB") or os.path.join(HERE, "libckrl.so")

LEVEL_CHUNK, LEVEL_ACTION, LEVEL_TOKEN = 0, 1, 2
DTYPE_F32, DTYPE_BF16, DTYPE_U8, DTYPE_I32, DTYPE_F64, DTYPE_TOKEN_ROWS = 0, 1, 2, 3, 4, 5
FLAG_TERMINATED, FLAG_TRUNCATED, FLAG_VALID = 1, 2, 4
DIAG_COUNT = 8
DIAG_NAMES = ("loss", "surrogate", "value_loss", "entropy", "clip_frac", "approx_kl", "units",
              "status")

vp = C.c_void_p


class Granularity(C.Structure):
    _fields_ = [("advantage_level", C.c_int32), ("logprob_level", C.c_int32),
                ("value_level", C.c_int32)]


class GaeParams(C.Structure):
    _fields_ = [("gamma", C.c_double), ("lambda_", C.c_double)]


class PpoParams(C.Structure):
    _fields_ = [("clip_eps", C.c_double), ("value_loss_coef", C.c_double),
                ("entropy_coef", C.c_double), ("advantage_normalization", C.c_int32)]


class GrpoParams(C.Structure):
    _fields_ = [("clip_eps", C.c_double)]


class GrpoOptions(C.Structure):
    _fields_ = [("eps_std", C.c_double), ("apply_filter", C.c_int32),
                ("filter_lower", C.c_double), ("filter_upper", C.c_double),
                ("length_normalized", C.c_int32), ("min_group_size", C.c_int32)]


class Rollout(C.Structure):
    _fields_ = [("num_envs", C.c_int32), ("num_chunks", C.c_int32), ("chunk_len", C.c_int32),
                ("tokens_per_action", C.c_int32), ("vocab", C.c_int32),
                ("token_dtype", C.c_int32), ("tokens", vp), ("old_logprob", vp),
                ("reward", vp), ("flags", vp), ("episode_id", vp), ("value_scalar", vp),
                ("value_vector", vp), ("bootstrap", vp)]


class PolicyOutputs(C.Structure):
    _fields_ = [("logits_dtype", C.c_int32), ("logits", vp), ("values", vp)]


class PolicyHead(C.Structure):
    _fields_ = [("hidden", C.c_int32), ("vocab", C.c_int32), ("feature", vp), ("w_pol", vp), ("b_pol", vp)]


class Episodes(C.Structure):
    _fields_ = [("count", C.c_int32), ("env_id", vp), ("episode_id", vp), ("start_step", vp),
                ("length", vp), ("total_reward", vp), ("first_success", vp), ("complete", vp),
                ("task_id", vp), ("reset_state_id", vp)]


class PpoBatchC(C.Structure):
    _fields_ = [("counted", vp), ("advantages", vp), ("returns", vp)]


class GrpoBatchC(C.Structure):
    _fields_ = [("env_group", vp), ("env_member", vp), ("env_episode", vp),
                ("env_advantage", vp), ("env_group_size", vp), ("slot_weight", vp),
                ("slot_member", vp), ("group_counts", vp)]


class LossOutputs(C.Structure):
    _fields_ = [("coeff_logprob", vp), ("coeff_entropy", vp), ("coeff_value", vp),
                ("token_logprob", vp), ("token_entropy", vp), ("dlogits", vp),
                ("action_entropy", vp), ("chunk_entropy", vp)]


class EnvConfig(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "kind", "num_envs", "max_episode_steps", "auto_reset", "ignore_terminations",
        "use_fixed_reset_state_ids", "chunk_len", "grid_size", "reward_shaping",
        "num_reset_states", "success_step", "deferred_reset")] + [("seed", C.c_uint64)]


class PolicyDesc(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("obs_dim", "hidden", "trunk_layers", "value_hidden",
                                         "vocab", "chunk_len", "tokens_per_action")]


SAMPLER_REFERENCE, SAMPLER_PARALLEL = 0, 1
PLACEMENT_COLOCATED, PLACEMENT_DISAGGREGATED, PLACEMENT_HYBRID = 0, 1, 2


class PipelineSpec(C.Structure):
    _fields_ = [("env", EnvConfig), ("policy", PolicyDesc), ("num_chunks", C.c_int32),
                ("stages", C.c_int32), ("sample_seed", C.c_uint64), ("reset_state_ids", vp),
                ("sampler", C.c_int32), ("placed", C.c_int32), ("gen_device", C.c_int32), ("gen_workspace", vp),
                ("gen_workspace_bytes", C.c_size_t)]


PIPELINE_OUTPUT_FIELDS = (
    "tokens", "old_logprob", "old_logprob_f64", "reward", "reward_f64", "flags", "episode_id",
    "value_scalar", "value_scalar_f64", "value_vector", "value_vector_f64", "boot_scalar",
    "boot_scalar_f64", "boot_vector0", "boot_vector0_f64", "episode_count", "ep_env_id",
    "ep_episode_id", "ep_start", "ep_length", "ep_total_reward", "ep_first_success",
    "ep_complete", "ep_task", "ep_reset_id", "status", "logits")


class PipelineOutputs(C.Structure):
    _fields_ = [(n, vp) for n in PIPELINE_OUTPUT_FIELDS]


# (name, restype, argtypes) for every exported symbol of ckrl.h
P = C.POINTER
SIGNATURES = {
    "ckrl_version": (C.c_char_p, []),
    "ckrl_status_string": (C.c_char_p, [C.c_int32]),
    "ckrl_last_error": (C.c_char_p, []),
    "ckrl_validate_granularity": (C.c_int32, [P(Granularity)]),
    "ckrl_workspace_bytes": (C.c_size_t, [C.c_int32] * 5),
    "ckrl_workspace_init": (C.c_int32, [vp, C.c_size_t, vp]),
    "ckrl_stats_record_bytes": (C.c_size_t, []),
    "ckrl_merge_stats_host": (C.c_int32, [vp, C.c_int32, P(C.c_double), P(C.c_double),
                                          P(C.c_int64)]),
    "ckrl_compute_gae": (C.c_int32, [C.c_int32, vp, vp, vp, vp, vp, P(GaeParams), vp, vp, vp]),
    "ckrl_assemble_ppo_batch": (C.c_int32, [P(Rollout), P(GaeParams), P(Granularity),
                                            P(PpoBatchC), vp, C.c_size_t, vp]),
    "ckrl_normalize_advantages": (C.c_int32, [P(Rollout), P(Granularity), P(PpoBatchC), vp,
                                              C.c_size_t, vp]),
    "ckrl_assemble_grpo_batch": (C.c_int32, [P(Rollout), P(Episodes), P(Granularity),
                                             P(GrpoOptions), P(GrpoBatchC), vp, C.c_size_t, vp]),
    "ckrl_token_stats": (C.c_int32, [C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, vp,
                                     C.c_int32, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "ckrl_project_token_stats": (C.c_int32, [C.c_int64, P(PolicyHead), C.c_int32, vp, vp, vp, vp, C.c_int32,
                                             vp, vp]),
    "ckrl_ppo_loss": (C.c_int32, [P(Rollout), P(PpoBatchC), P(PolicyOutputs), P(Granularity),
                                  P(PpoParams), P(LossOutputs), vp, vp, C.c_size_t, vp]),
    "ckrl_grpo_loss": (C.c_int32, [P(Rollout), P(GrpoBatchC), P(PolicyOutputs), P(Granularity),
                                   P(GrpoParams), P(LossOutputs), vp, vp, C.c_size_t, vp]),
    "ckrl_ppo_step": (C.c_int32, [P(Rollout), P(PolicyOutputs), P(GaeParams), P(Granularity),
                                  P(PpoParams), P(PpoBatchC), P(LossOutputs), vp, vp,
                                  C.c_size_t, vp, vp]),
    "ckrl_grpo_step": (C.c_int32, [P(Rollout), P(Episodes), P(PolicyOutputs), P(Granularity),
                                   P(GrpoOptions), P(GrpoParams), P(GrpoBatchC),
                                   P(LossOutputs), vp, vp, C.c_size_t, vp, vp]),
    "ckrl_ppo_step_assemble": (C.c_int32, [P(Rollout), P(GaeParams), P(Granularity), P(PpoBatchC), vp,
                                           C.c_size_t, vp, vp]),
    "ckrl_ppo_step_loss": (C.c_int32, [P(Rollout), P(PolicyOutputs), P(Granularity), P(PpoParams),
                                       P(PpoBatchC), P(LossOutputs), vp, vp, C.c_size_t, vp, vp]),
    "ckrl_grpo_step_assemble": (C.c_int32, [P(Rollout), P(Episodes), P(Granularity), P(GrpoOptions),
                                            P(GrpoBatchC), vp, C.c_size_t, vp, vp]),
    "ckrl_grpo_step_loss": (C.c_int32, [P(Rollout), P(PolicyOutputs), P(Granularity), P(GrpoParams),
                                        P(GrpoBatchC), P(LossOutputs), vp, vp, C.c_size_t, vp, vp]),
    "ckrl_read_diagnostics": (C.c_int32, [vp, vp, vp]),
    "ckrl_logits_grad": (C.c_int32, [C.c_int64, C.c_int32, C.c_int32, vp, C.c_int32, vp, vp, vp,
                                     C.c_int32, vp, vp, vp]),
    "ckrl_read_status": (C.c_int32, [vp, vp]),
    "ckrl_debug_cta_times": (C.c_int32, [vp, C.c_int32]),
    "ckrl_adam_workspace_bytes": (C.c_size_t, []),
    "ckrl_dump_slab": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, vp, vp, vp, vp,
                                   C.c_int32, C.c_char_p, C.c_size_t, P(C.c_size_t)]),
    "ckrl_save_checkpoint": (C.c_int32, [P(PolicyDesc), vp, C.c_char_p]),
    "ckrl_load_checkpoint": (C.c_int32, [C.c_char_p, P(PolicyDesc), vp, C.c_int64, P(C.c_int64)]),
    "ckrl_adam_step": (C.c_int32, [C.c_int32, C.c_int64, vp, vp, vp, vp, vp, C.c_int64, vp, vp, vp,
                                   C.c_size_t, vp, vp]),
    "ckrl_debug_timeline": (C.c_int32, [vp, C.c_int32]),
    "ckrl_select_records": (C.c_int32, [P(Rollout), P(PpoBatchC), P(PolicyOutputs), P(Granularity),
                                        C.c_int64, vp, P(Rollout), P(PpoBatchC), P(PolicyOutputs), vp,
                                        C.c_size_t, vp]),
    "ckrl_read_stats": (C.c_int32, [vp, C.c_size_t, C.c_int32, vp, vp, vp]),
    "ckrl_select_groups": (C.c_int32, [C.c_int32, vp, vp, C.c_int32, vp, vp, C.c_size_t, vp]),
    "ckrl_grpo_group_advantage": (C.c_int32, [C.c_int32, vp, vp, C.c_double, vp, vp, vp]),
    "ckrl_success_rate_filter": (C.c_int32, [C.c_int32, vp, vp, C.c_double, C.c_double, vp, vp,
                                             vp]),
    "ckrl_valid_action_mask": (C.c_int32, [C.c_int32, vp, vp, vp, vp, vp]),
    "ckrl_length_norm_weights": (C.c_int32, [C.c_int32, vp, vp, vp, C.c_int32, vp, vp]),
    "ckrl_slab_success_rate": (C.c_int32, [P(Episodes), vp, vp]),
    "ckrl_policy_num_params": (C.c_int64, [P(PolicyDesc)]),
    "ckrl_pipeline_workspace_bytes": (C.c_size_t, [P(PipelineSpec)]),
    "ckrl_pipeline_gen_workspace_bytes": (C.c_size_t, [P(PipelineSpec)]),
    "ckrl_placement_mode": (C.c_int32, [C.c_int32] * 8 + [P(C.c_int32)]),
    "ckrl_pipeline_run": (C.c_int32, [P(PipelineSpec), vp, P(PipelineOutputs), vp, C.c_size_t,
                                      vp]),
    "ckrl_comm_unique_id": (C.c_int32, [vp]),
    "ckrl_comm_create": (C.c_int32, [C.c_int32, C.c_int32, vp, P(vp)]),
    "ckrl_comm_ipc_handle": (C.c_int32, [vp, vp]),
    "ckrl_comm_open_peers": (C.c_int32, [vp, vp]),
    "ckrl_comm_set_peers": (C.c_int32, [vp, P(vp)]),
    "ckrl_comm_destroy": (C.c_int32, [vp]),
}

_LIB = None


def lib():
    """Load libckrl.so (once). Raises if the CUDA extension was not built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = h
    return _LIB


def check(status: int):
    """Map a ckrl status code to the reference's exception types (core/errors.hpp)."""
    if status != 0:
        msg = lib().ckrl_last_error().decode(errors="replace")
        raise errors.from_status(status, msg)
