"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU oracle and the reference shim.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
arm may import this module; the product path (paper_2510_06710_b200) never does.

* ``Oracle``  — oracle/liboracle.so, the C restatement (oracle/ckrl_oracle.c).
* ``RefScenario`` — oracle/_ref/libchunkrl_ref.so, the unmodified reference sources
  plus oracle/ref_shim.cpp. Only exists where /root/reference was present at build
  time (this container; the built .so travels to the GPU box with the snapshot).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libchunkrl_ref.so")

CHUNK, ACTION, TOKEN = 0, 1, 2
LEVELS = {"chunk": CHUNK, "action": ACTION, "token": TOKEN}


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class OrcRollout(C.Structure):
    _fields_ = [("E", C.c_int), ("Tc", C.c_int), ("C", C.c_int), ("M", C.c_int), ("V", C.c_int),
                ("tokens", C.c_void_p), ("old_logprob", C.c_void_p), ("reward", C.c_void_p),
                ("flags", C.c_void_p), ("episode_id", C.c_void_p), ("value_scalar", C.c_void_p),
                ("value_vector", C.c_void_p), ("bootstrap", C.c_void_p)]


class OrcEpisodes(C.Structure):
    _fields_ = [("count", C.c_int), ("env_id", C.c_void_p), ("episode_id", C.c_void_p),
                ("start_step", C.c_void_p), ("length", C.c_void_p), ("total_reward", C.c_void_p),
                ("first_success", C.c_void_p), ("complete", C.c_void_p), ("task_id", C.c_void_p),
                ("reset_state_id", C.c_void_p)]


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Oracle:
    """Double-precision restatement, driven on numpy SoA arrays (include/ckrl.h layout)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
        self.lib = C.CDLL(path)
        for name in ("orc_compute_gae", "orc_assemble_ppo", "orc_normalize_advantages",
                     "orc_ppo_loss", "orc_grpo_group_advantage", "orc_success_rate_filter",
                     "orc_assemble_grpo", "orc_grpo_loss", "orc_validate_granularity",
                     "orc_logits_grad", "orc_adam_step"):
            getattr(self.lib, name).restype = C.c_int

    # --- rollout marshalling -------------------------------------------------
    def rollout(self, d: dict, bootstrap: np.ndarray):
        keep = dict(
            tokens=np.ascontiguousarray(d["tokens"], dtype=np.int32),
            old_logprob=_c64(d["old_logprob"]), reward=_c64(d["reward"]),
            flags=np.ascontiguousarray(d["flags"], dtype=np.uint8),
            episode_id=np.ascontiguousarray(d["episode_id"], dtype=np.int32),
            value_scalar=_c64(d["value_scalar"]), value_vector=_c64(d["value_vector"]),
            bootstrap=_c64(bootstrap))
        E, Tc, Cn, M = keep["tokens"].shape[:4]
        V = int(d.get("V", d["logits"].shape[-1] if "logits" in d else 1))
        ro = OrcRollout(E, Tc, Cn, M, V, *[_p(keep[k]) for k in (
            "tokens", "old_logprob", "reward", "flags", "episode_id", "value_scalar",
            "value_vector", "bootstrap")])
        ro._keep = keep
        return ro

    def episodes(self, d: dict):
        keep = dict(
            env_id=np.ascontiguousarray(d["ep_env_id"], dtype=np.int32),
            episode_id=np.ascontiguousarray(d["ep_episode_id"], dtype=np.int32),
            start_step=np.ascontiguousarray(d["ep_start"], dtype=np.int64),
            length=np.ascontiguousarray(d["ep_length"], dtype=np.int64),
            total_reward=_c64(d["ep_total_reward"]),
            first_success=np.ascontiguousarray(d["ep_first_success"], dtype=np.int64),
            complete=np.ascontiguousarray(d["ep_complete"], dtype=np.uint8),
            task_id=np.ascontiguousarray(d["ep_task"], dtype=np.int32),
            reset_state_id=np.ascontiguousarray(d["ep_reset_id"], dtype=np.int32))
        ep = OrcEpisodes(len(keep["env_id"]), *[_p(keep[k]) for k in (
            "env_id", "episode_id", "start_step", "length", "total_reward", "first_success",
            "complete", "task_id", "reset_state_id")])
        ep._keep = keep
        return ep

    # --- ops -----------------------------------------------------------------
    def compute_gae(self, rewards, values, boot, term, trunc, gamma, lam):
        r, v, b = _c64(rewards), _c64(values), _c64(boot)
        te = np.ascontiguousarray(term, dtype=np.uint8)
        tr = np.ascontiguousarray(trunc, dtype=np.uint8)
        n = len(r)
        if not (len(v) == len(b) == len(te) == len(tr) == n):
            raise ValueError("compute_gae: input lengths differ")
        adv, ret = np.zeros(n), np.zeros(n)
        self.lib.orc_compute_gae(n, _p(r), _p(v), _p(b), _p(te), _p(tr), C.c_double(gamma),
                                 C.c_double(lam), _p(adv), _p(ret))
        return adv, ret

    def token_stats(self, logits, tokens):
        lg = _c64(logits)
        V = lg.shape[-1]
        rows = lg.size // V
        tk = np.ascontiguousarray(tokens, dtype=np.int32).reshape(-1)
        lp, ent = np.zeros(rows), np.zeros(rows)
        self.lib.orc_token_stats(C.c_int64(rows), V, _p(lg), _p(tk), _p(lp), _p(ent))
        return lp, ent

    def project_logits(self, feature, w_pol, b_pol=None):
        """logits_from_feature (policy_net.cpp:265-274) per row: [rows][H] x [V][H] -> [rows][V]."""
        f = _c64(feature)
        W = _c64(w_pol)
        V, H = W.shape
        f = f.reshape(-1, H)
        rows = f.shape[0]
        b = None if b_pol is None else _c64(b_pol).reshape(-1)
        out = np.zeros((rows, V))
        self.lib.orc_project_logits(C.c_int64(rows), H, V, _p(f), _p(W), _p(b), _p(out))
        return out

    def entropy_aggregates(self, ent, chunk_len, tokens_per_action, mask=None):
        """Per-token entropies [chunks*C*M] -> (action [chunks][C], chunk [chunks]) entropy in
        canonical order over the `mask` [chunks][C] slots (default all)."""
        Cn, M = chunk_len, tokens_per_action
        e = np.ascontiguousarray(ent, dtype=np.float64).reshape(-1)
        n = e.size // (Cn * M)
        act, chk = np.zeros((n, Cn)), np.zeros(n)
        mk = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8).reshape(-1)
        self.lib.orc_entropy_aggregates(C.c_int64(n), Cn, M, _p(e), _p(mk) if mk is not None else None,
                                        _p(act), _p(chk))
        return act, chk

    def logits_grad(self, logits, tokens, coeff_lp, coeff_ent):
        """dlogits per position (policy/policy_net.cpp:431-456); returns (status, [rows][V])."""
        lg = _c64(logits)
        V = lg.shape[-1]
        rows = lg.size // V
        tk = np.ascontiguousarray(tokens, dtype=np.int32).reshape(-1)
        kl, ke = _c64(np.reshape(coeff_lp, -1)), _c64(np.reshape(coeff_ent, -1))
        out = np.zeros((rows, V))
        st = self.lib.orc_logits_grad(C.c_int64(rows), V, _p(lg), _p(tk), _p(kl), _p(ke), _p(out))
        return st, out

    def adam_step(self, params, grad, m, v, t, lr, max_grad_norm=0.0, beta1=0.9, beta2=0.999, eps=1e-8):
        """Adam::step (optim/adam.cpp:15-41) in place on float64 arrays; returns (status, norm)."""
        norm = C.c_double(0.0)
        st = self.lib.orc_adam_step(C.c_int64(params.size), _p(params), _p(grad), _p(m), _p(v),
                                    C.c_double(lr), C.c_double(max_grad_norm), C.c_double(beta1),
                                    C.c_double(beta2), C.c_double(eps), C.c_int64(t), C.byref(norm))
        return st, norm.value

    def assemble_ppo(self, d, spec, gamma, lam):
        a, l, v = spec
        boot = d["boot_scalar"] if a == CHUNK else d["boot_vector0"]
        ro = self.rollout(d, boot)
        counted = np.zeros((ro.E, ro.Tc, ro.C), np.uint8)
        shape = (ro.E, ro.Tc) if a == CHUNK else (ro.E, ro.Tc, ro.C)
        adv, ret = np.zeros(shape), np.zeros(shape)
        st = self.lib.orc_assemble_ppo(C.byref(ro), a, l, v, C.c_double(gamma), C.c_double(lam),
                                       _p(counted), _p(adv), _p(ret))
        return st, counted, adv, ret

    def normalize_advantages(self, counted, adv, adv_level):
        E, Tc, Cn = counted.shape
        out = _c64(adv).copy()
        self.lib.orc_normalize_advantages(E, Tc, Cn, adv_level,
                                          _p(np.ascontiguousarray(counted, np.uint8)), _p(out))
        return out

    def ppo_loss(self, d, spec, counted, adv, ret, logits, new_values, clip, vcoef, ecoef):
        a, l, v = spec
        boot = d["boot_scalar"] if a == CHUNK else d["boot_vector0"]
        ro = self.rollout(d, boot)
        P = ro.C * ro.M
        coeff_lp = np.zeros((ro.E, ro.Tc, ro.C, ro.M))
        coeff_ent = np.zeros_like(coeff_lp)
        coeff_val = np.zeros((ro.E, ro.Tc) if v == CHUNK else (ro.E, ro.Tc, ro.C))
        diag = np.zeros(7)
        lg, nv = _c64(logits), _c64(new_values)
        cn = np.ascontiguousarray(counted, np.uint8)
        ad, rt = _c64(adv), _c64(ret)
        st = self.lib.orc_ppo_loss(C.byref(ro), a, l, v, _p(cn), _p(ad), _p(rt), _p(lg), _p(nv),
                                   C.c_double(clip), C.c_double(vcoef), C.c_double(ecoef),
                                   _p(coeff_lp), _p(coeff_ent), _p(coeff_val), _p(diag))
        del P
        return st, diag, coeff_lp, coeff_ent, coeff_val

    def grpo_group_advantage(self, rewards, eps):
        r = _c64(rewards)
        out = np.zeros(len(r))
        st = self.lib.orc_grpo_group_advantage(len(r), _p(r), C.c_double(eps), _p(out))
        return st, out

    def success_rate_filter(self, rewards, lower, upper):
        r = _c64(rewards)
        return bool(self.lib.orc_success_rate_filter(len(r), _p(r), C.c_double(lower), C.c_double(upper)))

    def valid_action_mask(self, length, success, fs):
        m = np.zeros(max(length, 0), np.uint8)
        self.lib.orc_valid_action_mask(C.c_int64(length), int(success), C.c_int64(fs), _p(m))
        return m.astype(bool)

    def length_norm_weights(self, length, success, fs, normalized):
        w = np.zeros(max(length, 0))
        self.lib.orc_length_norm_weights(C.c_int64(length), int(success), C.c_int64(fs),
                                         int(normalized), _p(w))
        return w

    def assemble_grpo(self, d, spec, eps_std=1e-8, apply_filter=True, lower=0.0, upper=1.0,
                      length_normalized=True, min_group_size=2):
        a, l, v = spec
        ro = self.rollout(d, d["boot_scalar"])
        ep = self.episodes(d)
        E = ro.E
        gt, gr = C.c_int(0), C.c_int(0)
        out = dict(env_group=np.zeros(E, np.int32), env_member=np.zeros(E, np.int32),
                   env_episode=np.zeros(E, np.int32), env_adv=np.zeros(E),
                   env_group_size=np.zeros(E, np.int32),
                   slot_weight=np.zeros((ro.E, ro.Tc, ro.C)),
                   slot_member=np.zeros((ro.E, ro.Tc, ro.C), np.uint8))
        st = self.lib.orc_assemble_grpo(
            C.byref(ro), C.byref(ep), a, l, v, C.c_double(eps_std), int(apply_filter),
            C.c_double(lower), C.c_double(upper), int(length_normalized), min_group_size,
            C.byref(gt), C.byref(gr), *[_p(out[k]) for k in (
                "env_group", "env_member", "env_episode", "env_adv", "env_group_size",
                "slot_weight", "slot_member")])
        out["groups_total"], out["groups_retained"] = gt.value, gr.value
        return st, out

    def grpo_loss(self, d, lp_level, asm, logits, clip):
        ro = self.rollout(d, d["boot_scalar"])
        coeff = np.zeros((ro.E, ro.Tc, ro.C, ro.M))
        diag = np.zeros(7)
        keep = {k: np.ascontiguousarray(asm[k]) for k in (
            "env_group", "env_member", "env_adv", "env_group_size", "slot_weight", "slot_member")}
        lg = _c64(logits)
        st = self.lib.orc_grpo_loss(
            C.byref(ro), lp_level, int(asm["groups_retained"]), _p(keep["env_group"]),
            _p(keep["env_member"]), _p(_c64(keep["env_adv"])), _p(keep["env_group_size"]),
            _p(_c64(keep["slot_weight"])), _p(keep["slot_member"].astype(np.uint8)), _p(lg),
            C.c_double(clip), _p(coeff), _p(diag))
        return st, diag, coeff


class RefCfg(C.Structure):
    _fields_ = [(n, C.c_int) for n in (
        "env_kind", "num_envs", "max_episode_steps", "auto_reset", "ignore_terminations",
        "use_fixed_reset_state_ids", "chunk_length", "grid_size", "num_reset_states",
        "success_step", "reward_shaping", "num_chunks", "deferred_reset", "group_size",
        "ids_with_replacement", "vocab", "tokens_per_action", "hidden", "trunk_layers",
        "value_hidden")] + [("env_seed", C.c_ulonglong), ("sample_seed", C.c_ulonglong),
                            ("net_seed", C.c_ulonglong), ("perturb", C.c_double)]


REF_DEFAULTS = dict(env_kind=0, num_envs=4, max_episode_steps=8, auto_reset=1,
                    ignore_terminations=0, use_fixed_reset_state_ids=0, chunk_length=2,
                    grid_size=5, num_reset_states=64, success_step=5, reward_shaping=0,
                    num_chunks=4, deferred_reset=0, group_size=1, ids_with_replacement=0,
                    vocab=4, tokens_per_action=2, hidden=6, trunk_layers=1, value_hidden=4,
                    env_seed=11, sample_seed=12, net_seed=13, perturb=0.05)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


_REF_LIB = None


def _ref_lib():
    global _REF_LIB
    if _REF_LIB is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_SO} missing (built by `make -C oracle ref` where /root/reference exists)")
        lib = C.CDLL(REF_SO)
        lib.refx_create.restype = C.c_void_p
        lib.refx_last_error.restype = C.c_char_p
        lib.refx_bpol_offset.restype = C.c_longlong
        lib.refx_adam.restype = C.c_int
        for n in ("refx_dump_slab", "refx_save_checkpoint", "refx_load_checkpoint"):
            getattr(lib, n).restype = C.c_int
        lib.refx_dump_slab.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]
        lib.refx_save_checkpoint.argtypes = [C.c_void_p, C.c_char_p]
        lib.refx_load_checkpoint.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_longlong,
                                             C.POINTER(C.c_longlong)]
        for n in ("refx_export", "refx_export_episodes", "refx_export_params", "refx_ppo_subset",
                  "refx_grpo_subset", "refx_ppo", "refx_grpo",
                  "refx_replay_ppo_grad", "refx_replay_grpo_grad"):
            getattr(lib, n).restype = C.c_int
        for n in ("refx_bench_ppo", "refx_bench_grpo"):
            getattr(lib, n).restype = C.c_double
        _REF_LIB = lib
    return _REF_LIB


def ref_adam(params, grads, lr, max_grad_norm=0.0, beta1=0.9, beta2=0.999, eps=1e-8):
    """The reference's optim::Adam over len(grads) steps (grads [steps][n], clipped in place);
    returns (status, params, grads, norms)."""
    lib = _ref_lib()
    p = _c64(params).copy()
    g = _c64(grads).copy()
    steps, n = g.shape
    norms = np.zeros(steps)
    st = lib.refx_adam(C.c_longlong(n), steps, _p(p), _p(g), C.c_double(lr), C.c_double(max_grad_norm),
                       C.c_double(beta1), C.c_double(beta2), C.c_double(eps), _p(norms))
    return st, p, g, norms


def ref_project_token_stats(feature, w_pol, b_pol, tokens):
    """The reference's forward_logits + evaluate_chunk on a head-only PolicyNet whose trunk
    input is each position's feature (ref_shim.cpp refx_project_token_stats)."""
    lib = _ref_lib()
    W = _c64(w_pol)
    V, H = W.shape
    f = _c64(feature).reshape(-1, H)
    rows = f.shape[0]
    b = None if b_pol is None else _c64(b_pol).reshape(-1)
    tk = np.ascontiguousarray(tokens, dtype=np.int32).reshape(-1)
    logits, lp, ent = np.zeros((rows, V)), np.zeros(rows), np.zeros(rows)
    st = lib.refx_project_token_stats(C.c_longlong(rows), H, V, _p(f), _p(W), _p(b), _p(tk), _p(logits),
                                      _p(lp), _p(ent))
    if st:
        raise RuntimeError(lib.refx_last_error().decode())
    return logits, lp, ent


def ref_load_checkpoint(path: str):
    """The reference's load_checkpoint: (status, descriptor 7-tuple, params)."""
    lib = _ref_lib()
    desc = (C.c_int * 7)()
    cnt = C.c_longlong(0)
    st = lib.refx_load_checkpoint(path.encode(), desc, None, 0, C.byref(cnt))
    if st:
        return st, None, None
    p = np.zeros(cnt.value)
    st = lib.refx_load_checkpoint(path.encode(), desc, _p(p), cnt, C.byref(cnt))
    return st, tuple(desc), p


class RefScenario:
    """A rollout produced by the reference's own StageSim/StageGen with a PolicyNet of
    arbitrary (vocab, M); exports everything in the SoA layout."""

    def __init__(self, **kw):
        cfg = dict(REF_DEFAULTS)
        cfg.update(kw)
        self.cfg = cfg
        self.lib = _ref_lib()
        st = C.c_int(0)
        self.h = self.lib.refx_create(C.byref(RefCfg(**cfg)), C.byref(st))
        if not self.h:
            raise RuntimeError(f"refx_create failed ({st.value}): {self.lib.refx_last_error().decode()}")
        dims = (C.c_longlong * 7)()
        self.lib.refx_dims(C.c_void_p(self.h), dims)
        self.E, self.Tc, self.C, self.M, self.V, self.n_ep, self.n_params = [int(x) for x in dims]

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.refx_destroy(C.c_void_p(self.h))
            self.h = None

    def export(self, with_logits: bool = True) -> dict:
        E, Tc, Cn, M, V = self.E, self.Tc, self.C, self.M, self.V
        d = dict(tokens=np.zeros((E, Tc, Cn, M), np.int32), old_logprob=np.zeros((E, Tc, Cn, M)),
                 reward=np.zeros((E, Tc, Cn)), flags=np.zeros((E, Tc, Cn), np.uint8),
                 episode_id=np.zeros((E, Tc, Cn), np.int32), value_scalar=np.zeros((E, Tc)),
                 value_vector=np.zeros((E, Tc, Cn)), boot_scalar=np.zeros((E, Tc, Cn)),
                 boot_vector0=np.zeros((E, Tc, Cn)), logits=np.zeros((E, Tc, Cn, M, V)),
                 new_value_scalar=np.zeros((E, Tc)), new_value_vector=np.zeros((E, Tc, Cn)),
                 lp_cur=np.zeros((E, Tc, Cn, M)), ent_cur=np.zeros((E, Tc, Cn, M)))
        st = self.lib.refx_export(C.c_void_p(self.h), *[_p(d[k]) for k in (
            "tokens", "old_logprob", "reward", "flags", "episode_id", "value_scalar",
            "value_vector", "boot_scalar", "boot_vector0", "logits", "new_value_scalar",
            "new_value_vector", "lp_cur", "ent_cur")])
        if st:
            raise RuntimeError(self.lib.refx_last_error().decode())
        n = self.n_ep
        ep = dict(ep_env_id=np.zeros(n, np.int32), ep_episode_id=np.zeros(n, np.int32),
                  ep_start=np.zeros(n, np.int64), ep_length=np.zeros(n, np.int64),
                  ep_total_reward=np.zeros(n), ep_first_success=np.zeros(n, np.int64),
                  ep_success=np.zeros(n, np.uint8), ep_complete=np.zeros(n, np.uint8),
                  ep_task=np.zeros(n, np.int32), ep_reset_id=np.zeros(n, np.int32))
        self.lib.refx_export_episodes(C.c_void_p(self.h), *[_p(ep[k]) for k in (
            "ep_env_id", "ep_episode_id", "ep_start", "ep_length", "ep_total_reward",
            "ep_first_success", "ep_success", "ep_complete", "ep_task", "ep_reset_id")])
        d.update(ep)
        d["V"] = V
        if not with_logits:
            d.pop("logits")
        return d

    def params(self):
        """(snapshot params f64, reset ids int32 or None) of the rollout."""
        p = np.zeros(self.n_params)
        ids = np.zeros(self.E, np.int32)
        has = self.lib.refx_export_params(C.c_void_p(self.h), _p(p), _p(ids))
        return p, (ids if has else None)

    def ppo(self, spec, gamma=0.99, lam=0.95, normalize=True, clip=0.2, vcoef=0.5, ecoef=0.01,
            want_grad=False):
        a, l, v = spec
        E, Tc, Cn = self.E, self.Tc, self.C
        shape = (E, Tc) if a == CHUNK else (E, Tc, Cn)
        out = dict(counted=np.zeros((E, Tc, Cn), np.uint8), adv_raw=np.zeros(shape),
                   ret=np.zeros(shape), adv_norm=np.zeros(shape), diag=np.zeros(7))
        grad = np.zeros(self.n_params) if want_grad else None
        st = self.lib.refx_ppo(C.c_void_p(self.h), a, l, v, C.c_double(gamma), C.c_double(lam),
                               int(normalize), C.c_double(clip), C.c_double(vcoef),
                               C.c_double(ecoef), _p(out["counted"]), _p(out["adv_raw"]),
                               _p(out["ret"]), _p(out["adv_norm"]), _p(out["diag"]), _p(grad))
        out["status"] = st
        out["grad"] = grad
        return out

    def ppo_subset(self, spec, idx, gamma=0.99, lam=0.95, normalize=True, clip=0.2, vcoef=0.5,
                   ecoef=0.01):
        """ppo_loss over record_indices `idx` (record = env * Tc + chunk)."""
        ix = np.ascontiguousarray(idx, np.int64)
        diag = np.zeros(7)
        st = self.lib.refx_ppo_subset(C.c_void_p(self.h), spec[0], spec[1], spec[2], C.c_double(gamma),
                                      C.c_double(lam), int(normalize), C.c_double(clip),
                                      C.c_double(vcoef), C.c_double(ecoef), C.c_longlong(ix.size),
                                      _p(ix), _p(diag))
        return st, diag

    def grpo_subset(self, spec, idx, eps_std=1e-8, apply_filter=True, lower=0.0, upper=1.0,
                    length_normalized=True, min_group_size=2, clip=0.2):
        ix = np.ascontiguousarray(idx, np.int64)
        diag = np.zeros(7)
        st = self.lib.refx_grpo_subset(C.c_void_p(self.h), spec[0], spec[1], spec[2],
                                       C.c_double(eps_std), int(apply_filter), C.c_double(lower),
                                       C.c_double(upper), int(length_normalized), min_group_size,
                                       C.c_double(clip), C.c_longlong(ix.size), _p(ix), _p(diag))
        return st, diag

    def dump_slab(self) -> str:
        """The reference's own dump_slab text (core/types.cpp:9-28) of this rollout."""
        n = C.c_size_t(0)
        self.lib.refx_dump_slab(C.c_void_p(self.h), None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value)
        self.lib.refx_dump_slab(C.c_void_p(self.h), buf, n.value, C.byref(n))
        return buf.raw[:n.value].decode()

    def save_checkpoint(self, path: str) -> None:
        if self.lib.refx_save_checkpoint(C.c_void_p(self.h), path.encode()):
            raise RuntimeError(self.lib.refx_last_error().decode())

    def bpol_offset(self) -> int:
        return int(self.lib.refx_bpol_offset(C.c_void_p(self.h)))

    def replay_ppo_grad(self, val_level, counted, coeff_lp, coeff_ent, coeff_val):
        g = np.zeros(self.n_params)
        st = self.lib.refx_replay_ppo_grad(
            C.c_void_p(self.h), val_level, _p(np.ascontiguousarray(counted, np.uint8)),
            _p(_c64(coeff_lp)), _p(_c64(coeff_ent)), _p(_c64(coeff_val)), _p(g))
        if st:
            raise RuntimeError(self.lib.refx_last_error().decode())
        return g

    def grpo(self, spec, eps_std=1e-8, apply_filter=True, lower=0.0, upper=1.0,
             length_normalized=True, min_group_size=2, clip=0.2, want_grad=False):
        a, l, v = spec
        E, Tc, Cn = self.E, self.Tc, self.C
        gt, gr = C.c_int(0), C.c_int(0)
        out = dict(env_group=np.zeros(E, np.int32), env_member=np.zeros(E, np.int32),
                   env_episode=np.zeros(E, np.int32), env_adv=np.zeros(E),
                   env_group_size=np.zeros(E, np.int32), slot_weight=np.zeros((E, Tc, Cn)),
                   slot_member=np.zeros((E, Tc, Cn), np.uint8), diag=np.zeros(7))
        grad = np.zeros(self.n_params) if want_grad else None
        st = self.lib.refx_grpo(
            C.c_void_p(self.h), a, l, v, C.c_double(eps_std), int(apply_filter),
            C.c_double(lower), C.c_double(upper), int(length_normalized), min_group_size,
            C.c_double(clip), C.byref(gt), C.byref(gr), *[_p(out[k]) for k in (
                "env_group", "env_member", "env_episode", "env_adv", "env_group_size",
                "slot_weight", "slot_member", "diag")], _p(grad))
        out.update(status=st, groups_total=gt.value, groups_retained=gr.value, grad=grad)
        return out

    def replay_grpo_grad(self, spec, coeff_lp, eps_std=1e-8, apply_filter=True, lower=0.0,
                         upper=1.0, length_normalized=True, min_group_size=2):
        g = np.zeros(self.n_params)
        st = self.lib.refx_replay_grpo_grad(
            C.c_void_p(self.h), spec[0], spec[1], C.c_double(eps_std), int(apply_filter),
            C.c_double(lower), C.c_double(upper), int(length_normalized), min_group_size,
            _p(_c64(coeff_lp)), _p(g))
        if st:
            raise RuntimeError(self.lib.refx_last_error().decode())
        return g

    def bench_ppo(self, spec, threads, iters, gamma=0.99, lam=0.95, clip=0.2, vcoef=0.5,
                  ecoef=0.01):
        diag = np.zeros(7)
        s = self.lib.refx_bench_ppo(C.c_void_p(self.h), spec[0], spec[1], spec[2],
                                    C.c_double(gamma), C.c_double(lam), C.c_double(clip),
                                    C.c_double(vcoef), C.c_double(ecoef), threads, iters, 1,
                                    _p(diag))
        return s, diag

    def bench_grpo(self, spec, threads, iters, align, eps_std=1e-8, length_normalized=True,
                   clip=0.2, apply_filter=True):
        diag = np.zeros(7)
        s = self.lib.refx_bench_grpo(C.c_void_p(self.h), spec[0], spec[1], C.c_double(eps_std),
                                     int(length_normalized), C.c_double(clip), threads, iters,
                                     align, _p(diag), int(apply_filter))
        return s, diag
