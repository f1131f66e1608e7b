"""Row f3: the wire / on-disk formats (host entry points of the C ABI; no device needed).

* dump_slab: the SoA slab of a reference rollout, formatted by ckrl_dump_slab, is the
  reference's own dump_slab text (core/types.cpp:9-28) byte-for-byte, in every rollout mode;
* CKRL checkpoint: files written by ckrl_save_checkpoint are byte-identical to the
  reference's save_checkpoint of the same parameters and load back through the reference's
  load_checkpoint, and the reference's files load through ckrl_load_checkpoint; the
  reference's error cases (magic, version, count, truncation) are errors here too.
The committed fixture tests/golden/dump_toyreach.npz pins the dump where /root/reference is
absent (the GPU box); tests/test_gpu_pipeline.py dumps a CUDA rollout against it.
"""
import os

import numpy as np
import pytest

from conftest import load_golden
from oracle.bindings import RefScenario, ref_available, ref_load_checkpoint
from paper_2510_06710_b200 import errors, formats
from paper_2510_06710_b200.pipeline import PolicyDescriptor

live = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")

MODES = {
    "partial": dict(auto_reset=1),
    "deferred": dict(auto_reset=1, deferred_reset=1, env_kind=1, success_step=2),
    "no_autoreset": dict(auto_reset=0, num_chunks=6),
    "v256_m7": dict(vocab=256, tokens_per_action=7, num_envs=3, chunk_length=4, num_chunks=3),
}


@live
@pytest.mark.parametrize("mode", sorted(MODES))
def test_dump_slab_matches_reference(mode):
    sc = RefScenario(**{**dict(num_envs=5, max_episode_steps=5, reward_shaping=1), **MODES[mode]})
    d = sc.export(with_logits=False)
    text = formats.dump_slab(d["tokens"], d["reward"], d["flags"], d["episode_id"])
    assert text == sc.dump_slab()
    assert formats.dump_slab(d["tokens"].astype(np.uint8), d["reward"], d["flags"], d["episode_id"]) == text


def test_dump_slab_golden_fixture():
    g = load_golden("dump_toyreach.npz")
    text = formats.dump_slab(g["tokens"], g["reward"], g["flags"], g["episode_id"])
    assert text == bytes(g["text"]).decode()


def test_dump_slab_partition_keeps_global_env_ids():
    """A VecEnv partition / rank shard whose first global env is 3 (vec_env.cpp:94): uids
    carry the global env id in their high word, the env column stays the slab row."""
    g = load_golden("dump_toyreach.npz")
    want = []
    for line in bytes(g["text"]).decode().splitlines(keepends=True):
        f = line.split(" ")
        if not line.startswith("#") and int(f[1]) >= 0:
            f[1] = str(int(f[1]) + (3 << 32))
        want.append(" ".join(f))
    text = formats.dump_slab(g["tokens"], g["reward"], g["flags"], g["episode_id"], first_env_id=3)
    assert text == "".join(want)


def _desc_of(sc):
    cfg = sc.cfg
    return PolicyDescriptor(obs_dim=6 if cfg["env_kind"] == 0 else 2, hidden=cfg["hidden"],
                            trunk_layers=cfg["trunk_layers"], value_hidden=cfg["value_hidden"],
                            vocab=cfg["vocab"], chunk_len=cfg["chunk_length"],
                            tokens_per_action=cfg["tokens_per_action"])


@live
def test_checkpoint_roundtrip_with_reference(tmp_path):
    sc = RefScenario(hidden=9, trunk_layers=2, vocab=7)
    p, _ = sc.params()
    ref_file, our_file = str(tmp_path / "ref.ckrl"), str(tmp_path / "ours.ckrl")
    sc.save_checkpoint(ref_file)
    desc = _desc_of(sc)
    formats.save_checkpoint(desc, p, our_file)
    assert open(ref_file, "rb").read() == open(our_file, "rb").read()
    d2, p2 = formats.load_checkpoint(ref_file)
    assert d2 == desc
    np.testing.assert_array_equal(p2, p)
    st, rdesc, rp = ref_load_checkpoint(our_file)
    assert st == 0 and rdesc == (desc.obs_dim, desc.hidden, desc.trunk_layers, desc.value_hidden,
                                 desc.vocab, desc.chunk_len, desc.tokens_per_action)
    np.testing.assert_array_equal(rp, p)


def test_checkpoint_errors(tmp_path):
    desc = PolicyDescriptor(obs_dim=6, hidden=4, trunk_layers=1, value_hidden=3, vocab=5,
                            chunk_len=2, tokens_per_action=2)
    p = np.arange(desc.num_params(), dtype=np.float64) * 0.5
    f = str(tmp_path / "a.ckrl")
    formats.save_checkpoint(desc, p, f)
    d2, p2 = formats.load_checkpoint(f)
    assert d2 == desc and np.array_equal(p2, p)
    raw = open(f, "rb").read()
    cases = {"magic": b"XKRL" + raw[4:], "version": raw[:4] + b"\x02" + raw[5:],
             "truncated": raw[:-5], "count": raw[:36] + (7).to_bytes(8, "little") + raw[44:]}
    for name, blob in cases.items():
        g = str(tmp_path / f"{name}.ckrl")
        open(g, "wb").write(blob)
        with pytest.raises(errors.Error):
            formats.load_checkpoint(g)
        if ref_available():
            assert ref_load_checkpoint(g)[0] != 0, name
    with pytest.raises(errors.Error):
        formats.load_checkpoint(str(tmp_path / "missing.ckrl"))
