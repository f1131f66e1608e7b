"""The C-ABI library loads and exports every symbol include/ckrl.h declares; host-only
helpers behave like the reference (error taxonomy); compute entry points fail loudly
instead of falling back to the CPU when no device is present."""
import ctypes as C
import os
import re

import pytest

import paper_2510_06710_b200 as ck
from paper_2510_06710_b200 import _lib, errors
from paper_2510_06710_b200.core import GranularitySpec, Level

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ckrl.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ckrl_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/ckrl.h but not exported"
    assert set(syms) == set(_lib.SIGNATURES), "ctypes binding out of sync with ckrl.h"


def test_version_and_status_strings():
    lib = ck.lib()
    assert b"sm_100a" in lib.ckrl_version()
    names = [lib.ckrl_status_string(i).decode() for i in range(0, 17)]
    assert names[1:13] == ["UnsupportedCombination", "GranularityOrderViolation", "LengthMismatch",
                           "BadResetId", "HeadMismatch", "NonFinite", "DegenerateGroup", "SkipUpdate",
                           "InvalidPlan", "MemoryOverflow", "EmptyTrace", "ConfigError"]
    for i in range(1, 13):  # exception classes mirror chunkrl/core/errors.hpp
        assert type(errors.from_status(i)).__name__ == names[i]


@pytest.mark.parametrize("adv,lp,val,ok", [
    (Level.Chunk, Level.Chunk, Level.Chunk, True), (Level.Chunk, Level.Action, Level.Chunk, True),
    (Level.Chunk, Level.Token, Level.Chunk, True), (Level.Action, Level.Action, Level.Action, True),
    (Level.Action, Level.Token, Level.Action, True),
    (Level.Action, Level.Chunk, Level.Action, False),  # the one rejected Table-1 cell
    (Level.Token, Level.Token, Level.Chunk, False), (Level.Chunk, Level.Chunk, Level.Token, False)])
def test_validate_granularity_table1(adv, lp, val, ok):
    # core/granularity.cpp:47-60, tests/test_core.cpp Table-1 cells
    if ok:
        ck.validate_granularity(GranularitySpec(adv, lp, val))
    else:
        with pytest.raises(errors.UnsupportedCombination):
            ck.validate_granularity(GranularitySpec(adv, lp, val))


def test_level_names():
    assert Level.from_name("chunk_level") == Level.Chunk and Level.from_name("token") == Level.Token
    with pytest.raises(errors.ConfigError):
        Level.from_name("episode_level")


def test_workspace_query_is_host_only_and_monotone():
    lib = ck.lib()
    a = lib.ckrl_workspace_bytes(256, 10, 8, 7, 1)
    b = lib.ckrl_workspace_bytes(4096, 10, 8, 7, 8)
    assert 0 < a <= b
    assert lib.ckrl_stats_record_bytes() == 64


def test_merge_stats_host_matches_numpy():
    import numpy as np
    from paper_2510_06710_b200.dist import StatsRecord, merge_stats
    rng = np.random.default_rng(1)
    parts = [rng.standard_normal(n) * 2 + 0.3 for n in (5, 11, 1, 7)]
    recs = [StatsRecord.from_units(p, n_val=len(p), n_pos=7 * len(p)) for p in parts]
    got = merge_stats(recs)
    allv = np.concatenate(parts)
    assert got["n_adv"] == len(allv) and got["n_pos"] == 7 * len(allv)
    assert abs(got["mean"] - allv.mean()) < 1e-12
    assert abs(got["denom"] - (allv.std() + 1e-8)) < 1e-12


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU behaviour")
def test_compute_entry_points_fail_loudly_without_device():
    lib = ck.lib()
    st = lib.ckrl_compute_gae(1, None, None, None, None, None, C.byref(_lib.GaeParams(0.9, 0.9)),
                              None, None, None)
    assert st == 14  # CKRL_ERR_CUDA: no CPU fallback
    assert b"no CPU fallback" in lib.ckrl_last_error()


def test_placement_mode_known_answers():
    """placement::derive_mode / validate_plan (placement/plan.cpp:49-68), the reference's own
    cases (tests/test_placement.cpp:71-74) plus validation errors."""
    from paper_2510_06710_b200 import errors
    from paper_2510_06710_b200.pipeline import COLOCATED, DISAGGREGATED, HYBRID, derive_mode
    assert derive_mode(8, "0-7", "0-7", "0-7") == COLOCATED
    assert derive_mode(8, "0-1", "2-3", "4-7") == DISAGGREGATED
    assert derive_mode(8, "0-3", "4-7", "0-7") == HYBRID
    assert derive_mode(1, "0", "0", "0") == COLOCATED
    with pytest.raises(errors.InvalidPlan):
        derive_mode(8, "0-8", "0-7", "0-7")
    with pytest.raises(errors.InvalidPlan):
        derive_mode(8, "3-2", "0-7", "0-7")
    with pytest.raises(errors.InvalidPlan):
        derive_mode(0, "0", "0", "0")
    with pytest.raises(errors.InvalidPlan):
        derive_mode(8, "0-7", "0-7", "0-7", pipeline_stage_num=0)
