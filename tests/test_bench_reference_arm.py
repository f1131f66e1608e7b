"""bench.py's reference arm (the reference's own CPU implementation, oracle/_ref, env-sharded
over the host threads) runs without a GPU: check its JSON line for a PPO and a GRPO config
(the GRPO shard re-indexing once crashed it)."""
import json
import os
import subprocess
import sys

import pytest

from oracle.bindings import ref_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_reference_arm_json_line(cfg):
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", cfg, "--steps", "1",
                          "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    j = json.loads(out.stdout.strip().splitlines()[-1])
    assert j["impl"] == "reference" and j["value"] > 0 and j["unit"] == "env-steps/s"
    assert j["cpu_baseline"]["kind"] == "reference" and j["cpu_baseline"]["value"] == j["value"]
    assert j["e2e"] == {"value": j["value"], "unit": j["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
