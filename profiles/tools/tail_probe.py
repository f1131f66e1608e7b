"""(Needs a probe build: `make -C paper_2510_06710_b200/csrc EXTRA=-DCKRL_PROBES`, or CKRL_LIB=<such a build>.)
Tail of the headline loss launch under graph replay: per-CTA start / roles-done / exit stamps
(ckrl_debug_cta_times) and the last CTA's reduction marks (timeline slots 28-31)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from paper_2510_06710_b200 import _lib, optim, synth  # noqa: E402
from paper_2510_06710_b200.core import (GaeParams, GranularitySpec, Level, PolicyOutputs,  # noqa: E402
                                        PpoParams, RolloutBuffer)

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = synth.CONFIGS[name]
a, l, v = synth.SPECS[name]
d = synth.episodes_numpy(cfg)
lg, tk, old = synth.token_tensors(cfg)
d["tokens"], d["old_logprob"] = tk, old
ro = RolloutBuffer.from_arrays(d, d["boot_scalar"] if a == 0 else d["boot_vector0"], 256)
nv = d["new_value_scalar"] if v == 0 else d["new_value_vector"]
pol = PolicyOutputs(lg, torch.tensor(nv, dtype=torch.float32, device="cuda"))
st = optim.PpoStep(ro, GaeParams(), GranularitySpec(Level(a), Level(l), Level(v)), PpoParams(0.2, 0.5, 0.01, True))
s_ = torch.cuda.Stream()
s_.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s_):
    for _ in range(3):
        st(ro, pol)
torch.cuda.current_stream().wait_stream(s_)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    st(ro, pol)
buf = (C.c_uint64 * (3 * 1184))()
tl = (C.c_uint64 * 32)()
for rep in range(4):
    g.replay()
    torch.cuda.synchronize()
    _lib.check(_lib.lib().ckrl_debug_cta_times(buf, 3 * 1184))
    _lib.check(_lib.lib().ckrl_debug_timeline(tl, 32))
    T = np.array(buf, dtype=np.int64).reshape(3, 1184)[:, :148]
    t0 = T[0].min()
    st_, dn, ex = (T[0] - t0) / 1e3, (T[1] - t0) / 1e3, (T[2] - t0) / 1e3
    last = [(tl[i] - t0) / 1e3 for i in range(28, 32)]
    print(f"{name} rep{rep}: start p50 {np.median(st_):.1f} max {st_.max():.1f} | roles done p50 "
          f"{np.median(dn):.1f} max {dn.max():.1f} | exit p50 {np.median(ex):.1f} max {ex.max():.1f} | "
          f"last CTA ticket {last[0]:.1f} loaded {last[1]:.1f} synced {last[2]:.1f} final {last[3]:.1f} us")
# start / roles-done by CTA index (does the late-start set sit at the top of the grid?)
T = np.array(buf, dtype=np.int64).reshape(3, 1184)[:, :148]
t0 = T[0].min()
order = np.argsort(T[0])
print("CTA ids by start time (first 10 / last 40):", order[:10].tolist(), order[-40:].tolist())
print("start us by id block of 16:", [round(float(np.mean((T[0][i:i + 16] - t0) / 1e3)), 1) for i in range(0, 148, 16)])
