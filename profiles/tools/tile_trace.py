"""(Needs a probe build: make -C paper_2510_06710_b200/csrc EXTRA=-DCKRL_PROBES, or CKRL_LIB=<it>.)
CTA 0's per-tile trace of the headline loss launch under graph replay: for each local tile,
when its row phase started (stage full) / finished, and when its unit phase started / finished
(us from the launch's first CTA start). Shows whether the row warps or the buffer warps
(unit phases) set the pace, and how far the unit phases lag at the end."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from paper_2510_06710_b200 import _lib, optim, synth  # noqa: E402
from paper_2510_06710_b200.core import (EpisodeTable, GaeParams, GranularitySpec, GrpoAssemblyOptions,  # noqa: E402
                                        GrpoParams, Level, PolicyOutputs, PpoParams, RolloutBuffer)

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
loss_only = len(sys.argv) > 2 and sys.argv[2] == "loss"  # graph of the loss launch alone
cfg = synth.CONFIGS[name]
a, l, v = synth.SPECS[name]
d = synth.episodes_numpy(cfg)
lg, tk, old = synth.token_tensors(cfg)
d["tokens"], d["old_logprob"] = tk, old
ro = RolloutBuffer.from_arrays(d, d["boot_scalar"] if a == 0 else d["boot_vector0"], 256)
spec = GranularitySpec(Level(a), Level(l), Level(v))
if cfg.algo == "ppo":
    nv = d["new_value_scalar"] if v == 0 else d["new_value_vector"]
    pol = PolicyOutputs(lg, torch.tensor(nv, dtype=torch.float32, device="cuda"))
    outs = os.environ.get("TRACE_NO_OUTPUTS") != "1"  # A/B: the loss without coefficient stores
    st = optim.PpoStep(ro, GaeParams(), spec, PpoParams(0.2, 0.5, 0.01, True), outputs=outs)
    run = lambda: st(ro, pol)  # noqa: E731
    if loss_only:
        st(ro, pol)
        run = lambda: optim.ppo_loss(ro, pol, st.batch, PpoParams(0.2, 0.5, 0.01, True), st.outputs,  # noqa: E731
                                     diag=st.diag)
else:
    ept = EpisodeTable.from_arrays(d)
    st = optim.GrpoStep(ro, GrpoAssemblyOptions(spec), GrpoParams(0.2))
    pol = PolicyOutputs(lg)
    run = lambda: st(ro, ept, pol)  # noqa: E731
s_ = torch.cuda.Stream()
s_.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s_):
    for _ in range(3):
        run()
torch.cuda.current_stream().wait_stream(s_)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    run()
n = 3 * 1184 + 7 * 64
buf = (C.c_uint64 * n)()
for rep in range(3):
    g.replay()
    torch.cuda.synchronize()
    _lib.check(_lib.lib().ckrl_debug_cta_times(buf, n))
    A = np.array(buf, dtype=np.int64)
    T = A[:3 * 1184].reshape(3, 1184)[:, :148]
    t0 = T[0].min()
    tt = A[3 * 1184:].reshape(7, 64)
    nt = int((tt[0] > 0).sum())
    print(f"{name} rep{rep}: CTA0 start {(T[0][0] - t0) / 1e3:.2f} roles done {(T[1][0] - t0) / 1e3:.2f} "
          f"exit {(T[2][0] - t0) / 1e3:.2f}; grid exit max {(T[2].max() - t0) / 1e3:.2f} us; {nt} tiles")
    for i in range(nt):
        r0, r1, u0, u1, um, ut, us = ((tt[:, i] - t0) / 1e3)
        print(f"  tile {i:2d}: rows {r0:6.2f}-{r1:6.2f} ({r1 - r0:4.2f})  unit {u0:6.2f}-{u1:6.2f} ({u1 - u0:4.2f}:"
              f" meta {um - u0:4.2f} tok {ut - um:4.2f} slot {us - ut:4.2f} rec {u1 - us:4.2f})  lag {u1 - r1:5.2f}")
