"""Per-CTA timing of the fused loss launch (%globaltimer): start skew, roles-done and exit
distribution across the 148 persistent CTAs, for the standalone loss (assembly done) and the
overlapped step. usage: cta_probe.py cfg3 [cfg4 ...]"""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2510_06710_b200 import _lib, advantage, optim, synth
from paper_2510_06710_b200.core import *

for name in sys.argv[1:] or ["cfg3"]:
    cfg = synth.CONFIGS[name]; a, l, v = synth.SPECS[name]
    d = synth.episodes_numpy(cfg); lg, tk, old = synth.token_tensors(cfg)
    d['tokens'], d['old_logprob'] = tk, old
    ro = RolloutBuffer.from_arrays(d, d['boot_scalar'] if a == 0 else d['boot_vector0'], 256)
    nv = torch.tensor(d['new_value_scalar'] if v == 0 else d['new_value_vector'], dtype=torch.float32, device='cuda')
    pol = PolicyOutputs(lg, nv)
    spec = GranularitySpec(Level(a), Level(l), Level(v))
    st = optim.PpoStep(ro, GaeParams(), spec, PpoParams(0.2, 0.5, 0.01, True))
    buf = (C.c_uint64 * (3 * 1184))()
    for mode in ("standalone", "step"):
        for _ in range(5):
            if mode == "step":
                st(ro, pol)
            else:
                advantage.assemble_ppo_batch(ro, PpoAssemblyOptions(GaeParams(), spec), out=st.batch)
                torch.cuda.synchronize()
                optim.ppo_loss(ro, pol, st.batch, PpoParams(0.2, 0.5, 0.01, True), st.outputs, diag=st.diag)
        torch.cuda.synchronize()
        _lib.check(_lib.lib().ckrl_debug_cta_times(buf, 3 * 1184))
        t = np.array(buf, dtype=np.int64).reshape(3, 1184)[:, :148]
        t0 = t[0].min()
        s, dn, ex = (t[0] - t0) / 1e3, (t[1] - t0) / 1e3, (t[2] - t0) / 1e3
        q = lambda x: "min %.1f p50 %.1f p90 %.1f max %.1f" % (x.min(), np.median(x), np.percentile(x, 90), x.max())
        print(f"{name} {mode}: start [{q(s)}] done [{q(dn)}] exit [{q(ex)}] us")
        print("   slowest CTAs:", np.argsort(-dn)[:8].tolist(), "done-start spread", q(dn - s))
