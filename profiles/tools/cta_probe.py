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
        tl = (C.c_uint64 * 32)()
        _lib.check(_lib.lib().ckrl_debug_timeline(tl, 32))
        vals = tuple((int(tl[i]) - int(t[1].max())) / 1e3 for i in (28, 29, 30, 31)) + (
            (int(t[2].max()) - int(t[1].max())) / 1e3,)
        print("   last CTA (us after the latest done): ticket %.2f loaded %.2f written %.2f finalised %.2f; exit max %.2f" % vals)

# overlapped step: where and when the assembly CTAs ran vs the loss CTAs' start
if os.environ.get("ASM_PROBE", "0") == "1" and hasattr(_lib.lib(), "ckrl_debug_asm_times"):
    asm = (C.c_uint64 * (3 * 1184))()
    smid = (C.c_uint32 * 1184)()
    g = torch.cuda.CUDAGraph()  # replayed like bench.py (no host submission gaps)
    s_ = torch.cuda.Stream()
    s_.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_):
        st(ro, pol)
    torch.cuda.current_stream().wait_stream(s_)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        st(ro, pol)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    _lib.check(_lib.lib().ckrl_debug_asm_times(asm, 3 * 1184, smid))
    _lib.check(_lib.lib().ckrl_debug_cta_times(buf, 3 * 1184))
    A = np.array(asm, dtype=np.int64).reshape(3, 1184)
    T = np.array(buf, dtype=np.int64).reshape(3, 1184)[:, :148]
    nA = int((A[0] > 0).sum())
    a0 = A[0][:nA].min()
    dn = (T[1] - a0) / 1e3
    ex = (T[2] - a0) / 1e3
    print(f"loss done max {dn.max():.1f} exit max {ex.max():.1f} us (rel. first assembly start)")
    print(f"assembly: {nA} CTAs, start [{(A[0][:nA]-a0).min()/1e3:.1f}..{(A[0][:nA]-a0).max()/1e3:.1f}] end [{(A[1][:nA]-a0).min()/1e3:.1f}..{(A[1][:nA]-a0).max()/1e3:.1f}] us")
    ls = (T[0] - a0) / 1e3
    asm_sms = set(A[2][:nA].tolist())
    on = np.array([int(smid[i]) in asm_sms for i in range(148)])
    print("(graph replay)")
    print(f"loss CTA start (rel. first assembly start): on assembly SMs p50 {np.median(ls[on]):.1f} max {ls[on].max():.1f} (n={on.sum()}); others p50 {np.median(ls[~on]) if (~on).any() else -1:.1f} max {ls[~on].max() if (~on).any() else -1:.1f}")
