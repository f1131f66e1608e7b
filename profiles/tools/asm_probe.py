"""Times PPO assembly alone and the full PPO step (CUDA events, warm, 500 iterations) for
cfg1 / cfg3; A/B the assembly schedule with CKRL_STAGED_GAE=0/1."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2510_06710_b200 import optim, synth, advantage
from paper_2510_06710_b200.core import *

for name in sys.argv[1:] or ["cfg3", "cfg1"]:
    cfg = synth.CONFIGS[name]; a, l, v = synth.SPECS[name]
    d = synth.episodes_numpy(cfg); lg, tk, old = synth.token_tensors(cfg)
    d['tokens'], d['old_logprob'] = tk, old
    ro = RolloutBuffer.from_arrays(d, d['boot_scalar'] if a == 0 else d['boot_vector0'], 256)
    nv = torch.tensor(d['new_value_scalar'] if v == 0 else d['new_value_vector'], dtype=torch.float32, device='cuda')
    spec = GranularitySpec(Level(a), Level(l), Level(v))
    opts = PpoAssemblyOptions(GaeParams(), spec)
    st = optim.PpoStep(ro, GaeParams(), spec, PpoParams(0.2, 0.5, 0.01, True))
    pol = PolicyOutputs(lg, nv)
    out = advantage.assemble_ppo_batch(ro, opts)
    def t(fn, n=500):
        for _ in range(20): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(n): fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / n
    ta = t(lambda: advantage.assemble_ppo_batch(ro, opts, out=out))
    ts = t(lambda: st(ro, pol))
    print(f"{name} staged={os.environ.get('CKRL_STAGED_GAE', '1')} assemble_us={ta:.2f} step_us={ts:.2f}")
