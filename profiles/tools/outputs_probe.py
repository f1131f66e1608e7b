"""A/B: the PPO step with and without materialised per-position outputs (token lp / entropy
and lp / entropy / value coefficients), CUDA-graph timed, to see what the unit phase's global
stores cost under the logits stream."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2510_06710_b200 import optim, synth
from paper_2510_06710_b200.core import *

for name in sys.argv[1:] or ["cfg3"]:
    cfg = synth.CONFIGS[name]; a, l, v = synth.SPECS[name]
    reps = []
    for r in range(3):
        c = synth.SynthConfig(**{**cfg.__dict__, "seed": cfg.seed + 101 * r})
        d = synth.episodes_numpy(c); lg, tk, old = synth.token_tensors(c)
        d['tokens'], d['old_logprob'] = tk, old
        ro = RolloutBuffer.from_arrays(d, d['boot_scalar'] if a == 0 else d['boot_vector0'], 256)
        nv = torch.tensor(d['new_value_scalar'] if v == 0 else d['new_value_vector'], dtype=torch.float32, device='cuda')
        reps.append((ro, PolicyOutputs(lg, nv)))
    for outputs in (True, False):
        st = optim.PpoStep(reps[0][0], GaeParams(), GranularitySpec(Level(a), Level(l), Level(v)),
                           PpoParams(0.2, 0.5, 0.01, True), outputs=outputs)
        for i in range(5): st(*reps[i % 3])
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(3): st(*reps[i])
        for _ in range(3): g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(50): g.replay()
        e1.record(); torch.cuda.synchronize()
        print(f"{name} outputs={outputs} step_us={e0.elapsed_time(e1) * 1e3 / 150:.2f}")
