"""Rollout epoch time vs env count (one CTA per env in gen_kernel): does per-position latency
depend on how many CTAs share an SM? python gen_scale.py [sampler]"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/profiles/", 1)[0])
import bench  # noqa: E402
from paper_2510_06710_b200.pipeline import RolloutPipeline, random_params  # noqa: E402

sampler = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for E in (32, 64, 128, 148, 256, 296, 444, 592):
    env, pol = bench.cfg5_specs(E, seed=3)
    params = random_params(pol, seed=7, device="cuda")
    pipe = RolloutPipeline(env, pol, bench.CFG5["num_chunks"], stages=1, sampler=sampler, keep_logits=False)
    for _ in range(2):
        pipe.launch(params)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        pipe.launch(params)
    e1.record()
    torch.cuda.synchronize()
    print(f"E={E} epoch {e0.elapsed_time(e1) / 3:.3f} ms")
