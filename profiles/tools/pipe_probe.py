"""One cfg5 rollout epoch (for ncu captures of the pipeline kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_06710_b200.pipeline import RolloutPipeline, random_params  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
env, pol = bench.cfg5_specs(bench.CFG5["num_envs"], seed=1000)
params = random_params(pol, seed=7)
pipe = RolloutPipeline(env, pol, bench.CFG5["num_chunks"], stages=k, sample_seed=77,
                       keep_logits=True)
for _ in range(2):
    pipe.launch(params)
torch.cuda.synchronize()
print("ok", int(pipe.out["episode_count"].item()))
