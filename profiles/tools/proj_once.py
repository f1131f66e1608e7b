"""One tcgen05 projection launch at the cfg3 token count (for ncu): python proj_once.py H [rows]."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/profiles/", 1)[0])
from paper_2510_06710_b200 import policy  # noqa: E402

H = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 256 * 80 * 7
g = torch.Generator(device="cuda").manual_seed(1)
f = torch.randn(rows, H, device="cuda", generator=g).to(torch.bfloat16)
W = (torch.randn(256, H, device="cuda", generator=g) / H ** 0.5).to(torch.bfloat16)
tok = torch.randint(0, 256, (rows,), device="cuda", generator=g, dtype=torch.int32)
out = torch.empty(rows, 2, dtype=torch.float64, device="cuda")
for _ in range(3):
    policy.project_token_stats(f, W, None, tok, rows_out=out)
torch.cuda.synchronize()
