"""cProfile of one batch-packed cryptonets_infer call (host-side cost breakdown)."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_01805_b200 as tt  # noqa: E402
from paper_2011_01805_b200 import nn  # noqa: E402

net = nn.cryptonets_network(42)
S = tt.Session(8192, 8)
batch = np.random.default_rng(1).uniform(0, 1, size=(784, 8192))
nn.cryptonets_infer(net, batch, (1, 1, 8192), S)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    nn.cryptonets_infer(net, batch, (1, 1, 8192), S)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
