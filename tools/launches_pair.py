"""One warm cfg1 pair (eager, no graph) for an ncu launch list."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_09459_b200 as rg  # noqa: E402
from paper_2404_09459_b200 import device as dv  # noqa: E402
from paper_2404_09459_b200.workloads import CONFIGS, make_pair  # noqa: E402

cfg = CONFIGS[os.environ.get("CFG", "cfg1")]
dv.USE_GRAPHS = False
g1, g2 = make_pair(cfg)
pair = rg.GmpPair.resident(torch.from_numpy(g1).cuda(), torch.from_numpy(g2).cuda())
opts = rg.GsvOptions(extraction=rg.ExtractionConfig.fixed_rank(cfg.k, 0, cfg.q))
for i in range(3):
    rg.compare(pair, opts)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("pair")
rg.compare(pair, opts)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
