"""bench.py's per-shard projection alone (development aid): every rank's shard at G = 1, 2, 4, 8
timed on this one GPU."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2003_02256_b200 as masw  # noqa: E402

print(json.dumps(bench.shard_projection(masw, torch, torch.device("cuda:0")), indent=1))
