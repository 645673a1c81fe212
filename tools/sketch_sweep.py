"""The bench's sketch sweep alone (causal 131k, bf16): tokens/s per (P, L) and the pass count.

    python tools/sketch_sweep.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

for r in bench.sketch_sweep(torch.device("cuda", 0), torch.bfloat16):
    print(json.dumps(r))
