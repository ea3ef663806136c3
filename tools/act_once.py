"""One act2pc layer exchange (bench.py's act2pc_layer workload) for ncu launch lists (development tool)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

print(bench.act2pc_layer(int(sys.argv[1]) if len(sys.argv) > 1 else 2, 2))
torch.cuda.synchronize()
