"""Config 4 as one rank of eight sees it (1 sequence x 32768 tokens): decode
launches for an ncu launch list (development tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda", 0)
wl = bench.DecodeWorkload(4, 8, 3, dev, layers=4)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    wl.decode(i)
torch.cuda.synchronize()
print("ok")
