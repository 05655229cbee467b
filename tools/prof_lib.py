"""ncu driver: eager steps with a chosen library build (argv[1]); no L2 flush between steps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_13727_b200 import PowerSGDEngine, _lib, catalogs  # noqa: E402

_lib._lib = _lib.load(sys.argv[1])
wl = os.environ.get("WL", "resnet18")
rank = int(os.environ.get("RANK_R", "2"))
specs = list(catalogs.get_catalog(wl).params)
eng = PowerSGDEngine(specs, rank, seed=0)
eng.g[0].normal_()
eng.bias_g[0].normal_()
for _ in range(3):
    eng.run()
torch.cuda.synchronize()
