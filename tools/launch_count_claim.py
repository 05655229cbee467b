import sys
sys.path.insert(0, ".")
import torch
from paper_1905_13727_b200 import PowerSGDEngine, catalogs
for wl, r in (("lstm", 4), ("resnet18", 2), ("resnet18", 4)):
    e = PowerSGDEngine(list(catalogs.get_catalog(wl).params), r)
    print(wl, r, "claimed launches/step", e.plan.info.launches_step_single)
