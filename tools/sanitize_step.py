"""Small PowerSGD steps for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family of libpsgd_b200.so on shapes that reach it, W = 1 and a
simulated W = 2, eager launches.  Usage: sanitize_step.py <case>"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_13727_b200 import ParamSpec, PowerSGDEngine, catalogs  # noqa: E402

CASES = {
    # K1 ef_p (chunks, multi-warp rows, bias), k2_gs warp + CTA items, k3_pipe (TMA + direct slabs)
    "resnet18": (list(catalogs.get_catalog("resnet18").params), 2),
    # tall: k2_gram / k2_apply, k3_slab tall, k3_tile, k4_tile, k4_tile2, k45_rows
    "tall": ([ParamSpec("t650", (2600, 650)), ParamSpec("b", (96,)), ParamSpec("t512", (2048, 512)),
              ParamSpec("t30", (1500, 30)), ParamSpec("c", (700, 48))], 4),
    # K1 split rows, unstaged Q, K1 column tiles (k1_tile + k1_tile_reduce)
    "wide": ([ParamSpec("long", (16, 20000)), ParamSpec("b", (16,)), ParamSpec("wide", (64, 4099)),
              ParamSpec("tile", (1024, 4096))], 8),
}

case = sys.argv[1]
specs, rank = CASES[case]
for workers in (1, 2):
    eng = PowerSGDEngine(specs, rank, workers=workers, seed=0)
    for w in range(workers):
        eng.g[w].normal_()
        eng.bias_g[w].normal_()
    eng.attach_optimizer(0.1, 0.9)
    for _ in range(2):
        eng.step()
        eng.optimizer_step()
    torch.cuda.synchronize()
    eng.check()
print("ok", case)
