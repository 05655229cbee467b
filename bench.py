#!/usr/bin/env python
"""bench.py — PowerSGD compress + all-reduce + decompress, ms/step (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--workload resnet18|lstm|stress]

N = 1: one B200, W = 1 (BASELINE.json configs[1], ResNet-18 rank 2: the
compress / orthogonalise / decompress kernels, no collective).  N > 1 (under
torchrun): one process per GPU = one data-parallel worker, NCCL all-reduces of
the packed P and q buffers (configs[2]); per-GPU work is fixed ("weak").

A step is one PowerSGD round over every parameter of the catalog with error
feedback: delta = g + e, P = delta Q, [AR1], P-hat = MGS(P), q = delta^T P-hat,
e = delta - P-hat q^T, [AR2], M-hat = P-hat Q-bar^T (optimizer.py:110-129).
Inputs are resident in HBM; L2 is flushed (256 MiB write) before every timed
step; each step is timed with CUDA events on the launching stream and the
result is the max over ranks.  `e2e` repeats the step through the same API
with the gradients copied in from pinned host memory and M-hat + bias mean
copied back, inside the timed region.

`--impl reference` times the reference algorithm on the host CPU (the float64
numpy oracle in oracle/powersgd.py, the reference being pure Python), W = N
simulated workers, rank 0 only.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PowerSGD compress+allreduce+decompress ms/step, ResNet-18 rank 2, 1/2/4/8 B200"
DEFAULT_RANK = {"resnet18": 2, "lstm": 4, "stress": 8}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["resnet18", "lstm", "stress"], default="resnet18")
    ap.add_argument("--rank", type=int, default=None)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-opt", action="store_true", help="skip the step + optimizer timing")
    a = ap.parse_args()
    a.warmup = max(3, a.warmup)
    if a.rank is None:
        a.rank = DEFAULT_RANK[a.workload]
    return a


def catalog_specs(workload):
    from paper_1905_13727_b200 import catalogs
    if workload == "stress":
        return list(catalogs.stress().params)
    return list(catalogs.get_catalog(workload).params)


def sizes(specs, rank):
    N = snr = smr = nb = 0
    for s in specs:
        if s.is_bias:
            nb += s.size
            continue
        n, m = s.matrix_shape
        r = min(n, m, rank)
        N += n * m
        snr += n * r
        smr += m * r
    return N, snr, smr, nb


def use_all_host_threads():
    """The CPU arms use every host core (torchrun exports OMP_NUM_THREADS=1)."""
    n = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    try:
        from threadpoolctl import threadpool_limits
        import numpy  # noqa: F401  (load the BLAS the limit applies to)
        threadpool_limits(limits=n, user_api="blas")
    except Exception:
        pass
    return n


def workload_name(workload, rank, world):
    """config.workload: the same string for both arms (ours and --impl reference)."""
    return f"{workload} rank {rank}, W={world}"


def host_info():
    """lscpu model, numpy and BLAS versions (state the CPU the baseline ran on)."""
    import numpy as np
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        for info in threadpool_info():
            if info.get("user_api") == "blas":
                blas = f"{info.get('internal_api')} {info.get('version')}"
                break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "numpy": np.__version__, "blas": blas}


def cpu_baseline_leg(specs, rank, world, budget_s, workload):
    """The float64 oracle port timed on the host: all BLAS threads, then 1 thread."""
    use_all_host_threads()
    times = oracle_steps(specs, rank, world, 1000, budget_s, warmup=1)
    cores = cpu_threads()
    one = None
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1, user_api="blas"):
            t1 = oracle_steps(specs, rank, world, 1000, max(2.0, budget_s / 3), warmup=1)
        one = round(1e3 * statistics.median(t1), 3)
    except Exception:
        pass
    return {"value": round(1e3 * statistics.median(times), 3), "unit": "ms/step", "cores": cores,
            "kind": "port", "value_1_thread": one,
            "sample": f"{len(times)} full {workload} r={rank} W={world} steps (median), float64 numpy "
                      f"oracle of optimizer.py:110-129 on {cores} OpenBLAS threads, ~{budget_s:.0f}s",
            **host_info()}


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        for info in threadpool_info():
            if info.get("internal_api") in ("openblas", "mkl", "blis"):
                return int(info["num_threads"])
    except Exception:
        pass
    return os.cpu_count() or 1


# --------------------------------------------------------------------------- CPU reference arm
def oracle_steps(specs, rank, world, steps, budget_s, warmup=1):
    """Time the reference algorithm (float64 oracle, optimizer.py:110-129 without the
    momentum update) with `world` simulated workers; returns per-step seconds."""
    import numpy as np
    from oracle import powersgd as O
    ospecs = [O.ParamSpec(s.name, s.shape) for s in specs]
    grads = [[O.derive_rng(0, "grad", 0, w, i).standard_normal(s.shape).astype(np.float32)
              for i, s in enumerate(ospecs)] for w in range(world)]
    comp = O.PowerSGD(rank)
    comm = O.Communicator(world)
    workers = [O.WorkerState(w) for w in range(world)]
    for t in range(warmup):
        O.ef_step(workers, grads, ospecs, comp, comm, 0, t)
    times = []
    t_start = time.perf_counter()
    for t in range(steps):
        t0 = time.perf_counter()
        O.ef_step(workers, grads, ospecs, comp, comm, 0, warmup + t)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s and len(times) >= 2:
            break
    return times


def run_reference(a):
    rank_env = int(os.environ.get("RANK", "0"))
    if rank_env != 0:
        return 0
    specs = catalog_specs(a.workload)
    world = a.gpus
    use_all_host_threads()
    budget = 150.0
    times = oracle_steps(specs, a.rank, world, a.steps, budget, warmup=a.warmup)
    ms = 1e3 * statistics.mean(times)
    cores = cpu_threads()
    sample = (f"{len(times)} full steps of {a.workload} r={a.rank} with {world} simulated workers "
              f"(float64 numpy oracle of optimizer.py:110-129, OpenBLAS {cores} threads)")
    line = {
        "metric": METRIC, "value": round(ms, 4), "unit": "ms/step", "n_gpus": a.gpus,
        "steps": len(times), "warmup": a.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": workload_name(a.workload, a.rank, world),
                   "detail": f"{world} simulated workers on the host CPU", "rank": a.rank, "world": world},
        "cpu_baseline": {"value": round(ms, 4), "unit": "ms/step", "cores": cores, "kind": "port",
                         "sample": sample, **host_info()},
        "e2e": {"value": round(ms, 4), "unit": "ms/step", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# --------------------------------------------------------------------------- GPU arm
def run_ours(a):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1905_13727_b200 import DistributedCommunicator, PowerSGDEngine, _lib
    from paper_1905_13727_b200.plan import ptr, stream_ptr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        print(f"warning: --gpus {a.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    if os.environ.get("PSGD_BENCH_BACKEND") == "gloo":  # test only: ranks may share a GPU
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # PSGD_BENCH_BACKEND=gloo exercises this path with several ranks on one GPU (test only)
        backend = os.environ.get("PSGD_BENCH_BACKEND", "nccl")
        dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
    comm = DistributedCommunicator() if world > 1 else None
    specs = catalog_specs(a.workload)
    N, snr, smr, nbias = sizes(specs, a.rank)
    eng = PowerSGDEngine(specs, a.rank, comm=comm, seed=0, device=dev)
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    eng.g[0].normal_(generator=gen)
    eng.bias_g[0].normal_(generator=gen)
    # (gloo, a test-only transport, runs on the host and cannot be captured)
    use_graph = not a.no_graph and not (world > 1 and os.environ.get("PSGD_BENCH_BACKEND") == "gloo")
    if use_graph:  # at N > 1 the graph holds the two NCCL all-reduces too
        eng.capture()
    flush = None if a.no_flush else torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # ---------------- warm-up
    for _ in range(a.warmup):
        if flush is not None:
            flush.zero_()
        eng.run()
    barrier()
    eng.check()

    # ---------------- timed region: K steps, L2 flushed before each
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    for k in range(a.steps):
        if flush is not None:
            flush.zero_()
        starts[k].record(stream)
        eng.run()
        ends[k].record(stream)
    barrier()
    clk = clocks.stop()
    per = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    # back-to-back steps (no flush between them): the L2 keeps part of the previous step
    bb0, bb1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    bb0.record(stream)
    for _ in range(a.steps):
        eng.run()
    bb1.record(stream)
    barrier()
    ms_b2b = bb0.elapsed_time(bb1) / a.steps
    ms_local = statistics.mean(per)
    t = torch.tensor([ms_local, statistics.median(per), ms_b2b], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, ms_median, ms_b2b = float(t[0]), float(t[1]), float(t[2])
    eng.check()
    info = eng.plan.info
    launches_per_step = (info.launches_step_single if world == 1 else
                         info.launches_ef_p + info.launches_q_ef + info.launches_decompress)

    # ---------------- per-kernel breakdown (eager, same stream, L2 flushed)
    lib = _lib.lib()
    h = eng.plan.handle
    sp = stream_ptr(stream)
    names = ["ef_p", "q_ef"] + (["allreduce_p", "allreduce_q", "decompress"] if world > 1 else [])
    acc = {k: [] for k in names}
    nb = max(5, min(a.steps, 30))
    for _ in range(nb):
        if flush is not None:
            flush.zero_()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        eng.status.zero_()
        ev[0].record(stream)
        _lib.check(lib.psgd_ef_p(h, ptr(eng.g[0]), ptr(eng.e[0]), ptr(eng.work[0]), ptr(eng.Q), ptr(eng.P[0]),
                                 ptr(eng.bias_g[0]), ptr(eng.status), sp), "ef_p")
        ev[1].record(stream)
        if world > 1:
            comm.all_reduce_sum_(eng.P[0])
        ev[2].record(stream)
        qout = eng.Q if world == 1 else eng.qbuf[0]
        _lib.check(lib.psgd_q_ef(h, ptr(eng.work[0]), ptr(eng.P[0]), world, ptr(eng.repl), ptr(eng.Phat),
                                 ptr(qout), ptr(eng.e[0]), ptr(eng.bias_out), ptr(eng.status), sp), "q_ef")
        ev[3].record(stream)
        if world > 1:
            comm.all_reduce_sum_(eng.qbuf[0])
            ev[4].record(stream)
            _lib.check(lib.psgd_decompress(h, ptr(eng.Phat), ptr(eng.qbuf[0]), world, ptr(eng.Q),
                                           ptr(eng.work[0]), ptr(eng.status), sp), "decomp")
            ev[5].record(stream)
        torch.cuda.synchronize(dev)
        acc["ef_p"].append(ev[0].elapsed_time(ev[1]))
        acc["q_ef"].append(ev[2].elapsed_time(ev[3]))
        if world > 1:
            acc["allreduce_p"].append(ev[1].elapsed_time(ev[2]))
            acc["allreduce_q"].append(ev[3].elapsed_time(ev[4]))
            acc["decompress"].append(ev[4].elapsed_time(ev[5]))
    kern_ms = {k: statistics.mean(v) for k, v in acc.items()}
    eng.check()

    # ---------------- NCCL small-message latency (context for the latency-bound collectives)
    nccl_us = None
    if world > 1:
        x = torch.zeros(2, dtype=torch.float32, device=dev)
        for _ in range(20):
            dist.all_reduce(x)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(100):
            dist.all_reduce(x)
        e1.record(stream)
        barrier()
        nccl_us = 1e3 * e0.elapsed_time(e1) / 100

    # ---------------- the step + heavy-ball update (optimizer.py:131-134), separate vs fused
    opt = None
    if world == 1 and N * 4 < (2 << 30) and not a.no_opt:
        opt = optimizer_timing(specs, a, dev, flush, barrier, stream)

    # ---------------- configs[0]: the reference's own workload, 2 simulated workers on this GPU
    sim2 = None
    if world == 1 and a.workload == "resnet18" and not a.no_opt:
        sim2 = simulated_w2_timing(specs, a, dev, flush, barrier, stream)

    # ---------------- the per-parameter drop-in (the reference's optimizer loop calling round_trip)
    dropin = None
    if world == 1 and a.workload == "resnet18" and not a.no_opt:
        dropin = dropin_timing(specs, a, dev)

    # ---------------- e2e: host gradients in, M-hat + bias mean out, every step
    if world == 1 and N * 4 < (2 << 30):  # the public host-pipelined API (pipeline.py)
        e2e_ms, h2d, d2h = e2e_pipelined(specs, a, dev, flush, barrier, stream)
    else:
        e2e_ms, h2d, d2h = e2e_serial(eng, a, world, dev, flush, barrier, stream, dist)

    # ---------------- roofline (measured peaks)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    # dominant single kernel: K1 (delta = g + e, P = delta Q), 12 B per matrix element
    # (read g, read e, write delta) + P written + Q read + bias; timed alone on the
    # launching stream above (eager, L2 flushed before it)
    k1_bytes = 12 * N + 4 * snr + 4 * smr + 8 * nbias
    dom = "ef_p"
    dom_bytes = k1_bytes
    achieved = dom_bytes / (kern_ms[dom] * 1e-3) / 1e9
    traffic, traffic_src = None, None
    prof_file = {("resnet18", 2): os.path.join("profiles", "ncu_summary.json"),
                 ("resnet18", 1): os.path.join("profiles", "r2", "ncu_summary_r1.json"),
                 ("resnet18", 4): os.path.join("profiles", "r2", "ncu_summary_r4.json"),
                 ("stress", 8): os.path.join("profiles", "r2", "ncu_summary_stress.json"),
                 ("lstm", 4): os.path.join("profiles", "r2", "ncu_summary_lstm.json")}.get((a.workload, a.rank))
    try:  # dram bytes per launch of the same kernel from the committed ncu capture of this workload
        with open(os.path.join(ROOT, prof_file)) as f:
            prof = json.load(f)
        ks = [v["traffic_bytes"] for name, v in prof["kernels"].items()
              if name.startswith("k1_ef_p") or name.startswith("k1_tile")]  # psgd_ef_p's launches
        if ks:
            traffic = float(sum(ks))
            traffic_src = f"{prof_file} (ncu --set full, one launch of each psgd_ef_p kernel)"
    except Exception:
        pass
    b_alg = 24 * N + 20 * snr + 16 * smr
    t_hbm_us = b_alg / (hbm * 1e9) * 1e6
    # ring all-reduce bytes per GPU per step over NVLink 5 (900 GB/s per direction)
    nvl_bytes = 2 * (world - 1) / world * 4 * (snr + nbias + smr) if world > 1 else 0.0
    t_nvl_us = nvl_bytes / 900e9 * 1e6
    t_roof_us = t_hbm_us + t_nvl_us

    cpu = None
    if rank == 0 and not a.no_cpu:  # N > 1: rank 0 times the W = N simulated-worker oracle
        cpu = cpu_baseline_leg(specs, a.rank, world, a.cpu_seconds if world == 1 else a.cpu_seconds / 2,
                               a.workload)
    if world > 1:
        dist.barrier()

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(ms, 5), "unit": "ms/step", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms, 5),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic: seeded N(0,1) fp32 gradients of the catalog shapes, resident in HBM",
            "impl": "ours",
            "config": {"workload": workload_name(a.workload, a.rank, world),
                       "detail": "one worker per GPU " + ("(configs[1], no collective)" if world == 1
                                                          else "(configs[2], NCCL all-reduce of packed P and q, "
                                                               "captured in the CUDA graph)"),
                       "rank": a.rank, "world": world, "matrix_elems": N, "bias_elems": nbias,
                       "l2": "flushed (256 MiB write) before every timed step" if flush is not None else "not flushed",
                       "cuda_graph": use_graph, "median_ms": round(ms_median, 5),
                       "back_to_back_ms": round(ms_b2b, 5)},
            "roofline": {"bound": "hbm", "kernel": "k1_ef_p (psgd_ef_p)", "achieved": round(achieved, 1),
                         "peak": hbm, "unit": "GB/s", "frac": round(achieved / hbm, 4), "traffic": traffic,
                         "algorithmic_bytes": dom_bytes, "peak_source": peak_src,
                         "traffic_source": traffic_src},
            "step_roofline": {"algorithmic_bytes": b_alg, "t_hbm_us": round(t_hbm_us, 2),
                              "nvlink_bytes_per_gpu": round(nvl_bytes), "t_nvlink_us": round(t_nvl_us, 3),
                              "t_roof_us": round(t_roof_us, 2), "t_measured_us": round(ms * 1e3, 2),
                              "frac": round(t_roof_us / (ms * 1e3), 4),
                              "frac_back_to_back": round(t_roof_us / (ms_b2b * 1e3), 4)},
            "kernels_ms": {k: round(v, 5) for k, v in kern_ms.items()},
            "optimizer_step": opt,
            "dropin": dropin,
            "simulated_w2": sim2,
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_ms, 4), "unit": "ms/step", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches_per_step * a.steps,
            "clocks": clk,
        }
        if nccl_us is not None:
            line["nccl_small_allreduce_us"] = round(nccl_us, 2)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0



def simulated_w2_timing(specs, a, dev, flush, barrier, stream):
    """BASELINE configs[0]: W = 2 simulated workers on one GPU (K1 x 2, tree mean of P,
    K2/K3 x 2, tree mean of q, K5), CUDA graph, L2 flushed before every step."""
    import statistics
    import torch
    from paper_1905_13727_b200 import Communicator, PowerSGDEngine
    eng = PowerSGDEngine(specs, a.rank, workers=2, comm=Communicator(2), seed=0, device=dev)
    gen = torch.Generator(device=dev).manual_seed(1000)
    for w in range(2):
        eng.g[w].normal_(generator=gen)
        eng.bias_g[w].normal_(generator=gen)
    eng.capture()
    for _ in range(a.warmup):
        eng.run()
    barrier()
    ts = []
    for _ in range(a.steps):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.run()
        e1.record(stream)
        ts.append((e0, e1))
    barrier()
    eng.check()
    return {"ms_per_step": round(statistics.mean(x.elapsed_time(y) for x, y in ts), 5),
            "note": "configs[0]: ResNet-18 r=2, 2 simulated workers on one GPU (the CPU reference's own "
                    "workload), CUDA graph, L2 flushed"}


def dropin_timing(specs, a, dev, steps=5):
    """The compression part of one optimizer step (optimizer.py:110-129: EF add,
    round_trip per matrix parameter, EF update, bias mean — the same work the
    reference arm times) through the drop-in `PowerSGD.round_trip`, once with numpy
    arrays on the host (the reference's own calling convention: one H2D/D2H round
    trip and one sync per parameter) and once with CUDA tensors (no per-parameter
    sync; errors at `check()`)."""
    import numpy as np
    import torch
    from paper_1905_13727_b200 import Communicator, CompressionContext, PowerSGD
    out = {}
    rng = np.random.default_rng(0)
    grads = [rng.standard_normal(s.shape).astype(np.float32) for s in specs]
    for mode in ("numpy", "torch"):
        comp, comm = PowerSGD(a.rank), Communicator(1)
        if mode == "numpy":
            xs = [None] * len(specs)
            errs = {}
            g = grads
        else:
            xs = [None] * len(specs)
            errs = {}
            g = [torch.from_numpy(x).to(dev) for x in grads]
        ts = []
        for t in range(steps + 1):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            for i, sp in enumerate(specs):
                if sp.is_bias:
                    upd = g[i] if mode == "torch" else g[i].astype(np.float64)
                else:
                    n, m = sp.matrix_shape
                    e = errs.get(i)
                    gi = g[i].reshape(n, m)
                    delta = (gi + e) if e is not None else (gi.clone() if mode == "torch" else gi.astype(np.float64))
                    trip = comp.round_trip([delta], CompressionContext(0, i, t), comm)
                    errs[i] = delta - trip.locals[0]
                    upd = trip.aggregated.reshape(sp.shape)
                xs[i] = upd  # the aggregated update the optimizer would apply (optimizer.py:130)
            if mode == "torch":
                comp.check()
            torch.cuda.synchronize(dev)
            if t > 0:
                ts.append(time.perf_counter() - t0)
        out[mode + "_ms"] = round(1e3 * statistics.median(ts), 3)
    out["note"] = ("optimizer.py:110-129 loop over the catalog calling PowerSGD.round_trip per matrix, "
                   "as the reference arm (numpy: float64 host arrays; torch: CUDA tensors); wall clock")
    return out


def optimizer_timing(specs, a, dev, flush, barrier, stream):
    """Compression step + heavy-ball update per step (CUDA graph, L2 flushed), with the
    update as the separate one-pass kernel vs fused into K3's M-hat epilogue."""
    import statistics
    import torch
    from paper_1905_13727_b200 import PowerSGDEngine
    out = {}
    for name, fused, keep in (("separate_ms", False, True), ("fused_ms", True, True),
                              ("fused_no_mhat_ms", True, False)):
        eng = PowerSGDEngine(specs, a.rank, seed=0, device=dev)
        gen = torch.Generator(device=dev).manual_seed(1000)
        eng.g[0].normal_(generator=gen)
        eng.bias_g[0].normal_(generator=gen)
        eng.attach_optimizer(0.01, 0.9, fused=fused, keep_update=keep)
        if fused:
            out["fused_in_kernel"] = eng.fused_in_kernel
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                eng._enqueue(s)
                eng.optimizer_step(s)
        stream.wait_stream(s)
        for _ in range(a.warmup):
            flush.zero_() if flush is not None else None
            g.replay()
        barrier()
        ts = []
        for _ in range(a.steps):
            if flush is not None:
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g.replay()
            e1.record(stream)
            ts.append((e0, e1))
        barrier()
        eng.check()
        out[name] = round(statistics.mean(x.elapsed_time(y) for x, y in ts), 5)
        del g, eng
    return out


def e2e_serial(eng, a, world, dev, flush, barrier, stream, dist):
    """host gradients in (pinned), step, M-hat + bias mean out, on one stream"""
    import statistics
    import torch
    g_host = torch.empty(eng.g[0].numel(), dtype=torch.float32, pin_memory=True)
    g_host.copy_(eng.g[0].cpu())
    b_host = torch.empty(eng.bias_g[0].numel(), dtype=torch.float32, pin_memory=True)
    b_host.copy_(eng.bias_g[0].cpu())
    m_host = torch.empty(eng.work[0].numel(), dtype=torch.float32, pin_memory=True)
    bo_host = torch.empty(eng.bias_out.numel(), dtype=torch.float32, pin_memory=True)
    st_host = torch.empty(1, dtype=torch.int32, pin_memory=True)
    ke = max(3, min(a.steps, 20))
    e_s = [torch.cuda.Event(enable_timing=True) for _ in range(ke)]
    e_e = [torch.cuda.Event(enable_timing=True) for _ in range(ke)]
    barrier()
    for k in range(ke):
        if flush is not None:
            flush.zero_()
        e_s[k].record(stream)
        eng.g[0].copy_(g_host, non_blocking=True)
        eng.bias_g[0].copy_(b_host, non_blocking=True)
        eng.run()
        m_host.copy_(eng.work[0], non_blocking=True)
        bo_host.copy_(eng.bias_out, non_blocking=True)
        st_host.copy_(eng.status, non_blocking=True)
        e_e[k].record(stream)
    barrier()
    if int(st_host.item()) != 0:
        raise RuntimeError(f"e2e step reported status {int(st_host.item())}")
    e2e_local = statistics.mean(s.elapsed_time(e) for s, e in zip(e_s, e_e))
    t = torch.tensor([e2e_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t[0])
    h2d = 4 * (g_host.numel() + b_host.numel())
    d2h = 4 * (m_host.numel() + bo_host.numel() + st_host.numel())
    return e2e_ms, h2d, d2h


def e2e_pipelined(specs, a, dev, flush, barrier, stream):
    """HostPipelinedEngine: per parameter group, H2D || compression || D2H on three streams,
    the whole step one CUDA graph"""
    import statistics
    import torch
    from paper_1905_13727_b200.pipeline import HostPipelinedEngine
    pipe = HostPipelinedEngine(specs, a.rank, groups=int(os.environ.get("PSGD_E2E_GROUPS", "10")), seed=0, device=dev)
    for t in pipe.g_host + pipe.bias_host:
        t.normal_()
    for _ in range(3):
        pipe.step()
    barrier()
    ke = max(3, min(a.steps, 20))
    e_s = [torch.cuda.Event(enable_timing=True) for _ in range(ke)]
    e_e = [torch.cuda.Event(enable_timing=True) for _ in range(ke)]
    for k in range(ke):
        if flush is not None:
            flush.zero_()
        e_s[k].record(stream)
        pipe.step()
        e_e[k].record(stream)
    barrier()
    pipe.check()
    return statistics.mean(s.elapsed_time(e) for s, e in zip(e_s, e_e)), pipe.h2d_bytes, pipe.d2h_bytes

def main():
    a = parse_args()
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
