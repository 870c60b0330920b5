"""Benchmark of the B200 tile-tensor hot path (driver contract: one JSON line).

Workload (BASELINE.json config 5, the throughput sweep):
  X = [2048/16,2048/32,512/32] (131072 tiles x 16384 fp64 slots, 16 GiB),
  W = [*/16,2048/32,512/32] (replicated along dim 1, 1024 tiles, 128 MiB).
  One step = tt_sum(tt_mul(X, W), k) for k = 1, 2, 3 in turn, each ONE fused
  sm_100a launch (external left fold + in-tile rotate-and-sum, product never
  stored).  value = streamed tile-slots per second = 3 * 2^31 per step per rank.

Weak scaling (one process per GPU): rank r owns external tiles
[128r, 128r+128) of dim 1 of a global [N*2048, 2048, 512] tensor (its own
seeded slab); sums over dims 2 and 3 need no communication, the sum over
dim 1 spans ranks and finishes with one NCCL all-reduce of the 128 MiB
partial result.

Inputs (16 GiB) exceed the 126 MB L2, so no flush is needed between steps.
Timing: CUDA events on the launching stream, barrier + synchronize around the
K timed steps, max over ranks.  `e2e` repeats the step through the public
API from pinned HOST buffers (H2D of the dense input, pack, the three fused
products, unpack, D2H of the results).  `--impl reference` times the
reference's own CPU implementation (oracle/_ref, else the C restatement) on
a bounded slab of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "tile-slots/sec and HBM GB/s (fraction of peak) for pack, mul+rotate-sum, matmul"
S5 = 16384
X_TILES = 131072
W_TILES = 1024
OUT_TILES = {1: 1024, 2: 2048, 3: 8192}
GIB = 1 << 30


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_summary():
    """Per-launch DRAM bytes from the committed ncu --set full summary, if any."""
    for p in sorted((ROOT / "profiles").glob("r*_ncu_summary.json"), reverse=True):
        try:
            return json.loads(p.read_text())
        except Exception:
            continue
    return {}


class ClockSampler:
    """SM clocks + throttle reasons sampled (NVML, every 10 ms) during the
    timed region; falls back to nvidia-smi if pynvml is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int):
        self.index = index
        self.sm, self.mx, self.reasons = [], [], set()
        self._stop = threading.Event()
        self.thread = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[self.index]) if vis else self.index
            h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self._stop.is_set():
                    try:
                        self.sm.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        self.mx.append(mx)
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for name, bit in self.REASONS.items():
                            if r & bit:
                                self.reasons.add(name)
                    except Exception:
                        pass
                    self._stop.wait(0.01)
            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx),
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


# ---- distributed plumbing -------------------------------------------------------------


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def init_dist(world, backend):
    import torch.distributed as dist
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return dist if world > 1 else None


def max_over_ranks(x: float, dist, device) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---- CPU baseline (reference) ----------------------------------------------------------


_REF = {}


def _ref_lib(threads: int):
    """oracle/_ref (the reference compiled here), with W packed once."""
    import ctypes
    if "lib" not in _REF:
        ref_lib = ROOT / "oracle" / "_ref" / "libttref.so"
        if not ref_lib.exists():
            _REF["lib"] = None
            return None
        lib = ctypes.CDLL(str(ref_lib))
        lib.ref_set_threads(int(threads))  # TILETENSOR_THREADS, read once (tile_tensor.hpp:53-61)
        _REF["lib"] = lib
    return _REF["lib"]


def cpu_slab_pipeline(slab_tiles: int, threads: int):
    """Reference CPU path on the config-5 slab X[0:16*slab_tiles]: pack X,
    tt_sum(tt_mul(X, W), k) for k = 1, 2, 3, unpack (W packed once, outside).
    Returns (kind, cores, seconds dict, streamed tile-slots)."""
    import ctypes

    import numpy as np

    from paper_2011_01805_b200 import configs, parse_shape
    from paper_2011_01805_b200.tiletensor import DimSpec, TileTensorShape

    rows = 16 * slab_tiles
    x = np.ascontiguousarray(configs.c5_x_slab(slice(0, rows)))
    sx = TileTensorShape([DimSpec(rows, 1, 16), DimSpec(2048, 1, 32), DimSpec(512, 1, 32)])
    sw = parse_shape(configs.C5_W_SHAPE)
    streamed = 3 * sx.tile_count() * S5
    lib = _ref_lib(threads)
    dp = ctypes.POINTER(ctypes.c_double)
    if lib is not None:
        if "w" not in _REF:
            w = np.ascontiguousarray(configs.c5_w())
            if lib.ref_bench_prepare_w(w.ctypes.data_as(dp), ctypes.byref(sw.to_c()),
                                       ctypes.c_int64(S5)) != 0:
                raise RuntimeError("reference W pack failed")
            _REF["w"] = True
        dims = (ctypes.c_int * 3)(1, 2, 3)
        secs = (ctypes.c_double * 4)()
        rc = lib.ref_bench_step(x.ctypes.data_as(dp), ctypes.byref(sx.to_c()), dims, 3, secs)
        if rc != 0:
            raise RuntimeError("reference pipeline failed")
        return ("reference", int(lib.ref_thread_hint()),
                {"pack": secs[0], "mul_sum": secs[1], "unpack": secs[2]}, streamed)
    # fall back to the C restatement (single-threaded port)
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import Oracle
    o = Oracle()
    if "w_port" not in _REF:
        _REF["w_port"] = o.pack(np.ascontiguousarray(configs.c5_w()), sw, S5)
    tw = _REF["w_port"]
    t0 = time.perf_counter()
    tx = o.pack(x, sx, S5)
    t1 = time.perf_counter()
    outs = [o.mul_sum(sx, tx, sw, tw, S5, k) for k in (1, 2, 3)]
    t2 = time.perf_counter()
    for so, ot, _ in outs:
        o.unpack(so, S5, ot)
    t3 = time.perf_counter()
    return ("port", 1, {"pack": t1 - t0, "mul_sum": t2 - t1, "unpack": t3 - t2}, streamed)


def run_reference(args):
    world, rank, _ = dist_env()
    if world > 1 and rank != 0:
        return  # rank 0 alone runs the CPU reference
    threads = min(64, os.cpu_count() or 1)
    slab = args.ref_slab_tiles
    for _ in range(args.warmup):
        cpu_slab_pipeline(slab, threads)
    times = []
    kind, cores, streamed = "reference", threads, 0
    for _ in range(args.steps):
        kind, cores, secs, streamed = cpu_slab_pipeline(slab, threads)
        times.append(secs["pack"] + secs["mul_sum"] + secs["unpack"])
    total = sum(times)
    value = streamed * len(times) / total
    sample = (f"config-5 slab X[0:{16 * slab}] ({slab * 64 * 16} of 131072 tiles): pack X, "
              "tt_sum(tt_mul(X,W),k) k=1,2,3, unpack, per step (W packed once)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tile-slots/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded splitmix64 U[-1,1])",
        "config": {"workload": "c5 [2048/16,2048/32,512/32] x [*/16,2048/32,512/32], sum dims 1,2,3 (CPU slab)",
                   "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": "tile-slots/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "tile-slots/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- our arm ----------------------------------------------------------------------------


def time_events(fn, reps, stream):
    import torch
    fn()  # warm-up outside the timed region (allocator growth, first-launch setup)
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(reps):
        fn()
    end.record(stream)
    end.synchronize()
    return start.elapsed_time(end) / 1e3 / reps


def run_ours(args):
    import numpy as np
    import torch

    import paper_2011_01805_b200 as tt
    from paper_2011_01805_b200 import configs

    world, rank, local = dist_env()
    # one process per GPU; more ranks than GPUs only for the gloo functional check
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # TT_BENCH_BACKEND=gloo: functional check of the N > 1 path with several
    # ranks on one GPU (NCCL refuses duplicate devices) -- never a measurement
    dist = init_dist(world, os.environ.get("TT_BENCH_BACKEND", "nccl"))
    stream = torch.cuda.current_stream(dev)
    hbm_peak, peak_src = peaks()

    from paper_2011_01805_b200 import sharding
    S = tt.Session(S5, 8, device=local)
    # weak scaling: the global X is [2048*N, 2048, 512]; rank r owns external
    # tiles [128r, 128r+128) of dim 1 (its own 16 GiB slab); W broadcasts.
    sx_global = tt.TileTensorShape([tt.DimSpec(2048 * world, 1, 16), tt.DimSpec(2048, 1, 32),
                                    tt.DimSpec(512, 1, 32)])
    plan = sharding.plan(sx_global, 1, world, rank)
    sx = plan.local_shape
    sw = tt.parse_shape(configs.C5_W_SHAPE)
    assert sharding.operand_plan(sw, plan) is None and sx.tile_count() == X_TILES
    # inputs generated on the device with the shared counter-based generator
    x_dense = torch.empty(configs.C5_DIMS, dtype=torch.float64, device=dev)
    w_dense = torch.empty((1, 2048, 512), dtype=torch.float64, device=dev)
    rank_offset = plan.row_slice.start * (2048 * 512)
    tt.fill_uniform(S, x_dense, configs.C5_SEED_X, -1.0, 1.0, offset=rank_offset)
    tt.fill_uniform(S, w_dense, configs.C5_SEED_W, -1.0, 1.0)  # same W on every rank
    X = tt.pack(x_dense, sx, S)
    W = tt.pack(w_dense, sw, S)

    def mul_sum(a, b, k):
        return tt.tt_mul_sum(a, b, k)

    def step():
        return [sharding.sharded_mul_sum(X, W, k, plan, mul_sum, lambda r: r.data())[0]
                for k in (1, 2, 3)]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()

    # per-launch timing of the fused kernel (one launch per dim)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    per_dim = {1: [], 2: [], 3: []}
    launches0 = S.launches()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for _ in range(args.steps):
            ev[0].record(stream)
            partial, work = None, None
            for k in (1, 2, 3):
                r = tt.tt_mul_sum(X, W, k)
                ev[k].record(stream)
                if k == plan.shard_dim:
                    partial = r
                    if world > 1:
                        # the one real exchange: the dim-1 sum spans the ranks'
                        # slabs (NCCL over NVLink), in flight while the dim-2
                        # and dim-3 products run
                        work = sharding.allreduce_partial(partial.data(), async_op=True)
            if work is not None:
                work.wait()
            # the sync below is per step only to read the per-launch events
            ev[3].synchronize()
            per_dim[1].append(ev[0].elapsed_time(ev[1]) / 1e3)
            per_dim[2].append(ev[1].elapsed_time(ev[2]) / 1e3)
            per_dim[3].append(ev[2].elapsed_time(ev[3]) / 1e3)
        t_end.record(stream)
        t_end.synchronize()
        elapsed = t_start.elapsed_time(t_end) / 1e3
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
    launches = S.launches() - launches0
    elapsed_max = max_over_ranks(elapsed, dist, dev)
    step_slots = 3 * X_TILES * S5
    value = world * step_slots * args.steps / elapsed_max

    # roofline of the dominant kernel (the fused group kernel, all three dims)
    alg = {k: (X_TILES + W_TILES + OUT_TILES[k]) * S5 * 8 for k in (1, 2, 3)}
    dur = {k: sum(v) / len(v) for k, v in per_dim.items()}
    achieved = sum(alg.values()) / sum(dur.values()) / 1e9
    traffic = traffic_summary()
    tr = traffic.get("c5_mul_sum_bytes_per_launch")

    ops = {}
    for k in (1, 2, 3):
        gbs = alg[k] / dur[k] / 1e9
        ops[f"mul_sum_dim{k}"] = {"ms": dur[k] * 1e3, "GB/s": gbs, "frac": gbs / hbm_peak,
                                  "frac_of_8TBps": gbs / 8000.0,
                                  "tile_slots_per_s": X_TILES * S5 / dur[k],
                                  "alg_bytes": alg[k]}

    # pack (dense -> tiles), same tensor
    try:
        if not args.skip_extra:
            t = time_events(lambda: tt.pack(x_dense, sx, S), max(1, args.steps), stream)
            pb = 2 * X_TILES * S5 * 8
            ops["pack"] = {"ms": t * 1e3, "GB/s": pb / t / 1e9, "frac": pb / t / 1e9 / hbm_peak,
                           "frac_of_8TBps": pb / t / 1e12 / 8.0, "tile_slots_per_s": X_TILES * S5 / t,
                           "alg_bytes": pb}
            del t
            # unfused elementwise (tt_mul with W broadcast along dim 1, tt_add): 16 GiB in, 16 GiB out
            for name, fn, nb in (("ew_mul_bcast", lambda: tt.tt_mul(X, W), (2 * X_TILES + W_TILES) * S5 * 8),
                                 ("ew_add", lambda: tt.tt_add(X, X), 2 * X_TILES * S5 * 8)):
                t = time_events(fn, max(1, args.steps), stream)
                ops[name] = {"ms": t * 1e3, "GB/s": nb / t / 1e9, "frac": nb / t / 1e9 / hbm_peak,
                             "tile_slots_per_s": X_TILES * S5 / t, "alg_bytes": nb}
            # the other tile passes on config-5-sized data (rows a8, a10, a12)
            reps = max(1, min(3, args.steps))
            for k in (1, 2, 3):
                t = time_events(lambda: tt.tt_sum(X, k), reps, stream)
                nb = (X_TILES + OUT_TILES[k]) * S5 * 8
                ops[f"sum_dim{k}"] = {"ms": t * 1e3, "GB/s": nb / t / 1e9, "frac": nb / t / 1e9 / hbm_peak}
            t = time_events(lambda: tt.tiles_rotate(S, X.data(), 5), reps, stream)
            ops["rotate"] = {"ms": t * 1e3, "GB/s": 2 * X_TILES * S5 * 8 / t / 1e9,
                             "frac": 2 * X_TILES * S5 * 8 / t / 1e9 / hbm_peak}
            R3 = tt.tt_sum(X, 3)  # [2048/16,2048/32,1?/32]: 8192 boundary tiles
            nb = 2 * OUT_TILES[3] * S5 * 8
            t = time_events(lambda: tt.clean_unknowns(R3), 10, stream)
            ops["clean_unknowns"] = {"ms": t * 1e3, "GB/s": nb / t / 1e9, "frac": nb / t / 1e9 / hbm_peak}
            C3 = tt.clean_unknowns(R3)
            t = time_events(lambda: tt.replicate_dim(C3, 3), 10, stream)
            ops["replicate_dim"] = {"ms": t * 1e3, "GB/s": nb / t / 1e9, "frac": nb / t / 1e9 / hbm_peak}
            del R3, C3
            ops.update(bench_matmul(tt, configs, S, stream, hbm_peak, max(3, args.steps)))
            ops.update(bench_small_configs(tt, configs, stream, hbm_peak, max(20, args.steps)))
    except Exception as exc:  # keep the bench line: report the failure instead
        print(f"[bench] extra failed: {exc!r}", file=sys.stderr)
        ops["extra_error"] = repr(exc)

    # end to end from pinned host memory through the public API
    e2e = None
    try:
        # every local rank stages its host input (x2 briefly while pinning): use
        # the largest slab of X (1, 1/2, 1/4, 1/8 of its dim-1 rows) that fits
        # the host's free memory, decided once for all ranks (the block below
        # has collectives) -- never drive the host out of memory
        frac = 1.0
        try:
            import psutil
            local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
            avail = psutil.virtual_memory().available
            if os.environ.get("TT_BENCH_HOST_GIB"):  # test hook: pretend a smaller host
                avail = float(os.environ["TT_BENCH_HOST_GIB"]) * 2**30
            while frac > 0.125 and 2.2 * x_dense.numel() * 8 * frac * local_world > avail:
                frac /= 2
        except Exception:
            pass
        frac = -max_over_ranks(-frac, dist, dev)
        if not args.skip_e2e:
            rows = int(x_dense.shape[0] * frac)
            sx_e = sx if frac == 1.0 else tt.TileTensorShape(
                [tt.DimSpec(rows, 1, 16), tt.DimSpec(2048, 1, 32), tt.DimSpec(512, 1, 32)])
            pinned = args.e2e_pinned
            host_x = x_dense[:rows].to("cpu")
            if pinned:
                try:  # fall back to pageable memory if the host cannot pin it
                    host_x = host_x.pin_memory()
                except RuntimeError as exc:
                    print(f"[bench] rank {rank}: pinning the host input failed ({exc}); pageable",
                          file=sys.stderr)
                    pinned = False
            host_w = w_dense.to("cpu").pin_memory() if pinned else w_dense.to("cpu")
            del x_dense
            torch.cuda.empty_cache()

            def e2e_step():
                Xh = tt.pack(host_x, sx_e, S)   # H2D of the dense input + pack kernel
                Wh = tt.pack(host_w, sw, S)
                d2h = 0
                for k in (1, 2, 3):
                    r, _ = sharding.sharded_mul_sum(Xh, Wh, k, plan, mul_sum, lambda t: t.data())
                    res = tt.unpack(r)          # unpack kernel + D2H
                    d2h += res.nbytes
                return d2h
            e2e_step()
            torch.cuda.synchronize(dev)
            reps = max(1, min(args.steps, args.e2e_steps))
            t0 = time.perf_counter()
            for _ in range(reps):
                d2h = e2e_step()
            torch.cuda.synchronize(dev)
            e_el = max_over_ranks((time.perf_counter() - t0) / reps, dist, dev)
            h2d = host_x.numel() * 8 + host_w.numel() * 8
            e2e = {"value": world * 3 * sx_e.tile_count() * S5 / e_el, "unit": "tile-slots/s",
                   "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                   "ms_per_step": e_el * 1e3, "steps": reps, "host_buffers": "pinned" if pinned else "pageable",
                   "x_slab_fraction": frac}
    except Exception as exc:  # keep the bench line: report the failure instead
        print(f"[bench] e2e failed: {exc!r}", file=sys.stderr)
        e2e = {"error": repr(exc)}

    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        threads = min(64, os.cpu_count() or 1)
        kind, cores, secs, streamed = cpu_slab_pipeline(args.cpu_slab_tiles, threads)
        cpu = {"value": streamed / secs["mul_sum"], "unit": "tile-slots/s", "cores": cores,
               "kind": kind,
               "sample": (f"reference tt_sum(tt_mul(X,W),k) k=1,2,3 on the config-5 slab "
                          f"X[0:{16 * args.cpu_slab_tiles}] ({args.cpu_slab_tiles * 1024} tiles), "
                          f"{secs['mul_sum']:.2f} s; pack {secs['pack']:.2f} s, "
                          f"unpack {secs['unpack']:.2f} s")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tile-slots/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed_max / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded splitmix64 U[-1,1] generated on device; 16 GiB input > 126 MB L2 (no flush needed)",
            "config": {"workload": "c5: tt_sum(tt_mul(X[2048/16,2048/32,512/32], W[*/16,2048/32,512/32]), k) for k=1,2,3",
                       "slots": S5, "x_tiles_per_rank": X_TILES, "global_x": [2048 * world, 2048, 512],
                       "parallelism": f"shard external dim 1 over {world} rank(s); NCCL all-reduce for the dim-1 sum",
                       "l2": "inputs larger than L2"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "frac_of_8TBps": achieved / 8000.0,
                         "peak_source": peak_src, "traffic": tr,
                         "kernel": "group_tma_kernel / group_tma_win_kernel (fused fold + rotate-and-sum, TMA ring)",
                         "alg_bytes_per_step": sum(alg.values())},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "ops": ops,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def bench_small_configs(tt, configs, stream, hbm_peak, reps):
    """Configs 1, 2 and 4 (device-resident operands): per-call latency of the
    op chain through the public API (CUDA events, averaged over `reps`).
    These are parity configs and latency-bound; reported beside
    the bench line, not as it."""
    import torch
    out = {}
    c1 = configs.config1()
    S1 = tt.Session(512, 8, device=torch.cuda.current_device())
    sA = tt.parse_shape(c1.shapes["A"])
    A, B = tt.pack(c1.tensors["A"], sA, S1), tt.pack(c1.tensors["B"], sA, S1)
    t = time_events(lambda: tt.tt_mul_sum(A, B, 2), reps, stream)
    out["c1_mul_sum"] = {"us": t * 1e6, "note": "[100/16,200/32] x same, sum dim 2 (49 tiles of 512)"}
    c2 = configs.config2()
    S2 = tt.Session(8192, 8, device=torch.cuda.current_device())
    M = tt.pack(c2.tensors["M"], tt.parse_shape(c2.shapes["M"]), S2)
    V = tt.pack(c2.tensors["V"], tt.parse_shape(c2.shapes["V"]), S2)
    t = time_events(lambda: tt.matvec_a(M, V), reps, stream)
    alg = (512 + 32 + 16) * 8192 * 8
    out["c2_matvec"] = {"us": t * 1e6, "GB/s": alg / t / 1e9, "frac": alg / t / 1e9 / hbm_peak,
                        "note": "M[1024/64,4096/128] x V[*/64,4096/128], sum dim 2 (35 MiB, L2-scale)"}
    c4 = configs.config4(True)
    S4 = tt.Session(8192, 8, device=torch.cuda.current_device())
    T = {k: tt.pack(c4.tensors[k], tt.parse_shape(v), S4) for k, v in c4.shapes.items()}

    def c4_chain():  # each layer one call: FC + bias (+ square), tail fused into the tree pass
        h = tt.tt_mul_sum_affine(T["W1t"], T["X"], 1, T["b1"], square=True)
        return tt.tt_mul_sum_affine(T["W2"], h, 2, T["b2"])

    def c4_unfused():  # the reference's five-call composition
        h = tt.tt_add(tt.tt_mul_sum(T["W1t"], T["X"], 1), T["b1"])
        h = tt.tt_mul(h, h)
        return tt.tt_add(tt.tt_mul_sum(T["W2"], h, 2), T["b2"])
    t = time_events(c4_chain, reps, stream)
    out["c4_fc_square_fc"] = {"us": t * 1e6, "samples_per_s": 4096 / t,
                              "unfused_us": time_events(c4_unfused, reps, stream) * 1e6,
                              "note": "784->100->square->10 on 4096 samples, batch interleaved (~) in "
                                      "tile dim 3; tt_mul_sum_affine per layer"}
    # the paper's network (CryptoNets: conv 5x5x5 -> square -> fc 845x100 -> square -> fc 100x10),
    # batch packed: every network scalar a tile of 8192 samples, batch resident on the device
    from paper_2011_01805_b200 import nn
    net = nn.cryptonets_network(42)
    S8 = tt.Session(8192, 8, device=torch.cuda.current_device())
    xb = torch.from_numpy(configs.uniform(784 * 8192, 8, 0.0, 1.0).reshape(784, 8192)).cuda()
    nn.cryptonets_infer(net, xb, (1, 1, 8192), S8)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        nn.cryptonets_infer(net, xb, (1, 1, 8192), S8)
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / 3
    comp = nn.CompiledBatchPacked(net, S8)
    comp.infer(xb)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        comp.infer(xb)
    torch.cuda.synchronize()
    tc = (time.perf_counter() - t0) / 5
    comp.close()
    # the paper's tiled layout for one sample (tile [32, 256, 1]), per call and
    # with the weights packed once (nn.CompiledTiled)
    one = configs.uniform(784, 13, 0.0, 1.0).reshape(784, 1)
    nn.cryptonets_infer(net, one, (32, 256, 1), S8)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        nn.cryptonets_infer(net, one, (32, 256, 1), S8)
    torch.cuda.synchronize()
    t_tiled = (time.perf_counter() - t0) / 5
    ct = nn.CompiledTiled(net, (32, 256, 1), S8)
    ct.infer(one)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        ct.infer(one)
    torch.cuda.synchronize()
    t_ctiled = (time.perf_counter() - t0) / 5
    out["cryptonets_tiled_1_sample"] = {"ms": t_tiled * 1e3, "compiled_ms": t_ctiled * 1e3,
                                        "note": "nn.cryptonets_infer tile [32,256,1], one sample, wall clock "
                                                "incl. host packing; compiled_ms: nn.CompiledTiled"}
    out["cryptonets_batch_packed"] = {"ms": t * 1e3, "samples_per_s": 8192 / t,
                                      "compiled_ms": tc * 1e3, "compiled_samples_per_s": 8192 / tc,
                                      "note": "nn.cryptonets_infer tile [1,1,8192], wall clock per call "
                                              "incl. host layer prep (batch already on the GPU); "
                                              "compiled_*: nn.CompiledBatchPacked (layers uploaded once)"}
    # the same chains captured once into CUDA graphs and replayed (no host launch cost)
    for name, fn in (("c1_mul_sum", lambda: tt.tt_mul_sum(A, B, 2)),
                     ("c2_matvec", lambda: tt.matvec_a(M, V)), ("c4_fc_square_fc", c4_chain)):
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(3):
                fn()
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        out[name]["graph_replay_us"] = time_events(g.replay, reps, stream) * 1e6
    return out


FP64_PEAK_OPS = 18.34e12  # B200, 148 SMs x 64 FP64 lanes at boost (profiles/r01_fp64_peak.txt)


def bench_matmul(tt, configs, S, stream, hbm_peak, reps):
    """Config 3 ('3b': matmul_b then matmul_a, no repacking) on 8192-slot tiles."""
    import torch
    c3 = configs.config3()
    S3 = tt.Session(8192, 8, device=torch.cuda.current_device())
    T = {k: tt.pack(c3.tensors[k], tt.parse_shape(v), S3) for k, v in c3.shapes.items()
         if k in ("A3", "Bt3", "C3")}

    def chain():
        s1 = tt.matmul_b(T["Bt3"], T["C3"])
        return tt.matmul_a(T["A3"], s1)
    chain()
    torch.cuda.synchronize()
    t = time_events(chain, reps, stream)
    # the same chain captured once into a CUDA graph (no host launch cost between kernels)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(3):
            chain()
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        chain()
    t_graph = time_events(g.replay, reps, stream)
    tile = 8192 * 8
    # unique operand tiles + out tiles of both stages
    alg = (1536 + 768 + 512 + 512 + 1024 + 512 + 512) * tile
    prod_tiles = 24576 + 16384
    # the fold is FP64-issue bound, not HBM bound: one DMUL + one DADD per
    # product slot (no contraction -- bit parity), against the measured
    # register-only DMUL+DADD rate (tools/micro/fp64_peak.cu,
    # profiles/r01_fp64_peak.txt)
    fp64_ops = 2 * prod_tiles * 8192
    # the literal chain ("3a"): matmul_a(A, B) -> clean_unknowns -> replicate_dim 2 -> x C^T, sum dim 3
    TA = {k: tt.pack(c3.tensors[k], tt.parse_shape(c3.shapes[k]), S3) for k in ("B3", "Ct3")}

    def chain_3a_calls():
        ra = tt.matmul_a(T["A3"], TA["B3"])
        rep = tt.replicate_dim(tt.clean_unknowns(ra), 2)
        return tt.tt_mul_sum(rep, TA["Ct3"], 3)

    def chain_3a():  # matmul_a + clean_unknowns as one call (the pipeline seam)
        rep = tt.replicate_dim(tt.tt_mul_sum_clean(T["A3"], TA["B3"], 2), 2)
        return tt.tt_mul_sum(rep, TA["Ct3"], 3)
    chain_3a()
    chain_3a_calls()
    t3a = time_events(chain_3a, reps, stream)
    t3a_calls = time_events(chain_3a_calls, reps, stream)
    fp64_3a = 2 * 8192 * (32 * 32 * 48 + 32 * 8 * 48)  # product tiles x slots, both products
    out_3a = {"ms": t3a * 1e3, "fp64_tops": fp64_3a / t3a / 1e12, "fp64_frac": fp64_3a / t3a / FP64_PEAK_OPS,
              "separate_calls_ms": t3a_calls * 1e3,
              "note": "literal config-3 chain: matmul_a(A3, B3) -> clean_unknowns -> replicate_dim(2) "
                      "-> tt_mul_sum(., Ct3, 3); the first two as one tt_mul_sum_clean call "
                      "(separate_calls_ms: four calls)"}
    return {"matmul_c3a": out_3a, "matmul_c3b": {"ms": t * 1e3, "GB/s": alg / t / 1e9, "frac": alg / t / 1e9 / hbm_peak,
                           "tile_slots_per_s": prod_tiles * 8192 / t, "alg_bytes": alg,
                           "graph_replay_ms": t_graph * 1e3,
                           "fp64_tops": fp64_ops / t / 1e12,
                           "fp64_frac": fp64_ops / t / FP64_PEAK_OPS,
                           "fp64_peak_source": "measured DMUL+DADD issue rate, 18.34e12 thread-ops/s",
                           "note": "Bt3[768/16,1024/32,*/16] x C3[768/16,*/32,256/16] -> matmul_a(A3, .)"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-extra", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-pinned", type=int, default=1)
    ap.add_argument("--cpu-slab-tiles", type=int, default=48)  # ~10 s of reference CPU work
    ap.add_argument("--ref-slab-tiles", type=int, default=4)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
