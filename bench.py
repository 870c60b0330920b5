"""Benchmark of the B200 tile-tensor hot path (driver contract: one JSON line).

Workload (BASELINE.json config 5, the throughput sweep):
  X = [2048/16,2048/32,512/32] (131072 tiles x 16384 fp64 slots, 16 GiB),
  W = [*/16,2048/32,512/32] (replicated along dim 1, 1024 tiles, 128 MiB).
  One step = tt_sum(tt_mul(X, W), k) for k = 1, 2, 3 in turn, each ONE fused
  sm_100a launch (external left fold + in-tile rotate-and-sum, product never
  stored).  value = streamed tile-slots per second over ALL ranks
  (3 * 2^31 per step for the whole job).

Strong scaling (default for N > 1, config 5 as named): the one 16 GiB X is
block-partitioned along external dim 1 -- rank r owns 128/N external rows --
and W is held whole on every rank.  Sums over dims 2 and 3 are local; the sum
over dim 1 spans ranks and finishes with one NCCL all-reduce of the 128 MiB
partial result (in flight while dims 2 and 3 run); its exact form (the left
folds chained rank to rank, sharding.chain_mul_sum) is timed beside it.
`--scaling weak`: every rank owns a whole 2048-row slab of [2048*N,2048,512].

Inputs (16 GiB) exceed the 126 MB L2, so no flush is needed between steps.
Timing: CUDA events on the launching stream, barrier + synchronize around the
K timed steps (no host sync inside), max over ranks.  `e2e` repeats the step through the public
API from pinned HOST buffers (H2D of the dense input, pack, the three fused
products, unpack, D2H of the results).  `--impl reference` times the
reference's own CPU implementation (oracle/_ref, else the C restatement) on
a bounded slab of the same workload, all host threads, the same three products
per step (pack / unpack reported separately); it never imports the product.
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
        """NVML is initialised and its queries warmed HERE -- construct the sampler
        before the warm-up steps, so that nothing but the synchronize and the barrier
        sits between the warm-up and the timed region (NVML's init and first queries
        take tens of ms and hold a driver lock the kernel launches also take: run
        beside the first timed launch they made it read 3-63 ms instead of 2.55 ms,
        and run before it they leave the GPU idle long enough to drop its clocks)."""
        self.index = index
        self.sm, self.mx, self.reasons = [], [], set()
        self._stop = threading.Event()
        self.thread = None
        self._sample = None
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[self.index]) if vis else self.index
            h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def sample(record=True):
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    if record:
                        self.sm.append(sm)
                        self.mx.append(mx)
                        for name, bit in self.REASONS.items():
                            if r & bit:
                                self.reasons.add(name)
                except Exception:
                    pass
            sample(record=False)
            self._sample = sample
        except Exception:
            self._sample = None

    def __enter__(self):
        if self._sample is not None:
            def run():  # first sample 10 ms into the timed region
                while not self._stop.wait(0.01):
                    self._sample()
            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
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


# ---- CPU reference legs (no import of the product package) ---------------------------
#
# The reference arm and the cpu_baseline leg load ONLY oracle/_ref/libttref.so
# (the unmodified reference headers compiled here, oracle/Makefile) -- or, when
# it is absent, the C restatement oracle/_build/libttoracle.so ("port").  The
# seeded inputs come from a local copy of the shared counter-based generator
# (splitmix64, bit-identical to tt_fill_uniform on the device), and shapes are
# plain tt_shape structs, so paper_2011_01805_b200 is never imported here.

import ctypes


class _CDim(ctypes.Structure):  # tt_dim, include/tiletensor_b200.h
    _fields_ = [("n", ctypes.c_int64), ("d", ctypes.c_int64), ("t", ctypes.c_int64),
                ("unknown", ctypes.c_int32), ("interleaved", ctypes.c_int32)]


class _CShape(ctypes.Structure):  # tt_shape
    _fields_ = [("rank", ctypes.c_int32), ("relaxed", ctypes.c_int32), ("dims", _CDim * 16)]  # TT_MAX_RANK


def _cshape(dims):
    sh = _CShape()
    sh.rank, sh.relaxed = len(dims), 0
    for i, (n, d, t) in enumerate(dims):
        sh.dims[i] = _CDim(n, d, t, 0, 0)
    return sh


C5_SEED_X, C5_SEED_W = 13, 14   # == paper_2011_01805_b200.configs


def _uniform_at(idx, seed, lo, hi):
    import numpy as np
    m1, m2, gold = np.uint64(0xBF58476D1CE4E5B9), np.uint64(0x94D049BB133111EB), np.uint64(0x9E3779B97F4A7C15)

    def sm(x):
        with np.errstate(over="ignore"):
            x = x + gold
            x = (x ^ (x >> np.uint64(30))) * m1
            x = (x ^ (x >> np.uint64(27))) * m2
            return x ^ (x >> np.uint64(31))
    key = sm(np.array([seed], dtype=np.uint64))[0]
    u = sm(np.asarray(idx, dtype=np.uint64) ^ key)
    return lo + (hi - lo) * ((u >> np.uint64(11)).astype(np.float64) * (2.0 ** -53))


def _c5_x_rows(r0, r1):
    import numpy as np
    idx = np.arange(r0 * 2048 * 512, r1 * 2048 * 512, dtype=np.uint64)
    return _uniform_at(idx, C5_SEED_X, -1.0, 1.0).reshape(r1 - r0, 2048, 512)


def _c5_w():
    import numpy as np
    return _uniform_at(np.arange(2048 * 512, dtype=np.uint64), C5_SEED_W, -1.0, 1.0).reshape(1, 2048, 512)


def cpu_leg(slab_tiles: int, steps: int, warmup: int):
    """The reference's CPU path on the config-5 slab X[0:16*slab_tiles]
    (slab_tiles external rows of dim 1 = slab_tiles*1024 tiles): pack X once,
    then `warmup` + `steps` x [tt_sum(tt_mul(X, W), k) for k = 1, 2, 3] --
    the same three products as one GPU step -- then unpack the results once.
    Threads: TILETENSOR_THREADS from the environment (read once per process
    by the reference, tile_tensor.hpp:53-61).  Returns a dict."""
    import numpy as np
    dp = ctypes.POINTER(ctypes.c_double)
    rows = 16 * slab_tiles
    x = np.ascontiguousarray(_c5_x_rows(0, rows))
    w = np.ascontiguousarray(_c5_w())
    sx = _cshape([(rows, 1, 16), (2048, 1, 32), (512, 1, 32)])
    sw = _cshape([(1, 16, 16), (2048, 1, 32), (512, 1, 32)])
    x_tiles = slab_tiles * 64 * 16
    ref_lib = ROOT / "oracle" / "_ref" / "libttref.so"
    out = {"slab_tiles": x_tiles, "streamed_slots_per_step": 3 * x_tiles * S5}
    if ref_lib.exists():
        lib = ctypes.CDLL(str(ref_lib))
        secs = (ctypes.c_double * 4)()
        if lib.ref_bench_prepare_w(w.ctypes.data_as(dp), ctypes.byref(sw), ctypes.c_int64(S5)) != 0:
            raise RuntimeError("reference W pack failed")
        if lib.ref_bench_pack_x(x.ctypes.data_as(dp), ctypes.byref(sx), secs) != 0:
            raise RuntimeError("reference X pack failed")
        out["pack_s"] = secs[0]
        dims = (ctypes.c_int * 3)(1, 2, 3)
        times = []
        for i in range(warmup + steps):
            if lib.ref_bench_mul_sum(dims, 3, secs) != 0:
                raise RuntimeError("reference mul+sum failed")
            if i >= warmup:
                times.append(secs[0])
        if lib.ref_bench_unpack(secs) != 0:
            raise RuntimeError("reference unpack failed")
        out.update(kind="reference", cores=int(lib.ref_thread_hint()), unpack_s=secs[0],
                   mul_sum_s=times)
        return out
    # the C restatement (single-threaded port of the same algorithm)
    lib = ctypes.CDLL(str(ROOT / "oracle" / "_build" / "libttoracle.so"))
    lib.or_tile_count.restype = ctypes.c_int64
    tx = np.zeros((x_tiles, S5))
    tw = np.zeros((lib.or_tile_count(ctypes.byref(sw)), S5))
    lib.or_pack(w.ctypes.data_as(dp), ctypes.byref(sw), ctypes.c_int64(S5), tw.ctypes.data_as(dp))
    t0 = time.perf_counter()
    lib.or_pack(x.ctypes.data_as(dp), ctypes.byref(sx), ctypes.c_int64(S5), tx.ctypes.data_as(dp))
    out["pack_s"] = time.perf_counter() - t0
    prod = np.zeros((x_tiles, S5))
    sp, so = _CShape(), _CShape()
    cost = (ctypes.c_uint64 * 6)()
    res = []
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        res = []
        for k in (1, 2, 3):
            lib.or_elementwise(1, ctypes.byref(sx), tx.ctypes.data_as(dp), ctypes.byref(sw),
                               tw.ctypes.data_as(dp), ctypes.c_int64(S5), ctypes.byref(sp),
                               prod.ctypes.data_as(dp), cost)
            r = np.zeros((x_tiles, S5))
            lib.or_sum(ctypes.byref(sp), prod.ctypes.data_as(dp), ctypes.c_int64(S5), k, -1,
                       ctypes.byref(so), r.ctypes.data_as(dp), cost)
            res.append((so, r))
        if i >= warmup:
            times.append(time.perf_counter() - t0)
    out.update(kind="port", cores=1, unpack_s=0.0, mul_sum_s=times)
    return out


def cpu_leg_subprocess(threads: int, slab_tiles: int, steps: int, warmup: int):
    """cpu_leg in a fresh process with TILETENSOR_THREADS=threads (the
    reference reads it once per process)."""
    env = dict(os.environ, TILETENSOR_THREADS=str(threads))
    proc = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--cpu-leg",
                           f"{slab_tiles},{steps},{warmup}"], env=env, capture_output=True,
                          text=True, timeout=900)
    if proc.returncode != 0:
        raise RuntimeError(f"cpu leg failed: {proc.stderr[-400:]}")
    return json.loads(proc.stdout.strip().splitlines()[-1])


def _leg_summary(leg):
    tps = leg["streamed_slots_per_step"] * len(leg["mul_sum_s"]) / sum(leg["mul_sum_s"])
    return tps, (f"reference tt_sum(tt_mul(X,W),k) k=1,2,3 on the config-5 slab "
                 f"({leg['slab_tiles']} of 131072 X tiles), {len(leg['mul_sum_s'])} step(s) of "
                 f"{statistics.mean(leg['mul_sum_s']):.3f} s; pack of the slab {leg['pack_s']:.2f} s, "
                 f"unpack of the results {leg['unpack_s']:.2f} s (reported, not in value)")


def host_threads() -> int:
    return min(64, os.cpu_count() or 1)  # the reference clamps to [1, 64]


def cpu_baseline_block(slab_all: int, slab_one: int):
    """cpu_baseline of the GPU arm: all host threads, plus 1 thread."""
    leg = cpu_leg_subprocess(host_threads(), slab_all, 1, 0)
    tps, sample = _leg_summary(leg)
    out = {"value": tps, "unit": "tile-slots/s", "cores": leg["cores"], "kind": leg["kind"],
           "sample": sample, "pack_tile_slots_per_s": leg["slab_tiles"] * S5 / leg["pack_s"]}
    try:
        one = cpu_leg_subprocess(1, slab_one, 1, 0)
        tps1, sample1 = _leg_summary(one)
        out["one_thread"] = {"value": tps1, "unit": "tile-slots/s", "cores": 1, "sample": sample1,
                             "pack_tile_slots_per_s": one["slab_tiles"] * S5 / one["pack_s"]}
    except Exception as exc:
        out["one_thread"] = {"error": repr(exc)}
    return out


def run_reference(args):
    """--impl reference: the reference's own CPU path, all host threads,
    on rank 0 only; the same config dict, metric and step content (the three
    fused products' work) as our arm."""
    world, rank, _ = dist_env()
    if world > 1 and rank != 0:
        return  # rank 0 alone runs the CPU reference
    threads = host_threads()
    os.environ["TILETENSOR_THREADS"] = str(threads)  # before the reference library loads
    leg = cpu_leg(args.ref_slab_tiles, args.steps, args.warmup)
    value, sample = _leg_summary(leg)
    one = None
    try:
        o = cpu_leg_subprocess(1, args.cpu_one_thread_slab_tiles, 1, 0)
        v1, s1 = _leg_summary(o)
        one = {"value": v1, "unit": "tile-slots/s", "cores": 1, "sample": s1}
    except Exception as exc:
        one = {"error": repr(exc)}
    scaling = resolve_scaling(args, world)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tile-slots/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(leg["mul_sum_s"]), "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": workload_config(world, scaling),
        "cpu_baseline": {"value": value, "unit": "tile-slots/s", "cores": leg["cores"],
                         "kind": leg["kind"], "sample": sample, "one_thread": one},
        "e2e": {"value": value, "unit": "tile-slots/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "phases": {"pack_s": leg["pack_s"], "unpack_s": leg["unpack_s"],
                   "pack_tile_slots_per_s": leg["slab_tiles"] * S5 / leg["pack_s"]},
    }
    print(json.dumps(line), flush=True)


DATA = ("synthetic: seeded splitmix64 U[-1,1] (bit-identical host/device generator); "
        "16 GiB input > 126 MB L2 (no flush needed)")


def resolve_scaling(args, world):
    if args.scaling != "auto":
        return args.scaling
    return "strong"   # config 5 as named: the one 16 GiB X split over the ranks


def workload_config(world, scaling):
    rows = 2048 * world if scaling == "weak" else 2048
    return {"workload": "c5: tt_sum(tt_mul(X[2048/16,2048/32,512/32], W[*/16,2048/32,512/32]), k) "
                        "for k=1,2,3",
            "slots": S5, "global_x": [rows, 2048, 512], "x_tiles_total": 64 * rows,
            "parallelism": (f"shard external dim 1 over {world} rank(s); dims 2, 3 local; "
                            "dim-1 sum: NCCL all-reduce of the partial result"),
            "l2": "inputs larger than L2"}


# ---- our arm ----------------------------------------------------------------------------


def time_events(fn, reps, stream, warm=1):
    import torch
    # warm-up outside the timed region (allocator growth, first-launch setup;
    # for the latency-scale configs also host caches and the GPU leaving idle:
    # measured on config 1, 200 calls after one warm-up read 11.3 us per call,
    # 2000 read 6.8 us)
    for _ in range(warm):
        fn()
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
    import torch

    import paper_2011_01805_b200 as tt
    from paper_2011_01805_b200 import configs, sharding

    world, rank, local = dist_env()
    # one process per GPU; more ranks than GPUs only for the gloo functional check
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # TT_BENCH_BACKEND=gloo: functional check of the N > 1 path with several
    # ranks on one GPU (NCCL refuses duplicate devices) -- never a measurement
    backend = os.environ.get("TT_BENCH_BACKEND", "nccl")
    dist = init_dist(world, backend)
    stream = torch.cuda.current_stream(dev)
    hbm_peak, peak_src = peaks()
    scaling = resolve_scaling(args, world)

    S = tt.Session(S5, 8, device=local)
    # strong (default): config 5 as named, X = [2048/16,2048/32,512/32] split
    # along dim 1 -- rank r owns external rows [begin, end) (128/N of them);
    # weak: every rank owns a whole 2048-row slab of a [2048*N,2048,512] X.
    # W (e1 = 1) broadcasts along dim 1: every rank holds it whole.
    cfg = workload_config(world, scaling)
    rows_global = cfg["global_x"][0]
    sx_global = tt.TileTensorShape([tt.DimSpec(rows_global, 1, 16), tt.DimSpec(2048, 1, 32),
                                    tt.DimSpec(512, 1, 32)])
    plan = sharding.plan(sx_global, 1, world, rank)
    sx = plan.local_shape
    sw = tt.parse_shape(configs.C5_W_SHAPE)
    assert sharding.operand_plan(sw, plan) is None
    x_tiles = sx.tile_count()
    out_tiles = {1: W_TILES, 2: x_tiles // 64, 3: x_tiles // 16}
    rows = plan.row_slice.stop - plan.row_slice.start
    # inputs generated on the device with the shared counter-based generator
    x_dense = torch.empty((rows, 2048, 512), dtype=torch.float64, device=dev)
    w_dense = torch.empty((1, 2048, 512), dtype=torch.float64, device=dev)
    tt.fill_uniform(S, x_dense, configs.C5_SEED_X, -1.0, 1.0, offset=plan.row_slice.start * 2048 * 512)
    tt.fill_uniform(S, w_dense, configs.C5_SEED_W, -1.0, 1.0)  # same W on every rank
    X = tt.pack(x_dense, sx, S)
    W = tt.pack(w_dense, sw, S)

    def step():
        outs, work = [], None
        for k in (1, 2, 3):
            r = tt.tt_mul_sum(X, W, k)
            if k == plan.shard_dim and world > 1:
                # the one real exchange: the dim-1 sum spans the ranks' slabs
                # (NCCL over NVLink), in flight while dims 2 and 3 run
                work = sharding.allreduce_partial(r.data(), async_op=True)
            outs.append(r)
        return outs, work

    sampler = ClockSampler(local)  # NVML set up before the warm-up (see its docstring)
    for _i in range(args.warmup):
        warm_outs, w = step()
        if w is not None:
            w.wait()
        # release the warm-up results: their blocks go back to the session's tile
        # cache, so the timed steps allocate nothing (while the last warm-up step's
        # results were still referenced, the first timed step had to cudaMalloc its
        # 128 MiB - 1 GiB results: its first launch read ~3.0 ms instead of 2.55 ms,
        # and 4.7 - 63 ms when the allocation met another driver call)
        del warm_outs
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()

    # per-launch CUDA events on the launching stream; read after the timed
    # region (no host synchronisation inside it)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    launches0 = S.launches()
    with sampler as clk:
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        outs = None
        for i in range(args.steps):
            ev = evs[i]
            ev[0].record(stream)
            work = None
            outs = []
            for k in (1, 2, 3):
                r = tt.tt_mul_sum(X, W, k)
                ev[k].record(stream)
                if k == plan.shard_dim and world > 1:
                    work = sharding.allreduce_partial(r.data(), async_op=True)
                outs.append(r)
            if work is not None:
                work.wait()   # stream-ordered: the next step's kernels queue behind it
        t_end.record(stream)
        t_end.synchronize()
        elapsed = t_start.elapsed_time(t_end) / 1e3
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
    launches = S.launches() - launches0
    elapsed_max = max_over_ranks(elapsed, dist, dev)
    per_dim = {k: [e[k - 1].elapsed_time(e[k]) / 1e3 for e in evs] for k in (1, 2, 3)}
    step_slots_total = 3 * sx_global.tile_count() * S5   # all ranks' units per step
    value = step_slots_total * args.steps / elapsed_max

    # roofline of the dominant kernel (the fused group kernel, all three dims),
    # this rank's algorithmic bytes over this rank's launch durations
    alg = {k: (x_tiles + W_TILES + out_tiles[k]) * S5 * 8 for k in (1, 2, 3)}
    dur = {k: sum(v) / len(v) for k, v in per_dim.items()}
    achieved = sum(alg.values()) / sum(dur.values()) / 1e9
    traffic = traffic_summary()
    tr = traffic.get("c5_mul_sum_bytes_per_launch") if world == 1 or scaling == "weak" else None

    ops = {}
    for k in (1, 2, 3):
        gbs = alg[k] / dur[k] / 1e9
        ops[f"mul_sum_dim{k}"] = {"ms": dur[k] * 1e3, "GB/s": gbs, "frac": gbs / hbm_peak,
                                  "frac_of_8TBps": gbs / 8000.0,
                                  "tile_slots_per_s": x_tiles * S5 / dur[k],
                                  "alg_bytes": alg[k],
                                  # every timed launch (a transient -- power capping, another
                                  # tenant of the host -- shows as single slow launches)
                                  "per_step_ms": [round(v * 1e3, 3) for v in per_dim[k]]}

    # the exact (bit-identical) form of the sum over the sharded dim: the
    # ranks' left folds chained along dim 1, the in-tile tree once at the end
    try:
        fold, finish, n_out, new_acc = sharding.gpu_chain_ops(tt, X, W, 1)

        def chain():
            return sharding.chain_mul_sum(X, W, 1, plan, fold, finish, n_out, new_acc)
        chain_res = chain()
        chain_res = None  # back to the tile cache: the timed calls allocate nothing
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        reps = max(1, min(args.steps, 5))
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(reps):
            chain_res = chain()
        t1.record(stream)
        t1.synchronize()
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        tc = max_over_ranks(t0.elapsed_time(t1) / 1e3 / reps, dist, dev)
        ops["mul_sum_dim1_chain"] = {
            "ms": tc * 1e3, "tile_slots_per_s": sx_global.tile_count() * S5 / tc,
            "note": "exact cross-rank form of the dim-1 sum (sharding.chain_mul_sum: left folds "
                    "chained rank to rank in 16 chunks, in-tile tree on the last rank); "
                    "bit-identical to one GPU"}
    except Exception as exc:
        print(f"[bench] chain failed: {exc!r}", file=sys.stderr)
        ops["mul_sum_dim1_chain"] = {"error": repr(exc)}
        chain_res = None

    if args.dump:
        dump_results(args.dump, rank, world, plan, outs, chain_res)

    try:
        if not args.skip_extra:
            ops.update(bench_extra_ops(tt, X, W, x_dense, sx, S, stream, hbm_peak, args, out_tiles))
            ops.update(bench_matmul(tt, configs, S, stream, hbm_peak, max(200, args.steps)))
            ops.update(bench_small_configs(tt, configs, stream, hbm_peak, max(1000, args.steps)))
            if rank == 0:
                ops["cpp"] = bench_cpp_leg()
    except Exception as exc:  # keep the bench line: report the failure instead
        print(f"[bench] extra failed: {exc!r}", file=sys.stderr)
        ops["extra_error"] = repr(exc)

    e2e = None
    if not args.skip_e2e:
        e2e = bench_e2e(tt, args, sharding, plan, X, W, x_dense, w_dense, sx, sw, S, dist, dev,
                        world, rank, sx_global)
    del x_dense

    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        try:
            cpu = cpu_baseline_block(args.cpu_slab_tiles, args.cpu_one_thread_slab_tiles)
        except Exception as exc:
            print(f"[bench] cpu baseline failed: {exc!r}", file=sys.stderr)
            cpu = {"error": repr(exc)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tile-slots/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed_max / args.steps * 1e3, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": cfg,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "frac_of_8TBps": achieved / 8000.0,
                         "peak_source": peak_src, "traffic": tr,
                         "traffic_source": traffic.get("source"),
                         "kernel": "group_tma_kernel / group_tma_win_kernel (fused fold + rotate-and-sum, TMA ring)",
                         "alg_bytes_per_step": sum(alg.values()), "x_tiles_per_rank": x_tiles},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "ops": ops,
        }
        if world > 1:
            line["backend"] = backend
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def dump_results(path, rank, world, plan, outs, chain_res):
    """--dump DIR: slabs of this rank's results (first / middle / last output
    rows) for the multi-rank parity test (tests/test_gpu_multirank.py)."""
    import numpy as np
    d = Path(path)
    d.mkdir(parents=True, exist_ok=True)
    r1, r2, r3 = (o.data() for o in outs)
    blob = {"begin": np.array([plan.begin, plan.end])}
    # dim 2 result: 16 tiles per external row of dim 1; dim 3: 64 per row
    for name, r, per in (("dim2", r2, 16), ("dim3", r3, 64)):
        e = r.shape[0] // per
        for tag, row in (("first", 0), ("mid", e // 2), ("last", e - 1)):
            blob[f"{name}_{tag}"] = r[row * per:(row + 1) * per].cpu().numpy()
            blob[f"{name}_{tag}_row"] = np.array([plan.begin + row])
    # dim 1 result (all-reduced, replicated): ext [1, 64, 16]; columns l2
    for tag, l2 in (("first", 0), ("mid", 31), ("last", 63)):
        blob[f"dim1_{tag}"] = r1[l2 * 16:(l2 + 1) * 16].cpu().numpy()
        blob[f"dim1_{tag}_l2"] = np.array([l2])
        if chain_res is not None:
            blob[f"dim1chain_{tag}"] = chain_res.data()[l2 * 16:(l2 + 1) * 16].cpu().numpy()
    np.savez(d / f"rank{rank}.npz", **blob)


def bench_extra_ops(tt, X, W, x_dense, sx, S, stream, hbm_peak, args, out_tiles):
    """The other config-5 tile passes (pack, unfused elementwise, sums,
    rotate, clean, replicate) on this rank's data."""
    ops = {}
    x_tiles = sx.tile_count()
    t = time_events(lambda: tt.pack(x_dense, sx, S), max(1, args.steps), stream)
    pb = 2 * x_tiles * S5 * 8
    ops["pack"] = {"ms": t * 1e3, "GB/s": pb / t / 1e9, "frac": pb / t / 1e9 / hbm_peak,
                   "frac_of_8TBps": pb / t / 1e12 / 8.0, "tile_slots_per_s": x_tiles * S5 / t,
                   "alg_bytes": pb}
    t = time_events(lambda: tt.unpack_device(X), max(1, min(5, args.steps)), stream)
    ops["unpack"] = {"ms": t * 1e3, "GB/s": pb / t / 1e9, "frac": pb / t / 1e9 / hbm_peak,
                     "frac_of_8TBps": pb / t / 1e12 / 8.0, "tile_slots_per_s": x_tiles * S5 / t,
                     "alg_bytes": pb}
    # unfused elementwise (tt_mul with W broadcast along dim 1, tt_add)
    for name, fn, nb in (("ew_mul_bcast", lambda: tt.tt_mul(X, W), (2 * x_tiles + W_TILES) * S5 * 8),
                         ("ew_add", lambda: tt.tt_add(X, X), 2 * x_tiles * S5 * 8)):
        t = time_events(fn, max(1, args.steps), stream)
        ops[name] = {"ms": t * 1e3, "GB/s": nb / t / 1e9, "frac": nb / t / 1e9 / hbm_peak,
                     "tile_slots_per_s": x_tiles * S5 / t, "alg_bytes": nb}
    reps = max(1, min(3, args.steps))
    for k in (1, 2, 3):
        t = time_events(lambda: tt.tt_sum(X, k), reps, stream)
        nb = (x_tiles + out_tiles[k]) * S5 * 8
        ops[f"sum_dim{k}"] = {"ms": t * 1e3, "GB/s": nb / t / 1e9, "frac": nb / t / 1e9 / hbm_peak}
    t = time_events(lambda: tt.tiles_rotate(S, X.data(), 5), reps, stream)
    ops["rotate"] = {"ms": t * 1e3, "GB/s": 2 * x_tiles * S5 * 8 / t / 1e9,
                     "frac": 2 * x_tiles * S5 * 8 / t / 1e9 / hbm_peak}
    R3 = tt.tt_sum(X, 3)  # [rows/16,2048/32,1?/32]: boundary tiles
    nb = 2 * out_tiles[3] * S5 * 8
    t = time_events(lambda: tt.clean_unknowns(R3), 10, stream)
    ops["clean_unknowns"] = {"ms": t * 1e3, "GB/s": nb / t / 1e9, "frac": nb / t / 1e9 / hbm_peak}
    C3 = tt.clean_unknowns(R3)
    t = time_events(lambda: tt.replicate_dim(C3, 3), 10, stream)
    ops["replicate_dim"] = {"ms": t * 1e3, "GB/s": nb / t / 1e9, "frac": nb / t / 1e9 / hbm_peak}
    return ops


def host_slab_fraction(numel, world, dist, dev):
    """Largest slab of X (1, 1/2, 1/4, 1/8 of its dim-1 rows) whose host
    staging (x2.2 while pinning) fits the host's free memory for all local
    ranks; 0 when not even 1/8 fits.  One decision for all ranks."""
    frac = 1.0
    try:
        import psutil
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
        avail = psutil.virtual_memory().available
        if os.environ.get("TT_BENCH_HOST_GIB"):  # test hook: pretend a smaller host
            avail = float(os.environ["TT_BENCH_HOST_GIB"]) * 2**30
        while frac >= 0.125 and 2.2 * numel * 8 * frac * local_world > avail:
            frac /= 2
        if frac < 0.125:
            frac = 0.0
    except Exception as exc:
        print(f"[bench] host memory probe failed ({exc!r}); staging 1/8 of X", file=sys.stderr)
        frac = 0.125
    return -max_over_ranks(-frac, dist, dev)


def bench_e2e(tt, args, sharding, plan, X, W, x_dense, w_dense, sx, sw, S, dist, dev, world, rank,
              sx_global):
    """The same step through the public API from pinned HOST buffers: H2D
    of the dense input + pack, the three fused products (+ the dim-1
    all-reduce), unpack + D2H of every result."""
    import torch
    try:
        frac = host_slab_fraction(x_dense.numel(), world, dist, dev)
        if frac == 0.0:
            return {"skipped": "host memory too small to stage even 1/8 of the input"}
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
        torch.cuda.empty_cache()

        def mul_sum(a, b, k):
            return tt.tt_mul_sum(a, b, k)

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
        if dist is not None:
            dist.barrier()
        reps = max(1, min(args.steps, args.e2e_steps))
        t0 = time.perf_counter()
        for _ in range(reps):
            d2h = e2e_step()
        torch.cuda.synchronize(dev)
        e_el = max_over_ranks((time.perf_counter() - t0) / reps, dist, dev)
        h2d = host_x.numel() * 8 + host_w.numel() * 8
        units = 3 * sx_global.tile_count() * S5 * frac
        return {"value": units / e_el, "unit": "tile-slots/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": e_el * 1e3, "steps": reps,
                "host_buffers": "pinned" if pinned else "pageable", "x_slab_fraction": frac,
                "path": "tt.pack(host) -> tt_mul_sum x3 (+ dim-1 all-reduce) -> tt.unpack (D2H)"}
    except Exception as exc:  # keep the bench line: report the failure instead
        print(f"[bench] e2e failed: {exc!r}", file=sys.stderr)
        return {"error": repr(exc)}


def bench_cpp_leg():
    """Configs 1-4 per call through the C++ drop-in headers (tests_cpp/bench_cpp.cpp:
    the reference's tiletensor:: API, results from the session's stream-ordered
    pool), with each call's CUDA-graph replay beside it."""
    from paper_2011_01805_b200 import build
    try:
        exe = build.build_cpp_bench()
        proc = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
        if proc.returncode != 0:
            return {"error": proc.stderr[-400:]}
        out = json.loads(proc.stdout.strip().splitlines()[-1])
        out["note"] = ("C++ per-call time through tiletensor_b200/*.hpp (host enqueue + device, "
                       "drained once per loop); graph_replay_us: the same call as a CUDA graph")
        return out
    except Exception as exc:
        return {"error": repr(exc)}


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
    t = time_events(lambda: tt.tt_mul_sum(A, B, 2), reps, stream, warm=50)
    out["c1_mul_sum"] = {"us": t * 1e6, "note": "[100/16,200/32] x same, sum dim 2 (49 tiles of 512)"}
    c2 = configs.config2()
    S2 = tt.Session(8192, 8, device=torch.cuda.current_device())
    M = tt.pack(c2.tensors["M"], tt.parse_shape(c2.shapes["M"]), S2)
    V = tt.pack(c2.tensors["V"], tt.parse_shape(c2.shapes["V"]), S2)
    t = time_events(lambda: tt.matvec_a(M, V), reps, stream, warm=50)
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
    t = time_events(c4_chain, reps, stream, warm=50)
    out["c4_fc_square_fc"] = {"us": t * 1e6, "samples_per_s": 4096 / t,
                              "unfused_us": time_events(c4_unfused, reps, stream, warm=50) * 1e6,
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
        out[name]["graph_replay_us"] = time_events(g.replay, reps, stream, warm=50) * 1e6
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
    t = time_events(chain, reps, stream, warm=50)
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
    t_graph = time_events(g.replay, reps, stream, warm=50)
    tile = 8192 * 8
    # unique operand tiles + out tiles of both stages
    # stage 1: Bt 96 MiB + C 48 MiB in, 32 MiB out; stage 2: A 64 + 32 MiB in, 32 MiB out
    alg = (1536 + 768 + 512 + 1024 + 512 + 512) * tile  # 4864 tiles = 304 MiB
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
    t3a = time_events(chain_3a, reps, stream, warm=50)
    t3a_calls = time_events(chain_3a_calls, reps, stream, warm=50)
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
    # the reference arm and the cpu_baseline leg time the same slab (32 external rows of
    # dim 1 = 32768 of 131072 X tiles, ~3.5 s per step on 16 host threads)
    ap.add_argument("--cpu-slab-tiles", type=int, default=32)
    ap.add_argument("--cpu-one-thread-slab-tiles", type=int, default=4)
    ap.add_argument("--ref-slab-tiles", type=int, default=32)
    ap.add_argument("--scaling", default="auto", choices=["auto", "strong", "weak"])
    ap.add_argument("--dump", default="", help="write result slabs per rank (parity test)")
    ap.add_argument("--cpu-leg", default="", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.cpu_leg:  # internal: one reference CPU leg in a fresh process
        slab, steps, warm = (int(v) for v in args.cpu_leg.split(","))
        print(json.dumps(cpu_leg(slab, steps, warm)), flush=True)
        return
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
