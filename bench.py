"""Benchmark of the B200 stochastic Barnes-Hut hot path (BASELINE.json metric).

Workload (BASELINE.json configs[3]): electrical (Coulomb)
potential of 2^22 area-uniform samples of one compact tilted torus
(torus(0.25, 0.06) rotated 0.7 rad about x, shifted (0.1, 0.05, -0.1); masses
1/M, seed 7) on a 1000 x 1000 slice plane at z = 0.03.  A step is one
stochastic S=1 evaluation of all 10^6 queries (FP32 terms / FP64
accumulation, tree prebuilt and resident) with the paper's GPU recipe for
the RNG streams (``--streams warp``, default: 32 shuffled queries share one
stream); the reference's per-query streams
(``--streams query``, draw-for-draw parity) are timed and error-matched beside
it under ``other_streams``.  Reported beside the step:

* median relative error of S=1 vs brute force (GPU brute force, FP64 accum.)
* the GPU deterministic BH (same API, f32) beta sweep, log-log interpolated
  to S=1's median error -> matched BH time and the speed-up
* e2e: the same step through the public API (``evaluate_field``) from pinned
  host queries to host results, copies inside the timed region
* roofline of the stochastic kernel, cpu_baseline (the C oracle port on the
  host cores, bounded sample), clocks sampled during the timed region.

``--impl reference`` times the reference algorithm's CPU implementation (the
C oracle port, all host threads) on the same workload, bounded sample/step.
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

N_SIDE = 1000
M_SOURCES = 2 ** 22
METRIC = "queries/s at matched median rel. error vs brute force; speedup over det. BH"
BETAS = (1.0, 1.5, 2.0, 3.0, 4.0, 6.0, 8.0, 10.0, 12.0, 16.0)
L2_READ_GBS = 16800.0  # L2-resident read bandwidth, measured by tools/micro/l2bw.cu


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def workload(m=M_SOURCES, side=N_SIDE):
    from paper_2506_02219_b200 import scenes as S
    from paper_2506_02219_b200.types import KernelSpec
    v, f = S.torus(0.25, 0.06)
    v = S.rotate_x(v, 0.7) + np.array([0.1, 0.05, -0.1])
    src = S.sample_mesh_surface(v, f, m, seed=7, kernel_kind="coulomb")
    qs = S.make_queries(S.GridSpec("slice_plane", resolution=(side, side), origin=(0.0, 0.0, 0.03)))
    return src, qs, KernelSpec("coulomb")


STREAM_NOTES = {
    "warp": ("warp-shared RNG streams, the paper's GPU recipe (PAPER.md:323, 392): 32 queries in a "
             "seeded shuffled order share the index and roulette streams (rng_sharing='warp')"),
    "query": ("per-query RNG streams, the reference's (rng.py:39-47, _core.py:219; "
              "rng_sharing='query', draw-for-draw parity)"),
}


def config_block(streams="warp"):
    return {"workload": "C4: coulomb, 2^22 tilted-torus surface samples, 1000^2 slice plane z=0.03",
            "sources": M_SOURCES, "queries": N_SIDE * N_SIDE, "method": "stochastic S=1 paper_ratio",
            "rng_streams": STREAM_NOTES[streams],
            "branching": {"stochastic": 4, "barnes_hut": 2}, "precision": "f32 terms, f64 accumulation",
            "l2": ("no flush in the timed loop (tree records ~0.3 GB > L2); the same steps "
                   "with L2 flushed before each (256 MB write) are reported as "
                   "l2_flushed_ms_per_step (within 1 %)"),
            "parallelism": "query slabs (replica tree per rank)"}


_NVML_POLLER = r"""
import sys, time
import pynvml as nv
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
print("max", nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM), flush=True)
w = sys.stdout.write
while True:
    try:
        w("%d %d %d\n" % (time.time_ns(), nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                           nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
    except Exception:
        break
    time.sleep(0.001)
"""


class Clocks:
    """SM clock + throttle-reason sampling DURING the timed region.

    NVML is polled every ~1 ms by a separate Python process (the timed region of
    a default run is only tens of ms, too short for ``nvidia-smi -lms``); its
    timestamped samples are kept when they fall between the moments ``active``
    is switched on and off.  A separate process keeps the poller off this
    process's GIL, so it never delays the enqueue of the timed steps.
    ``nvidia-smi`` runs beside it as the recipe's clocks line and is used when
    NVML is missing.
    """

    REASONS = (("hw_slowdown", 0x8), ("sw_power_cap", 0x4), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []  # (sm_mhz, reasons bitmask)
        self.sm_max = None
        self.smi_lines = []
        self._poller = None
        self._proc = None
        self._windows = []  # [t_on, t_off) in time.time_ns()
        self._active = False

    @property
    def active(self):
        return self._active

    @active.setter
    def active(self, on):  # set only while the timed region runs
        if on and not self._active:
            self._windows.append([time.time_ns(), None])
        elif not on and self._active:
            self._windows[-1][1] = time.time_ns()
        self._active = bool(on)

    def __enter__(self):
        try:
            self._poller = subprocess.Popen([sys.executable, "-c", _NVML_POLLER, str(self.gpu)],
                                            stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                            text=True)
            first = self._poller.stdout.readline().split()  # running before the region starts
            if len(first) == 2 and first[0] == "max":
                self.sm_max = int(first[1])
            else:
                self._poller.kill()
                self._poller = None
        except OSError:
            self._poller = None
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            # its start-up queries the driver heavily: let it reach its polling loop
            # (first line) before the timed region begins
            first = self._proc.stdout.readline()
            if first.strip():
                self.smi_lines.append(first.strip())
        except OSError:
            self._proc = None
        return self

    def __exit__(self, *exc):
        self.active = False
        for proc in (self._poller, self._proc):
            if proc is None:
                continue
            proc.terminate()
            try:
                out, _ = proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                proc.kill()
                out = ""
            if proc is self._proc:
                self.smi_lines += [ln for ln in out.splitlines() if ln.strip()]
                continue
            for ln in out.splitlines():
                parts = ln.split()
                if len(parts) != 3:
                    continue
                t = int(parts[0])
                if any(a <= t < (b if b is not None else t + 1) for a, b in self._windows):
                    self.samples.append((int(parts[1]), int(parts[2])))

    def summary(self):
        sm, mask = [], 0
        if self.samples:
            sm = [float(s) for s, _ in self.samples]
            for _, r in self.samples:
                mask |= int(r)
            reasons = sorted(nm for nm, bit in self.REASONS if mask & bit)
            src = "nvml (1 ms poll by a separate process during the timed region)"
            mx = float(self.sm_max) if self.sm_max else None
        else:
            reasons, mx = set(), None
            for ln in self.smi_lines:
                parts = [p.strip() for p in ln.split(",")]
                try:
                    sm.append(float(parts[0]))
                    mx = max(mx or 0.0, float(parts[1]))
                except (ValueError, IndexError):
                    continue
                for (nm, _), val in zip(self.REASONS, parts[2:6]):
                    if val.lower() == "active":
                        reasons.add(nm)
            reasons = sorted(reasons)
            src = "nvidia-smi -lms 50"
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "sm_mhz_min": float(min(sm)) if sm else None, "reasons": reasons,
                "samples": len(sm), "source": src}


class Gate:
    """Holds the current stream behind a one-thread gate kernel (fsb_gate) while the
    host enqueues a timed region, then opens it, so the region's steps run back to
    back on the GPU however long the host takes to enqueue them.  Used where every
    step is stream-ordered (one rank, or NCCL); the kernel gives up after ~2 s, so a
    host-side synchronisation inside a step cannot deadlock it."""

    def __init__(self, enabled=True):
        import torch
        # (FSB_BENCH_NO_GATE=1 under a profiler that serialises launches, where the
        # gate could only time out)
        self.enabled = enabled and not os.environ.get("FSB_BENCH_NO_GATE")
        self.flag = torch.zeros(1, dtype=torch.int32, pin_memory=True) if enabled else None

    def close(self):
        if self.enabled:
            import ctypes as C
            from paper_2506_02219_b200 import _device as dev, _lib
            self.flag[0] = 0
            _lib.check(_lib.lib().fsb_gate(C.c_void_p(self.flag.data_ptr()), 4_000_000_000,
                                           C.c_void_p(dev.stream_ptr())))

    def open(self):
        if self.enabled:
            self.flag[0] = 1


class quiet:
    """No garbage-collector pause inside a timed measurement."""

    def __enter__(self):
        self.was = gc.isenabled()
        gc.disable()

    def __exit__(self, *exc):
        if self.was:
            gc.enable()


def median_rel(est, ref):
    return float(np.median(np.abs(est - ref) / np.abs(ref)))


def loglog_interp(points, target):
    """(err, ms) points; time at `target` error by log-log linear interpolation."""
    pts = sorted(points)  # ascending error
    for (e0, t0), (e1, t1) in zip(pts, pts[1:]):
        if e0 <= target <= e1 and e0 > 0 and e1 > e0:
            w = (math.log(target) - math.log(e0)) / (math.log(e1) - math.log(e0))
            return math.exp(math.log(t0) + w * (math.log(t1) - math.log(t0)))
    return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


C5_SOURCES = 2 ** 24
C5_QUERIES = 10 ** 7


def workload_c5(m=C5_SOURCES, n=C5_QUERIES):
    """BASELINE configs[4] / SURVEY 8(d) C5: the C4 generator at 2^24 samples,
    default_rng(5).uniform(-1, 1, (10^7, 3)) queries."""
    from paper_2506_02219_b200 import scenes as S
    from paper_2506_02219_b200.types import KernelSpec, QuerySet
    v, f = S.torus(0.25, 0.06)
    v = S.rotate_x(v, 0.7) + np.array([0.1, 0.05, -0.1])
    src = S.sample_mesh_surface(v, f, m, seed=7, kernel_kind="coulomb")
    qs = QuerySet(np.random.default_rng(5).uniform(-1, 1, (n, 3)))
    return src, qs, KernelSpec("coulomb")


def c5_config(world):
    return {"workload": "C5: coulomb, 2^24 tilted-torus surface samples, 10^7 default_rng(5) "
                        "uniform [-1,1]^3 queries (BASELINE configs[4])",
            "sources": C5_SOURCES, "queries": C5_QUERIES, "method": "stochastic S=1 paper_ratio",
            "rng_streams": STREAM_NOTES["warp"], "branching": {"stochastic": 4, "barnes_hut": 2},
            "precision": "f32 terms, f64 accumulation",
            "l2": "inputs larger than L2 (tree ~0.9 GB, queries 240 MB); no flush",
            "parallelism": (f"strong scaling: {world} rank(s), query slabs on 2^16-position "
                            f"shuffle windows (query_offset = slab start), replica tree per rank, "
                            f"all_gather of the field inside every step (FP32 values, "
                            f"widened to FP64 after the collective: the same bits)")}


def run_c5(args, world, rank, local, anchor=False):
    """C5 strong scaling: a fixed 10^7 queries split into `world` slabs;
    every step evaluates this rank's slab (device-resident queries) and all-gathers
    the field (FP64 values, NCCL) -- both inside the timed region, max over ranks.
    Returns the JSON line (rank 0) or, with anchor=True at N=1, a compact object
    for the C4 line."""
    import torch
    import torch.distributed as dist
    import paper_2506_02219_b200 as fs
    from paper_2506_02219_b200 import _device as dev
    from paper_2506_02219_b200.estimators import evaluate_field_device
    from paper_2506_02219_b200.sharding import SHUFFLE_WINDOW, broadcast_tree, slab

    t0 = time.perf_counter()
    src, qs, kern = workload_c5()
    gen_s = time.perf_counter() - t0
    n = len(qs)
    a, b = slab(n, rank, world, SHUFFLE_WINDOW)
    widths = [slab(n, r, world, SHUFFLE_WINDOW)[1] - slab(n, r, world, SHUFFLE_WINDOW)[0]
              for r in range(world)]
    width = max(widths)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    barrier()
    t0 = time.perf_counter()
    tree = fs.build_tree(src, 4)
    torch.cuda.synchronize()
    build_ms = (time.perf_counter() - t0) * 1e3
    tmp = fs.build_tree(src, 4)  # (grows the memory pool for a second tree; freed)
    del tmp
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tmp = fs.build_tree(src, 4)
    e1.record()
    torch.cuda.synchronize()
    build_warm_ms = e0.elapsed_time(e1)
    del tmp
    tree_dist = None
    if world > 1:
        barrier()
        t0 = time.perf_counter()
        bt = broadcast_tree(src if rank == 0 else None, 4, src=0)
        barrier()
        bcast_ms = (time.perf_counter() - t0) * 1e3
        del bt
        tt = torch.tensor([build_ms, build_warm_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        tree_dist = {"replica_build_ms_max_over_ranks": float(tt[0]),
                     "replica_build_warm_ms_max_over_ranks": float(tt[1]),
                     "build_on_rank0_and_broadcast_ms": bcast_ms,
                     "backend": dist.get_backend(),
                     "used": "replica (deterministic per-rank build, no collective)"}
    cfg = fs.EstimatorConfig("stochastic", samples_per_subdomain=1, seed=1, precision="f32",
                             rng_sharing="warp")
    q_dev = dev.to_device(qs.positions[a:b])
    # the FP32 path's values are FP32 results widened to FP64: gathered as FP32 (4 B
    # per query) and widened after the collective -- the same bits
    full = torch.empty(world * width, dtype=torch.float32, device="cuda")
    pad = torch.zeros(width, dtype=torch.float32, device="cuda")

    def step():
        r = evaluate_field_device(cfg, src, kern, q_dev, tree, query_offset=a)
        if world == 1:
            return r.values
        pad[: b - a].copy_(r.values)  # exact: the values are FP32 numbers
        if dist.get_backend() == "nccl":
            dist.all_gather_into_tensor(full, pad)
        else:  # (gloo: several ranks sharing one GPU in tests)
            dist.all_gather(list(full.split(width)), pad)
        return full.double()

    for _ in range(args.warmup):
        step()
    barrier()
    launches = _count_launches(step)
    gate = Gate(world == 1 or dist.get_backend() == "nccl")
    with Clocks(local) as clk:
        barrier()
        ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # the start event, the K steps and the end event are enqueued behind a gate
        # that opens once they all are: a host-side stall while enqueueing cannot
        # idle the GPU inside the timed region (which holds exactly K steps)
        gate.close()  # the region runs once every step is enqueued
        gc.disable()  # no collector pause while the steps are enqueued
        ev_a.record()
        clk.active = True
        marks, host_t = [], [time.perf_counter()]
        for _ in range(args.steps):
            res = step()
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            marks.append(e)
            host_t.append(time.perf_counter())
        ev_b.record()
        gate.open()
        barrier()
        gc.enable()
        clk.active = False
    step_ms = ev_a.elapsed_time(ev_b) / args.steps
    # per-step GPU intervals and host enqueue times of the timed loop (diagnostic:
    # a gap in the GPU intervals with a long host interval is a host-side stall)
    gpu_iv = [ev_a.elapsed_time(marks[0])] + [marks[i - 1].elapsed_time(marks[i])
                                               for i in range(1, len(marks))]
    host_iv = [1e3 * (host_t[i + 1] - host_t[i]) for i in range(len(host_t) - 1)]
    step_spread = {"gpu_ms_min": min(gpu_iv), "gpu_ms_median": float(np.median(gpu_iv)),
                   "gpu_ms_max": max(gpu_iv), "host_enqueue_ms_max": max(host_iv),
                   "host_enqueue_ms_median": float(np.median(host_iv))}
    if world > 1:
        tt = torch.tensor([step_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        step_ms = float(tt.item())
    value = n / (step_ms * 1e-3)
    # the gathered field equals one process evaluating all 10^7 queries (rank 0, untimed)
    same = None
    if rank == 0:
        got = torch.cat([res[r * width: r * width + widths[r]] for r in range(world)])
        if world > 1:
            ref = evaluate_field_device(cfg, src, kern, dev.to_device(qs.positions), tree)
            same = bool(torch.equal(got, ref.values))
        else:
            same = True
        sub = np.linspace(0, n - 1, 65536).astype(np.int64)
        truth = fs.evaluate_field(fs.EstimatorConfig("brute_force", precision="f32"), src, kern,
                                  fs.QuerySet(qs.positions[sub])).values
        err = median_rel(got[torch.as_tensor(sub, device="cuda")].cpu().numpy(), truth)
    # e2e through the public multi-GPU API: host queries in, gathered host field out
    e2e = None
    if not anchor:
        from paper_2506_02219_b200.sharding import evaluate_field_sharded
        host = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
        host.numpy()[:] = qs.positions
        qset = fs.QuerySet(host.numpy())
        if world > 1:
            fn = lambda: evaluate_field_sharded(cfg, src, kern, qset, tree)  # noqa: E731
        else:
            fn = lambda: fs.evaluate_field(cfg, src, kern, qset, tree=tree).values  # noqa: E731
        for _ in range(max(2, args.warmup)):
            fn()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            vals = fn()
        barrier()
        dt = (time.perf_counter() - t0) / args.steps
        if world > 1:
            tt = torch.tensor([dt], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        e2e = {"value": n / dt, "unit": "queries/s", "h2d_bytes_per_step": int((b - a) * 24),
               "d2h_bytes_per_step": int(vals.nbytes), "ms_per_step": dt * 1e3,
               "api": ("paper_2506_02219_b200.sharding.evaluate_field_sharded (host slab in, "
                       "all_gather, host field out)" if world > 1 else
                       "paper_2506_02219_b200.evaluate_field (host numpy in/out)"),
               "bytes_note": "per rank per step (h2d: the rank's slab; d2h: the gathered field)"}
    if anchor:
        return {"workload": c5_config(1)["workload"], "n_gpus": 1, "ms_per_step": step_ms,
                "value": value, "unit": "queries/s", "s1_median_rel_err_65536_subset": err,
                "tree_build_ms": {"first_call": build_ms, "warm": build_warm_ms},
                "scene_generation_s": gen_s,
                "note": "C5 at one GPU: the anchor of the strong-scaling curve that "
                        "bench.py --gpus N (N > 1) measures on C5"}
    out = {"metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
           "step_spread": step_spread,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic (reference mesh generators, fixed seeds)",
           "config": c5_config(world), "clocks": clk.summary(), "e2e": e2e,
           "gathered_equals_single_process": same,
           "tree_build_ms": {"first_call": build_ms, "warm": build_warm_ms}}
    if rank == 0:
        out["accuracy"] = {"s1_median_rel_err": err,
                           "truth": "GPU brute force (FP32 terms, FP64 accumulation) on 65,536 "
                                    "queries spread over the 10^7"}
    if tree_dist is not None:
        out["tree_distribution"] = tree_dist
    if launches is not None:
        out["gpu_launches"] = launches * args.steps
    return out


# ----------------------------------------------------------------- our arm
def run_ours(args):
    import ctypes as C
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # FSB_BENCH_BACKEND=gloo lets several ranks share one GPU (tests of the
    # multi-rank path on a single-GPU box); the default is NCCL, one GPU per rank
    backend = os.environ.get("FSB_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    import paper_2506_02219_b200 as fs
    from paper_2506_02219_b200 import _device as dev
    from paper_2506_02219_b200 import _lib
    from paper_2506_02219_b200.estimators import evaluate_field_device

    wl = args.workload if args.workload != "auto" else ("c4" if world == 1 else "c5")
    if wl == "c5":
        out = run_c5(args, world, rank, local)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        if rank == 0:
            print(json.dumps(out), flush=True)
        return

    L = _lib.lib()
    src, qs, kern = workload()
    n = len(qs)
    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- tree builds (setup, timed separately).  The process's first build is
    # reported in parts: the sources' host->device copy (torch's pageable copy),
    # then the build itself (lazy module loading and memory-pool growth included)
    from paper_2506_02219_b200.octree import device_sources
    t0 = time.perf_counter()
    device_sources(src)
    torch.cuda.synchronize()
    sources_h2d_ms = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    tree4 = fs.build_tree(src, 4)
    torch.cuda.synchronize()
    build4_ms = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    tree2 = fs.build_tree(src, 2)
    torch.cuda.synchronize()
    build2_ms = (time.perf_counter() - t0) * 1e3
    # warm build: the first calls include lazy module loading and the growth of the
    # memory pool (a third tree while two are alive maps new memory), so one more
    # tree is built and freed first and the next build is timed
    tmp = fs.build_tree(src, 4)
    del tmp
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tmp = fs.build_tree(src, 4)
    e1.record()
    torch.cuda.synchronize()
    build4_warm_ms = e0.elapsed_time(e1)
    del tmp

    # N > 1: the alternative tree distribution, built on rank 0 and broadcast (NCCL over
    # NVLink), timed beside the per-rank replica build the step uses
    tree_dist = None
    if world > 1:
        from paper_2506_02219_b200.sharding import broadcast_tree
        barrier()
        t0 = time.perf_counter()
        bt = broadcast_tree(src if rank == 0 else None, 4, src=0)
        barrier()
        bcast_ms = (time.perf_counter() - t0) * 1e3
        del bt
        tt = torch.tensor([build4_ms, build4_warm_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        tree_dist = {"replica_build_ms_max_over_ranks": float(tt[0]),
                     "replica_build_warm_ms_max_over_ranks": float(tt[1]),
                     "build_on_rank0_and_broadcast_ms": bcast_ms,
                     "used": "replica (deterministic per-rank build, no collective)"}
    q_dev = dev.to_device(qs.positions)
    qoff = rank * n  # slab `rank` of a world*n query set: distinct RNG streams per rank
    other = "query" if args.streams == "warp" else "warp"
    cfgs = {m: fs.EstimatorConfig("stochastic", samples_per_subdomain=1, seed=1, precision="f32",
                                  rng_sharing=m) for m in ("warp", "query")}
    cfg_s1 = cfgs[args.streams]

    def step(mode=args.streams):
        return evaluate_field_device(cfgs[mode], src, kern, q_dev, tree4, query_offset=qoff)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # the headline must run the fast FP32 kernel: a silent fallback is reported
    os.environ["FSB_REQUIRE_FAST"] = "1"
    try:
        step()
        fast_path = True
    except Exception as exc:  # pragma: no cover
        log("WARNING: fast stochastic kernel declined:", exc)
        fast_path = False
    finally:
        del os.environ["FSB_REQUIRE_FAST"]
    torch.cuda.synchronize()

    # ---- timed region: K steps, barrier + sync both sides, max over ranks
    gate = Gate(world == 1 or dist.get_backend() == "nccl")
    with Clocks(local) as clk:
        barrier()
        ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # the start event, the K steps and the end event are enqueued behind a gate
        # that opens once they all are: a host-side stall while enqueueing cannot
        # idle the GPU inside the timed region (which holds exactly K steps)
        gate.close()  # the region runs once every step is enqueued
        gc.disable()  # no collector pause while the steps are enqueued
        ev_a.record()
        clk.active = True
        marks, host_t = [], [time.perf_counter()]
        for _ in range(args.steps):
            res = step()
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            marks.append(e)
            host_t.append(time.perf_counter())
        ev_b.record()
        gate.open()
        barrier()
        gc.enable()
        clk.active = False
    # ---- launch count of one step (CUPTI via torch.profiler), after the timed
    # region: a CUPTI session before it could leave work behind
    launches_per_step = None
    try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step()
            torch.cuda.synchronize()
        # our kernels: everything compiled into libfastsum_b200.so (fsb:: and its CUB sorts)
        launches_per_step = sum(1 for e in prof.events()
                                if e.device_type == torch.autograd.DeviceType.CUDA
                                and ("fsb" in e.name or "cub" in e.name.lower()))
    except Exception as exc:  # pragma: no cover
        log("profiler unavailable:", exc)

    step_ms = ev_a.elapsed_time(ev_b) / args.steps
    # per-step GPU intervals and host enqueue times of the timed loop (diagnostic:
    # a gap in the GPU intervals with a long host interval is a host-side stall)
    gpu_iv = [ev_a.elapsed_time(marks[0])] + [marks[i - 1].elapsed_time(marks[i])
                                               for i in range(1, len(marks))]
    host_iv = [1e3 * (host_t[i + 1] - host_t[i]) for i in range(len(host_t) - 1)]
    step_spread = {"gpu_ms_min": min(gpu_iv), "gpu_ms_median": float(np.median(gpu_iv)),
                   "gpu_ms_max": max(gpu_iv), "host_enqueue_ms_max": max(host_iv),
                   "host_enqueue_ms_median": float(np.median(host_iv))}
    # the same steps with L2 flushed before each (a 256 MB write, outside each
    # step's own event pair): reported beside the headline, which runs warm
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    for e0, e1 in evs:
        flush.fill_(1)
        e0.record()
        step()
        e1.record()
    torch.cuda.synchronize()
    cold_ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / args.steps
    del flush
    if world > 1:
        tt = torch.tensor([step_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        step_ms = float(tt.item())
    value = world * n / (step_ms * 1e-3)

    # ---- the stochastic kernel alone (events on the launching stream), for the roofline
    raw = dev.empty(n, torch.float32)
    vis = dev.empty(n, torch.int64)
    h = C.c_void_p(tree4._device_tree().handle)

    def kernel_only():
        if args.streams == "warp":  # k_sto_warp (shuffled order computed in-kernel)
            _lib.check(L.fsb_stochastic_batch_ex(
                h, 0, kern.alpha, kern.distance_floor, 1, C.c_void_p(dev.ptr(q_dev)), n,
                None, 1, 0, 1, qoff, 5, 2, C.c_void_p(dev.ptr(raw)),
                C.c_void_p(dev.ptr(vis)), None, None, sp))
        else:  # k_sto_fast
            _lib.check(L.fsb_stochastic_batch(h, 0, kern.alpha, kern.distance_floor, 1,
                                              C.c_void_p(dev.ptr(q_dev)), n, None, 1, 0, 1, qoff,
                                              C.c_void_p(dev.ptr(raw)), C.c_void_p(dev.ptr(vis)),
                                              None, None, sp))
    kernel_only()
    torch.cuda.synchronize()
    reps = max(3, args.steps)
    with quiet():
        gate.close()
        ev_a.record()
        for _ in range(reps):
            kernel_only()
        ev_b.record()
        gate.open()
        torch.cuda.synchronize()
    kern_ms = ev_a.elapsed_time(ev_b) / reps
    visited_mean = float(vis.double().mean().item())

    # ---- e2e through the public API from pinned host memory (all ranks)
    e2e = _e2e(args, fs, src, kern, qs, tree4, cfg_s1, world, rank)

    out = {"metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
           "step_spread": step_spread,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic (reference mesh generators, fixed seeds)",
           "config": config_block(args.streams), "clocks": clk.summary(), "e2e": e2e,
           "fast_kernel": fast_path,
           "l2_flushed_ms_per_step": cold_ms}
    if tree_dist is not None:
        out["tree_distribution"] = tree_dist
    if launches_per_step is not None:
        out["gpu_launches"] = launches_per_step * args.steps

    # ---- accuracy and the matched-error BH comparison (rank 0 only)
    if rank == 0:
        truth = dev.empty(n, torch.float64)
        pts_d, ms_d = dev.to_device(src.positions), dev.to_device(src.masses)
        t0 = time.perf_counter()
        _lib.check(L.fsb_brute_force_f32acc64(0, kern.alpha, kern.distance_floor,
                                               C.c_void_p(dev.ptr(pts_d)), C.c_void_p(dev.ptr(ms_d)),
                                               len(src), 1, C.c_void_p(dev.ptr(q_dev)), n,
                                               C.c_void_p(dev.ptr(truth)), sp))
        torch.cuda.synchronize()
        brute_ms = (time.perf_counter() - t0) * 1e3
        truth_h = truth.cpu().numpy()
        s1 = res.values.cpu().numpy()
        err_s1 = median_rel(s1, truth_h)
        # the other stream mode, timed the same way (device-resident steps)
        for _ in range(args.warmup):
            r_o = step(other)
        torch.cuda.synchronize()
        with quiet():
            gate.close()
            ev_a.record()
            for _ in range(args.steps):
                r_o = step(other)
            ev_b.record()
            gate.open()
            torch.cuda.synchronize()
        other_ms = ev_a.elapsed_time(ev_b) / args.steps
        err_other = median_rel(r_o.values.cpu().numpy(), truth_h)
        sweep = []
        for beta in BETAS:
            cfg = fs.EstimatorConfig("barnes_hut", beta=beta, precision="f32")
            t_w = time.perf_counter()
            for _ in range(2 if beta == BETAS[0] else 1):  # the first call packs the BH records
                r = evaluate_field_device(cfg, src, kern, q_dev, tree2)
            torch.cuda.synchronize()
            t_w = (time.perf_counter() - t_w) * 1e3
            with quiet():
                ev_a.record()
                r = evaluate_field_device(cfg, src, kern, q_dev, tree2)
                ev_b.record()
                torch.cuda.synchronize()
            ms = ev_a.elapsed_time(ev_b)
            if os.environ.get("FSB_BENCH_DEBUG"):
                log(f"  (warm-up call {t_w:.2f} ms)")
            err = median_rel(r.values.cpu().numpy(), truth_h)
            sweep.append({"beta": beta, "ms": ms, "median_rel_err": err,
                          "visited_mean": float(r.visited.double().mean().item())})
            log(f"BH beta={beta}: {ms:.2f} ms, median rel err {err:.3e}")
            if err < 0.5 * min(err_s1, err_other) or ms > 2000:
                break
        matched_ms = loglog_interp([(p["median_rel_err"], p["ms"]) for p in sweep], err_s1)
        matched_other = loglog_interp([(p["median_rel_err"], p["ms"]) for p in sweep], err_other)
        # the north star's warp-coherent BH (one query per lane, no work splitting),
        # bracketing the matched point: reported beside the load-balanced headline
        wc = []
        os.environ["FSB_BH_SPLIT"] = "0"
        try:
            for p in sweep:
                if p["median_rel_err"] < 0.5 * err_s1 or p["median_rel_err"] > 4 * err_s1:
                    continue
                cfg = fs.EstimatorConfig("barnes_hut", beta=p["beta"], precision="f32")
                evaluate_field_device(cfg, src, kern, q_dev, tree2)
                torch.cuda.synchronize()
                with quiet():
                    ev_a.record()
                    evaluate_field_device(cfg, src, kern, q_dev, tree2)
                    ev_b.record()
                    torch.cuda.synchronize()
                wc.append({"beta": p["beta"], "ms": ev_a.elapsed_time(ev_b),
                           "median_rel_err": p["median_rel_err"]})
        finally:
            del os.environ["FSB_BH_SPLIT"]
        wc_ms = loglog_interp([(p["median_rel_err"], p["ms"]) for p in wc], err_s1)
        # the paper's GPU BH: warp voting over Morton-ordered groups
        vote = []
        for beta in BETAS:
            cfg = fs.EstimatorConfig("barnes_hut", beta=beta, precision="f32", bh_warp_vote=True)
            evaluate_field_device(cfg, src, kern, q_dev, tree2)
            torch.cuda.synchronize()
            with quiet():
                ev_a.record()
                r = evaluate_field_device(cfg, src, kern, q_dev, tree2)
                ev_b.record()
                torch.cuda.synchronize()
            err = median_rel(r.values.cpu().numpy(), truth_h)
            vote.append({"beta": beta, "ms": ev_a.elapsed_time(ev_b), "median_rel_err": err})
            log(f"BH (warp vote) beta={beta}: {vote[-1]['ms']:.2f} ms, median rel err {err:.3e}")
            if err < 0.5 * err_s1 or vote[-1]["ms"] > 2000:
                break
        vote_ms = loglog_interp([(p["median_rel_err"], p["ms"]) for p in vote], err_s1)
        # the ground truth itself against the FP64 oracle brute force on a query subset
        from oracle import oracle as O
        sub = np.linspace(0, n - 1, 256).astype(np.int64)
        ref = np.zeros(len(sub))
        O.brute_force_batch(0, kern.alpha, kern.distance_floor, src.positions, src.masses,
                            np.ascontiguousarray(qs.positions[sub]), ref)
        truth_dev = float(np.max(np.abs(truth_h[sub] - ref) / np.abs(ref)))
        out["accuracy"] = {"s1_median_rel_err": err_s1, "s1_visited_mean": visited_mean,
                           "truth": "GPU brute force (FP32 terms, FP64 accumulation)",
                           "truth_ms": brute_ms,
                           "truth_vs_fp64_oracle_max_rel": truth_dev,
                           "truth_check": "256 queries spread over the plane vs the C oracle's "
                                          "FP64 brute force (reference Kahan recurrence)"}
        out["barnes_hut_sweep"] = sweep
        out["matched_bh_ms"] = matched_ms
        out["speedup_vs_bh_at_matched_error"] = (matched_ms / step_ms) if matched_ms else None
        out["bh_note"] = ("headline BH = load-balanced FP32 BH (warps hand large subtrees of long "
                          "union walks to other warps, csrc/fs_bh_split.cu)")
        out["other_streams"] = {
            "rng_streams": STREAM_NOTES[other], "ms_per_step": other_ms,
            "value": world * n / (other_ms * 1e-3), "s1_median_rel_err": err_other,
            "matched_bh_ms": matched_other,
            "speedup_vs_bh_at_matched_error": (matched_other / other_ms) if matched_other else None}
        out["warp_coherent_bh"] = {"sweep": wc, "matched_ms": wc_ms,
                                   "speedup_at_matched_error": (wc_ms / step_ms) if wc_ms else None,
                                   "note": "one query per lane, warp-union preorder walk, no "
                                           "splitting (the BH design BASELINE's north star names)"}
        out["paper_warp_vote_bh"] = {
            "sweep": vote, "matched_ms": vote_ms,
            "speedup_at_matched_error": (vote_ms / step_ms) if vote_ms else None,
            "note": "the paper's GPU BH (PAPER.md:322): a warp opens a node unless all 32 "
                    "Morton-ordered queries accept it (load-balanced FP32 kernel, d = 2)"}
        # BH roofline: 32 algorithmic bytes per visited node + 16 B per
        # query, at the sweep point nearest the matched error
        near = min(sweep, key=lambda p: abs(math.log(p["median_rel_err"] / err_s1)))
        bh_bytes = (32.0 * near["visited_mean"] + 16.0) * n
        bh_gbs = bh_bytes / (near["ms"] * 1e-3) / 1e9
        out["bh_roofline"] = {
            "bound": "l2", "beta": near["beta"], "ms": near["ms"], "achieved": bh_gbs,
            "peak": L2_READ_GBS, "unit": "GB/s", "frac": bh_gbs / L2_READ_GBS, "traffic": None,
            "note": ("algorithmic bytes = 32 B per visited node (two 16-byte records) + 16 B "
                     "per query; warps of Morton-ordered queries re-read the upper tree, so "
                     "the bound is L2, not HBM (achieved > the 6.65 TB/s HBM fallback); "
                     "peak = L2-resident float4 read bandwidth measured by "
                     "tools/micro/l2bw.cu (64 MB buffer)")}
        out["tree_build_ms"] = {"sources_h2d_first": sources_h2d_ms,
                                "d4_first_build": build4_ms, "d2_first_build": build2_ms,
                                "d4_warm": build4_warm_ms,
                                "note": ("first-in-process figures include the 168 MB pageable "
                                         "copy, lazy module loading and memory-pool growth and "
                                         "vary box to box; d4_warm is the build itself")}
        # the build is HBM-bound -- points/s, and the DRAM bytes of the
        # build kernels from the committed ncu capture of one warm d = 4 build
        out["tree_build"] = {"points_per_s_d4_warm": len(src) / (build4_warm_ms * 1e-3),
                             "from": ("the public build_tree on the same SourceSet with the "
                                      "memory pool grown: its FP64 arrays' device copies are "
                                      "cached (octree.device_sources), so a warm build reads "
                                      "device-resident inputs; the first call includes their "
                                      "168 MB host->device copy, module loading and pool growth"),
                             "dram_bytes": _profiled_build_traffic()}
        # the API-default precision (f64, types.py:205): the FP64 parity kernels on the
        # same workload, bitwise equal to the reference's cores
        f64 = {}
        for name, cfg in (("stochastic_s1", fs.EstimatorConfig("stochastic", seed=1)),
                          ("barnes_hut_beta2", fs.EstimatorConfig("barnes_hut", beta=2.0))):
            tr = tree4 if name.startswith("sto") else tree2
            for _ in range(3):  # first calls pack the FP64 records and grow the memory pool
                evaluate_field_device(cfg, src, kern, q_dev, tr)
            torch.cuda.synchronize()
            calls = []
            for _ in range(5):
                with quiet():
                    ev_a.record()
                    r64 = evaluate_field_device(cfg, src, kern, q_dev, tr)
                    ev_b.record()
                    torch.cuda.synchronize()
                calls.append(ev_a.elapsed_time(ev_b))
            ms = float(np.median(calls))
            f64[name] = {"ms_per_step": ms, "value": n / (ms * 1e-3), "calls_ms": calls,
                         "median_rel_err": median_rel(r64.values.cpu().numpy(), truth_h)}
        f64["note"] = ("precision='f64' (the reference's default): k_sto64 (FP64 queue kernel) and "
                       "k_bh<F64>, every operation in the reference's order (bitwise); "
                       "ms_per_step = median of 5 calls (calls_ms) after 3 warm-up calls")
        out["f64_default_precision"] = f64

        # ---- roofline of the stochastic kernel.  Work unit: one
        # node-term evaluation ("interaction": 8 FP32-pipe ops + 1 MUFU.RSQ, 10
        # flops).  Per query the kernel evaluates the N2 level-2 records (dense
        # part) plus the children of every walk step below level 2; the walk
        # part is visited - (n1 + S * sum_a(children(a) + 1)) (_core.py:195,205).
        pk = peaks()
        f_mhz = float(pk.get("sm_max_mhz", 1965.0))
        sms = torch.cuda.get_device_properties(local).multi_processor_count
        n1, n2, n_int = _level_sizes(tree4)
        S = 1
        visited_base = n1 + S * (n2 + n_int)
        walk_inter = max(visited_mean - visited_base, 0.0)
        inter_q = n2 + walk_inter
        samples_q = S * n_int
        ach = inter_q * n / (kern_ms * 1e-3)
        nominal = min(128 * sms * f_mhz * 1e6 / 8, 16 * sms * f_mhz * 1e6 / 1)  # coulomb I=8, U=1
        # measured on this GPU (fsb_micro_peaks): the Coulomb term at its best instruction
        # mix with every operand on chip, and the MUFU.RSQ rate
        mp = (C.c_double * 2)()
        _lib.check(L.fsb_micro_peaks(mp, sp))
        _lib.check(L.fsb_micro_peaks(mp, sp))
        limit = float(mp[1])
        # pipe floor with the integer RNG work (6 splitmix64 per sample: 6 IMAD on
        # the FMA-heavy pipe + 14 ALU ops each; once per warp with shared streams):
        # max over FMA / ALU / MUFU pipes
        share = 32.0 if args.streams == "warp" else 1.0
        fma_cyc = (7 * inter_q + 2 * 36 * samples_q / share) / 128.0
        alu_cyc = (1 * inter_q + 84 * samples_q / share) / 64.0
        mufu_cyc = (inter_q + samples_q / share) / 16.0
        floor_ms = max(fma_cyc, alu_cyc, mufu_cyc) * n / (sms * f_mhz * 1e6) * 1e3
        kname = "k_sto_warp" if args.streams == "warp" else "k_sto_fast"
        out["roofline"] = {
            "bound": "fp32+mufu", "achieved": ach * 10 / 1e12, "peak": limit * 10 / 1e12,
            "unit": "TFLOP/s", "frac": ach / limit,
            "traffic": _profiled_traffic(kname + "<0"),
            "kernel": f"{kname}<coulomb, paper_ratio> (FP32)", "kernel_ms": kern_ms,
            "work": (f"{inter_q:.1f} interactions/query = {n2} dense level-2 records + "
                     f"{walk_inter:.1f} walk children; 10 flops each"),
            "peak_source": ("measured on this GPU in this run: fsb_micro_peaks (csrc/fs_micro.cu) "
                            "-- Coulomb node terms/s of the packed-FP32 + "
                            "MUFU.RSQ loop with all operands on chip, x 10 flops (MEASURED_PEAKS."
                            "json has no FP32/MUFU entry)"),
            "measured_mufu_rsq_per_s": float(mp[0]),
            "nominal_peak": nominal * 10 / 1e12, "frac_of_nominal": ach / nominal,
            "nominal_source": (f"FP32 128/clk/SM over 8 ops, MUFU 16/clk/SM over 1 op, {sms} SMs "
                               f"x {f_mhz:.0f} MHz"),
            "survey_8d": {
                "flops_per_query": 10.0 * (n1 + n2) + 20.0 * S * n_int + 10.0 * walk_inter,
                "formula": ("SURVEY 8(d): (N1 + N2) F_k + S N_sub (2 x 10 flops for the two "
                            "far-field ratios) + sum over deeper levels (kids + 1) F_k, F_k = 10"),
                "achieved": (10.0 * (n1 + n2) + 20.0 * S * n_int + 10.0 * walk_inter) * n
                            / (kern_ms * 1e-3) / 1e12,
                "frac": (10.0 * (n1 + n2) + 20.0 * S * n_int + 10.0 * walk_inter) * n
                        / (kern_ms * 1e-3) / (limit * 10),
                "note": ("the survey's algorithmic count includes the N1 control-variate terms, "
                         "which the kernel's dense part cancels (never evaluated), and the "
                         "ratio arithmetic of every sample; `frac` above counts only the node "
                         "terms the kernel evaluates")},
            "pipe_floor_ms": floor_ms, "frac_of_pipe_floor": floor_ms / kern_ms,
            "pipe_floor_note": (f"FMA/ALU/MUFU pipe floor incl. {samples_q} samples/query x 6 "
                                f"splitmix64 mixes; cycles/query fma {fma_cyc:.1f} alu "
                                f"{alu_cyc:.1f} mufu {mufu_cyc:.1f}")}
        if args.cpu_baseline and world == 1:
            out["cpu_baseline"] = _cpu_baseline(tree4, src, qs, kern, args)
        if args.c5_anchor and world == 1:
            out["c5"] = run_c5(args, 1, 0, local, anchor=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


def _count_launches(fn):
    """Kernels of libfastsum_b200.so (fsb:: and its CUB sorts) one call of fn launches
    (CUPTI via torch.profiler, outside any timed region)."""
    import torch
    try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        return sum(1 for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
                   and ("fsb" in e.name or "cub" in e.name.lower()))
    except Exception as exc:  # pragma: no cover
        log("profiler unavailable:", exc)
        return None


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _profiled_traffic(kernel_key: str):
    """DRAM bytes per launch of the kernel from the newest committed ncu summary."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_kernels.json")), reverse=True):
        try:
            with open(path) as f:
                side = json.load(f)
        except (OSError, ValueError):
            continue
        for name, k in side.items():
            if kernel_key in name and "dram_bytes" in k:
                return {"bytes_per_launch": k["dram_bytes"], "source": os.path.relpath(path, ROOT)}
    return None


def _profiled_build_traffic():
    """Sum of dram__bytes over the build kernels of one warm d = 4 C4 build, from the
    newest committed profiles/r*_build.json (tools/profile_build.py)."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_build.json")), reverse=True):
        try:
            with open(path) as f:
                side = json.load(f)
            return {"bytes": side["dram_bytes_total"], "kernels": side["kernels"],
                    "gpu_time_ms": side["gpu_time_ms"], "source": os.path.relpath(path, ROOT)}
        except (OSError, ValueError, KeyError):
            continue
    return None


def _level_sizes(tree):
    """(n1, n2, internal level-1 nodes) of the d=4 tree: level-1 nodes, their children."""
    cc = tree.child_count
    cs = tree.child_start
    ci = tree.child_index
    lvl1 = ci[cs[0]:cs[0] + cc[0]]
    return int(len(lvl1)), int(sum(int(cc[a]) for a in lvl1)), int(np.count_nonzero(cc[lvl1]))


def _e2e(args, fs, src, kern, qs, tree, cfg, world, rank):
    """The step through the public API (evaluate_field, host numpy in / out): every
    rank evaluates its own slab (query_offset = rank * n), timed between barriers, max
    over ranks.  The headline input is a QuerySet over page-locked host memory (what a
    serving caller keeps); a plain (pageable) numpy QuerySet is timed beside it."""
    import torch
    import torch.distributed as dist
    n = len(qs)
    host = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
    host.numpy()[:] = qs.positions
    off = rank * n

    def timed(qset):
        """median of five trials of K steps after ten warm-up calls (the host side
        of the step -- worker threads, page-locked blocks, PCIe -- keeps warming up
        over the first tens of calls: trials of 1.27 / 1.07 / 0.91 ms after five)"""
        r = None
        for _ in range(max(10, args.warmup)):  # like the timed loop: the previous result stays alive
            r = fs.evaluate_field(cfg, src, kern, qset, tree=tree, query_offset=off)
        trials = []
        for _ in range(5):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            with quiet():
                t0 = time.perf_counter()
                for _ in range(args.steps):
                    r = fs.evaluate_field(cfg, src, kern, qset, tree=tree, query_offset=off)
                torch.cuda.synchronize()
                dt = (time.perf_counter() - t0) / args.steps
            if world > 1:
                tt = torch.tensor([dt], device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                dt = float(tt.item())
            trials.append(dt)
        return float(np.median(trials)), r, [t * 1e3 for t in trials]

    dt, r, tr = timed(fs.QuerySet(host.numpy()))
    dt_pg, _, tr_pg = timed(fs.QuerySet(np.array(qs.positions)))
    # bytes that cross PCIe: values, visited, path_steps (stochastic, non-smooth
    # kernel); raw (= values, identity post-transform), flagged (all false) and
    # path_count (query-independent) are written on the host by
    # fsb_evaluate_field_host while the pipeline runs
    out_bytes = sum(a.nbytes for a in (r.values, r.visited_nodes, r.path_steps))
    result_bytes = sum(a.nbytes for a in (r.values, r.raw, r.flagged, r.visited_nodes,
                                          r.path_steps, r.path_count))
    return {"value": world * n / dt, "unit": "queries/s",
            "h2d_bytes_per_step": int(n * 24), "d2h_bytes_per_step": int(out_bytes),
            "result_bytes_per_step": int(result_bytes),
            "ms_per_step": dt * 1e3, "trials_ms_per_step": tr,
            "api": ("paper_2506_02219_b200.evaluate_field (host numpy in/out, pipelined slabs); "
                    "QuerySet over page-locked host memory"),
            "pageable": {"value": world * n / dt_pg, "ms_per_step": dt_pg * 1e3,
                         "trials_ms_per_step": tr_pg,
                         "note": "the same call with a plain numpy (pageable) QuerySet"},
            "n_gpus": world, "bytes_note": "per rank per step"}


def _cpu_baseline(tree, src, qs, kern, args):
    """The C oracle port (reference algorithm) on the host cores, bounded sample."""
    from oracle import oracle as O
    n_sample = args.cpu_sample
    idx = np.unique(np.linspace(0, len(qs) - 1, n_sample).astype(np.int64))
    n_sample = len(idx)
    q = np.ascontiguousarray(qs.positions[idx])
    ca = tuple(np.ascontiguousarray(a) for a in tree.core_arrays())
    out = np.zeros(n_sample)
    z = [np.zeros(n_sample, dtype=np.int64) for _ in range(3)]
    O.stochastic_batch(*ca, 0, kern.alpha, kern.distance_floor, q[:64], 1, 0, 1, 0, out[:64],
                       z[0][:64], z[1][:64], z[2][:64])
    t0 = time.perf_counter()
    O.stochastic_batch(*ca, 0, kern.alpha, kern.distance_floor, q, 1, 0, 1, 0, out, *z)
    dt = time.perf_counter() - t0
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": n_sample / dt, "unit": "queries/s", "cores": cores, "kind": "port",
            "cpu_model": _cpu_model(), "nproc": os.cpu_count(),
            "sample": f"{n_sample} queries of the C4 plane, stochastic S=1 f64 "
                      f"(oracle/fastsum_oracle.c, OpenMP), tree from the GPU build"}


# ----------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from oracle import oracle as O
    src, qs, kern = workload()
    t0 = time.perf_counter()
    t = O.build_tree(src.positions, src.masses, src.weights, 4, 32)
    build_s = time.perf_counter() - t0
    ca = O.core_arrays(t)
    n_sample = args.cpu_sample
    rng = np.random.default_rng(0)
    z = [np.zeros(n_sample, dtype=np.int64) for _ in range(3)]
    out = np.zeros(n_sample)

    def step(k):
        idx = rng.integers(0, len(qs), n_sample)
        q = np.ascontiguousarray(qs.positions[idx])
        O.stochastic_batch(*ca, 0, kern.alpha, kern.distance_floor, q, 1, 0, 1, 0, out, *z)

    for k in range(args.warmup):
        step(k)
    t0 = time.perf_counter()
    for k in range(args.steps):
        step(k)
    dt = (time.perf_counter() - t0) / args.steps
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    v = n_sample / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference mesh generators, fixed seeds)",
            "config": config_block("query"), "cpu_baseline": {"value": v, "unit": "queries/s", "cores": cores, "kind": "port",
                             "cpu_model": _cpu_model(), "nproc": os.cpu_count(),
                             "sample": f"{n_sample} random queries of the C4 plane per step, "
                                       f"stochastic S=1 f64, oracle/fastsum_oracle.c (OpenMP)"},
            "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "tree_build_s": build_s}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--cpu-sample", type=int, default=N_SIDE * N_SIDE)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--workload", choices=("auto", "c4", "c5"), default="auto",
                    help="auto: C4 (the headline, BASELINE configs[3]) on one GPU, C5 strong "
                         "scaling (configs[4]) on N > 1")
    ap.add_argument("--no-c5-anchor", dest="c5_anchor", action="store_false",
                    help="skip the C5 one-GPU anchor in the C4 line")
    ap.add_argument("--streams", choices=("warp", "query"), default="warp",
                    help="RNG streams of the headline step (the other mode is reported beside)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
