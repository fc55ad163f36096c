#!/usr/bin/env python
"""Benchmark: RecSplit MPHF construction keys/s on B200 (BASELINE.json metric).

A "step" is one complete construction of the MPHF of the workload's keys: hash +
bucket sort, every split and leaf search, key redistribution, Golomb-Rice and
Elias-Fano encoding, serialization.  Default workload: C3 (n=5e6 keys, l=16, b=2000,
rotation fitting) -- the north-star target and the paper's 1.56 bits/object point.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C3]

value      keys/s with the keys already resident in HBM (device-pointer ABI entry),
           device time (CUDA events on the launch stream), L2 flushed between steps;
           for N>1: total keys of all ranks / max over ranks.
e2e        the same metric through recsplit_build with HOST keys (pinned), H2D and
           the result D2H inside the timed region (host wall clock around the call).
roofline   dominant kernel = the lower-level-1 split search (62% of the work at C3):
           algorithmic remix evaluations (sum over nodes of (minimal seed + 1) x keys)
           / that kernel's CUDA-event duration, against the INT32-pipe peak;
           at N > 1 from one extra single-GPU build of rank 0's key slice (the sharded build
           returns no per-kernel events).  Single-GPU builds of a configuration replay a
           captured CUDA graph after the first two (warm-up) builds.
cpu_baseline / --impl reference: the plain C oracle, as it stands, on this host's cores,
           on a bounded sample of the same workload (whole buckets).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

# the paper's own GPU figure, other hardware: context only, never the baseline (vs_baseline = null)
PAPER_CONTEXT = {"C3": "GPURecSplit RF, l=16 b=2000: 1.0 us/object = 1.0e6 keys/s on an RTX 3090 incl. transfers (P:581)"}
WORKLOAD_TEXT = {
    "C1": "C1: n=1e4 random u64 keys, l=8, b=100, rotation fitting",
    "C2": "C2: n=5e6 random u64 keys, l=8, b=100, rotation fitting",
    "C3": "C3: n=5e6 random u64 keys, l=16, b=2000, rotation fitting",
    "C5": "C5: n=1e8 random u64 keys, l=12, b=1000, rotation fitting",
}
# Scaling: strong by default (BASELINE.json: C3 "1 and 8 B200", C5 "sharded across 2/4/8"
# -- the total key count is the config's n for every N); --weak builds N x n keys.


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def mix_bound():
    """Measured roofline denominator: evaluations per clock per SM of the split
    loop's SASS mix under the per-opcode throughputs measured by tools/probe/pipes.cu
    (profiles/l1_mix_bound_r02.json, written by tools/probe/mix_bound.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "l1_mix_bound_r02.json")) as f:
            d = json.load(f)
        return float(d["evals_per_clk_per_sm"]), d
    except (OSError, ValueError, KeyError):
        return None, None


def int32_peak_evals(sm_count: int, mhz: float) -> float:
    """INT32 roofline in remix evaluations/s: the measured mix bound (mix_bound) if present,
    else the round-1 derived issue bound (21 integer instructions per evaluation, 64 lanes/clk
    per pipe -> 6.10 evaluations per clock per SM)."""
    per_clk, _ = mix_bound()
    return sm_count * mhz * 1e6 * (per_clk if per_clk else 64.0 / 10.5)


def executed_evals(cfg: dict, world: int):
    """Executed key evaluations per class of one build of the workload, from the counting
    build of the same kernels (build_var/count, -DRS_COUNT_EVALS) in a subprocess; None when
    that library is absent."""
    lib = os.path.join(ROOT, "build_var", "count", "librecsplit_b200.so")
    if world != 1 or not os.path.exists(lib):
        return None
    code = ("import sys, json, numpy as np, torch; sys.path.insert(0, %r)\n"
            "import paper_2212_09562_b200 as rs, synth\n"
            "k = synth.keys(%d, %d); kt = torch.from_numpy(k.view(np.int64)).cuda()\n"
            "b, s = rs.build_device(kt, %d, %d, stats=True)\n"
            "print(json.dumps(s['exec_evals']))" % (ROOT, cfg["n"], cfg["seed"], cfg["leaf"], cfg["bucket"]))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       env=dict(os.environ, RECSPLIT_LIB=lib), timeout=600)
    if r.returncode:
        return None
    return json.loads(r.stdout.strip().splitlines()[-1])


NVML_SAMPLER = r"""
import sys, time, pynvml as nv
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
while True:
    try:
        r = (nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM),
             nv.nvmlDeviceGetCurrentClocksEventReasons(h))
    except Exception:
        break
    print(*r, time.time(), flush=True)
    time.sleep(0.002)
"""


class NvmlClocks:
    """NVML sampler (every ~2 ms) in a separate process running during the timed region: SM
    clock, max SM clock and the active clock-event reasons -- enough samples even for a 30 ms
    timed region (C2), and no GIL shared with the timed thread (a sampler thread in this process
    once delayed a timed step by a whole GIL switch interval)."""

    NAMES = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
             ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
             ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
             ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap")]

    def __init__(self, index: int):
        import pynvml  # noqa: F401 -- fail here (fallback to nvidia-smi) if NVML is absent
        self.nv = pynvml
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".txt", delete=False)
        self.p = subprocess.Popen([sys.executable, "-c", NVML_SAMPLER, str(index)], stdout=self.f,
                                  stderr=subprocess.DEVNULL)
        t0 = time.time()
        while time.time() - t0 < 20:  # first sample before the timed region starts
            if os.path.getsize(self.f.name) > 0 or self.p.poll() is not None:
                break
            time.sleep(0.01)

    def stop(self, t_start: float = 0.0) -> dict:
        """Summary of the samples taken after t_start (time.time() at the timed region's start)."""
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = []
        for line in self.f.read().split("\n"):
            p = line.split()
            if len(p) == 4 and float(p[3]) >= t_start:
                rows.append((float(p[0]), float(p[1]), int(p[2])))
        os.unlink(self.f.name)
        reasons = sorted({nm for _, _, r in rows for nm, c in self.NAMES if r & getattr(self.nv, c)})
        busy = [s for s, _, _ in rows if s > 300] or [s for s, _, _ in rows]
        return {"sm_mhz": float(np.median(busy)) if busy else None,
                "sm_max_mhz": float(max(m for _, m, _ in rows)) if rows else None,
                "reasons": reasons, "samples": len(rows), "source": "nvml"}


def nvml_index(dev: int) -> int:
    """NVML (physical) index of CUDA device dev under CUDA_VISIBLE_DEVICES (integer lists)."""
    vis = [v.strip() for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
    return int(vis[dev]) if dev < len(vis) and vis[dev].isdigit() else dev


def clock_sampler(index: int):
    try:
        return NvmlClocks(index)
    except Exception:  # noqa: BLE001 -- no NVML: the nvidia-smi process sampler
        return Clocks(index)


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self, t_start: float = 0.0) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) < 9:
                continue
            for k, nm in enumerate(names):
                if r[5 + k].strip().lower() == "active":
                    reasons.add(nm)
        busy = [s for s in sm if s > 300] or sm
        return {"sm_mhz": float(np.median(busy)) if busy else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def cpu_sample(cfg: dict, keys: np.ndarray, budget_s: float, threads: int):
    """Run the oracle on whole buckets of the workload (largest-bucket-first order is
    avoided: buckets are taken in index order) until ~budget_s of wall time; returns
    (keys processed, seconds, buckets)."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor

    oracle.compile_oracle()
    n, leaf, b = cfg["n"], cfg["leaf"], cfg["bucket"]
    B = (n + b - 1) // b

    def remix(z):
        with np.errstate(over="ignore"):
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            return z ^ (z >> np.uint64(31))
    hi = remix(keys ^ np.uint64(0x9E3779B97F4A7C15))
    bucket = ((hi >> np.uint64(32)) * np.uint64(B)) >> np.uint64(32)
    order = np.argsort(bucket, kind="stable")
    sizes = np.bincount(bucket.astype(np.int64), minlength=B)
    starts = np.concatenate([[0], np.cumsum(sizes)])
    done_keys, nb = 0, 0
    t0 = time.perf_counter()
    i = 0
    with ThreadPoolExecutor(threads) as ex:
        while i < B and (nb == 0 or time.perf_counter() - t0 < budget_s):
            batch = list(range(i, min(B, i + threads)))
            i += len(batch)
            list(ex.map(lambda j: oracle.bucket_values(keys[order[starts[j]:starts[j + 1]]], leaf), batch))
            done_keys += int(sum(sizes[j] for j in batch))
            nb += len(batch)
    return done_keys, time.perf_counter() - t0, nb


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3", "C5"])
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--weak", action="store_true", help="n keys per rank (one MPHF of N x n keys)")
    ap.add_argument("--no-exec-count", action="store_true", help="skip the executed-evaluation count")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = synth.CONFIGS[args.config]
    threads = os.cpu_count() or 1

    if args.impl == "reference":
        # the oracle arm: rank 0 only, on host cores, bounded sample per step
        if rank != 0:
            return
        keys = synth.keys(cfg["n"], cfg["seed"])
        import oracle
        c1 = synth.CONFIGS["C1"]
        for _ in range(args.warmup):  # warm-up: one small build (page-in, thread start-up)
            oracle.build(synth.keys(c1["n"], c1["seed"]), c1["leaf"], c1["bucket"], threads=threads)
        tot_k, tot_t, tot_b = 0, 0.0, 0
        for _ in range(args.steps):  # each step: one round of `threads` whole buckets
            k, t, nb = cpu_sample(cfg, keys, 0.0, threads)
            tot_k, tot_t, tot_b = tot_k + k, tot_t + t, tot_b + nb
        v = tot_k / tot_t
        sample = f"{tot_b} whole buckets ({tot_k} keys) of the {args.config} workload over {args.steps} steps"
        print(json.dumps({
            "impl": "reference", "metric": "MPHF construction keys/s", "value": v, "unit": "keys/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_t / max(1, args.steps), "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": WORKLOAD_TEXT[args.config], "n": cfg["n"], "leaf": cfg["leaf"],
                       "bucket": cfg["bucket"]},
            "cpu_baseline": {"value": v, "unit": "keys/s", "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "keys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }))
        return

    import torch

    import paper_2212_09562_b200 as rs

    backend = os.environ.get("RS_BENCH_BACKEND", "nccl")  # gloo: functional runs of N ranks on 1 GPU
    if world > 1:
        import torch.distributed as dist
        dev_index = 0 if os.environ.get("RS_BENCH_SAME_DEVICE") else local
        torch.cuda.set_device(dev_index)
        dist.init_process_group(backend)
        # rank check: every rank prints its communicator size and device (stderr)
        nccl_v = ".".join(map(str, torch.cuda.nccl.version())) if backend == "nccl" else None
        print(f"[rank {rank}] backend={backend} world_size={dist.get_world_size()} nccl={nccl_v} "
              f"device={torch.cuda.current_device()} ({torch.cuda.get_device_name()})", file=sys.stderr, flush=True)
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    # run on the CPUs local to this GPU (pinned host buffers then live on its NUMA node; an H2D
    # from the far socket measured ~20 % slower end to end at C2)
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(nvml_index(dev))
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        cpus &= set(range(os.cpu_count()))
        if cpus:
            os.sched_setaffinity(0, cpus)
    except Exception:  # noqa: BLE001 -- no NVML / affinity: leave the scheduler's choice
        pass
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    # weak scaling: N ranks build ONE MPHF of N x n keys, each rank owning 1/N of the
    # buckets (bucket-range sharding).  Each rank starts from its own n-key slice of
    # the input; inside the build the keys are routed to their bucket owners with one
    # all-to-all, so per-rank memory and H2D stay at n keys.
    strong = not args.weak
    n_total = cfg["n"] if strong else cfg["n"] * world
    keys_all = synth.keys(n_total, cfg["seed"])
    keys = keys_all[rank * n_total // world:(rank + 1) * n_total // world]
    kt = torch.from_numpy(keys.view(np.int64).copy()).cuda()
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def build_once(keys_tensor):
        if world == 1:  # the result as a view of the library's buffer (no host copy)
            return rs.build_device(keys_tensor, cfg["leaf"], cfg["bucket"], stream=stream, stats=True, copy=False)
        blob = rs.build_sharded(keys_tensor, cfg["leaf"], cfg["bucket"], stream=stream, distribute=True)
        return blob, None

    def one_step():
        flush.zero_()  # L2 flush (inputs are 40 MB < 126 MB L2)
        if world > 1:
            torch.distributed.barrier()
        a = torch.cuda.Event(enable_timing=True)
        z = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        blob, st = build_once(kt)
        z.record(stream)
        z.synchronize()
        return a.elapsed_time(z) * 1e-3, blob, st

    # the clock sampler starts before the warm-up steps, so that the GPU is not left idle (and
    # its clocks ramping back up) between warm-up and timed steps; only the samples taken
    # during the timed region are reported
    clk = clock_sampler(nvml_index(dev)) if not os.environ.get("RS_BENCH_NO_CLOCKS") else None
    # the collector off in the timed loops (as timeit does): a full collection of this process's
    # objects (torch imported) took one timed C2 step from 2.6 to 18-22 ms
    import gc
    gc.collect()
    gc.disable()
    for _ in range(max(3, args.warmup)):
        one_step()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t_timed = time.time()
    times, stats = [], []
    blob = None
    for _ in range(args.steps):
        if world == 1:  # (the previous result's pinned buffer back to the library's pool first: a
            blob = b = None  # second live result costs a cudaMallocHost inside the timed step)
        t, b, st = one_step()
        times.append(t)
        stats.append(st)
        blob = b if b is not None else blob
    torch.cuda.synchronize()
    clocks = clk.stop(t_timed) if clk else {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["not sampled"], "samples": 0}
    print(f"[bench] step ms: {[round(1e3 * t, 4) for t in times]} graph replays: "
          f"{[int(x.get('graph_replay', 0)) for x in stats if x is not None]}", file=sys.stderr, flush=True)
    if world > 1:
        torch.distributed.barrier()
    mean_t = float(np.mean(times))
    t_all = torch.tensor([mean_t], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
    if world > 1:
        torch.distributed.all_reduce(t_all, op=torch.distributed.ReduceOp.MAX)
    t_max = float(t_all.item())
    value = n_total / t_max

    # ---- e2e: host keys through the public API, H2D + D2H inside the timed region
    pinned = torch.from_numpy(keys.view(np.int64)).pin_memory()
    pkeys = pinned.numpy().view(np.uint64)

    def e2e_once():
        if world == 1:
            return rs.build(pkeys, cfg["leaf"], cfg["bucket"], copy=False)
        kd = pinned.to("cuda", non_blocking=True)
        return rs.build_sharded(kd, cfg["leaf"], cfg["bucket"], stream=stream, distribute=True)

    for _ in range(max(3, args.warmup)):  # warm (the first builds of a configuration capture its CUDA graph)
        e2e_once()
    e2e_times = []
    eb = None
    for _ in range(args.steps):
        eb = None  # (as above: one result buffer in flight)
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        eb = e2e_once()
        e2e_times.append(time.perf_counter() - t0)
    print(f"[bench] e2e step ms: {[round(1e3 * t, 4) for t in e2e_times]}", file=sys.stderr, flush=True)
    gc.enable()
    e2e_t = torch.tensor([float(np.mean(e2e_times))], dtype=torch.float64,
                         device="cuda" if backend == "nccl" else "cpu")
    if world > 1:
        torch.distributed.all_reduce(e2e_t, op=torch.distributed.ReduceOp.MAX)
    e2e_value = n_total / float(e2e_t.item())
    if rank == 0:
        assert bytes(eb) == bytes(blob), "host-input and device-input builds differ"

    if rank != 0:
        torch.distributed.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (lower-level-1 split search), from the
    # single-GPU build's own CUDA events (N > 1: measured by one extra 1-GPU build)
    if stats[0] is None:
        rs.build_device(kt, cfg["leaf"], cfg["bucket"], stream=stream)  # warm (device tables)
        blob1, st1 = rs.build_device(kt, cfg["leaf"], cfg["bucket"], stream=stream, stats=True)
        stats = [st1]
    cls = 2
    tree = float(np.mean([s.get("t_search_tree", 0.0) for s in stats])) > 0
    if tree:  # small configurations: one whole-bucket kernel searches every node class
        evals = float(np.mean([sum(s["algo_evals"]) for s in stats]))
        kt_s = float(np.mean([s["t_search_tree"] for s in stats]))
    else:
        evals = float(np.mean([s["algo_evals"][cls] for s in stats]))
        kt_s = float(np.mean([s["t_search"][cls] for s in stats]))
    peaks = _peaks()
    if "sm_max_mhz" in peaks:
        max_mhz, mhz_src = float(peaks["sm_max_mhz"]), "MEASURED_PEAKS sm_max_mhz"
    elif clocks.get("sm_max_mhz"):
        max_mhz, mhz_src = float(clocks["sm_max_mhz"]), "nvidia-smi clocks.max.sm during the run"
    else:
        max_mhz, mhz_src = 1965.0, "fallback: B200 max SM clock"
    peak = int32_peak_evals(sms, max_mhz) / 1e9
    mix = mix_bound()
    achieved = evals / kt_s / 1e9
    ex = executed_evals(cfg, world) if not args.no_exec_count else None
    exec_l1 = (float(sum(ex)) if tree else float(ex[cls])) if ex and (sum(ex) if tree else ex[cls]) else None
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_l1_split_traffic.json")
    if os.path.exists(prof) and args.config == "C3":  # the ncu capture is of the C3 launch
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    st0 = stats[-1]
    line = {
        "metric": "MPHF construction keys/s", "value": value, "unit": "keys/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": 1e3 * t_max,
        "higher_is_better": True, "scaling": "strong" if strong else "weak",
        "vs_baseline": None,  # BASELINE.md publishes no B200 number for this metric
        "paper_context": PAPER_CONTEXT.get(args.config),
        "dtype": "u64", "data": "synthetic",
        "config": {"workload": WORKLOAD_TEXT[args.config], "n": n_total, "leaf": cfg["leaf"],
                   "bucket": cfg["bucket"], "keys_per_rank": len(keys), "l2": "flushed between steps",
                   "bits_per_key": rs.bits_per_key(blob),
                   "parallelism": f"bucket-range shards x{world} (one MPHF, work-balanced ranges)" if world > 1 else "1gpu",
                   "comm": ({"backend": backend, "world_size": world,
                             "nccl": ".".join(map(str, torch.cuda.nccl.version())) if backend == "nccl" else None}
                            if world > 1 else None)},
        "e2e": {"value": e2e_value, "unit": "keys/s", "h2d_bytes_per_step": int(n_total * 8),  # whole job
                "d2h_bytes_per_step": len(blob)},
        "gpu_launches": int(sum(s["kernel_launches"] for s in stats)) * (args.steps if world > 1 else 1),
        "roofline": {"bound": "alu", "kernel": ("k_bucket_tree (whole buckets per warp, every node class)" if tree
                                                else "k_search<SK_LOWER> (lower level 1 splits)"),
                     "achieved": achieved, "peak": peak, "unit": "Geval/s", "frac": achieved / peak,
                     "traffic": traffic,
                     "executed_frac": (exec_l1 / kt_s / 1e9 / peak) if exec_l1 else None,
                     "executed_over_algorithmic": (exec_l1 / evals) if exec_l1 else None,
                     "peak_note": (f"{sms} SMs x {max_mhz:.0f} MHz ({mhz_src}) x {mix[0]:.3f} evals/clk/SM: the split "
                                   f"loop's SASS mix ({mix[1]['loop_instructions']} instructions per 4 keys x 32 seeds) "
                                   f"under the per-opcode rates measured by tools/probe/pipes.cu "
                                   f"(profiles/l1_mix_bound_r02.json; FMA-pipe bound)") if mix[0] else
                                  f"{sms} SMs x {max_mhz:.0f} MHz ({mhz_src}) x 6.10 evals/clk/SM (derived issue bound)"},
        "phases_s": {"partition": st0["t_partition"], "tree": st0["t_tree"],
                     "search_bucket_tree": st0.get("t_search_tree", 0.0), "upper": st0["t_search"][0],
                     "lower2": st0["t_search"][1], "lower1": st0["t_search"][2], "leaves": st0["t_search"][3],
                     "reorder": st0["t_reorder"], "encode": st0["t_encode"], "d2h": st0["t_d2h"],
                     # the library's own device span (first enqueued operation to the end of the
                     # result D2H) and host wall time inside the C ABI call, means over the timed steps
                     "device_span": float(np.mean([x.get("t_device", 0.0) for x in stats])),
                     "abi_call": float(np.mean([x.get("t_total", 0.0) for x in stats]))},
        "algo_evals_per_step": [int(x) for x in st0["algo_evals"]],
        # INT32 fraction per search phase: that phase's algorithmic evaluations /
        # its CUDA-event time / the same peak; "step" = all evaluations / the whole step
        "int32_frac_by_phase": {
            nm: (float(np.mean([x["algo_evals"][k] for x in stats])) /
                 float(np.mean([x["t_search"][k] for x in stats])) / 1e9 / peak)
            if float(np.mean([x["t_search"][k] for x in stats])) > 0 else None
            for k, nm in enumerate(["upper", "lower2", "lower1", "leaves"])},
        "int32_frac_step": (float(np.mean([sum(x["algo_evals"]) for x in stats])) / t_max / 1e9 / peak)
        if world == 1 else None,
        # executed key evaluations (counting build) per phase / that phase's time / the same peak
        "int32_exec_frac_by_phase": ({
            nm: (float(ex[k]) / float(np.mean([x["t_search"][k] for x in stats])) / 1e9 / peak)
            if ex[k] and float(np.mean([x["t_search"][k] for x in stats])) > 0 else None
            for k, nm in enumerate(["upper", "lower2", "lower1", "leaves"])} if ex else None),
        "exec_evals_per_step": [int(x) for x in ex] if ex else None,
        "clocks": clocks,
    }
    if not args.no_cpu_baseline and world == 1:  # rank 0 at N = 1 only
        k, t, nb = cpu_sample(cfg, keys, args.cpu_budget, threads)
        # threads = 1: the same oracle on one core, on whole buckets
        # for about a third of the budget; per-key work is constant in n at fixed (l, b), so
        # keys/s on the sample is the single-thread rate (a full C3 build would take ~2 h)
        k1, t1, nb1 = cpu_sample(cfg, keys, args.cpu_budget / 3, 1)
        line["cpu_baseline"] = {"value": k / t, "unit": "keys/s", "cores": threads, "kind": "oracle",
                                "sample": f"{nb} whole buckets ({k} keys) of the {args.config} workload, "
                                          f"{threads} threads over contiguous buckets",
                                "single_thread": {"value": k1 / t1, "unit": "keys/s", "cores": 1,
                                                  "sample": f"{nb1} whole buckets ({k1} keys), one thread",
                                                  "full_build_s_extrapolated": cfg["n"] * t1 / k1}}
    print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
