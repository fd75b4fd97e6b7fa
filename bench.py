#!/usr/bin/env python
"""bench.py -- HyperBall hot path on B200 (driver contract in the task spec).

A step = one full HyperBall run (init -> iterate until max increase <= 0.5,
or the depth limit) over the synthetic C3 graph (open 486x486 grid, radius 87
cells: 236,196 cells, 4.79e9 directed edges, 4.83 GB LEB128 stream), p=10.

  value    edge-register updates/s = iterations * |E| * 2^p / time, CSR and
           counters resident in HBM, device time (CUDA events on the
           library's stream), max over ranks.
  e2e      same metric through the public C-ABI with HOST buffers: CSR upload
           (pinned H2D, chunked, validated per chunk) + run (its first run a
           wavefront over the upload chunks) + read-back of c / sum_d / sum_d2.
  roofline the fused decode-union kernel against the unit that binds it (SM
           instruction issue): ncu's warp-instructions per launch / the live
           CUDA-event launch time vs 1 instr/cycle/SMSP at the sampled clock;
           `dram_frac` (ncu DRAM bytes vs MEASURED_PEAKS.json hbm_gbs) and
           `hbm_algorithmic` (SURVEY §8(d) bytes) beside it.
  cpu_baseline  the reference's compiled primitives + SPEC loop
           (oracle/_ref) on this host's cores, bounded sample.

`--impl reference` times only the reference CPU path (rank 0) on the same
config and prints its own line.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (rows, cols, n_rects, rect_min, rect_max, seed, radius2, description)
    "c1": (64, 64, 20, 2, 9, 20261017, 0, "C1 64x64 grid, 20 rectangles, unlimited radius"),
    "c2": (212, 212, 60, 3, 10, 20261017, 44 * 44, "C2 212x212 grid, 60 rectangles (3-10 cells), radius 44 cells"),
    "c3": (486, 486, 0, 1, 1, 20261017, 87 * 87, "C3 open 486x486 grid, radius 87 cells"),
}
# BASELINE.json configs: C1 is quoted at depth limit 3, C2 / C3 at full depth.
DEFAULT_DEPTH = {"c1": 3}
METRIC = "HyperBall edge-register updates/s"
UNIT = "edge-register updates/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self, keep_busy=None):
        """keep_busy: for timed regions shorter than nvidia-smi's first sample (small
        configs), the same workload keeps running untimed until one sample exists."""
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        extended = False
        t0 = time.perf_counter()
        while keep_busy is not None and not self.lines and time.perf_counter() - t0 < 5.0:
            keep_busy()
            extended = True
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
               "reasons": sorted(reasons), "samples": len(sm)}
        if extended:
            out["note"] = "timed region shorter than the first nvidia-smi sample; sampled while the same runs continued untimed"
        return out


def build_graph(cfg, threads=0):
    from paper_2604_08374_b200 import CompressedCsr
    r, c, k, a, b, seed, rad2, _ = CONFIGS[cfg]
    t0 = time.perf_counter()
    g = CompressedCsr.synth_grid(r, c, k, a, b, seed, rad2, threads)
    log(f"[bench] generated {cfg}: {g} in {time.perf_counter() - t0:.1f} s")
    return g


def build_graph_reference(cfg, threads=0):
    """The same graph from the oracle's own generator (oracle/sb_synth.c, byte-identical:
    tests/test_oracle_synth.py), so the reference arm never maps the product library."""
    import oracle
    r, c, k, a, b, seed, rad2, _ = CONFIGS[cfg]
    t0 = time.perf_counter()
    g = oracle.SynthCsr(r, c, k, a, b, seed, rad2, threads)
    log(f"[bench] generated {cfg} (oracle generator): {g} in {time.perf_counter() - t0:.1f} s")
    return g


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def alg_bytes_per_iter(n, edges, stream_len, p):
    """CSR (stream + 8(N+1) + 4N) + |E| m/2 + N m/2 (own) + N m/2 (write)."""
    row = (1 << p) // 2
    return stream_len + 8 * (n + 1) + 4 * n + edges * row + 2 * n * row


def profile_entry(cfg, p):
    """The committed ncu --set full summary of the union kernel for this config (or None)."""
    path = os.path.join(ROOT, "profiles", "union_ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f).get(f"{cfg}_p{p}")
    except Exception:
        return None


def roofline_of(cfg, p, launch_s, bytes_launch, sm_mhz):
    """Roofline of the dominant kernel (the dense union) on the unit that binds it.

    The union's 2.46 TB of SURVEY 8(d) algorithmic row bytes per C3 launch never
    reach DRAM: each 16-node group gathers a row once per block of its cover and L2 serves it, so
    the ncu DRAM traffic is ~5 GB per launch (the stream + the planes) and an
    HBM "roofline" on algorithmic bytes reads > 1.  What bounds the kernel is the
    SM's instruction issue (ncu: issue slots ~77 % busy, ALU pipe ~70 %).  So:
      achieved = warp-instructions issued per launch (ncu, a per-launch constant
                 of this kernel on this graph) / the LIVE launch time (CUDA events)
      peak     = 1 warp-instruction / cycle / SMSP x 4 SMSPs x SMs x the SM clock
                 sampled during the timed region.
    The HBM view is kept beside it (`dram_frac` on measured DRAM bytes, and
    `hbm_algorithmic` on SURVEY 8(d) bytes), never as `frac`."""
    e = profile_entry(cfg, p)
    hbm, hbm_src = peaks()
    alg = {"bytes_per_launch": bytes_launch, "achieved_gbs": bytes_launch / launch_s / 1e9,
           "ratio_to_hbm_peak": bytes_launch / launch_s / 1e9 / hbm,
           "note": "SURVEY 8(d) algorithmic bytes (every edge's packed m/2-byte row) per launch / launch time; "
                   "> 1 because each row is gathered once per block of its 16-node group cover and served from L2 -- not a roofline"}
    if not e or not e.get("warp_instructions_issued"):
        return {"bound": "hbm", "achieved": None, "peak": hbm, "unit": "GB/s", "frac": None, "traffic": None,
                "note": "no committed ncu summary for this config (profiles/union_ncu_summary.json)"}, alg
    try:
        import torch
        sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    except Exception:
        sms = 148
    clk = (sm_mhz or e["sm_clock_ghz"] * 1e3) * 1e6
    peak = 4.0 * sms * clk
    achieved = e["warp_instructions_issued"] / launch_s
    traffic = e.get("dram_bytes_per_launch")
    stale = abs(launch_s * 1e3 - e["duration_ms"]) / e["duration_ms"] > 0.15
    return {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "warp-instructions/s",
            "frac": achieved / peak, "traffic": traffic,
            "dram_frac": (traffic / launch_s / 1e9 / hbm) if traffic else None, "hbm_peak_gbs": hbm,
            "hbm_peak_source": hbm_src,
            "pipes_pct_ncu": {k: e.get(k) for k in ("issue_active_pct", "alu_pipe_pct", "fma_pipe_pct",
                                                     "lsu_pipe_pct", "l1_throughput_pct", "l2_hit_rate_pct")},
            "warp_instructions_per_launch": e["warp_instructions_issued"], "launch_ms": launch_s * 1e3,
            "ncu_duration_ms": e["duration_ms"], "profile_stale": stale, "source": e.get("source"),
            "peak_def": f"1 warp-instruction/cycle/SMSP x 4 x {sms} SMs x {clk / 1e6:.0f} MHz (SM clock sampled "
                        f"in the timed region)"}, alg


# ------------------------------------------------------------------ CPU (reference) arm
def cpu_sample(g, p, target_s, threads):
    """Times iterate_once (t=1) of the reference CPU path over a node sample."""
    import oracle
    O = oracle.reference() if oracle.reference_available() else oracle.port()
    n = g.n
    cur, c0 = O.hb_init(n, p)
    nxt = np.zeros_like(cur)
    c1, sd, sd2 = np.zeros(n), np.zeros(n), np.zeros(n)
    mid = n // 2
    k = max(threads, 64)
    while True:  # calibrate
        v0, v1 = mid, min(n, mid + k)
        t0 = time.perf_counter()
        O.hb_iterate(g, p, 1, cur, nxt, c0, c1, sd, sd2, v0=v0, v1=v1, threads=threads)
        dt = time.perf_counter() - t0
        if dt > target_s / 8 or v1 == n:
            break
        k *= 4
    k = min(n - mid, max(1, int(k * target_s / max(dt, 1e-6))))
    v0, v1 = mid, mid + k
    edges = int(g.degrees[v0:v1].sum(dtype=np.uint64))
    return O, (v0, v1), edges, (cur, nxt, c0, c1, sd, sd2)


def run_cpu(g, p, target_s, threads, reps=1):
    O, (v0, v1), edges, bufs = cpu_sample(g, p, target_s, threads)
    cur, nxt, c0, c1, sd, sd2 = bufs
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.hb_iterate(g, p, 1, cur, nxt, c0, c1, sd, sd2, v0=v0, v1=v1, threads=threads)
        times.append(time.perf_counter() - t0)
    m = 1 << p
    return {
        "value": edges * m / statistics.median(times), "unit": UNIT, "cores": threads, "kind": O.kind,
        "cpu_model": cpu_model(), "nproc": os.cpu_count(),
        "sample": sample_text(v0, v1, edges, p, threads) + f", median of {reps} ({statistics.median(times):.2f} s)",
        "seconds": times,
    }


def sample_text(v0, v1, edges, p, threads):
    return (f"iterate_once (t=1) over nodes [{v0},{v1}) = {v1 - v0} nodes / {edges} edges of the same graph, "
            f"p={p}, {threads} threads (parallel_ranges). Representative of every pass: the reference's "
            f"iterate_once unions all neighbour rows whatever t is (SPEC.md:427-435), so its time per "
            f"edge does not depend on the iteration")


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    g = build_graph_reference(args.config, threads)
    O, (v0, v1), edges, bufs = cpu_sample(g, args.p, args.cpu_step_s, threads)
    cur, nxt, c0, c1, sd, sd2 = bufs
    for _ in range(args.warmup):
        O.hb_iterate(g, args.p, 1, cur, nxt, c0, c1, sd, sd2, v0=v0, v1=v1, threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.hb_iterate(g, args.p, 1, cur, nxt, c0, c1, sd, sd2, v0=v0, v1=v1, threads=threads)
        times.append(time.perf_counter() - t0)
    m = 1 << args.p
    v = edges * m / statistics.mean(times)
    cb = {"value": v, "unit": UNIT, "cores": threads, "kind": O.kind, "cpu_model": cpu_model(),
          "nproc": os.cpu_count(), "sample": sample_text(v0, v1, edges, args.p, threads)}
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic", "config": workload_config(args, g),
        "run": {"register_layout": "reference packed 4-bit (hll.hpp:31-32)",
                "parallelism": f"{threads} host threads (parallel_ranges)",
                "graph_generator": "oracle/sb_synth.c (byte-identical to the product generator)",
                "ops": O._opsname().decode() if O.kind == "reference" else "port"},
        "cpu_baseline": cb, "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    line["run"]["repo_libraries_mapped"] = repo_libraries_mapped()
    print(json.dumps(line), flush=True)
    return 0


def repo_libraries_mapped():
    """Shared objects under this repository mapped by this process (the reference arm
    must show only oracle/ ones)."""
    out = set()
    try:
        with open("/proc/self/maps") as f:
            for ln in f:
                path = ln.split()[-1] if ln.rstrip().endswith(".so") else ""
                if path.startswith(ROOT):
                    out.add(os.path.relpath(path, ROOT))
    except OSError:
        pass
    return sorted(out)


def workload_config(args, g):
    """Identical in both arms: only what defines the workload."""
    return {
        "workload": CONFIGS[args.config][7] + f", p={args.p}, depth {'unbounded' if not args.depth else args.depth}",
        "config": args.config, "nodes": g.n, "edges": g.edges, "stream_bytes": g.stream_len, "p": args.p,
        "depth_limit": args.depth or None,
        "l2": "inputs larger than L2 (4.8 GB CSR stream read every iteration; 121 MB plane)" if args.config == "c3"
        else "small graph",
    }


def pipeline_variant(args, P, device, hb_ref):
    """cmd_build_graph + cmd_analyze (BFS part) entirely on one GPU; wall seconds per phase."""
    import torch
    from paper_2604_08374_b200 import DeviceGraph, HyperBall, grid_mask
    r, c, k, a, b, seed, rad2, _ = CONFIGS[args.config]
    mask = grid_mask(r, c, k, a, b, seed)
    DeviceGraph.from_grid(grid_mask(16, 16, 0, 1, 1, 1), 9, device)  # warm the build kernels
    out = {"input": f"{r}x{c} obstacle mask ({mask.size} B H2D)",
           "timing": "host wall clock per phase, best of 2 (synchronous C-ABI calls)"}
    modes = ("interval", "dense")
    for mode in modes + modes:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dg = DeviceGraph.from_grid(mask, rad2, device)
        t1 = time.perf_counter()
        h = HyperBall(dg, P, args.depth or None, interval=(mode == "interval"))
        it = h.run()
        t2 = time.perf_counter()
        met = h.metrics(dg.node_count_of_component(), dg.degrees())
        t3 = time.perf_counter()
        same = bool(np.array_equal(h.state().sum_d, hb_ref.state().sum_d))
        rec = {"build_s": t1 - t0, "hyperball_s": t2 - t1, "metrics_s": t3 - t2, "total_s": t3 - t0,
               "iterations": it, "sum_d_identical_to_uploaded_graph": same,
               "md_mean": float(np.nanmean(met["md"]))}
        if args.local:
            t4 = time.perf_counter()
            dg.local_metrics()
            rec["local_metrics_s"] = time.perf_counter() - t4
        if mode in out:  # keep the faster of the two runs per field (timings only)
            prev = out[mode]
            for k, v in rec.items():
                if k.endswith("_s"):
                    prev[k] = min(prev[k], v)
            prev["sum_d_identical_to_uploaded_graph"] &= same
        else:
            out[mode] = rec
        del h, dg
    log(f"[bench] pipeline: {json.dumps(out)}")
    return out


# ------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--p", type=int, default=10)
    ap.add_argument("--depth", type=int, default=None,
                    help="depth limit d (0 = unbounded); default: the config's (C1: 3, C2/C3: full depth)")
    ap.add_argument("--cpu-sample-s", type=float, default=15.0)
    ap.add_argument("--cpu-step-s", type=float, default=6.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (1 run, no extras)")
    ap.add_argument("--no-pipeline", action="store_true", help="skip the grid -> device graph -> HyperBall pipeline")
    ap.add_argument("--local", action="store_true", help="also time the exact local metrics (slow on c3)")
    args = ap.parse_args()
    if args.depth is None:
        args.depth = DEFAULT_DEPTH.get(args.config, 0)
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    import torch.distributed as dist
    from paper_2604_08374_b200 import DeviceGraph, HllParams, HyperBall
    from paper_2604_08374_b200.distributed import (attach_peers, init_comm, reset_external_barrier,
                                                   run_external_barrier, sharded_hyperball)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = max(torch.cuda.device_count(), 1)
    local = local_rank % ndev
    # More ranks than GPUs (a functional run of the sharded path on a 1-GPU lease):
    # NCCL refuses two ranks on one device, so the rows travel as fused P2P stores
    # over CUDA IPC and a gloo all-reduce of the max increase is the iteration barrier.
    shared = world > ndev
    torch.cuda.set_device(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    g = build_graph(args.config, threads=max(1, (os.cpu_count() or 1) // max(world, 1)))
    P = HllParams(args.p)
    m = P.m
    bounds = g.partition(world)
    v0, v1 = int(bounds[rank]), int(bounds[rank + 1])

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    comm = None if shared else init_comm(rank, world, local)

    def make_hb(skip=False):
        return sharded_hyperball(g, P, args.depth or None, rank, world, local, comm, skip, bounds,
                                 external_barrier=shared)

    t0 = time.perf_counter()
    hb = make_hb()
    log(f"[bench] rank {rank}: upload+validate+init {time.perf_counter() - t0:.2f} s, items={hb.graph.n_items} "
        f"chunk={hb.graph.chunk}")
    stream = torch.cuda.ExternalStream(hb.stream_handle())

    def one_run(h):
        if shared:
            reset_external_barrier(h)
            return run_external_barrier(h)
        h.reset()
        return h.run()

    for _ in range(args.warmup if not args.profile else 1):
        iters = one_run(hb)
    if args.profile:
        log(f"[bench] profile run done: {iters} iterations")
        return 0
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    union_ms = []
    ev0.record(stream)
    for _ in range(args.steps):
        iters = one_run(hb)
    ev1.record(stream)
    ev1.synchronize()
    barrier()
    union_ms = [s["union_ms"] for s in hb.stats()]  # the last timed run (every run is identical)
    # (single process only: extra runs on one rank would desynchronise the collectives)
    clock_info = clocks.stop(keep_busy=(lambda: (one_run(hb), torch.cuda.synchronize())) if world == 1 else None)
    dev_s = max_over_ranks(ev0.elapsed_time(ev1) / 1e3)
    st = hb.stats()
    total_updates = args.steps * iters * g.edges * m
    value = total_updates / dev_s
    bytes_iter = alg_bytes_per_iter(g.n, g.edges, g.stream_len, args.p)
    # roofline of the dominant kernel (rank-local work / rank-local launch time)
    el = hb.graph.edges_local
    nl = hb.graph.n_local
    bytes_launch = hb.graph.stream_bytes_local + 8 * (nl + 1) + 4 * nl + el * P.row_bytes + 2 * nl * P.row_bytes
    avg_union_s = statistics.mean(union_ms) / 1e3
    achieved = bytes_launch / avg_union_s / 1e9
    log(f"[bench] {args.steps} runs x {iters} iterations in {dev_s:.3f} s; union avg {avg_union_s * 1e3:.2f} ms "
        f"-> {achieved:.0f} GB/s algorithmic")
    for s in st:
        log(f"[bench]   t={s['t']} union={s['union_ms']:.2f} ms est={s['estimate_ms']:.3f} ms "
            f"xchg={s['exchange_ms']:.3f} ms changed={s['changed_nodes']} max_inc={s['max_increase']:.3f}")

    # passes executed (Alg. 1 stops one pass after the last change) vs last changing pass
    last_changing = max_over_ranks(float(max([s["t"] for s in st if s["changed_nodes"] > 0], default=0)))
    from paper_2604_08374_b200.distributed import gather_to_root
    sd_all = gather_to_root(hb.state().sum_d, bounds, rank, world)  # identical for every N
    sum_d_sha = hashlib.sha256(sd_all.tobytes()).hexdigest() if rank == 0 else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dev_s / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload_config(args, g),
        "run": {"iterations": iters, "last_changing_pass": int(last_changing), "sum_d_sha256": sum_d_sha,
                "register_layout": "4-bit bit-sliced (reference density m/2 B per row)",
                "parallelism": f"node-range shards x{world}"},
        "end_to_end_s_device": dev_s / args.steps,
        "roofline": None,  # filled below (needs the sampled SM clock)
        "per_iteration_ms": [round(s["step_ms"], 3) for s in st],
        "exchange_ms": [round(s["exchange_ms"], 4) for s in st] if world > 1 else None,
        "exchange": getattr(hb, "exchange_mode", None) if world > 1 else None,
        "shared_device": ({"ranks": world, "gpus": ndev, "note": "functional run of the sharded path: ranks share "
                           "a GPU, so this is not a scaling point"} if shared else None),
        "clocks": clock_info,
        "gpu_launches": args.steps * (2 + 2 * iters),
    }

    # ---- end to end through the public API with host buffers
    if not args.no_e2e:
        t_pin = time.perf_counter()
        g.pin(True)  # page-lock the host CSR (a caller-side, once-per-graph cost)
        pin_s = time.perf_counter() - t_pin
        h2d = g.stream_len + 8 * (g.n + 1) + 4 * g.n
        d2h = 4 * 8 * nl + nl  # state(): c_t, c_(t-1), sum_d, sum_d2 (f64) + changed flags (u8)
        def e2e_once():
            t = time.perf_counter()
            dg = DeviceGraph(g, local, (v0, v1), async_upload=True)
            h = HyperBall(dg, P, args.depth or None)
            if shared:
                attach_peers(h, rank, world, bounds)
                it = run_external_barrier(h)
            else:
                if comm is not None:
                    h.attach_comm(comm, bounds)
                it = h.run()
            s = h.state()  # D2H c_t, c_(t-1), sum_d, sum_d2, changed
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            if shared:
                dist.barrier()  # no peer still holds this rank's IPC-exported planes
            del h, dg, s
            return dt, it
        cold_s, _ = e2e_once()  # first call: the device pool grows by the stream + planes
        cold_s = max_over_ranks(cold_s + pin_s)
        barrier()
        e2e_t = []
        for _ in range(args.steps):
            dt, it = e2e_once()
            e2e_t.append(dt)
        barrier()
        e2e_s = max_over_ranks(statistics.mean(e2e_t))
        line["e2e"] = {"value": iters * g.edges * m / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h, "seconds_per_step": e2e_s,
                       "path": "sb_graph_create_async(host CSR, pinned; chunked H2D + validation overlapped "
                               "with the first union pass) + sb_hb_create + sb_hb_run + sb_hb_read_state",
                       "warm": "mean of the timed calls: device buffers come from the retained pool, host CSR "
                               "already page-locked",
                       "cold": {"seconds": cold_s, "value": iters * g.edges * m / cold_s,
                                "includes": "page-locking the host CSR + the first call's pool allocation "
                                            "(the CUDA context already exists)"}}
        line["end_to_end_s"] = e2e_s
        g.pin(False)

    # ---- variant: skip unchanged neighbours (bit-exact; reported separately)
    if not args.no_variants:
        hs = make_hb(skip=True)
        one_run(hs)
        barrier()
        t = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2 = torch.cuda.ExternalStream(hs.stream_handle())
        e0.record(s2)
        its = one_run(hs)
        e1.record(s2)
        e1.synchronize()
        sk = max_over_ranks(e0.elapsed_time(e1) / 1e3)
        same = bool(np.array_equal(hs.state().sum_d, hb.state().sum_d))
        line["variants"] = {"skip_unchanged": {
            "seconds_per_run": sk, "iterations": its, "dense_equivalent_updates_per_s": its * g.edges * m / sk,
            "sum_d_identical_to_dense": same,
            "per_iteration_union_ms": [round(s["union_ms"], 3) for s in hs.stats()],
            "note": "gathers only neighbours whose registers changed last iteration; not used for value/roofline"}}
        del hs
        hi = sharded_hyperball(g, P, args.depth or None, rank, world, local, comm, False, bounds, interval=True,
                               external_barrier=shared)
        one_run(hi)
        barrier()
        s3 = torch.cuda.ExternalStream(hi.stream_handle())
        e0.record(s3)
        iti = one_run(hi)
        e1.record(s3)
        e1.synchronize()
        ti = max_over_ranks(e0.elapsed_time(e1) / 1e3)
        line["variants"]["interval"] = {
            "seconds_per_run": ti, "iterations": iti, "dense_equivalent_updates_per_s": iti * g.edges * m / ti,
            "sum_d_identical_to_dense": bool(np.array_equal(hi.state().sum_d, hb.state().sum_d)),
            "per_iteration_union_ms": [round(s["union_ms"], 3) for s in hi.stats()],
            "note": "runs of consecutive ids folded with 2 sparse-table rows (per-iteration table build "
                    "included); bit-exact; reported separately from value/roofline"}
        del hi
        if not args.no_e2e and world == 1:
            # the same end-to-end path as `e2e` (host CSR -> HBM -> run -> read-back) in interval
            # mode: the run index needs the whole stream, so the upload is not hidden here
            g.pin(True)

            def e2e_interval():
                t = time.perf_counter()
                dg = DeviceGraph(g, local, (v0, v1), async_upload=True)
                h = HyperBall(dg, P, args.depth or None, interval=True)
                it = h.run()
                sd = h.state().sum_d
                torch.cuda.synchronize()
                dt = time.perf_counter() - t
                del h, dg
                return dt, it, sd

            e2e_interval()
            ts = [e2e_interval() for _ in range(max(args.steps, 3))]
            es = statistics.mean(t for t, _, _ in ts)
            line["variants"]["interval"]["e2e"] = {
                "seconds_per_step": es, "dense_equivalent_updates_per_s": ts[-1][1] * g.edges * m / es,
                "sum_d_identical_to_dense": bool(np.array_equal(ts[-1][2], hb.state().sum_d)),
                "h2d_bytes_per_step": g.stream_len + 8 * (g.n + 1) + 4 * g.n,
                "path": "sb_graph_create_async + sb_hb_create(SB_HB_INTERVAL) (waits for the upload, builds "
                        "the run index) + sb_hb_run + sb_hb_read_state"}
            g.pin(False)

    # ---- paper pipeline on the device: raster obstacle mask -> visibility graph built in HBM
    # (sb_graph_build_grid) -> HyperBall -> BFS metrics; the only H2D copy is the mask.
    if not args.no_pipeline and world == 1:
        line["pipeline"] = pipeline_variant(args, P, local, hb)

    # ---- CPU baseline (rank 0, N=1)
    if not args.no_cpu and world == 1 and rank == 0:
        try:
            line["cpu_baseline"] = run_cpu(g, args.p, args.cpu_sample_s, os.cpu_count() or 1)
            line["cpu_baseline"].pop("seconds", None)
            one = run_cpu(g, args.p, min(5.0, args.cpu_sample_s), 1)  # per-core figure
            line["cpu_baseline"]["per_core"] = {"value": one["value"], "cores": 1, "sample": one["sample"]}
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "error": repr(e)}
    line["roofline"], line["hbm_algorithmic"] = roofline_of(args.config, args.p, avg_union_s, bytes_launch,
                                                            clock_info.get("sm_mhz"))
    line["roofline"]["kernel"] = f"sb::union_kernel<{args.p}> (fused decode-union, 16-node group path)"
    line["hbm_algorithmic"]["whole_run_gbs"] = bytes_iter * iters * args.steps / dev_s / 1e9
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
