#!/usr/bin/env python
"""bench.py — one step = the whole hot path over one batch.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--kernel tc|alu]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
    python bench.py --impl reference ...      # the CPU oracle arm (rank 0 only)

Workload (N=1): BASELINE.json configs[3] ("config 4": N = 100,000 synthetic protein
sequences, k = 3, p = 8 shards/buckets), the largest config the metric is quoted on
that fits one GPU; at N > 1 the same 8 shards are spread over N GPUs (strong scaling,
p = 8 fixed, bit-identical output).

Prints ONE JSON line on rank 0 (see the bench contract in DESIGN.md §7).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "pairwise k-mer similarities/s (whole rank+partition step)"
UNIT = "pairs/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--p", type=int, default=None)
    ap.add_argument("--kernel", default="tc", choices=["tc", "tc1", "tc8", "tc81", "tcfull", "tc8full", "alu"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rank-mode", default="ga", choices=["ga", "samples"],
                    help="ga: rank vs the global ancestor (north star); samples: SURVEY f1, vs the k*p samples")
    ap.add_argument("--f1-cuda-cores", action="store_true",
                    help="with --rank-mode samples: the rank against the samples on the CUDA cores")
    ap.add_argument("--e2e-sequential", action="store_true",
                    help="e2e as separately timed sequential steps (default at N=1: the double-buffered Pipeline)")
    ap.add_argument("--tile-split", action="store_true",
                    help="f2 across GPUs (SAD_F_TILE_SPLIT): every rank holds the whole input, the all-pairs tiles "
                         "are split over the ranks, T all-reduced (use with --p 1 for the centralized rank)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--oracle-threads", type=int, default=0,
                    help="reference arm / cpu_baseline: oracle threads (0 = all host cores)")
    ap.add_argument("--no-graph", action="store_true",
                    help="time eager steps instead of one CUDA graph replay per step (world == 1)")
    return ap.parse_args()


def workload_name(spec, p):
    return (f"{spec.name}: N={spec.n} {spec.alphabet} k={spec.k} p={p}, {spec.n_families} families "
            f"({spec.family_sizes}), roots {spec.root_len}, sub U{spec.sub}, indel {spec.indel}, seed {spec.seed}")


def total_pairs(n, p):
    from synth import gen
    sb = gen.shard_bounds(n, p)
    return sum((sb[s + 1] - sb[s]) * (sb[s + 1] - sb[s] - 1) // 2 for s in range(p))


# ----------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg and --impl reference)
# ----------------------------------------------------------------------------------------

def oracle_sample(a, o, spec, p, seconds, threads=0):
    """Size a prefix of the workload (same p) so that one oracle run takes about `seconds` on
    all host threads: grow the prefix until a probe run takes >= seconds/4, then scale by the
    pairs' n^2 growth."""
    import oracle
    cores = oracle.threads(threads)
    N = len(o) - 1
    n_sub = min(N, max(p * p, 800))
    while True:
        t0 = time.perf_counter()
        oracle.run(a[: o[n_sub]], o[: n_sub + 1], spec.alphabet, spec.k, p, nthreads=threads)
        dt = time.perf_counter() - t0
        if dt >= seconds / 4 or n_sub >= N:
            break
        n_sub = min(N, int(n_sub * min(3.0, max(1.2, (seconds / 4 / max(dt, 1e-3)) ** 0.5))))
    n_sub = int(min(N, max(p * p, n_sub * (seconds / max(dt, 1e-3)) ** 0.5)))
    return n_sub, cores


def run_oracle(a, o, spec, p, n_sub, threads=0):
    import oracle
    t0 = time.perf_counter()
    oracle.run(a[: o[n_sub]], o[: n_sub + 1], spec.alphabet, spec.k, p, nthreads=threads)
    return time.perf_counter() - t0


# ----------------------------------------------------------------------------------------
# clocks during the timed region
# ----------------------------------------------------------------------------------------

REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, device: int):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_dev{device}.csv") if os.path.isdir(
            os.path.join(ROOT, "gpurun_out")) else f"/tmp/clocks_dev{device}_{os.getpid()}.csv"
        self.device = device

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], [], set()
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 3:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
                r = int(parts[2], 16)
            except ValueError:
                continue
            sm.append(s)
            mx.append(m)
            for bit, name in REASONS.items():
                if r & bit and name != "gpu_idle":
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------------------

def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` launched without torchrun: re-launch this command as N ranks (one per
    GPU) through torch.distributed.run; fail loudly when fewer than N GPUs are visible."""
    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(json.dumps({"error": f"--gpus {n} needs {n} visible GPUs, found {have}"}), flush=True)
        return 2
    port = 29500 + os.getpid() % 2000
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    from synth import gen
    spec = gen.SPECS[args.config]
    p = args.p or (8 if args.config in (2, 3, 4) else spec.p)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return reference_arm(args, spec, p, world, rank)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_0901_2742_b200.runtime import Context

    a, o = gen.generate(spec)
    n = len(o) - 1
    if p % world and not args.tile_split:
        raise SystemExit(f"p={p} must be a multiple of the GPU count {world}")
    pl = p if args.tile_split else p // world
    sb = gen.shard_bounds(n, p)
    lo, hi = (0, n) if args.tile_split else (sb[rank * pl], sb[(rank + 1) * pl])
    a_loc = np.ascontiguousarray(a[o[lo]: o[hi]])
    o_loc = np.ascontiguousarray(o[lo: hi + 1] - o[lo])
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.Stream(dev)          # the context's own stream (graph capture needs a non-default one)
    d_a = torch.from_numpy(a_loc).to(dev)
    d_o = torch.from_numpy(o_loc).to(dev)
    h_a = torch.from_numpy(a_loc).pin_memory()
    h_o = torch.from_numpy(o_loc).pin_memory()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)       # 256 MB > 126 MB L2

    # world > 1: the library's own NCCL communicator runs every exchange (collective API)
    ctx = Context(spec.alphabet, spec.k, p, world=world, rank=rank, device=local_rank, stream=stream,
                  kernel=args.kernel, group=group, rank_mode=args.rank_mode, comm=world > 1,
                  f1_cuda_cores=args.f1_cuda_cores, tile_split=args.tile_split)
    R_glob = int(o[-1])

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    R_loc = int(o_loc[-1])

    def step_device():
        ctx.load(d_a, d_o, n, lo, residues=R_loc)
        ctx.run(sync=False, residues_global=R_glob)

    h_keys = None

    def step_e2e():
        nonlocal h_keys
        ctx.load(h_a.numpy(), h_o.numpy(), n, lo)                   # H2D from pinned host memory
        sizes = ctx.run(residues_global=R_glob)
        keys = ctx.out_keys()
        if h_keys is None or h_keys.shape != keys.shape:
            h_keys = torch.empty(keys.shape, dtype=keys.dtype, pin_memory=True)
        h_keys.copy_(keys)                                           # D2H of the step's result (pinned)
        return h_keys, sizes

    def timed(fn, steps, post=None):
        ev = []
        for _ in range(steps):
            barrier()
            flush.fill_(1)                                          # L2 flush between timed steps (untimed)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            s.record(stream)
            fn()
            e.record(stream)
            ev.append((s, e))
            if post is not None:                                    # after the step (untimed)
                barrier()
                post()
        barrier()
        ms = sum(s.elapsed_time(e) for s, e in ev)
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    for _ in range(args.warmup):
        step_device()
    graph = None
    if world == 1 and not args.no_graph:
        # the whole device-resident step (load .. partition) as ONE CUDA graph: no host
        # synchronization and no launch gaps inside the step
        barrier()
        graph = ctx.capture_step(d_a, d_o, R_loc)
        with torch.cuda.stream(stream):
            graph.replay()
        barrier()

    def replay():
        with torch.cuda.stream(stream):
            graph.replay()

    ctx.reset_stats()
    clocks = ClockSampler(local_rank)
    clocks.start()
    if graph is not None:
        ms_dev = timed(replay, args.steps, post=ctx.graph_account)
    else:
        ms_dev = timed(step_device, args.steps)
    clk = clocks.stop()
    st = ctx.stats()
    launches = st["launches"]
    ap_ms = st["allpairs_ms_total"] / max(st["calls"], 1)
    op_ms = st["operand_ms_total"] / max(st["calls"], 1)
    # e2e through the public API with host buffers
    for _ in range(max(1, args.warmup // 2)):
        step_e2e()
    e2e_h2d = int(h_a.numel() + h_o.numel() * 8)
    keys, sizes_all = step_e2e()
    # a12: the library's load report (sad_get_load_report: largest bucket vs 2w + p, < 2w when p | w;
    # PAPER.md:188, reading A23)
    load = dict(ctx.load_report(), bucket_sizes=[int(x) for x in sizes_all])
    e2e_d2h = int(keys.numel() * 8 + p * 8)
    e2e_mode = "sequential: load (pinned H2D) .. partition .. D2H of the keys per step, L2 flushed between steps"
    if world == 1 and not args.e2e_sequential:
        # the public double-buffered path (runtime.Pipeline): two contexts on two streams, the H2D and
        # k-mer counts of step k+1 overlap the device work of step k; every step still copies its own
        # inputs in and its keys out. One timed region over all steps (no flush inside it: the
        # per-step working set, ~1 GB of operand and excess rows, is far above the 126 MB L2).
        from paper_0901_2742_b200.runtime import Pipeline
        pipe = Pipeline(spec.alphabet, spec.k, p, depth=2, device=local_rank, kernel=args.kernel,
                        rank_mode=args.rank_mode, f1_cuda_cores=args.f1_cuda_cores)
        for _ in range(2):
            pipe.submit(h_a.numpy(), h_o.numpy(), n, lo)
        for _ in range(2):
            pipe.collect()
        barrier()
        flush.fill_(1)
        barrier()
        s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for k in range(args.steps):
            pipe.submit(h_a.numpy(), h_o.numpy(), n, lo)
            if k >= 1:
                pipe.collect()
        pipe.collect()
        barrier()
        e0.record()
        e0.synchronize()
        ms_e2e = s0.elapsed_time(e0)
        pipe.close()
        e2e_mode = ("double-buffered (runtime.Pipeline, 2 contexts / 2 streams): per step pinned H2D of the "
                    "inputs + load .. partition + D2H of the keys, step k+1's copy overlapping step k; one timed "
                    "region over all steps")
    else:
        ms_e2e = timed(step_e2e, args.steps)

    pairs_job = total_pairs(n, p)
    ms_step = ms_dev / args.steps
    value = pairs_job / (ms_step / 1e3)
    e2e_value = pairs_job / (ms_e2e / args.steps / 1e3)

    # roofline of the dominant kernel (the all-pairs kernel, K5 / K5')
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    measured = {}
    try:
        measured = json.load(open(os.path.join(ROOT, "profiles", "peaks_b200.json")))
    except Exception:
        pass
    _, _, kcols = ctx.profile_info()
    s0 = 0 if args.tile_split else rank * pl
    w_loc = [sb[s0 + s + 1] - sb[s0 + s] for s in range(pl)]
    fp4 = args.kernel in ("tc", "tc1", "tcfull")
    if args.kernel.startswith("tc"):
        # algorithmic dense work of the threshold-indicator SYRK: 2 * K_s ops per pair i <= j
        # (SURVEY §8(d) f_tc numerator: sum_s w_s (w_s + 1) K_s)
        ops = sum(2 * (w * (w + 1) // 2) * int(k) for w, k in zip(w_loc, kcols))
        if args.tile_split:                # this rank's share of the tiles (LPT-balanced row blocks)
            ops //= world
        bf16 = peaks.get("bf16_tflops")
        if bf16:
            # primary: the driver-measured bf16 burst x the nominal dense ratio of the operand dtype
            # (fp4 : bf16 = 9 : 2.25 = 4; int8 : bf16 = 4.5 : 2.25 = 2), B200_PROFILING.md
            ratio = 4.0 if fp4 else 2.0
            peak = ratio * bf16
            src = (f"MEASURED_PEAKS.json bf16_tflops (burst, {bf16:.1f}) x nominal "
                   f"{'fp4' if fp4 else 'int8'}:bf16 = {ratio:g}")
        else:
            peak = 9000.0 if fp4 else 4500.0
            src = "nominal dense B200 peak (MEASURED_PEAKS.json absent)"
        roof = {"bound": "tensor", "achieved": ops / (ap_ms / 1e3) / 1e12, "peak": peak, "unit": "TOPS",
                "frac": None, "traffic": None, "peak_source": src}
        # the all-pairs STAGE (a3 = K3 + K4 + K6 + K5: operand build and the contraction), SURVEY §8(d)
        roof["stage_ms"] = ap_ms + op_ms
        roof["stage_frac"] = ops / ((ap_ms + op_ms) / 1e3) / 1e12 / peak
        # operand bytes the contraction streams (rows padded to 128, K padded to one 128-byte block)
        bpc = 0.5 if fp4 else 1.0
        roof["operand_bytes"] = int(sum(((w + 127) // 128) * 128 * ((int(k) + 255) // 256 * 256) * bpc
                                        for w, k in zip(w_loc, kcols)))
        # context: the same kernel against this B200's own measured ceilings
        if fp4 and "fp4_mma_only_tops" in measured:
            roof["frac_of_mma_issue_rate"] = roof["achieved"] / measured["fp4_mma_only_tops"]
            roof["mma_issue_rate_tops"] = measured["fp4_mma_only_tops"]
        if "int8_tops" in measured:
            roof["frac_of_cublas_int8" + ("_x2" if fp4 else "")] = roof["achieved"] / (
                (2.0 if fp4 else 1.0) * measured["int8_tops"])
        roof["frac_of_nominal"] = roof["achieved"] / (9000.0 if fp4 else 4500.0)
        # DRAM traffic of one launch: ncu --set full of the same kernel on this workload
        suffix = "" if args.config == 4 and (args.p or 8) == 8 else f"_cfg{args.config}" + ("" if args.p is None else f"_p{args.p}")
        for tag in ("r02", "r01"):
            tr = os.path.join(ROOT, "profiles", f"{tag}_ncu_syrk_{args.kernel}{suffix}_summary.csv")
            if os.path.exists(tr):
                break
        if os.path.exists(tr):
            vals = {}
            for line in open(tr):
                parts = line.strip().split(",")
                if len(parts) == 3:
                    vals[parts[0]] = parts
            try:
                def gb(k):
                    v, u = float(vals[k][1]), vals[k][2]
                    return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}[u]
                roof["traffic"] = gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum")
                roof["traffic_source"] = f"ncu --set full, one k_syrk_tc launch ({os.path.relpath(tr, ROOT)})"
            except Exception:
                pass
    else:
        vpad = ((ctx_V(spec) + 63) // 64) * 64
        ops = sum((w * (w + 1) // 2) * vpad for w in w_loc)   # one VIMNMX.U16x2 + one VIADD.U16x2 per 2 k-mers
        peak = 148 * 128 * (peaks.get("sm_max_mhz", 1965.0) * 1e6) / 1e12
        roof = {"bound": "alu", "achieved": ops / (ap_ms / 1e3) / 1e12, "peak": peak, "unit": "Tops",
                "frac": None, "traffic": None,
                "peak_source": "148 SMs x 128 int32 lanes x sm_max_mhz (DESIGN.md §5)"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["kernel_ms"] = ap_ms
    roof["operand_build_ms"] = op_ms

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_sub, cores = oracle_sample(a, o, spec, p, args.cpu_seconds, threads=args.oracle_threads)
        dt = run_oracle(a, o, spec, p, n_sub, threads=args.oracle_threads)
        cpu = {"value": total_pairs(n_sub, p) / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"oracle.run (full pipeline, p={p}) on the first {n_sub} sequences of the workload, "
                         f"{dt:.1f} s; value = that subset's within-shard pairs / time"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": {"tc": "e2m1", "tc1": "e2m1", "tcfull": "e2m1", "tc8": "i8", "tc81": "i8", "tc8full": "i8",
                                               "alu": "u16"}[args.kernel], "data": "synthetic",
            "config": {"workload": workload_name(spec, p), "p": p, "kernel": args.kernel, "rank_mode": args.rank_mode,
                       "step": ("one CUDA graph replay (sad_load .. sad_partition captured)" if graph is not None
                                else "eager C-ABI calls (sad_load, sad_build_profiles, sad_rank, sad_partition)"),
                       "exchange": ("ncclAllReduce of T (tile split, f2)" if args.tile_split and world > 1 else
                                    "library NCCL communicator (collective API)" if world > 1 else "none (G = 1)"),
                       "pairs_per_step": pairs_job,
                       "l2": "L2 flushed (256 MB write) before every timed step; operand working set > L2"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": e2e_h2d, "d2h_bytes_per_step": e2e_d2h,
                    "ms_per_step": ms_e2e / args.steps, "mode": e2e_mode},
            "allpairs_pairs_per_s": pairs_job / world / (ap_ms / 1e3) * world if ap_ms > 0 else None,
            "roofline": roof,
            "load_report": load,
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": int(launches) * args.steps,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def ctx_V(spec):
    return (20 if spec.alphabet == "protein" else 4) ** spec.k


def reference_arm(args, spec, p, world, rank):
    """The oracle timed as it stands on the host cores, on this arm's config/metric."""
    if rank != 0:
        return 0
    from synth import gen
    a, o = gen.generate(spec)
    per_step = max(2.0, min(8.0, 120.0 / max(args.steps + args.warmup, 1)))
    th = args.oracle_threads
    n_sub, cores = oracle_sample(a, o, spec, p, per_step, th)
    for _ in range(args.warmup):
        run_oracle(a, o, spec, p, n_sub, th)
    t = sum(run_oracle(a, o, spec, p, n_sub, th) for _ in range(args.steps))
    value = total_pairs(n_sub, p) / (t / args.steps)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic", "impl": "reference",
            "config": {"workload": workload_name(spec, p), "p": p},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"each step: oracle.run on the first {n_sub} sequences of the workload"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main() or 0)
