#!/usr/bin/env python
"""bench.py — throughput of the hot path (paren_match + tree_bbox) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    (N > 1: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N)

Workload (BASELINE.json metric "G elements/s for paren_match+tree_bbox"): the
paper's random push/pop stream (configs[4], "random-depth stream"),
synthetic, 2^27 elements per GPU (weak scaling; N = 8 is the 1B-element
stream), 50 % leaves, 75 % of opens are clips, unbalanced tail kept.  One
step = paren_match_tree_bbox over the resident stream: match, parent and
node_bbox from one fused tile pass (csrc/fused.cu); N > 1: the sharded
paren_match then tree_bbox_matched.  Inputs (2.2 GB per GPU) exceed the 126 MB
L2, so no flush between steps.  --config C2|C3|C3L|C4 times another config of
SURVEY §8(d) on one GPU (with an L2 flush between steps when it fits in L2).

Printed (rank 0, one JSON line): value = elements x steps / max-over-ranks
device time; roofline of the dominant kernel (algorithmic bytes / its
event-timed duration vs the measured HBM copy peak); calls = paren_match,
tree_bbox and the pair timed separately (SURVEY §8(d) bytes: 9, 33, 42 per
element, fractions of 8 TB/s and of the measured peak); cpu_baseline = the
oracle (one pinned host thread, median of 3); e2e = the same metric through the
host-buffer C-ABI call (H2D + D2H inside the timed region).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

METRIC = "G elements/s for paren_match+tree_bbox"
UNIT = "Gelem/s"
BYTES_PM = 9     # paren_match: 1 B tag in, 4 B match + 4 B parent out
BYTES_TB = 33    # tree_bbox: 1 B tag + 16 B box in, 16 B box out
BYTES_PAIR = 42  # paren_match + tree_bbox as two calls
NOMINAL_GBS = 8000.0  # the north star's roofline denominator (8 TB/s)
# algorithmic bytes per element of each kernel (its share of the path's own
# inputs / outputs; workspace traffic is not algorithmic and shows up in traffic)
KERNEL_BYTES = {"fz_main": 41,     # tags + boxes in; match, parent, node_bbox out (the fused pass)
                "fz_reduce": 1,    # tags
                "pm_finish": 9, "pm_reduce": 1, "bbm_main": 33, "bbm_reduce": 1}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--log2n", type=int, default=27, help="elements per GPU = 2^log2n")
    ap.add_argument("--seed", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--config", default="C5", help="C5 (default, the metric's workload) or C2/C3/C3L/C4 (one GPU)")
    ap.add_argument("--no-calls", action="store_true", help="skip the separate paren_match / tree_bbox timings")
    return ap.parse_args()


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def pin_one_core():
    """Pin this process to one core for the oracle timing (restored after)."""
    try:
        old = os.sched_getaffinity(0)
        core = min(old)
        os.sched_setaffinity(0, {core})
        return old, core
    except Exception:
        return None, None


# ----------------------------------------------------------------------------
# clocks sampled during the timed region
# ----------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()
        # the timed region starts once nvidia-smi is sampling (a short region
        # would otherwise end before its first sample)
        t0 = time.time()
        while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
            time.sleep(0.01)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        n0 = len(self.lines)
        t0 = time.time()  # at least one sample at or after the end of the region
        while len(self.lines) <= n0 and time.time() - t0 < 1.0 and self.proc.poll() is None:
            time.sleep(0.01)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def profile_traffic(config="C5"):
    """DRAM bytes per launch of each kernel from the committed ncu launch list
    of this config (profiles/traffic.json for C5, traffic_<config>.json else)."""
    c = config.upper()
    path = os.path.join(ROOT, "profiles", "traffic.json" if c == "C5" else f"traffic_{c}.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return {}


# ----------------------------------------------------------------------------
# reference arm: the oracle on host cores
# ----------------------------------------------------------------------------
def bench_config(args, world, n=None, desc=None):
    """The workload description shared by both arms (the reference arm times a
    bounded sample of it, described in its cpu_baseline)."""
    if args.config.upper() != "C5":
        return {"workload": desc or args.config, "n_per_gpu": n, "config": args.config.upper(),
                "l2": "L2 flushed (512 MB write) before every timed step" if n * 17 < (256 << 20)
                else "inputs larger than L2; no flush",
                "parallelism": "single GPU"}
    return {"workload": f"C5 random-depth walk stream, 2^{args.log2n} elements per GPU "
                        f"(global stream {world} x 2^{args.log2n}); 50% leaves, 75% clips",
            "n_per_gpu": 1 << args.log2n, "seed": args.seed, "config": "C5",
            "l2": "inputs (2.2 GB/GPU) larger than L2; no flush",
            "parallelism": f"contiguous shards x{world}" if world > 1 else "single GPU"}


def make_inputs(args, rank, world, dev):
    """Tags / boxes of the timed config, generated on the device (seeded)."""
    import scenegen
    if args.config.upper() != "C5":
        tags, info = scenegen.config(args.config, device=dev)
        tags = tags.to(dev)
        n = tags.numel()
        boxes = scenegen.boxes(n, args.seed, tags, device=dev)
        return tags, boxes, n, info.get("workload")
    n = 1 << args.log2n
    offset = rank * n
    s_before = sum(scenegen.walk_step_sum(n, args.seed, offset=r * n, device=dev) for r in range(rank))
    tags = scenegen.walk_tags(n, args.seed, device=dev, offset=offset, s_before=s_before)
    boxes = scenegen.boxes(n, args.seed, tags, offset=offset, device=dev)
    return tags, boxes, n, None


def oracle_seconds(tags_np, boxes_np, reps):
    """The oracle (both walks) on one pinned host thread: median of reps runs."""
    import numpy as np
    import oracle
    n = len(tags_np)
    m_ = np.empty(n, np.int32)
    p_ = np.empty(n, np.int32)
    o_ = np.empty((n, 4), np.float32)
    old, core = pin_one_core()
    ts = []
    try:
        for _ in range(reps):
            t0 = time.perf_counter()
            oracle.paren_match(tags_np, m_, p_)
            oracle.tree_bbox(tags_np, boxes_np, o_)
            ts.append(time.perf_counter() - t0)
    finally:
        if old is not None:
            os.sched_setaffinity(0, old)
    return statistics.median(ts), core


def run_reference(args, rank, world):
    if rank != 0:
        return
    import scenegen
    dev = "cpu"
    if args.config.upper() != "C5":
        tags_t, info = scenegen.config(args.config)
        desc = info.get("workload")
    else:
        tags_t, desc = None, None
    if tags_t is None:
        log2s = min(args.log2n, 24)
        tags_t = scenegen.walk_tags(1 << log2s, args.seed)
        sample = (f"first 2^{log2s} elements of the bench stream per step (the oracle, oracle/oracle.c -O2, "
                  f"is sequential; its time is linear in the elements)")
    else:
        tags_t = tags_t[: 1 << 24].contiguous()
        sample = f"first {tags_t.numel()} elements of {args.config.upper()} per step"
    ns = tags_t.numel()
    tags = tags_t.numpy()
    boxes = scenegen.boxes(ns, args.seed, tags_t).numpy()
    import numpy as np
    import oracle
    match = np.empty(ns, np.int32)
    parent = np.empty(ns, np.int32)
    out = np.empty((ns, 4), np.float32)

    def step():
        oracle.paren_match(tags, match, parent)
        oracle.tree_bbox(tags, boxes, out)

    old, core = pin_one_core()
    try:
        for _ in range(args.warmup):
            step()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step()
        dt = time.perf_counter() - t0
    finally:
        if old is not None:
            os.sched_setaffinity(0, old)
    value = ns * args.steps / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "i32/f32",
        "data": "synthetic",
        "config": bench_config(args, world, None if args.config.upper() == "C5" else ns, desc),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model(), "pinned_core": core, "host_cpus": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.config.upper() != "C5":
        raise SystemExit("--config other than C5 runs on one GPU")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import paper_2205_11659_b200 as tb
    if world > 1:
        import torch.distributed as dist
        # the communicators' setup (ranks, transports, NVLS) on stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    lib = tb.load()
    lib.tb_launch_count.restype = ctypes.c_longlong
    lib.tb_profile_read.argtypes = [ctypes.c_char_p, ctypes.c_size_t]

    tags, boxes, n, desc = make_inputs(args, rank, world, dev)
    match = torch.empty(n, dtype=torch.int32, device=dev)
    parent = torch.empty(n, dtype=torch.int32, device=dev)
    out = torch.empty((n, 4), dtype=torch.float32, device=dev)
    shard = None
    if world > 1:
        shard = tb.ShardContext(world, rank, (1 << args.log2n) * rank, n)
    # inputs that fit in L2 get a 512 MB write between timed steps (outside the timing)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if n * 17 < (256 << 20) else None

    def step():
        if shard is None:
            tb.paren_match_tree_bbox(tags, boxes, match, parent, out)
        else:  # two fixed-size all-gathers, no host synchronisation (status checked after timing)
            shard.paren_match_tree_bbox(tags, boxes, match, parent, out, check=False)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def timed(fn, steps):
        """Device time of `steps` calls of fn (ms), CUDA events on this stream;
        with the L2 flush between calls when the inputs fit in L2."""
        if flush is None:
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(steps):
                fn()
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b)
        tot = 0.0
        for _ in range(steps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            tot += a.elapsed_time(b)
        return tot

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev.index if dev.index is not None else 0)
    clocks.start()
    launches0 = lib.tb_launch_count()
    ms = timed(step, args.steps)
    launches = lib.tb_launch_count() - launches0
    clk = clocks.stop()
    if shard is not None:
        shard.status()  # capacity overflow of any timed step would raise here
    barrier()
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = world * n * args.steps / (ms / 1e3) / 1e9
    peak, peak_src = measured_peak()

    # --- roofline: per-kernel event timing over a second run of the same steps
    lib.tb_profile_enable(1)
    lib.tb_profile_read(None, 0)
    for _ in range(args.steps):
        if flush is not None:
            flush.zero_()
        step()
    torch.cuda.synchronize()
    buf = ctypes.create_string_buffer(1 << 16)
    lib.tb_profile_read(buf, len(buf))
    lib.tb_profile_enable(0)
    per_kernel = json.loads(buf.value.decode() or "{}")
    dom = max(per_kernel.items(), key=lambda kv: kv[1][1])[0] if per_kernel else "fz_main"
    cnt, tot_ms = per_kernel.get(dom, [1, float("nan")])
    avg_ms = tot_ms / max(cnt, 1)
    kb = KERNEL_BYTES.get(dom, BYTES_PAIR)
    achieved = kb * n / (avg_ms / 1e3) / 1e9
    traffic = profile_traffic(args.config).get(dom)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "kernel_bytes_per_elem": kb, "kernel_ms": avg_ms,
                "frac_of_8TBs": achieved / NOMINAL_GBS,
                "step_share": tot_ms / max(sum(v[1] for v in per_kernel.values()), 1e-9),
                "per_kernel_ms": {k: v[1] / max(v[0], 1) for k, v in per_kernel.items()}}

    # --- the two calls of the north star timed separately, and the pair
    calls = None
    if not args.no_calls and shard is None:
        k = max(3, min(args.steps, 10))
        for _ in range(2):  # warm-up (workspace allocation of each call)
            tb.paren_match(tags, match, parent)
            tb.tree_bbox(tags, boxes, out)
        torch.cuda.synchronize()
        pm_ms = timed(lambda: tb.paren_match(tags, match, parent), k) / k
        tb_ms = timed(lambda: tb.tree_bbox(tags, boxes, out), k) / k

        def rec(nb, t):
            gbs = nb * n / (t / 1e3) / 1e9
            return {"ms": t, "Gelem_s": n / (t / 1e3) / 1e9, "bytes_per_elem": nb, "GBs": gbs,
                    "frac_of_8TBs": gbs / NOMINAL_GBS, "frac_of_measured": gbs / peak}
        calls = {"paren_match": rec(BYTES_PM, pm_ms), "tree_bbox": rec(BYTES_TB, tb_ms),
                 "pair_two_calls": rec(BYTES_PAIR, pm_ms + tb_ms),
                 "pair_fused_step": rec(BYTES_PAIR, ms_per_step)}

    # --- e2e through the host-buffer C ABI
    e2e = None
    if not args.no_e2e:
        h_tags = tags.cpu().pin_memory()
        h_boxes = boxes.cpu().pin_memory()
        h_match = torch.empty(n, dtype=torch.int32).pin_memory()
        h_parent = torch.empty(n, dtype=torch.int32).pin_memory()
        h_out = torch.empty((n, 4), dtype=torch.float32).pin_memory()
        e_steps = max(1, min(args.steps, 5))

        def estep():
            if shard is None:
                tb.paren_match_tree_bbox_host(h_tags, h_boxes, h_match, h_parent, h_out, device=dev)
            else:
                tags.copy_(h_tags, non_blocking=True)
                boxes.copy_(h_boxes, non_blocking=True)
                step()
                h_match.copy_(match, non_blocking=True)
                h_parent.copy_(parent, non_blocking=True)
                h_out.copy_(out, non_blocking=True)
                torch.cuda.current_stream(dev).synchronize()
        estep()
        torch.cuda.synchronize()
        barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(e_steps):
            estep()
        b.record()
        torch.cuda.synchronize()
        ems = a.elapsed_time(b)
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": world * n * e_steps / (ems / 1e3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 17 * n, "d2h_bytes_per_step": 24 * n,
               "steps": e_steps,
               "api": ("paren_match_tree_bbox_host (pinned host buffers)" if shard is None else
                       "pinned H2D + ShardContext.paren_match_tree_bbox + D2H")}

    # --- launch-bound configs (§8(d)): the same step replayed from a CUDA graph
    graph = None
    if shard is None and n <= (1 << 22):
        s2 = torch.cuda.Stream(dev)
        with torch.cuda.stream(s2):
            for _ in range(3):
                step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s2):
            step()
        torch.cuda.synchronize()
        k = max(args.steps, 20)
        gms = timed(g.replay, k) / k
        graph = {"ms_per_step": gms, "value": n / (gms / 1e3) / 1e9, "unit": UNIT, "steps": k}

    # --- oracle on the host (rank 0, N = 1 only): one pinned thread, median of 3
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sec, core = oracle_seconds(tags.cpu().numpy(), boxes.cpu().numpy(), 3)
        cpu = {"value": n / sec / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"the full bench workload ({n} elements), both oracle walks, median of 3 runs",
               "seconds": sec, "cpu_model": cpu_model(), "pinned_core": core, "host_cpus": os.cpu_count()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "i32/f32", "data": "synthetic",
            "config": bench_config(args, world, n, desc),
            "roofline": roofline,
            "calls": calls,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
            "graph": graph,
            "pair_bytes_per_elem": BYTES_PAIR,
            "pair_hbm_frac": BYTES_PAIR * n * world / (ms_per_step / 1e3) / 1e9 / (peak * world),
            "pair_frac_of_8TBs": BYTES_PAIR * n * world / (ms_per_step / 1e3) / 1e9 / (NOMINAL_GBS * world),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
