#!/usr/bin/env python
"""bench.py — throughput of the hot path (paren_match + tree_bbox) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    (N > 1: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N)

Workload (BASELINE.json metric "G elements/s for paren_match+tree_bbox"): the
paper's random push/pop stream (configs[4], "random-depth stream"),
synthetic, 2^27 elements per GPU (weak scaling; N = 8 is the 1B-element
stream), 50 % leaves, 75 % of opens are clips, unbalanced tail kept.  One
step = paren_match_tree_bbox over the resident stream: match / parent (as
paren_match) and node_bbox (as tree_bbox_matched on them) in one device call,
the box reduce pass overlapped with paren_match; N > 1: the sharded
paren_match then tree_bbox_matched.  Inputs (2.2 GB
per GPU) exceed the 126 MB L2, so no flush between steps.

Printed (rank 0, one JSON line): value = elements x steps / max-over-ranks
device time; roofline of the dominant kernel (algorithmic bytes / its
event-timed duration vs the measured HBM copy peak); cpu_baseline = the
oracle (single thread) on the host; e2e = the same metric through the
host-buffer C-ABI calls (H2D + D2H inside the timed region).
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
BYTES_PM = 9     # 1 B tag in, 4 B match + 4 B parent out
BYTES_TB = 41    # tree_bbox_matched: 1 B tag + 16 B box + 4 B match + 4 B parent in, 16 B box out
BYTES_PAIR = 41  # the step's own inputs and outputs: 1 B tag + 16 B box in; 4 + 4 + 16 B out


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
    return ap.parse_args()


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

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
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


def profile_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return {}


# ----------------------------------------------------------------------------
# reference arm: the oracle on host cores
# ----------------------------------------------------------------------------
def bench_config(args, world):
    """The workload description shared by both arms (the reference arm times a
    bounded sample of it, described in its cpu_baseline)."""
    return {"workload": f"C5 random-depth walk stream, 2^{args.log2n} elements per GPU "
                        f"(global stream {world} x 2^{args.log2n}); 50% leaves, 75% clips",
            "n_per_gpu": 1 << args.log2n, "seed": args.seed,
            "l2": "inputs (2.2 GB/GPU) larger than L2; no flush",
            "parallelism": f"contiguous shards x{world}" if world > 1 else "single GPU"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    import numpy as np
    import oracle
    import scenegen
    log2s = min(args.log2n, 24)
    ns = 1 << log2s
    tags = scenegen.walk_tags(ns, args.seed).numpy()
    boxes = scenegen.boxes(ns, args.seed, torch.from_numpy(tags)).numpy()
    match = np.empty(ns, np.int32)
    parent = np.empty(ns, np.int32)
    out = np.empty((ns, 4), np.float32)

    def step():
        oracle.paren_match(tags, match, parent)
        oracle.tree_bbox(tags, boxes, out)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    value = ns * args.steps / dt / 1e9
    sample = (f"first 2^{log2s} elements of the bench stream per step (the oracle, oracle/oracle.c -O2, "
              f"is sequential; its time is linear in the elements)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "i32/f32",
        "data": "synthetic",
        "config": bench_config(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
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
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import paper_2205_11659_b200 as tb
    import scenegen
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    lib = tb.load()
    lib.tb_launch_count.restype = ctypes.c_longlong
    lib.tb_profile_read.argtypes = [ctypes.c_char_p, ctypes.c_size_t]

    n = 1 << args.log2n
    offset = rank * n
    s_before = sum(scenegen.walk_step_sum(n, args.seed, offset=r * n, device=dev) for r in range(rank))
    tags = scenegen.walk_tags(n, args.seed, device=dev, offset=offset, s_before=s_before)
    boxes = scenegen.boxes(n, args.seed, tags, offset=offset, device=dev)
    match = torch.empty(n, dtype=torch.int32, device=dev)
    parent = torch.empty(n, dtype=torch.int32, device=dev)
    out = torch.empty((n, 4), dtype=torch.float32, device=dev)
    shard = None
    if world > 1:
        shard = tb.ShardContext(world, rank, offset, n)

    def step():
        if shard is None:
            tb.paren_match_tree_bbox(tags, boxes, match, parent, out)
        else:
            shard.paren_match(tags, match, parent)
            shard.tree_bbox_matched(tags, boxes, match, parent, out)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev.index if dev.index is not None else 0)
    clocks.start()
    launches0 = lib.tb_launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    launches = lib.tb_launch_count() - launches0
    ms = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    barrier()
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = world * n * args.steps / (ms / 1e3) / 1e9

    # --- roofline: per-kernel event timing over a second run of the same steps
    lib.tb_profile_enable(1)
    lib.tb_profile_read(None, 0)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    buf = ctypes.create_string_buffer(1 << 16)
    lib.tb_profile_read(buf, len(buf))
    lib.tb_profile_enable(0)
    per_kernel = json.loads(buf.value.decode() or "{}")
    alg_bytes = {"pm_finish": BYTES_PM * n, "pm_reduce": 1 * n, "bbm_main": BYTES_TB * n, "bbm_reduce": 5 * n,
                 "bb_finish": 33 * n, "bb_reduce": 1 * n}
    dom = max(per_kernel.items(), key=lambda kv: kv[1][1])[0] if per_kernel else "bbm_main"
    cnt, tot_ms = per_kernel.get(dom, [1, float("nan")])
    avg_ms = tot_ms / max(cnt, 1)
    peak, peak_src = measured_peak()
    achieved = alg_bytes.get(dom, BYTES_TB * n) / (avg_ms / 1e3) / 1e9
    traffic = profile_traffic().get(dom)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "kernel_ms": avg_ms,
                "step_share": tot_ms / max(sum(v[1] for v in per_kernel.values()), 1e-9),
                "per_kernel_ms": {k: v[1] / max(v[0], 1) for k, v in per_kernel.items()}}

    # --- e2e through the host-buffer C ABI
    e2e = None
    if not args.no_e2e:
        h_tags = tags.cpu().pin_memory()
        h_boxes = boxes.cpu().pin_memory()
        h_match = torch.empty(n, dtype=torch.int32).pin_memory()
        h_parent = torch.empty(n, dtype=torch.int32).pin_memory()
        h_out = torch.empty((n, 4), dtype=torch.float32).pin_memory()
        e_steps = max(1, min(args.steps, 3))

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
                       "pinned H2D + ShardContext.paren_match/tree_bbox + D2H")}

    # --- oracle on the host (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import numpy as np
        import oracle
        ht = tags.cpu().numpy()
        hb = boxes.cpu().numpy()
        m_ = np.empty(n, np.int32)
        p_ = np.empty(n, np.int32)
        o_ = np.empty((n, 4), np.float32)
        t0 = time.perf_counter()
        oracle.paren_match(ht, m_, p_)
        oracle.tree_bbox(ht, hb, o_)
        dt = time.perf_counter() - t0
        cpu = {"value": n / dt / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"the full bench workload (2^{args.log2n} elements), one pass of both oracle walks",
               "seconds": dt, "host_cpus": os.cpu_count()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "i32/f32", "data": "synthetic",
            "config": bench_config(args, world),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
            "pair_bytes_per_elem": BYTES_PAIR,
            "pair_hbm_frac": BYTES_PAIR * n * world / (ms_per_step / 1e3) / 1e9 / (peak * world),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
