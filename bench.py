"""Benchmark: keys/s sorting int32 n = 2^26 on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--family uniform] [--n 67108864] [--families]

One step = one full three-way partition sort of n = 2^26 int32 keys (the
BASELINE.json headline; generated like config 1 -- uniform over the full
int32 range -- at 2^26, see workloads.py), input resident in HBM.  The
pristine input is restored (device copy) before each step, outside the timed
window; the 256 MB input exceeds the 126 MB L2, so no extra flush is needed.
Steps are timed with CUDA events on the sorting stream; multi-GPU runs are
independent replicas (the sort path does not shard here) timed as the max
over ranks.

Also reported on the same JSON line:
  e2e          the same metric through the public API with pinned host
               buffers: T.sort_many over a batch of host arrays (every
               array's H2D + D2H inside the timed region, pipelined against
               the neighbouring sorts); single_call_ms = one T.sort(host)
  roofline     partition pass: algorithmic bytes (read n + write the < and >
               keys of every partitioned segment) / partition-kernel time,
               against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline the CPU restatement of the reference (oracle/, C + OpenMP
               tasks) on the box's host cores, on a bounded sample
--impl reference prints the reference arm's line: the same CPU restatement
timed alone (the reference itself is pure Python and not installed on the
GPU box).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "keys/sec sorted (int32, n=2^26) on 1 B200; achieved HBM GB/s vs peak"
FALLBACK_HBM_GBS = 6650.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for name, v in zip(names, s[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


def cpu_baseline(n_sample: int, threads: int, family: str):
    """The oracle (C restatement of the reference sort) on the host cores."""
    from oracle import oracle as O
    import workloads as W
    keys, _ = W.generate(family, n_sample)
    x = keys.copy()
    t0 = time.perf_counter()
    O.sort(x, seed=1, threads=threads)
    dt = time.perf_counter() - t0
    assert np.array_equal(x, np.sort(keys))
    return n_sample / dt, dt


def reference_arm(args, rank: int, world: int):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n_sample = 1 << args.sample_log2
    vals = []
    for i in range(args.warmup + args.steps):
        v, _ = cpu_baseline(n_sample, threads, args.family)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "keys/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": n_sample / value * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": f"{args.family} int32 n=2^26 (bounded sample "
                                f"n=2^{args.sample_log2} per step)",
                   "n": args.n, "sample_n": n_sample},
        "cpu_baseline": {"value": value, "unit": "keys/s", "cores": threads, "kind": "port",
                         "sample": f"{args.family} int32 n=2^{args.sample_log2} per step, "
                                   f"oracle/ C restatement with {threads} OpenMP threads"},
        "e2e": {"value": value, "unit": "keys/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def our_arm(args, rank: int, world: int):
    import torch
    import torch.distributed as dist
    import paper_1505_00558_b200 as T
    import workloads as W

    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    keys, _ = W.generate(args.family, args.n)
    src = torch.from_numpy(keys).cuda()
    work = torch.empty_like(src)
    sorter = T.Sorter(seed=1)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        work.copy_(src)
        sorter.sort(work)
    torch.cuda.synchronize()
    ok = bool(torch.all(work[1:] >= work[:-1]).item())

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    stats = []
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        for i in range(args.steps):
            work.copy_(src)                     # restore the pristine input (untimed)
            starts[i].record(stream)
            stats.append(sorter.sort_with_stats(work))
            ends[i].record(stream)
        torch.cuda.synchronize()
    barrier()
    # Device time of each step: the sort graph's own CUDA events, recorded on
    # the sorting stream before its first and after its last kernel
    # (stats.gpu["ms_total"]).  The outer events also enclose the host
    # round trip sort_with_stats makes after the graph (control-block
    # readback + stream sync); that synchronous per-call time is reported
    # as ms_per_step_sync.
    ms_steps = [float(s.gpu["ms_total"]) for s in stats]
    ms_sync = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms_total, ms_total_sync = sum(ms_steps), sum(ms_sync)
    if world > 1:
        t = torch.tensor([ms_total, ms_total_sync], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total, ms_total_sync = float(t[0].item()), float(t[1].item())
    ms_step = ms_total / args.steps
    value = world * args.n / (ms_step / 1e3)
    g = stats[-1].gpu
    # init + (partition, schedule) per level + 2 on-chip classes + retire
    launches_per_step = 2 * int(g["levels"]) + 4

    # roofline of the partition pass from a host-driven run (per-launch events)
    hl = T.Sorter(seed=1, gpu=T.GpuConfig(host_levels=True))
    work.copy_(src)
    hl.sort(work)
    trace = hl.last_level_trace or []
    part_ms = sum(lv["ms"] for lv in trace)
    part_bytes = sum(lv["bytes"] for lv in trace)
    peak, peak_kind = peaks()
    achieved = part_bytes / (part_ms / 1e3) / 1e9 if part_ms else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "partition_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                traffic = json.load(f).get("bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": "partition_kernel", "peak_kind": peak_kind,
                "launches": len(trace), "bytes_per_launch_avg": part_bytes / max(1, len(trace)),
                "ms_per_launch_avg": part_ms / max(1, len(trace))}

    # end to end through the public API with pinned host buffers.  Headline
    # e2e: T.sort_many over K pinned host arrays -- every array's H2D and
    # D2H inside the timed region, overlapped with the neighbours' sorts by
    # the pipeline (the copy engines run both directions at once).  Also the
    # latency of one synchronous T.sort(host) call.
    K = max(args.steps, 8)
    hosts = [torch.empty(args.n, dtype=torch.int32, pin_memory=True) for _ in range(K)]
    src_t = torch.from_numpy(keys)

    def refill():
        for h in hosts:
            h.copy_(src_t)

    refill()
    T.sort_many(hosts[:2])                     # warm the pipeline buffers
    refill()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    T.sort_many(hosts)
    e2e_ms_step = (time.perf_counter() - t0) * 1e3 / K
    e2e_ok = all(bool(np.all(h.numpy()[1:] >= h.numpy()[:-1])) for h in hosts)
    single_ms = []
    for i in range(3):
        hosts[0].copy_(src_t)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        T.sort(hosts[0])                       # H2D, device sort, D2H, synchronous
        single_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_ok = e2e_ok and bool(np.all(hosts[0].numpy()[1:] >= hosts[0].numpy()[:-1]))
    single_ms_call = statistics.median(single_ms)
    del hosts
    if world > 1:
        t = torch.tensor([e2e_ms_step], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms_step = float(t.item())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        v, dt = cpu_baseline(1 << 24, threads, args.family)
        cpu = {"value": v, "unit": "keys/s", "cores": threads, "kind": "port",
               "sample": f"{args.family} int32 n=2^24, oracle/ C restatement, "
                         f"{threads} OpenMP threads, {dt:.2f} s"}

    fams = None
    if args.families and rank == 0:
        fams = family_table(T, W, torch)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "ms_per_step_sync": ms_total_sync / args.steps,
            "timing": "sum over the K steps of each sort graph's CUDA events on the sorting "
                      "stream (device time); ms_per_step_sync adds the per-call host readback",
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int32", "data": "synthetic",
            "config": {"workload": f"{args.family} int32 n=2^{int(np.log2(args.n))} "
                                   "(C1 generator at the headline size)",
                       "n": args.n, "l2_flush": "input (256 MB) exceeds L2 (126 MB)",
                       "parallelism": f"replicas x{world}"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": world * args.n / (e2e_ms_step / 1e3), "unit": "keys/s",
                    "h2d_bytes_per_step": args.n * 4, "d2h_bytes_per_step": args.n * 4,
                    "ms_per_step": e2e_ms_step,
                    "mode": f"T.sort_many over {K} pinned host arrays (H2D/D2H of every "
                            "array timed, overlapped with neighbouring sorts)",
                    "single_call_ms": single_ms_call},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
            "sorted_ok": ok and e2e_ok,
            "levels": int(g["levels"]), "stages": int(g["stages"]),
            "device_ms_total": float(g["ms_total"]),
        }
        if fams:
            line["families"] = fams
        print(json.dumps(line), flush=True)


def family_table(T, W, torch):
    """Per input family at BASELINE.json sizes (device-resident, keys/s)."""
    out = {}
    s = T.Sorter(seed=1)
    for fam, n in W.FULL_N.items():
        keys, pay = W.generate(fam, n)
        src = torch.from_numpy(keys).cuda()
        psrc = torch.from_numpy(pay).cuda() if pay is not None else None
        d = torch.empty_like(src)
        p = torch.empty_like(psrc) if psrc is not None else None
        ms = []
        for i in range(4):
            d.copy_(src)
            if p is not None:
                p.copy_(psrc)
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            st = s.sort_with_stats(T.Records(d, p) if p is not None else d)
            b.record()
            torch.cuda.synchronize()
            if i:
                ms.append(a.elapsed_time(b))
        m = statistics.median(ms)
        out[fam] = {"n": n, "keys_per_s": n / (m / 1e3), "ms": m,
                    "levels": int(st.gpu["levels"]), "depth": int(st.max_depth)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--family", default="uniform")
    ap.add_argument("--n", type=int, default=1 << 26)
    ap.add_argument("--families", action="store_true", help="add a per-family table")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sample-log2", type=int, default=24,
                    help="reference arm: keys per timed CPU sample (2^k)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if args.impl == "reference":
            dist.init_process_group("gloo")
        else:
            import torch
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
            dist.init_process_group("nccl")
    if args.impl == "reference":
        reference_arm(args, rank, world)
    else:
        our_arm(args, rank, world)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
