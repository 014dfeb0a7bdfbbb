"""Benchmark: keys/s sorting int32 n = 2^26 on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--family uniform] [--n 67108864] [--no-families]

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
               tasks) on the box's host cores, on the same 2^26 workload
  families     every BASELINE.json config at its own size: keys/s,
               the partition-pass roofline from a host-driven run, the
               oracle's CPU time on the same input, and a bit-exact check
               against tests/golden/full.json
--impl reference prints the reference arm's line: the same CPU restatement
timed alone on the same workload (the reference itself is pure Python and
not installed on the GPU box).
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


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def full_golden():
    """tests/golden/full.json: the oracle's hashes of every config at full size."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "full.json")) as f:
            return {r["family"]: r for r in json.load(f)["data"]}
    except OSError:
        return {}


def cpu_sort_time(keys, payload, threads: int):
    """The oracle (C restatement of the reference sort) on the host cores:
    seconds to sort a copy of keys (+ payload) in place."""
    from oracle import oracle as O
    x = keys.copy()
    p = None if payload is None else payload.copy()
    t0 = time.perf_counter()
    O.sort(x, p, seed=1, threads=threads)
    dt = time.perf_counter() - t0
    return dt, x


def reference_arm(args, rank: int, world: int):
    """The reference's CPU path on this box's host cores, on our arm's
    workload (same generator, same n): the oracle port with all threads."""
    if rank != 0:
        return
    import workloads as W
    threads = os.cpu_count() or 1
    keys, _ = W.generate(args.family, args.n)
    ms = []
    ok = True
    for i in range(args.warmup + args.steps):
        dt, out = cpu_sort_time(keys, None, threads)
        if i == 0:
            ok = out.tobytes() == np.sort(keys).tobytes()
        if i >= args.warmup:
            ms.append(dt * 1e3)
    ms_step = statistics.median(ms)
    value = args.n / (ms_step / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "keys/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": f"{args.family} int32 n=2^{int(np.log2(args.n))} "
                                "(C1 generator at the headline size)",
                   "n": args.n, "same_config": True},
        "cpu_baseline": {"value": value, "unit": "keys/s", "cores": threads, "kind": "port",
                         "cpu": cpu_model(),
                         "sample": f"the full workload ({args.family} int32 n={args.n}) per "
                                   f"step, oracle/ C restatement with {threads} OpenMP "
                                   "threads; median step"},
        "e2e": {"value": value, "unit": "keys/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "sorted_ok": ok,
    }
    print(json.dumps(line), flush=True)


def partition_roofline(T, sorter_args, run, peak, peak_kind):
    """Roofline of the partition pass from a host-driven run (one event pair
    per partition launch): algorithmic bytes (read every live key, write the
    < and > keys; records add the payloads) / partition-kernel time."""
    hl = T.Sorter(seed=1, gpu=T.GpuConfig(host_levels=True, **sorter_args))
    run(hl)
    trace = hl.last_level_trace or []
    part_ms = sum(lv["ms"] for lv in trace)
    part_bytes = sum(lv["bytes"] for lv in trace)
    achieved = part_bytes / (part_ms / 1e3) / 1e9 if part_ms else 0.0
    levels = [{"ms": round(lv["ms"], 4), "GBps": round(lv["bytes"] / lv["ms"] / 1e6, 1)
               if lv["ms"] else 0.0, "segments": lv["segments"], "bytes": lv["bytes"]}
              for lv in trace]
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "kernel": "partition_kernel",
            "peak_kind": peak_kind, "launches": len(trace),
            "bytes_per_launch_avg": part_bytes / max(1, len(trace)),
            "ms_per_launch_avg": part_ms / max(1, len(trace)),
            "min_level_frac": round(min((lv["bytes"] / lv["ms"] / 1e6 for lv in trace
                                         if lv["ms"] > 0), default=0.0) / peak, 4),
            "levels": levels}


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
    # the last timed step's output: the sorted permutation of the input
    ok = bool(torch.equal(work, torch.sort(src).values))
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
    # init + (partition, schedule) per level + the drain round (2 on-chip
    # classes, retire, drain) per flush and at the end + the control-block
    # readback
    launches_per_step = 1 + 2 * int(g["levels"]) + 4 * (1 + int(g["flushes"])) + 1

    peak, peak_kind = peaks()

    def run_headline(s):
        work.copy_(src)
        s.sort(work)

    roofline = partition_roofline(T, {}, run_headline, peak, peak_kind)
    tp = os.path.join(ROOT, "profiles", "partition_traffic.json")
    roofline["traffic"] = None
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                roofline["traffic"] = json.load(f).get("bytes_per_launch")
        except Exception:
            pass

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
    want = np.sort(keys)
    e2e_ok = all(np.array_equal(h.numpy(), want) for h in hosts)
    single_ms = []
    for i in range(3):
        hosts[0].copy_(src_t)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        T.sort(hosts[0])                       # H2D, device sort, D2H, synchronous
        single_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_ok = e2e_ok and np.array_equal(hosts[0].numpy(), want)
    single_ms_call = statistics.median(single_ms)
    del hosts
    if world > 1:
        t = torch.tensor([e2e_ms_step], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms_step = float(t.item())

    cpu = None
    threads = os.cpu_count() or 1
    if rank == 0 and world == 1 and not args.no_cpu:
        dt, out = cpu_sort_time(keys, None, threads)
        cpu = {"value": args.n / dt, "unit": "keys/s", "cores": threads, "kind": "port",
               "cpu": cpu_model(),
               "sample": f"the full workload ({args.family} int32 n={args.n}), oracle/ C "
                         f"restatement with {threads} OpenMP threads, {dt:.2f} s",
               "sorted_ok": out.tobytes() == want.tobytes()}

    fams = None
    if not args.no_families and rank == 0:
        fams = family_table(T, W, torch, peak, peak_kind,
                            cpu_threads=0 if (args.no_cpu or world > 1) else threads)

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
                    "single_call_ms": single_ms_call,
                    "single_call_keys_per_s": args.n / (single_ms_call / 1e3)},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
            "sorted_ok": ok and e2e_ok,
            "levels": int(g["levels"]), "stages": int(g["stages"]),
            "device_ms_total": float(g["ms_total"]),
        }
        if fams:
            line["families"] = fams
        print(json.dumps(line), flush=True)


def family_table(T, W, torch, peak, peak_kind, cpu_threads: int):
    """Every BASELINE.json config at its own size (device-resident input):
    keys/s (median of 3 timed sorts after a warm-up), the partition-pass
    roofline of a host-driven run, the oracle's CPU time on the same input
    with `cpu_threads` threads, and a bit-exact check of the GPU output
    against tests/golden/full.json."""
    gold = full_golden()
    out = {}
    s = T.Sorter(seed=1)
    for fam, n in W.FULL_N.items():
        keys, pay = W.generate(fam, n)
        src = torch.from_numpy(keys).cuda()
        psrc = torch.from_numpy(pay).cuda() if pay is not None else None
        d = torch.empty_like(src)
        p = torch.empty_like(psrc) if psrc is not None else None

        def run(sorter):
            d.copy_(src)
            if p is not None:
                p.copy_(psrc)
            return sorter.sort_with_stats(T.Records(d, p) if p is not None else d)

        ms = []
        for i in range(4):
            st = run(s)
            if i:
                ms.append(float(st.gpu["ms_total"]))
        m = statistics.median(ms)
        got = d.cpu().numpy()
        ok = fam in gold and W.sha16(got) == gold[fam]["sorted_sha"]
        if p is not None:
            po = p.cpu().numpy().astype(np.int64)
            ok = ok and np.array_equal(keys[po], got) and \
                np.array_equal(np.bincount(po, minlength=n), np.ones(n, np.int64))
        rf = partition_roofline(T, {}, run, peak, peak_kind)
        rf.pop("levels")
        row = {"n": n, "dtype": str(keys.dtype) + ("+u32" if pay is not None else ""),
               "keys_per_s": n / (m / 1e3), "ms": m, "levels": int(st.gpu["levels"]),
               "depth": int(st.max_depth), "bit_exact_vs_oracle": bool(ok),
               "roofline": {k: rf[k] for k in ("achieved", "frac", "min_level_frac",
                                               "launches", "ms_per_launch_avg")}}
        if cpu_threads:
            dt, _ = cpu_sort_time(keys, pay, cpu_threads)
            row["cpu"] = {"keys_per_s": n / dt, "s": round(dt, 3), "cores": cpu_threads,
                          "kind": "port"}
            row["gpu_over_cpu"] = round((n / (m / 1e3)) / (n / dt), 1)
        out[fam] = row
        del src, psrc, d, p
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--family", default="uniform")
    ap.add_argument("--num-keys", "--n", dest="n", type=int, default=1 << 26)
    ap.add_argument("--no-families", action="store_true",
                    help="skip the per-config table (every BASELINE config at its size)")
    ap.add_argument("--no-cpu", action="store_true")
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
