#!/usr/bin/env python3
"""Benchmark of the DPG record-retrieval hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dpg|reference]
                    [--config c2|c1|c2L|c3a|c3b|c4|c4x|c5|h1] [--rec R]

N = 1 (default): one step = one dpg_retrieve call (the whole hot path: plan,
distribute, probe, gather) over BASELINE.json configs[1] --
Datamation-shaped sort phase 3, 1,048,576 x 100-byte records, rids = stable
argsort of the 10-byte keys -- with src and rids resident in HBM.  Before
every timed step L2 is flushed (a 512 MiB write, then a 512 MiB read, so no
dirty line of the flush is left for the step); after it, a second 512 MiB read
makes the L2 write back the step's own dirty output, and that write-back time
(measured against the same read after a clean L2) is added to the step.  The
line nests the same protocol on the other configurations (the record-size
sweep, the 2L row, the join, the single-GPU config-5 shard) with the direct
comparisons, so one run shows where DPG wins and where it does not.

N > 1: the driver launches this under torchrun (or, given --gpus N without
torchrun, it relaunches itself so); one step = the multi-GPU retrieval of
BASELINE.json configs[4] -- 2^30 x 100-byte records range-partitioned over
the ranks, rids a Feistel permutation (uint64) block-partitioned by output
position -- through the native C ABI (dpg_retrieve_dist: owner partition, NCCL
count all-gather and request send/recv, the owner's DPG writing replies into
the requesters' IPC windows over NVLink, Phase III); job time = max over ranks
of the CUDA-event time.

Every line carries the roofline of the dominant kernel (its own CUDA-event time
on the launching stream, from the library's phase events), the oracle's CPU
throughput (1 core and all cores), the end-to-end number through the
host-buffer C-ABI path and the SM clocks sampled during the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "record-retrieval effective GB/s vs HBM peak; records/s at 1/2/4/8 B200"
FALLBACK_HBM_GBS = 6650.0
NVLINK_GBS = 900.0            # per GPU per direction (NVLink 5 via NVSwitch)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="dpg", choices=["dpg", "reference"])
    ap.add_argument("--config", default=None,
                    choices=["c1", "c2", "c2L", "c3a", "c3b", "c4", "c4x", "c5", "h1"],
                    help="default: c2 on one GPU, c5 (multi-GPU exchange) under torchrun")
    ap.add_argument("--c5-log2", type=int, default=30, help="c5 total records = 2^c5_log2")
    ap.add_argument("--c5-rows", type=int, default=1 << 27,
                    help="c5 rows per rank per exchange call (bounds the windows: 13.4 GB)")
    ap.add_argument("--rec", type=int, default=None, help="record bytes for c3a/c3b")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="N=1: only the headline config")
    ap.add_argument("--extras", default="c2L,c3a4,c3a8,c3a16,c3a32,c3a64,c3a256,c3b8,c3a4n26,c3a8n26,c3a8n27,"
                                        "c3a16n26,c3a128,c4r256,c4,c4x,c5shard",
                    help="N=1: nested configurations")
    a = ap.parse_args()
    if a.config is None:
        a.config = "c5" if int(os.environ.get("WORLD_SIZE", "1")) > 1 or a.gpus > 1 else "c2"
    return a


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def relaunch_under_torchrun(args) -> int | None:
    """--gpus N > 1 outside torchrun: start N ranks of this script (one per GPU)
    via torch.distributed.run on 127.0.0.1 and return its exit code; fail loudly
    when fewer than N GPUs are visible."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import torch
    n = torch.cuda.device_count()
    if n < args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but {n} GPU(s) visible",
                          "n_gpus": args.gpus}), flush=True)
        sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, {n} visible\n")
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


# ---------------------------------------------------------------------------
# measurement helpers
# ---------------------------------------------------------------------------
class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    NAMES = {"applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
             "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
             "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100}

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.NAMES.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s)}


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def committed_traffic(key):
    """dram bytes per launch of the dominant kernel from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def host_cpu():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


class Steps:
    """The timing protocol of SURVEY 8(d): L2 flushed before every timed step
    (512 MiB write, then 512 MiB read), CUDA events on the launching stream,
    and the step's own dirty-output write-back added (a 512 MiB read after the
    step, minus the same read after a clean L2)."""

    def __init__(self, torch, dev):
        self.torch = torch
        self.w = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        self.r = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        self.r2 = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        self.stream = torch.cuda.current_stream()
        self.base = None

    def flush(self):
        self.w.fill_(1)
        self.r.view(self.torch.int32).max()

    def _read2(self):
        self.r2.view(self.torch.int32).max()

    def _ev(self):
        return self.torch.cuda.Event(enable_timing=True)

    def clean_read_ms(self, reps=5):
        if self.base is None:
            v = []
            for _ in range(reps):
                self.flush()
                a, b = self._ev(), self._ev()
                a.record(self.stream)
                self._read2()
                b.record(self.stream)
                self.torch.cuda.synchronize()
                v.append(a.elapsed_time(b))
            self.base = sorted(v)[len(v) // 2]
        return self.base

    def run(self, fn, steps, launches=None, phase_lib=None):
        """-> (per-step ms incl. write-back, per-step kernel-only ms, write-back ms,
        launches, phase times (I, II, III) per step or None)."""
        torch = self.torch
        base = self.clean_read_ms()
        evs = [(self._ev(), self._ev(), self._ev()) for _ in range(steps)]
        if phase_lib is not None:
            phase_lib.dpg_phase_times_ex()
            phase_lib.dpg_phase_timing(True)
        nl = 0
        for e0, e1, e2 in evs:
            self.flush()
            e0.record(self.stream)
            fn()
            e1.record(self.stream)
            self._read2()
            e2.record(self.stream)
            if launches is not None:
                nl += launches()
        torch.cuda.synchronize()
        ph = None
        if phase_lib is not None:
            phase_lib.dpg_phase_timing(False)
            a, b, c, calls = phase_lib.dpg_phase_times_ex()
            ph = (a / max(1, calls), b / max(1, calls), c / max(1, calls))
        step = [x.elapsed_time(y) for x, y, _ in evs]
        wb = [max(0.0, y.elapsed_time(z) - base) for _, y, z in evs]
        tot = [s + w for s, w in zip(step, wb)]
        return tot, step, wb, nl, ph


def med(v):
    v = sorted(v)
    return v[len(v) // 2]


# ---------------------------------------------------------------------------
# CPU baseline: the oracle on the host cores
# ---------------------------------------------------------------------------
def cpu_baseline(src, rids, alg_bytes_per_row, budget_s=8.0, sample=None, fk_join=None):
    """The oracle as it stands (single-threaded C loop) and the same loop split
    over all host cores (oracle_retrieve_threads), each repeated until
    ~budget_s of CPU work on the given (bounded) sample."""
    import oracle
    threads = host_threads()
    res = {}
    for label, fn in (("single", (lambda: oracle.retrieve(src, rids)) if fk_join is None else
                       (lambda: oracle.fk_join(*fk_join))),
                      ("all", (lambda: oracle.retrieve_threads(src, rids, threads))
                       if fk_join is None else None)):
        if fn is None:
            continue
        fn()
        reps, t0 = 0, time.perf_counter()
        while True:
            fn()
            reps += 1
            el = time.perf_counter() - t0
            if el >= budget_s / 2 or (reps >= 3 and el > budget_s / 4):
                break
        res[label] = el / reps
    n = (fk_join[1].size if fk_join is not None else rids.size)
    one = res["single"]
    out = {"value": n * alg_bytes_per_row / one / 1e9, "unit": "GB/s", "cores": 1,
           "kind": "oracle", "records_per_s": n / one,
           "sample": sample or f"{n} rows, oracle single-threaded C loop",
           "host_cpu": host_cpu(), "host_threads": threads}
    if "all" in res:
        out["all_cores"] = {"value": n * alg_bytes_per_row / res["all"] / 1e9, "unit": "GB/s",
                            "cores": threads, "records_per_s": n / res["all"],
                            "what": "oracle_retrieve_threads: the same loop over contiguous "
                                    "index ranges, one thread each"}
    return out


# ---------------------------------------------------------------------------
# reference arm: the oracle on the host cores (this tier has no reference code)
# ---------------------------------------------------------------------------
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import datagen
    import oracle
    cfg = args.config
    if cfg == "h1":
        w = datagen.hash_workload(1 << 24, 24, 1 << 26)
        q = w["queries"][: 1 << 24]
        times = []
        for _ in range(max(1, args.steps)):
            t0 = time.perf_counter()
            oracle.batch_lookup(w["keys"], q)
            times.append(time.perf_counter() - t0)
            if sum(times) > 120:
                break
        t = sum(times) / len(times)
        v = q.size / t
        print(json.dumps({
            "impl": "reference", "metric": "batch index lookups/s (hash index, DPG)", "value": v,
            "unit": "lookups/s", "n_gpus": world, "steps": len(times), "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (datagen.hash_workload, seed 0)",
            "config": {"workload": "h1 sample: 2^24 of the 2^26 queries"},
            "cpu_baseline": {"value": v, "unit": "lookups/s", "cores": 1, "kind": "oracle",
                             "sample": "2^24 queries, oracle.batch_lookup", "host_cpu": host_cpu()},
            "e2e": {"value": v, "unit": "lookups/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}), flush=True)
        return 0
    if cfg == "c5":
        # bounded sample of config 5 for the host oracle: 2^22 records of the
        # c5 source stream, rids = the c5 Feistel permutation of [0, 2^22)
        n = 1 << 22
        src = datagen.records(n, 100, datagen.STREAMS[("c5", "src")])
        rids = datagen.feistel(n, 0, n, datagen.STREAMS[("c5", "rids")])
        fn = lambda: oracle.retrieve(src, rids)
        n_out, per_row, sample = n, 2 * 100 + 8, "2^22 x 100 B sample of the c5 stream, 64-bit rids"
    else:
        w = make_inputs(cfg, args.rec)
        if cfg in ("c4", "c4x"):
            fn = lambda: oracle.fk_join(w["fact"], w["fk"], w["dim"])
            n_out, per_row = w["fk"].size, 4 + 16 + 64 + 80
        else:
            fn = lambda: oracle.retrieve(w["src"], w["rids"])
            n_out, per_row = w["rids"].size, 2 * w["src"].shape[1] + 4
        sample = f"full {cfg} workload"
    for _ in range(max(0, min(args.warmup, 3))):
        fn()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
        if sum(times) > 150:
            break
    t = sum(times) / len(times)
    value = n_out * per_row / t / 1e9
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": world, "steps": len(times), "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (datagen, seed 0)",
        "config": {"workload": workload_name(cfg, args.rec), "n_out": int(n_out)},
        "records_per_s": n_out / t,
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": f"{sample}, {len(times)} steps", "host_cpu": host_cpu()},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)
    return 0


def workload_name(cfg: str, rec: int | None) -> str:
    return {"c1": "c1: 65,536 x 100 B random records, uniform random permutation",
            "c2": "c2: Datamation sort phase 3, 1,048,576 x 100 B, rids = stable argsort of 10-B keys",
            "c2L": "2L: 16,777,216 x 100 B, uniform random permutation (SURVEY 8(d))",
            "c3a": f"c3a: 16,777,216 x {rec} B, uniform random permutation",
            "c3b": f"c3b: 16,777,216 x {rec} B, uniform rids with replacement",
            "c4": "c4: DPG-Move FK join, dim 16,777,216 x 64 B, fact 67,108,864 x (fk + 16 B)",
            "c4x": "c4x: config 4 with the paper's exponential join keys (P:890-892)",
            "c5": "c5: 2^30 x 100 B range-partitioned, rids = Feistel permutation (uint64) "
                  "block-partitioned"}.get(cfg, cfg)


def make_inputs(cfg: str, rec: int | None):
    import datagen
    if cfg in ("c3a", "c3b"):
        return datagen.make(cfg, rec=rec or 64)
    return datagen.make(cfg)


# ---------------------------------------------------------------------------
# N = 1
# ---------------------------------------------------------------------------
def measure_retrieval(torch, dpg, steps_obj, src, rids, steps, warmup, with_cmp=True):
    """DPG (the automatic plan) and the direct comparisons on resident inputs."""
    n_out, rec = rids.numel(), src.shape[1]
    alg = n_out * (2 * rec + 4)
    out = torch.empty((n_out, rec), dtype=torch.uint8, device=src.device)
    fns = {"dpg": lambda: dpg.dpg_retrieve(src, rids, dst=out)}
    if with_cmp:
        fns["naive"] = lambda: dpg.dpg_retrieve_direct(src, rids, dst=out)
        fns["direct_windowed"] = lambda: dpg.dpg_retrieve_direct_ex(src, rids, dst=out, hint=3)
    for _ in range(max(3, warmup)):
        for f in fns.values():
            f()
    torch.cuda.synchronize()
    dpg.dpg_sync_status()
    fns["dpg"]()
    path = dpg.last_path()
    res = {}
    for k, f in fns.items():
        tot, step, wb, nl, _ = steps_obj.run(f, steps, launches=dpg.last_launch_count)
        res[k] = {"ms": med(tot), "ms_kernels": med(step), "ms_writeback": med(wb),
                  "value": alg / (med(tot) * 1e-3) / 1e9, "unit": "GB/s",
                  "launches_per_step": nl / steps, "all_ms": tot, "phases_ms": None}
    res["dpg"]["plan_path"] = path
    res["dpg"]["phases_ms"] = phase_split(dpg, steps_obj, fns["dpg"], steps)
    return res, out, alg


def phase_split(dpg, steps_obj, fn, steps):
    """The per-phase kernel times (Phase I, II, III) of a plan from the
    library's own phase events, in a second timed pass: those events sit on
    the launching stream and each costs ~2.5 us of stream time
    (tools/launch_gap_probe.py: 59.4 -> 67.6 us for c2), so the step times
    above are taken without them."""
    _, _, _, _, ph = steps_obj.run(fn, steps, phase_lib=dpg)
    return ph


def roofline_for(dpg, plan_path, res_dpg, n_src, n_out, rec, pay, peak, peak_src, traffic_key):
    """The dominant kernel of the plan the call ran, its algorithmic bytes per
    launch over its own CUDA-event time."""
    ph = res_dpg["phases_ms"] or (0.0, res_dpg["ms_kernels"], 0.0)
    if res_dpg.get("launches_per_step") == 1 and plan_path in (1, 3):
        # one launch per step: the timed region's own events bracket exactly
        # that kernel (the phase pass only splits multi-kernel plans)
        ph = (0.0, res_dpg["ms_kernels"], 0.0)
    if plan_path == 6:
        # three kernels: Phase I (distribute + transpose), II (probe), III (gather)
        per = {"k3_distribute (Phase I)": (ph[0], n_out * (4 + 2 + 2)),
               "k3_probe (Phase II)": (ph[1], n_src * rec + n_out * (2 + rec)),
               "k3_gather (Phase III)": (ph[2], n_out * (2 + 2 * rec + pay))}
    elif plan_path == 3:
        per = {"k_dpg_l2run": (ph[1], n_out * (2 * rec + 4))}
    elif plan_path == 1:
        per = {"k_dpg_fused": (ph[1] + ph[0], n_out * (2 * rec + 4))}
    else:
        per = {f"path {plan_path} probe-gather": (ph[1], n_src * rec + n_out * (rec + 8))}
        if plan_path == 2 and ph[0] > 0:
            # Phase I: the rid list read, the 8-byte pairs written (the radix passes'
            # intermediate round trips are not algorithmic)
            per["path 2 Phase I (distribute)"] = (ph[0], n_out * (4 + 8))
    kernel = max(per, key=lambda k: per[k][0])
    ms, by = per[kernel]
    achieved = by / (ms * 1e-3) / 1e9 if ms > 0 else None
    return {"bound": "hbm", "kernel": kernel, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None, "traffic": committed_traffic(traffic_key),
            "peak_source": peak_src, "alg_bytes_per_launch": by, "launch_ms": ms,
            "share_of_step": ms / res_dpg["ms_kernels"] if res_dpg["ms_kernels"] else None,
            "phases_ms": ph,
            "kernels": {k: {"ms": v[0], "alg_bytes": v[1],
                            "frac": (v[1] / (v[0] * 1e-3) / 1e9 / peak) if v[0] > 0 else None}
                        for k, v in per.items()}}


def sampled_ok(out, want_fn, n, k=4096, seed=0):
    idx = np.unique(np.random.default_rng(seed).integers(0, n, k))
    import torch
    got = out[torch.from_numpy(idx.astype(np.int64)).to(out.device)].cpu().numpy()
    return bool(np.array_equal(got, want_fn(idx)))


def run_single(args):
    import torch
    torch.cuda.set_device(0)
    import datagen
    import oracle
    import paper_cs_0308004_b200 as dpg
    dev = torch.device("cuda", 0)
    peak, peak_src = hbm_peak()
    steps_obj = Steps(torch, dev)

    def to_dev(a):
        a = np.ascontiguousarray(a)
        if a.dtype == np.uint32:
            a = a.view(np.int32)
        return torch.from_numpy(a).to(dev)

    cfg = args.config
    if cfg in ("c4", "c4x"):
        return run_join_line(args, torch, dpg, steps_obj, cfg)
    w = make_inputs(cfg, args.rec)
    src, rids = to_dev(w["src"]), to_dev(w["rids"])
    n_out, rec = w["rids"].size, w["src"].shape[1]
    n_src = w["src"].shape[0]
    with ClockSampler(0) as clk:
        res, out, alg = measure_retrieval(torch, dpg, steps_obj, src, rids, args.steps, args.warmup)
    dpg.dpg_sync_status()
    ok = sampled_ok(out, lambda i: oracle.retrieve_at(w["src"], w["rids"], i.astype(np.uint64)), n_out)
    d = res["dpg"]
    roofline = roofline_for(dpg, d["plan_path"], d, n_src, n_out, rec, 0, peak, peak_src, cfg)

    # the paper's application of the path (section 3): the whole Datamation sort
    sort_res = None
    if cfg == "c2":
        for _ in range(2):
            dpg.dpg_sort(src, 0, 10, dst=out)
        torch.cuda.synchronize()
        srt_ok = sampled_ok(out, lambda i: oracle.retrieve_at(w["src"], w["rids"],
                                                               i.astype(np.uint64)), n_out, seed=1)
        tot, step, wb, nl, _ = steps_obj.run(lambda: dpg.dpg_sort(src, 0, 10, dst=out),
                                             max(3, args.steps // 2), launches=dpg.last_launch_count)
        sort_res = {"ms_per_sort": med(tot), "records_per_s": n_out / (med(tot) * 1e-3),
                    "launches_per_sort": nl / max(3, args.steps // 2), "parity_sampled_ok": srt_ok,
                    "what": "dpg_sort: 10-byte keys at offset 0, stable radix passes on the 4-byte prefix + fix-up of equal-prefix groups (full LSD sort if a group exceeds 32) + dpg_retrieve"}
        # the paper's comparison: the same phases 1-2, phase 3 by
        # the direct gather ("standard" key-pointer sort)
        srids = torch.empty(n_out, dtype=torch.int32, device="cuda")

        def naive_sort():
            dpg.dpg_sort_rids(src, 0, 10, rids=srids)
            dpg.dpg_retrieve_direct(src, srids, dst=out)
        naive_sort()
        torch.cuda.synchronize()
        ntot, _, _, _, _ = steps_obj.run(naive_sort, max(3, args.steps // 2))
        sort_res["naive_phase3_ms_per_sort"] = med(ntot)
        sort_res["dpg_over_naive"] = med(ntot) / med(tot)

    # end to end through the host-buffer C-ABI entries (PCIe copies inside):
    # the asynchronous entry on two streams in turn, so one step's device->host
    # copy overlaps the next step's host->device copy (every step still copies
    # its own inputs in and its result out); the synchronous entry beside it
    e2e = None
    if not args.no_e2e:
        hs = torch.from_numpy(w["src"]).pin_memory()
        hr = torch.from_numpy(w["rids"].view(np.int32)).pin_memory()
        ns = 2          # (3 or 4 streams: the same 89-90 GB/s, the PCIe limit)
        hd = [torch.empty((n_out, rec), dtype=torch.uint8).pin_memory() for _ in range(ns)]
        ss = [torch.cuda.Stream() for _ in range(ns)]
        for q in range(ns):
            dpg.dpg_retrieve_host(hs, hr, hd[q], stream=ss[q], synchronize=False)
        torch.cuda.synchronize()
        k = ns * max(2, min(args.steps, 12) // ns)
        t0 = time.perf_counter()
        for i in range(k):
            dpg.dpg_retrieve_host(hs, hr, hd[i % ns], stream=ss[i % ns], synchronize=False)
        torch.cuda.synchronize()
        el = (time.perf_counter() - t0) / k
        okh = all(np.array_equal(hd[q][:2000].numpy(), oracle.retrieve(w["src"], w["rids"][:2000]))
                  for q in range(ns))
        hd1 = hd[0]
        dpg.dpg_retrieve_host(hs, hr, hd1)          # (its stream's buffers allocated)
        t0 = time.perf_counter()
        for _ in range(3):
            dpg.dpg_retrieve_host(hs, hr, hd1)
        el_sync = (time.perf_counter() - t0) / 3
        e2e = {"value": alg / el / 1e9, "unit": "GB/s", "ms_per_step": el * 1e3,
               "h2d_bytes_per_step": int(w["src"].nbytes + w["rids"].nbytes),
               "d2h_bytes_per_step": int(n_out * rec),
               "entry": f"dpg_retrieve_host_async, {ns} streams in turn (wall clock over the steps)",
               "sync_entry": {"entry": "dpg_retrieve_host", "ms_per_step": el_sync * 1e3,
                              "value": alg / el_sync / 1e9},
               "parity_sampled_ok": bool(okh)}
        dpg.dpg_release_cache()

    cpu = None if args.no_cpu else cpu_baseline(
        w["src"], w["rids"], 2 * rec + 4, sample=f"full {cfg} workload")

    extras = {}
    if not args.no_extras and cfg == "c2":
        for name in [x for x in args.extras.split(",") if x]:
            try:
                extras[name] = run_extra(name, args, torch, dpg, steps_obj, peak)
            except Exception as e:  # noqa: BLE001 -- a failed extra is reported, not fatal
                extras[name] = {"error": repr(e)}
            torch.cuda.empty_cache()
            dpg.dpg_release_cache()      # each nested configuration starts from an empty pool

    line = {
        "metric": METRIC, "value": d["value"], "unit": "GB/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": d["ms"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (datagen, seed 0)",
        "config": {"workload": workload_name(cfg, args.rec), "n_src": n_src, "n_out": n_out,
                   "rec_bytes": rec, "rid_bytes": 4, "alg_bytes_per_step": alg,
                   "alg_bytes_formula": "N * (2 * rec + rid_bytes)",
                   "l2": "flushed before every step (512 MiB write, then 512 MiB read); the step's "
                         "dirty-output write-back is measured after it and included",
                   "parallelism": "single", "plan_path": d["plan_path"]},
        "records_per_s": n_out / (d["ms"] * 1e-3),
        "frac_of_hbm_peak": d["value"] / peak,
        "ms_kernels": d["ms_kernels"], "ms_writeback": d["ms_writeback"],
        "ms_min": min(d["all_ms"]), "ms_median": med(d["all_ms"]),
        "roofline": roofline,
        "naive": {k: v for k, v in res["naive"].items() if k not in ("all_ms", "phases_ms")},
        "direct_windowed": {k: v for k, v in res["direct_windowed"].items()
                            if k not in ("all_ms", "phases_ms")},
        "parity_sampled_ok": ok, "dpg_sort": sort_res, "e2e": e2e, "cpu_baseline": cpu,
        "configs": extras, "clocks": clk.summary(),
        "gpu_launches": int(round(d["launches_per_step"] * args.steps)),
        "gpu": torch.cuda.get_device_name(dev),
    }
    print(json.dumps(line), flush=True)
    return 0


def run_extra(name, args, torch, dpg, steps_obj, peak):
    """One nested configuration: DPG (automatic plan) vs the direct gather (and
    the three sequential passes where they apply), inputs generated on the
    device from the same counter-based streams, sampled parity against the
    oracle's definition for a generated source."""
    import datagen
    import oracle
    steps = max(3, min(args.steps, 8))
    if name in ("c4", "c4x"):
        return run_join_extra(args, torch, dpg, steps_obj, peak, steps, cfg=name)
    if name == "c5shard":
        return run_c5_shard(args, torch, dpg, steps_obj, peak, steps)
    if name.startswith("c4r"):                # config 4's retrieval shape with rec-byte records
        return run_c4r_extra(name, args, torch, dpg, steps_obj, peak, steps)
    log2n = 24
    if "n" in name[3:]:                       # e.g. c3a8n26: config 3's shape at 2^26 records
        name, log2n = name.split("n")[0], int(name.split("n")[1])
    if name == "c2L":
        rec, kind = 100, "c3a"
    else:
        kind, rec = name[:3], int(name[3:])
    n = 1 << log2n
    sid = datagen.STREAMS[("c3", "src")]
    src = torch.empty((n, rec), dtype=torch.uint8, device="cuda")
    datagen.random_bytes_cuda(src.view(-1), sid)
    rids_h = datagen.permutation(n, datagen.STREAMS[("c3a", "rids")]) if kind == "c3a" else \
        datagen.uniform(n, n, datagen.STREAMS[("c3b", "rids")])
    rids = torch.from_numpy(rids_h.view(np.int32)).cuda()
    res, out, alg = measure_retrieval(torch, dpg, steps_obj, src, rids, steps, args.warmup)
    dpg.dpg_sync_status()
    idx_fn = lambda i: oracle.retrieve_generated(rec, n, sid, rids_h[i].astype(np.uint64))
    ok = sampled_ok(out, idx_fn, n, k=512)
    d = res["dpg"]
    wl = workload_name("c2L" if name == "c2L" else kind, rec)
    if log2n != 24:
        wl = wl.replace("16,777,216", f"2^{log2n} = {n:,}") + \
            f" (source {n * rec / 1e6:.0f} MB, {n * rec / (126 << 20):.1f}x the L2)"
    r = {"workload": wl, "plan_path": d["plan_path"],
         "value": d["value"], "frac_of_hbm_peak": d["value"] / peak, "ms": d["ms"],
         "ms_kernels": d["ms_kernels"], "phases_ms": d["phases_ms"],
         "naive": {"value": res["naive"]["value"], "ms": res["naive"]["ms"]},
         "direct_windowed": {"value": res["direct_windowed"]["value"],
                             "ms": res["direct_windowed"]["ms"]},
         "dpg_over_naive": res["naive"]["ms"] / d["ms"], "parity_sampled_ok": ok,
         "roofline": roofline_for(dpg, d["plan_path"], d, n, n, rec, 0, peak, "", name)}
    del out, src, rids
    return r


def run_c4r_extra(name, args, torch, dpg, steps_obj, peak, steps):
    """Config 4's retrieval shape with wider dimension records (c4r256: 2^26
    uniform foreign keys into 2^24 x 256-byte records; four rids per record on
    average, the join's fan-in): DPG vs the direct gather."""
    import datagen
    import oracle
    rec = int(name[3:])
    n_src, n = 1 << 24, 1 << 26
    sid = datagen.STREAMS[("c4", "dim")]
    src = torch.empty((n_src, rec), dtype=torch.uint8, device="cuda")
    datagen.random_bytes_cuda(src.view(-1), sid)
    rids_h = datagen.uniform(n, n_src, datagen.STREAMS[("c4", "fk")])
    rids = torch.from_numpy(rids_h.view(np.int32)).cuda()
    res, out, alg = measure_retrieval(torch, dpg, steps_obj, src, rids, steps, args.warmup)
    dpg.dpg_sync_status()
    idx_fn = lambda i: oracle.retrieve_generated(rec, n_src, sid, rids_h[i].astype(np.uint64))
    ok = sampled_ok(out, idx_fn, n, k=512)
    d = res["dpg"]
    r = {"workload": f"c4r{rec}: 67,108,864 uniform rids into 16,777,216 x {rec} B "
                     "(config 4's fan-in, retrieval only)",
         "plan_path": d["plan_path"], "value": d["value"], "frac_of_hbm_peak": d["value"] / peak,
         "ms": d["ms"], "ms_kernels": d["ms_kernels"], "phases_ms": d["phases_ms"],
         "naive": {"value": res["naive"]["value"], "ms": res["naive"]["ms"]},
         "direct_windowed": {"value": res["direct_windowed"]["value"],
                             "ms": res["direct_windowed"]["ms"]},
         "dpg_over_naive": res["naive"]["ms"] / d["ms"], "parity_sampled_ok": ok,
         "roofline": roofline_for(dpg, d["plan_path"], d, n_src, n, rec, 0, peak, "", name)}
    del out, src, rids
    return r


def run_join_line(args, torch, dpg, steps_obj, cfg):
    """--config c4 / c4x as the main line (N = 1)."""
    peak, peak_src = hbm_peak()
    with ClockSampler(0) as clk:
        r = run_join_extra(args, torch, dpg, steps_obj, peak, args.steps, cfg=cfg, full=True)
    r.update({"metric": METRIC, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
              "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
              "data": "synthetic (datagen, seed 0)", "clocks": clk.summary(),
              "unit": "GB/s", "ms_per_step": r["ms"]})
    r["config"] = {"workload": workload_name(cfg, None), "alg_bytes_per_row": 164,
                   "plan_path": r.pop("plan_path")}
    r["e2e"] = None
    print(json.dumps(r), flush=True)
    return 0


def run_join_extra(args, torch, dpg, steps_obj, peak, steps, cfg="c4", full=False):
    import datagen
    import oracle
    w = datagen.make(cfg)
    fact = torch.from_numpy(w["fact"]).cuda()
    fk = torch.from_numpy(w["fk"].view(np.int32)).cuda()
    dim = torch.from_numpy(w["dim"]).cuda()
    n = w["fk"].size
    alg = n * (4 + 16 + 64 + 80)       # fk + fact payload + dim record read, 80-B row written
    out = torch.empty((n, 80), dtype=torch.uint8, device="cuda")
    fns = {"dpg": lambda: dpg.dpg_fk_join(fact, fk, dim, out=out),
           "direct": lambda: dpg.dpg_fk_join_direct(fact, fk, dim, out=out),
           "dpg_seq3": lambda: dpg.dpg_fk_join(fact, fk, dim, out=out, path=6),
           "dpg_sort_join": lambda: dpg.dpg_fk_join_sort(fact, fk, dim, out=out)}
    res = {}
    for k, f in fns.items():
        for _ in range(2):
            f()
        torch.cuda.synchronize()
        path = dpg.last_path()
        tot, step, wb, nl, _ = steps_obj.run(f, steps, launches=dpg.last_launch_count)
        ph = phase_split(dpg, steps_obj, f, steps) if k.startswith("dpg") else None
        if k != "dpg_sort_join":
            okk = sampled_ok(out, lambda i: oracle.fk_join(w["fact"][i], w["fk"][i], w["dim"]), n,
                             k=4096, seed=3)
        else:
            okk = None
        res[k] = {"ms": med(tot), "value": alg / (med(tot) * 1e-3) / 1e9, "unit": "GB/s",
                  "phases_ms": ph, "plan_path": path if k.startswith("dpg") else None,
                  "launches_per_step": nl / steps, "parity_sampled_ok": okk}
    dpg.dpg_sync_status()
    d = res["dpg"]
    r = {"workload": workload_name(cfg, None), "plan_path": d["plan_path"], "value": d["value"],
         "frac_of_hbm_peak": d["value"] / peak, "ms": d["ms"], "phases_ms": d["phases_ms"],
         "direct": res["direct"], "dpg_seq3": res["dpg_seq3"], "dpg_sort_join": res["dpg_sort_join"],
         "dpg_over_direct": res["direct"]["ms"] / d["ms"],
         "parity_sampled_ok": d["parity_sampled_ok"],
         "alg_bytes_formula": "N_fact * (4 + 16 + 64 + 80)"}
    del out, fact, fk, dim
    return r


def run_c5_shard(args, torch, dpg, steps_obj, peak, steps):
    """Config 5's per-GPU shard on one GPU (2^27 x 100 B, P = 1 through the
    native exchange) and the same exchange for virtual ranks (P = 2, 4, 8 on
    this GPU, dpg_retrieve_dist_loopback, 2^26 records): the single-GPU cost of
    the multi-GPU path (no NVLink involved)."""
    import datagen
    import oracle
    rec = 100
    out = {}
    n = 1 << 27
    sid_s, sid_r = datagen.STREAMS[("c5", "src")], datagen.STREAMS[("c5", "rids")]
    src = torch.empty((n, rec), dtype=torch.uint8, device="cuda")
    datagen.random_bytes_cuda(src.view(-1), sid_s)
    rids = datagen.feistel_cuda(n, 0, n, sid_r)
    comm = dpg.dpg_comm_create(dpg.dpg_get_unique_id(), 1, 0)
    try:
        dst = torch.empty((n, rec), dtype=torch.uint8, device="cuda")
        f = lambda: dpg.dpg_retrieve_dist(comm, src, n, rids, dst)
        f()
        torch.cuda.synchronize()
        idx = np.unique(np.random.default_rng(5).integers(0, n, 256))
        rh = rids[torch.from_numpy(idx).cuda()].cpu().numpy().astype(np.uint64)
        ok = bool(np.array_equal(dst[torch.from_numpy(idx).cuda()].cpu().numpy(),
                                 oracle.retrieve_generated(rec, n, sid_s, rh)))
        tot, _, _, nl, _ = steps_obj.run(f, max(2, steps // 2), launches=dpg.last_launch_count)
        out["P1_native"] = {"n_total": n, "ms": med(tot),
                            "value": n * (2 * rec + 8) / (med(tot) * 1e-3) / 1e9, "unit": "GB/s",
                            "parity_sampled_ok": ok}
        del dst
    finally:
        dpg.dpg_comm_destroy(comm)
    del src, rids
    torch.cuda.empty_cache()
    n = 1 << 26
    src_all = torch.empty((n, rec), dtype=torch.uint8, device="cuda")
    datagen.random_bytes_cuda(src_all.view(-1), sid_s)
    rids_all = datagen.feistel_cuda(n, 0, n, sid_r)
    for P in (2, 4, 8):
        S = 1 << ((n + P - 1) // P - 1).bit_length()
        shards = [src_all[r * S:min(n, (r + 1) * S)] for r in range(P)]
        blocks = [rids_all[r * n // P:(r + 1) * n // P] for r in range(P)]
        dsts = [torch.empty((b.numel(), rec), dtype=torch.uint8, device="cuda") for b in blocks]
        f = lambda: dpg.dpg_retrieve_dist_loopback(shards, n, blocks, dsts)
        f()
        torch.cuda.synchronize()
        b0 = blocks[1]
        idx = np.unique(np.random.default_rng(P).integers(0, b0.numel(), 256))
        rh = b0[torch.from_numpy(idx).cuda()].cpu().numpy().astype(np.uint64)
        ok = bool(np.array_equal(dsts[1][torch.from_numpy(idx).cuda()].cpu().numpy(),
                                 oracle.retrieve_generated(rec, n, sid_s, rh)))
        tot, _, _, nl, _ = steps_obj.run(f, max(2, steps // 2), launches=dpg.last_launch_count)
        out[f"P{P}_virtual"] = {"n_total": n, "ms": med(tot),
                                "value": n * (2 * rec + 8) / (med(tot) * 1e-3) / 1e9,
                                "unit": "GB/s", "parity_sampled_ok": ok,
                                "what": "P virtual ranks on one GPU (loopback copies, no NVLink)"}
        del dsts
    return out


# ---------------------------------------------------------------------------
# N > 1: config 5 through the native multi-GPU C ABI
# ---------------------------------------------------------------------------
def run_c5(args, rank, world, local):
    import torch
    import torch.distributed as dist
    import datagen
    import oracle
    import paper_cs_0308004_b200 as dpg
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rec = 100
    n_total = 1 << args.c5_log2
    sid_s, sid_r = datagen.STREAMS[("c5", "src")], datagen.STREAMS[("c5", "rids")]
    S = 1 << (max(1, -(-n_total // world)) - 1).bit_length()
    lo, hi = min(n_total, rank * S), min(n_total, (rank + 1) * S)
    src = torch.empty((max(1, hi - lo), rec), dtype=torch.uint8, device=dev)
    if hi > lo:
        datagen.random_bytes_cuda(src.view(-1), sid_s, offset=lo * rec)
    b0, b1 = rank * n_total // world, (rank + 1) * n_total // world
    rids = datagen.feistel_cuda(n_total, b0, b1 - b0, sid_r)
    dst = torch.empty((b1 - b0, rec), dtype=torch.uint8, device=dev)
    # one NCCL unique id, made on rank 0 and broadcast
    uid = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(dpg.dpg_get_unique_id()), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    comm = dpg.dpg_comm_create(bytes(uid.cpu().numpy()), world, rank)
    rows = args.c5_rows
    # every rank makes the same number of calls (the exchange is collective)
    ncall = max(1, -(-max((r + 1) * n_total // world - r * n_total // world for r in range(world)) // rows))

    def step():
        for k in range(ncall):
            a = min(b1 - b0, k * rows)
            e = min(b1 - b0, (k + 1) * rows)
            dpg.dpg_retrieve_dist(comm, src if hi > lo else src[:0], n_total, rids[a:e], dst[a:e])

    for _ in range(max(1, min(args.warmup, 3))):
        step()
    torch.cuda.synchronize()
    dpg.dpg_sync_status()
    idx = np.unique(np.random.default_rng(rank).integers(0, b1 - b0, 256))
    rh = rids[torch.from_numpy(idx).to(dev)].cpu().numpy().astype(np.uint64)
    parity_ok = bool(np.array_equal(dst[torch.from_numpy(idx).to(dev)].cpu().numpy(),
                                    oracle.retrieve_generated(rec, n_total, sid_s, rh)))
    dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    with ClockSampler(local) as clk:
        ev0.record()
        for _ in range(args.steps):
            step()
            launches += dpg.last_launch_count()
        ev1.record()
        torch.cuda.synchronize()
    dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    okt = torch.tensor([1 if parity_ok else 0], dtype=torch.int64, device=dev)
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    alg = n_total * (2 * rec + 8)
    value = alg / (ms * 1e-3) / 1e9
    peak, peak_src = hbm_peak()
    # NVLink all-to-all roofline per GPU per direction: requests out (4 B) and
    # replies (rec B) for the (P-1)/P of rows whose owner is another rank
    nvl_bytes = (world - 1) / world * (n_total / world) * (rec + 4)
    t_nvl = nvl_bytes / (NVLINK_GBS * 1e9) * 1e3
    t_hbm = alg / world / (peak * 1e9) * 1e3
    # NCCL all-to-all bus bandwidth on equal 256 MiB per-rank buffers (SV 8(e))
    a2a_in = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    a2a_out = torch.empty_like(a2a_in)
    for _ in range(3):
        dist.all_to_all_single(a2a_out, a2a_in)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        dist.all_to_all_single(a2a_out, a2a_in)
    e1.record()
    torch.cuda.synchronize()
    tb = torch.tensor([e0.elapsed_time(e1) / 10], dtype=torch.float64, device=dev)
    dist.all_reduce(tb, op=dist.ReduceOp.MAX)
    busbw = (256 << 20) * (world - 1) / world / (float(tb.item()) * 1e-3) / 1e9
    del a2a_in, a2a_out
    # end to end through the same API: the step's rids from pinned host memory,
    # the rows back to pinned host memory, chunk by chunk
    e2e = None
    if not args.no_e2e:
        hr = rids.cpu().pin_memory()
        sub = min(rows, b1 - b0, 1 << 24)          # pinned host rows buffer: 1.7 GB at most
        hd = torch.empty((max(1, sub), rec), dtype=torch.uint8).pin_memory()
        rbuf = torch.empty(min(rows, b1 - b0), dtype=torch.int64, device=dev)

        def step_e2e():
            for k in range(ncall):
                a = min(b1 - b0, k * rows)
                e = min(b1 - b0, (k + 1) * rows)
                rbuf[:e - a].copy_(hr[a:e], non_blocking=True)
                dpg.dpg_retrieve_dist(comm, src if hi > lo else src[:0], n_total, rbuf[:e - a],
                                      dst[:e - a])
                for c0 in range(0, e - a, sub):     # the rows back to the host, chunk by chunk
                    c1 = min(e - a, c0 + sub)
                    hd[:c1 - c0].copy_(dst[c0:c1], non_blocking=True)
                    torch.cuda.current_stream().synchronize()

        step_e2e()
        dist.barrier()
        k = max(1, min(3, args.steps))
        t0 = time.perf_counter()
        for _ in range(k):
            step_e2e()
        el = (time.perf_counter() - t0) / k
        te = torch.tensor([el], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        el = float(te.item())
        e2e = {"value": alg / el / 1e9, "unit": "GB/s", "ms_per_step": el * 1e3,
               "h2d_bytes_per_step": int(n_total * 8), "d2h_bytes_per_step": int(n_total * rec),
               "entry": "dpg_retrieve_dist (rids H2D and rows D2H per call, pinned host buffers)"}
    cpu = None
    if rank == 0 and not args.no_cpu:
        n = 1 << 22
        hs = datagen.records(n, rec, sid_s)
        hrid = datagen.feistel(n, 0, n, sid_r).astype(np.uint32)
        cpu = cpu_baseline(hs, hrid, 2 * rec + 8,
                           sample="2^22 x 100 B of the c5 source stream, rids = the c5 Feistel "
                                  "permutation of [0, 2^22)")
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (datagen on device, seed 0)",
            "config": {"workload": workload_name("c5", None) + f" (2^{args.c5_log2} records)",
                       "n_total": n_total, "rec_bytes": rec, "rid_bytes": 8,
                       "parallelism": f"ep{world} (range-partitioned source, owner exchange)",
                       "rows_per_call": rows, "calls_per_step": ncall,
                       "l2": "inputs >> L2", "exchange": "native C ABI dpg_retrieve_dist: NCCL "
                       "counts + requests, owner DPG writes replies into peers' IPC windows"},
            "records_per_s": n_total / (ms * 1e-3),
            "roofline": {"bound": "nvlink" if t_nvl > t_hbm else "hbm", "unit": "GB/s",
                         "hbm": {"achieved": value / world, "peak": peak,
                                 "frac": value / world / peak, "peak_source": peak_src},
                         "nvlink": {"roofline_ms": t_nvl, "bytes_per_gpu_per_direction": nvl_bytes,
                                    "peak_gbs_per_direction": NVLINK_GBS,
                                    "frac": t_nvl / ms if t_nvl else None},
                         "achieved": value / world, "peak": peak, "frac": value / world / peak,
                         "traffic": None},
            "nccl_alltoall_busbw_gbs": busbw, "parity_sampled_ok": bool(okt.item()),
            "e2e": e2e, "cpu_baseline": cpu, "clocks": clk.summary(),
            "gpu_launches": launches, "gpu": torch.cuda.get_device_name(dev)}), flush=True)
    dist.barrier()
    torch.cuda.synchronize()
    dpg.dpg_comm_destroy(comm)
    dist.destroy_process_group()
    return 0


def run_h1(args):
    """Batch lookup in a hash index (section 4), DPG beside the
    direct lookup."""
    import torch
    import datagen
    import oracle
    import paper_cs_0308004_b200 as dpg
    torch.cuda.set_device(0)
    w = datagen.hash_workload(1 << 24, 24, 1 << 26)
    t = torch.from_numpy(w["table"].view(np.int32)).cuda()
    p = torch.from_numpy(w["pool"].view(np.int32)).cuda()
    q = torch.from_numpy(w["queries"].view(np.int32)).cuda()
    out = torch.empty_like(q)
    n = q.numel()
    steps_obj = Steps(torch, torch.device("cuda", 0))
    res = {}
    with ClockSampler(0) as clk:
        for direct in (False, True):
            f = lambda: dpg.dpg_hash_lookup(t, p, q, out=out, direct=direct)
            for _ in range(max(3, args.warmup)):
                f()
            torch.cuda.synchronize()
            idx = np.random.default_rng(0).integers(0, n, 4096)
            ok = np.array_equal(out.cpu().numpy().view(np.uint32)[idx],
                                oracle.batch_lookup(w["keys"], w["queries"][idx]))
            tot, _, _, nl, _ = steps_obj.run(f, args.steps, launches=dpg.last_launch_count)
            res[direct] = (med(tot), ok, nl)
    ms, ok, launches = res[False]
    dms, dok, _ = res[True]
    peak, _ = hbm_peak()
    alg = n * (4 + 16 + 4)
    print(json.dumps({
        "metric": "batch index lookups/s (hash index, DPG)", "value": n / (ms * 1e-3),
        "unit": "lookups/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic (datagen.hash_workload, seed 0)",
        "config": {"workload": "h1: hash index of 2^24 keys, 2^26 queries (5% absent)"},
        "effective_gbs": alg / (ms * 1e-3) / 1e9, "frac_of_hbm_peak": alg / (ms * 1e-3) / 1e9 / peak,
        "direct": {"value": n / (dms * 1e-3), "unit": "lookups/s", "ms_per_step": dms,
                   "parity_sampled_ok": bool(dok)},
        "parity_sampled_ok": bool(ok), "gpu_launches": launches, "clocks": clk.summary()}),
        flush=True)
    return 0


def main():
    args = parse()
    rc = relaunch_under_torchrun(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    rank, world, local = dist_env()
    if world > 1 or args.config == "c5":
        if "MASTER_ADDR" not in os.environ:        # single process without torchrun
            s = socket.socket()
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
            s.close()
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0",
                              WORLD_SIZE="1", LOCAL_RANK="0")
        return run_c5(args, rank, world, local)
    if args.config == "h1":
        return run_h1(args)
    return run_single(args)


if __name__ == "__main__":
    sys.exit(main())
