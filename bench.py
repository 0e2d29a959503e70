#!/usr/bin/env python3
"""Benchmark of the DPG record-retrieval hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dpg|reference]
                    [--config c2] [--rec R]

One step = one pass of the whole hot path (plan,
distribute, fused probe+gather) over one batch of synthetic input already
resident in HBM: dpg_retrieve on BASELINE.json configs[1] (Datamation-shaped
sort phase 3, 1,048,576 x 100-byte records, rids = stable argsort of the
10-byte keys).  L2 is flushed (a 512 MiB write, then a 512 MiB read, so no
dirty flush line is left for the step to write back) before every timed step and
each step is timed alone with CUDA events on the launching stream; flush time
is excluded.  Multi-process (torchrun, N > 1): BASELINE.json config 5 --
2^30 x 100-byte records range-partitioned over the ranks, rids a global
permutation block-partitioned by output position -- through the multi-GPU
path (owner partition, NCCL all-to-alls, local DPG, reply scatter); job time
= max over ranks of the CUDA-event time.

The JSON line adds: roofline of the dominant kernel (k_dpg_fused) from its
own CUDA-event time inside the same timed steps, the naive direct-gather
comparison timed the same way, the end-to-end number through the host-buffer
C-ABI entry, the oracle's CPU throughput (cpu_baseline) and the SM clocks
sampled during the timed region.
"""
from __future__ import annotations

import argparse

import numpy as np
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "record-retrieval effective GB/s vs HBM peak; records/s at 1/2/4/8 B200"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="dpg", choices=["dpg", "reference"])
    ap.add_argument("--config", default=None, choices=["c1", "c2", "c3a", "c3b", "c4", "c4x", "c5", "h1"],
                    help="default: c2 on one GPU, c5 (multi-GPU exchange) under torchrun")
    ap.add_argument("--c5-log2", type=int, default=30, help="c5 total records = 2^c5_log2")
    ap.add_argument("--c5-round-rows", type=int, default=1 << 27,
                    help="c5 rows per exchange round (bounds the windows: 13.4 GB per rank)")
    ap.add_argument("--exchange", default="fused", choices=["fused", "nccl"],
                    help="c5: replies written into the requesters' windows over NVLink "
                         "(fused) or returned by an NCCL all-to-all")
    ap.add_argument("--rec", type=int, default=None, help="record bytes for c3a/c3b")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sort", action="store_true", help="skip the end-to-end DPG sort timing (c2)")
    a = ap.parse_args()
    if a.config is None:
        a.config = "c5" if int(os.environ.get("WORLD_SIZE", "1")) > 1 else "c2"
    return a


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_name(cfg: str, rec: int | None) -> str:
    return {"c1": "c1: 65,536 x 100 B random records, uniform random permutation",
            "c2": "c2: Datamation sort phase 3, 1,048,576 x 100 B, rids = stable argsort of 10-B keys",
            "c3a": f"c3a: 16,777,216 x {rec} B, uniform random permutation",
            "c3b": f"c3b: 16,777,216 x {rec} B, uniform rids with replacement",
            "c4": "c4: DPG-Move FK join, dim 16,777,216 x 64 B, fact 67,108,864 x (fk + 16 B)",
            "c4x": "c4x: config 4 with the paper's exponential join keys (P:890-892)",
            "c5": "c5 sample for the host oracle: 2^22 x 100 B of the c5 source stream, "
                  "rids = c5 Feistel permutation of [0, 2^22)"}[cfg]


def make_inputs(cfg: str, rec: int | None):
    import datagen
    if cfg in ("c3a", "c3b"):
        return datagen.make(cfg, rec=rec or 64)
    return datagen.make(cfg)


def units(cfg, w):
    """(n_out, rec, algorithmic bytes per step, rid bytes) per SURVEY 8(d):
    B = N * (2 * rec + rid_bytes)."""
    if cfg in ("c4", "c4x"):
        n_out = w["fk"].size
        rec = w["dim"].shape[1] + w["fact"].shape[1]          # 80-byte output rows
        # join rows: read fk (4) + fact payload (16) + dim record (64), write 80
        return n_out, rec, n_out * (4 + 16 + 64 + 80), 4
    n_out = w["rids"].size
    rec = w["src"].shape[1]
    return n_out, rec, n_out * (2 * rec + 4), 4


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

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
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
            "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
            "display_clock_setting": 0x100,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit and k != "gpu_idle":
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
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            v = float(json.load(f)["hbm_gbs"])
        return v, "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def committed_traffic(cfg):
    """dram bytes per probe-gather launch from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(cfg)
    except Exception:
        return None


def cpu_baseline(cfg, w, budget_s=10.0):
    """The oracle as it stands (single-threaded C loop, oracle/oracle.c) on this
    host, repeated over the full workload until ~budget_s of CPU work."""
    import oracle
    n_out, rec, alg_bytes, _ = units(cfg, w)
    fn = (lambda: oracle.fk_join(w["fact"], w["fk"], w["dim"])) if cfg in ("c4", "c4x") else \
        (lambda: oracle.retrieve(w["src"], w["rids"]))
    fn()  # warm (page in)
    reps, t0 = 0, time.perf_counter()
    while True:
        fn()
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or (reps >= 3 and el > budget_s / 2):
            break
    t = el / reps
    return {"value": alg_bytes / t / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "records_per_s": n_out / t,
            "sample": f"full {cfg} workload x {reps} repetitions ({el:.1f} s), "
                      f"oracle.retrieve single-threaded C loop",
            "host_cpu": host_cpu(), "host_threads": os.cpu_count()}


def host_cpu():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cfg = args.config
    if cfg == "h1":
        import datagen
        import oracle
        w = datagen.hash_workload(1 << 24, 24, 1 << 26)
        q = w["queries"][: 1 << 24]              # bounded sample: a quarter of the queries
        times = []
        for _ in range(max(1, args.steps)):
            t0 = time.perf_counter()
            oracle.batch_lookup(w["keys"], q)
            times.append(time.perf_counter() - t0)
            if sum(times) > 120:
                break
        t = sum(times) / len(times)
        value = q.size / t
        print(json.dumps({
            "impl": "reference", "metric": "batch index lookups/s (hash index, DPG)", "value": value,
            "unit": "lookups/s", "n_gpus": world, "steps": len(times), "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic (datagen.hash_workload, seed 0)",
            "config": {"workload": "h1 sample: 2^24 of the 2^26 queries"},
            "cpu_baseline": {"value": value, "unit": "lookups/s", "cores": 1, "kind": "oracle",
                             "sample": "2^24 queries, oracle.batch_lookup (sorted pairs + binary search)",
                             "host_cpu": host_cpu()},
            "e2e": {"value": value, "unit": "lookups/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}), flush=True)
        return 0
    if cfg == "c5":
        # bounded sample of the c5 workload for the host oracle: 2^22 records
        # of the c5 source stream, rids = the c5 Feistel permutation of [0, 2^22)
        import datagen
        n = 1 << 22
        w = {"src": datagen.records(n, 100, datagen.STREAMS[("c5", "src")]),
             "rids": datagen.feistel(n, 0, n, datagen.STREAMS[("c5", "rids")]).astype(np.uint32)}
        cfg = "c2"     # same shape of work (100-byte records, 4-byte rids) for units()
    else:
        w = make_inputs(cfg, args.rec)
    import oracle
    n_out, rec, alg_bytes, _ = units(cfg, w)
    fn = (lambda: oracle.fk_join(w["fact"], w["fk"], w["dim"])) if cfg in ("c4", "c4x") else \
        (lambda: oracle.retrieve(w["src"], w["rids"]))
    for _ in range(max(0, min(args.warmup, 3))):
        fn()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
        if sum(times) > 120:
            break
    t = sum(times) / len(times)
    value = alg_bytes / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": world, "steps": len(times), "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (datagen, seed 0)",
        "config": {"workload": workload_name(args.config, args.rec), "n_out": n_out, "rec_bytes": rec},
        "records_per_s": n_out / t,
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": f"full {cfg} workload, {len(times)} steps",
                         "host_cpu": host_cpu()},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_c5(args, rank, world):
    """BASELINE.json config 5: 2^30 x 100-byte records range-partitioned over the
    ranks, rids = a Feistel permutation of [0, 2^30) block-partitioned by output
    position; the multi-GPU path (paper_cs_0308004_b200/dist.py): owner
    partition, NCCL all-to-alls, local DPG, reply scatter.  Inputs are
    generated on each GPU by the counter-based generators (datagen)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import datagen
    from paper_cs_0308004_b200.dist import PeerWindows, owned_range, retrieve_dist
    dev = torch.device("cuda", torch.cuda.current_device())
    rec = 100
    n_total = 1 << args.c5_log2
    lo, hi = owned_range(rank, world, n_total)
    src = torch.empty((hi - lo, rec), dtype=torch.uint8, device=dev)
    datagen.random_bytes_cuda(src.view(-1), datagen.STREAMS[("c5", "src")], offset=lo * rec)
    b0, b1 = rank * n_total // world, (rank + 1) * n_total // world
    rids = datagen.feistel_cuda(n_total, b0, b1 - b0, datagen.STREAMS[("c5", "rids")])
    torch.cuda.synchronize()

    # fused exchange: one receive window per rank, mapped into every peer (CUDA
    # IPC); if any rank cannot map its peers, every rank uses the NCCL replies
    exchange, win = args.exchange, None
    if exchange == "fused":
        ok = 1
        try:
            win = PeerWindows(min(args.c5_round_rows, b1 - b0) * rec)
        except Exception as e:  # noqa: BLE001 -- reported in the JSON line
            print(f"fused exchange unavailable on rank {rank}: {e}", file=sys.stderr)
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int64, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if not flag.item():
            if win is not None:
                win.close()
            win, exchange = None, "nccl (fused windows unavailable)"

    def step():
        return retrieve_dist(src, rids, n_total, max_rows_per_round=args.c5_round_rows,
                             fused=win is not None, windows=win)

    out = None
    for _ in range(max(1, min(args.warmup, 3))):
        out = step()
    torch.cuda.synchronize()
    # sampled parity against the host generators (the definition, pointwise)
    idx = np.random.default_rng(rank).integers(0, b1 - b0, 256)
    got = out[torch.from_numpy(idx).to(dev)].cpu().numpy()
    want_r = datagen.feistel(n_total, b0, b1 - b0, datagen.STREAMS[("c5", "rids")])[idx] \
        if b1 - b0 <= (1 << 26) else np.array(
            [datagen.feistel(n_total, b0 + int(j), 1, datagen.STREAMS[("c5", "rids")])[0] for j in idx])
    want = np.stack([datagen.random_bytes(rec, datagen.STREAMS[("c5", "src")], offset=int(r) * rec)
                     for r in want_r])
    parity_ok = bool(np.array_equal(got, want))
    del out
    dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        ev0.record()
        for _ in range(args.steps):
            out = step()
            del out
        ev1.record()
        torch.cuda.synchronize()
    dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ok = torch.tensor([1 if parity_ok else 0], dtype=torch.int64, device=dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    alg = n_total * (2 * rec + 8)
    value = alg / (ms * 1e-3) / 1e9
    # NCCL all-to-all bus bandwidth on equal 256 MiB per-rank buffers (SV 8(e))
    busbw = None
    if world > 1:
        a2a_in = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        a2a_out = torch.empty_like(a2a_in)
        for _ in range(3):
            dist.all_to_all_single(a2a_out, a2a_in)
        torch.cuda.synchronize()
        b0e, b1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0e.record()
        for _ in range(10):
            dist.all_to_all_single(a2a_out, a2a_in)
        b1e.record()
        torch.cuda.synchronize()
        t = torch.tensor([b0e.elapsed_time(b1e) / 10], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        busbw = (256 << 20) * (world - 1) / world / (float(t.item()) * 1e-3) / 1e9
        del a2a_in, a2a_out
    peak, peak_src = hbm_peak()
    nvl = (world - 1) / world * (n_total / world) * (rec + 4) / 900e9 * 1e3 if world > 1 else 0.0
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (datagen on device, seed 0)",
            "config": {"workload": f"c5: 2^{args.c5_log2} x 100 B range-partitioned, rids = Feistel "
                                   "permutation (uint64) block-partitioned", "n_total": n_total,
                       "rec_bytes": rec, "rid_bytes": 8, "parallelism": f"ep{world} (owner exchange)",
                       "round_rows": args.c5_round_rows, "l2": "inputs >> L2",
                       "exchange": exchange},
            "records_per_s": n_total / (ms * 1e-3),
            "frac_of_hbm_peak_aggregate": value / (world * peak),
            "nvlink_roofline_ms": nvl, "frac_of_nvlink_roofline": (nvl / ms) if nvl else None,
            "nccl_alltoall_busbw_gbs": busbw,
            "parity_sampled_ok": bool(ok.item()),
            "clocks": clk.summary(), "gpu": torch.cuda.get_device_name(dev)}), flush=True)
    dist.barrier()
    if win is not None:
        torch.cuda.synchronize()
        dist.barrier()
        win.close()
    dist.destroy_process_group()
    return 0


def run_h1(args):
    """Batch lookup in a hash index (section 4): an index of 2^24
    distinct keys (2^24 slots of 16 B + slot-ordered overflow, 268 MB) and
    2^26 queries (5% absent).  DPG (distribute by partition, probe with the
    partition L2-resident, gather) beside the direct lookup."""
    import numpy as np
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
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    flush_rd = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def timed(direct):
        for _ in range(max(3, args.warmup)):
            dpg.dpg_hash_lookup(t, p, q, out=out, direct=direct)
        torch.cuda.synchronize()
        idx = np.random.default_rng(0).integers(0, n, 4096)
        ok = np.array_equal(out.cpu().numpy().view(np.uint32)[idx],
                            oracle.batch_lookup(w["keys"], w["queries"][idx]))
        ms = []
        launches = 0
        for _ in range(args.steps):
            flush.fill_(1)
            flush_rd.view(torch.int32).max()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dpg.dpg_hash_lookup(t, p, q, out=out, direct=direct)
            e1.record()
            launches += dpg.last_launch_count()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        return sum(ms) / len(ms), ok, launches

    with ClockSampler(0) as clk:
        ms, ok, launches = timed(False)
    dms, dok, _ = timed(True)
    alg = n * (4 + 16 + 4)        # key in, the key's 16-byte slot, rid out
    cpu = None
    if not args.no_cpu:
        qs = w["queries"][: 1 << 22]
        t0 = time.perf_counter()
        oracle.batch_lookup(w["keys"], qs)
        tc = time.perf_counter() - t0
        cpu = {"value": qs.size / tc, "unit": "lookups/s", "cores": 1, "kind": "oracle",
               "sample": "2^22 of the queries, oracle.batch_lookup (sorted pairs + binary search)",
               "host_cpu": host_cpu()}
    peak, peak_src = hbm_peak()
    print(json.dumps({
        "metric": "batch index lookups/s (hash index, DPG)", "value": n / (ms * 1e-3),
        "unit": "lookups/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic (datagen.hash_workload, seed 0)",
        "config": {"workload": "h1: hash index of 2^24 keys (2^24 slots x 16 B, overflow in slot "
                               "order), 2^26 queries (5% absent)", "slots": 1 << 24,
                   "pool_entries": int(w["pool"].shape[0]), "queries": n,
                   "l2": "flushed before every step"},
        "effective_gbs": alg / (ms * 1e-3) / 1e9, "frac_of_hbm_peak": alg / (ms * 1e-3) / 1e9 / peak,
        "direct": {"value": n / (dms * 1e-3), "unit": "lookups/s", "ms_per_step": dms,
                   "parity_sampled_ok": bool(dok)},
        "parity_sampled_ok": bool(ok), "gpu_launches": launches, "cpu_baseline": cpu,
        "clocks": clk.summary()}),
        flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "h1":
        return run_h1(args)
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world > 1 or args.config == "c5":
        torch.cuda.set_device(local)
        if "MASTER_ADDR" not in os.environ:        # single process without torchrun
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0", WORLD_SIZE="1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    import numpy as np
    import paper_cs_0308004_b200 as dpg

    cfg = args.config
    if cfg == "c5":
        return run_c5(args, rank, world)
    w = make_inputs(cfg, args.rec)
    n_out, rec, alg_bytes, rid_bytes = units(cfg, w)
    dev = torch.device("cuda", torch.cuda.current_device())

    def to_dev(a):
        a = np.ascontiguousarray(a)
        if a.dtype == np.uint32:
            a = a.view(np.int32)
        return torch.from_numpy(a).to(dev)

    if cfg in ("c4", "c4x"):
        fact, fk, dim = to_dev(w["fact"]), to_dev(w["fk"]), to_dev(w["dim"])
        out = torch.empty((n_out, rec), dtype=torch.uint8, device=dev)
        step = lambda: dpg.dpg_fk_join(fact, fk, dim, out=out)
        naive = windowed = None
        n_src = dim.shape[0]
    else:
        src, rids = to_dev(w["src"]), to_dev(w["rids"])
        out = torch.empty((n_out, rec), dtype=torch.uint8, device=dev)
        step = lambda: dpg.dpg_retrieve(src, rids, dst=out)
        naive = lambda: dpg.dpg_retrieve_direct(src, rids, dst=out)
        windowed = lambda: dpg.dpg_retrieve_direct_ex(src, rids, dst=out, hint=3)
        n_src = src.shape[0]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    flush_rd = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def flush_l2():
        # evict L2: write a buffer > 126 MB, then read another one, so that no
        # dirty line of the flush itself is left for the timed step to write back
        flush.fill_(1)
        flush_rd.view(torch.int32).max()

    def timed(fn, steps, phase=False):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        if phase:
            dpg.dpg_phase_times()
            dpg.dpg_phase_timing(True)
        launches = 0
        for e0, e1 in evs:
            flush_l2()
            e0.record(stream)
            fn()
            e1.record(stream)
            launches += dpg.last_launch_count()
        torch.cuda.synchronize()
        ph = None
        if phase:
            dpg.dpg_phase_timing(False)
            ph = dpg.dpg_phase_times()
        ms = [a.elapsed_time(b) for a, b in evs]
        return ms, launches, ph

    # warm-up
    for _ in range(max(3, args.warmup)):
        step()
        if naive:
            naive()
        if windowed:
            windowed()
    torch.cuda.synchronize()
    dpg.dpg_sync_status()

    step()
    ran_path = dpg.last_path()       # the plan the calls ran (after the skew check)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        ms, launches, _ = timed(step, args.steps)
    # the dominant kernel's own duration (CUDA events the library records on the
    # launching stream around its kernel), from a second pass of the same steps
    _, _, ph = timed(step, args.steps, phase=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    dpg.dpg_sync_status()
    total_ms = sum(ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * alg_bytes / (ms_per_step * 1e-3) / 1e9

    # naive comparison, same protocol
    naive_res = None
    if naive is not None:
        nms, nl, _ = timed(naive, args.steps)
        nt = sum(nms) / len(nms)
        naive_res = {"value": alg_bytes / (nt * 1e-3) / 1e9, "unit": "GB/s",
                     "ms_per_step": nt, "kernel": "k_direct", "launches_per_step": nl / args.steps}
    # the same direct retrieval on the best gather engine written here (the
    # L2-run kernel's 16-byte-window gather, no staging): the strongest
    # non-DPG comparison
    windowed_res = None
    if windowed is not None:
        wms, wl, _ = timed(windowed, args.steps)
        wt = sum(wms) / len(wms)
        windowed_res = {"value": alg_bytes / (wt * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": wt,
                        "kernel": "k_dpg_l2run (stage=0)", "launches_per_step": wl / args.steps}

    # the paper's application of the path (section 3): the whole Datamation
    # sort on the GPU -- key extraction + stable radix sort of the key-pointer
    # pairs (phases 1-2) + DPG retrieval (phase 3), timed the same way
    sort_res = None
    if cfg == "c2" and not args.no_sort:
        srids = torch.empty(n_out, dtype=torch.int32, device=dev)
        for _ in range(2):
            dpg.dpg_sort(src, 0, 10, dst=out)
        torch.cuda.synchronize()
        assert np.array_equal(out[:1000].cpu().numpy(), w["src"][w["rids"][:1000].astype(np.int64)])
        sms, sl, _ = timed(lambda: dpg.dpg_sort(src, 0, 10, dst=out), args.steps)
        rms, _, _ = timed(lambda: dpg.dpg_sort_rids(src, 0, 10, rids=srids), args.steps)
        st_ = sum(sms) / len(sms)
        sort_res = {"records_per_s": n_out / (st_ * 1e-3), "ms_per_sort": st_,
                    "ms_phases_1_2": sum(rms) / len(rms), "ms_phase_3": ms_per_step,
                    "launches_per_sort": sl / args.steps,
                    "what": "dpg_sort: 10-byte keys at offset 0, stable LSD radix sort "
                            "(10 passes) + dpg_retrieve"}
    # the paper's DPG-Sort join: the same join in fk order
    join_sort_res = None
    if cfg in ("c4", "c4x") and not args.no_sort:
        js = lambda: dpg.dpg_fk_join_sort(fact, fk, dim, out=out)
        for _ in range(2):
            js()
        torch.cuda.synchronize()
        dpg.dpg_sync_status()
        jms, jl, _ = timed(js, args.steps)
        jt = sum(jms) / len(jms)
        join_sort_res = {"value": alg_bytes / (jt * 1e-3) / 1e9, "unit": "GB/s",
                         "ms_per_step": jt, "launches_per_step": jl / args.steps,
                         "what": "dpg_fk_join_sort: stable radix sort of (rid_R, fk) pairs by "
                                 "fk + DPG retrieval of fact rows into a temporary file + "
                                 "zip with dim rows read in fk order"}
    peak, peak_src = hbm_peak()
    dist_ms, probe_ms, calls = ph
    pg_ms = probe_ms / max(1, calls)
    # (the join runs a DPG retrieval of dim rows -- no payload -- then a zip pass)
    plan = dpg.dpg_plan(rec if cfg not in ("c4", "c4x") else w["dim"].shape[1], n_src, n_out, 0,
                        torch.cuda.get_device_properties(dev).multi_processor_count)
    src_rec = w["dim"].shape[1] if cfg in ("c4", "c4x") else rec
    pay = 0
    if plan["path"] == 5:
        # K staged L2 runs probed into INTERNAL + the Phase III gather: the
        # L2-run kernel launches between the distribute and the end of the call
        kernel = "k_dpg_l2run (K runs + Phase III)"
        pg_bytes = alg_bytes
    elif plan["path"] == 3:
        # one run (the whole source) staged in L2, probed in rid order: one
        # kernel for the whole path, N * (2 * rec + rid_bytes)
        kernel = "k_dpg_l2run"
        pg_bytes = alg_bytes
    elif plan["path"] == 1:
        # one persistent kernel runs the whole path: its algorithmic bytes are
        # the path's, N * (2 * rec + rid_bytes)
        kernel = "k_dpg_fused" + (" + k_direct(INTERNAL)" if plan["gather"] == 2 else "")
        pg_bytes = alg_bytes
    else:
        # probe-gather kernel: every source record staged once + every output
        # row written once + its entry (and payload) read once
        kernel = "k_probe_gather"
        pg_bytes = n_src * src_rec + n_out * (rec + plan["pair_bytes"] + pay)
    achieved = pg_bytes / (pg_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": kernel, "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": committed_traffic(cfg),
                "peak_source": peak_src,
                "alg_bytes_per_launch": pg_bytes,
                "launch_ms": pg_ms,
                "share_of_step": probe_ms / max(1e-9, sum(ms)),
                "distribute_ms": dist_ms / max(1, calls),
                "path_frac_of_peak": value / world / peak}

    # end to end through the host-buffer C-ABI entry
    e2e = None
    if not args.no_e2e and cfg not in ("c4", "c4x"):
        hs = torch.from_numpy(w["src"]).pin_memory()
        hr = torch.from_numpy(w["rids"].view(np.int32)).pin_memory()
        hd = torch.empty((n_out, rec), dtype=torch.uint8).pin_memory()
        for _ in range(2):
            dpg.dpg_retrieve_host(hs, hr, hd)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            dpg.dpg_retrieve_host(hs, hr, hd)
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": world * alg_bytes / (el / args.steps) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": int(w["src"].nbytes + w["rids"].nbytes),
               "d2h_bytes_per_step": int(n_out * rec),
               "ms_per_step": el / args.steps * 1e3, "entry": "dpg_retrieve_host"}
        assert np.array_equal(hd[:1000].numpy(), w["src"][w["rids"][:1000].astype(np.int64)])
        dpg.dpg_release_cache()

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline(cfg, w)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic (datagen, seed 0)",
            "config": {"workload": workload_name(cfg, args.rec), "n_src": n_src, "n_out": n_out,
                       "rec_bytes": rec, "rid_bytes": rid_bytes,
                       "alg_bytes_per_step": alg_bytes,
                       "l2": "flushed before every step (512 MiB write, then 512 MiB read)",
                       "parallelism": "replicas" if world > 1 else "single",
                       "run_len": plan["run_len"], "num_runs": plan["num_runs"],
                       "pair_bytes": plan["pair_bytes"], "plan_path": ran_path},
            "records_per_s": world * n_out / (ms_per_step * 1e-3),
            "frac_of_hbm_peak": value / world / peak,
            "ms_min": min(ms), "ms_median": sorted(ms)[len(ms) // 2],
            "roofline": roofline, "naive": naive_res, "direct_windowed": windowed_res,
            "dpg_join_sort": join_sort_res,
            "dpg_sort": sort_res,
            "e2e": e2e, "cpu_baseline": cpu,
            "clocks": clk.summary(), "gpu_launches": launches,
            "gpu": torch.cuda.get_device_name(dev),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
