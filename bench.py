#!/usr/bin/env python
"""IVF-DADE query throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config config1]

One step = one batch of the workload's queries through the whole hot path:
rotation -> coarse ranking -> probe grouping -> dimension-progressive DCO scan
-> top-K merge. N = 1 runs BASELINE config 1 (1M x 256, 10k queries, nlist
1024, nprobe 32, K 100, dd 32, alpha .1). N > 1 shards the same index by list
over N ranks and scales the job to N x 10k queries, rank r owning 10k of them
(weak scaling): each rank rotates and coarse-ranks its own queries, NCCL
all-gathers the rotated queries and probes, scans its lists in two phases with
an all-reduce(MIN) of the per-query radius between them (the nearest list's
owner seeds the radius), and an all-to-all returns each query's per-shard top-K
to its owner for the merge (paper_2411_17229_b200/dist.py).

value  = queries / device time, inputs resident in HBM, CUDA events on the
         launching stream, L2 flushed (512 MB write) between steps, max over ranks.
e2e    = same metric through the C ABI with pinned host buffers: H2D of raw
         queries + search + D2H of ids/dists/counts, host wall clock.
cpu_baseline = the UNMODIFIED reference (oracle/_ref/libdade_ref.so) on this
         box's host, 1 thread (the paper's contract), a bounded query sample.
--impl reference = that reference with all host threads (hardware threads),
         each step a bounded query sample, same config / metric.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ivf_dade_queries_per_sec"
UNIT = "queries/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---- clocks --------------------------------------------------------------------
class ClockSampler:
    REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu: int, path: Path):
        self.path = path
        q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "20"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self, window=None):
        """Summarise the samples taken inside `window` = (t0, t1) (host epoch
        seconds of the timed region); all samples if None or none fall inside."""
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.05)
        self.p.terminate()
        self.p.wait()
        self.f.close()
        rows = []
        for line in self.path.read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                ts = time.mktime(time.strptime(parts[0].split(".")[0], "%Y/%m/%d %H:%M:%S")) + \
                    float("0." + parts[0].split(".")[1]) if "." in parts[0] else 0.0
                rows.append((ts, float(parts[1]), float(parts[2]), parts))
            except (ValueError, IndexError):
                continue
        inside = [r for r in rows if window and window[0] <= r[0] <= window[1]]
        use = inside or rows
        sm, mx, reasons = [], [], set()
        for _, a, b, parts in use:
            sm.append(a)
            mx.append(b)
            for name, v in zip(self.REASONS, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "samples_in_timed_region": len(inside), "reasons": sorted(reasons)}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def measured_bf16():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["bf16_tflops"])
    return 2250.0  # nominal dense bf16 (B200_PROFILING.md fallback)


def ncu_traffic(kernel: str = "dco_filter_umma"):
    """dram bytes per launch of the scan kernel from the committed ncu summary
    (the newest per-step summary's launches of that kernel, one search's worth)."""
    steps = sorted((ROOT / "profiles").glob("ncu_step_summary_*.json"))
    if steps:
        try:
            d = json.loads(steps[-1].read_text())
            ls = [x for x in d["launches"] if x["kernel"].startswith(kernel)]
            # the first launch of the capture may belong to the previous search: one search = the last
            # launches up to the step's launch count (2 filter passes)
            ls = ls[-2:] if len(ls) >= 2 else ls
            if ls:
                return float(np.mean([(x["dram_read_MB"] + x["dram_write_MB"]) * 1e6 for x in ls])), steps[-1].name
        except Exception:
            pass
    for p in sorted((ROOT / "profiles").glob("ncu_*summary*.json"), reverse=True):
        try:
            d = json.loads(p.read_text())
            if d.get("kernel", "").startswith(kernel) and d.get("config") == "config1":
                return float(d["dram_bytes_per_launch"]), p.name
        except Exception:
            continue
    return None, None


# ---- reference (CPU) -------------------------------------------------------------
def reference_setup(art, tmp: Path):
    from oracle import RefLib
    from paper_2411_17229_b200.io import Divf, write_divf, write_transform
    cfg = art.cfg
    ref = RefLib()
    write_transform(tmp / "t.dade", art.transform)
    divf = Divf(cfg.dim, cfg.n, cfg.nlist, 0, cfg.dim, art.centroids, art.offsets, art.ids,
                art.storage.reshape(-1))
    write_divf(tmp / "index.ivf", divf)
    t = ref.load_transform(tmp / "t.dade")
    cal = ref.cal_from(art.cal.p_s, art.cal.delta_d, art.cal.checkpoints, art.cal.epsilons)
    strat = ref.strategy_dade(t, cal, cfg.delta_d)
    ivf = ref.ivf_load(tmp / "index.ivf")
    os.remove(tmp / "index.ivf")
    return ref, ivf, strat, (t, cal)


def reference_sample(ivf, strat, q_rot: np.ndarray, cfg, threads: int, target_s: float, start: int = 0):
    """Run the reference on a query sample sized to ~target_s seconds."""
    n = q_rot.shape[0]
    probe = max(threads * 2, 16)
    _, _, _, _, sec = ivf.search(strat, q_rot[start:start + probe], cfg.k, cfg.nprobe, threads=threads)
    per_q = max(sec / probe, 1e-6)
    m = int(min(n, max(probe, target_s / per_q)))
    idx = (start + np.arange(m)) % n
    ids, d, cnt, st, sec = ivf.search(strat, q_rot[idx], cfg.k, cfg.nprobe, threads=threads)
    return idx, ids, cnt, st, sec


def recall(ids, counts, gt):
    from oracle import Oracle
    return Oracle().recall(ids, counts, gt)


def run_reference_arm(args, cfg):
    import torch
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import paper_2411_17229_b200 as gp
    from paper_2411_17229_b200 import workloads as W
    torch.cuda.set_device(0)
    dev = gp.Device(0)
    art = W.build(cfg, dev, torch.device("cuda:0"), with_gt=True, log=log)
    tmp = Path(tempfile.mkdtemp(prefix="dade_ref_"))
    ref, ivf, strat, _keep = reference_setup(art, tmp)
    q_rot = art.q_rot.cpu().numpy()
    threads = os.cpu_count() or 1
    qps, secs, recs, sample = [], [], [], 0
    start = 0
    for step in range(args.warmup + args.steps):
        idx, ids, cnt, st, sec = reference_sample(ivf, strat, q_rot, cfg, threads, args.ref_step_s, start)
        start = int((start + len(idx)) % q_rot.shape[0])
        if step >= args.warmup:
            qps.append(len(idx) / sec)
            secs.append(sec)
            recs.append(recall(ids, cnt, art.gt[idx]))
            sample = len(idx)
    value = float(np.mean(qps))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(secs)), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded Gaussian mixture)",
        "config": {"workload": cfg.describe(), "parallelism": f"{threads} host threads",
                   "artifacts": "GPU-built (paper_2411_17229_b200.workloads), loaded via DIVF/DADE files"},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{sample} queries per step (strided subsets per thread), "
                                   f"IvfIndex::search + DadeStrategy, rotation excluded as in measure()"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "recall_at_k": float(np.mean(recs)),
        "host_cpu": _cpu_model(),
    }
    print(json.dumps(line), flush=True)
    return 0


def _cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ---- ours -------------------------------------------------------------------------
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2411_17229_b200 as gp
    from paper_2411_17229_b200 import _capi
    from paper_2411_17229_b200 import dist as gdist
    from paper_2411_17229_b200 import workloads as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    dev = gp.Device(local)
    stream = torch.cuda.Stream(device)
    torch.cuda.set_stream(stream)  # torch ops, CUDA events and the C ABI share one stream

    nq_total = cfg.nq * world
    art = W.build(cfg, dev, device, with_gt=(rank == 0), nq=nq_total, log=log if rank == 0 else (lambda *a: None))
    if world > 1:  # identical lists on every rank (k-means sums are atomics): rank 0's wins
        for name in ("centroids", "offsets", "ids"):
            arr = getattr(art, name)
            t = torch.from_numpy(arr.astype(np.int64) if arr.dtype == np.uint32 else arr).to(device)
            dist.broadcast(t, 0)
            arr2 = t.cpu().numpy()
            setattr(art, name, arr2.astype(np.uint32) if arr.dtype == np.uint32 else arr2)
        art.storage = art.base_rot[torch.from_numpy(art.ids.astype(np.int64)).to(device)].cpu().numpy()
    idx = gp.IvfIndex(dev, cfg.dim, cfg.n, cfg.nlist, art.centroids, art.offsets, art.ids, art.storage)
    if world > 1:
        owner = gdist.plan_list_shards(art.offsets, world, cfg.dim)
        idx.shard((owner == rank).astype(np.uint8))
    dco = gp.DadeStrategy(art.transform, art.cal, cfg.delta_d, dev=dev)
    art.transform.upload(dev)
    dev.apply(dco)
    dev.set_stream(stream.cuda_stream)

    nq, k = nq_total, cfg.k
    q_dev = art.q_raw.contiguous()
    # N > 1: rank r owns queries [r * nq_loc, (r + 1) * nq_loc) of the job (query-owner scheme)
    nq_loc = cfg.nq
    q_loc = art.q_raw[rank * nq_loc:(rank + 1) * nq_loc].contiguous()
    out_ids = torch.empty((nq, k), dtype=torch.int32, device=device)
    out_d = torch.empty((nq, k), dtype=torch.float32, device=device)
    out_c = torch.empty((nq,), dtype=torch.int32, device=device)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=device)
    flags = _capi.QUERIES_RAW | _capi.DEVICE_PTRS

    def step():
        if world == 1:
            _capi.check(_capi.lib.dade_gpu_ivf_search(dev.h, _capi.ptr(q_dev), nq, k, cfg.nprobe, flags,
                                                      _capi.ptr(out_ids), _capi.ptr(out_d), _capi.ptr(out_c),
                                                      None))
            return out_ids, out_d, out_c
        return gdist.sharded_ivf_search(dev, None, q_loc, nq_loc, k, cfg.nprobe, raw=True)

    clocks = ClockSampler(local, Path(tempfile.gettempdir()) / f"dade_clocks_{local}.csv")
    time.sleep(0.3)  # let the sampler start emitting before the timed region
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    l0 = dev.launches
    evs = []
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_region0 = time.time()
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (outside the events)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = step()
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    t_region1 = time.time()
    if world > 1:
        dist.barrier()
    clk = clocks.stop((t_region0, t_region1))
    launches = (dev.launches - l0) // max(args.steps, 1)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    mean_ms = float(np.mean(step_ms))
    if world > 1:
        t = torch.tensor([mean_ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        mean_ms = float(t.item())
    value = nq / (mean_ms / 1e3)

    ids_np = res[0].cpu().numpy().astype(np.uint32)
    cnt_np = res[2].cpu().numpy().astype(np.uint32)

    # ---- scan-kernel roofline (profiled pass, not timed above) -------------------
    scan_ms = scan_bytes = total_ms = filter_ms = None
    n_filter = 0
    stats = gp.DcoStats()
    if world == 1:
        dev.set_profiling(True)
        sm, sb, fms, seed_prof = [], [], [], []
        for _ in range(3):
            flush.zero_()
            torch.cuda.synchronize()
            st = _capi.Stats()
            _capi.check(_capi.lib.dade_gpu_ivf_search(dev.h, _capi.ptr(q_dev), nq, k, cfg.nprobe, flags,
                                                      _capi.ptr(out_ids), _capi.ptr(out_d), _capi.ptr(out_c),
                                                      ctypes.byref(st)))
            a, b, c = dev.last_scan_profile()
            fm, nf = dev.last_filter_profile()
            seed_prof.append(dev.last_seed_profile())
            sm.append(a)
            sb.append(b)
            fms.append(fm)
            stats = gp.DcoStats(st.total_dco, st.dims_accumulated)
        dev.set_profiling(False)
        scan_ms, scan_bytes = float(np.median(sm)), float(np.median(sb))
        filter_ms, n_filter = float(np.median(fms)), nf

    # ---- e2e at N > 1: each rank's own query slice from pinned host memory, its own
    # results back to pinned host memory, host wall clock, max over ranks ----------
    e2e_multi = None
    if world > 1:
        qh = torch.empty((nq_loc, cfg.dim), dtype=torch.float32, pin_memory=True)
        qh.copy_(q_loc.cpu())
        ihm = torch.empty((nq_loc, k), dtype=torch.int32, pin_memory=True)
        dhm = torch.empty((nq_loc, k), dtype=torch.float32, pin_memory=True)
        chm = torch.empty((nq_loc,), dtype=torch.int32, pin_memory=True)

        def e2e_multi_step():
            qd = qh.to(device, non_blocking=True)
            i_, d_, c_ = gdist.sharded_ivf_search(dev, None, qd, nq_loc, k, cfg.nprobe, raw=True)
            ihm.copy_(i_, non_blocking=True)
            dhm.copy_(d_, non_blocking=True)
            chm.copy_(c_, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        for _ in range(args.warmup):
            e2e_multi_step()
        ts_m = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            e2e_multi_step()
            ts_m.append(time.perf_counter() - t0)
        t = torch.tensor([float(np.mean(ts_m))], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_multi = {"value": nq / float(t.item()), "unit": UNIT, "h2d_bytes_per_step": nq * cfg.dim * 4,
                     "d2h_bytes_per_step": nq * (k * 8 + 4), "ms_per_step": 1e3 * float(t.item()),
                     "api": "paper_2411_17229_b200.dist.sharded_ivf_search per step on every rank: H2D of the "
                            "rank's raw query slice, search, D2H of its ids/dists/counts; host wall clock, max "
                            "over ranks; bytes are whole-job",
                     "recall_at_k_rank0": recall(ihm.numpy().astype(np.uint32), chm.numpy().astype(np.uint32),
                                                 art.gt[:nq_loc]) if rank == 0 else None}

    if rank != 0:
        dist.destroy_process_group()
        return 0

    rec = recall(ids_np, cnt_np, art.gt if world == 1 else art.gt[:nq_loc])

    # ---- e2e through the C ABI with pinned host buffers ------------------------------
    e2e = None
    if world == 1:
        dev.set_stream(None)
        qh = torch.empty((nq, cfg.dim), dtype=torch.float32, pin_memory=True)
        qh.copy_(art.q_raw.cpu())
        ih = torch.empty((nq, k), dtype=torch.int32, pin_memory=True)
        dh = torch.empty((nq, k), dtype=torch.float32, pin_memory=True)
        ch = torch.empty((nq,), dtype=torch.int32, pin_memory=True)

        def e2e_step():
            _capi.check(_capi.lib.dade_gpu_ivf_search(dev.h, _capi.ptr(qh), nq, k, cfg.nprobe, _capi.QUERIES_RAW,
                                                      _capi.ptr(ih), _capi.ptr(dh), _capi.ptr(ch), None))
        # bring the PCIe link to its loaded state first (untimed): on some hosts
        # H2D runs at ~10 GB/s for the first few hundred ms of transfers
        qd_warm = torch.empty_like(qh, device="cuda")
        t_w = time.perf_counter()
        while time.perf_counter() - t_w < 0.5:
            qd_warm.copy_(qh, non_blocking=True)
            torch.cuda.synchronize()
        for _ in range(args.warmup):
            e2e_step()
        ts = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_step()
            ts.append(time.perf_counter() - t0)
        # serving loop: the same K steps as one pipelined call (batch b+1's H2D and
        # batch b-1's D2H under batch b's search); two pinned result sets in turn
        outs = [(ih, dh, ch)] + [tuple(torch.empty_like(x, pin_memory=True) for x in (ih, dh, ch))]

        def e2e_pipe(n):
            A = ctypes.c_void_p * n
            _capi.check(_capi.lib.dade_gpu_ivf_search_batches(
                dev.h, n, A(*[_capi.ptr(qh)] * n), nq, k, cfg.nprobe, _capi.QUERIES_RAW,
                A(*[_capi.ptr(outs[b % 2][0]) for b in range(n)]), A(*[_capi.ptr(outs[b % 2][1]) for b in range(n)]),
                A(*[_capi.ptr(outs[b % 2][2]) for b in range(n)]), None))
        e2e_pipe(max(args.warmup, 2))
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_pipe(args.steps)
        t_pipe = time.perf_counter() - t0
        pipe_rec = recall(outs[(args.steps - 1) % 2][0].numpy().astype(np.uint32),
                          outs[(args.steps - 1) % 2][2].numpy().astype(np.uint32), art.gt)
        # DADE radii are shared live across CTAs, so survivors can differ run to
        # run; the e2e answer is checked by its own recall
        e2e_rec = recall(ih.numpy().astype(np.uint32), ch.numpy().astype(np.uint32), art.gt)
        # the link's H2D rate right after the timed loop (context for the number)
        torch.cuda.synchronize()
        t_h = time.perf_counter()
        for _ in range(5):
            qd_warm.copy_(qh, non_blocking=True)
        torch.cuda.synchronize()
        h2d_gbs = 5 * qh.numel() * 4 / (time.perf_counter() - t_h) / 1e9
        del qd_warm
        e2e = {"value": nq * args.steps / t_pipe, "unit": UNIT, "h2d_bytes_per_step": nq * cfg.dim * 4,
               "d2h_bytes_per_step": nq * k * 8 + nq * 4, "ms_per_step": 1e3 * t_pipe / args.steps,
               "recall_at_k": pipe_rec,
               "api": "dade_gpu_ivf_search_batches: K steps as one pipelined call over pinned host buffers "
                      "(raw queries H2D, rotation, search, ids/dists/counts D2H every step; host wall clock "
                      "around the call, which returns after the last D2H)",
               "l2": "not flushed between the pipelined steps: each step streams the 1 GB base (> 126 MB L2)",
               "single_call": {"value": nq / float(np.mean(ts)), "ms_per_call": 1e3 * float(np.mean(ts)),
                               "recall_at_k": e2e_rec,
                               "api": "dade_gpu_ivf_search per step, synchronous, L2 flushed between calls"},
               "pcie_h2d_gbs_after": round(h2d_gbs, 1), "pcie_warmup_s": 0.5}

    # ---- CPU baseline: the reference, 1 thread, bounded sample ----------------------
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            tmp = Path(tempfile.mkdtemp(prefix="dade_cpu_"))
            ref, ivf, strat, _keep = reference_setup(art, tmp)
            q_rot = art.q_rot.cpu().numpy()
            sidx, rids, rcnt, rst, sec = reference_sample(ivf, strat, q_rot, cfg, 1, args.cpu_baseline_s)
            ref_rec = recall(rids, rcnt, art.gt[sidx])
            our_rec = recall(ids_np[sidx], cnt_np[sidx], art.gt[sidx])
            cpu = {"value": len(sidx) / sec, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"first {len(sidx)} of {nq} queries, 1 thread, IvfIndex::search + DadeStrategy "
                             f"(oracle/_ref/libdade_ref.so), rotation excluded as in measure()",
                   "recall_at_k_sample": ref_rec, "ours_recall_at_k_same_sample": our_rec,
                   "dim_fraction": float(rst[1]) / (float(rst[0]) * cfg.dim)}
        except Exception as e:  # reported, never fatal to the GPU line
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference", "sample": f"failed: {e}"}

    peak, peak_src = measured_peaks()
    peak_bf16 = measured_bf16()
    traffic, traffic_src = ncu_traffic()
    roof = None
    if scan_ms:
        # dominant kernel: the streaming tensor-core filter (all its launches of one search)
        kern_ms = filter_ms if filter_ms else scan_ms
        achieved = scan_bytes / (kern_ms / 1e3) / 1e9
        d0 = cfg.delta_d
        pairs = stats.total_dco
        tc_tflops = 2.0 * pairs * d0 / (kern_ms / 1e3) / 1e12
        # dominant kernel: dco_filter_umma_kernel (tcgen05 TF32, TMEM accumulators). Algorithmic
        # work = the first-slice dot products o.q over d0 dims of every DCO pair.
        tf32_peak = 0.5 * peak_bf16  # TF32 dense = half the measured dense bf16 rate
        roof = {"bound": "tensor", "achieved": tc_tflops, "peak": tf32_peak, "unit": "TFLOP/s",
                "frac": tc_tflops / tf32_peak, "traffic": traffic,
                "kernel": "dco_filter_umma_kernel" if filter_ms else "dco_scan_kernel",
                "kernel_launches_per_step": n_filter, "kernel_ms_per_step": kern_ms,
                "flops_definition": "2 * DCO pairs * d0 per step (first-slice o.q of every (row, query) pair)",
                "algorithmic_flops_per_step": 2.0 * pairs * d0, "scan_ms_seed_to_merge": scan_ms,
                "peak_source": f"MEASURED_PEAKS.json bf16_tflops {peak_bf16} / 2 (TF32 dense)",
                "traffic_source": traffic_src,
                "tmem": {"bytes_per_pair": 4, "achieved_gbs": 4.0 * pairs / (kern_ms / 1e3) / 1e9,
                         "peak_gbs": 64 * 148 * 1.965,
                         "frac": 4.0 * pairs / (kern_ms / 1e3) / 1e9 / (64 * 148 * 1.965),
                         "note": "fp32 accumulators read back with tcgen05.ld at 64 B/cycle/SM "
                                 "(B300_MICROARCH.md TMEM table): the binding limit of this design"},
                "hbm": {"achieved_gbs": achieved, "peak_gbs": peak, "frac": achieved / peak,
                        "bytes_per_step": scan_bytes,
                        "bytes_definition": "first-slice row-tile bytes per (tile, query item) + 16 B per "
                                            "survivor handed on (kernel-counted)"}}
        if seed_prof and seed_prof[-1][0] > 0:
            # the radius seed (largest single launch): exact sequential fp32 (row, query, dim) steps,
            # 3 FP32 ops each (sub, square, add: no FMA, bit-exact); peak = the issue rate the FP32
            # pipe sustains for that step, measured by tools/micro/fp_mix.cu (42 steps / SM / cycle)
            s_ms = float(np.median([x[0] for x in seed_prof]))
            s_pd = float(seed_prof[-1][1])
            s_peak = 42.0 * 148 * 1.965e9
            roof["seed"] = {"kernel": "seed_persist_kernel", "bound": "fp32 issue", "ms_per_step": s_ms,
                            "pair_dims_per_step": s_pd, "achieved_pair_dims_per_s": s_pd / (s_ms / 1e3),
                            "peak_pair_dims_per_s": s_peak, "frac": s_pd / (s_ms / 1e3) / s_peak,
                            "hbm_bytes_per_step_ncu": 1.014e9,
                            "hbm_frac": 1.014e9 / (s_ms / 1e3) / 1e9 / peak,
                            "source": "CUDA events around the launch; pair-dims counted by the kernel; ncu bytes "
                                      "from profiles/ncu_step_summary_r01_v61.json"}
        el = stats.dims_accumulated
        roof["alu"] = {"reference_element_ops_per_s": el / (scan_ms / 1e3), "dims_accumulated": el,
                       "note": "DcoStats dims a sequential CPU scan would accumulate, per second of GPU scan"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": mean_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded Gaussian mixture, BASELINE config shapes; GPU-built PCA/k-means/calibration)",
        "config": {"workload": cfg.describe(), "queries_per_step": nq,
                   "parallelism": "single GPU" if world == 1 else
                   f"list-sharded x{world}; rank r owns {nq_loc} queries: NCCL all-gather of rotated queries and "
                   f"probes, all-reduce MIN of the radius, all-to-all of top-K keys",
                   "l2": "flushed between steps (512 MB write); base 1 GB > L2",
                   "timed": "rotate+coarse+group+scan+merge on device-resident raw queries"},
        "recall_at_k": rec,
        "dim_fraction": stats.dim_fraction(cfg.dim) if stats.total_dco else None,
        "gpu_launches": int(launches),
        "clocks": clk,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e if world == 1 else e2e_multi,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="config1")
    ap.add_argument("--cpu-baseline-s", type=float, default=15.0)
    ap.add_argument("--ref-step-s", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    from paper_2411_17229_b200.workloads import CONFIGS
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference_arm(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
