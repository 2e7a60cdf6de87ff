#!/usr/bin/env python
"""IVF-DADE query throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config config1]

One step = one batch of the workload's queries through the whole hot path:
rotation -> coarse ranking -> probe grouping -> dimension-progressive DCO scan
-> top-K merge.

Workloads (BASELINE.json configs, seeded synthetic data of those shapes; the
artifacts -- PCA transform, calibration, IVF lists, ground truth -- are built
once per box on the GPU with the reference's arithmetic by
paper_2411_17229_b200.workloads and saved in the reference's file formats
under /tmp; both arms load the same files):
  * N = 1: config 1 (1M x 256, 10k queries, nlist 1024, nprobe 32, K 100,
    dd 32, p_s .1). The same line carries a `config2` block (1M x 960, 1k
    queries, nprobe 64, K 20, dd 64, p_s .05), the long-vector config the
    north_star's HBM target is about, and a `config4` block (the flat
    exhaustive scan, 2M x 768, 4096 queries per batch, K 10) with the
    reference's linear_scan timed on a query sample on all host threads.
  * N > 1 (one process per GPU; started here under torch.distributed.run when
    WORLD_SIZE is unset): config 3 (10M x 128, nlist 16384, 100k queries,
    nprobe 64, K 100) list-sharded over the N GPUs, strong scaling (the 100k
    queries split over the ranks): rank r ranks its own queries, NCCL
    all-gathers rotated queries and probes, scans its lists in two phases with
    an all-reduce(MIN) of the per-query radius, all-to-all of top-K keys to the
    queries' owners (paper_2411_17229_b200/dist.py). Rank 0 also reports the
    same workload unsharded on its own GPU (`n1_same_workload`).

value  = queries / device time, inputs resident in HBM, CUDA events on the
         launching stream, L2 flushed (512 MB write) between steps, max over ranks.
e2e    = same metric through the C ABI with pinned host buffers: H2D of raw
         queries + search + D2H of ids/dists/counts, host wall clock.
roofline = the DCO scan (seed -> merges) against HBM:
         achieved = B_read / scan time (kernel-counted slice bytes + metadata),
         scan_hbm_frac = ncu DRAM bytes of those kernels (newest committed
         profiles/ncu_step_summary_r*_<config>.json) / scan time / measured HBM
         peak; B_union and the over-fetch B_read / B_union.
cpu_baseline = the UNMODIFIED reference (oracle/_ref/libdade_ref.so) on this
         box's host, 1 thread (the paper's contract), a bounded query sample.
--impl reference = that reference with all host threads, each step a bounded
         query sample, same config / metric; it loads the artifacts with the
         reference's own loaders and never maps libdade_gpu.so.
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
GT_SAMPLE = 2000  # queries with exact ground truth (recall sample) per workload


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---- workloads (shared by both arms; no GPU library imported here) ---------------
def _configs_module():
    """paper_2411_17229_b200/configs.py loaded by path: importing the package
    would map libdade_gpu.so into the reference arm's process."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("_dade_configs", ROOT / "paper_2411_17229_b200" / "configs.py")
    mod = importlib.util.module_from_spec(spec)
    sys.modules["_dade_configs"] = mod  # (dataclasses resolve the module by name)
    spec.loader.exec_module(mod)
    return mod


CFGS = _configs_module()


def config_dict(cfg, n_gpus: int, queries_per_step: int) -> dict:
    """The `config` object of both arms' JSON lines (identical by construction)."""
    parallelism = "single GPU" if n_gpus == 1 else (
        f"list-sharded x{n_gpus} (strong scaling: {queries_per_step} queries over {n_gpus} ranks; NCCL all-gather of "
        f"rotated queries + probes, all-reduce MIN of the radius, all-to-all of top-K keys)")
    return {"workload": cfg.describe(), "queries_per_step": queries_per_step, "n_gpus": n_gpus,
            "parallelism": parallelism,
            "artifacts": "GPU-built with the reference's arithmetic (fit_pca covariance, calibrate, IvfIndex::build "
                         "k-means++/Lloyd, compute_ground_truth), saved as DADE / .cal / DIVF / fvecs / ivecs files "
                         "that both arms load",
            "l2": "flushed between timed steps (512 MB write)",
            "timed": "rotate + coarse + group + DCO scan + merge on device-resident raw queries"}


def ensure_artifacts_subprocess(cfg, nq=None) -> Path:
    """Build the artifacts in a child process (the reference arm must not load
    the GPU library itself)."""
    out = CFGS.artifact_dir(cfg, nq=nq)
    if (out / "DONE").exists():
        return out
    cmd = [sys.executable, "-m", "paper_2411_17229_b200.workloads", "--config", cfg.name, "--gt-queries",
           str(GT_SAMPLE)] + (["--nq", str(nq)] if nq else [])
    r = subprocess.run(cmd, cwd=ROOT, stdout=subprocess.PIPE, stderr=sys.stderr, text=True)
    if r.returncode != 0 or not (out / "DONE").exists():
        raise RuntimeError(f"artifact build failed ({r.returncode}): {' '.join(cmd)}")
    return out


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


def measured_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def measured_bf16():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["bf16_tflops"]), "MEASURED_PEAKS.json bf16_tflops"
    return 2250.0, "nominal dense bf16 (B200_PROFILING.md fallback)"


SCAN_KERNELS = ("seed_", "dco_filter", "advance_survivors", "merge_slots", "row_norms", "union_census")


def ncu_scan_traffic(cfg_name: str):
    """DRAM bytes of one search's DCO scan kernels (seed -> last slot merge) from
    the newest committed ncu --set full summary for this config, plus that
    summary's per-kernel bytes; None when no summary exists."""
    cands = sorted((ROOT / "profiles").glob(f"ncu_step_summary_r*_{cfg_name}.json"))
    if not cands:
        return None
    p = cands[-1]
    d = json.loads(p.read_text())
    ls = d["launches"]
    # one search: from its seed launch to the end of the list
    starts = [i for i, x in enumerate(ls) if x["kernel"].startswith(("seed_order", "seed_persist", "seed_radius"))]
    if starts:  # the seed order kernel (when present) directly precedes the seed
        while starts[-1] > 0 and ls[starts[-1] - 1]["kernel"].startswith("seed_order"):
            starts[-1] -= 1
    if starts:
        ls = ls[starts[-1]:]
    ls = [x for x in ls if x["kernel"].startswith(SCAN_KERNELS)]
    per = {}
    for x in ls:
        per[x["kernel"]] = per.get(x["kernel"], 0.0) + (x["dram_read_MB"] + x["dram_write_MB"]) * 1e6
    return {"bytes": sum(per.values()), "per_kernel_bytes": per, "source": f"profiles/{p.name}",
            "capture": d.get("source", "")}


# ---- reference arm (CPU) ---------------------------------------------------------------
def reference_load(art: Path, cfg):
    """The reference library on the saved artifacts, through its own loaders."""
    from oracle import RefLib, read_fvecs, read_ivecs
    ref = RefLib()
    t = ref.load_transform(art / "t.dade")
    cal = ref.cal_load(art / "c.cal")
    strat = ref.strategy_dade(t, cal, cfg.delta_d)
    ivf = ref.ivf_load(art / "index.ivf")
    q_rot = t.apply(read_fvecs(art / "queries.fvecs"))  # apply_transform, as measure()'s caller does
    gt = read_ivecs(art / "gt.ivecs").astype(np.uint32)
    return ref, ivf, strat, q_rot, gt, (t, cal)


def reference_sample(ivf, strat, q_rot, cfg, threads, target_s, start=0, limit=None):
    """Run the reference on a query sample sized to ~target_s seconds
    (steady_clock around the IvfIndex::search loop, as measure() does)."""
    n = q_rot.shape[0] if limit is None else min(limit, q_rot.shape[0])
    probe = max(threads * 2, 16)
    idx0 = (start + np.arange(probe)) % n
    _, _, _, _, sec = ivf.search(strat, q_rot[idx0], cfg.k, cfg.nprobe, threads=threads)
    per_q = max(sec / probe, 1e-6)
    m = int(min(n, max(probe, target_s / per_q)))
    idx = (start + np.arange(m)) % n
    ids, d, cnt, st, sec = ivf.search(strat, q_rot[idx], cfg.k, cfg.nprobe, threads=threads)
    return idx, ids, cnt, st, sec


def recall(ids, counts, gt):
    from oracle import Oracle
    return Oracle().recall(ids, counts, gt)


def _cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference_arm(args, cfg, n_gpus, nq_step):
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    art = ensure_artifacts_subprocess(cfg)
    ref, ivf, strat, q_rot, gt, _keep = reference_load(art, cfg)
    threads = os.cpu_count() or 1
    qps, secs, recs, sample = [], [], [], 0
    start = 0
    for step in range(args.warmup + args.steps):
        idx, ids, cnt, st, sec = reference_sample(ivf, strat, q_rot, cfg, threads, args.ref_step_s, start,
                                                  limit=gt.shape[0])
        start = int((start + len(idx)) % gt.shape[0])
        if step >= args.warmup:
            qps.append(len(idx) / sec)
            secs.append(sec)
            recs.append(recall(ids, cnt, gt[idx]))
            sample = len(idx)
    value = float(np.mean(qps))
    loaded = sorted({Path(l.split()[-1]).name for l in Path("/proc/self/maps").read_text().splitlines()
                     if l.endswith(".so") and ("dade" in l or "oracle" in l)})
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(secs)), "higher_is_better": True,
        "scaling": "strong" if n_gpus > 1 else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded Gaussian mixtures of the BASELINE config shapes)",
        "config": config_dict(cfg, n_gpus, nq_step),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{sample} queries per step (strided subsets per host thread), unmodified "
                                   f"IvfIndex::search + DadeStrategy (oracle/_ref/libdade_ref.so), artifacts loaded "
                                   f"with OrthoTransform::load / CalibrationTable::load / IvfIndex::load, queries "
                                   f"rotated by apply_transform outside the timed loop as in measure()"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "recall_at_k": float(np.mean(recs)),
        "host_cpu": _cpu_model(),
        "libraries_mapped": loaded,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---- ours: helpers -------------------------------------------------------------------
def load_ours(art: Path, cfg, dev, device):
    """Our arm on the same files: DIVF lists, DADE transform, .cal table, raw queries."""
    import torch

    import paper_2411_17229_b200 as gp
    from paper_2411_17229_b200.io import read_cal, read_divf, read_fvecs, read_ivecs, read_transform
    t = read_transform(art / "t.dade")
    cal = read_cal(art / "c.cal")
    dv = read_divf(art / "index.ivf")
    idx = gp.IvfIndex.from_divf(dev, dv)
    q_raw = torch.from_numpy(read_fvecs(art / "queries.fvecs")).to(device)
    gt = read_ivecs(art / "gt.ivecs").astype(np.uint32)
    return t, cal, dv, idx, q_raw, gt


def time_device(step, stream, flush, steps, warmup):
    import torch
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    evs = []
    for _ in range(steps):
        flush.zero_()  # L2 flush between timed steps (outside the events)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def profile_scan(dev, idx_search, reps=3):
    """Profiled searches (not timed above): scan / filter / seed device times,
    B_read, B_union, DcoStats."""
    import torch

    import paper_2411_17229_b200 as gp
    dev.set_profiling(True)
    rows = []
    try:
        for _ in range(reps):
            torch.cuda.synchronize()
            st = gp.DcoStats()
            idx_search(st)
            scan_ms, b_read, total_ms = dev.last_scan_profile()
            f_ms, n_f = dev.last_filter_profile()
            s_ms, s_pd = dev.last_seed_profile()
            b_union, u_rows = dev.last_union_profile()
            rows.append(dict(scan_ms=scan_ms, b_read=b_read, filter_ms=f_ms, n_filter=n_f, seed_ms=s_ms,
                             seed_pair_dims=s_pd, b_union=b_union, union_rows=u_rows, stats=st))
    finally:
        dev.set_profiling(False)
    med = {k: float(np.median([r[k] for r in rows])) for k in rows[0] if k != "stats"}
    med["stats"] = rows[-1]["stats"]
    return med


def roofline_block(cfg, prof, d0, dim):
    peak, peak_src = measured_hbm()
    bf16, bf16_src = measured_bf16()
    scan_s = prof["scan_ms"] / 1e3
    st = prof["stats"]
    ncu = ncu_scan_traffic(cfg.name)
    achieved = prof["b_read"] / scan_s / 1e9
    roof = {
        "bound": "hbm", "unit": "GB/s", "achieved": achieved, "peak": peak, "frac": achieved / peak,
        "kernel": "the DCO scan: seed_persist / seed_radius_list, dco_filter_umma (tcgen05), "
                  "advance_survivors_pipe, merge_slots (one search, seed through the last merge)",
        "scan_ms_per_step": prof["scan_ms"],
        "achieved_definition": "B_read / scan time: B_read = kernel-counted bytes of base-vector slices the "
                               "kernels loaded (filter tiles 4*d0*rows per work item, seed rows once per "
                               "16-query group, survivor row chunks from dim 0) + list/worklist metadata "
                               "(SURVEY.md §8d)",
        "b_read": prof["b_read"], "b_union": prof["b_union"],
        "overfetch_b_read_over_b_union": prof["b_read"] / prof["b_union"] if prof["b_union"] else None,
        "b_union_definition": "4 x sum over base rows of the most dims any (query, row) DCO of this search used "
                              "(our decisions; d0 for every row of a probed list, dim for seeded rows)",
        "reference_work_bytes": 4.0 * st.dims_accumulated,
        "effective_gbs": 4.0 * st.dims_accumulated / scan_s / 1e9,
        "peak_source": peak_src,
        "traffic": ncu["bytes"] if ncu else None,
        "scan_hbm_frac": (ncu["bytes"] / scan_s / 1e9 / peak) if ncu else None,
        "traffic_source": (f"{ncu['source']}: dram__bytes_read.sum + dram__bytes_write.sum of the scan kernels of "
                           f"one search ({ncu['capture']})") if ncu else "no committed ncu summary for this config",
        "traffic_per_kernel": ncu["per_kernel_bytes"] if ncu else None,
    }
    if prof["filter_ms"] > 0:
        pairs = st.total_dco
        tf = 2.0 * pairs * d0 / (prof["filter_ms"] / 1e3) / 1e12
        roof["tensor_view"] = {"kernel": "dco_filter_umma_kernel", "ms_per_step": prof["filter_ms"],
                               "launches_per_step": prof["n_filter"], "tf32_tflops": tf,
                               "peak_tflops": 0.5 * bf16, "frac": tf / (0.5 * bf16),
                               "definition": "2 * DCO pairs * d0 first-slice flops / filter time; peak = "
                                             f"{bf16_src} / 2 (TF32 dense)"}
    if prof["seed_ms"] > 0:
        seed_bytes = (sum(v for kname, v in ncu["per_kernel_bytes"].items() if kname.startswith("seed_persist"))
                      or None) if ncu else None  # (template instances: seed_persist_kernel<rows>)
        roof["seed_view"] = {"kernel": "seed_persist_kernel", "ms_per_step": prof["seed_ms"],
                             "pair_dims_per_step": prof["seed_pair_dims"],
                             "ncu_dram_bytes": seed_bytes,
                             "hbm_frac": (seed_bytes / (prof["seed_ms"] / 1e3) / 1e9 / peak) if seed_bytes else None}
    return roof


def e2e_block(dev, cfg, q_raw, nq, k, steps, warmup, flush, gt):
    """dade_gpu_ivf_search_batches over pinned host buffers (K steps in one
    pipelined call) and a synchronous single call per step."""
    import torch

    from paper_2411_17229_b200 import _capi
    dev.set_stream(None)
    qh = torch.empty((nq, cfg.dim), dtype=torch.float32, pin_memory=True)
    qh.copy_(q_raw.cpu())
    ih = torch.empty((nq, k), dtype=torch.int32, pin_memory=True)
    dh = torch.empty((nq, k), dtype=torch.float32, pin_memory=True)
    ch = torch.empty((nq,), dtype=torch.int32, pin_memory=True)

    def single():
        _capi.check(_capi.lib.dade_gpu_ivf_search(dev.h, _capi.ptr(qh), nq, k, cfg.nprobe, _capi.QUERIES_RAW,
                                                  _capi.ptr(ih), _capi.ptr(dh), _capi.ptr(ch), None))
    qd_warm = torch.empty_like(qh, device="cuda")
    t_w = time.perf_counter()
    while time.perf_counter() - t_w < 0.5:  # bring the PCIe link to its loaded state (untimed)
        qd_warm.copy_(qh, non_blocking=True)
        torch.cuda.synchronize()
    for _ in range(warmup):
        single()
    ts = []
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        single()
        ts.append(time.perf_counter() - t0)
    single_rec = recall(ih.numpy().astype(np.uint32)[:gt.shape[0]], ch.numpy().astype(np.uint32)[:gt.shape[0]], gt)
    outs = [(ih, dh, ch)] + [tuple(torch.empty_like(x, pin_memory=True) for x in (ih, dh, ch))]

    def pipe(n):
        A = ctypes.c_void_p * n
        _capi.check(_capi.lib.dade_gpu_ivf_search_batches(
            dev.h, n, A(*[_capi.ptr(qh)] * n), nq, k, cfg.nprobe, _capi.QUERIES_RAW,
            A(*[_capi.ptr(outs[b % 2][0]) for b in range(n)]), A(*[_capi.ptr(outs[b % 2][1]) for b in range(n)]),
            A(*[_capi.ptr(outs[b % 2][2]) for b in range(n)]), None))
    pipe(max(warmup, 2))
    flush.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pipe(steps)
    t_pipe = time.perf_counter() - t0
    last = outs[(steps - 1) % 2]
    pipe_rec = recall(last[0].numpy().astype(np.uint32)[:gt.shape[0]], last[2].numpy().astype(np.uint32)[:gt.shape[0]],
                      gt)
    torch.cuda.synchronize()
    t_h = time.perf_counter()
    for _ in range(5):
        qd_warm.copy_(qh, non_blocking=True)
    torch.cuda.synchronize()
    h2d_gbs = 5 * qh.numel() * 4 / (time.perf_counter() - t_h) / 1e9
    return {"value": nq * steps / t_pipe, "unit": UNIT, "h2d_bytes_per_step": nq * cfg.dim * 4,
            "d2h_bytes_per_step": nq * k * 8 + nq * 4, "ms_per_step": 1e3 * t_pipe / steps,
            "recall_at_k": pipe_rec,
            "api": "dade_gpu_ivf_search_batches: K steps as one pipelined call over pinned host buffers (raw "
                   "queries H2D, rotation, search, ids/dists/counts D2H every step; host wall clock around the "
                   "call, which returns after the last D2H)",
            "l2": "not flushed between the pipelined steps",
            "single_call": {"value": nq / float(np.mean(ts)), "ms_per_call": 1e3 * float(np.mean(ts)),
                            "recall_at_k": single_rec,
                            "api": "dade_gpu_ivf_search per step, synchronous, L2 flushed between calls"},
            "pcie_h2d_gbs_after": round(h2d_gbs, 1), "pcie_warmup_s": 0.5}


def cpu_baseline_block(art, cfg, ids_np, cnt_np, gt, target_s):
    try:
        ref, ivf, strat, q_rot, _, _keep = reference_load(art, cfg)
        sidx, rids, rcnt, rst, sec = reference_sample(ivf, strat, q_rot, cfg, 1, target_s, limit=gt.shape[0])
        return {"value": len(sidx) / sec, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": f"first {len(sidx)} queries, 1 thread, IvfIndex::search + DadeStrategy "
                          f"(oracle/_ref/libdade_ref.so), rotation excluded as in measure()",
                "recall_at_k_sample": recall(rids, rcnt, gt[sidx]),
                "ours_recall_at_k_same_sample": recall(ids_np[sidx], cnt_np[sidx], gt[sidx]),
                "dim_fraction": float(rst[1]) / (float(rst[0]) * cfg.dim)}
    except Exception as e:  # reported, never fatal to the GPU line
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "reference", "sample": f"failed: {e}"}


def single_gpu_workload(args, cfg, dev, device, stream, flush, with_e2e=True, with_cpu=True):
    """One workload on one GPU: device-timed value, profiled roofline, e2e, CPU baseline."""
    import torch

    import paper_2411_17229_b200 as gp
    from paper_2411_17229_b200 import _capi
    from paper_2411_17229_b200.workloads import artifact_dir, ensure_artifacts
    art = artifact_dir(cfg)
    if not (art / "DONE").exists():
        art = ensure_artifacts(cfg, gt_queries=GT_SAMPLE, log=log)
    t, cal, dv, idx, q_dev, gt = load_ours(art, cfg, dev, device)
    dco = gp.DadeStrategy(t, cal, cfg.delta_d, dev=dev)
    dev.apply(dco)
    dev.set_stream(stream.cuda_stream)
    nq, k = q_dev.shape[0], cfg.k
    out_ids = torch.empty((nq, k), dtype=torch.int32, device=device)
    out_d = torch.empty((nq, k), dtype=torch.float32, device=device)
    out_c = torch.empty((nq,), dtype=torch.int32, device=device)
    flags = _capi.QUERIES_RAW | _capi.DEVICE_PTRS

    def step(st=None):
        _capi.check(_capi.lib.dade_gpu_ivf_search(dev.h, _capi.ptr(q_dev), nq, k, cfg.nprobe, flags,
                                                  _capi.ptr(out_ids), _capi.ptr(out_d), _capi.ptr(out_c),
                                                  ctypes.byref(st) if st is not None else None))
    clocks = ClockSampler(device.index or 0, Path(tempfile.gettempdir()) / f"dade_clocks_{cfg.name}.csv")
    time.sleep(0.3)
    l0 = dev.launches
    t_region0 = time.time()
    ms = time_device(step, stream, flush, args.steps, args.warmup)
    t_region1 = time.time()
    clk = clocks.stop((t_region0, t_region1))
    launches = (dev.launches - l0) // max(args.steps + args.warmup, 1)
    mean_ms = float(np.mean(ms))
    ids_np = out_ids.cpu().numpy().astype(np.uint32)
    cnt_np = out_c.cpu().numpy().astype(np.uint32)
    rec = recall(ids_np[:gt.shape[0]], cnt_np[:gt.shape[0]], gt)

    def prof_search(st):
        s = _capi.Stats()
        step(s)
        st._add(s)
    prof = profile_scan(dev, prof_search)
    roof = roofline_block(cfg, prof, cfg.delta_d, cfg.dim)
    out = {"value": nq / (mean_ms / 1e3), "ms_per_step": mean_ms, "recall_at_k": rec,
           "recall_sample": f"first {gt.shape[0]} queries (exact GPU ground truth, compute_ground_truth semantics)",
           "dim_fraction": prof["stats"].dim_fraction(cfg.dim), "gpu_launches": int(launches), "clocks": clk,
           "roofline": roof, "queries_per_step": nq}
    if with_e2e:
        out["e2e"] = e2e_block(dev, cfg, q_dev, nq, k, args.steps, args.warmup, flush, gt)
    if with_cpu:
        out["cpu_baseline"] = cpu_baseline_block(art, cfg, ids_np, cnt_np, gt, args.cpu_baseline_s)
    dev.set_stream(stream.cuda_stream)
    return out


FLAT_PARTS, FLAT_PART_ITERS = 512, 10


def flat_workload(args, cfg, dev, device, stream, flush):
    """Config 4, the flat exhaustive DADE scan (dade_gpu_flat_search): device time
    per 4096-query batch (raw queries resident, L2 flushed, CUDA events), recall,
    and the reference's linear_scan (knn.cpp:31-41) on a bounded query sample
    with all host threads, on the same rotated base, transform and calibration."""
    import torch

    import paper_2411_17229_b200 as gp
    from oracle import RefLib, read_fvecs as ref_read_fvecs
    from paper_2411_17229_b200 import _capi
    from paper_2411_17229_b200.io import read_cal, read_fvecs, read_ivecs, read_transform
    from paper_2411_17229_b200.workloads import artifact_dir, ensure_artifacts
    art = artifact_dir(cfg)
    if not (art / "DONE").exists():
        art = ensure_artifacts(cfg, gt_queries=GT_SAMPLE, log=log)
    base = read_fvecs(art / "base.fvecs")
    idx = gp.FlatIndex(dev, base)
    dco = gp.DadeStrategy(read_transform(art / "t.dade"), read_cal(art / "c.cal"), cfg.delta_d, dev=dev)
    dev.apply(dco)
    dev.set_stream(stream.cuda_stream)
    q_raw = read_fvecs(art / "queries.fvecs")
    q_dev = torch.from_numpy(q_raw).to(device)
    gt = read_ivecs(art / "gt.ivecs").astype(np.uint32)
    nq, k = q_dev.shape[0], cfg.k
    out_ids = torch.empty((nq, k), dtype=torch.int32, device=device)
    out_d = torch.empty((nq, k), dtype=torch.float32, device=device)
    out_c = torch.empty((nq,), dtype=torch.int32, device=device)

    def step():
        _capi.check(_capi.lib.dade_gpu_flat_search(dev.h, _capi.ptr(q_dev), nq, k,
                                                   _capi.QUERIES_RAW | _capi.DEVICE_PTRS, _capi.ptr(out_ids),
                                                   _capi.ptr(out_d), _capi.ptr(out_c), None))
    ms = time_device(step, stream, flush, min(args.steps, 5), min(args.warmup, 3))
    row_ms = float(np.mean(ms))
    row_rec = recall(out_ids.cpu().numpy().astype(np.uint32)[:gt.shape[0]],
                     out_c.cpu().numpy().astype(np.uint32)[:gt.shape[0]], gt)
    # data-ordered scan: the base in k-means cells (dade_gpu_flat_partition), every
    # cell probed, each query's nearest first; the same dade_gpu_flat_search call
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    idx.partition(FLAT_PARTS, FLAT_PART_ITERS, 1)
    torch.cuda.synchronize()
    part_s = time.perf_counter() - t0
    dev.apply(dco)
    ms = time_device(step, stream, flush, min(args.steps, 5), min(args.warmup, 3))
    mean_ms = float(np.mean(ms))
    ids_np = out_ids.cpu().numpy().astype(np.uint32)
    cnt_np = out_c.cpu().numpy().astype(np.uint32)
    out = {"workload": cfg.describe(), "value": nq / (mean_ms / 1e3), "unit": UNIT, "ms_per_step": mean_ms,
           "recall_at_k": recall(ids_np[:gt.shape[0]], cnt_np[:gt.shape[0]], gt),
           "visit_order": f"data-ordered: {FLAT_PARTS} k-means cells of the base (dade_gpu_flat_partition, "
                          f"{FLAT_PART_ITERS} Lloyd iterations, built once in {part_s:.2f} s outside the timed "
                          "region), every cell probed, each query's nearest first",
           "row_order": {"value": nq / (row_ms / 1e3), "ms_per_step": row_ms, "recall_at_k": row_rec,
                         "visit_order": "base rows in id order (linear_scan's order), 4x-growing passes"},
           "timing": "CUDA events, raw queries resident, L2 flushed, mean of the timed batches"}
    try:
        ref = RefLib()
        t = ref.load_transform(art / "t.dade")
        cal = ref.cal_load(art / "c.cal")
        strat = ref.strategy_dade(t, cal, cfg.delta_d)
        threads = os.cpu_count() or 1
        m = min(gt.shape[0], max(2 * threads, 32))
        q_rot = t.apply(ref_read_fvecs(art / "queries.fvecs")[:m])
        rids, _, rcnt, _, sec = ref.linear_scan(base, strat, q_rot, k, threads=threads)
        out["reference"] = {"value": m / sec, "unit": UNIT, "cores": threads, "kind": "reference",
                            "sample": f"first {m} queries, linear_scan + DadeStrategy (oracle/_ref/libdade_ref.so) "
                                      f"over the same rotated base, {threads} host threads",
                            "recall_at_k_sample": recall(rids, rcnt, gt[:m]),
                            "ours_recall_at_k_same_sample": recall(ids_np[:m], cnt_np[:m], gt[:m])}
    except Exception as e:  # reported, never fatal to the GPU line
        out["reference"] = {"value": None, "sample": f"failed: {e}"}
    return out


# ---- ours ------------------------------------------------------------------------------
def run_ours_single(args, cfg):
    import torch

    import paper_2411_17229_b200 as gp
    CONFIGS = CFGS.CONFIGS
    torch.cuda.set_device(0)
    device = torch.device("cuda", 0)
    dev = gp.Device(0)
    stream = torch.cuda.Stream(device)
    torch.cuda.set_stream(stream)  # torch ops, CUDA events and the C ABI share one stream
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=device)
    main = single_gpu_workload(args, cfg, dev, device, stream, flush)
    line = {
        "metric": METRIC, "value": main["value"], "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": main["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded Gaussian mixtures of the BASELINE config shapes)",
        "config": config_dict(cfg, 1, main["queries_per_step"]),
        "recall_at_k": main["recall_at_k"], "recall_sample": main["recall_sample"],
        "dim_fraction": main["dim_fraction"], "gpu_launches": main["gpu_launches"], "clocks": main["clocks"],
        "roofline": main["roofline"], "cpu_baseline": main["cpu_baseline"], "e2e": main["e2e"],
    }
    if not args.no_config2 and cfg.name == "config1":
        try:
            del main
            torch.cuda.empty_cache()
            c2 = single_gpu_workload(args, CONFIGS["config2"], gp.Device(0), device, stream, flush)
            line["config2"] = {"workload": CONFIGS["config2"].describe(), "value": c2["value"],
                               "ms_per_step": c2["ms_per_step"], "e2e": c2["e2e"], "recall_at_k": c2["recall_at_k"],
                               "dim_fraction": c2["dim_fraction"], "roofline": c2["roofline"],
                               "cpu_baseline": c2["cpu_baseline"], "gpu_launches": c2["gpu_launches"],
                               "clocks": c2["clocks"]}
        except Exception as e:  # reported, never fatal to the headline line
            line["config2"] = {"error": repr(e)}
    if not args.no_config4 and cfg.name == "config1":
        try:
            torch.cuda.empty_cache()
            line["config4"] = flat_workload(args, CONFIGS["config4"], gp.Device(0), device, stream, flush)
        except Exception as e:  # reported, never fatal to the headline line
            line["config4"] = {"error": repr(e)}
    print(json.dumps(line), flush=True)
    return 0


def run_ours_multi(args, cfg):
    """N ranks (torch.distributed, NCCL): the list-sharded search, strong scaling."""
    import torch
    import torch.distributed as dist

    import paper_2411_17229_b200 as gp
    from paper_2411_17229_b200 import _capi
    from paper_2411_17229_b200 import dist as gdist
    from paper_2411_17229_b200.workloads import artifact_dir, ensure_artifacts
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=device)
    if rank == 0:
        ensure_artifacts(cfg, gt_queries=GT_SAMPLE, log=log)
    dist.barrier()
    art = artifact_dir(cfg)
    dev = gp.Device(local)
    stream = torch.cuda.Stream(device)
    torch.cuda.set_stream(stream)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=device)
    t, cal, dv, idx, q_all, gt = load_ours(art, cfg, dev, device)
    owner = gdist.plan_list_shards(dv.offsets, world, cfg.dim)
    dco = gp.DadeStrategy(t, cal, cfg.delta_d, dev=dev)
    n1 = None
    if rank == 0:  # the same workload unsharded on one GPU, for the scaling ratio
        dev.apply(dco)
        dev.set_stream(stream.cuda_stream)
        nq, k = q_all.shape[0], cfg.k
        oi = torch.empty((nq, k), dtype=torch.int32, device=device)
        od = torch.empty((nq, k), dtype=torch.float32, device=device)
        oc = torch.empty((nq,), dtype=torch.int32, device=device)

        def step1():
            _capi.check(_capi.lib.dade_gpu_ivf_search(dev.h, _capi.ptr(q_all), nq, k, cfg.nprobe,
                                                      _capi.QUERIES_RAW | _capi.DEVICE_PTRS, _capi.ptr(oi),
                                                      _capi.ptr(od), _capi.ptr(oc), None))
        ms1 = time_device(step1, stream, flush, max(3, args.steps // 4), args.warmup)
        n1 = {"value": nq / (float(np.mean(ms1)) / 1e3), "ms_per_step": float(np.mean(ms1)),
              "note": "rank 0 alone, unsharded index, same queries (the N = 1 point of this workload)"}
    dist.barrier()
    idx.shard((owner == rank).astype(np.uint8))
    dev.apply(dco)
    dev.set_stream(stream.cuda_stream)
    if q_all.shape[0] % world:
        raise SystemExit(f"{q_all.shape[0]} queries do not split evenly over {world} ranks")
    nq_loc = q_all.shape[0] // world  # strong scaling: the job's queries split over the ranks
    q_loc = q_all[rank * nq_loc:(rank + 1) * nq_loc].contiguous()

    def step():
        return gdist.sharded_ivf_search(dev, None, q_loc, nq_loc, cfg.k, cfg.nprobe, raw=True)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    clocks = ClockSampler(local, Path(tempfile.gettempdir()) / f"dade_clocks_r{rank}.csv")
    time.sleep(0.3)
    l0 = dev.launches
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.time()
    evs = []
    for _ in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = step()
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    t1 = time.time()
    dist.barrier()
    clk = clocks.stop((t0, t1))
    mean_ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    tt = torch.tensor([mean_ms], device=device)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    mean_ms = float(tt.item())
    launches = (dev.launches - l0) // max(args.steps, 1)
    ids0 = res[0].cpu().numpy().astype(np.uint32)
    cnt0 = res[2].cpu().numpy().astype(np.uint32)
    # e2e: each rank's raw query slice from pinned host memory, results back to pinned memory
    qh = torch.empty((nq_loc, cfg.dim), dtype=torch.float32, pin_memory=True)
    qh.copy_(q_loc.cpu())
    ihm = torch.empty((nq_loc, cfg.k), dtype=torch.int32, pin_memory=True)
    dhm = torch.empty((nq_loc, cfg.k), dtype=torch.float32, pin_memory=True)
    chm = torch.empty((nq_loc,), dtype=torch.int32, pin_memory=True)

    def e2e_step():
        qd = qh.to(device, non_blocking=True)
        i_, d_, c_ = gdist.sharded_ivf_search(dev, None, qd, nq_loc, cfg.k, cfg.nprobe, raw=True)
        ihm.copy_(i_, non_blocking=True)
        dhm.copy_(d_, non_blocking=True)
        chm.copy_(c_, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    for _ in range(args.warmup):
        e2e_step()
    ts = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        dist.barrier()
        ta = time.perf_counter()
        e2e_step()
        ts.append(time.perf_counter() - ta)
    tt = torch.tensor([float(np.mean(ts))], device=device)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e_s = float(tt.item())
    nq_total = q_all.shape[0]
    if rank == 0:
        m = min(gt.shape[0], nq_loc)
        line = {
            "metric": METRIC, "value": nq_total / (mean_ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Gaussian mixtures of the BASELINE config shapes)",
            "config": config_dict(cfg, world, nq_total),
            "recall_at_k": recall(ids0[:m], cnt0[:m], gt[:m]), "gpu_launches": int(launches), "clocks": clk,
            "n1_same_workload": n1,
            "e2e": {"value": nq_total / e2e_s, "unit": UNIT, "h2d_bytes_per_step": nq_total * cfg.dim * 4,
                    "d2h_bytes_per_step": nq_total * (cfg.k * 8 + 4), "ms_per_step": 1e3 * e2e_s,
                    "api": "dist.sharded_ivf_search per step on every rank: H2D of the rank's raw query slice, "
                           "search, D2H of its ids/dists/counts; host wall clock, max over ranks"},
            "roofline": None, "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


def relaunch_distributed(args) -> int:
    """--gpus N without a torch.distributed launcher: start N ranks here."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator lines (nranks) on stderr
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="default: config1 (N = 1), config3 (N > 1)")
    ap.add_argument("--cpu-baseline-s", type=float, default=12.0)
    ap.add_argument("--ref-step-s", type=float, default=6.0)
    ap.add_argument("--no-config2", action="store_true")
    ap.add_argument("--no-config4", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    n_gpus = max(args.gpus, world)
    cfg = CFGS.CONFIGS[args.config or ("config1" if n_gpus == 1 else "config3")]
    if args.impl == "reference":
        return run_reference_arm(args, cfg, n_gpus, cfg.nq)
    if n_gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args)
    if world > 1:
        return run_ours_multi(args, cfg)
    return run_ours_single(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
