"""Multi-GPU sharding of the IVF / flat scan.

One process per GPU. The base set is sharded by IVF list (or by contiguous
row blocks for the flat scan); centroids, transform and strategy tables are
replicated; every rank scans only its own lists for all queries and produces
a packed per-query top-K ((float_bits(dist) << 32) | id, ascending, empty =
UINT64_MAX). The exchange step is one NCCL all-gather of those keys over
NVLink followed by the on-device G·K -> K merge (dade_gpu_merge_keys).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi

EMPTY_KEY = np.uint64(0xFFFFFFFFFFFFFFFF)


def plan_list_shards(offsets: np.ndarray, world: int, dim: int = 1) -> np.ndarray:
    """Assign every list to a rank, balancing sum(len * dim) bytes: lists in
    descending size order go to the least-loaded rank (ties -> lowest rank,
    then lowest list id), so the plan is deterministic on every rank.
    Returns owner[n_lists]."""
    sizes = np.diff(np.asarray(offsets, dtype=np.int64)) * dim
    order = np.lexsort((np.arange(sizes.size), -sizes))
    load = np.zeros(world, dtype=np.int64)
    owner = np.zeros(sizes.size, dtype=np.int32)
    for l in order:
        r = int(np.argmin(load))
        owner[l] = r
        load[r] += sizes[l]
    return owner


def plan_row_shards(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous even row shards [start, end) for the flat scan."""
    base, rem = divmod(n, world)
    out, s = [], 0
    for r in range(world):
        e = s + base + (1 if r < rem else 0)
        out.append((s, e))
        s = e
    return out


def merge_keys_device(dev, keys_all, nq: int, k: int, ids, dists, counts) -> None:
    """keys_all: CUDA int64 tensor [G, nq, k] -> ids/dists/counts (CUDA)."""
    G = keys_all.shape[0]
    _capi.check(_capi.lib.dade_gpu_merge_keys(dev.h, _capi.ptr(keys_all), G, nq, k, _capi.ptr(ids),
                                              _capi.ptr(dists), _capi.ptr(counts)))


def ivf_search_keys(dev, d_queries, nq: int, k: int, n_probe: int, out_keys, raw: bool = False,
                    stats=None) -> None:
    flags = _capi.DEVICE_PTRS | (_capi.QUERIES_RAW if raw else 0)
    st = _capi.Stats()
    _capi.check(_capi.lib.dade_gpu_ivf_search_keys(dev.h, _capi.ptr(d_queries), nq, k, n_probe, flags,
                                                   _capi.ptr(out_keys), C.byref(st) if stats is not None else None))
    if stats is not None:
        stats._add(st)


def sharded_ivf_search(dev, group, d_queries, nq: int, k: int, n_probe: int, raw: bool = False):
    """Local scan + NCCL all-gather + device merge. Returns CUDA (ids, dists, counts)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    keys = torch.empty((nq, k), dtype=torch.int64, device=d_queries.device)
    ivf_search_keys(dev, d_queries, nq, k, n_probe, keys, raw=raw)
    gathered = torch.empty((world, nq, k), dtype=torch.int64, device=d_queries.device)
    dist.all_gather_into_tensor(gathered, keys, group=group)
    ids = torch.empty((nq, k), dtype=torch.int32, device=d_queries.device)
    dists = torch.empty((nq, k), dtype=torch.float32, device=d_queries.device)
    counts = torch.empty((nq,), dtype=torch.int32, device=d_queries.device)
    merge_keys_device(dev, gathered, nq, k, ids, dists, counts)
    return ids, dists, counts
