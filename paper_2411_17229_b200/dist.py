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


def flat_search_keys(dev, d_queries, nq: int, k: int, out_keys, raw: bool = False, stats=None) -> None:
    """linear_scan over this device's rows (FlatIndex, ids offset by its id_base) -> packed keys."""
    flags = _capi.DEVICE_PTRS | (_capi.QUERIES_RAW if raw else 0)
    st = _capi.Stats()
    _capi.check(_capi.lib.dade_gpu_flat_search_keys(dev.h, _capi.ptr(d_queries), nq, k, flags, _capi.ptr(out_keys),
                                                    C.byref(st) if stats is not None else None))
    if stats is not None:
        stats._add(st)


def sharded_flat_search(dev, group, d_queries, nq: int, k: int, raw: bool = False):
    """Row-sharded flat exhaustive scan (config 4): rank r holds the contiguous
    rows plan_row_shards(n, world)[r] as a FlatIndex with id_base = its first
    row and scans them for all nq queries (replicated) in two phases: the
    radius seed over its first rows, an NCCL all-reduce(MIN) of the per-query
    radius, the streaming passes; then an NCCL all-gather of the packed top-K
    keys ([world, nq, k], 8 B each) and the device merge. Every rank returns
    the global (ids, dists, counts)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    keys = torch.empty((nq, k), dtype=torch.int64, device=d_queries.device)
    radius = torch.empty((nq,), dtype=torch.int32, device=d_queries.device)
    flags = _capi.DEVICE_PTRS | (_capi.QUERIES_RAW if raw else 0)
    _capi.check(_capi.lib.dade_gpu_flat_search_keys_begin(dev.h, _capi.ptr(d_queries), nq, k, flags,
                                                          _capi.ptr(keys), _capi.ptr(radius)))
    dist.all_reduce(radius, op=dist.ReduceOp.MIN, group=group)  # every shard's seed bounds every query
    ivf_search_keys_end(dev, radius)
    gathered = torch.empty((world, nq, k), dtype=torch.int64, device=d_queries.device)
    dist.all_gather_into_tensor(gathered, keys, group=group)
    ids = torch.empty((nq, k), dtype=torch.int32, device=d_queries.device)
    dists = torch.empty((nq, k), dtype=torch.float32, device=d_queries.device)
    counts = torch.empty((nq,), dtype=torch.int32, device=d_queries.device)
    merge_keys_device(dev, gathered, nq, k, ids, dists, counts)
    return ids, dists, counts


def coarse_probes(dev, d_queries, nq: int, n_probe: int, q_rot_out, probes_out, raw: bool = False) -> None:
    """Rotation (raw) + coarse ranking of nq queries: rotated rows -> q_rot_out [nq, D],
    probe keys -> probes_out (int64 [nq, n_probe])."""
    flags = _capi.DEVICE_PTRS | (_capi.QUERIES_RAW if raw else 0)
    _capi.check(_capi.lib.dade_gpu_coarse_probes(dev.h, _capi.ptr(d_queries), nq, n_probe, flags,
                                                 _capi.ptr(q_rot_out), _capi.ptr(probes_out)))


def ivf_search_keys_begin(dev, d_queries, nq: int, k: int, n_probe: int, out_keys, radius,
                          raw: bool = False, probes=None) -> None:
    """Phase 1 of a shard's search: every query's nearest list if it is local
    (nearest LOCAL list without given probes); per-query radius -> radius (int32 [nq])."""
    flags = _capi.DEVICE_PTRS | (_capi.QUERIES_RAW if raw else 0)
    _capi.check(_capi.lib.dade_gpu_ivf_search_keys_begin(dev.h, _capi.ptr(d_queries), nq, k, n_probe, flags,
                                                         _capi.ptr(probes), _capi.ptr(out_keys), _capi.ptr(radius)))


def ivf_search_keys_end(dev, radius, stats=None) -> None:
    """Phase 2: the other local lists with the (min-reduced) radius; completes out_keys."""
    st = _capi.Stats()
    _capi.check(_capi.lib.dade_gpu_ivf_search_keys_end(dev.h, _capi.ptr(radius),
                                                       C.byref(st) if stats is not None else None))
    if stats is not None:
        stats._add(st)


def sharded_ivf_search(dev, group, d_queries, nq: int, k: int, n_probe: int, raw: bool = False):
    """List-sharded IVF-DADE search, query-owner scheme. Every rank owns nq
    queries (its slice of the job, d_queries on its GPU) and a shard of the
    lists (dade_gpu_set_ivf_shard):
      1. rotation + coarse ranking of its own slice (dade_gpu_coarse_probes);
      2. NCCL all-gather of the rotated slices and their probe keys;
      3. phase 1 over all queries: the shard owning a query's nearest list
         seeds it and scans that list; NCCL all-reduce(MIN) of the radius;
      4. phase 2: every shard scans its other probed lists with that radius;
      5. NCCL all-to-all of the packed top-K keys (each query's block goes to
         its owner) and the device merge of the world's blocks.
    Per-rank work stays that of one GPU on nq queries as the world grows
    (weak scaling). The context must run on torch's current stream
    (Device.set_stream), which NCCL uses too. Returns CUDA (ids, dists,
    counts) for this rank's own queries."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev_t = d_queries.device
    dim = d_queries.shape[1]
    q_rot = torch.empty((nq, dim), dtype=torch.float32, device=dev_t)
    probes = torch.empty((nq, n_probe), dtype=torch.int64, device=dev_t)
    coarse_probes(dev, d_queries, nq, n_probe, q_rot, probes, raw=raw)
    q_all = torch.empty((world * nq, dim), dtype=torch.float32, device=dev_t)
    p_all = torch.empty((world * nq, n_probe), dtype=torch.int64, device=dev_t)
    dist.all_gather_into_tensor(q_all, q_rot, group=group)
    dist.all_gather_into_tensor(p_all, probes, group=group)
    n_all = world * nq
    keys = torch.empty((n_all, k), dtype=torch.int64, device=dev_t)
    radius = torch.empty((n_all,), dtype=torch.int32, device=dev_t)
    ivf_search_keys_begin(dev, q_all, n_all, k, n_probe, keys, radius, probes=p_all)
    dist.all_reduce(radius, op=dist.ReduceOp.MIN, group=group)  # fp32 bits >= 0 order as int32
    ivf_search_keys_end(dev, radius)
    recv = torch.empty((world, nq, k), dtype=torch.int64, device=dev_t)
    dist.all_to_all_single(recv, keys, group=group)  # rows [j*nq, (j+1)*nq) -> rank j
    ids = torch.empty((nq, k), dtype=torch.int32, device=dev_t)
    dists = torch.empty((nq, k), dtype=torch.float32, device=dev_t)
    counts = torch.empty((nq,), dtype=torch.int32, device=dev_t)
    merge_keys_device(dev, recv, nq, k, ids, dists, counts)
    return ids, dists, counts


# ---- the same protocols through the C ABI's own NCCL layer (csrc/comm.cu) ---------------
class NcclComm:
    """dade_gpu_comm: an NCCL communicator owned by libdade_gpu on a Device, for
    dade_gpu_sharded_ivf_search / _flat_search (the C++ host's multi-GPU entry
    points). The unique id comes from rank 0 and is broadcast over `group`
    (torch.distributed, any backend), or passed in (`uid`, 128 bytes)."""

    def __init__(self, dev, world: int, rank: int, group=None, uid: bytes | None = None):
        if uid is None:
            buf = (C.c_uint8 * 128)()
            if rank == 0:
                _capi.check(_capi.lib.dade_gpu_nccl_unique_id(buf))
            if world > 1:
                import torch
                import torch.distributed as dist
                t = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
                dist.broadcast(t, 0, group=group)
                buf = (C.c_uint8 * 128)(*t.tolist())
            uid = bytes(buf)
        self.dev, self.world, self.rank = dev, world, rank
        h = C.c_void_p()
        idb = (C.c_uint8 * 128)(*uid)
        _capi.check(_capi.lib.dade_gpu_comm_create(dev.h, world, rank, idb, C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            _capi.lib.dade_gpu_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _run(self, fn, args, nq, k, queries, flags, stats):
        import torch
        dev_t = queries.device if getattr(queries, "is_cuda", False) else None
        if dev_t is not None:
            ids = torch.empty((nq, k), dtype=torch.int32, device=dev_t)
            dists = torch.empty((nq, k), dtype=torch.float32, device=dev_t)
            counts = torch.empty((nq,), dtype=torch.int32, device=dev_t)
            flags |= _capi.DEVICE_PTRS
        else:
            queries = np.ascontiguousarray(queries, np.float32)
            ids, dists, counts = (np.zeros((nq, k), np.uint32), np.zeros((nq, k), np.float32),
                                  np.zeros(nq, np.uint32))
        st = _capi.Stats()
        _capi.check(fn(self.h, _capi.ptr(queries), *args, flags, _capi.ptr(ids), _capi.ptr(dists),
                       _capi.ptr(counts), C.byref(st)))
        if stats is not None:
            stats._add(st)
        return ids, dists, counts

    def ivf_search(self, queries, nq: int, k: int, n_probe: int, raw: bool = False, stats=None):
        """dade_gpu_sharded_ivf_search: this rank's nq queries (host or CUDA)."""
        return self._run(_capi.lib.dade_gpu_sharded_ivf_search, (nq, k, n_probe), nq, k, queries,
                         _capi.QUERIES_RAW if raw else 0, stats)

    def flat_search(self, queries, nq: int, k: int, raw: bool = False, stats=None):
        """dade_gpu_sharded_flat_search: the same nq queries on every rank."""
        return self._run(_capi.lib.dade_gpu_sharded_flat_search, (nq, k), nq, k, queries,
                         _capi.QUERIES_RAW if raw else 0, stats)
