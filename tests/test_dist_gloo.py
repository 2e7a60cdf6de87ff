"""CPU, world_size 2 over gloo: the multi-GPU scheme of SURVEY.md §8e —
lists sharded by plan_list_shards, every rank scans its own lists for all
queries (centroids replicated), per-rank top-K packed as (float_bits << 32 | id)
keys, all-gathered, merged to the global top-K — gives exactly the unsharded
FD answer, also when every rank drops its candidates beyond the per-query
radius all-reduced (MIN) after its nearest local list, and when the per-shard
keys go to each query's owner rank by an all-to-all. The per-rank scan here is
the oracle (checker); on GPUs it is libdade_gpu's coarse_probes, NCCL
all-gathers, ivf_search_keys_begin, an NCCL all-reduce of the radius,
ivf_search_keys_end, an NCCL all-to-all and dade_gpu_merge_keys."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

EMPTY = np.uint64(0xFFFFFFFFFFFFFFFF)


def pack(ids, dists, counts, k):
    keys = np.full((ids.shape[0], k), EMPTY, np.uint64)
    for q in range(ids.shape[0]):
        c = int(counts[q])
        keys[q, :c] = (dists[q, :c].view(np.uint32).astype(np.uint64) << np.uint64(32)) | ids[q, :c].astype(np.uint64)
    return keys


def merge(blocks, k):  # [G, nq, k] -> [nq, k] smallest keys
    allk = np.concatenate(list(blocks), axis=1)
    return np.sort(allk, axis=1)[:, :k]


def shard_index(offsets, ids, storage, dim, keep):
    """Drop the lists this rank does not own (they become empty)."""
    new_off, new_ids, new_sto = [0], [], []
    for l in range(len(offsets) - 1):
        if keep[l]:
            a, b = offsets[l], offsets[l + 1]
            new_ids.append(ids[a:b])
            new_sto.append(storage.reshape(-1, dim)[a:b])
        new_off.append(new_off[-1] + (offsets[l + 1] - offsets[l] if keep[l] else 0))
    return (np.array(new_off, np.uint32), np.concatenate(new_ids).astype(np.uint32),
            np.concatenate(new_sto).astype(np.float32))


def worker(rank, world, port, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import Oracle
    from paper_2411_17229_b200.dist import plan_list_shards
    fx = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "ivf_fix.npz")))
    dim, k, npb = 16, 10, 5
    owner = plan_list_shards(fx["offsets"], world, dim)
    off, ids, sto = shard_index(fx["offsets"], fx["ids"], fx["storage"], dim, owner == rank)
    o = Oracle()
    li, ld, lc, _ = o.ivf_search(fx["centroids"], off, ids, sto, fx["queries"], k, npb)
    # two-phase scheme (dade_gpu_ivf_search_keys_begin/_end): phase 1 = each query's
    # nearest LOCAL probed list -> radius; all-reduce MIN of the radius' fp32 bits
    # as int32; phase 2 keeps only candidates within the reduced radius (FD: prune
    # iff dist > r), phase-1 results always kept
    qs = fx["queries"]
    cen = fx["centroids"].reshape(-1, dim).astype(np.float64)
    d2c = ((qs.astype(np.float64)[:, None, :] - cen[None]) ** 2).sum(2)
    probes = np.lexsort((np.tile(np.arange(cen.shape[0]), (qs.shape[0], 1)), d2c), axis=1)[:, :npb]
    nonempty = np.diff(off.astype(np.int64)) > 0
    rad = np.full(qs.shape[0], np.inf, np.float32)
    near = np.full(qs.shape[0], -1)
    rows = sto.reshape(-1, dim)
    for q in range(qs.shape[0]):
        loc = [l for l in probes[q] if nonempty[l]]
        if not loc:
            continue
        near[q] = loc[0]
        a, b = off[loc[0]], off[loc[0] + 1]
        dd = np.sqrt(((rows[a:b].astype(np.float64) - qs[q]) ** 2).sum(1))
        if b - a >= k:
            rad[q] = np.float32(np.sort(dd)[k - 1] * (1 + 1e-6))
    r_bits = torch.from_numpy(rad.view(np.int32).copy())
    dist.all_reduce(r_bits, op=dist.ReduceOp.MIN)
    r_glob = r_bits.numpy().view(np.float32)
    assert np.all(r_glob <= rad)
    for q in range(qs.shape[0]):
        keep = []
        for i in range(int(lc[q])):
            a, b = (off[near[q]], off[near[q] + 1]) if near[q] >= 0 else (0, 0)
            in_near = np.any(ids[a:b] == li[q, i])
            if in_near or ld[q, i] <= r_glob[q]:
                keep.append(i)
        li[q, :len(keep)], ld[q, :len(keep)] = li[q, keep], ld[q, keep]
        lc[q] = len(keep)
    keys = torch.from_numpy(pack(li, ld, lc, k).view(np.int64))
    # query-owner exchange (dist.sharded_ivf_search): all-to-all sends rows
    # [j * nq_loc, (j + 1) * nq_loc) of every rank's keys to rank j, which merges
    # its own queries; the owners' answers are gathered here only to check them
    nq_loc = qs.shape[0] // world
    recv = torch.empty((world, nq_loc, k), dtype=torch.int64)
    dist.all_to_all_single(recv, keys.contiguous())
    own = torch.from_numpy(merge([b.numpy().view(np.uint64) for b in recv], k).view(np.int64))
    gathered = [torch.empty_like(own) for _ in range(world)]
    dist.all_gather(gathered, own)
    if rank == 0:
        result.put(np.concatenate([g.numpy().view(np.uint64) for g in gathered]))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(300)
def test_list_sharded_search_equals_single_rank(ivf_fix, oracle_lib):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    fx = ivf_fix
    ri, rd, rc, _ = oracle_lib.ivf_search(fx["centroids"], fx["offsets"], fx["ids"], fx["storage"], fx["queries"], 10, 5)
    expect = pack(ri, rd, rc, 10)
    assert np.array_equal(merged, expect)
