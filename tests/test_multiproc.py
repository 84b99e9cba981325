"""N>1 host logic on CPU (gloo, world_size 2): bench.py's sharded path — every rank draws
the same batch list, takes its cost-balanced shard (shards.plan_shards), scores it (here
with the CPU oracle standing in for the GPU), scatters into the shared-memory host gather
(shards.HostGather) — and the max-over-ranks timing reduction.  Rank 0 then checks the
gathered result is bitwise the unsharded one.  No collective on the data path."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import bench
    from oracle import oracle
    from paper_2411_11547_b200 import datagen
    from paper_2411_11547_b200.shards import HostGather
    full = datagen.workload("c3", num_batches=6)
    shard = bench.shard_for_rank(full, ws, rank)
    name = "phmm_test_gather_%d" % port
    if rank == 0:
        gather = HostGather(name, full.num_pairs, create=True)
    dist.barrier()
    if rank != 0:
        gather = HostGather(name, full.num_pairs, create=False)
    acc, st = oracle.score_raw(oracle.Flat(**shard.flat.as_dict()), "f32", 120, threads=2)
    gather.put(shard.gids, oracle.finish(acc, st, 120), st)
    cells = int(bench.pair_cells(shard.flat).sum())
    t, c = bench.reduce_time_cells(0.5 + rank, cells, ws, "cpu")
    dist.barrier()
    if rank == 0:
        ref, kind = oracle.score(oracle.Flat(**full.as_dict()), "f32", threads=2)
        out["equal"] = bool(np.array_equal(gather.scores, ref, equal_nan=True) and
                            np.array_equal(gather.status, kind))
        out["all_cells"] = int(bench.pair_cells(full).sum())
    out[rank] = (t, c, shard.flat.num_pairs, shard.cost)
    dist.barrier()
    gather.close()
    dist.destroy_process_group()


def test_two_rank_gloo_shard_score_gather():
    ws = 2
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(ws, port, out), nprocs=ws, join=True)
    (t0, c0, n0, k0), (t1, c1, n1, k1) = out[0], out[1]
    assert t0 == t1 == 1.5                      # max over ranks
    assert c0 == c1 == out["all_cells"]         # cells summed over both shards = the whole list
    assert n0 > 0 and n1 > 0 and abs(k0 - k1) / (k0 + k1) < 0.05   # cost-balanced
    assert out["equal"]                         # gathered == unsharded, bitwise
