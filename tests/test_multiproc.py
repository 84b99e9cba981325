"""N>1 host logic on CPU (gloo, world_size 2): weak-scaling shards and the max-over-ranks
timing reduction used by bench.py.  The data path has no collective — pairs are independent."""
import os
import socket

import numpy as np
import pytest
import torch
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
    from paper_2411_11547_b200 import datagen
    flat = datagen.workload("c2", num_batches=2, seed_offset=bench.shard_seed_offset(rank))
    cells = int((flat.read_len[flat.pair_index()[0]] * flat.hap_len[flat.pair_index()[1]]).sum())
    t, c = bench.reduce_time_cells(0.5 + rank, cells, ws, "cpu")
    out[rank] = (t, c, int(flat.read_bases.astype(np.int64).sum()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_shards_and_reduction():
    ws = 2
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(ws, port, out), nprocs=ws, join=True)
    (t0, c0, s0), (t1, c1, s1) = out[0], out[1]
    assert t0 == t1 == 1.5                      # max over ranks
    assert c0 == c1 == 2 * (2 * 16 * 4 * 250 * 250)   # cells summed over both shards
    assert s0 != s1                             # each rank draws its own shard
