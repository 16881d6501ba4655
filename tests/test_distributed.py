"""World-size-2 gloo tests (CPU) of the multi-process host logic: sharding and
the exact mod-2^32 merge of partial encrypted models."""

import hashlib
import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN, REPO

sys.path.insert(0, GOLDEN)


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _worker(rank, world, port, q):
    sys.path.insert(0, REPO)
    sys.path.insert(0, GOLDEN)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from cases import TRAIN_CASES, train_inputs
        from oracle import wnn32
        from paper_2403_20190_b200 import distributed as D
        name = "train_cfg1"
        P, s1, bits, labels, stacks = train_inputs(name)
        s, l, a, r = TRAIN_CASES[name][2]
        mine = D.stripe(stacks, rank, world)
        rams, counts = wnn32.he_train(mine, s, l, a, r, P)              # partial model on this rank
        rt = torch.from_numpy(rams.view(np.int32).copy())
        ct = torch.from_numpy(counts.view(np.int32).copy())
        D.merge_models_(rt, ct)
        q.put((rank, sha(rt.numpy().view(np.uint32)), ct.numpy().view(np.uint32).copy()))
    finally:
        dist.destroy_process_group()


def test_sharded_training_merge_is_exact():
    from conftest import golden
    world = 2
    port = 29500 + (os.getpid() % 1000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = golden("train_cfg1.npz")
    for rank, rams_sha, counts in res:
        assert rams_sha == str(g["sha_rams"]), f"rank {rank} merged model differs from sequential training"
        assert np.array_equal(counts, g["counts_ct"])


@pytest.mark.parametrize("total,world", [(4096, 1), (4096, 8), (10, 3), (2, 4)])
def test_shard_range_partitions(total, world):
    from paper_2403_20190_b200.distributed import shard_range
    spans = [shard_range(total, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == total
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1


def test_allreduce_wraps_mod_2_32_single_process():
    # world size 1 gloo group: the wrap arithmetic of allreduce_u32_
    from paper_2403_20190_b200.distributed import allreduce_u32_
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(28500 + os.getpid() % 1000))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        t = torch.tensor([-1, 2 ** 31 - 1, 5], dtype=torch.int32)
        allreduce_u32_(t)
        assert t.tolist() == [-1, 2 ** 31 - 1, 5]
    finally:
        dist.destroy_process_group()
