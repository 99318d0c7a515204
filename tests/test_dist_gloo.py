"""Multi-process sharding logic on CPU (gloo, world_size 2): shard bounds cover the batch
contiguously with balanced cells, and the gathered results of the sharded run equal the
unsharded run.  The per-shard aligner in this test is the CPU oracle (test-only injection):
this exercises only the host-side shard/gather logic of paper_2002_04561_b200/dist.py."""
import os
import socket

import numpy as np
import pytest


def test_shard_bounds_properties():
    from paper_2002_04561_b200.dist import shard_bounds
    from synth import random_pairs
    q, qo, s, so = random_pairs(500, 0, 300, seed=3)
    cells = (np.diff(qo) + 1.0) * (np.diff(so) + 1.0)
    for world in (1, 2, 3, 4, 8):
        b = shard_bounds(qo, so, world)
        assert b[0] == 0 and b[-1] == 500 and np.all(np.diff(b) >= 0)
        per = [cells[b[r]:b[r + 1]].sum() for r in range(world)]
        assert abs(max(per) - sum(per) / world) <= cells.max() + 1e-9


def _free_port():
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        return s_.getsockname()[1]


def _worker(rank, world, port, out_path):
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2002_04561_b200.dist import align_sharded
    from synth import random_pairs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q, qo, s, so = random_pairs(120, 0, 200, seed=11)
    sch = O.Scheme("semi", "affine", 2, -1, 5, 1)

    def fn(qs, qo_, ss, so_):
        res, _ = O.batch(sch, qs, qo_, ss, so_, threads=1)
        return res["score"].astype(np.int32)

    full, (k0, k1) = align_sharded(fn, q, qo, s, so)
    if rank == 0:
        np.save(out_path, full)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_gather_equals_single(tmp_path):
    import torch.multiprocessing as mp
    from oracle import oracle as O
    from synth import random_pairs
    out = str(tmp_path / "scores.npy")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True,
                       start_method="spawn")
    full = np.load(out)
    q, qo, s, so = random_pairs(120, 0, 200, seed=11)
    res, _ = O.batch(O.Scheme("semi", "affine", 2, -1, 5, 1), q, qo, s, so, threads=2)
    assert np.array_equal(full, res["score"].astype(np.int32))
