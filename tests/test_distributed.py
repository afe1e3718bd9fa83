"""CPU: multi-rank host logic with the gloo backend (world size 2).

Frame batches (BASELINE configs[3]) shard round-robin with no data-path
collective; these tests check the sharding, the bookkeeping collectives and
that the gathered results equal a single-process run.  The per-frame solve is
the CPU oracle here (no GPU in this container); on a B200 box the same code
drives Solver.run_batch.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2110_03946_b200 import batch


def test_frames_for_rank_partition():
    for n in (0, 1, 5, 64):
        for world in (1, 2, 3, 8):
            owned = [batch.frames_for_rank(n, world, r) for r in range(world)]
            flat = sorted(k for o in owned for k in o)
            assert flat == list(range(n))
            assert all(k % world == r for r, o in enumerate(owned) for k in o)
    with pytest.raises(ValueError):
        batch.frames_for_rank(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _make_frame(k):
    import paper_2110_03946_b200 as si
    f = si.synthetic_test_image(48, 40, 2, 7 + k)
    m = si.random_mask(48, 40, 0.08, 11 + k)
    return f.data, m.known


def _solve(frames):
    from oracle import pyoracle
    return [pyoracle.oracle_solve(f, m, levels=2, block_size=16, overlap=4).image for f, m in frames]


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        local = batch.run_sharded(7, _make_frame, _solve, dist)
        merged = batch.gather_results(local, dist)
        assert sorted(local["frames"]) == batch.frames_for_rank(7, world, rank)
        assert local["slowest_s"] >= local["elapsed_s"]
        if rank == 0:
            np.savez(os.path.join(out_dir, "merged.npz"),
                     **{f"f{k}": v for k, v in merged.items()})
    finally:
        dist.destroy_process_group()


def test_sharded_batch_matches_single_process(tmp_path):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    merged = np.load(os.path.join(tmp_path, "merged.npz"))
    single = batch.run_sharded(7, _make_frame, _solve, None)
    assert sorted(int(k[1:]) for k in merged.files) == list(range(7))
    for k, img in single["frames"].items():
        assert np.array_equal(merged[f"f{k}"], img)
