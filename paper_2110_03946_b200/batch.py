"""Frame batches across GPUs (BASELINE configs[3], SURVEY.md §8e "C4").

Independent frames shard with no data-path collective: frame k goes to rank
k mod G, every rank solves its frames on its own GPU (one si_ctx per rank,
Solver.run_batch overlapping host<->device copies with the solves), and the
only communication is bookkeeping (which frames, how long) over
torch.distributed.  bench.py's end-to-end leg runs through run_sharded.
"""
from __future__ import annotations

import time
from typing import Callable, List, Optional, Sequence


def frames_for_rank(n_frames: int, world: int, rank: int) -> List[int]:
    """Frame indices owned by `rank`: k mod world == rank (round robin)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid world/rank")
    return list(range(rank, n_frames, world))


def run_sharded(n_frames: int, make_frame: Callable[[int], object],
                solve: Callable[[Sequence[object]], Sequence[object]],
                dist=None) -> dict:
    """Solve frames 0..n-1 across the ranks of `dist` (torch.distributed or None).

    make_frame(k) builds frame k on the host; solve(frames) returns one result
    per frame.  Returns this rank's {frame index: result} plus the wall time
    and the aggregate frames/s (frames over the slowest rank's time)."""
    world = dist.get_world_size() if dist is not None else 1
    rank = dist.get_rank() if dist is not None else 0
    mine = frames_for_rank(n_frames, world, rank)
    frames = [make_frame(k) for k in mine]
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    results = list(solve(frames)) if frames else []
    elapsed = time.perf_counter() - t0
    slowest = elapsed
    if dist is not None:
        import torch
        dev = None
        if dist.get_backend() == "nccl":  # NCCL reduces device tensors only
            dev = torch.device("cuda", torch.cuda.current_device())
        t = torch.tensor([elapsed], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        slowest = float(t.item())
    return {"rank": rank, "world": world, "frames": dict(zip(mine, results)),
            "elapsed_s": elapsed, "slowest_s": slowest,
            "frames_per_s": n_frames / slowest if slowest > 0 else float("inf")}


def gather_results(local: dict, dist=None) -> dict:
    """All frames' results on every rank (object all-gather); for checking."""
    if dist is None:
        return dict(local["frames"])
    parts: List[Optional[dict]] = [None] * dist.get_world_size()
    dist.all_gather_object(parts, local["frames"])
    merged = {}
    for p in parts:
        merged.update(p)
    return merged
