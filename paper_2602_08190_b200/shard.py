"""Multi-GPU partitioning of column chunks: chunks are self-contained, so decode shards
embarrassingly -- each rank takes a contiguous range of every column's chunks, balanced by COMPRESSED
bytes (the end-to-end path is PCIe-bound per GPU), and the only collective is one all-reduce of
per-rank metadata (rows, decoded bytes, compressed bytes, error bits) plus a MAX of the device time.
Host logic only; exercised with world_size 2 over gloo in tests/test_multiprocess.py."""
from __future__ import annotations


def shard_ranges(sizes: list[int], world: int) -> list[tuple[int, int]]:
    """Split one column's chunk list (compressed sizes, in row order) into `world` contiguous ranges
    [a, b) with near-equal byte totals.  Ranks may get an empty range when chunks < world."""
    n = len(sizes)
    if n <= world:  # one chunk per rank, the rest empty
        return [(min(r, n), min(r + 1, n)) for r in range(world)]
    total = sum(sizes)
    bounds = [0]
    acc = 0
    k = 1
    for i, s in enumerate(sizes):
        acc += s
        rest = n - (i + 1)  # chunks after this one
        # close range k-1 (never empty) once it holds its share of the bytes, as long as every later rank
        # still gets a chunk; close it anyway when exactly one chunk per later rank remains
        if k < world and bounds[-1] < i + 1 and rest >= world - k and (acc >= total * k / world or rest == world - k):
            bounds.append(i + 1)
            k += 1
    while len(bounds) < world:
        bounds.append(n)
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def shard_columns(columns: dict[str, list[int]], rank: int, world: int) -> dict[str, tuple[int, int]]:
    """Per column name -> this rank's chunk range."""
    return {name: shard_ranges(sizes, world)[rank] for name, sizes in columns.items()}


def reduce_metadata(rows: int, decoded: int, compressed: int, err_bits: int, seconds: float, group=None,
                    device=None):
    """One SUM all-reduce of the counters and one MAX of the elapsed time (torch.distributed; NCCL on
    GPUs, gloo in tests).  Error bits are OR-ed by summing one-hot bits per rank (each bit position summed,
    then tested for > 0)."""
    import torch
    import torch.distributed as dist
    bits = [(err_bits >> b) & 1 for b in range(8)]
    t = torch.tensor([rows, decoded, compressed, *bits], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    m = torch.tensor([seconds], dtype=torch.float64, device=device)
    dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
    v = [int(x) for x in t.tolist()]
    err = sum(1 << b for b in range(8) if v[3 + b] > 0)
    return {"rows": v[0], "decoded": v[1], "compressed": v[2], "error_bits": err, "seconds": float(m.item())}
