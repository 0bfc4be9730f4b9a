"""The N>1 path on CPU: world_size 2 over gloo.  Each rank decodes its shard of every column's chunks
(with the oracle -- no GPU here), the metadata all-reduce totals equal the single-process totals, and the
union of the rank outputs equals the whole column byte for byte."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2602_08190_b200.shard import shard_ranges


def test_shard_ranges_cover_and_balance():
    for sizes, world in [([5] * 10, 2), ([1, 100, 1, 1, 100], 2), ([3], 4), ([], 3), ([7] * 143, 8)]:
        rs = shard_ranges(sizes, world)
        assert len(rs) == world
        assert rs[0][0] == 0 and rs[-1][1] == len(sizes)
        for (a, b), (c, d) in zip(rs, rs[1:]):
            assert b == c and a <= b
        if len(sizes) >= world and len(set(sizes)) == 1:
            per = [b - a for a, b in rs]
            assert max(per) - min(per) <= 1


def test_shard_ranges_every_rank_gets_a_chunk():
    # a large leading chunk must not close several ranges at once: with chunks >= ranks, no rank
    # is left empty; with fewer chunks than ranks, each chunk goes to its own rank
    for sizes, world in [([100, 1, 1, 1], 4), ([1, 1, 1, 100], 2), ([1000, 1, 1, 1, 1, 1], 3), ([9, 9], 4)]:
        rs = shard_ranges(sizes, world)
        per = [b - a for a, b in rs]
        assert sum(per) == len(sizes)
        assert all(p >= 1 for p in per[:min(world, len(sizes))]), (sizes, world, rs)
    assert shard_ranges([100, 1, 1, 1], 4) == [(0, 1), (1, 2), (2, 3), (3, 4)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    import oracle
    from paper_2602_08190_b200 import encoder
    from paper_2602_08190_b200.inputs import TPCH
    from paper_2602_08190_b200.shard import shard_columns, reduce_metadata
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = TPCH(0.01)
    cols = {"l_orderkey": "RLE|[Delta|RLE|[BitPack,BitPack],BitPack]", "l_quantity": "Dict|BitPack",
            "l_comment": "Str|[LZ4,BitPack]"}
    chunks = {n: encoder.encode_chunks(s, g.column(n), 7_000) for n, s in cols.items()}
    ranges = shard_columns({n: [c.size for c in ch] for n, ch in chunks.items()}, rank, world)
    rows = dec = comp = 0
    mine = {}
    for n, (a, b) in ranges.items():
        outs = []
        for c in chunks[n][a:b]:
            payload, offs = oracle.decode_chunk(c)
            info = oracle.oracle._header(c)
            rows += info[2]
            dec += payload.size + (offs.size * 4 if offs is not None else 0)
            comp += c.size
            outs.append(payload.tobytes())
        mine[n] = (a, b, outs)
    meta = reduce_metadata(rows, dec, comp, 0, 0.5 + rank)
    q.put((rank, meta, mine))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_ranks_gloo_union_equals_whole():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    import oracle
    from paper_2602_08190_b200.inputs import TPCH
    g = TPCH(0.01)
    total_rows = sum(g.column(n).rows for n in ("l_orderkey", "l_quantity", "l_comment"))
    assert res[0][1] == res[1][1]                       # both ranks see the same reduced metadata
    assert res[0][1]["rows"] == total_rows              # all-reduced rows == generator rows
    assert res[0][1]["seconds"] == 1.5                  # MAX over ranks
    for n in ("l_orderkey", "l_quantity", "l_comment"):
        (a0, b0, o0), (a1, b1, o1) = res[0][2][n], res[1][2][n]
        assert b0 == a1
        union = b"".join(o0 + o1)
        col = g.column(n)
        assert union == col.data.tobytes()
