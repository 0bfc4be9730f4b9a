"""GPU parity: the CUDA path (through the C-ABI) == the CPU oracle, element by element (-m gpu).

Every chunk is decoded three ways on the device -- through the pipelined engine from pinned host memory
(cdm_submit_batch), through the same schedule captured as a CUDA graph (cdm_pipeline_*), and through the
device-resident batch API (cdm_batch_*) -- and compared byte for byte
with oracle/ on the same seeded inputs.  Integer/byte work must be bit-exact and Float2Int is one IEEE
division on both sides, so the tolerance is zero everywhere.  Outputs are pre-filled
with a sentinel so an element that is never written, or written outside [0, n), is caught.
"""
import os
import struct

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import cdm1
import oracle
from paper_2602_08190_b200 import cdm, encoder
from paper_2602_08190_b200.inputs import (TPCH, VARBYTES, Column, I32, I64, config1_column, rle_column,
                                          uniform_bits_column)

pytestmark = pytest.mark.gpu

SENTINEL = 0xA5


@pytest.fixture(scope="module")
def engine():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    e = cdm.Engine(0, n_slots=3, slot_bytes=256 << 20)
    yield e
    e.close()


def _outputs(chunk):
    info = cdm.chunk_info(chunk)
    out = torch.full((max(16, (info["payload_bytes"] + 15) // 16 * 16 + 64),), SENTINEL, dtype=torch.uint8,
                     device="cuda")
    offs = None
    if info["offsets_bytes"]:
        offs = torch.full((info["offsets_bytes"] // 4 + 4,), -7, dtype=torch.int32, device="cuda")
    return out, offs, info


def gpu_decode(engine, casc, chunks, resident=False, expect_error=False):
    """Decode chunks on the GPU; returns [(payload numpy, offsets numpy|None, result dict)].
    resident: False = cdm_submit_batch, True = cdm_batch_* on device copies, "pipeline" = cdm_pipeline_*,
    "graph" = cdm_batch_* in graph mode (captured on the first launch, replayed on the second)."""
    decs, bufs = [], []
    for ch in chunks:
        out, offs, info = _outputs(ch)
        d = cdm.Decode(casc, cdm.pinned(ch), out, offs)
        if resident is True or resident == "graph":
            d.dev_chunk = torch.from_numpy(ch).cuda()
        decs.append(d)
        bufs.append((out, offs, info))
    # the sentinel fills run on torch's (legacy) default stream, the engine on its own non-blocking streams:
    # the fills must be complete before the decode is enqueued (include/cdm.h: caller-owned outputs)
    torch.cuda.synchronize()
    if resident == "pipeline":
        p = cdm.Pipeline(engine, decs)
        p.launch()
        res = p.results(raise_on_error=not expect_error)
        p.close()
    elif resident == "graph":
        b = cdm.Batch(engine, decs)
        b.set_graph(True)
        stream = torch.cuda.Stream()
        for _ in range(2):  # capture + replay, then a replay over outputs reset to the sentinel
            b.launch(stream)
            res = b.results(stream, raise_on_error=not expect_error)
            for out, offs, _ in bufs:
                out.fill_(SENTINEL)
                if offs is not None:
                    offs.fill_(-7)
            torch.cuda.synchronize()
        b.launch(stream)
        res = b.results(stream, raise_on_error=not expect_error)
        b.close()
    elif resident:
        b = cdm.Batch(engine, decs)
        b.launch()
        res = b.results(raise_on_error=not expect_error)
        b.close()
    else:
        tickets = engine.submit_batch(decs)
        res = [engine.wait(t, raise_on_error=not expect_error) for t in tickets]
    torch.cuda.synchronize()
    outs = []
    for (out, offs, info), r in zip(bufs, res):
        o = out.cpu().numpy()
        p = info["payload_bytes"]
        # nothing written past the payload
        if not expect_error:
            assert np.all(o[p:] == SENTINEL), "write beyond the payload"
        outs.append((o[:p], None if offs is None else offs.cpu().numpy(), r))
    return outs


def check_parity(engine, spec, col_or_chunks, dtype=None, width=0, rows_per_chunk=None, both=True):
    if isinstance(col_or_chunks, Column):
        col = col_or_chunks
        chunks = encoder.encode_chunks(spec, col, rows_per_chunk or max(col.rows, 1))
        dtype, width = col.dtype, col.width
    else:
        chunks = col_or_chunks
    casc = cdm.Cascade(spec, dtype, width)
    modes = [False, "pipeline", True, "graph"] if both else [True]
    for resident in modes:
        got = gpu_decode(engine, casc, chunks, resident=resident)
        for ch, (payload, offs, r) in zip(chunks, got):
            exp, exp_offs = oracle.decode_chunk(ch)
            assert r["error_bits"] == 0
            assert payload.size == exp.size
            if not np.array_equal(payload, exp):
                bad = int(np.flatnonzero(payload != exp)[0])
                raise AssertionError(f"{spec} resident={resident}: first mismatch at byte {bad} "
                                     f"(got {payload[bad]}, oracle {exp[bad]})")
            if exp_offs is not None:
                assert np.array_equal(offs[: exp_offs.size], exp_offs), f"{spec} resident={resident}: offsets differ"
    return chunks


# ------------------------------------------------------------------------------ TPC-H columns, all cascades
TPCH_CASES = [
    ("l_orderkey", "RLE|[Delta|RLE|[BitPack,BitPack],BitPack]"),
    ("l_orderkey", "Delta|RLE|[BitPack,BitPack]"),
    ("l_orderkey", "Delta|BitPack"),
    ("l_orderkey", "BitPack"),
    ("l_partkey", "BitPack"),
    ("l_suppkey", "BitPack"),
    ("l_linenumber", "BitPack"),
    ("l_quantity", "Dict|BitPack"),
    ("l_discount", "Dict|BitPack"),
    ("l_tax", "Float2Int|BitPack"),
    ("l_extendedprice", "Float2Int|BitPack"),
    ("l_returnflag", "Dict|BitPack"),
    ("l_linestatus", "Dict|BitPack"),
    ("l_shipdate", "Dict|BitPack"),
    ("l_shipinstruct", "Dict|BitPack"),
    ("l_shipmode", "Dict|BitPack"),
    ("l_comment", "Str|[LZ4,BitPack]"),
    ("l_comment", "Str|[LZ4(sub=16384,hc=9),BitPack]"),  # the bench's cascade: liblz4 HC blocks (longer matches)
    ("l_comment", "Str|[Raw,BitPack]"),
    ("o_orderkey", "Delta|RLE|[BitPack,BitPack]"),
    ("o_orderkey", "DeltaStride|[Delta|RLE|[BitPack,BitPack],BitPack]"),                 # Table 2 O_ORDERKEY
    ("l_orderkey", "RLE|[DeltaStride|[Delta|RLE|[BitPack,BitPack],BitPack],BitPack]"),  # Table 2 L_ORDERKEY
    ("o_orderkey", "DeltaStride|[BitPack,BitPack]"),
    ("l_orderkey", "DeltaStride(stride=0)|[BitPack,BitPack]"),
    ("l_orderkey", "RLE|[RLE|[BitPack,BitPack],BitPack]"),
    ("l_orderkey", "RLE|[DeltaStride|[BitPack,BitPack],BitPack]"),
    ("o_custkey", "BitPack"),
    ("o_orderstatus", "Dict|BitPack"),
    ("o_totalprice", "Float2Int|BitPack"),
    ("o_orderdate", "RLE|[Dict|BitPack,BitPack]"),
    ("o_orderpriority", "Dict|BitPack"),
    ("o_clerk", "Dict|BitPack"),
    ("o_shippriority", "RLE|[BitPack,BitPack]"),
    ("o_comment", "Str|[LZ4,BitPack]"),
    ("o_totalprice", "RLE|[Float2Int|BitPack,BitPack]"),
    ("l_orderkey", "Raw"),
    ("l_returnflag", "ANS"),                      # Table 2 L_RETURNFLAG (NEXT-1: range ANS, 32 interleaved states)
    ("l_returnflag", "ANS(il=1,chunk=4096)"),     # one state per chunk (thread per chunk)
    ("l_linestatus", "ANS(chunk=1024)"),
    ("l_shipmode", "ANS(tl=10)"),
    ("o_orderstatus", "ANS(chunk=65536)"),
    ("l_comment", "Str|[ANS(chunk=2048),BitPack]"),
    ("l_comment", "Str|[ANS(il=1,chunk=2048),BitPack]"),
    ("o_comment", "Str|[StrDict|BitPack|ANS,BitPack]"),      # Table 2 O_COMMENT (NEXT-2 String-dictionary)
    ("o_comment", "Str|[StrDict|BitPack|ANS(il=1),BitPack]"),
    ("l_comment", "Str|[StrDict|BitPack,BitPack]"),
    ("ps_partkey", "RLE|[DeltaStride|[BitPack,BitPack],RLE|[BitPack,BitPack]]"),  # Table 2 PS_PARTKEY (R35)
    ("ps_suppkey", "Delta|Dict|BitPack"),                                          # Table 2 PS_SUPPKEY (R36)
    ("ps_supplycost", "Float2Int|BitPack"),
    ("ps_availqty", "BitPack"),
    ("ps_comment", "Str|[LZ4,BitPack]"),
]


@pytest.mark.parametrize("name,spec", TPCH_CASES)
def test_tpch_columns(engine, name, spec):
    col = TPCH(0.02).column(name)  # 120k lineitem rows: several tiles per chunk and a ragged tail
    check_parity(engine, spec, col, rows_per_chunk=50_001)


# ------------------------------------------------------------------------------ golden vectors on the GPU
def test_golden_vectors_gpu(engine, golden):
    g = golden("orderkey_nested.json")
    iv, ic, oc = g["bitpack_inner_values"], g["bitpack_inner_counts"], g["bitpack_outer_counts"]
    inner = cdm1.Node(cdm1.RLE, 10, [
        cdm1.Node(cdm1.BITPACK, 4, [cdm1.raw(bytes.fromhex(iv["bytes"]))], w=iv["w"], base=iv["for"]),
        cdm1.Node(cdm1.BITPACK, 4, [cdm1.raw(bytes.fromhex(ic["bytes"]))], w=ic["w"], base=ic["for"])],
        nruns=4, maxrun=7)
    root = cdm1.Node(cdm1.RLE, 20, [
        cdm1.Node(cdm1.DELTA, 10, [inner], base=g["delta_base"]),
        cdm1.Node(cdm1.BITPACK, 10, [cdm1.raw(bytes.fromhex(oc["bytes"]))], w=oc["w"], base=oc["for"])],
        nruns=10, maxrun=4)
    spec = g["cascade"]
    h = _hash(spec)
    ch = cdm1.build(root, cdm1.I64, 8, 20, cascade_hash=h)
    casc = cdm.Cascade(spec, cdm.I64)
    (payload, _, r), = gpu_decode(engine, casc, [ch], resident=True)
    assert payload.view(np.int64).tolist() == g["column"]

    s = golden("spec_bitpack.json")
    ch = cdm1.build(cdm1.Node(cdm1.BITPACK, 4, [cdm1.raw(bytes.fromhex(s["bitpack"]["bytes"]))], w=3, base=3),
                    cdm1.I32, 4, 4, cascade_hash=_hash("BitPack"))
    (payload, _, r), = gpu_decode(engine, cdm.Cascade("BitPack", cdm.I32), [ch], resident=True)
    assert payload.view(np.int32).tolist() == s["column"]


def _hash(spec):
    h = 14695981039346656037
    for b in encoder.canonical(spec).encode():
        h = ((h ^ b) * 1099511628211) & ((1 << 64) - 1)
    return h


# ------------------------------------------------------------------------------ bit widths / tile edges
@pytest.mark.parametrize("w", list(range(0, 65)))
def test_bitpack_every_width_tile_edges(engine, w):
    n = 3 * 4096 + 77
    col = uniform_bits_column(n, w, I64)
    chunks = [encoder.encode("BitPack", Column("x", I64, 8, m, col.data[:m])) for m in (1, 4095, 4096, 4097, n)]
    check_parity(engine, "BitPack", chunks, I64, both=False)
    if w <= 32:
        c32 = uniform_bits_column(n, w, I32)
        check_parity(engine, "BitPack", [encoder.encode("BitPack", c32)], I32, both=False)


def test_config1_parity(engine):
    check_parity(engine, "BitPack", config1_column())


@pytest.fixture(params=[0, 1, 2])
def scan_mode(request):
    """every H6 schedule (NEXT-3 knob scan_mode): 0 reduce-then-scan, 1 single-pass decoupled look-back, 2 warp
    tiles (three passes, no CTA barriers)"""
    prev = cdm.tune_get("scan_mode")
    cdm.tune_set("scan_mode", request.param)
    yield request.param
    cdm.tune_set("scan_mode", prev)


@pytest.mark.parametrize("w", [1, 3, 8, 17, 33, 64])
def test_delta_scan_many_tiles(engine, w, scan_mode):
    rng = np.random.default_rng(w)
    n = 300_000
    d = rng.integers(0, 1 << min(w, 62), size=n, dtype=np.uint64).astype(np.int64)
    col = Column("walk", I64, 8, n, np.cumsum(d))
    check_parity(engine, "Delta|BitPack", col, rows_per_chunk=123_457)
    col32 = Column("walk32", I32, 4, n, np.cumsum(d).astype(np.int32))
    check_parity(engine, "Delta|BitPack", col32, rows_per_chunk=200_000)


# ------------------------------------------------------------------------------ RLE distributions
RLE_DISTS = ["even-1", "even-2", "even-4", "even-64", "even-1024", "random-1-8", "random-1-1000",
             "outlier-1024-1", "outlier-100000-0.01", "mixed-even-2+random-1-64", "mixed-outlier-1024-1+even-8",
             "single"]


@pytest.mark.parametrize("cap", [1, 3, 8])
def test_gp_occupancy_knob(engine, cap):
    """the G.P. tuner knob (resident rle_kernel CTAs per SM) changes scheduling only, never bytes"""
    prev = cdm.tune_get("gp_ctas_per_sm")
    cdm.tune_set("gp_ctas_per_sm", cap)
    try:
        check_parity(engine, "RLE|[Delta|RLE|[BitPack,BitPack],BitPack]", TPCH(0.02).column("l_orderkey"),
                     rows_per_chunk=50_001, both=False)
        check_parity(engine, "RLE|[BitPack,BitPack]", rle_column("random-1-8", 300_000, I64), both=False)
    finally:
        cdm.tune_set("gp_ctas_per_sm", prev)


@pytest.mark.parametrize("dist", RLE_DISTS)
def test_rle_distributions(engine, dist):
    col = rle_column(dist, 1_000_003, I64)
    check_parity(engine, "RLE|[BitPack,BitPack]", col, rows_per_chunk=600_000)
    col32 = rle_column(dist, 400_000, I32)
    check_parity(engine, "RLE|[BitPack,BitPack]", col32, both=False)


def test_giant_runs(engine):
    # o_shippriority-like: one run per chunk and runs far above the big-tile limit
    n = 5_000_000
    col = Column("zeros", I32, 4, n, np.zeros(n, dtype=np.int32))
    check_parity(engine, "RLE|[BitPack,BitPack]", col, rows_per_chunk=4_194_304, both=False)
    counts = np.array([3, 2_000_000, 1, 1, 70_000, 5, 999_999], dtype=np.int64)
    vals = np.arange(len(counts), dtype=np.int64) * 7 + 1
    col = Column("big", I64, 8, int(counts.sum()), np.repeat(vals, counts))
    check_parity(engine, "RLE|[BitPack,BitPack]", col, both=False)
    check_parity(engine, "Delta|RLE|[BitPack,BitPack]", col, both=False)


@pytest.mark.parametrize("stride", [1, 3, -7, 0])
def test_dstride_random_runs(engine, stride):
    """DeltaStride over random arithmetic runs: many tiles, int64 and int32 (wrapping) output."""
    rng = np.random.default_rng(20 + stride)
    nr = 300_000
    counts = rng.integers(1, 9, size=nr)
    counts[rng.integers(0, nr, size=200)] = rng.integers(100, 5000, size=200)
    starts = rng.integers(-(1 << 40), 1 << 40, size=nr)
    n = int(counts.sum())
    idx = np.arange(n) - np.repeat(np.cumsum(counts) - counts, counts)
    v = np.repeat(starts, counts) + idx * stride
    spec = f"DeltaStride(stride={stride & ((1 << 64) - 1)})|[BitPack,BitPack]"
    check_parity(engine, spec, Column("ds", I64, 8, n, v.astype(np.int64)), rows_per_chunk=1_000_003)
    v32 = (np.repeat(starts % 1000, counts) + idx * stride).astype(np.int32)[:700_001]
    check_parity(engine, spec, Column("ds32", I32, 4, v32.size, v32), both=False)


def test_dstride_giant_runs(engine):
    """Arithmetic runs far above the big-tile limit (rle_big with a stride), at every lineage depth."""
    n = 5_000_000
    keys = np.arange(n, dtype=np.int64) * 3 + 11
    keys[2_000_000:] += 1000
    col = Column("seq", I64, 8, n, keys)
    check_parity(engine, "DeltaStride(stride=3)|[BitPack,BitPack]", col, rows_per_chunk=4_194_304, both=False)
    check_parity(engine, "DeltaStride(stride=3)|[Delta|RLE|[BitPack,BitPack],BitPack]", col, both=False)
    lines = np.repeat(keys[:1_000_000], np.tile([1, 2, 7], 333_334)[:1_000_000])
    check_parity(engine, "RLE|[DeltaStride(stride=3)|[Delta|RLE|[BitPack,BitPack],BitPack],BitPack]",
                 Column("lk", I64, 8, lines.size, lines), both=False)


def test_corrupt_dstride_counts_set_error(engine):
    spec = "RLE|[DeltaStride|[Delta|RLE|[BitPack,BitPack],BitPack],BitPack]"
    inner = cdm1.Node(cdm1.RLE, 4, [cdm1.bitpack([0, 32], 6, 0), cdm1.bitpack([1, 3], 2, 0)], nruns=2, maxrun=3)
    ds = cdm1.Node(cdm1.DSTRIDE, 32, [cdm1.Node(cdm1.DELTA, 4, [inner], base=1), cdm1.bitpack([8, 8, 8, 9], 4, 0)],
                   nruns=4, maxrun=9, stride=1)  # level-1 counts sum to 33 != 32
    root = cdm1.Node(cdm1.RLE, 64, [ds, cdm1.bitpack([2] * 32, 2, 0)], nruns=32, maxrun=2)
    ch = cdm1.build(root, cdm1.I64, 8, 64, cascade_hash=_hash(spec))
    (_, _, r), = gpu_decode(engine, cdm.Cascade(spec, cdm.I64), [ch], resident=True, expect_error=True)
    assert r["error_bits"] & cdm.ERR_RUN_SUM


def _counts_lineage_column(seed, nr, dtype=I64, arith=False):
    """Run counts that are themselves run-length coded (counts repeat in runs of 1..60, a few far above the
    big-tile limit), run values random (or an arithmetic sequence, arith=True)."""
    rng = np.random.default_rng(seed)
    cvals = rng.integers(1, 10, size=nr // 20 + 1)
    cvals[rng.integers(0, cvals.size, size=3)] = rng.integers(5000, 40_000, size=3)
    counts = np.repeat(cvals, rng.integers(1, 60, size=cvals.size))[:nr]
    vals = np.arange(counts.size, dtype=np.int64) * 3 + 17 if arith else rng.integers(-(1 << 40), 1 << 40,
                                                                                      size=counts.size)
    vals[1:] += (vals[1:] == vals[:-1])  # adjacent runs differ (maximal runs)
    v = np.repeat(vals, counts)
    return Column("cl", dtype, 8 if dtype == I64 else 4, v.size, v.astype(np.int64 if dtype == I64 else np.int32))


@pytest.mark.parametrize("spec,arith", [
    ("RLE|[BitPack,RLE|[BitPack,BitPack]]", False),
    ("RLE|[RLE|[BitPack,BitPack],RLE|[BitPack,BitPack]]", False),
    ("RLE|[DeltaStride(stride=3)|[BitPack,BitPack],RLE|[BitPack,BitPack]]", True),
    ("RLE|[DeltaStride(stride=3)|[Delta|RLE|[BitPack,BitPack],BitPack],RLE|[BitPack,BitPack]]", True),
    ("RLE|[BitPack,DeltaStride(stride=0)|[BitPack,BitPack]]", False),
    ("RLE|[BitPack,Delta|RLE|[BitPack,BitPack]]", False),
])
def test_counts_lineage(engine, spec, arith):
    """Table 2 PS_PARTKEY's shape (R35): the outer RLE's counts come from a lower RLE-family level (a u32 array
    in L2, its rle_sums launched after the round that writes it), next to a value lineage of depth 0-2; many
    tiles, ragged chunks, giant runs, int64 and int32 output."""
    col = _counts_lineage_column(5, 400_000, arith=arith)
    check_parity(engine, spec, col, rows_per_chunk=1_500_007)
    c32 = _counts_lineage_column(6, 60_000, dtype=I32, arith=arith)
    check_parity(engine, spec, c32, rows_per_chunk=250_001, both=False)


def test_ps_partkey_sf10_full(engine):
    """PS_PARTKEY at SF 10 (8 M rows) under Table 2's cascade: each chunk holds ONE DeltaStride run and ONE counts
    run of 1 M entries (both lineage levels are giant runs: rle_big), expanded into 4 M rows"""
    col = TPCH(10).column("ps_partkey")
    check_parity(engine, "RLE|[DeltaStride|[BitPack,BitPack],RLE|[BitPack,BitPack]]", col,
                 rows_per_chunk=1 << 22, both=False)


def test_corrupt_counts_lineage_sets_error(engine):
    """a counts level whose own counts overrun its element count, and an outer level whose lineage counts do
    not sum to its rows: both are CDM_ERR_RUN_SUM"""
    spec = "RLE|[BitPack,RLE|[BitPack,BitPack]]"
    for inner_counts, n in (([2, 3], 20), ([2, 2], 20), ([2, 3], 21)):  # 5 counts of 4 = 20 rows is the clean case
        cn = cdm1.Node(cdm1.RLE, 5, [cdm1.bitpack([4, 4], 3, 0), cdm1.bitpack(inner_counts, 2, 0)], nruns=2, maxrun=3)
        root = cdm1.Node(cdm1.RLE, n, [cdm1.bitpack([1, 2, 3, 4, 5], 3, 0), cn], nruns=5, maxrun=4)
        ch = cdm1.build(root, cdm1.I64, 8, n, cascade_hash=_hash(spec))
        exp_ok = inner_counts == [2, 3] and n == 20
        (payload, _, r), = gpu_decode(engine, cdm.Cascade(spec, cdm.I64), [ch], resident=True,
                                      expect_error=not exp_ok)
        if exp_ok:
            assert r["error_bits"] == 0 and np.array_equal(payload, oracle.decode_chunk(ch)[0])
        else:
            assert r["error_bits"] & cdm.ERR_RUN_SUM


@pytest.mark.parametrize("w", [1, 7, 13])
def test_delta_dict_scan(engine, w, scan_mode):
    """Table 2 PS_SUPPKEY's `Delta|Dict|BitPack` (R36): the deltas are dictionary entries gathered inside the scan
    (both H6 schedules); 2^w distinct deltas incl. negative ones (wrapping), many tiles, int64 and int32"""
    rng = np.random.default_rng(w)
    d = rng.integers(-(1 << 30), 1 << 30, size=1 << w)
    n = 700_001
    x = np.cumsum(d[rng.integers(0, d.size, size=n)]) + 12345
    check_parity(engine, "Delta|Dict|BitPack", Column("dd", I64, 8, n, x.astype(np.int64)), rows_per_chunk=300_007)
    check_parity(engine, "Delta|Dict|BitPack", Column("dd32", I32, 4, n, x.astype(np.int32)), both=False)


def test_delta_dict_bad_index_sets_error(engine, scan_mode):
    spec = "Delta|Dict|BitPack"
    n = 9000
    dn = cdm1.Node(cdm1.DICT, n, [cdm1.raw(np.arange(5, dtype=np.int64).tobytes(), eb=8),
                                  cdm1.bitpack([i % 7 for i in range(n)], 3, 0)], entries=5, E=8)
    root = cdm1.Node(cdm1.DELTA, n, [dn], base=0)
    ch = cdm1.build(root, cdm1.I64, 8, n, cascade_hash=_hash(spec))
    (_, _, r), = gpu_decode(engine, cdm.Cascade(spec, cdm.I64), [ch], resident=True, expect_error=True)
    assert r["error_bits"] & cdm.ERR_DICT_INDEX


def test_strdict_long_tokens_and_empty_strings(engine):
    """String-dictionary tiles past the staging size (32-byte tokens: direct stores), empty strings, one token."""
    rng = np.random.default_rng(9)
    alpha = np.frombuffer(b"abcdefghij", dtype=np.uint8)
    lens = rng.integers(0, 400, size=20_000)
    lens[rng.random(lens.size) < 0.1] = 0
    data = alpha[rng.integers(0, 3, size=int(lens.sum()))]  # few letters, no delimiters: long 32-byte tokens
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    col = Column("long", VARBYTES, 0, lens.size, data, offs)
    for spec in ("Str|[StrDict|BitPack,BitPack]", "Str|[StrDict|BitPack|ANS,BitPack]"):
        check_parity(engine, spec, col, rows_per_chunk=7_001, both=False)
    one = Column("one", VARBYTES, 0, 3, np.frombuffer(b"hello ", dtype=np.uint8).copy(),
                 np.array([0, 0, 6, 6], dtype=np.int64))
    check_parity(engine, "Str|[StrDict|BitPack,BitPack]", one, both=False)


@pytest.mark.parametrize("env", [{"CDM_SD_EXPAND": "1"}, {"CDM_SD_EXPAND": "2"}])
def test_strdict_expand_variants(env):
    """the opt-in String-dictionary expansions -- round 1's per-tile sd_expand (CDM_SD_EXPAND=1) and the
    word-parallel sd_expand2 (CDM_SD_EXPAND=2) -- decode the same bytes (fresh process: env read once)"""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, 'tests'); import test_gpu_parity as t; from paper_2602_08190_b200 import cdm; "
            "from paper_2602_08190_b200.inputs import TPCH; e = cdm.Engine(0); "
            "t.check_parity(e, 'Str|[StrDict|BitPack|ANS,BitPack]', TPCH(0.02).column('o_comment'), rows_per_chunk=50_001, both=False); "
            "t.test_strdict_long_tokens_and_empty_strings(e); print('ok')")
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True,
                       text=True, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_corrupt_strdict_sets_error(engine):
    spec = "Str|[StrDict|BitPack,BitPack]"
    blob = np.array([0, 2, 5], np.uint32).tobytes() + b"a b. "
    for ids, bit in (([0, 3, 0], cdm.ERR_DICT_INDEX), ([0, 1], cdm.ERR_LENGTHS)):
        sd = cdm1.Node(cdm1.STRDICT, 7, [cdm1.raw(blob), cdm1.bitpack(ids, 2, 0)], entries=2, E=5)
        root = cdm1.Node(cdm1.STR, 1, [sd, cdm1.bitpack([7], 3, 0)])
        ch = cdm1.build(root, cdm1.VARBYTES, 0, 1, payload=7, cascade_hash=_hash(spec))
        (_, _, r), = gpu_decode(engine, cdm.Cascade(spec, cdm.VARBYTES), [ch], resident=True, expect_error=True)
        assert r["error_bits"] & bit


def test_rle_zero_length_runs(engine):
    """Foreign encoders may emit zero-length runs; the decoder must skip them (decode parity only)."""
    rng = np.random.default_rng(12)
    nr = 5000
    counts = rng.integers(0, 4, size=nr)
    counts[100:200] = 0
    vals = rng.integers(0, 1 << 20, size=nr)
    n = int(counts.sum())
    spec = "RLE|[BitPack,BitPack]"
    root = cdm1.Node(cdm1.RLE, n, [cdm1.bitpack(vals, 20, 0), cdm1.bitpack(counts, 2, 0)], nruns=nr, maxrun=3)
    ch = cdm1.build(root, cdm1.I64, 8, n, cascade_hash=_hash(spec))
    check_parity(engine, spec, [ch], I64)


def test_nested_orderkey_sf1_full(engine):
    """Config 2's l_orderkey at full SF=1 size, every element against the oracle."""
    col = TPCH(1).column("l_orderkey")
    check_parity(engine, "RLE|[Delta|RLE|[BitPack,BitPack],BitPack]", col, rows_per_chunk=1 << 22)


def test_config2_full(engine):
    g = TPCH(1)
    for name in ("l_quantity", "l_discount"):
        check_parity(engine, "Dict|BitPack", g.column(name), rows_per_chunk=1 << 22, both=False)


# ------------------------------------------------------------------------------ LZ4
@pytest.mark.parametrize("sub", [4096, 65536, 1 << 20])
def test_lz4_subchunk_sizes(engine, sub):
    col = TPCH(0.01).column("l_comment")
    check_parity(engine, f"Str|[LZ4(sub={sub}),BitPack]", col, rows_per_chunk=40_000, both=False)


@pytest.fixture(params=["spec", "split", "split1", "split2", "split4", "split8", 1, 4, 2, 8, 16, 32])
def lz4_lanes(request):
    """every LZ4 schedule the tuner may select: the speculative-parse kernel (knob lz4_spec, sub-chunks <= 16 KiB;
    larger ones fall through to the split schedule), the split parse/copy kernel (knob lz4_split; lz4_split_g = 0
    automatic, 1, 2, 4, 8 sub-chunks per warp) and every lane-group width of the other schedules (knob
    lz4_lanes, lz4_split = 0)"""
    knobs = ("lz4_lanes", "lz4_split", "lz4_split_g", "lz4_spec")
    prev = {k: cdm.tune_get(k) for k in knobs}
    p = request.param
    cdm.tune_set("lz4_spec", 2 if p == "spec" else 0)
    if p == "spec":
        cdm.tune_set("lz4_split", 1)
        cdm.tune_set("lz4_split_g", 0)
    elif isinstance(p, str):
        cdm.tune_set("lz4_split", 1)
        cdm.tune_set("lz4_split_g", 0 if p == "split" else int(p[5:]))
    else:
        cdm.tune_set("lz4_split", 0)
        cdm.tune_set("lz4_lanes", p)
    yield p
    for k in knobs:
        cdm.tune_set(k, prev[k])


def test_lz4_lane_widths(engine, lz4_lanes):
    col = TPCH(0.01).column("l_comment")
    check_parity(engine, "Str|[LZ4(sub=4096),BitPack]", col, rows_per_chunk=30_001, both=False)


MIXED_CASES = [("l_comment", "Str|[LZ4(sub=16384,hc=9),BitPack]"), ("l_quantity", "Dict|BitPack"),
               ("l_shipmode", "Dict|BitPack"), ("l_orderkey", "RLE|[Delta|RLE|[BitPack,BitPack],BitPack]"),
               ("o_orderkey", "Delta|BitPack"), ("l_returnflag", "ANS"), ("o_comment", "Str|[StrDict|BitPack|ANS,BitPack]"),
               ("l_extendedprice", "Float2Int|BitPack")]


def mixed_batch_parity(engine, sf=0.01, rows_per_chunk=20_000, graph=False):
    """every kernel family in ONE device batch (one cdm_batch: all family streams, the phase schedule), each
    chunk's bytes and offsets against the oracle"""
    g = TPCH(sf)
    decs, exp = [], []
    for name, spec in MIXED_CASES:
        col = g.column(name)
        casc = cdm.Cascade(spec, col.dtype, col.width)
        for ch in encoder.encode_chunks(spec, col, rows_per_chunk):
            out, offs, info = _outputs(ch)
            decs.append(cdm.Decode(casc, cdm.pinned(ch), out, offs, dev_chunk=torch.from_numpy(ch).cuda()))
            exp.append((name, ch, out, offs, info))
    torch.cuda.synchronize()
    b = cdm.Batch(engine, decs)
    if graph:
        b.set_graph(True)
    stream = torch.cuda.Stream()
    for _ in range(2 if graph else 1):
        b.launch(stream)
        res = b.results(stream)
    b.close()
    torch.cuda.synchronize()
    for (name, ch, out, offs, info), r in zip(exp, res):
        e, eo = oracle.decode_chunk(ch)
        assert r["error_bits"] == 0, name
        assert np.array_equal(out.cpu().numpy()[: info["payload_bytes"]], e), name
        if eo is not None:
            assert np.array_equal(offs.cpu().numpy()[: eo.size], eo), name


def test_mixed_batch(engine):
    mixed_batch_parity(engine)
    mixed_batch_parity(engine, graph=True)


@pytest.mark.parametrize("env", [{"CDM_PHASES": "1"}, {"CDM_PHASES": "2"}, {"CDM_PHASES": "3"}, {"CDM_PHASES": "4"},
                                 {"CDM_SERIAL": "1"}, {"CDM_PDL": "0"}, {"CDM_RLE_PRIO": "hi"}])
def test_mixed_batch_phase_schedules(env):
    """every phase split of the batch schedule (CDM_PHASES; big batches use 2 by default, small ones one phase),
    the serial schedule, launches without programmatic dependencies and the RLE stream at high priority decode
    the same bytes (fresh process: the switches are read once)"""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, 'tests'); import test_gpu_parity as t; from paper_2602_08190_b200 import cdm; "
            "e = cdm.Engine(0); t.mixed_batch_parity(e); t.mixed_batch_parity(e, graph=True); print('ok')")
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True,
                       text=True, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]

def test_fp_pair_mapping_variant():
    """the opt-in pair-interleaved FP lane mapping (CDM_FP_PAIR=1) decodes the same rows (fresh process)"""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, 'tests'); import test_gpu_parity as t; from paper_2602_08190_b200 import cdm; "
            "from paper_2602_08190_b200.inputs import TPCH; e = cdm.Engine(0); g = TPCH(0.02); "
            "[t.check_parity(e, s, g.column(n), rows_per_chunk=50_001, both=False) for n, s in "
            "(('l_quantity', 'Dict|BitPack'), ('l_extendedprice', 'Float2Int|BitPack'), ('l_orderkey', 'BitPack'), "
            "('o_totalprice', 'Float2Int|BitPack'))]; print('ok')")
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, "CDM_FP_PAIR": "1"}, capture_output=True,
                       text=True, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_lz4_overlapping_matches(engine, lz4_lanes):
    from test_oracle_pins import _seq
    blocks, sizes = [], []
    for off, mlen in [(1, 4), (1, 300), (2, 19), (3, 1000), (5, 5), (7, 270), (31, 100), (32, 100), (33, 700)]:
        lit = bytes(range(65, 65 + off + 2))
        blocks.append(_seq(lit, off, mlen) + _seq(b"END", None, None))
        sizes.append(len(lit) + mlen + 3)
    payload = b"".join(blocks)
    tab = b""
    pos = 0
    for blk, dl in zip(blocks, sizes):
        tab += struct.pack("<III", pos, len(blk), dl)
        pos += len(blk)
    n = sum(sizes)
    lens = [n // 2, n - n // 2]
    spec = "Str|[LZ4,BitPack]"
    root = cdm1.Node(cdm1.STR, 2, [
        cdm1.Node(cdm1.LZ4, n, [cdm1.raw(payload), cdm1.raw(tab, eb=12)], nsub=len(blocks), sub=1 << 16),
        cdm1.bitpack(lens, 16, 0)])
    ch = cdm1.build(root, cdm1.VARBYTES, 1, 2, payload=n, cascade_hash=_hash(spec))
    check_parity(engine, spec, [ch], cdm.VARBYTES)


@pytest.mark.parametrize("spec", ["Str|[LZ4(sub=4096),BitPack]", "Str|[LZ4(sub=16384,hc=9),BitPack]",
                                  "Str|[LZ4(sub=65536,hc=12),BitPack]"])
def test_lz4_dependent_matches(engine, lz4_lanes, spec):
    """text built from a 6-word vocabulary, byte runs and long literal stretches: most matches are a few bytes
    to a few hundred bytes back, so the split kernel's matches depend on other lanes' matches of the same step
    (dependency rounds), short periods (< 16) are replicated, long literals and long matches cross 16-byte pieces"""
    rng = np.random.default_rng(77)
    words = [b"ab", b"abc ", b"the ", b"slyly ", b"x", b"carefully final "]
    parts = []
    for _ in range(12_000):
        r = rng.random()
        if r < 0.8:
            parts.append(words[rng.integers(0, len(words))])
        elif r < 0.9:
            parts.append(bytes([int(rng.integers(33, 127))]) * int(rng.integers(1, 300)))
        else:
            parts.append(rng.integers(0, 256, size=int(rng.integers(1, 200)), dtype=np.uint8).tobytes())
    data = np.frombuffer(b"".join(parts), dtype=np.uint8)
    cuts = np.sort(rng.choice(np.arange(1, data.size), size=2000, replace=False))
    offs = np.concatenate([[0], cuts, [data.size]]).astype(np.int64)
    col = Column("dep", VARBYTES, 1, offs.size - 1, data.copy(), offs)
    check_parity(engine, spec, col, rows_per_chunk=700, both=False)



def test_lz4_long_literals_and_incompressible(engine, lz4_lanes):
    """16 KiB sub-chunks whose compressed size exceeds the speculative kernel's shared input stage (random bytes:
    cl > 8 KiB, read through L1), literal runs longer than a parse segment (the true chain enters a segment past
    its end), and runs of one byte (period-1 matches of ~1 KiB)"""
    rng = np.random.default_rng(5)
    parts = []
    for _ in range(900):
        r = rng.random()
        if r < 0.3:
            parts.append(rng.integers(0, 256, size=int(rng.integers(500, 6000)), dtype=np.uint8).tobytes())
        elif r < 0.5:
            parts.append(bytes([int(rng.integers(0, 256))]) * int(rng.integers(4, 1500)))
        else:
            parts.append(b"furiously regular deposits " * int(rng.integers(1, 20)))
    data = np.frombuffer(b"".join(parts), dtype=np.uint8)
    cuts = np.sort(rng.choice(np.arange(1, data.size), size=300, replace=False))
    offs = np.concatenate([[0], cuts, [data.size]]).astype(np.int64)
    col = Column("lit", VARBYTES, 1, offs.size - 1, data.copy(), offs)
    for spec in ("Str|[LZ4(sub=16384),BitPack]", "Str|[LZ4(sub=16384,hc=9),BitPack]", "Str|[LZ4(sub=8000),BitPack]"):
        check_parity(engine, spec, col, rows_per_chunk=150, both=False)


def _stream_span(ch, i):
    nn = int(np.frombuffer(ch[6:8].tobytes(), np.uint16)[0])
    off, ln = struct.unpack_from("<QQ", ch.tobytes(), 64 + 32 * nn + 16 * i)
    return off, ln


def test_lz4_mutated_streams_match_oracle(engine, lz4_lanes):
    """byte mutations of valid LZ4 payloads (tokens, offsets, length extensions, literals): wherever the oracle
    rejects the chunk the GPU sets CDM_ERR_LZ4, wherever it decodes, the GPU's bytes equal the oracle's -- the
    speculative parse must find exactly the oracle's header chain even in garbage"""
    rng = np.random.default_rng(11)
    col = TPCH(0.002).column("l_comment")
    spec = "Str|[LZ4(sub=16384,hc=9),BitPack]"
    base = encoder.encode_chunks(spec, col, 3000)[:4]
    chunks = []
    for k in range(48):
        ch = base[k % len(base)].copy()
        off, ln = _stream_span(ch, 0)  # the LZ4 payload (first raw stream)
        for _ in range(int(rng.integers(1, 4))):
            pos = off + int(rng.integers(0, ln))
            ch[pos] = rng.integers(0, 256) if rng.random() < 0.7 else ch[pos] ^ (1 << int(rng.integers(0, 8)))
        chunks.append(ch)
    casc = cdm.Cascade(spec, VARBYTES)
    got = gpu_decode(engine, casc, chunks, resident=True, expect_error=True)
    n_err = 0
    for ch, (payload, offs, r) in zip(chunks, got):
        try:
            exp, _ = oracle.decode_chunk(ch)
        except oracle.OracleError:
            n_err += 1
            assert r["error_bits"] & cdm.ERR_LZ4, "oracle rejects the block, GPU did not flag it"
            continue
        assert r["error_bits"] == 0
        assert np.array_equal(payload, exp)
    assert 0 < n_err < len(chunks)

# ------------------------------------------------------------------------------ edge cases + corrupt data
def test_empty_and_tiny(engine):
    for n in (0, 1, 2, 31, 33):
        col = config1_column(n)
        check_parity(engine, "BitPack", col)
        check_parity(engine, "Delta|BitPack", col)
        check_parity(engine, "RLE|[BitPack,BitPack]", col)
    g = TPCH(0.0001)
    c = g.column("l_comment")
    empty = Column("e", cdm.VARBYTES, 1, 0, c.data[:0], c.offsets[:1] * 0)
    check_parity(engine, "Str|[LZ4,BitPack]", [encoder.encode("Str|[LZ4,BitPack]", empty)], cdm.VARBYTES)


def test_corrupt_dict_index_sets_error(engine):
    spec = "Dict|BitPack"
    root = cdm1.Node(cdm1.DICT, 5000, [cdm1.raw(np.arange(4, dtype=np.int64).tobytes(), eb=8),
                                       cdm1.bitpack([i % 5 for i in range(5000)], 3, 0)], entries=4, E=8)
    ch = cdm1.build(root, cdm1.I64, 8, 5000, cascade_hash=_hash(spec))
    casc = cdm.Cascade(spec, cdm.I64)
    for resident in (False, "pipeline", True):
        (_, _, r), = gpu_decode(engine, casc, [ch], resident=resident, expect_error=True)
        assert r["error_bits"] & cdm.ERR_DICT_INDEX


@pytest.mark.parametrize("E", [10, 15, 25])
def test_corrupt_char_dict_index_sets_error(engine, E):
    """CHAR(n) rows (row-group kernel, pre-shifted table): an index past the dictionary sets CDM_ERR_DICT_INDEX"""
    spec = "Dict|BitPack"
    words = np.frombuffer(b"".join(bytes([65 + k]) * E for k in range(4)), dtype=np.uint8)
    n = 9000
    root = cdm1.Node(cdm1.DICT, n, [cdm1.raw(words.tobytes(), eb=E),
                                    cdm1.bitpack([i % 5 for i in range(n)], 3, 0)], entries=4, E=E)
    ch = cdm1.build(root, cdm1.FIXED, E, n, cascade_hash=_hash(spec))
    casc = cdm.Cascade(spec, cdm1.FIXED, E)
    for resident in (False, True):
        (_, _, r), = gpu_decode(engine, casc, [ch], resident=resident, expect_error=True)
        assert r["error_bits"] & cdm.ERR_DICT_INDEX


def test_char_rows_plain_shared_dictionary_variant():
    """CDM_FPC_PRE=0 (fresh process): the TPC-H CHAR(n) columns through the plain shared dictionary copy"""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, 'tests'); import test_gpu_parity as t; from paper_2602_08190_b200 import cdm; "
            "from paper_2602_08190_b200.inputs import TPCH; e = cdm.Engine(0); g = TPCH(0.02); "
            "[t.check_parity(e, 'Dict|BitPack', g.column(n), rows_per_chunk=50_001, both=False) for n in "
            "('l_shipmode', 'l_shipinstruct', 'o_orderpriority')]; print('ok')")
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, "CDM_FPC_PRE": "0"}, capture_output=True,
                       text=True, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_corrupt_run_sum_sets_error(engine):
    spec = "RLE|[BitPack,BitPack]"
    for counts in ([3] * 4000, [3] * 4000 + [10 ** 6]):
        n = 12_001
        root = cdm1.Node(cdm1.RLE, n, [cdm1.bitpack(list(range(len(counts))), 20, 0),
                                       cdm1.bitpack(counts, 20, 0)], nruns=len(counts), maxrun=max(counts))
        ch = cdm1.build(root, cdm1.I64, 8, n, cascade_hash=_hash(spec))
        (payload, _, r), = gpu_decode(engine, cdm.Cascade(spec, cdm.I64), [ch], resident=True, expect_error=True)
        assert r["error_bits"] & cdm.ERR_RUN_SUM



# CHAR(n) dictionary rows (reading R14): every row width E -- the row-group kernel's widths (1, 2, 3, 10, 15,
# 25) and the generic byte path's (5, 7, 12, 31) -- with a tiny dictionary (shared-memory path), a large one
# (o_clerk-like, read through L1/L2) and an out-of-range index free column; ragged tails across several tiles.
@pytest.mark.parametrize("E", [1, 2, 3, 5, 7, 10, 12, 15, 25, 31])
@pytest.mark.parametrize("entries", [3, 7, 300, 2000])
def test_char_rows_every_width(engine, E, entries):
    """entries 3 / 7: the pre-shifted shared table (E >= 3), 300: the plain shared copy, 2000: read through L1"""
    rng = np.random.default_rng(E * 1000 + entries)
    words = rng.integers(32, 127, size=(entries, E), dtype=np.uint8)
    words = np.unique(words, axis=0)
    n = 3 * 8192 + 777
    data = words[rng.integers(0, words.shape[0], n)]
    col = Column("chr", cdm1.FIXED, E, n, np.ascontiguousarray(data))
    check_parity(engine, "Dict|BitPack", col, rows_per_chunk=20_011, both=False)


# A single symbol owns the whole ANS table (f = 2^tl): each decode step is the identity, no renormalisation
# word is read, and at tl = 12 the kernels decode it with tl = 11 (f = 2^12 does not fit their 12-bit f field).
# Also a near-degenerate two-symbol mix (f = 2^tl - 1 and 1) that exercises the widest f the field holds.
@pytest.mark.parametrize("spec", ["ANS", "ANS(il=1,chunk=4096)", "ANS(tl=10)", "ANS(il=1,tl=10,chunk=1024)"])
def test_ans_degenerate_tables(engine, spec):
    n = 100_003
    one = np.full((n, 1), 82, dtype=np.uint8)
    check_parity(engine, spec, Column("one", cdm1.FIXED, 1, n, one), rows_per_chunk=50_001)
    two = one.copy()
    two[np.random.default_rng(7).integers(0, n, 40), 0] = 65
    check_parity(engine, spec, Column("two", cdm1.FIXED, 1, n, two), rows_per_chunk=50_001)


@pytest.mark.parametrize("il", [1, 32])
def test_corrupt_ans_sets_error(engine, il):
    import test_ans_cpu as A
    data = np.random.default_rng(11).choice(np.array([65, 78, 82], np.uint8), 30000, p=[.25, .5, .25]).tobytes()
    good, _ = A.ans_chunk(data, 12, 4096, il=il)
    assert oracle.decode_chunk(good)[0].tobytes() == data
    casc = cdm.Cascade("ANS", cdm1.FIXED, 1)
    good[48:56] = np.frombuffer(struct.pack("<Q", _hash("ANS")), dtype=np.uint8)
    (payload, _, r), = gpu_decode(engine, casc, [good], resident=True)
    assert r["error_bits"] == 0 and payload.tobytes() == data
    for corrupt in ("word", "state", "truncate"):
        ch, _ = A.ans_chunk(data, 12, 4096, corrupt=corrupt, il=il)
        ch[48:56] = np.frombuffer(struct.pack("<Q", _hash("ANS")), dtype=np.uint8)
        (payload, _, r), = gpu_decode(engine, casc, [ch], resident=True, expect_error=True)
        assert r["error_bits"] & 0x20, corrupt


def test_varchar_offsets_scan_modes(engine, scan_mode):
    """VARCHAR offsets (exclusive scan + offsets[n]) over many tiles and a ragged tail, both schedules; a chunk
    whose lengths do not sum to its payload raises CDM_ERR_LENGTHS"""
    col = TPCH(0.01).column("l_comment")
    check_parity(engine, "Str|[LZ4,BitPack]", col, rows_per_chunk=40_961)
    lens = [7] * 9000
    n = sum(lens) + 1
    spec = "Str|[Raw,BitPack]"
    root = cdm1.Node(cdm1.STR, len(lens), [cdm1.raw(bytes(n)), cdm1.bitpack(lens, 3, 0)])
    ch = cdm1.build(root, cdm1.VARBYTES, 1, len(lens), payload=n, cascade_hash=_hash(spec))
    (_, _, r), = gpu_decode(engine, cdm.Cascade(spec, cdm.VARBYTES), [ch], resident=True, expect_error=True)
    assert r["error_bits"] & cdm.ERR_LENGTHS


def test_corrupt_lz4_sets_error(engine, lz4_lanes):
    from test_oracle_pins import _seq
    spec = "Str|[LZ4,BitPack]"
    for blk, dl in [(_seq(b"ABCDEFGH", 9, 4) + _seq(b"", None, None), 12),
                    (_seq(b"ABCDEFGH", 0, 4) + _seq(b"", None, None), 12),
                    (_seq(b"ABCDEFGH", 2, 40) + _seq(b"", None, None), 20)]:
        tab = struct.pack("<III", 0, len(blk), dl)
        root = cdm1.Node(cdm1.STR, 1, [cdm1.Node(cdm1.LZ4, dl, [cdm1.raw(blk), cdm1.raw(tab, eb=12)], nsub=1, sub=1 << 16),
                                       cdm1.bitpack([dl], 5, 0)])
        ch = cdm1.build(root, cdm1.VARBYTES, 1, 1, payload=dl, cascade_hash=_hash(spec))
        (_, _, r), = gpu_decode(engine, cdm.Cascade(spec, cdm.VARBYTES), [ch], resident=True, expect_error=True)
        assert r["error_bits"] & cdm.ERR_LZ4


def test_host_rejects_foreign_cascade(engine):
    col = config1_column(1000)
    ch = encoder.encode("Delta|BitPack", col)
    with pytest.raises(cdm.CdmError):
        gpu_decode(engine, cdm.Cascade("BitPack", cdm.I32), [ch])


# ------------------------------------------------------------------------------ pipeline invariance
def test_order_and_slots_do_not_change_bytes():
    """Pipelining changes time, never bytes: FIFO vs Johnson, 2 vs 6 slots."""
    col = TPCH(0.02).column("l_extendedprice")
    chunks = encoder.encode_chunks("Float2Int|BitPack", col, 10_000)
    ref = [oracle.decode_chunk(c)[0] for c in chunks]
    for order, slots in ((0, 2), (1, 6)):
        e = cdm.Engine(0, n_slots=slots, order_policy=order)
        got = gpu_decode(e, cdm.Cascade("Float2Int|BitPack", cdm.F64), chunks)
        e.close()
        for (p, _, _), r in zip(got, ref):
            assert np.array_equal(p, r)


def test_repeated_launches_graph_safe(engine):
    """The epoch|ticket counters survive repeated launches of one batch (and CUDA-graph replays)."""
    col = TPCH(0.05).column("l_orderkey")
    spec = "RLE|[Delta|RLE|[BitPack,BitPack],BitPack]"
    chunks = encoder.encode_chunks(spec, col, 100_000)
    casc = cdm.Cascade(spec, cdm.I64)
    decs, outs = [], []
    for ch in chunks:
        out, offs, _ = _outputs(ch)
        decs.append(cdm.Decode(casc, ch, out, offs, dev_chunk=torch.from_numpy(ch).cuda()))
        outs.append(out)
    b = cdm.Batch(engine, decs)
    s = torch.cuda.Stream()
    for _ in range(5):
        for o in outs:
            o.fill_(SENTINEL)
        b.launch(s)
        b.results(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        b.launch(s)
    for _ in range(3):
        for o in outs:
            o.fill_(SENTINEL)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        b.results(s)
        for ch, o in zip(chunks, outs):
            exp, _ = oracle.decode_chunk(ch)
            assert np.array_equal(o.cpu().numpy()[: exp.size], exp)
    b.close()


def test_pipeline_relaunch_and_error_positions(engine):
    """A captured pipeline re-copies and re-decodes on every launch; error words map back to job order."""
    g = TPCH(0.05)
    specs = [("l_orderkey", "RLE|[Delta|RLE|[BitPack,BitPack],BitPack]"), ("l_quantity", "Dict|BitPack"),
             ("l_comment", "Str|[LZ4,BitPack]"), ("l_extendedprice", "Float2Int|BitPack")]
    decs, outs, exps = [], [], []
    for name, spec in specs:
        col = g.column(name)
        casc = cdm.Cascade(spec, col.dtype, col.width)
        for ch in encoder.encode_chunks(spec, col, 120_000):
            out, offs, _ = _outputs(ch)
            decs.append(cdm.Decode(casc, cdm.pinned(ch), out, offs))
            outs.append((out, offs))
            exps.append(oracle.decode_chunk(ch))
    # a corrupt Dict chunk in the middle of the job list
    spec = "Dict|BitPack"
    root = cdm1.Node(cdm1.DICT, 5000, [cdm1.raw(np.arange(4, dtype=np.int64).tobytes(), eb=8),
                                       cdm1.bitpack([i % 5 for i in range(5000)], 3, 0)], entries=4, E=8)
    bad = cdm1.build(root, cdm1.I64, 8, 5000, cascade_hash=_hash(spec))
    bout, boffs, _ = _outputs(bad)
    k = len(decs) // 2
    decs.insert(k, cdm.Decode(cdm.Cascade(spec, cdm.I64), cdm.pinned(bad), bout, boffs))
    p = cdm.Pipeline(engine, decs)
    s = torch.cuda.Stream()
    for _ in range(3):
        for out, offs in outs:
            out.fill_(SENTINEL)
            if offs is not None:
                offs.fill_(-7)
        torch.cuda.synchronize()
        p.launch(s)
        res = p.results(raise_on_error=False)
        for i, r in enumerate(res):
            assert bool(r["error_bits"]) == (i == k), (i, r)
        j = 0
        for i in range(len(decs)):
            if i == k:
                continue
            (out, offs), (exp, exp_offs) = outs[j], exps[j]
            assert np.array_equal(out.cpu().numpy()[: exp.size], exp)
            if exp_offs is not None:
                assert np.array_equal(offs.cpu().numpy()[: exp_offs.size], exp_offs)
            j += 1
    with pytest.raises(cdm.CdmError):
        p.results()
    p.close()


# ------------------------------------------------------------------------------ every family in one graph
def test_all_families_one_batch_graph_and_timing(engine):
    """All 25 lineitem/orders cascades (config 4's map) in ONE device batch: FP, scan, RLE (two-level
    value lineage + big runs) and LZ4 run concurrently inside one captured graph; replays and the
    per-kernel timing mode (families serialised, events per launch) must not change a byte."""
    import bench
    g = TPCH(0.005)
    chunks_all, decs, bufs = [], [], []
    for name, spec in bench.WORKLOADS["config4"]["cols"]:
        col = g.column(name)
        casc = cdm.Cascade(spec, col.dtype, col.width)
        for ch in encoder.encode_chunks(spec, col, 9_999):
            out, offs, info = _outputs(ch)
            decs.append(cdm.Decode(casc, cdm.pinned(ch), out, offs, dev_chunk=torch.from_numpy(ch).cuda()))
            bufs.append((out, offs, info))
            chunks_all.append(ch)
    b = cdm.Batch(engine, decs)
    b.set_graph(True)
    stream = torch.cuda.Stream()
    for mode in (0, 1, 2, 0):
        b.set_timing(mode)
        for out, offs, _ in bufs:
            out.fill_(SENTINEL)
            if offs is not None:
                offs.fill_(-7)
        torch.cuda.synchronize()
        b.launch(stream)
        b.collect_timing()
        res = b.results(stream, raise_on_error=False)
        bad = [(i, r["error_bits"]) for i, r in enumerate(res) if r["error_bits"]]
        assert not bad, f"mode {mode}: error bits {bad}"
        for ch, (out, offs, info) in zip(chunks_all, bufs):
            exp, exp_offs = oracle.decode_chunk(ch)
            got = out.cpu().numpy()[: exp.size]
            assert np.array_equal(got, exp), f"mode {mode}: payload differs"
            if exp_offs is not None:
                assert np.array_equal(offs.cpu().numpy()[: exp_offs.size], exp_offs)
        if mode == 2:
            kt = b.kernel_times()
            for k in ("fp_kernel", "scan_kernel", "rle_sums_kernel", "rle_kernel(level0)", "rle_kernel",
                      "lz4_kernel"):
                assert kt[k][1] >= 1 and kt[k][0] > 0, k
        if mode == 1:
            km = b.kernel_ms()
            assert all(km[f][0] > 0 for f in ("fp", "scan", "rle", "lz4"))
    b.close()


# ------------------------------------------------------------------------------ H9 positional checksum
@pytest.mark.gpu
@pytest.mark.parametrize("name,spec", [("l_orderkey", "RLE|[DeltaStride|[Delta|RLE|[BitPack,BitPack],BitPack],BitPack]"),
                                       ("l_extendedprice", "Float2Int|BitPack"), ("l_shipmode", "Dict|BitPack"),
                                       ("o_comment", "Str|[StrDict|BitPack|ANS,BitPack]")])
def test_checksum_matches_oracle(engine, name, spec):
    """cdm_checksum of the device-decoded buffers == the oracle's checksum of its own decode."""
    col = TPCH(0.02).column(name)
    chunks = encoder.encode_chunks(spec, col, 50_001)
    casc = cdm.Cascade(spec, col.dtype, col.width)
    for ch in chunks:
        out, offs = cdm.output_buffers(ch)
        b = cdm.Batch(engine, [cdm.Decode(casc, ch, out, offs, dev_chunk=torch.from_numpy(ch).cuda())])
        b.launch()
        (r,) = b.results()
        b.close()
        cid = cdm.chunk_info(ch)["chunk_id"]
        exp, exp_offs = oracle.decode_chunk(ch)
        assert cdm.checksum(out[: exp.size], cid) == oracle.checksum(exp, cid)
        if exp_offs is not None:
            assert cdm.checksum(offs[: exp_offs.size], cid) == oracle.checksum(exp_offs, cid)
    # a misaligned pointer is rejected, not read
    with pytest.raises(cdm.CdmError):
        cdm.checksum(out[1:9], 0)


# ------------------------------------------------------------------------------ BASELINE full sizes
@pytest.mark.timeout(1200)
@pytest.mark.parametrize("workload", ["config3", "config4"])
def test_full_size_workload_every_chunk(engine, workload):
    """BASELINE configs 3 / 4 at SF 10 (config 3's full size; config 4's 25 columns at a tenth of the headline) in
    bench.py's launch configuration -- every chunk of the workload in ONE graph-mode device batch, decoded twice --
    with no device error bit, the H9 checksum of EVERY chunk equal to the oracle's checksum of the same chunk
    (oracle decodes on all host threads), and sampled chunks (first, last and two random per column) equal to the
    oracle byte for byte."""
    import random
    sys_path = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    import sys
    if sys_path not in sys.path:
        sys.path.insert(0, sys_path)
    import bench
    cols = bench.build_workload(0, workload, sf=10.0)
    decs, keep = [], []
    for name, spec, dtype, width, chunks, _ in cols:
        casc = cdm.Cascade(spec, dtype, width)
        for i, ch in enumerate(chunks):
            out, offs = cdm.output_buffers(ch)
            decs.append(cdm.Decode(casc, ch, out, offs, dev_chunk=torch.from_numpy(ch).cuda()))
            keep.append((name, i, len(chunks), ch, out, offs))
    b = cdm.Batch(engine, decs)
    b.set_graph(True)
    b.launch()
    res = b.results()
    b.launch()  # the replay bench.py times
    res = b.results()
    assert all(r["error_bits"] == 0 for r in res)
    torch.cuda.synchronize()
    # every chunk: device checksum == oracle checksum (payload under the chunk id, offsets under id ^ 2^63)
    gpu = []
    for name, i, _, ch, out, offs in keep:
        info = cdm.chunk_info(ch)
        cs = cdm.checksum(out[: info["payload_bytes"]], info["chunk_id"])
        if offs is not None:
            cs = (cs + cdm.checksum(offs, info["chunk_id"] ^ (1 << 63))) % (1 << 64)
        gpu.append(cs)
    threads = os.cpu_count() or 1
    for a in range(0, len(keep), 64):
        part = keep[a: a + 64]
        dec = oracle.decode_many([k[3] for k in part], nthreads=threads)
        for j, (k, (payload, offs)) in enumerate(zip(part, dec)):
            cid = int.from_bytes(k[3][56:64].tobytes(), "little")
            want = oracle.checksum(payload, cid)
            if offs is not None:
                want = (want + oracle.checksum(offs, cid ^ (1 << 63))) % (1 << 64)
            assert gpu[a + j] == want, f"{workload} {k[0]} chunk {k[1]}: checksum differs from the oracle's"
    rng = random.Random(7)
    by_col = {}
    for k in keep:
        by_col.setdefault(k[0], []).append(k)
    for name, ks in by_col.items():
        pick = {0, len(ks) - 1} | {rng.randrange(len(ks)) for _ in range(2)}
        for j in sorted(pick):
            _, i, _, ch, out, offs = ks[j]
            exp, exp_offs = oracle.decode_chunk(ch)
            got = out[: exp.size].cpu().numpy()
            assert np.array_equal(got, exp), f"{workload} {name} chunk {i}: payload differs"
            if exp_offs is not None:
                assert np.array_equal(offs[: exp_offs.size].cpu().numpy(), exp_offs), f"{name} chunk {i}: offsets"
    b.close()


@pytest.mark.parametrize("mode", ["submit", "pipeline"])
def test_contiguous_chunks_after_unaligned_total(engine, mode):
    """two host-contiguous chunks whose first total_bytes is NOT a multiple of 16 (a valid
    container: the header's total covers 8 trailing bytes) must not share one H2D copy -- the second chunk
    would land 8 bytes off a 16-byte boundary in the staging slot, where TMA and vector loads read it."""
    g = TPCH(0.002)
    spec = "Str|[LZ4,BitPack]"
    col = g.column("l_comment")
    a, b = encoder.encode_chunks(spec, col, 4000)[:2]
    a2 = np.concatenate([a, np.zeros(8, np.uint8)])
    struct.pack_into("<Q", a2, 40, a2.size)              # header total_bytes = 16k + 8
    host = cdm.pinned(np.concatenate([a2, b]))
    casc = cdm.Cascade(spec, col.dtype, col.width)
    parts = [host[: a2.size], host[a2.size:]]
    decs, bufs = [], []
    for ch in parts:
        out, offs, info = _outputs(ch.numpy())
        decs.append(cdm.Decode(casc, ch, out, offs))
        bufs.append((out, offs, info))
    if mode == "submit":
        res = [engine.wait(t) for t in engine.submit_batch(decs)]
    else:
        p = cdm.Pipeline(engine, decs)
        p.launch()
        res = p.results()
        p.close()
    torch.cuda.synchronize()
    for ch, (out, offs, info), r in zip((a2, b), bufs, res):
        assert r["error_bits"] == 0
        exp, exp_offs = oracle.decode_chunk(ch)
        assert np.array_equal(out[: exp.size].cpu().numpy(), exp)
        assert np.array_equal(offs[: exp_offs.size].cpu().numpy(), exp_offs)
