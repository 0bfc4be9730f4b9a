"""Encoder -> oracle round trip on TPC-H-shaped columns (generator == oracle(encode(generator))), plus the
encoder invariants of the north star: bit widths minimal and bounding the values, run lengths >= 1 and
maximal, dictionary indices < |dict|."""
import numpy as np
import pytest

import cdm1
import oracle
from paper_2602_08190_b200 import encoder
from paper_2602_08190_b200.inputs import TPCH, config1_column, rle_column, uniform_bits_column, I64

CASCADES = [
    ("l_orderkey", "RLE|[Delta|RLE|[BitPack,BitPack],BitPack]"),
    ("l_orderkey", "Delta|RLE|[BitPack,BitPack]"),
    ("l_orderkey", "Delta|BitPack"),
    ("l_partkey", "BitPack"),
    ("l_linenumber", "BitPack"),
    ("l_quantity", "Dict|BitPack"),
    ("l_discount", "Dict|BitPack"),
    ("l_tax", "Float2Int|BitPack"),
    ("l_extendedprice", "Float2Int|BitPack"),
    ("l_returnflag", "Dict|BitPack"),
    ("l_shipdate", "Dictionary encoding | Bit-packing"),
    ("l_shipinstruct", "Dict|BitPack"),
    ("l_shipmode", "Dict|BitPack"),
    ("l_comment", "Str|[LZ4,BitPack]"),
    ("l_comment", "Str|[LZ4(sub=4096),BitPack]"),
    ("l_comment", "Str|[LZ4(sub=16384,hc=9),BitPack]"),
    ("l_comment", "Str|[Raw,BitPack]"),
    ("o_orderkey", "Delta|RLE|[BitPack,BitPack]"),
    ("o_custkey", "BitPack"),
    ("o_clerk", "Dict|BitPack"),
    ("o_totalprice", "Float2Int|BitPack"),
    ("o_shippriority", "RLE|[BitPack,BitPack]"),
    ("o_comment", "Str|[LZ4,BitPack]"),
    ("o_orderdate", "RLE|[Dict|BitPack,BitPack]"),
    ("ps_partkey", "RLE|[DeltaStride|[BitPack,BitPack],RLE|[BitPack,BitPack]]"),  # Table 2 PS_PARTKEY (R35)
    ("ps_suppkey", "Delta|Dict|BitPack"),                                          # Table 2 PS_SUPPKEY (R36)
    ("ps_supplycost", "Float2Int|BitPack"),                                        # Table 2 PS_SUPPLYCOST
    ("ps_availqty", "BitPack"),
    ("ps_comment", "Str|[LZ4,BitPack]"),
]


def _check(col, chunks):
    dec = [oracle.decode_chunk(c) for c in chunks]
    payload = np.concatenate([d[0] for d in dec])
    assert np.array_equal(payload, col.data.reshape(-1).view(np.uint8))
    if col.offsets is not None:
        base, offs = 0, []
        for _, o in dec:
            offs.append(o[:-1].astype(np.int64) + base)
            base += int(o[-1])
        assert np.array_equal(np.concatenate(offs + [np.array([base])]), col.offsets)


@pytest.mark.parametrize("name,cascade", CASCADES)
def test_tpch_roundtrip(name, cascade):
    g = TPCH(0.01)
    col = g.column(name)
    _check(col, encoder.encode_chunks(cascade, col, 17_001))  # several ragged chunks


def _config4_cols():
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location("bench", os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    return bench.CONFIG4_COLS


@pytest.mark.parametrize("name,cascade", _config4_cols())
def test_config4_cascades_roundtrip(name, cascade):
    """the north-star workload's 25 columns under the exact cascades bench.py times (Table 2 mapped onto the
    hot-path codecs: DeltaStride order keys, ANS l_returnflag, String-dictionary|BitPack|ANS o_comment, ...):
    generator == oracle(encoder(generator)) over several ragged chunks"""
    g = TPCH(0.01)
    col = g.column(name)
    _check(col, encoder.encode_chunks(cascade, col, 23_017))


def test_ragged_and_empty():
    col = config1_column(1000)
    for rpc in (1, 7, 999, 1000, 5000):
        _check(col, encoder.encode_chunks("BitPack", col, rpc))
    empty = config1_column(0)
    ch = encoder.encode("BitPack", empty)
    out, _ = oracle.decode_chunk(ch)
    assert out.size == 0


@pytest.mark.parametrize("w", [0, 1, 7, 8, 13, 25, 31, 32, 33, 48, 63, 64])
def test_bitwidth_minimal_and_bounding(w):
    col = uniform_bits_column(5000, w)
    ch = encoder.encode("BitPack", col)
    h, nodes, streams = cdm1.parse(ch)
    assert nodes[0]["w"] == w  # both extremes are present, so w is forced
    v = col.data.view(np.uint64).astype(object)
    base = nodes[0]["base"]
    assert all(((int(x) - base) & ((1 << 64) - 1)) < (1 << w) or w == 64 for x in v[:200])
    _check(col, [ch])


@pytest.mark.parametrize("dist", ["even-1", "even-2", "even-64", "random-1-100", "outlier-1024-1",
                                  "mixed-even-4+random-1-32", "single"])
def test_rle_invariants(dist):
    col = rle_column(dist, 50_000, I64)
    ch = encoder.encode("RLE|[BitPack,BitPack]", col)
    _check(col, [ch])
    # decode the RLE children independently with numpy: counts >= 1, adjacent values differ, sum == n
    h, nodes, streams = cdm1.parse(ch)
    nr = nodes[0]["u32"][0]
    vals = _unpack(streams[0], nodes[1]["w"], nr) + nodes[1]["base"]
    cnts = _unpack(streams[1], nodes[3]["w"], nr) + nodes[3]["base"]
    assert cnts.min() >= 1 and int(cnts.sum()) == col.rows
    assert np.all(np.diff(vals) != 0)


def _unpack(b: bytes, w: int, n: int) -> np.ndarray:
    bits = np.unpackbits(np.frombuffer(b, np.uint8), bitorder="little")
    if w == 0:
        return np.zeros(n, dtype=np.int64)
    m = bits[: n * w].reshape(n, w).astype(np.int64)
    return (m << np.arange(w)).sum(axis=1)


def test_dict_indices_below_size():
    col = TPCH(0.01).column("l_shipdate")
    ch = encoder.encode("Dict|BitPack", col)
    h, nodes, streams = cdm1.parse(ch)
    entries = nodes[0]["u32"][0]
    idx = _unpack(streams[1], nodes[2]["w"], col.rows) + nodes[2]["base"]
    assert idx.max() < entries and (1 << (nodes[2]["w"] - 1)) < entries <= (1 << nodes[2]["w"])


def test_float2int_rejects_non_decimal():
    """SPEC.md:303 says pi is not representable; in IEEE doubles it is (pi == 3141592653589793/10^15
    rounds back to the same double, reading R13b).  1e-19 and 1e300 truly are not (d <= 18)."""
    from paper_2602_08190_b200.inputs import Column, F64
    for bad in ([0.5, 1e-19], [1e300]):
        col = Column("x", F64, 8, len(bad), np.array(bad))
        with pytest.raises(encoder.EncodeError):
            encoder.encode("Float2Int|BitPack", col)
    ok = encoder.encode("Float2Int|BitPack", Column("pi", F64, 8, 1, np.array([np.pi])))
    assert oracle.decode_chunk(ok)[0].view(np.float64)[0] == np.pi


@pytest.mark.parametrize("bad", ["RLE|[BitPack", "Bogus", "BitPack|[Raw,Raw]", "Dict|[BitPack,BitPack]", "LZ4|Raw"])
def test_cascade_grammar_errors(bad):
    with pytest.raises(encoder.EncodeError):
        encoder.canonical(bad)


def test_cascade_canonical_forms():
    assert encoder.canonical("Dictionary encoding | Bit-packing") == "DICT|[RAW,BITPACK|RAW]"
    assert encoder.canonical("RLE") == "RLE|[RAW,RAW]"
    assert encoder.canonical("RLE | [Bit-packing, Bit-packing]") == "RLE|[BITPACK|RAW,BITPACK|RAW]"


def test_partsupp_generator_shape():
    """partsupp (TPC-H 4.2.3): 4 rows per part, ps_partkey = part key, the 4 suppliers of a part distinct and in
    [1, S]; Table 2's PS_PARTKEY cascade keeps one DeltaStride run and one counts run per chunk of whole parts"""
    g = TPCH(0.05)
    pk = g.column("ps_partkey").data.astype(np.int64)
    sk = g.column("ps_suppkey").data.astype(np.int64)
    n = pk.size
    assert n == 4 * 10_000
    assert np.array_equal(pk, np.arange(n) // 4 + 1)
    S = 500
    assert sk.min() >= 1 and sk.max() <= S
    assert all(len(set(sk[4 * p: 4 * p + 4])) == 4 for p in range(0, n // 4, 97))
    col = g.column("ps_partkey")
    ch = encoder.encode_chunks("RLE|[DeltaStride|[BitPack,BitPack],RLE|[BitPack,BitPack]]", col, 20_000)
    assert len(ch) == 2 and all(c.size < 1024 for c in ch)  # 80 KB of keys -> a few hundred bytes per chunk
    _check(col, ch)
