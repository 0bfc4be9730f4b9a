"""Generator realism pins (PAPER.md facts + [ext] TPC-H rules) and determinism."""
import numpy as np

from paper_2602_08190_b200.inputs import TPCH, rle_counts, config1_column


def test_row_counts_and_lines_per_order():
    g = TPCH(0.1)
    assert g.rows(1) == 150_000
    ratio = g.rows(0) / g.rows(1)
    assert 3.95 < ratio < 4.05  # 1..7 lines per order, mean 4


def test_orderkey_counts_are_12_5_percent():
    # RLE count "only constitutes 12.5% of the original data" for int64 L_ORDERKEY;
    # with int32 counts that means runs/rows = 0.25.
    g = TPCH(0.1)
    k = g.column("l_orderkey").data
    runs = 1 + int(np.count_nonzero(np.diff(k)))
    assert abs(runs * 4 / (k.size * 8) - 0.125) < 0.002


def test_partkey_25_bits_at_sf100():
    # L_PARTKEY "compressed to a 25-bit width" at SF=100 (range 1..20,000,000)
    g = TPCH(100)
    pk = g.column("l_partkey", 0, 2_000_000).data.astype(np.int64)
    w = int(pk.max() - pk.min()).bit_length()
    assert w == 25 and pk.min() >= 1 and pk.max() <= 20_000_000


def test_cardinalities_and_ranges():
    g = TPCH(0.05)
    assert len(np.unique(g.column("l_shipmode").data, axis=0)) == 7
    assert len(np.unique(g.column("l_shipinstruct").data, axis=0)) == 4
    assert set(np.unique(g.column("l_returnflag").data).tobytes()) <= set(b"ARN")
    assert len(np.unique(g.column("l_quantity").data)) == 50
    assert len(np.unique(g.column("l_discount").data)) == 11
    assert len(np.unique(g.column("l_tax").data)) == 9
    sd = g.column("l_shipdate").data
    assert sd.min() >= 8035 + 1 and sd.max() <= 10591
    od = g.column("o_orderdate").data
    assert od.min() >= 8035 and od.max() <= 10440
    lens = np.diff(g.column("l_comment").offsets)
    assert lens.min() >= 10 and lens.max() <= 43


def test_row_ranges_are_independent():
    g = TPCH(0.02)
    for name in ("l_orderkey", "l_extendedprice", "l_comment", "o_totalprice"):
        full = g.column(name)
        n = full.rows
        a = g.column(name, 0, n // 3)
        b = g.column(name, n // 3, n - n // 3)
        if full.offsets is not None:
            assert np.array_equal(np.concatenate([a.data, b.data]), full.data)
        else:
            assert np.array_equal(np.concatenate([a.data, b.data]), full.data)


def test_rle_distributions_sum_to_n():
    for d in ("even-1", "even-2", "even-1024", "random-1-64", "outlier-1024-1", "mixed-even-4+random-1-32", "single"):
        c = rle_counts(d, 100_000)
        assert int(c.sum()) == 100_000 and c.min() >= 1


def test_config1_forces_w8():
    x = config1_column().data.astype(np.int64)
    assert int(x.max() - x.min()).bit_length() == 8
