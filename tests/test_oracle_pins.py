"""Pin the CPU oracle to things other than itself (-m "not gpu").

Each test constructs chunks WITHOUT the encoder (tests/cdm1.py hand-assembles streams from the plain
definitions or golden bytes) and checks the oracle's decode against: golden vectors printed in
SPEC/SURVEY (tests/golden/), library routines (numpy repeat/cumsum/take, liblz4), exact rational
arithmetic (fractions), brute force over every bit width, and invariants.  A plausible mistake in the
oracle (dropped FOR term, MSB-first bits, off-by-one delta, swapped RLE children, wrong LZ4 offset
direction) fails at least one of these.
"""
import ctypes
import struct
from fractions import Fraction

import numpy as np
import pytest

import cdm1
import oracle
from oracle import OracleError

MASK64 = (1 << 64) - 1


def dec(chunk):
    return oracle.decode_chunk(chunk)


def as_i64(payload):
    return payload.view(np.int64)


# ----------------------------------------------------------------------------- golden vectors

def test_golden_spec_bitpack(golden):
    g = golden("spec_bitpack.json")
    bp = g["bitpack"]
    assert cdm1.pack_bits(bp["fields"], bp["w"]).hex() == bp["bytes"]
    root = cdm1.Node(cdm1.BITPACK, 4, [cdm1.raw(bytes.fromhex(bp["bytes"]))], w=bp["w"], base=bp["for"])
    out, _ = dec(cdm1.build(root, cdm1.I32, 4, 4))
    assert out.view(np.int32).tolist() == g["column"]


def test_golden_orderkey_nested(golden):
    g = golden("orderkey_nested.json")
    iv, ic, oc = g["bitpack_inner_values"], g["bitpack_inner_counts"], g["bitpack_outer_counts"]
    inner = cdm1.Node(cdm1.RLE, 10, [
        cdm1.Node(cdm1.BITPACK, 4, [cdm1.raw(bytes.fromhex(iv["bytes"]))], w=iv["w"], base=iv["for"]),
        cdm1.Node(cdm1.BITPACK, 4, [cdm1.raw(bytes.fromhex(ic["bytes"]))], w=ic["w"], base=ic["for"])],
        nruns=4, maxrun=7)
    delta = cdm1.Node(cdm1.DELTA, 10, [inner], base=g["delta_base"])
    root = cdm1.Node(cdm1.RLE, 20, [
        delta, cdm1.Node(cdm1.BITPACK, 10, [cdm1.raw(bytes.fromhex(oc["bytes"]))], w=oc["w"], base=oc["for"])],
        nruns=10, maxrun=4)
    out, _ = dec(cdm1.build(root, cdm1.I64, 8, 20))
    assert as_i64(out).tolist() == g["column"]
    # the intermediate streams are what the paper's definitions say they are
    assert np.repeat(g["inner_values"], g["inner_counts"]).tolist() == g["deltas"]
    assert (g["delta_base"] + np.cumsum(g["deltas"])).tolist() == g["outer_values"]
    assert np.repeat(g["outer_values"], g["outer_counts"]).tolist() == g["column"]


def test_golden_orderkey_literal(golden):
    g = golden("orderkey_literal.json")
    bv, bc = g["bitpack_values"], g["bitpack_counts"]
    rle = cdm1.Node(cdm1.RLE, 20, [
        cdm1.Node(cdm1.BITPACK, 12, [cdm1.raw(bytes.fromhex(bv["bytes"]))], w=bv["w"], base=bv["for"]),
        cdm1.Node(cdm1.BITPACK, 12, [cdm1.raw(bytes.fromhex(bc["bytes"]))], w=bc["w"], base=bc["for"])],
        nruns=12, maxrun=3)
    root = cdm1.Node(cdm1.DELTA, 20, [rle], base=g["delta_base"])
    out, _ = dec(cdm1.build(root, cdm1.I64, 8, 20))
    assert as_i64(out).tolist() == g["column"]


def test_golden_shipmode_dict(golden):
    g = golden("shipmode_dict.json")
    W = g["width"]
    dictionary = b"".join(s.encode().ljust(W) for s in g["dictionary"])
    bi = g["bitpack_indices"]
    root = cdm1.Node(cdm1.DICT, 5, [
        cdm1.raw(dictionary, eb=W),
        cdm1.Node(cdm1.BITPACK, 5, [cdm1.raw(bytes.fromhex(bi["bytes"]))], w=bi["w"], base=bi["for"])],
        entries=len(g["dictionary"]), E=W)
    out, _ = dec(cdm1.build(root, cdm1.FIXED, W, 5))
    rows = [bytes(out[i * W:(i + 1) * W]).decode() for i in range(5)]
    assert rows == [s.ljust(W) for s in g["rows"]]


def test_spec_examples(golden):
    g = golden("spec_examples.json")
    # Delta: base 10, deltas [0,1,2] -> [10,11,13]
    d = g["delta"]
    root = cdm1.Node(cdm1.DELTA, 3, [cdm1.bitpack(d["deltas"], 2, 0)], base=d["base"])
    assert as_i64(dec(cdm1.build(root, cdm1.I64, 8, 3))[0]).tolist() == d["column"]
    # RLE
    r = g["rle"]
    root = cdm1.Node(cdm1.RLE, 5, [cdm1.bitpack(r["values"], 2, 7), cdm1.bitpack(r["counts"], 1, 2)], nruns=2, maxrun=3)
    assert as_i64(dec(cdm1.build(root, cdm1.I64, 8, 5))[0]).tolist() == r["column"]
    # Float2Int
    f = g["float2int"]
    root = cdm1.Node(cdm1.FLOAT2INT, 3, [cdm1.bitpack(f["ints"], 3, 0)], d=f["d"])
    assert dec(cdm1.build(root, cdm1.F64, 8, 3))[0].view(np.float64).tolist() == f["column"]
    # Prefix sum through the Str root: lengths [3,2,4] -> offsets [0,3,5,9]
    p = g["prefix"]
    root = cdm1.Node(cdm1.STR, 3, [cdm1.raw(b"abcdefghi"), cdm1.bitpack(p["counts"], 2, 2)])
    payload, offs = dec(cdm1.build(root, cdm1.VARBYTES, 1, 3, payload=9))
    assert offs.tolist() == p["offsets"] and bytes(payload) == b"abcdefghi"


# ----------------------------------------------------------------------------- BitPack + FOR brute force

@pytest.mark.parametrize("w", list(range(0, 65)))
def test_bitpack_every_width(w):
    rng = np.random.default_rng(w)
    for n in (0, 1, 2, 3, 7, 31, 32, 33, 65, 1023, 1025):
        if w == 0:
            fields = [0] * n
        else:
            fields = [int(x) for x in rng.integers(0, 1 << min(w, 62), size=n, dtype=np.uint64)]
            if w > 62:
                fields = [(f << (w - 62)) | int(rng.integers(0, 1 << (w - 62))) for f in fields]
            if n >= 2:
                fields[0], fields[-1] = 0, (1 << w) - 1
        base = int(rng.integers(-(1 << 62), 1 << 62))
        root = cdm1.Node(cdm1.BITPACK, n, [cdm1.raw(cdm1.pack_bits(fields, w))], w=w, base=base)
        out64, _ = dec(cdm1.build(root, cdm1.I64, 8, n))
        expect = [(base + f) & MASK64 for f in fields]
        assert out64.view(np.uint64).tolist() == expect
        out32, _ = dec(cdm1.build(root, cdm1.I32, 4, n))
        assert out32.view(np.uint32).tolist() == [e & 0xFFFFFFFF for e in expect]


def test_bitpack_short_stream_is_corrupt():
    root = cdm1.Node(cdm1.BITPACK, 9, [cdm1.raw(b"\xff")], w=1, base=0)  # 9 bits need 2 bytes
    with pytest.raises(OracleError):
        dec(cdm1.build(root, cdm1.I64, 8, 9))


# ----------------------------------------------------------------------------- Dict (np.take)

@pytest.mark.parametrize("E", [1, 4, 8, 10, 15, 25])
def test_dict_matches_np_take(E):
    rng = np.random.default_rng(E)
    entries, n = 37, 1000
    dictionary = rng.integers(0, 256, size=(entries, E), dtype=np.uint8)
    idx = rng.integers(0, entries, size=n)
    root = cdm1.Node(cdm1.DICT, n, [cdm1.raw(dictionary.tobytes(), eb=E), cdm1.bitpack(idx, 6, 0)], entries=entries, E=E)
    out, _ = dec(cdm1.build(root, cdm1.FIXED, E, n))
    assert np.array_equal(out.reshape(n, E), np.take(dictionary, idx, axis=0))


def test_dict_index_out_of_range():
    root = cdm1.Node(cdm1.DICT, 3, [cdm1.raw(b"\x01\x02", eb=1), cdm1.bitpack([0, 2, 1], 2, 0)], entries=2, E=1)
    with pytest.raises(OracleError, match="row 1"):
        dec(cdm1.build(root, cdm1.FIXED, 1, 3))


# ----------------------------------------------------------------------------- Float2Int (exact rationals)

def test_float2int_is_correctly_rounded_decimal():
    rng = np.random.default_rng(5)
    for d in (0, 1, 2, 3, 6, 9):
        ints = [int(x) for x in rng.integers(-(10 ** 12), 10 ** 12, size=400)] + [0, 1, -1, 10 ** 12]
        base = min(ints)
        w = (max(ints) - base).bit_length()
        root = cdm1.Node(cdm1.FLOAT2INT, len(ints), [cdm1.bitpack(ints, w, base)], d=d)
        out, _ = dec(cdm1.build(root, cdm1.F64, 8, len(ints)))
        # Fraction -> float is correctly rounded: exactly what one IEEE division of exact operands gives
        assert out.view(np.float64).tolist() == [float(Fraction(q, 10 ** d)) for q in ints]


def test_float2int_cents_identity():
    """Closed form: every cent amount c in the TPC-H range decodes to the double nearest c/100."""
    c = np.arange(0, 10_500_001, 997, dtype=np.int64)
    root = cdm1.Node(cdm1.FLOAT2INT, len(c), [cdm1.bitpack(c, 24, 0)], d=2)
    out, _ = dec(cdm1.build(root, cdm1.F64, 8, len(c)))
    assert out.view(np.float64).tolist() == [float(Fraction(int(x), 100)) for x in c]


# ----------------------------------------------------------------------------- Delta (np.cumsum mod 2^64)

def test_delta_matches_wrapping_cumsum():
    rng = np.random.default_rng(6)
    n = 5000
    deltas = rng.integers(-(1 << 40), 1 << 40, size=n)
    deltas[0] = 0
    base = int(rng.integers(-(1 << 62), 1 << 62))
    w = int(deltas.max() - deltas.min()).bit_length()
    root = cdm1.Node(cdm1.DELTA, n, [cdm1.bitpack(deltas, w, int(deltas.min()))], base=base)
    out, _ = dec(cdm1.build(root, cdm1.I64, 8, n))
    expect = (np.uint64(base & MASK64) + np.cumsum(deltas.astype(np.uint64)))  # numpy uint64 wraps mod 2^64
    assert np.array_equal(out.view(np.uint64), expect)
    out32, _ = dec(cdm1.build(root, cdm1.I32, 4, n))
    assert np.array_equal(out32.view(np.uint32), expect.astype(np.uint32))


# ----------------------------------------------------------------------------- RLE (np.repeat)

@pytest.mark.parametrize("seed", range(4))
def test_rle_matches_np_repeat(seed):
    rng = np.random.default_rng(seed)
    nr = 300
    counts = rng.integers(0 if seed == 3 else 1, 50, size=nr)  # seed 3: zero-length runs (foreign encoder)
    values = rng.integers(0, 1 << 30, size=nr)
    n = int(counts.sum())
    root = cdm1.Node(cdm1.RLE, n, [cdm1.bitpack(values, 30, 0), cdm1.bitpack(counts, 6, 0)], nruns=nr,
                     maxrun=int(counts.max()))
    out, _ = dec(cdm1.build(root, cdm1.I64, 8, n))
    assert np.array_equal(as_i64(out), np.repeat(values, counts))


def test_rle_even2_shape():
    # "even-2 yields an uncompressed sequence such as A-A-B-B-C-C"
    root = cdm1.Node(cdm1.RLE, 6, [cdm1.raw(b"ABC", eb=1), cdm1.bitpack([2, 2, 2], 0, 2)], nruns=3, maxrun=2)
    out, _ = dec(cdm1.build(root, cdm1.FIXED, 1, 6))
    assert bytes(out) == b"AABBCC"


def test_rle_count_sum_mismatch():
    for counts in ([3, 1], [3, 3]):  # sum 4 < 5 and 6 > 5
        root = cdm1.Node(cdm1.RLE, 5, [cdm1.bitpack([7, 9], 2, 7), cdm1.bitpack(counts, 2, 1)], nruns=2, maxrun=3)
        with pytest.raises(OracleError, match="run"):
            dec(cdm1.build(root, cdm1.I64, 8, 5))


# ----------------------------------------------------------------------------- DeltaStride (closed forms)
# PAPER.md:481 "(start, stride, count) triples"; reading R9 (children [starts, counts], one stride).

def _dstride(starts, counts, stride, wst=20, wc=8, rows=None):
    n = int(np.sum(counts)) if rows is None else rows
    return cdm1.Node(cdm1.DSTRIDE, n, [cdm1.bitpack(starts, wst, int(min(starts)) if len(starts) else 0),
                                       cdm1.bitpack(counts, wc, 0)],
                     nruns=len(starts), maxrun=int(max(counts)) if len(counts) else 0, stride=stride)


def test_dstride_spec_example():
    # SPEC.md:279's column [10,11,12,20,22,24]: with stride 1 the greedy runs are (10,3),(20,1),(22,1),(24,1);
    # with stride 2, (10,1),(11,1),(12,1),(20,3)
    for starts, counts, stride in (([10, 20, 22, 24], [3, 1, 1, 1], 1), ([10, 11, 12, 20], [1, 1, 1, 3], 2)):
        out, _ = dec(cdm1.build(_dstride(starts, counts, stride), cdm1.I64, 8, 6))
        assert as_i64(out).tolist() == [10, 11, 12, 20, 22, 24]


def test_dstride_tpch_orderkeys_closed_form():
    # TPC-H sparse order keys (first 8 of every 32): key(o) = 32*(o div 8) + (o mod 8) + 1 -- triples
    # (32q + 1, 1, 8); a chunk starting mid-group has a short first run
    o0, n = 5, 8 * 40 + 3
    o = np.arange(o0, o0 + n)
    keys = 32 * (o // 8) + (o % 8) + 1
    starts, counts, g = [], [], o0
    while g < o0 + n:
        k = min(8 - g % 8, o0 + n - g)
        starts.append(int(32 * (g // 8) + g % 8 + 1)); counts.append(k); g += k
    out, _ = dec(cdm1.build(_dstride(starts, counts, 1, wst=14, wc=4), cdm1.I64, 8, n))
    assert np.array_equal(as_i64(out), keys)


@pytest.mark.parametrize("stride", [0, 3, -7, (1 << 63) + 5])
def test_dstride_arithmetic_runs(stride):
    rng = np.random.default_rng(11)
    nr = 200
    counts = rng.integers(0, 40, size=nr)
    starts = rng.integers(0, 1 << 40, size=nr)
    n = int(counts.sum())
    out, _ = dec(cdm1.build(_dstride(list(starts), list(counts), stride, wst=41, wc=6), cdm1.I64, 8, n))
    exp = [(int(s) + j * stride) & MASK64 for s, c in zip(starts, counts) for j in range(int(c))]
    assert [int(x) & MASK64 for x in as_i64(out)] == exp
    # stride 0 is plain RLE (np.repeat)
    if stride == 0:
        assert np.array_equal(as_i64(out), np.repeat(starts, counts))


def test_dstride_under_rle_and_delta():
    # Table 2 L_ORDERKEY shape: RLE | [DeltaStride | [Delta | RLE | [BP, BP], BP], BP]
    # starts 1, 33, 65, 97 = Delta(base 1) of RLE(value 32 x 3 after a leading 0); counts 8 each
    inner = cdm1.Node(cdm1.RLE, 4, [cdm1.bitpack([0, 32], 6, 0), cdm1.bitpack([1, 3], 2, 0)], nruns=2, maxrun=3)
    starts = cdm1.Node(cdm1.DELTA, 4, [inner], base=1)
    ds = cdm1.Node(cdm1.DSTRIDE, 32, [starts, cdm1.bitpack([8, 8, 8, 8], 0, 8)], nruns=4, maxrun=8, stride=1)
    lines = [1 + (k % 7) for k in range(32)]
    root = cdm1.Node(cdm1.RLE, sum(lines), [ds, cdm1.bitpack(lines, 3, 0)], nruns=32, maxrun=7)
    out, _ = dec(cdm1.build(root, cdm1.I64, 8, sum(lines)))
    keys = [32 * (o // 8) + (o % 8) + 1 for o in range(32)]
    assert as_i64(out).tolist() == np.repeat(keys, lines).tolist()


def test_dstride_count_mismatch_and_arity():
    for counts in ([3, 1], [3, 3]):
        root = cdm1.Node(cdm1.DSTRIDE, 5, [cdm1.bitpack([7, 9], 2, 7), cdm1.bitpack(counts, 2, 1)], nruns=2, maxrun=3,
                         stride=1)
        with pytest.raises(OracleError, match="run"):
            dec(cdm1.build(root, cdm1.I64, 8, 5))
    root = cdm1.Node(cdm1.DSTRIDE, 2, [cdm1.bitpack([7, 9], 2, 7)], nruns=2, maxrun=1, stride=1)
    with pytest.raises(OracleError, match="2 children"):
        dec(cdm1.build(root, cdm1.I64, 8, 2))


# ----------------------------------------------------------------------------- String-dictionary
# PAPER.md:163 / 498 (tokens on spaces and periods, each token a group expanded from the dictionary);
# DESIGN.md reading R34 (dictionary = u32 offsets[E+1] + token bytes).  The tokenizer below is test-local.

def _tokens(s: bytes):
    out, k = [], 0
    for i in range(1, len(s) + 1):
        if i == len(s) or (s[i] not in b" ." and s[i - 1] in b" ."):
            out.append(s[k:i]); k = i
    return out


def _strdict_chunk(strings, ids_w=None, order=None):
    toks = [t for s in strings for t in _tokens(s)]
    vocab = order or list(dict.fromkeys(toks))
    ids = [vocab.index(t) for t in toks]
    offs = np.concatenate([[0], np.cumsum([len(t) for t in vocab])]).astype(np.uint32)
    blob = offs.tobytes() + b"".join(vocab)
    n = sum(len(s) for s in strings)
    w = ids_w if ids_w is not None else max(1, (len(vocab) - 1).bit_length())
    sd = cdm1.Node(cdm1.STRDICT, n, [cdm1.raw(blob), cdm1.bitpack(ids, w, 0)], entries=len(vocab),
                   E=int(offs[-1]))
    lens = [len(s) for s in strings]
    root = cdm1.Node(cdm1.STR, len(strings), [sd, cdm1.bitpack(lens, max(1, max(lens).bit_length()), 0)])
    return cdm1.build(root, cdm1.VARBYTES, 0, len(strings), payload=n), vocab, ids


def test_strdict_spec_example():
    # "a b. a " -> tokens "a ", "b. ", "a " (dictionary of 2 unique tokens, ids 0 1 0)
    ch, vocab, ids = _strdict_chunk([b"a b. a "])
    assert vocab == [b"a ", b"b. "] and ids == [0, 1, 0]
    out, offs = dec(ch)
    assert bytes(out) == b"a b. a " and offs.tolist() == [0, 7]


def test_strdict_reconstructs_strings():
    rng = np.random.default_rng(3)
    words = [b"furiously", b"slyly", b"ironic", b"deposits", b"packages", b"", b"x"]
    strings = []
    for _ in range(400):
        k = int(rng.integers(0, 9))
        s = b"".join(words[int(rng.integers(len(words)))] + (b". " if rng.random() < 0.2 else b" ") for _ in range(k))
        strings.append(s[: int(rng.integers(0, len(s) + 1))] if rng.random() < 0.3 else s)
    strings.append(b"")
    ch, vocab, _ = _strdict_chunk([s for s in strings] + [b"trailing"])
    out, offs = dec(ch)
    allb = b"".join(strings) + b"trailing"
    assert bytes(out) == allb
    assert offs.tolist() == np.concatenate([[0], np.cumsum([len(s) for s in strings] + [8])]).tolist()
    # a permuted dictionary with the ids remapped decodes to the same bytes (ids index, not order)
    perm = vocab[::-1]
    ch2, _, _ = _strdict_chunk([s for s in strings] + [b"trailing"], order=perm)
    assert bytes(dec(ch2)[0]) == allb


def test_strdict_errors():
    ch, vocab, ids = _strdict_chunk([b"a b. a "], ids_w=2)
    # id 3 >= 2 entries
    sd = cdm1.Node(cdm1.STRDICT, 7, [cdm1.raw(np.array([0, 2, 5], np.uint32).tobytes() + b"a b. "),
                                     cdm1.bitpack([0, 3, 0], 2, 0)], entries=2, E=5)
    root = cdm1.Node(cdm1.STR, 1, [sd, cdm1.bitpack([7], 3, 0)])
    with pytest.raises(OracleError, match="out of range"):
        dec(cdm1.build(root, cdm1.VARBYTES, 0, 1, payload=7))
    # tokens total 5 bytes != 7
    sd = cdm1.Node(cdm1.STRDICT, 7, [cdm1.raw(np.array([0, 2, 5], np.uint32).tobytes() + b"a b. "),
                                     cdm1.bitpack([0, 1], 1, 0)], entries=2, E=5)
    root = cdm1.Node(cdm1.STR, 1, [sd, cdm1.bitpack([7], 3, 0)])
    with pytest.raises(OracleError, match="token bytes"):
        dec(cdm1.build(root, cdm1.VARBYTES, 0, 1, payload=7))
    # decreasing dictionary offsets
    sd = cdm1.Node(cdm1.STRDICT, 7, [cdm1.raw(np.array([0, 4, 2], np.uint32).tobytes() + b"a b"),
                                     cdm1.bitpack([0, 1], 1, 0)], entries=2, E=3)
    root = cdm1.Node(cdm1.STR, 1, [sd, cdm1.bitpack([7], 3, 0)])
    with pytest.raises(OracleError, match="offsets"):
        dec(cdm1.build(root, cdm1.VARBYTES, 0, 1, payload=7))


# ----------------------------------------------------------------------------- LZ4 (liblz4 + hand sequences)

_lz4 = ctypes.CDLL("liblz4.so.1")
_lz4.LZ4_compress_default.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_int]


def lz4_compress(data: bytes) -> bytes:
    cap = len(data) + len(data) // 255 + 64
    dst = ctypes.create_string_buffer(cap)
    k = _lz4.LZ4_compress_default(data, dst, len(data), cap)
    assert k > 0
    return dst.raw[:k]


def lz4_chunk(blocks: list[bytes], sizes: list[int], sub: int) -> np.ndarray:
    payload = b"".join(blocks)
    tab = b""
    pos = 0
    for blk, dl in zip(blocks, sizes):
        tab += struct.pack("<III", pos, len(blk), dl)
        pos += len(blk)
    n = sum(sizes)
    lz = cdm1.Node(cdm1.LZ4, n, [cdm1.raw(payload), cdm1.raw(tab, eb=12)], nsub=len(blocks), sub=sub)
    return cdm1.build(lz, cdm1.FIXED, 1, n)


@pytest.mark.parametrize("kind", ["text", "random", "zeros", "mixed"])
def test_lz4_decodes_liblz4_output(kind):
    rng = np.random.default_rng(8)
    if kind == "text":
        words = [b"foxes ", b"sleep ", b"carefully ", b"among the ", b"ideas. ", b"quick "]
        data = b"".join(words[i] for i in rng.integers(0, len(words), size=20000))
    elif kind == "random":
        data = rng.integers(0, 256, size=100000, dtype=np.uint8).tobytes()
    elif kind == "zeros":
        data = bytes(70000)
    else:
        data = bytes(3000) + rng.integers(0, 4, size=50000, dtype=np.uint8).tobytes() + b"xyz" * 5000
    sub = 65536
    parts = [data[i:i + sub] for i in range(0, len(data), sub)]
    out, _ = dec(lz4_chunk([lz4_compress(p) for p in parts], [len(p) for p in parts], sub))
    assert bytes(out) == data


def test_lz4_brute_force_short_strings():
    import itertools
    for L in range(0, 9):
        for t in itertools.product(b"ab", repeat=L):
            s = bytes(t)
            out, _ = dec(lz4_chunk([lz4_compress(s)], [len(s)], 64))
            assert bytes(out) == s


def _seq(lit: bytes, off: int | None, mlen: int | None) -> bytes:
    """Hand-assembled LZ4 sequence (block format [ext]); mlen >= 4 or None for the last literals-only one."""
    ll = len(lit)
    tok_l = min(ll, 15)
    ml = 0 if mlen is None else mlen - 4
    tok_m = min(ml, 15)
    out = bytes([(tok_l << 4) | tok_m])
    if ll >= 15:
        r = ll - 15
        while r >= 255:
            out += b"\xff"
            r -= 255
        out += bytes([r])
    out += lit
    if mlen is None:
        return out
    out += struct.pack("<H", off)
    if ml >= 15:
        r = ml - 15
        while r >= 255:
            out += b"\xff"
            r -= 255
        out += bytes([r])
    return out


@pytest.mark.parametrize("off,mlen", [(1, 4), (1, 300), (2, 19), (3, 1000), (5, 5), (7, 270)])
def test_lz4_overlapping_matches(off, mlen):
    lit = bytes(range(65, 65 + max(off, 1) + 2))
    blk = _seq(lit, off, mlen) + _seq(b"END", None, None)
    expect = bytearray(lit)
    for _ in range(mlen):  # the definition: copy forward from `off` bytes back, one byte at a time
        expect.append(expect[-off])
    expect += b"END"
    out, _ = dec(lz4_chunk([blk], [len(expect)], 1 << 16))
    assert bytes(out) == bytes(expect)


@pytest.mark.parametrize("bad", ["offset0", "offset_far", "overrun", "short"])
def test_lz4_corrupt_blocks(bad):
    lit = b"ABCDEFGH"
    if bad == "offset0":
        blk, n = _seq(lit, 0, 4) + _seq(b"", None, None), 12
    elif bad == "offset_far":
        blk, n = _seq(lit, 9, 4) + _seq(b"", None, None), 12
    elif bad == "overrun":
        blk, n = _seq(lit, 2, 40) + _seq(b"", None, None), 20
    else:
        blk, n = _seq(lit, 2, 4)[:-1], 12
    with pytest.raises(OracleError):
        dec(lz4_chunk([blk], [n], 1 << 16))


# ----------------------------------------------------------------------------- container robustness

def _sample_chunks():
    from paper_2602_08190_b200 import encoder
    from paper_2602_08190_b200.inputs import Column, I64, VARBYTES
    col = np.array([1, 1, 1, 2, 2, 3, 4, 4, 4, 4, 5, 6, 6, 7, 8, 8, 33, 33, 33, 34], dtype=np.int64)
    a = encoder.encode("RLE|[Delta|RLE|[BitPack,BitPack],BitPack]", Column("k", I64, 8, 20, col))
    s = b"the quick brown fox jumps over the lazy dog"
    offs = np.array([0, 4, 10, 16, 20, 26, 31, 35, 40, len(s)], dtype=np.int64)
    b = encoder.encode("Str|[LZ4,BitPack]", Column("c", VARBYTES, 1, 9, np.frombuffer(s, np.uint8), offs))
    return [a, b]


def test_truncation_at_every_byte_fails_cleanly():
    for ch in _sample_chunks():
        dec(ch)
        for cut in range(ch.size):
            with pytest.raises(OracleError):
                dec(ch[:cut].copy())


def test_bad_magic_and_version():
    ch = _sample_chunks()[0]
    bad = ch.copy()
    bad[0] ^= 0xFF
    with pytest.raises(OracleError, match="magic"):
        dec(bad)
    bad = ch.copy()
    bad[4] = 9
    with pytest.raises(OracleError, match="version"):
        dec(bad)


def test_flipped_bytes_never_crash():
    rng = np.random.default_rng(9)
    for ch in _sample_chunks():
        for _ in range(300):
            bad = ch.copy()
            k = int(rng.integers(0, ch.size))
            bad[k] ^= np.uint8(1 << int(rng.integers(0, 8)))
            try:
                dec(bad)
            except OracleError:
                pass


# ----------------------------------------------------------------------------- H9 positional checksum
# h = sum_i splitmix64(chunk_id ^ i ^ w_i) mod 2^64 over little-endian 8-byte words.

def test_checksum_splitmix64_reference_value():
    # SplitMix64 seeded with 0: first output 0xE220A8397B1DCDAF (the generator's published first value);
    # one zero word at index 0 of chunk 0 hashes exactly that
    assert oracle.checksum(np.zeros(8, np.uint8), 0) == 0xE220A8397B1DCDAF
    # an empty buffer sums nothing
    assert oracle.checksum(np.zeros(0, np.uint8), 123) == 0


def test_checksum_invariants():
    rng = np.random.default_rng(4)
    a = rng.integers(0, 256, size=8 * 1000 + 5, dtype=np.uint8)
    h = oracle.checksum(a, 77)
    # additive over word-aligned pieces: the words keep their positions only if the pieces are placed at
    # their offsets -- a prefix plus the zero-extended rest equals the whole minus zero-word terms
    pre = a.copy(); pre[4000:] = 0
    post = a.copy(); post[:4000] = 0
    zero_terms = oracle.checksum(np.zeros_like(a), 77)
    assert (oracle.checksum(pre, 77) + oracle.checksum(post, 77) - zero_terms) % (1 << 64) == h
    # position-sensitive: swapping two different words changes it; so do the chunk id and one flipped bit
    sw = a.copy(); sw[0:8], sw[8:16] = a[8:16], a[0:8]
    assert oracle.checksum(sw, 77) != h
    assert oracle.checksum(a, 78) != h
    b = a.copy(); b[8 * 1000 + 4] ^= 1  # the zero-padded tail word counts
    assert oracle.checksum(b, 77) != h
