"""Range-ANS (NEXT-1, reading R32) pinned on the CPU (-m "not gpu").

The oracle's ANS decoder (oracle/cdm_oracle.c) is pinned against things other than itself:
  * a textbook range-ANS ENCODER written here (PAPER.md:176 entropy family; 32-bit state, 16-bit words,
    SPEC.md:322) -- chunks it builds must decode to their input, for several alphabets, skews, table
    logs and chunk sizes, including the zero-entropy case;
  * the information bound: payload bits >= n*H(empirical) - 32*chunks and, for the 90/10 two-symbol
    column of SPEC.md:326 (H = 0.469 bits/symbol), <= n*H*(1 + 2%) + 32*chunks;
  * the product encoder (encoder/cdm_encode.c) is cross-checked word for word against this encoder run
    with the table the product wrote;
  * corrupt words / states are rejected (a chunk must end at state 2^16 with every word read).
"""
import math
import struct

import numpy as np
import pytest

import cdm1
import oracle
from paper_2602_08190_b200 import encoder
from paper_2602_08190_b200.inputs import FIXED, Column

L = 1 << 16


def normalise(data: bytes, tl: int) -> list[int]:
    """Any valid normalised table: floor(count * 2^tl / n), present symbols >= 1, remainder on the max."""
    M = 1 << tl
    cnt = [0] * 256
    for b in data:
        cnt[b] += 1
    n = len(data)
    f = [max(1, c * M // n) if c else 0 for c in cnt]
    diff = M - sum(f)
    big = max(range(256), key=lambda s: f[s])
    f[big] += diff
    assert f[big] >= 1 and sum(f) == M
    return f


def rans_encode_chunk(sym: bytes, f: list[int], tl: int, il: int = 1) -> tuple[list[int], list[int]]:
    """Encode one chunk with `il` interleaved states (symbol i -> state i mod il), back to front from state L
    in the exact reverse of the decode order; returns (words in decode order, initial decoder states)."""
    cum = [0] * 257
    for s in range(256):
        cum[s + 1] = cum[s] + f[s]
    x = [L] * il
    out = []
    for i in reversed(range(len(sym))):
        s, k = sym[i], i % il
        fs = f[s]
        x_max = ((L >> tl) << 16) * fs
        while x[k] >= x_max:
            out.append(x[k] & 0xFFFF)
            x[k] >>= 16
        x[k] = (x[k] // fs << tl) + x[k] % fs + cum[s]
    assert all(L <= v < 1 << 32 for v in x)
    return out[::-1], x


def ans_chunk(data: bytes, tl: int = 12, chunk: int = 4096, f=None, corrupt=None, il: int = 1):
    """A FIXED(1) CDM1 chunk whose root is an ANS node (cascade text "ANS")."""
    f = f or normalise(data, tl)
    n = len(data)
    nch = (n + chunk - 1) // chunk
    words, tab = [], bytearray(struct.pack("<256H", *f))
    for c in range(nch):
        w, x = rans_encode_chunk(data[c * chunk:(c + 1) * chunk], f, tl, il)
        if corrupt == "state" and c == 0:
            x[il // 2] ^= 1
        tab += struct.pack("<II", len(words), len(w)) + struct.pack(f"<{il}I", *x)
        words += w
    if corrupt == "word" and words:
        words[len(words) // 2] ^= 0x40
    if corrupt == "truncate" and words:
        words = words[:-1]
    wbytes = struct.pack(f"<{len(words)}H", *words)
    root = cdm1.Node(cdm1.ANS, n, [cdm1.raw(wbytes, 2), cdm1.raw(bytes(tab))], nsub=nch, sub=chunk, tl=tl, il=il)
    return cdm1.build(root, cdm1.FIXED, 1, n), len(words)


def entropy_bits(data: bytes) -> float:
    n = len(data)
    cnt = np.bincount(np.frombuffer(data, dtype=np.uint8), minlength=256)
    p = cnt[cnt > 0] / n
    return float(-(p * np.log2(p)).sum() * n)


CASES = {
    "uniform256": lambda r, n: r.integers(0, 256, n, dtype=np.uint8),
    "skew9010": lambda r, n: np.where(r.random(n) < 0.9, 65, 66).astype(np.uint8),
    "returnflag": lambda r, n: np.array([78, 65, 82], np.uint8)[r.choice(3, n, p=[0.5, 0.25, 0.25])],
    "geometric": lambda r, n: np.minimum(r.geometric(0.3, n), 255).astype(np.uint8),
    "single": lambda r, n: np.full(n, 0x41, np.uint8),
}


@pytest.mark.parametrize("il", [1, 32])
@pytest.mark.parametrize("dist", sorted(CASES))
@pytest.mark.parametrize("tl,chunk,n", [(12, 4096, 30000), (8, 1024, 5000), (15, 16, 333), (10, 65536, 70001)])
def test_oracle_decodes_textbook_encoder(dist, tl, chunk, n, il):
    r = np.random.default_rng(hash((dist, tl, chunk)) & 0xFFFF)
    data = CASES[dist](r, n).tobytes()
    if dist == "uniform256" and tl == 8:
        data = bytes(b & 0x7F for b in data)  # 128 symbols fit a 2^8 table
    ch, _ = ans_chunk(data, tl, chunk, il=il)
    out, _ = oracle.decode_chunk(ch)
    assert out.tobytes() == data


@pytest.mark.parametrize("il", [1, 32])
def test_zero_entropy_needs_no_words(il):
    ch, nw = ans_chunk(b"\x41" * 50000, 12, 4096, il=il)
    assert nw == 0
    assert oracle.decode_chunk(ch)[0].tobytes() == b"\x41" * 50000


@pytest.mark.parametrize("il", [1, 32])
@pytest.mark.parametrize("dist", ["skew9010", "returnflag", "uniform256", "geometric"])
def test_entropy_bounds(dist, il):
    r = np.random.default_rng(7)
    n, chunk = 200_000, 16384 if il == 32 else 4096
    data = CASES[dist](r, n).tobytes()
    ch, nw = ans_chunk(data, 12, chunk, il=il)
    nch = (n + chunk - 1) // chunk
    H = entropy_bits(data)
    bits = 16 * nw
    assert bits + 32 * il * nch >= H - 1e-6 * n  # nothing beats the entropy (the final states carry <= 32 bits)
    assert bits <= H * 1.02 + 48 * il * nch
    if dist == "skew9010":
        assert abs(H / n - 0.469) < 0.01  # SPEC.md:326's H for 90/10


@pytest.mark.parametrize("il", [1, 32])
def test_product_encoder_matches_textbook_encoder(il):
    """The C encoder's words and states equal this file's encoder run with the table the C encoder chose."""
    r = np.random.default_rng(3)
    data = CASES["returnflag"](r, 50_000)
    col = Column("t", FIXED, 1, data.size, data.copy(), None)
    ch = encoder.encode(f"ANS(chunk=4096,tl=12,il={il})", col)
    hdr, nodes, streams = cdm1.parse(ch)
    assert nodes[0]["codec"] == cdm1.ANS
    words = np.frombuffer(streams[nodes[1]["stream"]], dtype=np.uint16).tolist()
    tab = streams[nodes[2]["stream"]]
    f = list(struct.unpack_from("<256H", tab, 0))
    assert sum(f) == 1 << 12
    rec = 8 + 4 * il
    pos = 0
    for c in range(len(tab[512:]) // rec):
        w0, nw = struct.unpack_from("<II", tab, 512 + rec * c)
        xs = list(struct.unpack_from(f"<{il}I", tab, 512 + rec * c + 8))
        ew, ex = rans_encode_chunk(data[c * 4096:(c + 1) * 4096].tobytes(), f, 12, il)
        assert (w0, nw, xs) == (pos, len(ew), ex)
        assert words[w0:w0 + nw] == ew
        pos += nw
    assert oracle.decode_chunk(ch)[0].tobytes() == data.tobytes()


@pytest.mark.parametrize("il", [1, 32])
@pytest.mark.parametrize("corrupt", ["word", "state", "truncate"])
def test_corrupt_ans_rejected(corrupt, il):
    r = np.random.default_rng(5)
    data = CASES["returnflag"](r, 20000).tobytes()
    ch, _ = ans_chunk(data, 12, 4096, corrupt=corrupt, il=il)
    with pytest.raises(Exception):
        out, _ = oracle.decode_chunk(ch)
        assert out.tobytes() == data  # a corruption that still decodes must not go unnoticed


def test_varbytes_round_trip_through_ans():
    from paper_2602_08190_b200.inputs import TPCH
    col = TPCH(0.002).column("l_comment")
    for ch in encoder.encode_chunks("Str|[ANS(chunk=1024),BitPack]", col, 5000):
        out, offs = oracle.decode_chunk(ch)
        assert offs[0] == 0 and offs.size == cdm1.parse(ch)[0]["rows"] + 1
    exp = col.data.tobytes()
    got = b"".join(oracle.decode_chunk(ch)[0].tobytes()
                   for ch in encoder.encode_chunks("Str|[ANS(chunk=1024),BitPack]", col, 5000))
    assert got == exp[:len(got)] and len(got) == len(exp)
