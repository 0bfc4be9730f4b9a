"""Host-side checks of the C-ABI library (-m "not gpu"): it loads, exports every symbol include/cdm.h
declares, compiles cascades to the documented fused plans, validates chunks on the host exactly like the
device path, and orders jobs by Johnson's rule.  No compute call needs a GPU here."""
import os
import re

import numpy as np
import pytest

import oracle
from paper_2602_08190_b200 import cdm, encoder
from paper_2602_08190_b200.inputs import TPCH, config1_column

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "cdm.h")).read()
    declared = set(re.findall(r"CDM_API\s+[\w\s\*]+?\b(cdm_\w+)\s*\(", hdr))
    assert len(declared) >= 20
    lib = cdm.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(cdm.SYMBOLS)
    assert "sm_100a" in cdm.version()


def test_kernels_are_sm100a_sass():
    import subprocess
    so = os.path.join(ROOT, "paper_2602_08190_b200", "_lib", "libcdm.so")
    cdm.lib()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    for k in ("fp_kernel", "scan_kernel", "rle_kernel", "rle_big_kernel", "rle_sums_kernel", "lz4_kernel"):
        assert k in sass
    assert "UBLKCP" in sass  # TMA bulk copies (cp.async.bulk) in the FP / scan kernels


@pytest.mark.parametrize("spec,dtype,plan", [
    ("BitPack", cdm.I32, "fp(unpack+FOR+cast)"),
    ("Dictionary encoding | Bit-packing", cdm.F64, "fp(unpack+FOR+dict gather)"),
    ("Float2Int|BitPack", cdm.F64, "fp(unpack+FOR+float2int)"),
    ("Delta|BitPack", cdm.I64, "scan("),
    ("RLE|[BitPack,BitPack]", cdm.I32, "rle("),
    ("RLE|[Delta|RLE|[BitPack,BitPack],BitPack]", cdm.I64, "run values -> u64 array"),
    ("RLE|[DeltaStride|[BitPack,BitPack],RLE|[BitPack,BitPack]]", cdm.I32, "run counts -> u32 array"),
    ("RLE|[BitPack,RLE|[BitPack,BitPack]]", cdm.I64, "counts = a lower level's array"),
    ("Delta|Dict|BitPack", cdm.I32, "dict gather+delta"),
    ("Delta|RLE|[BitPack,BitPack]", cdm.I64, "arithmetic runs"),
    ("DeltaStride|[BitPack,BitPack]", cdm.I64, "start + j*stride"),
    ("DeltaStride|[Delta|RLE|[BitPack,BitPack],BitPack]", cdm.I64, "rle level 1 (arithmetic runs"),
    ("RLE|[DeltaStride|[Delta|RLE|[BitPack,BitPack],BitPack],BitPack]", cdm.I64, "rle level 2"),
    ("RLE|[RLE|[BitPack,BitPack],BitPack]", cdm.I64, "rle level 1 (expand"),
    ("Str|[LZ4,BitPack]", cdm.VARBYTES, "lz4_group_decode"),
    ("Str|[ANS,BitPack]", cdm.VARBYTES, "ans_chunk_decode"),
    ("Str|[StrDict|BitPack|ANS,BitPack]", cdm.VARBYTES, "ans_chunk_decode(ids) + strdict_expand"),
    ("Str|[StrDict|BitPack,BitPack]", cdm.VARBYTES, "strdict_expand"),
    ("ANS", cdm.FIXED, "ans_chunk_decode"),
])
def test_cascade_plans(spec, dtype, plan):
    c = cdm.Cascade(spec, dtype, 1 if dtype == cdm.FIXED else 0)
    d = c.describe()
    assert plan in d
    assert d.split(" => ")[0] == encoder.canonical(spec)


@pytest.mark.parametrize("spec,code", [("RLE|[BitPack", 2), ("Nope", 2), ("BitPack|[Raw,Raw]", 2),
                                       ("Delta|Delta|BitPack", 3), ("BitPack|ANS", 3), ("Str|[LZ4,BitPack]", 3)])
def test_cascade_errors(spec, code):
    with pytest.raises(cdm.CdmError) as e:
        cdm.Cascade(spec, cdm.I64)
    assert e.value.status == code


def test_chunk_check_accepts_encoder_output_and_rejects_corruption():
    g = TPCH(0.005)
    for name, spec in [("l_orderkey", "RLE|[Delta|RLE|[BitPack,BitPack],BitPack]"), ("l_quantity", "Dict|BitPack"),
                       ("l_comment", "Str|[LZ4,BitPack]"), ("o_orderkey", "Delta|RLE|[BitPack,BitPack]")]:
        col = g.column(name)
        casc = cdm.Cascade(spec, col.dtype, col.width)
        ch = encoder.encode(spec, col)
        cdm.chunk_check(casc, ch)
        info = cdm.chunk_info(ch)
        assert info["rows"] == col.rows and info["compressed_bytes"] == ch.size
        # truncation at every 7th byte: rejected on the host (never reaches a kernel)
        for cut in range(0, ch.size, 7):
            with pytest.raises(cdm.CdmError):
                cdm.chunk_check(casc, ch[:cut].copy())
    # a chunk of another cascade is refused
    ch = encoder.encode("Delta|BitPack", config1_column(100))
    with pytest.raises(cdm.CdmError):
        cdm.chunk_check(cdm.Cascade("BitPack", cdm.I32), ch)


def test_host_and_oracle_agree_on_validity():
    """Flipped header/table bytes: whenever the host check accepts a chunk, the oracle must decode it
    cleanly or report a data error the device also detects (never a structural error)."""
    rng = np.random.default_rng(3)
    col = config1_column(3000)
    ch = encoder.encode("RLE|[BitPack,BitPack]", col)
    casc = cdm.Cascade("RLE|[BitPack,BitPack]", cdm.I32)
    hdr_end = 64 + 32 * 5 + 16 * 2
    for _ in range(400):
        bad = ch.copy()
        k = int(rng.integers(0, hdr_end))
        bad[k] ^= np.uint8(1 << int(rng.integers(0, 8)))
        try:
            cdm.chunk_check(casc, bad)
        except cdm.CdmError:
            continue
        try:
            oracle.decode_chunk(bad)
        except oracle.OracleError as e:
            assert "run" in e.detail or "row" in e.detail, e.detail


def test_johnson_matches_oracle_rule():
    rng = np.random.default_rng(4)
    for _ in range(100):
        n = int(rng.integers(0, 12))
        t = [float(rng.integers(0, 10)) for _ in range(n)]
        d = [float(rng.integers(0, 10)) for _ in range(n)]
        assert cdm.johnson_order(t, d) == oracle.johnson_order(list(zip(t, d)))
    assert cdm.johnson_order([4, 1], [1, 4]) == [1, 0]  # B before A
