import sys, numpy as np, torch
sys.path[:0] = ['tests', '.']
import oracle
from paper_2602_08190_b200 import cdm, encoder
from paper_2602_08190_b200.inputs import TPCH
import test_gpu_parity as T
eng = cdm.Engine(0)
col = TPCH(0.01).column("l_comment")
spec = "Str|[LZ4(sub=4096),BitPack]"
chs = encoder.encode_chunks(spec, col, 30_001)
casc = cdm.Cascade(spec, col.dtype, col.width)
for g in (1, 2, 4, 8):
    cdm.tune_set("lz4_split", 1); cdm.tune_set("lz4_split_g", g)
    got = T.gpu_decode(eng, casc, chs[:2], resident=True, expect_error=True)
    for ch, (p, o, r) in zip(chs[:2], got):
        exp, _ = oracle.decode_chunk(ch)
        bad = np.flatnonzero(p != exp)
        print(g, r["error_bits"], len(bad), bad[:3] // 4096 if len(bad) else "", flush=True)
