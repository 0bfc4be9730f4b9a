"""Paper-shaped microbenchmarks on B200 (SURVEY Sec. 8d "Extra sweeps", NEXT-3's measurement half).

Each case: synthetic column -> CDM1 chunks of 2^22 rows (host, untimed) -> device-resident batch in graph mode
-> K timed replays (CUDA events on the launching stream, 256 MiB L2-flush write between replays, outside the
events) -> decoded GB/s and the Eq. 1 roofline fraction ((compressed read + decoded written) / time / the
MEASURED_PEAKS copy peak).  Sweeps:
  E2  BitPack bit width w = 1..32, int32 output (uniform w-bit values)
  E2L BitPack bit width w = 1..64, int64 output
  E3  RLE group-size distributions even-X / random-L-R / outlier-X-P / mixed, int64
  E7  fused vs decoded-twice: Dict|BitPack and Float2Int|BitPack (PAPER.md:565-588's fusion question)
  CHR CHAR(n) dictionary rows: l_shipinstruct (25 B), l_shipmode (10), l_returnflag (1), o_orderpriority /
      o_clerk (15), o_orderstatus (1)
  SCAN H6 element-level Delta|BitPack / VARCHAR offsets: l_comment offsets, o_orderkey SF 100, config 1 sorted,
      random walks w = 4..32 (per-kernel times reported for every case)
  NP  LZ4 sub-chunk size and ANS chunk size (PAPER.md:411-416's chunk-size trade-off)
usage: python tools/microbench.py [sweeps] [--rows N] [--steps K]  -> JSON lines + a markdown table on stdout
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2602_08190_b200 import cdm, encoder  # noqa: E402
from paper_2602_08190_b200.inputs import (I32, I64, TPCH, Column, config1_column, rle_column,  # noqa: E402
                                          uniform_bits_column)

CHUNK = 1 << 22


def peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return float(json.load(open(p))["hbm_gbs"]) if os.path.exists(p) else 6650.0


FILTER = None


def run_case(eng, name, spec, col, steps, flush, stream):
    if FILTER and FILTER not in name:
        return None
    chunks = encoder.encode_chunks(spec, col, CHUNK)
    decs = []
    comp = dec = 0
    for ch in chunks:
        info = cdm.chunk_info(ch)
        out, offs = cdm.output_buffers(ch)
        decs.append(cdm.Decode(cdm.Cascade(spec, col.dtype, col.width), ch, out, offs,
                               dev_chunk=torch.from_numpy(ch).cuda()))
        comp += int(ch.size)
        dec += info["payload_bytes"] + info["offsets_bytes"]
    b = cdm.Batch(eng, decs)
    b.set_graph(True)
    for _ in range(3):
        b.launch(stream)
    b.results(stream)
    tot = 0.0
    for _ in range(steps):
        with torch.cuda.stream(stream):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            b.launch(stream)
            e1.record(stream)
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    res = b.results(stream, raise_on_error=False)
    # every kernel timed alone (events around each launch, families serialised), after L2 flushes
    b.set_timing(2)
    for _ in range(steps):
        with torch.cuda.stream(stream):
            flush.zero_()
            b.launch(stream)
        b.collect_timing()
    b.results(stream, raise_on_error=False)
    kt, kb = b.kernel_times(), b.kernel_bytes()
    # the RLE chain's kinds (sums, level launches, rle_big) report as one family: its bytes sit on one kind
    agg_t, agg_b = {}, {}
    for k, (kms, n) in kt.items():
        if not n:
            continue
        f = "rle_chain" if k.startswith("rle") else k
        agg_t[f] = agg_t.get(f, 0.0) + kms
        agg_b[f] = agg_b.get(f, 0) + kb.get(k, 0)
    kern = {}
    for k, kms in agg_t.items():
        if agg_b.get(k):
            per = kms / steps  # kernel_times sums over steps (a kind may launch several times per step)
            kern[k] = {"ms": round(per, 4), "gbs": round(agg_b[k] / per / 1e6, 1),
                       "frac": round(agg_b[k] / per / 1e6 / peak(), 3)}
    b.close()
    ms = tot / steps
    return {"case": name, "cascade": spec, "rows": col.rows, "decoded_mb": round(dec / 1e6, 1),
            "compressed_mb": round(comp / 1e6, 2), "cr": round(dec / comp, 2), "ms": round(ms, 4),
            "decoded_gbs": round(dec / ms / 1e6, 1), "eq1_frac": round((dec + comp) / ms / 1e6 / peak(), 3),
            "errors": int(any(r["error_bits"] for r in res)), "kernels": kern}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sweeps", nargs="*", default=["E2", "E3", "E7", "NP"])
    ap.add_argument("--rows", type=int, default=1 << 27)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--filter", default=None, help="only the cases whose name contains this")
    a = ap.parse_args()
    global FILTER
    FILTER = a.filter
    eng = cdm.Engine(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.Stream()
    n = a.rows
    rows = []

    def emit(r):
        if r is None:
            return
        rows.append(r)
        print(json.dumps(r), flush=True)

    if "E2" in a.sweeps:
        for w in (1, 2, 4, 8, 12, 16, 20, 24, 28, 32):
            emit(run_case(eng, f"E2 w={w}", "BitPack", uniform_bits_column(n, w, I32), a.steps, flush, stream))
    if "E2L" in a.sweeps:  # E2 on int64 output up to w = 64 (PAPER.md:356-371's bit-width sweep, 8-byte rows)
        for w in (1, 4, 8, 16, 24, 32, 40, 48, 56, 64):
            emit(run_case(eng, f"E2 i64 w={w}", "BitPack", uniform_bits_column(n // 2, w, I64), a.steps, flush, stream))
    if "E3" in a.sweeps:
        for dist in ("even-1", "even-4", "even-32", "even-1024", "random-1-8", "random-1-64", "outlier-1024-1",
                     "mixed-even-4+random-1-64"):
            emit(run_case(eng, f"E3 {dist}", "RLE|[BitPack,BitPack]", rle_column(dist, n // 2, I64), a.steps, flush,
                          stream))
    if "E7" in a.sweeps:
        g = TPCH(10.0)
        for name, spec in (("l_quantity", "Dict|BitPack"), ("l_extendedprice", "Float2Int|BitPack"),
                           ("l_shipinstruct", "Dict|BitPack"), ("l_shipdate", "Dict|BitPack")):
            emit(run_case(eng, f"E7 {name}", spec, g.column(name), a.steps, flush, stream))
    if "CHR" in a.sweeps:  # CHAR(n) Dict|BitPack rows (reading R14), SF 10
        g = TPCH(10.0)
        for name in ("l_shipinstruct", "l_shipmode", "l_returnflag", "o_orderpriority", "o_clerk", "o_orderstatus"):
            emit(run_case(eng, f"CHR {name}", "Dict|BitPack", g.column(name), a.steps, flush, stream))
    if "SCAN" in a.sweeps:  # H6 element-level scans (SURVEY Sec. 8d "Extra sweeps")
        g = TPCH(10.0)
        emit(run_case(eng, "SCAN l_comment offsets", "Str|[LZ4(sub=16384),BitPack]", g.column("l_comment"), a.steps,
                      flush, stream))
        emit(run_case(eng, "SCAN o_orderkey SF100 Delta|BitPack", "Delta|BitPack", TPCH(100.0).column("o_orderkey"),
                      a.steps, flush, stream))
        c1 = config1_column(n)
        c1s = Column("sorted", I32, 4, n, np.sort(c1.data))
        emit(run_case(eng, "SCAN config1 sorted Delta|BitPack", "Delta|BitPack", c1s, a.steps, flush, stream))
        rng = np.random.default_rng(5)
        for w in (4, 8, 16, 32):
            steps_w = rng.integers(-(1 << (w - 1)), 1 << (w - 1), size=n // 2, dtype=np.int64)
            walk = np.cumsum(steps_w).astype(np.int64)
            emit(run_case(eng, f"SCAN random walk w={w}", "Delta|BitPack", Column("walk", I64, 8, n // 2, walk), a.steps,
                          flush, stream))
    if "NP" in a.sweeps:
        g = TPCH(10.0)
        com = g.column("l_comment")
        for sub in (4096, 16384, 65536):
            emit(run_case(eng, f"NP lz4 sub={sub}", f"Str|[LZ4(sub={sub}),BitPack]", com, a.steps, flush, stream))
        # the bench's encoder setting: liblz4 HC level 9 (CR 1.86 -> 2.24 on the payload, 7.1 -> 8.9 bytes per sequence)
        emit(run_case(eng, "NP lz4 sub=16384 hc=9", "Str|[LZ4(sub=16384,hc=9),BitPack]", com, a.steps, flush, stream))
        # config 4's launch shape: ONE l_comment chunk of 2^22 rows (the bench decodes one such chunk per pipeline
        # group, ~6.9 K sub-chunks per launch)
        c4 = Column("l_comment", com.dtype, com.width, 1 << 22, com.data[: int(com.offsets[1 << 22])].copy(),
                    com.offsets[: (1 << 22) + 1].copy())
        emit(run_case(eng, "NP lz4 one 4M-row chunk sub=16384 hc=9", "Str|[LZ4(sub=16384,hc=9),BitPack]", c4,
                      a.steps, flush, stream))
        # single-sub-chunk latency: ONE sub-chunk (l_comment rows totalling ~sub bytes) per launch -- the length of
        # the chunk-sequential chain that bounds every LZ4 launch
        for sub in (4096, 16384, 65536):
            lens = np.diff(com.offsets)
            nrow = int(np.searchsorted(np.cumsum(lens), sub - 64))
            one = Column("l_comment", com.dtype, com.width, nrow, com.data[: int(com.offsets[nrow])].copy(),
                         com.offsets[: nrow + 1].copy())
            emit(run_case(eng, f"NP lz4 one sub-chunk sub={sub}", f"Str|[LZ4(sub={sub}),BitPack]", one, a.steps,
                          flush, stream))
        rf = g.column("l_returnflag")
        for chunk in (1024, 4096, 16384):
            emit(run_case(eng, f"NP ans chunk={chunk}", f"ANS(chunk={chunk})", rf, a.steps, flush, stream))
        emit(run_case(eng, "NP ans str chunk=4096", "Str|[ANS(chunk=4096),BitPack]", com, a.steps, flush, stream))
    print("\n| case | cascade | decoded MB | CR | ms | decoded GB/s | Eq.1 frac |")
    print("|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['case']} | `{r['cascade']}` | {r['decoded_mb']} | {r['cr']} | {r['ms']} | {r['decoded_gbs']} | "
              f"{r['eq1_frac']}{' ERR' if r['errors'] else ''} |")


if __name__ == "__main__":
    main()
