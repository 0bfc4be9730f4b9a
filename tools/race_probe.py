"""Probe for the round-1 racecheck finding: graph replays of `Str|[LZ4,BitPack]` (test_lz4_overlapping_matches)
left the VARCHAR offsets at the -7 fill under compute-sanitizer racecheck.

Runs the same chunk through cdm_batch in graph mode for --replays replays, refilling the outputs with the
sentinel between replays, and prints per replay whether payload / offsets came back right.
Usage: python tools/race_probe.py [--replays N] [--spec lz4|raw] [--lanes L] [--mode graph|direct]
"""
import argparse
import os
import struct
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np
import torch

import cdm1
import oracle
from paper_2602_08190_b200 import cdm
from test_oracle_pins import _seq


def _hash(spec):
    from test_gpu_parity import _hash as h
    return h(spec)


def build_chunk():
    blocks, sizes = [], []
    for off, mlen in [(1, 4), (1, 300), (2, 19), (3, 1000), (5, 5), (7, 270), (31, 100), (32, 100), (33, 700)]:
        lit = bytes(range(65, 65 + off + 2))
        blocks.append(_seq(lit, off, mlen) + _seq(b"END", None, None))
        sizes.append(len(lit) + mlen + 3)
    payload = b"".join(blocks)
    tab, pos = b"", 0
    for blk, dl in zip(blocks, sizes):
        tab += struct.pack("<III", pos, len(blk), dl)
        pos += len(blk)
    n = sum(sizes)
    lens = [n // 2, n - n // 2]
    spec = "Str|[LZ4,BitPack]"
    root = cdm1.Node(cdm1.STR, 2, [
        cdm1.Node(cdm1.LZ4, n, [cdm1.raw(payload), cdm1.raw(tab, eb=12)], nsub=len(blocks), sub=1 << 16),
        cdm1.bitpack(lens, 16, 0)])
    return spec, cdm1.build(root, cdm1.VARBYTES, 1, 2, payload=n, cascade_hash=_hash(spec))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--replays", type=int, default=8)
    ap.add_argument("--lanes", type=int, default=4)
    ap.add_argument("--mode", default="graph")
    ap.add_argument("--sync", default="device", help="device | stream: how the refill is ordered before a launch")
    ap.add_argument("--parity", action="store_true", help="run tests/test_gpu_parity.check_parity's four modes first")
    ap.add_argument("--scan-mode", type=int, default=None)
    a = ap.parse_args()
    if a.scan_mode is not None:
        cdm.tune_set("scan_mode", a.scan_mode)
    cdm.tune_set("lz4_lanes", a.lanes)
    spec, ch = build_chunk()
    exp, exp_offs = oracle.decode_chunk(ch)
    eng = cdm.Engine(0, n_slots=3, slot_bytes=256 << 20)
    casc = cdm.Cascade(spec, cdm.VARBYTES, 1)
    if a.parity:
        import test_gpu_parity as T
        for mode in (False, "pipeline", True, "graph"):
            got = T.gpu_decode(eng, casc, [ch], resident=mode)
            (payload, offs, r), = got
            print(f"check_parity mode {mode}: payload {'ok' if np.array_equal(payload, exp) else 'BAD'} offsets "
                  f"{'ok' if np.array_equal(offs[: exp_offs.size], exp_offs) else 'BAD ' + str(offs[:4].tolist())}",
                  flush=True)
    info = cdm.chunk_info(ch)
    out = torch.full(((info["payload_bytes"] + 15) // 16 * 16 + 64,), 0xA5, dtype=torch.uint8, device="cuda")
    offs = torch.full((info["offsets_bytes"] // 4 + 4,), -7, dtype=torch.int32, device="cuda")
    d = cdm.Decode(casc, cdm.pinned(ch), out, offs)
    d.dev_chunk = torch.from_numpy(ch).cuda()
    b = cdm.Batch(eng, [d])
    b.set_graph(a.mode == "graph")
    stream = torch.cuda.Stream()
    bad = 0
    for r in range(a.replays):
        if a.sync == "stream":
            with torch.cuda.stream(stream):
                out.fill_(0xA5)
                offs.fill_(-7)
        else:
            out.fill_(0xA5)
            offs.fill_(-7)
            torch.cuda.synchronize()
        b.launch(stream)
        res = b.results(stream, raise_on_error=False)
        torch.cuda.synchronize()
        o = out.cpu().numpy()[: exp.size]
        f = offs.cpu().numpy()[: exp_offs.size]
        ok_p = np.array_equal(o, exp)
        ok_o = np.array_equal(f, exp_offs)
        bad += not (ok_p and ok_o)
        print(f"replay {r}: payload {'ok' if ok_p else 'BAD'} offsets {'ok' if ok_o else 'BAD ' + str(f.tolist())} "
              f"err {res[0]['error_bits']}", flush=True)
    b.close()
    eng.close()
    print("probe", "ok" if not bad else f"FAILED {bad}/{a.replays}")


if __name__ == "__main__":
    main()
