"""NEXT-3 on B200: brute-force vs pruned search of the launch knobs (Table 3).

The B200 build fixes S (256 threads per CTA) and the tile shapes at compile time, so the runtime spaces are:
  F.P.  L = persistent fp_kernel CTAs per SM (knob fp_ctas_per_sm) in 2^0..2^4     (Table 3: L 2^0..2^4)
  G.P.  L = resident rle_kernel CTAs per SM (knob gp_ctas_per_sm) in 2^0..2^3   (Table 3: G.P. L = numCUs, S x C)
  N.P.  C = lanes per LZ4 sub-chunk (knob lz4_lanes) in {1, 2, 4, 8, 16, 32}       (Table 3: C 2^0..2^10)
        x the speculative-parse schedule (knob lz4_spec: 0 off, 2 always)
  H6    the scan schedule (knob scan_mode): reduce-then-scan vs single-pass look-back vs warp tiles
Each evaluation builds a fresh graph-mode batch over the workload (so the knob is captured), times K replays
with CUDA events after a 256 MiB L2-flush write each, and returns decoded GB/s.
usage: python tools/tune.py [--sf 10] [--steps 5] -> JSON lines + a summary table
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2602_08190_b200 import cdm, encoder, tune  # noqa: E402
from paper_2602_08190_b200.inputs import I64, TPCH, rle_column  # noqa: E402


def make_eval(eng, cols, steps, flush, stream, knob_names):
    decs, decoded = [], 0
    for spec, col in cols:
        for ch in encoder.encode_chunks(spec, col, 1 << 22):
            info = cdm.chunk_info(ch)
            out, offs = cdm.output_buffers(ch)
            decs.append(cdm.Decode(cdm.Cascade(spec, col.dtype, col.width), ch, out, offs,
                                   dev_chunk=torch.from_numpy(ch).cuda()))
            decoded += info["payload_bytes"] + info["offsets_bytes"]

    def evaluate(cfg):
        for k in knob_names:
            cdm.tune_set(k, cfg[k])
        b = cdm.Batch(eng, decs)
        b.set_graph(True)
        for _ in range(2):
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
        b.close()
        assert not any(r["error_bits"] for r in res)
        gbs = decoded * steps / tot / 1e6
        print(json.dumps({"config": cfg, "decoded_gbs": round(gbs, 1)}), flush=True)
        return gbs
    return evaluate


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sf", type=float, default=10.0)
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    eng = cdm.Engine(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.Stream()
    g = TPCH(a.sf)
    cases = {
        "FP": ({"fp_ctas_per_sm": [1, 2, 4, 8, 16]},
               [("Dict|BitPack", g.column("l_quantity")), ("Float2Int|BitPack", g.column("l_extendedprice"))]),
        "GP": ({"gp_ctas_per_sm": [1, 2, 4, 8]},
               [("RLE|[BitPack,BitPack]", rle_column("even-4", 1 << 26, I64)),
                ("RLE|[Delta|RLE|[BitPack,BitPack],BitPack]", g.column("l_orderkey"))]),
        "NP": ({"lz4_lanes": [1, 2, 4, 8, 16, 32], "lz4_spec": [0, 2]},
               [("Str|[LZ4(sub=16384,hc=9),BitPack]", g.column("l_comment"))]),
        "SCAN": ({"scan_mode": [0, 1, 2]}, [("Delta|BitPack", g.column("o_orderkey")),
                                         ("Str|[Raw,BitPack]", g.column("l_comment"))]),
    }
    rows = []
    defaults = {k: cdm.tune_get(k) for k in ("fp_ctas_per_sm", "lz4_lanes", "lz4_spec", "scan_mode", "gp_ctas_per_sm")}
    for pat, (space, cols) in cases.items():
        ev = make_eval(eng, cols, a.steps, flush, stream, list(space))
        bf = tune.brute_force(space, ev)
        pr = tune.pruned(space, ev)
        row = {"pattern": pat, "space": space, "bf_best": bf["best"], "bf_gbs": round(bf["best_metric"], 1),
               "bf_evaluations": bf["evaluations"], "pruned_best": pr["best"], "pruned_gbs": round(pr["best_metric"], 1),
               "pruned_evaluations": pr["evaluations"],
               "bf_trace": [(c, round(m, 1)) for c, m in bf["trace"]]}
        rows.append(row)
        print(json.dumps(row), flush=True)
        for k in space:  # restore the defaults
            cdm.tune_set(k, defaults[k])
    print("\n| pattern | space | B.F. evals | B.F. best (GB/s) | pruned evals | pruned best (GB/s) |")
    print("|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['pattern']} | {r['space']} | {r['bf_evaluations']} | {r['bf_best']} ({r['bf_gbs']}) | "
              f"{r['pruned_evaluations']} | {r['pruned_best']} ({r['pruned_gbs']}) |")


if __name__ == "__main__":
    main()
