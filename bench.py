#!/usr/bin/env python
"""bench.py -- effective decoded GB/s (host-compressed -> device-decoded) of the cascaded-columnar decode hot
path on B200.

Default workload = the north-star configuration (BASELINE.json configs[3], "config 4"): every TPC-H lineitem
and orders column (25) at SF=100 ("all experiments use a TPC-H scale factor of 100"), synthetic
dbgen-like data, row groups of 2^22 rows, each column under the SURVEY Sec. 8d cascade map (Table 2 mapped onto
the hot-path codecs: FP, Delta/VARCHAR scans, RLE / DeltaStride chains, LZ4, ANS, String-dictionary).  The
compressed chunks (~21.5 GB) are generated and encoded in parallel worker processes into ONE host buffer that
is page-locked in place (cdm_host_register) -- the paper's column store in pinned CPU memory.

One step = every chunk of the workload crosses PCIe and is decoded into its device output buffer.

  value      host-compressed -> device-decoded GB/s: decoded bytes / device time of one cdm_pipeline_launch
             (the H4 schedule: Johnson order, H2D copies from pinned host overlapped with the fused decodes of
             earlier groups, captured once as a CUDA graph), CUDA events on the launching stream; K steps.
  e2e        the same through the public API with the host in the loop: wall clock of cdm_pipeline_launch +
             cdm_pipeline_results (every chunk's error word read back on the host) per step.
  device_resident  decode only, compressed chunks already in HBM (cdm_batch graph replay), L2 flushed
             between steps -- the kernel-level number.
  serialized the non-pipelined schedule (E11): one H2D copy of all compressed bytes, then
             the decode -- what pipelining saves.
  roofline   the dominant kernel (alone) against the measured HBM peak; roofline.families = every kernel
             family's algorithmic bytes (Eq. 1, from cdm_batch_kernel_bytes) / its time alone.
  parity     H9 checksums of every chunk's device output; the oracle's checksums of the cpu_baseline sample.
  cpu_baseline  the CPU oracle (oracle/, plain C) on a bounded sample (the first chunk of every column), on 1
             thread and on every host core.

Multi-GPU (torchrun, one process per GPU, NCCL): strong scaling -- ONE dataset, each column's chunks split
into contiguous per-rank ranges balanced by row count (= compressed bytes for equal-size chunks; shard.py);
each rank builds, pins and decodes only its shard, CPU-bound to its GPU's affinity; the only collectives are
all-reduces of metadata, checksums and times.  checksum_total is the same for every N.

--impl reference: this tier's reference arm is the CPU oracle, timed as it stands on the host cores over the
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "effective decoded GB/s (host-compressed→device-decoded) at 1/2/4/8 B200 vs roofline"
CONFIG4_COLS = [
    ("l_orderkey", "RLE|[DeltaStride|[Delta|RLE|[BitPack,BitPack],BitPack],BitPack]"), ("l_partkey", "BitPack"),
    ("l_suppkey", "BitPack"), ("l_linenumber", "BitPack"), ("l_quantity", "Dict|BitPack"),
    ("l_extendedprice", "Float2Int|BitPack"), ("l_discount", "Dict|BitPack"), ("l_tax", "Dict|BitPack"),
    ("l_returnflag", "ANS"), ("l_linestatus", "Dict|BitPack"), ("l_shipdate", "Dict|BitPack"),
    ("l_commitdate", "Dict|BitPack"), ("l_receiptdate", "Dict|BitPack"), ("l_shipinstruct", "Dict|BitPack"),
    ("l_shipmode", "Dict|BitPack"), ("l_comment", "Str|[LZ4(sub=16384,hc=9),BitPack]"),
    ("o_orderkey", "DeltaStride|[Delta|RLE|[BitPack,BitPack],BitPack]"), ("o_custkey", "BitPack"),
    ("o_orderstatus", "Dict|BitPack"), ("o_totalprice", "Float2Int|BitPack"), ("o_orderdate", "Dict|BitPack"),
    ("o_orderpriority", "Dict|BitPack"), ("o_clerk", "Dict|BitPack"), ("o_shippriority", "RLE|[BitPack,BitPack]"),
    ("o_comment", "Str|[StrDict|BitPack|ANS,BitPack]")]
WORKLOADS = {
    # BASELINE configs[3] (the default / headline): all 25 lineitem + orders columns, SF=100 (north star)
    "config4": dict(sf=100.0, dtype="mixed", cols=CONFIG4_COLS,
                    desc="config 4: TPC-H lineitem + orders, all 25 columns at SF={sf} (SURVEY Sec. 8d cascade "
                         "map: l_returnflag ANS, l_/o_orderkey DeltaStride, o_comment String-dictionary|BitPack|ANS "
                         "per Table 2), streamed from pinned host"),
    # config 4 with Table 2's comment cascade (O_COMMENT's String-dictionary|Bit-packing|ANS) also on
    # l_comment: the cascade choice the paper's per-column selection would make for a comment column (P:499-500:
    # String-dictionary beats the LZ77 family on comments); the default config 4 keeps chunk-parallel LZ4
    "config4sd": dict(sf=100.0, dtype="mixed",
                      cols=[(n, "Str|[StrDict|BitPack|ANS,BitPack]" if n == "l_comment" else c) for n, c in CONFIG4_COLS],
                      desc="config 4 with l_comment under Table 2's comment cascade Str|[StrDict|BitPack|ANS,BitPack]: "
                           "TPC-H lineitem + orders, all 25 columns at SF={sf}, streamed from pinned host"),
    # BASELINE configs[4]: SF=1000 lineitem streamed through an output ring, 8 GPUs; one process decodes its
    # 1/8 slice (chunk ranges of every column), N processes take slices rank, rank + N, ... (see run_config5)
    "config5": dict(sf=1000.0, dtype="mixed", cols=[c for c in CONFIG4_COLS if c[0].startswith("l_")],
                    desc="config 5: TPC-H lineitem (16 columns) at SF={sf}, 1/8 slices streamed from pinned host "
                         "through an output ring (not retained)"),
    # BASELINE configs[1]: TPC-H SF=1 lineitem numeric columns
    "config2": dict(sf=1.0, dtype="int64", cols=[("l_orderkey", "RLE|[Delta|RLE|[BitPack,BitPack],BitPack]"),
                                                  ("l_quantity", "Dict|BitPack"), ("l_discount", "Dict|BitPack")],
                    desc="config 2: TPC-H SF={sf} lineitem numeric columns (l_orderkey RLE|[Delta|RLE|[BitPack,"
                         "BitPack],BitPack], l_quantity Dict|BitPack, l_discount Dict|BitPack)"),
    # BASELINE configs[2]: TPC-H SF=10 lineitem string columns (dictionary CHAR(n) + chunk-parallel LZ4)
    "config3": dict(sf=10.0, dtype="u8", cols=[("l_shipmode", "Dict|BitPack"), ("l_returnflag", "Dict|BitPack"),
                                                ("l_comment", "Str|[LZ4(sub=16384,hc=9),BitPack]")],
                    desc="config 3: TPC-H SF={sf} lineitem string columns (l_shipmode/l_returnflag Dict|BitPack "
                         "CHAR(n), l_comment Str|[LZ4(16 KiB sub-chunks),BitPack])"),
    # NEXT-2 Table 2's PS rows: partsupp at SF=100 (80 M rows), PS_PARTKEY RLE|[DeltaStride,RLE]
    # (count lineage, R35), PS_SUPPKEY Delta|Dict|BitPack (R36), PS_SUPPLYCOST Float2Int|BitPack, plus the other two
    "partsupp": dict(sf=100.0, dtype="mixed",
                     cols=[("ps_partkey", "RLE|[DeltaStride|[BitPack,BitPack],RLE|[BitPack,BitPack]]"),
                           ("ps_suppkey", "Delta|Dict|BitPack"), ("ps_availqty", "BitPack"),
                           ("ps_supplycost", "Float2Int|BitPack"), ("ps_comment", "Str|[LZ4(sub=16384,hc=9),BitPack]")],
                     desc="partsupp: TPC-H SF={sf} partsupp, all 5 columns under Table 2's PS cascades, streamed "
                          "from pinned host"),
    # NEXT-1 microbenchmark: the paper's ANS instance
    "ans": dict(sf=10.0, dtype="u8", cols=[("l_returnflag", "ANS(chunk=4096)"), ("l_linestatus", "ANS(chunk=4096)")],
                desc="ANS: TPC-H SF={sf} lineitem l_returnflag + l_linestatus CHAR(1) under range ANS (4 KiB chunks)"),
    # NEXT-2 microbenchmark: Table 2's O_COMMENT cascade
    "strdict": dict(sf=10.0, dtype="u8", cols=[("o_comment", "Str|[StrDict|BitPack|ANS,BitPack]")],
                    desc="String-dictionary: TPC-H SF={sf} orders o_comment under Str|[StrDict|BitPack|ANS,BitPack]"),
    # BASELINE configs[0]: the oracle-sized parity case (launch-bound: 4 MB decoded)
    "config1": dict(sf=1.0, dtype="int32", cols=[("config1", "BitPack")],
                    desc="config 1: 1M int32, FOR + 8-bit bit-packing, one chunk"),
}
CHUNK_ROWS = 1 << 22
# kernel kinds of cdm_batch_kernel_times / _bytes grouped into families (the RLE chain's bytes sit on rle_kernel)
FAMILY_OF = {"fp_kernel": "fp_numeric", "fp_kernel(char)": "fp_char", "scan_kernel": "scan",
             "rle_sums_kernel": "rle_chain", "rle_kernel(level0)": "rle_chain", "rle_kernel": "rle_chain",
             "rle_big_kernel": "rle_chain", "lz4_kernel": "lz4", "ans_kernel": "ans", "strdict_kernel": "strdict",
             "device_copy": "copy"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="cdm", choices=["cdm", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--workload", default="config4", choices=sorted(WORKLOADS))
    p.add_argument("--sf", type=float, default=None, help="scale factor override")
    p.add_argument("--workers", type=int, default=None, help="generator/encoder processes per rank")
    p.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                   help="torch.distributed backend for N>1 (gloo: the one-GPU multi-rank test)")
    p.add_argument("--ingest", default="", help="config5: comma-separated devices whose PCIe links carry the H2D "
                   "copies (NEXT-4 multi-link ingestion, cdm_engine_set_ingest); empty = the rank's own link")
    p.add_argument("--device-map", default="local", choices=["local", "zero"],
                   help="local: rank -> cuda:LOCAL_RANK; zero: every rank on cuda:0 (tests on a single GPU)")
    a = p.parse_args()
    if a.sf is not None:
        WORKLOADS[a.workload]["sf"] = a.sf
    return a


def desc_of(wl) -> str:
    return wl["desc"].format(sf=f"{wl['sf']:g}")


def shard_select(cols, sf, rank, world):
    """{column index: this rank's chunk indices}: contiguous ranges balanced by row count (shard.py)."""
    from paper_2602_08190_b200 import workload
    from paper_2602_08190_b200.inputs import MASTER_SEED, TPCH
    from paper_2602_08190_b200.shard import shard_ranges
    gen = TPCH(sf, MASTER_SEED)
    sel = {}
    for k, (name, _) in enumerate(cols):
        n = workload._row_count(gen, name)
        nch = max(1, -(-n // CHUNK_ROWS))
        rows = [min(CHUNK_ROWS, n - c * CHUNK_ROWS) for c in range(nch)]
        a, b = shard_ranges(rows, world)[rank]
        sel[k] = list(range(a, b))
    return sel


def bind_cpus(local: int) -> list[int]:
    """Bind this process (and the workers it forks) to the CPUs NVML reports as close to the GPU."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(local)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = [64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1]
        cpus = [c for c in cpus if c < (os.cpu_count() or 1)]
        if cpus:
            os.sched_setaffinity(0, cpus)
        return sorted(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001 -- no NVML (CPU box): leave the affinity alone
        return sorted(os.sched_getaffinity(0))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """SM clocks + throttle reasons sampled through NVML every 2 ms during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.sm = []
        self.max_mhz = None
        self.reasons = set()
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001 -- no NVML: clocks unknown
            self.nv = None
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join(timeout=2)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml, 2 ms"}


def measure_h2d(torch, nbytes=256 << 20, reps=5):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record()
            d.copy_(h, non_blocking=True)
            b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    del h, d
    return nbytes / best / 1e6


def chunk_checksum_oracle(payload, offs, chunk_id: int) -> int:
    """H9 checksum of a decoded chunk (payload words under chunk_id, offsets words under chunk_id ^ 2^63)."""
    import oracle
    cs = oracle.checksum(payload, chunk_id)
    if offs is not None:
        cs = (cs + oracle.checksum(offs, chunk_id ^ (1 << 63))) % (1 << 64)
    return cs


def oracle_sample(samples, threads_list):
    """The oracle as it stands on the sample chunks: (decoded bytes, {threads: seconds}, per-chunk checksums)."""
    import oracle
    decoded = 0
    for _, _, ch in samples:
        r = oracle.oracle._header(ch)
        decoded += int(r[3]) + (4 * (int(r[2]) + 1) if r[0] == 4 else 0)
    times, outs = {}, None
    for th in threads_list:
        t0 = time.perf_counter()
        o = oracle.decode_many([c for _, _, c in samples], nthreads=th)
        times[th] = time.perf_counter() - t0
        outs = o
    sums = {}
    for (k, c, ch), (payload, offs) in zip(samples, outs):
        cid = int.from_bytes(ch[56:64].tobytes(), "little")
        sums[(k, c)] = chunk_checksum_oracle(payload, offs, cid)
    return decoded, times, sums


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle on the bounded sample of this arm's workload, K timed steps after W."""
    if rank != 0:
        return
    from paper_2602_08190_b200 import workload
    from paper_2602_08190_b200.inputs import MASTER_SEED
    import oracle
    wl = WORKLOADS[args.workload]
    samples = workload.sample_chunks(wl["cols"], wl["sf"], MASTER_SEED, CHUNK_ROWS, per_column=1)
    chunks = [c for _, _, c in samples]
    decoded = 0
    for c in chunks:
        r = oracle.oracle._header(c)
        decoded += int(r[3]) + (4 * (int(r[2]) + 1) if r[0] == 4 else 0)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle.decode_many(chunks, nthreads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.decode_many(chunks, nthreads=threads)
    dt = time.perf_counter() - t0
    v = decoded * args.steps / dt / 1e9
    sample = (f"each step = one oracle pass over the first chunk of every column ({len(chunks)} chunks, "
              f"{decoded / 1e6:.1f} MB decoded) of the {desc_of(wl).split(':')[0]} workload at SF={wl['sf']:g}")
    line = {"metric": METRIC, "value": v, "unit": "GB/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": wl["dtype"],
            "data": "synthetic", "config": {"workload": desc_of(wl), "chunk_rows": CHUNK_ROWS,
                                            "decoded_bytes_per_step": decoded},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": threads, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_config5(args, rank, world, local, local_world):
    """BASELINE configs[4]: SF=1000 lineitem in 8 virtual slices (each column's chunks
    split into 8 contiguous ranges, shard.py); rank r streams slice r (weak scaling, N <= 8) from
    pinned host memory through cdm_submit_batch windows whose outputs land in a two-half OUTPUT RING (not
    retained): window j+1 is submitted before window j is waited, the engine computes every chunk's H9
    checksum on the device right after its decode (CDM_ENGINE_CHECKSUM), so the outputs can be overwritten.
    value = decoded bytes of all slices / wall time of the streaming pass (max over ranks); parity: the GPU
    checksums of a deterministic 1 % chunk sample equal the oracle's."""
    from paper_2602_08190_b200 import workload
    from paper_2602_08190_b200.inputs import MASTER_SEED
    wl = WORKLOADS["config5"]
    # weak scaling: rank r of N <= 8 decodes slice r (one GPU's share of the 8-GPU configuration)
    slices = [rank] if world <= 8 else ([rank] if rank < 8 else [])
    cpus = bind_cpus(local)
    sel = {}
    for s_ in slices:
        for k, idx in shard_select(wl["cols"], wl["sf"], s_, 8).items():
            sel.setdefault(k, []).extend(idx)
    workers = args.workers or max(1, len(cpus) // max(1, local_world))
    ds = workload.build(wl["cols"], wl["sf"], MASTER_SEED, CHUNK_ROWS, select=sel, workers=workers)
    import torch
    import torch.distributed as dist
    from paper_2602_08190_b200 import cdm
    dev = local if args.device_map == "local" else 0
    torch.cuda.set_device(dev)
    coll = "cuda" if args.dist_backend == "nccl" else "cpu"
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    pinned = cdm.PinnedBuffer(ds.used)
    src = ds.array()
    for a in range(0, ds.used, 1 << 28):
        pinned.array[a: a + (1 << 28)] = src[a: a + (1 << 28)]
    del src
    ds.rebind(pinned.array)
    host_all = pinned.array

    def up(x):
        return (x + 255) // 256 * 256
    # chunks per window (one submit_batch); windows in flight = output ring sections.  Measured on B200 (slice 0):
    # W 128 / DEPTH 2 / 4 staging slots 196 GB/s (bar 181); W 32 158-161 GB/s; DEPTH 3 with 12 slots 79 GB/s
    W = int(os.environ.get("CDM_C5_WINDOW", "128"))
    DEPTH = 2
    slot_out = max(up(max(c.payload, 16)) + up(c.offsets) for c in ds.chunks)
    ring = torch.empty(DEPTH * W * slot_out, dtype=torch.uint8, device="cuda")
    cascs = [cdm.Cascade(spec, dt, w) for (_, spec, dt, w) in ds.columns]
    max_chunk = max(c.size for c in ds.chunks)
    eng = cdm.Engine(dev, n_slots=4, slot_bytes=max(64 << 20, (max_chunk + (1 << 20) - 1) // (1 << 20) * (1 << 20)),
                     order_policy=1, checksum=True)
    if args.ingest:
        eng.set_ingest([int(x) for x in args.ingest.split(",")])
    order = sorted(range(len(ds.chunks)), key=lambda i: (ds.chunks[i].index, ds.chunks[i].column))  # row order
    windows = [order[a: a + W] for a in range(0, len(order), W)]
    decs = []
    for wi, win in enumerate(windows):
        half = (wi % DEPTH) * W
        row = []
        for j, i in enumerate(win):
            c = ds.chunks[i]
            base = (half + j) * slot_out
            out = ring[base: base + up(max(c.payload, 16))]
            offs = ring[base + up(max(c.payload, 16)): base + up(max(c.payload, 16)) + c.offsets].view(torch.int32) \
                if c.offsets else None
            row.append(cdm.Decode(cascs[c.column], host_all[c.offset: c.offset + c.size], out, offs))
        decs.append(row)
    sums, err = {}, 0

    def one_pass():
        nonlocal err
        pending = []

        def drain():
            nonlocal err
            pw, pt = pending.pop(0)
            for i, tk in zip(windows[pw], pt):
                r = eng.wait(tk, raise_on_error=False)
                err |= r["error_bits"]
                sums[i] = r["checksum"]
        for wi, row in enumerate(decs):
            if len(pending) == DEPTH:  # its ring section is reused by this window
                drain()
            pending.append((wi, eng.submit_batch(row)))
        while pending:
            drain()
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        one_pass()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    walls = []
    l0 = eng.launches()
    with ClockSampler(dev) as clocks:
        for _ in range(args.steps):
            t0 = time.perf_counter()
            one_pass()
            walls.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    launches = eng.launches() - l0
    wall = sum(walls)
    decoded, compressed = ds.decoded, ds.compressed
    checksum_total = sum(sums.values()) % (1 << 64)
    h2d = measure_h2d(torch)
    # parity + cpu_baseline: a deterministic 1 % chunk sample (every 100th chunk of the slice in row order)
    sample = [order[i] for i in range(0, len(order), 100)]
    samples = [(ds.chunks[i].column, ds.chunks[i].index, ds.host(ds.chunks[i]).copy()) for i in sample]
    threads = os.cpu_count() or 1
    sdec, stimes, osums = oracle_sample(samples, [threads])
    gsum = {(ds.chunks[i].column, ds.chunks[i].index): sums[i] for i in sample}
    mism = [k for k, v in osums.items() if gsum.get(k) != v]
    n_chunks = len(ds.chunks)
    if world > 1:
        meta = torch.tensor([decoded, compressed, n_chunks, err, len(mism)], dtype=torch.int64, device=coll)
        dist.all_reduce(meta)
        t = torch.tensor([wall], dtype=torch.float64, device=coll)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        decoded, compressed, n_chunks, err, nmism = [int(x) for x in meta.tolist()]
        wall = float(t.item())
    else:
        nmism = len(mism)
    if rank == 0:
        value = decoded * args.steps / wall / 1e9
        cr = decoded / compressed
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(wall * 1e3 / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": wl["dtype"], "data": "synthetic",
            "config": {"workload": desc_of(wl), "sf": wl["sf"], "slices": slices, "slices_total": 8,
                       "chunk_rows": CHUNK_ROWS, "columns": len(ds.columns), "chunks": n_chunks,
                       "decoded_bytes_per_step": decoded, "compressed_bytes_per_step": compressed,
                       "compression_ratio": round(cr, 3), "window_chunks": W, "windows_in_flight": DEPTH,
                       "ingest_devices": args.ingest or None,
                       "output_ring_bytes": int(ring.numel()),
                       "parallelism": f"{world} rank(s) x their 1/8 slices of one SF=1000 dataset",
                       "l2": "inputs and outputs exceed the 126 MB L2",
                       "timing": "host wall clock of a streaming pass (submit_batch windows + waits), max over ranks",
                       "host": {"build_s": round(ds.build_s, 1), "build_workers": ds.workers,
                                "pinned_bytes": ds.used}},
            "e2e": {"value": round(value, 2), "unit": "GB/s", "h2d_bytes_per_step": compressed,
                    "d2h_bytes_per_step": 12 * n_chunks, "pcie_h2d_gbs_measured": round(h2d, 1),
                    "bar_cr_x_0.8_x_pcie": round(cr * 0.8 * h2d * world, 1),
                    "how": "the value is already end to end: pinned host -> H2D -> decode -> per-chunk error word and "
                           "checksum read back (cdm_submit_batch / cdm_wait)"},
            "parity": {"chunks_checked_vs_oracle": len(osums) * (world if world > 1 else 1), "mismatches": nmism,
                       "checksum_total_rank0": f"{checksum_total:016x}", "errors": err,
                       "sample": "every 100th chunk of each slice in row order (1 %)"},
            "cpu_baseline": {"value": round(sdec / stimes[threads] / 1e9, 4), "unit": "GB/s", "cores": threads,
                             "kind": "oracle", "cpu_model": cpu_model(),
                             "sample": f"{len(samples)} chunks (1 % of rank 0's slice), {sdec / 1e6:.1f} MB decoded, "
                                       f"{stimes[threads]:.2f} s on {threads} threads"},
            "gpu_launches": launches, "clocks": clocks.summary(), "errors": err}
        print(json.dumps(line), flush=True)
    eng.close()
    del decs, ring
    pinned.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.workload == "config5":
        run_config5(args, rank, world, local, local_world)
        return
    from paper_2602_08190_b200 import workload
    from paper_2602_08190_b200.inputs import MASTER_SEED
    wl = WORKLOADS[args.workload]
    cpus = bind_cpus(local)

    # ------------------------------------------------------------ this rank's shard (untimed; forks workers,
    # so it runs before CUDA is initialised)
    sel = shard_select(wl["cols"], wl["sf"], rank, world) if world > 1 else None
    workers = args.workers or max(1, len(cpus) // max(1, local_world) if world > 1 else len(cpus))
    ds = workload.build(wl["cols"], wl["sf"], MASTER_SEED, CHUNK_ROWS, select=sel, workers=workers)

    import torch
    import torch.distributed as dist
    from paper_2602_08190_b200 import cdm

    dev = local if args.device_map == "local" else 0
    torch.cuda.set_device(dev)
    coll = "cuda" if args.dist_backend == "nccl" else "cpu"  # device of the collectives' tensors
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    # the column store moves into page-locked host memory (cudaHostAlloc through cdm_host_alloc: registering
    # the workers' shared mapping in place is refused by the driver on this VM)
    t0 = time.perf_counter()
    pinned = cdm.PinnedBuffer(ds.used)
    pin_s = time.perf_counter() - t0
    src = ds.array()
    step = 1 << 28
    for a in range(0, ds.used, step):
        pinned.array[a: a + step] = src[a: a + step]
    host_all = pinned.array
    copy_s = time.perf_counter() - t0 - pin_s
    del src
    ds.rebind(host_all)
    host_t = torch.from_numpy(host_all)

    compressed, decoded, n_chunks = ds.compressed, ds.decoded, len(ds.chunks)
    # one device buffer for every chunk's outputs (payload + offsets, 256-byte aligned slices) and one for the
    # device-resident copy of the compressed chunks
    def up(x):
        return (x + 255) // 256 * 256
    out_bytes = sum(up(max(c.payload, 16)) + up(c.offsets) for c in ds.chunks)
    out_all = torch.empty(max(out_bytes, 256), dtype=torch.uint8, device="cuda")
    dev_all = torch.empty(max(ds.used, 256), dtype=torch.uint8, device="cuda")
    copy_stream = torch.cuda.Stream()
    with torch.cuda.stream(copy_stream):
        dev_all[: ds.used].copy_(host_t, non_blocking=True)
    copy_stream.synchronize()

    max_chunk = max(c.size for c in ds.chunks)
    slot = max(64 << 20, (max_chunk + (1 << 20) - 1) // (1 << 20) * (1 << 20))
    eng = cdm.Engine(dev, n_slots=4, slot_bytes=slot, order_policy=1)
    cascs = [cdm.Cascade(spec, dt, w) for (_, spec, dt, w) in ds.columns]
    decs_dev, decs_host, views = [], [], []
    pos = 0
    for c in ds.chunks:
        pb = up(max(c.payload, 16))
        out = out_all[pos: pos + pb]
        pos += pb
        offs = None
        if c.offsets:
            offs = out_all[pos: pos + c.offsets].view(torch.int32)
            pos += up(c.offsets)
        host = host_all[c.offset: c.offset + c.size]
        decs_dev.append(cdm.Decode(cascs[c.column], host, out, offs, dev_chunk=dev_all[c.offset: c.offset + c.size]))
        decs_host.append(cdm.Decode(cascs[c.column], host, out, offs))
        views.append((out, offs))
    stream = torch.cuda.Stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    err_bits = 0

    # ------------------------------------------------------------ (value) pipelined host -> device decode
    pipe = cdm.Pipeline(eng, decs_host)
    pinfo = pipe.info()
    for _ in range(args.warmup):
        pipe.launch(stream)
        for r in pipe.results(raise_on_error=False):
            err_bits |= r["error_bits"]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    wall = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clocks:
        for k in range(args.steps):
            t0 = time.perf_counter()
            ev[k][0].record(stream)
            pipe.launch(stream)                     # every compressed byte crosses PCIe + every chunk decodes
            ev[k][1].record(stream)
            for r in pipe.results(raise_on_error=False):  # per-chunk error words on the host
                err_bits |= r["error_bits"]
            wall.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    pipe_ms = sum(a.elapsed_time(b) for a, b in ev)
    e2e_s = sum(wall)
    launches = pinfo["kernel_launches"] * args.steps

    # ------------------------------------------------------------ H9 parity: checksums of every chunk output
    gpu_sums = {}
    for c, (out, offs) in zip(ds.chunks, views):
        cs = cdm.checksum(out[: c.payload], c.chunk_id, stream)
        if offs is not None:
            cs = (cs + cdm.checksum(offs, c.chunk_id ^ (1 << 63), stream)) % (1 << 64)
        gpu_sums[(c.column, c.index)] = cs
    checksum_total = sum(gpu_sums.values()) % (1 << 64)

    # ------------------------------------------------------------ device-resident decode (kernel level)
    batch = cdm.Batch(eng, decs_dev)
    batch.set_graph(True)
    kbytes = batch.kernel_bytes()
    for _ in range(args.warmup):
        batch.launch(stream)
    for r in batch.results(stream, raise_on_error=False):
        err_bits |= r["error_bits"]
    dev_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    with ClockSampler(dev) as dev_clocks:
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()                      # L2 flush (256 MiB write), outside the events
                dev_ev[k][0].record(stream)
                batch.launch(stream)
                dev_ev[k][1].record(stream)
        torch.cuda.synchronize()
    dev_ms = sum(a.elapsed_time(b) for a, b in dev_ev)
    for r in batch.results(stream, raise_on_error=False):
        err_bits |= r["error_bits"]

    # ------------------------------------------------------------ serialized (E11): copy everything, then decode
    ser_ev = []
    for k in range(max(2, min(args.steps, 3))):
        a, m, b = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        with torch.cuda.stream(stream):
            a.record(stream)
            dev_all[: ds.used].copy_(host_t, non_blocking=True)
            m.record(stream)
            batch.launch(stream)
            b.record(stream)
        ser_ev.append((a, m, b))
    torch.cuda.synchronize()
    ser_ms = [a.elapsed_time(b) for a, _, b in ser_ev]
    ser_copy_ms = [a.elapsed_time(m) for a, m, _ in ser_ev]
    for r in batch.results(stream, raise_on_error=False):
        err_bits |= r["error_bits"]

    # ------------------------------------------------------------ per-kernel (alone) and per-family timing
    tsteps = max(1, min(args.steps, 3))
    timing = {}
    batch.set_graph(False)
    for mode in (2, 1):
        batch.set_timing(mode)
        batch.launch(stream)
        batch.results(stream, raise_on_error=False)
        batch.set_timing(mode)
        for k in range(tsteps):
            with torch.cuda.stream(stream):
                flush.zero_()
                batch.launch(stream)
        for r in batch.results(stream, raise_on_error=False):
            err_bits |= r["error_bits"]
        timing[mode] = batch.kernel_times() if mode == 2 else batch.kernel_ms()
    ktimes, fams_conc = timing[2], timing[1]
    batch.close()
    h2d_alone = measure_h2d(torch) if rank == 0 or world == 1 else None
    # H2D denominators: each rank alone (one after another), then all ranks concurrently
    h2d_each = None
    h2d_conc = None
    if world > 1:
        h2d_each = []
        for r in range(world):
            dist.barrier()
            v = measure_h2d(torch) if rank == r else 0.0
            t = torch.tensor([v], dtype=torch.float64, device=coll)
            dist.all_reduce(t)
            h2d_each.append(round(float(t.item()), 1))
        dist.barrier()
        v = measure_h2d(torch)
        t = torch.zeros(world, dtype=torch.float64, device=coll)
        t[rank] = v
        dist.all_reduce(t)
        h2d_conc = [round(float(x), 1) for x in t.tolist()]
        h2d_alone = h2d_each[rank]

    # ------------------------------------------------------------ reduce over ranks (metadata only)
    pipe_s, dev_s = pipe_ms / 1e3, dev_ms / 1e3
    if world > 1:
        meta = torch.tensor([decoded, compressed, n_chunks, err_bits], dtype=torch.int64, device=coll)
        dist.all_reduce(meta, op=dist.ReduceOp.SUM)
        cs = torch.tensor([checksum_total & 0xFFFFFFFF, checksum_total >> 32], dtype=torch.int64, device=coll)
        dist.all_reduce(cs, op=dist.ReduceOp.SUM)  # 32-bit halves summed exactly, recombined mod 2^64
        tmax = torch.tensor([pipe_s, e2e_s, dev_s], dtype=torch.float64, device=coll)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tot_decoded, tot_comp, tot_chunks, tot_err = [int(x) for x in meta.tolist()]
        lo, hi = [int(x) for x in cs.tolist()]
        checksum_total = (lo + (hi << 32)) % (1 << 64)
        pipe_s, e2e_s, dev_s = [float(x) for x in tmax.tolist()]
    else:
        tot_decoded, tot_comp, tot_chunks, tot_err = decoded, compressed, n_chunks, err_bits

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # bounded sample: the first chunk of every column, decoded by the oracle on 1 thread and on all cores
        samples = [(c.column, c.index, ds.host(c).copy()) for c in ds.chunks if c.index == 0]
        threads = os.cpu_count() or 1
        sdec, stimes, osums = oracle_sample(samples, [1, threads])
        mism = [k for k, v in osums.items() if gpu_sums.get(k) != v]
        cpu = {"value": round(sdec / stimes[threads] / 1e9, 4), "unit": "GB/s", "cores": threads, "kind": "oracle",
               "one_thread": {"value": round(sdec / stimes[1] / 1e9, 4), "cores": 1},
               "cpu_model": cpu_model(),
               "sample": f"the first chunk (2^22 rows) of each of the {len(samples)} columns, {sdec / 1e6:.1f} MB "
                         f"decoded, one oracle pass on {threads} threads ({stimes[threads]:.2f} s) and one on 1 "
                         f"thread ({stimes[1]:.2f} s)"}
        parity = {"chunks_checked_vs_oracle": len(osums), "mismatches": len(mism),
                  "mismatched": [list(k) for k in mism[:8]]}
    else:
        parity = {"chunks_checked_vs_oracle": 0, "mismatches": 0}

    if rank == 0:
        peak, peak_src = load_peaks()
        value = tot_decoded * args.steps / pipe_s / 1e9
        e2e = tot_decoded * args.steps / e2e_s / 1e9
        dev_v = tot_decoded * args.steps / dev_s / 1e9
        cr = tot_decoded / tot_comp
        # rooflines: each kernel kind alone (events around each launch) against its algorithmic bytes
        fam_ms, fam_bytes, fam_n = {}, {}, {}
        for kname, (ms, n) in ktimes.items():
            f = FAMILY_OF[kname]
            if n:
                fam_ms[f] = fam_ms.get(f, 0.0) + ms / tsteps
                fam_n[f] = fam_n.get(f, 0) + n / tsteps
            fam_bytes[f] = fam_bytes.get(f, 0) + kbytes.get(kname, 0)
        families = {}
        for f, ms in sorted(fam_ms.items(), key=lambda x: -x[1]):
            b = fam_bytes.get(f, 0)
            gbs = b / (ms / 1e3) / 1e9 if ms > 0 else 0.0
            families[f] = {"ms_per_step": round(ms, 4), "algorithmic_bytes": b, "achieved_gbs": round(gbs, 1),
                           "frac": round(gbs / peak, 4), "launches_per_step": round(fam_n.get(f, 0), 2)}
        dom = max(families, key=lambda f: families[f]["ms_per_step"])
        lanes = cdm.tune_get("lz4_lanes")
        kern_of = {"fp_numeric": "fp_kernel", "fp_char": "fpc_kernel (CHAR(n) row groups)",
                   "scan": "scan_sums_kernel+scan_kernel_rts" if cdm.tune_get("scan_mode") == 0 else "scan_kernel_lb",
                   "rle_chain": "rle_sums_kernel+rle_kernel(+level0, rle_big_kernel)",
                   "lz4": "lz4_thread_kernel" if lanes == 1 else "lz4_kernel" if lanes == 32 else "lz4_group_kernel",
                   "ans": "ans_warp_kernel", "strdict": "sd_sums+sd_scan+sd_expand", "copy": "cudaMemcpyAsync D2D"}
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                traffic = json.load(f).get(f"{args.workload}:{kern_of[dom]}")
        conc = {k: round(v[0] / tsteps, 4) for k, v in fams_conc.items() if v[1]}
        crit = max(conc, key=conc.get) if conc else None
        cfg = {"workload": desc_of(wl), "sf": wl["sf"], "chunk_rows": CHUNK_ROWS, "columns": len(ds.columns),
               "chunks": tot_chunks, "decoded_bytes_per_step": tot_decoded, "compressed_bytes_per_step": tot_comp,
               "compression_ratio": round(cr, 3),
               "parallelism": f"dp{world}: one dataset, per-rank contiguous chunk ranges (strong scaling)",
               "l2": f"inputs ({tot_comp / 1e9:.1f} GB compressed) and outputs ({tot_decoded / 1e9:.1f} GB) exceed the "
                     "126 MB L2; the device-resident pass also flushes L2 (256 MiB write) before each step",
               "timing": "value: CUDA events on the launching stream around each cdm_pipeline_launch (sum over "
                         "steps, max over ranks); e2e: host wall clock of launch + results",
               "host": {"cpus_bound": len(cpus), "build_s": round(ds.build_s, 1), "build_workers": ds.workers,
                        "pin_alloc_s": round(pin_s, 2), "pin_copy_s": round(copy_s, 2), "pinned_bytes": ds.used},
               "pipeline": pinfo}
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(pipe_s * 1e3 / args.steps, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": wl["dtype"], "data": "synthetic", "config": cfg,
            "e2e": {"value": round(e2e, 2), "unit": "GB/s", "h2d_bytes_per_step": tot_comp,
                    "d2h_bytes_per_step": 4 * tot_chunks, "ms_per_step": round(e2e_s * 1e3 / args.steps, 3),
                    "how": "cdm_pipeline_launch + cdm_pipeline_results per step, host wall clock: every compressed "
                           "chunk copied H2D from pinned host and decoded, every chunk's error word read back",
                    "pcie_h2d_gbs_measured": round(h2d_alone, 1) if h2d_alone else None,
                    "pcie_h2d_gbs_achieved_in_pipeline": round(tot_comp * args.steps / e2e_s / 1e9 / max(world, 1), 1),
                    "pcie_h2d_gbs_each_rank_alone": h2d_each, "pcie_h2d_gbs_all_ranks_concurrent": h2d_conc,
                    "bar_cr_x_0.8_x_pcie": round(cr * 0.8 * h2d_alone * (world if world > 1 else 1), 1)
                    if h2d_alone else None,
                    "serialized": {"value": round(tot_decoded / (statistics.median(ser_ms) / 1e3) / 1e9, 2)
                                   if world == 1 else None,
                                   "ms_per_step": round(statistics.median(ser_ms), 3),
                                   "copy_ms": round(statistics.median(ser_copy_ms), 3),
                                   "how": "E11 (PAPER.md:654-657): one H2D copy of all compressed bytes, then the "
                                          "device-resident decode, no overlap (rank 0)"}},
            "device_resident": {"value": round(dev_v, 2), "unit": "GB/s",
                                "ms_per_step": round(dev_s * 1e3 / args.steps, 3),
                                "decoded_written_over_8tbs": round(dev_v / 8000.0, 4),
                                "clocks": dev_clocks.summary(),
                                "how": "one CUDA-graph replay of the whole fused decode of every chunk already in "
                                       "HBM, CUDA events on the launching stream, L2 flushed between steps"},
            "roofline": {"bound": "hbm", "achieved": families[dom]["achieved_gbs"], "peak": peak, "unit": "GB/s",
                         "frac": families[dom]["frac"], "traffic": traffic, "kernel": kern_of[dom], "family": dom,
                         "launches_per_step": families[dom]["launches_per_step"],
                         "algorithmic_bytes_per_launch": int(families[dom]["algorithmic_bytes"] /
                                                             max(families[dom]["launches_per_step"], 1)),
                         "traffic_how": "ncu --set full DRAM read + write bytes of ONE launch of this kernel in this "
                                        "workload (profiles/ncu_traffic.json), per launch like algorithmic_bytes_per_launch",
                         "algorithmic_bytes_per_step": families[dom]["algorithmic_bytes"],
                         "kernel_ms_per_step": families[dom]["ms_per_step"], "peak_source": peak_src,
                         "families": families, "families_concurrent_ms": conc, "critical_path_family": crit,
                         "timing": f"CUDA events around each kernel launch (each kernel alone, families serialised) "
                                   f"over {tsteps} device-resident steps after L2 flushes; bytes from "
                                   "cdm_batch_kernel_bytes (Eq. 1)"},
            "parity": dict(parity, checksum_total=f"{checksum_total:016x}", chunks_checksummed_on_gpu=tot_chunks,
                           errors=tot_err),
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "errors": tot_err,
        }
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    pipe.close()
    eng.close()
    del decs_host, decs_dev, host_t
    pinned.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def build_workload(rank: int, workload: str = "config2", sf: float | None = None):
    """Compatibility helper for tests: [(name, spec, dtype, width, [chunk numpy arrays], plain bytes)]."""
    from paper_2602_08190_b200 import workload as W
    from paper_2602_08190_b200.inputs import MASTER_SEED
    wl = WORKLOADS[workload]
    ds = W.build(wl["cols"], sf if sf is not None else wl["sf"], MASTER_SEED + 1000 * rank, CHUNK_ROWS)
    out = []
    for k, (name, spec, dt, w) in enumerate(ds.columns):
        chs = [ds.host(c).copy() for c in ds.chunks if c.column == k]
        plain = sum(c.plain for c in ds.chunks if c.column == k)
        out.append((name, spec, dt, w, chs, plain))
    return out


if __name__ == "__main__":
    main()
