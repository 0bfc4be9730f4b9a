"""The C-ABI boundary's concurrency and completion contract on the GPU (include/cdm.h):
thread-safe cdm_submit* / cdm_wait on one engine, cdm_ticket_event for consumers that chain on a decode without a
host synchronisation, and the H9 checksum an engine created with CDM_ENGINE_CHECKSUM returns in cdm_result.
Every decoded byte is compared with the CPU oracle (-m gpu)."""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
from paper_2602_08190_b200 import cdm, encoder
from paper_2602_08190_b200.inputs import TPCH

pytestmark = pytest.mark.gpu

CASES = [("l_orderkey", "RLE|[Delta|RLE|[BitPack,BitPack],BitPack]"), ("l_quantity", "Dict|BitPack"),
         ("l_shipmode", "Dict|BitPack"), ("l_comment", "Str|[LZ4,BitPack]"), ("o_orderkey", "Delta|BitPack")]


def _chunks():
    g = TPCH(0.01)
    out = []
    for name, spec in CASES:
        col = g.column(name)
        casc = cdm.Cascade(spec, col.dtype, col.width)
        for ch in encoder.encode_chunks(spec, col, 20_011):
            out.append((casc, ch))
    return out


def _decodes(items):
    decs, bufs = [], []
    for casc, ch in items:
        out, offs = cdm.output_buffers(ch)
        decs.append(cdm.Decode(casc, cdm.pinned(ch), out, offs))
        bufs.append((ch, out, offs))
    return decs, bufs


def _check(bufs):
    for ch, out, offs in bufs:
        exp, exp_offs = oracle.decode_chunk(ch)
        assert np.array_equal(out.cpu().numpy()[: exp.size], exp)
        if exp_offs is not None:
            assert np.array_equal(offs.cpu().numpy()[: exp_offs.size], exp_offs)


@pytest.fixture(scope="module")
def items():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return _chunks()


def test_concurrent_submit_and_wait(items):
    """four host threads drive ONE engine (cdm_submit_batch / cdm_submit / cdm_wait interleaved)"""
    eng = cdm.Engine(0, n_slots=3, slot_bytes=64 << 20)
    errors = []

    def worker(k):
        try:
            for rep in range(3):
                sel = items[k::4]
                decs, bufs = _decodes(sel)
                if rep % 2 == 0:
                    tickets = eng.submit_batch(decs)
                else:
                    tickets = [eng.submit(d) for d in decs]
                for t in reversed(tickets):  # waits out of order
                    eng.wait(t)
                torch.cuda.synchronize()
                _check(bufs)
        except Exception as e:  # noqa: BLE001 -- reported by the main thread
            errors.append(repr(e))

    ths = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    eng.close()
    assert not errors, errors[:3]


def test_ticket_event_orders_a_consumer_stream(items):
    """a consumer stream that waits on cdm_ticket_event's event sees the decoded bytes (no host sync first)"""
    from cuda.bindings import runtime as rt
    eng = cdm.Engine(0)
    decs, bufs = _decodes(items)
    tickets = eng.submit_batch(decs)
    consumer = torch.cuda.Stream()
    copies = []
    for t, (ch, out, offs) in zip(tickets, bufs):
        ev = eng.ticket_event(t)
        assert ev
        err, = rt.cudaStreamWaitEvent(consumer.cuda_stream, ev, 0)
        assert err == rt.cudaError_t.cudaSuccess
        with torch.cuda.stream(consumer):
            copies.append((ch, out.clone(), None if offs is None else offs.clone()))
    consumer.synchronize()
    _check(copies)
    for t in tickets:
        eng.wait(t)
    # a consumed ticket has no event; a harvested group's tickets get an event that has completed
    with pytest.raises(cdm.CdmError):
        eng.ticket_event(tickets[0])
    t2 = eng.submit_batch(decs[:2])
    eng.synchronize()
    ev = eng.ticket_event(t2[0])
    assert rt.cudaEventQuery(ev)[0] == rt.cudaError_t.cudaSuccess
    for t in t2:
        eng.wait(t)
    eng.close()


def test_engine_checksum_matches_oracle(items):
    """CDM_ENGINE_CHECKSUM: cdm_result.checksum == the oracle's H9 checksum of the same chunk"""
    eng = cdm.Engine(0, checksum=True)
    decs, bufs = _decodes(items)
    res = [eng.wait(t) for t in eng.submit_batch(decs)]
    for r, (ch, _, _) in zip(res, bufs):
        exp, exp_offs = oracle.decode_chunk(ch)
        cid = int.from_bytes(ch[56:64].tobytes(), "little")
        want = oracle.checksum(exp, cid)
        if exp_offs is not None:
            want = (want + oracle.checksum(exp_offs, cid ^ (1 << 63))) % (1 << 64)
        assert r["checksum"] == want
    plain = cdm.Engine(0)
    r0 = plain.wait(plain.submit(decs[0]))
    assert r0["checksum"] == 0
    plain.close()
    eng.close()


def test_multi_link_ingestion_path(items):
    """NEXT-4: cdm_engine_set_ingest routes each group's H2D copy through an ingest device's own
    staging buffer and stream, then a peer (here device-to-device) copy into the engine's slot.  With one GPU the
    ingest devices are the engine's own device twice (two buffers / streams, round-robin): every byte still equals
    the oracle's, the checksum path is unchanged, and clearing the list restores direct copies."""
    eng = cdm.Engine(0, n_slots=3, slot_bytes=64 << 20, checksum=True)
    eng.set_ingest([0, 0])
    for rep in range(2):
        decs, bufs = _decodes(items)
        res = [eng.wait(t) for t in eng.submit_batch(decs)]
        torch.cuda.synchronize()
        _check(bufs)
        assert all(r["error_bits"] == 0 for r in res)
    eng.set_ingest([])
    decs, bufs = _decodes(items[:3])
    for t in eng.submit_batch(decs):
        eng.wait(t)
    torch.cuda.synchronize()
    _check(bufs)
    with pytest.raises(cdm.CdmError):
        eng.set_ingest([99])
    eng.close()
