"""The speculative parallel header parse of `lz4_spec_kernel`, modelled on the CPU and checked
against the plain sequential chain on real (liblz4 HC-9) and byte-mutated LZ4 blocks.

The kernel's claim: 32 segment walks started at arbitrary bytes, a fix-up that re-walks each segment from its true
entry only until it meets a position marked by its own speculative walk, iterated until no segment exit changes,
leave a bitmask that is EXACTLY the set of header positions of the sequential parse (the LZ4 block format).
This model follows the kernel's steps (word-aligned segments, marks, fix-up rounds, clear-and-set) in plain
Python; the reference is the obvious sequential walk."""
import struct

import numpy as np
import pytest

from paper_2602_08190_b200 import encoder
from paper_2602_08190_b200.inputs import TPCH

import cdm1


def nxt(c: bytes, p: int) -> int:
    """position of the next header after a header at p (len(c): a literal-only last sequence; len(c)+1: overrun)"""
    cl = len(c)
    t = c[p]
    q, lit = p + 1, t >> 4
    if lit == 15:
        while True:
            if q >= cl:
                return cl + 1
            b = c[q]
            q += 1
            lit += b
            if b != 255:
                break
    if lit > cl - q:
        return cl + 1
    q += lit
    if q == cl:
        return cl
    if cl - q < 2:
        return cl + 1
    q += 2
    if t & 15 == 15:
        while True:
            if q >= cl:
                return cl + 1
            b = c[q]
            q += 1
            if b != 255:
                break
    return q


def sequential_headers(c: bytes) -> set:
    out, p = set(), 0
    while p < len(c):
        out.add(p)
        p = nxt(c, p)
    return out


def speculative_headers(c: bytes) -> tuple:
    cl = len(c)
    nwords = (cl + 31) // 32
    L = 32 * ((nwords + 31) // 32)
    marks = [set() for _ in range(32)]
    ex = [0] * 32
    for j in range(32):  # speculative walks
        s0, e = j * L, min(j * L + L, cl)
        p = s0
        while p < e:
            marks[j].add(p)
            p = nxt(c, p)
        ex[j] = p if s0 < cl else s0
    E = ex[:]
    entry, mpos, walked, tprev = [j * L for j in range(32)], [j * L for j in range(32)], [False] * 32, [0] * 32
    rounds = 0
    for _ in range(33):  # fix-up rounds (all lanes in parallel: entries from the previous round's exits)
        rounds += 1
        prev = E[:]
        changed = False
        for j in range(32):
            s0, e = j * L, min(j * L + L, cl)
            if s0 >= cl:
                continue
            t = 0 if j == 0 else prev[j - 1]
            if walked[j] and t == tprev[j]:
                continue
            p = t
            while p < e and p not in marks[j]:
                p = nxt(c, p)
            nE = ex[j] if p < e else p
            entry[j], mpos[j] = t, (p if p < e else e)
            changed |= nE != E[j]
            E[j], tprev[j], walked[j] = nE, t, True
        if not changed:
            break
    heads = set()
    for j in range(32):  # clear [s0, mpos), set the re-walked chain [entry, mpos)
        s0 = j * L
        if s0 >= cl:
            continue
        keep = {p for p in marks[j] if p >= mpos[j]}
        p = entry[j]
        while p < mpos[j]:
            keep.add(p)
            p = nxt(c, p)
        heads |= keep
    return heads, rounds


def _blocks(spec: str, sf: float = 0.002, limit: int = 24):
    col = TPCH(sf).column("l_comment")
    subs = []
    for ch in encoder.encode_chunks(spec, col, 3000)[:4]:
        _, _, streams = cdm1.parse(ch)
        pay, tab = streams[0], streams[1]
        for s in range(len(tab) // 12):
            co, cl, _ = struct.unpack_from("<III", tab, 12 * s)
            subs.append(bytes(pay[co:co + cl]))
    return subs[:limit]


@pytest.mark.parametrize("spec", ["Str|[LZ4(sub=16384,hc=9),BitPack]", "Str|[LZ4(sub=4096),BitPack]"])
def test_speculative_parse_finds_the_sequential_chain(spec):
    for c in _blocks(spec):
        heads, rounds = speculative_headers(c)
        assert heads == sequential_headers(c)
        assert rounds < 33  # converged before the kernel's iteration cap (16 KiB HC-9 blocks: 1-3 rounds; 4 KiB
        # blocks have 32-byte segments, where a wrong chain may cross a whole segment before merging: up to ~6)


def test_speculative_parse_on_mutated_and_adversarial_bytes():
    rng = np.random.default_rng(3)
    base = _blocks("Str|[LZ4(sub=16384,hc=9),BitPack]", limit=6)
    cases = []
    for c in base:
        for _ in range(6):
            b = bytearray(c)
            for _ in range(int(rng.integers(1, 6))):
                b[int(rng.integers(0, len(b)))] = int(rng.integers(0, 256))
            cases.append(bytes(b))
    # long literal runs spanning several segments, and random bytes
    cases.append(bytes([0xF0, 255, 255, 255, 255, 10]) + bytes(1040))
    cases += [rng.integers(0, 256, size=int(n), dtype=np.uint8).tobytes() for n in (1, 2, 31, 33, 1000, 5000)]
    for c in cases:
        heads, _ = speculative_headers(c)
        assert heads == sequential_headers(c)
