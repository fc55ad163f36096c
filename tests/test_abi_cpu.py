"""CPU-side checks of the C-ABI library (no compute calls that need a GPU).

* the library loads and exports every symbol include/recsplit.h declares;
* its host tables (tau) agree with the oracle's for every reachable node class;
* its host query reads the oracle's serialized format (cross-check of two
  independent readers/writers of DESIGN.md section 6);
* without a GPU the build fails loudly (RECSPLIT_E_CUDA) -- there is no CPU fallback.
"""
from __future__ import annotations

import os
import re

import numpy as np
import pytest
import torch

import oracle
import paper_2212_09562_b200 as rs
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "recsplit.h")).read()
    declared = set(re.findall(r"RECSPLIT_API[^;(]*?\b(recsplit_\w+)\s*\(", hdr))
    assert declared == set(rs.SYMBOLS)
    L = rs.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert L.recsplit_version() == 1
    assert L.recsplit_max_bucket_keys() == 65536


@pytest.mark.parametrize("leaf", [2, 3, 5, 8, 12, 16, 20, 24])
@pytest.mark.parametrize("rf", [True, False])
def test_tau_tables_match_oracle(leaf, rf):
    """Library (log-factorial sums, expm1) vs oracle (lgamma, squaring) tau for every
    node size up to 2600 -- the tie margin is ~7e-6 so any faithful evaluation agrees."""
    for s in list(range(1, 400)) + list(range(400, 2600, 7)):
        assert rs.tau(leaf, s, rf) == oracle.tau(leaf, s, rf), (leaf, s, rf)


@pytest.mark.parametrize("leaf,b,rf,n", [(8, 100, True, 10000), (5, 5, True, 3000), (16, 300, False, 2000),
                                          (3, 1, True, 500), (24, 50, True, 100), (12, 1000, True, 3000)])
def test_library_query_reads_oracle_format(leaf, b, rf, n):
    keys = synth.keys(n, leaf * 7 + b)
    blob = oracle.build(keys, leaf, b, rf=rf, threads=4)
    q = rs.query_many(blob, keys)
    assert np.array_equal(q, oracle.query_many(blob, keys))
    assert np.array_equal(np.sort(q), np.arange(n, dtype=np.uint64))
    assert rs.query(blob, int(keys[0])) == int(q[0])


def test_corrupt_blob_is_format_error():
    keys = synth.keys(1000, 3)
    blob = oracle.build(keys, 8, 100)
    for bad in (blob[:50], b"XXXX" + blob[4:], blob[:-8], blob + b"\0" * 8):
        with pytest.raises(rs.RecSplitError) as e:
            rs.query_many(bad, keys[:10])
        assert e.value.code == rs.E_FORMAT


def test_bits_per_key_accounting():
    keys = synth.keys(10000, 1)
    blob = oracle.build(keys, 8, 100)
    from test_oracle_pins import bits_per_object
    assert rs.bits_per_key(blob) == pytest.approx(bits_per_object(blob))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    keys = synth.keys(100, 1)
    with pytest.raises(rs.RecSplitError) as e:
        rs.build(keys, 8, 100)
    assert e.value.code == rs.E_CUDA
    with pytest.raises(rs.RecSplitError) as e:
        rs.search_leaves(np.zeros(4, np.uint64), np.zeros(4, np.uint8), [0, 4])
    assert e.value.code == rs.E_CUDA


def test_argument_validation():
    keys = synth.keys(10, 1)
    for leaf, b in [(1, 10), (25, 10), (8, 0)]:
        with pytest.raises(rs.RecSplitError) as e:
            rs.build(keys, leaf, b)
        assert e.value.code == rs.E_INVALID
    with pytest.raises(rs.RecSplitError) as e:
        rs.build(np.zeros(0, np.uint64), 8, 100)
    assert e.value.code == rs.E_INVALID


def test_library_string_query_reads_oracle_format():
    """String keys (N4, R16): the library's host string query reads the oracle's string-key
    MPHFs (independent implementations of the string hash) and rejects u64 queries."""
    data, off = synth.strings(4000, 21)
    blob = oracle.build_strings(data, off, 8, 100, threads=2)
    q = rs.query_strings(blob, data, off)
    assert np.array_equal(q, oracle.query_strings(blob, data, off))
    assert np.array_equal(np.sort(q), np.arange(4000, dtype=np.uint64))
    with pytest.raises(rs.RecSplitError) as e:
        rs.query_many(blob, np.array([1], dtype=np.uint64))
    assert e.value.code == rs.E_FORMAT


def test_host_handle_matches_blob_query():
    """recsplit_open with device < 0 (no GPU needed): the handle's query equals the
    per-call query and the oracle's; bad blobs fail at open; close is NULL-safe."""
    keys = synth.keys(20000, 5)
    blob = oracle.build(keys, 12, 1000, threads=4)
    with rs.Handle(blob) as h:
        assert np.array_equal(h.query_many(keys), oracle.query_many(blob, keys))
        # host-only handle: the device query is refused, not emulated
        assert rs.lib().recsplit_handle_query_device(h._h, None, 0, None, None) == rs.E_INVALID
    with pytest.raises(rs.RecSplitError) as e:
        rs.Handle(blob[:-8])
    assert e.value.code == rs.E_FORMAT
    rs.lib().recsplit_close(None)


def test_corrupt_blob_rejected_or_in_range():
    """A corrupt blob never makes the query read past the data: every bucket's
    unary region must hold exactly N(s) ones after its F(s) fixed bits (format.cpp), so a
    flipped bit in a unary region -> RECSPLIT_E_FORMAT; a flipped fixed bit leaves a valid
    structure whose queries stay in [0, n) (header contract).  Host parser = the same code
    the GPU query's recsplit_open uses."""
    keys = synth.keys(10_000, 1)
    blob = oracle.build(keys, 8, 100)
    n = len(keys)
    rng = np.random.default_rng(5)
    data_bits = int.from_bytes(blob[40:48], "little")
    data_start = len(blob) - 8 * ((data_bits + 63) // 64)
    rejected = 0
    for _ in range(200):
        b = bytearray(blob)
        bit = int(rng.integers(0, data_bits))
        b[data_start + bit // 8] ^= 1 << (bit % 8)
        try:
            q = rs.query_many(bytes(b), keys[:500])
        except rs.RecSplitError as e:
            assert e.code == rs.E_FORMAT
            rejected += 1
            continue
        assert (q < n).all()
    assert 0 < rejected < 200
    # truncated / bit-flipped index words are rejected too
    with pytest.raises(rs.RecSplitError):
        rs.query_many(blob[:-8], keys[:10])


def test_trim_without_gpu():
    """recsplit_trim only releases what exists: without a GPU (or before any build) it succeeds."""
    rs.trim()
    rs.trim()
