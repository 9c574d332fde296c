"""Worker wire protocol (protocol.py) and the GPU worker's failure paths that
need no GPU; byte-compatibility with the reference's own encoder is pinned by
tests/golden/protocol_frames.json (generated from the reference)."""

import io
import json
import struct

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle
import paper_1605_01584_b200 as pc
from paper_1605_01584_b200 import protocol
from paper_1605_01584_b200.errors import ProtocolError
from paper_1605_01584_b200.worker import serve

from conftest import GOLDEN, random_values


def test_frames_byte_identical_to_reference():
    g = json.loads((GOLDEN / "protocol_frames.json").read_text())
    vals = np.array(g["blocks_values"])
    assert protocol.encode_assign(3, 17, 4, 1000, "/data/expr.lpcc").hex() == g["assign"]
    assert protocol.encode_assign(0, 0, 1, 1, "déjà.lpcc").hex() == g["assign_unicode"]
    assert protocol.encode_blocks(12, vals, 4).hex() == g["blocks"]
    assert protocol.encode_done(123456789).hex() == g["done"]
    assert protocol.encode_error("ValueError: boom").hex() == g["error"]


def test_round_trips():
    a = protocol.decode_assign(protocol.encode_assign(5, 9, 3, 77, "x.lpcc"))
    assert (a.j_start, a.j_end, a.t, a.capacity, a.dataset_path) == (5, 9, 3, 77, "x.lpcc")
    v = np.random.default_rng(0).random(3 * 4)
    first, count, back = protocol.decode_blocks(protocol.encode_blocks(11, v, 2), 2)
    assert (first, count) == (11, 3) and np.array_equal(back, v)
    assert protocol.decode_done(protocol.encode_done(42)) == 42
    assert protocol.decode_error(protocol.encode_error("oops")) == "oops"
    buf = io.BytesIO()
    protocol.write_frame(buf, protocol.FRAME_DONE, protocol.encode_done(7))
    buf.seek(0)
    assert protocol.read_frame(buf) == (protocol.FRAME_DONE, protocol.encode_done(7))
    assert protocol.read_frame(buf) is None


def test_truncation_and_garbage_rejected():
    with pytest.raises(ProtocolError):
        protocol.read_frame(io.BytesIO(b"\x01\x00"))
    with pytest.raises(ProtocolError):
        protocol.read_frame(io.BytesIO(struct.pack("<BI", 2, 10) + b"abc"))
    for bad in [b"", b"\x00" * 10,
                struct.pack("<QQIQH", 9, 5, 1, 1, 0),            # inverted range
                struct.pack("<QQIQH", 0, 5, 0, 1, 0),            # t = 0
                struct.pack("<QQIQH", 0, 5, 1, 0, 0),            # capacity = 0
                struct.pack("<QQIQH", 0, 5, 1, 1, 4) + b"ab",    # path length mismatch
                struct.pack("<QQIQH", 0, 5, 1, 1, 2) + b"\xff\xfe"]:  # not utf-8
        with pytest.raises(ProtocolError):
            protocol.decode_assign(bad)
    with pytest.raises(ProtocolError):
        protocol.decode_blocks(struct.pack("<QI", 0, 2) + b"\x00" * 8, 2)
    with pytest.raises(ProtocolError):
        protocol.encode_blocks(0, np.zeros(5), 2)
    with pytest.raises(ProtocolError):
        protocol.decode_done(b"\x00" * 4)


@given(st.binary(max_size=64))
@settings(max_examples=300, deadline=None)
def test_read_frame_never_crashes(data):
    stream = io.BytesIO(data)
    while True:
        try:
            frame = protocol.read_frame(stream)
        except ProtocolError:
            break
        if frame is None:
            break


def _frames(buf: bytes):
    s = io.BytesIO(buf)
    out = []
    while (f := protocol.read_frame(s)) is not None:
        out.append(f)
    return out


def test_worker_reports_protocol_failures_as_error_frames(tmp_path, rng):
    out = io.BytesIO()
    assert serve(io.BytesIO(b""), out) == 1
    (kind, msg), = _frames(out.getvalue())
    assert kind == protocol.FRAME_ERROR and "ASSIGN" in protocol.decode_error(msg)

    out = io.BytesIO()
    buf = io.BytesIO()
    protocol.write_frame(buf, protocol.FRAME_DONE, protocol.encode_done(1))
    buf.seek(0)
    assert serve(buf, out) == 1
    assert _frames(out.getvalue())[0][0] == protocol.FRAME_ERROR

    out = io.BytesIO()
    buf = io.BytesIO()
    protocol.write_frame(buf, protocol.FRAME_ASSIGN, protocol.encode_assign(0, 1, 2, 10, str(tmp_path / "missing")))
    buf.seek(0)
    assert serve(buf, out) == 1
    assert _frames(out.getvalue())[0][0] == protocol.FRAME_ERROR

    path = tmp_path / "d.lpcc"
    pc.save_dataset(path, pc.Dataset(values=random_values(rng, 6, 4)))
    out = io.BytesIO()
    buf = io.BytesIO()
    protocol.write_frame(buf, protocol.FRAME_ASSIGN, protocol.encode_assign(0, 99, 2, 10, str(path)))
    buf.seek(0)
    assert serve(buf, out) == 1
    (kind, msg), = _frames(out.getvalue())
    assert kind == protocol.FRAME_ERROR and "exceeds" in protocol.decode_error(msg)


def test_merge_detects_every_missing_or_duplicated_tile(rng):
    x = random_values(rng, 12, 6)
    u, _ = oracle.normalize(x)
    geom = pc.TileGeometry(n=12, t=4)  # 6 tiles

    def reports():
        out = []
        for i, (lo, hi) in enumerate(pc.partition(geom.total_tiles, 2)):
            flat = oracle.compute_pass(u, 4, lo, hi)
            blocks = [pc.TileBlock(lo + k, flat[k * 16:(k + 1) * 16]) for k in range(hi - lo)]
            out.append(pc.WorkerReport(worker_index=i, tiles_done=hi - lo, blocks=blocks))
        return out

    ref, _ = oracle.allpairs(x)
    assert np.array_equal(pc.merge(reports(), geom).packed, ref)
    for victim in range(geom.total_tiles):
        r = reports()
        for rep in r:
            rep.blocks = [b for b in rep.blocks if b.tile_id != victim]
        with pytest.raises(pc.IntegrityError, match=str(victim)):
            pc.merge(r, geom)
        r = reports()
        r[-1].blocks.append(next(b for rep in r for b in rep.blocks if b.tile_id == victim))
        with pytest.raises(pc.IntegrityError, match=str(victim)):
            pc.merge(r, geom)
    r = reports()
    r[0].status, r[0].message = "error", "boom"
    with pytest.raises(pc.WorkerError):
        pc.merge(r, geom)
