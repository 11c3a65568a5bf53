"""Wire format and the GPU worker handler against frames
the reference produced (tests/golden/make_wire_golden.py: pmflow.wire
encode_request / encode_response and the reference worker's answer,
rpc.py:147-195).  Mirrors the reference's tests/test_wire.py themes:
round trips, one status per malformed-input class, framing."""

from __future__ import annotations

import io
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1509_06004_b200 import wire
from paper_1509_06004_b200.grid import BorderEdgeError


def frames():
    with open(os.path.join(GOLDEN, "wire_frames.json")) as f:
        return json.load(f)["frames"]


FRAMES = frames()
GOOD = [f for f in FRAMES if f["status"] == 0]
DECODE_BAD = [f for f in FRAMES if f["status"] in (1, 2, 3, 4)]


@pytest.mark.parametrize("f", GOOD, ids=lambda f: f["name"])
def test_request_round_trip_is_byte_exact(f):
    payload = bytes.fromhex(f["request"])
    req = wire.decode_request(payload)
    assert wire.encode_request(req) == payload
    wp = wire.decode_planes(payload)
    assert wp.planes.dtype == np.int32 and not wp.planes.flags.writeable
    assert np.shares_memory(wp.planes, np.frombuffer(payload, np.uint8))   # zero copy
    assert np.array_equal(wp.planes[0], req.graph.src_cap)
    assert np.array_equal(wp.planes[2:6], req.graph.nbr_cap)
    assert wire.request_payload_size(req.graph.n, len(req.layout.segments)) == len(payload)


@pytest.mark.parametrize("f", GOOD, ids=lambda f: f["name"])
def test_response_round_trip_is_byte_exact(f):
    payload, resp = bytes.fromhex(f["request"]), bytes.fromhex(f["response"])
    n = wire.decode_planes(payload).planes.shape[1]
    r = wire.decode_response(resp, n)
    assert r.status == wire.Status.OK and r.labels.shape == (n,)
    assert wire.encode_response(r) == resp
    assert wire.response_payload_size(n) == len(resp)


@pytest.mark.parametrize("f", DECODE_BAD, ids=lambda f: f["name"])
def test_malformed_request_status_matches_reference(f):
    payload = bytes.fromhex(f["request"])
    with pytest.raises(wire.WireError) as ei:
        wire.decode_planes(payload)
    assert int(ei.value.status) == f["status"]
    # the worker's answer for a frame that fails to decode (rpc.py:186-195)
    answer = wire.encode_response(wire.WireResponse(wire.peek_task_id(payload), ei.value.status, 0, None))
    assert answer == bytes.fromhex(f["response"])


def test_border_arc_is_rejected_like_admit():
    f = next(f for f in FRAMES if f["name"] == "border_arc")
    wp = wire.decode_planes(bytes.fromhex(f["request"]))
    with pytest.raises(BorderEdgeError) as ei:
        wire._check_border(wp)
    assert wire.status_for_exception(ei.value) == wire.Status.GRAPH_REJECTED == f["status"]


def test_bits_and_frames():
    rng = np.random.default_rng(5)
    for n in (1, 7, 8, 9, 100):
        bits = rng.integers(0, 2, n).astype(np.uint8)
        data = wire.pack_bits(bits)
        assert len(data) == (n + 7) // 8
        assert np.array_equal(wire.unpack_bits(data, n), bits)
    with pytest.raises(wire.FrameLengthError):
        wire.unpack_bits(b"\xff", 7)          # nonzero padding
    with pytest.raises(wire.FrameLengthError):
        wire.unpack_bits(b"\x00\x00", 7)      # wrong byte count
    stream = io.BytesIO(wire.frame(b"abc") + wire.frame(b"") + b"\x05\x00")
    assert wire.read_frame(stream) == b"abc"
    assert wire.read_frame(stream) == b""
    with pytest.raises(wire.FrameLengthError):
        wire.read_frame(stream)               # partial header
    assert wire.read_frame(io.BytesIO(b"")) is None
    with pytest.raises(wire.FrameLengthError):
        wire.read_frame(io.BytesIO(b"\x09\x00\x00\x00abc"))   # partial payload


@pytest.mark.gpu
@pytest.mark.parametrize("f", FRAMES, ids=lambda f: f["name"])
def test_gpu_worker_answers_like_the_reference(f):
    """serve_payload (decode in place -> pmf_solve_composites_i32 -> encode)
    returns the reference worker's response bytes, for solved requests
    (flow + LSB-first label bits) and for every rejection."""
    assert wire.serve_payload(bytes.fromhex(f["request"])) == bytes.fromhex(f["response"])


@pytest.mark.gpu
def test_gpu_solve_fn_matches_the_wire_answer():
    """gpu_solve_fn (the WorkerServer(solve_fn=...) hook, rpc.py:94,100) on
    the reference's decoded request gives the same cut as the wire path."""
    f = FRAMES[[g["name"] for g in FRAMES].index("composite_3seg")]
    req = wire.decode_request(bytes.fromhex(f["request"]))
    cut = wire.gpu_solve_fn(req.graph, req.layout)
    r = wire.decode_response(bytes.fromhex(f["response"]), req.graph.n)
    assert cut.flow == r.flow
    assert np.array_equal(np.asarray(cut.labels, np.uint8).reshape(-1), r.labels)


def test_encoder_rejects_capacities_the_wire_cannot_carry():
    """encode_request refuses planes outside [0, CAP_MAX] (wire.py:131-134)."""
    from paper_1509_06004_b200.grid import CAP_MAX, GridGraph
    f = next(f for f in FRAMES if f["name"] == "whole_6x9")
    req = wire.decode_request(bytes.fromhex(f["request"]))
    g = req.graph
    for bad in (-1, CAP_MAX + 1):
        src = g.src_cap.copy()
        src[3] = bad
        g2 = GridGraph(g.width, g.height, src, g.snk_cap, g.nbr_cap)
        with pytest.raises(wire.CapacityRangeError):
            wire.encode_request(wire.WireRequest(1, g2, None))


@pytest.mark.parametrize("f", [f for f in GOOD if f["name"].startswith("wide_")], ids=lambda f: f["name"])
def test_oracle_pinned_on_wide_frames(f):
    """The oracle (the GPU tests' checker) reproduces the reference worker's
    answers on requests whose excess leaves int32 (CAP_MAX arc pairs)."""
    import oracle
    req = wire.decode_request(bytes.fromhex(f["request"]))
    g = req.graph
    segs = [(s.offset, s.width, s.swapped) for s in req.layout.segments]
    flow, labels, _ = oracle.solve(g.width, g.height, g.src_cap, g.snk_cap, g.nbr_cap, segs)
    r = wire.decode_response(bytes.fromhex(f["response"]), g.n)
    assert flow == r.flow
    assert np.array_equal(labels, r.labels)
