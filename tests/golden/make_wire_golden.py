"""Golden wire frames from the REFERENCE package (pmflow.wire / rpc).

    python tests/golden/make_wire_golden.py

Writes wire_frames.json next to this script: request payloads the
reference's ``encode_request`` (wire.py:137) produced, the response payload
its worker would send (``solve_composite`` + ``encode_response``,
rpc.py:147-162), and malformed payloads with the status the reference's
``decode_request`` raises for each (wire.py:189-228, ``status_for_exception``
:281).  Run in the build container (reference mounted at /root/reference).
"""

from __future__ import annotations

import json
import os
import struct
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

from conftest import random_grid  # noqa: E402  (reference test helper)
from pmflow import wire  # noqa: E402
from pmflow.grid import admit  # noqa: E402
from pmflow.supergraph import apply_swap, join, solve_composite  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "wire_frames.json")


def wide_grid(rng, w, h):
    """Random admitted grid with capacities drawn from {0, small, up to
    CAP_MAX, CAP_MAX}: most pixels' excess bound is far past 2**31."""
    cap = 1 << 30

    def draw(shape):
        kind = rng.integers(0, 4, shape)
        v = np.where(kind == 0, 0, np.where(kind == 1, rng.integers(1, 100, shape),
                                            np.where(kind == 2, rng.integers(1, cap + 1, shape), cap)))
        return v.astype(np.int64)

    src, snk, nbr = draw(w * h), draw(w * h), draw((4, w * h)).reshape(4, h, w)
    nbr[0][:, 0] = 0
    nbr[1][:, -1] = 0
    nbr[2][0, :] = 0
    nbr[3][-1, :] = 0
    from pmflow.grid import GridGraph
    return admit(GridGraph(w, h, src, snk, nbr.reshape(4, w * h)))


def served(payload: bytes) -> bytes:
    """What the reference worker answers for one payload (rpc.py:147-195)."""
    try:
        req = wire.decode_request(payload)
    except wire.WireError as exc:
        tid = struct.unpack_from("<Q", payload, 8)[0] if len(payload) >= 16 and payload[:4] == wire.MAGIC else 0
        return wire.encode_response(wire.WireResponse(tid, exc.status, 0, None))
    try:
        cut = solve_composite(admit(req.graph), req.layout)
        resp = wire.WireResponse(req.task_id, wire.Status.OK, cut.flow, cut.labels)
    except Exception as exc:
        resp = wire.WireResponse(req.task_id, wire.status_for_exception(exc), 0, None)
    return wire.encode_response(resp)


def main():
    rng = np.random.default_rng(2024)
    frames = []
    # a composite of three constituents, the middle one embedded swapped
    parts = [random_grid(rng, 7, 6, cap_hi=30), random_grid(rng, 5, 6, cap_hi=30), random_grid(rng, 9, 6, cap_hi=30)]
    comp, layout = join([parts[0], apply_swap(parts[1]), parts[2]], swapped=[False, True, False])
    frames.append(("composite_3seg", wire.encode_request(wire.WireRequest(77, comp, layout))))
    # single graphs (whole-graph layout)
    for k, (w, h) in enumerate([(1, 1), (8, 1), (6, 9), (13, 11)]):
        g = random_grid(rng, w, h, cap_hi=50)
        frames.append((f"whole_{w}x{h}", wire.encode_request(wire.WireRequest(1000 + k, g, None))))
    # graphs the reference admits whose excess leaves int32 (CAP_MAX arc
    # pairs and CAP_MAX terminals next to them): the engine's int64 variant
    for k, (w, h) in enumerate([(7, 5), (12, 9)]):
        frames.append((f"wide_{w}x{h}", wire.encode_request(wire.WireRequest(2000 + k, wide_grid(rng, w, h), None))))
    wparts = [wide_grid(rng, 6, 5), wide_grid(rng, 4, 5)]
    wcomp, wlay = join([wparts[0], apply_swap(wparts[1])], swapped=[False, True])
    frames.append(("wide_composite_2seg", wire.encode_request(wire.WireRequest(2100, wcomp, wlay))))
    good = frames[0][1]
    # malformed payloads, one per failure class
    bad = {
        "bad_magic": b"XXXX" + good[4:],
        "version_2": good[:4] + struct.pack("<H", 2) + good[6:],
        "flags_set": good[:6] + struct.pack("<H", 1) + good[8:],
        "truncated": good[:-3],
        "trailing": good + b"\0",
        "header_only": good[:20],
    }
    n = comp.n
    planes_at = len(good) - 24 * n
    neg = bytearray(good)
    neg[planes_at + 4 * 5: planes_at + 4 * 6] = struct.pack("<i", -1)
    bad["negative_src"] = bytes(neg)
    big = bytearray(good)
    big[planes_at + 4 * n: planes_at + 4 * n + 4] = struct.pack("<i", (1 << 30) + 1)
    bad["snk_above_cap_max"] = bytes(big)
    border = bytearray(good)
    border[planes_at + 8 * n: planes_at + 8 * n + 4] = struct.pack("<i", 5)   # LEFT arc of pixel 0
    bad["border_arc"] = bytes(border)
    # a range error together with a framing error: the reference's decode
    # reports the range error when the planes are complete and the framing
    # error when they are not (decode_request's order, wire.py:189-228)
    bad["range_and_trailing"] = bytes(big) + b"\0"
    bad["range_and_truncated"] = bytes(neg)[:-3]
    frames += sorted(bad.items())
    out = []
    for name, payload in frames:
        resp = served(payload)
        out.append({"name": name, "request": payload.hex(), "response": resp.hex(),
                    "status": struct.unpack_from("<H", resp, 8)[0]})
    with open(OUT, "w") as f:
        json.dump({"generator": "tests/golden/make_wire_golden.py (reference pmflow.wire, rpc)",
                   "frames": out}, f, indent=1)
    print(OUT, len(out), "frames")


if __name__ == "__main__":
    main()
