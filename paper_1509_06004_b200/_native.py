"""ctypes binding of libpmflow_b200.so (the C ABI in include/pmflow_b200.h).

The shared library is built in-tree (``python -m paper_1509_06004_b200.build``
or ``__graft_entry__.build()``).  There is no CPU fallback: if the library or
a CUDA device is missing, every solver entry point raises
``NativeUnavailable``.  Status codes map onto the reference's exception
classes (solvers.py:33-38, grid.py:45-46).
"""

from __future__ import annotations

import ctypes
import os
import sys
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PMF_LIB") or os.path.join(HERE, "libpmflow_b200.so")

PMF_OK, PMF_ERR_ARG, PMF_ERR_CUDA, PMF_ERR_NOCONV, PMF_ERR_NONMAX, PMF_ERR_RANGE = 0, -1, -2, -3, -4, -5
SWAP_MODES = {"auto": 0, "on": 1, "off": 2}

EXPORTS = ("pmf_solver_create", "pmf_solver_destroy", "pmf_solver_set", "pmf_last_error",
           "pmf_solver_stats", "pmf_solver_stream", "pmf_solve_composites", "pmf_solve_seed_batch",
           "pmf_seed_stage", "pmf_seed_run", "pmf_seed_launch", "pmf_seed_wait", "pmf_seed_fetch",
           "pmf_synth_stage", "pmf_debug_planes", "pmf_solver_depend", "pmf_seed_kind",
           "pmf_debug_state",
           "pmf_debug_trace", "pmf_debug_busy", "pmf_seed_score", "pmf_debug_phases",
           "pmf_solve_composites_i32", "pmf_composite_bits", "pmf_plane_stats")


class NativeUnavailable(RuntimeError):
    """The CUDA engine cannot run here (library not built or no GPU)."""


class PmfStats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in (
        "cycles", "push_tile_passes", "bfs_tile_passes", "label_tile_passes", "push_sweeps",
        "bfs_sweeps", "full_passes", "grids", "tiles", "pixels")] + [
        ("edge_bytes", ctypes.c_int32), ("timed", ctypes.c_int32)] + [
        (k, ctypes.c_double) for k in ("ms_total", "ms_build", "ms_push", "ms_bfs", "ms_labels",
                                       "ms_seed", "ms_h2d", "ms_d2h", "ms_device")] + [
        (k, ctypes.c_int64) for k in ("launches", "h2d_bytes", "d2h_bytes", "graph_builds",
                                       "kernels", "steps", "scan_tile_passes")] + [
        ("ms_async", ctypes.c_double), ("async_mode", ctypes.c_int32), ("wide_mode", ctypes.c_int32)] + [
        (k, ctypes.c_int64) for k in ("binit_tile_passes", "seed_tile_passes", "linit_tile_passes",
                                       "emit_tile_passes")]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load (once) and type the shared library.  Raises NativeUnavailable."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is not built; run __graft_entry__.build() (no CPU fallback exists)")
        lib = ctypes.CDLL(path)
        P = ctypes.POINTER
        i32, i64, u8, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint8, ctypes.c_void_p
        lib.pmf_solver_create.argtypes = [i32, P(vp)]
        lib.pmf_solver_destroy.argtypes = [vp]
        lib.pmf_solver_set.argtypes = [vp, ctypes.c_char_p, i64]
        lib.pmf_last_error.argtypes = []
        lib.pmf_last_error.restype = ctypes.c_char_p
        lib.pmf_solver_stats.argtypes = [vp, P(PmfStats)]
        lib.pmf_solve_composites.argtypes = [
            vp, i32, P(i32), P(i32), P(vp), P(vp), P(vp), P(i32), P(vp), P(vp), P(vp),
            P(i64), P(vp)]
        lib.pmf_solve_composites_i32.argtypes = lib.pmf_solve_composites.argtypes
        lib.pmf_composite_bits.argtypes = [vp, i32, P(u8), i64]
        lib.pmf_solve_seed_batch.argtypes = [
            vp, i32, i32, i32, P(vp), P(vp), P(vp), P(vp), P(vp), P(i32), P(vp), P(i32),
            i32, P(i64), i32, P(u8), P(i64), P(u8)]
        lib.pmf_seed_stage.argtypes = [
            vp, i32, i32, i32, P(vp), P(vp), P(vp), P(vp), P(vp), P(i32), P(vp), P(i32),
            i32, P(i64), i32]
        lib.pmf_seed_run.argtypes = [vp]
        lib.pmf_seed_launch.argtypes = [vp, vp]
        lib.pmf_solver_depend.argtypes = [vp, vp]
        lib.pmf_seed_kind.argtypes = [vp, P(i32), P(i32)]
        lib.pmf_debug_planes.argtypes = [vp, P(i32), P(i64), P(i32), P(i64)]
        lib.pmf_synth_stage.argtypes = [vp, i32, i32, i32, P(u8), i32, P(i32), i32, P(i32), i32, P(i64), i32]
        lib.pmf_seed_wait.argtypes = [vp]
        lib.pmf_seed_fetch.argtypes = [vp, P(u8), P(i64), P(u8)]
        lib.pmf_solver_stream.argtypes = [vp, P(vp)]
        lib.pmf_debug_state.argtypes = [vp, vp, vp, vp, vp, P(i64)]
        lib.pmf_debug_trace.argtypes = [vp, vp, vp, vp, vp, P(i32)]
        lib.pmf_debug_busy.argtypes = [vp, P(ctypes.c_double)]
        lib.pmf_debug_phases.argtypes = [vp, i64, P(ctypes.c_uint64), P(i32)]
        lib.pmf_seed_score.argtypes = [vp, P(vp), P(i64), P(i64), P(i64)]
        lib.pmf_plane_stats.argtypes = [i32, P(vp), P(i64), P(i64)]
        for name in EXPORTS:
            if name != "pmf_last_error":
                getattr(lib, name).restype = ctypes.c_int
        _lib = lib
        return lib


def _raise_for(rc: int):
    from .grid import CapacityOverflowError
    from .solvers import NonMaximalFlowError, SolverError
    msg = load_library().pmf_last_error().decode(errors="replace")
    if rc == PMF_ERR_NOCONV:
        raise SolverError(msg)
    if rc == PMF_ERR_NONMAX:
        raise NonMaximalFlowError(msg)
    if rc == PMF_ERR_RANGE:
        raise CapacityOverflowError(msg)
    if rc == PMF_ERR_ARG:
        raise ValueError(msg)
    raise RuntimeError(f"pmflow_b200 CUDA failure: {msg}")


def _ptrs(arrays, ctype=ctypes.c_void_p):
    return (ctype * len(arrays))(*[None if a is None else a.ctypes.data for a in arrays])


class _LabelBuffers:
    """Reuse of large label output buffers across calls.  A fresh multi-MB
    numpy array costs a page fault and a kernel zero-fill per 4 KiB on first
    touch, which dominated the host side of large batches.  A buffer is
    handed out again only once nothing but this pool references it: every
    numpy view of it (the per-cut label arrays) holds a reference to it, so
    ``sys.getrefcount`` shows when the caller has dropped them all."""

    MIN_BYTES = 16 << 20
    KEEP = 2          # buffers kept per size

    def __init__(self):
        self._free = {}
        self._lock = threading.Lock()

    def take(self, shape):
        nbytes = int(np.prod(shape))
        if nbytes < self.MIN_BYTES:
            return np.empty(shape, np.uint8)
        with self._lock:
            bufs = self._free.setdefault(nbytes, [])
            for b in bufs:
                # refs: the list entry, the loop variable, getrefcount's argument
                if sys.getrefcount(b) <= 3:
                    return b.reshape(shape)
            b = np.empty(nbytes, np.uint8)
            if len(bufs) < self.KEEP:
                bufs.append(b)
            return b.reshape(shape)


class Solver:
    """One device + one CUDA stream + its workspaces.  Not thread-safe: use
    one per host thread (``solver_for_thread``)."""

    def __init__(self, device: int = 0, **knobs):
        lib = load_library()
        h = ctypes.c_void_p()
        rc = lib.pmf_solver_create(int(device), ctypes.byref(h))
        if rc:
            raise NativeUnavailable(lib.pmf_last_error().decode(errors="replace"))
        self._lib, self._h, self.device = lib, h, device
        self._labels = _LabelBuffers()
        for k, v in knobs.items():
            self.set(k, v)

    def set(self, name: str, value: int):
        rc = self._lib.pmf_solver_set(self._h, name.encode(), int(value))
        if rc:
            _raise_for(rc)

    def stats(self) -> dict:
        st = PmfStats()
        self._lib.pmf_solver_stats(self._h, ctypes.byref(st))
        return st.as_dict()

    def close(self):
        if self._h:
            self._lib.pmf_solver_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- solves
    def solve_composites(self, items, i32: bool = False, labels: bool = True):
        """items: [(width, height, src, snk, nbr, segments)] with segments a
        list of (offset, width, swapped) or None.  Returns [(flow, labels)].
        i32: the planes are int32 (wire requests) and are read in place.
        labels=False: labels stay on the device (None returned; see
        composite_bits)."""
        k = len(items)
        self._staged = None   # a composite solve replaces the staged seed batch on the device
        dt = np.int32 if i32 else np.int64
        keep = []
        widths = np.array([it[0] for it in items], np.int32)
        heights = np.array([it[1] for it in items], np.int32)
        srcs, snks, nbrs, nsegs, offs, wids, sws, labs = [], [], [], [], [], [], [], []
        for (w, h, src, snk, nbr, segs) in items:
            srcs.append(np.ascontiguousarray(src, dt))
            snks.append(np.ascontiguousarray(snk, dt))
            nbrs.append(np.ascontiguousarray(nbr, dt))
            segs = list(segs or ())
            nsegs.append(len(segs))
            offs.append(np.array([s[0] for s in segs] or [0], np.int32))
            wids.append(np.array([s[1] for s in segs] or [0], np.int32))
            sws.append(np.array([1 if s[2] else 0 for s in segs] or [0], np.uint8))
            labs.append(np.empty(w * h, np.uint8) if labels else None)
        keep += [srcs, snks, nbrs, offs, wids, sws, labs]
        flows = np.zeros(k, np.int64)
        nseg = np.array(nsegs, np.int32)
        P = ctypes.POINTER
        fn = self._lib.pmf_solve_composites_i32 if i32 else self._lib.pmf_solve_composites
        rc = fn(
            self._h, k, widths.ctypes.data_as(P(ctypes.c_int32)),
            heights.ctypes.data_as(P(ctypes.c_int32)), _ptrs(srcs), _ptrs(snks), _ptrs(nbrs),
            nseg.ctypes.data_as(P(ctypes.c_int32)), _ptrs(offs), _ptrs(wids), _ptrs(sws),
            flows.ctypes.data_as(P(ctypes.c_int64)), _ptrs(labs))
        if rc:
            _raise_for(rc)
        return [(int(f), l) for f, l in zip(flows, labs)]

    def composite_bits(self, c: int, n: int) -> bytes:
        """Labels of composite c of the last composite solve (n pixels) as
        LSB-first bits (the wire's response body), packed on the device."""
        out = np.empty((n + 7) // 8, np.uint8)
        rc = self._lib.pmf_composite_bits(self._h, c, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                                          ctypes.c_int64(out.size))
        if rc:
            _raise_for(rc)
        return out.tobytes()

    def debug_state(self):
        """(w, h, r, lab) tile-major arrays of the last run (diagnostics)."""
        nt = ctypes.c_int64()
        self._lib.pmf_debug_state(self._h, None, None, None, None, ctypes.byref(nt))
        P_ = nt.value * 1024
        eb = self.stats()["edge_bytes"]
        w = np.empty(P_, np.int32)
        h = np.empty(P_, np.int32)
        r = np.empty(P_, np.uint32) if eb == 4 else np.empty((P_, 4), np.int32)
        lab = np.empty(P_, np.uint8)
        rc = self._lib.pmf_debug_state(self._h, w.ctypes.data, h.ctypes.data, r.ctypes.data,
                                       lab.ctypes.data, ctypes.byref(nt))
        if rc:
            _raise_for(rc)
        return w, h, r, lab

    def trace(self):
        """[(kind, us, tile_passes, start_us)] of the first tile-kernel launches
        of the last run (kind: 0 discharge, 1 sink BFS, 2 label BFS; start_us
        relative to the first traced launch)."""
        cap = 1 << 16   # PMF_KTRACE of diagnostics builds; the library clamps to its own
        n = ctypes.c_int32(cap)
        kind = np.zeros(cap, np.int32)
        us = np.zeros(cap, np.float64)
        t0 = np.zeros(cap, np.float64)
        tiles = np.zeros(cap, np.int64)
        self._lib.pmf_debug_trace(self._h, kind.ctypes.data, us.ctypes.data, t0.ctypes.data,
                                  tiles.ctypes.data, ctypes.byref(n))
        return [(int(kind[i]), round(float(us[i]), 1), int(tiles[i]), round(float(t0[i]), 1))
                for i in range(n.value)]

    def busy(self):
        """Async runs: CTA-busy ms per phase kind, summed over CTAs."""
        out = np.zeros(16, np.float64)
        self._lib.pmf_debug_busy(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        names = ("binit", "bfs", "seed", "push", "linit", "lab", "emit", "-", "wait", "handoff", "transition")
        d = {k: round(float(v), 2) for k, v in zip(names, out) if k != "-"}
        d["push_iterations"] = int(out[15])
        d["spec_tries"] = int(out[7])
        d["spec_spoiled"] = int(out[11])
        d["relax_ms"] = round(float(out[13]), 2)
        d["relax_calls"] = int(out[14])
        d["relax_sweeps"] = int(out[12])
        return d

    def phases(self, grid: int):
        """Phase timeline [(phase name, us since the first entry)] of one grid
        of the last asynchronous run (knob phase_log=1)."""
        out = np.zeros(512, np.uint64)
        n = ctypes.c_int32(512)
        rc = self._lib.pmf_debug_phases(self._h, grid, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                        ctypes.byref(n))
        if rc:
            _raise_for(rc)
        names = ("binit", "bfs", "seed", "push", "linit", "lab", "emit", "done")
        v = out[:n.value]
        ts = (v & np.uint64((1 << 56) - 1)).astype(np.int64)
        return [(names[int(x >> np.uint64(56))], round(float(t - ts[0]) / 1e3, 1)) for x, t in zip(v, ts)]

    def stream_handle(self) -> int:
        """The solver's cudaStream_t as an integer (torch.cuda.ExternalStream)."""
        out = ctypes.c_void_p()
        self._lib.pmf_solver_stream(self._h, ctypes.byref(out))
        return int(out.value or 0)

    def seed_stage(self, width, height, problems, lambdas, swap_mode="auto"):
        """Validate/convert seed problems and copy them to the device."""
        ub = [np.ascontiguousarray(p.unary_base, np.int64) for p in problems]
        us = [np.ascontiguousarray(p.unary_slope, np.int64) for p in problems]
        sb = [np.ascontiguousarray(p.sink_base, np.int64) for p in problems]
        pw = [np.ascontiguousarray(p.pairwise, np.int64) for p in problems]
        fg = [np.ascontiguousarray(p._fg_idx, np.int64) for p in problems]
        bg = [np.ascontiguousarray(p._bg_idx, np.int64) for p in problems]
        nfg = np.array([a.size for a in fg], np.int32)
        nbg = np.array([a.size for a in bg], np.int32)
        fgp = [a if a.size else np.zeros(1, np.int64) for a in fg]
        bgp = [a if a.size else np.zeros(1, np.int64) for a in bg]
        lam = np.ascontiguousarray(lambdas, np.int64)
        Pt = ctypes.POINTER
        rc = self._lib.pmf_seed_stage(
            self._h, len(problems), width, height, _ptrs(ub), _ptrs(us), _ptrs(sb), _ptrs(pw),
            _ptrs(fgp), nfg.ctypes.data_as(Pt(ctypes.c_int32)), _ptrs(bgp),
            nbg.ctypes.data_as(Pt(ctypes.c_int32)), lam.size,
            lam.ctypes.data_as(Pt(ctypes.c_int64)), SWAP_MODES[swap_mode])
        if rc:
            _raise_for(rc)
        self._staged = (width * height, len(problems), lam.size)

    def synth_stage(self, images, coords, types, lambdas, swap_mode="auto"):
        """Stage synthetic CPMC images (k, H, W) whose planes the device
        derives (pmf_synth_stage); coords: seed (x, y) pixels; types: "A" /
        "B" seed types.  Problems image-major, seed, type-minor."""
        imgs = np.ascontiguousarray(images, np.uint8)
        k, H, W = imgs.shape
        xy = np.ascontiguousarray(np.asarray(coords, np.int32).reshape(-1))
        ty = np.array([{"A": 0, "B": 1}[t] for t in types], np.int32)
        lam = np.ascontiguousarray(lambdas, np.int64)
        P = ctypes.POINTER
        rc = self._lib.pmf_synth_stage(self._h, k, W, H, imgs.ctypes.data_as(P(ctypes.c_uint8)), xy.size // 2,
                                       xy.ctypes.data_as(P(ctypes.c_int32)), ty.size,
                                       ty.ctypes.data_as(P(ctypes.c_int32)), lam.size,
                                       lam.ctypes.data_as(P(ctypes.c_int64)), SWAP_MODES[swap_mode])
        if rc:
            _raise_for(rc)
        self._staged = (W * H, k * (xy.size // 2) * ty.size, lam.size)

    def debug_planes(self):
        """(planes, pairwise) int32 arrays of the staged batch on the device
        (diagnostics; synthetic batches: valid after a run)."""
        P = ctypes.POINTER
        a, b = ctypes.c_int64(0), ctypes.c_int64(0)
        rc = self._lib.pmf_debug_planes(self._h, None, ctypes.byref(a), None, ctypes.byref(b))
        if rc:
            _raise_for(rc)
        pl, pw = np.empty(a.value, np.int32), np.empty(b.value, np.int32)
        rc = self._lib.pmf_debug_planes(self._h, pl.ctypes.data_as(P(ctypes.c_int32)), ctypes.byref(a),
                                        pw.ctypes.data_as(P(ctypes.c_int32)), ctypes.byref(b))
        if rc:
            _raise_for(rc)
        return pl, pw

    def seed_run(self):
        """Build + solve the staged batch; results stay on the device."""
        rc = self._lib.pmf_seed_run(self._h)
        if rc:
            _raise_for(rc)

    def seed_launch(self, after=None):
        """Enqueue the run of the staged batch and return at once; with
        ``after`` (another Solver of the device) the run starts when that
        solver's last launched run has finished."""
        rc = self._lib.pmf_seed_launch(self._h, after._h if after is not None else None)
        if rc:
            _raise_for(rc)
        self._launched = True

    def depend(self, other):
        """The next launched run starts after ``other``'s last launched run."""
        rc = self._lib.pmf_solver_depend(self._h, other._h)
        if rc:
            _raise_for(rc)

    def seed_kind(self):
        """(staged batch runs asynchronously, last launched run was asynchronous)."""
        a, b = ctypes.c_int32(), ctypes.c_int32()
        rc = self._lib.pmf_seed_kind(self._h, ctypes.byref(a), ctypes.byref(b))
        if rc:
            _raise_for(rc)
        return bool(a.value), bool(b.value)

    def seed_wait(self):
        """Block until the launched run is done (device errors raised here)."""
        self._launched = False
        rc = self._lib.pmf_seed_wait(self._h)
        if rc:
            _raise_for(rc)

    def abandon(self):
        """Wait for a launched run nobody will fetch (errors dropped)."""
        if getattr(self, "_launched", False):
            try:
                self.seed_wait()
            except Exception:  # noqa: BLE001 -- the stream that launched it has ended
                pass

    def seed_fetch(self, labels=True):
        """(swapped (P,), flows (P, K), labels (P, K, n) uint8 or None)."""
        if getattr(self, "_staged", None) is None:
            raise ValueError("no staged seed batch (a composite solve replaced it)")
        n, P_, K = self._staged
        Pt = ctypes.POINTER
        swapped = np.zeros(P_, np.uint8)
        flows = np.zeros(P_ * K, np.int64)
        lab = self._labels.take((P_, K, n)) if labels else None
        rc = self._lib.pmf_seed_fetch(
            self._h, swapped.ctypes.data_as(Pt(ctypes.c_uint8)),
            flows.ctypes.data_as(Pt(ctypes.c_int64)),
            lab.ctypes.data_as(Pt(ctypes.c_uint8)) if labels else None)
        if rc:
            _raise_for(rc)
        return swapped.astype(bool), flows.reshape(P_, K), lab

    def seed_score(self, truths):
        """Device scores of the last seed run against one 0/1 truth mask per
        problem: (foreground, intersection, union) int64 arrays (P, K)."""
        n, P_, K = self._staged
        if len(truths) != P_:
            raise ValueError(f"need one truth mask per problem ({P_}), got {len(truths)}")
        keep = [np.ascontiguousarray(np.asarray(t).reshape(-1) != 0, np.uint8) for t in truths]
        if any(k.size != n for k in keep):
            raise ValueError("truth mask size differs from the problems' pixel count")
        fg, inter, uni = (np.zeros(P_ * K, np.int64) for _ in range(3))
        Pt = ctypes.POINTER
        rc = self._lib.pmf_seed_score(self._h, _ptrs(keep), fg.ctypes.data_as(Pt(ctypes.c_int64)),
                                      inter.ctypes.data_as(Pt(ctypes.c_int64)),
                                      uni.ctypes.data_as(Pt(ctypes.c_int64)))
        if rc:
            _raise_for(rc)
        return fg.reshape(P_, K), inter.reshape(P_, K), uni.reshape(P_, K)

    def solve_seed_batch(self, width, height, problems, lambdas, swap_mode="auto"):
        """problems: objects with unary_base, unary_slope, sink_base, pairwise
        (int64) and _fg_idx/_bg_idx.  Returns (swapped (P,), flows (P, K),
        labels (P, K, n) uint8)."""
        self.seed_stage(width, height, problems, lambdas, swap_mode)
        self.seed_run()
        return self.seed_fetch(True)


_tls = threading.local()
_knobs = {}


def configure(**knobs):
    """Set default knobs for solvers created afterwards (and existing ones
    of the calling thread)."""
    _knobs.update(knobs)
    s = getattr(_tls, "solvers", {})
    for sv in s.values():
        for k, v in knobs.items():
            sv.set(k, v)


def solver_for_thread(device: int = 0) -> Solver:
    """The calling thread's solver for ``device`` (created on first use)."""
    pool = getattr(_tls, "solvers", None)
    if pool is None:
        pool = _tls.solvers = {}
    s = pool.get(device)
    if s is None:
        s = pool[device] = Solver(device, **_knobs)
    return s


def pipeline_solvers(device: int, depth: int, lease: bool = False):
    """``depth`` solvers for ``device`` from the calling thread's pool, used
    by the batch stream (supergraph.solve_seed_supergraphs) and created on
    first use.  lease=True hands out a set no running stream of this thread
    holds (nested streams get their own solvers; give it back with
    release_solvers); without it, the most recent set (its statistics)."""
    pool = getattr(_tls, "pipes", None)
    if pool is None:
        pool = _tls.pipes = {}
    sets = pool.setdefault(device, [])
    if not lease:
        return sets[-1][1][:depth] if sets else []
    for ent in sets:
        if not ent[0]:
            break
    else:
        ent = [False, []]
        sets.append(ent)
    while len(ent[1]) < depth:
        ent[1].append(Solver(device, **_knobs))
    ent[0] = True
    sets.remove(ent)
    sets.append(ent)   # most recent last
    return ent[1][:depth]


def release_solvers(device: int, solvers) -> None:
    """Give a leased solver set back to the calling thread's pool."""
    for ent in getattr(_tls, "pipes", {}).get(device, []):
        if ent[1][:len(solvers)] == list(solvers):
            ent[0] = False
            return


_dev_locks = {}
_dev_locks_mu = threading.Lock()


def device_lock(device: int) -> threading.Lock:
    """Process-wide lock serialising device solves of one GPU: solvers of
    different threads may stage and fetch concurrently, but their persistent
    and cooperative kernels never share the device."""
    with _dev_locks_mu:
        lk = _dev_locks.get(device)
        if lk is None:
            lk = _dev_locks[device] = threading.Lock()
        return lk


def plane_stats(planes):
    """[(min, max, sum, sum below CAP_MAX)] of int64 planes, reduced on all
    host cores by the native library (pmf_plane_stats)."""
    lib = load_library()
    arrs = [np.ascontiguousarray(a, np.int64).reshape(-1) for a in planes]
    sizes = np.array([a.size for a in arrs], np.int64)
    out = np.zeros((len(arrs), 4), np.int64)
    P = ctypes.POINTER
    rc = lib.pmf_plane_stats(len(arrs), _ptrs(arrs), sizes.ctypes.data_as(P(ctypes.c_int64)),
                             out.ctypes.data_as(P(ctypes.c_int64)))
    if rc:
        _raise_for(rc)
    return [tuple(int(v) for v in row) for row in out]
