"""Dynamic FIFO dispatch of supergraph tasks onto GPUs.

Mirror of the in-scope part of /root/reference/pkg/src/pmflow/scheduler.py:
``Task`` / ``WorkerHandle`` / ``TaskRecord`` / ``TaskSchedule`` /
``Completion`` (:44-95), ``ThreadedBackend`` (:137-200) and ``run_dynamic``
(:253-292) with the same policy: worker tokens (``slots`` per worker) in a
FIFO; the head token takes the next pending task and re-enters at the tail
when it completes; a failed worker is retired and its task retried once at
the front; a second failure aborts the batch.

B200 side: a worker of kind ``"gpu"`` is one CUDA device (``endpoint`` holds
the device ordinal).  ``GpuBackend`` gives each device one executor thread
with its own solver/stream; tasks dispatched to a device while it is busy
are coalesced into the next device batch (every grid of every coalesced
supergraph is discharged by the same kernel launches), so ``slots`` tokens
per GPU become batch depth instead of idle threads (composite tasks share
one device batch; seed-supergraph tasks run as a batch stream whose host
staging and decoding overlap the device).  CUDA errors surface as
``WorkerFailure`` and go through the reference's retry path.
"""

from __future__ import annotations

import queue
import threading
import time
from collections import deque
from concurrent.futures import FIRST_COMPLETED, ThreadPoolExecutor, wait as futures_wait
from dataclasses import dataclass

from .grid import CutResult, GridGraph
from .supergraph import (SupergraphLayout, solve_composite, solve_composites, solve_seed_supergraph,
                         solve_seed_supergraphs)


class SchedulerError(RuntimeError):
    pass


class WorkerFailure(SchedulerError):
    """A worker failed while executing a task."""


class BatchAborted(SchedulerError):
    """The policy gave up on the batch."""


@dataclass(frozen=True)
class Task:
    """One unit of work: a (composite) graph, or -- device-built -- a seed
    supergraph given by its problems and schedule."""

    id: int
    graph: GridGraph | None = None
    layout: SupergraphLayout | None = None
    duration: int = 1
    problems: tuple | None = None
    schedule: object = None
    swap_mode: str = "auto"


@dataclass(frozen=True)
class WorkerHandle:
    id: int
    kind: str = "local"  # "local" | "gpu"
    endpoint: str | None = None
    slots: int = 1


@dataclass(frozen=True)
class TaskRecord:
    task_id: int
    worker_id: int
    start: float
    finish: float
    attempt: int = 1


@dataclass(frozen=True)
class TaskSchedule:
    records: tuple

    @property
    def makespan(self) -> float:
        return max((r.finish for r in self.records), default=0)

    def record_for(self, task_id: int) -> TaskRecord:
        for r in self.records:
            if r.task_id == task_id:
                return r
        raise KeyError(task_id)


@dataclass(frozen=True)
class Completion:
    task: Task
    worker: WorkerHandle
    attempt: int
    start: float
    finish: float
    cut: object
    error: Exception | None


def _wrap(exc: Exception) -> WorkerFailure:
    if isinstance(exc, WorkerFailure):
        return exc
    err = WorkerFailure(str(exc))
    err.__cause__ = exc
    return err


def _solve_one(task: Task, device: int = 0):
    if task.problems is not None:
        return solve_seed_supergraph(task.problems, task.schedule, task.swap_mode, device=device)
    return solve_composite(task.graph, task.layout, device=device)


class ThreadedBackend:
    """Per-worker thread pools, ``slots`` wide; local tasks run the device
    solve_composite on the calling thread's solver (the reference's local
    solver hook, scheduler.py:141-142, is kept: ``local_solver(task)``)."""

    def __init__(self, local_solver=None):
        self._solve = local_solver or (lambda t: _solve_one(t, 0))
        self._pools = {}
        self._outstanding = {}
        self._t0 = time.monotonic()

    def _now(self) -> float:
        return time.monotonic() - self._t0

    def _run(self, worker: WorkerHandle, task: Task, attempt: int) -> Completion:
        start = self._now()
        cut, err = None, None
        try:
            if worker.kind == "gpu":
                cut = _solve_one(task, int(worker.endpoint or 0))
            else:
                cut = self._solve(task)
        except Exception as exc:  # noqa: BLE001 -- surfaced as a worker failure
            err = _wrap(exc)
        return Completion(task, worker, attempt, start, self._now(), cut, err)

    def submit(self, worker: WorkerHandle, task: Task, attempt: int = 1) -> None:
        pool = self._pools.get(worker.id)
        if pool is None:
            pool = self._pools[worker.id] = ThreadPoolExecutor(max_workers=worker.slots)
        self._outstanding[pool.submit(self._run, worker, task, attempt)] = None

    def wait_any(self) -> Completion:
        if not self._outstanding:
            raise SchedulerError("wait_any with nothing outstanding")
        done, _ = futures_wait(list(self._outstanding), return_when=FIRST_COMPLETED)
        fut = next(iter(done))
        del self._outstanding[fut]
        return fut.result()

    def close(self) -> None:
        for pool in self._pools.values():
            pool.shutdown(wait=True, cancel_futures=True)
        self._pools.clear()
        self._outstanding.clear()


class GpuBackend:
    """One executor thread per GPU; everything dispatched to a GPU while it
    is busy is solved together in its next device batch."""

    def __init__(self, max_batch: int = 64, solver=None):
        self._max_batch = max_batch
        self._inbox = {}
        self._threads = {}
        self._done = queue.Queue()
        self._pending = 0
        self._t0 = time.monotonic()
        self._solver = solver     # optional fn(list[Task], device) -> list[result]
        self._stop = False

    def _now(self):
        return time.monotonic() - self._t0

    def _loop(self, worker: WorkerHandle):
        dev = int(worker.endpoint or 0)
        inbox = self._inbox[worker.id]
        while True:
            first = inbox.get()
            if first is None:
                return
            batch = [first]
            while len(batch) < self._max_batch:
                try:
                    nxt = inbox.get_nowait()
                except queue.Empty:
                    break
                if nxt is None:
                    inbox.put(None)
                    break
                batch.append(nxt)
            start = self._now()
            try:
                results = self._run_batch([t for t, _ in batch], dev)
                errs = [None] * len(batch)
            except Exception as exc:  # noqa: BLE001
                if len(batch) == 1:
                    results, errs = [None], [_wrap(exc)]
                else:
                    # a coalesced batch failed: solve its tasks one at a time so
                    # the failure is charged to the task that caused it (the
                    # reference charges only the failing task, scheduler.py:270-279)
                    results, errs = [], []
                    for t, _ in batch:
                        try:
                            results.append(self._run_batch([t], dev)[0])
                            errs.append(None)
                        except Exception as exc1:  # noqa: BLE001
                            results.append(None)
                            errs.append(_wrap(exc1))
            fin = self._now()
            for (task, attempt), res, err in zip(batch, results, errs):
                self._done.put(Completion(task, worker, attempt, start, fin, res, err))

    def _run_batch(self, tasks, dev):
        if self._solver is not None:
            return self._solver(tasks, dev)
        out = [None] * len(tasks)
        comp = [i for i, t in enumerate(tasks) if t.problems is None]
        if comp:
            for i, r in zip(comp, solve_composites([(tasks[i].graph, tasks[i].layout)
                                                    for i in comp], device=dev)):
                out[i] = r
        # seed supergraphs: one batch stream per (schedule, swap mode), so the
        # admission / staging of task k+1 and the decode of task k-1 overlap
        # the device solve of task k (an error fails the coalesced batch,
        # which _loop then re-solves task by task)
        groups = {}
        for i, t in enumerate(tasks):
            if t.problems is not None:
                groups.setdefault((tuple(t.schedule.values), t.swap_mode), []).append(i)
        for idx in groups.values():
            if len(idx) == 1:
                out[idx[0]] = _solve_one(tasks[idx[0]], dev)
                continue
            t0 = tasks[idx[0]]
            for i, res in zip(idx, solve_seed_supergraphs([tasks[i].problems for i in idx], t0.schedule,
                                                          t0.swap_mode, device=dev)):
                out[i] = res
        return out

    def submit(self, worker: WorkerHandle, task: Task, attempt: int = 1) -> None:
        if worker.id not in self._threads:
            self._inbox[worker.id] = queue.Queue()
            th = threading.Thread(target=self._loop, args=(worker,), daemon=True)
            self._threads[worker.id] = th
            th.start()
        self._pending += 1
        self._inbox[worker.id].put((task, attempt))

    def wait_any(self) -> Completion:
        if self._pending == 0:
            raise SchedulerError("wait_any with nothing outstanding")
        comp = self._done.get()
        self._pending -= 1
        return comp

    def close(self) -> None:
        for q in self._inbox.values():
            q.put(None)
        for th in self._threads.values():
            th.join()
        self._threads.clear()
        self._inbox.clear()


def run_dynamic(tasks, workers, backend):
    """FIFO work queue over worker tokens; one retry per task."""
    pending = deque(tasks)
    workers = list(workers)
    if not workers:
        raise SchedulerError("no workers")
    tokens = deque(w for w in workers for _ in range(w.slots))
    records, cuts = [], {}
    retried, dead = set(), set()
    in_flight = 0
    while pending or in_flight:
        while pending and tokens:
            w = tokens.popleft()
            t = pending.popleft()
            backend.submit(w, t, attempt=2 if t.id in retried else 1)
            in_flight += 1
        if in_flight == 0:
            raise BatchAborted(f"{len(pending)} tasks pending and every worker retired")
        comp = backend.wait_any()
        in_flight -= 1
        if comp.error is not None:
            dead.add(comp.worker.id)
            tokens = deque(w for w in tokens if w.id not in dead)
            if comp.task.id in retried:
                raise BatchAborted(f"task {comp.task.id} failed twice; batch aborted") from comp.error
            retried.add(comp.task.id)
            pending.appendleft(comp.task)
            continue
        records.append(TaskRecord(comp.task.id, comp.worker.id, comp.start, comp.finish,
                                  comp.attempt))
        cuts[comp.task.id] = comp.cut
        if comp.worker.id not in dead:
            tokens.append(comp.worker)
    return TaskSchedule(tuple(records)), cuts


def gpu_workers(devices, slots: int = 4):
    """One WorkerHandle per CUDA device ordinal."""
    return [WorkerHandle(id=i, kind="gpu", endpoint=str(d), slots=slots)
            for i, d in enumerate(devices)]
