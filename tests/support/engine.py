"""Test doubles for the trajectory manager's collaborators (TEST INFRASTRUCTURE).

The reference drives TrajectoryManager with a deterministic mock LLM engine
(rolloutlab/engine.py:150-379) and a rollout controller (rollout.py:163-386); both
are out of scope for the B200 path, but the drop-in manager needs something with
the same protocol on the GPU box (where /root/reference does not exist).  These are
compact restatements of that protocol — pinned to the reference's frozen token
streams and to tests/golden/engine_vectors.json (tests/test_engine_double.py).

Token function (engine.py:35-46, frozen byte layout):
    sha256(b"tokgen1" + le64(seed) + le32(version) + le32(len(ctx)) + le32(t)...)[:8]
    as big-endian uint64, mod vocab.
"""

from __future__ import annotations

import hashlib
import itertools
import struct
import threading
from dataclasses import dataclass, field
from enum import Enum

import numpy as np


def next_token(context, seed: int, version: int, vocab_size: int) -> int:
    h = hashlib.sha256()
    h.update(b"tokgen1" + struct.pack("<qII", seed, version, len(context)))
    h.update(np.asarray(context, dtype="<u4").tobytes())
    return int.from_bytes(h.digest()[:8], "big") % vocab_size


def oracle_generate(input_tokens, params, version, vocab_size, prefix=()):
    out = list(prefix)
    while len(out) < params.max_new_tokens:
        t = next_token(list(input_tokens) + out, params.seed, version, vocab_size)
        out.append(t)
        if params.stop_condition is not None and t == params.stop_condition:
            break
    return out[len(prefix):]


class WaitSignal(Exception):
    """Engine is switching weights; retry later (engine.py:103-109)."""


class StepOutcome(Enum):
    TOKEN = "token"
    FINISHED = "finished"
    INTERRUPTED = "interrupted"


@dataclass
class Result:
    output_tokens: list
    version_per_token: list
    finished: bool
    request_id: str | None = None


@dataclass
class _Job:
    request_id: str | None
    input_tokens: list
    prefix: list
    params: object
    produced: list = field(default_factory=list)
    versions: list = field(default_factory=list)
    interrupted: bool = False
    stopped: bool = False

    def remaining(self):
        return self.params.max_new_tokens - len(self.prefix) - len(self.produced)


class Engine:
    """Token-at-a-time engine with interrupt / weight-switch semantics."""

    def __init__(self, vocab_size=4096):
        self.vocab_size = vocab_size
        self.step_hook = None
        self._lock = threading.RLock()
        self._serving = threading.Event()
        self._serving.set()
        self._switching = False
        self._version = 0
        self._jobs: dict[str, _Job] = {}
        self._ids = itertools.count()
        self._log: list[tuple[str | None, Result]] = []

    @property
    def current_version(self):
        with self._lock:
            return self._version

    def wait_serving(self, timeout=None):
        return self._serving.wait(timeout)

    def oracle_log(self, request_id):
        with self._lock:
            return [r for rid, r in self._log if rid == request_id]

    def begin_switch(self):
        with self._lock:
            assert not self._switching
            self._switching = True
            self._serving.clear()
            for j in self._jobs.values():
                j.interrupted = True

    def complete_switch(self, v):
        with self._lock:
            assert self._switching and v > self._version
            self._version = v
            self._switching = False
            self._serving.set()

    def interrupt(self, job_ids=None):
        with self._lock:
            for jid in (list(self._jobs) if job_ids is None else job_ids):
                if jid in self._jobs:
                    self._jobs[jid].interrupted = True

    def start_job(self, input_tokens, params, *, prefix=(), request_id=None):
        params.validate()
        with self._lock:
            if self._switching:
                raise WaitSignal()
            jid = f"job-{next(self._ids)}"
            self._jobs[jid] = _Job(request_id, list(input_tokens), list(prefix), params)
            return jid

    def step_job(self, jid):
        with self._lock:
            job = self._jobs[jid]
        if self.step_hook is not None:
            self.step_hook(jid, len(job.produced))
        with self._lock:
            if job.interrupted or self._switching:
                job.interrupted = True
                return StepOutcome.INTERRUPTED
            if job.stopped or job.remaining() <= 0:
                return StepOutcome.FINISHED
            t = next_token(job.input_tokens + job.prefix + job.produced, job.params.seed, self._version,
                           self.vocab_size)
            job.produced.append(t)
            job.versions.append(self._version)
            if job.params.stop_condition is not None and t == job.params.stop_condition:
                job.stopped = True
                return StepOutcome.FINISHED
            return StepOutcome.FINISHED if job.remaining() <= 0 else StepOutcome.TOKEN

    def finish_job(self, jid):
        with self._lock:
            job = self._jobs.pop(jid)
            r = Result(list(job.produced), list(job.versions), not job.interrupted, job.request_id)
            self._log.append((job.request_id, r))
            return r


class Control:
    """Rollout gate: pause / resume / weight update (rollout.py:190-386 protocol)."""

    def __init__(self, engine: Engine):
        self.engine = engine
        self._lock = threading.RLock()
        self._tasks: dict[str, dict] = {}
        self._order: list[str] = []

    def admit_task(self, tid, snapshot=None):
        with self._lock:
            self._tasks[tid] = dict(snapshot=snapshot, job=None, paused=False)

    def release_task(self, tid):
        with self._lock:
            self._tasks.pop(tid, None)
            if tid in self._order:
                self._order.remove(tid)

    def note_job(self, tid, jid):
        with self._lock:
            if tid in self._tasks:
                self._tasks[tid]["job"] = jid

    def is_runnable(self, tid):
        with self._lock:
            t = self._tasks.get(tid)
            return t is None or not t["paused"]

    def pause_rollouts(self):
        with self._lock:
            for tid, t in self._tasks.items():
                if t["paused"]:
                    continue
                produced_now = 0
                if t["job"] is not None:
                    job = self.engine._jobs.get(t["job"])
                    produced_now = len(job.produced) if job else 0
                    self.engine.interrupt([t["job"]])
                if t["snapshot"] is not None:
                    snap = t["snapshot"]()
                    if snap.budget_remaining - produced_now <= 0:
                        continue  # budget spent: the owner finalizes instead
                t["paused"] = True
                self._order.append(tid)

    def resume_rollouts(self):
        with self._lock:
            for tid in self._order:
                if tid in self._tasks:
                    self._tasks[tid]["paused"] = False
            self._order.clear()

    def coordinate_update(self, v):
        with self._lock:
            self.pause_rollouts()
            self.engine.begin_switch()
            self.engine.complete_switch(v)
            self.resume_rollouts()
