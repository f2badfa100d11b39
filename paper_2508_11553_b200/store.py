"""Batched Python front end of the B200 session-history store (libtmstore.so).

``DeviceStore`` owns one tm_store on one GPU.  Host-array calls are synchronous
(they are what the drop-in SessionTrie / TrajectoryManager use); the ``*_device``
variants take CUDA tensors and enqueue on a stream (trainer handoff, benchmarks).
PyTorch is used only to hand device memory and streams across; all compute is in
the CUDA kernels behind the C ABI.
"""

from __future__ import annotations

import array
import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import TM_MEM_DEVICE, TM_MEM_HOST, TM_ORDER_INSERT, TM_ORDER_LEX, check


def _ptr(a: np.ndarray | None):
    # the address as an int (c_void_p argtypes take ints; 2x cheaper than ctypes.data_as)
    return None if a is None else a.__array_interface__["data"][0]


def _addr(x, dtype):
    """Address of a contiguous buffer of ``dtype`` (array.array or numpy), and the object
    that keeps it alive."""
    if isinstance(x, array.array):
        if x.itemsize != np.dtype(dtype).itemsize:
            x = np.asarray(x, dtype)
        else:
            return x.buffer_info()[0], x
    x = np.ascontiguousarray(x, dtype)
    return x.__array_interface__["data"][0], x


def _tptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def runs_from_per_token(origins: np.ndarray, versions: np.ndarray):
    """Per-token (origin code, version) -> run starts / origins / versions."""
    n = len(origins)
    if n == 0:
        return np.zeros(0, np.int32), np.zeros(0, np.uint8), np.zeros(0, np.int32)
    o = np.asarray(origins, dtype=np.int64)
    v = np.asarray(versions, dtype=np.int64)
    cut = np.flatnonzero((o[1:] != o[:-1]) | (v[1:] != v[:-1])) + 1
    starts = np.concatenate(([0], cut))
    return starts.astype(np.int32), o[starts].astype(np.uint8), v[starts].astype(np.int32)


@dataclass
class RecordResult:
    """Per-entry outputs of a record batch (numpy arrays, batch order)."""

    matched: np.ndarray   # int64, InsertResult.matched_prefix_length
    row: np.ndarray       # int64 global row id
    local: np.ndarray     # int32 session-local ordinal (node_id of the drop-in API)
    parent: np.ndarray    # int64 global parent row, -1 if none
    parent_local: np.ndarray  # int32
    added: np.ndarray     # int64, InsertResult.added_tokens


@dataclass
class Packed:
    """cu_seqlens-style packed trajectories."""

    offsets: np.ndarray  # int64 [n+1]
    tokens: object       # int32 [total]  (numpy on host, torch tensor on device)
    loss_mask: object    # uint8 [total]
    versions: object     # int32 [total]
    resp_start: object   # int64 [n]: where the trailing model response starts


class DeviceStore:
    """A GPU-resident store of many sessions (one per device per process)."""

    def __init__(self, device: int = 0, *, arena_words: int = 1 << 22, row_capacity: int = 1 << 12,
                 run_capacity: int = 1 << 14, session_capacity: int = 1 << 10):
        self.lib = _lib.load()
        cfg = _lib.TmConfig(device, arena_words, row_capacity, run_capacity, session_capacity)
        h = C.c_void_p()
        check(self.lib.tm_store_create(C.byref(cfg), C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.lib.tm_store_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- sessions ----------------------------------------------------------------
    def new_session(self) -> int:
        sid = C.c_int32()
        check(self.lib.tm_session_create(self.h, C.byref(sid)))
        return sid.value

    def session_stats(self, sid: int) -> tuple[int, int, int]:
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(self.lib.tm_session_stats(self.h, sid, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def session_rows(self, sid: int, order: str = "insert") -> np.ndarray:
        _, _, n = self.session_stats(sid)
        out = np.empty(max(n, 1), np.int64)
        got = C.c_int64()
        code = TM_ORDER_LEX if order == "lex" else TM_ORDER_INSERT
        check(self.lib.tm_session_rows(self.h, sid, code, _ptr(out), n, C.byref(got)))
        return out[: got.value]

    def row_info(self, row: int):
        sid, loc = C.c_int32(), C.c_int32()
        par, m, L = C.c_int64(), C.c_int64(), C.c_int64()
        check(self.lib.tm_row_info(self.h, row, C.byref(sid), C.byref(loc), C.byref(par), C.byref(m), C.byref(L)))
        return dict(session=sid.value, local=loc.value, parent=par.value, matched=m.value, length=L.value)

    def stats(self) -> dict:
        r, u, c, d = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        check(self.lib.tm_store_stats(self.h, C.byref(r), C.byref(u), C.byref(c), C.byref(d)))
        return dict(rows=r.value, arena_used=u.value, arena_cap=c.value, max_depth=d.value)

    def counters(self) -> dict:
        """Calls / items / tokens seen by this store (observability)."""
        c = np.zeros(8, np.int64)
        check(self.lib.tm_store_counters(self.h, _ptr(c)))
        keys = ("record_calls", "records", "record_tokens", "match_calls", "queries", "export_calls", "export_rows",
                "export_tokens")
        return dict(zip(keys, c.tolist()))

    def h2d_stats(self) -> dict:
        """How host-memory token inputs crossed PCIe: packed 18-bit planes or raw int32
        (tm_store_h2d_stats)."""
        c = np.zeros(6, np.int64)
        check(self.lib.tm_store_h2d_stats(self.h, _ptr(c)))
        keys = ("packed_calls", "packed_tokens", "raw_calls", "raw_tokens", "pack_fallbacks", "token_bytes")
        return dict(zip(keys, c.tolist()))

    def stream(self) -> int:
        s = C.c_void_p()
        check(self.lib.tm_store_stream(self.h, C.byref(s)))
        return s.value or 0

    def save(self, path: str) -> None:
        """Snapshot the store (arena, rows, runs, counters) to ``path``."""
        check(self.lib.tm_store_save(self.h, str(path).encode()))

    @classmethod
    def load(cls, path: str, device: int = 0) -> "DeviceStore":
        """A new store on ``device`` restored from a snapshot (branch index rebuilt)."""
        st = cls(device)
        check(st.lib.tm_store_load(st.h, str(path).encode()))
        return st

    KERNELS = {"walk": 0, "commit": 1, "export": 2, "plan": 3, "route": 4, "route_pack": 5, "route_wait": 6,
               "record_copy": 7, "block_hash": 8}

    def profile_begin(self, reserve: int = 0):
        """Start recording CUDA events around every kernel launch of this store (with
        ``reserve``: create the event pairs of that many launches per kernel kind now)."""
        if reserve:
            check(self.lib.tm_profile_reserve(self.h, int(reserve)))
        check(self.lib.tm_profile_begin(self.h))

    def profile_end(self, kernel: str = "walk") -> tuple[float, int]:
        """(summed device ms, launches) of one kernel kind since profile_begin."""
        ms, n = C.c_double(), C.c_int64()
        check(self.lib.tm_profile_end(self.h, self.KERNELS[kernel], C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def synchronize(self):
        check(self.lib.tm_synchronize(self.h))

    # -- record (batched lpm_insert) ------------------------------------------------
    def record_packed(self, sids, tokens, tok_off, tok_len, run_off, run_start, run_origin, run_version) -> RecordResult:
        sids = np.ascontiguousarray(sids, np.int32)
        tokens = np.ascontiguousarray(tokens, np.int32)
        tok_off = np.ascontiguousarray(tok_off, np.int64)
        tok_len = np.ascontiguousarray(tok_len, np.int64)
        run_off = np.ascontiguousarray(run_off, np.int64)
        run_start = np.ascontiguousarray(run_start, np.int32)
        run_origin = np.ascontiguousarray(run_origin, np.uint8)
        run_version = np.ascontiguousarray(run_version, np.int32)
        n = len(sids)
        if not (len(tok_off) >= n and len(tok_len) == n and len(run_off) == n + 1):
            raise ValueError("inconsistent batch arrays")
        r = RecordResult(np.empty(n, np.int64), np.empty(n, np.int64), np.empty(n, np.int32),
                         np.empty(n, np.int64), np.empty(n, np.int32), np.empty(n, np.int64))
        check(self.lib.tm_record_batch(
            self.h, n, TM_MEM_HOST, _ptr(sids), _ptr(tokens), _ptr(tok_off), _ptr(tok_len), _ptr(run_off),
            _ptr(run_start), _ptr(run_origin), _ptr(run_version), _ptr(r.matched), _ptr(r.row), _ptr(r.local),
            _ptr(r.parent), _ptr(r.parent_local), _ptr(r.added), None))
        return r

    def record_device(self, sids, tokens, tok_off, tok_len, run_off, run_start, run_origin, run_version,
                      stream=None) -> RecordResult:
        """record_packed with the token buffer already on the GPU (a CUDA tensor, every
        sequence starting at a multiple of 32 words); other arrays are host arrays.  The
        tokens are read after the work queued on ``stream`` (default: torch's current)."""
        if stream is None:
            import torch

            stream = torch.cuda.current_stream(self.device).cuda_stream
        sids = np.ascontiguousarray(sids, np.int32)
        tok_off = np.ascontiguousarray(tok_off, np.int64)
        tok_len = np.ascontiguousarray(tok_len, np.int64)
        run_off = np.ascontiguousarray(run_off, np.int64)
        run_start = np.ascontiguousarray(run_start, np.int32)
        run_origin = np.ascontiguousarray(run_origin, np.uint8)
        run_version = np.ascontiguousarray(run_version, np.int32)
        n = len(sids)
        r = RecordResult(np.empty(n, np.int64), np.empty(n, np.int64), np.empty(n, np.int32),
                         np.empty(n, np.int64), np.empty(n, np.int32), np.empty(n, np.int64))
        check(self.lib.tm_record_batch(
            self.h, n, TM_MEM_DEVICE, _ptr(sids), _tptr(tokens), _ptr(tok_off), _ptr(tok_len), _ptr(run_off),
            _ptr(run_start), _ptr(run_origin), _ptr(run_version), _ptr(r.matched), _ptr(r.row), _ptr(r.local),
            _ptr(r.parent), _ptr(r.parent_local), _ptr(r.added), self._stream_arg(stream)))
        return r

    def record_one(self, sid: int, tokens, runs) -> RecordResult:
        """Single-sequence record (the per-request path) through tm_record_one: no batch
        arrays.  ``tokens``: int32 numpy array or array.array('i'); ``runs``: (starts,
        origin codes, versions)."""
        st, org, ver = runs
        pt, kt = _addr(tokens, np.int32)
        ps, ks = _addr(st, np.int32)
        po, ko = _addr(org, np.uint8)
        pv, kv = _addr(ver, np.int32)
        out = (C.c_int64 * 6)()
        check(self.lib.tm_record_one(self.h, sid, pt, len(kt), ps, po, pv, len(ks), C.addressof(out)))
        m, row, local, par, par_local, added = out
        # one-element lists, not arrays: this is the per-request path and every microsecond shows
        return RecordResult([m], [row], [local], [par], [par_local], [added])

    def record(self, sids, seqs, runs) -> RecordResult:
        """seqs: list of int sequences; runs: list of (starts, origins, versions)."""
        lens = np.fromiter((len(s) for s in seqs), np.int64, len(seqs))
        off = np.zeros(len(seqs) + 1, np.int64)
        np.cumsum(lens, out=off[1:])
        tokens = np.concatenate([np.asarray(s, np.int64) for s in seqs]) if seqs else np.zeros(0, np.int64)
        if tokens.size and (tokens.min() < -(2**31) or tokens.max() >= 2**31):
            raise ValueError("token ids must fit in int32")
        rc = np.fromiter((len(r[0]) for r in runs), np.int64, len(runs))
        roff = np.zeros(len(runs) + 1, np.int64)
        np.cumsum(rc, out=roff[1:])
        cat = lambda i, dt: np.concatenate([np.asarray(r[i], dt) for r in runs]) if runs else np.zeros(0, dt)  # noqa: E731
        return self.record_packed(sids, tokens, off[:-1], lens, roff, cat(0, np.int32), cat(1, np.uint8), cat(2, np.int32))

    # -- read-only match --------------------------------------------------------------
    def match(self, sids, tokens, tok_off, tok_len):
        sids = np.ascontiguousarray(sids, np.int32)
        tokens = np.ascontiguousarray(tokens, np.int32)
        tok_off = np.ascontiguousarray(tok_off, np.int64)
        tok_len = np.ascontiguousarray(tok_len, np.int64)
        n = len(sids)
        m = np.empty(n, np.int64)
        p = np.empty(n, np.int64)
        d = np.empty(n, np.int64)
        check(self.lib.tm_match_batch(self.h, n, TM_MEM_HOST, _ptr(sids), _ptr(tokens), _ptr(tok_off), _ptr(tok_len),
                                      _ptr(m), _ptr(p), _ptr(d), None))
        return m, p, d

    def match_lists(self, sids, seqs):
        """match() for Python callers holding token lists (the reference's argument type):
        the lists are flattened into one int32 buffer by host threads (csrc/tmfast.c), then
        one host-buffer match call."""
        from . import _tmfast

        tok, off = _tmfast.pack_lists(seqs, os.cpu_count() or 1)
        off = np.frombuffer(off, np.int64)
        return self.match(sids, np.frombuffer(tok, np.int32), off[:-1], np.diff(off))

    @staticmethod
    def _stream_arg(stream):
        # torch reports the legacy default stream as 0; the C ABI reads NULL as "the
        # store's own stream", so pass cudaStreamLegacy (0x1) explicitly
        return C.c_void_p(1 if stream == 0 else stream)

    def match_device(self, sids, tokens, tok_off, tok_len, out_matched, out_parent, out_dup, stream=None):
        """All CUDA tensors on this store's device; tok_off multiples of 32; enqueued on
        ``stream`` (a cudaStream_t int, default: torch's current stream)."""
        if stream is None:
            import torch

            stream = torch.cuda.current_stream(self.device).cuda_stream
        check(self.lib.tm_match_batch(self.h, sids.numel(), TM_MEM_DEVICE, _tptr(sids), _tptr(tokens), _tptr(tok_off),
                                      _tptr(tok_len), _tptr(out_matched), _tptr(out_parent), _tptr(out_dup),
                                      self._stream_arg(stream)))

    def block_hashes(self, tokens, out, stream=None):
        """Per-128-word block hashes of a device token buffer (tm_block_hashes)."""
        if stream is None:
            import torch

            stream = torch.cuda.current_stream(self.device).cuda_stream
        check(self.lib.tm_block_hashes(self.h, _tptr(tokens), tokens.numel(), _tptr(out), self._stream_arg(stream)))

    # -- export (trajectory assembly) ---------------------------------------------------
    def rows_total(self, rows) -> int:
        rows = np.ascontiguousarray(rows, np.int64)
        t = C.c_int64()
        check(self.lib.tm_rows_total(self.h, len(rows), _ptr(rows), C.byref(t)))
        return t.value

    def _pinned_views(self, specs):
        """Numpy arrays carved out of this store's page-locked export pool (grown x2 on
        demand): the copy engine writes them at full PCIe rate, with no pinned -> pageable
        pass.  The views are reused by the next pinned export of this store."""
        import torch

        sizes = [((int(n) * np.dtype(dt).itemsize + 255) // 256) * 256 for n, dt in specs]
        need = max(256, sum(sizes))
        pool = getattr(self, "_pin_pool", None)
        if pool is None or pool.numel() < need:
            self._pin_pool = pool = torch.empty(max(need, 2 * (pool.numel() if pool is not None else 0)),
                                                dtype=torch.uint8, pin_memory=True)
        base = pool.numpy()
        out, o = [], 0
        for (n, dt), sz in zip(specs, sizes):
            out.append(base[o: o + int(n) * np.dtype(dt).itemsize].view(dt))
            o += sz
        return out

    def export(self, rows, total: int | None = None, *, pinned: bool = False) -> Packed:
        """Packed trajectories of ``rows`` in host numpy arrays (``total``: their summed
        length when the caller already knows it, saving a round trip).  ``pinned``: the
        arrays are views of the store's page-locked export pool (written directly by the
        copy engine; valid until the next pinned export of this store - copy to keep)."""
        rows = np.ascontiguousarray(rows, np.int64)
        n = len(rows)
        if total is None:
            total = self.rows_total(rows) if n else 0
        off = np.zeros(n + 1, np.int64)
        if pinned:
            tok, msk, ver, resp = self._pinned_views([(total, np.int32), (total, np.uint8), (total, np.int32),
                                                       (n, np.int64)])
        else:
            tok = np.empty(total, np.int32)
            msk = np.empty(total, np.uint8)
            ver = np.empty(total, np.int32)
            resp = np.empty(n, np.int64)
        check(self.lib.tm_export_rows(self.h, n, _ptr(rows), TM_MEM_HOST, _ptr(off), _ptr(tok), _ptr(msk), _ptr(ver),
                                      _ptr(resp), None))
        return Packed(off, tok, msk, ver, resp)

    def export_ndjson(self, rows, session_ids, *, as_array: bool = False, pinned: bool = False):
        """Canonical NDJSON lines of ``rows`` (one per row, "\n"-terminated), formatted on
        the GPU; byte-identical to trajectory_to_line (core.py:182-183).  ``session_ids``:
        the session id string of each row."""
        import json

        rows = np.ascontiguousarray(rows, np.int64)
        n = len(rows)
        if n == 0:
            return np.zeros(0, np.uint8) if as_array else b""
        lits = [json.dumps(s).encode("ascii") for s in session_ids]
        sid_off = np.zeros(n + 1, np.int64)
        np.cumsum([len(x) for x in lits], out=sid_off[1:])
        sid = np.frombuffer(b"".join(lits) or b"\0", np.uint8)
        size = C.c_int64()
        check(self.lib.tm_export_ndjson(self.h, n, _ptr(rows), _ptr(sid), _ptr(sid_off), TM_MEM_HOST, None, 0,
                                        C.byref(size), None))
        out = self._pinned_views([(max(size.value, 1), np.uint8)])[0] if pinned else np.empty(max(size.value, 1), np.uint8)
        got = C.c_int64()
        check(self.lib.tm_export_ndjson(self.h, n, _ptr(rows), _ptr(sid), _ptr(sid_off), TM_MEM_HOST, _ptr(out),
                                        size.value, C.byref(got), None))
        return out[: got.value] if as_array else out[: got.value].tobytes()

    def export_device(self, rows, stream=None) -> Packed:
        """Packed trajectories left on the GPU as torch tensors (trainer handoff)."""
        import torch

        rows = np.ascontiguousarray(rows, np.int64)
        n = len(rows)
        total = self.rows_total(rows) if n else 0
        dev = torch.device("cuda", self.device)
        tok = torch.empty(total, dtype=torch.int32, device=dev)
        msk = torch.empty(total, dtype=torch.uint8, device=dev)
        ver = torch.empty(total, dtype=torch.int32, device=dev)
        resp = torch.empty(n, dtype=torch.int64, device=dev)
        off = np.zeros(n + 1, np.int64)
        if stream is None:
            stream = torch.cuda.current_stream(self.device).cuda_stream
        check(self.lib.tm_export_rows(self.h, n, _ptr(rows), TM_MEM_DEVICE, _ptr(off), _tptr(tok), _tptr(msk), _tptr(ver),
                                      _tptr(resp), self._stream_arg(stream)))
        return Packed(off, tok, msk, ver, resp)


    def export_device_with_host_rows(self, rows, host_rows, stream=None) -> Packed:
        """export_device of ``rows`` followed, in the same packed device batch, by rows that
        live on the host (open / paused requests, trajectory.py:329-340): ``host_rows`` is a
        list of (tokens, n_input, context_version, versions_of_the_output) - the input span
        at the context version, then MODEL_OUTPUT positions at their per-token versions
        (tm_export_host_rows)."""
        import torch

        rows = np.ascontiguousarray(rows, np.int64)
        n = len(rows)
        total = self.rows_total(rows) if n else 0
        nh = len(host_rows)
        hl = np.fromiter((len(t) for t, *_ in host_rows), np.int64, nh)
        tok_off = np.zeros(nh + 1, np.int64)
        np.cumsum(hl, out=tok_off[1:])
        htotal = int(tok_off[-1])
        dev = torch.device("cuda", self.device)
        tok = torch.empty(total + htotal, dtype=torch.int32, device=dev)
        msk = torch.empty(total + htotal, dtype=torch.uint8, device=dev)
        ver = torch.empty(total + htotal, dtype=torch.int32, device=dev)
        resp = torch.empty(n + nh, dtype=torch.int64, device=dev)
        off = np.zeros(n + nh + 1, np.int64)
        if stream is None:
            stream = torch.cuda.current_stream(self.device).cuda_stream
        sa = self._stream_arg(stream)
        if n:
            check(self.lib.tm_export_rows(self.h, n, _ptr(rows), TM_MEM_DEVICE, _ptr(off), _tptr(tok), _tptr(msk),
                                          _tptr(ver), _tptr(resp), sa))
        off[n + 1:] = total + tok_off[1:]
        if nh:
            tokens = np.concatenate([np.asarray(t, np.int32) for t, *_ in host_rows]) if htotal else np.zeros(1, np.int32)
            n_in = np.fromiter((int(x[1]) for x in host_rows), np.int64, nh)
            cv = np.fromiter((int(x[2]) for x in host_rows), np.int32, nh)
            starts, vers, roff = [], [], [0]
            for (t, ni, _, v) in host_rows:
                v = np.asarray(v, np.int64)
                if len(v):
                    cut = np.flatnonzero(v[1:] != v[:-1]) + 1
                    st = np.concatenate(([0], cut))
                    starts.append(st + int(ni))
                    vers.append(v[st])
                roff.append(roff[-1] + (len(starts[-1]) if len(v) else 0))
            rs = np.concatenate(starts).astype(np.int32) if starts else np.zeros(1, np.int32)
            rv = np.concatenate(vers).astype(np.int32) if vers else np.zeros(1, np.int32)
            roff = np.asarray(roff, np.int64)
            out_off = np.ascontiguousarray(off[n:n + nh])
            check(self.lib.tm_export_host_rows(self.h, nh, _ptr(tokens), _ptr(tok_off), _ptr(n_in), _ptr(cv),
                                               _ptr(roff), _ptr(rs), _ptr(rv), _ptr(out_off), _tptr(tok), _tptr(msk),
                                               _tptr(ver), C.c_void_p(resp.data_ptr() + 8 * n), sa))
        return Packed(off, tok, msk, ver, resp)

_default: dict[int, DeviceStore] = {}


def default_store(device: int = 0) -> DeviceStore:
    """Process-wide store for stand-alone SessionTrie objects."""
    st = _default.get(device)
    if st is None:
        st = _default[device] = DeviceStore(device)
    return st
