"""ctypes loader for the C restatement of the reference radix tree (TEST INFRASTRUCTURE).

See oracle/radix_oracle.c.  Built by ``make -C oracle`` (called from
``__graft_entry__.build()``); tests and bench.py's CPU leg load it here.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libradix_oracle.so")

_P = C.c_void_p
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        l = C.CDLL(LIB)
        l.ro_create.restype = _P
        l.ro_destroy.argtypes = [_P]
        l.ro_insert_batch.argtypes = [_P, C.c_int64] + [_P] * 11 + [C.c_int]
        l.ro_match_batch.argtypes = [_P, C.c_int64] + [_P] * 6 + [C.c_int]
        l.ro_stats.argtypes = [_P, C.c_int64, _P, _P, _P]
        l.ro_row_len.argtypes = [_P, C.c_int64, C.c_int32]
        l.ro_row_len.restype = C.c_int64
        l.ro_export_row.argtypes = [_P, C.c_int64, C.c_int32, _P, _P, _P]
        l.ro_lex_rows.argtypes = [_P, C.c_int64, _P, _P]
        l.ro_export_batch.argtypes = [_P, C.c_int64, _P, _P, _P, _P, _P, _P, C.c_int]
        _lib = l
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class CRadixStore:
    """Many sessions of the reference radix tree, in C.  Session ids are ints."""

    def __init__(self):
        self.h = lib().ro_create()

    def close(self):
        if self.h:
            lib().ro_destroy(self.h)
            self.h = None

    __del__ = close

    def insert_batch(self, sids, tokens, tok_off, run_off, run_start, run_origin, run_version, nthreads=1):
        n = len(sids)
        sids = np.ascontiguousarray(sids, np.int32)
        tokens = np.ascontiguousarray(tokens, np.int32)
        tok_off = np.ascontiguousarray(tok_off, np.int64)
        run_off = np.ascontiguousarray(run_off, np.int64)
        run_start = np.ascontiguousarray(run_start, np.int32)
        run_origin = np.ascontiguousarray(run_origin, np.uint8)
        run_version = np.ascontiguousarray(run_version, np.int32)
        m = np.zeros(n, np.int32)
        row = np.zeros(n, np.int32)
        par = np.zeros(n, np.int32)
        add = np.zeros(n, np.int32)
        rc = lib().ro_insert_batch(self.h, n, _p(sids), _p(tokens), _p(tok_off), _p(run_off), _p(run_start),
                                   _p(run_origin), _p(run_version), _p(m), _p(row), _p(par), _p(add), nthreads)
        if rc:
            raise ValueError("cannot insert an empty sequence")
        return m, row, par, add

    def match_batch(self, sids, tokens, tok_off, nthreads=1):
        n = len(sids)
        sids = np.ascontiguousarray(sids, np.int32)
        tokens = np.ascontiguousarray(tokens, np.int32)
        tok_off = np.ascontiguousarray(tok_off, np.int64)
        m = np.zeros(n, np.int64)
        par = np.zeros(n, np.int32)
        dup = np.zeros(n, np.int32)
        lib().ro_match_batch(self.h, n, _p(sids), _p(tokens), _p(tok_off), _p(m), _p(par), _p(dup), nthreads)
        return m, par, dup

    def stats(self, sid):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int32()
        if lib().ro_stats(self.h, sid, C.byref(a), C.byref(b), C.byref(c)):
            raise KeyError(sid)
        return a.value, b.value, c.value

    def export_row(self, sid, row):
        L = lib().ro_row_len(self.h, sid, row)
        if L < 0:
            raise KeyError((sid, row))
        t = np.empty(L, np.int32)
        m = np.empty(L, np.uint8)
        v = np.empty(L, np.int32)
        lib().ro_export_row(self.h, sid, row, _p(t), _p(m), _p(v))
        return t, m, v

    def export_batch(self, sids, rows, nthreads=1):
        """Rows (sids[k], rows[k]) packed: (offsets[n+1], tokens, mask, versions)."""
        sids = np.ascontiguousarray(sids, np.int64)
        rows = np.ascontiguousarray(rows, np.int32)
        lens = np.array([lib().ro_row_len(self.h, int(s), int(r)) for s, r in zip(sids, rows)], np.int64)
        if np.any(lens < 0):
            raise KeyError("unknown row")
        off = np.zeros(len(rows) + 1, np.int64)
        np.cumsum(lens, out=off[1:])
        t = np.empty(off[-1], np.int32)
        m = np.empty(off[-1], np.uint8)
        v = np.empty(off[-1], np.int32)
        if lib().ro_export_batch(self.h, len(rows), _p(sids), _p(rows), _p(off), _p(t), _p(m), _p(v), nthreads):
            raise KeyError("unknown row")
        return off, t, m, v

    def lex_rows(self, sid):
        _, _, nrows = self.stats(sid)
        out = np.empty(max(nrows, 1), np.int32)
        n = C.c_int32()
        lib().ro_lex_rows(self.h, sid, _p(out), C.byref(n))
        return out[: n.value]
