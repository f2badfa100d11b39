"""Seeded synthetic workloads for the five BASELINE.json configs,
plus packing helpers shared by tests and bench.py.

Token ids are uniform in [0, 151,936) (Qwen3 vocabulary), drawn from
numpy PCG64 with seed = 20251018 + config_index.  Nothing here is on the product
path; it only builds inputs.
"""

from __future__ import annotations

import numpy as np

VOCAB = 151_936
SEED0 = 20251018
ALIGN = 32  # words; the store wants 128-byte aligned sequence starts


def per_token_runs(origins, versions):
    """Per-token (origin 0/1, version) -> (relative starts, origins, versions) runs."""
    o = np.asarray(origins, dtype=np.int64)
    v = np.asarray(versions, dtype=np.int64)
    if len(o) == 0:
        return np.zeros(0, np.int32), np.zeros(0, np.uint8), np.zeros(0, np.int32)
    chg = np.flatnonzero((o[1:] != o[:-1]) | (v[1:] != v[:-1])) + 1
    starts = np.concatenate([[0], chg])
    return starts.astype(np.int32), o[starts].astype(np.uint8), v[starts].astype(np.int32)


def pack_records(sids, seqs, origins, versions, align=1):
    """Pack a list of sequences (+ per-token meta) into the flat batch layout the
    oracle and the store take: (sids, tokens, tok_off[n+1], run_off[n+1],
    run_start, run_origin, run_version).  With align>1 every sequence starts at a
    multiple of ``align`` words (padding is zero and not part of any sequence);
    tok_off then holds starts and ``tok_len`` must be derived from the lengths."""
    n = len(seqs)
    lens = np.array([len(s) for s in seqs], np.int64)
    if align > 1:
        padded = (lens + align - 1) // align * align
        starts = np.concatenate([[0], np.cumsum(padded)])
    else:
        starts = np.concatenate([[0], np.cumsum(lens)])
    tokens = np.zeros(int(starts[-1]), np.int32)
    rs, ro, rv, roff = [], [], [], [0]
    for k in range(n):
        tokens[starts[k]: starts[k] + lens[k]] = seqs[k]
        a, b, c = per_token_runs(origins[k], versions[k])
        rs.append(a)
        ro.append(b)
        rv.append(c)
        roff.append(roff[-1] + len(a))
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt)  # noqa: E731
    tok_off = starts if align == 1 else np.concatenate([starts[:-1], [starts[-1]]])
    return (
        np.asarray(sids, np.int32),
        tokens,
        tok_off.astype(np.int64),
        np.asarray(roff, np.int64),
        cat(rs, np.int32),
        cat(ro, np.uint8),
        cat(rv, np.int32),
    )
