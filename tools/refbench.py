"""CPU baselines timed by bench.py beside the GPU numbers (never the measured product path).

Two CPU implementations of the same hot path, each on the box's host cores:

* the UNMODIFIED reference (rolloutlab.trie.SessionTrie / rolloutlab.core, installed in
  baseline/_ref by tools/install_reference.sh): one process, and a multiprocessing pool of
  os.cpu_count() workers over session-disjoint shards (sessions are independent, so this is
  the fair all-core figure) - BASELINE.md §3;
* the C restatement of the reference trie (oracle/radix_oracle.c, kind "port"), threaded.

Work units follow SURVEY.md §8(d): c4 = one lpm_insert per query into a trie holding that
query's session history (the history insert is setup, not timed); c1-c3 = the configs'
records in order per session (lpm_insert), then extract() and trajectory_to_line per session.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

_G: dict = {}  # fork-inherited state of the pool workers


def reference_modules():
    """(rolloutlab.trie, rolloutlab.core) of the unmodified reference, or None."""
    if not os.path.isdir(os.path.join(REF, "rolloutlab")):
        return None
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import rolloutlab.core as core
    import rolloutlab.trie as trie

    if not trie.__file__.startswith(REF):  # aliased to the drop-in: not the reference
        return None
    return trie, core


def _origins(core, codes):
    a, o = core.SpanOrigin.AGENT_INPUT, core.SpanOrigin.MODEL_OUTPUT
    return [o if c else a for c in codes]


def _per_token(run_start, run_origin, run_version, L):
    st = np.r_[run_start, L]
    return (np.repeat(run_origin.astype(np.int64), np.diff(st)).tolist(),
            np.repeat(run_version.astype(np.int64), np.diff(st)).tolist())


# ---- c4 / c5 shard: prefix-match queries ------------------------------------------------

def _match_job(idx):
    trie_mod, core = _G["mods"]
    hist, queries = _G["hist"], _G["queries"]
    tries = {}
    for i in idx:  # setup: each query's session history (not timed)
        s = queries[i][0]
        if s not in tries:
            toks, org, ver = hist(s)
            t = trie_mod.SessionTrie(f"s{s}")
            t.lpm_insert(toks, _origins(core, org), ver)
            tries[s] = t
    work = []
    for i in idx:
        s, q = queries[i]
        work.append((tries[s], q, [core.SpanOrigin.AGENT_INPUT] * len(q), [0] * len(q)))
    warm = trie_mod.SessionTrie("warm")  # first-call costs out of the timed loop
    warm.lpm_insert(work[0][1], work[0][2], work[0][3])
    warm.lpm_insert(work[0][1], work[0][2], work[0][3])
    t0 = time.perf_counter()
    for t, q, o, v in work:
        t.lpm_insert(q, o, v)
    return len(idx), time.perf_counter() - t0


def time_reference_match(hist, queries, procs=None):
    """Unmodified reference on a query sample: {single, pool} queries/s, or None.
    hist(s) -> (tokens list, origin codes, versions); queries = [(session, tokens list)]."""
    mods = reference_modules()
    if mods is None:
        return None
    _G.update(mods=mods, hist=hist, queries=queries)
    n = len(queries)
    one_n = max(1, n // 8)
    n1, dt1 = _match_job(list(range(one_n)))
    procs = procs or (os.cpu_count() or 1)
    chunks = [list(range(k, n, procs)) for k in range(procs) if k < n]
    with mp.get_context("fork").Pool(len(chunks)) as pool:
        res = pool.map(_match_job, chunks)
    tot = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    return {"single": n1 / dt1, "pool": tot / wall, "procs": len(chunks), "queries_single": n1, "queries_pool": tot}


# ---- c1-c3: record + extract + NDJSON -----------------------------------------------------

def _record_job(sessions):
    trie_mod, core = _G["mods"]
    recs = _G["recs"]  # session -> [(tokens list, origins, versions)]
    ntok = nrec = nexp = 0
    t0 = time.perf_counter()
    tries = []
    for s in sessions:
        t = trie_mod.SessionTrie(f"s{s}")
        for k, (toks, org, ver) in enumerate(recs[s]):
            t.lpm_insert(toks, org, ver, completion_id=f"r{k}")
            ntok += len(toks)
            nrec += 1
        tries.append(t)
    t_rec = time.perf_counter() - t0
    t0 = time.perf_counter()
    trajs = []
    for t in tries:
        for _, tr in t.extract():
            trajs.append(tr)
            nexp += len(tr.tokens)
    t_exp = time.perf_counter() - t0
    t0 = time.perf_counter()
    for tr in trajs:
        core.trajectory_to_line(tr)
    t_json = time.perf_counter() - t0
    return nrec, ntok, t_rec, nexp, t_exp, t_json


def time_reference_records(wl, n_sessions_single, n_sessions_pool, procs=None):
    """Unmodified reference on a session sample of a RecordWorkload: records/s, record
    tokens/s, export tokens/s (extract) and NDJSON tokens/s, one process and a pool."""
    mods = reference_modules()
    if mods is None:
        return None
    _, core = mods
    recs: dict = {}
    want = set(range(min(wl.n_sessions, max(n_sessions_single, n_sessions_pool))))
    for k, s in enumerate(wl.sids):
        if s in want:
            st, org, ver = wl.runs[k]
            o, v = _per_token(st, org, ver, len(wl.seqs[k]))
            recs.setdefault(s, []).append((wl.seqs[k].tolist(), _origins(core, o), v))
    _G.update(mods=mods, recs=recs)
    r = _record_job(list(range(min(n_sessions_single, wl.n_sessions))))
    single = {"records_per_s": r[0] / r[2], "record_tokens_per_s": r[1] / r[2], "export_tokens_per_s": r[3] / r[4],
              "ndjson_tokens_per_s": r[3] / r[5], "sessions": min(n_sessions_single, wl.n_sessions)}
    procs = procs or (os.cpu_count() or 1)
    ns = min(n_sessions_pool, wl.n_sessions)
    chunks = [list(range(k, ns, procs)) for k in range(procs) if k < ns]
    with mp.get_context("fork").Pool(len(chunks)) as pool:
        res = pool.map(_record_job, chunks)
    pool_d = {"records_per_s": sum(x[0] for x in res) / max(x[2] for x in res),
              "record_tokens_per_s": sum(x[1] for x in res) / max(x[2] for x in res),
              "export_tokens_per_s": sum(x[3] for x in res) / max(x[4] for x in res),
              "ndjson_tokens_per_s": sum(x[3] for x in res) / max(x[5] for x in res),
              "sessions": ns, "procs": len(chunks)}
    return {"single": single, "pool": pool_d}


# ---- the C port (threads) ----------------------------------------------------------------

def time_port_records(wl, nthreads):
    """C restatement: record every record of the workload, then export every row."""
    from oracle.cport import CRadixStore

    ora = CRadixStore()
    packed = wl.packed()
    t0 = time.perf_counter()
    m, row, par, add = ora.insert_batch(*packed, nthreads=nthreads)
    t_rec = time.perf_counter() - t0
    sess = np.asarray(wl.sids, np.int64)
    t0 = time.perf_counter()
    off, tok, msk, ver = ora.export_batch(sess, row, nthreads=nthreads)
    t_exp = time.perf_counter() - t0
    n = len(wl.seqs)
    ntok = int(np.diff(packed[2]).sum())
    out = {"records_per_s": n / t_rec, "record_tokens_per_s": ntok / t_rec, "export_tokens_per_s": float(off[-1]) / t_exp,
           "threads": nthreads}
    ora.close()
    return out, (m, row, par, add)
