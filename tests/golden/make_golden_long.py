"""Golden vectors at long lengths, from the UNMODIFIED reference.

The JSON fixtures of make_golden.py hold sequences of at most ~1k tokens; this script pins
the path at the lengths the configs use (8k - 40k tokens: turn-by-turn growth, branches deep
inside long histories, re-records, strict prefixes, metadata runs of several versions).
It runs ``rolloutlab.trie.SessionTrie`` from /root/reference in this container and writes
``long_cases.npz`` next to itself (committed; the GPU box never reads /root/reference):

  tokens, tok_off      every inserted sequence (int32, concatenated) and its offsets
  sess                 session index of every insert
  run_off, run_start, run_origin, run_version   its (origin, version) runs
  matched, row, added, parent                   InsertResult (node ids canonicalised to
                                                rows in order of first appearance) and the
                                                earliest-row-with-LCP == matched parent
  stored, naive        StorageStats after every insert
  ext_sess, ext_row, ext_off, ext_mask, ext_ver  extract() of every session: rows in
                                                lexicographic order with their loss masks
                                                and versions (tokens = the row's sequence)

    python tests/golden/make_golden_long.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from rolloutlab.core import SpanOrigin  # noqa: E402
from rolloutlab.trie import SessionTrie  # noqa: E402

IN, OUT = SpanOrigin.AGENT_INPUT, SpanOrigin.MODEL_OUTPUT


def lcp(a, b):
    a, b = np.asarray(a), np.asarray(b)
    n = min(len(a), len(b))
    d = np.flatnonzero(a[:n] != b[:n])
    return int(d[0]) if len(d) else n


def session_stream(rng, n_turns):
    """Turn-by-turn growth with versions bumped mid-session, then branches off deep
    positions, a re-record and a strict prefix of a long row."""
    seqs = []
    ctx = []
    ver = 0
    for t in range(n_turns):
        user = rng.integers(0, 151936, int(rng.integers(500, 3000))).tolist()
        out = rng.integers(0, 151936, int(rng.integers(2000, 7000))).tolist()
        if t == n_turns // 2:
            ver += 1
        seq = ctx + user + out
        org = [0] * (len(ctx) + len(user)) + [1] * len(out)
        vers = [0] * len(ctx) + [ver] * len(user)
        k = int(rng.integers(1, len(out)))  # a switch inside the output: two legs
        vers += [ver] * k + [ver + 1] * (len(out) - k)
        seqs.append((seq, org, vers))
        ctx = seq
    base = seqs[-1][0]
    for _ in range(3):  # branches deep inside the longest history
        cut = int(rng.integers(len(base) // 2, len(base) - 1))
        tail = rng.integers(0, 151936, int(rng.integers(100, 4000))).tolist()
        tail[0] = (base[cut] + 1) % 151936
        seq = base[:cut] + tail
        seqs.append((seq, [0] * cut + [1] * len(tail), [1] * cut + [2] * len(tail)))
    seqs.append(seqs[1])  # a re-record
    p = seqs[-2][0][: len(seqs[-2][0]) - 77]  # a strict prefix of a branch
    seqs.append((p, [1] * len(p), [3] * len(p)))
    return seqs


def main():
    rng = np.random.default_rng(20251022)
    out = {k: [] for k in ("tokens", "tok_len", "sess", "run_start", "run_origin", "run_version", "run_cnt", "matched",
                           "row", "added", "parent", "stored", "naive", "ext_sess", "ext_row", "ext_len", "ext_mask",
                           "ext_ver")}
    for s in range(3):
        trie = SessionTrie(f"long-{s}")
        node_to_row, row_seqs = {}, []
        for toks, org, vers in session_stream(rng, 4 + s):
            res = trie.lpm_insert(toks, [OUT if o else IN for o in org], vers, completion_id=f"c{len(out['sess'])}")
            parent = -1
            if res.matched_prefix_length > 0:
                for r, q in enumerate(row_seqs):
                    if lcp(q, toks) == res.matched_prefix_length:
                        parent = r
                        break
            if res.node_id not in node_to_row:
                node_to_row[res.node_id] = len(row_seqs)
                row_seqs.append(toks)
            st = trie.stats()
            o = np.asarray(org, np.int64)
            v = np.asarray(vers, np.int64)
            starts = np.flatnonzero(np.r_[True, (o[1:] != o[:-1]) | (v[1:] != v[:-1])])
            out["tokens"].append(np.asarray(toks, np.int32))
            out["tok_len"].append(len(toks))
            out["sess"].append(s)
            out["run_start"].append(starts.astype(np.int32))
            out["run_origin"].append(o[starts].astype(np.uint8))
            out["run_version"].append(v[starts].astype(np.int32))
            out["run_cnt"].append(len(starts))
            out["matched"].append(res.matched_prefix_length)
            out["row"].append(node_to_row[res.node_id])
            out["added"].append(res.added_tokens)
            out["parent"].append(parent)
            out["stored"].append(st.stored_tokens)
            out["naive"].append(st.naive_tokens)
        for nid, traj in trie.extract():
            out["ext_sess"].append(s)
            out["ext_row"].append(node_to_row[nid])
            out["ext_len"].append(len(traj.loss_mask))
            out["ext_mask"].append(np.asarray(traj.loss_mask, np.uint8))
            out["ext_ver"].append(np.asarray(traj.version_tags, np.int32))
            assert traj.tokens == row_seqs[node_to_row[nid]]
    cat = lambda k, dt: np.concatenate(out[k]).astype(dt)  # noqa: E731
    arr = lambda k, dt: np.asarray(out[k], dt)  # noqa: E731
    np.savez_compressed(
        os.path.join(HERE, "long_cases.npz"),
        tokens=cat("tokens", np.int32), tok_len=arr("tok_len", np.int64), sess=arr("sess", np.int32),
        run_start=cat("run_start", np.int32), run_origin=cat("run_origin", np.uint8),
        run_version=cat("run_version", np.int32), run_cnt=arr("run_cnt", np.int64), matched=arr("matched", np.int64),
        row=arr("row", np.int64), added=arr("added", np.int64), parent=arr("parent", np.int64),
        stored=arr("stored", np.int64), naive=arr("naive", np.int64), ext_sess=arr("ext_sess", np.int32),
        ext_row=arr("ext_row", np.int64), ext_len=arr("ext_len", np.int64), ext_mask=cat("ext_mask", np.uint8),
        ext_ver=cat("ext_ver", np.int32))
    print("inserts", len(out["sess"]), "tokens", int(sum(out["tok_len"])), "extract rows", len(out["ext_row"]))


if __name__ == "__main__":
    main()
