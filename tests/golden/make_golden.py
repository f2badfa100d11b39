"""Generate the golden vectors that pin the oracle and the B200 store.

Runs the UNMODIFIED reference (``/root/reference/pkg/src/rolloutlab``) in this
container and writes its outputs as JSON fixtures next to this script.  The
fixtures are committed; ``/root/reference`` does not exist on the GPU box, so no
test reads the reference at run time.

    python tests/golden/make_golden.py

Fixtures:

* ``trie_cases.json``    — per-session insert streams through ``SessionTrie.lpm_insert``
  (trie.py:120-179) with every ``InsertResult``, ``stats()`` after every insert,
  ``extract()`` (trie.py:210-216) and ``path_trajectory`` (trie.py:203-208) for every
  returned node, plus the canonical NDJSON line (core.py:182-183) of each row.
  Node ids are canonicalised to *rows* (order of first appearance) because the
  store numbers rows, not trie nodes (SURVEY.md §8(b) node_id contract).  The
  ``parent`` column is the SURVEY.md §0.1-fact-3 definition (earliest row with
  LCP == matched), computed here by brute force from the reference's own rows.
* ``manager_cases.json`` — ``TrajectoryManager`` (trajectory.py) driven by the
  reference MockEngine/RolloutManager with switches and pauses; the stream of
  ``_finalize`` records (session, input, produced, versions, context version,
  request id) is logged together with ``extract_trajectories``, ``storage_stats``
  and ``drain_batch`` outputs, so the B200 manager can replay the same records.
* ``engine_vectors.json`` — ``next_token`` (engine.py:35-46) values used to pin the
  test-double engine in ``tests/support``.
"""

from __future__ import annotations

import json
import os
import random
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from rolloutlab.core import GenParams, SpanOrigin, trajectory_to_line  # noqa: E402
from rolloutlab.engine import MockEngine, next_token  # noqa: E402
from rolloutlab.rollout import RolloutManager  # noqa: E402
from rolloutlab.trajectory import PumpStatus, TrajectoryManager  # noqa: E402
from rolloutlab.trie import SessionTrie  # noqa: E402

IN, OUT = SpanOrigin.AGENT_INPUT, SpanOrigin.MODEL_OUTPUT


def lcp(a, b):
    n = 0
    for x, y in zip(a, b):
        if x != y:
            break
        n += 1
    return n


def run_trie_case(name, inserts):
    """inserts: list of (tokens, origins01, versions, completion_id|None)."""
    trie = SessionTrie("sess-" + name)
    node_to_row: dict[int, int] = {}
    row_seqs: list[tuple] = []
    results = []
    for toks, org, ver, cid in inserts:
        origins = [OUT if o else IN for o in org]
        # parent: earliest row (by first appearance) with LCP == matched
        res = trie.lpm_insert(toks, origins, ver, cid)
        parent = -1
        if res.matched_prefix_length > 0:
            for r, s in enumerate(row_seqs):
                if lcp(s, toks) == res.matched_prefix_length:
                    parent = r
                    break
        if res.node_id not in node_to_row:
            node_to_row[res.node_id] = len(row_seqs)
            row_seqs.append(tuple(toks))
        st = trie.stats()
        results.append(
            dict(
                matched=res.matched_prefix_length,
                row=node_to_row[res.node_id],
                parent=parent,
                added=res.added_tokens,
                stored=st.stored_tokens,
                naive=st.naive_tokens,
            )
        )
    extract = []
    for node_id, traj in trie.extract():
        extract.append(
            dict(
                row=node_to_row[node_id],
                tokens=traj.tokens,
                loss_mask=[1 if m else 0 for m in traj.loss_mask],
                versions=list(traj.version_tags),
                line=trajectory_to_line(traj),
            )
        )
    paths = {}
    for node_id, row in node_to_row.items():
        traj = trie.path_trajectory(node_id)
        paths[str(row)] = dict(
            tokens=traj.tokens,
            loss_mask=[1 if m else 0 for m in traj.loss_mask],
            versions=list(traj.version_tags),
        )
    assert trie.check_well_formed() == []
    st = trie.stats()
    return dict(
        name=name,
        session_id=trie.session_id,
        inserts=[dict(tokens=list(t), origins=list(o), versions=list(v), completion_id=c) for t, o, v, c in inserts],
        results=results,
        extract=extract,
        paths=paths,
        stored=st.stored_tokens,
        naive=st.naive_tokens,
        dedup_ratio=st.dedup_ratio,
    )


def ins(tokens, cid=None, version=0, origin=1):
    return (list(tokens), [origin] * len(tokens), [version] * len(tokens), cid)


def unit_cases():
    """The scenarios of tests/test_trie.py:47-138, as golden streams."""
    cases = [
        ("empty_then_one", [ins([10, 11, 12, 13], "a")]),
        ("divergence_split", [ins([10, 11, 12, 13], "a"), ins([10, 11, 20, 21], "b")]),
        ("duplicate", [ins([10, 11, 12, 13], "a"), ins([10, 11, 12, 13], "b")]),
        ("prefix_of_existing", [ins([1, 2, 3, 4], "long"), ins([1, 2], "short")]),
        ("extension", [ins([1, 2], "a"), ins([1, 2, 3], "b")]),
        ("leaf_id_stable", [ins([5, 6, 7, 8], "a"), ins([5, 6, 9], "b")]),
        (
            "version_boundary_inside_node",
            [([1, 2, 3, 4], [1, 1, 1, 1], [0, 0, 1, 1], "a")],
        ),
        # mid-output divergence keeps first-writer mask
        (
            "mid_output_branch_mask",
            [([1, 2, 3, 4], [0, 0, 1, 1], [0] * 4, "a"), ([1, 2, 3, 9, 5, 6], [0, 0, 0, 0, 1, 1], [0] * 6, "b")],
        ),
        # prefix recorded after a branch point already split the node
        (
            "prefix_at_split_point",
            [ins([1, 2, 3, 4], "a"), ins([1, 2, 5], "b"), ins([1, 2], "c"), ins([1, 2], "d"), ins([1, 2, 5, 6], "e")],
        ),
        ("unmarked_inserts", [ins([7, 8, 9]), ins([7, 8], "x"), ins([7, 8, 9, 10])]),
    ]
    P, S, K = 16, 8, 4
    prefix = list(range(100, 100 + P))
    cases.append(("closed_form_P16_S8_K4", [ins(prefix + [1000 * (k + 1) + j for j in range(S)], f"c{k}") for k in range(K)]))
    for K in (2, 4, 8):
        for P in (16, 256):
            for S in (16, 64):
                pre = [(7 * i) % 4096 for i in range(P)]
                seq = []
                for k in range(K):
                    seq.append(ins(pre + [5000 + 97 * k + j for j in range(S)], f"b{k}"))
                cases.append((f"closed_form_K{K}_P{P}_S{S}", seq))
    return cases


def random_small(rng, n):
    """Hypothesis-like streams (tests/test_trie.py:141-164): tiny alphabet, many ties."""
    out = []
    for s in range(n):
        seqs = []
        for k in range(rng.randint(1, 25)):
            L = rng.randint(1, 12)
            toks = [rng.randint(0, 5) for _ in range(L)]
            org = [rng.randint(0, 1) for _ in range(L)]
            v0 = rng.randint(0, 3)
            ver = []
            for _ in range(L):
                v0 += 1 if rng.random() < 0.15 else 0
                ver.append(v0)
            cid = None if rng.random() < 0.2 else f"c{k}"
            seqs.append((toks, org, ver, cid))
        out.append((f"small_{s}", seqs))
    return out


def random_multiturn(rng, n, vocab=1000):
    """Agent-like sessions: turns extend an earlier context, branches reuse it."""
    out = []
    for s in range(n):
        contexts = [([], [], [])]
        seqs = []
        version = 0
        for turn in range(rng.randint(2, 12)):
            ct, co, cv = rng.choice(contexts)
            user = [rng.randrange(vocab) for _ in range(rng.randint(1, 40))]
            outp = [rng.randrange(vocab) for _ in range(rng.randint(1, 80))]
            if rng.random() < 0.3:
                version += 1
            toks = ct + user + outp
            org = co + [0] * len(user) + [1] * len(outp)
            # replayed context is re-tagged with the current version (trajectory.py:226-230)
            ver = [version] * (len(ct) + len(user)) + [version] * len(outp)
            seqs.append((toks, org, ver, f"t{turn}"))
            contexts.append((toks, org, ver))
            if rng.random() < 0.15:  # re-record an old context verbatim (duplicate)
                t2, o2, v2 = rng.choice(contexts[1:])
                seqs.append((t2, o2, v2, f"dup{turn}"))
            if rng.random() < 0.15 and len(toks) > 2:  # record a strict prefix
                cut = rng.randint(1, len(toks) - 1)
                seqs.append((toks[:cut], org[:cut], ver[:cut], f"pre{turn}"))
        out.append((f"multiturn_{s}", seqs))
    return out


def make_trie_cases():
    rng = random.Random(20251018)
    cases = unit_cases() + random_small(rng, 300) + random_multiturn(rng, 60)
    return [run_trie_case(name, seqs) for name, seqs in cases]


# --------------------------------------------------------------------------- manager


def make_manager_cases():
    """Criterion-1-like capture (tests/test_acceptance.py:64-115), smaller, with the
    _finalize stream logged so the B200 manager can replay identical records."""
    VOCAB = 4096
    cases = []
    for case_idx, (n_sessions, seed) in enumerate([(40, 20250810), (25, 777)]):
        engine = MockEngine(vocab_size=VOCAB)
        rm = RolloutManager(engine)
        tm = TrajectoryManager(engine, control=rm, pending_timeout=10.0)
        records = []
        orig_finalize = tm._finalize

        def logging_finalize(req, _orig=orig_finalize):
            records.append(
                dict(
                    session_id=req.session_id,
                    request_id=req.request_id,
                    input_tokens=list(req.input_tokens),
                    produced=list(req.produced),
                    versions=list(req.versions),
                    context_version=req.context_version,
                )
            )
            _orig(req)

        tm._finalize = logging_finalize
        rng = random.Random(seed)
        switch_at = {"step": None}
        steps = {"n": 0}

        def hook(job_id, pos):
            steps["n"] += 1
            if switch_at["step"] is not None and steps["n"] >= switch_at["step"]:
                switch_at["step"] = None
                rm.coordinate_update(engine.current_version + 1)

        engine.step_hook = hook
        drains = []
        for s in range(n_sessions):
            sid = f"sess-{s}"
            contexts = [[]]
            for turn in range(rng.randint(1, 6)):
                ctx = list(rng.choice(contexts))
                user = [rng.randrange(VOCAB) for _ in range(rng.randint(2, 5))]
                inp = ctx + user
                params = GenParams(max_new_tokens=rng.randint(4, 9), seed=rng.randrange(1_000_000))
                if rng.random() < 0.25:
                    switch_at["step"] = steps["n"] + rng.randint(1, params.max_new_tokens)
                out = tm.proxy_generate(sid, inp, params, request_id=f"{sid}-t{turn}")
                contexts.append(inp + out)
            if s % 7 == 6:
                batch = tm.drain_batch(3)
                drains.append(
                    dict(after_record=len(records), lines=None if batch is None else [trajectory_to_line(t) for t in batch])
                )
        engine.step_hook = None
        final = tm.drain_batch(1)
        drains.append(dict(after_record=len(records), lines=None if final is None else [trajectory_to_line(t) for t in final]))
        sessions = {}
        for sid in tm.session_ids():
            st = tm.storage_stats(sid)
            sessions[sid] = dict(
                extract=[trajectory_to_line(t) for t in tm.extract_trajectories(sid)],
                extract_min_v1=[trajectory_to_line(t) for t in tm.extract_trajectories(sid, min_version=1)],
                stored=st.stored_tokens,
                naive=st.naive_tokens,
            )
        cases.append(dict(name=f"capture_{case_idx}", records=records, drains=drains, sessions=sessions))

    # partial-rollout pause/resume with a version change mid-turn (config 3 in miniature)
    engine = MockEngine(vocab_size=VOCAB)
    rm = RolloutManager(engine)
    tm = TrajectoryManager(engine, control=rm, pending_timeout=10.0)
    records = []
    orig_finalize = tm._finalize

    def logging_finalize2(req, _orig=orig_finalize):
        records.append(
            dict(
                session_id=req.session_id,
                request_id=req.request_id,
                input_tokens=list(req.input_tokens),
                produced=list(req.produced),
                versions=list(req.versions),
                context_version=req.context_version,
            )
        )
        _orig(req)

    tm._finalize = logging_finalize2
    rng = random.Random(31337)
    for s in range(12):
        sid = f"pr-{s}"
        t1 = [rng.randrange(VOCAB) for _ in range(6)]
        out1 = tm.proxy_generate(sid, t1, GenParams(max_new_tokens=8, seed=s))
        t2 = t1 + out1 + [rng.randrange(VOCAB) for _ in range(3)]
        req = tm.open_request(sid, t2, GenParams(max_new_tokens=12, seed=100 + s))
        k = rng.randint(1, 10)
        n = 0
        while n < k:
            if tm.pump(req) is PumpStatus.PROGRESS:
                n += 1
        rm.coordinate_update(engine.current_version + 1)
        guard = 0
        while tm.pump(req) is not PumpStatus.DONE:
            guard += 1
            assert guard < 10000
    sessions = {}
    for sid in tm.session_ids():
        st = tm.storage_stats(sid)
        sessions[sid] = dict(
            extract=[trajectory_to_line(t) for t in tm.extract_trajectories(sid)],
            extract_min_v1=[trajectory_to_line(t) for t in tm.extract_trajectories(sid, min_version=1)],
            stored=st.stored_tokens,
            naive=st.naive_tokens,
        )
    final = tm.drain_batch(1)
    cases.append(
        dict(
            name="partial_rollout_stitch",
            records=records,
            drains=[dict(after_record=len(records), lines=[trajectory_to_line(t) for t in final])],
            sessions=sessions,
        )
    )
    return cases


def make_engine_vectors():
    rng = random.Random(5)
    vecs = []
    for _ in range(40):
        ctx = [rng.randrange(4096) for _ in range(rng.randint(0, 30))]
        seed = rng.randrange(-(2**40), 2**40)
        version = rng.randint(0, 5)
        vecs.append(dict(context=ctx, seed=seed, version=version, vocab=4096, token=next_token(ctx, seed, version, 4096)))
    return vecs


def main():
    trie_cases = make_trie_cases()
    with open(os.path.join(HERE, "trie_cases.json"), "w") as fh:
        json.dump(trie_cases, fh, separators=(",", ":"))
    mgr = make_manager_cases()
    with open(os.path.join(HERE, "manager_cases.json"), "w") as fh:
        json.dump(mgr, fh, separators=(",", ":"))
    with open(os.path.join(HERE, "engine_vectors.json"), "w") as fh:
        json.dump(make_engine_vectors(), fh, separators=(",", ":"))
    print(f"trie cases: {len(trie_cases)}  manager cases: {len(mgr)}")


if __name__ == "__main__":
    main()
