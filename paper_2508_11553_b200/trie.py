"""Drop-in ``SessionTrie`` (reference: rolloutlab/trie.py:90-255) backed by the B200 store.

A session's recorded sequences live in the GPU arena as rows (novel suffix + parent
pointer); matching, recording and reconstruction run in CUDA kernels.  This class
keeps the reference's public surface:

* ``lpm_insert(tokens, origins, versions, completion_id=None) -> InsertResult``
* ``stats() -> StorageStats``; ``total_stored_tokens`` / ``total_naive_tokens``
* ``extract() -> [(node_id, Trajectory)]`` in lexicographic order (marked rows)
* ``path_trajectory(node_id)``, ``mark``, ``marked_nodes``, ``check_well_formed``
* ``root`` / ``nodes``: a radix-tree VIEW materialised from the rows on demand
  (debug and API fidelity only; never on the hot path).

``node_id`` is the session-local row ordinal: identical sequences get the same id,
extensions a new one, and ids survive later branching.
"""

from __future__ import annotations

import array
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from .core import ORIGIN_CODE, ModelVersion, SpanOrigin, TokenId, Trajectory
from .store import DeviceStore, default_store, runs_from_per_token

try:  # host-side argument marshalling in C (csrc/tmfast.c); the pure-Python paths below remain
    from . import _tmfast
except ImportError:  # pragma: no cover - the extension is built with libtmstore.so
    _tmfast = None

MetaRun = tuple[int, SpanOrigin, ModelVersion]


@dataclass
class InsertResult:
    matched_prefix_length: int
    node_id: int
    added_tokens: int


@dataclass
class StorageStats:
    stored_tokens: int
    naive_tokens: int

    @property
    def dedup_ratio(self) -> float:
        if self.naive_tokens == 0:
            return 1.0
        return self.stored_tokens / self.naive_tokens


@dataclass
class TrieNode:
    """Node of the materialised radix view (same fields as trie.py:58-68)."""

    node_id: int
    tokens: list[TokenId]
    runs: list[MetaRun]
    children: dict[TokenId, "TrieNode"] = field(default_factory=dict)
    leaf_marks: set[str] = field(default_factory=set)

    @property
    def is_marked(self) -> bool:
        return bool(self.leaf_marks)


def _as_int32(values):
    """Token ids -> an int32 buffer at C speed (array.array for lists, numpy arrays as
    int32), rejecting ids outside int32."""
    if isinstance(values, np.ndarray):
        if values.size and (values.min() < -(2**31) or values.max() >= 2**31):
            raise ValueError("token ids must fit in int32")
        return np.ascontiguousarray(values, np.int32)
    if _tmfast is not None and isinstance(values, (list, tuple)):
        return np.frombuffer(_tmfast.pack_i32(values), np.int32)
    try:
        return array.array("i", values)
    except OverflowError:
        raise ValueError("token ids must fit in int32") from None


def meta_runs(origins, versions):
    """Per-token (origin, version) -> run starts / origin codes / versions.

    Runs are found at C speed: origin changes with list.index (two values), version
    changes from an int64 view (skipped when every token has the same version)."""
    n = len(origins)
    if _tmfast is not None and n and isinstance(origins, (list, tuple)) and isinstance(versions, (list, tuple)):
        st, org, ver, k = _tmfast.meta_runs(origins, versions, SpanOrigin.MODEL_OUTPUT, SpanOrigin.AGENT_INPUT)
        return np.frombuffer(st, np.int32, k), np.frombuffer(org, np.uint8, k), np.frombuffer(ver, np.int32, k)
    if isinstance(origins, np.ndarray) or not n:
        o = np.asarray([ORIGIN_CODE.get(x, 1 if getattr(x, "value", x) in (1, True, "model_output") else 0)
                        for x in origins] if not isinstance(origins, np.ndarray) else origins, np.int64)
        return runs_from_per_token(o, np.asarray(versions, np.int64))
    first = origins[0]
    o_starts, o_vals = [0], [first]
    cur, i = first, 0
    other = {SpanOrigin.AGENT_INPUT: SpanOrigin.MODEL_OUTPUT, SpanOrigin.MODEL_OUTPUT: SpanOrigin.AGENT_INPUT}
    if cur not in other:  # not this package's SpanOrigin (0/1, bools, the reference's own enum): by value
        return runs_from_per_token(
            np.asarray([1 if getattr(x, "value", x) in (1, True, "model_output") else 0 for x in origins], np.int64),
            np.asarray(versions, np.int64))
    while True:
        nxt = other[cur]
        try:
            i = origins.index(nxt, i)
        except ValueError:
            break
        o_starts.append(i)
        o_vals.append(nxt)
        cur = nxt
    if isinstance(versions, list) and versions.count(versions[0]) == n:
        v_starts, v_vals = [0], [versions[0]]
    else:
        v = np.frombuffer(array.array("q", versions), np.int64) if isinstance(versions, list) else np.asarray(versions, np.int64)
        cut = np.flatnonzero(v[1:] != v[:-1]) + 1
        v_starts = [0] + cut.tolist()
        v_vals = v[[0] + cut.tolist()].tolist()
    starts = sorted(set(o_starts) | set(v_starts))
    oi = np.searchsorted(np.asarray(o_starts), starts, side="right") - 1
    vi = np.searchsorted(np.asarray(v_starts), starts, side="right") - 1
    codes = np.asarray([ORIGIN_CODE[x] for x in o_vals], np.uint8)[oi]
    return np.asarray(starts, np.int32), codes, np.asarray(v_vals, np.int32)[vi]


class SessionTrie:
    """One session of the B200 store, with the reference SessionTrie API."""

    def __init__(self, session_id: str, *, store: DeviceStore | None = None):
        self.session_id = session_id
        self.store = store if store is not None else default_store()
        self.sid = self.store.new_session()
        self._marks: dict[int, set[str]] = {}
        self._rows: list[int] = []  # local ordinal -> global row
        self._lens: list[int] = []  # local ordinal -> sequence length

    # -- record -------------------------------------------------------------------
    def lpm_insert(self, tokens: Sequence[TokenId], origins: Sequence[SpanOrigin], versions: Sequence[ModelVersion],
                   completion_id: str | None = None) -> InsertResult:
        """Insert one recorded sequence, merging with stored content by LPM (trie.py:120-179)."""
        if len(tokens) == 0:
            raise ValueError("cannot insert an empty sequence")
        if not (len(tokens) == len(origins) == len(versions)):
            raise ValueError("tokens, origins, versions must be parallel")
        return self.insert_runs(tokens, meta_runs(origins, versions), completion_id)

    def insert_runs(self, tokens, runs, completion_id: str | None = None) -> InsertResult:
        """lpm_insert with metadata already as (starts, origins 0/1, versions) runs."""
        r = self.store.record_one(self.sid, _as_int32(tokens), runs)
        return self._absorb(r, 0, completion_id, len(tokens))

    def _absorb(self, r, k: int, completion_id, length: int):
        local = int(r.local[k])
        if local == len(self._rows):
            self._rows.append(int(r.row[k]))
            self._lens.append(int(length))
        if completion_id is not None:
            self._marks.setdefault(local, set()).add(completion_id)
        return InsertResult(int(r.matched[k]), local, int(r.added[k]))

    def mark(self, node_id: int, completion_id: str) -> None:
        self._global(node_id)
        self._marks.setdefault(node_id, set()).add(completion_id)

    # -- accounting -----------------------------------------------------------------
    def stats(self) -> StorageStats:
        stored, naive, _ = self.store.session_stats(self.sid)
        return StorageStats(stored, naive)

    @property
    def total_stored_tokens(self) -> int:
        return self.store.session_stats(self.sid)[0]

    @property
    def total_naive_tokens(self) -> int:
        return self.store.session_stats(self.sid)[1]

    # -- reconstruction ----------------------------------------------------------------
    def _global(self, node_id: int) -> int:
        if not (0 <= node_id < len(self._rows)):
            raise KeyError(f"node {node_id} not in trie")
        return self._rows[node_id]

    def row_of(self, node_id: int) -> int:
        """Global store row of a node id."""
        return self._global(node_id)

    def path_trajectory(self, node_id: int) -> Trajectory:
        """Rebuild the trajectory for the root->node path (trie.py:203-208)."""
        p = self.store.export([self._global(node_id)], total=self._lens[node_id])
        return Trajectory.from_packed(self.session_id, p.tokens, p.loss_mask, p.versions)

    def lex_node_ids(self) -> list[int]:
        """All node ids of the session in lexicographic sequence order."""
        base = {g: k for k, g in enumerate(self._rows)}
        return [base[int(g)] for g in self.store.session_rows(self.sid, "lex")]

    def marked_node_ids(self) -> list[int]:
        """Node ids carrying a completion mark, in lexicographic order."""
        return [k for k in self.lex_node_ids() if self._marks.get(k)]

    def marked_nodes(self) -> list[TrieNode]:
        """Marked nodes of the radix view in path order (trie.py:200-201)."""
        nodes = self.nodes
        return [nodes[k] for k in self.marked_node_ids()]

    def extract(self) -> list[tuple[int, Trajectory]]:
        """One trajectory per marked node, in lexicographic order (trie.py:210-216)."""
        ids = self.marked_node_ids()
        if not ids:
            return []
        p = self.store.export([self._rows[k] for k in ids], total=sum(self._lens[k] for k in ids))
        out = []
        for i, k in enumerate(ids):
            a, b = p.offsets[i], p.offsets[i + 1]
            out.append((k, Trajectory.from_packed(self.session_id, p.tokens[a:b], p.loss_mask[a:b], p.versions[a:b])))
        return out

    # -- radix view (debug / API fidelity) ----------------------------------------------
    def _materialise(self):
        """Build the reference-shaped radix tree from the rows (insertion order)."""
        root = TrieNode(node_id=-1, tokens=[], runs=[])
        nodes = {root.node_id: root}
        if not self._rows:
            return root, nodes
        p = self.store.export(self._rows)
        next_interior = [-2]

        def new_interior(tokens, runs):
            n = TrieNode(node_id=next_interior[0], tokens=tokens, runs=runs)
            next_interior[0] -= 1
            nodes[n.node_id] = n
            return n

        def runs_of(a, b):
            mk, vs = p.loss_mask[a:b], p.versions[a:b]
            out = []
            for m, v in zip(mk.tolist(), vs.tolist()):
                o = SpanOrigin.MODEL_OUTPUT if m else SpanOrigin.AGENT_INPUT
                if out and out[-1][1] is o and out[-1][2] == v:
                    out[-1] = (out[-1][0] + 1, o, v)
                else:
                    out.append((1, o, v))
            return out

        for local, _ in enumerate(self._rows):
            a, b = int(p.offsets[local]), int(p.offsets[local + 1])
            toks = p.tokens[a:b].tolist()
            node, i = root, 0
            while True:
                if i == len(toks):
                    end = node
                    break
                child = node.children.get(toks[i])
                if child is None:
                    end = TrieNode(node_id=local, tokens=toks[i:], runs=runs_of(a + i, b))
                    nodes[local] = end
                    node.children[toks[i]] = end
                    break
                c = 0
                lim = min(len(child.tokens), len(toks) - i)
                while c < lim and child.tokens[c] == toks[i + c]:
                    c += 1
                if c == len(child.tokens):
                    node, i = child, i + c
                    continue
                head_runs, tail_runs, seen = [], [], 0
                for ln, o, v in child.runs:
                    if seen + ln <= c:
                        head_runs.append((ln, o, v))
                    elif seen >= c:
                        tail_runs.append((ln, o, v))
                    else:
                        head_runs.append((c - seen, o, v))
                        tail_runs.append((ln - (c - seen), o, v))
                    seen += ln
                head = new_interior(child.tokens[:c], head_runs)
                node.children[head.tokens[0]] = head
                child.tokens, child.runs = child.tokens[c:], tail_runs
                head.children = {child.tokens[0]: child}
                i += c
                if i == len(toks):
                    end = head
                    break
                end = TrieNode(node_id=local, tokens=toks[i:], runs=runs_of(a + i, b))
                nodes[local] = end
                head.children[toks[i]] = end
                break
            if end.node_id != local:  # the sequence ends on an interior node: it becomes the row's node
                del nodes[end.node_id]
                end.node_id = local
                nodes[local] = end
            end.leaf_marks = set(self._marks.get(local, set()))
        return root, nodes

    @property
    def root(self) -> TrieNode:
        return self._materialise()[0]

    @property
    def nodes(self) -> dict[int, TrieNode]:
        return self._materialise()[1]

    def check_well_formed(self) -> list[str]:
        """Structural invariants of the materialised view + store accounting (trie.py:228-255)."""
        root, _ = self._materialise()
        problems: list[str] = []
        seen = 0
        stack = [root]
        while stack:
            node = stack.pop()
            if node is not root:
                if not node.tokens:
                    problems.append(f"node {node.node_id} has empty span")
                seen += len(node.tokens)
                if sum(r[0] for r in node.runs) != len(node.tokens):
                    problems.append(f"node {node.node_id} runs do not cover its tokens")
            for key, child in node.children.items():
                if not child.tokens or child.tokens[0] != key:
                    problems.append(f"child of node {node.node_id} keyed {key} but starts with {child.tokens[:1]}")
                stack.append(child)
        st = self.stats()
        if seen != st.stored_tokens:
            problems.append(f"stored-token accounting off: counted {seen}, recorded {st.stored_tokens}")
        if st.stored_tokens > st.naive_tokens:
            problems.append("stored exceeds naive total")
        return problems
