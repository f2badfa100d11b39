"""CPU oracle (TEST INFRASTRUCTURE ONLY) — pure-Python restatement of the reference
session radix tree, extended with the row/parent numbering the B200 store reports.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this module, and only as the checker.  The
product (``paper_2508_11553_b200``) never imports ``oracle/``.

Parity pinned: ``tests/test_oracle_golden.py`` checks this restatement against the
golden vectors in ``tests/golden/`` that ``tests/golden/make_golden.py`` produced by
running the unmodified reference (``/root/reference/pkg/src/rolloutlab``).

What it restates (file:line in /root/reference/pkg/src/rolloutlab):

* ``RadixOracle.insert``   — ``SessionTrie.lpm_insert`` trie.py:120-179 (walk by first
  token :140, per-token compare :151-154, descend :155-158, split :159-166 via
  ``_split`` :106-118, novel-suffix node :141-149 / :164-168, counters :145-146, :168-176).
* run splitting           — ``_runs_from`` :26-33, ``_split_runs`` :36-49, ``_merge_runs`` :258-265.
* ``RadixOracle.extract``  — ``_walk`` :189-198 (children in ascending first token,
  pre-order) + ``extract`` :210-216 (marked nodes only).
* ``RadixOracle.path``     — ``path_trajectory`` :203-208.
* ``RadixOracle.stats``    — ``stats`` :184-185 / ``StorageStats`` :78-87.

Additions the reference does not define:

* **row** — the session-local ordinal of a distinct recorded sequence, in order of
  first appearance.  A re-recorded identical sequence returns the same row; the
  reference returns the same ``node_id`` (tests/test_trie.py:66-74).
* **parent** — the earliest-inserted row whose LCP with the new sequence equals the
  matched length ``m`` (``-1`` when ``m == 0``).  Equivalently, the row that first
  wrote position ``m-1`` on this path: every trie node remembers the row that created
  its tokens (a split head inherits it, trie.py:112-113), and the parent is the
  creator of the node holding position ``m-1``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

INPUT, OUTPUT = 0, 1  # SpanOrigin.AGENT_INPUT / MODEL_OUTPUT (core.py:17-19)


def runs_from(origins, versions):
    """(length, origin, version) runs — restates trie.py:26-33."""
    runs = []
    for o, v in zip(origins, versions):
        if runs and runs[-1][1] == o and runs[-1][2] == v:
            runs[-1] = (runs[-1][0] + 1, o, v)
        else:
            runs.append((1, o, v))
    return runs


def split_runs(runs, k):
    """Cut a run list at token offset ``k`` — restates trie.py:36-49."""
    left, right, seen = [], [], 0
    for n, o, v in runs:
        if seen + n <= k:
            left.append((n, o, v))
        elif seen >= k:
            right.append((n, o, v))
        else:
            left.append((k - seen, o, v))
            right.append((n - (k - seen), o, v))
        seen += n
    return left, right


def merge_runs(runs):
    """Maximal runs — restates trie.py:258-265."""
    out = []
    for n, o, v in runs:
        if out and out[-1][1] == o and out[-1][2] == v:
            out[-1] = (out[-1][0] + n, o, v)
        else:
            out.append((n, o, v))
    return out


@dataclass
class _Node:
    tokens: list
    runs: list
    creator: int  # row that first wrote these tokens
    children: dict = field(default_factory=dict)
    row: int | None = None  # row ordinal when a recorded sequence ends here
    marks: set = field(default_factory=set)


@dataclass
class InsertOut:
    matched: int
    row: int
    parent: int
    added: int
    new_row: bool


class RadixOracle:
    """One session's radix tree (the reference ``SessionTrie``) plus row numbering."""

    def __init__(self):
        self.root = _Node([], [], -1)
        self.rows: list[_Node] = []  # row ordinal -> end node
        self.row_len: list[int] = []
        self.stored = 0
        self.naive = 0

    def _new_row(self, node, length):
        node.row = len(self.rows)
        self.rows.append(node)
        self.row_len.append(length)
        return node.row

    def insert(self, tokens, origins, versions, mark=None) -> InsertOut:
        """``lpm_insert`` (trie.py:120-179) returning (matched, row, parent, added)."""
        if len(tokens) == 0:
            raise ValueError("cannot insert an empty sequence")
        if not (len(tokens) == len(origins) == len(versions)):
            raise ValueError("tokens, origins, versions must be parallel")
        tokens = list(tokens)
        L = len(tokens)
        node, i = self.root, 0
        while True:
            if i == L:  # ended exactly at a node boundary (trie.py:137-139, 175-179)
                end, matched = node, L
                parent = node.creator
                break
            child = node.children.get(tokens[i])
            if child is None:  # novel suffix hangs off ``node`` (trie.py:141-149)
                row_id = len(self.rows)
                end = _Node(tokens[i:], runs_from(origins[i:], versions[i:]), row_id)
                node.children[tokens[i]] = end
                self.stored += L - i
                self.naive += L
                parent = node.creator if i > 0 else -1
                self._new_row(end, L)
                if mark is not None:
                    end.marks.add(mark)
                return InsertOut(i, row_id, parent, L - i, True)
            lim = min(len(child.tokens), L - i)
            c = 0
            while c < lim and child.tokens[c] == tokens[i + c]:
                c += 1
            if c == len(child.tokens):  # descend (trie.py:155-158)
                node, i = child, i + c
                continue
            # divergence or sequence end inside child's span: split (trie.py:159-166)
            parent = child.creator  # position i+c-1 lies in child's span (c >= 1)
            head_runs, tail_runs = split_runs(child.runs, c)
            head = _Node(child.tokens[:c], head_runs, child.creator)
            node.children[head.tokens[0]] = head
            child.tokens, child.runs = child.tokens[c:], tail_runs
            head.children = {child.tokens[0]: child}
            i += c
            if i == L:
                end, matched = head, L
                break
            row_id = len(self.rows)
            end = _Node(tokens[i:], runs_from(origins[i:], versions[i:]), row_id)
            head.children[tokens[i]] = end
            self.stored += L - i
            self.naive += L
            self._new_row(end, L)
            if mark is not None:
                end.marks.add(mark)
            return InsertOut(i, row_id, parent, L - i, True)
        # sequence ends at ``end`` (duplicate, or a prefix of stored content)
        self.naive += L
        new = end.row is None
        if new:
            self._new_row(end, L)
        if mark is not None:
            end.marks.add(mark)
        return InsertOut(matched, end.row, parent, 0, new)

    def stats(self):
        return self.stored, self.naive

    def _walk(self):
        """Pre-order DFS, children in ascending first token (trie.py:189-198)."""
        stack = [(self.root, [], [])]
        while stack:
            node, toks, runs = stack.pop()
            if node is not self.root:
                yield node, toks, runs
            for key in sorted(node.children, reverse=True):
                ch = node.children[key]
                stack.append((ch, toks + ch.tokens, runs + ch.runs))

    @staticmethod
    def _expand(toks, runs):
        mask, vers = [], []
        for n, o, v in merge_runs(runs):
            mask.extend([o == OUTPUT] * n)
            vers.extend([v] * n)
        return list(toks), mask, vers

    def extract(self, marked_only=True):
        """[(row, tokens, loss_mask, versions)] in lexicographic order (trie.py:210-216)."""
        out = []
        for node, toks, runs in self._walk():
            if node.row is None:
                continue
            if marked_only and not node.marks:
                continue
            out.append((node.row,) + self._expand(toks, runs))
        return out

    def path(self, row):
        """Full (tokens, loss_mask, versions) of one row (trie.py:203-208)."""
        target = self.rows[row]
        for node, toks, runs in self._walk():
            if node is target:
                return self._expand(toks, runs)
        raise KeyError(row)


class FlatOracle:
    """Independent flat restatement: distinct rows with
    parent pointers; ``meta[:m]`` inherited from the parent, ``meta[m:]`` own.

    Restates the reference's NaiveStore LCP oracle (tests/test_trie.py:18-44)
    extended with insertion order and first-writer metadata (trie.py:9-11).
    """

    def __init__(self):
        self.seqs: list[tuple] = []
        self.meta: list[tuple[list, list]] = []
        self.index: dict[tuple, int] = {}
        self.stored = 0
        self.naive = 0

    @staticmethod
    def _lcp(a, b):
        n = 0
        for x, y in zip(a, b):
            if x != y:
                break
            n += 1
        return n

    def insert(self, tokens, origins, versions):
        t = tuple(tokens)
        best, parent = 0, -1
        for r, s in enumerate(self.seqs):
            l = self._lcp(s, t)
            if l > best:
                best, parent = l, r
        self.naive += len(t)
        if t in self.index:
            return InsertOut(best, self.index[t], parent, 0, False)
        pm, pv = (self.meta[parent] if parent >= 0 else ([], []))
        mask = list(pm[:best]) + [o == OUTPUT for o in origins[best:]]
        vers = list(pv[:best]) + list(versions[best:])
        row = len(self.seqs)
        self.seqs.append(t)
        self.meta.append((mask, vers))
        self.index[t] = row
        self.stored += len(t) - best
        return InsertOut(best, row, parent, len(t) - best, True)
