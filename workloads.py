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


# ----------------------------------------------------------------------------- configs


def turn_runs(hist_len: int, turns: int, in_frac: float = 0.125, bump_at: int = 5):
    """Meta runs of an agent history: per turn an AGENT_INPUT run then a MODEL_OUTPUT
    run; versions bumped from turn ``bump_at`` on (a policy update mid-session)."""
    per = hist_len // turns
    n_in = max(1, int(per * in_frac))
    starts, origins, versions = [], [], []
    for t in range(turns):
        v = 0 if t < bump_at else 1
        starts += [t * per, t * per + n_in]
        origins += [0, 1]
        versions += [v, v]
    return np.asarray(starts, np.int32), np.asarray(origins, np.uint8), np.asarray(versions, np.int32)


class MatchWorkload:
    """Config 4 (and the per-shard slice of config 5): sessions with one stored history
    each, and batches of read-only match queries — 75% full history + 256 new tokens
    (matched = history length), 25% branches at d ~ U[0, len) with a forced mismatch."""

    def __init__(self, n_sessions=10_000, hist_len=32_768, n_queries=4096, ext_frac=0.75, new_tokens=256,
                 seed=SEED0 + 4, mixed=None):
        rng = np.random.default_rng(seed)
        self.n_sessions = n_sessions
        if mixed is None:
            lens = np.full(n_sessions, hist_len, np.int64)
        else:  # log-uniform lengths in [lo, hi] (config 5)
            lo, hi = mixed
            lens = np.exp(rng.uniform(np.log(lo), np.log(hi), n_sessions)).astype(np.int64)
        self.hist_len = lens
        padded = (lens + ALIGN - 1) // ALIGN * ALIGN
        self.hist_off = np.zeros(n_sessions + 1, np.int64)
        np.cumsum(padded, out=self.hist_off[1:])
        self.hist_tokens = np.zeros(int(self.hist_off[-1]), np.int32)
        for s in range(n_sessions):  # chunked generation keeps peak memory low
            self.hist_tokens[self.hist_off[s]: self.hist_off[s] + lens[s]] = rng.integers(0, VOCAB, int(lens[s]), dtype=np.int32)
        runs = [turn_runs(int(L), 8) if L >= 64 else (np.array([0], np.int32), np.array([1], np.uint8), np.array([0], np.int32)) for L in lens]
        self.run_off = np.zeros(n_sessions + 1, np.int64)
        np.cumsum([len(r[0]) for r in runs], out=self.run_off[1:])
        self.run_start = np.concatenate([r[0] for r in runs])
        self.run_origin = np.concatenate([r[1] for r in runs])
        self.run_version = np.concatenate([r[2] for r in runs])
        self.n_queries = n_queries
        self.ext_frac, self.new_tokens = ext_frac, new_tokens
        self.set_queries(self.make_queries(rng))

    def make_queries(self, rng):
        """One batch: 75% full history + new tokens, 25% branches with a forced mismatch."""
        n, lens, new_tokens = self.n_queries, self.hist_len, self.new_tokens
        qs = rng.integers(0, self.n_sessions, n)
        ext = rng.random(n) < self.ext_frac
        depth = np.where(ext, lens[qs], (rng.random(n) * lens[qs]).astype(np.int64))
        qlen = depth + new_tokens
        qpad = (qlen + ALIGN - 1) // ALIGN * ALIGN
        q_off = np.zeros(n + 1, np.int64)
        np.cumsum(qpad, out=q_off[1:])
        q_tokens = np.zeros(int(q_off[-1]), np.int32)
        for i in range(n):
            s, d, o = qs[i], int(depth[i]), int(q_off[i])
            h = self.hist_tokens[self.hist_off[s]: self.hist_off[s] + lens[s]]
            q_tokens[o: o + d] = h[:d]
            tail = rng.integers(0, VOCAB, new_tokens, dtype=np.int32)
            if d < lens[s]:  # forced mismatch at d
                tail[0] = (int(h[d]) + 1 + int(rng.integers(0, VOCAB - 1))) % VOCAB
            q_tokens[o + d: o + d + new_tokens] = tail
        return dict(q_sess=qs.astype(np.int32), q_len=qlen, q_depth=depth, q_off=q_off, q_tokens=q_tokens)

    def set_queries(self, q):
        self.q_sess, self.q_len, self.q_depth = q["q_sess"], q["q_len"], q["q_depth"]
        self.q_off, self.q_tokens = q["q_off"], q["q_tokens"]

    def compared_tokens(self, matched, parent_len):
        """c_q = min(m+1, |q|, |parent|) per query."""
        return np.minimum(np.minimum(matched + 1, self.q_len), parent_len)


class RecordWorkload:
    """Record streams for configs 1-3 as flat batches (sids, sequences, meta runs) in
    recording order, ready for pack_records / DeviceStore.record / the C oracle.

    c1: 1 session, 8 turns x (128 user + 384 output) -> 4,096 tokens; each turn's
        input = the previous full sequence + user tokens; version bumped from turn 5.
    c2: sessions x 16 branches: shared prefix P=6,144 (input), per-branch S=2,048
        (512 user + 1,536 output), pairwise-distinct first suffix tokens.
    c3: sessions x 2 turns: turn 1 = 1,024 in + 1,024 out @v0; turn 2 = turn 1 + 512
        user @v0 (context version) + 1,536 out split at k ~ U[1, 1535]: leg 1 @v0,
        leg 2 @v1 (a weight switch mid-turn: the partial-rollout stitch).
    """

    def __init__(self, config: int, n_sessions: int | None = None, seed: int | None = None):
        rng = np.random.default_rng(SEED0 + config if seed is None else seed)
        self.sids, self.seqs, self.runs = [], [], []
        self.config = config
        if config == 1:
            n_sessions = n_sessions or 1
            for s in range(n_sessions):
                ctx = np.zeros(0, np.int32)
                runs_s, runs_o, runs_v = [], [], []
                for t in range(8):
                    v = 0 if t < 5 else 1
                    user = rng.integers(0, VOCAB, 128, dtype=np.int32)
                    out = rng.integers(0, VOCAB, 384, dtype=np.int32)
                    # the recorded sequence is input ++ output; input runs are re-tagged
                    # with the current version (trajectory.py:226-230)
                    seq = np.concatenate([ctx, user, out])
                    n_in = len(ctx) + 128
                    self._add(s, seq, [0, n_in], [0, 1], [v, v])
                    ctx = seq
        elif config == 2:
            n_sessions = n_sessions or 1000
            P, S, K = 6144, 2048, 16
            for s in range(n_sessions):
                prefix = rng.integers(0, VOCAB, P, dtype=np.int32)
                firsts = rng.choice(VOCAB, size=K, replace=False).astype(np.int32)
                for k in range(K):
                    suf = rng.integers(0, VOCAB, S, dtype=np.int32)
                    suf[0] = firsts[k]
                    self._add(s, np.concatenate([prefix, suf]), [0, P + 512], [0, 1], [0, 0])
        elif config == 3:
            n_sessions = n_sessions or 4000
            self.split = []
            for s in range(n_sessions):
                t1 = rng.integers(0, VOCAB, 2048, dtype=np.int32)
                self._add(s, t1, [0, 1024], [0, 1], [0, 0])
                user = rng.integers(0, VOCAB, 512, dtype=np.int32)
                out = rng.integers(0, VOCAB, 1536, dtype=np.int32)
                k = int(rng.integers(1, 1536))
                self.split.append(k)
                n_in = 2048 + 512
                self._add(s, np.concatenate([t1, user, out]), [0, n_in, n_in + k], [0, 1, 1], [0, 0, 1])
        else:
            raise ValueError(config)
        self.n_sessions = n_sessions

    def _add(self, s, seq, starts, origins, versions):
        self.sids.append(s)
        self.seqs.append(np.asarray(seq, np.int32))
        self.runs.append((np.asarray(starts, np.int32), np.asarray(origins, np.uint8), np.asarray(versions, np.int32)))

    def packed(self, sid_map=None):
        """(sids, tokens, tok_off[n+1], run_off[n+1], run_start, run_origin, run_version)."""
        sids = np.asarray(self.sids if sid_map is None else [sid_map[s] for s in self.sids], np.int32)
        lens = np.array([len(x) for x in self.seqs], np.int64)
        off = np.zeros(len(lens) + 1, np.int64)
        np.cumsum(lens, out=off[1:])
        rc = np.array([len(r[0]) for r in self.runs], np.int64)
        roff = np.zeros(len(rc) + 1, np.int64)
        np.cumsum(rc, out=roff[1:])
        return (sids, np.concatenate(self.seqs), off, roff, np.concatenate([r[0] for r in self.runs]),
                np.concatenate([r[1] for r in self.runs]), np.concatenate([r[2] for r in self.runs]))

    def per_token_meta(self, k):
        """Own (mask, versions) of record k over its full length."""
        st, org, ver = self.runs[k]
        L = len(self.seqs[k])
        ends = np.append(st[1:], L)
        mask = np.repeat(org, ends - st)
        vers = np.repeat(ver, ends - st)
        return mask, vers


# ------------------------------------------------------------------ config 5 (on device)


def synth_tokens(g, p, salt: int = 0):
    """Counter-based synthetic token of session g at position p (torch int64 tensors ->
    int32), so any rank can regenerate any session's history without storing it."""
    import torch

    x = (g * 0x9E3779B1 + p * 0x7FEB352D + 0x165667B1 + salt * 0x27D4EB2F) & 0xFFFFFFFF
    x = x ^ (x >> 15)
    x = (x * 0x2C1B3C6D) & 0xFFFFFFFF
    x = x ^ (x >> 12)
    x = (x * 0x297A2D39) & 0xFFFFFFFF
    x = x ^ (x >> 15)
    return (x % VOCAB).to(torch.int32)


def turn_runs_batch(lens: np.ndarray, turns: int = 8, bump_at: int = 5):
    """turn_runs for many sessions at once (sessions shorter than 64 tokens: one run)."""
    n = len(lens)
    per = lens // turns
    n_in = np.maximum(1, (per * 0.125).astype(np.int64))
    t = np.arange(turns)
    starts = np.stack([t[None, :] * per[:, None], t[None, :] * per[:, None] + n_in[:, None]], axis=2).reshape(n, -1)
    origins = np.tile(np.array([0, 1], np.uint8), (n, turns))
    vers = np.repeat((t >= bump_at).astype(np.int32), 2)[None, :].repeat(n, 0)
    short = lens < 64
    run_cnt = np.where(short, 1, 2 * turns)
    run_off = np.zeros(n + 1, np.int64)
    np.cumsum(run_cnt, out=run_off[1:])
    keep = np.ones((n, 2 * turns), bool)
    keep[short, 1:] = False
    starts[short, 0] = 0
    origins[short, 0] = 1
    vers[short, 0] = 0
    return run_off, starts[keep].astype(np.int32), origins[keep], vers[keep].astype(np.int32)


class C5Workload:
    """Config 5: S sessions with log-uniform lengths in [lo, hi], sharded by session hash
    over nranks; each rank originates a batch of queries for sessions owned anywhere."""

    def __init__(self, n_sessions=1_000_000, lo=1024, hi=131072, nranks=1, rank=0, n_queries=4096,
                 ext_frac=0.75, new_tokens=256):
        from paper_2508_11553_b200.routing import owner_of

        rng = np.random.default_rng(SEED0 + 5)
        self.n_sessions, self.nranks, self.rank = n_sessions, nranks, rank
        self.lens = np.exp(rng.uniform(np.log(lo), np.log(hi), n_sessions)).astype(np.int64)
        self.owner = owner_of(np.arange(n_sessions), nranks)
        self.owned = np.flatnonzero(self.owner == rank)
        self.g2l = np.full(n_sessions, -1, np.int32)
        self.g2l[self.owned] = np.arange(len(self.owned), dtype=np.int32)
        q = np.random.default_rng(SEED0 + 55 + 1000 * rank)
        self.q_g = q.integers(0, n_sessions, n_queries)
        L = self.lens[self.q_g]
        ext = q.random(n_queries) < ext_frac
        self.q_depth = np.where(ext, L, (q.random(n_queries) * L).astype(np.int64))
        self.q_len = self.q_depth + new_tokens
        pad = (self.q_len + ALIGN - 1) // ALIGN * ALIGN
        self.q_off = np.zeros(n_queries + 1, np.int64)
        np.cumsum(pad, out=self.q_off[1:])
        self.n_queries = n_queries

    def build_shard(self, store, chunk_tokens=1 << 28):
        """Record this rank's sessions (one history row each) into ``store``."""
        import torch

        dev = torch.device("cuda", store.device)
        sids = [store.new_session() for _ in range(len(self.owned))]
        assert sids == list(range(len(self.owned)))
        k0 = 0
        while k0 < len(self.owned):
            lens = self.lens[self.owned[k0:]]
            pad = (lens + ALIGN - 1) // ALIGN * ALIGN
            k1 = k0 + max(1, int(np.searchsorted(np.cumsum(pad), chunk_tokens)))
            k1 = min(k1, len(self.owned))
            g = self.owned[k0:k1]
            lens, pad = self.lens[g], (self.lens[g] + ALIGN - 1) // ALIGN * ALIGN
            starts = np.zeros(len(g) + 1, np.int64)
            np.cumsum(pad, out=starts[1:])
            tot = int(starts[-1])
            gi = torch.repeat_interleave(torch.as_tensor(g, device=dev), torch.as_tensor(pad, device=dev))
            base = torch.repeat_interleave(torch.as_tensor(starts[:-1], device=dev), torch.as_tensor(pad, device=dev))
            pos = torch.arange(tot, device=dev, dtype=torch.int64) - base
            tok = synth_tokens(gi, pos)
            del gi, base, pos
            roff, rs, ro, rv = turn_runs_batch(lens)
            r = store.record_device(np.arange(k0, k1, dtype=np.int32), tok, starts[:-1], lens, roff, rs, ro, rv)
            assert np.all(r.matched == 0) and np.all(r.added == lens)
            del tok
            k0 = k1

    def fill_queries(self, router):
        """Generate this rank's query batch straight into its routing region."""
        import torch

        dev = router.gsid.device
        n = self.n_queries
        router.gsid[:n].copy_(torch.as_tensor(self.q_g, device=dev))
        router.qoff[:n].copy_(torch.as_tensor(self.q_off[:-1], device=dev))
        router.qlen[:n].copy_(torch.as_tensor(self.q_len, device=dev))
        pad = np.diff(self.q_off)
        tot = int(self.q_off[-1])
        gi = torch.repeat_interleave(torch.as_tensor(self.q_g, device=dev), torch.as_tensor(pad, device=dev))
        base = torch.repeat_interleave(torch.as_tensor(self.q_off[:-1], device=dev), torch.as_tensor(pad, device=dev))
        pos = torch.arange(tot, device=dev, dtype=torch.int64) - base
        d = torch.repeat_interleave(torch.as_tensor(self.q_depth, device=dev), torch.as_tensor(pad, device=dev))
        Lh = torch.repeat_interleave(torch.as_tensor(self.lens[self.q_g], device=dev), torch.as_tensor(pad, device=dev))
        hist = synth_tokens(gi, pos)
        fresh = synth_tokens(gi, pos, salt=1)
        # forced mismatch at d when the history continues there
        forced = ((hist.to(torch.int64) + 1 + synth_tokens(gi, pos, salt=2).to(torch.int64) % (VOCAB - 1)) % VOCAB).to(torch.int32)
        tok = torch.where(pos < d, hist, torch.where((pos == d) & (d < Lh), forced, fresh))
        router.tokens[:tot].copy_(tok)


class C5CpuSample:
    """A config-5-shaped sample for the CPU baseline (the 1M-session store
    does not fit the host as Python objects, so a seeded sample of sessions with the same
    log-uniform length law is timed): histories from synth_tokens (the same counter-based
    generator as the GPU shards, on the CPU), a batch of queries on those sessions,
    75 % extensions + 256 new tokens / 25 % branches with a forced mismatch."""

    def __init__(self, nranks=1, n_sessions=10_000, n_queries=4096, lo=1024, hi=131072, ext_frac=0.75,
                 new_tokens=256):
        import torch

        rng = np.random.default_rng(SEED0 + 5)
        lens_all = np.exp(rng.uniform(np.log(lo), np.log(hi), 1_000_000)).astype(np.int64)
        self.g = np.arange(n_sessions, dtype=np.int64)  # the first sessions of the 1M (same lengths)
        self.lens = lens_all[: n_sessions]
        self.n_sessions, self.n_queries = n_sessions, n_queries
        q = np.random.default_rng(SEED0 + 56)
        self.q_sess = q.integers(0, n_sessions, n_queries).astype(np.int32)
        L = self.lens[self.q_sess]
        ext = q.random(n_queries) < ext_frac
        self.q_depth = np.where(ext, L, (q.random(n_queries) * L).astype(np.int64))
        self.q_len = self.q_depth + new_tokens
        self._torch = torch

    def _hist(self, s):
        t = self._torch
        return synth_tokens(t.full((int(self.lens[s]),), int(self.g[s]), dtype=t.int64),
                            t.arange(int(self.lens[s]), dtype=t.int64)).numpy()

    def build_port(self, nthreads):
        """(C port store holding the sample's histories, query tokens, query offsets)."""
        from oracle.cport import CRadixStore

        t = self._torch
        off = np.zeros(self.n_sessions + 1, np.int64)
        np.cumsum(self.lens, out=off[1:])
        g = t.repeat_interleave(t.as_tensor(self.g), t.as_tensor(self.lens))
        base = t.repeat_interleave(t.as_tensor(off[:-1]), t.as_tensor(self.lens))
        pos = t.arange(int(off[-1]), dtype=t.int64) - base
        toks = synth_tokens(g, pos).numpy()
        roff, rs, ro, rv = turn_runs_batch(self.lens)
        st = CRadixStore()
        st.insert_batch(np.arange(self.n_sessions, dtype=np.int32), toks, off, roff, rs, ro, rv, nthreads=nthreads)
        qo = np.zeros(self.n_queries + 1, np.int64)
        np.cumsum(self.q_len, out=qo[1:])
        qt = np.empty(int(qo[-1]), np.int32)
        qrng = np.random.default_rng(SEED0 + 57)
        for i in range(self.n_queries):
            s, d = int(self.q_sess[i]), int(self.q_depth[i])
            h = toks[off[s]: off[s + 1]]
            tail = qrng.integers(0, VOCAB, self.q_len[i] - d, dtype=np.int32)
            if d < len(h):
                tail[0] = (int(h[d]) + 1) % VOCAB
            qt[qo[i]: qo[i] + d] = h[:d]
            qt[qo[i] + d: qo[i + 1]] = tail
        self.qt, self.qo = qt, qo
        return st, qt, qo
