"""The synthetic workloads are the BASELINE.json configs (shapes asserted, CPU only):
c1 one session of 8 turns to 4,096 tokens; c2 1k sessions x 16 branches of 8,192 tokens
sharing a 6,144-token prefix with pairwise-distinct first suffix tokens; c3 4k sessions x
2 turns with a mid-turn version switch; c4 10k x 32,768-token histories and 4,096-query
batches (75 % extend the full history); c5 1M sessions, log-uniform 1k-128k."""

import numpy as np

from workloads import C5Workload, MatchWorkload, RecordWorkload


def test_c1_c2_c3_shapes():
    c1 = RecordWorkload(1)
    assert c1.n_sessions == 1 and len(c1.seqs) == 8 and len(c1.seqs[-1]) == 4096
    assert all(np.array_equal(c1.seqs[k][: len(c1.seqs[k - 1])], c1.seqs[k - 1]) for k in range(1, 8))
    c2 = RecordWorkload(2, n_sessions=20)
    assert len(c2.seqs) == 20 * 16 and all(len(x) == 8192 for x in c2.seqs)
    for s in range(20):
        rows = [c2.seqs[k] for k in range(len(c2.seqs)) if c2.sids[k] == s]
        assert all(np.array_equal(r[:6144], rows[0][:6144]) for r in rows)
        assert len({int(r[6144]) for r in rows}) == 16  # pairwise-distinct first suffix tokens
    c3 = RecordWorkload(3, n_sessions=30)
    assert len(c3.seqs) == 60
    for s in range(30):
        t1, t2 = c3.seqs[2 * s], c3.seqs[2 * s + 1]
        assert len(t1) == 2048 and len(t2) == 4096 and np.array_equal(t2[:2048], t1)
        st, org, ver = c3.runs[2 * s + 1]
        assert org.tolist() == [0, 1, 1] and ver.tolist() == [0, 0, 1] and 2560 < st[2] < 4096  # the stitch


def test_c4_and_c5_shapes():
    wl = MatchWorkload(n_sessions=200, hist_len=32_768, n_queries=512)
    ext = wl.q_depth == 32_768
    assert 0.6 < ext.mean() < 0.9 and np.all(wl.q_len == wl.q_depth + 256)
    c5 = C5Workload(20_000, n_queries=256)
    assert c5.lens.min() >= 1024 and c5.lens.max() <= 131_072
    assert np.log(c5.lens).std() > 1.0  # log-uniform spread, not a constant length
