"""The reference's trajectory-manager tests (pkg/tests/test_trajectory.py,
test_integration_edges.py, test_acceptance.py criteria 1-4), run against the B200
drop-in TrajectoryManager with the test-double engine/controller (tests/support)."""

import random
import threading

import pytest

from tests.support.engine import Control, Engine, next_token, oracle_generate

pytestmark = pytest.mark.gpu
VOCAB = 4096


@pytest.fixture(scope="module")
def store():
    from paper_2508_11553_b200 import DeviceStore

    s = DeviceStore(0)
    yield s
    s.close()


@pytest.fixture
def stack(store):
    from paper_2508_11553_b200 import TrajectoryManager

    engine = Engine(VOCAB)
    rm = Control(engine)
    tm = TrajectoryManager(engine, control=rm, pending_timeout=5.0, store=store)
    return engine, rm, tm


def P(n, seed=0, stop=None):
    from paper_2508_11553_b200 import GenParams

    return GenParams(max_new_tokens=n, seed=seed, stop_condition=stop)


def oracle_run(inp, seed, version, n, prefix=()):
    out = list(prefix)
    while len(out) < n:
        out.append(next_token(list(inp) + out, seed, version, VOCAB))
    return out[len(prefix):]


def test_single_turn_pass_through(stack):
    _, _, tm = stack
    out = tm.proxy_generate("s1", [1, 2, 3], P(6, 7))
    assert out == oracle_run([1, 2, 3], 7, 0, 6)
    trie = tm.trie_for("s1")
    assert len(trie.root.children) == 1
    (child,) = trie.root.children.values()
    assert child.tokens == [1, 2, 3] + out


def test_switch_mid_turn_is_invisible_to_agent(stack):
    from paper_2508_11553_b200 import validate_trajectory

    engine, rm, tm = stack
    fired = []

    def hook(job_id, pos):
        if pos == 4 and not fired:
            fired.append(True)
            rm.coordinate_update(1)

    engine.step_hook = hook
    out = tm.proxy_generate("s1", [9, 9], P(10, 5))
    engine.step_hook = None
    head = oracle_run([9, 9], 5, 0, 10)[:4]
    assert out == head + oracle_run([9, 9], 5, 1, 10, prefix=head)
    (traj,) = tm.extract_trajectories("s1")
    assert traj.version_tags == [0, 0] + [0] * 4 + [1] * 6
    assert validate_trajectory(traj, vocab_size=VOCAB).ok


def test_branches_share_prefix_once(stack):
    _, _, tm = stack
    a = tm.proxy_generate("s1", [1, 2, 3, 4], P(4, 1))
    b = tm.proxy_generate("s1", [1, 2, 3, 4], P(4, 2))
    assert a != b
    st = tm.storage_stats("s1")
    assert st.naive_tokens == 16 and st.stored_tokens == 4 + len(a) + len(b) and 0 < st.dedup_ratio < 1


def test_multi_turn_extends_single_path(stack):
    _, _, tm = stack
    t1 = [5, 6]
    o1 = tm.proxy_generate("s1", t1, P(4, 3))
    t2 = t1 + o1 + [7]
    o2 = tm.proxy_generate("s1", t2, P(4, 3))
    trajs = tm.extract_trajectories("s1")
    assert {tuple(t.tokens) for t in trajs} == {tuple(t1 + o1), tuple(t2 + o2)}
    assert tm.storage_stats("s1").stored_tokens == len(t2 + o2)
    long = max(trajs, key=len)
    assert long.loss_mask[len(t1): len(t1) + len(o1)] == [True] * len(o1)  # first-writer mask
    assert long.loss_mask[len(t2) - 1] is False


def test_version_step_at_turn_boundary(stack):
    from paper_2508_11553_b200 import validate_trajectory

    _, rm, tm = stack
    t1 = [1]
    o1 = tm.proxy_generate("s1", t1, P(3))
    rm.coordinate_update(1)
    tm.proxy_generate("s1", t1 + o1 + [2], P(3))
    two = sorted(tm.extract_trajectories("s1"), key=len)[-1]
    assert validate_trajectory(two).ok
    b = len(t1) + len(o1)
    assert set(two.version_tags[:b]) == {0} and set(two.version_tags[b:]) == {1}


def test_unknown_and_empty_sessions(stack):
    from paper_2508_11553_b200 import UnknownSessionError

    _, _, tm = stack
    with pytest.raises(UnknownSessionError):
        tm.extract_trajectories("nope")
    with pytest.raises(UnknownSessionError):
        tm.storage_stats("nope")
    tm.open_request("s1", [1], P(2))
    assert tm.extract_trajectories("s1") == []


def test_partials_behind_flag(stack):
    from paper_2508_11553_b200 import PumpStatus, validate_trajectory

    _, rm, tm = stack
    req = tm.open_request("s1", [1], P(8))
    for _ in range(4):
        tm.pump(req)
    rm.pause_rollouts()
    while tm.pump(req) is PumpStatus.PROGRESS:
        pass
    assert tm.extract_trajectories("s1") == []
    parts = tm.extract_trajectories("s1", include_partials=True)
    assert len(parts) == 1 and parts[0].tokens[0] == 1 and validate_trajectory(parts[0]).ok


def test_min_version_filter(stack):
    _, rm, tm = stack
    tm.proxy_generate("s1", [1], P(2, 1))
    rm.coordinate_update(1)
    tm.proxy_generate("s1", [2], P(2, 1))
    assert len(tm.extract_trajectories("s1")) == 2
    assert len(tm.extract_trajectories("s1", min_version=1)) == 1


def test_drain_semantics(stack):
    _, _, tm = stack
    assert tm.drain_batch(4) is None
    for i in range(5):
        tm.proxy_generate(f"s{i}", [i + 1], P(2))
    assert len(tm.drain_batch(4)) == 5
    assert tm.drain_batch(1) is None
    tm.proxy_generate("s0", [1], P(2))  # identical turn: same leaf, not redelivered
    assert tm.drain_batch(1) is None
    out = tm.proxy_generate("s0", [1] + oracle_run([1], 0, 0, 2) + [2], P(2))
    assert len(out) == 2 and len(tm.drain_batch(1)) == 1
    with pytest.raises(ValueError):
        tm.drain_batch(0)


def test_concurrent_drains_are_disjoint(stack):
    _, _, tm = stack
    for i in range(40):
        tm.proxy_generate(f"s{i}", [i + 1], P(2))
    got = []

    def drain():
        while (b := tm.drain_batch(1)) is not None:
            got.append(b)

    ts = [threading.Thread(target=drain) for _ in range(6)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    ids = [tuple(t.tokens) for b in got for t in b]
    assert len(ids) == 40 == len(set(ids))


def test_capture_matches_engine_oracle_log(stack):
    engine, rm, tm = stack
    fired = []

    def hook(job_id, pos):
        if pos == 3 and not fired:
            fired.append(True)
            rm.coordinate_update(1)

    engine.step_hook = hook
    out = tm.proxy_generate("s1", [3, 1], P(7, 2), request_id="r1")
    engine.step_hook = None
    legs = engine.oracle_log("r1")
    assert len(legs) == 2 and [t for l in legs for t in l.output_tokens] == out
    (traj,) = tm.extract_trajectories("s1")
    assert traj.tokens == [3, 1] + out
    assert traj.version_tags[2:] == [v for l in legs for v in l.version_per_token]


def test_concurrent_branched_turns_share_prefix_once(store):
    from paper_2508_11553_b200 import TrajectoryManager

    engine = Engine(VOCAB)
    tm = TrajectoryManager(engine, control=Control(engine), pending_timeout=5.0, store=store)
    prefix = list(range(50, 66))
    res = {}

    def branch(seed):
        res[seed] = tm.proxy_generate("scale", prefix, P(8, seed))

    ts = [threading.Thread(target=branch, args=(s,)) for s in range(6)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    seqs = [tuple(prefix + res[s]) for s in res]
    st = tm.storage_stats("scale")
    assert st.naive_tokens == 6 * 24
    assert st.stored_tokens == len({q[:i] for q in seqs for i in range(1, len(q) + 1)})
    assert tm.trie_for("scale").check_well_formed() == []
    assert {tuple(t.tokens) for t in tm.extract_trajectories("scale")} == set(seqs)


def test_pending_request_times_out_as_retryable(store):
    from paper_2508_11553_b200 import ProxyRetryableError, TrajectoryManager

    engine = Engine(VOCAB)
    tm = TrajectoryManager(engine, pending_timeout=0.15, poll_interval=0.005, store=store)
    engine.begin_switch()
    with pytest.raises(ProxyRetryableError):
        tm.proxy_generate("s", [1], P(4))
    assert tm.extract_trajectories("s", include_partials=True) == []
    engine.complete_switch(1)
    assert len(tm.proxy_generate("s", [1], P(4))) == 4


def test_criterion_1_bit_exact_capture(store):
    """test_acceptance.py:64-115 (200 sessions here): extracted trajectories equal the
    engine's own log, with random weight switches mid-turn."""
    from paper_2508_11553_b200 import TrajectoryManager, validate_trajectory

    engine = Engine(VOCAB)
    rm = Control(engine)
    tm = TrajectoryManager(engine, control=rm, pending_timeout=10.0, store=store)
    rng = random.Random(20250810)
    sw = {"step": None}
    steps = {"n": 0}

    def hook(job_id, pos):
        steps["n"] += 1
        if sw["step"] is not None and steps["n"] >= sw["step"]:
            sw["step"] = None
            rm.coordinate_update(engine.current_version + 1)

    engine.step_hook = hook
    for s in range(200):
        sid = f"sess-{s}"
        contexts, expected = [[]], set()
        for turn in range(rng.randint(1, 6)):
            inp = list(rng.choice(contexts)) + [rng.randrange(VOCAB) for _ in range(rng.randint(2, 5))]
            params = P(rng.randint(4, 9), rng.randrange(1_000_000))
            if rng.random() < 0.25:
                sw["step"] = steps["n"] + rng.randint(1, params.max_new_tokens)
            rid = f"{sid}-t{turn}"
            out = tm.proxy_generate(sid, inp, params, request_id=rid)
            assert out == [t for l in engine.oracle_log(rid) for t in l.output_tokens]
            contexts.append(inp + out)
            expected.add(tuple(inp + out))
        ext = tm.extract_trajectories(sid)
        assert {tuple(t.tokens) for t in ext} == expected
        assert all(validate_trajectory(t, vocab_size=VOCAB).ok for t in ext)
    engine.step_hook = None


def test_criterion_3_switch_at_every_position(store):
    from paper_2508_11553_b200 import TrajectoryManager

    N = 32
    for k in range(N + 1):
        engine = Engine(VOCAB)
        rm = Control(engine)
        tm = TrajectoryManager(engine, control=rm, pending_timeout=10.0, store=store)
        fired = []

        def hook(job_id, pos, k=k):
            if pos == k and not fired:
                fired.append(True)
                rm.coordinate_update(1)

        engine.step_hook = hook
        params = P(N, k * 131 + 7)
        out = tm.proxy_generate("s", [11, 22], params)
        head = oracle_generate([11, 22], params, 0, VOCAB)[:k]
        if k < N:
            assert out == head + oracle_generate([11, 22], params, 1, VOCAB, prefix=head)
        (traj,) = tm.extract_trajectories("s")
        assert traj.version_tags[2:] == [0] * k + [1] * (N - k)


def test_criterion_4_pause_resume_is_bit_exact(store):
    from paper_2508_11553_b200 import PumpStatus, TrajectoryManager

    rng = random.Random(4242)
    for case in range(100):
        engine = Engine(VOCAB)
        rm = Control(engine)
        tm = TrajectoryManager(engine, control=rm, pending_timeout=10.0, store=store)
        inp = [rng.randrange(VOCAB) for _ in range(rng.randint(1, 6))]
        params = P(rng.randint(4, 24), rng.randrange(10**9))
        base = oracle_generate(inp, params, 0, VOCAB)
        stops = sorted(rng.sample(range(1, params.max_new_tokens + 1), rng.randint(1, min(4, params.max_new_tokens))))
        n = {"n": 0}

        def hook(job_id, pos):
            n["n"] += 1
            if stops and n["n"] >= stops[0]:
                stops.pop(0)
                rm.pause_rollouts()

        engine.step_hook = hook
        req = tm.open_request("s", inp, params)
        for _ in range(10_000):
            st = tm.pump(req)
            if st is PumpStatus.DONE:
                break
            if st is PumpStatus.WAITING:
                rm.resume_rollouts()
        assert req.response == base, case
        (traj,) = tm.extract_trajectories("s")
        assert traj.tokens == inp + base
