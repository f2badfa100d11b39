"""Pin the test-double engine to the reference's frozen token streams (CPU)."""

from tests.support.engine import Engine, next_token


class _P:
    def __init__(self, n, seed, stop=None):
        self.max_new_tokens, self.seed, self.stop_condition = n, seed, stop

    def validate(self):
        assert self.max_new_tokens >= 1


def _run(engine, inp, params, prefix=()):
    jid = engine.start_job(inp, params, prefix=prefix)
    while engine.step_job(jid).value == "token":
        pass
    return engine.finish_job(jid)


def test_golden_token_vectors():
    from tests.conftest import load_golden

    for v in load_golden("engine_vectors.json"):
        assert next_token(v["context"], v["seed"], v["version"], v["vocab"]) == v["token"]


def test_frozen_streams():
    # tests/test_engine.py:54-55, 193-194 in the reference
    e = Engine()
    assert _run(e, [1, 2, 3], _P(8, 7)).output_tokens == [4037, 2817, 2147, 3737, 3615, 3838, 2964, 2384]
    e.begin_switch()
    e.complete_switch(1)
    assert _run(e, [1, 2, 3], _P(8, 7)).output_tokens == [572, 2994, 3703, 2183, 203, 1762, 2946, 1444]
    e2 = Engine()
    full = _run(e2, [5], _P(10, 7)).output_tokens
    assert full == [2842, 3194, 379, 355, 2388, 3269, 2388, 1921, 3027, 2323]
    e2.begin_switch()
    e2.complete_switch(1)
    assert _run(e2, [5], _P(10, 7), prefix=full[:4]).output_tokens == [1042, 764, 2208, 823, 2072, 98]
