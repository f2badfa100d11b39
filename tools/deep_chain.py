"""A long agent session recorded turn by turn (each turn extends the previous one):
per-insert latency and export time as the row chain grows (deep-chain behaviour)."""

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(turns=2000, per=32):
    from paper_2508_11553_b200 import DeviceStore, SessionTrie, SpanOrigin

    store = DeviceStore(0)
    trie = SessionTrie("deep", store=store)
    rng = np.random.default_rng(0)
    seq = []
    marks = {1, 10, 100, 500, 1000, 2000}
    for t in range(1, turns + 1):
        seq = seq + rng.integers(0, 151936, per).tolist()
        t0 = time.perf_counter()
        r = trie.lpm_insert(seq, [SpanOrigin.MODEL_OUTPUT] * len(seq), [0] * len(seq), f"t{t}")
        dt = time.perf_counter() - t0
        assert r.matched_prefix_length == len(seq) - per
        if t in marks:
            t0 = time.perf_counter()
            p = trie.path_trajectory(r.node_id)
            de = time.perf_counter() - t0
            assert p.tokens == seq
            t0 = time.perf_counter()
            trie.store.export([trie.row_of(r.node_id)], total=len(seq))  # the C-ABI part alone
            dx = time.perf_counter() - t0
            print(f"turn {t:5d} ({len(seq):6d} tokens, chain depth {t - 1:5d}): lpm_insert {dt * 1e3:7.2f} ms  "
                  f"path_trajectory {de * 1e3:7.2f} ms (export call {dx * 1e3:6.2f} ms)", flush=True)


if __name__ == "__main__":
    main()
