"""Per-call latency of the drop-in API (single lpm_insert / path_trajectory / extract)
next to the reference's own Python implementation (a C restatement is not the right
comparison for per-call overhead; the pure-Python oracle restates trie.py)."""

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2508_11553_b200 import DeviceStore, SessionTrie, SpanOrigin
    from paper_2508_11553_b200.trie import _as_int32, meta_runs
    from tools.refbench import reference_modules

    mods = reference_modules()
    if mods is None:
        from oracle.radix import RadixOracle
    store = DeviceStore(0)
    rng = np.random.default_rng(0)
    for L in (16, 512, 4096, 32768):
        trie = SessionTrie("lat", store=store)
        base = rng.integers(0, 151936, L).tolist()
        org = [SpanOrigin.AGENT_INPUT] * (L // 2) + [SpanOrigin.MODEL_OUTPUT] * (L - L // 2)
        ver = [0] * L
        seqs = [base[: L - 8] + rng.integers(0, 151936, 8).tolist() for _ in range(50)]
        trie.lpm_insert(seqs[0], org, ver, "w")
        t0 = time.perf_counter()
        for s in seqs[1:]:
            trie.lpm_insert(s, org, ver, "c")
        t_ins = (time.perf_counter() - t0) / (len(seqs) - 1)
        # breakdown: Python-side argument preparation vs the C-ABI call
        t0 = time.perf_counter()
        for s in seqs[1:]:
            runs = meta_runs(org, ver)
            toks = _as_int32(s)
        t_prep = (time.perf_counter() - t0) / (len(seqs) - 1)
        t0 = time.perf_counter()
        for s in seqs[1:]:
            store.record_one(trie.sid, toks, runs)
        t_c = (time.perf_counter() - t0) / (len(seqs) - 1)
        if mods is not None:
            trie_mod, core = mods
            ref = trie_mod.SessionTrie("lat")
            rorg = [core.SpanOrigin.AGENT_INPUT] * (L // 2) + [core.SpanOrigin.MODEL_OUTPUT] * (L - L // 2)
            ref.lpm_insert(seqs[0], rorg, ver, "w")
            t0 = time.perf_counter()
            for s in seqs[1:]:
                ref.lpm_insert(s, rorg, ver, "c")
            t_ref = (time.perf_counter() - t0) / (len(seqs) - 1)
            t0 = time.perf_counter()
            for k in range(20):
                ref.path_trajectory(k + 1)
            t_ref_path = (time.perf_counter() - t0) / 20
            kind = "reference"
        else:
            ora = RadixOracle()
            o01 = [0] * (L // 2) + [1] * (L - L // 2)
            t0 = time.perf_counter()
            for s in seqs:
                ora.insert(s, o01, ver, "c")
            t_ref = (time.perf_counter() - t0) / len(seqs)
            t_ref_path = float("nan")
            kind = "restatement"
        t0 = time.perf_counter()
        for k in range(20):
            trie.path_trajectory(k)
        t_path = (time.perf_counter() - t0) / 20
        trie.extract()  # warm: first call at a new size grows the staging buffers
        t0 = time.perf_counter()
        ext = trie.extract()
        t_ext = time.perf_counter() - t0
        print(f"L={L:6d}  lpm_insert {t_ins*1e6:8.1f} us (python prep {t_prep*1e6:6.1f} + C call {t_c*1e6:6.1f}; "
              f"{kind} {t_ref*1e6:8.1f} us)  path_trajectory {t_path*1e6:8.1f} us ({kind} {t_ref_path*1e6:8.1f} us)  "
              f"extract({len(ext)} rows) {t_ext*1e3:7.2f} ms", flush=True)


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def ingest_throughput(threads=16, per=100, L=4096):
    """Records/s when `threads` finalizers record concurrently: per-record vs micro-batched."""
    import threading

    from paper_2508_11553_b200 import DeviceStore, TrajectoryManager

    class E:
        current_version = 0

    rng = np.random.default_rng(1)
    base = [rng.integers(0, 151936, L).tolist() for _ in range(threads)]
    for batched in (False, True):
        store = DeviceStore(0)
        tm = TrajectoryManager(E(), store=store, batched_ingest=batched)

        def worker(t):
            ctx = base[t]
            for k in range(per):
                out = rng.integers(0, 151936, 64).tolist()
                tm.record(f"s{t}", ctx, out, [0] * 64, 0, f"r{t}-{k}")  # branches off a shared context

        ths = [threading.Thread(target=worker, args=(t,)) for t in range(threads)]
        t0 = time.perf_counter()
        [x.start() for x in ths]
        [x.join() for x in ths]
        dt = time.perf_counter() - t0
        tm.close()
        print(f"ingest {'batched' if batched else 'per-record'}: {threads * per / dt:10.0f} records/s "
              f"({threads} threads x {per} records of {L}+64 tokens)")
        store.close()


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "ingest":
    for L in (256, 4096):
        ingest_throughput(L=L)
