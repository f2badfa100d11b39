"""Benchmark: prefix-match queries/s and tokens compared/s (HBM GB/s vs peak) on B200.

One JSON line (rank 0).  Headline workload by GPU count (BASELINE.json configs):

  N = 1  c4 (configs[3]): 10,000 sessions x one 32,768-token history, batches of 4,096
         read-only match queries (75 % full history + 256 new tokens, 25 % branches at a
         uniform depth with a forced mismatch).  One step = one batch through K1.
  N > 1  c5 (configs[4]): 1,000,000 sessions, log-uniform 1k-128k histories, sharded by
         session hash; every rank originates 4,096 queries for sessions owned anywhere,
         routed over NVLink by the fused P2P match (pipelined batches).  One step = one
         batch per rank.  The c4 weak-scaling shards are measured beside it (c4_shards).

  value         queries/s with queries resident in HBM (device-timed, CUDA events on the
                launching stream, max over ranks; W warm-up steps, then exactly K)
  e2e           (N = 1) the same through the C-ABI host-buffer call: query tokens cross PCIe
                inside the timed region, results come back
  roofline      K1 algorithmic bytes (8 B per compared token, c_q = min(m+1,|q|,|parent|)) /
                device time per batch, against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the C restatement of the reference trie (oracle/, "port"), all host threads,
                same batch; reference_unmodified: the reference's own Python trie from
                baseline/_ref, one process and a pool over all cores, on a query sample
  configs       (N = 1) c1 / c2 / c3: record (K2), export (K3), NDJSON and - c3 - the
                include_partials export, device and call rates with their rooflines, next to
                the C port and the unmodified reference
  c5_routed     (N = 1) config 5 at one GPU (1M sessions in one 107 GB store, routed path)
  c4_shards,    (N > 1) weak-scaling shards beside the routed headline: every rank its own
  config_shards c4 match shard, and its own copy of configs 2 / 3 recorded and exported

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG", "WARN")  # NCCL's "NCCL version ..." banner would land on stdout beside the JSON line

METRIC = "prefix-match queries/s (c4: 10k sessions x 32k-token histories, 4096-query batches)"
METRIC_C5 = "prefix-match queries/s (c5: 1M sessions, 1k-128k tokens, routed)"
LINK_PEAK = 670.0  # GB/s per GPU, SM peer reads with both directions busy (tools/p2p_probe)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--sessions", type=int, default=10_000)
    ap.add_argument("--hist", type=int, default=32_768)
    ap.add_argument("--queries", type=int, default=4096)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="N=1: skip the c1-c3 record/export measurements")
    ap.add_argument("--no-c5", action="store_true", help="N=1: skip the config-5 routed measurement")
    ap.add_argument("--workload", default=None, choices=["c4", "c5"],
                    help="headline workload (default: c4 at N=1, c5 at N>1)")
    ap.add_argument("--c5-sessions", type=int, default=1_000_000)
    ap.add_argument("--pipeline", action=argparse.BooleanOptionalAction, default=True,
                    help="c5, N>1, fused routing: two routing regions, batch k+1 bucketed + packed while batch k "
                         "is matched (--no-pipeline: one region, batches back to back)")
    ap.add_argument("--routing", default="fused", choices=["fused", "push", "fused-nccl-barrier", "nccl"],
                    help="c5 exchange: fused P2P K1 (owners pull the planes), push (requesters write the planes "
                         "into the owners' inboxes) or NCCL all-to-all + local match (baseline)")
    ap.add_argument("--mixed", default=None,
                    help="lo,hi: log-uniform history lengths (config-5 shard) instead of fixed --hist")
    a = ap.parse_args()
    if a.warmup < 3:
        ap.error("--warmup must be >= 3")
    return a


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def log(*a):
    print("[bench]", *a, file=sys.stderr, flush=True)


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.p = None

    def __enter__(self):
        if os.environ.get("BENCH_CLOCKS", "1") == "0":  # diagnostics only: no sampler
            return self
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p is not None:
            time.sleep(0.15)
            self.p.terminate()
            out, _ = self.p.communicate(timeout=5)
            self.rows = [r.split(", ") for r in out.strip().splitlines() if r.strip()]
        else:
            self.rows = []

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
                for n, v in zip(names, r[3:7]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------- configs

def c4_config(args, world, mixed=None):
    """The config object both arms print (the driver compares the arms on it)."""
    arena_gb = args.sessions * ((args.hist + 31) // 32 * 32) * 4 / 1e9
    query_gb = args.queries * (0.75 * (args.hist + 256) + 0.25 * (args.hist / 2 + 256)) * 4 / 1e9
    return {"workload": "c4" if mixed is None else "c5-shard", "sessions": args.sessions,
            "history_tokens": args.hist if mixed is None else f"log-uniform {mixed}",
            "batch_queries": args.queries, "ext_frac": 0.75, "parallelism": f"session-shard x{world}",
            "l2": "inputs larger than L2 (arena %.2f GB + queries ~%.2f GB per rank)" % (arena_gb, query_gb)}


def c5_config(args, world):
    return {"workload": "c5", "sessions_total": args.c5_sessions, "history_tokens": "log-uniform [1024, 131072]",
            "batch_queries_per_rank": args.queries, "owner": "splitmix64(gsid) mod N", "n_ranks": world,
            "routing": {"fused": "fused P2P K1: owners read requester HBM over NVLink, write results back; "
                                 "device-side epoch-flag barriers (no collective call per batch)",
                        "push": "push P2P: requesters pack remote queries' 18-bit planes straight into the owners' "
                                "inboxes (P2P stores, beside the previous batch's walk); owners walk from local HBM "
                                "and write results back; device-side epoch-flag barriers",
                        "fused-nccl-barrier": "fused P2P K1 bracketed by two one-element NCCL all-reduces",
                        "nccl": "BASELINE: NCCL all-to-all of query tokens, local K1, all-to-all of results"}[
                args.routing] if world > 1 else "one rank: every query is local",
            "pipelined": bool(args.pipeline and args.routing in ("fused", "push")),
            "l2": "inputs larger than L2 (~%.0f GB arena per rank)" % (107.0 / world)}


# ------------------------------------------------------------------------- CPU baselines

_cpu_store = {}


def cpu_port_bench_reuse(wl, nthreads):
    from oracle.cport import CRadixStore

    st = _cpu_store.get("st")
    if st is None:
        st = CRadixStore()
        ns = wl.n_sessions
        toks = np.concatenate([wl.hist_tokens[wl.hist_off[s]: wl.hist_off[s] + wl.hist_len[s]] for s in range(ns)])
        off = np.zeros(ns + 1, np.int64)
        np.cumsum(wl.hist_len, out=off[1:])
        st.insert_batch(np.arange(ns, dtype=np.int32), toks, off, wl.run_off, wl.run_start, wl.run_origin,
                        wl.run_version, nthreads=nthreads)
        n = wl.n_queries
        qt = np.concatenate([wl.q_tokens[wl.q_off[i]: wl.q_off[i] + wl.q_len[i]] for i in range(n)])
        qo = np.zeros(n + 1, np.int64)
        np.cumsum(wl.q_len, out=qo[1:])
        _cpu_store.update(st=st, qt=qt, qo=qo)
    t0 = time.perf_counter()
    res = st.match_batch(wl.q_sess, _cpu_store["qt"], _cpu_store["qo"], nthreads=nthreads)
    return wl.n_queries, time.perf_counter() - t0, res


def reference_match_sample(hist_of, qlist, per_core=16):
    """The UNMODIFIED reference (baseline/_ref) on a sample of match queries: one process
    and a pool over all cores.  Falls back to the pure-Python restatement (oracle/radix.py,
    labelled) when baseline/_ref is not installed."""
    from tools.refbench import time_reference_match

    cores = os.cpu_count() or 1
    q = qlist[: max(8, per_core * cores)]
    r = time_reference_match(hist_of, q)
    if r is not None:
        return {"value": r["pool"], "unit": "queries/s", "cores": r["procs"], "kind": "reference",
                "single_process": r["single"],
                "sample": f"{r['queries_pool']} queries (pool of {r['procs']} processes over session-disjoint "
                          f"shards) / {r['queries_single']} (one process): one lpm_insert each into a trie holding "
                          "the query's session history, the unmodified reference rolloutlab.trie from baseline/_ref"}
    from oracle.radix import RadixOracle  # restatement fallback (labelled)

    tries, work = {}, []
    for s, toks in q[:64]:
        if s not in tries:
            t, o, v = hist_of(s)
            tries[s] = RadixOracle()
            tries[s].insert(t, o, v)
        work.append((s, toks))
    t0 = time.perf_counter()
    for s, toks in work:
        tries[s].insert(toks, [0] * len(toks), [0] * len(toks))
    dt = time.perf_counter() - t0
    return {"value": len(work) / dt, "unit": "queries/s", "cores": 1, "kind": "port",
            "sample": f"{len(work)} queries, pure-Python restatement (oracle/radix.py): baseline/_ref not installed"}


def c4_hist_sampler(wl):
    def hist_of(s):
        a, b = wl.run_off[s], wl.run_off[s + 1]
        st = np.r_[wl.run_start[a:b], wl.hist_len[s]]
        org = np.repeat(wl.run_origin[a:b].astype(np.int64), np.diff(st)).tolist()
        ver = np.repeat(wl.run_version[a:b].astype(np.int64), np.diff(st)).tolist()
        return wl.hist_tokens[wl.hist_off[s]: wl.hist_off[s] + wl.hist_len[s]].tolist(), org, ver
    qlist = [(int(wl.q_sess[i]), wl.q_tokens[wl.q_off[i]: wl.q_off[i] + wl.q_len[i]].tolist())
             for i in range(min(wl.n_queries, 4096))]
    return hist_of, qlist


# ----------------------------------------------------------------------------- reference arm

def run_reference(args):
    """--impl reference: the CPU implementation of the path on this box's host cores, same
    config / metric / unit as the b200 arm (rank 0 only; other ranks exit 0)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from workloads import MatchWorkload

    cores = os.cpu_count() or 1
    workload = args.workload or ("c5" if world > 1 else "c4")
    if workload == "c5":
        from workloads import C5CpuSample

        smp = C5CpuSample(world, n_sessions=10_000, n_queries=args.queries)
        st, qt, qo = smp.build_port(cores)
        times = []
        st.match_batch(smp.q_sess, qt, qo, nthreads=cores)
        for _ in range(max(1, args.steps)):
            t0 = time.perf_counter()
            st.match_batch(smp.q_sess, qt, qo, nthreads=cores)
            times.append(time.perf_counter() - t0)
        v = smp.n_queries * len(times) / sum(times)
        line = {"impl": "reference", "metric": METRIC_C5, "value": v, "unit": "queries/s", "n_gpus": world,
                "steps": len(times), "warmup": 1, "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
                "config": c5_config(args, world),
                "cpu_baseline": {"value": v, "unit": "queries/s", "cores": cores, "kind": "port",
                                 "sample": f"sampled: {smp.n_sessions} of the 1M config-5 sessions (same length law), "
                                           f"{smp.n_queries}-query batches per step on their sessions, C radix-tree "
                                           f"restatement (oracle/radix_oracle.c), {cores} threads; the store is one "
                                           "host's memory, so N GPUs' batches run on the same cores"},
                "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return
    wl = MatchWorkload(args.sessions, args.hist, args.queries)
    times = []
    cpu_port_bench_reuse(wl, cores)  # warm: build the C store + one pass
    for _ in range(max(1, args.steps)):
        _, dt, _ = cpu_port_bench_reuse(wl, cores)
        times.append(dt)
    total = sum(times)
    v = wl.n_queries * len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "queries/s", "n_gpus": world,
        "steps": len(times), "warmup": 1, "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": c4_config(args, world),
        "cpu_baseline": {"value": v, "unit": "queries/s", "cores": cores, "kind": "port",
                         "sample": f"full c4 batch ({wl.n_queries} queries) per step, C radix-tree restatement "
                                   f"(oracle/radix_oracle.c), {cores} threads"},
        "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_cpu and args.sessions >= 1000:
        hist_of, qlist = c4_hist_sampler(wl)
        line["reference_unmodified"] = reference_match_sample(hist_of, qlist)
    print(json.dumps(line))


# ------------------------------------------------------------------------------- c4 (N = 1)

def measure_c4(args, rank, world, local, dev):
    import torch

    from paper_2508_11553_b200 import DeviceStore
    from workloads import SEED0, MatchWorkload

    mixed = tuple(int(x) for x in args.mixed.split(",")) if args.mixed else None
    t0 = time.perf_counter()
    wl = MatchWorkload(args.sessions, args.hist, args.queries, seed=SEED0 + 4 + 1000 * rank, mixed=mixed)
    store = DeviceStore(local, arena_words=int(wl.hist_off[-1]) + (1 << 20), row_capacity=args.sessions + 64,
                        run_capacity=len(wl.run_start) + 64, session_capacity=args.sessions + 16)
    sids = [store.new_session() for _ in range(args.sessions)]
    assert sids[0] == 0 and sids[-1] == args.sessions - 1
    rec = store.record_packed(np.arange(args.sessions, dtype=np.int32), wl.hist_tokens, wl.hist_off[:-1].copy(),
                              wl.hist_len, wl.run_off, wl.run_start, wl.run_origin, wl.run_version)
    assert np.all(rec.matched == 0) and np.all(rec.added == wl.hist_len)
    row_len = wl.hist_len  # row id == session id here (one row per session, recorded in order)
    log(f"rank {rank}: c4 store built in {time.perf_counter() - t0:.1f} s")

    # two device-resident batches with different queries (A is the workload's own batch);
    # consecutive steps alternate A / B so no batch re-reads what the previous one did
    qsets = [dict(q_sess=wl.q_sess, q_len=wl.q_len, q_depth=wl.q_depth, q_off=wl.q_off, q_tokens=wl.q_tokens),
             wl.make_queries(np.random.default_rng(SEED0 + 44 + 1000 * rank))]

    def to_dev(q):
        return (torch.from_numpy(q["q_sess"]).to(dev), torch.from_numpy(q["q_tokens"]).to(dev),
                torch.from_numpy(q["q_off"][:-1].copy()).to(dev), torch.from_numpy(q["q_len"]).to(dev))

    dq = [to_dev(q) for q in qsets]
    om = torch.empty(wl.n_queries, dtype=torch.int64, device=dev)
    # Batches are independent and read-only, so consecutive batches alternate between two
    # streams (each its own output buffers): batch k+1's ramp-up overlaps batch k's tail.
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    stream = streams[0]
    torch.cuda.set_stream(stream)
    outs = [(om, torch.empty_like(om), torch.empty_like(om)), tuple(torch.empty_like(om) for _ in range(3))]
    nstep = [0]

    def step():
        i = nstep[0] & 1
        nstep[0] += 1
        o = outs[i]
        store.match_device(*dq[i], o[0], o[1], o[2], stream=streams[i].cuda_stream)

    # exactly W warm-up steps; the launch profiler's event pairs for the timed region are
    # created up front (cudaEventCreate inside the timed region made N>1 host-bound)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    nstep[0] = 0
    # correctness of the benchmarked batches (size-independent truth) and their bytes
    alg = []
    for i in range(2):
        m = outs[i][0].cpu().numpy()
        par = outs[i][1].cpu().numpy()
        assert np.array_equal(m, qsets[i]["q_depth"]), "matched length != constructed depth"
        assert np.all((par == qsets[i]["q_sess"]) | (m == 0)), "parent row != query session's row"
        plen = np.where(par >= 0, row_len[np.maximum(par, 0)], 0)
        alg.append(np.minimum(np.minimum(m + 1, qsets[i]["q_len"]), plen))
    m = outs[0][0].cpu().numpy()
    cq = (alg[0] + alg[1]) / 2.0  # steps alternate A/B: mean compared tokens per batch
    alg_bytes = 8.0 * float(cq.sum())

    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    store.profile_begin(reserve=args.steps + 64)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        time.sleep(0.3)  # let the sampler start before the timed region
        t_wall = time.perf_counter()
        # Device-side gate before e0: the host enqueues all K steps while the GPU spins, so
        # the events time the steps back to back and not the host's launch jitter.
        if os.environ.get("BENCH_GATE", "1") != "0":
            torch.cuda._sleep(int(1.9e6 * min(1000.0, 20.0 + 2.0 * args.steps)))
        prof = os.environ.get("BENCH_PROFILE_RANGE") == "1"  # ncu --replay-mode range over exactly this region
        if prof:
            torch.cuda.synchronize()
            torch.cuda.profiler.start()
        e0.record(stream)
        streams[1].wait_stream(streams[0])
        t_enq = time.perf_counter()
        for _ in range(args.steps):
            step()
        streams[0].wait_stream(streams[1])
        e1.record(stream)
        t_enq = time.perf_counter() - t_enq
        torch.cuda.synchronize()
        if prof:
            torch.cuda.profiler.stop()
        walk_ms, walk_n = store.profile_end("walk")
        plan_ms, plan_n = store.profile_end("plan")
        # short regions: keep the identical load running so the sampler sees >= 1 s of it
        while time.perf_counter() - t_wall < 1.0:
            for _ in range(50):
                step()
            torch.cuda.synchronize()
    elapsed = e0.elapsed_time(e1) / 1e3
    # A/B of the north star's hash-first filter: the per-128-token block
    # hashes of the query batch it would have to compute before it could filter anything
    nq = (dq[0][1].numel() // 128) * 128
    hashes = torch.empty(nq // 128, dtype=torch.int64, device=dev)
    for _ in range(3):
        store.block_hashes(dq[0][1][:nq], hashes, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    store.profile_begin(reserve=64)
    for _ in range(args.steps):
        store.block_hashes(dq[0][1][:nq], hashes, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    hash_ms, hash_n = store.profile_end("block_hash")
    log(f"rank {rank}: c4 device-timed region {1e3 * elapsed:.3f} ms for {args.steps} steps (walk {walk_ms:.3f} ms "
        f"over {walk_n} launches; host enqueue {1e3 * t_enq:.3f} ms)")
    if world > 1:
        t = torch.tensor([elapsed], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        elapsed = float(t.item())
    value = world * wl.n_queries * args.steps / elapsed
    toks_per_s = world * float(cq.sum()) * args.steps / elapsed

    # e2e: the public host-buffer API, pinned inputs, copies inside the timed region
    pin_tok = torch.from_numpy(wl.q_tokens).pin_memory()
    pin_np = pin_tok.numpy()
    q_off = wl.q_off[:-1].copy()
    store.match(wl.q_sess, pin_np, q_off, wl.q_len)  # warm
    tok_bytes0 = store.h2d_stats()["token_bytes"]
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        mh, ph, dh = store.match(wl.q_sess, pin_np, q_off, wl.q_len)
    e2e_elapsed = time.perf_counter() - t0
    assert np.array_equal(mh, wl.q_depth)
    if world > 1:
        t = torch.tensor([e2e_elapsed], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_elapsed = float(t.item())
    e2e_value = world * wl.n_queries * args.e2e_steps / e2e_elapsed
    # token bytes that crossed PCIe (packed 18-bit planes when the library packs them, see
    # DESIGN.md "PCIe path") + the per-query session ids, offsets and lengths
    h2d = (store.h2d_stats()["token_bytes"] - tok_bytes0) // args.e2e_steps + wl.n_queries * (4 + 8 + 8)
    d2h = wl.n_queries * 24
    # e2e from Python-list callers (the reference's own argument type): tokens as lists
    lists = None
    if world == 1 and not args.no_cpu:
        qtl = [wl.q_tokens[wl.q_off[i]: wl.q_off[i] + wl.q_len[i]].tolist() for i in range(wl.n_queries)]
        t0 = time.perf_counter()
        mh2, _, _ = store.match_lists(wl.q_sess, qtl)
        dt_l = time.perf_counter() - t0
        assert np.array_equal(mh2, wl.q_depth)
        lists = {"value": wl.n_queries / dt_l, "unit": "queries/s",
                 "note": "one batch of Python int lists (the reference's lpm_insert argument type) through "
                         "DeviceStore.match_lists: list -> int32 conversion and PCIe inside the timed call"}

    peak, peak_kind = peaks()
    traffic = None
    try:  # DRAM bytes per K1 launch from the committed ncu capture of this command (profiles/traffic.json)
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tr = json.load(fh).get("k_walk:c4")
        if tr and args.sessions == 10_000 and args.hist == 32_768 and args.queries == 4096:
            traffic = tr["dram_bytes_per_launch"]
    except Exception:
        pass
    # Consecutive batches overlap on two streams, so per-launch event intervals include
    # time shared with the neighbouring batch; the kernel time charged to one batch is
    # the timed region divided by the batches in it (an upper bound on K1's own time).
    k_avg = elapsed / args.steps
    achieved = alg_bytes / k_avg / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": c4_config(args, world, mixed),
        "tokens_compared_per_s": toks_per_s,
        "alg_GBps": world * alg_bytes * args.steps / elapsed / 1e9,
        "roofline": {"bound": "hbm", "kernel": "k_walk_tma", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_kind": peak_kind, "frac_of_8TBps": achieved / 8000.0,
                     "alg_bytes_per_launch": alg_bytes, "kernel_ms_avg": k_avg * 1e3, "traffic": traffic,
                     "traffic_source": "profiles/traffic.json: dram__bytes_read.sum + dram__bytes_write.sum per k_walk_tma "
                                       "launch, ncu --set full of this command (profiles/r02_*)",
                     "kernel_time_basis": "timed region / batches (batches overlap on 2 streams)",
                     "event_ms_avg_per_launch": walk_ms / max(walk_n, 1),
                     "planner_ms_avg": plan_ms / max(plan_n, 1)},
        "e2e": {"value": e2e_value, "unit": "queries/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "hash_filter_ab": {"k1_ms_per_batch": k_avg * 1e3, "block_hash_ms_per_batch": hash_ms / max(hash_n, 1),
                           "hash_first_ms_per_batch_lower_bound": k_avg * 1e3 + hash_ms / max(hash_n, 1),
                           "query_words_hashed": nq,
                           "note": "tm_block_hashes over the batch's query buffer (what a hash-first filter computes "
                                   "before it can prune); an equal hash never proves a match, so the exact compare "
                                   "that follows reads the same 8 B per compared token: hash-first can only add time"},
        "gpu_launches": int(walk_n + plan_n),  # our kernels in the timed region (CUDA-event bracketed)
        "timing": ("CUDA events on the launching stream around K back-to-back steps, enqueued behind a "
                   "device-side spin gate (host launch jitter excluded); max over ranks"
                   if os.environ.get("BENCH_GATE", "1") != "0" else
                   "CUDA events on the launching stream around K steps as launched; max over ranks"),
        "clocks": clk.summary(),
    }
    if lists:
        line["e2e_python_lists"] = lists
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        n, dt, res = cpu_port_bench_reuse(wl, cores)
        n, dt2, res = cpu_port_bench_reuse(wl, cores)
        dt = min(dt, dt2)
        assert np.array_equal(res[0], m), "CPU port disagrees with the GPU"
        line["cpu_baseline"] = {"value": n / dt, "unit": "queries/s", "cores": cores, "kind": "port",
                                "sample": f"full c4 batch ({n} queries), best of 2, C radix-tree restatement "
                                          f"(oracle/radix_oracle.c), {cores} threads"}
        if args.sessions >= 1000 and not args.mixed:
            hist_of, qlist = c4_hist_sampler(wl)
            line["reference_unmodified"] = reference_match_sample(hist_of, qlist)
    store.close()
    _cpu_store.clear()
    torch.cuda.set_stream(torch.cuda.default_stream(dev))
    return line


# ------------------------------------------------------------------------- c1-c3 (N = 1)

def measure_config(cfg, reps=3, with_cpu=True):
    """Record (K2 = k_record_tma, one launch), export (K3), NDJSON and - c3 - the
    include_partials export on one BASELINE config, device time (CUDA events around the
    launches) and call time (host arrays through the C ABI), with rooflines."""
    import torch

    from paper_2508_11553_b200 import DeviceStore
    from workloads import RecordWorkload

    peak, _ = peaks()
    wl = RecordWorkload(cfg)
    sids, tok, off, roff, rs, ro, rv = wl.packed()
    lens = np.diff(off)
    pad = (lens + 31) // 32 * 32
    aoff = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(pad, out=aoff[1:])
    atok = np.zeros(int(aoff[-1]), np.int32)
    for k in range(len(lens)):
        atok[aoff[k]: aoff[k] + lens[k]] = tok[off[k]: off[k + 1]]
    dtok = torch.from_numpy(atok).cuda()
    n_rec = len(lens)
    store = DeviceStore(0, arena_words=(2 * reps + 3) * int(aoff[-1]) + (1 << 22), row_capacity=(2 * reps + 3) * n_rec + 64,
                        run_capacity=(2 * reps + 3) * len(rs) + 64, session_capacity=(2 * reps + 3) * wl.n_sessions + 16)
    store.profile_begin(reserve=64)
    best: dict = {}

    def keep(k, v):
        best[k] = min(best.get(k, v), v)

    rng = np.random.default_rng(20251021)
    paused = np.sort(rng.choice(wl.n_sessions, wl.n_sessions // 10, replace=False)) if cfg == 3 else None
    for rep in range(reps + 1):
        smap = [store.new_session() for _ in range(wl.n_sessions)]
        g_sids = np.asarray([smap[s] for s in sids], np.int32)
        torch.cuda.synchronize()
        store.profile_begin()
        t0 = time.perf_counter()
        r = store.record_device(g_sids, dtok, aoff[:-1], lens, roff, rs, ro, rv)
        t_dev_call = time.perf_counter() - t0
        k2_ms, _ = store.profile_end("commit")
        cp_ms, _ = store.profile_end("record_copy")
        # the same records through the host-array call (PCIe inside), into fresh sessions
        smap2 = [store.new_session() for _ in range(wl.n_sessions)]
        g2 = np.asarray([smap2[s] for s in sids], np.int32)
        t0 = time.perf_counter()
        store.record_packed(g2, tok, off[:-1], lens, roff, rs, ro, rv)
        t_call = time.perf_counter() - t0
        rows = np.asarray(r.row, np.int64) if cfg != 1 else np.asarray(store.session_rows(smap[0], "lex"), np.int64)
        n_out = int(store.rows_total(rows))
        torch.cuda.synchronize()
        store.profile_begin()
        t0 = time.perf_counter()
        p = store.export_device(rows)
        torch.cuda.synchronize()
        t_exp_dev = time.perf_counter() - t0
        ex_ms, _ = store.profile_end("export")
        t0 = time.perf_counter()
        store.export(rows, total=n_out)
        t_exp_host = time.perf_counter() - t0
        t0 = time.perf_counter()
        store.export(rows, total=n_out, pinned=True)
        t_exp_pin = time.perf_counter() - t0
        names = [f"sess-{int(s)}" for s in sids] if cfg != 1 else ["sess-0"] * len(rows)
        t0 = time.perf_counter()
        text = store.export_ndjson(rows, names, as_array=True)
        t_json = time.perf_counter() - t0
        t0 = time.perf_counter()
        store.export_ndjson(rows, names, as_array=True, pinned=True)
        t_json_pin = time.perf_counter() - t0
        part = None
        if cfg == 3:  # 10 % of the sessions paused inside turn 2: completed rows + partials
            keep_rows, host_rows = [], []
            pset = set(paused.tolist())
            for s in range(wl.n_sessions):
                keep_rows.append(int(r.row[2 * s]))
                if s in pset:
                    t2 = wl.seqs[2 * s + 1]
                    k = wl.split[s]
                    host_rows.append((t2[: 2560 + k], 2560, 0, [0] * k))
                else:
                    keep_rows.append(int(r.row[2 * s + 1]))
            torch.cuda.synchronize()
            store.profile_begin()
            t0 = time.perf_counter()
            pp = store.export_device_with_host_rows(keep_rows, host_rows)
            torch.cuda.synchronize()
            t_part = time.perf_counter() - t0
            part_ms, _ = store.profile_end("export")
            part = (t_part, part_ms, int(pp.offsets[-1]), len(keep_rows) + len(host_rows),
                    sum(len(h[0]) for h in host_rows))
        del p
        if rep == 0:
            continue  # warm-up
        keep("k2_ms", k2_ms + cp_ms)
        keep("k_record_ms", k2_ms)
        keep("copy_ms", cp_ms)
        keep("t_dev_call", t_dev_call)
        keep("t_call", t_call)
        keep("ex_ms", ex_ms)
        keep("t_exp_dev", t_exp_dev)
        keep("t_exp_host", t_exp_host)
        keep("t_exp_pin", t_exp_pin)
        keep("t_json", t_json)
        keep("t_json_pin", t_json_pin)
        if part:
            keep("t_part", part[0])
            keep("part_ms", part[1])
    m = r.matched.astype(np.int64)
    # |parent| per record: lengths of each session's rows by local ordinal (rows are new in order)
    by_local: dict = {}
    plen = np.zeros(n_rec, np.int64)
    for k in range(n_rec):
        rows_s = by_local.setdefault(int(sids[k]), [])
        if r.parent_local[k] >= 0:
            plen[k] = rows_s[int(r.parent_local[k])]
        if int(r.local[k]) == len(rows_s):
            rows_s.append(int(lens[k]))
    cq = np.where(r.parent_local >= 0, np.minimum(np.minimum(m + 1, lens), plen), 0)
    novel = (lens - m).astype(np.float64)
    rec_bytes = float((8 * cq + 8 * novel).sum())
    exp_bytes = 13.0 * n_out + 8.0 * len(rows)

    def roof(nbytes, ms, kernel):
        a = nbytes / ms / 1e6
        return {"bound": "hbm", "kernel": kernel, "achieved": a, "peak": peak, "unit": "GB/s", "frac": a / peak,
                "alg_bytes": nbytes}

    out = {
        "records": n_rec, "sessions": wl.n_sessions, "record_tokens": int(lens.sum()), "novel_tokens": int(novel.sum()),
        "record": {"device_ms": best["k2_ms"], "k_record_ms": best["k_record_ms"], "k_record_copy_ms": best["copy_ms"],
                   "records_per_s_device": n_rec / best["k2_ms"] * 1e3,
                   "call_ms_device_tokens": 1e3 * best["t_dev_call"], "call_ms_host_arrays": 1e3 * best["t_call"],
                   "records_per_s_call": n_rec / best["t_call"],
                   "roofline": roof(rec_bytes, best["k2_ms"], "k_record_tma")},
        "export": {"rows": int(len(rows)), "tokens": n_out, "device_ms": best["ex_ms"],
                   "call_ms_device_out": 1e3 * best["t_exp_dev"], "call_ms_host_out": 1e3 * best["t_exp_host"],
                   "host_GBps": 9.0 * n_out / best["t_exp_host"] / 1e9,
                   "call_ms_host_pinned_out": 1e3 * best["t_exp_pin"],
                   "host_pinned_GBps": 9.0 * n_out / best["t_exp_pin"] / 1e9,
                   "roofline": roof(exp_bytes, best["ex_ms"], "k_export_plan + k_export_tma")},
        "ndjson": {"call_ms": 1e3 * best["t_json"], "bytes": int(len(text)), "tokens_per_s": n_out / best["t_json"],
                   "call_ms_pinned_out": 1e3 * best["t_json_pin"], "pinned_GBps": len(text) / best["t_json_pin"] / 1e9},
    }
    if cfg == 3:
        _, _, ptok, prow, htok = part
        out["export_include_partials"] = {
            "rows": prow, "tokens": ptok, "partial_rows": len(paused), "partial_tokens": htok,
            "device_ms": best["part_ms"], "call_ms": 1e3 * best["t_part"],
            "roofline": roof(13.0 * ptok + 8.0 * prow, best["part_ms"], "k_export_tma + k_fill_host_rows"),
            "note": "10 % of the sessions paused inside turn 2: their turn-1 rows from the store plus the open "
                    "request (input + first leg) assembled on the GPU (trajectory.py:317-340)"}
    store.close()
    if with_cpu:
        from tools.refbench import time_port_records, time_reference_records

        cores = os.cpu_count() or 1
        port, _ = time_port_records(wl, cores)
        out["cpu_baseline"] = {"value": port["records_per_s"], "unit": "records/s", "cores": cores, "kind": "port",
                               "export_tokens_per_s": port["export_tokens_per_s"],
                               "sample": f"all {n_rec} records then every row exported, C restatement "
                                         f"(oracle/radix_oracle.c), {cores} threads"}
        n1 = {1: 1, 2: 4, 3: 40}[cfg]
        refd = time_reference_records(wl, n1, n1 * cores)
        if refd is not None:
            out["reference_unmodified"] = dict(refd, unit="records/s and tokens/s", kind="reference",
                                               sample="sessions of this config recorded in order (lpm_insert), then "
                                                      "extract() and trajectory_to_line, unmodified rolloutlab from "
                                                      "baseline/_ref: one process, and a pool over all cores")
    return out


# ------------------------------------------------------------------------------------- c5

def measure_config_shards(cfg, rank, world, local, dev, reps=3):
    """N > 1: configs 2 / 3 as weak-scaling shards - every rank records and exports its own
    copy of the config's sessions (sessions are independent) into its own
    store; device time of K2 and K3 (CUDA events), max over ranks; aggregate rates."""
    import torch
    import torch.distributed as dist

    from paper_2508_11553_b200 import DeviceStore
    from workloads import SEED0, RecordWorkload

    peak, _ = peaks()
    wl = RecordWorkload(cfg, seed=SEED0 + 100 * cfg + rank)
    sids, tok, off, roff, rs, ro, rv = wl.packed()
    lens = np.diff(off)
    pad = (lens + 31) // 32 * 32
    aoff = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(pad, out=aoff[1:])
    atok = np.zeros(int(aoff[-1]), np.int32)
    for k in range(len(lens)):
        atok[aoff[k]: aoff[k] + lens[k]] = tok[off[k]: off[k + 1]]
    dtok = torch.from_numpy(atok).to(dev)
    n_rec = len(lens)
    store = DeviceStore(local, arena_words=(reps + 2) * int(aoff[-1]) + (1 << 22), row_capacity=(reps + 2) * n_rec + 64,
                        run_capacity=(reps + 2) * len(rs) + 64, session_capacity=(reps + 2) * wl.n_sessions + 16)
    store.profile_begin(reserve=64)
    best_k2 = best_ex = float("inf")
    r = rows = None
    n_out = 0
    for _ in range(reps + 1):
        smap = [store.new_session() for _ in range(wl.n_sessions)]
        g = np.asarray([smap[x] for x in sids], np.int32)
        torch.cuda.synchronize()
        store.profile_begin()
        r = store.record_device(g, dtok, aoff[:-1], lens, roff, rs, ro, rv)
        k2, _ = store.profile_end("commit")
        rows = np.asarray(r.row, np.int64)
        n_out = int(store.rows_total(rows))
        torch.cuda.synchronize()
        store.profile_begin()
        store.export_device(rows)
        torch.cuda.synchronize()
        ex, _ = store.profile_end("export")
        best_k2, best_ex = min(best_k2, k2), min(best_ex, ex)
    m = r.matched.astype(np.int64)
    cq = np.where(r.parent_local >= 0, np.minimum(m + 1, lens), 0)  # (upper bound on |parent|: the own length)
    rec_bytes = float((8 * cq + 8 * (lens - m)).sum())
    exp_bytes = 13.0 * n_out + 8.0 * len(rows)
    t = torch.tensor([best_k2, best_ex], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    k2_max, ex_max = float(t[0]), float(t[1])
    store.close()
    return {"workload": f"c{cfg} x {world} shards (every rank its own {wl.n_sessions} sessions)",
            "records_per_s": world * n_rec / k2_max * 1e3, "record_ms_max_over_ranks": k2_max,
            "record_frac_per_rank": rec_bytes / k2_max / 1e6 / peak,
            "export_tokens_per_s": world * n_out / ex_max * 1e3, "export_ms_max_over_ranks": ex_max,
            "export_frac_per_rank": exp_bytes / ex_max / 1e6 / peak, "peak_GBps": peak,
            "timing": "CUDA events around K2 / K3 on each rank (best of reps), max over ranks"}


def measure_c5(args, steps, warmup):
    """Config 5: 1M sessions (log-uniform 1k-128k tokens) sharded by session hash; every
    rank originates 4096 queries for sessions owned anywhere; Router.match routes them
    (fused P2P K1 over NVLink).  value = all ranks' queries / max-over-ranks time."""
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    own_pg = False
    if not dist.is_initialized():
        own_pg = True
        if world == 1 and "MASTER_ADDR" not in os.environ:  # plain `python bench.py` (under torchrun: env://)
            dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29533", rank=0, world_size=1, device_id=dev)
        else:
            dist.init_process_group("nccl", device_id=dev)
    from paper_2508_11553_b200 import DeviceStore
    from paper_2508_11553_b200.routing import Router
    from workloads import C5Workload

    wl = C5Workload(args.c5_sessions, nranks=world, rank=rank, n_queries=args.queries)
    owned_tokens = int(((wl.lens[wl.owned] + 31) // 32 * 32).sum())
    store = DeviceStore(local, arena_words=owned_tokens + (1 << 22), row_capacity=len(wl.owned) + 64,
                        run_capacity=16 * len(wl.owned) + 64, session_capacity=len(wl.owned) + 16)
    t0 = time.perf_counter()
    wl.build_shard(store)
    build_s = time.perf_counter() - t0
    log(f"rank {rank}: c5 shard ({len(wl.owned)} sessions, {owned_tokens * 4 / 1e9:.1f} GB) built in {build_s:.1f} s")
    tok_need = torch.tensor([int(wl.q_off[-1])], device=dev)
    dist.all_reduce(tok_need, op=dist.ReduceOp.MAX)
    push = args.routing == "push"
    router = Router(store, dist.group.WORLD, n_max=args.queries, tokens_max=int(tok_need.item()), g2l=wl.g2l,
                    push=push)
    wl.fill_queries(router)
    routers = [router]
    if args.pipeline and args.routing in ("fused", "push"):
        # a second region: the next batch is bucketed + packed while this one is matched
        routers.append(Router(store, dist.group.WORLD, n_max=args.queries, tokens_max=int(tok_need.item()),
                              g2l=wl.g2l, push=push))
        wl.fill_queries(routers[1])
    torch.cuda.synchronize()
    if len(routers) > 1:
        from paper_2508_11553_b200.routing import match_pipelined

        side = torch.cuda.Stream(dev)
        defer = os.environ.get("BENCH_DEFER_DONE", "0") == "1"  # A/B knob: done waits on their own stream (measured neutral)
        run_batches = lambda k: match_pipelined(routers, wl.n_queries, k, side, defer_done=defer)  # noqa: E731
    else:
        route = {"fused": router.match, "push": router.match,
                 "fused-nccl-barrier": lambda n: router.match(n, sync="nccl"),
                 "nccl": router.match_nccl}[args.routing]

        def run_batches(k):
            for _ in range(k):
                route(wl.n_queries)
    run_batches(warmup)
    torch.cuda.synchronize()
    m = np.concatenate([r.out_matched[: wl.n_queries].cpu().numpy() for r in routers])
    bad = np.flatnonzero(m != np.tile(wl.q_depth, len(routers))) % wl.n_queries
    if len(bad):
        print(f"rank {rank}: {len(bad)} mismatches, e.g.", [(int(i), int(m[i]), int(wl.q_depth[i])) for i in bad[:8]],
              file=sys.stderr)
    assert len(bad) == 0, "routed matched length != constructed depth"
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.current_stream(dev)
    dist.barrier()
    torch.cuda.synchronize()
    store.profile_begin(reserve=steps + 64)
    with Clocks(local) as clk:
        time.sleep(0.3)
        t_wall = time.perf_counter()
        # no device-side gate here (unlike c4): routed batches are device-bound (host enqueue
        # ~50 us per batch vs 280-380 us on the GPU) and a per-rank gate only adds the ranks'
        # gate-end skew to the routed barriers (profiles/r01_bench_c5_gate_check.txt)
        e0.record(stream)
        t_enq = time.perf_counter()
        run_batches(steps)
        e1.record(stream)
        t_enq = time.perf_counter() - t_enq
        torch.cuda.synchronize()
        walk_ms, walk_n = store.profile_end("walk")
        phase_ms = {k: store.profile_end(k) for k in ("route", "route_pack", "route_wait")}
        # keep the clocks sampler running for >= 1 s under load; every rank must make the
        # same number of (collective) routed calls, so the count is agreed on first
        left = torch.tensor([max(0.0, 1.0 - (time.perf_counter() - t_wall))], device=dev, dtype=torch.float64)
        per = torch.tensor([e0.elapsed_time(e1) / 1e3 / steps], device=dev, dtype=torch.float64)
        dist.all_reduce(left, op=dist.ReduceOp.MAX)
        dist.all_reduce(per, op=dist.ReduceOp.MAX)
        run_batches(int(float(left.item()) / max(float(per.item()), 1e-6)) + 1)
        torch.cuda.synchronize()
    elapsed = e0.elapsed_time(e1) / 1e3
    log(f"rank {rank}: c5 device-timed region {1e3 * elapsed:.3f} ms for {steps} routed batches "
        f"(host enqueue {1e3 * t_enq:.3f} ms)")
    t = torch.tensor([elapsed], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed = float(t.item())
    L = wl.lens[wl.q_g]
    cq = np.minimum(np.minimum(wl.q_depth + 1, wl.q_len), L)
    remote = wl.owner[wl.q_g] != rank
    pushed = float(((wl.q_len[remote] + 31) // 32 * 32).sum())  # push: whole queries cross, not compared prefixes
    stats = torch.tensor([float(cq.sum()), float(cq[remote].sum()), float(remote.mean()), pushed], device=dev,
                         dtype=torch.float64)
    dist.all_reduce(stats)
    toks, remote_toks, xfrac = float(stats[0]), float(stats[1]), float(stats[2]) / world
    if push and world > 1:
        remote_toks = float(stats[3])
    value = world * wl.n_queries * steps / elapsed
    wire_b = 2.25 if (world > 1 and args.routing != "nccl" and os.environ.get("TM_ROUTE_PACK", "1") != "0") else 4.0
    peak, peak_kind = peaks()
    per_gpu_alg = 8.0 * toks / world  # HBM+link bytes per rank per batch (average)
    line = {
        "metric": METRIC_C5, "value": value, "unit": "queries/s", "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": 1e3 * elapsed / steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": c5_config(args, world),
        "cross_shard_frac": xfrac, "shard_build_s": build_s, "arena_GB_per_rank": owned_tokens * 4 / 1e9,
        "tokens_compared_per_s": toks * steps / elapsed,
        "alg_GBps_per_rank": per_gpu_alg * steps / elapsed / 1e9,
        "nvlink_query_GBps_per_rank": 4.0 * remote_toks / world * steps / elapsed / 1e9,
        # bytes that actually cross the links: remote queries move as 18-bit planes (2.25 B per
        # compared position) unless the exchange is the NCCL baseline (int32)
        "nvlink_wire_bytes_per_position": wire_b,
        "nvlink_wire_GBps_per_rank": wire_b * remote_toks / world * steps / elapsed / 1e9,
        "routed_walk_ms_avg_rank0": walk_ms / max(walk_n, 1),
        "phase_ms_avg_rank0": {k: (ms / n if n else 0.0) for k, (ms, n) in phase_ms.items()},
        "roofline": {"bound": "nvlink" if world > 1 else "hbm", "kernel": "k_walk_routed",
                     "achieved": (wire_b * remote_toks / world if world > 1 else per_gpu_alg) * steps / elapsed / 1e9,
                     "peak": LINK_PEAK if world > 1 else peak, "unit": "GB/s",
                     "frac": ((wire_b * remote_toks / world) / LINK_PEAK if world > 1 else per_gpu_alg / peak)
                     * steps / elapsed / 1e9,
                     "peak_kind": "measured SM peer reads per GPU with both directions busy (tools/p2p_probe)"
                     if world > 1 else peak_kind,
                     "hbm_frac": per_gpu_alg * steps / elapsed / 1e9 / peak,
                     "traffic": None,
                     "note": "N>1: achieved = bytes on the wire (remote compared positions x nvlink_wire_bytes_per_"
                             "position) over the whole step; history bytes come from local HBM (tools/p2p_probe: SM "
                             "peer reads 780 GB/s one direction, 670 GB/s per GPU both directions at once)"},
        # ours per batch: k_route + k_walk_routed (+ k_route_pack with peers, + k_route_arrive +
        # k_route_wait_done with device barriers)
        "gpu_launches": steps * ((4 if args.routing in ("fused", "push") else 2) + (1 if world > 1 and
                                                                        args.routing != "nccl" else 0)),
        "clocks": clk.summary(),
        "timing": "CUDA events on the launching stream around K routed batches; max over ranks",
    }
    for r in routers:
        r.close()
    store.close()
    if own_pg:
        dist.destroy_process_group()
    return line


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    workload = args.workload or ("c5" if world > 1 else "c4")
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    if workload == "c5":
        line = measure_c5(args, args.steps, args.warmup)
        if world > 1:  # the host-routed weak-scaling shards beside it (every rank its own c4 shard)
            line["c4_shards"] = {k: v for k, v in measure_c4(args, rank, world, local, dev).items()
                                 if k in ("value", "ms_per_step", "config", "roofline", "e2e", "tokens_compared_per_s")}
            if not args.no_configs:  # record / export of configs 2 and 3 as shards
                line["config_shards"] = {f"c{c}": measure_config_shards(c, rank, world, local, dev) for c in (2, 3)}
    else:
        line = measure_c4(args, rank, world, local, dev)
        if world == 1 and not args.no_configs:
            line["configs"] = {}
            for cfg in (1, 2, 3):
                t0 = time.perf_counter()
                line["configs"][f"c{cfg}"] = measure_config(cfg, with_cpu=not args.no_cpu)
                log(f"c{cfg} record/export measured in {time.perf_counter() - t0:.1f} s")
        if world == 1 and not args.no_c5:
            c5 = measure_c5(args, args.steps, args.warmup)
            line["c5_routed"] = {k: c5[k] for k in ("value", "unit", "ms_per_step", "config", "roofline",
                                                    "tokens_compared_per_s", "shard_build_s", "arena_GB_per_rank")}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
