"""Record (K1+K2) and export (K3) throughput on configs 1-3, next to the CPU port.

Not the driver's bench line (bench.py is); this measures the other hot-path kernels on
the BASELINE.json configs and prints one JSON object per measurement:

  python tools/bench_paths.py [--configs 1,2,3] [--reps 3]

Algorithmic bytes:
  record  8*c_q (match) + 4*(L-m) (read novel suffix) + 4*(L-m) (arena write)
  export  13 B per emitted token + 8 B per row offset
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    import torch

    from oracle.cport import CRadixStore
    from paper_2508_11553_b200 import DeviceStore
    from workloads import RecordWorkload

    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    cores = os.cpu_count() or 1
    for cfg in [int(c) for c in args.configs.split(",")]:
        wl = RecordWorkload(cfg)
        packed = wl.packed()
        sids, tok, off, roff, rs, ro, rv = packed
        lens = np.diff(off)
        # device-resident tokens with aligned offsets (the engine-produced case)
        pad = (lens + 31) // 32 * 32
        aoff = np.zeros(len(lens) + 1, np.int64)
        np.cumsum(pad, out=aoff[1:])
        atok = np.zeros(int(aoff[-1]), np.int32)
        for k in range(len(lens)):
            atok[aoff[k]: aoff[k] + lens[k]] = tok[off[k]: off[k + 1]]
        dtok = torch.from_numpy(atok).cuda()
        best = {}
        store = DeviceStore(0, arena_words=(args.reps + 2) * int(aoff[-1]) + (1 << 22),
                            row_capacity=(args.reps + 2) * len(lens) + 64, run_capacity=(args.reps + 2) * len(rs) + 64,
                            session_capacity=(args.reps + 2) * wl.n_sessions + 16)
        for rep in range(args.reps + 1):
            smap = [store.new_session() for _ in range(wl.n_sessions)]
            g_sids = np.asarray([smap[s] for s in sids], np.int32)
            torch.cuda.synchronize()
            store.profile_begin()
            t0 = time.perf_counter()
            r = store.record_device(g_sids, dtok, aoff[:-1], lens, roff, rs, ro, rv)
            t_rec = time.perf_counter() - t0
            walk_ms, walk_n = store.profile_end("walk")
            commit_ms, commit_n = store.profile_end("commit")
            copy_ms, _ = store.profile_end("record_copy")
            commit_ms += copy_ms
            rows = store.session_rows(smap[0], "insert") if cfg == 1 else r.row
            rows = np.asarray(rows, np.int64)
            n_out = int(store.rows_total(rows))
            store.profile_begin()
            t0 = time.perf_counter()
            p = store.export_device(rows)
            torch.cuda.synchronize()
            t_exp = time.perf_counter() - t0
            exp_ms, exp_n = store.profile_end("export")
            t0 = time.perf_counter()
            ph = store.export(rows)
            t_exp_host = time.perf_counter() - t0
            names = [f"sess-{int(sids[k])}" for k in range(len(rows))] if cfg != 1 else ["sess-0"] * len(rows)
            t0 = time.perf_counter()
            text = store.export_ndjson(rows, names, as_array=True)
            t_json = time.perf_counter() - t0
            if rep == 0:
                continue  # warm-up
            cur = dict(t_rec=t_rec, walk_ms=walk_ms, commit_ms=commit_ms, copy_ms=copy_ms, commit_n=commit_n, t_exp=t_exp,
                       exp_ms=exp_ms,
                       t_exp_host=t_exp_host, t_json=t_json)
            for k, v in cur.items():
                best[k] = min(best.get(k, v), v)
        store.close()
        m = r.matched
        novel = (lens - m).astype(np.float64)
        cq = np.minimum(m + 1, lens)  # compared tokens (parent length >= m+1 or the row end)
        rec_bytes = float((8 * cq + 8 * novel).sum())
        exp_bytes = 13.0 * n_out + 8.0 * len(rows)
        dev_rec_ms = best["commit_ms"]
        line = {
            "config": f"c{cfg}", "records": int(len(lens)), "sessions": int(wl.n_sessions),
            "record_tokens": int(lens.sum()), "novel_tokens": int(novel.sum()),
            "record": {"waves": int(np.bincount(sids).max()), "launches": int(best["commit_n"]), "k1_k2_ms": best["commit_ms"],
                       "k2_copy_ms": best["copy_ms"],
                       "device_ms": dev_rec_ms, "call_ms": 1e3 * best["t_rec"], "alg_bytes": rec_bytes,
                       "device_GBps": rec_bytes / dev_rec_ms / 1e6, "frac_of_peak": rec_bytes / dev_rec_ms / 1e6 / peak,
                       "records_per_s_call": len(lens) / best["t_rec"]},
            "export": {"rows": int(len(rows)), "tokens": n_out, "k3_ms": best["exp_ms"], "alg_bytes": exp_bytes,
                       "device_GBps": exp_bytes / best["exp_ms"] / 1e6,
                       "frac_of_peak": exp_bytes / best["exp_ms"] / 1e6 / peak,
                       "device_call_ms": 1e3 * best["t_exp"], "host_call_ms": 1e3 * best["t_exp_host"],
                       "host_tokens_per_s": n_out / best["t_exp_host"],
                       "ndjson_call_ms": 1e3 * best["t_json"], "ndjson_bytes": len(text),
                       "ndjson_tokens_per_s": n_out / best["t_json"]},
        }
        if not args.no_cpu:
            ora = CRadixStore()
            t0 = time.perf_counter()
            ora.insert_batch(*packed, nthreads=cores)
            t_cpu_rec = time.perf_counter() - t0
            t0 = time.perf_counter()
            n_exp = 0
            for s in range(min(wl.n_sessions, 200)):
                for k in ora.lex_rows(s):
                    n_exp += len(ora.export_row(s, int(k))[0])
            t_cpu_exp = time.perf_counter() - t0
            # reference-format JSON on the CPU (json.dumps, as trajectory_to_line does) for a sample
            import json as _json
            t0 = time.perf_counter()
            nj = 0
            for k in range(min(len(rows), 200)):
                a, b = ph.offsets[k], ph.offsets[k + 1]
                _json.dumps({"session_id": names[k], "tokens": ph.tokens[a:b].tolist(),
                             "loss_mask": ph.loss_mask[a:b].tolist(), "versions": ph.versions[a:b].tolist()},
                            separators=(",", ":"))
                nj += b - a
            t_cpu_json = time.perf_counter() - t0
            line["cpu_port"] = {"cores": cores, "record_s": t_cpu_rec, "records_per_s": len(lens) / t_cpu_rec,
                                "export_tokens_per_s": n_exp / t_cpu_exp,
                                "export_sample": f"{min(wl.n_sessions, 200)} sessions, 1 thread (ctypes per row)",
                                "json_dumps_tokens_per_s": nj / t_cpu_json}
            ora.close()
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
