"""Per-phase trace (TM_TRACE_CALLS) of the c2 / c3 record call with device tokens."""
import os
import sys

import numpy as np

os.environ.setdefault("TM_TRACE_CALLS", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import torch

    from paper_2508_11553_b200 import DeviceStore
    from workloads import RecordWorkload

    for cfg in (3, 2):
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
        store = DeviceStore(0, arena_words=5 * int(aoff[-1]) + (1 << 22), row_capacity=5 * len(lens) + 64,
                            run_capacity=5 * len(rs) + 64, session_capacity=5 * wl.n_sessions + 16)
        for rep in range(4):
            smap = [store.new_session() for _ in range(wl.n_sessions)]
            g = np.asarray([smap[s] for s in sids], np.int32)
            print(f"c{cfg} rep {rep}", file=sys.stderr, flush=True)
            store.record_device(g, dtok, aoff[:-1], lens, roff, rs, ro, rv)
        store.close()


if __name__ == "__main__":
    main()
