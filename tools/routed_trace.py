"""Summarise TM_ROUTED_TRACE files (tools/gpurun/trace_n2.sh): per routed call, the link
bytes in flight over time (remote items' compared positions x 2.25 B spread over their
[start, end) intervals), the walk span, the busy-CTA profile and the tail."""
import glob
import sys

import numpy as np


def calls(path):
    raw = np.fromfile(path, np.int64)
    i = 0
    while i < len(raw):
        n, ep = int(raw[i]), int(raw[i + 1])
        rec = raw[i + 2: i + 2 + 4 * n].reshape(n, 4)
        i += 2 + 4 * n
        yield ep, rec


def main():
    for path in sorted(glob.glob(sys.argv[1] + ".*")):
        cs = list(calls(path))
        for ep, rec in cs[-2:]:
            rec = rec[rec[:, 1] > 0]
            t0 = rec[:, 0].min()
            s, e = (rec[:, 0] - t0) / 1e3, (rec[:, 1] - t0) / 1e3  # us
            L = rec[:, 2] & ((1 << 40) - 1)
            remote = (rec[:, 2] >> 40) & 1
            m = rec[:, 2] >> 41
            cmp_ = np.minimum(m + 1, L)
            span = e.max()
            rb = (cmp_ * 2.25 * remote).sum()
            lb = (cmp_ * 8 * (1 - remote)).sum() + (cmp_ * 4 * remote).sum()
            dur = e - s
            # link-bytes rate profile in 10 us bins
            bins = np.arange(0, span + 10, 10)
            rate = np.zeros(len(bins))
            for a, b, by in zip(s[remote == 1], e[remote == 1], (cmp_ * 2.25)[remote == 1]):
                i0, i1 = int(a // 10), int(b // 10)
                for k in range(i0, i1 + 1):
                    lo, hi = max(a, bins[k]), min(b, bins[k] + 10)
                    if hi > lo:
                        rate[k] += by * (hi - lo) / max(b - a, 1e-9)
            rate = rate / 10e-6 / 1e9  # GB/s
            busy = [int(((s <= t) & (e > t)).sum()) for t in bins]
            busy_r = [int(((s <= t) & (e > t) & (remote == 1)).sum()) for t in bins]
            hrate = np.zeros(len(bins))
            hb = np.where(remote == 1, cmp_ * 4.0, cmp_ * 8.0)
            for a, b, by in zip(s, e, hb):
                i0, i1 = int(a // 10), int(b // 10)
                for k in range(i0, i1 + 1):
                    lo, hi = max(a, bins[k]), min(b, bins[k] + 10)
                    if hi > lo:
                        hrate[k] += by * (hi - lo) / max(b - a, 1e-9)
            hrate = hrate / 10e-6 / 1e12  # TB/s
            # start time of items by length class
            for lab, sel in (("remote", remote == 1), ("local", remote == 0)):
                order = np.argsort(s[sel])
                Ls = cmp_[sel][order]
                print(f"  {lab} items: last start {s[sel].max():.1f} us; compared length of the last 20 started: "
                      f"{Ls[-20:].tolist()}; longest ending item ends {e[sel][np.argmax(cmp_[sel])]:.1f}")
            print(f"{path} epoch {ep}: {len(rec)} items ({int(remote.sum())} remote), span {span:.1f} us, "
                  f"link {rb / 1e6:.1f} MB -> {rb / span / 1e3:.0f} GB/s avg, HBM {lb / 1e6:.0f} MB")
            print("  remote item us: p50 %.1f p90 %.1f max %.1f; per-item us per KB link %.3f" % (
                np.percentile(dur[remote == 1], 50), np.percentile(dur[remote == 1], 90), dur[remote == 1].max(),
                np.median(dur[remote == 1] / np.maximum(cmp_[remote == 1] * 2.25 / 1024, 1e-9))))
            print("  local  item us: p50 %.1f p90 %.1f max %.1f" % (
                np.percentile(dur[remote == 0], 50), np.percentile(dur[remote == 0], 90), dur[remote == 0].max()))
            print("  short items (<2k compared): n=%d mean us %.1f" % (
                int((cmp_ < 2048).sum()), dur[cmp_ < 2048].mean() if (cmp_ < 2048).any() else 0))
            print("  t(us) : " + " ".join(f"{b:5.0f}" for b in bins[::2]))
            print("  GB/s  : " + " ".join(f"{r:5.0f}" for r in rate[::2]))
            print("  busy  : " + " ".join(f"{b:5d}" for b in busy[::2]))
            print("  busyR : " + " ".join(f"{b:5d}" for b in busy_r[::2]))
            print("  HBM TB/s: " + " ".join(f"{r:5.2f}" for r in hrate[::2]))


if __name__ == "__main__":
    main()
