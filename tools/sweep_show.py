"""Print the c5 bench lines of a knob sweep (gpurun_out/sw_*.json)."""
import glob
import json
import sys

for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sw_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        ph = {k: round(v, 3) for k, v in d.get("phase_ms_avg_rank0", {}).items()}
        print(f"{f:40s} {d['value'] / 1e6:6.2f} M q/s  {d['ms_per_step']:.3f} ms  walk {d['routed_walk_ms_avg_rank0']:.3f}"
              f"  {ph}  frac {d['roofline']['frac']:.3f}")
    except Exception as e:  # noqa: BLE001
        print(f, "failed", e)
