"""Print kernel ms / roofline fraction of every bench line in a gpurun_out dir."""
import glob
import json
import os
import sys

for f in sorted(glob.glob(os.path.join(sys.argv[1], "*.json"))):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]
        print(f"{os.path.basename(f):50s} step {d['ms_per_step']:.4f} kern {r['kernel_ms']:.4f} "
              f"frac {r['frac']:.3f} sm {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
    except Exception as e:  # noqa: BLE001
        err = f[:-5] + ".err"
        tail = open(err).read().strip().splitlines()[-2:] if os.path.exists(err) else []
        print(f"{os.path.basename(f):50s} FAILED {e!r} {tail}")
