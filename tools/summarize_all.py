"""Table of every BASELINE config from the bench.py lines of one round
(gpurun_out/<tag>_all_<cfg>_<rule>.json, written by tools/round_evidence.sh).

    python tools/summarize_all.py r01b > profiles/r01b_all_configs.txt
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01b"
cfgs = ["c0", "c1", "c2", "c3", "c4p2", "c4p4", "c4p6"]
out = {}


def f(x, fmt):
    return format(x, fmt) if isinstance(x, (int, float)) and not (isinstance(x, float) and math.isnan(x)) else "-"


print(f"{'cfg':6s} {'rule':9s} {'EQP/s':>10s} {'step ms':>9s} {'bound':>6s} {'kern.roof':>9s} {'step-roof':>9s} "
      f"{'e2e EQP/s':>10s} {'CPU EQP/s':>10s} {'GPU/CPU':>8s} {'blocks ms':>9s} {'blk roof':>8s} {'launches':>8s}")
for rule in ("gauss", "reference"):
    for c in cfgs:
        p = os.path.join(ROOT, "gpurun_out", f"{tag}_all_{c}_{rule}.json")
        try:
            d = json.loads(open(p).read().strip().splitlines()[-1])
        except Exception as exc:
            print(f"{c:6s} {rule:9s} missing ({exc.__class__.__name__})")
            continue
        out[f"{c}_{rule}"] = d
        cpu = (d.get("cpu_baseline") or {}).get("value")
        blk = d.get("blocks") or {}
        roof = d.get("roofline") or {}
        e2e = (d.get("e2e") or {}).get("value")
        ratio = d["value"] / cpu if cpu else None
        print(f"{c:6s} {rule:9s} {d['value']:10.3e} {d['ms_per_step']:9.4f} {roof.get('bound', '-'):>6s} "
              f"{f(roof.get('frac'), '9.3f'):>9s} {f(d.get('step_roofline_frac'), '9.3f'):>9s} "
              f"{f(e2e, '10.3e'):>10s} {f(cpu, '10.3e'):>10s} {f(ratio, '8.0f'):>8s} "
              f"{f(blk.get('ms'), '9.3f'):>9s} {f(blk.get('roofline_frac'), '8.3f'):>8s} "
              f"{f(d.get('gpu_launches'), '8d'):>8s}")
with open(os.path.join(ROOT, "profiles", f"{tag}_all_configs.json"), "w") as fh:
    json.dump(out, fh, indent=1)
