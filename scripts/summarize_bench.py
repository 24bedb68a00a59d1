"""One row per bench JSON line found under profiles/ (the evidence behind the
DESIGN.md §8 table): config, parallelism, samples/s, step roofline, GEMM
roofline fraction, e2e, clocks.

    python scripts/summarize_bench.py [profiles/r01]
"""
import glob
import json
import os
import sys


def rows(root):
    for path in sorted(glob.glob(os.path.join(root, "**", "*.log"), recursive=True) +
                       glob.glob(os.path.join(root, "*.json"))):
        try:
            lines = [ln for ln in open(path) if ln.startswith("{") and '"metric"' in ln]
        except (OSError, UnicodeDecodeError):
            continue
        for ln in lines:
            try:
                d = json.loads(ln)
            except json.JSONDecodeError:
                continue
            if d.get("impl") == "reference" or "value" not in d:
                continue
            c = d.get("config", {})
            yield {"file": os.path.relpath(path, root), "config": c.get("workload", "")[:2],
                   "par": c.get("parallelism"), "split": c.get("stage_layers") or c.get("last_stage_layers"),
                   "head": c.get("head_place", "last_stage"), "samples_s": round(d["value"], 2),
                   "step_roofline": round(d.get("step_roofline", {}).get("frac", 0), 3),
                   "gemm_frac": round((d.get("roofline") or {}).get("frac", 0), 3),
                   "e2e": round(d["e2e"]["value"], 2) if d.get("e2e") else None,
                   "sm_mhz": (d.get("clocks") or {}).get("sm_mhz")}


def main():
    root = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "profiles", "r01")
    keys = ["file", "config", "par", "split", "head", "samples_s", "step_roofline", "gemm_frac", "e2e", "sm_mhz"]
    print(" | ".join(keys))
    for r in rows(root):
        print(" | ".join(str(r[k]) for k in keys))


if __name__ == "__main__":
    main()
