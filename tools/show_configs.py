"""Print the per-phase breakdown of tools/run_configs.py JSON lines (stdin)."""
import json
import sys

for line in sys.stdin:
    r = json.loads(line)
    ph = {k: (round(v["GBs"]), round(v["ns"] / 1e3, 1)) for k, v in r.get("phases", {}).items()}
    print(r["config"], "ms/step", round(r["ms_per_step"], 3), "valid", r["valid_every_checked_step"],
          "phases (GB/s, us/step):", ph)
    print("   work/step:", {k: round(v, 1) for k, v in r.get("work_per_step", {}).items() if not k.startswith("t_")})
