"""Write profiles/traffic.json from an ncu --set full capture summary of fd_mode_kernel.

    python tools/traffic_from_ncu.py <summary.txt> <config id> <source text>
The summary is tools/ncu_summary.py output (one JSON object per captured launch, dram in
bytes).  bench.py reports the mean dram read+write bytes per launch as roofline.traffic.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path, cfg, src = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [json.loads(l) for l in open(path) if l.startswith("{")]
rows = [r for r in rows if "fd_mode" in r["kernel"] or "fd_time" in r["kernel"]]
assert rows and rows[0]["dram_unit"] in ("byte", "B"), rows[:1]
b = sum(r["dram_read"] + r["dram_write"] for r in rows) / len(rows)
out_path = os.path.join(ROOT, "profiles", "traffic.json")
data = json.load(open(out_path)) if os.path.exists(out_path) else {}
data[f"config{cfg}"] = {"bytes_per_launch": b, "launches": len(rows), "source": src}
json.dump(data, open(out_path, "w"), indent=1)
print(data)
