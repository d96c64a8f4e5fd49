"""Print the headline numbers of a bench.py JSON line (last line of the file)."""
import json
import sys
d = json.loads(open(sys.argv[1]).read().strip().split("\n")[-1])
tag = sys.argv[2] if len(sys.argv) > 2 else ""
print(tag, round(d["value"], 2), round(d["ms_per_step"], 3),
      {k: (round(v["ms_per_call"], 4), round(v.get("GB_per_s") or 0)) for k, v in d["kernels"].items() if v["launches"]})
