"""Print the headline fields of a bench.py JSON line: python tools/bench_line.py FILE [tag]"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
tag = sys.argv[2] if len(sys.argv) > 2 else ""
r = d.get("roofline", {})
print(tag, "s/epoch", d.get("value"), "ms/batch", d.get("ms_per_step"), "e2e", d.get("e2e", {}).get("value"),
      "pass_us", r.get("kernel_us"), "prep_us", r.get("prep_us"), "frac", r.get("frac"))
