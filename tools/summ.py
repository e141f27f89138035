"""Print a one-line summary of a bench.py JSON line read from stdin."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    tag = sys.argv[1] if len(sys.argv) > 1 else ""
    print(tag, "value", d.get("value"), d.get("unit"), "us/layer", d.get("us_per_layer"),
          "frac", (d.get("roofline") or {}).get("frac"), "e2e", (d.get("e2e") or {}).get("value"),
          "clocks", d.get("clocks"))
