"""Print the compact summary of a bench JSON line read from stdin (tag in argv[1])."""
import json
import sys

d = json.loads(sys.stdin.read())
print(sys.argv[1] if len(sys.argv) > 1 else "", round(d["ms_per_step"], 2), round(d.get("value", 0)),
      {k: round(v, 2) for k, v in (d.get("kernel_ms") or {}).items()})
