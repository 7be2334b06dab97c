"""One-line summary of a bench.py JSON line on stdin (tuning runs): value, clocks, solve breakdown."""
import json
import sys

tag = " ".join(sys.argv[1:])
j = json.loads(sys.stdin.read().strip().splitlines()[-1])
s = j.get("solve") or {}
it = s.get("inner") or 1
print(f"{tag}: {j['value'] * 1e3:.2f} ms/step, sm {j.get('clocks', {}).get('sm_mhz')} MHz, outer {s.get('outer')}, "
      f"inner {s.get('inner')}, pcg {s.get('t_pcg_ms', 0):.2f} ms ({s.get('t_pcg_ms', 0) / it * 1e3:.2f} us/it), "
      f"sketch {s.get('t_sketch_ms', 0):.2f} ms, other {s.get('t_other_ms', 0):.2f} ms")
