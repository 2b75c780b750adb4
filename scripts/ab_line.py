"""One A/B line from a bench.py JSON: stage times and clock-normalised ms x GHz."""
import json
import sys

lib, path = sys.argv[1], sys.argv[2]
d = json.load(open(path))
c = (d["clocks"]["sm_mhz"] or 0) / 1000
dense = d.get("dense_fa_ms") or 0
st = d["stage_ms"]
print(f"{lib.split('/')[-2]:24s} value {d['value']:.2f} est {st['estimate']:.2f} sel {st['select']:.2f} "
      f"att {st['attention']:.2f} dense {dense:.2f} clk {c:.3f} | att*GHz {st['attention'] * c:.1f} "
      f"value*GHz {d['value'] * c:.1f} dense*GHz {dense * c:.1f}")
