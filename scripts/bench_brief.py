"""Print the key numbers of a bench.py JSON line (last line of the given file)."""
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d["roofline"]
print("ms/step %.3f  prepass %.3f  cull %.3f  classify %.3f  frac %.4f" % (
    d["ms_per_step"], r["prepass_ms"], r.get("cull_ms") or 0, r["kernel_ms"], r["frac"]))
print(d["cascade"])
