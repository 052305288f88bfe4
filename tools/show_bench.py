import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d["roofline"]
print("value", round(d["value"]), "ms", round(d["ms_per_step"], 4), "e2e", round(d["e2e"]["value"]),
      "dominant", r.get("kernel"), r.get("bound"), round(r.get("frac", 0), 4))
for k, v in r.get("stages", {}).items():
    print("  ", k, v["ms"], v["bound"], round(v["achieved"], 3), v["unit"], "frac", round(v["frac"], 4))
t = d["tucker"]
print("tucker ms", round(t["ms_per_solve"], 3), {k: round(v, 3) for k, v in t["stage_ms"].items()},
      "tflops", round(t["algorithmic_tflops"], 3))
