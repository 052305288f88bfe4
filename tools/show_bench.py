import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], "stages", d["roofline"]["stage_ms"], "e2e", d["e2e"]["value"])
print("tucker ms", d["tucker"]["ms_per_solve"], d["tucker"]["stage_ms"], "tflops", d["tucker"]["algorithmic_tflops"])
