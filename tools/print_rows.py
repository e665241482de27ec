"""Print the headline numbers and the secondary rows of a bench.py --rows JSON line."""
import json, sys
d = json.loads(open(sys.argv[1]).read())
print("value", d["value"], "ms/step", d["ms_per_step"], "frac", d["roofline"]["frac"], "e2e ms", d["e2e"]["ms_per_step"])
for k, v in d.get("rows", {}).items():
    print(k, json.dumps(v))
