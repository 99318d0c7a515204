"""Print the key numbers of the last bench.py JSON line in gpurun_out/.last_call.json."""
import json
d = json.load(open("gpurun_out/.last_call.json"))
lines = [l for l in d["stdout_tail"].split("\n") if l.startswith("{")]
for line in lines:
    j = json.loads(line)
    if "roofline" in j:
        print("value", j["value"], "fill", j["roofline"]["achieved"], "frac", j["roofline"]["frac"],
              "e2e", j["e2e"]["value"], "ms", j["ms_per_step"])
    else:
        print(line[:300])
