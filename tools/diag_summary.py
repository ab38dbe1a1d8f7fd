"""Print tools/diag_thresholds.py output compactly."""
import json
import sys

for l in open(sys.argv[1]):
    try:
        d = json.loads(l)
    except Exception:
        print(l.strip())
        continue
    if "error" in d:
        print(d)
        continue
    if d["it"] == 0:
        print(d["case"], d["set"], "init relX %.2e" % d["relX"])
        continue
    print(d["case"], d["set"], d["it"], "relX %.2e e %.1e A %.1e C %.1e dCabs %.1e dk %.1e dp %.1e dw %.1e flips %d gap %.1e" % (
        d["relX"], d["rel_e"], d["rel_A"], d["rel_C"], d["max_dC_abs"], d["max_dk"], d["dp"], d["dw"], d["flipsC"],
        d["min_gap_C"]), {k: "%.1e" % v for k, v in d["em_rel"].items()})
    print("   bins", {k: (v[0], "%.1e" % v[1]) for k, v in d["bins"].items()})
