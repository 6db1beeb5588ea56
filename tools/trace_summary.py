import json, sys
for f in sys.argv[1:]:
    d = json.load(open(f))
    print(f, round(d["makespan_us"]), "us", round(d["gflops"]), "GF/s busy", round(d["sm_busy_frac"], 3), "wait", round(d["sm_wait_frac"], 3), d["busy_by_decile"])
    for k, v in d["per_kind"].items():
        print("  ", k, v["n"], "mean", round(v["mean_us"], 1), "p90", round(v["p90_us"], 1), "wait", round(v["mean_wait_us"], 1))
    for k, v in d.get("panel_phases_us", {}).items():
        print("  phases", k, v)
