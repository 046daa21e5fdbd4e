import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f, "ms/step=%.2f" % d["ms_per_step"], "Gbases/s=%.2f" % (d["value"] / 1e9), "Gkmers/s=%.2f" % (d["kmers_per_s"] / 1e9))
    print("  stages", {k: round(v, 2) for k, v in d["stage_ms"].items()}, "waves", d["config"]["waves"], "bins", d["config"]["n_bins"])
    print("  result", d["result"])
    r = d["roofline"]
    print("  roofline frac=%.3f achieved=%.0f GB/s avg_launch=%.3f ms launches=%d share=%.2f" % (r["frac"] or 0, r["achieved"] or 0, r["avg_launch_ms"], r["launches_per_step"], r["share_of_step"]))
    if d.get("e2e"): print("  e2e", {k: d["e2e"][k] for k in ("value", "ms_per_step")})
    print("  clocks", d["clocks"], "launches", d["gpu_launches"])
