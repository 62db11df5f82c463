import json, sys
for f in sys.argv[1:]:
    for ln in open(f):
        if ln.startswith('{'):
            d = json.loads(ln)
            print(f, {k: d.get(k) for k in ("value", "ms_per_step", "setup_ms", "solve_ms", "iterations", "apply_ms", "kappa")},
                  "e2e", d["e2e"]["value"])
            print("   roof", d.get("roofline"))
            print("   ", {k: (v["avg_ms"], v.get("frac")) for k, v in d["phases"].items()})
            break
    else:
        print(f, open(f).read()[-1200:])
