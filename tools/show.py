import json, sys, glob, os
d = sys.argv[1]
for f in sorted(glob.glob(os.path.join(d, "bench_n*.json"))):
    try:
        x = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    print(os.path.basename(f), x["value"], {k: round(v * 1000, 1) for k, v in x["stage_ms"].items()},
          "roof", x["roofline"]["frac"], "emu", (x.get("emulated_local") or {}).get("ms_per_sync_one_gpu"),
          (x.get("emulated_local") or {}).get("stage_ms"))
