# CFG3 sweep with and without the 2-SM halo conv (incl. stride-2 convs), same box, twice
for p in 0 1 0 1; do SLIM_HALO_PAIR=$p timeout 900 python bench.py --workload sweep > gpurun_out/sw_pair$p.json 2>/dev/null; python - "$p" <<'PY'
import json, sys
p = sys.argv[1]
for l in open(f"gpurun_out/sw_pair{p}.json"):
    if l.startswith("{"):
        d = json.loads(l); c = d["config"]
        if c["batch"] >= 128: print(p, c["batch"], c["width"], round(d["us_per_call"], 1))
PY
done
