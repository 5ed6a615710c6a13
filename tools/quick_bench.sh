# quick per-config numbers: value, e2e, stage avg ms
for c in ${CONFIGS:-c1 c2 c3 c4 c5}; do
  steps=10; [ $c = c5 ] && steps=3
  python bench.py --config $c --steps $steps --warmup 3 --no-cpu-baseline 2>gpurun_out/qb_$c.err | tail -1 > gpurun_out/qb_$c.json
  python - $c <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/qb_{c}.json").read())
except Exception as e:
    print(c, "FAILED", open(f"gpurun_out/qb_{c}.err").read()[-800:]); sys.exit()
st = {k: round(v["avg_ms"], 4) for k, v in d["stages"].items()}; rs = d.get("roofline_search") or {}
print(c, "value %.4g" % d["value"], "e2e %.4g" % d["e2e"]["value"], st, "roof", d["roofline"].get("kernel"), round(d["roofline"]["frac"], 3), "iso", round(d["roofline"].get("frac_isolated") or 0, 3), "search_roof", rs.get("kernel"), round(rs.get("frac") or 0, 3), round(rs.get("frac_isolated") or 0, 3), "ok", d["parity_in_run"]["status_ok"], "/", d["parity_in_run"]["records"])
PY
done
