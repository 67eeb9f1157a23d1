#!/bin/bash
# every BASELINE config through bench.py (our arm + the reference arm), one GPU
cd "${GRAFT_REPO_ROOT:-.}"
O=${BENCH_OUT:-gpurun_out/r02_all}; mkdir -p $O
for c in 1 2 3 5 4; do
  timeout 1200 python bench.py --config $c --steps 10 --warmup 3 > $O/ours_c$c.json 2> $O/ours_c$c.err
  echo "config $c rc=$?" >> $O/rc.txt
done
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --impl reference --config $c --steps 3 --warmup 1 > $O/ref_c$c.json 2> $O/ref_c$c.err
  echo "ref config $c rc=$?" >> $O/rc.txt
done
cat $O/rc.txt
for c in 1 2 3 4 5; do python - "$O" "$c" <<'PY'
import json, sys
O, c = sys.argv[1], sys.argv[2]
try:
    d = json.load(open(f"{O}/ours_c{c}.json")); r = json.load(open(f"{O}/ref_c{c}.json"))
    print(c, round(d["value"], 2), round(d["ms_per_step"], 2), round(d["effective_GBps"]), {k: round(v["GBps"]) for k, v in d["roofline"]["per_kernel"].items()},
          "e2e", round(d["e2e"]["value"], 2), "cpu", round(d["cpu_baseline"]["value"], 3), "ref", round(r["value"], 3), d["clocks"]["sm_mhz"])
except Exception as e:
    print(c, "error", e)
PY
done
