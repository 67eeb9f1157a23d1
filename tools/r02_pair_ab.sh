#!/bin/bash
# paired CGS2 step: parity suites (bounded) then a same-box A/B: serialised
# (KSVD_PAIR=0), paired with the separate finalisation (KSVD_TAILFIN=0),
# paired with the finalisation in k_gemv_n's tail (default)
cd "${GRAFT_REPO_ROOT:-.}"
O=${OUT:-gpurun_out/pair5}; mkdir -p $O
for i in 1 2; do
  for v in "KSVD_PAIR=0" "KSVD_TAILFIN=0" "X=1"; do
    env $v timeout 300 python tools/la_timing.py > $O/gk_${v%%=*}_$i.json 2>> $O/t.err
  done
done
python - "$O" <<'PY'
import json, sys
O=sys.argv[1]
for i in (1,2):
  row=[]
  for v in ("KSVD_PAIR", "KSVD_TAILFIN", "X"):
    try:
      d=json.load(open(f"{O}/gk_{v}_{i}.json")); row.append(v+" "+"/".join("%.1f" % (1e3*d[k]["ms_per_step"]) for k in d))
    except Exception as e:
      row.append(v+" err")
  print(i, " | ".join(row))
PY
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -3 $O/tests.log
for i in 1 2; do
  for v in "KSVD_PAIR=0" "KSVD_TAILFIN=0" "X=1"; do
    env $v timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/c2_${v%%=*}_$i.json 2>> $O/ab.err
  done
done
for f in $O/c2_*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['ms_per_step'],2), round(d['roofline']['share_of_device_time'].get('cgs'),4), d['clocks']['sm_mhz'])" 2>&1 | tail -1; done
