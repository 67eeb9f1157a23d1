#!/bin/bash
# paired CGS2 step: parity suites (bounded) then a same-box A/B against the
# serialised step (KSVD_PAIR=0) on GK runs and config-2/3 bench lines
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/pair; mkdir -p $O
for i in 1 2; do
  KSVD_PAIR=0 timeout 300 python tools/la_timing.py > $O/off_$i.json 2>> $O/t.err
  timeout 300 python tools/la_timing.py > $O/on_$i.json 2>> $O/t.err
done
python - <<'PY'
import json, numpy as np
O="gpurun_out/pair"
for i in (1,2):
  try:
    off=json.load(open(f"{O}/off_{i}.json")); on=json.load(open(f"{O}/on_{i}.json"))
  except Exception as e:
    print("err", e); continue
  for k in off:
    a0=np.array(off[k]["alphas"]); a1=np.array(on[k]["alphas"])
    b0=np.array(off[k]["betas"]); b1=np.array(on[k]["betas"])
    print(i, k, "off %.2f us/step on %.2f us/step" % (1e3*off[k]["ms_per_step"], 1e3*on[k]["ms_per_step"]),
          "alpha rel diff: first 8 %.1e all %.1e" % (np.max(np.abs(a0-a1)[:8]/a0[:8]), np.max(np.abs(a0-a1)/a0)),
          "beta %.1e" % np.max(np.abs(b0-b1)/b0))
PY
tail -3 $O/t.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -5 $O/tests.log
for c in 2 3; do
  for i in 1 2; do
    KSVD_PAIR=0 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/off_c${c}_$i.json 2>> $O/ab.err
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/on_c${c}_$i.json 2>> $O/ab.err
  done
done
for f in $O/off_c*.json $O/on_c*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['ms_per_step'],2), d['roofline']['share_of_device_time'].get('cgs'), d['clocks']['sm_mhz'])" 2>&1 | tail -1; done
