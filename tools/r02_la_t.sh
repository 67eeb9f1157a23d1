#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/la_t3; mkdir -p $O
for i in 1 2; do
KSVD_LOOKAHEAD=0 timeout 300 python tools/la_timing.py > $O/off_$i.json 2> $O/off.err
timeout 300 python tools/la_timing.py > $O/on_$i.json 2> $O/on.err
done
python - <<'PY'
import json
O="gpurun_out/la_t3"
for i in (1,2):
  off=json.load(open(f"{O}/off_{i}.json")); on=json.load(open(f"{O}/on_{i}.json"))
  for k in off:
    a0=off[k]["alphas"]; a1=on[k]["alphas"]
    import numpy as np
    d=np.max(np.abs(np.array(a0)-np.array(a1))/np.abs(np.array(a0)))
    print(i, k, "off %.2f us/step on %.2f us/step" % (1e3*off[k]["ms_per_step"], 1e3*on[k]["ms_per_step"]), "max rel alpha diff %.2e" % d)
PY
for i in 1; do
KSVD_CARVEOUT=0 timeout 300 python tools/la_timing.py > $O/nocarve_$i.json 2> $O/nocarve.err
python -c "
import json; d=json.load(open('$O/nocarve_1.json'))
print('carveout off, lookahead on:', {k: round(v['ms_per_step']*1e3,2) for k,v in d.items()})"
done
