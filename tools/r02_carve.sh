#!/bin/bash
# GK step time vs the L1/shared carveout of the step kernels, lookahead on/off
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/carve; mkdir -p $O
for cv in -1 30 50 70 86; do
  for la in 0 1; do
    KSVD_CARVEOUT=$cv KSVD_LOOKAHEAD=$la timeout 300 python tools/la_timing.py > $O/cv${cv}_la$la.json 2>> $O/err.txt
    python -c "
import json; d=json.load(open('$O/cv${cv}_la$la.json'))
print('carveout $cv lookahead $la', {k: round(v['ms_per_step']*1e3,2) for k,v in d.items()})" >> $O/sum.txt 2>&1
  done
done
cat $O/sum.txt
