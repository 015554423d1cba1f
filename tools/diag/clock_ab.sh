#!/bin/bash
# A/B: C2 bench with and without the NVML clock sampler (host stalls?)
for i in 1 2; do
  for f in "" "--no-clocks"; do
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $f 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$f' or 'clocks', d['ms_per_step'], [round(p['t_solve_ms']) for p in d['per_problem']])"
  done
done
