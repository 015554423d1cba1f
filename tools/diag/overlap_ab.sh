#!/bin/bash
# A/B: C2 bench with and without the side-stream reduction overlap (variance)
for i in 1 2 3; do
  for f in "" "--no-overlap"; do
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks $f 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$f' or 'overlap', round(d['ms_per_step'],1), [round(p['t_solve_ms']) for p in d['per_problem']])"
  done
done
