#!/bin/bash
# RR near-diagonal regime bound sweep: RR device time and fast-path count per problem (C2)
for b in 0.1 0.3 0.5 1.0; do
  CHFSI_RR_BAIL=$b python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('bail $b', round(d['ms_per_step'],1), [(p['loops'], p['rr_fast_eigs'], round(p['dev_ms']['rr'],1)) for p in d['per_problem']])"
done
