python -m pytest tests/test_gpu_solve.py -q -x 2>&1 | tail -2
for i in 1 2; do
  for q in 1 0; do
    CHFSI_QR_DEFER=$q python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-scale-base --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('defer=$q', round(d['ms_per_step'],1), round(d['value']), d['step_ms'], [p['loops'] for p in d['per_problem']])"
  done
done
