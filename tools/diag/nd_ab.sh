python -m pytest tests/test_gpu_kernels.py -q -x -k "near_diagonal or rayleigh or hermitian_eig" 2>&1 | tail -25
python tools/diag/rr_eig_bench.py
for i in 1 2; do
  for p in 1 0; do
    CHFSI_ND_PERSIST=$p python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-scale-base --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('persist=$p', round(d['ms_per_step'],1), round(d['value']), d['step_ms'], [p['rr_fast_eigs'] for p in d['per_problem']], [p['loops'] for p in d['per_problem']])"
  done
done
