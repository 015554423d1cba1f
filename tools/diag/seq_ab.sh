# A/B of driver changes: bench C2 twice + the sequence-driver GPU tests
python -m pytest tests/test_gpu_solve.py -q -x -k "sequence or c1_chained or slots or releases" > gpurun_out/ab_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/ab_tests.log
for i in 1 2; do
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-scale-base --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],1), round(d['value']), d['step_ms'], d['step_problem_ms'][-1])"
done
