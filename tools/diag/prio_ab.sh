for i in 1 2; do
  for p in 1 0; do
    CHFSI_STREAM_PRIORITY=$p python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-scale-base --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('prio=$p', round(d['ms_per_step'],1), round(d['value']), d['step_ms'])"
  done
done
python tools/diag/kernel_mix.py --top 30 > gpurun_out/r02j_mix_prio.txt 2>&1
