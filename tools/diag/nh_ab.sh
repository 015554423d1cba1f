# K1 k-slab depth A/B: sweep at the C2/C3/C4 shapes, then the C2 sequence, NH=2 vs NH=4
for nh in 2 4; do
  CHFSI_K1_NH=$nh python tools/k1_sweep.py --products 3 --no-cublas --chains 2 --shapes 2048x160,2048x131,2048x100,2048x64,2048x40,5000x600,12000x1400 2>/dev/null | sed "s/^/nh=$nh /"
done
for i in 1 2; do
  for nh in 4 2; do
    CHFSI_K1_NH=$nh python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-scale-base --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('nh=$nh', round(d['ms_per_step'],1), round(d['value']), round(d['roofline']['achieved'],2), d['step_ms'])"
  done
done
CHFSI_K1_NH=4 python -m pytest tests/test_gpu_kernels.py -q -x -k "cheb_step or filter" 2>&1 | tail -2
