for env in "X=1" "CHFSI_QR_DEFER=0" "CHFSI_ND_PERSIST=0" "CHFSI_STREAM_PRIORITY=0"; do
  r=$(env $env python -m pytest tests/test_gpu_solve.py -q -x 2>&1 | tail -1)
  echo "$env: $r"
done
