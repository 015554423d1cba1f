T="tests/test_gpu_solve.py::test_sequence_side_worker_matches_inline_and_serial tests/test_gpu_solve.py::test_c2_chained_sequence_bitwise_reproducible"
for env in "X=1" "CHFSI_QR_DEFER=0" "CHFSI_ND_PERSIST=0" "CHFSI_STREAM_PRIORITY=0" "CHFSI_K1_NH=2" "CHFSI_QR_DEFER=0 CHFSI_ND_PERSIST=0"; do
  r=$(env $env python -m pytest $T -q 2>&1 | tail -1)
  echo "$env: $r"
done
