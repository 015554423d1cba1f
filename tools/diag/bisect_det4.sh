for sel in "c2_harness or side_worker" "angle_report or side_worker"; do
  r=$(python -m pytest tests/test_gpu_solve.py -q -k "$sel" 2>&1 | tail -1)
  echo "[$sel]: $r"
done
