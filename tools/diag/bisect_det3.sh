W="side_worker"
for sel in "solve_matches_reference_golden or $W" "known_diagonal or deterministic or hp_reuse or guess_width or rank_repair or $W" "c1_ or $W" "c2_harness or angle_report or $W" "c3_harness or $W" "raises_reference or c2_chained or $W"; do
  r=$(python -m pytest tests/test_gpu_solve.py -q -k "$sel" 2>&1 | tail -1)
  echo "[$sel]: $r"
done
