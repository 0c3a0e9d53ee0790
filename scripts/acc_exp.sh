for acc in 2 3; do
  IVFTQ_SCAN_ACC=$acc timeout 300 python -m pytest tests -m gpu -q -x -k "search_matches or random_configs" 2>&1 | tail -1
  IVFTQ_SCAN_ACC=$acc timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_acc$acc.log 2>&1
  tail -1 gpurun_out/bench_acc$acc.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('acc', $acc, d['value'], d['roofline']['kernel_ms'], d['recall_at_10'])"
done
